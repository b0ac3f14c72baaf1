#!/bin/bash
# interleaved env A/B on the experiment build (liboz2_exp.so, -DOZ2_EXPERIMENTS)
export OZ2_LIB=$PWD/paper_2504_08009_b200/liboz2_exp.so
for rep in $(seq ${REPS:-2}); do
for kv in $AB_VARS; do
  env $kv OZ2_GEMM_DEBUG=${DBG:-0} timeout 600 python bench.py --steps ${STEPS:-10} --warmup 4 --no-e2e --no-cpu-baseline --no-context $BARGS > /tmp/ab.json 2> /tmp/ab.err
  python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$kv', round(d['value'],1), round(d['stage_ms']['gemm'],3), d['clocks']['sm_mhz'])"
  grep "gemm dbg" /tmp/ab.err | tail -1
done; done
