#!/bin/bash
# interleaved A/B of environment settings (REPS rounds), one bench each
python -c "from paper_2504_08009_b200 import build; build.build()" > /dev/null 2>&1
for rep in $(seq ${REPS:-2}); do
for kv in $AB_VARS; do
  env $kv timeout 600 python bench.py --steps ${STEPS:-10} --warmup 4 --no-e2e --no-cpu-baseline --no-context $BARGS > /tmp/ab.json 2> /tmp/ab.err
  python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$kv', round(d['value'],1), round(d['stage_ms']['gemm'],3), d['clocks']['sm_mhz'])"
done; done
