#!/bin/bash
# GEMM wait-cycle counters and epilogue attribution (experiment build liboz2_exp.so, -DOZ2_EXPERIMENTS)
export OZ2_LIB=$PWD/paper_2504_08009_b200/liboz2_exp.so
for n in ${DBG_SIZES:-16384 4096}; do
for cfg in ${EXP_CFGS:-"OZ2_X=0" "OZ2_EPI_NOP=1" "OZ2_EXP_NO_CRT=1"}; do
  echo "== n=$n $cfg"; env $cfg OZ2_GEMM_DEBUG=1 timeout 300 python bench.py --n $n --steps ${EXP_STEPS:-5} --warmup 3 --no-e2e --no-context --no-cpu-baseline 2> /tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'TFLOPS', {k: round(v,3) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"; grep "gemm dbg" /tmp/err.txt | tail -1
done; done
