#!/bin/bash
# GEMM experiment sweep: knobs via env (see csrc/gemm.cu make_params), wait-cycle counters via OZ2_GEMM_DEBUG
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps ${EXP_STEPS:-3} --warmup 3 --no-e2e --no-context --no-cpu-baseline"
for cfg in ${EXP_CFGS:-"OZ2_X=0" "OZ2_EPI_NOP=1" "OZ2_SYNC_KB=0" "OZ2_SYNC_LAG=2" "OZ2_GROUP_TM=4" "OZ2_GROUP_TM=16"}; do
  echo "== $cfg"; env $cfg OZ2_GEMM_DEBUG=1 timeout 300 $B 2> /tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'TFLOPS', {k: round(v,2) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"; grep "gemm dbg" /tmp/err.txt | tail -1
done
