#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-context --no-cpu-baseline"
for cfg in "OZ2_SYNC_LAG=0" "OZ2_EPI_NOP=1" "OZ2_SYNC_LAG=1" "OZ2_GROUP_TM=4"; do
  echo "== $cfg"; env $cfg timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'TFLOPS', {k: round(v,2) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'], round(d['roofline']['achieved']), d['compwise_err'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:modmul -s 1 -c 1 -o gpurun_out/prof_gemm4 python bench.py --steps 1 --warmup 1 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
