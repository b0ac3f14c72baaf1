#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-context --no-cpu-baseline"
for cfg in "OZ2_PF_DIST=16" "OZ2_PF_DIST=0" "OZ2_PF_DIST=32" "OZ2_PF_DIST=8" "OZ2_PF_DIST=64" "OZ2_PF_DIST=32 OZ2_SYNC_LAG=1" "OZ2_PF_DIST=32 OZ2_SYNC_KB=64" "OZ2_PF_DIST=32 OZ2_EPI_NOP=1"; do
  echo "== $cfg"; env $cfg OZ2_GEMM_DEBUG=1 timeout 300 $B 2> /tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'TFLOPS', {k: round(v,2) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'])"; grep "gemm dbg" /tmp/err.txt | tail -1
done
