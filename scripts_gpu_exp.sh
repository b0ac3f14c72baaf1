#!/bin/bash
# experiments: CTA-pair GEMM correctness + schedule variants
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest(CG=2) rc=$?"; tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-context --no-cpu-baseline"
for cfg in "OZ2_CG=2" "OZ2_CG=2 OZ2_GROUP_TM=4" "OZ2_CG=2 OZ2_GROUP_TM=16" "OZ2_CG=1" "OZ2_CG=2 OZ2_TILE_MAJOR=0 OZ2_GROUP_TM=8"; do
  echo "== $cfg"; env $cfg timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'TFLOPS', {k: round(v,2) for k,v in d['stage_ms'].items()}, d['clocks'].get('sm_mhz'), d['clocks'].get('power_w_max'), d['compwise_err'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:modmul -s 1 -c 1 -o gpurun_out/prof_cg2 python bench.py --steps 1 --warmup 1 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
