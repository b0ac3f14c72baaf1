#!/bin/bash
# quick check: smoke, stage/fused parity tests, bench (fast)
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build(); import oracle; oracle.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_q.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-context > gpurun_out/bench_q$i.json 2> gpurun_out/bench_q$i.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_q$i.json')); print(round(d['value'],1), d['ms_per_step'], {k: round(v,3) for k,v in d['stage_ms'].items()}, d.get('clocks'))"; done
