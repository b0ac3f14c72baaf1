#!/bin/bash
# round-2 check: build, smoke, GPU tests (new fused/safety tests first), bench
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -i "model name" >> gpurun_out/nproc.txt
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_fused.py -q -x --durations=10 > gpurun_out/pytest_fused.log 2>&1; echo "fused rc=$?"; tail -15 gpurun_out/pytest_fused.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 --deselect tests/test_gpu_fused.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -20 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
