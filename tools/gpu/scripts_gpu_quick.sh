#!/bin/bash
# quick GPU check: tests, then an env-knob sweep of the bench (EXP_CFGS)
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
bash tools/gpu/scripts_gpu_exp.sh
