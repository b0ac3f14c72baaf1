#!/bin/bash
# the FP64 prime-modulus regime tests + the multi-GPU functional check (2 ranks, 1 GPU, gloo)
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_fp64mod.py tests/test_gpu_ksplit.py -q -x > gpurun_out/pytest_f4.log 2>&1; echo "f4 rc=$?"; tail -25 gpurun_out/pytest_f4.log
N=4096 bash tools/gpu/dist_check.sh
