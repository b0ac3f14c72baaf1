#!/bin/bash
# multi-GPU functional checks on one GPU (2 ranks over gloo): small and c4-size
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
N=4096 bash tools/gpu/dist_check.sh
N=32768 bash tools/gpu/dist_check.sh
