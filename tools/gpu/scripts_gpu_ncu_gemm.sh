#!/bin/bash
# one ncu --set full capture of the GEMM (source counters for stall attribution)
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"modmul" -s 1 -c 1 -o gpurun_out/prof_gemm ${NCU_ENV} python bench.py --steps 1 --warmup 1 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1; echo "ncu rc=$?"
