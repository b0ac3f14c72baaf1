#!/bin/bash
# ncu source-level capture of the fused GEMM at 4096^3 (epilogue stall attribution)
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:modmul -s 3 -c 1 -o /tmp/prof_g4096 python bench.py --n ${NCU_N:-4096} --steps 1 --warmup 3 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_g4096.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_g4096.ncu-rep --page raw --csv > gpurun_out/ncu_g4096_raw.csv 2>/dev/null
ncu -i /tmp/prof_g4096.ncu-rep --page source --csv > gpurun_out/ncu_g4096_src.csv 2>/dev/null
ls -la gpurun_out/ncu_g4096*
