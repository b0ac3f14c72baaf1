#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|cols_stats|cols_residues" -s 3 -c 3 -o gpurun_out/prof_conv python bench.py --steps 1 --warmup 1 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_conv.log 2>&1; echo "ncu rc=$?"
