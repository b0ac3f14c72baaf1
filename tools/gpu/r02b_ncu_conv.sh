#!/bin/bash
# ncu --set full of the two residue kernels inside a bench step
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-rows_kernel|cols_residues}" -s 2 -c 2 -o /tmp/prof_conv python bench.py --steps 1 --warmup 1 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_conv.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_conv.ncu-rep --page raw --csv > gpurun_out/ncu_conv_raw.csv 2>/dev/null
ncu -i /tmp/prof_conv.ncu-rep --page details --csv > gpurun_out/ncu_conv_details.csv 2>/dev/null
ncu -i /tmp/prof_conv.ncu-rep --page source --csv -k regex:cols_residues > gpurun_out/ncu_conv_src_cols.csv 2>/dev/null
ncu -i /tmp/prof_conv.ncu-rep --page source --csv -k regex:rows_kernel > gpurun_out/ncu_conv_src_rows.csv 2>/dev/null
cp /tmp/prof_conv.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out
