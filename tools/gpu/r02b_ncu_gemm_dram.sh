#!/bin/bash
# DRAM bytes of the fused GEMM at 16384^3 for liboz2.so and $ALT (one launch each)
ALT=${ALT:-$PWD/paper_2504_08009_b200/liboz2_alt.so}
for lib in main alt; do
  if [ $lib = alt ]; then export OZ2_LIB=$ALT; else unset OZ2_LIB; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:modmul -s 2 -c 1 python bench.py --steps 1 --warmup 2 --no-e2e --no-context --no-cpu-baseline 2>/dev/null | grep -E "dram__bytes|duration" | sed "s/^/$lib /"
done
