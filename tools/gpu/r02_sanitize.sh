#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small products
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build(); import oracle; oracle.build()" > gpurun_out/build.log 2>&1
export OZ2_SYNC_KB=48
for shape in "64 64 64" "256 256 256" "2560 3900 300"; do
  tag=$(echo $shape | tr ' ' 'x')
  for tool in memcheck racecheck synccheck; do
    to=1200; [ "$tool" = "racecheck" ] && to=2400
    timeout $to compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
        python tools/sanitize_case.py $shape > gpurun_out/sanitize_${tool}_${tag}.log 2>&1
    echo "$tool $tag rc=$?"; grep -E "ERROR SUMMARY|mismatches|Error|error" gpurun_out/sanitize_${tool}_${tag}.log | head -5
  done
done
