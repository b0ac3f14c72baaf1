#!/bin/bash
# A/B of residue-kernel builds: parity subset + bench stage times for each, ncu of the conversion kernels
mkdir -p gpurun_out
LIBS=${LIBS:-"liboz2.so liboz2_minb3.so liboz2_dp4a.so"}
for lib in $LIBS; do
  L=$(realpath paper_2504_08009_b200/$lib)
  echo "== $lib"
  OZ2_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q -x \
     -k "stage_parity or edge or extreme or every_N or c2_sampled_256 or certificate" > gpurun_out/ab_pytest_$lib.log 2>&1
  echo "pytest rc=$?"; tail -n 2 gpurun_out/ab_pytest_$lib.log
  for r in 1 2; do
    OZ2_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ab_bench_${lib}_$r.json 2>&1
    python - <<PY
import json
d = json.loads(open("gpurun_out/ab_bench_${lib}_$r.json").read().strip().splitlines()[-1])
print("$lib run $r:", round(d["value"], 2), "TFLOPS", {k: round(v, 3) for k, v in d["stage_ms"].items()}, d["clocks"]["sm_mhz"])
PY
  done
done
L=$(realpath paper_2504_08009_b200/liboz2.so)
OZ2_LIB=$L timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|cols_residues|cols_stats" -s 3 -c 3 -o /tmp/conv python bench.py --steps 1 --warmup 1 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_conv.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/conv.ncu-rep > gpurun_out/ncu_conv_summary.txt 2>&1
ncu -i /tmp/conv.ncu-rep --page raw --csv > gpurun_out/ncu_conv_raw.csv 2>/dev/null
ncu -i /tmp/conv.ncu-rep --page source --csv --kernel-name regex:rows_kernel > gpurun_out/ncu_conv_src_rows.csv 2>/dev/null
