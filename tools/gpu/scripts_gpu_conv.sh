#!/bin/bash
# conversion-kernel experiment: GPU tests, then the bench's stage times under env knobs (EXP_CFGS)
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps ${EXP_STEPS:-5} --warmup 3 --no-e2e --no-context --no-cpu-baseline"
for cfg in ${EXP_CFGS:-"OZ2_X=0"}; do
  echo "== $cfg"; env $cfg timeout 300 $B 2> /tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'TFLOPS', {k: round(v,3) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'])"; tail -2 /tmp/err.txt
done
if [ -n "$EXP_NCU" ]; then
  env $EXP_NCU timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|cols_stats|cols_residues" -s 3 -c 3 -o /tmp/prof_conv python bench.py --steps 1 --warmup 1 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_conv.log 2>&1; echo "ncu rc=$?"
  python tools/ncu_summary.py /tmp/prof_conv.ncu-rep > gpurun_out/ncu_conv_summary.txt 2>&1
  ncu -i /tmp/prof_conv.ncu-rep --page details --csv > gpurun_out/ncu_conv_details.csv 2>/dev/null
  ncu -i /tmp/prof_conv.ncu-rep --page source --csv --kernel-name regex:rows_kernel > gpurun_out/ncu_conv_rows_source.csv 2>/dev/null
fi
