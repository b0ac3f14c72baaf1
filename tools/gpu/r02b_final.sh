#!/bin/bash
# round-2 evidence: smoke, GPU tests, bench (fast, accu, reference arm), FP64-regime
# bench, ncu launch list + one ncu --set full capture of the step's kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/smi.txt
python -c "from paper_2504_08009_b200 import build; build.build(); import oracle; oracle.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --mode accu --no-e2e --no-context --no-cpu-baseline > gpurun_out/bench_accu.json 2>&1; echo "bench accu rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
timeout 900 python tools/fp64mod_bench.py 4096 1.0 > gpurun_out/fp64mod_bench.json 2> gpurun_out/fp64mod_bench.err; echo "fp64mod bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"modmul|rows_kernel|cols_stats|cols_residues" -s 5 -c 4 -o /tmp/prof_full python bench.py --steps 1 --warmup 3 --no-e2e --no-context --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py /tmp/prof_full.ncu-rep > gpurun_out/ncu_full_summary.txt 2>&1
ncu -i /tmp/prof_full.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv 2>/dev/null
ls -la gpurun_out | head -40
