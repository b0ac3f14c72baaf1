#!/bin/bash
# host-pipeline experiment: the host-path GPU tests, then e2e through oz2_dgemm_host under env knobs (EXP_CFGS)
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "host" > gpurun_out/pytest_host.log 2>&1; echo "pytest host rc=$?"; tail -2 gpurun_out/pytest_host.log
timeout 300 python tools/e2e_check.py 2>&1 | tail -8
for cfg in ${EXP_CFGS:-"OZ2_X=0"}; do
  echo "== $cfg"; env $cfg timeout 300 python bench.py --steps 3 --warmup 3 --no-context --no-cpu-baseline 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'TFLOPS device;', 'e2e', round(d['e2e']['value'],1), 'TFLOPS', round(d['e2e']['ms_per_step'],1), 'ms')"; tail -2 /tmp/err.txt
done
