#!/bin/bash
# A/B of environment knobs on the bench step: AB_VARS="VAR=a VAR=b ..." (one bench per setting)
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for kv in $AB_VARS; do
  for rep in 1 2; do
    env $kv timeout 600 python bench.py --steps 10 --warmup 4 --no-e2e --no-cpu-baseline --no-context > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$kv', round(d['value'],1), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
