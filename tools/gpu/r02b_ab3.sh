#!/bin/bash
# interleaved A/B/C of liboz2.so, liboz2_alt.so, liboz2_alt2.so (REPS rounds)
for rep in $(seq ${REPS:-2}); do
  for lib in main alt alt2; do
    if [ $lib = main ]; then unset OZ2_LIB; else export OZ2_LIB=$PWD/paper_2504_08009_b200/lib${lib/main/}oz2_$lib.so; export OZ2_LIB=$PWD/paper_2504_08009_b200/liboz2_$lib.so; fi
    timeout 600 python bench.py --steps ${STEPS:-10} --warmup 4 --no-e2e --no-cpu-baseline --no-context $BARGS > /tmp/ab.json 2> /tmp/ab.err
    python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$lib', round(d['value'],1), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
