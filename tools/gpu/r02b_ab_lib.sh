#!/bin/bash
# A/B of two in-tree builds on the same box: liboz2.so vs $ALT (default liboz2_alt.so),
# interleaved, REPS rounds of one bench each; extra bench args in $BARGS
ALT=${ALT:-$PWD/paper_2504_08009_b200/liboz2_alt.so}
for rep in $(seq ${REPS:-3}); do
  for lib in main alt; do
    if [ $lib = alt ]; then export OZ2_LIB=$ALT; else unset OZ2_LIB; fi
    timeout 600 python bench.py --steps ${STEPS:-10} --warmup 4 --no-e2e --no-cpu-baseline --no-context $BARGS > /tmp/ab.json 2> /tmp/ab.err
    python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$lib', round(d['value'],1), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
