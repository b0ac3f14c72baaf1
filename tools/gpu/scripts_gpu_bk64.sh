L64=$PWD/paper_2504_08009_b200/liboz2_bk64.so
OZ2_LIB=$L64 timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2; echo "smoke64 rc=$?"
OZ2_LIB=$L64 timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for i in 1 2; do
for lib in paper_2504_08009_b200/liboz2.so $L64; do
  echo "== $lib"; OZ2_LIB=$(realpath $lib) timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-context --no-cpu-baseline 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'TFLOPS', {k: round(v,3) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'])"; tail -2 /tmp/err.txt
done; done
