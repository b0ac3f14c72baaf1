ALT=paper_2504_08009_b200/liboz2_er.so
OZ2_LIB=$(realpath $ALT) timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_syrk.py -q -x 2>&1 | tail -1
for i in 1 2 3 4; do
for lib in paper_2504_08009_b200/liboz2.so $ALT; do
  OZ2_LIB=$(realpath $lib) timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-context --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], round(d['value'],1), round(d['stage_ms']['gemm'],2))"
done; done
