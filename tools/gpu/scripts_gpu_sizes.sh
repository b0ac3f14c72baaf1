for sz in 4096 8192; do for up in 74 148 300; do
 echo "== size $sz up_tiles $up"; OZ2_UP_TILES=$up python bench.py --size $sz --steps 10 --no-e2e --no-context --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'TFLOPS', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['stage_ms'].items()})"
done; done
