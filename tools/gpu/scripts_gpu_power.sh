nvidia-smi -q -d POWER,CLOCK | grep -i -E "limit|power draw|SM  |Graphics" | head -20
python -c "from paper_2504_08009_b200 import build; build.build()"
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,temperature.gpu --format=csv,noheader -lms 50 > gpurun_out/pw.csv &
P=$!
python bench.py --steps 60 --warmup 3 --no-e2e --no-context --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['stage_ms'], d['clocks'])"
kill $P
python - <<'P2'
rows=[l.split(',') for l in open('gpurun_out/pw.csv')]
import statistics
sm=[float(r[0].split()[0]) for r in rows]; pw=[float(r[1].split()[0]) for r in rows]
hi=[i for i,p in enumerate(pw) if p>300]
print(len(rows),'samples; loaded', len(hi))
print('sm median loaded', statistics.median([sm[i] for i in hi]) if hi else None, 'power median', statistics.median([pw[i] for i in hi]) if hi else None, 'max', max(pw))
print('pcap active frac', sum(1 for i in hi if 'Active' in rows[i][2])/max(1,len(hi)))
P2
