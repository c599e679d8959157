#!/bin/bash
# Power / clock behaviour during a long bench run (run under gpurun).
nvidia-smi -q -d POWER,CLOCK | grep -iE "limit|Power Draw|SM  |Graphics|Max Clocks" | head -30
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.sw_power_cap,temperature.gpu --format=csv,noheader -lms 50 > gpurun_out/power_trace.csv &
P=$!
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 60 --warmup 3 "$@" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'xterm', d['roofline']['ms_per_launch'], d['clocks'])"
kill $P
python - <<'PY'
import statistics
rows=[l.strip().split(', ') for l in open('gpurun_out/power_trace.csv') if l.strip()]
sm=[float(r[1].split()[0]) for r in rows]; pw=[float(r[2].split()[0]) for r in rows]
busy=[(s,p) for s,p in zip(sm,pw) if p>300]
print('samples', len(rows), 'busy', len(busy))
if busy:
    print('busy sm MHz median %.0f min %.0f max %.0f; power median %.0f max %.0f' % (statistics.median([b[0] for b in busy]), min(b[0] for b in busy), max(b[0] for b in busy), statistics.median([b[1] for b in busy]), max(b[1] for b in busy)))
PY
