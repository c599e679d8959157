# a4/a5 overlap modes on C4 (run under gpurun)
for mode in 0 1 2; do
  for rep in 1 2; do
  timeout -s KILL 300 python bench.py --overlap-mode $mode --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('mode $mode ms/step %.3f xterm %.3f frac %.3f moments %.3f hbm %s' % (d['ms_per_step'], r['ms_per_launch'], r['frac'], d['phases_ms_per_step']['moments'], {k: round(v or 0) for k,v in d['hbm'].items()}))"
  done
done
