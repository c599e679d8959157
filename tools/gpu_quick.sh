# parity tests, racecheck on C1, short C4 + W48 bench lines
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
bash tools/racecheck.sh > /dev/null 2>&1; grep "SUMMARY" gpurun_out/racecheck_c1.log
for cfg in C4 W48; do
  timeout -s KILL 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/bench_$cfg.log 2>&1
  tail -1 gpurun_out/bench_$cfg.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$cfg ms/step %.3f  xterm %.3f ms frac %.3f  phases %s key %s hbm %s clocks %s' % (d['ms_per_step'], r['ms_per_launch'], r['frac'], {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['key_recovered'], {k: round(v or 0) for k,v in d['hbm'].items()}, d.get('clocks')))"
done
