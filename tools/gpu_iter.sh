# fast iteration (under gpurun): build, one parity file, C4 bench line(s)
# usage: bash tools/gpu_iter.sh [test file] [extra bench args]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
T=${1:-tests/test_parity_gpu.py}; shift
timeout -s KILL 600 python -m pytest $T -q -x --timeout 300 2>&1 | tail -4
for i in 1 2; do
timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('ms/step %.2f  xterm %.2f ms  %.0f TOPS frac %.3f ceil %.3f phases %s key %s clocks %s' % (d['ms_per_step'], r['ms_per_launch'], r['achieved'], r['frac'], r.get('frac_of_mma_rate_ceiling', 0), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['key_recovered'], d.get('clocks')))"
done
