# class-sum path (HW models): parity tests, then C4-HW bench per library variant
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -q -x --timeout 300 -k "class_sums" 2>&1 | tail -3
for lib in "" $LIBS; do
timeout -s KILL 300 env CPA_LIB_PATH=$lib python bench.py --config C4-HW --class-sums 1 --no-e2e --no-cpu-baseline --steps 5 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('${lib:-default} cs ms/step %.2f  xterm %.2f ms phases %s key %s' % (d['ms_per_step'], r['ms_per_launch'], {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['key_recovered']))"
done
