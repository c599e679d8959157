timeout 600 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -1
for cfg in C4 W48; do for rep in 1 2; do for lib in "" tools/libcpa_finold.so; do
  timeout -s KILL 300 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('$cfg ${lib:-new}', 'step %.3f fin %.4f GBps %s' % (d['ms_per_step'], p['finalize'], d['hbm']['finalize_GBps']))"
done; done; done
for lib in "" tools/libcpa_finold.so; do
  timeout -s KILL 600 env CPA_LIB_PATH=$lib python bench.py --config C5 --steps 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('C5 ${lib:-new}', 'step %.3f' % d['ms_per_step'], {k: round(v,3) for k,v in p.items()})"
done
