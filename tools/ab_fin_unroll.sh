for cfg in W48 C4; do for rep in 1 2; do for lib in "" tools/lib_fin8.so tools/lib_fin2.so; do
  timeout -s KILL 300 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('$cfg ${lib:-new}', 'step %.3f fin %.4f GBps %.0f' % (d['ms_per_step'], p['finalize'], d['hbm']['finalize_GBps']))"
done; done; done
