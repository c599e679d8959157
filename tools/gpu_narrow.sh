# CPA_OPT_NARROW: all GPU tests, then bench A/B of narrow on/off and finalize variants
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_narrow.log 2>&1
tail -3 gpurun_out/pytest_narrow.log
for lib in "" tools/alt_minb4.so tools/alt_ux2.so; do for cfg in W48 C2; do for nar in 0 1; do
  timeout -s KILL 300 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 10 --narrow $nar 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${lib:-default} $cfg narrow=$nar', 'step %.3f xterm %.3f ms fin %.3f ms fin GBps %.0f clk %s key %s' % (d['ms_per_step'], r['ms_per_launch'], d['phases_ms_per_step']['finalize'], d['hbm']['finalize_GBps'], d['clocks']['sm_mhz'], d['key_recovered']))"
done; done
for nar in 0 1; do
  timeout -s KILL 400 env CPA_LIB_PATH=$lib python bench.py --config C5 --no-e2e --no-cpu-baseline --steps 3 --narrow $nar 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default} C5 narrow=$nar', 'step %.3f phases %s key %s' % (d['ms_per_step'], {k: round(v,3) for k,v in d.get('phases_ms_per_step',{}).items()}, d['key_recovered']))"
done; done
