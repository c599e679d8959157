# narrow first-touch spill: 2 rows x 64 B per store (default) vs 4 rows x 32 B (tools/alt_st4.so)
timeout -s KILL 600 python -m pytest tests/test_narrow_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -2
for cfg in W48 C2; do for lib in "" tools/alt_st4.so "" tools/alt_st4.so; do
  timeout -s KILL 300 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${lib:-default} $cfg', 'step %.3f xterm %.4f ms fin %.3f clk %s key %s' % (d['ms_per_step'], r['ms_per_launch'], d['phases_ms_per_step']['finalize'], d['clocks']['sm_mhz'], d['key_recovered']))"
done; done
