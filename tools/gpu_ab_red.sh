# narrow red.add.u32 spill: 2 rows x 64 B per warp instruction (default) vs 4 rows x 32 B (tools/alt_red4.so)
timeout -s KILL 900 python -m pytest tests/test_narrow_gpu.py tests/test_parity_gpu.py tests/test_stream.py -m gpu -x -q 2>&1 | tail -2
for cfg in C4 C5 C2; do for lib in "" tools/alt_red4.so "" tools/alt_red4.so; do
  timeout -s KILL 400 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${lib:-default} $cfg', 'step %.3f xterm/launch %.4f phases %s clk %s key %s' % (d['ms_per_step'], r['ms_per_launch'], {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['key_recovered']))"
done; done
