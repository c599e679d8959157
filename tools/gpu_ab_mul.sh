# finalize numerator: 32-bit-operand multiplies (default) vs int64 multiplies (tools/alt_mul64.so)
timeout -s KILL 900 python -m pytest tests/test_parity_gpu.py tests/test_narrow_gpu.py tests/test_fullsize_gpu.py -m gpu -x -q 2>&1 | tail -2
for lib in "" tools/alt_mul64.so "" tools/alt_mul64.so; do for nar in 0 1; do
  FIN_RHO=0 FIN_NARROW=$nar CPA_LIB_PATH=$lib timeout -s KILL 300 python tools/fin_bench.py 2>/dev/null | sed "s#^#${lib:-default} narrow=$nar maxima #" | cut -c1-200
  FIN_RHO=1 FIN_M=48000 FIN_NARROW=$nar CPA_LIB_PATH=$lib timeout -s KILL 300 python tools/fin_bench.py 2>/dev/null | sed "s#^#${lib:-default} narrow=$nar rho #" | cut -c1-200
done; done
for cfg in C5 W48; do for lib in "" tools/alt_mul64.so; do
  timeout -s KILL 400 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default} $cfg', 'step %.3f phases %s clk %s key %s' % (d['ms_per_step'], {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['key_recovered']))"
done; done
