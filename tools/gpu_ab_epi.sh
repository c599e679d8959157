# epilogue store loop: unswitched (default build) vs per-element branches (tools/alt_branchy.so)
for cfg in W48 C2 C4; do for lib in "" tools/alt_branchy.so "" tools/alt_branchy.so; do for nar in 0 1; do
  timeout -s KILL 300 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 10 --narrow $nar 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${lib:-default} $cfg narrow=$nar', 'step %.3f xterm %.3f ms fin %.3f clk %s key %s' % (d['ms_per_step'], r['ms_per_launch'], d['phases_ms_per_step']['finalize'], d['clocks']['sm_mhz'], d['key_recovered']))"
done; done; done
