# int64-row maxima kernel (narrow off: multi-GPU checkpoints): U = 4 / 4 blocks (default) vs U = 2, U = 2 / 5 blocks
for rep in 1 2; do for lib in "" tools/alt_w2.so tools/alt_w2b5.so; do
  FIN_RHO=0 FIN_NARROW=0 CPA_LIB_PATH=$lib timeout -s KILL 300 python tools/fin_bench.py 2>/dev/null | sed "s#^#${lib:-default} #" | cut -c1-160
done; done
for lib in "" tools/alt_w2.so tools/alt_w2b5.so; do
  timeout -s KILL 400 env CPA_LIB_PATH=$lib python bench.py --config C5 --narrow 0 --no-e2e --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default} C5 narrow=0', 'step %.3f finalize %.3f clk %s key %s' % (d['ms_per_step'], d['phases_ms_per_step']['finalize'], d['clocks']['sm_mhz'], d['key_recovered']))"
done
