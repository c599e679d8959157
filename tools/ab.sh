# A/B of library variants (under gpurun): LIBS="tools/x.so ..." CFGS="C4 C3" REPS=3 bash tools/ab.sh
for cfg in ${CFGS:-C4}; do
for rep in $(seq ${REPS:-3}); do
for lib in "" $LIBS; do
  timeout -s KILL 300 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps ${STEPS:-10} $BENCH_ARGS 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg ${lib:-default}', 'step %.3f xterm %.3f ms clk %s key %s' % (d['ms_per_step'], r['ms_per_launch'], d['clocks']['sm_mhz'], d['key_recovered']))"
done; done; done
