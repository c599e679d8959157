# A/B of library variants with the per-phase times (under gpurun):
#   LIBS="tools/x.so ..." CFGS="C3" REPS=3 PHASE=moments bash tools/ab_phase.sh
for cfg in ${CFGS:-C4}; do
for rep in $(seq ${REPS:-3}); do
for lib in "" $LIBS; do
  timeout -s KILL 300 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps ${STEPS:-10} $BENCH_ARGS 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('$cfg ${lib:-default}', 'step %.3f' % d['ms_per_step'], ' '.join('%s %.3f' % (k, v) for k, v in p.items()), 'key', d['key_recovered'])"
done; done; done
