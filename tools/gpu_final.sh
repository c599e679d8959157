# final evidence (tools/gpu_evidence.sh) + C4 / C5 A/B of the narrow 2-row spill against 4 rows (tools/alt_st4.so)
bash tools/gpu_evidence.sh
for cfg in C4 C5; do for lib in tools/alt_st4.so "" tools/alt_st4.so ""; do
  timeout -s KILL 400 env CPA_LIB_PATH=$lib python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default} $cfg', 'step %.3f phases %s clk %s key %s' % (d['ms_per_step'], {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['key_recovered']))"
done; done
