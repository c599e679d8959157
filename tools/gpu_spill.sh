# A/B of the int8 cross-term spill (CPA_OPT_SPILL) + parity, under gpurun
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 900 -k "parity or fullsize or sharded" > gpurun_out/pytest_spill.log 2>&1; tail -2 gpurun_out/pytest_spill.log
for cfg in W48 C2 C4; do for sp in 0 1 0 1; do
  timeout 300 python bench.py --config $cfg --spill $sp --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sp_${cfg}_${sp}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sp_${cfg}_${sp}.log').read().strip().splitlines()[-1]);print('$cfg spill=$sp', round(d['ms_per_step'],3), 'xterm', round(d['phases_ms_per_step']['xterm'],3), 'TOPS', round(d['roofline']['achieved']), 'clk', d['roofline'].get('kernel_sm_mhz'))"
done; done
