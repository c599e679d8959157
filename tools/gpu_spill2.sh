for cfg in W48 C2; do for sp in 1 1; do
  timeout 300 python bench.py --config $cfg --spill $sp --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sp_${cfg}_${sp}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sp_${cfg}_${sp}.log').read().strip().splitlines()[-1]);print('$cfg spill=$sp', round(d['ms_per_step'],3), 'xterm', round(d['phases_ms_per_step']['xterm'],3), 'TOPS', round(d['roofline']['achieved']), 'clk', d['roofline'].get('kernel_sm_mhz'))"
done; done
