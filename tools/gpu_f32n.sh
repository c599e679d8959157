mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_float_gpu.py tests/test_bench_gpu.py -q -x --timeout 900 -k "float" > gpurun_out/pytest_f32n.log 2>&1; tail -2 gpurun_out/pytest_f32n.log
for xt in 1 2 1 2; do
  timeout 300 python bench.py --config C3 --xt-tiles $xt --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c3_$xt.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/c3_$xt.log').read().strip().splitlines()[-1]);print('C3 xt=$xt', round(d['ms_per_step'],3), 'xterm', round(d['phases_ms_per_step']['xterm'],3), 'frac', round(d['roofline']['frac_of_mma_ceiling_at_kernel_clock'],3), 'clk', d['roofline'].get('kernel_sm_mhz'), d['key_recovered'])"
done
