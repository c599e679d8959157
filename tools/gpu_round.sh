# new GPU tests, sanitizer, and bench lines (C4 default, W48)
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py --config W48 --steps 10 --warmup 3 > gpurun_out/bench_w48.log 2>&1; tail -1 gpurun_out/bench_w48.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log
bash tools/sanitize.sh > /dev/null 2>&1; tail -60 gpurun_out/sanitize.log
