set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
(echo "== tools/pair_bench (tcgen05.mma cta_group::2 kind::i8 issue rate)"; timeout 120 ./tools/pair_bench; echo "== tools/mma_bench (cta_group::1, kind::i8 / kind::f16)"; timeout 120 ./tools/mma_bench; echo "== tools/peak_int8.py (cuBLASLt)"; timeout 120 python tools/peak_int8.py) > gpurun_out/mma_bench.txt 2>&1
timeout 300 python tools/combine_proxy.py > gpurun_out/combine_proxy.json 2> gpurun_out/combine_proxy.err
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout -s KILL 1200 python -m pytest tests/test_bench_gpu.py -q --timeout 900 > gpurun_out/pytest_bench.log 2>&1
tail -3 gpurun_out/pytest_bench.log
