# usage (under gpurun): bash tools/gpu_tests.sh [pytest -k expr]
mkdir -p gpurun_out
K=${1:+-k "$1"}
eval timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 900 $K 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
