# gen-drain variants: parity tests on the variant library, then A/B against the default
mkdir -p gpurun_out
CPA_LIB_PATH=tools/alt_gdb.so timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -m gpu -x -q > gpurun_out/pytest_gd.log 2>&1
tail -2 gpurun_out/pytest_gd.log
LIBS="${LIBS:-tools/alt_gdb.so tools/alt_gdb36.so}" CFGS="${CFGS:-W48 C2 C4 C5}" REPS=2 STEPS=${STEPS:-5} bash tools/ab.sh
