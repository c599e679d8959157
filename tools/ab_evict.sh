CPA_LIB_PATH=tools/libcpa_evl.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "c1_full or split_k or c2" 2>&1 | tail -1
LIBS=tools/libcpa_evl.so CFGS=C4 REPS=3 bash tools/ab.sh
for lib in "" tools/libcpa_evl.so; do
CPA_LIB_PATH=$lib timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_xterm -s 2 -c 1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | grep -E "dram__bytes_read|gpu__time" 
done
