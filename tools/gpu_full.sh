# Full round evidence (under gpurun): smoke, all GPU tests, bench lines, ncu.
# usage: TAG=r01h bash tools/gpu_full.sh
TAG=${TAG:-r01h}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-400
timeout -s KILL 600 python bench.py --config C3 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-300
timeout -s KILL 900 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1; tail -1 gpurun_out/bench_c5.log | cut -c1-300
timeout -s KILL 600 python bench.py --config W48 --steps 10 --warmup 3 > gpurun_out/bench_w48.log 2>&1; tail -1 gpurun_out/bench_w48.log | cut -c1-300
timeout -s KILL 600 python bench.py --config C4-HW --no-e2e --no-cpu-baseline > gpurun_out/bench_c4hw.log 2>&1; tail -1 gpurun_out/bench_c4hw.log | cut -c1-300
timeout -s KILL 600 python bench.py --config C4-HW --class-sums 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4hw_cs.log 2>&1; tail -1 gpurun_out/bench_c4hw_cs.log | cut -c1-300
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
bash profiles/run_ncu.sh $TAG > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:k_cs_sum -s 1 -c 1 -o gpurun_out/k_cs_sum_$TAG -f python bench.py --config C4-HW --class-sums 1 --no-e2e --no-cpu-baseline --no-clocks --steps 1 --warmup 1 > /dev/null 2>&1

# float path (C3): full captures of the cross term and the split pre-pass
BC3="python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_xterm -s 1 -c 1 -o gpurun_out/k_xterm_c3_$TAG -f $BC3 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_split_f32 -s 1 -c 1 -o gpurun_out/k_split_f32_c3_$TAG -f $BC3 > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_$TAG.csv python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1

ls gpurun_out
