# Round-2 evidence on HEAD (final kernels; + sanitizers) (under gpurun): smoke, all GPU tests, bench lines, ncu launch lists + captures
TAG=${TAG:-r02l}
mkdir -p gpurun_out/$TAG
O=gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > $O/smoke_$TAG.txt 2>&1; tail -2 $O/smoke_$TAG.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -25 > $O/pytest_gpu_$TAG.txt; tail -3 $O/pytest_gpu_$TAG.txt
for cfg in C4 C3 C5 W48 C2; do
  timeout -s KILL 900 python bench.py --config $cfg > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench_${TAG}_$cfg.json
  tail -1 $O/bench.log | cut -c1-200
done
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench_${TAG}_ref.json
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_c5_$TAG.csv python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1
TAG=$TAG bash tools/ncu_r02.sh > /dev/null 2>&1
ls gpurun_out/*$TAG* | head -30
