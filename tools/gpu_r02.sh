# Round-2 evidence run on HEAD (under gpurun): smoke, GPU tests, bench lines, launch list.
# usage: TAG=r02a bash tools/gpu_r02.sh
TAG=${TAG:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -25 > gpurun_out/pytest_gpu_${TAG}.log
tail -2 gpurun_out/pytest_gpu_${TAG}.log
for cfg in C4 C3 C5 W48 C2; do
  timeout -s KILL 900 python bench.py --config $cfg $( [ $cfg != C4 ] && echo --no-cpu-baseline ) > gpurun_out/bench_${TAG}_${cfg}.log 2>&1
  tail -1 gpurun_out/bench_${TAG}_${cfg}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_${TAG}_ref.log 2>&1; tail -1 gpurun_out/bench_${TAG}_ref.log | cut -c1-200
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1
ls gpurun_out | head -50
