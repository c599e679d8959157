#!/bin/bash
# Profiling recipe (B200_PROFILING.md), run under gpurun from the repo root.
# $1 = tag (round/change name).  Writes into gpurun_out/.
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
# launch list of the bench command (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/launches_${TAG}.log 2>&1
# full capture of the top kernel
ncu --set full --clock-control none --import-source on -k regex:k_xterm -s 1 -c 1 -o gpurun_out/xterm_${TAG} -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/xterm_${TAG}.log 2>&1
ncu --set full --clock-control none -k regex:k_moments -s 1 -c 1 -o gpurun_out/moments_${TAG} -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/moments_${TAG}.log 2>&1
