#!/bin/bash
# Profiling recipe (B200_PROFILING.md), run under gpurun from the repo root:
#   bash profiles/run_ncu.sh <tag>
# Writes gpurun_out/{launches,xterm,moments,modelsums,finalize}_<tag>.* ; the
# summaries are then copied into profiles/ (tracked).
TAG=${1:-r01}
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
# every launch with its device time (cold-cache, serialised: compare SHARES)
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks \
    > gpurun_out/launches_${TAG}.log 2>&1
# full capture of each kernel of the step (second step = warm)
KERNELS=${KERNELS:-"k_xterm k_moments_i8 k_texthist k_hist_contract k_repack k_finalize_i8"}
for k in $KERNELS; do
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${k}_${TAG} -f $B > gpurun_out/${k}_${TAG}.log 2>&1
done
ls -la gpurun_out
