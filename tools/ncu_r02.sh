# Round-2 profiling (under gpurun): launch lists of the C4 and C3 steps and full
# captures of their kernels; then `python profiles/summarize.py <tag>` here.
TAG=${TAG:-r02}
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks \
    > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3_${TAG}.csv python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks \
    > /dev/null 2>&1
for k in k_xterm k_texthist k_hist_contract k_finalize_rows; do
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${k}_${TAG} -f $B > /dev/null 2>&1
done
for k in k_xterm k_split_f32; do
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${k}_c3_${TAG} -f $B --config C3 > /dev/null 2>&1
done
timeout -s KILL 300 ncu --set full --clock-control none -k regex:k_finalize_maxima -s 3 -c 1 \
    -o gpurun_out/k_finalize_maxima_c5_${TAG} -f python bench.py --config C5 --steps 1 --warmup 0 --no-clocks > /dev/null 2>&1
ls gpurun_out/*${TAG}*
