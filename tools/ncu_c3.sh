mkdir -p gpurun_out
for xt in 1 2; do
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_xterm -s 1 -c 1 \
   -o gpurun_out/xterm_c3_xt${xt} -f python bench.py --config C3 --xt-tiles $xt --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_c3_xt${xt}.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
