# ncu capture of one k_cs_sum launch (class-sum path, C4-HW); under gpurun
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_cs_sum -s 1 -c 1 -o gpurun_out/cs_sum_full -f python bench.py --config C4-HW --class-sums 1 --no-e2e --no-cpu-baseline --no-clocks --steps 1 --warmup 1 > gpurun_out/cs_full.log 2>&1; tail -2 gpurun_out/cs_full.log
