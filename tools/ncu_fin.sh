# ncu full capture of the finalize kernels (tools/fin_bench.py cases), under gpurun
mkdir -p gpurun_out
for v in 14 14nf; do
  FIN_M=20000 FIN_RHO=0 FIN_VARIANTS=$v timeout -s KILL 300 ncu --set full --clock-control none --import-source on \
     -k regex:k_finalize_rows -s 3 -c 1 -o gpurun_out/fin_${v}_r02 -f python tools/fin_bench.py > gpurun_out/fin_${v}.log 2>&1
done
FIN_M=48000 FIN_RHO=1 FIN_VARIANTS=14 timeout -s KILL 300 ncu --set full --clock-control none --import-source on \
     -k regex:k_finalize_rows -s 3 -c 1 -o gpurun_out/fin_rho_r02 -f python tools/fin_bench.py > gpurun_out/fin_rho.log 2>&1
ls gpurun_out
