# rho-writing finalize on int32 rows: 16-byte loads in flight per thread U = 4 (default) vs 2 / 6 / 8
for rep in 1 2; do for lib in "" tools/alt_r2.so tools/alt_r6.so tools/alt_r8.so; do
  FIN_RHO=1 FIN_NARROW=1 FIN_M=48000 CPA_LIB_PATH=$lib timeout -s KILL 300 python tools/fin_bench.py 2>/dev/null | sed "s#^#${lib:-default} M48000 #" | cut -c1-150
  FIN_RHO=1 FIN_NARROW=1 FIN_M=20000 CPA_LIB_PATH=$lib timeout -s KILL 300 python tools/fin_bench.py 2>/dev/null | sed "s#^#${lib:-default} M20000 #" | cut -c1-150
done; done
