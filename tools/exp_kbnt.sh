# KB/NT variants of the int8 cross term (run under gpurun): parity + C4 bench per lib
for lib in "" ${LIBS:-tools/libcpa_kb2nt1.so}; do
  CPA_LIB_PATH=$lib timeout 300 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -1
  for mode in ${MODES:-3 1}; do
  for i in 1 2; do
    CPA_LIB_PATH=$lib timeout 200 python bench.py --no-e2e --no-cpu-baseline --steps 10 --overlap-mode $mode 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${lib:-normal} mode $mode', 'step %.2f xterm %.3f ms clk %s key %s' % (d['ms_per_step'], r['ms_per_launch'], d['clocks']['sm_mhz'], d['key_recovered']))"
  done; done
done
