#!/bin/bash
# Cross-term bottleneck experiments (run under gpurun): xterm ms per launch for
# the normal build and the XT_EXP builds (tools/libcpa_exp<N>.so; see xterm.cu).
for lib in "" ${LIBS:-tools/libcpa_exp1.so tools/libcpa_exp2.so tools/libcpa_exp3.so}; do
  CPA_LIB_PATH=$lib timeout 200 python bench.py --no-e2e --no-cpu-baseline --no-clocks --steps ${STEPS:-5} --no-overlap "$@" 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-normal}', 'xterm %.3f ms' % d['roofline']['ms_per_launch'])"
done
