for rep in 1 2; do for lib in tools/fm_head.so tools/fm_r1u4.so; do
  FIN_RHO=0 FIN_ROUNDS=3 CPA_LIB_PATH=$lib timeout 300 python tools/fin_bench.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); v=d['variants']['default']; print('${lib:-default}', d['M'], d['dtype'], v['ms_min'], v['GBps_min_t'])"
done; done
