# A/B of the int8 cross-term variants (CPA_OPT_XT_TILES 1 = NT 2, 2 = NT 1 overlapped)
# usage (under gpurun): bash tools/ab_xt.sh
mkdir -p gpurun_out
for cfg in W48 C2 C4; do
  for xt in 1 2 0; do
    timeout -s KILL 600 python bench.py --config $cfg --xt-tiles $xt --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_xt_${cfg}_${xt}.log 2>&1
    python - "$cfg" "$xt" gpurun_out/ab_xt_${cfg}_${xt}.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    ph = d["phases_ms_per_step"]
    print(sys.argv[1], "xt", sys.argv[2], "step %.3f ms" % d["ms_per_step"], "xterm %.3f" % ph["xterm"],
          "moments %.3f" % ph["moments"], "mhz", d["roofline"].get("kernel_sm_mhz"))
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
  done
done
