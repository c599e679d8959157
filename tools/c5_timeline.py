"""GPU timeline of the streamed C5 step (CUPTI via torch.profiler): kernel
start/end times of two steps, the busy fraction and the largest gaps between
consecutive GPU activities.  Usage: python tools/c5_timeline.py [config]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    sys.argv = ["bench.py", "--config", cfg, "--steps", "2", "--warmup", "2", "--no-clocks", "--no-phase-times",
                "--no-e2e", "--no-cpu-baseline"]
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        bench.main()
    out = os.path.join(ROOT, "gpurun_out", f"timeline_{cfg}.json")
    prof.export_chrome_trace(out)
    ev = json.load(open(out))["traceEvents"]
    k = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")],
               key=lambda e: e["ts"])
    # the last 40% of the trace: the timed steps (after warm-up and data generation)
    t_end = k[-1]["ts"] + k[-1]["dur"]
    k = [e for e in k if e["ts"] > t_end - 0.45 * (t_end - k[0]["ts"])]
    span = k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]
    busy, gaps, prev_end = 0.0, [], k[0]["ts"]
    for e in k:
        gaps.append((e["ts"] - prev_end, e["name"][:60]))
        busy += e["dur"]
        prev_end = max(prev_end, e["ts"] + e["dur"])
    gaps.sort(reverse=True)
    tot_gap = sum(g for g, _ in gaps if g > 0)
    print(json.dumps({"events": len(k), "span_ms": span / 1e3, "busy_ms": busy / 1e3, "gaps_ms": tot_gap / 1e3,
                      "largest_gaps_us": [(round(g, 1), n) for g, n in gaps[:15]]}, indent=1))
    by = {}
    for e in k:
        by.setdefault(e["name"][:50], [0, 0.0])
        by[e["name"][:50]][0] += 1
        by[e["name"][:50]][1] += e["dur"] / 1e3
    for n, (c, t) in sorted(by.items(), key=lambda x: -x[1][1])[:12]:
        print(f"{t:9.3f} ms {c:5d}  {n}")


if __name__ == "__main__":
    main()
