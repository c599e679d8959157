"""One-GPU proxy of the multi-GPU combine at the G = 8 shard size of C4
(N = 1.5M / 8 = 187,500 traces per rank, M = 5000): the cross-term kernel's
time with its rows spilled into its own accumulator (red.add.u64, the 'rows' /
'allreduce' combines, which then run NCCL) and with row owners set to its own
accumulator (system-scope red.add, the 'fused' combine's epilogue, here without
NVLink), plus the unit schedule each uses.  Prints one JSON line.

    python tools/combine_proxy.py [--shards 8] [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1412_7682_b200 as P  # noqa: E402
from synth import synth as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    w = S.CONFIGS["C4"]
    n = w.n // a.shards
    texts, lv = S.texts(w, 0, n)
    ld = (w.m + 15) // 16 * 16
    dW = torch.empty((n, ld), dtype=torch.int8, device="cuda")
    S.dev_traces(w, torch.from_numpy(lv).cuda(), 0, n, dW, ld)
    dT = torch.from_numpy(texts).cuda()
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    out = {"config": f"C4 shard: {n} traces x {w.m} samples (G = {a.shards})"}
    for mode in ("own", "owners_self"):
        eng.set_row_owners([0] * 16 if mode == "owners_self" else None)
        for _ in range(3):
            eng.reset()
            eng.accumulate(dW[:, :w.m], dT)
        eng.sync()
        eng.set_timing(True)
        eng.phase_times()
        for _ in range(a.reps):
            eng.reset()
            eng.accumulate(dW[:, :w.m], dT)
        ms, cnt = eng.phase_times()
        eng.set_timing(False)
        xt = ms["xterm"] / cnt["xterm"]
        ops = 2.0 * 4096 * n * w.m
        out[mode] = {"xterm_ms": xt, "tops": ops / (xt * 1e-3) / 1e12,
                     "step_ms": sum(ms.values()) / a.reps}
    eng.set_row_owners(None)
    out["sum_hw_bytes_per_rank"] = 4096 * w.m * 8
    out["note"] = ("own: each unit's int64 tile red.add'ed into the local accumulator (then NCCL reduce-scatter "
                   "or all-reduce moves (G-1)/G or 2(G-1)/G of it); owners_self: the fused combine's "
                   "system-scope red.add path and longer units (auto_kchunk's remote-epilogue model) into the "
                   "local accumulator -- the NVLink leg is not in this proxy")
    print(json.dumps(out))
    eng.close()


if __name__ == "__main__":
    main()
