"""Step time of the device-resident attack, direct calls vs CUDA-graph replay
(include/cpa.h cpa_graph_*): reset + accumulate + finalize (direct) against
graph_launch of the captured reset + accumulate + finalize_async, each followed
by the key readback (best[32] D2H, key-schedule inversion on the host).  CUDA
events on the context's stream over K steps after W warm-up steps.  One JSON
line per config.  Usage: python tools/graph_bench.py [C2 C3 ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_7682_b200 as P  # noqa: E402
from synth import synth as S  # noqa: E402


def run(cfg, steps=20, warmup=5):
    w = S.CONFIGS[cfg]
    f32 = w.dtype == S.F32
    texts, lv = S.texts(w)
    ld = (w.m + 3) // 4 * 4 if f32 else (w.m + 15) // 16 * 16
    dW = torch.empty((w.n, ld), dtype=torch.float32 if f32 else torch.int8, device="cuda")
    S.dev_traces(w, torch.from_numpy(lv).cuda(), 0, w.n, dW, ld)
    dT = torch.from_numpy(texts).cuda()
    st = torch.cuda.Stream()
    eng = P.Engine(w.m, P.CPA_F32 if f32 else P.CPA_S8, w.leak_model, 0, stream=st)
    rank = torch.empty(4096, dtype=torch.int32, device="cuda")
    mx = torch.empty(4096, dtype=torch.float64, device="cuda")
    am = torch.empty(4096, dtype=torch.int32, device="cuda")
    best = torch.empty(32, dtype=torch.int32, device="cuda")
    best_h = torch.empty(32, dtype=torch.int32, pin_memory=True)
    torch.cuda.synchronize()

    def direct():
        eng.reset()
        eng.accumulate(dW[:, :w.m], dT)
        return bytes(P.cpa_finalize(eng.ctx, None, mx, am, rank).master_key)

    def replay():
        eng.graph_launch()
        with torch.cuda.stream(st):
            best_h.copy_(best, non_blocking=True)
        st.synchronize()
        rk = bytes(best_h[:16].numpy().astype(np.uint8))
        return bytes(P.cpa_aes_invert_key_schedule(rk, 10)) if w.leak_model != P.CPA_HW_FIRST else rk

    def timed(fn):
        for _ in range(warmup):
            key = fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            key = fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps, key

    t_direct, k1 = timed(direct)
    eng.graph_begin()
    eng.reset()
    eng.accumulate(dW[:, :w.m], dT)
    P.cpa_finalize_async(eng.ctx, None, mx, am, rank, best)
    eng.graph_end()
    t_graph, k2 = timed(replay)
    eng.close()
    return {"config": cfg, "ms_direct": round(t_direct, 4), "ms_graph": round(t_graph, 4),
            "key_ok": k1 == w.key and k2 == w.key}


if __name__ == "__main__":
    for cfg in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
        print(json.dumps(run(cfg)), flush=True)
