"""Phase-3 finalize (a8) timing: for each M, sums from N synthetic traces,
then cpa_finalize_rows(0, 4096) with and without rho, timed by the library's
CUDA events (phase 3) over FIN_ROUNDS rounds.  Kernel variants are compared by
running it against differently built libraries (CPA_LIB_PATH, tools/ab.sh);
DESIGN.md records the results.  One JSON line per (M, rho)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_7682_b200 as P  # noqa: E402
from synth import synth as S  # noqa: E402

VARIANTS = ["default"]


def main():
    cases = ((5000, 4096, False), (20000, 4096, False), (48000, 2048, False), (5000, 4096, True))
    only = os.environ.get("FIN_M")            # e.g. FIN_M=20000 (int path only)
    if only:
        cases = [c for c in cases if c[0] == int(only) and not c[2]]
    rhos = {"1": (True,), "0": (False,)}.get(os.environ.get("FIN_RHO", ""), (True, False))
    for M, n, f32 in cases:
        w = S.CONFIGS["C3" if f32 else "C2"].replace(n=n, m=M)
        texts, lv = S.texts(w)
        ld = (M + 15) // 16 * 16
        dW = torch.empty((n, ld), dtype=torch.float32 if f32 else torch.int8, device="cuda")
        S.dev_traces(w, torch.from_numpy(lv).cuda(), 0, n, dW, ld)
        eng = P.Engine(M, P.CPA_F32 if f32 else P.CPA_S8, P.CPA_HD_LAST, 0)
        if os.environ.get("FIN_NARROW") == "1":   # int32 sum_hw rows (CPA_OPT_NARROW)
            eng.set_narrow(True)
        eng.accumulate(dW[:, :M], torch.from_numpy(texts).cuda())
        eng.sync()
        for want_rho in rhos:
            ref = None
            times = {v: [] for v in VARIANTS}
            mx, am, pk = (t[0] for t in eng.maxima_buffers(1))
            for rnd in range(int(os.environ.get("FIN_ROUNDS", "5"))):   # interleaved: clock drift hits all alike
                for v in VARIANTS:
                    if rnd == 0:
                        rho = eng.finalize_rows(0, 4096, mx, am, pk, want_rho)
                        out = (rho, mx.clone(), am.clone(), pk.clone())
                        if ref is None:
                            ref = out
                        else:
                            same = all(torch.equal(a, b) for a, b in zip(out[1:], ref[1:])) and (
                                not want_rho or torch.equal(out[0], ref[0]))
                            assert same, f"variant {v} differs"
                    eng.set_timing(True)
                    eng.phase_times()
                    reps = 10
                    for _ in range(reps):
                        eng.finalize_rows(0, 4096, mx, am, pk, want_rho)
                    ms, cnt = eng.phase_times()
                    eng.set_timing(False)
                    times[v].append(ms["finalize"] / reps)
            nbytes = 4096 * M * (16 if want_rho else 8)
            res = {v: {"ms_min": round(min(t), 4), "ms_med": round(sorted(t)[len(t) // 2], 4),
                       "GBps_min_t": round(nbytes / (min(t) * 1e-3) / 1e9, 1)} for v, t in times.items()}
            print(json.dumps({"M": M, "dtype": "f64" if f32 else "i64", "rho": want_rho, "variants": res}), flush=True)
        eng.close()


if __name__ == "__main__":
    main()
