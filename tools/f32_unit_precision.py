"""Float path (a6): max |rho_gpu - rho_oracle| at full C3 (100K x 5000, sampled
columns incl. the leak samples) and at small N, for several fp32 TMEM
accumulation lengths (CPA_OPT_KCHUNK) -- the precision side of the unit-length
choice.  Run with a library built with -DF32_MAX_UNIT_NT2=32768 (CPA_LIB_PATH)
to allow units beyond the default bound.  One JSON line per case."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_7682_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from synth import synth as S  # noqa: E402


def run(w, kc, cols=None):
    texts, lv = S.texts(w)
    dW = torch.empty((w.n, w.m), dtype=torch.float32, device="cuda")
    S.dev_traces(w, torch.from_numpy(lv).cuda(), 0, w.n, dW, w.m)
    eng = P.Engine(w.m, P.CPA_F32, P.CPA_HD_LAST, 0)
    if kc:
        eng.set_kchunk(kc)
    eng.accumulate(dW, torch.from_numpy(texts).cuda())
    out = eng.finalize(want_rho=True)
    cols = np.arange(w.m, dtype=np.int32) if cols is None else cols
    Wc = S.traces(w, lv, 0, cols)
    shw, sw, sw2 = O.sums_f32(O.HD_LAST, texts, Wc)
    sh, sh2 = O.model_sums(O.HD_LAST, texts)
    ref = O.rho_eq1_f64_grid(w.n, shw, sh, sh2, sw, sw2)
    err = float(np.max(np.abs(out["rho"].cpu().numpy()[:, cols] - ref)))
    eng.close()
    return err, out["master_key"] == w.key


def main():
    kcs = [int(x) for x in os.environ.get("KCS", "4096,8192,16384,32768").split(",")]
    w3 = S.CONFIGS["C3"]
    cols = np.array(sorted(set(w3.leak_positions()) | {0, 1, 2500, 4999}), np.int32)
    for kc in kcs:
        err, ok = run(w3, kc, cols)
        print(json.dumps({"case": "C3 full, 20 columns", "kchunk": kc, "max_abs_drho": err, "key": ok}), flush=True)
    for n, m in ((3000, 160), (65, 257)):
        w = S.CONFIGS["C3"].replace(n=n, m=m, a=0.02)
        err, _ = run(w, 0)
        print(json.dumps({"case": f"{n}x{m}", "kchunk": "auto", "max_abs_drho": err}), flush=True)


if __name__ == "__main__":
    main()
