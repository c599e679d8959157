"""Run one accumulate+finalize on a synthetic config (debug / sanitizer aid).
usage: python tools/repro.py C2 [n] [kchunk] [a] [m]   (C3 runs the float path; a = leak amplitude;
m >= 8192 also takes the maxima-only finalize kernel in the finalize_rows call below)
REPRO_CLASS_SUMS=1 with an HW workload (C2-HW) takes the class-sum cross term."""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1412_7682_b200 as P
from synth import synth as S

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = S.CONFIGS[name]
if len(sys.argv) > 2:
    w = w.replace(n=int(sys.argv[2]))
if len(sys.argv) > 4 and float(sys.argv[4]) > 0:
    w = w.replace(a=float(sys.argv[4]))
if len(sys.argv) > 5:
    w = w.replace(m=int(sys.argv[5]))
texts, W = S.dataset(w)
f32 = w.dtype == S.F32
ld = (w.m + 3) // 4 * 4 if f32 else (w.m + 15) // 16 * 16
Wp = np.zeros((w.n, ld), W.dtype); Wp[:, :w.m] = W
eng = P.Engine(w.m, P.CPA_F32 if f32 else P.CPA_S8, w.leak_model, 0)
if os.environ.get("REPRO_CLASS_SUMS") == "1":
    eng.set_class_sums(True)
if len(sys.argv) > 3 and int(sys.argv[3]):
    eng.set_kchunk(int(sys.argv[3]))
eng.accumulate(torch.from_numpy(Wp).cuda()[:, :w.m], torch.from_numpy(texts).cuda())
out = eng.finalize(want_rho=True)
mx, am, pk = (t[0] for t in eng.maxima_buffers(1))
eng.finalize_rows(100, 900, mx, am, pk)
sel = eng.select(*(t.view(1, -1).repeat(2, 1) for t in (out["maxabs"], out["argmax"], out["maxabs"])))
print("key", out["master_key"].hex(), "ok" if out["master_key"] == w.key else "WRONG")
