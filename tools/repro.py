"""Run one accumulate+finalize on a synthetic config (debug / sanitizer aid).
usage: python tools/repro.py C2 [n] [kchunk]"""
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
texts, W = S.dataset(w)
ld = (w.m + 15) // 16 * 16
Wp = np.zeros((w.n, ld), np.int8); Wp[:, :w.m] = W
eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
if len(sys.argv) > 3:
    eng.set_kchunk(int(sys.argv[3]))
eng.accumulate(torch.from_numpy(Wp).cuda()[:, :w.m], torch.from_numpy(texts).cuda())
out = eng.finalize()
print("key", out["master_key"].hex(), "ok" if out["master_key"] == w.key else "WRONG")
