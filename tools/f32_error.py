# max |rho_gpu - rho_oracle| for C3 at full size on sampled columns (float path precision)
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1412_7682_b200 as P
from oracle import oracle as O
from synth import synth as S
w = S.CONFIGS["C3"]
texts, lv = S.texts(w)
dW = torch.empty((w.n, w.m), dtype=torch.float32, device="cuda")
S.dev_traces(w, torch.from_numpy(lv).cuda(), 0, w.n, dW, w.m)
eng = P.Engine(w.m, P.CPA_F32, P.CPA_HD_LAST, 0)
eng.accumulate(dW, torch.from_numpy(texts).cuda())
out = eng.finalize(want_rho=True)
cols = np.array(sorted(set(w.leak_positions()[:4]) | {0, 7, 2500, w.m - 1}), np.int32)
Wc = S.traces(w, lv, 0, cols)
shw, sw, sw2 = O.sums_f32(O.HD_LAST, texts, Wc)
sh, sh2 = O.model_sums(O.HD_LAST, texts)
ref = O.rho_eq1_f64_grid(w.n, shw, sh, sh2, sw, sw2)
rho = out["rho"].cpu().numpy()[:, cols]
print("max|drho| %.3e" % np.max(np.abs(rho - ref)), "key", out["master_key"] == w.key)
