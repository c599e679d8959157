# Float-path split diagnostics: per-column-block max |drho| vs the fp64 oracle,
# and the same error for a bf16-hi-only split simulated in numpy (the level a
# lost lo term would give).
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1412_7682_b200 as P
from oracle import oracle as O
from synth import synth as S


def bf16(x):
    b = np.asarray(x, np.float32).view(np.uint32)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def rho_of(texts, W):
    shw, sw, sw2 = O.sums_f32(O.HD_LAST, texts, W)
    sh, sh2 = O.model_sums(O.HD_LAST, texts)
    return O.rho_eq1_f64_grid(W.shape[0], shw, sh, sh2, sw, sw2)


for n, m in [(2000, 300), (65, 257), (1500, 200), (3000, 160)]:
    w = S.CONFIGS["C3"].replace(n=n, m=m, a=0.02)
    texts, W = S.dataset(w)
    eng = P.Engine(m, P.CPA_F32, P.CPA_HD_LAST, 0)
    eng.accumulate(torch.from_numpy(np.ascontiguousarray(W)).cuda(), torch.from_numpy(texts).cuda())
    out = eng.finalize(want_rho=True)
    rho = out["rho"].cpu().numpy()
    eng.close()
    ref = rho_of(texts, W)
    Wc = (W - W[0:1]).astype(np.float32)
    hi_only = rho_of(texts, bf16(Wc))
    e = np.abs(rho - ref).max(axis=0)
    eb = np.abs(hi_only - ref).max(axis=0)
    blocks = [(j, min(m, j + 32)) for j in range(0, m, 32)]
    print(f"n={n} m={m}: max {e.max():.3g} (bf16-hi-only sim {eb.max():.3g}); worst col {int(e.argmax())}")
    print("   per 32-col block:", " ".join(f"{e[a:b].max():.1e}" for a, b in blocks))
    print("   hi-only         :", " ".join(f"{eb[a:b].max():.1e}" for a, b in blocks))
