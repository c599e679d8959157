"""The seeded input generator: determinism, noise statistics [S:330-338],
independent-AES agreement with the oracle's AES [S:343], and column-subset
consistency (the property the full-size parity tests rely on)."""
import numpy as np

from oracle import oracle as O
from synth import synth as S


def test_gauss_table_moments():
    g = S.gauss_table().astype(np.float64) / 65536.0
    assert np.all(np.diff(g) >= 0) and np.allclose(g, -g[::-1])
    assert abs(g.mean()) < 1e-9 and abs(g.var() - 1.0) < 1e-4   # quantised N(0, 1)
    # draws through the counter hash: 10^6 samples
    w = S.CONFIGS["C2"].replace(n=200, m=5000, a=0.0, sigma=1.0, mu_lo=0, mu_hi=0, dtype=S.F32)
    _, lv = S.texts(w)
    z = S.traces(w, lv).ravel().astype(np.float64)
    assert abs(z.mean()) < 0.005 and 0.99 < z.var() < 1.01       # [S:337-338]


def test_determinism_and_subset():
    w = S.CONFIGS["C1"]
    t1, W1 = S.dataset(w)
    t2, W2 = S.dataset(w)
    assert np.array_equal(t1, t2) and np.array_equal(W1, W2)    # [S:330]
    cols = np.array([3, 29, 400, 499], np.int32)
    _, lv = S.texts(w)
    assert np.array_equal(S.traces(w, lv, 0, cols), W1[:, cols])
    t3, lv3 = S.texts(w, 100, 50)
    assert np.array_equal(t3, t1[100:150])
    assert np.array_equal(S.traces(w, lv3, 100), W1[100:150])
    assert not np.array_equal(S.dataset(w.replace(seed=2))[1], W1)


def test_ciphertexts_match_oracle_aes():
    w = S.CONFIGS["C1"].replace(n=200)
    ct, _ = S.texts(w)
    pt, _ = S.texts(w.replace(leak_model=S.LEAK_HW_FIRST))
    for i in range(200):
        c, _ = O.encrypt_with_states(pt[i].tobytes(), w.key)
        assert c.tobytes() == ct[i].tobytes()
