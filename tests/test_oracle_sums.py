"""Pins for the oracle's Phase 1 / Phase 2 exact integer sums [P:75, P:79;
S:230-243]: brute force, an independent numpy int64 contraction, closed forms
and the SPEC's special cases."""
import numpy as np
import pytest

from oracle import oracle as O


def h_matrix(model, texts):
    """Independent numpy evaluation of H[i, 256b+k] from the FIPS-pinned tables."""
    s, inv = O.aes_tables()
    sr = O.shiftrows_src()
    k = np.arange(256)
    pop = np.array([bin(v).count("1") for v in range(256)], np.int64)
    cols = []
    for b in range(16):
        x = texts[:, b:b + 1].astype(np.int64) ^ k[None, :]
        if model == O.HD_LAST:
            v = inv[x] ^ texts[:, sr[b]:sr[b] + 1]
        elif model == O.HW_LAST:
            v = inv[x]
        else:
            v = s[x]
        cols.append(pop[v])
    return np.concatenate(cols, axis=1)


def rand_data(n, m, seed, dtype=np.int8):
    rng = np.random.default_rng(seed)
    t = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    lo, hi = (-128, 128) if dtype == np.int8 else (0, 256)
    W = rng.integers(lo, hi, (n, m)).astype(dtype)
    return t, W


def test_triple_loop_brute_force():
    t, W = rand_data(20, 8, 0)                                   # [S:243]
    shw = O.cross_sums_i8(O.HD_LAST, t, W)
    sw, sw2 = O.trace_sums_i8(W)
    sh, sh2 = O.model_sums(O.HD_LAST, t)
    for h in (0, 1, 255, 256, 1000, 4095):
        b, k = divmod(h, 256)
        H = [O.selection(O.HD_LAST, t[i].tobytes(), b, k) for i in range(20)]
        assert sh[h] == sum(H) and sh2[h] == sum(x * x for x in H)
        for j in range(8):
            assert shw[h, j] == sum(H[i] * int(W[i, j]) for i in range(20))
    for j in range(8):
        assert sw[j] == sum(int(W[i, j]) for i in range(20))
        assert sw2[j] == sum(int(W[i, j]) ** 2 for i in range(20))


@pytest.mark.parametrize("model", [O.HD_LAST, O.HW_LAST, O.HW_FIRST])
@pytest.mark.parametrize("dtype", [np.int8, np.uint8])
def test_numpy_contraction(model, dtype):
    t, W = rand_data(300, 40, 1 + model, dtype)
    H = h_matrix(model, t)
    assert np.array_equal(O.cross_sums_i8(model, t, W), H.T @ W.astype(np.int64))
    sh, sh2 = O.model_sums(model, t)
    assert np.array_equal(sh, H.sum(0)) and np.array_equal(sh2, (H * H).sum(0))


def test_column_subset_matches_full():
    t, W = rand_data(100, 30, 5)
    cols = np.array([0, 3, 17, 29], np.int32)
    full = O.cross_sums_i8(O.HD_LAST, t, W)
    assert np.array_equal(O.cross_sums_i8(O.HD_LAST, t, W, cols), full[:, cols])


def test_closed_forms():
    """sum_k sumH = 1024 N, sum_k sumH2 = 4608 N, sum_k sumHW[b,k,j] = 1024 sumW[j]."""
    t, W = rand_data(200, 16, 6)
    for model in (O.HD_LAST, O.HW_LAST, O.HW_FIRST):
        sh, sh2 = O.model_sums(model, t)
        shw = O.cross_sums_i8(model, t, W)
        sw, _ = O.trace_sums_i8(W)
        assert (sh.reshape(16, 256).sum(1) == 1024 * 200).all()
        assert (sh2.reshape(16, 256).sum(1) == 4608 * 200).all()
        assert (shw.reshape(16, 256, 16).sum(1) == 1024 * sw[None, :]).all()
        assert (sh <= sh2).all() and (sh2 <= 8 * sh).all()          # [S:201]
        assert (200 * sh2 - sh * sh >= 0).all()                       # [S:202]


def test_special_cases():
    t, W = rand_data(1, 6, 7)                                      # n = 1 [S:234, S:242]
    sh, sh2 = O.model_sums(O.HD_LAST, t)
    shw = O.cross_sums_i8(O.HD_LAST, t, W)
    H = h_matrix(O.HD_LAST, t)[0]
    assert np.array_equal(sh, H) and np.array_equal(sh2, H * H)
    assert np.array_equal(shw, H[:, None] * W[0].astype(np.int64)[None, :])
    t, W = rand_data(50, 6, 8)                                     # duplicates [S:235]
    t2, W2 = np.concatenate([t, t]), np.concatenate([W, W])
    assert np.array_equal(O.model_sums(O.HD_LAST, t2)[0], 2 * O.model_sums(O.HD_LAST, t)[0])
    assert np.array_equal(O.cross_sums_i8(O.HD_LAST, t2, W2), 2 * O.cross_sums_i8(O.HD_LAST, t, W))
    Z = np.zeros_like(W)                                           # zero traces [S:241]
    assert not O.cross_sums_i8(O.HD_LAST, t, Z).any() and not any(O.trace_sums_i8(Z)[0])


def test_chunk_and_permutation_invariance():
    t, W = rand_data(120, 10, 9)
    full = O.cross_sums_i8(O.HD_LAST, t, W)
    parts = O.cross_sums_i8(O.HD_LAST, t[:37], W[:37]) + O.cross_sums_i8(O.HD_LAST, t[37:], W[37:])
    assert np.array_equal(full, parts)
    perm = np.random.default_rng(0).permutation(120)
    assert np.array_equal(full, O.cross_sums_i8(O.HD_LAST, t[perm], W[perm]))


def test_hypothesis_subset_sums_match_full():
    t, W = rand_data(150, 12, 21)
    hyps = np.array([0, 17, 256, 3333, 4095], np.int32)
    cols = np.array([2, 5, 11], np.int32)
    full = O.cross_sums_i8(O.HD_LAST, t, W)
    assert np.array_equal(O.cross_sums_hyps_i8(O.HD_LAST, t, W, hyps, cols), full[hyps][:, cols])
    sh, sh2 = O.model_sums(O.HD_LAST, t)
    a, b = O.model_sums_hyps(O.HD_LAST, t, hyps)
    assert np.array_equal(a, sh[hyps]) and np.array_equal(b, sh2[hyps])
