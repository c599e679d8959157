"""Pins for the selection function H [P:67; S:83-103].

The worked example is FIPS-197 App. B: with the true round-10 key the HD_LAST
value must equal the Hamming distance between the printed round-10 start state
and the printed ciphertext at register position SR(b) [S:96]."""
import numpy as np

from oracle import oracle as O
from synth import synth as S


def popcount(v):
    return bin(int(v)).count("1")


def test_fips_b_worked_example(fips):
    ct, start, rk10 = fips["b_ct"], fips["b_r10_start"], fips["b_r10_key"]
    sr = O.shiftrows_src()
    hd = [O.selection(O.HD_LAST, ct, b, rk10[b]) for b in range(16)]
    assert hd == [popcount(start[sr[b]] ^ ct[sr[b]]) for b in range(16)]
    assert hd == [4, 5, 4, 3, 5, 3, 3, 2, 5, 4, 5, 7, 1, 4, 3, 3]
    hw = [O.selection(O.HW_LAST, ct, b, rk10[b]) for b in range(16)]
    assert hw == [popcount(start[sr[b]]) for b in range(16)]
    # first-round model with the plaintext: HW of the printed round-1 SubBytes state
    hf = [O.selection(O.HW_FIRST, fips["b_pt"], b, fips["a1_key"][b]) for b in range(16)]
    assert hf == [popcount(x) for x in fips["b_r1_sbox"]]


def test_per_bit_brute_force():
    s, inv = O.aes_tables()
    sr = O.shiftrows_src()
    rng = np.random.default_rng(1)
    for _ in range(300):
        c = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        b, k = int(rng.integers(16)), int(rng.integers(256))
        x, y = inv[c[b] ^ k], c[sr[b]]
        bits = sum(((x >> i) & 1) != ((y >> i) & 1) for i in range(8))  # [S:89]
        assert O.selection(O.HD_LAST, c, b, k) == bits


def test_zero_when_register_unchanged():
    s, inv = O.aes_tables()
    sr = O.shiftrows_src()
    c = bytearray(16)
    for b in (1, 6, 11):
        k = 0x3c
        c[sr[b]] = inv[c[b] ^ k]          # [S:88]
        assert O.selection(O.HD_LAST, bytes(c), b, k) == 0


def test_xor_mask_invariance():
    rng = np.random.default_rng(2)
    for _ in range(200):                  # [S:102]
        c = bytearray(rng.integers(0, 256, 16, dtype=np.uint8).tobytes())
        b, k, m = int(rng.integers(16)), int(rng.integers(256)), int(rng.integers(256))
        h0 = O.selection(O.HD_LAST, bytes(c), b, k)
        c2 = bytearray(c)
        c2[b] ^= m
        if O.shiftrows_src()[b] == b:     # bytes 0,4,8,12: c[b] also is c[SR(b)]
            continue
        assert O.selection(O.HD_LAST, bytes(c2), b, k ^ m) == h0


def test_closed_form_sum_over_keys():
    """Each model is HW of a bijection of (text byte ^ k): over the 256 keys,
    sum H = 8 * 128 = 1024 and sum H^2 = 256 * (8 + 8*7/4) = 4608."""
    rng = np.random.default_rng(3)
    for model in (O.HD_LAST, O.HW_LAST, O.HW_FIRST):
        for _ in range(20):
            c = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
            for b in (0, 5, 12):
                hs = [O.selection(model, c, b, k) for k in range(256)]
                assert sum(hs) == 1024 and sum(h * h for h in hs) == 4608


def test_true_key_equals_register_hd():
    """[S:96, S:103]: for the true key, HD_LAST equals the HD of the round-10
    register transition, for >= 1000 random encryptions."""
    rng = np.random.default_rng(4)
    sr = O.shiftrows_src()
    key = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
    rk10 = O.expand_key(key)[10]
    for _ in range(1000):
        pt = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        ct, st = O.encrypt_with_states(pt, key)
        for b in range(16):
            assert O.selection(O.HD_LAST, ct.tobytes(), b, int(rk10[b])) == popcount(st[sr[b]] ^ ct[sr[b]])


def test_synth_planted_leak_matches_selection():
    """The generator's planted value is the selection value at the true key."""
    w = S.CONFIGS["C1"].replace(n=64)
    for model, lm in ((O.HD_LAST, S.LEAK_HD_LAST), (O.HW_LAST, S.LEAK_HW_LAST), (O.HW_FIRST, S.LEAK_HW_FIRST)):
        t, lv = S.texts(w.replace(leak_model=lm))
        kk = O.expand_key(w.key)[0 if model == O.HW_FIRST else 10]
        for i in range(64):
            assert [O.selection(model, t[i].tobytes(), b, int(kk[b])) for b in range(16)] == lv[i].tolist()
