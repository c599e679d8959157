"""Pins for Eq. (1) [P:69] (reference B, from exact integers) and the two-pass
Pearson (reference A) [S:244-251, S:274-285, S:455]; and Phases 3/4
[P:83; S:252-265]."""
from decimal import Decimal, getcontext

import numpy as np
import pytest

from oracle import oracle as O
from synth import synth as S
from tests.test_oracle_sums import h_matrix, rand_data


def test_perfect_and_anti_correlation():
    t, _ = rand_data(60, 1, 11)
    H = h_matrix(O.HD_LAST, t)
    h = 256 * 3 + 77
    W = np.stack([H[:, h], -H[:, h], np.full(60, 5)], 1).astype(np.int8)  # [S:248-250]
    r = O.attack_i8(O.HD_LAST, t, W)["rho"][h]
    assert r[0] == 1.0 and r[1] == -1.0 and r[2] == 0.0
    ra = O.rho_two_pass_i8(O.HD_LAST, t, W, hyps=[h])[0]
    assert abs(ra[0] - 1) <= 1e-12 and abs(ra[1] + 1) <= 1e-12 and ra[2] == 0.0


def test_numpy_corrcoef_tiny():
    t, W = rand_data(40, 5, 12)
    H = h_matrix(O.HD_LAST, t).astype(float)
    r = O.attack_i8(O.HD_LAST, t, W)["rho"]
    for h in (0, 500, 4095):
        for j in range(5):
            ref = np.corrcoef(H[:, h], W[:, j].astype(float))[0, 1]
            assert abs(r[h, j] - ref) <= 1e-12


def test_exact_rational_spot_cells():
    """rho_B is within 1 ulp of the exact value num / sqrt(dw dh) (50 digits)."""
    getcontext().prec = 50
    t, W = rand_data(500, 4, 13)
    a = O.attack_i8(O.HD_LAST, t, W)
    n = 500
    for h in (7, 1234, 3000):
        for j in range(4):
            num = n * int(a["sum_hw"][h, j]) - int(a["sum_h"][h]) * int(a["sum_w"][j])
            dw = n * int(a["sum_w2"][j]) - int(a["sum_w"][j]) ** 2
            dh = n * int(a["sum_h2"][h]) - int(a["sum_h"][h]) ** 2
            exact = Decimal(num) / (Decimal(dw).sqrt() * Decimal(dh).sqrt())
            got = a["rho"][h, j]
            assert abs(Decimal(got) - exact) <= Decimal(np.spacing(abs(got))) * 2


def test_two_pass_agreement_acceptance_1():
    """SPEC acceptance 1: n=50, m=64, all 4096x64 cells within 1e-9."""
    t, W = rand_data(50, 64, 14)
    rb = O.attack_i8(O.HD_LAST, t, W)["rho"]
    ra = O.rho_two_pass_i8(O.HD_LAST, t, W)
    assert np.max(np.abs(ra - rb)) <= 1e-9
    assert np.all(np.abs(rb) <= 1.0)


def test_affine_invariance_exact():
    """Integer offset: num and dw unchanged exactly -> bit-identical rho_B;
    negation: exact sign flip; duplication: bit-identical [S:285]."""
    t, W = rand_data(300, 12, 15)
    W = np.clip(W, -100, 100).astype(np.int8)
    r0 = O.attack_i8(O.HD_LAST, t, W)["rho"]
    r1 = O.attack_i8(O.HD_LAST, t, (W.astype(np.int16) + 27).astype(np.int8))["rho"]
    assert np.array_equal(r0, r1)
    rn = O.attack_i8(O.HD_LAST, t, (-W.astype(np.int16)).astype(np.int8))["rho"]
    assert np.array_equal(rn, -r0)
    ru = O.attack_i8(O.HD_LAST, t, (W.astype(np.int16) + 128).astype(np.uint8))["rho"]
    assert np.array_equal(ru, r0)                         # u8 = s8 + 128
    rd = O.attack_i8(O.HD_LAST, np.concatenate([t, t]), np.concatenate([W, W]))["rho"]
    assert np.array_equal(rd, r0)


def test_eq1_overflow_guard():
    with pytest.raises(OverflowError):
        O.rho_eq1(2**40, 2**40, 2**40, 2**41, 2**40, 2**50)


def test_phase3_phase4_constructed_surfaces():
    rho = np.zeros((4096, 3))
    for b in range(16):
        rho[256 * b + b, 1] = -1.0                           # [S:263]
    mx, am, pk = O.phase3(rho)
    best, rank = O.phase4(mx)
    assert best.tolist() == list(range(16))
    assert all(am[256 * b + b] == 1 and pk[256 * b + b] == -1.0 for b in range(16))
    best, rank = O.phase4(np.zeros(4096))                    # all equal -> 0x00 [S:264]
    assert best.tolist() == [0] * 16 and rank[:256].tolist() == list(range(1, 257))
    rho = np.full((4096, 4), 0.25)                           # ties -> lowest sample
    mx, am, _ = O.phase3(rho, np.array([3, 5, 8, 9], np.int32))
    assert (am == 3).all()


def test_end_to_end_noiseless_and_noisy():
    """[S:331, S:341, S:456-457]: noiseless -> rho = 1 exactly at the planted
    sample for all 16 bytes; noisy C1 -> the true round-10 key, master key."""
    for name in ("C1-0", "C1"):
        w = S.CONFIGS[name]
        t, W = S.dataset(w)
        a = O.attack_i8(O.HD_LAST, t, W)
        rk = O.expand_key(w.key)[10].astype(int)
        assert a["best"].tolist() == rk.tolist()
        assert O.invert_key_schedule(a["best"].tobytes()).tobytes() == w.key
        hs = [256 * b + rk[b] for b in range(16)]
        assert a["argmax"][hs].tolist() == w.leak_positions()
        assert (a["rank"][hs] == 1).all()
        if name == "C1-0":
            assert np.all(np.abs(a["maxabs"][hs] - 1.0) <= 1e-12)


def test_float_oracle_pins():
    """Float-trace oracle [S:297]: fp64 sums equal an independent numpy fp64
    contraction; on integer-valued float traces the float and int oracles agree;
    Eq. (1) in fp64 agrees with the two-pass reference."""
    rng = np.random.default_rng(21)
    t = rng.integers(0, 256, (300, 16), dtype=np.uint8)
    Wf = (rng.normal(1.0, 0.05, (300, 20))).astype(np.float32)
    H = h_matrix(O.HD_LAST, t).astype(np.float64)
    shw, sw, sw2 = O.sums_f32(O.HD_LAST, t, Wf)
    assert np.allclose(shw, H.T @ Wf.astype(np.float64), rtol=1e-14, atol=0)
    assert np.allclose(sw, Wf.astype(np.float64).sum(0), rtol=1e-14)
    assert np.allclose(sw2, (Wf.astype(np.float64) ** 2).sum(0), rtol=1e-14)
    sh, sh2 = O.model_sums(O.HD_LAST, t)
    rb = O.rho_eq1_f64_grid(300, shw, sh, sh2, sw, sw2)
    ra = O.rho_two_pass_f32(O.HD_LAST, t, Wf)
    assert np.max(np.abs(ra - rb)) <= 1e-9
    Wi = rng.integers(-100, 100, (300, 20)).astype(np.int8)
    ri = O.rho_two_pass_i8(O.HD_LAST, t, Wi)
    rf = O.rho_two_pass_f32(O.HD_LAST, t, Wi.astype(np.float32))
    assert np.array_equal(ri, rf)


def degenerate_columns(n=400, seed=31):
    """Float columns on both sides of SPEC's degenerate-variance rule [S:293]
    (rho = 0 iff n*sum w^2 - (sum w)^2 <= 1e-12 * n * sum w^2, RAW sums), each
    >= 4x away from the boundary: a DC level far above the noise makes a column
    degenerate although its variance is not 0.  Returns (W [n][6] f32, expected
    degenerate flags decided in exact rational arithmetic on the f32 values)."""
    from fractions import Fraction
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((n, 6))
    dc = np.array([1000.0, 1000.0, 1.0, 1.0, 0.0, 3.0])
    sd = np.array([0.0, 0.05, 3e-7, 4e-6, 1.0, 1e-3])
    W = (dc + sd * z).astype(np.float32)
    W[::7, 0] = np.nextafter(np.float32(1000.0), np.float32(2000.0))  # var > 0, 1 ulp steps
    flags = []
    for j in range(6):
        v = [Fraction(float(x)) for x in W[:, j]]
        s1, s2 = sum(v), sum(x * x for x in v)
        dw = n * s2 - s1 * s1
        ratio = dw / (n * s2)
        eps = Fraction(1, 10**12)
        assert ratio <= eps / 4 or ratio >= 4 * eps, (j, float(ratio))
        flags.append(ratio <= eps)
    assert flags == [True, False, True, False, False, False]
    return W, flags


def test_float_degenerate_rule_pinned():
    """The eps branch of both float oracle functions [S:293]: columns whose
    variance is below 1e-12 of their raw second moment give rho = 0 exactly,
    the others the textbook Pearson value (numpy.corrcoef)."""
    W, flags = degenerate_columns()
    rng = np.random.default_rng(32)
    t = rng.integers(0, 256, (W.shape[0], 16), dtype=np.uint8)
    H = h_matrix(O.HD_LAST, t).astype(np.float64)
    shw, sw, sw2 = O.sums_f32(O.HD_LAST, t, W)
    sh, sh2 = O.model_sums(O.HD_LAST, t)
    rb = O.rho_eq1_f64_grid(W.shape[0], shw, sh, sh2, sw, sw2)
    hyps = np.array([0, 77, 1000, 4095], np.int32)
    ra = O.rho_two_pass_f32(O.HD_LAST, t, W, hyps=hyps)
    for j, deg in enumerate(flags):
        if deg:
            assert np.all(rb[:, j] == 0.0) and np.all(ra[:, j] == 0.0), j
        else:
            for a, h in enumerate(hyps):
                ref = np.corrcoef(H[:, h], W[:, j].astype(np.float64))[0, 1]
                assert abs(ra[a, j] - ref) <= 1e-9, (j, h)
                assert abs(rb[h, j] - ref) <= 1e-4, (j, h)
                assert ref != 0.0
