"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bar: int64 sums bit-exact; rho
bit-exact to Eq. (1)-from-integers (reference B) and within 1e-9 relative
(+1e-12 abs) of the two-pass reference A; max/argmax/ranks/key identical."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from synth import synth as S  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1412_7682_b200 as P
    return P


MODEL = {O.HD_LAST: 0, O.HW_LAST: 1, O.HW_FIRST: 2}


def run_gpu(P, texts, W, model=0, kchunk=0, chunks=None, want_rho=True, overlap=True, mode=None, fuse_hist=None,
            xt=None, spill=None, narrow=None):
    dtype = {np.int8: P.CPA_S8, np.uint8: P.CPA_U8}[W.dtype.type]
    eng = P.Engine(W.shape[1], dtype, model, 0)
    if narrow is not None:
        eng.set_narrow(narrow)
    if xt is not None:
        eng.set_xt_tiles(xt)
    if spill is not None:
        eng.set_spill(spill)
    if kchunk:
        eng.set_kchunk(kchunk)
    if not overlap:
        eng.set_overlap(False)
    if mode is not None:
        eng.set_overlap(mode)
    if fuse_hist is not None:
        eng.set_fuse_hist(fuse_hist)
    bounds = chunks or [0, W.shape[0]]
    # pad rows to a 16-byte multiple (TMA stride rule); ld > M exercises strides
    ld = (W.shape[1] + 15) // 16 * 16
    Wp = np.zeros((W.shape[0], ld), W.dtype)
    Wp[:, :W.shape[1]] = W
    dW = torch.from_numpy(Wp).cuda()
    dT = torch.from_numpy(np.ascontiguousarray(texts)).cuda()
    for a, b in zip(bounds[:-1], bounds[1:]):
        eng.accumulate(dW[a:b, :W.shape[1]], dT[a:b])
    out = eng.finalize(want_rho=want_rho) if W.shape[0] >= 2 else None
    sums = dict(sum_hw=eng.sum_hw.cpu().numpy(), sum_w=eng.sum_w.cpu().numpy(),
                sum_w2=eng.sum_w2.cpu().numpy(), sum_h=eng.sum_h.cpu().numpy(),
                sum_h2=eng.sum_h2.cpu().numpy(), n=int(eng.n.cpu().numpy()[0]))
    eng.close()
    return sums, out


def assert_parity(sums, out, ref, rho_exact=True):
    for k in ("sum_hw", "sum_w", "sum_w2", "sum_h", "sum_h2"):
        assert np.array_equal(sums[k], ref[k]), k
    assert sums["n"] == ref["n"]
    if out is None:
        return
    rho = out["rho"].cpu().numpy()
    if rho_exact:
        assert np.array_equal(rho, ref["rho"])          # bit-exact vs reference B
    assert np.array_equal(out["maxabs"].cpu().numpy(), ref["maxabs"])
    assert np.array_equal(out["argmax"].cpu().numpy(), ref["argmax"])
    assert np.array_equal(out["rank"].cpu().numpy(), ref["rank"])
    assert out["round_key"] == ref["best"].tobytes()


def test_c1_full_parity(P):
    w = S.CONFIGS["C1"]
    texts, W = S.dataset(w)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    sums, out = run_gpu(P, texts, W)
    assert_parity(sums, out, ref)
    assert out["master_key"] == w.key
    rk = O.expand_key(w.key)[10].astype(int)
    assert out["peak_sample"] == w.leak_positions()
    # reference A (two-pass) on the true-key rows and a spread of others
    hyps = np.array([256 * b + rk[b] for b in range(16)] + list(range(0, 4096, 97)), np.int32)
    ra = O.rho_two_pass_i8(O.HD_LAST, texts, W, hyps=hyps)
    rg = out["rho"].cpu().numpy()[hyps]
    assert np.all(np.abs(rg - ra) <= 1e-9 * np.abs(ra) + 1e-12)


def test_c1_noiseless_rho_one(P):
    w = S.CONFIGS["C1-0"]
    texts, W = S.dataset(w)
    _, out = run_gpu(P, texts, W)
    rk = O.expand_key(w.key)[10].astype(int)
    mx = out["maxabs"].cpu().numpy()
    am = out["argmax"].cpu().numpy()
    for b in range(16):
        assert abs(mx[256 * b + rk[b]] - 1.0) <= 1e-12 and am[256 * b + rk[b]] == w.leak_positions()[b]
    assert out["master_key"] == w.key


@pytest.mark.parametrize("xt,spill", [(1, 1), (1, 2), (1, 3), (2, 1), (2, 2), (2, 3)])
@pytest.mark.parametrize("model", [O.HD_LAST, O.HW_LAST, O.HW_FIRST])
@pytest.mark.parametrize("dtype", [np.int8, np.uint8])
def test_models_dtypes_ragged(P, model, dtype, xt, spill):
    rng = np.random.default_rng(100 + model)
    n, m = 333, 300                     # ragged: 333 = 5*64+13 traces, 300 = 256+44 samples
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    lo, hi = (-128, 128) if dtype == np.int8 else (0, 256)
    W = rng.integers(lo, hi, (n, m)).astype(dtype)
    ref = O.attack_i8(model, texts, W)
    sums, out = run_gpu(P, texts, W, model=MODEL[model], xt=xt, spill=spill)
    assert_parity(sums, out, ref)


@pytest.mark.parametrize("xt,spill", [(1, 1), (1, 2), (1, 3), (2, 1), (2, 2), (2, 3)])
@pytest.mark.parametrize("n,m", [(2, 1), (3, 17), (64, 256), (65, 257), (65, 258), (130, 513), (130, 514), (1000, 16)])
def test_edge_shapes(P, n, m, xt, spill):
    rng = np.random.default_rng(n * 1000 + m)
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    W = rng.integers(-128, 128, (n, m)).astype(np.int8)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    sums, out = run_gpu(P, texts, W, xt=xt, spill=spill)   # spill 2 needs M even (odd M falls back to red.add)
    assert_parity(sums, out, ref)


def test_degenerate_columns(P):
    """Constant columns (dw = 0) give rho = 0 exactly [S:250, S:293]."""
    rng = np.random.default_rng(5)
    texts = rng.integers(0, 256, (200, 16), dtype=np.uint8)
    W = rng.integers(-128, 128, (200, 40)).astype(np.int8)
    W[:, 3] = 7
    W[:, 39] = -128
    ref = O.attack_i8(O.HD_LAST, texts, W)
    sums, out = run_gpu(P, texts, W)
    assert_parity(sums, out, ref)
    rho = out["rho"].cpu().numpy()
    assert not rho[:, 3].any() and not rho[:, 39].any()


def test_split_k_chunks_and_permutation_bit_identical(P):
    """Integer sums are order-independent: split-K units, several accumulate
    calls and a trace permutation all give bit-identical results."""
    rng = np.random.default_rng(9)
    n, m = 9000, 700
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    W = rng.integers(-128, 128, (n, m)).astype(np.int8)
    base, out0 = run_gpu(P, texts, W)
    for kw in (dict(kchunk=128), dict(kchunk=1024), dict(chunks=[0, 1, 700, 4097, 9000]),
               dict(overlap=False), dict(overlap=False, chunks=[0, 5000, 9000]),
               dict(xt=1), dict(xt=2), dict(xt=1, kchunk=256), dict(xt=2, kchunk=256),
               dict(xt=2, chunks=[0, 1, 700, 4097, 9000]), dict(spill=1), dict(spill=2, kchunk=128),
               dict(spill=2, xt=2, kchunk=256), dict(spill=3), dict(spill=3, kchunk=128),
               dict(spill=3, xt=2, kchunk=256), dict(spill=3, chunks=[0, 1, 700, 4097, 9000])):
        s, o = run_gpu(P, texts, W, **kw)
        for k in base:
            assert np.array_equal(base[k], s[k]), (kw, k)
        assert np.array_equal(out0["rho"].cpu().numpy(), o["rho"].cpu().numpy())
    perm = rng.permutation(n)
    s, o = run_gpu(P, texts[perm], W[perm])
    assert np.array_equal(out0["rho"].cpu().numpy(), o["rho"].cpu().numpy())
    # oracle on a column subset
    cols = np.array([0, 1, 255, 256, 511, 699], np.int32)
    ref_hw = O.cross_sums_i8(O.HD_LAST, texts, W, cols)
    assert np.array_equal(base["sum_hw"][:, cols], ref_hw)


def test_c2_subset_and_closed_form(P):
    w = S.CONFIGS["C2"]
    texts, W = S.dataset(w)
    cols = np.array(sorted(set(w.leak_positions()) | {0, 1, 255, 256, 4095, 4999}), np.int32)
    sums, out = run_gpu(P, texts, W)
    assert np.array_equal(sums["sum_hw"][:, cols], O.cross_sums_i8(O.HD_LAST, texts, W, cols))
    sw, sw2 = O.trace_sums_i8(W)
    assert np.array_equal(sums["sum_w"], sw) and np.array_equal(sums["sum_w2"], sw2)
    sh, sh2 = O.model_sums(O.HD_LAST, texts)
    assert np.array_equal(sums["sum_h"], sh) and np.array_equal(sums["sum_h2"], sh2)
    # closed form over ALL columns: sum_k sumHW[b,k,j] = 1024 sumW[j]
    assert (sums["sum_hw"].reshape(16, 256, -1).sum(1) == 1024 * sums["sum_w"][None, :]).all()
    rho_ref = O.rho_eq1_grid(w.n, sums["sum_hw"][:, cols], sh, sh2, sw[cols], sw2[cols])
    assert np.array_equal(out["rho"].cpu().numpy()[:, cols], rho_ref)
    assert out["master_key"] == w.key


def test_unaligned_device_input_is_staged(P):
    """ld*1 not a multiple of 16 (TMA rule): the library stages the rows."""
    w = S.CONFIGS["C1"]
    texts, W = S.dataset(w)                  # ld = 500
    ref = O.attack_i8(O.HD_LAST, texts, W)
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.accumulate(torch.from_numpy(W).cuda(), torch.from_numpy(texts).cuda())
    out = eng.finalize(want_rho=True)
    assert np.array_equal(eng.sum_hw.cpu().numpy(), ref["sum_hw"])
    assert np.array_equal(out["rho"].cpu().numpy(), ref["rho"])
    eng.close()


def test_host_buffer_path_matches_device(P):
    w = S.CONFIGS["C2"].replace(n=3000)
    texts, W = S.dataset(w)
    s_dev, o_dev = run_gpu(P, texts, W)
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.accumulate_host(W, texts)
    o = eng.finalize(want_rho=True)
    assert np.array_equal(eng.sum_hw.cpu().numpy(), s_dev["sum_hw"])
    assert np.array_equal(o["rho"].cpu().numpy(), o_dev["rho"].cpu().numpy())
    eng.close()


@pytest.mark.parametrize("m,ld,stage", [(300, 300, 0), (300, 300, 300 * 97), (301, 301, 320 * 50),
                                        (320, 320, 320 * 64), (300, 333, 320 * 41), (5000, 5000, 5008 * 700)])
def test_staging_chunks_linear_repack_and_pitched(P, m, ld, stage):
    """a1 staging: linear copy + repack (row not a 16-byte multiple), linear
    copy in place (row a 16-byte multiple) and the pitched 2D copy (ld > M),
    over many double-buffered chunks, all bit-exact with the oracle."""
    rng = np.random.default_rng(m + ld)
    n = 2311
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    base = rng.integers(-128, 128, (n, ld)).astype(np.int8)
    W = base[:, :m]
    cols = np.array([0, 1, m // 2, m - 1], np.int32)
    ref_hw = O.cross_sums_i8(O.HD_LAST, texts, np.ascontiguousarray(W), cols)
    for src in ("host", "device"):
        eng = P.Engine(m, P.CPA_S8, P.CPA_HD_LAST, 0)
        eng.set_stage_bytes(stage)
        if src == "host":
            eng.accumulate_host(W, texts)
        else:  # an odd byte offset forces the staged path for device input too
            raw = torch.from_numpy(np.concatenate([np.zeros(1, np.int8), base.reshape(-1)])).cuda()
            dW = raw[1:].view(n, ld)[:, :m]
            eng.accumulate(dW, torch.from_numpy(texts).cuda())
        eng.sync()
        assert np.array_equal(eng.sum_hw.cpu().numpy()[:, cols], ref_hw), src
        assert np.array_equal(eng.sum_w.cpu().numpy(), W.astype(np.int64).sum(0)), src
        assert np.array_equal(eng.sum_w2.cpu().numpy(), (W.astype(np.int64) ** 2).sum(0)), src
        assert int(eng.n.cpu().numpy()[0]) == n
        eng.close()


def test_errors(P):
    eng = P.Engine(100, P.CPA_S8, P.CPA_HD_LAST, 0)
    W = torch.zeros((10, 100), dtype=torch.int8, device="cuda")
    T = torch.zeros((10, 16), dtype=torch.uint8, device="cuda")
    with pytest.raises(P.CpaError, match="INVALID_ARG"):
        P.cpa_accumulate(eng.ctx, W, 99, T, 10)           # ld < M
    with pytest.raises(P.CpaError, match="TOO_FEW"):
        eng.finalize()                                     # N = 0 < 2
    eng.accumulate(W[:1], T[:1])
    rk = torch.empty(4096, dtype=torch.int32, device="cuda")
    with pytest.raises(P.CpaError, match="TOO_FEW"):
        eng.finalize_async(rk)                             # N = 1, checked without blocking
    eng.close()
    # the exact-int64 bound of Eq. (1) on the running total (not only per call)
    eng = P.Engine(16, P.CPA_S8, P.CPA_HD_LAST, 0)
    n = 1 << 23
    W = torch.zeros((n, 16), dtype=torch.int8, device="cuda")
    T = torch.zeros((n, 16), dtype=torch.uint8, device="cuda")
    eng.accumulate(W[: n // 2], T[: n // 2])
    eng.accumulate(W[n // 2:], T[n // 2:])                # exactly 2^23: allowed
    with pytest.raises(P.CpaError, match="OVERFLOW"):
        eng.accumulate(W[:1], T[:1])
    eng.reset()
    eng.accumulate(W[:1], T[:1])                          # the reset restarts the count
    eng.close()
    # host buffers: the element type must match the context's
    eng = P.Engine(100, P.CPA_S8, P.CPA_HD_LAST, 0)
    with pytest.raises(TypeError):
        eng.accumulate_host(np.zeros((10, 100), np.float64), np.zeros((10, 16), np.uint8))
    with pytest.raises(ValueError):
        eng.accumulate_host(np.zeros((10, 100), np.int8), np.zeros((10, 15), np.uint8))
    eng.close()


def test_synth_device_generator_matches_host(P):
    for name in ("C1", "C3"):
        w = S.CONFIGS[name].replace(n=300)
        texts, lv = S.texts(w)
        Wh = S.traces(w, lv)
        d = torch.empty(Wh.shape, dtype={S.S8: torch.int8, S.F32: torch.float32}[w.dtype], device="cuda")
        S.dev_traces(w, torch.from_numpy(lv).cuda(), 0, w.n, d, w.m)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), Wh)


@pytest.mark.parametrize("model", [O.HD_LAST, O.HW_LAST, O.HW_FIRST])
def test_model_sums_histogram_path(P, model):
    """N >= 65536 in one call takes the byte-pair histogram path for a3, with the
    pairs counted by a separate pass (default) or inside the cross-term kernel
    (CPA_OPT_FUSE_HIST; M = 600 spans two N-tile groups, only group 0 counts);
    both must equal the oracle and the direct path (chunks < 65536) bit for bit."""
    rng = np.random.default_rng(31 + model)
    n, m = 70001, 600
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    W = rng.integers(-128, 128, (n, m)).astype(np.int8)
    one, _ = run_gpu(P, texts, W, model=MODEL[model], want_rho=False)
    sep, _ = run_gpu(P, texts, W, model=MODEL[model], want_rho=False, fuse_hist=True)
    chunked, _ = run_gpu(P, texts, W, model=MODEL[model], chunks=[0, 30000, 60000, n], want_rho=False)
    sh, sh2 = O.model_sums(model, texts)
    for s in (one, sep, chunked):
        assert np.array_equal(s["sum_h"], sh) and np.array_equal(s["sum_h2"], sh2)
        assert s["n"] == n
    assert np.array_equal(one["sum_hw"], chunked["sum_hw"])


@pytest.mark.parametrize("dt", [np.int8, np.uint8])
def test_moment_modes_exact(P, dt):
    """a4 trace moments in every CPA_OPT_OVERLAP mode (0 serial, 1 low-priority
    side stream, 2 co-resident, 3 fused into the cross-term kernel) equal the
    oracle's exact sums [P:79], including the extreme values (-128/127, 0/255)
    whose squares bound the per-thread 32-bit partials, a ragged last sample
    tile (M = 300: the second CTA of the second tile is entirely past M) and
    ragged trace counts / split-K units."""
    rng = np.random.default_rng(21)
    n, m = 5 * 128 + 77, 300
    lo, hi = (-128, 128) if dt is np.int8 else (0, 256)
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    W = rng.integers(lo, hi, (n, m)).astype(dt)
    W[:, 7] = lo                     # constant extreme columns
    W[:, 299] = hi - 1
    W[:300, 11] = lo
    sw, sw2 = O.trace_sums_i8(W)
    ref_hw = O.cross_sums_i8(O.HD_LAST, texts, W, np.array([0, 7, 11, 255, 256, 299], np.int32))
    for mode in (0, 1, 2, 3):
        for kw in (dict(), dict(kchunk=128), dict(chunks=[0, 3, 400, n]), dict(xt=2), dict(xt=2, kchunk=128)):
            # xt = 1 forces the NT = 2 kernel, the one that fuses a4 (mode 3)
            s, _ = run_gpu(P, texts, W, mode=mode, want_rho=False, **dict(dict(xt=1), **kw))
            assert np.array_equal(s["sum_w"], sw), (mode, kw)
            assert np.array_equal(s["sum_w2"], sw2), (mode, kw)
            assert np.array_equal(s["sum_hw"][:, [0, 7, 11, 255, 256, 299]], ref_hw), (mode, kw)


@pytest.mark.parametrize("dt,v", [(np.int8, -128), (np.uint8, 255)])
def test_fused_moments_32bit_bound(P, dt, v):
    """Worst case of the fused a4 partials (xterm.cu moments_pass): constant
    extreme traces over one 2^20-trace split-K unit, the largest allowed, so a
    thread's 32-bit sum W^2 reaches 2^15 * 65025 (u8) / 2^29 (s8).  Closed form:
    sum W = N v, sum W^2 = N v^2, and sum_k sum HW = 1024 sum W per byte."""
    n, m = (1 << 20) + 5, 16
    texts = np.random.default_rng(3).integers(0, 256, (n, 16), dtype=np.uint8)
    W = np.full((n, m), v, dt)
    s, _ = run_gpu(P, texts, W, kchunk=1 << 20, mode=3, want_rho=False, xt=1)
    assert np.all(s["sum_w"] == n * v) and np.all(s["sum_w2"] == n * v * v)
    hw = s["sum_hw"].reshape(16, 256, m).sum(axis=1)
    assert np.all(hw == 1024 * n * v)


def run_cs(P, texts, W, model, chunks=None, class_sums=True):
    dtype = {np.int8: P.CPA_S8, np.uint8: P.CPA_U8}[W.dtype.type]
    eng = P.Engine(W.shape[1], dtype, model, 0)
    eng.set_class_sums(class_sums)
    ld = (W.shape[1] + 15) // 16 * 16
    Wp = np.zeros((W.shape[0], ld), W.dtype)
    Wp[:, :W.shape[1]] = W
    dW = torch.from_numpy(Wp).cuda()
    dT = torch.from_numpy(np.ascontiguousarray(texts)).cuda()
    bounds = chunks or [0, W.shape[0]]
    for a, b in zip(bounds[:-1], bounds[1:]):
        eng.accumulate(dW[a:b, :W.shape[1]], dT[a:b])
    out = eng.finalize(want_rho=True)
    sums = dict(sum_hw=eng.sum_hw.cpu().numpy(), sum_w=eng.sum_w.cpu().numpy(),
                sum_w2=eng.sum_w2.cpu().numpy(), sum_h=eng.sum_h.cpu().numpy(),
                sum_h2=eng.sum_h2.cpu().numpy(), n=int(eng.n.cpu().numpy()[0]))
    eng.close()
    return sums, out


@pytest.mark.parametrize("model", [O.HW_LAST, O.HW_FIRST])
@pytest.mark.parametrize("dt", [np.int8, np.uint8])
def test_class_sums_exact(P, model, dt):
    """Class-sum cross term (CPA_OPT_CLASS_SUMS): for the
    single-byte models sum_i H W = sum_x f(x ^ k) S_b[x][j] exactly, so every
    sum, rho, maximum and rank equals the oracle's (and the tensor-core path's)
    bit for bit.  Ragged N and M (half-empty last column tile), several calls."""
    rng = np.random.default_rng(31 + model)
    n, m = 3 * 128 + 61, 300
    lo, hi = (-128, 128) if dt is np.int8 else (0, 256)
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    texts[:40, 3] = 7                                  # a heavy class
    W = rng.integers(lo, hi, (n, m)).astype(dt)
    W[:, 5] = lo
    ref = O.attack_i8(model, texts, W)
    for chunks in (None, [0, 1, 200, n]):
        sums, out = run_cs(P, texts, W, MODEL[model], chunks)
        assert_parity(sums, out, ref)
    s0, o0 = run_cs(P, texts, W, MODEL[model], class_sums=False)
    assert np.array_equal(s0["sum_hw"], sums["sum_hw"])


def test_class_sums_column_blocks_and_key(P):
    """M > 8192 (two column blocks of the class-sum scratch) on HW_LAST leakage:
    closed form over every column, oracle on sampled columns, key recovered."""
    w = S.CONFIGS["C2-HW"].replace(n=600, m=8200, a=6.0)
    texts, W = S.dataset(w)
    sums, out = run_cs(P, texts, W, 1)
    cols = np.array(sorted(set(w.leak_positions()) | {0, 8191, 8192, 8199}), np.int32)
    assert np.array_equal(sums["sum_hw"][:, cols], O.cross_sums_i8(O.HW_LAST, texts, W, cols))
    sw, _ = O.trace_sums_i8(W)
    assert np.array_equal(sums["sum_hw"].reshape(16, 256, -1).sum(axis=1), 1024 * np.broadcast_to(sw, (16, w.m)))
    assert out["master_key"] == w.key


def test_class_sums_chunked_sort_and_errors(P):
    """> 2^20 traces in one call (two super-chunks, ragged sort chunks), closed form; class sums on
    an HD_LAST context are refused with CPA_E_INVALID_ARG."""
    n, m = (1 << 20) + 300, 16
    rng = np.random.default_rng(5)
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    W = rng.integers(-128, 128, (n, m)).astype(np.int8)
    sums, _ = run_cs(P, texts, W, 1)
    sw, sw2 = O.trace_sums_i8(W)
    assert np.array_equal(sums["sum_w"], sw)
    assert np.array_equal(sums["sum_hw"].reshape(16, 256, m).sum(axis=1), 1024 * np.broadcast_to(sw, (16, m)))
    ref = O.cross_sums_i8(O.HW_LAST, texts, W, np.array([15], np.int32))
    assert np.array_equal(sums["sum_hw"][:, [15]], ref)
    eng = P.Engine(16, P.CPA_S8, 0, 0)
    with pytest.raises(Exception):
        eng.set_class_sums(True)
    eng.close()


@pytest.mark.parametrize("spill", [1, 2, 3])
def test_first_touch_store_then_add(P, spill):
    """After cpa_init / cpa_reset the first int8 accumulate with one trace chunk
    per work unit stores its sums (include/cpa.h); later calls add.  The same
    traces accumulated twice give exactly twice the sums, and a reset restarts."""
    rng = np.random.default_rng(77)
    n, m = 700, 600
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    W = rng.integers(-128, 128, (n, m)).astype(np.int8)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    eng = P.Engine(m, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.set_spill(spill)
    dW, dT = torch.from_numpy(W).cuda(), torch.from_numpy(texts).cuda()
    for rounds in (1, 2, 3):
        eng.reset()
        for _ in range(rounds):
            eng.accumulate(dW, dT)
        eng.sync()
        assert np.array_equal(eng.sum_hw.cpu().numpy(), rounds * ref["sum_hw"]), rounds
        assert np.array_equal(eng.sum_w.cpu().numpy(), rounds * ref["sum_w"]), rounds
    eng.close()


@pytest.mark.parametrize("dtype", ["s8", "f32"])
@pytest.mark.parametrize("m,dup", [(8192, False), (9002, True), (20000, False), (8193, False)])
def test_maxima_only_finalize_equals_rho_maxima(P, dtype, m, dup):
    """Without rho (checkpoints, M >= 8192) the finalize runs the filtered maxima
    kernel (most cells skip the division against a row-wide threshold): its max
    |rho|, argmax, signed peak and ranks equal those of the rho-writing kernel
    (bit-exact against the oracle elsewhere) bit for bit, ties to the lowest
    sample [S:298] (dup, int8: the second half of the columns repeats the first,
    so every maximum ties exactly), also for a partial row range."""
    rng = np.random.default_rng(m + (7 if dup else 0))
    n = 300
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    half = m // 2 if dup else m
    W = rng.integers(-128, 128, (n, half)).astype(np.int8)
    if dtype == "f32":
        W = W.astype(np.float32) + 0.01 * rng.standard_normal(W.shape).astype(np.float32)
    if dup:
        W = np.concatenate([W, W], axis=1)
    eng = P.Engine(m, P.CPA_S8 if dtype == "s8" else P.CPA_F32, P.CPA_HD_LAST, 0)
    eng.accumulate(torch.from_numpy(np.ascontiguousarray(W)).cuda(), torch.from_numpy(texts).cuda())
    full = eng.finalize(want_rho=True)
    fast = eng.finalize(want_rho=False)
    rho = full["rho"].cpu().numpy()
    a = np.abs(rho)
    assert np.array_equal(full["maxabs"].cpu().numpy(), a.max(axis=1))
    assert np.array_equal(full["argmax"].cpu().numpy(), a.argmax(axis=1))   # first maximum
    for k in ("maxabs", "argmax", "rank"):
        assert np.array_equal(fast[k].cpu().numpy(), full[k].cpu().numpy()), k
    assert fast["peak_rho"] == full["peak_rho"] and fast["peak_sample"] == full["peak_sample"]
    if dup and dtype == "s8":                       # exact sums: the copies tie exactly
        assert np.all(full["argmax"].cpu().numpy() < half)
    mx, am, pk = (t[0] for t in eng.maxima_buffers(1))
    h0, h1 = 5, 1003                                   # a partial last row group
    eng.finalize_rows(h0, h1, mx, am, pk)
    assert np.array_equal(mx[h0:h1].cpu().numpy(), a.max(axis=1)[h0:h1])
    assert np.array_equal(am[h0:h1].cpu().numpy(), a.argmax(axis=1)[h0:h1])
    assert np.array_equal(pk[h0:h1].cpu().numpy(), rho[np.arange(h0, h1), a.argmax(axis=1)[h0:h1]])
    assert not mx[:h0].any() and not mx[h1:].any()
    eng.close()


@pytest.mark.parametrize("n,m", [(40000, 2600), (34000, 5000)])
def test_tail_split_bit_identical(P, n, m):
    """One trace chunk per tile, long units, more tiles than CTA pairs and not a
    whole number of waves: the last wave's tiles are cut into pieces
    (xterm.cu tail_split).  Every sum equals a two-chunk run (no tail split) bit
    for bit, and sampled columns of the split tiles (the last tile groups) equal
    the oracle."""
    rng = np.random.default_rng(n + m)
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    W = rng.integers(-128, 128, (n, m)).astype(np.int8)
    # one trace chunk per tile (kchunk >= n); a first 1-trace call, so the second
    # adds (long units and no first touch: the tail split applies)
    split, out0 = run_gpu(P, texts, W, chunks=[0, 1, n], kchunk=(n + 127) // 128 * 128)
    kc = ((n + 1) // 2 + 127) // 128 * 128
    two, out1 = run_gpu(P, texts, W, kchunk=kc)
    for k in split:
        assert np.array_equal(split[k], two[k]), k
    assert np.array_equal(out0["rho"].cpu().numpy(), out1["rho"].cpu().numpy())
    cols = np.array(sorted({0, 511, m - 512, m - 300, m - 1}), np.int32)
    assert np.array_equal(split["sum_hw"][:, cols], O.cross_sums_i8(O.HD_LAST, texts, W, cols))
    sw, sw2 = O.trace_sums_i8(W)
    assert np.array_equal(split["sum_w"], sw) and np.array_equal(split["sum_w2"], sw2)
