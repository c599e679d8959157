"""CPA_OPT_NARROW (include/cpa.h): the int8 cross term kept in an int32 shadow
of sum_hw while N max|H| max|W| < 2^31.  Every result -- the int64 sums after
cpa_flush, rho (bit-exact to reference B), maxima, ranks, key -- equals the
oracle's exactly as without the option: the int32 sums are the same integers
(Eq. (1) [P:69] is evaluated from them unchanged).  Also: the flush
when a call would pass the bound (capped low here with NARROW > 1), the zeroed
shadow of a multi-chunk first call, reset, host staging, the maxima-only
finalize reading the shadow, and graph replay."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from synth import synth as S  # noqa: E402

from tests.test_parity_gpu import MODEL, assert_parity, run_gpu  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1412_7682_b200 as P
    return P


def _data(seed, n, m, dtype=np.int8):
    rng = np.random.default_rng(seed)
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    lo, hi = (-128, 128) if dtype == np.int8 else (0, 256)
    return texts, rng.integers(lo, hi, (n, m)).astype(dtype)


@pytest.mark.parametrize("xt", [1, 2])
@pytest.mark.parametrize("model", [O.HD_LAST, O.HW_LAST, O.HW_FIRST])
@pytest.mark.parametrize("dtype", [np.int8, np.uint8])
def test_narrow_models_dtypes_ragged(P, model, dtype, xt):
    texts, W = _data(300 + model, 333, 300, dtype)      # ragged traces and samples
    ref = O.attack_i8(model, texts, W)
    sums, out = run_gpu(P, texts, W, model=MODEL[model], xt=xt, narrow=1)
    assert_parity(sums, out, ref)


@pytest.mark.parametrize("n,m", [(2, 1), (3, 17), (65, 257), (130, 514), (1000, 16)])
def test_narrow_edge_shapes(P, n, m):
    texts, W = _data(n * 7 + m, n, m)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    sums, out = run_gpu(P, texts, W, narrow=1)
    assert_parity(sums, out, ref)


@pytest.mark.parametrize("cap,chunks", [
    (0, [0, 400, 401, 900]),       # no cap: every call stays in the shadow
    (500, [0, 400, 401, 900]),     # the third call passes the cap: flush, then int64
    (450, [0, 300, 900]),          # the second call passes it
    (100, [0, 300, 900]),          # the first call already exceeds it: int64 throughout
])
def test_narrow_flush_at_bound(P, cap, chunks):
    texts, W = _data(cap + len(chunks), 900, 520)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    sums, out = run_gpu(P, texts, W, chunks=chunks, narrow=cap or 1)
    assert_parity(sums, out, ref)


@pytest.mark.parametrize("kchunk", [128, 256])
def test_narrow_multichunk_first_call(P, kchunk):
    """A first call split into several trace chunks per tile cannot first-touch
    store: the shadow is zeroed and added to."""
    texts, W = _data(kchunk, 700, 600)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    sums, out = run_gpu(P, texts, W, kchunk=kchunk, narrow=1)
    assert_parity(sums, out, ref)


@pytest.mark.parametrize("spill", [2, 3])
def test_narrow_yields_to_explicit_spill(P, spill):
    texts, W = _data(spill, 500, 512)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    sums, out = run_gpu(P, texts, W, spill=spill, narrow=1, chunks=[0, 200, 500])
    assert_parity(sums, out, ref)


def test_narrow_reset_rounds_and_toggle(P):
    texts, W = _data(5, 640, 700)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    eng = P.Engine(700, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.set_narrow(True)
    dW, dT = torch.from_numpy(W).cuda(), torch.from_numpy(texts).cuda()
    for rounds in (2, 1, 3):
        eng.reset()
        for _ in range(rounds):
            eng.accumulate(dW, dT)
        assert np.array_equal(eng.sum_hw.cpu().numpy(), rounds * ref["sum_hw"]), rounds
    # flushed (sum_hw above), then more traces into a fresh shadow, then the option
    # turned off (flushes): the accumulator holds all four passes
    eng.accumulate(dW, dT)
    eng.set_narrow(False)
    eng.sync()
    assert np.array_equal(eng.sum_hw.cpu().numpy(), 4 * ref["sum_hw"])
    eng.close()


def test_narrow_host_staging(P):
    """cpa_accumulate_host in several staging chunks: each chunk adds into the shadow."""
    texts, W = _data(9, 3000, 1000)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    eng = P.Engine(1000, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.set_narrow(True)
    eng.set_stage_bytes(700 * 1024)                        # 700 traces of 1 KB per chunk
    eng.accumulate_host(W, texts)
    out = eng.finalize(want_rho=True)
    assert np.array_equal(out["rho"].cpu().numpy(), ref["rho"])
    assert np.array_equal(out["rank"].cpu().numpy(), ref["rank"])
    assert np.array_equal(eng.sum_hw.cpu().numpy(), ref["sum_hw"])
    eng.close()


@pytest.mark.parametrize("m,dup", [(8192, False), (9002, True), (8193, False)])
def test_narrow_maxima_only_finalize(P, m, dup):
    """The filtered maxima kernel reading int32 rows gives the maxima of the
    rho-writing kernel reading int64 rows, bit for bit (ties to the lowest j)."""
    rng = np.random.default_rng(m)
    n = 300
    texts = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    half = m // 2 if dup else m
    W = rng.integers(-128, 128, (n, half)).astype(np.int8)
    if dup:
        W = np.concatenate([W, W], axis=1)
    dW, dT = torch.from_numpy(np.ascontiguousarray(W)).cuda(), torch.from_numpy(texts).cuda()
    wide = P.Engine(m, P.CPA_S8, P.CPA_HD_LAST, 0)
    wide.accumulate(dW, dT)
    full = wide.finalize(want_rho=True)
    eng = P.Engine(m, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.set_narrow(True)
    eng.accumulate(dW, dT)
    fast = eng.finalize(want_rho=False)
    for k in ("maxabs", "argmax", "rank"):
        assert np.array_equal(fast[k].cpu().numpy(), full[k].cpu().numpy()), k
    assert fast["peak_rho"] == full["peak_rho"] and fast["peak_sample"] == full["peak_sample"]
    mx, am, pk = (t[0] for t in eng.maxima_buffers(1))
    eng.finalize_rows(5, 1003, mx, am, pk)
    a = np.abs(full["rho"].cpu().numpy())
    assert np.array_equal(mx[5:1003].cpu().numpy(), a.max(axis=1)[5:1003])
    assert np.array_equal(am[5:1003].cpu().numpy(), a.argmax(axis=1)[5:1003])
    assert torch.equal(eng.sum_hw, wide.sum_hw)
    eng.close()
    wide.close()


def test_narrow_graph_replay(P):
    w = S.CONFIGS["C2"].replace(n=3000, m=1200)
    texts, W = S.dataset(w)
    st = torch.cuda.Stream()
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0, stream=st)
    eng.set_narrow(True)
    dW = torch.from_numpy(np.ascontiguousarray(W)).cuda()
    dT = torch.from_numpy(texts).cuda()
    rank = torch.empty(4096, dtype=torch.int32, device="cuda")
    mx = torch.empty(4096, dtype=torch.float64, device="cuda")
    am = torch.empty(4096, dtype=torch.int32, device="cuda")
    best = torch.empty(32, dtype=torch.int32, device="cuda")
    eng.reset()
    eng.accumulate(dW, dT)
    ref = eng.finalize()
    ref_hw = eng.sum_hw.clone()
    eng.graph_begin()
    eng.reset()
    eng.accumulate(dW, dT)
    eng.finalize_async(rank, mx, am, best)
    eng.graph_end()
    for _ in range(3):
        eng.graph_launch()
        eng.sync()
        assert torch.equal(rank, ref["rank"]) and torch.equal(mx, ref["maxabs"]) and torch.equal(am, ref["argmax"])
        assert torch.equal(eng.sum_hw, ref_hw)              # flushes the replay's shadow
    assert ref["master_key"] == w.key
    cols = np.arange(0, w.m, 97, dtype=np.int32)
    assert np.array_equal(ref_hw.cpu().numpy()[:, cols], O.cross_sums_i8(O.HD_LAST, texts, W, cols))
    eng.close()


def test_narrow_contexts_over_trace_shards_flush_and_sum(P):
    """Two contexts on trace halves, each with a live shadow: after cpa_flush the
    int64 accumulators add up to the whole run's (the multi-GPU combine's
    precondition), and the summed accumulator finalizes to the oracle's rho."""
    texts, W = _data(11, 900, 640)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    engs = [P.Engine(640, P.CPA_S8, P.CPA_HD_LAST, 0) for _ in range(2)]
    for e, (a, b) in zip(engs, [(0, 450), (450, 900)]):
        e.set_narrow(True)
        e.accumulate(torch.from_numpy(W[a:b]).cuda(), torch.from_numpy(texts[a:b]).cuda())
        e.flush()
        e.sync()
    engs[0].accum += engs[1].accum
    torch.cuda.synchronize()
    engs[0].set_narrow(False)      # no live shadow left: finalize reads the summed accumulator
    out = engs[0].finalize(want_rho=True)
    assert np.array_equal(engs[0].sum_hw.cpu().numpy(), ref["sum_hw"])
    assert np.array_equal(out["rho"].cpu().numpy(), ref["rho"])
    assert np.array_equal(out["rank"].cpu().numpy(), ref["rank"])
    for e in engs:
        e.close()
