"""CUDA-graph replay of a fixed-shape step (include/cpa.h cpa_graph_*): the
captured reset + accumulate + finalize_async replays to the same sums, maxima,
ranks and key as the direct calls, bit for bit (int path) / identically (float
path: the same kernels on the same data), reads its input buffers at replay
time, and the calls that cannot be captured are refused."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from synth import synth as S  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available()
    import paper_1412_7682_b200 as P
    return P


def _step_buffers(dev="cuda"):
    return (torch.empty(4096, dtype=torch.int32, device=dev), torch.empty(4096, dtype=torch.float64, device=dev),
            torch.empty(4096, dtype=torch.int32, device=dev), torch.empty(32, dtype=torch.int32, device=dev))


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_graph_replay_equals_direct_calls(P, cfg):
    w = S.CONFIGS[cfg].replace(n=3000, m=1000, a=0.02) if cfg == "C3" else S.CONFIGS[cfg].replace(n=3000, m=1200)
    texts, W = S.dataset(w)
    f32 = w.dtype == S.F32
    st = torch.cuda.Stream()
    eng = P.Engine(w.m, P.CPA_F32 if f32 else P.CPA_S8, P.CPA_HD_LAST, 0, stream=st)
    dW = torch.from_numpy(np.ascontiguousarray(W)).cuda()
    dT = torch.from_numpy(texts).cuda()
    rank, mx, am, best = _step_buffers()

    def direct():
        eng.reset()
        eng.accumulate(dW, dT)
        out = eng.finalize()
        return (eng.sum_hw.clone(), out["rank"].clone(), out["maxabs"].clone(), out["argmax"].clone(),
                out["round_key"], out["master_key"])

    ref = direct()                                   # also allocates what the capture needs
    eng.graph_begin()
    eng.reset()
    eng.accumulate(dW, dT)
    eng.finalize_async(rank, mx, am, best)
    eng.graph_end()
    rk10 = O.expand_key(w.key)[10].astype(int)
    true_h = torch.tensor([256 * b + rk10[b] for b in range(16)], device="cuda")

    def same(got_hw, got_rank, got_mx, got_am, r):
        if f32:   # fp64 atomics: the order of the adds (and so the last bits) may differ
            assert torch.allclose(got_hw, r[0], rtol=1e-12, atol=0)
            assert torch.allclose(got_mx, r[2], rtol=1e-12, atol=0)
            assert torch.equal(got_rank[true_h], r[1][true_h]) and torch.equal(got_am[true_h], r[3][true_h])
        else:     # exact integer sums: bit for bit
            assert torch.equal(got_hw, r[0]) and torch.equal(got_rank, r[1])
            assert torch.equal(got_mx, r[2]) and torch.equal(got_am, r[3])

    for _ in range(3):
        eng.graph_launch()
        eng.sync()
        same(eng.sum_hw, rank, mx, am, ref)
        assert bytes(best[:16].cpu().numpy().astype(np.uint8)) == ref[4]
    assert ref[5] == w.key
    # the graph reads its buffers at replay time: new traces in place -> new result
    W2 = np.ascontiguousarray(np.roll(W, 7, axis=1))   # other traces, same shape
    T2 = np.ascontiguousarray(np.roll(texts, 3, axis=0))
    dW.copy_(torch.from_numpy(W2))
    dT.copy_(torch.from_numpy(T2))
    torch.cuda.synchronize()
    eng.graph_launch()
    eng.sync()
    got = (eng.sum_hw.clone(), rank.clone(), mx.clone(), am.clone())
    ref2 = direct()
    same(*got, ref2)
    assert not torch.equal(got[0], ref[0])
    if not f32:
        cols = np.arange(0, w.m, 97, dtype=np.int32)
        assert np.array_equal(got[0].cpu().numpy()[:, cols], O.cross_sums_i8(O.HD_LAST, T2, W2, cols))
    eng.close()


def test_graph_capture_rules(P):
    w = S.CONFIGS["C1"].replace(m=512)    # 16-byte rows: the aligned (capturable) path
    texts, W = S.dataset(w)
    dW = torch.from_numpy(W).cuda()
    dT = torch.from_numpy(texts).cuda()
    eng0 = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0, stream=torch.cuda.default_stream())
    if torch.cuda.default_stream().cuda_stream == 0:   # legacy default stream: not capturable
        with pytest.raises(P.CpaError, match="INVALID_ARG"):
            eng0.graph_begin()
    eng0.close()
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0, stream=torch.cuda.Stream())
    with pytest.raises(P.CpaError, match="INVALID_ARG"):
        eng.graph_launch()                               # nothing captured
    eng.reset()
    eng.accumulate(dW, dT)
    eng.finalize()
    eng.graph_begin()
    with pytest.raises(P.CpaError, match="INVALID_ARG"):
        eng.accumulate(dW, dT)                           # no captured reset before it
    eng.reset()
    eng.accumulate(dW, dT)
    mx, am, rank = (torch.empty(4096, dtype=t, device="cuda") for t in (torch.float64, torch.int32, torch.int32))
    for call in (lambda: P.cpa_finalize(eng.ctx, None, mx, am, rank), lambda: P.cpa_sync(eng.ctx),
                 lambda: P.cpa_phase_times(eng.ctx), lambda: P.cpa_accumulate_host(eng.ctx, W, w.m, texts, w.n)):
        with pytest.raises(P.CpaError, match="INVALID_ARG"):
            call()
    with pytest.raises(P.CpaError, match="INVALID_ARG"):
        eng.graph_begin()                                # already capturing
    wide = torch.zeros((w.n, w.m + 16), dtype=torch.int8, device="cuda")
    with pytest.raises(P.CpaError, match="not capturable"):    # unaligned rows: staging buffers
        P.cpa_accumulate(eng.ctx, wide[:, 1:1 + w.m], w.m + 16, dT, w.n)
    eng.graph_end()
    eng.graph_launch()
    eng.sync()
    ref = O.attack_i8(O.HD_LAST, texts, W)
    assert np.array_equal(eng.sum_hw.cpu().numpy(), ref["sum_hw"])
    eng.close()
