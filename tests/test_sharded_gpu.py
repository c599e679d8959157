"""Sharded Phase 3/4 through the C ABI (include/cpa.h "sharded Phase 3/4",
SURVEY §8e) and the wide-trace workload (the paper's
48000-sample dataset2 shape [P:168]), against the CPU oracle.

The multi-rank collectives are covered on CPU (tests/test_multigpu_gloo.py);
here every "rank" is a slice of the work on the one GPU: cpa_finalize_rows over
row blocks must reproduce cpa_finalize bit for bit, and G column-shard contexts
(CPA_OPT_COL0) merged by cpa_select must equal one context over all columns."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_1412_7682_b200 import multigpu as MG  # noqa: E402
from synth import synth as S  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1412_7682_b200 as P
    return P


def _padded(W):
    ld = (W.shape[1] + 15) // 16 * 16
    Wp = np.zeros((W.shape[0], ld), W.dtype)
    Wp[:, :W.shape[1]] = W
    return torch.from_numpy(Wp).cuda()


@pytest.fixture(scope="module")
def c1():
    w = S.CONFIGS["C1"]
    texts, W = S.dataset(w)
    return w, texts, W, O.attack_i8(O.HD_LAST, texts, W)


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_finalize_rows_equals_finalize(P, c1, G):
    w, texts, W, ref = c1
    dW = _padded(W)
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.accumulate(dW[:, :w.m], torch.from_numpy(texts).cuda())
    mx, am, pk = (t[0] for t in eng.maxima_buffers(1))
    for r in range(G):
        h0, h1 = MG.row_range(r, G)
        rho = eng.finalize_rows(h0, h1, mx, am, pk, want_rho=True)
        assert np.array_equal(rho.cpu().numpy(), ref["rho"][h0:h1])      # bit-exact Eq. (1)
    assert np.array_equal(mx.cpu().numpy(), ref["maxabs"])
    assert np.array_equal(am.cpu().numpy(), ref["argmax"])
    assert np.array_equal(pk.cpu().numpy(), ref["peak"])
    out = eng.select(mx, am, pk)
    assert np.array_equal(out["rank"].cpu().numpy(), ref["rank"])
    assert out["round_key"] == ref["best"].tobytes() and out["master_key"] == w.key
    assert out["peak_sample"] == w.leak_positions() and out["n_traces"] == w.n
    eng.close()


def _column_sharded(P, texts, W, G, dW=None):
    """G contexts, each over all traces and its own columns; merged by cpa_select."""
    M = W.shape[1]
    dW = _padded(W) if dW is None else dW
    dT = torch.from_numpy(np.ascontiguousarray(texts)).cuda()
    engs, shards = [], []
    for r in range(G):
        j0, j1 = MG.column_range(M, r, G)
        e = P.Engine(j1 - j0, P.CPA_S8, P.CPA_HD_LAST, 0)
        e.set_col0(j0)
        e.accumulate(dW[:, j0:j1], dT)          # column slice read in place (16-byte aligned)
        mx, am, pk = (t[0] for t in e.maxima_buffers(1))
        e.finalize_rows(0, 4096, mx, am, pk)
        shards.append((mx, am, pk))
        engs.append(e)
    stacked = [torch.stack([s[i] for s in shards]) for i in range(3)]
    out = engs[0].select(*stacked)
    for e in engs:
        e.close()
    return out


@pytest.mark.parametrize("G", [2, 3, 7])
def test_column_shards_merge_equals_single(P, c1, G):
    w, texts, W, ref = c1
    out = _column_sharded(P, texts, W, G)
    assert np.array_equal(out["maxabs"].cpu().numpy(), ref["maxabs"])
    assert np.array_equal(out["argmax"].cpu().numpy(), ref["argmax"])
    assert np.array_equal(out["peak"].cpu().numpy(), ref["peak"])
    assert np.array_equal(out["rank"].cpu().numpy(), ref["rank"])
    assert out["master_key"] == w.key and out["peak_sample"] == w.leak_positions()


def test_column_shards_tie_goes_to_lowest_sample(P, c1):
    """Both shards hold the same 256 columns, so every hypothesis' maximum ties
    across shards: the merge must keep shard 0's (lower) sample [S:298]."""
    w, texts, W, _ = c1
    W2 = np.concatenate([W[:, :256], W[:, :256]], axis=1)
    ref = O.attack_i8(O.HD_LAST, texts, W2)
    assert np.all(ref["argmax"] < 256)
    out = _column_sharded(P, texts, W2, 2)
    assert np.array_equal(out["argmax"].cpu().numpy(), ref["argmax"])
    assert np.array_equal(out["maxabs"].cpu().numpy(), ref["maxabs"])
    assert np.array_equal(out["rank"].cpu().numpy(), ref["rank"])


def test_select_and_rows_errors(P, c1):
    w, texts, W, _ = c1
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    mx, am, pk = (t[0] for t in eng.maxima_buffers(1))
    with pytest.raises(P.CpaError, match="N=0"):        # nothing accumulated yet
        eng.finalize_rows(0, 4096, mx, am, pk)
    eng.accumulate(_padded(W)[:, :w.m], torch.from_numpy(texts).cuda())
    for h0, h1 in ((-1, 10), (0, 4097), (20, 10)):
        with pytest.raises(P.CpaError, match="INVALID|invalid"):
            eng.finalize_rows(h0, h1, mx, am, pk)
    with pytest.raises(P.CpaError):
        P.cpa_finalize_rows(eng.ctx, 0, 4096, None, None, am, pk)
    with pytest.raises(P.CpaError):
        P.cpa_select(eng.ctx, 0, mx, am, pk)
    with pytest.raises(P.CpaError):
        P.cpa_set_option(eng.ctx, P.CPA_OPT_COL0, -1)
    eng.finalize_rows(5, 5, mx, am, pk)                 # empty range: no-op
    eng.close()


def test_wide_traces_w48_sampled_parity_and_column_shards(P):
    """Paper's wide-trace shape at bench's W48 size (8000 traces x 48000
    samples, one trace chunk per tile: first-touch stores); sampled sums and
    rho bit-exact against the oracle (all 4096 hypotheses), closed form over
    every column, key at the planted samples, and G = 4 column shards equal to
    the single context."""
    w = S.CONFIGS["W48"]
    texts, W = S.dataset(w)
    dW = _padded(W)
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.accumulate(dW[:, :w.m], torch.from_numpy(texts).cuda())
    out = eng.finalize(want_rho=True)
    hw = eng.sum_hw.view(16, 256, w.m)
    assert torch.equal(hw.sum(1), 1024 * eng.sum_w.view(1, -1).expand(16, -1))
    rng = np.random.default_rng(1)
    cols = np.array(sorted(set(w.leak_positions()) | set(rng.integers(0, w.m, 48).tolist()) | {0, w.m - 1}),
                    np.int32)
    ref = O.attack_i8(O.HD_LAST, texts, W, cols)
    assert np.array_equal(eng.sum_hw.cpu().numpy()[:, cols], ref["sum_hw"])
    assert np.array_equal(eng.sum_w.cpu().numpy()[cols], ref["sum_w"])
    assert np.array_equal(eng.sum_w2.cpu().numpy()[cols], ref["sum_w2"])
    assert np.array_equal(eng.sum_h.cpu().numpy(), ref["sum_h"])
    assert np.array_equal(out["rho"].cpu().numpy()[:, cols], ref["rho"])
    assert out["master_key"] == w.key and out["peak_sample"] == w.leak_positions()
    sh = _column_sharded(P, texts, W, 4, dW=dW)
    for k in ("maxabs", "argmax", "rank"):
        assert torch.equal(sh[k], out[k]), k
    assert sh["round_key"] == out["round_key"]
    eng.close()


def test_finalize_rho_buffer_alignment(P, c1):
    """The finalize kernel's 16-byte vector path (M even, aligned rho) and its
    scalar path (rho only 8-byte aligned) give bit-identical results."""
    w, texts, W, ref = c1
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.accumulate(_padded(W)[:, :w.m], torch.from_numpy(texts).cuda())
    buf = torch.zeros(4096 * w.m + 1, dtype=torch.float64, device="cuda")
    mx = torch.empty(4096, dtype=torch.float64, device="cuda")
    am = torch.empty(4096, dtype=torch.int32, device="cuda")
    for off in (0, 1):
        rho = buf[off:off + 4096 * w.m]
        P.cpa_finalize(eng.ctx, rho, mx, am)
        assert np.array_equal(rho.view(4096, w.m).cpu().numpy(), ref["rho"]), off
        assert np.array_equal(mx.cpu().numpy(), ref["maxabs"]) and np.array_equal(am.cpu().numpy(), ref["argmax"])
    eng.close()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_fused_row_owner_combine_equals_one_gpu(P, c1, G):
    """Fused combine (cpa_set_row_owners): G trace-shard contexts on the one GPU,
    each routing key byte b's cross-term rows into the accumulator of its owner
    (MG.byte_owner; same-device pointers stand in for the NVLink-mapped peer
    buffers), then only the small fields are summed.  Each owner's rows, the
    small fields and the Phase 3/4 results equal one context's bit for bit."""
    w, texts, W, ref = c1
    dW, dT = _padded(W)[:, :w.m], torch.from_numpy(texts).cuda()
    engs = [P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0) for _ in range(G)]
    addrs = [e.accum.data_ptr() for e in engs]
    for r, e in enumerate(engs):
        e.set_row_owners(MG.owner_table(addrs, G, r))
    for r, e in enumerate(engs):
        i0, i1 = MG.shard_range(w.n, r, G)
        e.accumulate(dW[i0:i1], dT[i0:i1])
    torch.cuda.synchronize()
    n_hw = 4096 * w.m
    small = sum(e.accum[n_hw:] for e in engs)
    for r, e in enumerate(engs):
        e.accum[n_hw:] = small
    torch.cuda.synchronize()
    mx, am, pk = (t[0] for t in engs[0].maxima_buffers(1))
    for r, e in enumerate(engs):
        h0, h1 = MG.row_range(r, G)
        assert np.array_equal(e.sum_hw[h0:h1].cpu().numpy(), ref["sum_hw"][h0:h1]), r
        e.finalize_rows(h0, h1, mx, am, pk)
    assert np.array_equal(engs[0].sum_w.cpu().numpy(), ref["sum_w"])
    out = engs[0].select(mx, am, pk)
    assert np.array_equal(out["maxabs"].cpu().numpy(), ref["maxabs"])
    assert np.array_equal(out["rank"].cpu().numpy(), ref["rank"])
    assert out["master_key"] == w.key
    with pytest.raises(P.CpaError):
        engs[0].set_class_sums(True)   # class sums cannot route rows
    for e in engs:
        e.set_row_owners(None)
        e.close()
