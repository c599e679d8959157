"""The N>1 path on CPU: world_size-2 gloo process group.  Each rank computes
its shard's exact partial sums (with the oracle standing in for the GPU
accumulate), packs them in the include/cpa.h layout, and the production
all-reduce (paper_1412_7682_b200.multigpu) combines them; the result must equal
the single-process sums bit for bit, and Eq. (1) from it the single-process rho."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1412_7682_b200 import multigpu as MG


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _collect(q, procs, n, timeout=300):
    """n results from the workers; fails fast if one of them died."""
    import queue
    import time
    out, t_end = [], time.time() + timeout
    while len(out) < n:
        try:
            out.append(q.get(timeout=2))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead and time.time() < t_end, f"worker exit codes {dead}"
    return out


def _worker(rank, world, port, name, ret):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    from synth import synth as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = S.CONFIGS[name]
    i0, i1 = MG.shard_range(w.n, rank, world)
    texts, lv = S.texts(w, i0, i1 - i0)
    W = S.traces(w, lv, i0)
    sh, sh2 = O.model_sums(O.HD_LAST, texts)
    sw, sw2 = O.trace_sums_i8(W)
    shw = O.cross_sums_i8(O.HD_LAST, texts, W)
    acc = MG.pack(w.m, dict(sum_hw=shw, sum_w=sw, sum_w2=sw2, sum_h=sh, sum_h2=sh2, n=[i1 - i0]),
                  torch.zeros(1, dtype=torch.int64))
    MG.allreduce_accumulator(acc)
    if rank == 0:
        ret.put(acc.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_allreduce_equals_single_process(world):
    from oracle import oracle as O
    from synth import synth as S
    name = "C1"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    acc = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = S.CONFIGS[name]
    texts, W = S.dataset(w)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    got = MG.unpack(w.m, torch.from_numpy(acc))
    for k in ("sum_hw", "sum_w", "sum_w2", "sum_h", "sum_h2"):
        assert np.array_equal(got[k].numpy(), ref[k]), k
    assert int(got["n"][0]) == w.n
    rho = O.rho_eq1_grid(w.n, got["sum_hw"].numpy(), got["sum_h"].numpy(), got["sum_h2"].numpy(),
                         got["sum_w"].numpy(), got["sum_w2"].numpy())
    assert np.array_equal(rho, ref["rho"])


def test_shard_ranges_cover_exactly():
    for n in (1, 2, 7, 500, 1_500_000):
        for world in (1, 2, 3, 4, 8):
            rs = [MG.shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_layout_matches_library():
    import paper_1412_7682_b200 as P
    for M in (1, 500, 5000):
        f = MG.accum_fields(M)
        assert MG.accum_words(M) == P.cpa_accum_words(M)
        for i, k in enumerate(("sum_hw", "sum_w", "sum_w2", "sum_h", "sum_h2", "n")):
            assert f[k][0] == P.cpa_accum_offset(M, i)


# ---- sharded Phase 3/4: row-sharded finalize and sample-axis sharding ---------
class OracleEngine:
    """Stands in for paper_1412_7682_b200.Engine on CPU: the accumulator holds
    the oracle's exact partial sums of this rank's data; finalize_rows / select
    follow include/cpa.h with the oracle's Eq. (1), phase 3 and phase 4 (the
    shard merge written out in numpy).  Exercises multigpu's collectives and
    index ranges; the library's own kernels are checked in test_sharded_gpu."""

    def __init__(self, texts, W, cols):
        from oracle import oracle as O
        self.O, self.cols, self.M = O, np.asarray(cols, np.int32), len(cols)
        sh, sh2 = O.model_sums(O.HD_LAST, texts)
        sw, sw2 = O.trace_sums_i8(W, self.cols)
        shw = O.cross_sums_i8(O.HD_LAST, texts, W, self.cols)
        self.accum = MG.pack(self.M, dict(sum_hw=shw, sum_w=sw, sum_w2=sw2, sum_h=sh, sum_h2=sh2,
                                          n=[W.shape[0]]), torch.zeros(1, dtype=torch.int64))

    def maxima_buffers(self, G=1):
        return (torch.zeros((G, 4096), dtype=torch.float64), torch.zeros((G, 4096), dtype=torch.int32),
                torch.zeros((G, 4096), dtype=torch.float64))

    def finalize_rows(self, h0, h1, mx, am, pk, want_rho=False):
        s = MG.unpack(self.M, self.accum)
        rho = self.O.rho_eq1_grid(int(s["n"][0]), s["sum_hw"].numpy(), s["sum_h"].numpy(), s["sum_h2"].numpy(),
                                  s["sum_w"].numpy(), s["sum_w2"].numpy())
        m, a, p = self.O.phase3(rho, self.cols)
        mx[h0:h1], am[h0:h1], pk[h0:h1] = (torch.from_numpy(x[h0:h1]) for x in (m, a, p))
        return torch.from_numpy(rho[h0:h1]) if want_rho else None

    def select(self, mx, am, pk):
        mx, am, pk = (t.reshape(-1, 4096).clone() for t in (mx, am, pk))
        for g in range(1, mx.shape[0]):     # largest max|rho|, ties to the lowest sample
            win = (mx[g] > mx[0]) | ((mx[g] == mx[0]) & (am[g] < am[0]))
            mx[0][win], am[0][win], pk[0][win] = mx[g][win], am[g][win], pk[g][win]
        best, rank = self.O.phase4(mx[0].numpy())
        return dict(maxabs=mx[0], argmax=am[0], peak=pk[0], rank=torch.from_numpy(rank), round_key=best.tobytes())


def _sharded_worker(rank, world, port, mode, ret):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from synth import synth as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = S.CONFIGS["C1"]
    if mode == "rows":              # trace shard, all columns
        i0, i1 = MG.shard_range(w.n, rank, world)
        texts, lv = S.texts(w, i0, i1 - i0)
        eng = OracleEngine(texts, S.traces(w, lv, i0), np.arange(w.m))
        out = MG.finalize_rows_sharded(eng, want_rho=True)
    else:                           # all traces, this rank's columns
        j0, j1 = MG.column_range(w.m, rank, world)
        texts, W = S.dataset(w)
        eng = OracleEngine(texts, W, np.arange(j0, j1))
        out = MG.finalize_columns_sharded(eng)
    ret.put((rank, {k: (v.numpy() if torch.is_tensor(v) else v) for k, v in out.items() if k != "rows"},
             out.get("rows")))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,world", [("rows", 2), ("rows", 3), ("rows", 4), ("columns", 2), ("columns", 3)])
def test_gloo_sharded_finalize_equals_single_process(mode, world):
    from oracle import oracle as O
    from synth import synth as S
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = _collect(q, procs, world)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = S.CONFIGS["C1"]
    texts, W = S.dataset(w)
    ref = O.attack_i8(O.HD_LAST, texts, W)
    for rank, out, rows in outs:        # every rank holds the full, identical selection
        assert np.array_equal(out["maxabs"], ref["maxabs"])
        assert np.array_equal(out["argmax"], ref["argmax"])
        assert np.array_equal(out["peak"], ref["peak"])
        assert np.array_equal(out["rank"], ref["rank"])
        assert out["round_key"] == ref["best"].tobytes()
        if mode == "rows":
            h0, h1 = rows
            assert (h0, h1) == MG.row_range(rank, world)
            assert np.array_equal(out["rho"], ref["rho"][h0:h1])


def test_column_ranges_aligned_cover():
    for M in (16, 500, 5000, 48000, 20000):
        for world in (1, 2, 3, 4, 8):
            if M < 16 * world:
                continue
            rs = [MG.column_range(M, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(j0 % 16 == 0 and j1 > j0 for j0, j1 in rs)
    assert [MG.row_range(r, 8) for r in range(8)][3] == (1536, 2048)


def test_byte_owner_table_matches_row_ranges():
    """Fused combine bookkeeping: byte b's owner holds rows [256 b, 256 b + 256)
    inside its row_range, for every G dividing 16; other G are refused."""
    for G in (1, 2, 4, 8, 16):
        for b in range(16):
            h0, h1 = MG.row_range(MG.byte_owner(b, G), G)
            assert h0 <= 256 * b and 256 * (b + 1) <= h1
        tab = MG.owner_table([1000 + r for r in range(G)], G, 0)
        assert [0 if MG.byte_owner(b, G) == 0 else 1000 + MG.byte_owner(b, G) for b in range(16)] == tab
    for G in (3, 5, 6):
        with pytest.raises(ValueError):
            MG.byte_owner(0, G)


class _FakeEng:
    def __init__(self):
        self.accum = torch.zeros(8, dtype=torch.int64)
        self.owner_calls = []

    def set_row_owners(self, owners):
        self.owner_calls.append(owners)


class _Flaky(MG.FusedOwners):
    """Rank 0 maps its peers; rank 1 cannot (as on a box without peer atomics)."""
    closed = 0

    def __init__(self, eng, group=None):
        if dist.get_rank() == 1:
            raise RuntimeError("no native peer atomics")
        self.eng, self.mapped, self.owners = eng, [], [0] * 16
        eng.set_row_owners(self.owners)

    def close(self):
        _Flaky.closed += 1
        self.eng.set_row_owners(None)


def _fused_consensus_worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = _FakeEng()
    owners, why = _Flaky.try_create(eng)
    ret.put((rank, owners is None, why, eng.owner_calls[-1] if eng.owner_calls else "none", _Flaky.closed))
    dist.barrier()
    dist.destroy_process_group()


def test_fused_combine_consensus_falls_back_on_every_rank():
    """FusedOwners.try_create is collective: when one rank cannot map its peers,
    every rank falls back to the NCCL combine (no rank is left routing rows)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_consensus_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, none0, why0, last0, closed0), (r1, none1, why1, last1, _) = res
    assert none0 and none1                       # both fall back
    assert last0 is None and closed0 == 1        # rank 0 undid its routing
    assert "peer atomics" in why1 and why0       # the reason is reported on both


def _float_worker(rank, world, port, shared, ret):
    """Float traces (a6) on a trace shard: the sums are of the CENTRED samples
    fl32(w - o_j), as the library computes them (k_split_f32), packed in the
    fp64 accumulator layout and combined by the production reduce-scatter.
    shared=True: o = rank 0's first trace, broadcast (multigpu.broadcast_offsets,
    what bench.py / share_offsets do); False: each rank's own first trace (the
    library default, wrong across ranks)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    from synth import synth as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = S.CONFIGS["C3"].replace(n=3000, m=24, a=0.02)
    i0, i1 = MG.shard_range(w.n, rank, world)
    texts, lv = S.texts(w, i0, i1 - i0)
    W = S.traces(w, lv, i0)
    if shared:
        o = MG.broadcast_offsets(torch.from_numpy(W[0]), w.m, "cpu").numpy()
        MG.assert_same_offsets(torch.from_numpy(o))
    else:
        o = W[0].copy()
        try:
            MG.assert_same_offsets(torch.from_numpy(o))
            raised = False
        except RuntimeError:
            raised = True
        assert raised, "differing offsets must be rejected"
    C = (W - o[None, :]).astype(np.float32)        # fp32 subtraction, as on the GPU
    sh, sh2 = O.model_sums(O.HD_LAST, texts)
    shw, sw, sw2 = O.sums_f32(O.HD_LAST, texts, C)
    acc = MG.pack(w.m, dict(sum_hw=shw, sum_w=sw, sum_w2=sw2, sum_h=sh, sum_h2=sh2, n=[i1 - i0]),
                  torch.zeros(1, dtype=torch.float64))
    h0, h1 = MG.reduce_scatter_rows(acc, w.m)
    ret.put((rank, h0, h1, acc.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shared", [True, False])
def test_gloo_float_combine_needs_shared_offsets(shared):
    """World 2, float traces [P:201-217, P:230]: with one set of offsets the
    combined rows give rho within 1e-9 of the single-process oracle on the raw
    traces; with per-rank offsets (the library default) they do not (>1e-3)."""
    from oracle import oracle as O
    from synth import synth as S
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_float_worker, args=(r, world, port, shared, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = _collect(q, procs, world)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = S.CONFIGS["C3"].replace(n=3000, m=24, a=0.02)
    texts, W = S.dataset(w)
    shw, sw, sw2 = O.sums_f32(O.HD_LAST, texts, W)
    sh, sh2 = O.model_sums(O.HD_LAST, texts)
    ref = O.rho_eq1_f64_grid(w.n, shw, sh, sh2, sw, sw2)
    err = 0.0
    for rank, h0, h1, acc in res:
        got = MG.unpack(w.m, torch.from_numpy(acc))
        assert int(got["n"][0]) == w.n
        rho = O.rho_eq1_f64_grid(w.n, got["sum_hw"].numpy(), got["sum_h"].numpy().astype(np.int64),
                                 got["sum_h2"].numpy().astype(np.int64), got["sum_w"].numpy(),
                                 got["sum_w2"].numpy())
        err = max(err, float(np.max(np.abs(rho[h0:h1] - ref[h0:h1]))))
    if shared:
        assert err <= 1e-9, err
    else:
        assert err > 1e-3, err
