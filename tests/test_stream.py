"""Streamed accumulation with checkpoints (BASELINE config C5's key-rank curve,
SURVEY §8a row a9 "known-key rank for curves").

CPU: the chunk schedule, the curve bookkeeping, and the multi-rank checkpoint
combine over a gloo group (the oracle stands in for the GPU accumulate).  GPU:
StreamingAttack's checkpoint ranks equal the oracle's on every trace prefix and
the streamed sums equal the one-shot sums bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1412_7682_b200 import multigpu as MG
from paper_1412_7682_b200.stream import Curve, chunk_rounds, known_key_ranks


@pytest.mark.parametrize("n,chunk,world", [(1, 1, 1), (10, 3, 1), (10, 3, 2), (10, 3, 4), (1_500_000, 65536, 8),
                                           (1_500_000, 65536, 1), (65536, 65536, 3)])
def test_chunk_rounds_cover_in_order(n, chunk, world):
    rounds = chunk_rounds(n, chunk, world)
    flat = [c for rnd in rounds for c in rnd]
    assert [c[1] for c in flat] == list(range(0, n, chunk))          # global chunk order
    assert all(i1 - i0 == min(chunk, n - i0) for _, i0, i1 in flat)  # exact cover
    assert flat[-1][2] == n
    for rnd in rounds:
        assert [r for r, _, _ in rnd] == list(range(len(rnd)))       # chunk j*G + r -> rank r
    with pytest.raises(ValueError):
        chunk_rounds(10, 0, 1)


def test_known_key_ranks_and_curve():
    table = np.arange(4096, dtype=np.int32) % 256 + 1   # rank = k + 1
    key = bytes(range(16))
    assert known_key_ranks(table, key) == [b + 1 for b in range(16)]
    c = Curve()
    c.add(100, [2] + [1] * 15)
    c.add(200, [1] * 16)
    c.add(300, [3] + [1] * 15)   # falls back: not yet stable
    c.add(400, [1] * 16)
    c.add(500, [1] * 16)
    assert c.traces_to_key() == 400
    assert c.summary()[0] == [100, 2, 15]
    assert Curve().traces_to_key() is None


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, chunk, ret):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    from synth import synth as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = S.CONFIGS["C1"]
    acc = torch.zeros(MG.accum_words(w.m), dtype=torch.int64)
    scratch = torch.zeros_like(acc)
    outs = []
    for rnd in chunk_rounds(w.n, chunk, world):
        for r, i0, i1 in rnd:
            if r == rank:   # this rank's chunk: oracle partial sums added to the running acc
                texts, lv = S.texts(w, i0, i1 - i0)
                W = S.traces(w, lv, i0)
                sh, sh2 = O.model_sums(O.HD_LAST, texts)
                sw, sw2 = O.trace_sums_i8(W)
                shw = O.cross_sums_i8(O.HD_LAST, texts, W)
                acc += MG.pack(w.m, dict(sum_hw=shw, sum_w=sw, sum_w2=sw2, sum_h=sh, sum_h2=sh2,
                                         n=[i1 - i0]), acc)
        before = acc.clone()
        rows = MG.reduce_scatter_rows(acc, w.m, out=scratch)
        assert torch.equal(acc, before)            # running partials untouched
        outs.append((rows, scratch.clone().numpy()))
    if rank == 0:
        ret.put(outs)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_checkpoints_equal_prefix_sums(world):
    """Every checkpoint of a world-G streamed run (out-of-place reduce-scatter
    of the running partials) holds exactly the sums of the trace prefix
    processed so far in this rank's rows and the small fields (no double
    counting of the running partials)."""
    from oracle import oracle as O
    from synth import synth as S
    chunk = 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, chunk, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = S.CONFIGS["C1"]
    texts, W = S.dataset(w)
    rounds = chunk_rounds(w.n, chunk, world)
    assert len(outs) == len(rounds)
    for rnd, ((h0, h1), got) in zip(rounds, outs):
        n = rnd[-1][2]
        assert (h0, h1) == MG.row_range(0, world)
        ref_hw = O.cross_sums_i8(O.HD_LAST, texts[:n], W[:n])
        sh, sh2 = O.model_sums(O.HD_LAST, texts[:n])
        sw, sw2 = O.trace_sums_i8(W[:n])
        g = MG.unpack(w.m, torch.from_numpy(got))
        assert np.array_equal(g["sum_hw"].numpy()[h0:h1], ref_hw[h0:h1])   # this rank's rows
        for k, v in (("sum_h", sh), ("sum_h2", sh2), ("sum_w", sw), ("sum_w2", sw2)):
            assert np.array_equal(g[k].numpy(), v), k
        assert int(g["n"][0]) == n


@pytest.mark.gpu
def test_streaming_checkpoint_ranks_match_oracle_prefixes():
    from oracle import oracle as O
    from synth import synth as S
    import paper_1412_7682_b200 as P
    w = S.CONFIGS["C1"]
    texts, W = S.dataset(w)
    rk = O.expand_key(w.key)[10]
    ld = (w.m + 15) // 16 * 16
    Wp = np.zeros((w.n, ld), np.int8)
    Wp[:, :w.m] = W
    dW = torch.from_numpy(Wp).cuda()[:, :w.m]
    dT = torch.from_numpy(texts).cuda()
    st = P.StreamingAttack(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    curve = Curve()
    chunk = 128
    for rnd in chunk_rounds(w.n, chunk):
        for _, i0, i1 in rnd:
            st.add(dW[i0:i1], dT[i0:i1])
        n = rnd[-1][2]
        out = st.checkpoint()
        ref = O.attack_i8(O.HD_LAST, texts[:n], W[:n])
        assert np.array_equal(out["rank"].cpu().numpy(), ref["rank"]), n
        assert np.array_equal(out["maxabs"].cpu().numpy(), ref["maxabs"]), n
        curve.add(n, known_key_ranks(out["rank"].cpu().numpy(), rk))
    ref = O.attack_i8(O.HD_LAST, texts, W)
    assert np.array_equal(st.eng.sum_hw.cpu().numpy(), ref["sum_hw"])
    assert curve.points[-1][1] == known_key_ranks(ref["rank"], rk)
    assert curve.traces_to_key() is not None   # C1 recovers the key at N = 500
    st.close()


@pytest.mark.gpu
def test_async_checkpoints_equal_blocking_ones():
    """cpa_finalize_async (the non-blocking streamed checkpoint) enqueues the
    same Phase 3-4 kernels as cpa_finalize: the ranks written at every
    checkpoint, while later chunks are accumulated on the same stream, equal
    those of a blocking finalize at that prefix (and the oracle's at the end)."""
    from oracle import oracle as O
    from synth import synth as S
    import paper_1412_7682_b200 as P
    w = S.CONFIGS["C1"]
    texts, W = S.dataset(w)
    ld = (w.m + 15) // 16 * 16
    Wp = np.zeros((w.n, ld), np.int8)
    Wp[:, :w.m] = W
    dW = torch.from_numpy(Wp).cuda()[:, :w.m]
    dT = torch.from_numpy(texts).cuda()
    rounds = chunk_rounds(w.n, 96)
    a = P.StreamingAttack(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    b = P.StreamingAttack(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    buf = torch.full((len(rounds), 4096), -1, dtype=torch.int32, device="cuda")
    blocking = []
    for j, rnd in enumerate(rounds):
        for _, i0, i1 in rnd:
            a.add(dW[i0:i1], dT[i0:i1])
            b.add(dW[i0:i1], dT[i0:i1])
        assert a.checkpoint_async(buf[j])
        blocking.append(b.checkpoint()["rank"].cpu().numpy())
    a.eng.sync()
    got = buf.cpu().numpy()
    for j in range(len(rounds)):
        assert np.array_equal(got[j], blocking[j]), j
    ref = O.attack_i8(O.HD_LAST, texts, W)
    assert np.array_equal(got[-1], ref["rank"])
    a.close()
    b.close()
