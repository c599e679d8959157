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
