"""Host-side logic of the multi-GPU combine (a7, [P:230] "multiple GPUs"):
traces shard over ranks by contiguous ranges; each rank's packed accumulator
(include/cpa.h layout) holds exact partial sums; ONE all-reduce(SUM) combines
them.  Integer sums are associative, so the result is bit-identical for any
rank count and any reduction order (ring / tree / NVLS).

No CPA arithmetic happens here -- only index ranges, the accumulator layout and
the collective call (which runs on whatever device the tensor lives on: NCCL
on the GPUs, gloo in the CPU tests)."""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous trace range [i0, i1) of `rank` among `world` (sizes differ by <= 1)."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world {world}")
    return n * rank // world, n * (rank + 1) // world


def accum_fields(M: int) -> dict[str, tuple[int, int]]:
    """(offset, length) in 8-byte words of each field of the packed accumulator."""
    return {
        "sum_hw": (0, 4096 * M),
        "sum_w": (4096 * M, M),
        "sum_w2": (4097 * M, M),
        "sum_h": (4098 * M, 4096),
        "sum_h2": (4098 * M + 4096, 4096),
        "n": (4098 * M + 8192, 1),
    }


def accum_words(M: int) -> int:
    return 4098 * M + 8193


def pack(M: int, sums: dict, like):
    """Pack a dict of sums (any array-likes) into a flat tensor shaped like `like`."""
    import torch
    out = torch.zeros(accum_words(M), dtype=like.dtype, device=like.device)
    for k, (o, n) in accum_fields(M).items():
        v = torch.as_tensor(sums[k], dtype=like.dtype).reshape(-1)
        assert v.numel() == n, (k, v.numel(), n)
        out[o:o + n] = v.to(like.device)
    return out


def unpack(M: int, acc) -> dict:
    f = accum_fields(M)
    d = {k: acc[o:o + n] for k, (o, n) in f.items()}
    d["sum_hw"] = d["sum_hw"].view(4096, M)
    return d


def allreduce_accumulator(acc, group=None):
    """Combine the per-rank partial sums: one all-reduce(SUM) of the packed buffer."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


# ---- float traces: one set of per-sample offsets for every rank ---------------
# The CPA_F32 sums are of centred samples w - o_j (include/cpa.h cpa_set_offsets);
# partial sums of different ranks add up to the sums of ONE data set only if
# every rank centred on the same o_j.  The library's default (from each context's
# own first traces) differs per rank, so a float multi-GPU run shares rank 0's.

def broadcast_offsets(first_trace, M: int, device, group=None, src: int = 0):
    """Collective: rank `src` passes its offsets ([M] float32, any device; e.g.
    its first trace, or Engine.default_offsets), the others anything (ignored);
    every rank returns the same [M] float32 tensor on `device`."""
    import torch
    import torch.distributed as dist
    world, rank = _world(group)
    buf = torch.empty(M, dtype=torch.float32, device=device)
    if rank == src:
        buf.copy_(first_trace.reshape(-1)[:M])
    if world > 1:
        dist.broadcast(buf, src=src, group=group)
    return buf


def share_offsets(engine, traces=None, group=None, src: int = 0):
    """Set the offsets rank `src`'s engine would choose for its shard (the
    library's default: the per-sample mean of its first <= 1024 traces,
    cpa_default_offsets) on every rank, before the first accumulate.  Returns
    them."""
    _, rank = _world(group)
    t0 = engine.default_offsets(traces) if (rank == src and traces is not None) else None
    o = broadcast_offsets(t0, engine.M, engine.device, group, src)
    engine.set_offsets(o)
    return o


def check_same_offsets(engine, group=None):
    """Raise unless every rank's float engine has its offsets set and equal."""
    o, ok = engine.offsets()
    assert_same_offsets(o, ok, group)


def assert_same_offsets(o, ok: bool = True, group=None):
    """Collective: raise on every rank unless all ranks' offsets `o` ([M]) are
    equal and set (all-reduce of MIN/MAX of `o` and of the 'set' flag)."""
    import torch
    import torch.distributed as dist
    world, _ = _world(group)
    if world == 1:
        return
    lo, hi = o.clone(), o.clone()
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=o.device)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag.item()) == 0 or not torch.equal(lo, hi):
        raise RuntimeError("float ranks centred their sums on different offsets: call "
                           "multigpu.share_offsets(engine, traces) on every rank before the first accumulate")


# ---- sharded Phase 3/4 (include/cpa.h "sharded Phase 3/4") -------
# The engine protocol used below (paper_1412_7682_b200.Engine implements it):
#   .accum, .M, .maxima_buffers(G), .finalize_rows(h0, h1, mx, am, pk, want_rho),
#   .select(mx, am, pk)
# Only index ranges and collectives live here; Eq. (1), the shard merge and the
# ranking run in the library.

def row_range(rank: int, world: int) -> tuple[int, int]:
    """Hypothesis rows [h0, h1) whose Phase 3 `rank` computes."""
    return shard_range(4096, rank, world)


def column_range(M: int, rank: int, world: int, align: int = 16) -> tuple[int, int]:
    """Sample columns [j0, j1) of `rank` for sample-axis sharding: balanced in
    units of `align` columns so every shard starts 16-byte aligned (the TMA
    fast path reads an int8 column slice in place).  Empty when
    M < world * align (callers require M >= world * align)."""
    units = -(-M // align)
    u0, u1 = shard_range(units, rank, world)
    return min(M, u0 * align), min(M, u1 * align)


def _world(group):
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def reduce_scatter_rows(acc, M: int, group=None, out=None) -> tuple[int, int]:
    """Combine trace-sharded partial sums for a row-sharded finalize: ONE
    reduce-scatter of the sum_hw rows (this rank receives its rows) and an
    all-reduce of the small fields (sum_w, sum_w2, sum_h, sum_h2, N).  Moves
    (G-1)/G of sum_hw per rank instead of the all-reduce's 2(G-1)/G.
    In place by default; with `out` (another packed accumulator) the combined
    rows and small fields land there and `acc` is left untouched (checkpoints
    of a running accumulation).  Returns this rank's rows [h0, h1)."""
    import torch.distributed as dist
    world, rank = _world(group)
    dst = acc if out is None else out
    n_hw = 4096 * M
    if world == 1:
        if out is not None:
            out.copy_(acc)
        return 0, 4096
    if out is not None:
        out[n_hw:].copy_(acc[n_hw:])
    dist.all_reduce(dst[n_hw:], op=dist.ReduceOp.SUM, group=group)
    h0, h1 = row_range(rank, world)
    if 4096 % world == 0:
        inp = acc[:n_hw]
        if out is None and dist.get_backend(group) != "nccl":
            inp = inp.clone()     # NCCL reduce-scatters in place; gloo gets a copy
        dist.reduce_scatter_tensor(dst[h0 * M:h1 * M], inp, op=dist.ReduceOp.SUM, group=group)
    else:                         # unequal row blocks: plain all-reduce of the rows
        if out is not None:
            out[:n_hw].copy_(acc[:n_hw])
        dist.all_reduce(dst[:n_hw], op=dist.ReduceOp.SUM, group=group)
    return h0, h1


def _pack_maxima(mx, am, pk):
    import torch
    return torch.stack([mx, am.to(torch.float64), pk])   # int32 -> f64 is exact


def gather_rows(mx, am, pk, h0: int, h1: int, group=None):
    """After each rank wrote rows [h0, h1) of the [4096] maxima: one
    all-reduce(SUM) of the packed rows, zero elsewhere, fills in every row
    (each entry has exactly one nonzero contributor, so the sum is exact)."""
    import torch
    import torch.distributed as dist
    world, _ = _world(group)
    if world == 1:
        return mx, am, pk
    buf = torch.zeros((3, 4096), dtype=torch.float64, device=mx.device)
    buf[:, h0:h1] = _pack_maxima(mx[h0:h1], am[h0:h1], pk[h0:h1])
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    mx.copy_(buf[0])
    am.copy_(buf[1].to(torch.int32))
    pk.copy_(buf[2])
    return mx, am, pk


def gather_shards(mx, am, pk, group=None):
    """Sample-axis sharding: all-gather every rank's [4096] maxima into
    stacked [G][4096] arrays (rank order = column order)."""
    import torch
    import torch.distributed as dist
    world, _ = _world(group)
    if world == 1:
        return mx.view(1, -1), am.view(1, -1), pk.view(1, -1)
    buf = _pack_maxima(mx, am, pk)
    out = torch.empty((world * buf.shape[0], buf.shape[1]), dtype=buf.dtype, device=buf.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    out = out.view(world, buf.shape[0], buf.shape[1])
    return (out[:, 0].contiguous(), out[:, 1].to(torch.int32).contiguous(), out[:, 2].contiguous())


def finalize_rows_sharded(engine, group=None, want_rho: bool = False) -> dict:
    """Trace-sharded run, row-sharded finalize: reduce-scatter + all-reduce of
    the sums, Phase 3 on this rank's hypothesis rows, gather of the maxima,
    Phase 4.  Every rank returns the same key; rho (if wanted) covers only
    this rank's rows (`rows`)."""
    from . import _binding as B
    if getattr(engine, "dtype", None) == B.CPA_F32:
        check_same_offsets(engine, group)
    if hasattr(engine, "flush"):
        engine.flush()  # CPA_OPT_NARROW: the int32 shadow into the accumulator
    h0, h1 = reduce_scatter_rows(engine.accum, engine.M, group)
    mx, am, pk = (t[0] for t in engine.maxima_buffers(1))
    rho = engine.finalize_rows(h0, h1, mx, am, pk, want_rho)
    gather_rows(mx, am, pk, h0, h1, group)
    out = engine.select(mx, am, pk)
    out.update(rows=(h0, h1), rho=rho)
    return out


def finalize_columns_sharded(engine, group=None, want_rho: bool = False) -> dict:
    """Sample-axis sharded run (engine holds ALL traces over its columns, its
    CPA_OPT_COL0 set): local Phase 3, all-gather of the maxima, merge + Phase 4."""
    mx, am, pk = (t[0] for t in engine.maxima_buffers(1))
    rho = engine.finalize_rows(0, 4096, mx, am, pk, want_rho)
    out = engine.select(*gather_shards(mx, am, pk, group))
    out.update(rho=rho)
    return out



# ---- fused combine: the cross term writes each key byte's rows to their owner ----
# (include/cpa.h cpa_set_row_owners).  Rank r owns hypothesis rows
# [4096 r/G, 4096 (r+1)/G), i.e. key bytes [16 r/G, 16 (r+1)/G), so G must divide
# 16.  Each rank maps its peers' accumulators (CUDA IPC) once; per step only the
# small fields need a collective, and that collective is also the cross-GPU
# ordering point (a rank's kernels, and thus its peer atomics, complete before its
# contribution enters the all-reduce).

def byte_owner(b: int, world: int) -> int:
    """Rank owning key byte b's hypothesis rows (row_range of that rank)."""
    if 16 % world:
        raise ValueError(f"fused combine needs world | 16, got {world}")
    return b // (16 // world)


def owner_table(addrs: list[int], world: int, rank: int) -> list[int]:
    """owners[b] for cpa_set_row_owners: the mapped address of byte b's owner's
    accumulator (0 = this rank's own)."""
    return [0 if byte_owner(b, world) == rank else addrs[byte_owner(b, world)] for b in range(16)]


class FusedOwners:
    """Map the peers' accumulators into this process (CUDA IPC) and route this
    engine's cross-term rows to their owners."""

    def __init__(self, eng, group=None):
        import torch.distributed as dist
        from . import _binding as B
        self.world, self.rank = _world(group)
        byte_owner(0, self.world)                  # validates world | 16
        h, off = B.cpa_ipc_export(eng.accum)
        dev = eng.accum.device.index
        allh = [None] * self.world
        dist.all_gather_object(allh, (h, off, dev), group=group)
        for r, (_, _, pdev) in enumerate(allh):   # system-scope atomics must work on every peer
            if not B.cpa_peer_atomics(dev, pdev):
                raise RuntimeError(f"no native peer atomics from device {dev} to rank {r}'s device {pdev}")
        self.mapped = []                           # (base, ptr) of opened peer buffers
        addrs = []
        for r, (hr, offr, _) in enumerate(allh):
            if r == self.rank:
                addrs.append(eng.accum.data_ptr())
                continue
            ptr = B.cpa_ipc_open(hr, offr)
            self.mapped.append((ptr - offr, ptr))
            addrs.append(ptr)
        self.owners = owner_table(addrs, self.world, self.rank)
        eng.set_row_owners(self.owners)
        self.eng = eng

    def close(self):
        from . import _binding as B
        self.eng.set_row_owners(None)
        for base, _ in self.mapped:
            B.cpa_ipc_close(base)
        self.mapped = []

    @classmethod
    def try_create(cls, eng, group=None):
        """Collective: every rank maps its peers, or (if any rank cannot: no peer
        access, no native peer atomics, no IPC) none does.  Returns (owners or
        None, reason or None)."""
        import torch
        import torch.distributed as dist
        owners, why = None, None
        try:
            owners = cls(eng, group)
        except Exception as e:  # noqa: BLE001 -- any failure means: use the NCCL combine
            why = f"{type(e).__name__}: {e}"
        ok = torch.tensor([0 if owners is None else 1], dtype=torch.int32, device=eng.accum.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            if owners is not None:
                owners.close()
                owners = None
            why = why or "a peer rank cannot map the accumulators"
        return owners, why


def device_barrier(t, group=None):
    """Stream-ordered cross-GPU barrier: a 1-element all-reduce.  On return (in
    stream order) every rank's earlier work on its stream has completed."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def allreduce_small_fields(acc, M: int, group=None) -> tuple[int, int]:
    """Fused combine, after the accumulation: the sum_hw rows already sit in
    their owners' accumulators; all-reduce only the small fields (sum_w,
    sum_w2, sum_h, sum_h2, N).  Returns this rank's rows [h0, h1)."""
    import torch.distributed as dist
    world, rank = _world(group)
    if world > 1:
        dist.all_reduce(acc[4096 * M:], op=dist.ReduceOp.SUM, group=group)
    return row_range(rank, world)
