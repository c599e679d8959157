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


def combined_copy(acc, scratch, group=None):
    """Checkpoint of a running multi-rank accumulation: copy this rank's partial
    sums into `scratch` and all-reduce the copy, leaving `acc` (the running
    partials) untouched so later chunks are not double counted."""
    scratch.copy_(acc)
    return allreduce_accumulator(scratch, group)
