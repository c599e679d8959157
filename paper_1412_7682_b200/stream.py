"""Streamed accumulation with checkpoints -> the key-rank-vs-trace-count curve.

BASELINE config C5 ("1.5M traces x 20,000 samples streamed in 64K-trace chunks
with key-rank-vs-trace-count curve") and SURVEY §8a row a9 ("known-key rank for
curves"): traces arrive in chunks; after each round of chunks the attack is
finalized from the sums so far (Phases 3-4 [P:81-87] on a prefix of the traces)
and the rank of the known key byte among the 256 guesses is recorded per byte.
The traces-to-key point is the first checkpoint from which every byte ranks 1.

Multi-GPU [P:230]: global chunk c covers traces [c*chunk, (c+1)*chunk); round j
gives chunk j*G + r to rank r.  With the fused combine (fused=True) every rank's
cross term adds each key byte's rows into the owner rank's running accumulator
over NVLink (multigpu.FusedOwners), so a checkpoint only all-reduces the small
fields into a scratch accumulator and copies the rank's own, already combined
rows.  Otherwise each rank keeps its own partial sums and a checkpoint
reduce-scatters them (out of place) into the scratch accumulator, so the running
partials are never double counted.  Either way each rank then finalizes its
4096/G hypothesis rows, the maxima are gathered and Phase 4 ranks them
(SURVEY §8e (ii)).

Only index bookkeeping and orchestration live here; every sum, rho and rank is
computed by libcpa through the C ABI."""
from __future__ import annotations

from dataclasses import dataclass, field


def chunk_rounds(n_total: int, chunk: int, world: int = 1) -> list[list[tuple[int, int, int]]]:
    """Rounds of (rank, i0, i1): global chunk c = [c*chunk, min(n, (c+1)*chunk)),
    chunk j*world + r goes to rank r in round j.  The last round may leave some
    ranks without a chunk."""
    if chunk <= 0 or world <= 0:
        raise ValueError("chunk and world must be positive")
    n_chunks = (n_total + chunk - 1) // chunk
    rounds = []
    for j in range((n_chunks + world - 1) // world):
        rnd = []
        for r in range(world):
            c = j * world + r
            if c < n_chunks:
                rnd.append((r, c * chunk, min(n_total, (c + 1) * chunk)))
        rounds.append(rnd)
    return rounds


def known_key_ranks(rank_table, key_bytes) -> list[int]:
    """Rank (1 = best) of the known sub-key of each byte, from the 4096-entry
    rank table cpa_finalize returns (h = 256*b + k)."""
    return [int(rank_table[256 * b + int(key_bytes[b])]) for b in range(16)]


@dataclass
class Curve:
    """(traces so far, rank of the known key byte per byte) at each checkpoint."""
    points: list[tuple[int, list[int]]] = field(default_factory=list)

    def add(self, n: int, ranks: list[int]):
        self.points.append((n, list(ranks)))

    def traces_to_key(self) -> int | None:
        """First checkpoint from which all 16 bytes stay at rank 1 (None if never)."""
        first = None
        for n, ranks in self.points:
            if all(r == 1 for r in ranks):
                if first is None:
                    first = n
            else:
                first = None
        return first

    def summary(self) -> list[list[int]]:
        """[[n, worst rank over the 16 bytes, bytes at rank 1], ...]"""
        return [[n, max(r), sum(1 for x in r if x == 1)] for n, r in self.points]


class StreamingAttack:
    """Chunked accumulate + checkpoint finalize on one rank of a (possibly
    multi-GPU) run.  `group` is a torch.distributed group (None = default when
    initialized; single process otherwise)."""

    def __init__(self, M: int, dtype: int, model: int, device: int = 0, group=None, fused: bool = False,
                 narrow: bool | None = None):
        import torch
        import torch.distributed as dist

        from . import multigpu as MG
        from .engine import Engine
        self.group = group
        self.world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
        self.eng = Engine(M, dtype, model, device)
        # CPA_OPT_NARROW (int8): the cross term in int32 while exact -- half the
        # sum_hw bytes in every chunk's spill and every checkpoint's finalize.
        # Default: one rank (a multi-GPU checkpoint combines the int64 accumulator)
        from . import _binding as B
        if (self.world == 1 if narrow is None else narrow) and dtype != B.CPA_F32:
            self.eng.set_narrow(True)
        # multi-GPU checkpoints finalize from an all-reduced copy of the partials
        self.view = Engine(M, dtype, model, device, stream=self.eng.stream) if self.world > 1 else None
        self.n_local = 0
        # fused combine: every chunk's cross-term rows go straight to their owner
        # rank's running accumulator (MG.FusedOwners); a checkpoint then only
        # all-reduces the small fields
        self.owners, self.fused_note = (MG.FusedOwners.try_create(self.eng, group) if (fused and self.world > 1)
                                        else (None, None))
        self._bar = torch.zeros(1, dtype=torch.int32, device=self.eng.device)

    def share_offsets(self, traces=None, src: int = 0):
        """Float traces, multi-GPU (collective, before the first add): centre
        every rank's sums on rank `src`'s default offsets (multigpu.share_offsets);
        the checkpoint view finalizes with the same offsets."""
        from . import multigpu as MG
        o = MG.share_offsets(self.eng, traces, self.group, src)
        if self.view is not None:
            self.view.set_offsets(o)
        self._offsets_shared = True

    def add(self, traces, texts):
        from . import _binding as B
        if self.view is not None and self.eng.dtype == B.CPA_F32 and not getattr(self, "_offsets_shared", False):
            raise RuntimeError("float multi-GPU stream: call share_offsets() on every rank before the first add "
                               "(each rank's sums must be centred on the same offsets)")
        self.eng.accumulate(traces, texts)
        self.n_local += traces.shape[0]

    def checkpoint(self, want_rho: bool = False) -> dict:
        if self.view is None:
            return self.eng.finalize(want_rho=want_rho)
        import torch

        from . import multigpu as MG
        self.eng.flush()  # CPA_OPT_NARROW: the int32 shadow into the accumulator
        with torch.cuda.stream(self.eng.stream):
            if self.owners is not None:
                # small fields: all-reduced copy (also the point after which every
                # peer's atomics into this rank's rows are complete); then this
                # rank's rows, already combined; then a barrier so that no peer
                # starts the next round's atomics into them before the copy
                M = self.eng.M
                n_hw = 4096 * M
                self.view.accum[n_hw:].copy_(self.eng.accum[n_hw:])
                h0, h1 = MG.allreduce_small_fields(self.view.accum, M, self.group)
                self.view.accum[h0 * M:h1 * M].copy_(self.eng.accum[h0 * M:h1 * M])
                MG.device_barrier(self._bar, self.group)
            else:
                h0, h1 = MG.reduce_scatter_rows(self.eng.accum, self.eng.M, self.group, out=self.view.accum)
            mx, am, pk = (t[0] for t in self.view.maxima_buffers(1))
            rho = self.view.finalize_rows(h0, h1, mx, am, pk, want_rho)
            MG.gather_rows(mx, am, pk, h0, h1, self.group)
            out = self.view.select(mx, am, pk)
        out.update(rows=(h0, h1), rho=rho)
        return out

    def checkpoint_async(self, rank_out) -> bool:
        """Single GPU: enqueue the checkpoint's Phases 3-4 without blocking, the
        4096 ranks into rank_out (a device int32 [4096] view), and return True;
        the caller reads them after its last checkpoint (one D2H for the whole
        curve).  Multi-GPU checkpoints block (collectives + sharded finalize):
        returns False and the caller uses checkpoint()."""
        if self.view is not None:
            return False
        self.eng.finalize_async(rank_out)
        return True

    def reset(self):
        self.eng.reset()
        self.n_local = 0
        if self.owners is not None:   # every owner is zeroed before any peer adds into it
            import torch

            from . import multigpu as MG
            with torch.cuda.stream(self.eng.stream):
                MG.device_barrier(self._bar, self.group)

    @property
    def launches(self) -> int:
        return self.eng.launches + (self.view.launches if self.view is not None else 0)

    def close(self):
        if self.owners is not None:
            self.owners.close()
        if self.view is not None:
            self.view.close()
        self.eng.close()
