"""Engine: a convenience wrapper over the C ABI for PyTorch callers.

PyTorch supplies device memory, streams and process groups only; the CPA
arithmetic runs in libcpa.so.  Multi-GPU (traces sharded over ranks [P:230]):
every rank calls ``accumulate`` on its shard, then ``allreduce`` (one NCCL
all-reduce(SUM) of the packed accumulator), then ``finalize``.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _binding as B

_TORCH_DTYPE = {B.CPA_S8: torch.int8, B.CPA_U8: torch.uint8, B.CPA_F32: torch.float32}


class Engine:
    def __init__(self, M: int, dtype: int = B.CPA_S8, model: int = B.CPA_HD_LAST,
                 device: int | torch.device = 0, stream: torch.cuda.Stream | None = None):
        self.device = torch.device("cuda", device if isinstance(device, int) else device.index)
        self.M, self.dtype, self.model = M, dtype, model
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        words = B.cpa_accum_words(M)
        acc_t = torch.float64 if dtype == B.CPA_F32 else torch.int64
        self.accum = torch.zeros(words, dtype=acc_t, device=self.device)
        self.ctx = B.cpa_init(M, dtype, model, self.device.index, self.stream.cuda_stream, self.accum)

    # ---- views into the packed accumulator (include/cpa.h layout) ----
    def _field(self, f, n):
        o = B.cpa_accum_offset(self.M, f)
        return self.accum[o:o + n]

    @property
    def sum_hw(self):
        self.flush()  # CPA_OPT_NARROW: the int32 shadow into the accumulator first
        return self._field(B.FIELD_HW, 4096 * self.M).view(4096, self.M)

    @property
    def sum_w(self):
        return self._field(B.FIELD_W, self.M)

    @property
    def sum_w2(self):
        return self._field(B.FIELD_W2, self.M)

    @property
    def sum_h(self):
        return self._field(B.FIELD_H, 4096)

    @property
    def sum_h2(self):
        return self._field(B.FIELD_H2, 4096)

    @property
    def n(self):
        return self._field(B.FIELD_N, 1)

    # ---- the path ----
    def set_kchunk(self, k: int):
        B.cpa_set_option(self.ctx, B.CPA_OPT_KCHUNK, k)

    def set_timing(self, on: bool = True):
        B.cpa_set_option(self.ctx, B.CPA_OPT_TIMING, int(on))

    def set_stage_bytes(self, nbytes: int):
        B.cpa_set_option(self.ctx, B.CPA_OPT_STAGE_BYTES, nbytes)

    def set_col0(self, col0: int):
        """Global index of this context's sample 0 (sample-axis sharding)."""
        B.cpa_set_option(self.ctx, B.CPA_OPT_COL0, col0)

    def set_fuse_hist(self, on: bool = True):
        """CPA_OPT_FUSE_HIST: a3's byte-pair histogram counted inside the cross-term kernel (default off)."""
        B.cpa_set_option(self.ctx, B.CPA_OPT_FUSE_HIST, int(bool(on)))

    def set_xt_tiles(self, v: int):
        """CPA_OPT_XT_TILES: int8 cross-term variant (0 model, 1 two sample tiles per unit, 2 one tile, overlapped spill)."""
        B.cpa_set_option(self.ctx, B.CPA_OPT_XT_TILES, v)

    def set_spill(self, mode: int):
        """CPA_OPT_SPILL: 0 auto (default), 1 red.add per element, 2 bulk tensor reduce-add,
        3 per-chunk partial stores + one reduce pass (include/cpa.h)."""
        B.cpa_set_option(self.ctx, B.CPA_OPT_SPILL, mode)

    def set_narrow(self, on: bool | int = True):
        """CPA_OPT_NARROW: int32 cross-term sums while exact (half the sum_hw bytes);
        the accumulator's HW field is stale until flush() (include/cpa.h).  An int
        > 1 also caps the shadow at that many traces (tests)."""
        B.cpa_set_option(self.ctx, B.CPA_OPT_NARROW, int(on))

    def flush(self):
        """cpa_flush: add a live int32 shadow (CPA_OPT_NARROW) into the accumulator
        (on the context's stream; torch's current stream then waits for it, so a
        read of the accumulator in torch sees the flushed sums)."""
        B.cpa_flush(self.ctx)
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def set_row_owners(self, owners):
        """cpa_set_row_owners: 16 device addresses (0 = own accumulator) or None."""
        B.cpa_set_row_owners(self.ctx, owners)

    def set_class_sums(self, on: bool = True):
        """CPA_OPT_CLASS_SUMS: class-sum cross term for HW_LAST / HW_FIRST (exact)."""
        B.cpa_set_option(self.ctx, B.CPA_OPT_CLASS_SUMS, int(bool(on)))

    def set_overlap(self, mode: int | bool = True):
        """CPA_OPT_OVERLAP: 0 serial, 1 (True) low-priority side stream, 2 co-resident, 3 fused (default)."""
        B.cpa_set_option(self.ctx, B.CPA_OPT_OVERLAP, int(mode))

    def phase_times(self):
        """({phase: ms}, {phase: launches}) of the CUDA-event-timed launches
        since the last call (needs set_timing(True))."""
        return B.cpa_phase_times(self.ctx)

    def accumulate(self, traces: torch.Tensor, texts: torch.Tensor):
        assert traces.device == self.device and texts.device == self.device
        assert traces.dtype == _TORCH_DTYPE[self.dtype] and texts.dtype == torch.uint8
        assert traces.dim() == 2 and traces.shape[1] == self.M and traces.stride(1) == 1
        assert texts.shape == (traces.shape[0], 16) and texts.is_contiguous()
        B.cpa_accumulate(self.ctx, traces, traces.stride(0), texts, traces.shape[0])

    def accumulate_host(self, traces: np.ndarray | torch.Tensor, texts: np.ndarray | torch.Tensor):
        """Host (ideally pinned) buffers: the library stages them (cpa_accumulate_host).
        The element type must be the context's: raw bytes are passed through."""
        want = _TORCH_DTYPE[self.dtype]
        if isinstance(traces, np.ndarray):
            ok = traces.dtype == np.dtype(str(want).replace("torch.", ""))
            row_ok = traces.ndim == 2 and traces.strides[1] == traces.itemsize
            ld = traces.strides[0] // traces.itemsize if traces.ndim == 2 else 0
        else:
            ok = traces.dtype == want and traces.device.type == "cpu"
            row_ok = traces.dim() == 2 and traces.stride(1) == 1
            ld = traces.stride(0) if traces.dim() == 2 else 0
        if not ok:
            raise TypeError(f"traces dtype {traces.dtype} does not match the context's {want} (host buffer)")
        if not row_ok or traces.shape[1] != self.M:
            raise ValueError(f"traces must be [N][{self.M}] with unit column stride")
        n = traces.shape[0]
        tx_dtype = texts.dtype == (np.uint8 if isinstance(texts, np.ndarray) else torch.uint8)
        tx_contig = texts.flags["C_CONTIGUOUS"] if isinstance(texts, np.ndarray) else texts.is_contiguous()
        if not tx_dtype or tuple(texts.shape) != (n, 16) or not tx_contig:
            raise ValueError("texts must be a contiguous uint8 [N][16] host buffer")
        B.cpa_accumulate_host(self.ctx, traces, ld, texts, n)

    # ---- float path: per-sample offsets (include/cpa.h cpa_set_offsets) ----
    def set_offsets(self, offsets: torch.Tensor | None):
        """CPA_F32: centre every sample on offsets[j] (device float32 [M]; None =
        0).  Multi-GPU: every rank must use the SAME offsets, see
        multigpu.share_offsets."""
        if offsets is not None:
            assert offsets.device == self.device and offsets.dtype == torch.float32
            assert offsets.is_contiguous() and offsets.numel() == self.M
        B.cpa_set_offsets(self.ctx, offsets)

    def default_offsets(self, traces: torch.Tensor) -> torch.Tensor:
        """The offsets the library would choose for these device traces (the
        per-sample mean of the first <= 1024 rows), without setting them."""
        assert traces.device == self.device and traces.dtype == torch.float32 and traces.stride(1) == 1
        out = torch.empty(self.M, dtype=torch.float32, device=self.device)
        B.cpa_default_offsets(self.ctx, traces, traces.stride(0), traces.shape[0], out)
        self.sync()
        return out

    def offsets(self) -> tuple[torch.Tensor, bool]:
        """(the offsets in force [M] float32, whether they were set)."""
        out = torch.empty(self.M, dtype=torch.float32, device=self.device)
        ok = B.cpa_get_offsets(self.ctx, out)
        self.sync()
        return out, ok

    def allreduce(self, group=None, check_offsets: bool = True):
        """Combine partial sums over ranks: one all-reduce(SUM) [a7].  Exact
        for the int64 accumulator under any reduction order.  Float contexts:
        the ranks' sums must be centred on the same offsets (checked first
        unless the caller already did, check_offsets=False)."""
        from .multigpu import allreduce_accumulator, check_same_offsets
        if self.dtype == B.CPA_F32 and check_offsets:
            check_same_offsets(self, group)
        self.flush()
        with torch.cuda.stream(self.stream):
            allreduce_accumulator(self.accum, group)

    def finalize(self, want_rho: bool = False):
        dev = self.device
        rho = torch.empty((4096, self.M), dtype=torch.float64, device=dev) if want_rho else None
        maxabs = torch.empty(4096, dtype=torch.float64, device=dev)
        argmax = torch.empty(4096, dtype=torch.int32, device=dev)
        rank = torch.empty(4096, dtype=torch.int32, device=dev)
        res = B.cpa_finalize(self.ctx, rho, maxabs, argmax, rank)
        return dict(rho=rho, maxabs=maxabs, argmax=argmax, rank=rank,
                    round_key=bytes(res.round_key), master_key=bytes(res.master_key),
                    peak_sample=list(res.peak_sample), peak_rho=list(res.peak_rho),
                    n_traces=res.n_traces)

    def finalize_async(self, rank, maxabs=None, argmax=None, best=None, rho=None):
        """Phase 3 + 4 enqueued without blocking (cpa_finalize_async): rank [4096]
        int32 (and the optional maxabs/argmax/best[32]/rho) fill in stream order."""
        B.cpa_finalize_async(self.ctx, rho, maxabs, argmax, rank, best)

    # ---- CUDA-graph replay of a fixed-shape step (include/cpa.h cpa_graph_*) ----
    def graph_begin(self):
        """Start capturing this context's stream (needs a non-default stream):
        reset / accumulate / finalize_async are recorded until graph_end."""
        B.cpa_graph_begin(self.ctx)

    def graph_end(self):
        B.cpa_graph_end(self.ctx)

    def graph_launch(self):
        """Replay the captured calls as one graph launch (asynchronous)."""
        B.cpa_graph_launch(self.ctx)

    def maxima_buffers(self, G: int = 1):
        """Zeroed per-hypothesis maxima (maxabs, argmax, peak) for G stacked shards."""
        dev = self.device
        return (torch.zeros((G, 4096), dtype=torch.float64, device=dev),
                torch.zeros((G, 4096), dtype=torch.int32, device=dev),
                torch.zeros((G, 4096), dtype=torch.float64, device=dev))

    def finalize_rows(self, h0: int, h1: int, maxabs, argmax, peak, want_rho: bool = False):
        """Phase 3 for hypothesis rows [h0, h1) into the [4096] maxima arrays
        (sharded finalize, include/cpa.h); returns rho [h1-h0][M] or None."""
        rho = (torch.empty((h1 - h0, self.M), dtype=torch.float64, device=self.device)
               if want_rho else None)
        B.cpa_finalize_rows(self.ctx, h0, h1, rho, maxabs, argmax, peak)
        return rho

    def select(self, maxabs, argmax, peak):
        """Phase 4 from G stacked shards of maxima ([G][4096]; merged in place
        into shard 0 when G > 1)."""
        G = maxabs.shape[0] if maxabs.dim() == 2 else 1
        rank = torch.empty(4096, dtype=torch.int32, device=self.device)
        res = B.cpa_select(self.ctx, G, maxabs, argmax, peak, rank)
        m = (lambda t: t[0] if t.dim() == 2 else t)
        return dict(maxabs=m(maxabs), argmax=m(argmax), peak=m(peak), rank=rank,
                    round_key=bytes(res.round_key), master_key=bytes(res.master_key),
                    peak_sample=list(res.peak_sample), peak_rho=list(res.peak_rho),
                    n_traces=res.n_traces)

    def reset(self):
        B.cpa_reset(self.ctx)

    def sync(self):
        B.cpa_sync(self.ctx)

    @property
    def launches(self) -> int:
        return B.cpa_launch_count(self.ctx)

    def close(self):
        if self.ctx:
            B.cpa_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
