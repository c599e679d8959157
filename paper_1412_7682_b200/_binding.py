"""Thin ctypes binding of libcpa.so -- same names as include/cpa.h.

Argument marshalling only: every step of the CPA hot path runs in the CUDA
kernels behind the C ABI.  There is no CPU fallback: importing this module
without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CPA_LIB_PATH") or os.path.join(_PKG, "libcpa.so")  # override: debugging only

CPA_OK = 0
CPA_E_INVALID_ARG, CPA_E_BAD_STATE, CPA_E_CUDA, CPA_E_NO_MEMORY = 1, 2, 3, 4
CPA_E_TOO_FEW_TRACES, CPA_E_OVERFLOW, CPA_E_UNSUPPORTED_DEVICE, CPA_E_NONFINITE = 5, 6, 7, 8
CPA_S8, CPA_U8, CPA_F32 = 0, 1, 2
CPA_HD_LAST, CPA_HW_LAST, CPA_HW_FIRST = 0, 1, 2
(CPA_OPT_KCHUNK, CPA_OPT_TIMING, CPA_OPT_OVERLAP, CPA_OPT_STAGE_BYTES, CPA_OPT_COL0, CPA_OPT_CLASS_SUMS,
 CPA_OPT_FUSE_HIST, CPA_OPT_XT_TILES, CPA_OPT_SPILL, CPA_OPT_NARROW) = 1, 2, 3, 4, 5, 6, 7, 8, 9, 10
CPA_NUM_PHASES = 6
PHASE_NAMES = ("modelsums", "moments", "xterm", "finalize", "phase4", "spill_reduce")
FIELD_HW, FIELD_W, FIELD_W2, FIELD_H, FIELD_H2, FIELD_N = range(6)

# every symbol include/cpa.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = (
    "cpa_accum_words", "cpa_accum_bytes", "cpa_accum_offset", "cpa_init", "cpa_accumulate",
    "cpa_accumulate_host", "cpa_finalize", "cpa_finalize_async", "cpa_finalize_rows", "cpa_select",
    "cpa_set_row_owners", "cpa_ipc_export", "cpa_ipc_open", "cpa_ipc_close", "cpa_xterm_clock", "cpa_peer_atomics", "cpa_reset", "cpa_sync", "cpa_flush", "cpa_destroy",
    "cpa_get_offsets", "cpa_default_offsets",
    "cpa_set_offsets", "cpa_set_option", "cpa_phase_times", "cpa_launch_count", "cpa_status_str", "cpa_last_error",
    "cpa_aes_expand_key", "cpa_aes_invert_key_schedule", "cpa_graph_begin", "cpa_graph_end", "cpa_graph_launch",
)


class CpaError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = _lib.cpa_last_error().decode(errors="replace")
        super().__init__(f"{where}: {_lib.cpa_status_str(status).decode()} ({detail})")


class cpa_result(C.Structure):
    _fields_ = [("round_key", C.c_uint8 * 16), ("master_key", C.c_uint8 * 16),
                ("peak_sample", C.c_int32 * 16), ("peak_rho", C.c_double * 16),
                ("n_traces", C.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the CUDA path has no fallback)")
    L = C.CDLL(LIB_PATH)
    P, I64, I32, ST = C.c_void_p, C.c_int64, C.c_int32, C.c_int
    sig = {
        "cpa_accum_words": (C.c_size_t, [I32]),
        "cpa_accum_bytes": (C.c_size_t, [I32]),
        "cpa_accum_offset": (C.c_size_t, [I32, C.c_int]),
        "cpa_init": (ST, [C.POINTER(P), I32, C.c_int, C.c_int, C.c_int, P, P]),
        "cpa_accumulate": (ST, [P, P, I64, P, I64]),
        "cpa_accumulate_host": (ST, [P, P, I64, P, I64]),
        "cpa_finalize": (ST, [P, P, P, P, P, C.POINTER(cpa_result)]),
        "cpa_finalize_rows": (ST, [P, I32, I32, P, P, P, P]),
        "cpa_finalize_async": (ST, [P, P, P, P, P, P]),
        "cpa_graph_begin": (ST, [P]),
        "cpa_graph_end": (ST, [P]),
        "cpa_graph_launch": (ST, [P]),
        "cpa_select": (ST, [P, I32, P, P, P, P, C.POINTER(cpa_result)]),
        "cpa_set_row_owners": (ST, [P, P]),
        "cpa_ipc_export": (ST, [P, P, C.POINTER(C.c_uint64)]),
        "cpa_ipc_open": (ST, [P, C.c_uint64, C.POINTER(P)]),
        "cpa_ipc_close": (ST, [P]),
        "cpa_xterm_clock": (ST, [P, C.POINTER(C.c_double)]),
        "cpa_peer_atomics": (ST, [C.c_int, C.c_int, C.POINTER(C.c_int)]),
        "cpa_reset": (ST, [P]),
        "cpa_sync": (ST, [P]),
        "cpa_flush": (ST, [P]),
        "cpa_destroy": (ST, [P]),
        "cpa_set_offsets": (ST, [P, P]),
        "cpa_get_offsets": (ST, [P, P, C.POINTER(C.c_int)]),
        "cpa_default_offsets": (ST, [P, P, I64, I64, P]),
        "cpa_set_option": (ST, [P, C.c_int, I64]),
        "cpa_phase_times": (ST, [P, P, P]),
        "cpa_launch_count": (I64, [P]),
        "cpa_status_str": (C.c_char_p, [C.c_int]),
        "cpa_last_error": (C.c_char_p, []),
        "cpa_aes_expand_key": (None, [P, P]),
        "cpa_aes_invert_key_schedule": (None, [P, C.c_int, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


_lib = _load()


def _ptr(x):
    """Raw address of a torch tensor / int / None for the C ABI."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(type(x))


def _check(st: int, where: str):
    if st != CPA_OK:
        raise CpaError(st, where)


# ---- same-name wrappers ------------------------------------------------------
def cpa_accum_words(M: int) -> int:
    return _lib.cpa_accum_words(M)


def cpa_accum_bytes(M: int) -> int:
    return _lib.cpa_accum_bytes(M)


def cpa_accum_offset(M: int, field: int) -> int:
    return _lib.cpa_accum_offset(M, field)


def cpa_init(M: int, dtype: int, model: int, device: int, stream: int, d_accum) -> int:
    h = C.c_void_p()
    _check(_lib.cpa_init(C.byref(h), M, dtype, model, device, stream, _ptr(d_accum)), "cpa_init")
    return h.value


def cpa_accumulate(ctx, d_traces, ld: int, d_texts, N: int):
    _check(_lib.cpa_accumulate(ctx, _ptr(d_traces), ld, _ptr(d_texts), N), "cpa_accumulate")


def cpa_accumulate_host(ctx, h_traces, ld: int, h_texts, N: int):
    _check(_lib.cpa_accumulate_host(ctx, _ptr(h_traces), ld, _ptr(h_texts), N), "cpa_accumulate_host")


def cpa_finalize(ctx, d_rho=None, d_maxabs=None, d_argmax=None, d_rank=None) -> cpa_result:
    res = cpa_result()
    _check(_lib.cpa_finalize(ctx, _ptr(d_rho), _ptr(d_maxabs), _ptr(d_argmax), _ptr(d_rank),
                             C.byref(res)), "cpa_finalize")
    return res


def cpa_finalize_async(ctx, d_rho=None, d_maxabs=None, d_argmax=None, d_rank=None, d_best=None):
    _check(_lib.cpa_finalize_async(ctx, _ptr(d_rho), _ptr(d_maxabs), _ptr(d_argmax), _ptr(d_rank), _ptr(d_best)),
           "cpa_finalize_async")


def cpa_finalize_rows(ctx, h0: int, h1: int, d_rho, d_maxabs, d_argmax, d_peak):
    _check(_lib.cpa_finalize_rows(ctx, h0, h1, _ptr(d_rho), _ptr(d_maxabs), _ptr(d_argmax), _ptr(d_peak)),
           "cpa_finalize_rows")


def cpa_set_row_owners(ctx, owners):
    """owners: 16 device addresses (int; 0 = this context's accumulator) or None (off)."""
    if owners is None:
        _check(_lib.cpa_set_row_owners(ctx, None), "cpa_set_row_owners")
        return
    arr = (C.c_void_p * 16)(*[int(o) or None for o in owners])
    _check(_lib.cpa_set_row_owners(ctx, arr), "cpa_set_row_owners")


def cpa_xterm_clock(ctx) -> float:
    mhz = C.c_double(0.0)
    _check(_lib.cpa_xterm_clock(ctx, C.byref(mhz)), "cpa_xterm_clock")
    return mhz.value


def cpa_peer_atomics(dev: int, peer: int) -> bool:
    ok = C.c_int(0)
    _check(_lib.cpa_peer_atomics(dev, peer, C.byref(ok)), "cpa_peer_atomics")
    return bool(ok.value)


def cpa_ipc_export(d_ptr) -> tuple[bytes, int]:
    h = (C.c_uint8 * 64)()
    off = C.c_uint64(0)
    _check(_lib.cpa_ipc_export(_ptr(d_ptr), h, C.byref(off)), "cpa_ipc_export")
    return bytes(h), off.value


def cpa_ipc_open(handle: bytes, offset: int) -> int:
    h = (C.c_uint8 * 64).from_buffer_copy(bytes(handle))
    out = C.c_void_p()
    _check(_lib.cpa_ipc_open(h, offset, C.byref(out)), "cpa_ipc_open")
    return out.value


def cpa_ipc_close(d_base: int):
    _check(_lib.cpa_ipc_close(C.c_void_p(d_base)), "cpa_ipc_close")


def cpa_select(ctx, G: int, d_maxabs, d_argmax, d_peak, d_rank=None) -> cpa_result:
    res = cpa_result()
    _check(_lib.cpa_select(ctx, G, _ptr(d_maxabs), _ptr(d_argmax), _ptr(d_peak), _ptr(d_rank), C.byref(res)),
           "cpa_select")
    return res


def cpa_reset(ctx):
    _check(_lib.cpa_reset(ctx), "cpa_reset")


def cpa_sync(ctx):
    _check(_lib.cpa_sync(ctx), "cpa_sync")


def cpa_flush(ctx):
    _check(_lib.cpa_flush(ctx), "cpa_flush")


def cpa_graph_begin(ctx):
    _check(_lib.cpa_graph_begin(ctx), "cpa_graph_begin")


def cpa_graph_end(ctx):
    _check(_lib.cpa_graph_end(ctx), "cpa_graph_end")


def cpa_graph_launch(ctx):
    _check(_lib.cpa_graph_launch(ctx), "cpa_graph_launch")


def cpa_destroy(ctx):
    _check(_lib.cpa_destroy(ctx), "cpa_destroy")


def cpa_set_offsets(ctx, d_offsets):
    _check(_lib.cpa_set_offsets(ctx, _ptr(d_offsets)), "cpa_set_offsets")


def cpa_get_offsets(ctx, d_out=None) -> bool:
    """Copy the offsets in force into d_out (device float32 [M], optional);
    return whether they were set (explicitly or by the first accumulate)."""
    ok = C.c_int(0)
    _check(_lib.cpa_get_offsets(ctx, _ptr(d_out), C.byref(ok)), "cpa_get_offsets")
    return bool(ok.value)


def cpa_default_offsets(ctx, d_traces, ld: int, N: int, d_out):
    """The library's default offsets for these device traces (mean of the first
    <= 1024 rows) into d_out (device float32 [M]); asynchronous on the stream."""
    _check(_lib.cpa_default_offsets(ctx, _ptr(d_traces), ld, N, _ptr(d_out)), "cpa_default_offsets")


def cpa_set_option(ctx, option: int, value: int):
    _check(_lib.cpa_set_option(ctx, option, value), "cpa_set_option")


def cpa_phase_times(ctx):
    """({phase: ms}, {phase: launches}) since the last call (CPA_OPT_TIMING)."""
    ms = (C.c_double * CPA_NUM_PHASES)()
    n = (C.c_int64 * CPA_NUM_PHASES)()
    _check(_lib.cpa_phase_times(ctx, ms, n), "cpa_phase_times")
    return dict(zip(PHASE_NAMES, list(ms))), dict(zip(PHASE_NAMES, list(n)))


def cpa_launch_count(ctx) -> int:
    return _lib.cpa_launch_count(ctx)


def cpa_status_str(st: int) -> str:
    return _lib.cpa_status_str(st).decode()


def cpa_last_error() -> str:
    return _lib.cpa_last_error().decode()


def cpa_aes_expand_key(key: bytes) -> list[bytes]:
    k = (C.c_uint8 * 16).from_buffer_copy(bytes(key))
    rk = (C.c_uint8 * 176)()
    _lib.cpa_aes_expand_key(k, rk)
    raw = bytes(rk)
    return [raw[16 * r:16 * r + 16] for r in range(11)]


def cpa_aes_invert_key_schedule(rk: bytes, round_index: int = 10) -> bytes:
    r = (C.c_uint8 * 16).from_buffer_copy(bytes(rk))
    k = (C.c_uint8 * 16)()
    _lib.cpa_aes_invert_key_schedule(r, round_index, k)
    return bytes(k)
