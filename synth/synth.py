"""Seeded synthetic CPA workloads (inputs only) -- ctypes wrapper over synth/.

The recipe: uniform seeded plaintexts, AES-128 with a
known key (FIPS-197 App. A key by default), one leak sample per key byte at
L_b = floor((b+1) M / 17) carrying the true last-round register Hamming
distance [S:327, S:346], a per-sample baseline mu_j, and Gaussian noise drawn
through a counter-based hash of (seed, i, j).  Both the oracle and the CUDA
path consume these inputs; this module contains none of the CPA arithmetic.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(HERE, "libsynth.so")
DEV_LIB = os.path.join(HERE, "libsynth_dev.so")

LEAK_HD_LAST, LEAK_HW_LAST, LEAK_HW_FIRST = 0, 1, 2
S8, U8, F32 = 0, 1, 2
DEFAULT_KEY = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")  # FIPS-197 App. A.1


class SyParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("m", C.c_int32), ("leak", C.c_int32 * 16),
                ("mu_lo_q32", C.c_int64), ("mu_hi_q32", C.c_int64),
                ("a_q32", C.c_int64), ("sigma_q16", C.c_int64)]


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    n: int
    m: int
    dtype: int            # S8 / U8 / F32
    a: float              # leak amplitude
    sigma: float          # noise sigma
    mu_lo: float
    mu_hi: float
    seed: int = 1
    key: bytes = DEFAULT_KEY
    leak_model: int = LEAK_HD_LAST

    def leak_positions(self):
        return [((b + 1) * self.m) // 17 for b in range(16)]

    def params(self) -> SyParams:
        p = SyParams()
        p.seed = self.seed
        p.m = self.m
        for b, L in enumerate(self.leak_positions()):
            p.leak[b] = L
        p.mu_lo_q32 = int(round(self.mu_lo * 2**32))
        p.mu_hi_q32 = int(round(self.mu_hi * 2**32))
        p.a_q32 = int(round(self.a * 2**32))
        p.sigma_q16 = int(round(self.sigma * 2**16))
        return p

    def replace(self, **kw) -> "Workload":
        return dataclasses.replace(self, **kw)

    @property
    def np_dtype(self):
        return {S8: np.int8, U8: np.uint8, F32: np.float32}[self.dtype]


# BASELINE.json configs[0..4]; calibration in SURVEY.md Sec. 8(d)
CONFIGS = {
    "C1": Workload("C1", 500, 500, S8, 5.0, 16.0, -40, 40),
    "C1-0": Workload("C1-0", 500, 500, S8, 1.0, 0.0, -40, 40),
    "C2": Workload("C2", 2000, 5000, S8, 3.0, 16.0, -40, 40),
    "C3": Workload("C3", 100_000, 5000, F32, 1e-3, 0.045, 0.5, 1.5),
    "C4": Workload("C4", 1_500_000, 5000, S8, 0.25, 32.0, -40, 40),
    "C5": Workload("C5", 1_500_000, 20000, S8, 0.25, 32.0, -40, 40),
    # the paper's wide-trace shape (dataset2: 48000 samples
    # per trace [P:168]; Fig. 5's largest run, 8000 traces [P:188, P:199])
    "W48": Workload("W48", 8000, 48000, S8, 3.0, 16.0, -40, 40),
    # C4 / C2 with last-round Hamming-WEIGHT leakage, attacked
    # with the HW_LAST model (class-sum cross term)
    "C4-HW": Workload("C4-HW", 1_500_000, 5000, S8, 0.25, 32.0, -40, 40, leak_model=LEAK_HW_LAST),
    "C2-HW": Workload("C2-HW", 2000, 5000, S8, 3.0, 16.0, -40, 40, leak_model=LEAK_HW_LAST),
}


def build(force: bool = False, device: bool = True):
    srcs = [os.path.join(HERE, f) for f in ("synth.c", "synth.h", "synth_core.h")]
    if force or not os.path.exists(HOST_LIB) or os.path.getmtime(HOST_LIB) < max(map(os.path.getmtime, srcs)):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-o", HOST_LIB,
                               os.path.join(HERE, "synth.c"), "-lm"])
    if device:
        dsrc = srcs + [os.path.join(HERE, "synth_dev.cu")]
        if force or not os.path.exists(DEV_LIB) or os.path.getmtime(DEV_LIB) < max(map(os.path.getmtime, dsrc)):
            subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                                   "-Xcompiler", "-fPIC", "-shared", "-o", DEV_LIB,
                                   os.path.join(HERE, "synth_dev.cu")])


_host = None
_dev = None


def _hlib():
    global _host
    if _host is None:
        build(device=False)
        _host = C.CDLL(HOST_LIB)
        P = C.c_void_p
        _host.sy_texts.argtypes = [P, P, C.c_int, C.c_int64, C.c_int64, P, P]
        _host.sy_traces.argtypes = [P, C.c_int, P, P, C.c_int64, C.c_int64, P, C.c_int, P, C.c_int64]
        _host.sy_gauss_table.argtypes = [P]
    return _host


def _dlib():
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_LIB):
            build(device=True)
        _dev = C.CDLL(DEV_LIB)
        P = C.c_void_p
        _dev.sy_dev_traces.argtypes = [P, C.c_int, P, P, C.c_int64, C.c_int64, P, C.c_int64, P]
        _dev.sy_dev_traces.restype = C.c_int
    return _dev


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


_gauss_cache = None


def gauss_table() -> np.ndarray:
    global _gauss_cache
    if _gauss_cache is None:
        t = np.zeros(65536, np.int32)
        _hlib().sy_gauss_table(_p(t))
        _gauss_cache = t
    return _gauss_cache


def texts(w: Workload, i0: int = 0, n: int | None = None):
    """(texts N x 16 u8, planted leak values N x 16 u8) for traces [i0, i0+n)."""
    n = w.n - i0 if n is None else n
    t = np.zeros((n, 16), np.uint8); lv = np.zeros((n, 16), np.uint8)
    p = w.params()
    _hlib().sy_texts(C.byref(p), bytes(w.key), w.leak_model, i0, n, _p(t), _p(lv))
    return t, lv


def traces(w: Workload, leakv: np.ndarray, i0: int = 0, cols=None) -> np.ndarray:
    """Host traces for rows [i0, i0+len(leakv)) and the given columns (all if None)."""
    n = leakv.shape[0]
    leakv = np.ascontiguousarray(leakv, np.uint8)
    p = w.params()
    if cols is None:
        out = np.zeros((n, w.m), w.np_dtype)
        _hlib().sy_traces(C.byref(p), w.dtype, _p(gauss_table()), _p(leakv), i0, n, None, 0,
                          _p(out), w.m)
    else:
        cols = np.ascontiguousarray(cols, np.int32)
        out = np.zeros((n, len(cols)), w.np_dtype)
        _hlib().sy_traces(C.byref(p), w.dtype, _p(gauss_table()), _p(leakv), i0, n, _p(cols),
                          len(cols), _p(out), len(cols))
    return out


def dataset(w: Workload, cols=None):
    """Host (texts, traces) for the whole workload (small configs only)."""
    t, lv = texts(w)
    return t, traces(w, lv, 0, cols)


def dev_traces(w: Workload, d_leakv, i0: int, n: int, d_out, ld: int, stream_ptr: int = 0,
               d_gauss=None):
    """Generate all M columns of traces [i0, i0+n) on the device.

    d_leakv / d_out / d_gauss are torch CUDA tensors (d_gauss optional)."""
    import torch
    if d_gauss is None:
        d_gauss = torch.from_numpy(gauss_table()).to(d_out.device)
    p = w.params()
    rc = _dlib().sy_dev_traces(C.byref(p), w.dtype, C.c_void_p(d_gauss.data_ptr()),
                               C.c_void_p(d_leakv.data_ptr()), i0, n,
                               C.c_void_p(d_out.data_ptr()), ld, C.c_void_p(stream_ptr))
    if rc != 0:
        raise RuntimeError(f"sy_dev_traces failed ({rc})")
    return d_out
