"""ctypes wrapper around oracle/liboracle.so -- the plain CPU CPA oracle.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package (paper_1412_7682_b200/).  The C source (oracle.c) cites the passages of
PAPER.md / SPEC.md each function follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

HD_LAST, HW_LAST, HW_FIRST = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (single-threaded, no FMA contraction)."""
    src = os.path.join(HERE, "oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off",
             "-fno-fast-math", "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        i64, i32 = C.c_int64, C.c_int
        L.or_selection.restype = C.c_int
        L.or_selection.argtypes = [C.c_int, P, C.c_int, C.c_int]
        L.or_rho_eq1.restype = C.c_int
        L.or_rho_eq1.argtypes = [i64] * 6 + [P]
        L.or_rho_eq1_grid.restype = C.c_int
        L.or_rho_eq1_grid.argtypes = [i64, P, P, P, P, P, i32, P]
        L.or_model_sums.argtypes = [i32, P, i64, P, P]
        L.or_trace_sums_i8.argtypes = [P, i32, i64, i64, P, i32, P, P]
        L.or_cross_sums_i8.argtypes = [i32, P, P, i32, i64, i64, P, i32, P]
        L.or_rho_two_pass_i8.argtypes = [i32, P, P, i32, i64, i64, P, i32, P, i32, P]
        L.or_rho_two_pass_f32.argtypes = [i32, P, P, i64, i64, P, i32, P, i32, P]
        L.or_sums_f32.argtypes = [i32, P, P, i64, i64, P, i32, P, P, P]
        L.or_rho_eq1_f64_grid.argtypes = [i64, P, P, P, P, P, i32, P]
        L.or_model_sums_hyps.argtypes = [i32, P, i64, P, i32, P, P]
        L.or_cross_sums_hyps_i8.argtypes = [i32, P, P, i32, i64, i64, P, i32, P, i32, P]
        L.or_phase3.argtypes = [P, i32, P, P, P, P]
        L.or_phase4.argtypes = [P, P, P]
        L.or_invert_key_schedule.argtypes = [P, C.c_int, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"] or a.ndim == 0
    return a.ctypes.data_as(C.c_void_p)


# ---- AES ------------------------------------------------------------------
def aes_tables():
    s = np.zeros(256, np.uint8); i = np.zeros(256, np.uint8)
    lib().or_aes_tables(_p(s), _p(i))
    return s, i


def shiftrows_src():
    sr = np.zeros(16, np.uint8)
    lib().or_shiftrows_src(_p(sr))
    return sr


def expand_key(key) -> np.ndarray:
    k = np.frombuffer(bytes(key), np.uint8).copy()
    rk = np.zeros((11, 16), np.uint8)
    lib().or_expand_key(_p(k), _p(rk))
    return rk


def invert_key_schedule(rk, round_index: int = 10) -> np.ndarray:
    r = np.frombuffer(bytes(rk), np.uint8).copy()
    k = np.zeros(16, np.uint8)
    lib().or_invert_key_schedule(_p(r), round_index, _p(k))
    return k


def encrypt_with_states(pt, key):
    p = np.frombuffer(bytes(pt), np.uint8).copy()
    k = np.frombuffer(bytes(key), np.uint8).copy()
    ct = np.zeros(16, np.uint8); st = np.zeros(16, np.uint8)
    lib().or_encrypt_with_states(_p(p), _p(k), _p(ct), _p(st))
    return ct, st


# ---- selection and sums ---------------------------------------------------
def selection(model: int, text, b: int, k: int) -> int:
    t = np.frombuffer(bytes(text), np.uint8).copy()
    return lib().or_selection(model, _p(t), b, k)


def model_sums(model: int, texts: np.ndarray):
    texts = np.ascontiguousarray(texts, np.uint8)
    n = texts.shape[0]
    sh = np.zeros(4096, np.int64); sh2 = np.zeros(4096, np.int64)
    lib().or_model_sums(model, _p(texts), n, _p(sh), _p(sh2))
    return sh, sh2


def _cols(W: np.ndarray, cols):
    if cols is None:
        cols = np.arange(W.shape[1], dtype=np.int32)
    return np.ascontiguousarray(cols, np.int32)


def trace_sums_i8(W: np.ndarray, cols=None):
    W = np.ascontiguousarray(W)
    assert W.dtype in (np.int8, np.uint8)
    cols = _cols(W, cols)
    sw = np.zeros(len(cols), np.int64); sw2 = np.zeros(len(cols), np.int64)
    lib().or_trace_sums_i8(_p(W), int(W.dtype == np.int8), W.shape[0], W.shape[1],
                           _p(cols), len(cols), _p(sw), _p(sw2))
    return sw, sw2


def cross_sums_i8(model: int, texts: np.ndarray, W: np.ndarray, cols=None):
    W = np.ascontiguousarray(W); texts = np.ascontiguousarray(texts, np.uint8)
    assert W.dtype in (np.int8, np.uint8) and texts.shape == (W.shape[0], 16)
    cols = _cols(W, cols)
    shw = np.zeros((4096, len(cols)), np.int64)
    lib().or_cross_sums_i8(model, _p(texts), _p(W), int(W.dtype == np.int8),
                           W.shape[0], W.shape[1], _p(cols), len(cols), _p(shw))
    return shw


def model_sums_hyps(model: int, texts: np.ndarray, hyps):
    texts = np.ascontiguousarray(texts, np.uint8)
    hyps = np.ascontiguousarray(hyps, np.int32)
    sh = np.zeros(len(hyps), np.int64); sh2 = np.zeros(len(hyps), np.int64)
    lib().or_model_sums_hyps(model, _p(texts), texts.shape[0], _p(hyps), len(hyps), _p(sh), _p(sh2))
    return sh, sh2


def cross_sums_hyps_i8(model: int, texts: np.ndarray, W: np.ndarray, hyps, cols=None):
    W = np.ascontiguousarray(W); texts = np.ascontiguousarray(texts, np.uint8)
    cols = _cols(W, cols)
    hyps = np.ascontiguousarray(hyps, np.int32)
    shw = np.zeros((len(hyps), len(cols)), np.int64)
    lib().or_cross_sums_hyps_i8(model, _p(texts), _p(W), int(W.dtype == np.int8), W.shape[0], W.shape[1],
                                _p(cols), len(cols), _p(hyps), len(hyps), _p(shw))
    return shw


def rho_eq1(n, s_hw, s_h, s_h2, s_w, s_w2) -> float:
    out = np.zeros((), np.float64)
    rc = lib().or_rho_eq1(n, int(s_hw), int(s_h), int(s_h2), int(s_w), int(s_w2), _p(out))
    if rc:
        raise OverflowError("Eq. (1) intermediate does not fit int64")
    return float(out)


def rho_eq1_grid(n, sum_hw, sum_h, sum_h2, sum_w, sum_w2) -> np.ndarray:
    ncols = sum_hw.shape[1]
    rho = np.zeros((4096, ncols), np.float64)
    args = [np.ascontiguousarray(a, np.int64) for a in (sum_hw, sum_h, sum_h2, sum_w, sum_w2)]
    rc = lib().or_rho_eq1_grid(n, *[_p(a) for a in args], ncols, _p(rho))
    if rc:
        raise OverflowError("Eq. (1) intermediate does not fit int64")
    return rho


def rho_two_pass_i8(model, texts, W, cols=None, hyps=None) -> np.ndarray:
    W = np.ascontiguousarray(W); texts = np.ascontiguousarray(texts, np.uint8)
    cols = _cols(W, cols)
    hyps = np.arange(4096, dtype=np.int32) if hyps is None else np.ascontiguousarray(hyps, np.int32)
    rho = np.zeros((len(hyps), len(cols)), np.float64)
    lib().or_rho_two_pass_i8(model, _p(texts), _p(W), int(W.dtype == np.int8), W.shape[0],
                             W.shape[1], _p(cols), len(cols), _p(hyps), len(hyps), _p(rho))
    return rho


def rho_two_pass_f32(model, texts, W, cols=None, hyps=None) -> np.ndarray:
    W = np.ascontiguousarray(W, np.float32); texts = np.ascontiguousarray(texts, np.uint8)
    cols = _cols(W, cols)
    hyps = np.arange(4096, dtype=np.int32) if hyps is None else np.ascontiguousarray(hyps, np.int32)
    rho = np.zeros((len(hyps), len(cols)), np.float64)
    lib().or_rho_two_pass_f32(model, _p(texts), _p(W), W.shape[0], W.shape[1], _p(cols),
                              len(cols), _p(hyps), len(hyps), _p(rho))
    return rho


def sums_f32(model, texts, W, cols=None):
    W = np.ascontiguousarray(W, np.float32); texts = np.ascontiguousarray(texts, np.uint8)
    cols = _cols(W, cols)
    shw = np.zeros((4096, len(cols)), np.float64)
    sw = np.zeros(len(cols), np.float64); sw2 = np.zeros(len(cols), np.float64)
    lib().or_sums_f32(model, _p(texts), _p(W), W.shape[0], W.shape[1], _p(cols), len(cols),
                      _p(shw), _p(sw), _p(sw2))
    return shw, sw, sw2


def rho_eq1_f64_grid(n, sum_hw, sum_h, sum_h2, sum_w, sum_w2):
    ncols = sum_hw.shape[1]
    rho = np.zeros((4096, ncols), np.float64)
    a = [np.ascontiguousarray(sum_hw, np.float64), np.ascontiguousarray(sum_h, np.int64),
         np.ascontiguousarray(sum_h2, np.int64), np.ascontiguousarray(sum_w, np.float64),
         np.ascontiguousarray(sum_w2, np.float64)]
    lib().or_rho_eq1_f64_grid(n, *[_p(x) for x in a], ncols, _p(rho))
    return rho


def phase3(rho: np.ndarray, cols=None):
    rho = np.ascontiguousarray(rho, np.float64)
    ncols = rho.shape[1]
    cols = np.arange(ncols, dtype=np.int32) if cols is None else np.ascontiguousarray(cols, np.int32)
    mx = np.zeros(4096, np.float64); am = np.zeros(4096, np.int32); pk = np.zeros(4096, np.float64)
    lib().or_phase3(_p(rho), ncols, _p(cols), _p(mx), _p(am), _p(pk))
    return mx, am, pk


def phase4(maxabs: np.ndarray):
    maxabs = np.ascontiguousarray(maxabs, np.float64)
    best = np.zeros(16, np.uint8); rank = np.zeros(4096, np.int32)
    lib().or_phase4(_p(maxabs), _p(best), _p(rank))
    return best, rank


def attack_i8(model, texts, W, cols=None):
    """Full oracle pipeline (Phases 1-4) over the listed columns.

    Returns a dict of every intermediate: exact sums, rho_B grid, phase-3 and
    phase-4 results."""
    W = np.ascontiguousarray(W)
    n = W.shape[0]
    cols = _cols(W, cols)
    sh, sh2 = model_sums(model, texts)
    sw, sw2 = trace_sums_i8(W, cols)
    shw = cross_sums_i8(model, texts, W, cols)
    rho = rho_eq1_grid(n, shw, sh, sh2, sw, sw2)
    mx, am, pk = phase3(rho, cols)
    best, rank = phase4(mx)
    return dict(n=n, cols=cols, sum_h=sh, sum_h2=sh2, sum_w=sw, sum_w2=sw2, sum_hw=shw,
                rho=rho, maxabs=mx, argmax=am, peak=pk, best=best, rank=rank)
