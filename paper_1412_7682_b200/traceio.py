"""Trace and ciphertext files (SPEC trace_model [S:119-185]).

The paper assumes the traces already sit in host RAM [P:166] and names no file
format; these are the steps either side of the hot path: captured traces in,
correlation curves out.  Host-side plumbing only (no CPA arithmetic).

"CPA1" binary [S:177]: magic b"CPA1", little-endian u32 n, u32 m, u8 precision
code, u8 layout code (0 = trace-major, 1 = sample-major), 2 zero bytes, then the
raw little-endian samples.  Precision codes: 4 = float32 and 8 = float64 (SPEC),
plus this build's 8-bit ADC codes 0x81 = int8 and 0x01 = uint8 (the int path).
Loading maps the payload (numpy memmap, no copy for trace-major files), checks
the length against the header, and rejects non-finite float samples [S:140].

CSV: one trace per row, comma-separated decimals [S:179].  Ciphertexts: one
32-hex-character line per trace [S:152]; keys print as 32 lowercase hex
characters [S:441].
"""
from __future__ import annotations

import dataclasses
import os
import struct

import numpy as np

MAGIC = b"CPA1"
HEADER = struct.Struct("<4sIIBBH")   # 16 bytes
PREC = {4: np.float32, 8: np.float64, 0x81: np.int8, 0x01: np.uint8}
CODE = {np.dtype(v): k for k, v in PREC.items()}
TRACE_MAJOR, SAMPLE_MAJOR = 0, 1


class TraceFileError(ValueError):
    """Malformed or inconsistent trace / ciphertext file (message says which)."""


@dataclasses.dataclass
class TraceSet:
    """n traces x m samples; `samples` is (n, m) trace-major (a view when loaded
    from a trace-major binary file)."""
    samples: np.ndarray

    @property
    def n(self) -> int:
        return self.samples.shape[0]

    @property
    def m(self) -> int:
        return self.samples.shape[1]


def read_header(path: str) -> dict:
    with open(path, "rb") as f:
        raw = f.read(HEADER.size)
    if len(raw) < HEADER.size:
        raise TraceFileError(f"{path}: truncated header ({len(raw)} of {HEADER.size} bytes)")
    magic, n, m, prec, layout, rsv = HEADER.unpack(raw)
    if magic != MAGIC:
        raise TraceFileError(f"{path}: bad magic {magic!r} (expected {MAGIC!r})")
    if prec not in PREC:
        raise TraceFileError(f"{path}: unknown precision code {prec:#x}")
    if layout not in (TRACE_MAJOR, SAMPLE_MAJOR):
        raise TraceFileError(f"{path}: unknown layout code {layout}")
    if n < 1 or m < 1:
        raise TraceFileError(f"{path}: empty trace set (n={n}, m={m})")
    if rsv != 0:
        raise TraceFileError(f"{path}: reserved header bytes are not zero")
    return dict(n=n, m=m, dtype=np.dtype(PREC[prec]), precision_code=prec,
                layout="trace-major" if layout == TRACE_MAJOR else "sample-major")


def _check_finite(a: np.ndarray, what: str):
    if a.dtype.kind == "f":
        step = max(1, (1 << 24) // max(1, a.shape[1]))
        for i in range(0, a.shape[0], step):           # bounded memory on large maps
            if not np.isfinite(a[i:i + step]).all():
                bad = i + int(np.argwhere(~np.isfinite(a[i:i + step]))[0][0])
                raise TraceFileError(f"{what}: non-finite sample in trace {bad}")


def load_traces(path: str, fmt: str | None = None, dtype=np.float32) -> TraceSet:
    """Binary ("CPA1") or CSV (`dtype` for CSV values).  Errors: TraceFileError
    for a malformed header, a payload length that disagrees with it, a
    non-finite sample or a ragged CSV; OSError for an unreadable file."""
    fmt = fmt or ("csv" if path.endswith(".csv") else "binary")
    if fmt == "csv":
        rows = []
        with open(path) as f:
            for ln, line in enumerate(f, 1):
                line = line.strip()
                if not line:
                    continue
                try:
                    rows.append([float(x) for x in line.split(",")])
                except ValueError as e:
                    raise TraceFileError(f"{path}:{ln}: {e}") from None
        if not rows:
            raise TraceFileError(f"{path}: no traces")
        if len({len(r) for r in rows}) != 1:
            raise TraceFileError(f"{path}: rows have different sample counts")
        a = np.asarray(rows, dtype=np.float64)
        _check_finite(a, path)
        dt = np.dtype(dtype)
        if dt.kind in "iu":
            info = np.iinfo(dt)
            if not (np.all(a == np.round(a)) and a.min() >= info.min and a.max() <= info.max):
                raise TraceFileError(f"{path}: values do not fit {dt}")
        return TraceSet(a.astype(dt))
    if fmt != "binary":
        raise ValueError(f"unknown trace format {fmt!r}")
    h = read_header(path)
    n, m, dt = h["n"], h["m"], h["dtype"]
    want = HEADER.size + n * m * dt.itemsize
    size = os.path.getsize(path)
    if size != want:
        raise TraceFileError(f"{path}: length mismatch: {size} bytes, header implies {want}")
    if h["layout"] == "trace-major":
        a = np.memmap(path, dtype=dt.newbyteorder("<"), mode="r", offset=HEADER.size, shape=(n, m))
    else:
        a = np.ascontiguousarray(np.memmap(path, dtype=dt.newbyteorder("<"), mode="r", offset=HEADER.size,
                                           shape=(m, n)).T)
    _check_finite(a, path)
    return TraceSet(a)


def save_traces(ts: TraceSet | np.ndarray, path: str, fmt: str = "binary", layout: str = "trace-major"):
    a = ts.samples if isinstance(ts, TraceSet) else np.asarray(ts)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("traces must be a non-empty 2-D array")
    if fmt == "csv":
        with open(path, "w") as f:
            if a.dtype.kind == "f":
                for row in a:
                    f.write(",".join(repr(float(x)) for x in row) + "\n")   # shortest round-trip decimal
            else:
                for row in a:
                    f.write(",".join(str(int(x)) for x in row) + "\n")
        return
    if a.dtype not in CODE:
        raise ValueError(f"no CPA1 precision code for {a.dtype}")
    lay = TRACE_MAJOR if layout == "trace-major" else SAMPLE_MAJOR
    with open(path, "wb") as f:
        f.write(HEADER.pack(MAGIC, a.shape[0], a.shape[1], CODE[a.dtype], lay, 0))
        body = a if lay == TRACE_MAJOR else a.T
        np.ascontiguousarray(body, dtype=a.dtype.newbyteorder("<")).tofile(f)


def load_ciphertexts(path: str) -> np.ndarray:
    """(n, 16) uint8 from hex lines; errors name the line."""
    out = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            line = line.strip()
            if not line:
                continue
            if len(line) != 32:
                raise TraceFileError(f"{path}:{ln}: wrong line length {len(line)} (expected 32 hex chars)")
            try:
                out.append(bytes.fromhex(line))
            except ValueError:
                raise TraceFileError(f"{path}:{ln}: bad hex") from None
    if not out:
        raise TraceFileError(f"{path}: no ciphertexts")
    return np.frombuffer(b"".join(out), dtype=np.uint8).reshape(-1, 16).copy()


def save_ciphertexts(texts: np.ndarray, path: str):
    with open(path, "w") as f:
        for row in np.asarray(texts, np.uint8).reshape(-1, 16):
            f.write(row.tobytes().hex() + "\n")


def parse_key(s: str) -> bytes:
    s = s.strip()
    if len(s) != 32:
        raise ValueError(f"key must be 32 hex characters, got {len(s)}")
    return bytes.fromhex(s)
