"""Command line around the C ABI (SPEC cli [S:397-451]).

    python -m paper_1412_7682_b200 attack --traces T.cpa1 --ciphertexts T.ct [--json]
                                          [--model hd_last|hw_last|hw_first] [--export-curves out.csv]
    python -m paper_1412_7682_b200 export-curves --traces ... --ciphertexts ... --out curves.csv
    python -m paper_1412_7682_b200 simulate --key HEX32 --n N --m M [--dtype s8|u8|f32] --out-prefix P
    python -m paper_1412_7682_b200 inspect T.cpa1

attack streams the (memory-mapped) trace file through cpa_accumulate_host in
chunks, then cpa_finalize: the Phase-1..4 arithmetic runs on the GPU only
(there is no CPU fallback).  Diagnostics go to stderr, data to stdout / files;
exit status 0 iff the command completed [S:445].
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from . import traceio as IO

MODELS = {"hd_last": 0, "hw_last": 1, "hw_first": 2}


def _die(msg: str, code: int = 2):
    print(f"error: {msg}", file=sys.stderr)
    sys.exit(code)


def run_attack(traces: np.ndarray, texts: np.ndarray, model: int = 0, device: int = 0,
               chunk_bytes: int = 1 << 30, want_rho: bool = False) -> dict:
    """Host arrays in, attack result out (Phases 1-4 on the GPU through the C ABI)."""
    import torch

    from . import _binding as B
    from .engine import Engine
    n, m = traces.shape
    if texts.shape != (n, 16):
        raise ValueError(f"trace count {n} != ciphertext count {texts.shape[0]}")
    if n < 2:
        raise ValueError(f"N={n} < 2 traces: Eq. (1) is undefined")
    kind = {np.dtype(np.int8): B.CPA_S8, np.dtype(np.uint8): B.CPA_U8, np.dtype(np.float32): B.CPA_F32}
    if traces.dtype == np.float64:
        print("note: float64 traces are narrowed to float32 (the float path's input type)", file=sys.stderr)
    if traces.dtype not in kind and traces.dtype != np.float64:
        raise TypeError(f"unsupported trace dtype {traces.dtype} (int8, uint8, float32 or float64)")
    dt = kind.get(traces.dtype, B.CPA_F32)
    eng = Engine(m, dt, model, device)
    if dt != B.CPA_F32:
        eng.set_narrow(True)   # int32 cross-term sums while exact (one GPU, no combine)
    rows = max(1, chunk_bytes // (m * traces.dtype.itemsize))
    texts = np.ascontiguousarray(texts, np.uint8)
    for i0 in range(0, n, rows):
        i1 = min(n, i0 + rows)
        w = traces[i0:i1]
        if w.dtype == np.float64:
            w = w.astype(np.float32)
        eng.accumulate_host(np.ascontiguousarray(w), texts[i0:i1])
    out = eng.finalize(want_rho=want_rho)
    mx = out["maxabs"].view(16, 256).cpu().numpy()
    rank = out["rank"].view(16, 256).cpu().numpy()
    table = []
    for b in range(16):
        order = np.argsort(rank[b], kind="stable")
        k1, k2 = int(order[0]), int(order[1])
        table.append(dict(byte=b, subkey=k1, maxabs=float(mx[b, k1]), margin=float(mx[b, k1] - mx[b, k2]),
                          second=k2, peak_sample=int(out["peak_sample"][b]), peak_rho=float(out["peak_rho"][b])))
    res = dict(n_traces=int(out["n_traces"]), n_samples=m, model=model, table=table,
               round_key=out["round_key"].hex(), master_key=out["master_key"].hex())
    if want_rho:
        best = [t["subkey"] for t in table]
        res["curves"] = out["rho"].view(16, 256, m)[torch.arange(16), torch.tensor(best)].cpu().numpy()
    eng.close()
    return res


def write_curves(path: str, res: dict):
    """Plot-ready long CSV: m rows per byte position, for its top-ranked sub-key."""
    with open(path, "w") as f:
        f.write("byte,subkey,sample,rho\n")
        for b, t in enumerate(res["table"]):
            for j, r in enumerate(res["curves"][b]):
                f.write(f"{b},{t['subkey']:02x},{j},{float(r)!r}\n")


def cmd_attack(a, curves_path=None):
    try:
        ts = IO.load_traces(a.traces, a.format)
        texts = IO.load_ciphertexts(a.ciphertexts)
    except (IO.TraceFileError, OSError) as e:
        _die(str(e))
    if ts.n != texts.shape[0]:
        _die(f"trace count {ts.n} != ciphertext count {texts.shape[0]}")
    curves_path = curves_path or a.export_curves
    try:
        res = run_attack(ts.samples, texts, MODELS[a.model], a.device, a.chunk_bytes, want_rho=bool(curves_path))
    except ValueError as e:
        _die(str(e))
    if curves_path:
        write_curves(curves_path, res)
        res.pop("curves")
    if a.json:
        print(json.dumps(res))
        return
    print(f"N = {res['n_traces']} traces x M = {res['n_samples']} samples, model {a.model}")
    print("byte  subkey  max|rho|    margin      peak_sample  peak_rho")
    for t in res["table"]:
        print(f"{t['byte']:4d}  {t['subkey']:02x}      {t['maxabs']:.6f}  {t['margin']:.6f}    "
              f"{t['peak_sample']:11d}  {t['peak_rho']:+.6f}")
    print(f"round-10 key: {res['round_key']}" if a.model != "hw_first" else f"round-0 key: {res['round_key']}")
    print(f"master key:   {res['master_key']}")


def cmd_simulate(a):
    from synth import synth as S   # the seeded input generator (no CPA arithmetic)
    try:
        key = IO.parse_key(a.key)
    except ValueError as e:
        _die(str(e))
    dt = {"s8": S.S8, "u8": S.U8, "f32": S.F32}[a.dtype]
    lo, hi = (0.5, 1.5) if dt == S.F32 else (-40, 40)
    if dt == S.U8:
        lo, hi = 88, 168
    leak = {"hd_last": S.LEAK_HD_LAST, "hw_last": S.LEAK_HW_LAST, "hw_first": S.LEAK_HW_FIRST}[a.leak]
    w = S.Workload("sim", a.n, a.m, dt, a.a, a.sigma, lo, hi, seed=a.seed, key=key, leak_model=leak)
    texts, W = S.dataset(w)
    IO.save_traces(W, a.out_prefix + ".traces")
    IO.save_ciphertexts(texts, a.out_prefix + ".ct")
    print(json.dumps({"traces": a.out_prefix + ".traces", "ciphertexts": a.out_prefix + ".ct", "n": a.n,
                      "m": a.m, "dtype": a.dtype, "leak_samples": w.leak_positions(), "key": key.hex()}))


def cmd_inspect(a):
    try:
        h = IO.read_header(a.path)
    except (IO.TraceFileError, OSError) as e:
        _die(str(e))
    print(json.dumps({"n": h["n"], "m": h["m"], "dtype": str(h["dtype"]), "precision_code": h["precision_code"],
                      "layout": h["layout"]}))


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1412_7682_b200",
                                 description="CPA on AES-128 (arXiv:1412.7682) on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def attack_args(p):
        p.add_argument("--traces", required=True)
        p.add_argument("--ciphertexts", required=True, help="hex lines (plaintexts for --model hw_first)")
        p.add_argument("--format", choices=["binary", "csv"], default=None)
        p.add_argument("--model", choices=sorted(MODELS), default="hd_last")
        p.add_argument("--device", type=int, default=0)
        p.add_argument("--chunk-bytes", type=int, default=1 << 30)
        p.add_argument("--json", action="store_true")

    p = sub.add_parser("attack")
    attack_args(p)
    p.add_argument("--export-curves", default=None, metavar="CSV")
    p = sub.add_parser("export-curves")
    attack_args(p)
    p.add_argument("--out", required=True)
    p = sub.add_parser("simulate")
    p.add_argument("--key", required=True)
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--m", type=int, required=True)
    p.add_argument("--a", type=float, default=5.0, help="leak amplitude")
    p.add_argument("--sigma", type=float, default=16.0, help="Gaussian noise sigma")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--dtype", choices=["s8", "u8", "f32"], default="s8")
    p.add_argument("--leak", choices=sorted(MODELS), default="hd_last",
                   help="leakage planted (hw_first writes plaintexts to the .ct file)")
    p.add_argument("--out-prefix", required=True)
    p = sub.add_parser("inspect")
    p.add_argument("path")
    a = ap.parse_args(argv)
    if a.cmd == "attack":
        cmd_attack(a)
    elif a.cmd == "export-curves":
        cmd_attack(a, curves_path=a.out)
    elif a.cmd == "simulate":
        cmd_simulate(a)
    else:
        cmd_inspect(a)


if __name__ == "__main__":
    main()
