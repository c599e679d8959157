#!/usr/bin/env python
"""bench.py -- the BASELINE.json metric on B200: hypothesis x sample
correlations per second at 1.5M traces (workload C4: 1.5M x 5000 int8
traces, HD last-round model), plus time-to-key end to end.

One step = the whole hot path over the workload: cpa_reset -> cpa_accumulate
(a3 model sums, a4 trace moments, a5 tcgen05 cross term) -> [N>1: one NCCL
all-reduce of the packed int64 accumulator (a7)] -> cpa_finalize (a8 Eq. (1)
rho [4096][M] in fp64 + max/argmax, a9 ranking, key D2H).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Traces are sharded over ranks (strong scaling, fixed 1.5M total).  Inputs
(7.5 GB) exceed L2 (126 MB), so no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
INT8_PER_BF16 = 4.5 / 2.25  # nominal dense int8 : bf16 ratio (B200_PROFILING.md)
MODEL_NAMES = ("HD last-round", "HW last-round", "HW first-round")
# tcgen05 MAC/clk/SM (tools/pair_bench: kind::i8 8192, kind::f16 4096, both measured 100% reachable)
MMA_MACS_PER_CLK_SM = {False: 8192, True: 4096}
# float path: per multiply-add of the contraction, one kind::f16 MAC (fp16 hi) and
# one kind::f8f6f4 MAC (e4m3 lo) at twice the f16 rate = 1.5 f16-MAC equivalents
F32_EXEC = 1.5
OVERLAP_DEFAULT = 3   # CPA_OPT_OVERLAP: a4 fused into the cross-term kernel (int8 traces)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-phase-times", action="store_true",
                    help="no per-launch CUDA events inside the timed steps (the phase split and the "
                         "roofline's kernel time are then unavailable)")
    ap.add_argument("--combine", choices=["auto", "fused", "rows", "allreduce"], default="auto",
                    help="N>1 trace shards: 'fused' = the cross-term kernel adds each key byte's rows "
                         "into the owner rank's accumulator over NVLink (cpa_set_row_owners), then "
                         "an all-reduce of the small fields, row-sharded finalize, gather of the "
                         "maxima; 'rows' = the same with an NCCL reduce-scatter of the rows after "
                         "the kernel; 'allreduce' = one all-reduce of the whole accumulator, "
                         "finalize on every rank; 'auto' = rows (north_star's NCCL combine); the "
                         "others are timed after it in the same run (combine_ms_per_step)")
    ap.add_argument("--no-combine-sweep", action="store_true",
                    help="N>1 trace shards: skip timing the other combines after the headline one")
    ap.add_argument("--shard", choices=["auto", "traces", "samples"], default="auto",
                    help="N>1: split the traces (partial sums combined per --combine) or the sample "
                         "columns (every rank all traces of M/G columns; only the per-hypothesis maxima "
                         "are exchanged).  auto: samples for the wide-trace W48 workload, else traces")
    ap.add_argument("--no-overlap", action="store_true",
                    help="serialise the a4 moments pass with the cross term")
    ap.add_argument("--overlap-mode", type=int, default=None, choices=[0, 1, 2, 3],
                    help="CPA_OPT_OVERLAP (include/cpa.h); default: the library's")
    ap.add_argument("--class-sums", choices=["0", "1"], default="0",
                    help="CPA_OPT_CLASS_SUMS=1: class-sum cross term for HW_LAST/HW_FIRST workloads "
                         "(C4-HW); default: the tensor-core contraction (faster on B200, DESIGN.md)")
    ap.add_argument("--fuse-hist", choices=["0", "1"], default="0",
                    help="CPA_OPT_FUSE_HIST: a3's byte-pair histogram counted inside the cross-term kernel")
    ap.add_argument("--xt-tiles", type=int, default=0, choices=[0, 1, 2],
                    help="CPA_OPT_XT_TILES: int8 cross-term variant (0 = the library's cost model, 1 = two "
                         "sample tiles per unit, 2 = one tile with the spill overlapped)")
    ap.add_argument("--kchunk", type=int, default=0,
                    help="CPA_OPT_KCHUNK: traces per cross-term work unit (0 = the library's model)")
    ap.add_argument("--spill", type=int, default=0, choices=[0, 1, 2, 3],
                    help="CPA_OPT_SPILL: cross-term spill, 0 = auto (default), 1 = red.add per "
                         "element, 2 = bulk tensor reduce-add, 3 = per-chunk partial stores + one reduce pass")
    ap.add_argument("--narrow", choices=["auto", "0", "1"], default="auto",
                    help="CPA_OPT_NARROW: int8 cross-term sums in an int32 shadow while exact (half the "
                         "sum_hw bytes); auto = on for one rank / sample shards (no accumulator combine)")
    ap.add_argument("--chunk", type=int, default=0,
                    help="stream the traces in chunks of this many, finalizing after every round "
                         "(key-rank curve); default for C5: 65536")
    return ap.parse_args()


def metric_name(w) -> str:
    """BASELINE.json's metric (quoted at N = 1.5M traces: C4, C5); other
    configs state their own N."""
    at = "1.5M" if w.n == 1_500_000 else f"{w.n}"
    return f"hypothesis x sample correlations/s at {at} traces"


DATASHEET_TOPS = {False: 4500.0, True: 2250.0}   # B200 dense int8 / fp16-bf16 (B200_PROFILING.md)


def cublaslt_peak_tops(dev, int8: bool = True, n: int = 8192, reps: int = 5) -> float:
    """The library GEMM on this GPU, measured in this run: cuBLASLt int8
    (torch._int_mm, int32 out) or bf16 (torch.matmul) at n^3, best of `reps`
    after a warm-up (2 n^3 ops each).  A reference point for the roofline of
    the cross term, not part of the path."""
    import torch
    if int8:
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t()
        fn = lambda: torch._int_mm(a, b)  # noqa: E731
    else:
        a = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
        fn = lambda: torch.matmul(a, a)  # noqa: E731
    for _ in range(2):
        fn()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return dict(PEAK_FALLBACK), "fallback"


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, enabled: bool = True):
        self.enabled = enabled
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        if self.enabled:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                     "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
            except OSError:
                self.proc = None
            time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.proc:
            return None
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3] not in ("[N/A]",))}


# ---------------------------------------------------------- cpu baseline ----
# SURVEY 8d's CPU protocol: the oracle as it stands, single-threaded, on the 16
# leak samples + 48 seeded random columns of the workload (all columns for the
# small configs C1/C2), on the first CPU_SAMPLE_TRACES traces (bounded: ~5 s
# per run on a Xeon core).  Its cost is t(c) = a + b c per run (a: the per-trace
# Phase-1 / selection work, shared by all columns; b: per column), so it is also
# timed on the 16 leak columns alone, and the time of the FULL workload (all M
# columns, all N traces) is extrapolated as (a + b M) N / n -- stated as such.
CPU_SAMPLE_TRACES = 16384
CPU_COLS_RANDOM = 48
CPU_FULL_MAX_CELLS = 2000 * 5000   # C1, C2: the oracle runs on the whole workload


def oracle_columns(w, n_random=CPU_COLS_RANDOM, seed=1412):
    """The 16 leak samples + n_random seeded distinct other columns (sorted)."""
    import numpy as np
    lp = sorted(set(w.leak_positions()))
    rest = np.setdiff1d(np.arange(w.m), lp)
    rnd = np.random.default_rng(seed).choice(rest, min(n_random, len(rest)), replace=False)
    return np.array(sorted(lp + rnd.tolist()), np.int32), np.array(lp, np.int32)


def oracle_attack(O, texts, Ws, model=0):
    """The oracle's Phases 1-4 on the sampled columns (int or float traces)."""
    import numpy as np
    if Ws.dtype == np.float32:
        sh, sh2 = O.model_sums(model, texts)
        shw, sw, sw2 = O.sums_f32(model, texts, Ws)
        rho = O.rho_eq1_f64_grid(Ws.shape[0], shw, sh, sh2, sw, sw2)
        mx, am, pk = O.phase3(rho)
        best, rank = O.phase4(mx)
        return {"best": best, "argmax": am}
    return O.attack_i8(model, texts, Ws, np.arange(Ws.shape[1], dtype=np.int32))


class OracleSample:
    """A bounded sample of workload w for the oracle: texts + the chosen
    columns of the first n traces (host generator), and the timing model."""

    def __init__(self, w, n_traces=CPU_SAMPLE_TRACES):
        import numpy as np
        from synth import synth as S
        self.w = w
        self.full = w.n * w.m <= CPU_FULL_MAX_CELLS
        self.n = w.n if self.full else min(n_traces, w.n)
        self.texts, lv = S.texts(w, 0, self.n)
        if self.full:
            self.cols, self.leak = np.arange(w.m, dtype=np.int32), np.array(w.leak_positions(), np.int32)
        else:
            self.cols, self.leak = oracle_columns(w)
        self.W = S.traces(w, lv, 0, self.cols)
        lidx = np.searchsorted(self.cols, self.leak)
        self.W16 = np.ascontiguousarray(self.W[:, lidx])
        self.describe = (f"all {w.m} columns x all {w.n} traces of {w.name} (measured, no extrapolation)"
                         if self.full else
                         f"{len(self.cols)} columns (the 16 leak samples + {len(self.cols) - 16} seeded random) x "
                         f"first {self.n} traces of {w.name}; also timed on the 16 leak columns alone to split "
                         f"the per-trace cost a from the per-column cost b; full step (all {w.m} columns, "
                         f"{w.n} traces) extrapolated as (a + b*{w.m}) x {w.n / self.n:.2f}")

    def run(self, leak_only=False):
        """(seconds, key bytes ranked first) of one oracle pass over the sample."""
        from oracle import oracle as O
        W = self.W16 if leak_only else self.W
        t0 = time.perf_counter()
        a = oracle_attack(O, self.texts, W, self.w.leak_model)
        t = time.perf_counter() - t0
        return t, int(sum(a["best"] == O.expand_key(self.w.key)[10]))

    def full_step_seconds(self, t_all, t_leak):
        """Extrapolated seconds of one oracle pass over the whole workload."""
        if self.full:
            return t_all
        c = len(self.cols)
        b = max(0.0, (t_all - t_leak) / (c - 16))
        a = max(0.0, t_all - b * c)
        return (a + b * self.w.m) * (self.w.n / self.n)


def cpu_baseline(w, repeats=None):
    """The oracle as it stands (single-threaded C, oracle/oracle.c) on the
    bounded sample; rate = 4096 M / (extrapolated full-step time)."""
    smp = OracleSample(w)
    reps = repeats or (3 if smp.full and w.n * w.m <= 500 * 500 else 1)
    ts, ok = [], 0
    for _ in range(reps):
        t, ok = smp.run()
        ts.append(t)
    t_all = statistics.median(ts)
    t_leak = t_all if smp.full else smp.run(leak_only=True)[0]
    t_full = smp.full_step_seconds(t_all, t_leak)
    return {"value": 4096 * w.m / t_full, "unit": "correlations/s", "cores": 1, "kind": "oracle",
            "sample": smp.describe, "sample_columns": len(smp.cols), "sample_traces": smp.n,
            "seconds_sample": t_all, "seconds_leak_columns": t_leak, "repeats": reps,
            "full_step_seconds": t_full, "extrapolated": not smp.full, "key_bytes_ranked_first": ok,
            "rate_on_sample_columns": 4096 * len(smp.cols) / (t_all * w.n / smp.n)}


def host_cpu_info():
    """CPU model and socket count of this host (for the all-cores baseline)."""
    info = {"model": None, "sockets": None, "logical_cpus": os.cpu_count()}
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in txt.splitlines():
            k, _, v = line.partition(":")
            if k.strip() == "Model name":
                info["model"] = v.strip()
            elif k.strip() == "Socket(s)":
                info["sockets"] = int(v.strip()) if v.strip().isdigit() else v.strip()
    except Exception:  # noqa: BLE001
        pass
    return info


def cpu_baseline_all_cores(w):
    """SURVEY 8d's all-cores CPU baseline (the paper's multi-threaded server
    comparison [P:164]): the oracle's own Phase 1-2 functions (single-threaded
    C that releases the GIL) over one contiguous block of the sample's traces
    per host thread -- every thread does a whole pass over its traces, like the
    serial oracle -- the exact partial sums added, then Phases 3-4.  Same
    sample and the same full-step extrapolation as cpu_baseline."""
    import concurrent.futures as cf
    import numpy as np
    from oracle import oracle as O
    smp = OracleSample(w)
    threads = max(1, min(len(os.sched_getaffinity(0)), 128))
    is_f32 = smp.W.dtype == np.float32
    model = w.leak_model

    def one_pass(W):
        bl = [(smp.n * t // threads, smp.n * (t + 1) // threads) for t in range(threads)]
        bl = [(i0, i1) for i0, i1 in bl if i1 > i0]

        def phase12(r):
            i0, i1 = r
            tx, Wb = smp.texts[i0:i1], np.ascontiguousarray(W[i0:i1])
            sh, sh2 = O.model_sums(model, tx)
            if is_f32:
                shw, sw, sw2 = O.sums_f32(model, tx, Wb)
            else:
                sw, sw2 = O.trace_sums_i8(Wb)
                shw = O.cross_sums_i8(model, tx, Wb)
            return sh, sh2, shw, sw, sw2

        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(max_workers=len(bl)) as ex:
            parts = list(ex.map(phase12, bl))
        sh, sh2, shw, sw, sw2 = (sum(p[k] for p in parts) for k in range(5))
        rho = (O.rho_eq1_f64_grid if is_f32 else O.rho_eq1_grid)(smp.n, shw, sh, sh2, sw, sw2)
        mx, _, _ = O.phase3(rho)
        best, _ = O.phase4(mx)
        return time.perf_counter() - t0, int(sum(np.asarray(best) == O.expand_key(w.key)[10]))

    t_all, ok = one_pass(smp.W)
    t_leak = t_all if smp.full else one_pass(smp.W16)[0]
    t_full = smp.full_step_seconds(t_all, t_leak)
    return {"value": 4096 * w.m / t_full, "unit": "correlations/s", "cores": threads,
            "kind": "oracle, Phases 1-2 over one trace block per host thread (exact partial sums added)",
            "sample": smp.describe, "seconds_sample": t_all, "seconds_leak_columns": t_leak,
            "full_step_seconds": t_full, "extrapolated": not smp.full, "host": host_cpu_info(),
            "key_bytes_ranked_first": ok}


def run_reference(args, w):
    """--impl reference: the oracle on the host cores (single thread), one
    bounded sample of the workload per step (OracleSample).  ms_per_step is the
    MEASURED time of the sample step; value is the metric at the workload's
    full size, from the extrapolated full-step time (the 16-leak-column pass
    that splits the cost is timed once, with the warm-up)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    smp = OracleSample(w)
    t_leak = None
    ts = []
    ok = 0
    for s in range(args.warmup + args.steps):
        t, ok = smp.run()
        if s >= args.warmup:
            ts.append(t)
        elif s == 0 and not smp.full:
            t_leak = smp.run(leak_only=True)[0]
    t = statistics.mean(ts)
    t_full = smp.full_step_seconds(t, t_leak if t_leak is not None else t)
    val = 4096 * w.m / t_full
    line = {"metric": metric_name(w), "impl": "reference", "value": val,
            "unit": "correlations/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if w.dtype == 2 else "int64", "data": "synthetic",
            "config": {"workload": f"{w.name}: {w.n} traces x {w.m} samples "
                                   f"{'float32' if w.dtype == 2 else 'int8'}, {MODEL_NAMES[w.leak_model]} model",
                       "n_traces": w.n, "n_samples": w.m},
            "step": f"one oracle pass (Phases 1-4) over the sample: {smp.describe}",
            "extrapolation": {"full_step_ms": t_full * 1e3, "sample_step_ms": t * 1e3,
                              "leak_columns_ms": (t_leak or t) * 1e3, "extrapolated": not smp.full},
            "key_bytes_ranked_first_on_sample": ok,
            "cpu_baseline": {"value": val, "unit": "correlations/s", "cores": 1, "kind": "oracle",
                             "sample": smp.describe},
            "e2e": {"value": val, "unit": "correlations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours ----
def main():
    args = parse()
    from synth import synth as S
    w = S.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, w)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks (tests/test_bench_gpu.py): run a multi-rank bench on ONE GPU with
    # every rank on cuda:0 over gloo.  Production runs use NCCL, one GPU per rank.
    if os.environ.get("CPA_BENCH_SAME_DEVICE") == "1":
        local = 0
    backend = os.environ.get("CPA_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_1412_7682_b200 as P

    from paper_1412_7682_b200 import multigpu as MG
    from paper_1412_7682_b200.multigpu import shard_range
    dev = torch.device("cuda", local)
    if args.chunk or w.name == "C5":
        return run_stream(args, w, dev, world, rank, local)
    shard = args.shard if args.shard != "auto" else ("samples" if w.name == "W48" else "traces")
    if world == 1:
        shard = "traces"
    if shard == "samples":      # all traces, this rank's columns [j0, j1) (16-aligned)
        i0, i1 = 0, w.n
        j0, j1 = MG.column_range(w.m, rank, world)
        assert j1 > j0, f"M={w.m} too small for {world} column shards"
    else:
        i0, i1 = shard_range(w.n, rank, world)
        j0, j1 = 0, w.m
    n_local, m_local = i1 - i0, j1 - j0
    # ---- inputs: texts + planted leakage on the host, traces generated on device
    is_f32 = w.dtype == S.F32
    tdt = torch.float32 if is_f32 else torch.int8
    texts, lv = S.texts(w, i0, n_local)
    ld = (w.m + 3) // 4 * 4 if is_f32 else (w.m + 15) // 16 * 16  # 16-byte rows for TMA
    dW = torch.empty((n_local, ld), dtype=tdt, device=dev)
    dT = torch.from_numpy(texts).to(dev)
    S.dev_traces(w, torch.from_numpy(lv).to(dev), i0, n_local, dW, ld)
    dWv = dW[:, j0:j1]
    torch.cuda.synchronize()

    eng = P.Engine(m_local, P.CPA_F32 if is_f32 else P.CPA_S8, w.leak_model, local)  # model = the leakage's
    class_sums = args.class_sums == "1" and not is_f32
    if class_sums:
        eng.set_class_sums(True)
    eng.set_fuse_hist(args.fuse_hist == "1")
    eng.set_xt_tiles(args.xt_tiles)
    if args.kchunk:
        eng.set_kchunk(args.kchunk)
    eng.set_spill(args.spill)
    eng.set_col0(j0)
    combine0 = ("columns" if shard == "samples" else args.combine) if world > 1 else "none"
    narrow = not is_f32 and not class_sums and (args.narrow == "1" or (args.narrow == "auto" and
                                                                     combine0 in ("none", "columns")))
    if narrow:
        eng.set_narrow(True)
    ovl_mode = 0 if args.no_overlap else (args.overlap_mode if args.overlap_mode is not None else OVERLAP_DEFAULT)
    eng.set_overlap(ovl_mode)
    if is_f32 and world > 1:
        # float sums are centred per sample: every rank must use the same offsets
        # (rank 0's default ones), or the combined sums mix differently-shifted data
        MG.share_offsets(eng, dWv if rank == 0 else None)
    combine = ("columns" if shard == "samples" else args.combine) if world > 1 else "none"
    fused_note = None
    if combine == "auto":   # north_star's NCCL combine: reduce-scatter of the rows (+ small-field all-reduce)
        combine = "rows"
    owners = None
    fused_ok = not is_f32 and not class_sums and 16 % world == 0

    def use_owners(on: bool):
        """Map the peers' accumulators (CUDA IPC) and route the rows to their
        owners (on), or unmap (off).  Collective.  Returns why not, or None."""
        nonlocal owners
        if on and owners is None:
            owners, why = MG.FusedOwners.try_create(eng)
            return why if owners is None else None
        if not on and owners is not None:
            barrier()
            owners.close()
            owners = None
        return None

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if combine == "fused":
        why = use_owners(True) if fused_ok else "float or class-sum path, or G does not divide 16"
        if owners is None:      # no peer mapping on this box (every rank agrees): NCCL reduce-scatter
            fused_note, combine = f"fused combine unavailable ({why}); rows", "rows"
    h0, h1 = MG.row_range(rank, world) if combine in ("rows", "fused") else (0, 4096)
    bar_t = torch.zeros(1, dtype=torch.int32, device=dev)
    rho = torch.empty((h1 - h0, m_local), dtype=torch.float64, device=dev)   # this rank's block of rho
    maxabs = torch.empty(4096, dtype=torch.float64, device=dev)
    argmax = torch.empty(4096, dtype=torch.int32, device=dev)
    peak = torch.empty(4096, dtype=torch.float64, device=dev)
    rank_t = torch.empty(4096, dtype=torch.int32, device=dev)
    stream = eng.stream

    def step(host=None):
        eng.reset()
        if combine == "fused":  # every owner's accumulator is zero before any peer adds to it
            MG.device_barrier(bar_t)
        if host is None:
            eng.accumulate(dWv, dT)
        else:
            eng.accumulate_host(*host)
        if narrow and combine in ("fused", "rows"):
            eng.flush()         # the int32 shadow into the accumulator the combine reads
        if combine == "fused":  # rows already with their owners; small fields + ordering point
            MG.allreduce_small_fields(eng.accum, w.m)
            P.cpa_finalize_rows(eng.ctx, h0, h1, rho, maxabs, argmax, peak)
            MG.gather_rows(maxabs, argmax, peak, h0, h1)
            return P.cpa_select(eng.ctx, 1, maxabs, argmax, peak, rank_t)
        if combine == "rows":   # reduce-scatter rows, sharded Eq. (1), gather maxima, select
            MG.reduce_scatter_rows(eng.accum, w.m)
            P.cpa_finalize_rows(eng.ctx, h0, h1, rho, maxabs, argmax, peak)
            MG.gather_rows(maxabs, argmax, peak, h0, h1)
            return P.cpa_select(eng.ctx, 1, maxabs, argmax, peak, rank_t)
        if combine == "columns":    # local Eq. (1) over this rank's columns, gather maxima, merge
            P.cpa_finalize_rows(eng.ctx, 0, 4096, rho, maxabs, argmax, peak)
            return P.cpa_select(eng.ctx, world, *MG.gather_shards(maxabs, argmax, peak), rank_t)
        if combine == "allreduce":
            eng.allreduce(check_offsets=False)   # float: checked once before the timed steps
        return P.cpa_finalize(eng.ctx, rho, maxabs, argmax, rank_t)

    def timed_steps(k):
        """k steps between a barrier + synchronize on both sides, CUDA events on
        the library's stream; the max over ranks (ms)."""
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            r = step()
        e1.record(stream)
        barrier()
        t = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t, r

    for _ in range(args.warmup):
        res = step()
    if is_f32 and world > 1 and shard == "traces":
        MG.check_same_offsets(eng)   # every rank's sums centred on the same offsets
    eng.set_timing(not args.no_phase_times)
    eng.phase_times()  # clear
    barrier()
    launches0 = eng.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, not args.no_clocks) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res = step()
        ev1.record(stream)
        barrier()
    ms_total = ev0.elapsed_time(ev1)
    launches = eng.launches - launches0
    phase_ms, phase_n = eng.phase_times()
    eng.set_timing(False)
    xt_mhz = P.cpa_xterm_clock(eng.ctx)   # SM clock of the last timed cross-term launch (in-kernel probe)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    # N>1 trace shards: every other combine timed in the same invocation (the
    # headline is `combine`), so one multi-GPU run compares them directly
    combine_ms = None
    if world > 1 and shard == "traces" and not args.no_combine_sweep:
        head = (combine, h0, h1, rho)
        combine_ms = {combine: ms_total / args.steps}
        k2 = max(3, min(args.steps, 10))
        for c in ("rows", "allreduce", "fused"):
            if c == head[0]:
                continue
            if c == "fused":
                why = use_owners(True) if fused_ok else "not applicable (float / class sums / G does not divide 16)"
                if owners is None:
                    combine_ms[c] = f"unavailable: {why}"
                    continue
            else:
                use_owners(False)   # the NCCL combines: rows stay in this rank's accumulator
            combine = c
            h0, h1 = MG.row_range(rank, world) if c in ("rows", "fused") else (0, 4096)
            rho = torch.empty((h1 - h0, m_local), dtype=torch.float64, device=dev)
            for _ in range(2):
                step()
            t2, r2 = timed_steps(k2)
            # every rank holds the same result after the combine, so all take the same
            # branch here: a mismatch is recorded, never raised (a raise on some ranks
            # would leave the others waiting in a collective)
            same = bytes(r2.master_key) == bytes(res.master_key)
            combine_ms[c] = t2 / k2 if same else f"key mismatch ({t2 / k2:.3f} ms)"
        combine, h0, h1, rho = head
        if combine == "fused":
            use_owners(True)
        elif owners is not None:
            use_owners(False)
    # a4 alone: the timed steps overlap it with a5 on a low-priority side stream,
    # which hides its own HBM rate; two untimed extra steps serialise it
    solo = None
    if ovl_mode:
        eng.set_overlap(0)
        eng.set_timing(True)
        eng.phase_times()
        for _ in range(2):
            step()
        barrier()
        sm, sn = eng.phase_times()
        solo = sm["moments"] / max(1, sn["moments"])
        eng.set_timing(False)
        eng.set_overlap(ovl_mode)
    ms_step = ms_total / args.steps
    value = 4096 * w.m / (ms_step * 1e-3)
    key_ok = bytes(res.master_key) == w.key

    # ---- roofline of the dominant kernel (cross term, tensor-bound)
    peaks, src = load_peaks()
    xt_ms = phase_ms["xterm"] / max(1, phase_n["xterm"]) or float("nan")   # nan: --no-phase-times
    ops = 2.0 * 4096 * n_local * m_local   # algorithmic: one multiply-add per (h, i, j)
    achieved = ops / (xt_ms * 1e-3) / 1e12
    ratio = 1.0 if is_f32 else INT8_PER_BF16
    # the burst figure: the measured sustained bf16 one (a power-capped cuBLAS
    # run) is below what this int8 kernel sustains, so it cannot be a ceiling
    peak = peaks["bf16_tflops"] * ratio
    traffic = None
    ncu_xt = None
    tp = os.path.join(ROOT, "profiles", "xterm_traffic.json" if w.name == "C4" else f"xterm_traffic_{w.name}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        if tj.get("config") == w.name and tj.get("n_gpus", 1) == world:
            traffic = tj.get("dram_bytes_per_launch")
            ncu_xt = {k: tj.get(k) for k in ("tensor_active_pct", "sm_mhz", "duration_ms", "tag")}
    roofline = {"kernel": "k_xterm<F32>" if is_f32 else "k_xterm<I8>", "bound": "tensor", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": (f"{src} bf16_tflops (burst)" if is_f32 else
                                f"{src} bf16_tflops (burst) x {INT8_PER_BF16:g} (int8:bf16 nominal ratio)"),
                "frac_of_sustained": achieved / (peaks["bf16_tflops_sustained"] * ratio),
                "algorithmic_ops_per_launch": ops, "ms_per_launch": xt_ms}
    if xt_mhz > 0 and not class_sums:
        # the tcgen05 issue ceiling at the clock the kernel itself measured (clock64 over
        # %globaltimer in its first CTA): what the 1000 W cap left it
        ceil_k = MMA_MACS_PER_CLK_SM[is_f32] * 2 * 148 * xt_mhz * 1e6 / 1e12
        roofline["kernel_sm_mhz"] = xt_mhz
        roofline["mma_ceiling_at_kernel_clock"] = ceil_k
        roofline["frac_of_mma_ceiling_at_kernel_clock"] = (F32_EXEC * achieved if is_f32 else achieved) / ceil_k
    if ncu_xt and ncu_xt.get("sm_mhz"):
        # the same kernel under ncu: tensor-pipe activity and its own SM clock; the
        # tcgen05 issue ceiling at that clock is what the 1000 W cap allows
        ceil = MMA_MACS_PER_CLK_SM[is_f32] * 2 * 148 * ncu_xt["sm_mhz"] * 1e6 / 1e12
        roofline["ncu"] = dict(ncu_xt, mma_ceiling_at_kernel_clock=ceil,
                               frac_of_ceiling_under_ncu=ops / (ncu_xt["duration_ms"] * 1e-3) / 1e12 / ceil)
    roofline["frac_vs_datasheet"] = (F32_EXEC * achieved if is_f32 else achieved) / DATASHEET_TOPS[is_f32]
    roofline["datasheet_tops"] = DATASHEET_TOPS[is_f32]
    try:   # the library GEMM of the same precision class, measured now on this GPU
        lib = cublaslt_peak_tops(dev, int8=not is_f32)
        key = "cublaslt_bf16_tflops" if is_f32 else "cublaslt_int8_tops"
        roofline[key] = lib
        roofline["frac_vs_cublaslt"] = (F32_EXEC * achieved if is_f32 else achieved) / lib
    except Exception as ex:  # noqa: BLE001
        roofline["cublaslt_error"] = f"{type(ex).__name__}: {ex}"
    roofline["mma_rate_source"] = ("tools/pair_bench.cu + tools/mma_bench.cu: kind::i8 8192, kind::f16 4096 "
                                   "MAC/clk/SM reachable (profiles/mma_bench_r02.txt)")
    if class_sums:  # NEXT-4 path: HBM-bound by design (16 adds per trace byte), so report it as such
        gbs = n_local * m_local / (xt_ms * 1e-3) / 1e9
        roofline = {"kernel": "class sums (k_cs_sort + k_cs_sum + k_cs_contract)", "bound": "hbm",
                    "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"],
                    "traffic": None, "algorithmic_bytes_per_launch": n_local * m_local, "ms_per_launch": xt_ms,
                    "note": "each trace byte is gathered once per key byte (16x) through L2; see DESIGN.md"}
    if is_f32:
        # fp16-equivalent ops issued: the fp16 hi MMAs + the e4m3 lo MMAs at 2x rate
        roofline["executed_ops_per_launch"] = F32_EXEC * ops
        roofline["executed_frac"] = F32_EXEC * achieved / peak
    step_phase_ms = {k: v / args.steps for k, v in phase_ms.items()}
    tot = sum(step_phase_ms.values()) or 1.0
    # HBM-bound kernels: achieved GB/s on their algorithmic bytes
    mo_launch_ms = phase_ms["moments"] / max(1, phase_n["moments"])
    # (the NT = 1 cross-term variant, CPA_OPT_XT_TILES, runs a4 as its own pass)
    fused = ovl_mode == 3 and not is_f32 and not class_sums and not phase_n["moments"]
    mo_solo = solo or mo_launch_ms
    mo_bytes = n_local * m_local * (7 if is_f32 else 1)  # f32: k_split_f32 reads 4 B, writes 2 B (fp16) + 1 B (e4m3)
    hbm = {"moments_GBps": mo_bytes / (mo_solo * 1e-3) / 1e9 if mo_solo else None,
           "moments_GBps_overlapped": mo_bytes / (mo_launch_ms * 1e-3) / 1e9 if (solo and mo_launch_ms) else None,
           "moments_in_step": ("fused into k_xterm (no separate pass; moments_GBps is the unfused k_moments_i8 "
                               "measured in two extra serialised steps)") if fused else
                              ("k_split_f32 pre-pass (centring, fp16 hi + e4m3 lo planes, fp64 sums)" if is_f32
                               else "separate k_moments_i8 pass"),
           # bytes per cell: the sum_hw read (4 B narrow / 8 B) + the rho write (8 B)
           "finalize_GBps": ((h1 - h0) * m_local * (12 if narrow else 16)) / (step_phase_ms["finalize"] * 1e-3) / 1e9 if step_phase_ms["finalize"] else None,
           "hbm_peak_GBps": peaks["hbm_gbs"]}

    # ---- end to end through the public API: host (pinned) buffers -> key on host
    e2e = None
    if not args.no_e2e:
        try:
            hW = torch.empty((n_local, m_local), dtype=tdt, pin_memory=True)
            hW.copy_(dWv)
            hT = torch.from_numpy(texts).pin_memory()
            step((hW, hT))  # warm the staging buffers
            barrier()
            ts = []
            for _ in range(args.e2e_steps):
                barrier()
                t0 = time.perf_counter()
                r2 = step((hW, hT))
                barrier()
                ts.append(time.perf_counter() - t0)
            te = max(ts) if world == 1 else ts[-1]
            if world > 1:
                t = torch.tensor([statistics.mean(ts)], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                te = float(t.item())
            else:
                te = statistics.mean(ts)
            e2e = {"value": 4096 * w.m / te, "unit": "correlations/s",
                   "h2d_bytes_per_step": n_local * (m_local * hW.element_size() + 16),
                   "d2h_bytes_per_step": 8 + 32 * 4 + 16 * 8,
                   "ms_per_step": te * 1e3, "time_to_key_s": te, "key_recovered": bytes(r2.master_key) == w.key,
                   "host_buffers": "pinned"}
            del hW
        except Exception as ex:  # noqa: BLE001
            e2e = {"value": None, "unit": "correlations/s", "error": f"{type(ex).__name__}: {ex}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w)
        try:
            cpu["all_cores"] = cpu_baseline_all_cores(w)
        except Exception as ex:  # noqa: BLE001
            cpu["all_cores"] = {"error": f"{type(ex).__name__}: {ex}"}

    if rank == 0:
        line = {
            "metric": metric_name(w), "value": value,
            "unit": "correlations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f16+e4m3 (f32 traces: fp16 hi + e4m3 lo MMAs, fp32 accum, fp64 sums)" if is_f32 else "s8",
            "data": "synthetic",
            "config": {"workload": f"{w.name}: {w.n} traces x {w.m} samples "
                                   f"{'float32' if is_f32 else 'int8 (s8)'}, {MODEL_NAMES[w.leak_model]} model"
                                   f"{' (class-sum cross term)' if class_sums else ''}, "
                                   f"AES-128 key {w.key.hex()}",
                       "n_traces": w.n, "n_samples": w.m, "hypotheses": 4096, "parallelism": (f"{'sample' if shard == 'samples' else 'trace'}-shard x{world}"
                                       + (f", {combine} combine" if world > 1 else "")
                                       + (f" [{fused_note}]" if fused_note else "")),
                       "l2": f"inputs {n_local * m_local * dW.element_size() / 1e9:.2f} GB per rank > 126 MB L2, "
                             "no flush needed",
                       "rho_written": True,
                       "sum_hw": "int32 shadow (CPA_OPT_NARROW, exact)" if narrow else ("fp64" if is_f32 else "int64")},
            "key_recovered": key_ok, "gpu_launches": launches,
            "phases_ms_per_step": step_phase_ms,
            "phase_share": {k: v / tot for k, v in step_phase_ms.items()},
            "roofline": roofline, "hbm": hbm, "e2e": e2e, "cpu_baseline": cpu,
            "combine_ms_per_step": combine_ms,
            "cell_trace_macs_per_s": 4096 * w.m * w.n / (ms_step * 1e-3),
        }
        if not args.no_clocks:
            line["clocks"] = clk.summary()
            mhz = (line["clocks"] or {}).get("sm_mhz")
            if mhz:
                # tcgen05 issue-rate ceiling at the observed SM clock (tools/pair_bench:
                # kind::i8 8192, kind::f16 4096 MAC/clk/SM, both measured 100% reachable)
                macs = MMA_MACS_PER_CLK_SM[is_f32]
                ceil = 2.0 * macs * torch.cuda.get_device_properties(dev).multi_processor_count * mhz * 1e6 / 1e12
                roofline["mma_rate_ceiling_at_clock"] = ceil
                roofline["frac_of_mma_rate_ceiling"] = (roofline["executed_ops_per_launch"] if is_f32 else ops) \
                    / (xt_ms * 1e-3) / 1e12 / ceil
        print(json.dumps(line), flush=True)
    if owners is not None:
        barrier()
        owners.close()
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def run_stream(args, w, dev, world, rank, local):
    """Streamed workload (BASELINE config C5): global 64K-trace chunks, chunk
    j*G + r on rank r, and after every round a checkpoint finalize from the
    (all-reduced) sums so far -> the known-key rank curve.  One step = every
    chunk + every checkpoint (the last one writes rho)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from synth import synth as S
    import paper_1412_7682_b200 as P
    from paper_1412_7682_b200.stream import Curve, StreamingAttack, chunk_rounds

    chunk = args.chunk or 65536
    rounds = chunk_rounds(w.n, chunk, world)
    mine = [(i0, i1) for rnd in rounds for r, i0, i1 in rnd if r == rank]
    n_local = sum(i1 - i0 for i0, i1 in mine)
    ld = (w.m + 15) // 16 * 16
    dW = torch.empty((max(n_local, 1), ld), dtype=torch.int8, device=dev)
    dT = torch.empty((max(n_local, 1), 16), dtype=torch.uint8, device=dev)
    off = 0
    for i0, i1 in mine:   # traces generated on the device, chunk by chunk
        t, lv = S.texts(w, i0, i1 - i0)
        dT[off:off + i1 - i0].copy_(torch.from_numpy(t))
        S.dev_traces(w, torch.from_numpy(lv).to(dev), i0, i1 - i0, dW[off:off + i1 - i0], ld)
        off += i1 - i0
    torch.cuda.synchronize()
    rk10 = P.cpa_aes_expand_key(w.key)[10]   # the known round key (library host helper)
    key_idx = torch.tensor([256 * b + rk10[b] for b in range(16)], device=dev)
    # default (auto): reduce-scatter checkpoints (NCCL); the fused combine is
    # timed after the headline in the same run (combine_ms_per_step)
    fused = world > 1 and args.combine == "fused" and 16 % world == 0
    narrow = args.narrow == "1" or (args.narrow == "auto" and world == 1)
    st = StreamingAttack(w.m, P.CPA_S8, P.CPA_HD_LAST, local, fused=fused, narrow=narrow)
    if fused and st.owners is None:   # peers not mappable: NCCL reduce-scatter checkpoints
        print(f"fused combine unavailable ({st.fused_note}); reduce-scatter checkpoints", file=sys.stderr)
        fused = False
    stream = st.eng.stream

    # non-final checkpoints run without blocking (one GPU): their ranks land in
    # rank_buf and are read once per step; multi-GPU checkpoints block
    rank_buf = torch.empty((len(rounds), 4096), dtype=torch.int32, device=dev)

    def step():
        """One streamed pass; returns (final result, the ranks of the blocking
        checkpoints).  The non-blocking checkpoints' ranks stay in rank_buf."""
        st.reset()
        o = 0
        sync_ranks = {}
        for j, rnd in enumerate(rounds):
            for r, i0, i1 in rnd:
                if r == rank:
                    st.add(dW[o:o + i1 - i0, :w.m], dT[o:o + i1 - i0])
                    o += i1 - i0
            last = j == len(rounds) - 1
            if last or not st.checkpoint_async(rank_buf[j]):
                out = st.checkpoint(want_rho=last)
                sync_ranks[j] = out["rank"]
        return out, sync_ranks

    def read_curve(sync_ranks):
        """The key-rank curve of the last step (device reads: outside the timed region)."""
        curve = Curve()
        for j, rnd in enumerate(rounds):
            rk = sync_ranks.get(j, rank_buf[j])
            curve.add(rnd[-1][2], rk[key_idx].tolist())
        return curve

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    st.eng.set_timing(not args.no_phase_times)
    st.eng.phase_times()
    barrier()
    launches0 = st.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, not args.no_clocks) as clk:
        ev0.record(stream)
        for s_ in range(args.steps):
            out, sync_ranks = step()
        ev1.record(stream)
        barrier()
    ms_total = ev0.elapsed_time(ev1)
    curve = read_curve(sync_ranks)
    launches = st.launches - launches0
    phase_ms, phase_n = st.eng.phase_times()
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    # the other checkpoint combine, timed in the same invocation
    combine_ms = None
    if world > 1 and not args.no_combine_sweep:
        name = "fused" if fused else "rows"
        combine_ms = {name: ms_step}
        other = not fused
        if other and 16 % world:
            combine_ms["fused"] = "not applicable: G does not divide 16"
        else:
            st_main = st
            st = StreamingAttack(w.m, P.CPA_S8, P.CPA_HD_LAST, local, fused=other)
            if other and st.owners is None:
                combine_ms["fused"] = f"unavailable: {st.fused_note}"
            else:
                k2 = max(2, min(args.steps, 5))
                step()
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st.eng.stream)
                for _ in range(k2):
                    o2, _ = step()
                e1.record(st.eng.stream)
                barrier()
                t = torch.tensor([e0.elapsed_time(e1) / k2], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                combine_ms["fused" if other else "rows"] = float(t.item())
                if bytes(o2["master_key"]) != bytes(out["master_key"]):   # recorded, never raised (collectives)
                    combine_ms["fused" if other else "rows"] = f"key mismatch ({float(t.item()):.3f} ms)"
            st.close()
            st = st_main
    peaks, src = load_peaks()
    xt_ms = phase_ms["xterm"] / max(1, phase_n["xterm"]) or float("nan")   # nan: --no-phase-times
    ops = 2.0 * 4096 * n_local * w.m / max(1, phase_n["xterm"] // args.steps)  # per launch (one per chunk)
    achieved = ops / (xt_ms * 1e-3) / 1e12
    peak = peaks["bf16_tflops"] * INT8_PER_BF16
    if rank == 0:
        line = {
            "metric": metric_name(w), "value": 4096 * w.m / (ms_step * 1e-3),
            "unit": "correlations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "s8", "data": "synthetic",
            "config": {"workload": f"{w.name}: {w.n} traces x {w.m} samples int8, streamed in {chunk}-trace chunks, "
                                   f"checkpoint finalize after every round of {world}, HD last-round model",
                       "n_traces": w.n, "n_samples": w.m, "chunk": chunk, "checkpoints": len(rounds),
                       "parallelism": f"trace-chunk round-robin x{world}"
                                      + (", fused row combine" if fused else (", reduce-scatter checkpoints" if world > 1 else "")),
                       "l2": f"inputs {w.n * w.m / 1e9:.0f} GB > 126 MB L2, no flush needed",
                       "sum_hw": "int32 shadow (CPA_OPT_NARROW, exact)" if narrow else "int64"},
            "key_recovered": bytes(out["master_key"]) == w.key,
            "traces_to_key": curve.traces_to_key(),
            "rank_curve": {"columns": ["traces", "worst_rank", "bytes_at_rank_1"], "points": curve.summary()},
            "gpu_launches": launches,
            "phases_ms_per_step": {k: v / args.steps for k, v in phase_ms.items()},
            "roofline": {"kernel": "k_xterm<I8>", "bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                         "peak_source": f"{src} bf16_tflops (burst) x {INT8_PER_BF16:g}",
                         "ms_per_launch": xt_ms, "algorithmic_ops_per_launch": ops},
            "e2e": None, "cpu_baseline": None, "combine_ms_per_step": combine_ms,
        }
        if not args.no_clocks:
            line["clocks"] = clk.summary()
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
