"""bench.py's contract on a real GPU: the JSON line of a single-GPU run, and the
multi-rank path (sharding, all-reduce, max-over-ranks timing, one line from
rank 0) run as 2 ranks on one GPU over gloo (the production path is NCCL with
one GPU per rank; the driver's scaling run exercises that)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches"}


def _run(cmd, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_single_gpu_line():
    d = _run([sys.executable, "bench.py", "--config", "C2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["key_recovered"] is True
    assert d["gpu_launches"] > 0 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1.5 and r["unit"] == "TFLOP/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 2000 * (5000 + 16) and d["e2e"]["key_recovered"] is True


@pytest.mark.gpu
@pytest.mark.parametrize("combine,port", [("rows", 29533), ("allreduce", 29535), ("fused", 29538)])
def test_bench_two_ranks_one_gpu_gloo(combine, port):
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--config", "C2",
              "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--combine", combine],
             env={"CPA_BENCH_SAME_DEVICE": "1", "CPA_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["key_recovered"] is True
    assert KEYS <= set(d) and combine in d["config"]["parallelism"]
    assert "unavailable" not in d["config"]["parallelism"]   # fused: CUDA IPC between the ranks worked
    cm = d["combine_ms_per_step"]   # every combine timed in the same invocation
    assert set(cm) == {"rows", "allreduce", "fused"} and all(isinstance(v, float) for v in cm.values()), cm


@pytest.mark.gpu
def test_bench_stream_two_ranks_one_gpu_gloo():
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", "29534", "bench.py", "--gpus", "2", "--config", "C1",
              "--chunk", "64", "--steps", "3", "--warmup", "3", "--no-clocks"],
             env={"CPA_BENCH_SAME_DEVICE": "1", "CPA_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["key_recovered"] is True
    pts = d["rank_curve"]["points"]
    assert pts[-1][0] == 500 and d["config"]["checkpoints"] == len(pts)
    assert "reduce-scatter checkpoints" in d["config"]["parallelism"]   # the default (north_star's NCCL combine)
    cm = d["combine_ms_per_step"]   # and the fused one (rows routed to their owner by CUDA IPC), same run
    assert isinstance(cm["rows"], float) and isinstance(cm["fused"], float), cm


@pytest.mark.gpu
@pytest.mark.parametrize("config,port", [("C2", 29536), ("W48", 29537)])
def test_bench_sample_shards_two_ranks_one_gpu_gloo(config, port):
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--config", config,
              "--shard", "samples", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"],
             env={"CPA_BENCH_SAME_DEVICE": "1", "CPA_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["key_recovered"] is True
    assert d["config"]["parallelism"].startswith("sample-shard x2")


@pytest.mark.gpu
@pytest.mark.parametrize("combine,port", [("rows", 29541), ("allreduce", 29542)])
def test_bench_float_two_ranks_one_gpu_gloo(combine, port):
    """north_star config 3 at 2 GPUs (C3, float traces): rank 0's offsets are
    shared before the first accumulate (multigpu.share_offsets), the combined
    sums recover the key; the line says float."""
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--config", "C3",
              "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--combine", combine],
             env={"CPA_BENCH_SAME_DEVICE": "1", "CPA_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["key_recovered"] is True
    assert combine in d["config"]["parallelism"] and "float32" in d["config"]["workload"]


@pytest.mark.gpu
@pytest.mark.parametrize("combine,port", [("rows", 29543), ("allreduce", 29544)])
def test_bench_two_ranks_narrow_flush_before_combine(combine, port):
    """--narrow 1 with an accumulator combine: every rank flushes its int32
    shadow (CPA_OPT_NARROW) into the int64 accumulator before the NCCL / gloo
    combine reads it; the key and the line are as without the option."""
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--config", "C2",
              "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--combine", combine,
              "--narrow", "1", "--no-combine-sweep"],
             env={"CPA_BENCH_SAME_DEVICE": "1", "CPA_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["key_recovered"] is True
    assert d["config"]["sum_hw"].startswith("int32 shadow")


@pytest.mark.gpu
def test_bench_stream_two_ranks_narrow():
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", "29545", "bench.py", "--gpus", "2", "--config", "C1",
              "--chunk", "64", "--steps", "3", "--warmup", "3", "--no-clocks", "--narrow", "1", "--no-combine-sweep"],
             env={"CPA_BENCH_SAME_DEVICE": "1", "CPA_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["key_recovered"] is True
    assert d["config"]["sum_hw"].startswith("int32 shadow")
    assert d["rank_curve"]["points"][-1][0] == 500
