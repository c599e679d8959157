"""Trace / ciphertext files and the command line (SPEC
trace_model examples [S:138-165] and cli examples [S:409-438]).  CPU tests:
formats, errors, simulate / inspect; GPU tests: attack and export-curves."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1412_7682_b200 import traceio as IO
from tests.conftest import ROOT


def test_binary_smallest_round_trip(tmp_path):
    a = np.arange(6, dtype=np.float64).reshape(2, 3)            # [S:142]
    p = str(tmp_path / "t.cpa1")
    IO.save_traces(a, p)
    assert os.path.getsize(p) == 16 + 6 * 8
    h = IO.read_header(p)
    assert (h["n"], h["m"], h["dtype"], h["layout"]) == (2, 3, np.float64, "trace-major")
    assert np.array_equal(IO.load_traces(p).samples, a)


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.int8, np.uint8])
@pytest.mark.parametrize("layout", ["trace-major", "sample-major"])
def test_binary_round_trip_bit_exact(tmp_path, dt, layout):
    rng = np.random.default_rng(3)
    a = (rng.normal(size=(10, 10)) * 50).astype(dt) if np.dtype(dt).kind == "f" else \
        rng.integers(np.iinfo(dt).min, np.iinfo(dt).max, (10, 10), endpoint=True).astype(dt)
    p = str(tmp_path / "t.cpa1")
    IO.save_traces(a, p, layout=layout)
    b = IO.load_traces(p).samples
    assert b.dtype == a.dtype and np.array_equal(b.view(np.uint8), np.ascontiguousarray(a).view(np.uint8))


def test_sample_major_storage_order(tmp_path):
    a = np.arange(1, 7, dtype=np.float32).reshape(2, 3)        # [S:160]
    p = str(tmp_path / "t.cpa1")
    IO.save_traces(a, p, layout="sample-major")
    raw = np.fromfile(p, dtype=np.float32, offset=16)
    assert raw.tolist() == [1, 4, 2, 5, 3, 6]
    assert np.array_equal(IO.load_traces(p).samples, a)


def test_binary_errors(tmp_path):
    p = str(tmp_path / "t.cpa1")
    IO.save_traces(np.ones((2, 3), np.float64), p)
    data = open(p, "rb").read()
    open(p, "wb").write(data[:-8])                                # one value short [S:143]
    with pytest.raises(IO.TraceFileError, match="length mismatch"):
        IO.load_traces(p)
    open(p, "wb").write(b"CPA2" + data[4:])
    with pytest.raises(IO.TraceFileError, match="magic"):
        IO.load_traces(p)
    open(p, "wb").write(data[:5])
    with pytest.raises(IO.TraceFileError, match="truncated"):
        IO.load_traces(p)
    bad = np.ones((2, 3), np.float32)
    bad[1, 2] = np.nan
    IO.save_traces(bad, p)
    with pytest.raises(IO.TraceFileError, match="non-finite sample in trace 1"):
        IO.load_traces(p)
    with pytest.raises(OSError):
        IO.load_traces(str(tmp_path / "missing.cpa1"))


def test_csv_fixture_and_round_trip(tmp_path):
    p = str(tmp_path / "t.csv")
    with open(p, "w") as f:                                       # 4 x 5 fixture [S:144]
        for i in range(4):
            f.write(",".join(str(10 * i + j) for j in range(5)) + "\n")
    ts = IO.load_traces(p, dtype=np.int8)
    assert (ts.n, ts.m) == (4, 5) and ts.samples[3, 4] == 34 and ts.samples.dtype == np.int8
    a = np.random.default_rng(0).normal(size=(3, 7))
    IO.save_traces(a, p, fmt="csv")
    assert np.array_equal(IO.load_traces(p, dtype=np.float64).samples, a)   # shortest repr: exact
    with open(p, "w") as f:
        f.write("1,2,3\n4,5\n")
    with pytest.raises(IO.TraceFileError, match="different sample counts"):
        IO.load_traces(p)
    with open(p, "w") as f:
        f.write("1,300\n")
    with pytest.raises(IO.TraceFileError, match="do not fit"):
        IO.load_traces(p, dtype=np.int8)


def test_ciphertext_lines(tmp_path):
    p = str(tmp_path / "c.ct")
    open(p, "w").write("0" * 32 + "\n")                           # [S:151]
    assert IO.load_ciphertexts(p).tolist() == [[0] * 16]
    t = np.random.default_rng(1).integers(0, 256, (3, 16), dtype=np.uint8)
    IO.save_ciphertexts(t, p)
    assert np.array_equal(IO.load_ciphertexts(p), t)
    open(p, "w").write("0" * 31 + "\n")                           # [S:152]
    with pytest.raises(IO.TraceFileError, match="wrong line length"):
        IO.load_ciphertexts(p)
    open(p, "w").write("zz" * 16 + "\n")
    with pytest.raises(IO.TraceFileError, match="bad hex"):
        IO.load_ciphertexts(p)


def _cli(*args, check=True):
    r = subprocess.run([sys.executable, "-m", "paper_1412_7682_b200", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stderr[-2000:]
    return r


def test_cli_simulate_inspect_deterministic(tmp_path):
    key = "2b7e151628aed2a6abf7158809cf4f3c"
    for d in ("a", "b"):
        _cli("simulate", "--key", key, "--n", "10", "--m", "16", "--seed", "7",
             "--out-prefix", str(tmp_path / d))
    assert os.path.getsize(tmp_path / "a.traces") == 16 + 10 * 16                 # int8 samples
    assert open(tmp_path / "a.traces", "rb").read() == open(tmp_path / "b.traces", "rb").read()
    assert open(tmp_path / "a.ct").read() == open(tmp_path / "b.ct").read()
    info = json.loads(_cli("inspect", str(tmp_path / "a.traces")).stdout)
    assert (info["n"], info["m"], info["dtype"], info["layout"]) == (10, 16, "int8", "trace-major")
    _cli("simulate", "--key", key, "--n", "4", "--m", "8", "--dtype", "f32", "--out-prefix", str(tmp_path / "f"))
    assert os.path.getsize(tmp_path / "f.traces") == 16 + 4 * 8 * 4


def test_cli_errors(tmp_path):
    r = _cli("simulate", "--key", "0" * 31, "--n", "2", "--m", "2", "--out-prefix", str(tmp_path / "x"),
             check=False)
    assert r.returncode != 0 and "32 hex" in r.stderr
    r = _cli("inspect", str(tmp_path / "nope"), check=False)
    assert r.returncode != 0 and "error" in r.stderr
    r = _cli("attack", "--traces", "x", check=False)               # missing required flag
    assert r.returncode != 0 and "usage" in r.stderr
    IO.save_traces(np.zeros((3, 4), np.int8), str(tmp_path / "t.cpa1"))
    IO.save_ciphertexts(np.zeros((2, 16), np.uint8), str(tmp_path / "t.ct"))
    r = _cli("attack", "--traces", str(tmp_path / "t.cpa1"), "--ciphertexts", str(tmp_path / "t.ct"), check=False)
    assert r.returncode != 0 and "3" in r.stderr and "2" in r.stderr   # both counts named [S:412]


@pytest.mark.gpu
def test_cli_attack_recovers_key_and_exports_curves(tmp_path):
    key = "000102030405060708090a0b0c0d0e0f"
    _cli("simulate", "--key", key, "--n", "500", "--m", "500", "--a", "1", "--sigma", "0",
         "--out-prefix", str(tmp_path / "s"))                      # noiseless [S:331]
    out = _cli("attack", "--traces", str(tmp_path / "s.traces"), "--ciphertexts", str(tmp_path / "s.ct"),
               "--json", "--export-curves", str(tmp_path / "c.csv")).stdout
    res = json.loads(out)
    assert res["master_key"] == key
    leaks = [((b + 1) * 500) // 17 for b in range(16)]
    assert [t["peak_sample"] for t in res["table"]] == leaks
    rows = [l.split(",") for l in open(tmp_path / "c.csv").read().splitlines()[1:]]
    assert len(rows) == 16 * 500                                   # m rows per byte [S:438]
    for b in range(16):
        curve = [float(r[3]) for r in rows if int(r[0]) == b]
        assert abs(curve[leaks[b]] - 1.0) <= 1e-9 and max(abs(c) for c in curve) <= 1.0
    text = _cli("attack", "--traces", str(tmp_path / "s.traces"), "--ciphertexts", str(tmp_path / "s.ct")).stdout
    assert f"master key:   {key}" in text


@pytest.mark.gpu
def test_cli_attack_float_and_csv(tmp_path):
    key = "2b7e151628aed2a6abf7158809cf4f3c"
    _cli("simulate", "--key", key, "--n", "2000", "--m", "64", "--dtype", "f32", "--a", "0.05", "--sigma", "0.02",
         "--out-prefix", str(tmp_path / "f"))
    res = json.loads(_cli("attack", "--traces", str(tmp_path / "f.traces"), "--ciphertexts", str(tmp_path / "f.ct"),
                          "--json").stdout)
    assert res["master_key"] == key
    IO.save_traces(np.ones((2000, 40), np.int8), str(tmp_path / "c.csv"), fmt="csv")
    r = _cli("attack", "--traces", str(tmp_path / "c.csv"), "--ciphertexts", str(tmp_path / "f.ct"), "--json")
    assert all(t["maxabs"] == 0.0 for t in json.loads(r.stdout)["table"])   # constant columns -> rho = 0 [S:250]
