"""The C-ABI library loads and exports every symbol include/cpa.h declares;
host-only helpers and layout arithmetic (no GPU needed)."""
import ctypes
import os
import re

import pytest

from tests.conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "cpa.h")).read()
    return sorted(set(re.findall(r"CPA_API\s+[\w\s\*]*?\b(cpa_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import paper_1412_7682_b200 as P
    syms = header_symbols()
    assert len(syms) >= 16
    lib = ctypes.CDLL(P._binding.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(P._binding.ABI_SYMBOLS) == syms


def test_library_is_sm100a():
    import subprocess
    import paper_1412_7682_b200 as P
    out = subprocess.run(["cuobjdump", "--list-elf", P._binding.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", P._binding.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass and "UTMALDG" in sass  # tcgen05.mma kind::i8 + TMA


def test_host_key_schedule_helpers(fips):
    import paper_1412_7682_b200 as P
    rk = P.cpa_aes_expand_key(fips["a1_key"])
    assert rk[0] == fips["a1_key"] and rk[10] == fips["a1_rk10"]
    assert P.cpa_aes_expand_key(fips["c1_key"])[10] == fips["c1_rk10"]
    assert P.cpa_aes_invert_key_schedule(fips["a1_rk10"]) == fips["a1_key"]
    assert P.cpa_aes_invert_key_schedule(fips["c1_rk10"], 10) == fips["c1_key"]
    assert P.cpa_aes_invert_key_schedule(rk[4], 4) == fips["a1_key"]


def test_accumulator_layout():
    import paper_1412_7682_b200 as P
    for M in (1, 500, 5000):
        assert P.cpa_accum_words(M) == 4098 * M + 8193
        assert P.cpa_accum_bytes(M) == 8 * P.cpa_accum_words(M)
        offs = [P.cpa_accum_offset(M, f) for f in range(6)]
        assert offs == [0, 4096 * M, 4097 * M, 4098 * M, 4098 * M + 4096, 4098 * M + 8192]


def test_status_strings_and_no_gpu_error():
    import paper_1412_7682_b200 as P
    assert P.cpa_status_str(0) == "CPA_OK"
    assert P.cpa_status_str(6) == "CPA_E_OVERFLOW"
    with pytest.raises(P.CpaError):
        P.cpa_init(0, P.CPA_S8, P.CPA_HD_LAST, 0, 0, 0)  # invalid M, no GPU needed
