"""Pins for the oracle's AES-128 pieces against FIPS-197 printed values
(tests/golden/fips197.txt) and exhaustive properties [S:48-103, S:463]."""
import numpy as np

from oracle import oracle as O


def test_sbox_bijection_and_spot_values(fips):
    s, inv = O.aes_tables()
    assert sorted(s.tolist()) == list(range(256))          # permutation [S:61]
    assert all(inv[s[x]] == x for x in range(256))          # round trip [S:53, S:60]
    assert s[0x00] == 0x63 and inv[0x63] == 0x00            # [S:52, S:59]
    assert s[0x53] == fips["sbox_53"][0]                    # FIPS-197 Sec. 5.1.1
    assert all(s[x] != x for x in range(256))               # AES S-box has no fixed point


def test_sbox_against_fips_round_states(fips):
    s, _ = O.aes_tables()
    for start, sb in (("b_r1_start", "b_r1_sbox"), ("b_r10_start", "b_r10_sbox"),
                      ("c1_r10_start", "c1_r10_sbox")):
        assert bytes(s[x] for x in fips[start]) == fips[sb]


def test_shiftrows_map(fips):
    sr = O.shiftrows_src()
    assert sr.tolist() == [0, 5, 10, 15, 4, 9, 14, 3, 8, 13, 2, 7, 12, 1, 6, 11]  # [S:67]
    assert sorted(sr.tolist()) == list(range(16))
    assert all(sr[b] == b for b in (0, 4, 8, 12))                                 # [S:100]
    for sb, srow in (("b_r10_sbox", "b_r10_srow"), ("c1_r10_sbox", "c1_r10_srow")):
        assert bytes(fips[sb][sr[b]] for b in range(16)) == fips[srow]


def test_key_schedule_fips(fips):
    rk = O.expand_key(fips["a1_key"])
    assert rk[0].tobytes() == fips["a1_key"]
    assert rk[10].tobytes() == fips["a1_rk10"] == fips["b_r10_key"]
    assert O.expand_key(fips["c1_key"])[10].tobytes() == fips["c1_rk10"]
    assert O.invert_key_schedule(fips["a1_rk10"]).tobytes() == fips["a1_key"]
    assert O.invert_key_schedule(fips["c1_rk10"]).tobytes() == fips["c1_key"]


def test_key_schedule_round_trip_random():
    rng = np.random.default_rng(7)
    seen = set()
    for _ in range(1000):                                    # [S:80, S:101]
        key = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        rk = O.expand_key(key)
        for r in (1, 5, 10):
            assert O.invert_key_schedule(rk[r], r).tobytes() == key
        seen.add(rk[10].tobytes())
    assert len(seen) == 1000                                  # [S:75]


def test_encrypt_fips_vectors(fips):
    ct, st = O.encrypt_with_states(fips["b_pt"], fips["a1_key"])
    assert ct.tobytes() == fips["b_ct"] and st.tobytes() == fips["b_r10_start"]
    ct, st = O.encrypt_with_states(fips["c1_pt"], fips["c1_key"])
    assert ct.tobytes() == fips["c1_ct"] and st.tobytes() == fips["c1_r10_start"]
