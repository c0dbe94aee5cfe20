"""GPU scale runs as tests, checked against the oracle on sampled rows
and against closed forms that hold at any size:

* the whole 512x256 frame as both arms (P_a = P_b = 131,072; Gamma 68.7 GB in HBM), full GEMM
  and the SYRK path (CPI_SYRK=1): sampled rows equal the oracle (exact sums -> Gamma <= 1e-6),
  Gamma symmetric, the two paths bit-identical on samples;
* many batches at configs[1]'s RoIs (4 x 16,384 frames, N_TOT > 46,340 -> the int64-numerator Gamma):
  sum_pq S_ab = sum_i n_A(i) n_B(i) exactly, sampled rows equal the oracle accumulated batch by
  batch, and cpi_finalize's Gamma on them is within 1e-6 of the exact rational."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "-m gpu selected but no CUDA device"
    from paper_2407_20692_b200 import build
    build.build()


def _assert_rel(got, exact):
    got = got.astype(np.float64)
    zero = exact == 0
    assert np.all(got[zero] == 0)
    assert (np.abs(got - exact) / np.where(zero, 1, np.abs(exact))).max() <= 1e-6


def _whole_frame(n, syrk, monkeypatch):
    from paper_2407_20692_b200 import Context
    if syrk:
        monkeypatch.setenv("CPI_SYRK", "1")
    else:
        monkeypatch.delenv("CPI_SYRK", raising=False)
    roi = (0, 0, 512, 256)
    fr = synth.bernoulli_frames(n, 0.05, seed=synth.SEED_ARMS)
    ctx = Context(roi, roi, n, variant="fp4")
    g = ctx.new_gamma()
    ctx.load_frames(fr)
    ctx.correlate(g)
    torch.cuda.synchronize()
    return fr, ctx, g


def test_whole_frame_full_and_syrk(monkeypatch):
    n = 1536
    p = 512 * 256
    rng = np.random.default_rng(20692)
    rows = np.sort(rng.choice(p, 3, replace=False))
    ri, ci = rng.integers(0, p, 4096), rng.integers(0, p, 4096)
    samples = {}
    for syrk in (False, True):
        fr, ctx, g = _whole_frame(n, syrk, monkeypatch)
        it, jt = torch.from_numpy(ri).cuda(), torch.from_numpy(ci).cuda()
        assert torch.equal(g[it, jt], g[jt, it]), "Gamma must be exactly symmetric"
        samples[syrk] = (g[it, jt].cpu().numpy(), g[torch.from_numpy(rows).cuda()].cpu().numpy())
        del g, ctx
        torch.cuda.empty_cache()
    np.testing.assert_array_equal(samples[True][0], samples[False][0])
    np.testing.assert_array_equal(samples[True][1], samples[False][1])
    want = oracle.correlate(fr, (0, 0, 512, 256), (0, 0, 512, 256), rows=rows)
    _assert_rel(samples[False][1], want["gamma"])


def test_many_batches_int64_numerator():
    from paper_2407_20692_b200 import Context
    roi_a, roi_b = synth.ROI_FULL_A, synth.ROI_FULL_B
    nb, bs = 4, 16384
    ctx = Context(roi_a, roi_b, bs, variant="fp4", keep_counts=True)
    rows = np.array([0, 40_001, 65_535])
    want_sab = np.zeros((rows.size, 65536), dtype=np.int64)
    sum_nanb = 0
    sa_tot = np.zeros(65536, dtype=np.int64)
    sb_tot = np.zeros(65536, dtype=np.int64)
    popc = np.array([bin(b).count("1") for b in range(256)], dtype=np.int64)
    for b in range(nb):
        fr = synth.bernoulli_frames(bs, 0.05, seed=synth.SEED_ARMS, frame0=b * bs)
        ctx.load_frames(fr)
        ctx.correlate()
        w = oracle.correlate(fr, roi_a, roi_b, rows=rows)
        want_sab += w["s_ab"]
        sa_tot += w["s_a"]
        sb_tot += w["s_b"]
        na = popc[fr[:, :, :32]].sum(axis=(1, 2))
        nbb = popc[fr[:, :, 32:]].sum(axis=(1, 2))
        sum_nanb += int((na * nbb).sum())
        torch.cuda.synchronize()
    s_ab, s_a, s_b = ctx.counts_views()
    total = sum(int(s_ab[r:r + 4096].sum(dtype=torch.int64).item()) for r in range(0, s_ab.shape[0], 4096))
    assert total == sum_nanb, "sum of S_ab must equal sum_i n_A(i) n_B(i)"
    np.testing.assert_array_equal(s_ab[torch.from_numpy(rows).cuda()].cpu().numpy(), want_sab)
    np.testing.assert_array_equal(s_a.cpu().numpy(), sa_tot)
    np.testing.assert_array_equal(s_b.cpu().numpy(), sb_tot)
    g = ctx.new_gamma()
    n = ctx.finalize(g)
    torch.cuda.synchronize()
    assert n == nb * bs > 46340
    exact = oracle.gamma(want_sab, sa_tot[rows], sb_tot, n)
    _assert_rel(g[torch.from_numpy(rows).cuda()].cpu().numpy(), exact)
