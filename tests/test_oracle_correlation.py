"""Pins of the correlation oracle (oracle.unpack / marginals / pair_sums / gamma) against
things other than itself: the paper's/SPEC's hand values, a per-frame fp64 brute force
in numpy, exact identities, bounds, algebraic closed forms and light statistics.

Eq. (1) is PAPER.md:100-111.  Each test names the passage it pins.
"""
import json
import math
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import oracle
import synth
from tests._util import pack, unpack_np

GOLDEN = Path(__file__).parent / "golden"


def _one_by_one(a_bits, b_bits):
    """N frames of an 8x1 layout: A = col 0, B = col 1 (1x1 RoIs)."""
    n = len(a_bits)
    bits = np.zeros((n, 1, 8), dtype=np.uint8)
    bits[:, 0, 0] = a_bits
    bits[:, 0, 1] = b_bits
    return pack(bits), (0, 0, 1, 1), (1, 0, 1, 1)


def test_hand_values_frames():
    """hand evaluations of Eq. (1)."""
    cases = json.loads((GOLDEN / "eq1_hand_values.json").read_text())["frame_cases"]
    for c in cases:
        fr, ra, rb = _one_by_one(c["a"], c["b"])
        r = oracle.correlate(fr, ra, rb)
        assert Fraction(r["gamma"][0, 0]) == Fraction(c["gamma"]), c["cite"]
        if "s_ab" in c:
            assert r["s_ab"][0, 0] == c["s_ab"], c["cite"]


def test_hand_values_counts():
    """finalize examples; exact rational reproduced in fp64."""
    for c in json.loads((GOLDEN / "eq1_hand_values.json").read_text())["count_cases"]:
        g = oracle.gamma(np.array([[c["s_ab"]]]), np.array([c["s_a"]]), np.array([c["s_b"]]), c["n"])
        assert Fraction(g[0, 0]) == Fraction(c["gamma"]), c["cite"]


def test_zero_frames_rejected():
    """SPEC.md:230 finalize errors ZeroFrames when n_tot = 0."""
    with pytest.raises(ValueError):
        oracle.gamma(np.zeros((1, 1)), np.zeros(1), np.zeros(1), 0)


@pytest.mark.parametrize("trial", range(20))
def test_brute_force_vs_per_frame_fp64(trial):
    """SPEC.md:483 acceptance 1: >= 20 random datasets, RoIs <= 16x16, frames <= 4096,
    against SPEC correlate_naive (per-frame fp64 accumulation, numpy) and against an
    independent numpy unpack + matmul of the integer sums."""
    rng = np.random.default_rng([77, trial])
    W, H = 64, 24
    n = int(rng.integers(1, 4097 if trial % 5 == 0 else 700))
    wa, ha = int(rng.integers(1, 17)), int(rng.integers(1, 17))
    wb, hb = int(rng.integers(1, 17)), int(rng.integers(1, 17))
    ra = (int(rng.integers(0, W - wa + 1)), int(rng.integers(0, H - ha + 1)), wa, ha)
    rb = (int(rng.integers(0, W - wb + 1)), int(rng.integers(0, H - hb + 1)), wb, hb)
    f = float(rng.choice([0.03, 0.2, 0.5, 0.9]))
    frames = pack(rng.random((n, H, W)) < f)
    r = oracle.correlate(frames, ra, rb)
    A, B = unpack_np(frames, ra).astype(np.int64), unpack_np(frames, rb).astype(np.int64)
    np.testing.assert_array_equal(r["s_ab"], A.T @ B)
    np.testing.assert_array_equal(r["s_a"], A.sum(0))
    np.testing.assert_array_equal(r["s_b"], B.sum(0))
    naive = oracle.correlate_naive_fp64(frames, ra, rb)
    # per-frame fp64 sums of 0/1 are exact; only the final expression rounds
    np.testing.assert_allclose(r["gamma"], naive, rtol=0, atol=4e-16)


def test_exact_identities_single_frame_and_zero():
    """N=1 -> Gamma == 0; all-zero frames -> Gamma == 0."""
    rng = np.random.default_rng(5)
    fr = pack(rng.random((1, 8, 32)) < 0.5)
    r = oracle.correlate(fr, (0, 0, 8, 8), (8, 0, 8, 8))
    assert np.all(r["gamma"] == 0.0)
    fr0 = np.zeros((50, 8, 4), dtype=np.uint8)
    r0 = oracle.correlate(fr0, (0, 0, 4, 4), (16, 2, 4, 4))
    assert np.all(r0["gamma"] == 0.0) and np.all(r0["s_ab"] == 0)


def test_constant_pixel_row_is_zero():
    """an always-on (or always-off) pixel has zero covariance with all."""
    rng = np.random.default_rng(6)
    bits = rng.random((300, 8, 32)) < 0.3
    bits[:, 2, 3] = True   # A pixel (3,2) always on
    bits[:, 4, 5] = False  # A pixel (5,4) always off
    r = oracle.correlate(pack(bits), (0, 0, 8, 8), (16, 0, 8, 8))
    assert np.all(r["gamma"][2 * 8 + 3] == 0.0)
    assert np.all(r["gamma"][4 * 8 + 5] == 0.0)


def test_identical_and_complementary_arms():
    """SURVEY §8(c) pins: B_q == A_p bit for bit -> Gamma = f(1-f) exactly;
    B_q == NOT A_p -> Gamma = -f(1-f) exactly, with f = S_a/N."""
    rng = np.random.default_rng(8)
    n = 997
    a = rng.random((n, 6, 6)) < 0.37
    bits = np.zeros((n, 6, 16), dtype=bool)
    bits[:, :, 0:6] = a
    bits[:, :, 8:14] = ~a
    fr = pack(bits)
    # identical region on both arms
    r = oracle.correlate(fr, (0, 0, 6, 6), (0, 0, 6, 6))
    s = r["s_a"]
    diag = np.diag(r["gamma"])
    for p in range(36):
        # correctly rounded fp64 of the rational S(N-S)/N^2 (Python float(Fraction) rounds once)
        assert diag[p] == float(Fraction(int(s[p]) * (n - int(s[p])), n * n))
    # complement arm
    rc = oracle.correlate(fr, (0, 0, 6, 6), (8, 0, 6, 6))
    assert np.all(np.diag(rc["s_ab"]) == 0)
    dc = np.diag(rc["gamma"])
    np.testing.assert_array_equal(dc, -diag)


def test_bounds_and_symmetry():
    """S:197-198 count bounds, S:204 Gamma in [-1/4, 1/4]; same RoI on both arms ->
    S_ab symmetric, Gamma symmetric under arm swap (BASELINE.json north_star)."""
    rng = np.random.default_rng(9)
    fr = pack(rng.random((1500, 10, 24)) < 0.2)
    ra, rb = (1, 1, 7, 6), (12, 2, 9, 5)
    r = oracle.correlate(fr, ra, rb)
    sa, sb, sab, n = r["s_a"][:, None], r["s_b"][None, :], r["s_ab"], r["n"]
    assert np.all(sab <= np.minimum(sa, sb)) and np.all(sab >= np.maximum(0, sa + sb - n))
    assert np.all(np.abs(r["gamma"]) <= 0.25)
    rs = oracle.correlate(fr, ra, ra)
    np.testing.assert_array_equal(rs["s_ab"], rs["s_ab"].T)
    np.testing.assert_array_equal(rs["gamma"], rs["gamma"].T)
    # swapping the arms transposes Gamma exactly
    r_ba = oracle.correlate(fr, rb, ra)
    np.testing.assert_array_equal(r_ba["gamma"], r["gamma"].T)


def test_row_column_total_closed_forms():
    """Algebraic identities of the pair sums (exact, O(N P)), SURVEY §8(c):
    sum_q S_ab[p][q] = sum_i A^i_p n_B(i),  sum_p S_ab[p][q] = sum_i B^i_q n_A(i),
    sum_pq S_ab = sum_i n_A(i) n_B(i); n_X(i) = number of fired pixels of arm X in frame i
    (counted here with a byte popcount table, not via the oracle)."""
    rng = np.random.default_rng(10)
    fr = pack(rng.random((2000, 16, 32)) < 0.1)
    ra, rb = (0, 0, 16, 16), (16, 0, 16, 16)   # byte-aligned halves
    r = oracle.correlate(fr, ra, rb)
    popc = np.array([bin(b).count("1") for b in range(256)], dtype=np.int64)
    n_a = popc[fr[:, :, 0:2]].sum(axis=(1, 2))
    n_b = popc[fr[:, :, 2:4]].sum(axis=(1, 2))
    A = unpack_np(fr, ra).astype(np.int64)
    B = unpack_np(fr, rb).astype(np.int64)
    np.testing.assert_array_equal(r["s_ab"].sum(1), A.T @ n_b)
    np.testing.assert_array_equal(r["s_ab"].sum(0), B.T @ n_a)
    assert r["s_ab"].sum() == int(n_a @ n_b)
    assert r["s_a"].sum() == n_a.sum() and r["s_b"].sum() == n_b.sum()


def test_additivity_and_order_invariance():
    """S:235-243 accumulate_chunk: sums over frame slices add exactly; Eq. (1) is invariant
    under frame order."""
    rng = np.random.default_rng(11)
    fr = pack(rng.random((999, 8, 16)) < 0.25)
    ra, rb = (0, 0, 5, 8), (8, 1, 6, 7)
    full = oracle.correlate(fr, ra, rb)
    cuts = [0, 100, 101, 640, 999]
    acc = sum(oracle.pair_sums(fr[a:b], ra, rb) for a, b in zip(cuts, cuts[1:]))
    np.testing.assert_array_equal(acc, full["s_ab"])
    perm = rng.permutation(999)
    np.testing.assert_array_equal(oracle.pair_sums(fr[perm], ra, rb), full["s_ab"])


def test_row_subset_and_threads():
    """rows= selects A pixels; result rows equal the full computation's rows."""
    rng = np.random.default_rng(12)
    fr = pack(rng.random((300, 8, 16)) < 0.3)
    ra, rb = (0, 0, 8, 8), (8, 0, 8, 8)
    full = oracle.pair_sums(fr, ra, rb, threads=1)
    rows = [63, 0, 17, 17]
    np.testing.assert_array_equal(oracle.pair_sums(fr, ra, rb, rows=rows, threads=3), full[rows])


def test_unpack_non_byte_aligned_and_msb():
    """S:83 per-pixel scalar re-read: RoIs not aligned to bytes (BASELINE configs[0]
    x0 = 124, 382); msb_first flips the bit index (S:29 bit_order)."""
    rng = np.random.default_rng(13)
    bits = rng.random((5, 256, 512)) < 0.5
    fr = pack(bits)
    for roi in (synth.ROI_TINY_A, synth.ROI_TINY_B, (3, 5, 13, 2)):
        x0, y0, w, h = roi
        u = oracle.unpack(fr, roi)
        np.testing.assert_array_equal(u, bits[:, y0:y0 + h, x0:x0 + w].reshape(5, -1))
    frm = np.packbits(bits.astype(np.uint8), axis=-1, bitorder="big")
    np.testing.assert_array_equal(oracle.unpack(frm, (3, 5, 13, 2), msb=True),
                                  bits[:, 5:7, 3:16].reshape(5, -1))


def test_cumulative_preview_is_marginal():
    """Fig. 2 cumulative sum of 512 frames = single-pixel sums; max <= 512."""
    fr = synth.bernoulli_frames(512, 0.3, seed=3, width=64, height=16)
    s = oracle.marginals(fr, (0, 0, 64, 16))
    allbits = np.unpackbits(fr, axis=-1, bitorder="little").astype(np.int64)
    np.testing.assert_array_equal(s, allbits.sum(0).reshape(-1))
    assert s.max() <= 512


def test_spec_finalize_distance_from_exact():
    """SPEC's fp64 expression is within a few ulps of the exact
    rational but is not exact; bound |spec - exact| <= 4 eps (S/N + S_a S_b/N^2)."""
    rng = np.random.default_rng(14)
    fr = pack(rng.random((299, 6, 16)) < 0.6)
    r = oracle.correlate(fr, (0, 0, 6, 6), (8, 0, 6, 6))
    spec = oracle.gamma_spec(r["s_ab"], r["s_a"], r["s_b"], r["n"])
    n = r["n"]
    bound = 4 * 2.0**-53 * (r["s_ab"] / n + np.outer(r["s_a"], r["s_b"]) / n**2)
    assert np.all(np.abs(spec - r["gamma"]) <= bound)


def test_independent_bernoulli_statistics():
    """BASELINE north_star: Gamma ~ 0 for independent frames.  For independent
    Bernoulli(f) pixels the estimator has mean -f(1-f)/N ~ 0 and std ~ f(1-f)/sqrt(N)."""
    f, n = 0.05, 20000
    fr = synth.bernoulli_frames(n, f, seed=21, width=32, height=8)
    r = oracle.correlate(fr, (0, 0, 16, 8), (16, 0, 16, 8))
    g = r["gamma"]
    sd = f * (1 - f) / math.sqrt(n)
    assert abs(g.mean()) < 5 * sd / math.sqrt(g.size) + 3 * f * (1 - f) / n
    assert 0.85 * sd < g.std() < 1.15 * sd


@pytest.mark.parametrize("f", [0.5, 0.2])
def test_chaotic_light_known_correlation(f):
    """BASELINE north_star: a synthetic chaotic-light source with known correlation is
    recovered.  Thresholded unit Gaussian speckle with grain g has pairwise correlation
    rho = (1-|dx|/g)(1-|dy|/g); Eq. (1) then equals Phi2(-tau,-tau;rho) - f^2, which for
    f = 1/2 is Sheppard's arcsin(rho)/(2 pi).  Checked within 5 sigma per pair."""
    from scipy.stats import multivariate_normal, norm
    n, g = 30000, 2
    ra = (0, 0, 6, 5)
    rb = (16, 0, 6, 5)
    fr = synth.speckle_frames(n, ra, rb, f=f, grain=g, shift_b=(1, 0), width=32, height=8)
    r = oracle.correlate(fr, ra, rb)
    tau = norm.ppf(1 - f)
    worst = 0.0
    cache = {}
    for p in range(30):
        ja, ma = p % 6, p // 6
        for q in range(30):
            kb, nb = q % 6, q // 6
            dx, dy = ja - (kb + 1), ma - nb
            rho = max(0.0, 1 - abs(dx) / g) * max(0.0, 1 - abs(dy) / g)
            if rho not in cache:
                if f == 0.5:
                    cache[rho] = math.asin(rho) / (2 * math.pi)
                elif rho == 0:
                    cache[rho] = 0.0
                elif rho == 1:
                    cache[rho] = f - f * f
                else:
                    cache[rho] = multivariate_normal(mean=[0, 0], cov=[[1, rho], [rho, 1]]).cdf([-tau, -tau]) - f * f
            expect = cache[rho]
            p11 = expect + f * f
            sigma = math.sqrt(max(p11 * (1 - p11), 1e-12) / n)   # std of mean(A B), conservative
            worst = max(worst, abs(r["gamma"][p, q] - expect) / sigma)
    assert worst < 5.0
    # the strongest pairs are the co-located ones (rho = 1): Gamma = f(1-f)
    assert abs(r["gamma"][1, 0] - f * (1 - f)) < 0.01
