"""Pins of the refocusing oracle (oracle.refocus / oracle.interp4).

The paper describes refocusing only as "an algorithm based on Radon transformations"
 implemented in the prototype by "4D multilinear interpolation"
(PAPER.md:270).  The transform itself is the declared convention of SURVEY §8(c)
Q10-Q14 (SPEC.md:274 default map, centred coordinates, skip_and_renormalize).  These
tests pin the oracle to that convention through closed forms that do not re-run its
code: the alpha=1 ghost image computed straight from frames, affine (ramp) data on which
multilinear interpolation is exact, integer-shear data that must be reproduced
bit-for-bit, deltas, constants, and a separately written dense numpy evaluation.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
import synth
from tests._util import pack, unpack_np

GOLDEN = Path(__file__).parent / "golden"


def _dense_refocus_np(G, dims, alpha, clamp=False):
    """Independent dense evaluation (SPEC.md:307 'precompute all coordinates, interpolate
    from materialised arrays'): coordinate arrays for every (x,u) and (y,v), the
    bilinear interpolation on the A axes (B coordinates are integers under the default
    map), skip_and_renormalize, or (clamp=True, S:279 / SURVEY §8(c) c2 "CPI_CLAMP") each A
    coordinate clamped into [0, W-1] with every sample counted.  numpy, vectorised, no shared
    code with the C oracle."""
    Wa, Ha, Wb, Hb = dims
    G4 = np.asarray(G, dtype=np.float64).reshape(Ha, Wa, Hb, Wb)   # [m][j][v][u]
    cax, cay, cbx, cby = (Wa - 1) / 2, (Ha - 1) / 2, (Wb - 1) / 2, (Hb - 1) / 2
    x = np.arange(Wa, dtype=np.float64)[:, None]
    u = np.arange(Wb, dtype=np.float64)[None, :]
    y = np.arange(Ha, dtype=np.float64)[:, None]
    v = np.arange(Hb, dtype=np.float64)[None, :]
    CX = (alpha * (x - cax)) + ((1 - alpha) * (u - cbx)) + cax          # [x][u]
    CY = (alpha * (y - cay)) + ((1 - alpha) * (v - cby)) + cay          # [y][v]
    VX = (CX >= 0) & (CX <= Wa - 1)
    VY = (CY >= 0) & (CY <= Ha - 1)
    if clamp:
        CX, CY = np.clip(CX, 0, Wa - 1), np.clip(CY, 0, Ha - 1)
        VX, VY = np.ones_like(VX), np.ones_like(VY)
    J0 = np.clip(np.minimum(np.floor(CX), Wa - 2), 0, None).astype(int)
    M0 = np.clip(np.minimum(np.floor(CY), Ha - 2), 0, None).astype(int)
    TX, TY = CX - J0, CY - M0
    out = np.zeros((Ha, Wa))
    cnt = np.zeros((Ha, Wa), dtype=np.int64)
    uu = np.arange(Wb)
    for yy in range(Ha):
        for vv in range(Hb):
            if not VY[yy, vv]:
                continue
            m0, ty = M0[yy, vv], TY[yy, vv]
            # rows of G at (m0, :, vv, :) and (m0+1, :, vv, :)
            r0 = G4[m0, :, vv, :]
            r1 = G4[m0 + 1, :, vv, :]
            for xx in range(Wa):
                sel = VX[xx]
                j0, tx = J0[xx, sel], TX[xx, sel]
                us = uu[sel]
                val = ((1 - ty) * ((1 - tx) * r0[j0, us] + tx * r0[j0 + 1, us])
                       + ty * ((1 - tx) * r1[j0, us] + tx * r1[j0 + 1, us]))
                out[yy, xx] += val.sum()
                cnt[yy, xx] += sel.sum()
    return np.where(cnt > 0, out / np.maximum(cnt, 1), 0.0), cnt


def test_interp4_golden_examples():
    """SPEC.md:296-298."""
    ex = json.loads((GOLDEN / "refocus_examples.json").read_text())["interp4"]
    rng = np.random.default_rng(1)
    for e in ex:
        Wa, Wb, Ha, Hb = e["dims_jkmn"]
        dims = (Wa, Ha, Wb, Hb)
        j, k, m, n = e["coord"]
        if e["kind"] == "lattice":
            G = rng.random((Wa * Ha, Wb * Hb))
            assert oracle.interp4(G, dims, j, k, m, n) == G[m * Wa + j, n * Wb + k], e["cite"]
        elif e["kind"] == "constant":
            G = np.full((Wa * Ha, Wb * Hb), e["c"])
            assert oracle.interp4(G, dims, j, k, m, n) == e["c"], e["cite"]
        else:
            G = np.zeros((Wa * Ha, Wb * Hb))
            G[1 * Wa + 2, 1 * Wb + 1] = 1.0   # entry at (j=2,k=1,m=1,n=1); (j=1,...) is 0
            assert oracle.interp4(G, dims, j, k, m, n) == e["value"], e["cite"]


def test_interp4_partition_of_unity():
    """the 16 weights sum to 1 within 1e-15 for random fractional coordinates."""
    rng = np.random.default_rng(2)
    dims = (5, 4, 6, 3)
    G = np.ones((20, 18))
    for _ in range(200):
        c = rng.random(4) * (np.array([dims[0], dims[2], dims[1], dims[3]]) - 1)
        assert abs(oracle.interp4(G, dims, *c) - 1.0) <= 1e-15


def test_alpha1_is_ghost_image_from_frames():
    """BASELINE north_star: refocusing at the focused plane reproduces the direct ghost
    image.  At alpha = 1 every sample is valid and lands on the lattice, so
    R_1(p) = (1/P_b) sum_q Gamma[p][q] = (N sum_i A^i_p n_B(i) - S_a[p] sum_i n_B(i))/(N^2 P_b),
    evaluated here directly from the frames with numpy (n_B(i) = fired B pixels in frame i)."""
    rng = np.random.default_rng(3)
    n = 3000
    ra, rb = (0, 0, 10, 7), (16, 1, 6, 5)
    fr = pack(rng.random((n, 8, 32)) < 0.15)
    r = oracle.correlate(fr, ra, rb)
    R = oracle.refocus(r["gamma"], (10, 7, 6, 5), [1.0])[0]
    A = unpack_np(fr, ra).astype(np.int64)
    nB = unpack_np(fr, rb).astype(np.int64).sum(1)
    ghost = (n * (A.T @ nB) - A.sum(0) * nB.sum()) / (n * n * 30.0)
    np.testing.assert_allclose(R.reshape(-1), ghost, rtol=0, atol=1e-17)


@pytest.mark.parametrize("alpha", [0.5, 0.75, 1.0, 1.3, 2.0])
def test_sheared_ramp_closed_form(alpha):
    """Gamma(j,u,m,v) = a + b (j' - s u') + c (m' - s v') (primes: centred coordinates)
    refocused at alpha = 1 - s equals a + b alpha x' + c alpha y' wherever a sample is
    valid: multilinear interpolation is exact on affine data (SURVEY §8(c) pins)."""
    Wa, Ha, Wb, Hb = 11, 9, 7, 6
    a, b, c, s = 0.01, -0.003, 0.002, 1 - alpha
    j = np.arange(Wa) - (Wa - 1) / 2
    m = np.arange(Ha) - (Ha - 1) / 2
    u = np.arange(Wb) - (Wb - 1) / 2
    v = np.arange(Hb) - (Hb - 1) / 2
    G4 = (a + b * (j[None, :, None, None] - s * u[None, None, None, :])
          + c * (m[:, None, None, None] - s * v[None, None, :, None]))    # [m][j][v][u]
    G = G4.reshape(Ha * Wa, Hb * Wb)
    R, cnt = oracle.refocus(G, (Wa, Ha, Wb, Hb), [alpha], return_counts=True)
    expect = a + b * alpha * j[None, :] + c * alpha * m[:, None]
    ok = cnt[0] > 0
    assert ok.any()
    np.testing.assert_allclose(R[0][ok], expect[ok], rtol=0, atol=1e-15)
    assert np.all(R[0][~ok] == 0.0)


def test_integer_shear_bit_exact():
    """Gamma(j,u,m,v) = O(j+u, m+v) for arbitrary fp32 O, equal arm sizes, alpha = 2:
    c_A = 2x - u is an integer, so R(x,y) = O(2x, 2y) exactly wherever count > 0
    (each partial sum is count * an fp32 value, exact in fp64) — zero tolerance."""
    W, H = 9, 7
    rng = np.random.default_rng(4)
    O = rng.standard_normal((2 * W - 1, 2 * H - 1)).astype(np.float32)   # O[sx][sy]
    jj, uu = np.meshgrid(np.arange(W), np.arange(W), indexing="ij")
    mm, vv = np.meshgrid(np.arange(H), np.arange(H), indexing="ij")
    G4 = O[(jj + uu)[None, :, None, :], (mm + vv)[:, None, :, None]]        # [m][j][v][u]
    G = np.ascontiguousarray(G4.reshape(H * W, H * W), dtype=np.float32)
    R, cnt = oracle.refocus(G, (W, H, W, H), [2.0], return_counts=True)
    ok = cnt[0] > 0
    xs, ys = np.meshgrid(np.arange(W), np.arange(H))
    expect = O[2 * xs, 2 * ys].astype(np.float64)
    assert np.array_equal(R[0][ok], expect[ok])


def test_delta_alpha1():
    """a delta at (j0,k0,m0,n0), alpha=1 -> 1/|U| at (j0,m0), zero elsewhere."""
    e = json.loads((GOLDEN / "refocus_examples.json").read_text())["delta_alpha1"]
    Wa, Ha, Wb, Hb = e["dims"]
    j0, k0, m0, n0 = e["at"]
    G = np.zeros((Wa * Ha, Wb * Hb))
    G[m0 * Wa + j0, n0 * Wb + k0] = 1.0
    R = oracle.refocus(G, (Wa, Ha, Wb, Hb), [1.0])[0]
    expect = np.zeros((Ha, Wa))
    expect[m0, j0] = 1.0 / (Wb * Hb)
    assert np.array_equal(R, expect), e["cite"]


def test_constant_and_clamp():
    """S:297 constant tensor -> constant where count > 0; clamp: every sample
    counts (count = P_b) and a constant stays constant everywhere."""
    dims = (8, 6, 5, 4)
    G = np.full((48, 20), 0.0625)
    R, cnt = oracle.refocus(G, dims, [0.6, 1.7], return_counts=True)
    assert np.all(R[cnt > 0] == 0.0625) and np.all(R[cnt == 0] == 0.0)
    Rc, cc = oracle.refocus(G, dims, [0.6, 1.7], boundary=oracle.BOUNDARY_CLAMP, return_counts=True)
    assert np.all(cc == 20) and np.all(np.abs(Rc - 0.0625) <= 1e-17)


@pytest.mark.parametrize("alpha", json.loads((GOLDEN / "refocus_examples.json").read_text())["dense_alphas"]["alphas"] + [1.0, 1.75])
def test_dense_materialised_oracle(alpha):
    """SPEC.md:487 acceptance 5: vs a dense materialised-coordinate evaluation within
    1e-12 absolute — a delta tensor and a random tensor."""
    dims = (7, 6, 5, 4)
    Wa, Ha, Wb, Hb = dims
    rng = np.random.default_rng(5)
    for G in (np.zeros((Wa * Ha, Wb * Hb)), rng.random((Wa * Ha, Wb * Hb)) - 0.5):
        if not G.any():
            G[3 * Wa + 2, 1 * Wb + 3] = 1.0
        R, cnt = oracle.refocus(G, dims, [alpha], return_counts=True)
        D, dcnt = _dense_refocus_np(G, dims, alpha)
        np.testing.assert_array_equal(cnt[0], dcnt)
        np.testing.assert_allclose(R[0], D, rtol=0, atol=1e-12)


@pytest.mark.parametrize("alpha", [0.6, 1.3, 2.0, -0.8])
def test_dense_materialised_oracle_clamp(alpha):
    """CPI_CLAMP branch on RANDOM Gamma vs the dense numpy evaluation
    with its own clamp: counts are P_b everywhere and values agree within 1e-12.  Random data
    detects a wrong clamp bound (e.g. W instead of W - 1), which constant data cannot."""
    dims = (7, 6, 5, 4)
    Wa, Ha, Wb, Hb = dims
    G = np.random.default_rng(15).random((Wa * Ha, Wb * Hb)) - 0.5
    R, cnt = oracle.refocus(G, dims, [alpha], boundary=oracle.BOUNDARY_CLAMP, return_counts=True)
    D, dcnt = _dense_refocus_np(G, dims, alpha, clamp=True)
    assert np.all(cnt[0] == Wb * Hb) and np.all(dcnt == Wb * Hb)
    np.testing.assert_allclose(R[0], D, rtol=0, atol=1e-12)


@pytest.mark.parametrize("alpha", [0.6, 1.3, 2.0])
def test_clamp_ramp_closed_form(alpha):
    """Closed form of the clamp branch: on affine Gamma = a + b j' + c m' (primes: centred),
    interpolation is exact and every sample counts, so
        R(x, y) = a + b mean_u(clip(c_x(x,u), 0, W_a-1) - c_ax) + c mean_v(clip(c_y(y,v), 0, H_a-1) - c_ay)
    with c_x, c_y the default map.  Linear extrapolation is exact on affine data too, so
    a clamp to the wrong bound changes the coordinate means and fails here."""
    Wa, Ha, Wb, Hb = 11, 9, 7, 6
    a, b, c = 0.01, -0.003, 0.002
    cax, cay, cbx, cby = (Wa - 1) / 2, (Ha - 1) / 2, (Wb - 1) / 2, (Hb - 1) / 2
    j = np.arange(Wa) - cax
    m = np.arange(Ha) - cay
    G4 = (a + b * j[None, :, None, None] + c * m[:, None, None, None]) * np.ones((1, 1, Hb, Wb))
    G = G4.reshape(Ha * Wa, Hb * Wb)
    R = oracle.refocus(G, (Wa, Ha, Wb, Hb), [alpha], boundary=oracle.BOUNDARY_CLAMP)[0]
    x, u = np.arange(Wa)[:, None], np.arange(Wb)[None, :]
    y, v = np.arange(Ha)[:, None], np.arange(Hb)[None, :]
    mx = np.clip(alpha * (x - cax) + (1 - alpha) * (u - cbx) + cax, 0, Wa - 1).mean(1) - cax
    my = np.clip(alpha * (y - cay) + (1 - alpha) * (v - cby) + cay, 0, Ha - 1).mean(1) - cay
    expect = a + b * mx[None, :] + c * my[:, None]
    np.testing.assert_allclose(R, expect, rtol=0, atol=1e-15)


def test_counts_are_separable():
    """The skip rule is per axis, so count(x,y) = cnt_x(x) * cnt_y(y) with
    cnt_x(x) = #{u : 0 <= alpha(x - c_a) + (1-alpha)(u - c_b) + c_a <= W_a - 1} (brute force)."""
    Wa, Ha, Wb, Hb = 13, 8, 9, 6
    G = np.zeros((Wa * Ha, Wb * Hb))
    for alpha in (0.4, 0.9, 1.6, 2.5, -0.7):
        _, cnt = oracle.refocus(G, (Wa, Ha, Wb, Hb), [alpha], return_counts=True)
        def axis(W, Wb_):
            c, cb = (W - 1) / 2, (Wb_ - 1) / 2
            return np.array([sum(0 <= (alpha * (x - c)) + ((1 - alpha) * (u - cb)) + c <= W - 1
                                 for u in range(Wb_)) for x in range(W)])
        np.testing.assert_array_equal(cnt[0], np.outer(axis(Ha, Hb), axis(Wa, Wb)))


def test_linearity_permutation_duplicates():
    """S:328 linearity (1e-12 rel); S:332 permuting alphas permutes planes bit-identically;
    S:315 duplicated alpha -> bit-identical planes."""
    dims = (6, 5, 4, 4)
    rng = np.random.default_rng(6)
    G1, G2 = rng.random((30, 16)), rng.random((30, 16))
    al = [0.55, 1.0, 1.45, 0.55]
    R1, R2 = oracle.refocus(G1, dims, al), oracle.refocus(G2, dims, al)
    R12 = oracle.refocus(2.0 * G1 - 3.0 * G2, dims, al)
    np.testing.assert_allclose(R12, 2 * R1 - 3 * R2, rtol=1e-12, atol=1e-14)
    assert np.array_equal(R1[0], R1[3])
    perm = [2, 0, 3, 1]
    assert np.array_equal(oracle.refocus(G1, dims, [al[i] for i in perm]), R1[perm])


def test_pixel_subset_matches_full_plane():
    dims = (6, 5, 4, 3)
    G = np.random.default_rng(7).random((30, 12)).astype(np.float32)
    full = oracle.refocus(G, dims, [0.8, 1.9])
    pix = [(0, 0), (5, 4), (2, 3)]
    sub = oracle.refocus(G, dims, [0.8, 1.9], pixels=pix)
    for k, (x, y) in enumerate(pix):
        assert sub[0, k] == full[0, y, x] and sub[1, k] == full[1, y, x]


def test_degenerate_alpha_rejected():
    """S:303 DegenerateAlpha: alpha = 0 (or non-finite) under the default map."""
    G = np.zeros((4, 4))
    for bad in (0.0, float("nan"), float("inf")):
        with pytest.raises(ValueError):
            oracle.refocus(G, (2, 2, 2, 2), [bad])


# ---- general affine maps (S:273 RefocusMap) ---------------------------

def _coords_np(mp, dims):
    """Coordinate arrays of a general map (inputs of the check: the map's definition)."""
    Wa, Ha, Wb, Hb = dims
    cax, cay, cbx, cby = (Wa - 1) / 2, (Ha - 1) / 2, (Wb - 1) / 2, (Hb - 1) / 2
    xr = np.arange(Wa, dtype=np.float64)[:, None] - cax
    ur = np.arange(Wb, dtype=np.float64)[None, :] - cbx
    yr = np.arange(Ha, dtype=np.float64)[:, None] - cay
    vr = np.arange(Hb, dtype=np.float64)[None, :] - cby
    CAX = mp[0] * xr + mp[1] * ur + mp[2] + cax        # [x][u]
    CBX = mp[3] * xr + mp[4] * ur + mp[5] + cbx
    CAY = mp[6] * yr + mp[7] * vr + mp[8] + cay        # [y][v]
    CBY = mp[9] * yr + mp[10] * vr + mp[11] + cby
    VX = (CAX >= 0) & (CAX <= Wa - 1) & (CBX >= 0) & (CBX <= Wb - 1)
    VY = (CAY >= 0) & (CAY <= Ha - 1) & (CBY >= 0) & (CBY <= Hb - 1)
    return CAX, CBX, CAY, CBY, VX, VY


def _dense_affine_np(G, dims, mp, clamp=False):
    """Independent dense evaluation for a general map: materialised coordinates, the 16-corner
    multilinear weights as separate per-axis 1D linear weights (numpy), skip_and_renormalize
    (or clamp=True: every coordinate clamped onto its lattice interval, every sample counted)."""
    Wa, Ha, Wb, Hb = dims
    G4 = np.asarray(G, dtype=np.float64).reshape(Ha, Wa, Hb, Wb)     # [m][j][n][k]
    CAX, CBX, CAY, CBY, VX, VY = _coords_np(mp, dims)
    if clamp:
        CAX, CBX = np.clip(CAX, 0, Wa - 1), np.clip(CBX, 0, Wb - 1)
        CAY, CBY = np.clip(CAY, 0, Ha - 1), np.clip(CBY, 0, Hb - 1)
        VX, VY = np.ones_like(VX), np.ones_like(VY)

    def lin(c, W):   # lower corner and weights of 1D linear interpolation on [0, W-1]
        i0 = np.clip(np.minimum(np.floor(c), W - 2), 0, None).astype(int)
        return i0, c - i0
    J0, TJ = lin(CAX, Wa)
    K0, TK = lin(CBX, Wb)
    M0, TM = lin(CAY, Ha)
    N0, TN = lin(CBY, Hb)
    out = np.zeros((Ha, Wa))
    cnt = np.zeros((Ha, Wa), dtype=np.int64)
    for y in range(Ha):
        for v in range(Hb):
            if not VY[y, v]:
                continue
            for x in range(Wa):
                for u in range(Wb):
                    if not VX[x, u]:
                        continue
                    acc = 0.0
                    for dm, wm in ((0, 1 - TM[y, v]), (1, TM[y, v])):
                        for dn, wn in ((0, 1 - TN[y, v]), (1, TN[y, v])):
                            for dj, wj in ((0, 1 - TJ[x, u]), (1, TJ[x, u])):
                                for dk, wk in ((0, 1 - TK[x, u]), (1, TK[x, u])):
                                    acc += wm * wn * wj * wk * G4[M0[y, v] + dm, J0[x, u] + dj,
                                                                   N0[y, v] + dn, K0[x, u] + dk]
                    out[y, x] += acc
                    cnt[y, x] += 1
    return np.where(cnt > 0, out / np.maximum(cnt, 1), 0.0), cnt


@pytest.mark.parametrize("boundary", [0, 1])
def test_affine_default_map_is_bit_identical(boundary):
    """The default map written as a general map gives the default refocus bit for bit."""
    dims = (9, 7, 8, 5)
    G = synth.random_gamma(63, 40, seed=21)
    al = [0.5, 0.8, 1.0, 1.37, 2.0]
    for g in (G, G.astype(np.float64)):
        R = oracle.refocus(g, dims, al, boundary=boundary)
        Ra = oracle.refocus_affine(g, dims, [oracle.default_map(a) for a in al], boundary=boundary)
        np.testing.assert_array_equal(Ra, R)


MAPS = [
    [0.7, 0.3, 0.25, 0.0, 0.5, -0.3, 1.3, -0.3, -0.4, 0.1, 0.8, 0.2],     # fractional B coordinates
    [1.0, 0.0, 0.0, 0.25, 0.75, 0.1, 0.9, 0.1, 0.0, -0.2, 1.1, 0.0],
    [2.0, -1.0, 0.5, 0.0, 1.0, 0.0, 0.5, 0.5, 0.0, 0.0, 1.0, 0.0],        # integral B (GPU fast path)
]


@pytest.mark.parametrize("mp", MAPS)
def test_affine_dense_materialised(mp):
    """General maps vs the dense numpy evaluation (values and counts)."""
    dims = (6, 5, 7, 4)
    G = synth.random_gamma(30, 28, seed=8)
    R, C = oracle.refocus_affine(G, dims, [mp], return_counts=True)
    Rd, Cd = _dense_affine_np(G, dims, np.array(mp))
    np.testing.assert_array_equal(C[0], Cd)
    np.testing.assert_allclose(R[0], Rd, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("mp", MAPS)
def test_affine_exact_on_affine_gamma(mp):
    """Multilinear interpolation reproduces affine data exactly: for
    Gamma(j,k,m,n) = c0 + c1 j + c2 k + c3 m + c4 n the refocused pixel is the mean over valid
    samples of c0 + c1 c_Ax + c2 c_Bx + c3 c_Ay + c4 c_By (closed form, no interpolation)."""
    dims = (8, 6, 7, 5)
    Wa, Ha, Wb, Hb = dims
    c0, c1, c2, c3, c4 = 0.3, 0.25, -0.5, 0.125, 1.0
    m, j, n, k = np.meshgrid(np.arange(Ha), np.arange(Wa), np.arange(Hb), np.arange(Wb), indexing="ij")
    G = (c0 + c1 * j + c2 * k + c3 * m + c4 * n).reshape(Wa * Ha, Wb * Hb)
    R = oracle.refocus_affine(G, dims, [mp])[0]
    CAX, CBX, CAY, CBY, VX, VY = _coords_np(np.array(mp), dims)
    for y in range(Ha):
        for x in range(Wa):
            vals = [c0 + c1 * CAX[x, u] + c2 * CBX[x, u] + c3 * CAY[y, v] + c4 * CBY[y, v]
                    for v in range(Hb) for u in range(Wb) if VX[x, u] and VY[y, v]]
            want = np.mean(vals) if vals else 0.0
            assert abs(R[y, x] - want) <= 1e-12 * (1 + abs(want))


@pytest.mark.parametrize("mp", [MAPS[0], MAPS[2]])
def test_affine_dense_materialised_clamp(mp):
    """General maps under CPI_CLAMP vs the dense numpy evaluation with its own clamp (every
    sample counts)."""
    dims = (6, 5, 7, 4)
    G = synth.random_gamma(30, 28, seed=9)
    R, C = oracle.refocus_affine(G, dims, [mp], boundary=oracle.BOUNDARY_CLAMP, return_counts=True)
    Rd, Cd = _dense_affine_np(G, dims, np.array(mp), clamp=True)
    assert np.all(C[0] == 28) and np.all(Cd == 28)
    np.testing.assert_allclose(R[0], Rd, rtol=1e-12, atol=1e-15)


def test_affine_identity_map_is_angular_mean():
    """a = 1, b = 0 on the A axes and the identity on the B axes: R(x,y) = mean over (u,v) of
    Gamma[(y, x)][(v, u)] (plain angular marginal)."""
    dims = (5, 4, 6, 3)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(20, 18, seed=3)
    ident = [1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0, 0.0]
    R = oracle.refocus_affine(G, dims, [ident])[0]
    want = np.asarray(G, dtype=np.float64).reshape(Ha, Wa, Hb * Wb).mean(axis=2)
    np.testing.assert_allclose(R, want, rtol=1e-13)


def test_affine_nonfinite_rejected():
    with pytest.raises(ValueError):
        oracle.refocus_affine(np.zeros((4, 4), np.float32), (2, 2, 2, 2), [[np.nan] + [0.0] * 11])


def _resample_b_np(G, dims, ex, fx, ey, fy):
    """Gamma resampled onto the B lattice (DESIGN R15): G'[(m, j)][(v, u)] = bilinear of
    G[(m, j)][(., .)] at (c_By(v), c_Bx(u)), coordinates clamped to the lattice.  numpy."""
    Wa, Ha, Wb, Hb = dims
    G4 = np.asarray(G, dtype=np.float64).reshape(Ha * Wa, Hb, Wb)
    cbx, cby = (Wb - 1) / 2, (Hb - 1) / 2
    cu = np.clip(ex * (np.arange(Wb) - cbx) + fx + cbx, 0, Wb - 1)
    cv = np.clip(ey * (np.arange(Hb) - cby) + fy + cby, 0, Hb - 1)
    k0 = np.minimum(np.floor(cu), Wb - 2).astype(int)
    n0 = np.minimum(np.floor(cv), Hb - 2).astype(int)
    tu, tv = cu - k0, cv - n0
    rows = (1 - tv)[None, :, None] * G4[:, n0, :] + tv[None, :, None] * G4[:, n0 + 1, :]     # [p][v][k]
    out = (1 - tu)[None, None, :] * rows[:, :, k0] + tu[None, None, :] * rows[:, :, k0 + 1]  # [p][v][u]
    return out.reshape(Wa * Ha, Hb * Wb)


@pytest.mark.parametrize("boundary,bmap", [(0, (0.8, 0.3, 0.6, -0.5)), (1, (0.8, 0.3, 0.6, -0.5)),
                                           (1, (1.3, -0.7, 1.6, 0.9))])
def test_fractional_b_factorises_through_b_resample(boundary, bmap):
    """R15: with B coordinates depending on u, v only, the 16-corner weight factorises into
    A corners x B corners, so refocusing Gamma with the fractional-B map equals refocusing the
    B-resampled Gamma' with the identity B map (the GPU's default route).  Skip policy: B maps
    that stay on the lattice (so no sample is dropped for its B coordinate); clamp: any map."""
    dims = (7, 6, 7, 5)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=41)
    ex, fx, ey, fy = bmap
    amaps = [(0.7, 0.3, 0.25, 1.3, -0.3, -0.4), (1.6, -0.45, -1.5, 0.55, 0.5, 2.0), (1.0, 0.0, 0.0, 1.0, 0.0, 0.0)]
    frac = [[a[0], a[1], a[2], 0.0, ex, fx, a[3], a[4], a[5], 0.0, ey, fy] for a in amaps]
    ident = [[a[0], a[1], a[2], 0.0, 1.0, 0.0, a[3], a[4], a[5], 0.0, 1.0, 0.0] for a in amaps]
    R = oracle.refocus_affine(G, dims, frac, boundary=boundary)
    Rr = oracle.refocus_affine(_resample_b_np(G, dims, ex, fx, ey, fy), dims, ident, boundary=boundary)
    np.testing.assert_allclose(Rr, R, rtol=1e-11, atol=1e-15)
