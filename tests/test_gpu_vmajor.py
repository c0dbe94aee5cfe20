"""GPU parity of the v-major B order (include/cpi.h CPI_GAMMA_VMAJOR) and of the window stage 1
(KB5w, csrc/refocus_w.cu) it feeds, through the C ABI, against the CPU oracle.

Bars as tests/test_gpu_parity.py: S_ab / S_a / S_b bit-exact (here: bit-identical to the
row-major context after un-permuting the B index), Gamma bit-identical, refocused planes within
1e-6 M of the oracle (M = the oracle's refocusing of |Gamma|, per output).  Gamma given to a
v-major context is the row-major Gamma with its columns permuted by ctx.b_index().
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _ctx(roi_a, roi_b, n, **kw):
    from paper_2407_20692_b200 import Context
    return Context(roi_a, roi_b, n, **kw)


def _to_ctx_order(ctx, G):
    """Row-major Gamma [P_a][P_b] -> the context's column order."""
    out = np.empty_like(G)
    out[:, ctx.b_index()] = G
    return out


def _refocus_vmajor(G, dims, alphas=None, boundary=0, affine=None, row0=0, rows=None, row_block=0, row_stride=0):
    Wa, Ha, Wb, Hb = dims
    ctx = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1, gamma_order="vmajor")
    g = torch.from_numpy(np.ascontiguousarray(_to_ctx_order(ctx, np.asarray(G, dtype=np.float32)))).cuda()
    n = len(affine) if affine is not None else len(alphas)
    planes = ctx.new_planes(n)
    ctx.refocus(alphas, g, planes, boundary=boundary, affine=affine, row0=row0, rows=rows, row_block=row_block,
                row_stride=row_stride)
    torch.cuda.synchronize()
    return planes.cpu().numpy().astype(np.float64)


def _assert_planes(R, G, dims, alphas=None, boundary=0, affine=None):
    if affine is not None:
        Ro = oracle.refocus_affine(G, dims, affine, boundary=boundary)
        M = oracle.refocus_affine(np.abs(np.asarray(G, dtype=np.float64)), dims, affine, boundary=boundary)
    else:
        Ro = oracle.refocus(G, dims, alphas, boundary=boundary)
        M = oracle.refocus(np.abs(np.asarray(G, dtype=np.float64)), dims, alphas, boundary=boundary)
    err = np.abs(R - Ro)
    assert np.all(err <= 1e-6 * M + 1e-30), f"max err/M {np.max(err / np.maximum(M, 1e-300)):.3e}"


ALPHAS = [0.5, 0.61, 0.75, 0.93, 1.0, 1.07, 1.3, 1.52, 1.77, 2.0, -0.6]


@pytest.mark.parametrize("dims", [(24, 20, 16, 12), (7, 5, 9, 4), (40, 33, 37, 8), (64, 10, 20, 128),
                                  (130, 6, 12, 256), (256, 4, 9, 20), (96, 7, 256, 8)])
@pytest.mark.parametrize("boundary", [0, 1])
def test_vmajor_refocus_random_gamma(dims, boundary):
    """Random Gamma, 11 planes (two full groups of 4 and a ragged group of 3, one negative
    alpha), ragged x tiles (W_a = 7, 24, 40, 130), v blocks (H_b = 4 .. 132 across the 128-row
    block), W_a = 256 full width and W_b = 256."""
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=sum(dims) + boundary)
    R = _refocus_vmajor(G, dims, ALPHAS, boundary)
    _assert_planes(R, G, dims, ALPHAS, boundary)


def test_vmajor_refocus_large_slope_fallback():
    """A-axis slopes whose span exceeds the window stage (alpha = 2.9, -2.5 at W_a = 200) run the
    plain staged stage 1 in v-major order; the mixed stack still matches the oracle."""
    dims = (200, 6, 24, 8)
    G = synth.random_gamma(200 * 6, 24 * 8, seed=5)
    al = [0.8, 2.9, 1.0, -2.5, 1.9]
    R = _refocus_vmajor(G, dims, al)
    _assert_planes(R, G, dims, al)


def test_vmajor_integer_shear_bit_exact_rows():
    """Integer shear at alpha = 2 (all t = 0): the window stage 1 must reproduce O(2x, 2y) to the
    fp32 Gamma's precision (every tap weight is 0 or 1)."""
    W, H = 33, 20
    rng = np.random.default_rng(4)
    O = (rng.random((2 * W - 1, 2 * H - 1)) + 0.5).astype(np.float32)
    jj, uu = np.meshgrid(np.arange(W), np.arange(W), indexing="ij")
    mm, vv = np.meshgrid(np.arange(H), np.arange(H), indexing="ij")
    G = np.ascontiguousarray(O[(jj + uu)[None, :, None, :], (mm + vv)[:, None, :, None]].reshape(H * W, H * W))
    R = _refocus_vmajor(G, (W, H, W, H), [2.0])[0]
    _, cnt = oracle.refocus(G, (W, H, W, H), [2.0], return_counts=True)
    ok = cnt[0] > 0
    xs, ys = np.meshgrid(np.arange(W), np.arange(H))
    np.testing.assert_allclose(R[ok], O[2 * xs, 2 * ys][ok], rtol=1e-6)


@pytest.mark.parametrize("boundary", [0, 1])
def test_vmajor_affine_and_fractional_b(boundary):
    """General maps: integral B (window kernel) and fractional B (B resample in v-major order,
    then the window kernel), consecutive planes sharing a B map."""
    dims = (48, 12, 20, 16)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=77 + boundary)
    maps = [[0.7, 0.3, 0.25, 0.0, 1.0, 0.0, 1.3, -0.3, -0.4, 0.0, 1.0, 0.0],
            [1.6, -0.6, 0.0, 0.0, 1.0, 0.0, 0.5, 0.5, 0.0, 0.0, 1.0, 0.0],
            [0.8, 0.2, 0.0, 0.0, 0.9, 0.3, 0.8, 0.2, 0.0, 0.0, 0.8, -0.2],
            [1.2, -0.2, 0.5, 0.0, 0.9, 0.3, 0.9, 0.1, 0.0, 0.0, 0.8, -0.2],
            [1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0, 0.0]]
    R = _refocus_vmajor(G, dims, boundary=boundary, affine=maps)
    _assert_planes(R, G, dims, boundary=boundary, affine=maps)


def test_vmajor_cyclic_shards_sum_to_whole():
    """Block-cyclic row shards (block 2 of 4 ranks): each shard equals the oracle on its rows and
    the shards sum to the whole plane (SURVEY §8(e) load balance)."""
    dims = (40, 16, 12, 8)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=31)
    al = [0.55, 1.0, 1.45, 1.9, 0.8]
    whole = _refocus_vmajor(G, dims, al)
    world, block = 4, 2
    total = np.zeros_like(whole)
    for rank in range(world):
        stride = world * block
        m = np.array([rank * block + (l // block) * stride + l % block for l in range(Ha // world)])
        pix = (m[:, None] * Wa + np.arange(Wa)[None, :]).reshape(-1)
        R = _refocus_vmajor(G[pix], dims, al, row0=rank * block * Wa, rows=pix.size, row_block=block,
                            row_stride=stride)
        Gs = np.zeros_like(G)
        Gs[pix] = G[pix]
        _assert_planes(R, Gs, dims, al)
        total += R
    _assert_planes(total, G, dims, al)       # the shards' sum meets the whole-plane bar


@pytest.mark.parametrize("variant", ["tc", "fp4"])
def test_vmajor_counts_and_gamma_are_a_permutation(variant):
    """Frames -> counts / Gamma in the v-major order equal the row-major context's after the
    B index permutation (same integers, same normalisation), and the planes match the oracle."""
    roi_a, roi_b = (0, 0, 24, 16), (256, 0, 20, 12)
    fr = synth.bernoulli_frames(900, 0.2, seed=61)
    ref = _ctx(roi_a, roi_b, 900, variant=variant, keep_counts=True)
    vm = _ctx(roi_a, roi_b, 900, variant=variant, keep_counts=True, gamma_order="vmajor")
    g_ref, g_vm = ref.new_gamma(), vm.new_gamma()
    for c, g in ((ref, g_ref), (vm, g_vm)):
        c.load_frames(fr)
        c.correlate(g)
    idx = vm.b_index()
    assert sorted(idx.tolist()) == list(range(roi_b[2] * roi_b[3]))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g_vm.cpu().numpy()[:, idx], g_ref.cpu().numpy())
    sr, sv = ref.counts_views(), vm.counts_views()
    np.testing.assert_array_equal(sv[0].cpu().numpy()[:, idx], sr[0].cpu().numpy())
    np.testing.assert_array_equal(sv[2].cpu().numpy()[idx], sr[2].cpu().numpy())
    want = oracle.correlate(fr, roi_a, roi_b)
    np.testing.assert_array_equal(sv[0].cpu().numpy()[:, idx], want["s_ab"])
    al = [0.6, 1.0, 1.7]
    p_vm = vm.new_planes(3)
    vm.refocus(al, g_vm, p_vm)
    torch.cuda.synchronize()
    G = g_ref.cpu().numpy()
    _assert_planes(p_vm.cpu().numpy().astype(np.float64), G, (24, 16, 20, 12), al)


def test_vmajor_repeat_bit_identical():
    """The window stage 1 is deterministic (fixed summation order, no atomics): repeated runs
    give bit-identical planes (guards the stage-release ordering)."""
    dims = (64, 24, 32, 128)
    G = synth.random_gamma(64 * 24, 32 * 128, seed=9)
    al = list(np.linspace(0.5, 2.0, 12))
    ref = _refocus_vmajor(G, dims, al)
    for _ in range(3):
        assert np.array_equal(_refocus_vmajor(G, dims, al), ref)
