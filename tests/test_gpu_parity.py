"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star):
  * S_a, S_b, S_ab: bit-exact (integers).
  * Gamma (fp32) vs the oracle's exact rational rounded to fp64: |g - G| <= 1e-6 |G|, and
    G == 0 => g == 0 exactly.
  * Refocused planes (fp32): |R - R_o| <= 1e-6 * M + 1e-30 with M(x,y) the oracle's
    refocusing of |Gamma| (mean absolute contribution; M >= |R_o|, = |R_o| when no
    cancellation), stated per output.
"""
import numpy as np
import pytest

import oracle
import synth
from tests._util import pack

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "-m gpu selected but no CUDA device: GPU parity cannot run"
    from paper_2407_20692_b200 import build
    build.build()


def _ctx(roi_a, roi_b, max_frames, **kw):
    from paper_2407_20692_b200 import Context
    return Context(roi_a, roi_b, max_frames, **kw)


def _gpu_sums(frames, roi_a, roi_b, variant="tc", batches=None, width=512, height=256, gamma=True):
    n = frames.shape[0]
    batches = batches or [n]
    ctx = _ctx(roi_a, roi_b, max(max(batches), 1), variant=variant, keep_counts=True,
               width=width, height=height)
    g = ctx.new_gamma() if gamma else None
    off = 0
    for b in batches:
        ctx.load_frames(np.ascontiguousarray(frames[off:off + b]))
        ctx.correlate(g)
        off += b
    s_ab = torch.empty((ctx.p_a, ctx.p_b), dtype=torch.int32, device="cuda")
    s_a = torch.empty(ctx.p_a, dtype=torch.int32, device="cuda")
    s_b = torch.empty(ctx.p_b, dtype=torch.int32, device="cuda")
    n_tot = ctx.get_counts(s_ab, s_a, s_b)
    torch.cuda.synchronize()
    out = dict(s_ab=s_ab.cpu().numpy(), s_a=s_a.cpu().numpy(), s_b=s_b.cpu().numpy(), n=n_tot,
               gamma=g.cpu().numpy() if gamma else None, ctx=ctx)
    return out


def _assert_gamma(g_gpu, g_exact):
    g_gpu = g_gpu.astype(np.float64)
    zero = g_exact == 0
    assert np.all(g_gpu[zero] == 0.0), "exact zeros must stay zero"
    rel = np.abs(g_gpu - g_exact) / np.where(zero, 1.0, np.abs(g_exact))
    assert rel.max() <= 1e-6, f"max rel err {rel.max():.3e}"


def _check_sums(got, want):
    np.testing.assert_array_equal(got["s_a"], want["s_a"])
    np.testing.assert_array_equal(got["s_b"], want["s_b"])
    np.testing.assert_array_equal(got["s_ab"], want["s_ab"])
    assert got["n"] == want["n"]


@pytest.mark.parametrize("variant", ["tc", "popc", "fp4", "bits"])
def test_tiny_config_bit_exact(variant):
    """BASELINE configs[0]: 8x8 rho_a x 4x4 rho_b (non byte-aligned), 1000 frames."""
    fr = synth.bernoulli_frames(1000, 0.05, seed=synth.SEED_ARMS)
    want = oracle.correlate(fr, synth.ROI_TINY_A, synth.ROI_TINY_B)
    got = _gpu_sums(fr, synth.ROI_TINY_A, synth.ROI_TINY_B, variant)
    _check_sums(got, want)
    _assert_gamma(got["gamma"], want["gamma"])


@pytest.mark.parametrize("variant", ["tc", "popc", "fp4", "bits"])
@pytest.mark.parametrize("n", [1, 31, 127, 129, 255, 257, 1000, 2600, 12500])
def test_ragged_tiles_and_k_tails(variant, n):
    """Several M/N tiles with ragged edges (P_a = 1500, P_b = 380) and K tails (N not a
    multiple of 128): zero padding must be inert."""
    roi_a, roi_b = (3, 7, 50, 30), (261, 2, 20, 19)
    fr = synth.bernoulli_frames(n, 0.3, seed=n)
    want = oracle.correlate(fr, roi_a, roi_b)
    got = _gpu_sums(fr, roi_a, roi_b, variant)
    _check_sums(got, want)
    _assert_gamma(got["gamma"], want["gamma"])


@pytest.mark.parametrize("knobs", [{"CPI_GEMM_1CTA": "1"}, {"CPI_GEMM_CACHE": "3"},
                                   {"CPI_GEMM_CACHE": "1", "CPI_GEMM_1CTA": "1"}])
@pytest.mark.parametrize("variant", ["tc", "fp4"])
def test_gemm_knobs(knobs, variant, monkeypatch):
    """GEMM implementation knobs: the 1-CTA int8 kernel (ignored by FP4, which
    always runs CTA pairs) and the L2 cache-policy bits give the same exact sums."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    roi_a, roi_b = (3, 7, 50, 30), (261, 2, 20, 19)
    fr = synth.bernoulli_frames(1300, 0.3, seed=77)
    want = oracle.correlate(fr, roi_a, roi_b)
    got = _gpu_sums(fr, roi_a, roi_b, variant)
    _check_sums(got, want)
    _assert_gamma(got["gamma"], want["gamma"])


@pytest.mark.parametrize("variant", ["tc", "fp4"])
def test_chaotic_light_dense_and_identities(variant):
    """Correlated (speckle) data with exact identities: same RoI on both arms -> S_ab
    symmetric; Gamma diagonal = f(1-f) (exact rational), checked through the GPU path."""
    roi = (10, 20, 40, 24)
    fr = synth.speckle_frames(3000, roi, (300, 20, 40, 24), f=0.3, grain=3, shift_b=(0, 0))
    want = oracle.correlate(fr, roi, roi)
    got = _gpu_sums(fr, roi, roi, variant)
    _check_sums(got, want)
    np.testing.assert_array_equal(got["s_ab"], got["s_ab"].T)
    _assert_gamma(got["gamma"], want["gamma"])


def test_multi_batch_accumulation_and_virtual_ranks():
    """S:235-243 accumulate_chunk: three batches == one batch, bit for bit; and the
    frame-sharded decomposition: G slices in separate contexts, summed,
    equal the single-context sums (the multi-GPU contract, emulated on one GPU)."""
    roi_a, roi_b = (0, 0, 64, 20), (256, 0, 30, 20)
    fr = synth.bernoulli_frames(3000, 0.1, seed=5)
    one = _gpu_sums(fr, roi_a, roi_b, "tc")
    three = _gpu_sums(fr, roi_a, roi_b, "tc", batches=[1000, 1, 1999])
    three_f4 = _gpu_sums(fr, roi_a, roi_b, "fp4", batches=[1000, 1, 1999])
    _check_sums(three_f4, one)
    np.testing.assert_array_equal(three_f4["gamma"], one["gamma"])
    three_bits = _gpu_sums(fr, roi_a, roi_b, "bits", batches=[1000, 1, 1999])   # f1: unpacked inside the GEMM
    _check_sums(three_bits, one)
    np.testing.assert_array_equal(three_bits["gamma"], one["gamma"])
    _check_sums(three, one)
    np.testing.assert_array_equal(three["gamma"], one["gamma"])
    parts = [_gpu_sums(fr[a:b], roi_a, roi_b, "tc", gamma=False) for a, b in [(0, 700), (700, 2048), (2048, 3000)]]
    np.testing.assert_array_equal(sum(p["s_ab"] for p in parts), one["s_ab"])
    np.testing.assert_array_equal(sum(p["s_a"] for p in parts), one["s_a"])


def test_device_frames_in_place_and_finalize():
    """CPI_DEVICE frames are used in place; cpi_finalize from kept counts equals the fused
    epilogue's Gamma bit for bit; cpi_finalize_counts of a row shard equals its rows."""
    roi_a, roi_b = (5, 5, 33, 17), (300, 1, 12, 12)
    fr = synth.bernoulli_frames(777, 0.2, seed=9)
    ctx = _ctx(roi_a, roi_b, 777, keep_counts=True)
    d = torch.from_numpy(fr).cuda()
    ctx.load_frames(d)
    g1 = ctx.new_gamma()
    ctx.correlate(g1)
    g2 = ctx.new_gamma()
    n = ctx.finalize(g2)
    assert n == 777
    assert torch.equal(g1, g2)
    s_ab = torch.empty((ctx.p_a, ctx.p_b), dtype=torch.int32, device="cuda")
    s_a = torch.empty(ctx.p_a, dtype=torch.int32, device="cuda")
    s_b = torch.empty(ctx.p_b, dtype=torch.int32, device="cuda")
    ctx.get_counts(s_ab, s_a, s_b)
    rows = torch.empty((66, ctx.p_b), dtype=torch.float32, device="cuda")
    ctx.finalize_counts(s_ab[33:99].contiguous(), 33, s_a, s_b, n, rows)
    assert torch.equal(rows, g1[33:99])


def test_error_paths_on_device():
    from paper_2407_20692_b200 import CpiError
    ctx = _ctx((0, 0, 8, 8), (8, 0, 8, 8), 10)
    with pytest.raises(CpiError, match="STATE"):
        ctx.correlate(ctx.new_gamma())            # nothing loaded
    with pytest.raises(CpiError, match="CAPACITY"):
        ctx.load_frames(np.zeros((11, 256, 64), np.uint8))
    with pytest.raises(CpiError, match="SIZE_MISMATCH"):
        ctx.load_frames(np.zeros(16385, np.uint8))
    ctx.load_frames(np.zeros((0, 256, 64), np.uint8))
    with pytest.raises(CpiError, match="ZERO_FRAMES"):
        ctx.correlate(ctx.new_gamma())
    ctx.load_frames(np.zeros((3, 256, 64), np.uint8))
    g = ctx.new_gamma()
    ctx.correlate(g)
    assert torch.all(g == 0)
    with pytest.raises(CpiError, match="STATE"):
        ctx.load_frames(np.zeros((3, 256, 64), np.uint8))
        ctx.correlate(g)                          # second batch without KEEP_COUNTS
    planes = ctx.new_planes(1)
    with pytest.raises(CpiError, match="DEGENERATE_ALPHA"):
        ctx.refocus([0.0], g, planes)
    with pytest.raises(CpiError, match="EMPTY_ANGULAR_GRID"):
        ctx.refocus([], g, planes)


# ------------------------------------------------------------------ refocusing ---------

def _refocus_gpu(G, dims, alphas, boundary=0, row0=0, rows=None):
    Wa, Ha, Wb, Hb = dims
    ctx = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1)
    g = torch.from_numpy(np.ascontiguousarray(G, dtype=np.float32)).cuda()
    planes = ctx.new_planes(len(alphas))
    ctx.refocus(alphas, g[row0:] if row0 else g, planes, row0=row0, rows=rows, boundary=boundary)
    torch.cuda.synchronize()
    return planes.cpu().numpy().astype(np.float64)


def _assert_planes(R, G, dims, alphas, boundary=0):
    Ro = oracle.refocus(G, dims, alphas, boundary=boundary)
    M = oracle.refocus(np.abs(G.astype(np.float64)), dims, alphas, boundary=boundary)
    err = np.abs(R - Ro)
    assert np.all(err <= 1e-6 * M + 1e-30), f"max err/M {np.max(err / np.maximum(M, 1e-300)):.3e}"


@pytest.mark.parametrize("dims", [(24, 20, 16, 12), (7, 5, 9, 3), (40, 33, 37, 10)])
@pytest.mark.parametrize("boundary", [0, 1])
def test_refocus_random_gamma(dims, boundary):
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=sum(dims))
    alphas = [0.5, 0.75, 1.0, 1.3, 2.0, -0.6]
    R = _refocus_gpu(G, dims, alphas, boundary)
    _assert_planes(R, G, dims, alphas, boundary)


def test_refocus_integer_shear_and_ramp():
    """Closed forms through the GPU path: integer shear at alpha=2 reproduces O(2x,2y)
    (fp32 taps; within 1e-6 rel), the sheared ramp reproduces a + b alpha x' + c alpha y'."""
    W, H = 33, 21
    rng = np.random.default_rng(4)
    O = (rng.random((2 * W - 1, 2 * H - 1)) + 0.5).astype(np.float32)
    jj, uu = np.meshgrid(np.arange(W), np.arange(W), indexing="ij")
    mm, vv = np.meshgrid(np.arange(H), np.arange(H), indexing="ij")
    G = np.ascontiguousarray(O[(jj + uu)[None, :, None, :], (mm + vv)[:, None, :, None]].reshape(H * W, H * W))
    R = _refocus_gpu(G, (W, H, W, H), [2.0])[0]
    xs, ys = np.meshgrid(np.arange(W), np.arange(H))
    _, cnt = oracle.refocus(G, (W, H, W, H), [2.0], return_counts=True)
    ok = cnt[0] > 0
    np.testing.assert_allclose(R[ok], O[2 * xs, 2 * ys][ok], rtol=1e-6)
    assert np.all(R[~ok] == 0)
    # sheared ramp
    Wa, Ha, Wb, Hb = 30, 26, 22, 14
    for alpha in (0.6, 1.4):
        s = 1 - alpha
        j = np.arange(Wa) - (Wa - 1) / 2
        m = np.arange(Ha) - (Ha - 1) / 2
        u = np.arange(Wb) - (Wb - 1) / 2
        v = np.arange(Hb) - (Hb - 1) / 2
        G4 = (0.02 + 0.001 * (j[None, :, None, None] - s * u[None, None, None, :])
              - 0.0007 * (m[:, None, None, None] - s * v[None, None, :, None]))
        R = _refocus_gpu(G4.reshape(Ha * Wa, Hb * Wb), (Wa, Ha, Wb, Hb), [alpha])[0]
        _, cnt = oracle.refocus(G4.reshape(Ha * Wa, Hb * Wb), (Wa, Ha, Wb, Hb), [alpha], return_counts=True)
        expect = 0.02 + 0.001 * alpha * j[None, :] - 0.0007 * alpha * m[:, None]
        ok = cnt[0] > 0
        M = oracle.refocus(np.abs(G4.reshape(Ha * Wa, Hb * Wb)), (Wa, Ha, Wb, Hb), [alpha])[0]
        assert np.all(np.abs(R[ok] - expect[ok]) <= 1e-6 * M[ok])     # closed form, 1e-6 M bar


def test_refocus_row_shards_sum_to_whole():
    """Row-sharded refocus: the planes of A-row shards add up to the plane of
    the whole Gamma (linearity), so an all-reduce of shard planes is the multi-GPU merge."""
    dims = (20, 16, 12, 10)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=3)
    al = [0.7, 1.0, 1.6]
    whole = _refocus_gpu(G, dims, al)
    parts = sum(_refocus_gpu(G, dims, al, row0=r0 * Wa, rows=(r1 - r0) * Wa) for r0, r1 in [(0, 5), (5, 11), (11, 16)])
    _assert_planes(parts, G, dims, al)
    _assert_planes(whole, G, dims, al)


def test_end_to_end_frames_to_planes_alpha1_ghost():
    """frames -> GPU Gamma -> GPU planes; alpha = 1 equals the direct ghost image computed
    from the frames (closed form), and every plane matches the oracle pipeline."""
    roi_a, roi_b = (0, 0, 32, 24), (256, 0, 20, 16)
    fr = synth.bernoulli_frames(4000, 0.1, seed=12)
    ctx = _ctx(roi_a, roi_b, 4000)
    ctx.load_frames(fr)
    g = ctx.correlate(ctx.new_gamma())
    al = [0.5, 1.0, 1.5]
    planes = ctx.new_planes(3)
    ctx.refocus(al, g, planes)
    torch.cuda.synchronize()
    R = planes.cpu().numpy().astype(np.float64)
    want = oracle.correlate(fr, roi_a, roi_b)
    dims = (32, 24, 20, 16)
    _assert_planes(R, want["gamma"], dims, al)
    from tests._util import unpack_np
    A = unpack_np(fr, roi_a).astype(np.int64)
    nB = unpack_np(fr, roi_b).astype(np.int64).sum(1)
    n = 4000
    ghost = (n * (A.T @ nB) - A.sum(0) * nB.sum()) / (n * n * 320.0)
    M = oracle.refocus(np.abs(want["gamma"]), dims, [1.0])[0].reshape(-1)
    assert np.all(np.abs(R[1].reshape(-1) - ghost) <= 1e-6 * M + 1e-30)


@pytest.mark.parametrize("fuse", [1, 2, 3, 4])
def test_refocus_fused_plane_groups(fuse, monkeypatch):
    """The TMA stage 1 fuses F planes per pass over Gamma (CPI_REFOCUS_FUSE); every group size,
    including a ragged last group (7 planes), matches the oracle per plane.  The alpha set spans
    alpha < 1 (all samples valid, narrow j spans), alpha = 1 and alpha > 1 (skipped samples,
    warp-level x-block skipping)."""
    monkeypatch.setenv("CPI_REFOCUS_FUSE", str(fuse))
    dims = (64, 40, 48, 24)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=40 + fuse)
    alphas = [0.5, 0.77, 1.0, 1.31, 1.62, 2.0, 2.9]
    R = _refocus_gpu(G, dims, alphas)
    _assert_planes(R, G, dims, alphas)


@pytest.mark.parametrize("fuse,n_planes", [(4, 70), (3, 50), (1, 9)])
def test_refocus_many_planes_fused_groups(fuse, n_planes, monkeypatch):
    """Long stacks in fused groups of F planes (ragged last group): every plane matches the
    oracle and equals the same plane refocused alone, bit for bit (a plane's taps, their order
    and its fp32 / fp64 sums do not depend on the planes it shares a pass over Gamma with)."""
    monkeypatch.setenv("CPI_REFOCUS_FUSE", str(fuse))
    dims = (48, 20, 32, 16)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=70 + fuse)
    alphas = list(np.linspace(0.5, 2.0, n_planes))
    R = _refocus_gpu(G, dims, alphas)
    _assert_planes(R, G, dims, alphas)
    monkeypatch.setenv("CPI_REFOCUS_FUSE", "1")
    for p in (0, n_planes // 2, n_planes - 1):
        np.testing.assert_array_equal(_refocus_gpu(G, dims, [alphas[p]])[0], R[p])


@pytest.mark.parametrize("knobs", [{"CPI_STAGE1_SIMPLE": "1"}, {"CPI_STAGE2_SIMPLE": "1"},
                                   {"CPI_STAGE1_SIMPLE": "1", "CPI_STAGE2_SIMPLE": "1"}, {"CPI_S1_NOSKIP": "1"},
                                   {"CPI_S1_L2PROMO": "0"}, {"CPI_S1_L2PROMO": "128"}, {"CPI_REFOCUS_FUSE": "3"}])
@pytest.mark.parametrize("boundary", [0, 1])
def test_refocus_fallback_kernels(knobs, boundary, monkeypatch):
    """The fallback kernels (plain stage 1 for W_a > 256, W_b % 4 != 0 or unaligned Gamma;
    warp-per-pixel stage 2 for H_a > 256) and the no-skip stage 1 agree with the oracle."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    dims = (40, 33, 36, 10)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=5)
    alphas = [0.5, 1.0, 1.3, 2.0]
    R = _refocus_gpu(G, dims, alphas, boundary=boundary)
    _assert_planes(R, G, dims, alphas, boundary=boundary)


def test_refocus_repeat_bit_identical():
    """Every refocus kernel is deterministic (fixed summation order, no atomics in the value
    path), so repeated runs must agree bit for bit.  Catches pipeline races: e.g. a stage
    released to the TMA producer before its shared-memory loads have returned (the reads are
    generic-proxy, the refill async-proxy).  W_a = 256 exercises the full-x kernel; alphas
    near 2 maximise skipped samples."""
    dims = (256, 64, 256, 64)
    Wa, Ha, Wb, Hb = dims
    ctx = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1)
    g = torch.from_numpy(synth.random_gamma(Wa * Ha, Wb * Hb, seed=1)).cuda()
    al = synth.alpha_grid(64)
    ref = ctx.new_planes(64)
    ctx.refocus(al, g, ref)
    for _ in range(3):
        p = ctx.new_planes(64)
        ctx.refocus(al, g, p)
        torch.cuda.synchronize()
        assert torch.equal(p, ref)
    same = ctx.new_planes(4)
    ctx.refocus([1.9] * 4, g, same)
    torch.cuda.synchronize()
    for s in range(1, 4):
        assert torch.equal(same[s], same[0])


@pytest.mark.parametrize("variant", ["tc", "popc", "fp4"])
def test_correlate_rows_panels_match_full(variant):
    """cpi_correlate_rows (SURVEY §8(e) panelised GEMM): covering A pixels with aligned row
    panels, over two accumulated batches with different panel splits, gives counts and
    Gamma bit-identical to cpi_correlate, and the borrowed count views alias the library's."""
    roi_a, roi_b = (3, 5, 64, 20), (260, 7, 24, 10)          # P_a = 1280 (5 x 256 rows), P_b = 240
    fr = synth.bernoulli_frames(700, 0.2, seed=44)
    full = _gpu_sums(fr, roi_a, roi_b, variant=variant, batches=[300, 400])
    ctx = _ctx(roi_a, roi_b, 400, variant=variant, keep_counts=True)
    al = ctx.row_align()
    assert al > 0 and ctx.p_a % al == 0
    g = ctx.new_gamma()
    splits = [[(0, al), (al, 3 * al), (3 * al, ctx.p_a - 3 * al)], [(0, ctx.p_a)]]
    for (lo, hi), panels in zip([(0, 300), (300, 700)], splits):
        ctx.load_frames(np.ascontiguousarray(fr[lo:hi]))
        for r0, rows in panels[::-1]:                         # any order
            ctx.correlate_rows(r0, rows, g)
    s_ab, s_a, s_b = ctx.counts_views()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(s_ab.cpu().numpy(), full["s_ab"])
    np.testing.assert_array_equal(s_a.cpu().numpy(), full["s_a"])
    np.testing.assert_array_equal(s_b.cpu().numpy(), full["s_b"])
    np.testing.assert_array_equal(g.cpu().numpy(), full["gamma"])
    # errors: misaligned panel, whole-batch correlate after a panel of the same batch
    from paper_2407_20692_b200 import CpiError
    ctx.load_frames(np.ascontiguousarray(fr[:10]))
    with pytest.raises(CpiError, match="INVALID_ARG"):
        ctx.correlate_rows(1, al)
    ctx.correlate_rows(0, al)
    with pytest.raises(CpiError, match="STATE"):
        ctx.correlate(g)


@pytest.mark.parametrize("block", [1, 2])
def test_refocus_block_cyclic_shards(block):
    """Block-cyclic A-row shards (cpi_refocus_spec row_block / row_stride, the multi-GPU
    ownership of parallel.ShardPlan): each shard's planes equal the oracle's planes of Gamma
    restricted to the shard's rows, and the shards of all ranks add up to the whole plane."""
    dims = (20, 16, 12, 12)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=9)
    al = [0.6, 1.0, 1.7]
    world = 4
    whole = _refocus_gpu(G, dims, al)
    total = np.zeros_like(whole)
    ctx = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1)
    for rank in range(world):
        stride = world * block
        m = np.array([rank * block + (l // block) * stride + l % block for l in range(Ha // world)])
        pix = (m[:, None] * Wa + np.arange(Wa)[None, :]).reshape(-1)
        rows_g = torch.from_numpy(np.ascontiguousarray(G[pix], dtype=np.float32)).cuda()
        planes = ctx.new_planes(len(al))
        ctx.refocus(al, rows_g, planes, row0=rank * block * Wa, rows=pix.size, row_block=block, row_stride=stride)
        torch.cuda.synchronize()
        R = planes.cpu().numpy().astype(np.float64)
        Gs = np.zeros_like(G)
        Gs[pix] = G[pix]
        Ro = oracle.refocus(Gs, dims, al)
        M = oracle.refocus(np.abs(Gs.astype(np.float64)), dims, al)
        assert np.all(np.abs(R - Ro) <= 1e-6 * M + 1e-30)
        total += R
    _assert_planes(total, G, dims, al)       # the shards' sum meets the whole-plane bar


@pytest.mark.parametrize("variant,roi_b", [("tc", (256, 0, 16, 12)), ("fp4", (256, 0, 24, 10)),
                                            ("popc", (260, 3, 40, 6))])
def test_gamma_ublocked_layout(variant, roi_b):
    """CPI_GAMMA_UBLOCKED: B pixels in u-blocked order everywhere (S_b, S_ab and Gamma columns,
    fused epilogue, panels, cpi_finalize, cpi_finalize_counts) hold exactly the row-major
    values at the permuted indices, and refocusing gives planes bit-identical to the
    row-major path."""
    roi_a = (0, 0, 24, 16)
    fr = synth.bernoulli_frames(900, 0.2, seed=61)
    ref = _ctx(roi_a, roi_b, 900, variant=variant, keep_counts=True)
    blk = _ctx(roi_a, roi_b, 900, variant=variant, keep_counts=True, gamma_blocked=True)
    g_ref, g_blk = ref.new_gamma(), blk.new_gamma()
    for c, g in ((ref, g_ref), (blk, g_blk)):
        c.load_frames(fr)
        c.correlate(g)
    idx = blk.b_index()
    assert sorted(idx.tolist()) == list(range(roi_b[2] * roi_b[3]))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g_blk.cpu().numpy()[:, idx], g_ref.cpu().numpy())
    sr, sb = ref.counts_views(), blk.counts_views()
    np.testing.assert_array_equal(sb[0].cpu().numpy()[:, idx], sr[0].cpu().numpy())
    np.testing.assert_array_equal(sb[1].cpu().numpy(), sr[1].cpu().numpy())
    np.testing.assert_array_equal(sb[2].cpu().numpy()[idx], sr[2].cpu().numpy())
    al = [0.6, 1.0, 1.7]
    p_ref, p_blk = ref.new_planes(3), blk.new_planes(3)
    ref.refocus(al, g_ref, p_ref)
    blk.refocus(al, g_blk, p_blk)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(p_blk.cpu().numpy(), p_ref.cpu().numpy())
    # cpi_finalize and cpi_finalize_counts on the blocked sums
    for c in (ref, blk):
        c.load_frames(fr[:10])
        c.correlate(None)
    g2, g2r, g3 = blk.new_gamma(), ref.new_gamma(), blk.new_gamma()
    blk.finalize(g2)
    ref.finalize(g2r)
    s_ab, s_a, s_b = blk.counts_views()
    blk.finalize_counts(s_ab, 0, s_a, s_b, 910, g3)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g2.cpu().numpy()[:, idx], g2r.cpu().numpy())
    np.testing.assert_array_equal(g3.cpu().numpy(), g2.cpu().numpy())


@pytest.mark.parametrize("boundary", [0, 1])
def test_refocus_affine_maps(boundary):
    """General RefocusMap rows (cpi_refocus_spec.affine) with integral B coordinates:
    per-plane A-axis maps (a, b, c) on x and y, vs the oracle's general 16-corner refocus; the
    default map written as affine rows is bit-identical to the alphas path; fractional B
    coordinates are refused (CPI_ERR_UNSUPPORTED)."""
    dims = (24, 20, 16, 12)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=17)
    maps = [[0.7, 0.3, 0.25, 0.0, 1.0, 0.0, 1.3, -0.3, -0.4, 0.0, 1.0, 0.0],
            [1.6, -0.45, -1.5, 0.0, 1.0, 0.0, 0.55, 0.5, 2.0, 0.0, 1.0, 0.0],
            [1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0, 0.0],
            [2.0, -1.0, 0.5, 0.0, 1.0, 0.0, -0.8, 1.2, 3.0, 0.0, 1.0, 0.0],
            [0.5, 0.5, 0.0, 0.0, 1.0, 0.0, 0.5, 0.5, 0.0, 0.0, 1.0, 0.0],
            [1.2, 0.1, -0.7, 0.0, 1.0, 0.0, 0.9, 0.0, 0.3, 0.0, 1.0, 0.0]]
    ctx = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1)
    g = torch.from_numpy(np.ascontiguousarray(G, dtype=np.float32)).cuda()
    planes = ctx.new_planes(len(maps))
    ctx.refocus(None, g, planes, boundary=boundary, affine=maps)
    torch.cuda.synchronize()
    R = planes.cpu().numpy().astype(np.float64)
    Ro = oracle.refocus_affine(G, dims, maps, boundary=boundary)
    M = oracle.refocus_affine(np.abs(G.astype(np.float64)), dims, maps, boundary=boundary)
    assert np.all(np.abs(R - Ro) <= 1e-6 * M + 1e-30), np.max(np.abs(R - Ro) / np.maximum(M, 1e-300))
    al = [0.5, 1.0, 1.45]
    p1, p2 = ctx.new_planes(3), ctx.new_planes(3)
    ctx.refocus(al, g, p1, boundary=boundary)
    ctx.refocus(None, g, p2, boundary=boundary, affine=[oracle.default_map(a) for a in al])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(p2.cpu().numpy(), p1.cpu().numpy())


@pytest.mark.parametrize("boundary", [0, 1])
@pytest.mark.parametrize("dims", [(24, 20, 16, 12), (40, 12, 170, 9), (9, 33, 6, 200)])
def test_refocus_output_dependent_b(boundary, dims):
    """General maps whose B coordinates depend on the output pixel (dx, dy != 0, all
    twelve coefficients free) through refocus_gen.cu vs the oracle's 16-corner refocus, incl.
    B RoIs wider than one shared-memory column window (170, 200 > 160) and mixed stacks (a
    default-map plane evaluated by the same route); row shards; the u-blocked order refuses."""
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=sum(dims))
    maps = [[1.0, 0.0, 0.0, 0.1, 1.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0, 0.0],
            [0.7, 0.3, 0.25, -0.2, 0.9, 0.4, 1.3, -0.3, -0.4, 0.35, 1.1, -0.6],
            [1.6, -0.45, -1.5, 0.5, 0.5, 0.0, 0.55, 0.5, 2.0, -0.5, 0.75, 1.5],
            oracle.default_map(1.2),
            [-0.8, 1.2, 3.0, 1.0, 0.0, 0.0, 2.0, -1.0, 0.5, 0.05, 1.0, 0.0]]
    ctx = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1)
    g = torch.from_numpy(np.ascontiguousarray(G, dtype=np.float32)).cuda()
    planes = ctx.new_planes(len(maps))
    ctx.refocus(None, g, planes, boundary=boundary, affine=maps)
    torch.cuda.synchronize()
    R = planes.cpu().numpy().astype(np.float64)
    Ro = oracle.refocus_affine(G, dims, maps, boundary=boundary)
    M = oracle.refocus_affine(np.abs(G.astype(np.float64)), dims, maps, boundary=boundary)
    assert np.all(np.abs(R - Ro) <= 1e-6 * M + 1e-30), np.max(np.abs(R - Ro) / np.maximum(M, 1e-300))
    # contiguous row shards sum to the whole
    r1 = Ha // 3
    parts = np.zeros_like(R)
    for a, b in [(0, r1), (r1, Ha)]:
        pp = ctx.new_planes(len(maps))
        ctx.refocus(None, g[a * Wa:], pp, row0=a * Wa, rows=(b - a) * Wa, boundary=boundary, affine=maps)
        torch.cuda.synchronize()
        parts += pp.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(parts - Ro) <= 1e-6 * M + 1e-30)   # M is additive over row shards
    if Wb % 8 == 0:
        from paper_2407_20692_b200 import CpiError
        ub = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1, gamma_order="ublocked")
        with pytest.raises(CpiError, match="UNSUPPORTED"):
            ub.refocus(None, g, planes, affine=maps)


@pytest.mark.parametrize("boundary", [0, 1])
@pytest.mark.parametrize("route", ["band", "gather", "direct"])
def test_refocus_affine_fractional_b(boundary, route, monkeypatch):
    """General maps with fractional B coordinates (ex, fx, ey, fy arbitrary; dx = dy = 0) vs the
    oracle's 16-corner refocus, 1e-6 M.  Default route: Gamma resampled onto the B lattice once
    per distinct B map (planes 0-2 share one and run as one fused group, plane 7 repeats it after
    other maps), then the separable fast path; the resample runs banded in shared memory, or as
    a gather (CPI_RESAMPLE_GATHER, and always for |ey| > 2.4 such as plane 9's); direct = the
    general-B kernels (CPI_GENB_DIRECT)."""
    if route == "direct":
        monkeypatch.setenv("CPI_GENB_DIRECT", "1")
    elif route == "gather":
        monkeypatch.setenv("CPI_RESAMPLE_GATHER", "1")
    dims = (24, 20, 16, 12)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=23)
    maps = [[0.7, 0.3, 0.25, 0.0, 0.5, -0.3, 1.3, -0.3, -0.4, 0.0, 0.8, 0.2],
            [1.1, -0.1, 0.0, 0.0, 0.5, -0.3, 0.9, 0.1, 0.3, 0.0, 0.8, 0.2],
            [0.6, 0.4, -0.2, 0.0, 0.5, -0.3, 1.0, 0.0, 0.0, 0.0, 0.8, 0.2],
            [1.0, 0.0, 0.0, 0.0, 0.75, 0.1, 0.9, 0.1, 0.0, 0.0, 1.1, 0.0],
            [1.6, -0.45, -1.5, 0.0, 1.25, 0.5, 0.55, 0.5, 2.0, 0.0, 0.6, -1.0],
            [2.0, -1.0, 0.5, 0.0, -0.9, 0.0, 0.5, 0.5, 0.0, 0.0, 1.9, 0.3],
            [0.8, 0.2, 0.0, 0.0, 1.0, 0.0, 1.2, -0.2, 0.0, 0.0, 1.0, 0.0],   # integral B in a mixed call
            [0.9, 0.1, 0.1, 0.0, 0.5, -0.3, 0.7, 0.3, 0.0, 0.0, 0.8, 0.2],
            [1.0, 0.0, 0.0, 0.0, 1.0, 2.0, 1.0, 0.0, 0.0, 0.0, 1.0, -1.0],   # integer B shift
            [0.9, 0.1, 0.0, 0.0, -0.6, 0.2, 1.1, -0.1, 0.0, 0.0, -3.0, 0.4]]   # |ey| > 2.4: gather form
    ctx = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1)
    g = torch.from_numpy(np.ascontiguousarray(G, dtype=np.float32)).cuda()
    planes = ctx.new_planes(len(maps))
    ctx.refocus(None, g, planes, boundary=boundary, affine=maps)
    torch.cuda.synchronize()
    R = planes.cpu().numpy().astype(np.float64)
    Ro = oracle.refocus_affine(G, dims, maps, boundary=boundary)
    M = oracle.refocus_affine(np.abs(G.astype(np.float64)), dims, maps, boundary=boundary)
    assert np.all(np.abs(R - Ro) <= 1e-6 * M + 1e-30), np.max(np.abs(R - Ro) / np.maximum(M, 1e-300))


@pytest.mark.parametrize("boundary", [0, 1])
def test_refocus_fractional_b_ublocked_block_cyclic(boundary):
    """Fractional B through the resample route on u-blocked Gamma columns and block-cyclic
    A-row shards (the multi-GPU layout): each shard matches the oracle on Gamma restricted to
    its rows, and the shards add up to the unsharded row-major result."""
    dims = (24, 16, 16, 12)
    Wa, Ha, Wb, Hb = dims
    G = synth.random_gamma(Wa * Ha, Wb * Hb, seed=29)
    maps = [[0.7, 0.3, 0.25, 0.0, 0.5, -0.3, 1.3, -0.3, -0.4, 0.0, 0.8, 0.2],
            [1.2, -0.2, 0.0, 0.0, 0.5, -0.3, 0.8, 0.2, 0.0, 0.0, 0.8, 0.2],
            [1.6, -0.45, -1.5, 0.0, 1.25, 0.5, 0.55, 0.5, 2.0, 0.0, 0.6, -1.0]]
    row = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1)
    whole = row.new_planes(len(maps))
    row.refocus(None, torch.from_numpy(np.ascontiguousarray(G, dtype=np.float32)).cuda(), whole,
                boundary=boundary, affine=maps)
    blk = _ctx((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1, gamma_blocked=True)
    idx = blk.b_index()
    world, block = 4, 2
    total = np.zeros((len(maps), Ha, Wa))
    for rank in range(world):
        stride = world * block
        m = np.array([rank * block + (l // block) * stride + l % block for l in range(Ha // world)])
        pix = (m[:, None] * Wa + np.arange(Wa)[None, :]).reshape(-1)
        Gb = np.empty((pix.size, Wb * Hb), dtype=np.float32)
        Gb[:, idx] = G[pix]
        planes = blk.new_planes(len(maps))
        blk.refocus(None, torch.from_numpy(Gb).cuda(), planes, boundary=boundary, affine=maps,
                    row0=rank * block * Wa, rows=pix.size, row_block=block, row_stride=stride)
        torch.cuda.synchronize()
        R = planes.cpu().numpy().astype(np.float64)
        Gs = np.zeros_like(G)
        Gs[pix] = G[pix]
        Ro = oracle.refocus_affine(Gs, dims, maps, boundary=boundary)
        M = oracle.refocus_affine(np.abs(Gs.astype(np.float64)), dims, maps, boundary=boundary)
        assert np.all(np.abs(R - Ro) <= 1e-6 * M + 1e-30), np.max(np.abs(R - Ro) / np.maximum(M, 1e-300))
        total += R
    torch.cuda.synchronize()
    Rw = oracle.refocus_affine(G, dims, maps, boundary=boundary)
    Mw = oracle.refocus_affine(np.abs(G.astype(np.float64)), dims, maps, boundary=boundary)
    assert np.all(np.abs(total - Rw) <= 1e-6 * Mw + 1e-30)   # the shards' sum meets the whole-plane bar


def test_refocus_from_current_totals():
    """cpi_refocus with gamma_dev = NULL (SURVEY §8(b) CPI_FROM_COUNTS) refocuses the context's
    current totals: the fused Gamma of the last correlate, or Gamma finalised from the kept
    counts after further batches -- bit-identical to passing that Gamma explicitly."""
    from paper_2407_20692_b200 import CpiError
    roi_a, roi_b = (0, 0, 32, 24), (256, 0, 20, 16)
    fr = synth.bernoulli_frames(1500, 0.1, seed=71)
    al = [0.6, 1.0, 1.4]
    ctx = _ctx(roi_a, roi_b, 1000, keep_counts=True)
    g = ctx.new_gamma()
    ctx.load_frames(fr[:1000])
    ctx.correlate(g)
    p_none, p_expl = ctx.new_planes(3), ctx.new_planes(3)
    ctx.refocus(al, None, p_none)
    ctx.refocus(al, g, p_expl)
    ctx.load_frames(fr[1000:])
    ctx.correlate(None)                       # totals move on; Gamma now only in the counts
    p2_none = ctx.new_planes(3)
    ctx.refocus(al, None, p2_none)
    g2 = ctx.new_gamma()
    ctx.finalize(g2)
    p2_expl = ctx.new_planes(3)
    ctx.refocus(al, g2, p2_expl)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(p_none.cpu().numpy(), p_expl.cpu().numpy())
    np.testing.assert_array_equal(p2_none.cpu().numpy(), p2_expl.cpu().numpy())
    want = oracle.correlate(fr, roi_a, roi_b)
    _assert_planes(p2_none.cpu().numpy().astype(np.float64), want["gamma"], (32, 24, 20, 16), al)
    bare = _ctx(roi_a, roi_b, 100)
    with pytest.raises(CpiError, match="ZERO_FRAMES|STATE"):
        bare.refocus(al, None, bare.new_planes(3))


@pytest.mark.parametrize("variant", ["tc", "fp4", "popc"])
def test_msb_first_and_unaligned_rois(variant):
    """bit_order = CPI_MSB_FIRST (S:110 configurable flag) with RoIs that start and end inside
    bytes: sums bit-exact vs the oracle reading the same bit order."""
    from paper_2407_20692_b200 import Context, _lib
    roi_a, roi_b = (5, 3, 27, 9), (301, 250, 19, 6)
    fr = synth.bernoulli_frames(777, 0.25, seed=19)
    want = oracle.correlate(fr, roi_a, roi_b, msb=True)
    ctx = Context(roi_a, roi_b, 777, variant=variant, keep_counts=True, bit_order=_lib.CPI_MSB_FIRST)
    ctx.load_frames(fr)
    g = ctx.correlate(ctx.new_gamma())
    s_ab, s_a, s_b = ctx.counts_views()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(s_ab.cpu().numpy(), want["s_ab"])
    np.testing.assert_array_equal(s_a.cpu().numpy(), want["s_a"])
    np.testing.assert_array_equal(s_b.cpu().numpy(), want["s_b"])
    _assert_gamma(g.cpu().numpy(), want["gamma"])
