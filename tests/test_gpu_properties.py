"""Property-based parity (hypothesis) of the CUDA path against the oracle on random shapes:
random RoIs (any alignment, both arms, any size up to 48 x 24), random frame counts (K tails),
every GEMM variant, and random refocus maps with both boundary policies.  Bounded example
counts keep the GPU tier within a minute."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402

roi = st.tuples(st.integers(0, 200), st.integers(0, 200), st.integers(1, 48), st.integers(1, 24))


@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck))
@given(ra=roi, rb=roi, n=st.integers(1, 700), f=st.floats(0.01, 0.6), seed=st.integers(0, 2**31 - 1),
       variant=st.sampled_from(["tc", "popc", "fp4"]))
def test_random_rois_counts_and_gamma(ra, rb, n, f, seed, variant):
    from paper_2407_20692_b200 import Context
    roi_a = (ra[0], ra[1], ra[2], ra[3])
    roi_b = (256 + rb[0] % 200, rb[1], rb[2], rb[3])
    fr = synth.bernoulli_frames(n, f, seed=seed)
    want = oracle.correlate(fr, roi_a, roi_b)
    ctx = Context(roi_a, roi_b, n, variant=variant, keep_counts=True)
    ctx.load_frames(fr)
    g = ctx.correlate(ctx.new_gamma())
    s_ab, s_a, s_b = ctx.counts_views()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(s_ab.cpu().numpy(), want["s_ab"])
    np.testing.assert_array_equal(s_a.cpu().numpy(), want["s_a"])
    np.testing.assert_array_equal(s_b.cpu().numpy(), want["s_b"])
    G, E = g.cpu().numpy().astype(np.float64), want["gamma"]
    zero = E == 0
    assert np.all(G[zero] == 0)
    assert np.all(np.abs(G - E) <= 1e-6 * np.abs(E))


@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck))
@given(wa=st.integers(2, 40), ha=st.integers(2, 30), wb=st.integers(1, 20), hb=st.integers(1, 12),
       alphas=st.lists(st.floats(0.3, 2.5), min_size=1, max_size=6), boundary=st.sampled_from([0, 1]),
       seed=st.integers(0, 2**31 - 1))
def test_random_refocus(wa, ha, wb, hb, alphas, boundary, seed):
    from paper_2407_20692_b200 import Context
    dims = (wa, ha, wb, hb)
    G = synth.random_gamma(wa * ha, wb * hb, seed=seed)
    ctx = Context((0, 0, wa, ha), (0, 0, wb, hb), 1)
    g = torch.from_numpy(np.ascontiguousarray(G, dtype=np.float32)).cuda()
    planes = ctx.new_planes(len(alphas))
    ctx.refocus(alphas, g, planes, boundary=boundary)
    torch.cuda.synchronize()
    R = planes.cpu().numpy().astype(np.float64)
    Ro = oracle.refocus(G, dims, alphas, boundary=boundary)
    M = oracle.refocus(np.abs(G.astype(np.float64)), dims, alphas, boundary=boundary)
    assert np.all(np.abs(R - Ro) <= 1e-6 * M + 1e-30)


coef = st.floats(-1.5, 1.5)


@settings(max_examples=40, deadline=None, suppress_health_check=list(HealthCheck))
@given(wa=st.integers(2, 24), ha=st.integers(2, 20), wb=st.integers(2, 16), hb=st.integers(2, 10),
       n_planes=st.integers(1, 3), boundary=st.sampled_from([0, 1]), integral_b=st.booleans(),
       route=st.sampled_from(["", "CPI_RESAMPLE_GATHER", "CPI_GENB_DIRECT"]),
       seed=st.integers(0, 2**31 - 1), data=st.data())
def test_random_affine_maps(wa, ha, wb, hb, n_planes, boundary, integral_b, route, seed, data):
    """Random general RefocusMap rows (dx = dy = 0), integral or fractional B, vs the oracle;
    fractional B through the banded or gather B resample, or the direct general-B kernels."""
    import os
    from paper_2407_20692_b200 import Context
    maps = []
    for _ in range(n_planes):
        ax, bx, cx, ay, by, cy = (data.draw(coef) for _ in range(6))
        if integral_b:
            ex, fx, ey, fy = 1.0, 0.0, 1.0, 0.0
        else:
            ex, fx, ey, fy = (data.draw(st.floats(0.3, 1.8)), data.draw(coef), data.draw(st.floats(0.3, 1.8)),
                              data.draw(coef))
        maps.append([ax, bx, cx, 0.0, ex, fx, ay, by, cy, 0.0, ey, fy])
    dims = (wa, ha, wb, hb)
    G = synth.random_gamma(wa * ha, wb * hb, seed=seed)
    ctx = Context((0, 0, wa, ha), (0, 0, wb, hb), 1)
    g = torch.from_numpy(np.ascontiguousarray(G, dtype=np.float32)).cuda()
    planes = ctx.new_planes(n_planes)
    if route:
        os.environ[route] = "1"
    try:
        ctx.refocus(None, g, planes, boundary=boundary, affine=maps)
        torch.cuda.synchronize()
    finally:
        os.environ.pop(route, None)
    R = planes.cpu().numpy().astype(np.float64)
    Ro = oracle.refocus_affine(G, dims, maps, boundary=boundary)
    M = oracle.refocus_affine(np.abs(G.astype(np.float64)), dims, maps, boundary=boundary)
    assert np.all(np.abs(R - Ro) <= 1e-6 * M + 1e-30)


@settings(max_examples=15, deadline=None, suppress_health_check=list(HealthCheck))
@given(h=st.integers(1, 40), w=st.integers(8, 40), n=st.integers(1, 600), variant=st.sampled_from(["tc", "fp4", "popc"]),
       cuts=st.lists(st.integers(1, 8), min_size=0, max_size=4), seed=st.integers(0, 2**31 - 1))
def test_random_row_panels(h, w, n, variant, cuts, seed):
    """cpi_correlate_rows over random aligned panel splits equals cpi_correlate bit for bit."""
    from paper_2407_20692_b200 import Context
    roi_a, roi_b = (0, 0, w, h), (300, 10, 12, 9)
    fr = synth.bernoulli_frames(n, 0.3, seed=seed)
    full = Context(roi_a, roi_b, n, variant=variant, keep_counts=True)
    full.load_frames(fr)
    gf = full.correlate(full.new_gamma())
    part = Context(roi_a, roi_b, n, variant=variant, keep_counts=True)
    al, pa = part.row_align(), part.p_a
    bounds = sorted({min(pa, c * al) for c in cuts} | {0, pa})
    gp = part.new_gamma()
    part.load_frames(fr)
    for r0, r1 in zip(bounds[:-1], bounds[1:]):
        if r1 > r0:
            part.correlate_rows(r0, r1 - r0, gp)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(part.counts_views()[0].cpu().numpy(), full.counts_views()[0].cpu().numpy())
    np.testing.assert_array_equal(gp.cpu().numpy(), gf.cpu().numpy())
