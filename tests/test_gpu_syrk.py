"""Symmetric pair sums (SYRK): with roi_a == roi_b one expanded operand serves
both arms, the CTA-pair GEMM computes only the tiles that touch the upper triangle and the
epilogue mirrors each element (r, c > r) to (c, r).  S_ab is symmetric by Eq. (1) (P:100-102:
A^i_p B^i_q with A = B), so the result must equal the full GEMM's bit for bit."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(autouse=True)
def _syrk_on(monkeypatch):
    monkeypatch.setenv("CPI_SYRK", "1")   # opt-in knob


def _run(roi, frames, variant, batches=1, env=None, monkeypatch=None, rows_panels=None):
    from paper_2407_20692_b200 import Context
    if env and monkeypatch:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
    n = frames.shape[0]
    c = Context(roi, roi, n, variant=variant, keep_counts=True)
    g = c.new_gamma()
    off = 0
    for b in range(batches):
        part = frames[off:off + n // batches if b < batches - 1 else n]
        off += part.shape[0]
        c.load_frames(np.ascontiguousarray(part))
        if rows_panels:
            for r0 in range(0, c.p_a, rows_panels):
                c.correlate_rows(r0, min(rows_panels, c.p_a - r0), g)
        else:
            c.correlate(g)
    s_ab, s_a, s_b = c.counts_views()
    torch.cuda.synchronize()
    out = (s_ab.cpu().numpy(), s_a.cpu().numpy(), s_b.cpu().numpy(), g.cpu().numpy())
    c.close()
    return out


@pytest.mark.parametrize("roi", [(0, 0, 32, 24), (3, 5, 37, 19), (0, 0, 64, 40), (0, 0, 512, 2)])
@pytest.mark.parametrize("variant", ["tc", "fp4"])
def test_syrk_matches_oracle(roi, variant):
    """Ragged sizes around the 256-row / 224-column tiles (P = 768 .. 2560, 1024 as 2 rows of the
    whole frame width), two batches (mirrored accumulation of kept counts)."""
    frames = synth.bernoulli_frames(700, 0.25, seed=sum(roi) + len(variant))
    s_ab, s_a, s_b, g = _run(roi, frames, variant, batches=2)
    want = oracle.correlate(frames, roi, roi)
    np.testing.assert_array_equal(s_ab, want["s_ab"])
    np.testing.assert_array_equal(s_a, want["s_a"])
    np.testing.assert_array_equal(s_b, want["s_b"])
    G = want["gamma"]
    zero = G == 0
    assert np.all(g[zero] == 0)
    assert np.max(np.abs(g.astype(np.float64) - G) / np.where(zero, 1, np.abs(G))) <= 1e-6
    assert np.array_equal(g, g.T) and np.array_equal(s_ab, s_ab.T)


def test_syrk_equals_full_gemm_and_panels(monkeypatch):
    """The same context without SYRK (CPI_SYRK=0), and row panels (which run the plain GEMM on the
    shared operand), give bit-identical counts and Gamma."""
    roi = (0, 0, 48, 32)
    frames = synth.bernoulli_frames(900, 0.3, seed=5)
    a = _run(roi, frames, "fp4")
    b = _run(roi, frames, "fp4", rows_panels=512)
    c = _run(roi, frames, "fp4", env={"CPI_SYRK": "0"}, monkeypatch=monkeypatch)
    for x, y in ((a, b), (a, c)):
        for u, v in zip(x, y):
            np.testing.assert_array_equal(u, v)
