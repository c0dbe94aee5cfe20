"""GPU: a dataset of .bin files streamed through the context (dataset.correlate_files:
cpi_read_bin into pinned buffers -> cpi_load_frames -> cpi_correlate, batches spanning file
boundaries) gives the oracle's exact sums and Gamma, and the same bits as one in-memory batch."""
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


@pytest.mark.parametrize("variant,batch", [("fp4", 700), ("tc", 256), ("fp4", 1500)])
def test_correlate_files_matches_oracle(tmp_path, variant, batch):
    from paper_2407_20692_b200 import Context, dataset
    roi_a, roi_b = (3, 5, 40, 16), (270, 1, 24, 16)
    fr = synth.bernoulli_frames(1500, 0.2, seed=61)
    for i in range(5):                               # 5 files x 300 frames, written out of order
        (tmp_path / f"frames_{4 - i:04d}.bin").write_bytes(fr[300 * (4 - i):300 * (5 - i)].tobytes())
    m = dataset.scan_dataset(str(tmp_path))
    assert m.n_tot == 1500
    ctx = Context(roi_a, roi_b, batch, variant=variant, keep_counts=True)
    g = ctx.new_gamma()
    assert dataset.correlate_files(ctx, m, gamma=g) == 1500
    s_ab = torch.empty((ctx.p_a, ctx.p_b), dtype=torch.int32, device="cuda")
    s_a = torch.empty(ctx.p_a, dtype=torch.int32, device="cuda")
    s_b = torch.empty(ctx.p_b, dtype=torch.int32, device="cuda")
    n = ctx.get_counts(s_ab, s_a, s_b)
    torch.cuda.synchronize()
    want = oracle.correlate(fr, roi_a, roi_b)
    assert n == want["n"] == 1500
    np.testing.assert_array_equal(s_ab.cpu().numpy(), want["s_ab"])
    np.testing.assert_array_equal(s_a.cpu().numpy(), want["s_a"])
    np.testing.assert_array_equal(s_b.cpu().numpy(), want["s_b"])
    gg, ge = g.cpu().numpy().astype(np.float64), want["gamma"]
    zero = ge == 0
    assert np.all(gg[zero] == 0)
    assert (np.abs(gg - ge) / np.where(zero, 1, np.abs(ge))).max() <= 1e-6
