"""SURVEY §4 tier T3: the frame-sharded pipeline on 2-8 real GPUs (one rank per GPU, NCCL,
launched with torch.distributed.run).  Gamma gathered from the ranks' block-cyclic shards is
bit-identical to one GPU's Gamma (integer sums), and the all-reduced planes equal the
single-GPU planes to fp32 summation order.  Skipped when fewer than 2 GPUs are visible (the
gloo tests cover the orchestration on CPU; test_gpu_sharded.py covers it on one GPU)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tmp_path, variant, world, mode="rows"):
    sys.path.insert(0, HERE)
    import _mgpu_worker as w
    import synth
    from paper_2407_20692_b200 import Context
    out = tmp_path / "mgpu.npz"
    env = dict(os.environ, CPI_MGPU_VARIANT=variant, CPI_MGPU_MODE=mode)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           os.path.join(HERE, "_mgpu_worker.py"), str(out)]
    subprocess.run(cmd, check=True, env=env, timeout=900)
    got = np.load(out)
    frames = synth.bernoulli_frames(w.N, 0.1, seed=99)
    ctx = Context(w.ROI_A, w.ROI_B, w.N, variant=variant, gamma_blocked=True)
    ctx.load_frames(frames)
    g = ctx.correlate(ctx.new_gamma())
    planes = ctx.new_planes(len(w.ALPHAS))
    ctx.refocus(w.ALPHAS, g, planes)
    torch.cuda.synchronize()
    assert int(got["n_tot"]) == w.N and int(got["panels"]) >= 1
    np.testing.assert_array_equal(got["gamma"], g.cpu().numpy())
    import oracle
    G = g.cpu().numpy()
    if ctx.gamma_blocked:                    # oracle wants the row-major B order
        Gr = np.empty_like(G)
        Gr[:] = G[:, ctx.b_index()]
        G = Gr
    dims = (w.ROI_A[2], w.ROI_A[3], w.ROI_B[2], w.ROI_B[3])
    sel = np.random.default_rng(0).integers(0, dims[0] * dims[1], 64)
    pix = np.stack([sel % dims[0], sel // dims[0]], 1)
    R = oracle.refocus(G, dims, w.ALPHAS, pixels=pix)
    M = oracle.refocus(np.abs(G.astype(np.float64)), dims, w.ALPHAS, pixels=pix)
    got_p = got["planes"].astype(np.float64)[:, pix[:, 1], pix[:, 0]]
    err = np.abs(got_p - R)                  # fp64 plane all-reduce: 1e-6 M
    assert np.all(err <= 1e-6 * M + 1e-30), np.max(err / np.maximum(M, 1e-300))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs (one rank per GPU)")
@pytest.mark.parametrize("variant,mode", [("fp4", "rows"), ("tc", "rows"), ("fp4", "tiles")])
def test_frame_sharded_nccl_matches_single_gpu(tmp_path, variant, mode):
    _run(tmp_path, variant, min(torch.cuda.device_count(), 8), mode)


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
@pytest.mark.parametrize("mode", ["rows", "tiles"])
def test_nccl_single_rank_pipeline(tmp_path, mode):
    """The NCCL code path of both pipelines (async reduce-scatter on the library's count views /
    all-gather of frames, all-reduces) as a one-rank group under torch.distributed.run."""
    _run(tmp_path, "fp4", 1, mode)
