"""The frame-sharded multi-GPU contract inside the C ABI (include/cpi.h cpi_config rank / world /
nccl_id, cpi_finalize with the C2 all-reduce and the panelised C1 reduce-scatter, cpi_refocus from
the totals with the fp64 plane all-reduce).

One GPU is available here, so the library's NCCL path runs as a one-rank group (world = 1 with an
nccl_id: the same code path); it must be bit-identical to a plain single-GPU context and to the
torch.distributed orchestration (paper_2407_20692_b200.parallel) at world 1.  The >= 2-GPU variant
(one process per GPU, the unique id shared through torch.distributed) runs when the box has them.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
HERE = os.path.dirname(os.path.abspath(__file__))

ROI_A, ROI_B = (0, 0, 48, 32), (256, 0, 24, 16)
N = 1500
ALPHAS = [0.6, 1.0, 1.45, 1.9, 0.8]


def _single(frames, order):
    from paper_2407_20692_b200 import Context
    c = Context(ROI_A, ROI_B, N, gamma_order=order)
    c.load_frames(frames)
    g = c.correlate(c.new_gamma())
    planes = c.new_planes(len(ALPHAS))
    c.refocus(ALPHAS, g, planes)
    torch.cuda.synchronize()
    return c, g.cpu().numpy(), planes.cpu().numpy()


@pytest.mark.parametrize("order", ["ublocked", "vmajor"])
def test_abi_one_rank_group_matches_single_gpu(order):
    from paper_2407_20692_b200 import Context, nccl_unique_id
    frames = synth.bernoulli_frames(N, 0.2, seed=101)
    single, G, P = _single(frames, order)
    c = Context(ROI_A, ROI_B, N, keep_counts=True, gamma_order=order, rank=0, world=1, nccl_id=nccl_unique_id())
    c.load_frames(frames[:700])       # two batches: accumulation before the reduction
    c.correlate(None)
    c.load_frames(frames[700:])
    c.correlate(None)
    with pytest.raises(Exception):    # partial sums: no fused Gamma in multi-GPU mode
        c.load_frames(frames[:10])
        c.correlate(c.new_gamma())
    c.reset()
    c.load_frames(frames)
    c.correlate(None)
    rows_g = torch.empty((ROI_A[2] * ROI_A[3], ROI_B[2] * ROI_B[3]), dtype=torch.float32, device="cuda")
    n = c.finalize(rows_g)
    assert n == N and c.shard_rows == (0, ROI_A[2] * ROI_A[3])
    pix = c.shard_pixel_rows()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(rows_g.cpu().numpy(), G[pix])          # integer sums: bit-identical
    planes = c.new_planes(len(ALPHAS))
    c.refocus(ALPHAS, None, planes)                                        # own rows + fp64 all-reduce
    torch.cuda.synchronize()
    np.testing.assert_array_equal(planes.cpu().numpy(), P)
    Gr = G[:, single.b_index()]
    dims = (ROI_A[2], ROI_A[3], ROI_B[2], ROI_B[3])
    R = oracle.refocus(Gr, dims, ALPHAS)
    M = oracle.refocus(np.abs(Gr.astype(np.float64)), dims, ALPHAS)
    assert np.all(np.abs(planes.cpu().numpy().astype(np.float64) - R) <= 1e-6 * M + 1e-30)


def test_abi_one_rank_group_matches_torch_orchestration():
    """The library's C1/C2/C3 vs parallel.correlate_and_refocus over torch.distributed (NCCL, one
    rank): same Gamma rows, same planes."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29700 + os.getpid() % 200))
    code = f"""
import sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {os.path.dirname(HERE)!r})
import synth
from paper_2407_20692_b200 import Context, nccl_unique_id, parallel
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
A, B, N, AL = {ROI_A!r}, {ROI_B!r}, {N}, {ALPHAS!r}
fr = synth.bernoulli_frames(N, 0.2, seed=101)
be = parallel.CudaBackend(A, B, N, device=0, gamma_order="ublocked")
res = parallel.correlate_and_refocus(be, torch.from_numpy(fr).cuda(), A, B, AL)
c = Context(A, B, N, keep_counts=True, gamma_order="ublocked", rank=0, world=1, nccl_id=nccl_unique_id())
c.load_frames(fr); c.correlate(None)
g = torch.empty_like(res.gamma_rows); c.finalize(g)
p = c.new_planes(len(AL)); c.refocus(AL, None, p)
torch.cuda.synchronize()
gl = np.empty((A[2] * A[3], B[2] * B[3]), np.float32); gl[c.shard_pixel_rows()] = g.cpu().numpy()
gt = np.empty_like(gl); gt[res.plan.pixel_rows().numpy()] = res.gamma_rows.cpu().numpy()
assert np.array_equal(gl, gt)
np.testing.assert_allclose(p.cpu().numpy(), res.planes.cpu().numpy(), rtol=0, atol=1e-9)
dist.destroy_process_group()
print("ok")
"""
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs (one rank per GPU)")
@pytest.mark.parametrize("fused", [False, True])
def test_abi_multi_gpu_matches_single_gpu(tmp_path, fused):
    """One rank per GPU: library NCCL reduce-scatter (fused = False) or the GEMM epilogue adding into
    the owners' shards over NVLink peer memory (CPI_FUSED_REDUCE, f2)."""
    world = min(torch.cuda.device_count(), 8)
    out = tmp_path / "abi_mgpu.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29800 + os.getpid() % 100),
           os.path.join(HERE, "_abi_mgpu_worker.py"), str(out)]
    subprocess.run(cmd, check=True, timeout=900, env=dict(os.environ, CPI_ABI_FUSED="1" if fused else "0"))
    got = np.load(out)
    frames = synth.bernoulli_frames(int(got["n"]), 0.2, seed=101)
    _, G, P = _single(frames, "vmajor")
    np.testing.assert_array_equal(got["gamma"], G)
    np.testing.assert_allclose(got["planes"], P, rtol=0, atol=float(np.abs(P).max()) * 1e-6)
