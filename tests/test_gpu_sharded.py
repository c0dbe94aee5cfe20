"""Frame-sharded pipeline through the CUDA backend (paper_2407_20692_b200.parallel.CudaBackend)
with 2 ranks sharing one GPU over gloo.  No kernel waits on another rank (the collectives run on
the host through gloo), so this is safe on one device; it exercises the product's multi-GPU
code path end to end: per-rank int32 partial sums, all-reduce of the marginals, row
reduce-scatter of GEMM row panels (cpi_correlate_rows), cpi_finalize_counts of the owned
block-cyclic rows, block-cyclic refocusing and the plane all-reduce.  Result: Gamma rows bit-identical to the single-context run, planes within 1e-6 M of the
oracle (shard planes are summed in fp64)."""
import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROI_A, ROI_B = (0, 0, 32, 32), (256, 0, 24, 12)      # P_a = 1024: four 256-row panels at world 2
N = 1500
ALPHAS = [0.6, 1.0, 1.45]
MAPS = [[0.7, 0.3, 0.25, 0.0, 0.5, -0.3, 1.3, -0.3, -0.4, 0.0, 0.8, 0.2],      # fractional B
        [1.2, -0.2, 0.0, 0.0, 0.5, -0.3, 0.8, 0.2, 0.0, 0.0, 0.8, 0.2]]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, mode="rows", affine=False, order="rowmajor", variant="tc"):
    import torch.distributed as dist
    import synth
    from paper_2407_20692_b200 import parallel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = synth.bernoulli_frames(N, 0.2, seed=77)
        lo, hi = parallel.frame_slice(N, rank, world)
        be = parallel.CudaBackend(ROI_A, ROI_B, N if mode == "tiles" else hi - lo, device=0,
                                  keep_counts=mode != "tiles", gamma_order=order, variant=variant)

        class GlooCuda:
            """gloo collectives need host tensors: stage through the host (plumbing only)."""
            device = torch.device("cpu")
            row_align = be.row_align

            def begin(self, fr):
                be.begin(fr)

            def panel_counts(self, row0, rows):
                return be.panel_counts(row0, rows).cpu()

            def marginals(self):
                s_a, s_b, n = be.marginals()
                return s_a.cpu(), s_b.cpu(), n

            def rows_to(self, row0, rows, out):
                tmp = torch.empty(tuple(out.shape), dtype=torch.float32, device="cuda")
                out.copy_(be.rows_to(row0, rows, tmp).cpu())
                return out

            def finalize_rows(self, s_ab_rows, s_a_rows, s_b, n_tot):
                return be.finalize_rows(s_ab_rows.cuda(), s_a_rows.cuda(), s_b.cuda(), n_tot).cpu()

            def refocus(self, alphas, gamma_rows, row0, rows, row_block, row_stride, affine=None):
                return be.refocus(alphas, gamma_rows.cuda(), row0, rows, row_block, row_stride, affine=affine).cpu()

        run = parallel.correlate_and_refocus_tiles if mode == "tiles" else parallel.correlate_and_refocus
        res = run(GlooCuda(), np.ascontiguousarray(frames[lo:hi]), ROI_A, ROI_B, ALPHAS, min_panel_rows=1,
                  affine=MAPS if affine else None)
        q.put((rank, res.n_tot, res.plan.pixel_rows().numpy(), res.plan.panels, res.gamma_rows.numpy(),
               res.planes.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,affine,order,variant", [("rows", False, "rowmajor", "tc"), ("tiles", False, "rowmajor", "tc"),
                                                       ("rows", True, "rowmajor", "tc"),
                                                       ("tiles", False, "vmajor", "fp4"),   # bench.py's --gpus N step
                                                       ("rows", False, "vmajor", "fp4")])
def test_two_ranks_on_one_gpu_match_single_context(mode, affine, order, variant):
    import torch.multiprocessing as mp
    import synth
    from paper_2407_20692_b200 import Context
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode, affine, order, variant)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    frames = synth.bernoulli_frames(N, 0.2, seed=77)
    c = Context(ROI_A, ROI_B, N, gamma_order=order, variant=variant)
    c.load_frames(frames)
    g = c.correlate(c.new_gamma())
    planes = c.new_planes(len(MAPS) if affine else len(ALPHAS))
    if affine:
        c.refocus(None, g, planes, affine=MAPS)
    else:
        c.refocus(ALPHAS, g, planes)
    torch.cuda.synchronize()
    G = g.cpu().numpy()
    P = planes.cpu().numpy()
    dims = (ROI_A[2], ROI_A[3], ROI_B[2], ROI_B[3])
    G_rm = G[:, c.b_index()]                        # the oracle reads row-major B columns
    Gabs = np.abs(G_rm.astype(np.float64))
    R = oracle.refocus_affine(G_rm, dims, MAPS) if affine else oracle.refocus(G_rm, dims, ALPHAS)
    M = oracle.refocus_affine(Gabs, dims, MAPS) if affine else oracle.refocus(Gabs, dims, ALPHAS)
    for rank, n_tot, rows, panels, g_rows, pl in out:
        assert n_tot == N and panels > 1           # several row panels, block-cyclic ownership
        np.testing.assert_array_equal(g_rows, G[rows])
        err = np.abs(pl.astype(np.float64) - R)     # fp64 plane all-reduce: 1e-6 M
        assert np.all(err <= 1e-6 * M + 1e-30), np.max(err / np.maximum(M, 1e-300))
        np.testing.assert_allclose(pl, P, rtol=0, atol=float(np.max(4e-7 * M)) + 1e-30)
