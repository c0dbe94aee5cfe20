"""Frame-sharded multi-rank orchestration (paper_2407_20692_b200.parallel) on CPU with gloo,
world sizes 2 and 4.  Each rank's compute backend is the CPU oracle (tests may use it); the
collectives, frame slicing, row sharding and plane merging are the product's.  The result
must equal the single-process oracle: Gamma rows exactly (integer sums are additive), planes
to fp rounding (the row shards' partial planes add up, refocusing being linear in Gamma)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2407_20692_b200 import parallel

ROI_A, ROI_B = (0, 0, 12, 8), (256, 0, 10, 6)
DIMS = (12, 8, 10, 6)
N = 900
ALPHAS = [0.6, 1.0, 1.7]
# general RefocusMap rows (include/cpi.h), fractional B coordinates on both axes
MAPS = [[0.7, 0.3, 0.25, 0.0, 0.5, -0.3, 1.3, -0.3, -0.4, 0.0, 0.8, 0.2],
        [1.6, -0.45, -1.5, 0.0, 1.25, 0.5, 0.55, 0.5, 2.0, 0.0, 0.6, -1.0]]


class OracleBackend:
    """The pipeline steps computed by the CPU oracle (test stand-in for CudaBackend)."""
    device = torch.device("cpu")
    row_align = 1

    def begin(self, frames):
        self.r = oracle.correlate(frames, ROI_A, ROI_B)

    def panel_counts(self, row0, rows):
        return torch.from_numpy(self.r["s_ab"][row0:row0 + rows].astype(np.int32))

    def marginals(self):
        return (torch.from_numpy(self.r["s_a"].astype(np.int32)), torch.from_numpy(self.r["s_b"].astype(np.int32)),
                int(self.r["n"]))

    def rows_to(self, row0, rows, out):
        out.copy_(torch.from_numpy(self.r["gamma"][row0:row0 + rows].astype(np.float32)))
        return out

    def finalize_rows(self, s_ab_rows, s_a_rows, s_b, n_tot):
        g = oracle.gamma(s_ab_rows.numpy(), s_a_rows.numpy(), s_b.numpy(), n_tot)
        return torch.from_numpy(g.astype(np.float32))

    def refocus(self, alphas, gamma_rows, row0, rows, row_block, row_stride, affine=None):
        Wa, Ha, Wb, Hb = DIMS
        G = np.zeros((Wa * Ha, Wb * Hb), dtype=np.float32)
        l = np.arange(rows // Wa)                     # include/cpi.h cpi_refocus_spec row map
        m = row0 // Wa + (l // row_block) * row_stride + l % row_block
        pix = (m[:, None] * Wa + np.arange(Wa)[None, :]).reshape(-1)
        G[pix] = gamma_rows.numpy()
        if affine is not None:
            return torch.from_numpy(oracle.refocus_affine(G, DIMS, affine).astype(np.float32))
        return torch.from_numpy(oracle.refocus(G, DIMS, alphas).astype(np.float32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, min_panel_rows, affine=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = synth.bernoulli_frames(N, 0.3, seed=31)
        lo, hi = parallel.frame_slice(N, rank, world)
        res = parallel.correlate_and_refocus(OracleBackend(), frames[lo:hi], ROI_A, ROI_B, ALPHAS,
                                             min_panel_rows=min_panel_rows, affine=MAPS if affine else None)
        q.put((rank, res.n_tot, res.plan, res.gamma_rows.numpy(), res.planes.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,min_panel_rows,affine", [(2, 8192, False), (4, 8192, False), (2, 1, False),
                                                         (4, 1, False), (2, 1, True)])
def test_frame_sharded_pipeline_matches_single_process(world, min_panel_rows, affine):
    """min_panel_rows = 1: one A row per rank per panel (cyclic ownership, several panels);
    8192: one panel of contiguous blocks at this small RoI; affine: general maps (fractional
    B) instead of alphas."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, min_panel_rows, affine)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    frames = synth.bernoulli_frames(N, 0.3, seed=31)
    full = oracle.correlate(frames, ROI_A, ROI_B)
    G = full["gamma"].astype(np.float32)
    want_planes = oracle.refocus_affine(G, DIMS, MAPS) if affine else oracle.refocus(G, DIMS, ALPHAS)
    Gabs = np.abs(G.astype(np.float64))
    M = oracle.refocus_affine(Gabs, DIMS, MAPS) if affine else oracle.refocus(Gabs, DIMS, ALPHAS)
    covered = np.zeros(G.shape[0], dtype=int)
    for rank, n_tot, plan, g_rows, planes in out:
        assert n_tot == N and plan.rank == rank and plan.world == world
        if min_panel_rows == 1:
            assert plan.block == 1 and plan.panels == DIMS[1] // world      # cyclic A rows
        rows = plan.pixel_rows().numpy()
        assert g_rows.shape[0] == rows.size == G.shape[0] // world
        np.testing.assert_array_equal(g_rows, G[rows])
        covered[rows] += 1
        err = np.abs(planes.astype(np.float64) - want_planes)
        assert np.all(err <= 1e-6 * M + 1e-30), np.max(err / np.maximum(M, 1e-300))   # SURVEY Q17 bar
    assert np.all(covered == 1)


def test_slicing_helpers():
    for n in (0, 1, 7, 10_000):
        for world in (1, 2, 3, 8):
            sl = [parallel.frame_slice(n, r, world) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
            assert max(h - l for l, h in sl) - min(h - l for l, h in sl) <= 1
    assert parallel.row_shard(256, 256, 3, 8) == (3 * 32 * 256, 32 * 256)
    with pytest.raises(ValueError):
        parallel.row_shard(256, 250, 0, 8)
    # block-cyclic plans: every A row owned exactly once, panels aligned to the GEMM tile
    for (W, H, world, align) in [(256, 256, 8, 256), (256, 256, 2, 256), (128, 128, 4, 256), (12, 8, 4, 256),
                                 (12, 8, 2, 1), (32, 16, 2, 128)]:
        owned = np.zeros(H, dtype=int)
        for r in range(world):
            p = parallel.shard_plan(W, H, r, world, align)
            assert p.panel_rows % align == 0 or p.panels == 1
            assert p.m_count * world == H
            owned[p.a_rows().numpy()] += 1
        assert np.all(owned == 1)
    p = parallel.shard_plan(256, 256, 3, 8, 256)
    assert (p.block, p.panels, p.stride, p.m_base) == (4, 8, 32, 12)
    assert p.a_rows()[:6].tolist() == [12, 13, 14, 15, 44, 45]


def _worker_tiles(rank, world, port, q, affine=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = synth.bernoulli_frames(N, 0.3, seed=31)
        lo, hi = parallel.frame_slice(N, rank, world)
        res = parallel.correlate_and_refocus_tiles(OracleBackend(), frames[lo:hi], ROI_A, ROI_B, ALPHAS,
                                                   min_panel_rows=1, affine=MAPS if affine else None)
        q.put((rank, res.n_tot, res.plan, res.gamma_rows.numpy(), res.planes.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,affine", [(2, False), (4, False), (2, True)])
def test_output_tile_sharding_matches_single_process(world, affine):
    """Output-tile sharding (SURVEY §8(e) control): frames all-gathered, each rank computes its
    own block-cyclic Gamma rows over all frames; rows equal the single-process oracle, planes
    merge by all-reduce."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_tiles, args=(r, world, port, q, affine)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    frames = synth.bernoulli_frames(N, 0.3, seed=31)
    full = oracle.correlate(frames, ROI_A, ROI_B)
    G = full["gamma"].astype(np.float32)
    want_planes = oracle.refocus_affine(G, DIMS, MAPS) if affine else oracle.refocus(G, DIMS, ALPHAS)
    Gabs = np.abs(G.astype(np.float64))
    M = oracle.refocus_affine(Gabs, DIMS, MAPS) if affine else oracle.refocus(Gabs, DIMS, ALPHAS)
    covered = np.zeros(G.shape[0], dtype=int)
    for rank, n_tot, plan, g_rows, planes in out:
        assert n_tot == N
        rows = plan.pixel_rows().numpy()
        np.testing.assert_array_equal(g_rows, G[rows])
        covered[rows] += 1
        err = np.abs(planes.astype(np.float64) - want_planes)
        assert np.all(err <= 1e-6 * M + 1e-30), np.max(err / np.maximum(M, 1e-300))   # SURVEY Q17 bar
    assert np.all(covered == 1)
