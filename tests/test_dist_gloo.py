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


class OracleBackend:
    """The five pipeline steps computed by the CPU oracle (test stand-in for CudaBackend)."""
    device = torch.device("cpu")

    def local_sums(self, frames):
        r = oracle.correlate(frames, ROI_A, ROI_B)
        return (torch.from_numpy(r["s_ab"].astype(np.int32)), torch.from_numpy(r["s_a"].astype(np.int32)),
                torch.from_numpy(r["s_b"].astype(np.int32)), int(r["n"]))

    def finalize_rows(self, s_ab_rows, row0, s_a, s_b, n_tot):
        rows = s_ab_rows.shape[0]
        g = oracle.gamma(s_ab_rows.numpy(), s_a.numpy()[row0:row0 + rows], s_b.numpy(), n_tot)
        return torch.from_numpy(g.astype(np.float32))

    def refocus(self, alphas, gamma_rows, row0, rows):
        Wa, Ha, Wb, Hb = DIMS
        G = np.zeros((Wa * Ha, Wb * Hb), dtype=np.float32)
        G[row0:row0 + rows] = gamma_rows.numpy()
        return torch.from_numpy(oracle.refocus(G, DIMS, alphas).astype(np.float32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = synth.bernoulli_frames(N, 0.3, seed=31)
        lo, hi = parallel.frame_slice(N, rank, world)
        res = parallel.correlate_and_refocus(OracleBackend(), frames[lo:hi], ROI_A, ROI_B, ALPHAS)
        q.put((rank, res.n_tot, res.row0, res.rows, res.gamma_rows.numpy(), res.planes.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_frame_sharded_pipeline_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    frames = synth.bernoulli_frames(N, 0.3, seed=31)
    full = oracle.correlate(frames, ROI_A, ROI_B)
    G = full["gamma"].astype(np.float32)
    want_planes = oracle.refocus(G, DIMS, ALPHAS)
    covered = np.zeros(G.shape[0], dtype=int)
    for rank, n_tot, row0, rows, g_rows, planes in out:
        assert n_tot == N
        assert row0 == rank * rows and rows == G.shape[0] // world
        np.testing.assert_array_equal(g_rows, G[row0:row0 + rows])
        covered[row0:row0 + rows] += 1
        np.testing.assert_allclose(planes, want_planes, rtol=1e-5, atol=1e-7)
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
