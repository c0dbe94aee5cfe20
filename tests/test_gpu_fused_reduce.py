"""f2: the cross-rank reduction fused into the pair-sum GEMM epilogue
(include/cpi.h CPI_FUSED_REDUCE).  Every rank's epilogue adds its partial tiles straight into
the shard of the rank that owns those A rows (red.global.add.s32 into CUDA-IPC-mapped peer
memory), so no rank writes a full-size partial and no reduce-scatter pass runs.

One GPU is available here: two processes share it (CUDA IPC works between processes on the same
device), in the library's external mode (the handles and the rank ordering go through gloo on the
host; no kernel waits on another rank).  Result: each rank's Gamma rows bit-identical to a single
context's.  The NCCL one-rank group runs the library-managed flow (handle all-gather over the
communicator, cpi_reset / cpi_finalize ordering, refocus from the totals).
"""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROI_A, ROI_B = (0, 0, 32, 32), (256, 0, 24, 12)
N = 1500
ALPHAS = [0.6, 1.0, 1.45]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, variant, batches):
    import torch.distributed as dist
    from paper_2407_20692_b200 import Context
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        frames = synth.bernoulli_frames(N, 0.2, seed=77)
        lo, hi = rank * N // world, (rank + 1) * N // world
        c = Context(ROI_A, ROI_B, N, variant=variant, rank=rank, world=world, fused_reduce=True)
        hs = [None] * world
        dist.all_gather_object(hs, c.shard_ipc_handle())
        c.open_peer_shards(hs)
        c.reset()                                  # zero this rank's shard ...
        torch.cuda.synchronize()
        dist.barrier()                             # ... before any rank's GEMM adds into it
        mine = frames[lo:hi]
        for b in range(batches):                   # several batches accumulate into the shards
            part = np.ascontiguousarray(mine[b * len(mine) // batches:(b + 1) * len(mine) // batches])
            c.load_frames(part)
            c.correlate(None)
        torch.cuda.synchronize()
        dist.barrier()                             # every rank's adds are done
        shard, s_a, s_b = c.counts_views()
        marg = torch.cat([s_a.cpu().long(), s_b.cpu().long(), torch.tensor([hi - lo])])
        dist.all_reduce(marg)
        p_a = ROI_A[2] * ROI_A[3]
        s_a_tot, s_b_tot, n_tot = marg[:p_a].int(), marg[p_a:-1].int(), int(marg[-1])
        rows = c.shard_pixel_rows()
        g = torch.empty((rows.size, ROI_B[2] * ROI_B[3]), dtype=torch.float32, device="cuda")
        c.finalize_counts(shard, 0, s_a_tot[torch.from_numpy(rows)].contiguous().cuda(), s_b_tot.cuda(), n_tot, g)
        torch.cuda.synchronize()
        q.put((rank, n_tot, rows, g.cpu().numpy(), shard.cpu().numpy()))
        c.close()
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("variant,batches", [("fp4", 1), ("tc", 2)])
def test_fused_reduce_two_ranks_share_one_gpu(variant, batches):
    import multiprocessing as mp
    from paper_2407_20692_b200 import Context
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, variant, batches)) for r in range(world)]
    for p in procs:
        p.start()
    out = []
    import queue as _queue
    while len(out) < world:   # fail fast if a rank dies instead of waiting for the queue timeout
        try:
            out.append(q.get(timeout=10))
        except _queue.Empty:
            assert all(p.is_alive() or p.exitcode == 0 for p in procs), "a rank failed"
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    frames = synth.bernoulli_frames(N, 0.2, seed=77)
    c = Context(ROI_A, ROI_B, N, variant=variant, keep_counts=True)
    c.load_frames(frames)
    g = c.correlate(c.new_gamma())
    s_ab = c.counts_views()[0]
    torch.cuda.synchronize()
    G, S = g.cpu().numpy(), s_ab.cpu().numpy()
    covered = np.zeros(G.shape[0], dtype=int)
    for rank, n_tot, rows, g_rows, shard in out:
        assert n_tot == N
        np.testing.assert_array_equal(shard, S[rows])     # exact integer sums, reduced in the epilogue
        np.testing.assert_array_equal(g_rows, G[rows])
        covered[rows] += 1
    assert np.all(covered == 1)


@pytest.mark.parametrize("order", ["ublocked", "vmajor"])
def test_fused_reduce_one_rank_group(order):
    """Library-managed flow over NCCL (one-rank group): the handle all-gather, cpi_reset's barrier,
    cpi_finalize without a reduce-scatter, refocus from the totals."""
    from paper_2407_20692_b200 import Context, nccl_unique_id
    frames = synth.bernoulli_frames(N, 0.2, seed=78)
    ref = Context(ROI_A, ROI_B, N, gamma_order=order)
    ref.load_frames(frames)
    G = ref.correlate(ref.new_gamma()).cpu().numpy()
    P = ref.new_planes(len(ALPHAS))
    ref.refocus(ALPHAS, torch.from_numpy(G).cuda(), P)
    c = Context(ROI_A, ROI_B, N, gamma_order=order, rank=0, world=1, nccl_id=nccl_unique_id(), fused_reduce=True)
    for _ in range(2):   # the second acquisition starts from zeroed shards
        c.reset()
        c.load_frames(frames[:800])
        c.correlate(None)
        c.load_frames(frames[800:])
        c.correlate(None)
        g = torch.empty((ROI_A[2] * ROI_A[3], ROI_B[2] * ROI_B[3]), dtype=torch.float32, device="cuda")
        assert c.finalize(g) == N
        torch.cuda.synchronize()
        np.testing.assert_array_equal(g.cpu().numpy(), G[c.shard_pixel_rows()])
        planes = c.new_planes(len(ALPHAS))
        c.refocus(ALPHAS, None, planes)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(planes.cpu().numpy(), P.cpu().numpy())
