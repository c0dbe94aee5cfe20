"""Frame-sharded multi-GPU CPI over torch.distributed (NCCL on B200s, gloo in CPU tests).

SURVEY §8(e) / BASELINE north_star: frames shard naturally.  Rank g of G takes a
contiguous frame slice, accumulates int32 partial S_ab, S_a, S_b, N over it (Eq. (1)'s
sums are exactly additive), then
  1. all-reduce(sum) of [S_a | S_b | N]                    (tiny),
  2. reduce-scatter(sum) of S_ab by A-row blocks            (the one real exchange),
  3. finalise its own Gamma row shard (cpi_finalize_counts),
  4. refocus its own rows into partial planes (refocusing is linear in Gamma and the
     normalisation is geometry-only, so shard planes add up),
  5. all-reduce(sum) of the planes.
Shards are whole A rows (multiples of W_a) so each rank's refocus stage 1 sees complete
(m, v) blocks.

The compute steps are supplied by a backend object so the same orchestration runs with
the CUDA library (``CudaBackend``) or, in CPU tests, with any other implementation of
the five methods (the tests plug in the oracle).  This module does no arithmetic on
pixel data itself.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist


def frame_slice(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced slice [lo, hi) of the global frame sequence for a rank."""
    base, rem = divmod(n_frames, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def row_shard(width_a: int, height_a: int, rank: int, world: int) -> tuple[int, int]:
    """A-row block [row0, row0 + rows) of Gamma owned by a rank (whole A rows, equal
    blocks: reduce-scatter needs equal chunks, so H_a must be divisible by world)."""
    if height_a % world:
        raise ValueError(f"H_a = {height_a} must be divisible by the world size {world}")
    m_per = height_a // world
    return rank * m_per * width_a, m_per * width_a


@dataclass
class ShardResult:
    n_tot: int
    row0: int
    rows: int
    gamma_rows: torch.Tensor          # [rows][P_b] fp32
    planes: Optional[torch.Tensor]    # [P][H_a][W_a] fp32 (summed over ranks) or None


def _reduce_scatter_rows(full: torch.Tensor, rows: int, group) -> torch.Tensor:
    out = torch.empty((rows, full.shape[1]), dtype=full.dtype, device=full.device)
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, full, op=dist.ReduceOp.SUM, group=group)
    else:   # gloo has no reduce_scatter_tensor: all-reduce then keep the own block
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
        r = dist.get_rank(group)
        out.copy_(full[r * rows:(r + 1) * rows])
    return out


def correlate_and_refocus(backend, frames_local, roi_a, roi_b, alphas=None, group=None) -> ShardResult:
    """Run the frame-sharded pipeline on this rank.  ``backend`` provides:
         local_sums(frames) -> (s_ab [P_a][P_b] int32, s_a [P_a] int32, s_b [P_b] int32, n)
         finalize_rows(s_ab_rows, row0, s_a, s_b, n_tot) -> gamma rows fp32
         refocus(alphas, gamma_rows, row0, rows) -> planes [P][H_a][W_a] fp32
    all tensors on ``backend.device``."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    s_ab, s_a, s_b, n = backend.local_sums(frames_local)
    p_a, p_b = s_a.numel(), s_b.numel()
    marg = torch.cat([s_a.to(torch.int64), s_b.to(torch.int64),
                      torch.tensor([n], dtype=torch.int64, device=s_a.device)])
    dist.all_reduce(marg, op=dist.ReduceOp.SUM, group=group)
    s_a_tot = marg[:p_a].to(torch.int32)
    s_b_tot = marg[p_a:p_a + p_b].to(torch.int32)
    n_tot = int(marg[-1].item())
    row0, rows = row_shard(roi_a[2], roi_a[3], rank, world)
    s_ab_rows = _reduce_scatter_rows(s_ab, rows, group)
    gamma_rows = backend.finalize_rows(s_ab_rows, row0, s_a_tot, s_b_tot, n_tot)
    planes = None
    if alphas is not None and len(alphas):
        planes = backend.refocus(alphas, gamma_rows, row0, rows)
        dist.all_reduce(planes, op=dist.ReduceOp.SUM, group=group)
    return ShardResult(n_tot, row0, rows, gamma_rows, planes)


class CudaBackend:
    """The five pipeline steps on one B200 through the C ABI (libcpi.so)."""

    def __init__(self, roi_a, roi_b, max_frames: int, device: int = 0, variant: str = "tc"):
        from .cpi import Context
        self.ctx = Context(roi_a, roi_b, max_frames, device=device, variant=variant, keep_counts=True)
        self.device = torch.device(f"cuda:{device}")
        self.roi_a = roi_a

    def local_sums(self, frames):
        c = self.ctx
        c.reset()
        c.load_frames(frames)
        c.correlate(None)
        s_ab = torch.empty((c.p_a, c.p_b), dtype=torch.int32, device=self.device)
        s_a = torch.empty(c.p_a, dtype=torch.int32, device=self.device)
        s_b = torch.empty(c.p_b, dtype=torch.int32, device=self.device)
        n = c.get_counts(s_ab, s_a, s_b)
        return s_ab, s_a, s_b, n

    def finalize_rows(self, s_ab_rows, row0, s_a, s_b, n_tot):
        g = torch.empty(s_ab_rows.shape, dtype=torch.float32, device=self.device)
        self.ctx.finalize_counts(s_ab_rows.contiguous(), row0, s_a.contiguous(), s_b.contiguous(), n_tot, g)
        return g

    def refocus(self, alphas, gamma_rows, row0, rows):
        planes = self.ctx.new_planes(len(alphas))
        self.ctx.refocus(alphas, gamma_rows, planes, row0=row0, rows=rows)
        return planes
