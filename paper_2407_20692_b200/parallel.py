"""Frame-sharded multi-GPU CPI over torch.distributed (NCCL on B200s, gloo in CPU tests).

SURVEY §8(e) / BASELINE north_star: frames shard naturally.  Rank g of G takes a
contiguous frame slice, accumulates int32 partial S_ab, S_a, S_b, N over it (Eq. (1)'s
sums are exactly additive), then
  1. runs the pair-sum GEMM in row panels and reduce-scatters(sum) each panel as soon as it
     is done (the one real exchange, overlapped with the next panels' GEMM),
  2. all-reduce(sum) of [S_a | S_b | N]                    (tiny),
  3. finalises its own Gamma rows (cpi_finalize_counts),
  4. refocuses its own rows into partial planes (refocusing is linear in Gamma and the
     normalisation is geometry-only, so shard planes add up),
  5. all-reduce(sum) of the planes.
Ownership is block-cyclic over whole A rows (``ShardPlan``): every rank holds rows spread
over the whole RoI, which balances the refocusing work for alpha < 1.

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
    """Contiguous A-row block [row0, row0 + rows) of a rank (whole A rows, equal blocks).
    Kept for callers that want contiguous ownership; the pipeline uses ``shard_plan``."""
    if height_a % world:
        raise ValueError(f"H_a = {height_a} must be divisible by the world size {world}")
    m_per = height_a // world
    return rank * m_per * width_a, m_per * width_a


@dataclass(frozen=True)
class ShardPlan:
    """Block-cyclic ownership of Gamma's A rows (SURVEY §8(e) load balance + panelised RS).
    The GEMM runs in ``panels`` row panels of ``world * block`` A rows; in every panel rank g
    owns the g-th block of ``block`` consecutive A rows, so its shard is the A rows
        m(l) = m_base + (l // block) * stride + l % block,   l < m_count,
    with m_base = g * block, stride = world * block.  Every panel's reduce-scatter can start
    as soon as that panel's GEMM is done, and every rank owns rows spread over the whole
    A RoI (refocusing work per rank balanced for every alpha)."""
    width_a: int
    height_a: int
    world: int
    rank: int
    block: int
    panels: int

    @property
    def m_base(self) -> int:
        return self.rank * self.block

    @property
    def stride(self) -> int:
        return self.world * self.block

    @property
    def m_count(self) -> int:
        return self.block * self.panels

    @property
    def panel_rows(self) -> int:          # A pixels per panel
        return self.world * self.block * self.width_a

    def a_rows(self):
        """Global A-row index of each local A row of the shard."""
        l = torch.arange(self.m_count)
        return self.m_base + (l // self.block) * self.stride + l % self.block

    def pixel_rows(self):
        """Global Gamma row (A pixel) of each local row of the shard."""
        m = self.a_rows()
        return (m[:, None] * self.width_a + torch.arange(self.width_a)[None, :]).reshape(-1)


def shard_plan(width_a: int, height_a: int, rank: int, world: int, row_align: int = 1,
               min_panel_rows: int = 8192, block_aligned: bool = False) -> ShardPlan:
    """Smallest block (A rows per rank per panel) whose panel is a multiple of the GEMM's row
    alignment and holds at least ``min_panel_rows`` A pixels (launch / collective overhead vs
    pipelining); one panel of contiguous blocks if none qualifies (always valid).
    block_aligned: each rank's block itself must be row-aligned (output-tile sharding runs
    the GEMM on the rank's own blocks)."""
    if height_a % world:
        raise ValueError(f"H_a = {height_a} must be divisible by the world size {world}")
    m_per = height_a // world
    if world > 1:
        for block in range(1, m_per + 1):
            rows = world * block * width_a
            unit = block * width_a if block_aligned else rows
            if m_per % block == 0 and unit % row_align == 0 and rows >= min(min_panel_rows, width_a * height_a):
                return ShardPlan(width_a, height_a, world, rank, block, m_per // block)
        # every rank raises (none may enter a collective the others never reach)
        if block_aligned and (m_per * width_a) % row_align:
            raise ValueError(f"no row-aligned block-cyclic plan for W_a = {width_a}, H_a = {height_a}, "
                             f"world {world}, alignment {row_align}")
    return ShardPlan(width_a, height_a, world, rank, m_per, 1)


@dataclass
class ShardResult:
    n_tot: int
    plan: ShardPlan
    gamma_rows: torch.Tensor          # [m_count * W_a][P_b] fp32, rows plan.pixel_rows()
    planes: Optional[torch.Tensor]    # [P][H_a][W_a] fp32 (summed over ranks) or None


def _reduce_scatter_async(out: torch.Tensor, full: torch.Tensor, group):
    """Sum `full` over ranks and keep this rank's equal chunk in `out` (async on NCCL)."""
    if dist.get_backend(group) == "nccl":
        return dist.reduce_scatter_tensor(out, full, op=dist.ReduceOp.SUM, group=group, async_op=True)
    # gloo has no reduce_scatter_tensor: all-reduce a copy, keep the own chunk
    tmp = full.clone()
    dist.all_reduce(tmp, op=dist.ReduceOp.SUM, group=group)
    r, rows = dist.get_rank(group), out.shape[0]
    out.copy_(tmp[r * rows:(r + 1) * rows])
    return None


def correlate_and_refocus(backend, frames_local, roi_a, roi_b, alphas=None, group=None,
                          min_panel_rows: int = 8192, affine=None) -> ShardResult:
    """Run the frame-sharded pipeline on this rank.  ``backend`` provides
         row_align                          GEMM row-panel alignment (A pixels)
         begin(frames)                      load this rank's frames
         panel_counts(row0, rows)           int32 [rows][P_b] pair sums of A pixels [row0, +rows)
                                            over this rank's frames (launched on the current stream)
         marginals() -> (s_a, s_b, n)       this rank's S_a, S_b (int32), frame count
         finalize_rows(s_ab_rows, s_a_rows, s_b, n_tot) -> Gamma rows fp32
         refocus(alphas, gamma_rows, row0, rows, row_block, row_stride, affine) -> planes fp32
    with all tensors on ``backend.device``.  affine: optional [planes][12] general RefocusMap
    rows (include/cpi.h) used instead of alphas."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    Wa, Ha = roi_a[2], roi_a[3]
    p_a, p_b = Wa * Ha, roi_b[2] * roi_b[3]
    plan = shard_plan(Wa, Ha, rank, world, backend.row_align, min_panel_rows)
    dev = backend.device
    backend.begin(frames_local)
    chunk = plan.block * Wa
    shard = torch.empty((plan.panels, chunk, p_b), dtype=torch.int32, device=dev)
    works = []
    for k in range(plan.panels):
        panel = backend.panel_counts(k * plan.panel_rows, plan.panel_rows)
        works.append(_reduce_scatter_async(shard[k], panel, group))
    s_a, s_b, n = backend.marginals()
    marg = torch.cat([s_a.to(torch.int64), s_b.to(torch.int64),
                      torch.tensor([n], dtype=torch.int64, device=s_a.device)])
    dist.all_reduce(marg, op=dist.ReduceOp.SUM, group=group)
    for w in works:
        if w is not None:
            w.wait()
    s_a_tot = marg[:p_a].to(torch.int32)
    s_b_tot = marg[p_a:p_a + p_b].to(torch.int32)
    n_tot = int(marg[-1].item())
    s_a_rows = s_a_tot[plan.pixel_rows().to(s_a_tot.device)].contiguous()
    gamma_rows = backend.finalize_rows(shard.view(-1, p_b), s_a_rows, s_b_tot, n_tot)
    planes = _refocus_shard(backend, plan, Wa, gamma_rows, alphas, affine, group)
    return ShardResult(n_tot, plan, gamma_rows, planes)


def _refocus_shard(backend, plan, Wa, gamma_rows, alphas, affine, group):
    """Refocus this rank's block-cyclic Gamma rows and sum the partial planes over ranks
    (refocusing is linear in Gamma).  affine rows replace alphas when given.
    The partial planes are summed in fp64 and rounded once to fp32: each
    rank's fp32 plane is within 2^-24 of its fp64 value relative to that rank's M, M is additive
    over row shards, so the sum stays within ~2^-23 M of the single-GPU plane."""
    if affine is None and (alphas is None or not len(alphas)):
        return None
    args = (gamma_rows, plan.m_base * Wa, plan.m_count * Wa, plan.block, plan.stride)
    planes = backend.refocus(alphas, *args) if affine is None else backend.refocus(None, *args, affine=affine)
    p64 = planes.to(torch.float64)
    dist.all_reduce(p64, op=dist.ReduceOp.SUM, group=group)
    return p64.to(torch.float32)


def _gather_frames(frames_local, group, device) -> torch.Tensor:
    """All ranks' frame slices concatenated in rank order (= the global frame order)."""
    world = dist.get_world_size(group)
    t = torch.as_tensor(frames_local).to(device)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(x.item()) for x in ns]
    n_max = max(ns)
    padded = torch.zeros((n_max,) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
    padded[:t.shape[0]] = t
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * n_max,) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
        dist.all_gather_into_tensor(out, padded, group=group)
        parts = [out[r * n_max:r * n_max + ns[r]] for r in range(world)]
    else:
        lst = [torch.empty_like(padded) for _ in range(world)]
        dist.all_gather(lst, padded, group=group)
        parts = [lst[r][:ns[r]] for r in range(world)]
    return torch.cat(parts).contiguous()


def correlate_and_refocus_tiles(backend, frames_local, roi_a, roi_b, alphas=None, group=None,
                                min_panel_rows: int = 8192, affine=None) -> ShardResult:
    """Output-tile sharding (SURVEY §8(e) control measurement): the packed frames are
    all-gathered (each rank's slice is 16 KB per frame, ~1.3 GB per rank at 10^5 frames), then
    every rank runs the GEMM with the fused exact normalisation on its own block-cyclic Gamma
    rows over all frames (``backend.rows_to``), refocuses them and the planes are all-reduced.
    No reduce-scatter of the 4 P_a P_b-byte partial sums.  ``backend`` as for
    correlate_and_refocus plus rows_to(row0, rows, out) -> Gamma rows [row0, +rows) into out."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    Wa, Ha = roi_a[2], roi_a[3]
    p_b = roi_b[2] * roi_b[3]
    plan = shard_plan(Wa, Ha, rank, world, backend.row_align, min_panel_rows, block_aligned=True)
    frames_all = _gather_frames(frames_local, group, backend.device)
    backend.begin(frames_all)
    chunk = plan.block * Wa
    gamma_rows = torch.empty((plan.panels * chunk, p_b), dtype=torch.float32, device=backend.device)
    for k in range(plan.panels):
        backend.rows_to(k * plan.panel_rows + rank * chunk, chunk, gamma_rows[k * chunk:(k + 1) * chunk])
    planes = _refocus_shard(backend, plan, Wa, gamma_rows, alphas, affine, group)
    return ShardResult(int(frames_all.shape[0]), plan, gamma_rows, planes)


class CudaBackend:
    """The pipeline steps on one B200 through the C ABI (libcpi.so): the GEMM runs in row
    panels (cpi_correlate_rows) whose pair sums are handed to the collectives in place
    (cpi_counts_dev views, no copies)."""

    def __init__(self, roi_a, roi_b, max_frames: int, device: int = 0, variant: str = "tc",
                 gamma_blocked: bool = False, keep_counts: bool = True, gamma_order=None):
        """gamma_order (or gamma_blocked = "ublocked"): the B pixel order (faster refocusing);
        S_b and the columns of ShardResult.gamma_rows then follow ctx.b_index()."""
        from .cpi import Context
        self.ctx = Context(roi_a, roi_b, max_frames, device=device, variant=variant, keep_counts=keep_counts,
                           gamma_blocked=gamma_blocked, gamma_order=gamma_order)
        self.device = torch.device(f"cuda:{device}")
        self.roi_a = roi_a
        self.row_align = self.ctx.row_align()
        self._s_ab, self._s_a, self._s_b = self.ctx.counts_views()   # s_ab None without kept counts
        self._n = 0

    def begin(self, frames):
        c = self.ctx
        c.reset()
        self._n = c.load_frames(frames)

    def panel_counts(self, row0, rows):
        self.ctx.correlate_rows(row0, rows)
        return self._s_ab[row0:row0 + rows]

    def marginals(self):
        return self._s_a, self._s_b, self._n

    def rows_to(self, row0, rows, out):
        self.ctx.correlate_rows_to(row0, rows, out)
        return out

    def finalize_rows(self, s_ab_rows, s_a_rows, s_b, n_tot):
        g = torch.empty(s_ab_rows.shape, dtype=torch.float32, device=self.device)
        self.ctx.finalize_counts(s_ab_rows.contiguous(), 0, s_a_rows.contiguous(), s_b.contiguous(), n_tot, g)
        return g

    def refocus(self, alphas, gamma_rows, row0, rows, row_block=0, row_stride=0, affine=None):
        planes = self.ctx.new_planes(len(affine) if affine is not None else len(alphas))
        self.ctx.refocus(alphas, gamma_rows, planes, row0=row0, rows=rows, row_block=row_block,
                         row_stride=row_stride, affine=affine)
        return planes
