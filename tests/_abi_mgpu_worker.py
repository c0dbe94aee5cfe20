"""One rank of the C-ABI multi-GPU test (tests/test_gpu_abi_multi.py): rank 0 creates the NCCL
unique id with cpi_nccl_unique_id and shares it over torch.distributed (plumbing); every rank then
creates a multi-GPU context, correlates its frame slice, finalises its rows and refocuses."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2407_20692_b200 import Context, nccl_unique_id  # noqa: E402
from test_gpu_abi_multi import ALPHAS, N, ROI_A, ROI_B  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("gloo")
    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    frames = synth.bernoulli_frames(N, 0.2, seed=101)
    lo, hi = rank * N // world, (rank + 1) * N // world
    fused = os.environ.get("CPI_ABI_FUSED", "0") == "1"
    c = Context(ROI_A, ROI_B, N, keep_counts=not fused, gamma_order="vmajor", device=int(os.environ["LOCAL_RANK"]),
                rank=rank, world=world, nccl_id=box[0], fused_reduce=fused)
    c.load_frames(np.ascontiguousarray(frames[lo:hi]))
    c.correlate(None)
    rows = c.shard_pixel_rows()
    g = torch.empty((rows.size, ROI_B[2] * ROI_B[3]), dtype=torch.float32, device="cuda")
    n = c.finalize(g)
    planes = c.new_planes(len(ALPHAS))
    c.refocus(ALPHAS, None, planes)
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, (rows, g.cpu().numpy()))
    if rank == 0:
        G = np.empty((ROI_A[2] * ROI_A[3], ROI_B[2] * ROI_B[3]), dtype=np.float32)
        for r, gg in parts:
            G[r] = gg
        np.savez(sys.argv[1], gamma=G, planes=planes.cpu().numpy(), n=n)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
