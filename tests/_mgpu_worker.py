"""Worker of tests/test_multi_gpu.py (SURVEY §4 tier T3): one rank per GPU over NCCL, the
frame-sharded pipeline of paper_2407_20692_b200.parallel with the CUDA backend.  Rank 0 writes
the gathered Gamma rows and planes to the path in argv[1] for the parent test to compare with
a single-GPU run.  Launched by torch.distributed.run."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2407_20692_b200 import parallel  # noqa: E402

ROI_A, ROI_B = (0, 0, 64, 64), (256, 0, 48, 40)
N = 6000
ALPHAS = [0.6, 1.0, 1.55]


def main(out_path: str) -> None:
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    frames = synth.bernoulli_frames(N, 0.1, seed=99)
    lo, hi = parallel.frame_slice(N, rank, world)
    tiles = os.environ.get("CPI_MGPU_MODE", "rows") == "tiles"
    be = parallel.CudaBackend(ROI_A, ROI_B, N if tiles else hi - lo, device=local,
                              variant=os.environ.get("CPI_MGPU_VARIANT", "fp4"), gamma_blocked=True,
                              keep_counts=not tiles)
    run = parallel.correlate_and_refocus_tiles if tiles else parallel.correlate_and_refocus
    res = run(be, np.ascontiguousarray(frames[lo:hi]), ROI_A, ROI_B, ALPHAS, min_panel_rows=256)
    rows = res.plan.pixel_rows().to(res.gamma_rows.device)
    gathered_g = [torch.empty_like(res.gamma_rows) for _ in range(world)]
    gathered_r = [torch.empty_like(rows) for _ in range(world)]
    dist.all_gather(gathered_g, res.gamma_rows)
    dist.all_gather(gathered_r, rows)
    if rank == 0:
        G = torch.empty((ROI_A[2] * ROI_A[3], res.gamma_rows.shape[1]), dtype=torch.float32, device=rows.device)
        for g, r in zip(gathered_g, gathered_r):
            G[r] = g
        np.savez(out_path, gamma=G.cpu().numpy(), planes=res.planes.cpu().numpy(), n_tot=res.n_tot,
                 panels=res.plan.panels, b_index=be.ctx.b_index())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
