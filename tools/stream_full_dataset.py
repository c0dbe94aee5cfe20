"""Full-dataset scale (7808 files x 512 frames = 3,997,696 frames, RoI 256x256):
stream the frames through one context in batches (cpi_load_frames from pinned host memory, double-
buffered copy overlapping the previous batch) accumulating int32 counts (CPI_KEEP_COUNTS), then
cpi_finalize to Gamma.  3,997,696 = 61 x 65,536: two distinct synthetic 65,536-frame batches are
alternated (generation of 65 GB of distinct frames would dominate the run); throughput does not depend
on the bit values.  Checks the closed form total: sum_pq S_ab = sum_i n_A(i) n_B(i)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2407_20692_b200 import Context
from paper_2407_20692_b200._lib import KC_GEMM, KC_EXPAND, KC_FINALIZE

B = int(os.environ.get("CPI_STREAM_BATCH", 65536))
n_batches = int(os.environ.get("CPI_STREAM_BATCHES", 61))
t0 = time.time()
host = [torch.from_numpy(synth.bernoulli_frames(B, 0.05, seed=synth.SEED_ARMS, frame0=k * B)).pin_memory() for k in range(2)]
gen_s = time.time() - t0
popc = torch.tensor([bin(b).count("1") for b in range(256)], dtype=torch.int64)
ctx = Context(synth.ROI_FULL_A, synth.ROI_FULL_B, B, keep_counts=True)
# warm-up batch, then reset
ctx.load_frames(host[0]); ctx.correlate(None); torch.cuda.synchronize(); ctx.reset()
ctx.set_timing(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(n_batches):
    ctx.load_frames(host[k % 2])
    ctx.correlate(None)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
gemm_ms, gemm_n = ctx.kernel_time_ms(KC_GEMM)
exp_ms, _ = ctx.kernel_time_ms(KC_EXPAND)
gamma = ctx.new_gamma()
f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
f0.record(); n_tot = ctx.finalize(gamma); f1.record(); torch.cuda.synchronize()
fin_ms = f0.elapsed_time(f1)
s_ab = torch.empty((65536, 65536), dtype=torch.int32, device="cuda")
ctx.get_counts(s_ab)
total = int(s_ab.sum(dtype=torch.int64).item())

# exact expected total: batches alternate host[0], host[1]
na0 = popc[host[0][:, :, 0:32].long()].sum(dim=(1, 2)); nb0 = popc[host[0][:, :, 32:64].long()].sum(dim=(1, 2))
na1 = popc[host[1][:, :, 0:32].long()].sum(dim=(1, 2)); nb1 = popc[host[1][:, :, 32:64].long()].sum(dim=(1, 2))
p0, p1 = int((na0 * nb0).sum()), int((na1 * nb1).sum())
expect_total = p0 * ((n_batches + 1) // 2) + p1 * (n_batches // 2)
ops = 2.0 * 65536 * 65536 * B * n_batches
print(json.dumps({
    "workload": f"{n_batches} x {B} = {n_batches * B} frames (PAPER.md:61 full dataset = 3,997,696), RoI 256x256 halves",
    "n_tot": n_tot, "stream_ms": ms, "frames_per_s": n_batches * B / (ms / 1e3),
    "gemm_ms": gemm_ms, "gemm_tops": ops / (gemm_ms / 1e3) / 1e12, "expand_ms": exp_ms,
    "finalize_ms": fin_ms, "end_to_end_s": (ms + fin_ms) / 1e3,
    "total_pairs_check": {"gpu": total, "closed_form": expect_total, "equal": total == expect_total},
    "host_generation_s": gen_s}))
