"""Race detector: every kernel of the path is deterministic, so repeated runs on the same
input must agree bit for bit.  Reports mismatches of Gamma (GEMM) and of the planes (refocus)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2407_20692_b200 import Context

fr = torch.from_numpy(synth.bernoulli_frames(10_000, 0.05)).cuda()
ctx = Context(synth.ROI_FULL_A, synth.ROI_FULL_B, 10_000)
g1 = ctx.new_gamma(); g2 = ctx.new_gamma()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for r in range(reps):
    ctx.reset(); ctx.load_frames(fr); ctx.correlate(g1 if r == 0 else g2)
    torch.cuda.synchronize()
    if r:
        ne = (g1 != g2)
        n = int(ne.sum())
        print(f"gamma rep {r}: mismatches {n}", flush=True)
        if n:
            idx = ne.nonzero()[:10].tolist()
            print("  first", idx, [(g1[i, j].item(), g2[i, j].item()) for i, j in idx[:5]])
alphas = synth.alpha_grid(64)
p1 = ctx.new_planes(64); p2 = ctx.new_planes(64)
for r in range(reps):
    ctx.refocus(alphas, g1, p1 if r == 0 else p2)
    torch.cuda.synchronize()
    if r:
        ne = (p1 != p2)
        n = int(ne.sum())
        print(f"planes rep {r}: mismatches {n}", flush=True)
        if n:
            pl = ne.any(dim=2).any(dim=1).nonzero().flatten().tolist()
            print("  planes", pl[:20])
            idx = ne.nonzero()[:10].tolist()
            print("  first", idx, [(p1[a, b, c].item(), p2[a, b, c].item()) for a, b, c in idx[:5]])
