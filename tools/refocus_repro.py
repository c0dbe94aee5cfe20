"""Small refocus determinism repro: random Gamma, W_a = 256 (full-x kernel path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2407_20692_b200 import Context

Wa, Ha, Wb, Hb = [int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 32, 256, 16))]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
ctx = Context((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1)
g = torch.from_numpy(synth.random_gamma(Wa * Ha, Wb * Hb, seed=1)).cuda()
al = synth.alpha_grid(64)
ref = ctx.new_planes(64); ctx.refocus(al, g, ref); torch.cuda.synchronize()
for r in range(reps):
    p = ctx.new_planes(64); p.fill_(float("nan")); ctx.refocus(al, g, p); torch.cuda.synchronize()
    ne = ref != p
    print(f"rep {r}: mismatches {int(ne.sum())} planes {ne.any(2).any(1).nonzero().flatten().tolist()[:16]}", flush=True)
