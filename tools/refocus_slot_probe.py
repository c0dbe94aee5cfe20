"""Is the F=4 refocus error tied to the plane slot or to alpha?  Groups of identical alphas must
give identical planes in every slot; reversed alpha order must give the same planes permuted."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2407_20692_b200 import Context

Wa, Ha, Wb, Hb = 256, 64, 256, 64
ctx = Context((0, 0, Wa, Ha), (0, 0, Wb, Hb), 1)
g = torch.from_numpy(synth.random_gamma(Wa * Ha, Wb * Hb, seed=1)).cuda()
for a in (1.83, 1.9, 2.0, 1.5, 0.7):
    for rep in range(2):
        p = ctx.new_planes(4); ctx.refocus([a] * 4, g, p); torch.cuda.synchronize()
        d = [(int((p[0] != p[s]).sum())) for s in range(1, 4)]
        print(f"alpha {a} rep {rep}: slot mismatches vs slot 0: {d}", flush=True)
al = synth.alpha_grid(64)
p1 = ctx.new_planes(64); ctx.refocus(al, g, p1)
p2 = ctx.new_planes(64); ctx.refocus(al[::-1].copy(), g, p2); torch.cuda.synchronize()
p2 = p2.flip(0)
ne = p1 != p2
print("reversed order mismatching planes:", ne.any(2).any(1).nonzero().flatten().tolist())
