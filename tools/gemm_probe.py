"""Probe KB2 timing at configs[1]: fused Gamma epilogue vs counts-only epilogue, interleaved
rounds in one process, min over rounds (CUDA events inside the library)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2407_20692_b200 import Context
from paper_2407_20692_b200._lib import KC_GEMM

fr = torch.from_numpy(synth.bernoulli_frames(10_000, 0.05)).cuda()
modes = {"gamma": Context(synth.ROI_FULL_A, synth.ROI_FULL_B, 10_000),
         "counts": Context(synth.ROI_FULL_A, synth.ROI_FULL_B, 10_000, keep_counts=True)}
g = modes["gamma"].new_gamma()
best = {k: 1e9 for k in modes}
for rnd in range(4):
    for k, ctx in modes.items():
        ctx.set_timing(True)
        for _ in range(2):
            ctx.reset(); ctx.load_frames(fr); ctx.correlate(g if k == "gamma" else None)
        torch.cuda.synchronize()
        ms, n = ctx.kernel_time_ms(KC_GEMM)
        if rnd:
            best[k] = min(best[k], ms / n)
        ctx.set_timing(False)
print(json.dumps({k: {"ms": v, "tops": 2 * 65536**2 * 1e4 / v / 1e9} for k, v in best.items()}))
