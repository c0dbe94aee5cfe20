"""Refocusing benchmark grid of PAPER.md:306-321 (Figs. 11-12): RoI 128x128 and 256x256, a Gamma from
11 files' worth of frames (11 x 512 = 5632), 100 / 261 / 1000 refocusing planes,
alpha = linspace(0.5, 2, P).  Device-resident Gamma; CUDA events around cpi_refocus; prints one JSON
line per point, for each B pixel order in $CPI_SWEEP_ORDERS (default "vmajor ublocked": KB5w / KB5).
(The paper's own times are figure-only; this is the B200 analog.)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import bench
from paper_2407_20692_b200 import Context
from paper_2407_20692_b200._lib import KC_STAGE1, KC_STAGE2, KC_COORDS

n = 11 * 512
cases = [(o, name, ra, rb) for o in os.environ.get("CPI_SWEEP_ORDERS", "vmajor ublocked").split()
         for name, ra, rb in (("128x128", synth.ROI_128_A, synth.ROI_128_B), ("256x256", synth.ROI_FULL_A, synth.ROI_FULL_B))]
for order, name, ra, rb in cases:
    fr = torch.from_numpy(synth.bernoulli_frames(n, 0.05)).cuda()
    ctx = Context(ra, rb, n, variant="fp4", gamma_order=order)
    ctx.load_frames(fr)
    g = ctx.correlate(ctx.new_gamma())
    dims = (ra[2], ra[3], rb[2], rb[3])
    for P in (100, 261, 1000):
        al = synth.alpha_grid(P)
        planes = ctx.new_planes(P)
        ctx.refocus(al[:8], g, planes)                     # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.set_timing(True)
        e0.record()
        ctx.refocus(al, g, planes)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        s1 = ctx.kernel_time_ms(KC_STAGE1)[0]
        s2 = ctx.kernel_time_ms(KC_STAGE2)[0]
        co = ctx.kernel_time_ms(KC_COORDS)[0]
        ctx.set_timing(False)
        span, taps = bench.refocus_work(dims, al)
        print(json.dumps({"order": order, "roi": name, "frames": n, "planes": P, "ms": ms, "planes_per_s": P / (ms / 1e3),
                          "ms_per_plane": ms / P, "stage1_ms": s1, "stage2_ms": s2, "coords_ms": co,
                          "span_bytes": span, "span_gbs": span / (ms / 1e3) / 1e9,
                          "taps_per_s": taps / (s1 / 1e3)}), flush=True)
    del g, ctx
    torch.cuda.empty_cache()
