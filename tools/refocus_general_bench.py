"""Time cpi_refocus on general RefocusMap rows at the 256^2 x 256^2 RoI:
default map (alphas), the same maps as affine rows with integral B (fast separable kernels),
and maps with fractional B coordinates: one B map shared by the stack (one resample of Gamma onto
the B lattice, then the fused fast path), a distinct B map per plane (one resample per plane),
and the direct general-B kernels (CPI_GENB_DIRECT).  Gamma: a seeded random fp32 matrix already
in HBM.  Prints one JSON line (ms per plane per kind, and the resample kernel's ms per launch)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_20692_b200 import Context  # noqa: E402
from paper_2407_20692_b200._lib import KC_RESAMPLE  # noqa: E402


def main():
    W = 256
    ctx = Context((0, 0, W, W), (256, 0, W, W), 1)
    g = torch.empty((W * W, W * W), dtype=torch.float32, device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(7)
    g.uniform_(-1.0, 1.0, generator=gen)
    P = 8
    al = np.linspace(0.5, 2.0, P)
    integral = [[a, 1 - a, 0.0, 0.0, 1.0, 0.0, a, 1 - a, 0.0, 0.0, 1.0, 0.0] for a in al]
    frac = [[a, 1 - a, 0.25, 0.0, 0.9, 0.3, a, 1 - a, -0.25, 0.0, 0.8, -0.2] for a in al]
    frac_each = [[a, 1 - a, 0.25, 0.0, 0.8 + 0.05 * i, 0.3, a, 1 - a, -0.25, 0.0, 0.8, -0.2]
                 for i, a in enumerate(al)]
    planes = ctx.new_planes(P)
    out = {"roi": "256x256 / 256x256", "planes": P}
    for name, kw in (("default", dict(alphas=al)), ("affine_integral_b", dict(alphas=None, affine=integral)),
                     ("affine_fractional_b", dict(alphas=None, affine=frac)),
                     ("affine_fractional_b_per_plane", dict(alphas=None, affine=frac_each)),
                     ("affine_fractional_b_direct", dict(alphas=None, affine=frac, direct=True))):
        alphas = kw.pop("alphas")
        if kw.pop("direct", False):
            os.environ["CPI_GENB_DIRECT"] = "1"
        else:
            os.environ.pop("CPI_GENB_DIRECT", None)
        for _ in range(2):
            ctx.refocus(alphas, g, planes, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 3
        for _ in range(reps):
            ctx.refocus(alphas, g, planes, **kw)
        e1.record()
        torch.cuda.synchronize()
        out[name + "_ms_per_plane"] = e0.elapsed_time(e1) / reps / P
    os.environ.pop("CPI_GENB_DIRECT", None)
    ctx.set_timing(True)
    ctx.refocus(None, g, planes, affine=frac_each)
    ms, n = ctx.kernel_time_ms(KC_RESAMPLE)
    out["resample_ms_per_launch"] = ms / max(n, 1)
    out["resample_gb_per_s"] = 2 * 4 * (W ** 4) / (ms / max(n, 1)) / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
