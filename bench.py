#!/usr/bin/env python3
"""bench.py — CPI hot path on B200: frames -> Gamma (Eq. 1) -> refocused plane stack.

One *step* = one pass of the whole hot path over one batch:
  N frames resident in HBM -> expand + marginals (KB1) -> S_ab on tcgen05 tensor cores
  (default kind::mxf4 on E2M1 0/1 operands, exact; --variant tc = kind::i8) with the fused
  exact normalisation (KB2) -> fp32 Gamma -> refocus into a P-plane stack (KB5a/KB5/KB6).
Workload at N=1 (BASELINE.json configs[1] + configs[3]): SwissSPAD2 256x512 frames,
rho_a = left 256x256 half, rho_b = right 256x256 half, 10^4
Bernoulli(0.05) frames per step, 64 refocus planes alpha = linspace(0.5, 2, 64).
Metric: frames/s into Gamma (whole step), with the correlation-only frames/s, planes/s and
the two kernels' roofline fractions alongside.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cb200|reference]
Multi-GPU: launched by torch.distributed.run; frames shard across ranks (weak scaling:
10^4 frames per rank); the pair-sum GEMM runs in row panels whose NCCL reduce-scatter starts
as each panel finishes (overlapping the next panels), Gamma rows are owned block-cyclically,
each rank refocuses its rows and the planes are all-reduced (paper_2407_20692_b200.parallel).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import synth  # noqa: E402

METRIC = "frames/s into Gamma (and % int8 TC peak); refocused planes/s (% HBM BW)"
# the step's default configuration (tests/test_gpu_fullsize.py runs exactly this against the oracle)
STEP_VARIANT = "fp4"
STEP_GAMMA_ORDER = "vmajor"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="cb200", choices=["cb200", "reference"])
    p.add_argument("--frames", type=int, default=10_000,
                   help="frames per step, split across the ranks (strong scaling of the configs[1] step)")
    p.add_argument("--planes", type=int, default=64, help="refocus planes per step")
    p.add_argument("--occupancy", type=float, default=0.05, help="Bernoulli f of the synthetic bits")
    p.add_argument("--variant", default=STEP_VARIANT, choices=["tc", "popc", "fp4", "bits"],
                   help="pair-sum GEMM: fp4 = tcgen05 kind::mxf4 on E2M1 0/1 (default, exact), "
                        "tc = kind::i8, popc = popcount(AND), bits = kind::i8 on bit streams unpacked in "
                        "shared memory (f1)")
    p.add_argument("--roi", default="full", choices=["full", "128", "tiny"])
    p.add_argument("--gamma-order", default=STEP_GAMMA_ORDER, choices=["ublocked", "rowmajor", "vmajor"],
                   help="column order of the step's Gamma (include/cpi.h CPI_GAMMA_UBLOCKED)")
    p.add_argument("--parallel-mode", default="auto", choices=["auto", "lib", "rows", "tiles"],
                   help="multi-GPU: lib = frame sharding with the library's own NCCL reduce-scatter / all-reduces "
                        "(cpi_config rank/world, north_star); rows = the same over torch.distributed "
                        "(parallel.py); auto = tiles when all-gathering the packed frames moves fewer bytes than "
                        "reduce-scattering the int32 partial S_ab (N * 16 KB < 4 P_a P_b), else lib; tiles = "
                        "all-gather of frames + each rank's own Gamma rows (SURVEY §8(e) control)")
    p.add_argument("--no-fused-reduce", action="store_true",
                   help="lib mode: reduce-scatter the partial pair sums with NCCL instead of adding them into the "
                        "owners' shards from the GEMM epilogue (CPI_FUSED_REDUCE, default)")
    p.add_argument("--sharded", action="store_true",
                   help="run the frame-sharded multi-GPU pipeline (NCCL) even at one rank (tests its code path)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-pixels", type=int, default=48, help="oracle sample: refocused output pixels per alpha")
    return p.parse_args()


def frame_bytes_of(args):
    return synth.frame_bytes()


def rois(name):
    if name == "full":
        return synth.ROI_FULL_A, synth.ROI_FULL_B
    if name == "128":
        return synth.ROI_128_A, synth.ROI_128_B
    return synth.ROI_TINY_A, synth.ROI_TINY_B


def load_traffic():
    """ncu DRAM bytes per launch of the dominant kernels (profiles/r02_traffic.json, else r01's)."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            return json.loads((ROOT / "profiles" / name).read_text())
        except Exception:
            pass
    return {}


def issue_view(prof, ms_per_launch, f_clk):
    """Issue-slot and shared-memory views of a kernel from its committed ncu capture: the capture's
    warp instructions and shared-memory wavefronts per launch over this run's live launch time,
    against 4 warp instructions and 1 wavefront per clock per SM (148 SMs, this run's median clock)."""
    inst, wav = prof.get("warp_instructions_per_launch"), prof.get("smem_wavefronts_per_launch")
    if not inst or not ms_per_launch:
        return None
    slots = 148 * f_clk * ms_per_launch / 1e3
    return {"issue_frac": inst / (4 * slots), "smem_wavefront_frac": wav / slots if wav else None,
            "warp_instructions_per_launch": inst, "smem_wavefronts_per_launch": wav,
            "source": prof.get("source"),
            "note": "counts from the ncu capture named in source, time from this run"}


def load_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks ----------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if s > 0]
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------ roofline helpers -------
def _axis_tables(W, Wb_, alpha):
    """Per-axis support of the default map, as the kernels use it: for every
    B coordinate the used outputs, their lower taps and the span [min i0, max i0 + 1]."""
    c, cb = (W - 1) / 2.0, (Wb_ - 1) / 2.0
    x = np.arange(W, dtype=np.float64)[None, :]
    u = np.arange(Wb_, dtype=np.float64)[:, None]
    cc = (alpha * (x - c)) + ((1.0 - alpha) * (u - cb)) + c
    ok = (cc >= 0) & (cc <= W - 1)
    j0 = np.minimum(np.floor(cc), W - 2)
    lo = np.where(ok, j0, np.inf).min(1)
    hi = np.where(ok, j0 + 1, -np.inf).max(1)
    span = np.where(hi >= lo, hi - lo + 1, 0)
    return ok, span


def refocus_work(dims, alphas):
    """Per-plane algorithmic work of refocus stage 1 (SURVEY §8(d) 'per unit of work'):
      bytes = 4 B x Gamma entries inside the separable stencil span
            = 4 (sum_u |J_u|)(sum_v |M_v|), J_u = [min j0, max j0 + 1] over outputs using u;
      taps  = 2 x (valid (x, u) samples) x (sum_v |M_v|)  — one fp32 tap = one 4-byte
              shared-memory load + one FMA in the kernel.
    Returns (bytes, taps) summed over the planes."""
    Wa, Ha, Wb, Hb = dims
    tot_b = tot_t = 0.0
    for a in alphas:
        okx, sx = _axis_tables(Wa, Wb, a)
        _, sy = _axis_tables(Ha, Hb, a)
        tot_b += 4.0 * sx.sum() * sy.sum()
        tot_t += 2.0 * okx.sum() * sy.sum()
    return tot_b, tot_t


def refocus_span_bytes(dims, alphas):
    return refocus_work(dims, alphas)[0]


# ------------------------------------------------------------------ CPU baseline ----------
def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_step_estimate(oracle, frames_np, roi_a, roi_b, alphas, step_planes, threads, n_s, rows_pair, n_pix, G):
    """One timed pass of the oracle over a bounded sample of the step, extrapolated to the step.
    Every phase is linear in what is sampled: single-pixel sums and pair sums in the frame count
    (first n_s frames), pair sums also in the A pixels (rows_pair and 2 rows_pair rows, all B
    pixels: fixed unpacking + per-row part), refocusing in output pixels and planes (n_pix pixels
    at each of 8 alphas spread over the stack's grid)."""
    n = frames_np.shape[0]
    fs = frames_np[:n_s]
    p_a = roi_a[2] * roi_a[3]
    t0 = time.perf_counter()
    s_a = oracle.marginals(fs, roi_a)
    s_b = oracle.marginals(fs, roi_b)
    t_marg = (time.perf_counter() - t0) * n / n_s
    r1 = np.linspace(0, p_a - 1, rows_pair).astype(np.int64)
    r2 = np.linspace(0, p_a - 1, 2 * rows_pair).astype(np.int64)
    t0 = time.perf_counter()
    oracle.pair_sums(fs, roi_a, roi_b, rows=r1, threads=threads)
    t1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    s_ab = oracle.pair_sums(fs, roi_a, roi_b, rows=r2, threads=threads)
    g = oracle.gamma(s_ab, s_a[r2], s_b, n_s)                      # Eq. (1) on the sampled rows
    t2 = time.perf_counter() - t0
    per_row = max(t2 - t1, 1e-9) / rows_pair
    fixed = max(t1 - rows_pair * per_row, 0.0)
    t_pairs = (fixed + per_row * p_a) * n / n_s
    Wa, Ha, Wb, Hb = roi_a[2], roi_a[3], roi_b[2], roi_b[3]
    if G[0, 0] != G[0, 0]:                                            # first pass: fill the refocus input
        G[:] = g[np.arange(p_a) % g.shape[0]].astype(np.float32)      # (refocus cost is data-independent)
    sel = np.unique(np.linspace(0, len(alphas) - 1, 8).astype(int))
    rng = np.random.default_rng(0)
    pix = np.stack([rng.integers(0, Wa, n_pix), rng.integers(0, Ha, n_pix)], 1)
    t0 = time.perf_counter()
    oracle.refocus(G, (Wa, Ha, Wb, Hb), np.asarray(alphas)[sel], pixels=pix, threads=threads)
    t_ref = (time.perf_counter() - t0) / (len(sel) * n_pix) * (Wa * Ha) * step_planes
    return {"marginals": t_marg, "pair_sums": t_pairs, "refocus": t_ref}


def cpu_baseline(frames_np, roi_a, roi_b, alphas, n_pix, step_planes, reps=3, one_core=True):
    """The oracle as it stands, timed on the box's host cores on a bounded sample of the same
    workload (rank 0, N = 1; SURVEY §8(d) "oracle timed beside it"): >= 3 repetitions on all
    cores (median), plus one repetition on 1 core; CPU model and core count reported."""
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1
    n = frames_np.shape[0]
    n_s = min(n, 512)
    G = np.empty((roi_a[2] * roi_a[3], roi_b[2] * roi_b[3]), dtype=np.float32)   # one refocus input for all passes
    G[0, 0] = np.nan
    runs = [_oracle_step_estimate(oracle, frames_np, roi_a, roi_b, alphas, step_planes, cores, n_s, cores, n_pix, G)
            for _ in range(reps)]
    tot = [sum(r.values()) for r in runs]
    med = runs[int(np.argsort(tot)[len(tot) // 2])]
    est = sum(med.values())
    out = {"value": n / est, "unit": "frames/s", "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
           "reps": reps, "rep_step_s": tot,
           "sample": (f"first {n_s} of {n} frames; single-pixel sums over all {roi_a[2] * roi_a[3]}+"
                      f"{roi_b[2] * roi_b[3]} pixels; pair sums for {cores} and {2 * cores} A pixels x all B "
                      f"pixels; refocus of {n_pix} output pixels at 8 alphas spread over the {len(alphas)}-plane "
                      f"grid; each phase extrapolated linearly (frames, A pixels, output pixels x planes) to the "
                      f"step; median of {reps} repetitions on {cores} threads"),
           "extrapolated_step_s": est, "extrapolated_parts_s": med}
    if one_core:
        r1 = _oracle_step_estimate(oracle, frames_np, roi_a, roi_b, alphas, step_planes, 1, min(n_s, 256), 1,
                                   max(4, n_pix // 8), G)
        out["one_core"] = {"value": n / sum(r1.values()), "unit": "frames/s", "extrapolated_parts_s": r1,
                           "sample": "first 256 frames, pair sums for 1 and 2 A pixels, refocus of "
                                     f"{max(4, n_pix // 8)} pixels at 8 alphas, 1 repetition on 1 thread"}
    return out


# ------------------------------------------------------------------ reference arm ---------
def run_reference(args, json_out=None):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    roi_a, roi_b = rois(args.roi)
    alphas = synth.alpha_grid(args.planes)
    frames = synth.bernoulli_frames(args.frames, args.occupancy, seed=synth.SEED_ARMS)
    vals = []
    last = None
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(frames, roi_a, roi_b, alphas, max(8, args.cpu_pixels // 4), args.planes, reps=1,
                         one_core=False)
        if i >= args.warmup:
            vals.append(r["value"])
            last = r
    v = float(np.median(vals))
    last["value"] = v
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
           "config": {"workload": f"configs[1]+configs[3]: {args.frames} frames, RoI {roi_a}/{roi_b}, "
                                  f"{args.planes} planes", "frames_per_step": args.frames,
                      "planes_per_step": args.planes},
           "cpu_baseline": last,
           "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), file=json_out or sys.stdout, flush=True)


# ------------------------------------------------------------------ main arm --------------
def _claim_stdout():
    """Route fd 1 to stderr for the rest of the run (NCCL, CUDA and library messages) and return
    a stream on the original stdout for the one JSON line of the contract."""
    out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    return out


def main():
    args = parse()
    json_out = _claim_stdout()
    if args.impl == "reference":
        run_reference(args, json_out)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run (one rank per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    use_dist = world > 1 or args.sharded
    if use_dist:
        os.environ.setdefault("NCCL_DEBUG", "WARN")   # keep stdout to the one JSON line
        if world == 1:   # one-rank NCCL group (no launcher): rendezvous on localhost
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29400 + os.getpid() % 500))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)

    from paper_2407_20692_b200 import Context
    from paper_2407_20692_b200._lib import KC_GEMM, KC_EXPAND, KC_STAGE1, KC_STAGE2, KC_COORDS, KC_FINALIZE
    from paper_2407_20692_b200 import parallel

    roi_a, roi_b = rois(args.roi)
    p_a, p_b = roi_a[2] * roi_a[3], roi_b[2] * roi_b[3]
    Wa, Ha, Wb, Hb = roi_a[2], roi_a[3], roi_b[2], roi_b[3]
    alphas = synth.alpha_grid(args.planes)
    n_total = args.frames
    # this rank's contiguous slice of the step's frames (strong scaling: the same configs[1] step at
    # every N; Eq. (1)'s sums are additive over slices)
    f_lo, f_hi = parallel.frame_slice(n_total, rank, world)
    n = f_hi - f_lo
    frames_np = synth.bernoulli_frames(n, args.occupancy, seed=synth.SEED_ARMS, frame0=f_lo)
    frames_host = torch.from_numpy(frames_np).pin_memory()
    frames_dev = frames_host.to(dev)
    stream = torch.cuda.current_stream(dev)

    mode, tiles = "single", False
    if not use_dist:
        ctx = Context(roi_a, roi_b, n, device=local, variant=args.variant,
                      gamma_order=args.gamma_order)
        gamma = ctx.new_gamma()
        planes = ctx.new_planes(args.planes)
    else:
        mode = args.parallel_mode
        if mode == "auto":   # DESIGN §9 cost model: bytes each rank sends per step
            mode = "tiles" if n_total * frame_bytes_of(args) < 4 * p_a * p_b else "lib"
        tiles = mode == "tiles"
        if mode == "lib":
            # the library's own multi-GPU contract (include/cpi.h cpi_config rank / world / nccl_id):
            # cpi_finalize reduce-scatters the partial S_ab and all-reduces [S_a|S_b|N] over its NCCL
            # communicator, cpi_refocus from the totals refocuses the owned rows and all-reduces planes
            from paper_2407_20692_b200 import nccl_unique_id
            box = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            fused = not args.no_fused_reduce and args.variant in ("tc", "fp4")
            ctx = Context(roi_a, roi_b, n, device=local, variant=args.variant, gamma_order=args.gamma_order,
                          keep_counts=not fused, rank=rank, world=world, nccl_id=box[0], fused_reduce=fused)
            planes = ctx.new_planes(args.planes)
        else:
            # torch.distributed orchestration (parallel.py): rows = GEMM row panels reduce-scattered as
            # they finish; tiles = all-gather of the packed frames, each rank its own Gamma rows
            backend = parallel.CudaBackend(roi_a, roi_b, n_total if tiles else n, device=local, variant=args.variant,
                                           gamma_order=args.gamma_order, keep_counts=not tiles)
            ctx = backend.ctx
    planes_host = torch.empty((args.planes, Ha, Wa), dtype=torch.float32).pin_memory()

    def step(src):
        """one pass of a1..a6; src = device frames (resident) or pinned host frames (e2e);
        returns the plane stack"""
        if not use_dist:
            ctx.reset()          # a new acquisition: zero S_a, S_b, N (memsets)
            ctx.load_frames(src)
            ctx.correlate(gamma)
            ctx.refocus(alphas, gamma, planes)
            return planes
        if mode == "lib":
            ctx.reset()
            ctx.load_frames(src)
            ctx.correlate(None)
            ctx.finalize(None)
            ctx.refocus(alphas, None, planes)
            return planes
        run = parallel.correlate_and_refocus_tiles if tiles else parallel.correlate_and_refocus
        res = run(backend, src, roi_a, roi_b, alphas)
        return res.planes

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step(frames_dev)
    barrier()

    clocks = ClockSampler(local)
    ctx.set_timing(True)
    launches0 = ctx.launch_count()
    clocks.start()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(frames_dev)
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count() - launches0
    t_ms = ev0.elapsed_time(ev1)
    kt = {k: ctx.kernel_time_ms(c) for k, c in (("gemm", KC_GEMM), ("expand", KC_EXPAND), ("stage1", KC_STAGE1),
                                                 ("stage2", KC_STAGE2), ("coords", KC_COORDS),
                                                 ("finalize", KC_FINALIZE))}
    ctx.set_timing(False)
    if use_dist:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    ms_step = t_ms / args.steps
    value = n_total / (ms_step / 1e3)

    # ---- end to end through the public API with host buffers --------------------------
    e2e = None
    if not args.no_e2e:
        for _ in range(1):
            planes_host.copy_(step(frames_host), non_blocking=True)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            planes_host.copy_(step(frames_host), non_blocking=True)
        e1.record(stream)
        barrier()
        te = e0.elapsed_time(e1)
        if use_dist:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": n_total / (te / args.steps / 1e3), "unit": "frames/s",
               "h2d_bytes_per_step": int(frames_np.nbytes), "d2h_bytes_per_step": int(planes_host.numel() * 4),
               "ms_per_step": te / args.steps}

    if rank != 0:
        if use_dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peak_src = load_peaks()
    traffic = load_traffic()
    hbm = peaks["hbm_gbs"]
    f_clk = (clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)) * 1e6
    gemm_ms, gemm_n = kt["gemm"]
    # algorithmic ops of this rank's GEMM: one AND/MAC per pair per frame (tiles: own rows, all frames)
    ops = 2.0 * p_a * p_b * n if not (use_dist and tiles) else 2.0 * (p_a // world) * p_b * n_total
    gemm_tops = ops / (gemm_ms / gemm_n / 1e3) / 1e12 if gemm_n else None
    clock_peak_tops = 148 * 8192 * 2 * f_clk / 1e12  # tcgen05 kind::i8: 8192 MAC/clk/SM
    s1_ms, s1_n = kt["stage1"]
    rows_here = p_a if world == 1 else p_a // world
    span, taps = refocus_work((Wa, Ha, Wb, Hb), alphas)
    span *= rows_here / p_a
    taps *= rows_here / p_a
    s1_s = s1_ms / args.steps / 1e3
    s1_gbs = span / s1_s / 1e9 if s1_n else None
    s1_gtaps = taps / s1_s / 1e9 if s1_n else None
    lds_peak_gtaps = 148 * 32 * f_clk / 1e9          # 32 four-byte LDS lanes per clock per SM
    corr_ms = (kt["expand"][0] + gemm_ms) / args.steps
    ref_ms = (kt["coords"][0] + s1_ms + kt["stage2"][0]) / args.steps
    # the FP4 variant runs kind::mxf4: its own peak is 4 x bf16 (nominal 9 / 2.25 PFLOP/s)
    ratio, dname = (4.0, "fp4 (e2m1, kind::mxf4)") if args.variant == "fp4" else (2.0, "int8")
    tc_burst, tc_sustained = ratio * peaks["bf16_tflops"], ratio * peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    if args.variant == "fp4":
        clock_peak_tops *= 2.0                        # 16384 e2m1 MAC/clk/SM
    roof_gemm = {"kernel": {"tc": "gemm_i8_tc2 (KB2, cta_group::2, kind::i8)", "popc": "gemm_popc (KB3)",
                            "bits": "gemm_i8_tc2<bits> (f1: bit streams unpacked in shared memory, kind::i8)",
                            "fp4": "gemm_i8_tc2<fp4> (KB2, cta_group::2, kind::mxf4)"}[args.variant],
                 "bound": "tensor", "achieved": gemm_tops, "peak": tc_burst, "unit": "TOPS",
                 "frac": gemm_tops / tc_burst if gemm_tops else None,
                 "peak_note": (f"{dname} dense = {ratio:g} x {peak_src} bf16 burst {peaks['bf16_tflops']} TFLOP/s "
                               f"(guide ratio {ratio * 2.25:g}/2.25); the sustained bf16 figure "
                               f"({peaks.get('bf16_tflops_sustained')}) was taken at a 1327 MHz median clock, this "
                               f"run's median was {clk.get('sm_mhz')} MHz"),
                 "frac_of_sustained": gemm_tops / tc_sustained if gemm_tops else None,
                 "frac_of_clock_peak": gemm_tops / clock_peak_tops if gemm_tops else None,
                 "clock_peak_tops": clock_peak_tops,
                 "smem_view": ({"ceiling_tops": 448.0 / 578.0 * clock_peak_tops,
                                "frac": gemm_tops / (448.0 / 578.0 * clock_peak_tops) if gemm_tops else None,
                                "note": ("shared-memory roof of the CTA-pair FP4 tile: 74 KB of operand traffic "
                                         "(TMA writes + tensor-core reads) per 256-frame k-block at 128 B/clk = 578 "
                                         "clocks vs 448 clocks of MMAs (DESIGN.md §17.2)")}
                               if args.variant == "fp4" else None),
                 "ops_per_launch": ops, "ms_per_launch": gemm_ms / gemm_n if gemm_n else None,
                 "traffic": traffic.get("gemm_i8_tc2_kernel<fp4>" if args.variant == "fp4" else
                                        "gemm_i8_tc2_kernel<i8>", {}).get("bytes_per_launch")
                 if args.variant in ("tc", "fp4") else None,
                 "traffic_note": "ncu dram read + write bytes per launch (profiles/r02_traffic.json)"}
    fma_peak_gtaps = 148 * 128 * f_clk / 1e9         # 128 fp32 FMA lanes per clock per SM
    vm = args.gamma_order == "vmajor"
    s1_key = "stage1_w_kernel" if vm else "stage1_tma_kernel<1,4,1,256>"
    roof_s1 = {"kernel": ("refocus_stage1_w (KB5w, v-major window stage 1: 8 planes per staged slab, one launch "
                          "per 64 planes)" if vm else "refocus_stage1_tma (KB5, 4 planes per pass)"),
               "bound": "alu",
               "achieved": s1_gtaps, "peak": lds_peak_gtaps, "unit": "Gtap/s",
               "frac": s1_gtaps / lds_peak_gtaps if s1_gtaps else None,
               "peak_note": ("taps per second at one 4-byte shared-memory load per tap (+1 FFMA): 148 SMs x 32 "
                             "LDS lanes/clk x median SM clock of this run (DESIGN.md §5)" +
                             ("; KB5w loads alpha/2 bytes per tap (rows reused from registers), so this is the "
                              "one-load-per-tap design's roof kept across rounds; fma_view is the FP32 FMA-lane "
                              "roof" if vm else "")),
               "fma_view": {"peak": fma_peak_gtaps, "frac": s1_gtaps / fma_peak_gtaps if s1_gtaps else None,
                            "note": "one FFMA lane per tap: 148 SMs x 128 FP32 lanes/clk x median SM clock"},
               "taps_per_step": taps, "ms_per_step": s1_ms / args.steps,
               "hbm_view": {"algorithmic_bytes_per_step": span, "achieved_gbs": s1_gbs, "peak_gbs": hbm,
                            "frac": s1_gbs / hbm if s1_gbs else None,
                            "note": "per-plane span bytes / time; > 1 possible because planes share HBM passes"},
               "issue_view": issue_view(traffic.get(s1_key, {}), s1_ms / args.steps, f_clk),
               "traffic": traffic.get(s1_key, {}).get("bytes_per_launch"),
               "traffic_note": (f"ncu dram read + write bytes per launch of {s1_key} (profiles/r02_traffic.json); "
                                + ("one launch per step" if vm else "achieved is per step (16 launches)"))}
    dominant = roof_s1 if (s1_ms > gemm_ms) else roof_gemm
    # north_star's correlation metric is the kind::i8 kernel's fraction of the int8 peak: when
    # the step runs the FP4 GEMM, time the kind::i8 GEMM on the same frames too (after the timed
    # region, not part of value)
    int8_side = None
    if args.variant == "fp4" and not use_dist:
        c8 = Context(roi_a, roi_b, n, device=local, variant="tc", gamma_order=args.gamma_order)
        for it in range(5):
            if it == 2:
                c8.set_timing(True)
            c8.reset()
            c8.load_frames(frames_dev)
            c8.correlate(gamma)
        g8_ms, g8_n = c8.kernel_time_ms(KC_GEMM)
        c8.close()
        i8_tops = ops / (g8_ms / g8_n / 1e3) / 1e12
        i8_peak = 2.0 * peaks["bf16_tflops"]
        int8_side = {"kernel": "gemm_i8_tc2 (KB2, cta_group::2, kind::i8, int32 accumulation)",
                     "ms_per_launch": g8_ms / g8_n, "achieved": i8_tops, "peak": i8_peak, "unit": "TOPS",
                     "frac": i8_tops / i8_peak, "frac_of_clock_peak": i8_tops / (148 * 8192 * 2 * f_clk / 1e12),
                     "note": "same frames, epilogue and Gamma, timed after the step loop; not part of value"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(frames_np, roi_a, roi_b, alphas, args.cpu_pixels, args.planes)
    out = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": {"tc": "u8 x u8 -> s32 (S_ab)", "popc": "u32 popc(and) -> s32 (S_ab)",
                  "bits": "1-bit streams -> u8 in smem, u8 x u8 -> s32 (S_ab)",
                  "fp4": "e2m1 {0,1} x e2m1 -> f32 exact integers -> s32 (S_ab)"}[args.variant]
                 + ", f64 -> f32 (Gamma), f32/f64 (refocus)",
        "data": "synthetic",
        "config": {"workload": (f"configs[1] (+configs[3] stack): SwissSPAD2 256x512 frames, rho_a {roi_a}, "
                                f"rho_b {roi_b}, {n_total} Bernoulli({args.occupancy}) frames per step "
                                f"(split across {world} rank(s)) -> Gamma {p_a}x{p_b} -> {args.planes}-plane "
                                f"refocus stack"),
                   "frames_per_step": n_total, "frames_per_step_per_rank": n, "planes_per_step": args.planes,
                   "alphas": "linspace(0.5, 2.0, P)", "variant": args.variant, "gamma_order": args.gamma_order,
                   "parallelism": (f"frame-sharded x{world} (" + {"lib": "library: GEMM-epilogue reduction into the "
                                                                          "owners' shards over peer memory"
                                                                   if not args.no_fused_reduce else
                                                                   "library NCCL reduce-scatter",
                                                                   "rows": "torch.distributed panelised reduce-scatter",
                                                                   "tiles": "output-tile sharding"}[mode] + ")")
                   if use_dist else "single GPU",
                   "l2": "inputs larger than L2 (Gamma 17 GB, operands 1.3 GB) - no flush needed"},
        "gpu_launches": launches,
        "roofline": dominant,
        "rooflines": [roof_gemm, roof_s1],
        "int8_gemm": int8_side,
        "stages_ms_per_step": {"expand": kt["expand"][0] / args.steps, "gemm": gemm_ms / args.steps,
                               "refocus_coords": kt["coords"][0] / args.steps,
                               "refocus_stage1": s1_ms / args.steps, "refocus_stage2": kt["stage2"][0] / args.steps,
                               "finalize": kt["finalize"][0] / args.steps},
        "correlation_frames_per_s": n_total / (corr_ms / 1e3) if corr_ms else None,
        "planes_per_s": args.planes / (ref_ms / 1e3) if ref_ms else None,
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "paper_context": "paper: 20x (correlation) / 500x (refocus) OpenCL-GPU vs CPU on RTX 2080 Ti vs "
                         "i7-9700K (PAPER.md:38, 52, 279-292); no absolute timings in the text",
    }
    if cpu and corr_ms and ref_ms:
        parts = cpu["extrapolated_parts_s"]
        out["speedup_vs_oracle"] = {
            "correlation": (parts["marginals"] + parts["pair_sums"]) / (corr_ms / 1e3),
            "refocus": parts["refocus"] / (ref_ms / 1e3),
            "note": (f"oracle stage times on {cpu['cores']} host cores (extrapolated, see cpu_baseline) / GPU "
                     "stage times of this run; the paper's 20x / 500x compare OpenCL on an RTX 2080 Ti with "
                     "its own CPU code on an i7-9700K")}
    print(json.dumps(out), file=json_out, flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
