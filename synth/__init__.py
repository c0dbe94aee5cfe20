"""Seeded synthetic inputs for the CPI hot path (shared by the oracle tests, the GPU
parity tests and bench.py).

This module holds NONE of the method's arithmetic: no pair sums, no marginals, no
correlation, no refocusing.  It only draws frames / correlation tensors / plane grids
with stated seeds so that both sides of a parity test consume identical bytes.

Frame layout (§2 "Input Dataset"; SPEC.md:28-33 FrameLayout):
  * a frame is 256 rows x 512 columns, 1 bit per pixel, row stride 64 bytes,
    16,384 bytes per frame; frames are stored frame-major then row-major;
  * bit order inside a byte is lsb_first: column c of a row is bit (c % 8) of byte
    c // 8 (declared convention — the paper does not state it);
  * a "file" holds 512 frames, so frame index i lives in file i // 512.

Generators are keyed by (seed, file index) so any frame slice [frame0, frame0+n) is
reproducible independently of how the sequence was sharded (frame-sharded multi-GPU
runs draw their own slices).
"""
from __future__ import annotations

import math
import os
import statistics
from concurrent.futures import ThreadPoolExecutor

import numpy as np

FRAME_W = 512          # PAPER.md:65  "Frame size: 256 x 512 px"
FRAME_H = 256
FRAMES_PER_FILE = 512  # PAPER.md:64  "512 binary frames"
SEED_ARMS = 2407       # seed for arm data
SEED_NOISE = 20692     # seed for independent noise


def frame_bytes(width: int = FRAME_W, height: int = FRAME_H) -> int:
    return height * (width // 8)


def _pack_lsb(bits: np.ndarray) -> np.ndarray:
    """bool [..., W] -> uint8 [..., W/8], column c -> bit c%8 of byte c//8."""
    return np.packbits(bits, axis=-1, bitorder="little")


def _bernoulli_file(seed: int, file_idx: int, f: float, width: int, height: int) -> np.ndarray:
    rng = np.random.default_rng([seed, file_idx])
    if f == 0.5:
        # every bit an independent fair coin: random bytes are exactly that
        return rng.integers(0, 256, size=(FRAMES_PER_FILE, height, width // 8), dtype=np.uint8)
    u = rng.random((FRAMES_PER_FILE, height, width), dtype=np.float32)
    return _pack_lsb(u < np.float32(f))


def bernoulli_frames(n_frames: int, f: float = 0.05, seed: int = SEED_ARMS, frame0: int = 0,
                     width: int = FRAME_W, height: int = FRAME_H,
                     threads: int | None = None) -> np.ndarray:
    """i.i.d. Bernoulli(f) bits in SwissSPAD2 layout -> uint8 [n_frames][height][width/8].

    Throughput workload of SURVEY §8(d): f = 0.05 (sparse SPAD-like) or 0.5.
    Frames [frame0, frame0 + n_frames) of the infinite seeded sequence.
    """
    if width % 8 or height <= 0 or width <= 0:
        raise ValueError("width must be a positive multiple of 8")
    out = np.empty((n_frames, height, width // 8), dtype=np.uint8)
    if n_frames == 0:
        return out
    first = frame0 // FRAMES_PER_FILE
    last = (frame0 + n_frames - 1) // FRAMES_PER_FILE
    files = list(range(first, last + 1))

    def fill(k: int) -> None:
        blk = _bernoulli_file(seed, k, f, width, height)
        lo = max(frame0, k * FRAMES_PER_FILE)
        hi = min(frame0 + n_frames, (k + 1) * FRAMES_PER_FILE)
        out[lo - frame0:hi - frame0] = blk[lo - k * FRAMES_PER_FILE:hi - k * FRAMES_PER_FILE]

    nthreads = threads or min(len(files), os.cpu_count() or 1)
    if nthreads <= 1 or len(files) == 1:
        for k in files:
            fill(k)
    else:
        with ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(fill, files))
    return out


def speckle_frames(n_frames: int, roi_a, roi_b, f: float = 0.5, grain: int = 2,
                   shift_b=(0, 0), seed: int = SEED_NOISE,
                   width: int = FRAME_W, height: int = FRAME_H) -> np.ndarray:
    """Chaotic-light (thresholded Gaussian speckle) frames with a known correlation.

    Model (SURVEY §8(d) "Correctness data"): per frame i an i.i.d. N(0,1) field W_i is
    drawn on integer source cells; Z_i(s) = (1/g) * sum_{a,b < g} W_i(s + (a, b)) has unit
    variance.  Pixel (j, m) of arm A samples Z_i at source (j, m); pixel (k, n) of arm B
    samples Z_i at source (k + dx, n + dy).  A pixel fires when Z_i > tau with
    tau = Phi^{-1}(1 - f).  Pixels outside both RoIs are 0.

    Two samples at source offset (Dx, Dy) have correlation rho = (1-|Dx|/g)(1-|Dy|/g)
    for |Dx|,|Dy| < g, else 0 (fraction of shared cells).  The expected value of Eq. (1)
    under this model is a property checked in tests, not computed here.
    roi = (x0, y0, w, h) in frame coordinates.
    """
    ax0, ay0, aw, ah = roi_a
    bx0, by0, bw, bh = roi_b
    dx, dy = shift_b
    g = int(grain)
    tau = statistics.NormalDist().inv_cdf(1.0 - f) if 0.0 < f < 1.0 else (math.inf if f <= 0 else -math.inf)
    # source window covering both arms' samples
    sx0 = min(0, dx)
    sy0 = min(0, dy)
    sx1 = max(aw, bw + dx) + g
    sy1 = max(ah, bh + dy) + g
    rng = np.random.default_rng([seed, 7])
    out = np.zeros((n_frames, height, width // 8), dtype=np.uint8)
    chunk = 256
    for c0 in range(0, n_frames, chunk):
        c1 = min(n_frames, c0 + chunk)
        w = rng.standard_normal((c1 - c0, sy1 - sy0, sx1 - sx0))
        # box filter of width g along both axes (cumulative sums), scaled by 1/g
        cs = np.cumsum(np.pad(w, ((0, 0), (1, 0), (0, 0))), axis=1)
        w = cs[:, g:, :] - cs[:, :-g, :]
        cs = np.cumsum(np.pad(w, ((0, 0), (0, 0), (1, 0))), axis=2)
        z = (cs[:, :, g:] - cs[:, :, :-g]) / g
        bits = np.zeros((c1 - c0, height, width), dtype=bool)
        za = z[:, (0 - sy0):(0 - sy0) + ah, (0 - sx0):(0 - sx0) + aw]
        zb = z[:, (dy - sy0):(dy - sy0) + bh, (dx - sx0):(dx - sx0) + bw]
        bits[:, ay0:ay0 + ah, ax0:ax0 + aw] = za > tau
        bits[:, by0:by0 + bh, bx0:bx0 + bw] = zb > tau
        out[c0:c1] = _pack_lsb(bits)
    return out


def random_gamma(p_a: int, p_b: int, seed: int = SEED_NOISE, scale: float = 0.25) -> np.ndarray:
    """A dense fp32 tensor with values in [-scale, scale) shaped like Gamma [P_a][P_b]
    (Eq. (1) entries lie in [-1/4, 1/4]).  Used as refocus input where the
    refocus stage is tested in isolation."""
    rng = np.random.default_rng([seed, 11])
    return (rng.random((p_a, p_b), dtype=np.float32) * np.float32(2 * scale) - np.float32(scale))


def alpha_grid(n_planes: int, lo: float = 0.5, hi: float = 2.0) -> np.ndarray:
    """Refocusing parameters alpha_p = lo + (hi - lo) * p / (P - 1) in fp64 (SURVEY Q12:
    the paper gives plane counts 100/261/1000, but not the alpha range).
    The 64-plane grid hits alpha = 1.0 exactly at p = 21."""
    if n_planes == 1:
        return np.array([1.0])
    p = np.arange(n_planes, dtype=np.float64)
    return lo + (hi - lo) * p / (n_planes - 1)


# Workload geometry of BASELINE.json configs (SURVEY §8 sizes).
ROI_FULL_A = (0, 0, 256, 256)      # left half, "pixel 1 to pixel 256"
ROI_FULL_B = (256, 0, 256, 256)    # right half, "pixel 257 to 512"
ROI_TINY_A = (124, 124, 8, 8)      # configs[0]: 8x8 rho_a, not byte-aligned
ROI_TINY_B = (382, 126, 4, 4)      # configs[0]: 4x4 rho_b, not byte-aligned
ROI_128_A = (64, 64, 128, 128)     # P:307 128x128 refocus RoI, centred
ROI_128_B = (320, 64, 128, 128)
