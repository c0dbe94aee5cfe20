"""Small helpers shared by tests (no method arithmetic beyond what each test states)."""
from fractions import Fraction

import numpy as np


def pack(bits: np.ndarray) -> np.ndarray:
    """bool/uint8 [N][H][W] -> packed lsb-first uint8 [N][H][W/8] (layout of P:65-69)."""
    return np.packbits(np.asarray(bits, dtype=np.uint8), axis=-1, bitorder="little")


def unpack_np(frames: np.ndarray, roi) -> np.ndarray:
    """Independent numpy unpack of one RoI -> uint8 [N][P] (np.unpackbits, not the oracle)."""
    x0, y0, w, h = roi
    allbits = np.unpackbits(frames, axis=-1, bitorder="little")
    return allbits[:, y0:y0 + h, x0:x0 + w].reshape(frames.shape[0], w * h)


def frac(s: str) -> Fraction:
    return Fraction(s)


def exact_gamma(s_ab, s_a, s_b, n) -> Fraction:
    return Fraction(int(n) * int(s_ab) - int(s_a) * int(s_b), int(n) * int(n))
