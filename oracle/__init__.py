"""CPU oracle for the CPI hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  It is independent of the CUDA path
(paper_2407_20692_b200): the two share no code, and neither imports the other; both
consume inputs from the ``synth`` module only.

Layers:
  * ``cpi_oracle.c`` (plain C loops, fp64, -ffp-contract=off) — unpack, sums, exact
    Gamma, 4D-multilinear refocusing; built into ``liboracle.so`` by ``build()``.
  * this module — ctypes marshalling plus one pure-numpy reference,
    ``correlate_naive_fp64`` (SPEC.md:208-211 per-frame fp64 accumulation), used as the
    brute-force cross-check of the C sums on tiny inputs.

Parity status per function (see DESIGN.md §Oracle pins):
  * unpack / marginals / pair_sums / gamma — pinned (hand values, brute force, closed
    forms, invariants, chaotic-light statistics).
  * refocus — pinned to the declared convention by closed forms
    (alpha=1 ghost image, sheared ramp, integer shear, delta, constant, interp4 examples);
    physical fidelity of the refocusing transform: "parity unpinned" (the paper defers
    the transform to cited references).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "cpi_oracle.c"
_LIB = _HERE / "liboracle.so"
_lock = threading.Lock()
_lib = None

BOUNDARY_SKIP = 0   # skip_and_renormalize (S:279, S:336 default)
BOUNDARY_CLAMP = 1  # clamp


class _Roi(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_int32), ("y0", ctypes.c_int32),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


def build(force: bool = False) -> Path:
    """Compile cpi_oracle.c with gcc (plain C17, OpenMP, no FMA contraction)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        cmd = ["gcc", "-std=c17", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", str(_SRC), "-o", str(_LIB) + ".tmp", "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(str(_LIB) + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(str(_LIB))
            P = ctypes.c_void_p
            i64, i32 = ctypes.c_int64, ctypes.c_int
            lib.oracle_unpack.argtypes = [P, i64, i32, i32, i32, _Roi, P]
            lib.oracle_marginals.argtypes = [P, i64, i32, i32, i32, _Roi, P]
            lib.oracle_pair_sums.argtypes = [P, i64, i32, i32, i32, _Roi, _Roi, P, i64, P, i32]
            lib.oracle_gamma.argtypes = [P, P, P, i64, i64, i64, P]
            lib.oracle_gamma_spec.argtypes = [P, P, P, i64, i64, i64, P]
            lib.oracle_interp4.argtypes = [P, i32, i32, i32, i32, i32, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_double]
            lib.oracle_interp4.restype = ctypes.c_double
            lib.oracle_refocus.argtypes = [P, i32, i32, i32, i32, i32, P, i32, i32, P, i64, P, P, i32]
            lib.oracle_refocus_affine.argtypes = [P, i32, i32, i32, i32, i32, P, i32, i32, P, i64, P, P, i32]
            for f in ("oracle_unpack", "oracle_marginals", "oracle_pair_sums", "oracle_gamma",
                      "oracle_gamma_spec", "oracle_refocus", "oracle_refocus_affine"):
                getattr(lib, f).restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _frames(frames: np.ndarray):
    f = np.ascontiguousarray(frames, dtype=np.uint8)
    if f.ndim != 3:
        raise ValueError("frames must be uint8 [N][H][W/8]")
    n, h, wb = f.shape
    return f, n, wb * 8, h


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed (rc={rc})")


def unpack(frames: np.ndarray, roi, msb: bool = False) -> np.ndarray:
    """A^i_p -> uint8 [N][P], p = m*width + j."""
    f, n, W, H = _frames(frames)
    out = np.empty((n, roi[2] * roi[3]), dtype=np.uint8)
    _check(_load().oracle_unpack(_ptr(f), n, W, H, int(msb), _Roi(*roi), _ptr(out)), "unpack")
    return out


def marginals(frames: np.ndarray, roi, msb: bool = False) -> np.ndarray:
    """S[p] = sum_i A^i_p (Eq. 1 single-pixel sums) -> int64 [P]."""
    f, n, W, H = _frames(frames)
    out = np.empty(roi[2] * roi[3], dtype=np.int64)
    _check(_load().oracle_marginals(_ptr(f), n, W, H, int(msb), _Roi(*roi), _ptr(out)), "marginals")
    return out


def pair_sums(frames: np.ndarray, roi_a, roi_b, rows=None, msb: bool = False,
              threads: int = 0) -> np.ndarray:
    """S_ab[r][q] = sum_i A^i_{rows[r]} B^i_q (Eq. 1 pair sums) -> int64 [R][P_b]."""
    f, n, W, H = _frames(frames)
    pb = roi_b[2] * roi_b[3]
    if rows is None:
        rows_arr = None
        nrows = roi_a[2] * roi_a[3]
    else:
        rows_arr = np.ascontiguousarray(rows, dtype=np.int64)
        nrows = rows_arr.size
    out = np.empty((nrows, pb), dtype=np.int64)
    rc = _load().oracle_pair_sums(_ptr(f), n, W, H, int(msb), _Roi(*roi_a), _Roi(*roi_b),
                                  None if rows_arr is None else _ptr(rows_arr), nrows,
                                  _ptr(out), int(threads))
    _check(rc, "pair_sums")
    return out


def gamma(s_ab: np.ndarray, s_a_rows: np.ndarray, s_b: np.ndarray, n: int) -> np.ndarray:
    """Exact-rational Gamma of Eq. (1) rounded once to fp64 -> float64 [R][P_b]."""
    s_ab = np.ascontiguousarray(s_ab, dtype=np.int64)
    s_a_rows = np.ascontiguousarray(s_a_rows, dtype=np.int64)
    s_b = np.ascontiguousarray(s_b, dtype=np.int64)
    out = np.empty(s_ab.shape, dtype=np.float64)
    _check(_load().oracle_gamma(_ptr(s_ab), _ptr(s_a_rows), _ptr(s_b), int(n), s_ab.shape[0],
                                s_ab.shape[1], _ptr(out)), "gamma")
    return out


def gamma_spec(s_ab, s_a_rows, s_b, n) -> np.ndarray:
    """SPEC finalize expression, for comparison only."""
    s_ab = np.ascontiguousarray(s_ab, dtype=np.int64)
    s_a_rows = np.ascontiguousarray(s_a_rows, dtype=np.int64)
    s_b = np.ascontiguousarray(s_b, dtype=np.int64)
    out = np.empty(s_ab.shape, dtype=np.float64)
    _check(_load().oracle_gamma_spec(_ptr(s_ab), _ptr(s_a_rows), _ptr(s_b), int(n),
                                     s_ab.shape[0], s_ab.shape[1], _ptr(out)), "gamma_spec")
    return out


def correlate(frames: np.ndarray, roi_a, roi_b, rows=None, msb: bool = False, threads: int = 0):
    """Full Eq. (1) pipeline: returns dict(s_ab, s_a, s_b, n, gamma) for the chosen A rows."""
    s_a = marginals(frames, roi_a, msb)
    s_b = marginals(frames, roi_b, msb)
    s_ab = pair_sums(frames, roi_a, roi_b, rows, msb, threads)
    n = frames.shape[0]
    rows_idx = np.arange(s_a.size) if rows is None else np.asarray(rows, dtype=np.int64)
    g = gamma(s_ab, s_a[rows_idx], s_b, n) if n > 0 else None
    return dict(s_ab=s_ab, s_a=s_a, s_b=s_b, n=n, gamma=g, rows=rows_idx)


def correlate_naive_fp64(frames: np.ndarray, roi_a, roi_b) -> np.ndarray:
    """SPEC correlate_naive: per-frame fp64 accumulation of A^i (x) B^i and of
    the two mean images in frame order, then Eq. (1).  Pure numpy; tiny inputs only.
    Independent of the C code (own unpack via numpy bit ops)."""
    n = frames.shape[0]
    def arm(roi):
        x0, y0, w, h = roi
        cols = np.arange(x0, x0 + w)
        sub = frames[:, y0:y0 + h, :][:, :, cols // 8]
        return ((sub >> (cols % 8)) & 1).reshape(n, w * h).astype(np.float64)
    A, B = arm(roi_a), arm(roi_b)
    sab = np.zeros((A.shape[1], B.shape[1]))
    sa = np.zeros(A.shape[1])
    sb = np.zeros(B.shape[1])
    for i in range(n):
        sab += np.outer(A[i], B[i])
        sa += A[i]
        sb += B[i]
    return sab / n - np.outer(sa / n, sb / n)


def interp4(g: np.ndarray, dims, cAx, cBx, cAy, cBy) -> float:
    """S:290 interp4 at one 4D point; dims = (Wa, Ha, Wb, Hb); g is [Pa][Pb] fp32/fp64."""
    g = np.ascontiguousarray(g)
    f32 = g.dtype == np.float32
    if not f32:
        g = g.astype(np.float64, copy=False)
    Wa, Ha, Wb, Hb = dims
    return _load().oracle_interp4(_ptr(g), int(f32), Wa, Ha, Wb, Hb, cAx, cBx, cAy, cBy)


def refocus(g: np.ndarray, dims, alphas, boundary: int = BOUNDARY_SKIP, pixels=None,
            threads: int = 0, return_counts: bool = False):
    """Refocused planes -> float64 [P][Ha][Wa] (pixels None) or [P][K] for a
    list of K (x, y) output pixels.  Gamma fp32 is widened exactly to fp64."""
    g = np.ascontiguousarray(g)
    f32 = g.dtype == np.float32
    if not f32:
        g = np.ascontiguousarray(g, dtype=np.float64)
    Wa, Ha, Wb, Hb = dims
    if g.shape != (Wa * Ha, Wb * Hb):
        raise ValueError("gamma must be [Wa*Ha][Wb*Hb]")
    al = np.ascontiguousarray(alphas, dtype=np.float64).ravel()
    if pixels is None:
        pix = None
        npix = Wa * Ha
    else:
        pix = np.ascontiguousarray(pixels, dtype=np.int32).reshape(-1, 2)
        npix = pix.shape[0]
    out = np.empty((al.size, npix), dtype=np.float64)
    cnt = np.empty((al.size, npix), dtype=np.int64)
    rc = _load().oracle_refocus(_ptr(g), int(f32), Wa, Ha, Wb, Hb, _ptr(al), al.size,
                                int(boundary), None if pix is None else _ptr(pix), npix,
                                _ptr(out), _ptr(cnt), int(threads))
    if rc == -2:
        raise ValueError("DegenerateAlpha: alpha must be finite and non-zero (S:303)")
    _check(rc, "refocus")
    if pixels is None:
        out = out.reshape(al.size, Ha, Wa)
        cnt = cnt.reshape(al.size, Ha, Wa)
    return (out, cnt) if return_counts else out


def default_map(alpha: float):
    """The SPEC default map as a general affine map row (refocus_affine layout)."""
    a = float(alpha)
    b = 1.0 - a
    return [a, b, 0.0, 0.0, 1.0, 0.0, a, b, 0.0, 0.0, 1.0, 0.0]


def refocus_affine(g: np.ndarray, dims, maps, boundary: int = BOUNDARY_SKIP, pixels=None,
                   threads: int = 0, return_counts: bool = False):
    """Refocused planes under general affine maps (S:273 RefocusMap):
    maps = [P][12] rows {ax, bx, cx, dx, ex, fx, ay, by, cy, dy, ey, fy} (see
    cpi_oracle.c refocus_pixel_affine).  Output as refocus()."""
    g = np.ascontiguousarray(g)
    f32 = g.dtype == np.float32
    if not f32:
        g = np.ascontiguousarray(g, dtype=np.float64)
    Wa, Ha, Wb, Hb = dims
    if g.shape != (Wa * Ha, Wb * Hb):
        raise ValueError("gamma must be [Wa*Ha][Wb*Hb]")
    mp = np.ascontiguousarray(maps, dtype=np.float64).reshape(-1, 12)
    if pixels is None:
        pix = None
        npix = Wa * Ha
    else:
        pix = np.ascontiguousarray(pixels, dtype=np.int32).reshape(-1, 2)
        npix = pix.shape[0]
    out = np.empty((mp.shape[0], npix), dtype=np.float64)
    cnt = np.empty((mp.shape[0], npix), dtype=np.int64)
    rc = _load().oracle_refocus_affine(_ptr(g), int(f32), Wa, Ha, Wb, Hb, _ptr(mp), mp.shape[0],
                                       int(boundary), None if pix is None else _ptr(pix), npix,
                                       _ptr(out), _ptr(cnt), int(threads))
    if rc == -2:
        raise ValueError("map coefficients must be finite")
    _check(rc, "refocus_affine")
    if pixels is None:
        out = out.reshape(mp.shape[0], Ha, Wa)
        cnt = cnt.reshape(mp.shape[0], Ha, Wa)
    return (out, cnt) if return_counts else out
