"""ctypes loader for libcpi.so (include/cpi.h).  Fails loudly: there is no fallback path."""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libcpi.so"

CPI_OK = 0
STATUS = {
    0: "CPI_OK", -1: "CPI_ERR_INVALID_ARG", -2: "CPI_ERR_LAYOUT", -3: "CPI_ERR_ROI_OUT_OF_BOUNDS",
    -4: "CPI_ERR_SIZE_MISMATCH", -5: "CPI_ERR_CAPACITY", -6: "CPI_ERR_ZERO_FRAMES",
    -7: "CPI_ERR_DEGENERATE_ALPHA", -8: "CPI_ERR_EMPTY_ANGULAR_GRID", -9: "CPI_ERR_STATE",
    -10: "CPI_ERR_CUDA", -11: "CPI_ERR_OOM", -12: "CPI_ERR_UNSUPPORTED", -13: "CPI_ERR_NCCL",
}
CPI_NCCL_ID_BYTES = 128
CPI_LSB_FIRST, CPI_MSB_FIRST = 0, 1
CPI_HOST, CPI_DEVICE = 0, 1
CPI_VARIANT_TC, CPI_VARIANT_POPC, CPI_KEEP_COUNTS, CPI_VARIANT_FP4, CPI_GAMMA_UBLOCKED = 0, 1, 2, 4, 8
CPI_VARIANT_TC_BITS = 64   # f1: bit-stream operands unpacked inside the CTA-pair kind::i8 GEMM
CPI_GAMMA_VMAJOR = 16
CPI_FUSED_REDUCE = 32
CPI_SHARD_HANDLE_BYTES = 64
CPI_SKIP_RENORMALIZE, CPI_CLAMP = 0, 1
KC_GEMM, KC_EXPAND, KC_STAGE1, KC_STAGE2, KC_FINALIZE, KC_COORDS, KC_RESAMPLE = range(7)

# every symbol include/cpi.h declares
EXPORTS = ["cpi_create", "cpi_destroy", "cpi_last_error", "cpi_status_string", "cpi_load_frames",
           "cpi_correlate", "cpi_finalize", "cpi_finalize_counts", "cpi_get_counts", "cpi_reset",
           "cpi_refocus", "cpi_launch_count", "cpi_set_timing", "cpi_kernel_time_ms",
           "cpi_abi_version", "cpi_correlate_rows", "cpi_row_align", "cpi_counts_dev", "cpi_correlate_rows_to",
           "cpi_shard_layout", "cpi_nccl_unique_id", "cpi_shard_ipc_handle", "cpi_open_peer_shards",
           "cpi_bin_frames", "cpi_read_bin"]


class CpiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {msg}")


class Roi(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_int32), ("y0", ctypes.c_int32),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class Layout(ctypes.Structure):
    _fields_ = [("width_px", ctypes.c_int32), ("height_px", ctypes.c_int32),
                ("bit_order", ctypes.c_int32)]


class Config(ctypes.Structure):
    _fields_ = [("layout", Layout), ("roi_a", Roi), ("roi_b", Roi), ("max_frames", ctypes.c_int64),
                ("device", ctypes.c_int32), ("flags", ctypes.c_uint32), ("rank", ctypes.c_int32),
                ("world", ctypes.c_int32), ("nccl_id", ctypes.c_void_p)]


class RefocusSpec(ctypes.Structure):
    _fields_ = [("alphas", ctypes.POINTER(ctypes.c_double)), ("n_planes", ctypes.c_int32),
                ("boundary", ctypes.c_int32), ("gamma_dev", ctypes.c_void_p),
                ("row0", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("row_block", ctypes.c_int32), ("row_stride", ctypes.c_int32),
                ("affine", ctypes.POINTER(ctypes.c_double))]


_lib = None


def load():
    """Load libcpi.so (building it first if the sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if os.environ.get("CPI_NO_BUILD") != "1":
        try:
            from . import build as _b
            if _b._stale() and Path(_b.NVCC).exists():
                _b.build()
        except Exception:
            if not LIB_PATH.exists():
                raise
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2407_20692_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "cpi_create": ([ctypes.POINTER(Config), ctypes.POINTER(P)], i32),
        "cpi_destroy": ([P], None),
        "cpi_last_error": ([P], ctypes.c_char_p),
        "cpi_status_string": ([i32], ctypes.c_char_p),
        "cpi_load_frames": ([P, P, i64, i32, P], i32),
        "cpi_correlate": ([P, P, P], i32),
        "cpi_finalize": ([P, P, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64), P], i32),
        "cpi_shard_layout": ([P, ctypes.POINTER(i32), ctypes.POINTER(i32)], i32),
        "cpi_nccl_unique_id": ([P], i32),
        "cpi_shard_ipc_handle": ([P, P], i32),
        "cpi_open_peer_shards": ([P, P], i32),
        "cpi_finalize_counts": ([P, P, i64, i64, P, P, i64, P, P], i32),
        "cpi_get_counts": ([P, P, P, P, ctypes.POINTER(i64), P], i32),
        "cpi_reset": ([P, P], i32),
        "cpi_refocus": ([P, ctypes.POINTER(RefocusSpec), P, P], i32),
        "cpi_launch_count": ([P], i64),
        "cpi_set_timing": ([P, i32], i32),
        "cpi_kernel_time_ms": ([P, i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)], i32),
        "cpi_abi_version": ([], i32),
        "cpi_correlate_rows": ([P, i64, i64, P, P], i32),
        "cpi_correlate_rows_to": ([P, i64, i64, P, P], i32),
        "cpi_row_align": ([P], i64),
        "cpi_counts_dev": ([P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P)], i32),
        "cpi_bin_frames": ([ctypes.c_char_p, ctypes.POINTER(Layout), ctypes.POINTER(i64)], i32),
        "cpi_read_bin": ([ctypes.c_char_p, ctypes.POINTER(Layout), i64, i64, P], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib
