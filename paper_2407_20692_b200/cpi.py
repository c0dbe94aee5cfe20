"""Python binding of the CPI C ABI (include/cpi.h) — argument marshalling only.

Every step of the hot path runs in libcpi.so's CUDA kernels; this module only converts
torch tensors / numpy arrays into pointers, picks the current torch CUDA stream, and turns
status codes into exceptions.  torch supplies device memory and streams (plumbing).
Names follow the C functions: load_frames / correlate / finalize / refocus / get_counts.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import CpiError

FRAME_W, FRAME_H = 512, 256   # SwissSPAD2 frame
# B pixel (Gamma column) orders, include/cpi.h: row-major q = v W_b + u, u-blocked, v-major u H_b + v
GAMMA_ORDERS = {"rowmajor": 0, "ublocked": _lib.CPI_GAMMA_UBLOCKED, "vmajor": _lib.CPI_GAMMA_VMAJOR}


def _torch():
    import torch
    return torch


class Context:
    """One CPI accumulation context on one GPU (cpi_create ... cpi_destroy)."""

    def __init__(self, roi_a, roi_b, max_frames: int, *, width: int = FRAME_W, height: int = FRAME_H,
                 bit_order: int = _lib.CPI_LSB_FIRST, device: int = 0, variant: str = "tc",
                 keep_counts: bool = False, gamma_blocked: bool = False, gamma_order: Optional[str] = None,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None, fused_reduce: bool = False):
        """rank / world / nccl_id: frame-sharded multi-GPU mode (include/cpi.h cpi_config; world >= 2
        needs keep_counts and the same nccl_unique_id() bytes on every rank; cpi_create is
        collective).  fused_reduce: CPI_FUSED_REDUCE (the GEMM epilogue adds into the owners'
        shards; without nccl_id the caller maps the peers with open_peer_shards)."""
        self._lib = _lib.load()
        if variant not in ("tc", "popc", "fp4", "bits"):
            raise ValueError("variant must be 'tc', 'popc', 'fp4' or 'bits'")
        flags = {"tc": _lib.CPI_VARIANT_TC, "popc": _lib.CPI_VARIANT_POPC, "fp4": _lib.CPI_VARIANT_FP4,
                 "bits": _lib.CPI_VARIANT_TC_BITS}[variant]
        if keep_counts:
            flags |= _lib.CPI_KEEP_COUNTS
        if fused_reduce:
            flags |= _lib.CPI_FUSED_REDUCE
        if gamma_order is None:
            gamma_order = "ublocked" if gamma_blocked else "rowmajor"
        if gamma_order not in GAMMA_ORDERS:
            raise ValueError(f"gamma_order must be one of {sorted(GAMMA_ORDERS)}")
        flags |= GAMMA_ORDERS[gamma_order]   # B pixel (Gamma column) order, include/cpi.h
        self._id_buf = None
        if nccl_id is not None:
            if len(nccl_id) != _lib.CPI_NCCL_ID_BYTES:
                raise ValueError(f"nccl_id must be {_lib.CPI_NCCL_ID_BYTES} bytes (nccl_unique_id())")
            self._id_buf = ctypes.create_string_buffer(bytes(nccl_id), _lib.CPI_NCCL_ID_BYTES)
        elif world > 1 and not fused_reduce:
            raise ValueError("world > 1 needs nccl_id (nccl_unique_id()), or fused_reduce=True (external mode)")
        cfg = _lib.Config(_lib.Layout(width, height, bit_order), _lib.Roi(*roi_a), _lib.Roi(*roi_b),
                          int(max_frames), int(device), flags, int(rank), int(world),
                          ctypes.cast(self._id_buf, ctypes.c_void_p) if self._id_buf is not None else None)
        h = ctypes.c_void_p()
        st = self._lib.cpi_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != 0:
            raise CpiError(st, self._lib.cpi_last_error(None).decode())
        self._h = h
        self.roi_a, self.roi_b = tuple(roi_a), tuple(roi_b)
        self.p_a = roi_a[2] * roi_a[3]
        self.p_b = roi_b[2] * roi_b[3]
        self.device = device
        self.width, self.height = width, height
        self.frame_bytes = (width // 8) * height
        self.max_frames = int(max_frames)
        self.variant = variant
        self.keep_counts = keep_counts
        self.rank, self.world = (int(rank), int(world)) if world > 1 else (0, 1)
        self.sharded = self._id_buf is not None or (world > 1 and fused_reduce)
        self.fused_reduce = fused_reduce
        self.shard_rows = (0, self.p_a)    # owned Gamma rows (A pixels) of the last finalize
        self.gamma_order = gamma_order
        self.gamma_blocked = gamma_order == "ublocked"
        self._keep = []   # host buffers that must outlive an async copy

    # -- helpers ----------------------------------------------------------------------
    def _check(self, st: int):
        if st != 0:
            raise CpiError(st, self._lib.cpi_last_error(self._h).decode())

    def _stream(self, stream=None):
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    @staticmethod
    def _ptr(t) -> ctypes.c_void_p:
        if t is None:
            return ctypes.c_void_p(0)
        if isinstance(t, np.ndarray):
            return ctypes.c_void_p(t.ctypes.data)
        return ctypes.c_void_p(t.data_ptr())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.cpi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- C ABI -------------------------------------------------------------------------
    def load_frames(self, frames, n_frames: Optional[int] = None, stream=None):
        """cpi_load_frames.  frames: packed uint8 [N][H][W/8] as a numpy array / CPU tensor
        (host copy, pinned = async) or a CUDA tensor (used in place)."""
        torch = _torch()
        if isinstance(frames, np.ndarray):
            nbytes = frames.nbytes
            where = _lib.CPI_HOST
            self._keep = [frames]
        else:
            nbytes = frames.numel() * frames.element_size()
            where = _lib.CPI_DEVICE if frames.is_cuda else _lib.CPI_HOST
            if not frames.is_contiguous():
                raise ValueError("frames must be contiguous")
            self._keep = [frames]
        if n_frames is None:
            if nbytes % self.frame_bytes:
                raise CpiError(-4, f"{nbytes} bytes is not a whole number of {self.frame_bytes}-byte frames")
            n_frames = nbytes // self.frame_bytes
        self._check(self._lib.cpi_load_frames(self._h, self._ptr(frames), int(n_frames), where,
                                              self._stream(stream)))
        return n_frames

    def correlate(self, gamma=None, stream=None):
        """cpi_correlate: accumulate the loaded batch; write Gamma [P_a][P_b] fp32 if given."""
        if gamma is not None:
            self._check_gamma(gamma)
        self._check(self._lib.cpi_correlate(self._h, self._ptr(gamma), self._stream(stream)))
        return gamma

    def correlate_rows(self, row0: int, rows: int, gamma=None, stream=None):
        """cpi_correlate_rows: the loaded batch's pair sums for A pixels [row0, row0+rows)
        (the first call of a batch also expands it and adds S_a, S_b, N)."""
        if gamma is not None:
            self._check_gamma(gamma)
        self._check(self._lib.cpi_correlate_rows(self._h, int(row0), int(rows), self._ptr(gamma),
                                                 self._stream(stream)))
        return gamma

    def correlate_rows_to(self, row0: int, rows: int, gamma_rows, stream=None):
        """cpi_correlate_rows_to: as correlate_rows, Gamma rows written compactly to
        gamma_rows (CUDA float32 [rows][P_b])."""
        torch = _torch()
        if not (gamma_rows.is_cuda and gamma_rows.dtype == torch.float32 and gamma_rows.is_contiguous()
                and gamma_rows.numel() >= rows * self.p_b):
            raise ValueError("gamma_rows must be a contiguous CUDA float32 tensor with rows * P_b elements")
        self._check(self._lib.cpi_correlate_rows_to(self._h, int(row0), int(rows), self._ptr(gamma_rows),
                                                    self._stream(stream)))
        return gamma_rows

    def row_align(self) -> int:
        """cpi_row_align: A-pixel alignment of correlate_rows panels."""
        return int(self._lib.cpi_row_align(self._h))

    def counts_views(self):
        """cpi_counts_dev as torch tensors viewing the library's buffers (no copy):
        (s_ab [P_a][P_b] or None, s_a [P_a], s_b [P_b]), int32, valid until close()."""
        torch = _torch()
        pab, pa, pb = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        self._check(self._lib.cpi_counts_dev(self._h, ctypes.byref(pab), ctypes.byref(pa), ctypes.byref(pb)))

        def view(ptr, shape):
            if not ptr.value:
                return None
            n = int(np.prod(shape))

            class _Arr:   # __cuda_array_interface__ wrapper of a borrowed device pointer
                __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<i4", "data": (ptr.value, False),
                                            "version": 3, "strides": None}
            t = torch.as_tensor(_Arr(), device=f"cuda:{self.device}")
            assert t.numel() == n and t.data_ptr() == ptr.value
            return t
        rows_ab = self.p_a // self.world if self.fused_reduce else self.p_a   # fused: this rank's shard
        return view(pab, (rows_ab, self.p_b)), view(pa, (self.p_a,)), view(pb, (self.p_b,))

    def finalize(self, gamma=None, stream=None) -> int:
        """cpi_finalize: Gamma from the accumulated sums; returns N_TOT.  Multi-GPU: the cross-rank
        reduction runs here and gamma (optional) receives this rank's rows [rows][P_b]
        (self.shard_rows = (row0, rows), layout from shard_layout())."""
        if gamma is not None and not self.sharded:
            self._check_gamma(gamma)
        n, r0, rows = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
        self._check(self._lib.cpi_finalize(self._h, self._ptr(gamma), ctypes.byref(n), ctypes.byref(r0),
                                           ctypes.byref(rows), self._stream(stream)))
        self.shard_rows = (r0.value, rows.value)
        return n.value

    def shard_ipc_handle(self) -> bytes:
        """cpi_shard_ipc_handle (CPI_FUSED_REDUCE): this rank's shard handle for the other ranks."""
        buf = ctypes.create_string_buffer(_lib.CPI_SHARD_HANDLE_BYTES)
        self._check(self._lib.cpi_shard_ipc_handle(self._h, buf))
        return buf.raw

    def open_peer_shards(self, handles):
        """cpi_open_peer_shards: handles[r] = shard_ipc_handle() bytes of rank r."""
        blob = b"".join(bytes(h) for h in handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        self._check(self._lib.cpi_open_peer_shards(self._h, buf))

    def shard_layout(self):
        """cpi_shard_layout: (row_block, row_stride) of this rank's block-cyclic A rows."""
        b, st = ctypes.c_int32(0), ctypes.c_int32(0)
        self._check(self._lib.cpi_shard_layout(self._h, ctypes.byref(b), ctypes.byref(st)))
        return b.value, st.value

    def shard_pixel_rows(self):
        """Global A pixel of each local Gamma row owned by this rank (include/cpi.h cpi_finalize)."""
        block, stride = self.shard_layout()
        Wa, Ha = self.roi_a[2], self.roi_a[3]
        row0, rows = self.shard_rows
        if self.sharded:   # include/cpi.h cpi_finalize: rank r owns blocks r of every panel
            row0, rows = self.rank * block * Wa, (Ha // self.world) * Wa
        lr = np.arange(rows // Wa)
        m = row0 // Wa + (lr // block) * stride + lr % block
        return (m[:, None] * Wa + np.arange(Wa)[None, :]).reshape(-1)

    def finalize_counts(self, s_ab_rows, row0: int, s_a, s_b, n_tot: int, gamma_rows, stream=None):
        """cpi_finalize_counts: stateless Gamma of an externally reduced row shard."""
        rows = s_ab_rows.shape[0]
        self._check(self._lib.cpi_finalize_counts(self._h, self._ptr(s_ab_rows), int(row0), int(rows),
                                                  self._ptr(s_a), self._ptr(s_b), int(n_tot),
                                                  self._ptr(gamma_rows), self._stream(stream)))
        return gamma_rows

    def get_counts(self, s_ab=None, s_a=None, s_b=None, stream=None) -> int:
        """cpi_get_counts into caller CUDA int32 tensors; returns N_TOT."""
        n = ctypes.c_int64(0)
        self._check(self._lib.cpi_get_counts(self._h, self._ptr(s_ab), self._ptr(s_a), self._ptr(s_b),
                                             ctypes.byref(n), self._stream(stream)))
        return n.value

    def reset(self, stream=None):
        self._check(self._lib.cpi_reset(self._h, self._stream(stream)))

    def refocus(self, alphas: Optional[Sequence[float]], gamma, planes, row0: int = 0, rows: Optional[int] = None,
                boundary: int = _lib.CPI_SKIP_RENORMALIZE, row_block: int = 0, row_stride: int = 0,
                affine=None, stream=None):
        """cpi_refocus: planes [n_planes][H_a][W_a] fp32 from a Gamma row shard of `rows` pixel
        rows (leading dimension P_b) starting at A row row0 / W_a; row_block > 0 makes the
        shard block-cyclic (local A row l -> row0/W_a + (l // row_block) * row_stride + l % row_block).
        affine: optional [n_planes][12] general maps (include/cpi.h) instead of alphas."""
        if affine is not None:
            mp = np.ascontiguousarray(affine, dtype=np.float64).reshape(-1, 12)
            n = mp.shape[0]
            al_ptr = ctypes.POINTER(ctypes.c_double)()
            aff_ptr = mp.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            keep = mp
        else:
            al = np.ascontiguousarray(alphas, dtype=np.float64).ravel()
            n = al.size
            al_ptr = al.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            aff_ptr = ctypes.POINTER(ctypes.c_double)()
            keep = al
        if rows is None:
            rows = self.p_a - row0
        spec = _lib.RefocusSpec(al_ptr, n, int(boundary), self._ptr(gamma), int(row0), int(rows), int(row_block),
                                int(row_stride), aff_ptr)
        self._check(self._lib.cpi_refocus(self._h, ctypes.byref(spec), self._ptr(planes), self._stream(stream)))
        del keep
        return planes

    def launch_count(self) -> int:
        return int(self._lib.cpi_launch_count(self._h))

    def set_timing(self, enable: bool):
        self._check(self._lib.cpi_set_timing(self._h, int(bool(enable))))

    def kernel_time_ms(self, cls: int):
        ms = ctypes.c_double(0)
        n = ctypes.c_int64(0)
        self._check(self._lib.cpi_kernel_time_ms(self._h, int(cls), ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    # -- conveniences -------------------------------------------------------------------
    def _check_gamma(self, g):
        torch = _torch()
        if not (g.is_cuda and g.dtype == torch.float32 and g.is_contiguous() and g.numel() >= self.p_a * self.p_b):
            raise ValueError("gamma must be a contiguous CUDA float32 tensor with P_a*P_b elements")

    def b_index(self):
        """Index of every B pixel q = v * W_b + u in S_b and in the columns of S_ab / Gamma
        (identity for the row-major order; include/cpi.h CPI_GAMMA_UBLOCKED, CPI_GAMMA_VMAJOR)."""
        Wb, Hb = self.roi_b[2], self.roi_b[3]
        q = np.arange(Wb * Hb)
        if self.gamma_order == "rowmajor":
            return q
        v, u = q // Wb, q % Wb
        if self.gamma_order == "vmajor":   # include/cpi.h: blocks of 128 B rows (kernels.h vmajor_slot)
            vb = min(Hb, 128)
            return (v // vb) * (Wb * vb) + u * vb + v % vb
        return (u // 8) * (8 * Hb) + 8 * v + (u % 8)

    def new_gamma(self):
        torch = _torch()
        return torch.empty((self.p_a, self.p_b), dtype=torch.float32, device=f"cuda:{self.device}")

    def new_planes(self, n_planes: int):
        torch = _torch()
        return torch.empty((n_planes, self.roi_a[3], self.roi_a[2]), dtype=torch.float32,
                           device=f"cuda:{self.device}")


def abi_version() -> int:
    return int(_lib.load().cpi_abi_version())


def nccl_unique_id() -> bytes:
    """cpi_nccl_unique_id: a new NCCL unique id for a multi-GPU group (share it with every rank)."""
    buf = ctypes.create_string_buffer(_lib.CPI_NCCL_ID_BYTES)
    st = _lib.load().cpi_nccl_unique_id(buf)
    if st != 0:
        raise CpiError(st, "cpi_nccl_unique_id failed (libnccl.so.2 unavailable?)")
    return buf.raw
