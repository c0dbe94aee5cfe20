"""Dataset files of the paper's input ("Input Dataset": sets of headerless .bin
files, 8 MiB = 512 SwissSPAD2 frames each; SPEC.md:57-64 parse_bin_file, S:91-100 scan_dataset).

Argument marshalling over libcpi's host-side readers (`cpi_bin_frames`, `cpi_read_bin`,
include/cpi.h) plus the directory walk and the batch streaming loop: files are read into two
pinned host buffers while the GPU correlates the previous batch (cpi_load_frames copies
asynchronously from pinned memory).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import CpiError

FRAME_W, FRAME_H = 512, 256


def _layout(width: int, height: int, bit_order: int):
    return _lib.Layout(width, height, bit_order)


def _err(st: int) -> CpiError:
    msg = _lib.load().cpi_last_error(None)
    return CpiError(st, msg.decode() if msg else "")


def bin_frames(path: str, *, width: int = FRAME_W, height: int = FRAME_H, bit_order: int = 0) -> int:
    """cpi_bin_frames: number of whole frames in a .bin file (SizeMismatch otherwise)."""
    n = ctypes.c_int64()
    lay = _layout(width, height, bit_order)
    st = _lib.load().cpi_bin_frames(os.fsencode(path), ctypes.byref(lay), ctypes.byref(n))
    if st != 0:
        raise _err(st)
    return int(n.value)


def read_bin(path: str, frame0: int = 0, n_frames: Optional[int] = None, out=None, *, width: int = FRAME_W,
             height: int = FRAME_H, bit_order: int = 0):
    """cpi_read_bin: frames [frame0, frame0 + n_frames) of a file, bit for bit, into `out` (a
    contiguous uint8 numpy array or CPU tensor of n_frames * frame bytes; allocated if None)."""
    if n_frames is None:
        n_frames = bin_frames(path, width=width, height=height, bit_order=bit_order) - frame0
    fb = width // 8 * height
    if out is None:
        out = np.empty((n_frames, height, width // 8), dtype=np.uint8)
    if isinstance(out, np.ndarray):
        if not out.flags["C_CONTIGUOUS"] or out.nbytes < n_frames * fb:
            raise ValueError("out must be contiguous and hold n_frames frames")
        ptr = out.ctypes.data
    else:
        if not out.is_contiguous() or out.is_cuda or out.numel() * out.element_size() < n_frames * fb:
            raise ValueError("out must be a contiguous host tensor holding n_frames frames")
        ptr = out.data_ptr()
    lay = _layout(width, height, bit_order)
    st = _lib.load().cpi_read_bin(os.fsencode(path), ctypes.byref(lay), int(frame0), int(n_frames),
                                  ctypes.c_void_p(ptr))
    if st != 0:
        raise _err(st)
    return out


@dataclass
class Manifest:
    """SPEC DatasetManifest: N_TOT = N_files x frames_per_file."""
    file_paths: List[str]
    frames_per_file: int
    width: int = FRAME_W
    height: int = FRAME_H
    bit_order: int = 0

    @property
    def n_files(self) -> int:
        return len(self.file_paths)

    @property
    def n_tot(self) -> int:
        return self.n_files * self.frames_per_file


def scan_dataset(directory: str, *, width: int = FRAME_W, height: int = FRAME_H, bit_order: int = 0,
                 suffix: str = ".bin") -> Manifest:
    """SPEC scan_dataset: the directory's `suffix` files in lexicographic order;
    every file must hold the same whole number of frames (SizeMismatch names the file);
    EmptyDataset (CpiError INVALID_ARG) when there is none."""
    names = sorted(n for n in os.listdir(directory) if n.endswith(suffix))
    if not names:
        raise CpiError(-1, f"EmptyDataset: no {suffix} files in {directory}")
    paths = [os.path.join(directory, n) for n in names]
    per = None
    for p in paths:
        n = bin_frames(p, width=width, height=height, bit_order=bit_order)
        if per is None:
            per = n
        elif n != per:
            raise CpiError(-4, f"{p}: {n} frames, the dataset's files have {per}")
    return Manifest(paths, per, width, height, bit_order)


def _batches(manifest: Manifest, batch_frames: int):
    """(file, frame0, n, offset in batch) pieces of consecutive batches of batch_frames frames."""
    pieces: list = []
    filled = 0
    for p in manifest.file_paths:
        f0 = 0
        while f0 < manifest.frames_per_file:
            n = min(manifest.frames_per_file - f0, batch_frames - filled)
            pieces.append((p, f0, n, filled))
            filled += n
            f0 += n
            if filled == batch_frames:
                yield pieces, filled
                pieces, filled = [], 0
    if filled:
        yield pieces, filled


def correlate_files(ctx, manifest: Manifest, batch_frames: Optional[int] = None, gamma=None, stream=None,
                    threads: Optional[int] = None) -> int:
    """Stream a dataset through a context: batches of up to ctx.max_frames frames are read into
    two pinned host buffers (the next batch is read while the GPU correlates the current one),
    loaded (cpi_load_frames, asynchronous from pinned memory) and accumulated (cpi_correlate).
    The context needs CPI_KEEP_COUNTS for more than one batch; `gamma`, if given, receives Gamma
    of the totals from the last batch's fused epilogue.  A batch's file pieces are read by
    `threads` host threads at once (cpi_read_bin releases the GIL).  Returns the number of frames."""
    from concurrent.futures import ThreadPoolExecutor
    import torch
    if (manifest.width, manifest.height) != (ctx.width, ctx.height):
        raise ValueError("manifest layout differs from the context's")
    batch_frames = int(batch_frames or ctx.max_frames)
    if batch_frames > ctx.max_frames:
        raise ValueError(f"batch_frames {batch_frames} exceeds the context's max_frames {ctx.max_frames}")
    batches = list(_batches(manifest, batch_frames))
    if len(batches) > 1 and not ctx.keep_counts:
        raise ValueError("more than one batch needs a context with keep_counts=True (CPI_KEEP_COUNTS)")
    if not ctx.keep_counts and gamma is None:
        raise ValueError("a context without kept counts needs a gamma output")
    fb = ctx.frame_bytes
    bufs = [torch.empty(batch_frames * fb, dtype=torch.uint8).pin_memory() for _ in range(2)]
    done: list = [None, None]
    st = stream if stream is not None else torch.cuda.current_stream(ctx.device)
    total = 0
    with ThreadPoolExecutor(max(1, threads or min(8, os.cpu_count() or 1))) as pool:
        for b, (pieces, n) in enumerate(batches):
            k = b & 1
            if done[k] is not None:
                done[k].synchronize()   # the GPU finished with this buffer's previous batch
            buf = bufs[k]
            list(pool.map(lambda pc: read_bin(pc[0], pc[1], pc[2], buf[pc[3] * fb:(pc[3] + pc[2]) * fb],
                                              width=manifest.width, height=manifest.height,
                                              bit_order=manifest.bit_order), pieces))
            ctx.load_frames(buf[:n * fb], n, stream=st)
            ctx.correlate(gamma if b == len(batches) - 1 else None, stream=st)
            ev = torch.cuda.Event()
            ev.record(st)
            done[k] = ev
            total += n
    return total
