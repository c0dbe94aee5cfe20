"""Host-side dataset readers (include/cpi.h cpi_bin_frames / cpi_read_bin, dataset.py):
SPEC.md:57-64 parse_bin_file and S:91-100 scan_dataset examples, bytes round-trip exactly.
CPU only (the readers need no device)."""
import os

import numpy as np
import pytest

from paper_2407_20692_b200 import dataset
from paper_2407_20692_b200._lib import CpiError
from synth import bernoulli_frames


def _write(path, arr):
    with open(path, "wb") as f:
        f.write(np.ascontiguousarray(arr).tobytes())


def test_bin_frames_paper_file_size(tmp_path):
    # an 8,388,608-byte file of the 256x512 layout is 512 frames of 16,384 bytes
    p = tmp_path / "f.bin"
    with open(p, "wb") as f:
        f.truncate(8_388_608)
    assert dataset.bin_frames(str(p)) == 512


def test_bin_frames_empty_and_mismatch(tmp_path):
    e = tmp_path / "empty.bin"
    e.write_bytes(b"")
    assert dataset.bin_frames(str(e)) == 0
    m = tmp_path / "odd.bin"
    m.write_bytes(b"\0" * 16_385)                          # one byte over a frame
    with pytest.raises(CpiError) as ei:
        dataset.bin_frames(str(m))
    assert ei.value.name == "CPI_ERR_SIZE_MISMATCH"
    with pytest.raises(CpiError) as ei:
        dataset.bin_frames(str(tmp_path / "missing.bin"))
    assert ei.value.name == "CPI_ERR_INVALID_ARG"
    with pytest.raises(CpiError) as ei:
        dataset.bin_frames(str(e), width=12)
    assert ei.value.name == "CPI_ERR_LAYOUT"


def test_read_bin_round_trip(tmp_path):
    fr = bernoulli_frames(37, 0.3, seed=5)                 # [37][256][64] packed frames
    p = tmp_path / "a.bin"
    _write(p, fr)
    out = dataset.read_bin(str(p))
    assert out.shape == fr.shape and np.array_equal(out, fr)
    part = dataset.read_bin(str(p), 11, 7)
    assert np.array_equal(part, fr[11:18])
    for f0, n in [(-1, 1), (30, 8), (38, 0)]:
        with pytest.raises(CpiError):
            dataset.read_bin(str(p), f0, n)
    assert dataset.read_bin(str(p), 37, 0).shape[0] == 0


def test_scan_dataset_order_and_errors(tmp_path):
    fr = bernoulli_frames(8, 0.5, seed=9)
    names = ["b.bin", "a.bin", "c.bin", "notes.txt"]
    for i, n in enumerate(names):
        _write(tmp_path / n, fr[2 * i:2 * i + 2])
    m = dataset.scan_dataset(str(tmp_path))
    assert [os.path.basename(p) for p in m.file_paths] == ["a.bin", "b.bin", "c.bin"]   # lexicographic
    assert m.frames_per_file == 2 and m.n_tot == 6                                        # N_TOT = N x N_file
    _write(tmp_path / "d.bin", fr[:3])
    with pytest.raises(CpiError) as ei:
        dataset.scan_dataset(str(tmp_path))
    assert ei.value.name == "CPI_ERR_SIZE_MISMATCH" and "d.bin" in str(ei.value)
    empty = tmp_path / "sub"
    empty.mkdir()
    with pytest.raises(CpiError, match="EmptyDataset"):
        dataset.scan_dataset(str(empty))


def test_batches_cover_every_frame_once():
    m = dataset.Manifest(["f0", "f1", "f2"], 5)
    got = []
    for pieces, n in dataset._batches(m, 4):
        assert n == sum(p[2] for p in pieces) and n <= 4
        off = 0
        for path, f0, cnt, o in pieces:
            assert o == off
            off += cnt
            got += [(path, f0 + k) for k in range(cnt)]
    assert got == [(f"f{i}", k) for i in range(3) for k in range(5)]


def test_correlate_files_argument_checks(tmp_path):
    class _Ctx:   # host-side checks run before any device work
        width, height, frame_bytes, max_frames, keep_counts, device = 512, 256, 16384, 4, False, 0
    m = dataset.Manifest(["f0", "f1"], 5)
    with pytest.raises(ValueError, match="max_frames"):
        dataset.correlate_files(_Ctx(), m, batch_frames=8)
    with pytest.raises(ValueError, match="keep_counts"):
        dataset.correlate_files(_Ctx(), m)
    c = _Ctx()
    c.max_frames = 10
    with pytest.raises(ValueError, match="gamma"):
        dataset.correlate_files(c, m)
