"""Host-side checks of the C-ABI library (no compute calls): it builds for sm_100a, loads,
exports every symbol include/cpi.h declares, and rejects bad configurations with the
documented status codes before touching a device."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2407_20692_b200 import _lib, build
    build.build()
    return _lib.load()


def _declared():
    hdr = (ROOT / "include" / "cpi.h").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(cpi_[a-z_]+)\s*\(", hdr)))


def test_header_symbols_exported(lib):
    from paper_2407_20692_b200 import _lib
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), f"libcpi.so does not export {name}"
    assert sorted(_lib.EXPORTS) == declared


def test_abi_version_and_status_names(lib):
    assert lib.cpi_abi_version() == 201
    assert lib.cpi_status_string(0) == b"CPI_OK"
    assert lib.cpi_status_string(-7) == b"CPI_ERR_DEGENERATE_ALPHA"
    assert lib.cpi_status_string(-12) == b"CPI_ERR_UNSUPPORTED"


def test_sass_is_tcgen05(lib):
    """The shipped library holds sm_100a tensor-core (UTC*MMA), TMA (UTMALDG) and TMEM
    load (LDTM) instructions — the tcgen05 path, not a legacy mma.sync one."""
    import subprocess
    from paper_2407_20692_b200._lib import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "UTCIMMA" in out and "UTMALDG" in out and "LDTM" in out
    assert "arch = sm_100a" in out
    assert " HMMA" not in out and " IMMA" not in out


def _cfg(lib_mod, roi_a=(0, 0, 256, 256), roi_b=(256, 0, 256, 256), w=512, h=256, max_frames=1000,
         flags=0, order=0):
    return lib_mod.Config(lib_mod.Layout(w, h, order), lib_mod.Roi(*roi_a), lib_mod.Roi(*roi_b),
                          max_frames, 0, flags)


@pytest.mark.parametrize("kw,status", [
    (dict(w=500), -2),                              # CPI_ERR_LAYOUT
    (dict(h=0), -2),
    (dict(roi_a=(300, 0, 256, 256)), -3),           # CPI_ERR_ROI_OUT_OF_BOUNDS
    (dict(roi_b=(0, 250, 8, 8)), -3),
    (dict(roi_a=(0, 0, 0, 4)), -3),
    (dict(max_frames=0), -1),                       # CPI_ERR_INVALID_ARG
    (dict(flags=0x80), -1),
    (dict(flags=0x1 | 0x4), -1),                    # POPC and FP4 are exclusive
    (dict(flags=0x40 | 0x4), -1),                   # f1 (TC_BITS) and FP4 are exclusive
    (dict(flags=0x4, max_frames=1 << 24), -1),      # FP4: exact fp32 sums need N < 2^24
    (dict(flags=0x8, roi_b=(256, 0, 12, 8)), -12),  # u-blocked Gamma needs W_b % 8 == 0
    (dict(order=5), -1),
])
def test_create_rejects_bad_config(lib, kw, status):
    from paper_2407_20692_b200 import _lib
    h = ctypes.c_void_p()
    cfg = _cfg(_lib, **kw)
    st = lib.cpi_create(ctypes.byref(cfg), ctypes.byref(h))
    assert st == status, (st, lib.cpi_last_error(None))
    assert h.value is None
    assert lib.cpi_last_error(None)


def test_null_handles(lib):
    assert lib.cpi_create(None, None) == -1
    lib.cpi_destroy(None)
    assert lib.cpi_launch_count(None) == 0
    assert lib.cpi_load_frames(None, None, 0, 0, None) == -1
    assert lib.cpi_correlate(None, None, None) == -1
    assert lib.cpi_correlate_rows(None, 0, 256, None, None) == -1
    assert lib.cpi_row_align(None) == 0
    assert lib.cpi_counts_dev(None, None, None, None) == -1
    assert lib.cpi_finalize(None, None, None, None, None, None) == -1
    assert lib.cpi_shard_layout(None, None, None) == -1
    assert lib.cpi_nccl_unique_id(None) == -1
    assert lib.cpi_finalize_counts(None, None, 0, 0, None, None, 1, None, None) == -1
    assert lib.cpi_get_counts(None, None, None, None, None, None) == -1
    assert lib.cpi_reset(None, None) == -1
    assert lib.cpi_refocus(None, None, None, None) == -1
    assert lib.cpi_set_timing(None, 1) == -1
