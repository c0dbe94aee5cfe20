"""B200-native (sm_100a) hot path of Correlation Plenoptic Imaging (arXiv 2407.20692).

binary SwissSPAD2 frames -> on-device expansion -> S_ab on tcgen05 kind::i8 tensor cores
with fused exact normalisation -> Gamma (Eq. 1) -> refocused plane stack.

The compute lives in libcpi.so (C ABI: include/cpi.h); this package is its thin binding
(`cpi`), the dataset-file readers (`dataset`: .bin files) and the frame-sharded
multi-GPU orchestration over torch.distributed (`parallel`).
"""
from ._lib import CpiError, CPI_CLAMP, CPI_SKIP_RENORMALIZE  # noqa: F401
from .cpi import Context, abi_version, nccl_unique_id  # noqa: F401

__all__ = ["Context", "CpiError", "abi_version", "nccl_unique_id", "CPI_CLAMP", "CPI_SKIP_RENORMALIZE"]
