import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (minutes)")


def pytest_runtest_setup(item):
    """GPU tests fail loudly (never skip) when they run on a box without a CUDA device, so a
    CPU-only run can never masquerade as GPU parity.  The CPU tier deselects them with
    -m "not gpu"."""
    if item.get_closest_marker("gpu") is not None:
        import torch
        if not torch.cuda.is_available():
            pytest.fail("GPU test selected but no CUDA device is visible (run the CPU tier with -m 'not gpu')",
                        pytrace=False)


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle
