import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def native():
    """The product library, built in-tree if stale (nvcc works without a GPU)."""
    from paper_1710_08314_b200 import _build

    _build.build()
    from paper_1710_08314_b200 import _lib

    return _lib.lib()


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle

    oracle.build_oracle()
    return oracle


@pytest.fixture(scope="session")
def ref_lib():
    """The compiled, unmodified reference (oracle/_ref), or skip."""
    from oracle import oracle

    try:
        oracle.Reference.lib()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"reference not available: {e}")
    return oracle


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a host without CUDA")
    return torch


def rough_llrs(rng, n, nframes, precision):
    """Adversarial LLRs of test_sc.cpp:18-37 / test_list.cpp:26-45: exact
    zeros, +-127 and tiny magnitudes (ties everywhere)."""
    pick = rng.integers(0, 8, (nframes, n))
    mag = np.where(pick == 0, 0, np.where(pick == 1, 127, rng.integers(0, 8, (nframes, n))))
    s = np.where(rng.integers(0, 2, (nframes, n)) == 1, -1, 1)
    v = s * mag
    if precision == "i8":
        return v.astype(np.int8)
    return (v * 0.5).astype(np.float32)
