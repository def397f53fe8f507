"""Test configuration.

Markers: ``gpu`` — needs a CUDA device (run with -m gpu on a B200);
everything else runs on CPU (oracle vs golden fixtures, host C++ page table,
C-ABI exports, scene I/O, multi-process gloo logic).
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200 / sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    d = os.path.join(ROOT, "tests", "golden")

    class G:
        def __getitem__(self, name):
            return np.load(os.path.join(d, f"{name}.npz"))

    return G()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_19415_b200 import _lib

    _lib.load()
    return torch
