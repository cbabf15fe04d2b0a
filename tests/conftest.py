"""Shared fixtures.  CPU tests (-m "not gpu") exercise the oracle, golden
vectors, host logic and the C ABI's exported symbols; GPU tests (-m gpu) are
the parity tests proper and call the product through its C ABI."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    oracle.load()
    return oracle


@pytest.fixture(scope="session")
def pam():
    import paper_2509_08383_b200 as pam

    return pam


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    torch.cuda.init()
    return torch


def normwise(z, zref):
    """max|z - zref| / max|zref|."""
    z = np.asarray(z, dtype=np.float64)
    zref = np.asarray(zref, dtype=np.float64)
    return float(np.max(np.abs(z - zref)) / max(np.max(np.abs(zref)), 1e-300))
