"""Shared pytest configuration.

* ``gpu`` marker: tests that need a B200 (sm_100a) and the built CUDA
  library; the driver runs ``-m gpu`` on a GPU box and ``-m "not gpu"`` here.
* The repo root is put on ``sys.path`` so ``oracle`` (test infrastructure)
  and the product package import without installation.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libpolar_b200.so")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


def bf16_bits_to_f32(a):
    return (np.asarray(a, np.uint16).astype(np.uint32) << 16).view(np.float32)
