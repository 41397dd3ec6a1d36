"""Shared test plumbing.

Markers: ``gpu`` = needs a B200 (run with ``-m gpu`` on the GPU box);
everything else runs on CPU.  The oracle (``oracle/``) is importable here as
the checker only.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def random_walks(count: int, n: int, seed: int) -> np.ndarray:
    """z-normalised random walks, independent of the package generator
    (same recipe as the reference tests' conftest.random_walks)."""
    rng = np.random.default_rng(seed)
    walks = np.cumsum(rng.standard_normal((count, n)), axis=1)
    mu = walks.mean(axis=1, keepdims=True)
    sd = walks.std(axis=1, keepdims=True)
    return ((walks - mu) / sd).astype(np.float32)


@pytest.fixture(scope="session")
def oracle():
    import oracle as o  # noqa: WPS433  (oracle/oracle.py)

    o.lib()
    return o


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
