"""Shared test configuration.

Markers: ``gpu`` tests need a B200 (run with ``-m gpu``); everything else runs
on the CPU container (``-m "not gpu"``). The hypothesis profile mirrors the
reference's (pkg/tests/conftest.py:7-14).
"""

import os
import sys

import numpy as np
import pytest
from hypothesis import HealthCheck, settings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

settings.register_profile("warmgray", max_examples=60, deadline=None, derandomize=True,
                          suppress_health_check=[HealthCheck.too_slow])
settings.load_profile("warmgray")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def rand_rgb(rng, height, width):
    from paper_2108_13656_b200 import PlanarImage

    return PlanarImage(rng.random((height, width, 3)))


def rand_u8_rgb(rng, height, width):
    from paper_2108_13656_b200 import PlanarImage

    return PlanarImage(rng.integers(0, 256, (height, width, 3)).astype(np.float64) / 255.0)


def u8_mismatch(got: np.ndarray, want: np.ndarray):
    """(max |diff|, fraction of differing pixels) for uint8 arrays."""
    d = np.abs(got.astype(np.int16) - want.astype(np.int16))
    return int(d.max()) if d.size else 0, float((d != 0).mean()) if d.size else 0.0


# north-star parity bar: u8 identical except +-1 on <= 0.01% of pixels
U8_MAX_FRAC = 1e-4
F32_TOL = 1e-6   # fp32 gray vs fp64 oracle (test_core.py:199 binds tighter than the 1e-5 north star)
