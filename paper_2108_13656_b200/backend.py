"""Kernel-backend registry and worker-count resolution.

Drop-in for /root/reference/pkg/src/warmgray/backend.py. The reference keeps
two interchangeable kernel modules ("compiled" Cython, "python" NumPy) behind
``get_kernels`` (backend.py:25-52) and fans row chunks out over a thread pool
(``run_rows``, backend.py:65-81). Here there is exactly ONE backend, the
sm_100a CUDA library (no multi-backend dispatch, no CPU fallback):

* ``get_kernels()`` returns :mod:`paper_2108_13656_b200._kernels_cuda`, whose
  ``decolor_rows(rgb, out, beta_r, beta_k, row0, row1)`` has the reference
  plugin signature (_kernels.pyx:47-56).
* The name ``"compiled"`` is accepted as an alias of ``"cuda"`` so callers
  written against the reference keep working; any other name raises
  ``ValueError`` like the reference (backend.py:50-52).
* ``threads`` / ``WARMGRAY_THREADS`` are still resolved and validated
  (backend.py:55-62) but cannot change results: one launch covers the image.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from typing import Callable

from . import _lib

THREADS_ENV = "WARMGRAY_THREADS"
DEVICE_ENV = "WARMGRAY_DEVICE"
BACKEND_NAME = "cuda"
_ALIASES = {"cuda": BACKEND_NAME, "compiled": BACKEND_NAME}

_device: int | None = None


def compiled_available() -> bool:
    """True when the sm_100a library is built and loadable."""
    return _lib.available()


def available_backends() -> tuple[str, ...]:
    """Backend names usable in this process (the CUDA backend, or nothing)."""
    return (BACKEND_NAME,) if _lib.available() else ()


def active_backend() -> str:
    """Name of the backend used when none is requested explicitly."""
    _lib.load()  # raises ExtensionMissing: there is no CPU fallback
    return BACKEND_NAME


def get_kernels(name: str | None = None):
    """Return the kernel module for ``name`` (default and only: the CUDA backend)."""
    if name is not None and name not in _ALIASES:
        known = ", ".join(sorted(_ALIASES))
        raise ValueError(f"unknown or unavailable backend {name!r} (have: {known})")
    _lib.load()
    from . import _kernels_cuda

    return _kernels_cuda


def resolve_threads(threads: int | None = None) -> int:
    """Worker count: explicit value, else $WARMGRAY_THREADS, else 1 (validated >= 1)."""
    if threads is None:
        raw = os.environ.get(THREADS_ENV, "").strip()
        threads = int(raw) if raw else 1
    if threads < 1:
        raise ValueError(f"thread count must be >= 1, got {threads}")
    return threads


def run_rows(height: int, threads: int, fn: Callable[[int, int], None]) -> None:
    """Call ``fn(row0, row1)`` over disjoint contiguous row spans covering [0, height).

    Kept for API compatibility with the reference's host utility; the CUDA
    path itself issues one call per image. Worker exceptions propagate.
    """
    if height <= 0:
        return
    n = max(1, min(threads, height))
    step = -(-height // n)
    spans = [(r, min(r + step, height)) for r in range(0, height, step)]
    if len(spans) == 1:
        fn(*spans[0])
        return
    with ThreadPoolExecutor(max_workers=len(spans)) as pool:
        for fut in [pool.submit(fn, r0, r1) for r0, r1 in spans]:
            fut.result()


def set_device(index: int) -> None:
    """Select the GPU used by the host-array (drop-in) entry points."""
    global _device
    if index < 0:
        raise ValueError(f"device index must be >= 0, got {index}")
    _device = int(index)


def get_device() -> int:
    """GPU used by host-array entry points: set_device(), else $WARMGRAY_DEVICE,
    else torch's current device if torch.cuda is initialised, else 0."""
    if _device is not None:
        return _device
    raw = os.environ.get(DEVICE_ENV, "").strip()
    if raw:
        return int(raw)
    import sys

    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        return int(torch.cuda.current_device())
    return 0
