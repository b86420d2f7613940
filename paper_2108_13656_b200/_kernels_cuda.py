"""The CUDA kernel module returned by ``backend.get_kernels()``.

Same module surface as the reference's plugin modules (``NAME`` plus
``decolor_rows``; /root/reference/pkg/src/warmgray/_kernels.pyx:12,47-56).
``decolor_rows`` takes host fp64 arrays exactly like the Cython kernel and
runs the fp64 device kernel through the C ABI (wg_host_decolor_rows_f64),
which is bit-identical to the reference's compiled backend.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .backend import get_device

NAME = "cuda"


def _require(arr, ndim: int, what: str) -> None:
    # mirrors the Cython memoryview checks: dtype, ndim, C-contiguity
    if not isinstance(arr, np.ndarray):
        raise TypeError(f"{what}: expected a numpy.ndarray, got {type(arr).__name__}")
    if arr.dtype != np.float64:
        raise ValueError(f"{what}: Buffer dtype mismatch, expected 'double' but got {arr.dtype}")
    if arr.ndim != ndim:
        raise ValueError(f"{what}: Buffer has wrong number of dimensions (expected {ndim}, got {arr.ndim})")
    if not arr.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{what}: ndarray is not C-contiguous")


def decolor_rows(rgb, out, beta_r, beta_k, row0, row1) -> None:
    """Warm/cool weighted blending of the RGB channels into one gray value.

    Fills ``out[row0:row1]`` in place from ``rgb[row0:row1]``.
    """
    _require(rgb, 3, "rgb")
    _require(out, 2, "out")
    if not out.flags["WRITEABLE"]:
        raise ValueError("out: buffer source array is read-only")
    h, w = rgb.shape[0], rgb.shape[1]
    if rgb.shape[2] != 3 or out.shape[0] < h or out.shape[1] != w:
        raise ValueError(f"shape mismatch: rgb {rgb.shape} vs out {out.shape}")
    _lib.call("wg_host_decolor_rows_f64", rgb.ctypes.data, out.ctypes.data, h, w,
              float(beta_r), float(beta_k), int(row0), int(row1), get_device())
