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


def _rows_checks(rgb, out, out_ndim):
    _require(rgb, 3, "rgb")
    _require(out, out_ndim, "out")
    if not out.flags["WRITEABLE"]:
        raise ValueError("out: buffer source array is read-only")
    h, w = rgb.shape[0], rgb.shape[1]
    if rgb.shape[2] != 3 or out.shape[0] < h or out.shape[1] != w or (out_ndim == 3 and out.shape[2] != 3):
        raise ValueError(f"shape mismatch: rgb {rgb.shape} vs out {out.shape}")
    return h, w


def _luma_rows(method: int, rgb, out, row0, row1) -> None:
    h, w = _rows_checks(rgb, out, 2)
    _lib.call("wg_host_luma_rows_f64", rgb.ctypes.data, out.ctypes.data, h, w, method, int(row0), int(row1),
              get_device())


def bt601_rows(rgb, out, row0, row1) -> None:
    """BT.601 weighted sum, clamped (_kernels.pyx:59-68)."""
    _luma_rows(0, rgb, out, row0, row1)


def hsv_value_rows(rgb, out, row0, row1) -> None:
    """V of HSV: max(r, g, b) (_kernels.pyx:71-84)."""
    _luma_rows(1, rgb, out, row0, row1)


def lab_lightness_rows(rgb, out, row0, row1) -> None:
    """CIELAB lightness of the sRGB input, rescaled to [0, 1] (_kernels.pyx:99-112)."""
    _luma_rows(2, rgb, out, row0, row1)


def lab_rows(rgb, out, row0, row1) -> None:
    """Full CIELAB coordinates into out[row0:row1] of shape (..., 3) (_kernels.pyx:115-132)."""
    h, w = _rows_checks(rgb, out, 3)
    _lib.call("wg_host_lab_rows_f64", rgb.ctypes.data, out.ctypes.data, h, w, int(row0), int(row1), get_device())


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
