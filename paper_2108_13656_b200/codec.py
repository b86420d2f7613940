"""uint8 <-> float conversion semantics of the reference codec (codec.py:22-29).

``quantize_u8``: floor(clip(v, 0, 1) * 255 + 0.5) (round half up);
``dequantize_u8``: k / 255.0. Both run as device kernels through the C ABI;
inside the fused u8 kernels the same rounding happens in registers. File
I/O (PNG / PNM, codec.py:37-140) is host format handling outside the
data-parallel path.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .backend import get_device


def quantize_u8(data) -> np.ndarray:
    """[0, 1] float samples to uint8 with clamping and round-half-up."""
    src = np.ascontiguousarray(data, dtype=np.float64)
    out = np.empty(src.shape, dtype=np.uint8)
    if out.size:
        _lib.call("wg_host_quantize_u8_f64", src.ctypes.data, out.ctypes.data, out.size, get_device())
    return out


def dequantize_u8(data) -> np.ndarray:
    """uint8 samples to float64 k / 255."""
    src = np.ascontiguousarray(data, dtype=np.uint8)
    out = np.empty(src.shape, dtype=np.float64)
    if out.size:
        _lib.call("wg_host_dequantize_u8_f64", src.ctypes.data, out.ctypes.data, out.size, get_device())
    return out
