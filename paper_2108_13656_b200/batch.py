"""Flat-batch API: the throughput path.

Two flavours over the same C ABI (include/warmgray_b200.h):

* ``decolor`` / ``decolor_tone`` / ``hdr_tonemap`` / ``sigmoid`` take CUDA
  ``torch.Tensor`` batches that are already resident in HBM (N, H, W, 3)
  (or any (..., 3) shape) and launch on the caller's current stream. One
  launch covers the whole batch: images are independent and the kernels
  are per-pixel maps (HDR adds a per-image statistic), so there is no
  per-image launch overhead.
* ``decolor_host`` / ``decolor_tone_host`` / ``hdr_tonemap_host`` take host
  NumPy arrays and run the pipelined host->device->host path
  (wg_host_*), the batch analogue of the reference's ``decolor_rows``
  plugin call on host memory.

uint8 inputs produce uint8 outputs bit-for-bit equal to
``quantize_u8(decolor_image(dequantize_u8(x)))`` except for at most +-1 on
rounding ties; fp32 inputs produce fp32 gray within 1e-6 of the fp64
reference; fp64 inputs reproduce the reference's compiled backend exactly.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .backend import get_device
from .core import DEFAULT_PARAMS, DecolorParams
from .tonemap import SigmoidCurve

_DECOLOR_FN = {"uint8": "wg_decolor_u8", "float32": "wg_decolor_f32", "float64": "wg_decolor_f64"}


def _torch():
    import torch

    return torch


def _check_rgb_tensor(rgb, dtypes):
    torch = _torch()
    if not isinstance(rgb, torch.Tensor):
        raise TypeError(f"expected a torch.Tensor, got {type(rgb).__name__}")
    if not rgb.is_cuda:
        raise ValueError("expected a CUDA tensor (use the *_host functions for host arrays)")
    if rgb.dim() < 1 or rgb.shape[-1] != 3:
        raise ValueError(f"rgb needs a trailing channel axis of 3, got shape {tuple(rgb.shape)}")
    if not rgb.is_contiguous():
        raise ValueError("rgb must be contiguous (interleaved HWC)")
    name = str(rgb.dtype).replace("torch.", "")
    if name not in dtypes:
        raise ValueError(f"unsupported dtype {rgb.dtype} (have: {', '.join(dtypes)})")
    return name


def _stream(stream, device):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _check_out(out, shape, like, dtype=None):
    """A caller-supplied output tensor: contiguous, ``shape``, ``like``'s device, ``dtype`` (default like's)."""
    dtype = like.dtype if dtype is None else dtype
    if tuple(out.shape) != tuple(shape) or out.dtype != dtype or not out.is_contiguous() \
            or out.device != like.device:
        raise ValueError(f"out must be a contiguous {dtype} tensor of shape {tuple(shape)} on {like.device}")
    return out


def decolor(rgb, params: DecolorParams = DEFAULT_PARAMS, out=None, stream=None, exact: bool = False):
    """Gray of a device-resident (..., 3) uint8 / float32 / float64 batch.

    uint8: identical to quantize_u8 of the reference except +-1 on rounding
    ties (5e-6 of colours); ``exact=True`` makes it bit-identical (~10%
    slower). float64 is always bit-identical; float32 within 1e-6.
    """
    torch = _torch()
    name = _check_rgb_tensor(rgb, _DECOLOR_FN)
    out = _check_out(out, rgb.shape[:-1], rgb) if out is not None else \
        torch.empty(rgb.shape[:-1], dtype=rgb.dtype, device=rgb.device)
    n = out.numel()
    fn = "wg_decolor_u8_exact" if exact and name == "uint8" else _DECOLOR_FN[name]
    with torch.cuda.device(rgb.device):
        _lib.call(fn, rgb.data_ptr(), out.data_ptr(), n, params.beta_r, params.beta_k, _stream(stream, rgb.device))
    return out


def decolor_tone(rgb, curve: SigmoidCurve = SigmoidCurve(), params: DecolorParams = DEFAULT_PARAMS,
                 return_gray: bool = False, return_rgb: bool = False, stream=None, exact: bool = False,
                 out=None):
    """Fused decolor + global sigmoid on a device batch.

    uint8 -> toned uint8 (and gray uint8 if ``return_gray``; with
    ``return_rgb`` also the reinstated colour image as uint8, i.e.
    quantize_u8 of tonemap_image(mode="global")[0]). The default uint8 route
    meets the north-star bar (+-1 on <= 0.01% of pixels); ``exact=True`` (and
    every ``return_rgb`` call) is bit-identical to the reference (fp32 with a
    rigorous error bound, the fp64 chain for pixels in doubt).
    float32 -> toned float32 (+ gray, + reinstated rgb if requested).
    Returns the toned tensor, or a tuple ``(toned, gray, rgb_out)`` with
    ``None`` for outputs not requested when either flag is set. ``out``: a
    preallocated toned tensor (contiguous, rgb's dtype and device, shape
    ``rgb.shape[:-1]``).
    """
    torch = _torch()
    name = _check_rgb_tensor(rgb, ("uint8", "float32"))
    shape = rgb.shape[:-1]
    toned = _check_out(out, shape, rgb) if out is not None else torch.empty(shape, dtype=rgb.dtype, device=rgb.device)
    gray = torch.empty(shape, dtype=rgb.dtype, device=rgb.device) if return_gray else None
    rgb_out = None
    with torch.cuda.device(rgb.device):
        st = _stream(stream, rgb.device)
        if name == "uint8" and (return_rgb or exact):
            # bit-identical route (wg_decolor_tone_rgb_u8; the colour image only when asked)
            rgb_out = torch.empty_like(rgb) if return_rgb else None
            _lib.call("wg_decolor_tone_rgb_u8", rgb.data_ptr(), rgb_out.data_ptr() if rgb_out is not None else None,
                      toned.data_ptr(), gray.data_ptr() if gray is not None else None, toned.numel(), params.beta_r,
                      params.beta_k, curve.midpoint, curve.slope, st)
        elif name == "uint8":
            _lib.call("wg_decolor_tone_u8", rgb.data_ptr(), toned.data_ptr(),
                      gray.data_ptr() if gray is not None else None, toned.numel(),
                      params.beta_r, params.beta_k, curve.midpoint, curve.slope, st)
        else:
            rgb_out = torch.empty_like(rgb) if return_rgb else None
            _lib.call("wg_decolor_tone_f32", rgb.data_ptr(), toned.data_ptr(),
                      gray.data_ptr() if gray is not None else None,
                      rgb_out.data_ptr() if rgb_out is not None else None, toned.numel(),
                      params.beta_r, params.beta_k, curve.midpoint, curve.slope, st)
    if return_gray or return_rgb:
        return toned, gray, rgb_out
    return toned


def sigmoid(lum, curve: SigmoidCurve = SigmoidCurve(), stream=None):
    """apply_sigmoid on a device float32 / float64 tensor."""
    torch = _torch()
    if not isinstance(lum, torch.Tensor) or not lum.is_cuda or not lum.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    fn = {torch.float32: "wg_sigmoid_f32", torch.float64: "wg_sigmoid_f64"}.get(lum.dtype)
    if fn is None:
        raise ValueError(f"unsupported dtype {lum.dtype}")
    out = torch.empty_like(lum)
    with torch.cuda.device(lum.device):
        _lib.call(fn, lum.data_ptr(), out.data_ptr(), lum.numel(), curve.midpoint, curve.slope,
                  _stream(stream, lum.device))
    return out


_LUMA_METHOD = {"y": 0, "weighted": 0, "v": 1, "lab": 2}


def _luma_code(method: str) -> int:
    if method not in _LUMA_METHOD:
        raise ValueError(f"unknown luma method {method!r} (have: {', '.join(_LUMA_METHOD)})")
    return _LUMA_METHOD[method]


def luma(rgb, method: str = "y", stream=None):
    """Baseline gray of a device (..., 3) uint8 / float64 batch.

    float64 follows the reference's bt601_rows / hsv_value_rows /
    lab_lightness_rows; uint8 is quantize_u8 of that on dequantized input.
    """
    torch = _torch()
    name = _check_rgb_tensor(rgb, ("uint8", "float64"))
    code = _luma_code(method)
    out = torch.empty(rgb.shape[:-1], dtype=rgb.dtype, device=rgb.device)
    with torch.cuda.device(rgb.device):
        _lib.call("wg_luma_u8" if name == "uint8" else "wg_luma_f64", rgb.data_ptr(), out.data_ptr(),
                  out.numel(), code, _stream(stream, rgb.device))
    return out


def lab(rgb, stream=None):
    """CIELAB (L*, a*, b*) of a device (..., 3) float64 sRGB batch (lab_rows)."""
    torch = _torch()
    _check_rgb_tensor(rgb, ("float64",))
    out = torch.empty_like(rgb)
    with torch.cuda.device(rgb.device):
        _lib.call("wg_lab_f64", rgb.data_ptr(), out.data_ptr(), rgb.numel() // 3, _stream(stream, rgb.device))
    return out


def _grid_for(h, w, grid):
    from .tonemap import LocalHistogramGrid

    return grid or LocalHistogramGrid.for_image(w, h)


def _nhw(shape):
    if len(shape) == 3:
        return 1, shape[0], shape[1]
    if len(shape) == 4:
        return shape[0], shape[1], shape[2]
    raise ValueError(f"expected (H, W, 3) or (N, H, W, 3), got shape {tuple(shape)}")


def decolor_tone_local(rgb, grid=None, params: DecolorParams = DEFAULT_PARAMS, return_gray: bool = False,
                       scratch=None, stream=None, out=None):
    """Fused decolor + local tone map of a device uint8 (N, H, W, 3) / (H, W, 3) batch.

    Per image: toned = quantize_u8(apply_local_lhe(decolor_image(rgb / 255), grid)),
    bit-identical to the fp64 reference; ``return_gray`` adds quantize_u8 of the
    gray. ``grid`` defaults to LocalHistogramGrid.for_image(W, H); ``out``: optional
    destination for the toned batch (contiguous uint8, rgb.shape[:-1]).
    """
    torch = _torch()
    _check_rgb_tensor(rgb, ("uint8",))
    n, h, w = _nhw(rgb.shape)
    g = _grid_for(h, w, grid)
    toned = torch.empty(rgb.shape[:-1], dtype=torch.uint8, device=rgb.device) if out is None \
        else _check_out(out, rgb.shape[:-1], rgb)
    gray = torch.empty_like(toned) if return_gray else None
    need = int(_lib.load().wg_lhe_scratch_bytes(n, h, w, g.tile_w, g.tile_h, g.bins))
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(max(need, 1), dtype=torch.uint8, device=rgb.device)
    with torch.cuda.device(rgb.device):
        _lib.call("wg_decolor_tone_local_u8", rgb.data_ptr(), toned.data_ptr(),
                  gray.data_ptr() if gray is not None else None, n, h, w, params.beta_r, params.beta_k,
                  g.tile_w, g.tile_h, g.bins, g.strength, scratch.data_ptr(), scratch.numel(),
                  _stream(stream, rgb.device))
    return (toned, gray) if return_gray else toned


class HdrScratch:
    """Reusable device scratch for :func:`hdr_tonemap` (gray plane + per-block partials)."""

    def __init__(self, nimg: int, pix_per_img: int, device=None):
        torch = _torch()
        self.nbytes = int(_lib.load().wg_hdr_scratch_bytes(nimg, pix_per_img))
        self.buf = torch.empty(max(self.nbytes, 1), dtype=torch.uint8,
                               device=device if device is not None else "cuda")


def hdr_tonemap(rgb, params: DecolorParams = DEFAULT_PARAMS, curve: SigmoidCurve = SigmoidCurve(),
                scratch: HdrScratch | None = None, out=None, stream=None):
    """HDR adapter on a device (N, H, W, 3) float32 radiance batch -> uint8."""
    torch = _torch()
    _check_rgb_tensor(rgb, ("float32",))
    if rgb.dim() < 2:
        raise ValueError("hdr_tonemap expects a batch (N, ..., 3)")
    n = rgb.shape[0]
    ppi = rgb[0].numel() // 3 if n else 0
    if out is None:
        out = torch.empty(rgb.shape[:-1], dtype=torch.uint8, device=rgb.device)
    else:
        _check_out(out, rgb.shape[:-1], rgb, dtype=torch.uint8)
    need = int(_lib.load().wg_hdr_scratch_bytes(n, ppi))
    if scratch is None or scratch.nbytes < need:
        scratch = HdrScratch(n, ppi, device=rgb.device)
    with torch.cuda.device(rgb.device):
        _lib.call("wg_hdr_tonemap_u8", rgb.data_ptr(), out.data_ptr(), n, ppi, params.beta_r,
                  params.beta_k, curve.midpoint, curve.slope, scratch.buf.data_ptr(),
                  scratch.nbytes, _stream(stream, rgb.device))
    return out


# ---------------------------------------------------------------- host-array flavour

def _host_rgb(rgb, dtypes):
    arr = np.asarray(rgb)
    if arr.ndim < 1 or arr.shape[-1] != 3:
        raise ValueError(f"rgb needs a trailing channel axis of 3, got shape {arr.shape}")
    if arr.dtype.name not in dtypes:
        raise ValueError(f"unsupported dtype {arr.dtype} (have: {', '.join(dtypes)})")
    return np.ascontiguousarray(arr)


def decolor_host(rgb, params: DecolorParams = DEFAULT_PARAMS, out=None, device: int | None = None,
                 exact: bool = False):
    """Gray of a host (..., 3) uint8 / float32 / float64 array via the pipelined host path (see :func:`decolor`)."""
    arr = _host_rgb(rgb, ("uint8", "float32", "float64"))
    if out is None:
        out = np.empty(arr.shape[:-1], dtype=arr.dtype)
    elif out.shape != arr.shape[:-1] or out.dtype != arr.dtype or not out.flags["C_CONTIGUOUS"]:
        raise ValueError("out must be C-contiguous with shape rgb.shape[:-1] and rgb's dtype")
    dev = get_device() if device is None else device
    n = out.size
    if n:
        if arr.dtype == np.uint8:
            _lib.call("wg_host_decolor_u8_exact" if exact else "wg_host_decolor_u8", arr.ctypes.data,
                      out.ctypes.data, n, params.beta_r, params.beta_k, dev)
        elif arr.dtype == np.float32:
            _lib.call("wg_host_decolor_f32", arr.ctypes.data, out.ctypes.data, n, params.beta_r,
                      params.beta_k, dev)
        else:
            _lib.call("wg_host_decolor_rows_f64", arr.ctypes.data, out.ctypes.data, 1, n,
                      params.beta_r, params.beta_k, 0, 1, dev)
    return out


def luma_host(rgb, method: str = "y", device: int | None = None):
    """Baseline gray of a host uint8 (..., 3) array -> uint8 via the pipelined host path."""
    arr = _host_rgb(rgb, ("uint8",))
    code = _luma_code(method)
    out = np.empty(arr.shape[:-1], dtype=np.uint8)
    if out.size:
        _lib.call("wg_host_luma_u8", arr.ctypes.data, out.ctypes.data, out.size, code,
                  get_device() if device is None else device)
    return out


def _host_out(out, shape):
    """A caller's destination array (pinned keeps the copies asynchronous) or a new one."""
    if out is None:
        return np.empty(shape, dtype=np.uint8)
    if out.shape != tuple(shape) or out.dtype != np.uint8 or not out.flags["C_CONTIGUOUS"]:
        raise ValueError(f"out must be C-contiguous uint8 of shape {tuple(shape)}")
    return out


def decolor_tone_local_host(rgb, grid=None, params: DecolorParams = DEFAULT_PARAMS, return_gray: bool = False,
                            device: int | None = None, out=None):
    """:func:`decolor_tone_local` on a host uint8 (N, H, W, 3) / (H, W, 3) array (pipelined per image);
    ``out``: optional destination for the toned batch."""
    arr = _host_rgb(rgb, ("uint8",))
    n, h, w = _nhw(arr.shape)
    g = _grid_for(h, w, grid)
    toned = _host_out(out, arr.shape[:-1])
    gray = np.empty_like(toned) if return_gray else None
    _lib.call("wg_host_decolor_tone_local_u8", arr.ctypes.data, toned.ctypes.data,
              gray.ctypes.data if gray is not None else None, n, h, w, params.beta_r, params.beta_k,
              g.tile_w, g.tile_h, g.bins, g.strength, get_device() if device is None else device)
    return (toned, gray) if return_gray else toned


def decolor_tone_host(rgb, curve: SigmoidCurve = SigmoidCurve(),
                      params: DecolorParams = DEFAULT_PARAMS, return_gray: bool = False,
                      device: int | None = None, return_rgb: bool = False, out=None, exact: bool = False):
    """Fused decolor + global sigmoid of a host uint8 (..., 3) array -> toned uint8 (+ gray).

    With ``return_rgb`` returns ``(toned, gray, rgb_out)`` (gray None unless
    requested), rgb_out the reinstated colour image as uint8. ``out``:
    optional destination for the toned array. ``exact``: bit-identical toned
    (and gray) bytes, as with ``return_rgb``.
    """
    arr = _host_rgb(rgb, ("uint8",))
    toned = _host_out(out, arr.shape[:-1])
    gray = np.empty_like(toned) if return_gray else None
    rgb_out = np.empty_like(arr) if return_rgb else None
    dev = get_device() if device is None else device
    if toned.size and (return_rgb or exact):  # bit-identical route
        _lib.call("wg_host_decolor_tone_rgb_u8", arr.ctypes.data,
                  rgb_out.ctypes.data if rgb_out is not None else None, toned.ctypes.data,
                  gray.ctypes.data if gray is not None else None, toned.size, params.beta_r,
                  params.beta_k, curve.midpoint, curve.slope, dev)
    elif toned.size:
        _lib.call("wg_host_decolor_tone_u8", arr.ctypes.data, toned.ctypes.data,
                  gray.ctypes.data if gray is not None else None, toned.size, params.beta_r,
                  params.beta_k, curve.midpoint, curve.slope, dev)
    if return_rgb:
        return toned, gray, rgb_out
    return (toned, gray) if return_gray else toned


def hdr_tonemap_host(rgb, params: DecolorParams = DEFAULT_PARAMS,
                     curve: SigmoidCurve = SigmoidCurve(), device: int | None = None, out=None):
    """HDR adapter on a host (N, H, W, 3) float32 batch -> (N, H, W) uint8.

    ``out`` (optional, C-contiguous uint8 of shape rgb.shape[:-1]): pass a
    pinned buffer to keep the device -> host copies asynchronous (a pageable
    destination serialises the copy pipeline).
    """
    arr = _host_rgb(rgb, ("float32",))
    if arr.ndim < 2:
        raise ValueError("hdr_tonemap_host expects a batch (N, ..., 3)")
    if out is None:
        out = np.empty(arr.shape[:-1], dtype=np.uint8)
    elif out.shape != arr.shape[:-1] or out.dtype != np.uint8 or not out.flags["C_CONTIGUOUS"]:
        raise ValueError("out must be C-contiguous uint8 with shape rgb.shape[:-1]")
    n = arr.shape[0]
    ppi = out.size // n if n else 0
    if out.size:
        _lib.call("wg_host_hdr_tonemap_u8", arr.ctypes.data, out.ctypes.data, n, ppi,
                  params.beta_r, params.beta_k, curve.midpoint, curve.slope,
                  get_device() if device is None else device)
    return out
