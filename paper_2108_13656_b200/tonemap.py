"""Tone mapping of the gray channel and ratio-based colour reinstatement.

Drop-in for /root/reference/pkg/src/warmgray/tonemap.py: ``SigmoidCurve``
(tonemap.py:22-33), ``LocalHistogramGrid`` (:36-69), ``apply_sigmoid``
(:72-83), ``apply_local_lhe`` (:103-169), ``reinstate_color`` (:172-192) and
``tonemap_image`` (:195-216). All image work runs in fp64 device kernels (the
reference's own precision, bit-identical results):

* ``tonemap_image(mode="global")`` is ONE fused device pass
  (decolor -> sigmoid -> reinstate) instead of three NumPy passes;
* ``mode="local"`` runs decolor, the tile-histogram equalisation
  (histograms -> CDF curves -> bilinear blend; csrc/wg_lhe.cu) and the
  reinstatement back to back on the device with the gray kept resident.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .backend import get_device, get_kernels, resolve_threads
from .core import DEFAULT_PARAMS, DecolorParams, PlanarImage


@dataclass(frozen=True)
class SigmoidCurve:
    """Logistic tone curve renormalised to map 0 to 0 and 1 to 1."""

    midpoint: float = 0.5
    slope: float = 8.0

    def __post_init__(self):
        if not 0.0 <= self.midpoint <= 1.0:
            raise ValueError(f"midpoint must lie in [0, 1], got {self.midpoint!r}")
        if not self.slope > 0.0 or math.isinf(self.slope):
            raise ValueError(f"slope must be a positive finite value, got {self.slope!r}")


@dataclass(frozen=True)
class LocalHistogramGrid:
    """Tile layout and blend strength for local histogram equalisation (tonemap.py:36-69)."""

    tile_w: int
    tile_h: int
    bins: int = 256
    strength: float = 0.7

    def __post_init__(self):
        if self.tile_w < 1 or self.tile_h < 1:
            raise ValueError(f"tile size must be >= 1, got {self.tile_w}x{self.tile_h}")
        if self.bins < 2:
            raise ValueError(f"bins must be >= 2, got {self.bins}")
        if not 0.0 <= self.strength <= 1.0:
            raise ValueError(f"strength must lie in [0, 1], got {self.strength!r}")

    @classmethod
    def for_image(cls, width: int, height: int, tiles_x: int = 8, tiles_y: int = 8,
                  bins: int = 256, strength: float = 0.7) -> "LocalHistogramGrid":
        """Grid sized so the image splits into about tiles_x by tiles_y tiles."""
        return cls(tile_w=max(1, -(-width // tiles_x)), tile_h=max(1, -(-height // tiles_y)),
                   bins=bins, strength=strength)


def apply_sigmoid(img: PlanarImage, curve: SigmoidCurve = SigmoidCurve()) -> PlanarImage:
    """Monotone global remap of a luminance image through the curve (GPU, fp64)."""
    if img.kind != "luminance":
        raise ValueError("apply_sigmoid expects a luminance image")
    out = np.empty_like(img.data)
    if out.size:
        _lib.call("wg_host_sigmoid_f64", img.data.ctypes.data, out.ctypes.data, out.size,
                  float(curve.midpoint), float(curve.slope), get_device())
    return PlanarImage._from_kernel(out)


def reinstate_color(rgb: PlanarImage, l_in: PlanarImage, l_out: PlanarImage) -> PlanarImage:
    """Rescale RGB by the luminance ratio l_out / max(l_in, 1e-6); l_in == 0 stays black."""
    if rgb.kind != "rgb" or l_in.kind != "luminance" or l_out.kind != "luminance":
        raise ValueError("reinstate_color expects (rgb, luminance, luminance) images")
    dims = (rgb.width, rgb.height)
    if dims != (l_in.width, l_in.height) or dims != (l_out.width, l_out.height):
        raise ValueError("reinstate_color requires matching image dimensions")
    out = np.empty_like(rgb.data)
    if out.size:
        _lib.call("wg_host_reinstate_f64", rgb.data.ctypes.data, l_in.data.ctypes.data,
                  l_out.data.ctypes.data, out.ctypes.data, l_in.data.size, get_device())
    return PlanarImage._from_kernel(out)


def apply_local_lhe(img: PlanarImage, grid: LocalHistogramGrid, threads: int | None = None) -> PlanarImage:
    """Local histogram equalisation with bilinearly blended tile curves.

    Each tile's cumulative histogram, stretched over its occupied range, is a
    tone curve; per pixel the four surrounding tile curves are blended and
    the result mixed with the identity by ``grid.strength``. Single-bin tiles
    (constant content) keep their values; tiles larger than the image are
    clamped to it. ``threads`` is validated only: the GPU result does not
    depend on it (the reference's test_thread_count_invariance).
    """
    if img.kind != "luminance":
        raise ValueError("apply_local_lhe expects a luminance image")
    resolve_threads(threads)
    data = img.data
    h, w = data.shape
    out = np.empty_like(data)
    if h and w:
        _lib.call("wg_host_local_lhe_f64", data.ctypes.data, out.ctypes.data, h, w, int(grid.tile_w),
                  int(grid.tile_h), int(grid.bins), float(grid.strength), get_device())
    else:
        out = data.copy()
    return PlanarImage._from_kernel(out)


def tonemap_image(
    rgb: PlanarImage,
    mode: str = "global",
    params: DecolorParams = DEFAULT_PARAMS,
    curve: SigmoidCurve | None = None,
    grid: LocalHistogramGrid | None = None,
    threads: int | None = None,
    backend: str | None = None,
) -> tuple[PlanarImage, PlanarImage]:
    """Decolorize, tone-map the luminance, reinstate colour -> ``(rgb_out, toned_luminance)``."""
    if rgb.kind != "rgb":
        raise ValueError("decolor_image expects an rgb image")
    get_kernels(backend)
    resolve_threads(threads)
    if mode == "global":
        c = curve or SigmoidCurve()
        l_out = np.empty((rgb.height, rgb.width), dtype=np.float64)
        rgb_out = np.empty_like(rgb.data)
        if l_out.size:
            _lib.call("wg_host_tonemap_global_f64", rgb.data.ctypes.data, l_out.ctypes.data,
                      rgb_out.ctypes.data, l_out.size, params.beta_r, params.beta_k,
                      float(c.midpoint), float(c.slope), get_device())
        return PlanarImage._from_kernel(rgb_out), PlanarImage._from_kernel(l_out)
    if mode == "local":
        g = grid or LocalHistogramGrid.for_image(rgb.width, rgb.height)
        l_out = np.empty((rgb.height, rgb.width), dtype=np.float64)
        rgb_out = np.empty_like(rgb.data)
        if l_out.size:
            _lib.call("wg_host_tonemap_local_f64", rgb.data.ctypes.data, l_out.ctypes.data,
                      rgb_out.ctypes.data, rgb.height, rgb.width, params.beta_r, params.beta_k,
                      int(g.tile_w), int(g.tile_h), int(g.bins), float(g.strength), get_device())
        return PlanarImage._from_kernel(rgb_out), PlanarImage._from_kernel(l_out)
    raise ValueError(f"unknown tonemap mode {mode!r} (use 'global' or 'local')")
