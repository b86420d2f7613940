"""CPU oracle bindings -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/_build/liboracle.so`` (built from
``oracle/warmgray_oracle.c`` by ``oracle/Makefile``), the fp64 restatement
of the reference's hot path (/root/reference/pkg/src/warmgray/_kernels.pyx:31-56,
codec.py:22-29, tonemap.py:72-83,172-216). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs import this
module, as the checker or as the timed CPU baseline. The product package
``paper_2108_13656_b200`` never imports it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

_c_dp = ctypes.POINTER(ctypes.c_double)
_c_fp = ctypes.POINTER(ctypes.c_float)
_c_u8p = ctypes.POINTER(ctypes.c_uint8)
_c_i32p = ctypes.POINTER(ctypes.c_int32)
_i64 = ctypes.c_int64
_d = ctypes.c_double
_i = ctypes.c_int

_SIGS = {
    "or_decolor_f64": [_c_dp, _c_dp, _i64, _d, _d, _i],
    "or_decolor_f32in": [_c_fp, _c_dp, _i64, _d, _d, _i],
    "or_decolor_u8": [_c_u8p, _c_u8p, _i64, _d, _d, _i],
    "or_luma_f64": [_c_dp, _c_dp, _i64, _i, _i],
    "or_lab_f64": [_c_dp, _c_dp, _i64, _i],
    "or_luma_u8": [_c_u8p, _c_u8p, _i64, _i, _i],
    "or_local_lhe_f64": [_c_dp, _c_dp, _i64, _i64, _i64, _i64, _i64, _i, _d, _i],
    "or_tone_local_u8": [_c_u8p, _c_u8p, _c_u8p, _i64, _i64, _i64, _d, _d, _i64, _i64, _i, _d, _i],
    "or_metric_counts_f64": [_c_dp, _c_dp, _i64, _c_dp, _i, ctypes.POINTER(ctypes.c_int64),
                             ctypes.POINTER(ctypes.c_int64), _i64, ctypes.POINTER(ctypes.c_int64), _i],
    "or_sigmoid_f64": [_c_dp, _c_dp, _i64, _d, _d],
    "or_reinstate_f64": [_c_dp, _c_dp, _c_dp, _c_dp, _i64],
    "or_tone_u8": [_c_u8p, _c_u8p, _c_u8p, _i64, _d, _d, _d, _d, _i],
    "or_tonemap_global_f64": [_c_dp, _c_dp, _c_dp, _i64, _d, _d, _d, _d],
    "or_tone_rgb_u8": [_c_u8p, _c_u8p, _c_u8p, _c_u8p, _i64, _d, _d, _d, _d, _i],
    "or_hdr_u8": [_c_fp, _c_u8p, _i64, _i64, _d, _d, _d, _d, _i],
    "or_synth_uniform_u8": [_c_u8p, _i64, _i64, ctypes.c_uint32, _i64],
    "or_synth_voronoi_u8": [_c_u8p, _i64, ctypes.c_int32, ctypes.c_int32, _c_i32p, _c_u8p,
                            ctypes.c_int32, ctypes.c_uint32, _i64],
}

_lib = None


def build() -> None:
    """Compile the oracle with its Makefile (gcc is in the image)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        handle = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = None
        _lib = handle
    return _lib


def _ptr(a: np.ndarray, ctype):
    assert a.flags["C_CONTIGUOUS"], "oracle expects C-contiguous arrays"
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def decolor_f64(rgb: np.ndarray, beta_r=0.55, beta_k=0.8, threads: int = 1) -> np.ndarray:
    """fp64 gray of fp64 rgb (..., 3); bit-identical to _kernels.decolor_rows."""
    rgb = np.ascontiguousarray(rgb, dtype=np.float64)
    out = np.empty(rgb.shape[:-1], dtype=np.float64)
    lib().or_decolor_f64(_ptr(rgb, ctypes.c_double), _ptr(out, ctypes.c_double),
                         out.size, beta_r, beta_k, threads)
    return out


def decolor_f32in(rgb: np.ndarray, beta_r=0.55, beta_k=0.8, threads: int = 1) -> np.ndarray:
    """fp64 gray of fp32 rgb (exact promotion, as PlanarImage would do)."""
    rgb = np.ascontiguousarray(rgb, dtype=np.float32)
    out = np.empty(rgb.shape[:-1], dtype=np.float64)
    lib().or_decolor_f32in(_ptr(rgb, ctypes.c_float), _ptr(out, ctypes.c_double),
                           out.size, beta_r, beta_k, threads)
    return out


def decolor_u8(rgb: np.ndarray, beta_r=0.55, beta_k=0.8, threads: int = 1) -> np.ndarray:
    """quantize_u8(decolor_image(PlanarImage(dequantize_u8(rgb))).data)."""
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    out = np.empty(rgb.shape[:-1], dtype=np.uint8)
    lib().or_decolor_u8(_ptr(rgb, ctypes.c_uint8), _ptr(out, ctypes.c_uint8),
                        out.size, beta_r, beta_k, threads)
    return out


LUMA_METHODS = {"y": 0, "weighted": 0, "v": 1, "lab": 2}


def luma_f64(rgb: np.ndarray, method: str, threads: int = 1) -> np.ndarray:
    """bt601_rows / hsv_value_rows / lab_lightness_rows (_kernels.pyx:59-112) on fp64 rgb."""
    rgb = np.ascontiguousarray(rgb, dtype=np.float64)
    out = np.empty(rgb.shape[:-1], dtype=np.float64)
    lib().or_luma_f64(_ptr(rgb, ctypes.c_double), _ptr(out, ctypes.c_double), out.size,
                      LUMA_METHODS[method], threads)
    return out


def lab_f64(rgb: np.ndarray, threads: int = 1) -> np.ndarray:
    """lab_rows (_kernels.pyx:115-132): (..., 3) CIELAB of fp64 rgb."""
    rgb = np.ascontiguousarray(rgb, dtype=np.float64)
    out = np.empty_like(rgb)
    lib().or_lab_f64(_ptr(rgb, ctypes.c_double), _ptr(out, ctypes.c_double), rgb.size // 3, threads)
    return out


def luma_u8(rgb: np.ndarray, method: str, threads: int = 1) -> np.ndarray:
    """quantize_u8(luminance_image(dequantize_u8(rgb), method).data)."""
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    out = np.empty(rgb.shape[:-1], dtype=np.uint8)
    lib().or_luma_u8(_ptr(rgb, ctypes.c_uint8), _ptr(out, ctypes.c_uint8), out.size,
                     LUMA_METHODS[method], threads)
    return out


def local_lhe_f64(lum: np.ndarray, tile_w: int, tile_h: int, bins: int = 256, strength: float = 0.7,
                  threads: int = 1) -> np.ndarray:
    """apply_local_lhe (tonemap.py:103-169) on (H, W) or (N, H, W) fp64 luminance."""
    lum = np.ascontiguousarray(lum, dtype=np.float64)
    n, h, w = (1,) + lum.shape if lum.ndim == 2 else lum.shape
    out = np.empty_like(lum)
    lib().or_local_lhe_f64(_ptr(lum, ctypes.c_double), _ptr(out, ctypes.c_double), n, h, w, tile_w, tile_h,
                           bins, strength, threads)
    return out


def tone_local_u8(rgb: np.ndarray, tile_w: int, tile_h: int, bins: int = 256, strength: float = 0.7,
                  beta_r=0.55, beta_k=0.8, threads: int = 1, with_gray: bool = False):
    """quantize_u8(apply_local_lhe(decolor_image(dequantize_u8(rgb)))) per image of (N, H, W, 3) / (H, W, 3)."""
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    n, h, w = (1,) + rgb.shape[:2] if rgb.ndim == 3 else rgb.shape[:3]
    toned = np.empty(rgb.shape[:-1], dtype=np.uint8)
    gray = np.empty_like(toned) if with_gray else None
    lib().or_tone_local_u8(_ptr(rgb, ctypes.c_uint8), _ptr(toned, ctypes.c_uint8),
                           _ptr(gray, ctypes.c_uint8) if gray is not None else None, n, h, w, beta_r, beta_k,
                           tile_w, tile_h, bins, strength, threads)
    return (toned, gray) if with_gray else toned


def metric_counts(rgb: np.ndarray, gray: np.ndarray, taus, pairs=None, threads: int = 1) -> np.ndarray:
    """_sweep_counts (metrics.py:118-135): (ntau, 4) counts; pairs = (i, j) arrays or None for all pairs."""
    rgb = np.ascontiguousarray(rgb, dtype=np.float64)
    gray = np.ascontiguousarray(gray, dtype=np.float64)
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    out = np.zeros((len(taus), 4), dtype=np.int64)
    pi = pj = None
    npairs = 0
    if pairs is not None:
        pi = np.ascontiguousarray(pairs[0], dtype=np.int64)
        pj = np.ascontiguousarray(pairs[1], dtype=np.int64)
        npairs = len(pi)
    lib().or_metric_counts_f64(_ptr(rgb, ctypes.c_double), _ptr(gray, ctypes.c_double), gray.size,
                               _ptr(taus, ctypes.c_double), len(taus),
                               _ptr(pi, ctypes.c_int64) if pi is not None else None,
                               _ptr(pj, ctypes.c_int64) if pj is not None else None, npairs,
                               _ptr(out, ctypes.c_int64), threads)
    return out


def sigmoid_f64(x: np.ndarray, midpoint=0.5, slope=8.0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().or_sigmoid_f64(_ptr(x, ctypes.c_double), _ptr(out, ctypes.c_double), x.size,
                         midpoint, slope)
    return out


def reinstate_f64(rgb: np.ndarray, l_in: np.ndarray, l_out: np.ndarray) -> np.ndarray:
    rgb = np.ascontiguousarray(rgb, dtype=np.float64)
    l_in = np.ascontiguousarray(l_in, dtype=np.float64)
    l_out = np.ascontiguousarray(l_out, dtype=np.float64)
    out = np.empty_like(rgb)
    lib().or_reinstate_f64(_ptr(rgb, ctypes.c_double), _ptr(l_in, ctypes.c_double),
                           _ptr(l_out, ctypes.c_double), _ptr(out, ctypes.c_double), l_in.size)
    return out


def tone_u8(rgb: np.ndarray, beta_r=0.55, beta_k=0.8, midpoint=0.5, slope=8.0,
            threads: int = 1, with_gray: bool = False):
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    toned = np.empty(rgb.shape[:-1], dtype=np.uint8)
    gray = np.empty_like(toned) if with_gray else None
    lib().or_tone_u8(_ptr(rgb, ctypes.c_uint8), _ptr(toned, ctypes.c_uint8),
                     _ptr(gray, ctypes.c_uint8) if gray is not None else None,
                     toned.size, beta_r, beta_k, midpoint, slope, threads)
    return (toned, gray) if with_gray else toned


def tone_rgb_u8(rgb: np.ndarray, beta_r=0.55, beta_k=0.8, midpoint=0.5, slope=8.0, threads: int = 1):
    """(rgb_out, toned, gray) u8: quantize_u8 of tonemap_image(mode='global') on dequantize_u8(rgb)."""
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    out = np.empty_like(rgb)
    toned = np.empty(rgb.shape[:-1], dtype=np.uint8)
    gray = np.empty_like(toned)
    lib().or_tone_rgb_u8(_ptr(rgb, ctypes.c_uint8), _ptr(out, ctypes.c_uint8), _ptr(toned, ctypes.c_uint8),
                         _ptr(gray, ctypes.c_uint8), toned.size, beta_r, beta_k, midpoint, slope, threads)
    return out, toned, gray


def tonemap_global_f64(rgb: np.ndarray, beta_r=0.55, beta_k=0.8, midpoint=0.5, slope=8.0):
    """(rgb_out, l_out) of tonemap_image(mode='global')."""
    rgb = np.ascontiguousarray(rgb, dtype=np.float64)
    l_out = np.empty(rgb.shape[:-1], dtype=np.float64)
    rgb_out = np.empty_like(rgb)
    lib().or_tonemap_global_f64(_ptr(rgb, ctypes.c_double), _ptr(l_out, ctypes.c_double),
                                _ptr(rgb_out, ctypes.c_double), l_out.size, beta_r, beta_k,
                                midpoint, slope)
    return rgb_out, l_out


def hdr_u8(rgb: np.ndarray, beta_r=0.55, beta_k=0.8, midpoint=0.5, slope=8.0,
           threads: int = 1) -> np.ndarray:
    """HDR adapter over a batch (N, H, W, 3) float32 -> (N, H, W) u8."""
    rgb = np.ascontiguousarray(rgb, dtype=np.float32)
    n = rgb.shape[0]
    ppi = int(np.prod(rgb.shape[1:-1]))
    out = np.empty(rgb.shape[:-1], dtype=np.uint8)
    lib().or_hdr_u8(_ptr(rgb, ctypes.c_float), _ptr(out, ctypes.c_uint8), n, ppi, beta_r, beta_k,
                    midpoint, slope, threads)
    return out


def synth_uniform_u8(nimg: int, height: int, width: int, seed: int, first_image: int = 0):
    out = np.empty((nimg, height, width, 3), dtype=np.uint8)
    lib().or_synth_uniform_u8(_ptr(out, ctypes.c_uint8), nimg, height * width * 3, seed,
                              first_image)
    return out


def synth_voronoi_u8(height: int, width: int, seeds_xy: np.ndarray, colors: np.ndarray,
                     seed: int, first_image: int = 0):
    seeds_xy = np.ascontiguousarray(seeds_xy, dtype=np.int32)
    colors = np.ascontiguousarray(colors, dtype=np.uint8)
    nimg, nseeds = seeds_xy.shape[0], seeds_xy.shape[1]
    out = np.empty((nimg, height, width, 3), dtype=np.uint8)
    lib().or_synth_voronoi_u8(_ptr(out, ctypes.c_uint8), nimg, width, height,
                              _ptr(seeds_xy, ctypes.c_int32), _ptr(colors, ctypes.c_uint8),
                              nseeds, seed, first_image)
    return out


def color_cube_u8() -> np.ndarray:
    """All 2^24 uint8 colours as a 4096x4096 image, index i -> (i>>16, (i>>8)&255, i&255)."""
    i = np.arange(1 << 24, dtype=np.uint32)
    cube = np.empty((1 << 24, 3), dtype=np.uint8)
    cube[:, 0] = i >> 16
    cube[:, 1] = (i >> 8) & 255
    cube[:, 2] = i & 255
    return cube.reshape(4096, 4096, 3)
