"""ctypes binding of ``libwarmgray_b200.so`` (the C ABI in include/warmgray_b200.h).

The shared library is built in-tree by :func:`paper_2108_13656_b200.build.build`
(nvcc, ``-gencode arch=compute_100a,code=sm_100a``). There is no CPU fallback:
if the library is missing, or no CUDA device is present, every compute call
raises instead of silently computing something elsewhere.

Status convention (warmgray_b200.h): 0 ok; negative = argument error, raised
as ``ValueError`` like the reference's validation errors; positive = a
``cudaError_t``, raised as :class:`CudaError` (a ``RuntimeError``).
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "_build", "libwarmgray_b200.so")


WG_EINVAL, WG_EALIGN, WG_ESCRATCH, ENODEV, WG_ECODEC, WG_EIO = -1, -2, -3, -4, -5, -6


class CudaError(RuntimeError):
    """A CUDA runtime failure reported by the B200 kernels."""


class CodecError(Exception):
    """Unsupported or malformed image file (the reference's codec.CodecError)."""


class ExtensionMissing(ImportError):
    """The sm_100a library has not been built (run __graft_entry__.build())."""


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_f = ctypes.c_float
_d = ctypes.c_double
_i = ctypes.c_int
_u32 = ctypes.c_uint32
_sz = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/warmgray_b200.h
SIGNATURES = {
    "wg_version": (_i, []),
    "wg_last_error": (ctypes.c_char_p, []),
    "wg_device_count": (_i, []),
    "wg_sm_count": (_i, [_i]),
    "wg_decolor_u8": (_i, [_vp, _vp, _i64, _d, _d, _vp]),
    "wg_decolor_u8_exact": (_i, [_vp, _vp, _i64, _d, _d, _vp]),
    "wg_host_check_unit_f64": (_i, [_vp, _i64, ctypes.POINTER(ctypes.c_int)]),
    "wg_u8_exact_info": (_i, [_d, _d, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                              ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]),
    "wg_decolor_f32": (_i, [_vp, _vp, _i64, _f, _f, _vp]),
    "wg_decolor_f64": (_i, [_vp, _vp, _i64, _d, _d, _vp]),
    "wg_sigmoid_f64": (_i, [_vp, _vp, _i64, _d, _d, _vp]),
    "wg_sigmoid_f32": (_i, [_vp, _vp, _i64, _f, _f, _vp]),
    "wg_reinstate_f64": (_i, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "wg_tonemap_global_f64": (_i, [_vp, _vp, _vp, _i64, _d, _d, _d, _d, _vp]),
    "wg_decolor_tone_u8": (_i, [_vp, _vp, _vp, _i64, _f, _f, _f, _f, _vp]),
    "wg_decolor_tone_rgb_u8": (_i, [_vp, _vp, _vp, _vp, _i64, _d, _d, _d, _d, _vp]),
    "wg_host_decolor_tone_rgb_u8": (_i, [_vp, _vp, _vp, _vp, _i64, _d, _d, _d, _d, _i]),
    "wg_decolor_tone_f32": (_i, [_vp, _vp, _vp, _vp, _i64, _f, _f, _f, _f, _vp]),
    "wg_quantize_u8_f64": (_i, [_vp, _vp, _i64, _vp]),
    "wg_dequantize_u8_f64": (_i, [_vp, _vp, _i64, _vp]),
    "wg_hdr_scratch_bytes": (_sz, [_i64, _i64]),
    "wg_hdr_tonemap_u8": (_i, [_vp, _vp, _i64, _i64, _f, _f, _f, _f, _vp, _sz, _vp]),
    "wg_hdr_debug_trace": (_i64, [_vp]),
    "wg_ipc_alloc": (_i, [_sz, _i, _vp, _vp]),
    "wg_ipc_open": (_i, [_vp, _i, _vp]),
    "wg_ipc_close": (_i, [_vp]),
    "wg_ipc_free": (_i, [_vp, _i]),
    "wg_luma_f64": (_i, [_vp, _vp, _i64, _i, _vp]),
    "wg_lab_f64": (_i, [_vp, _vp, _i64, _vp]),
    "wg_luma_u8": (_i, [_vp, _vp, _i64, _i, _vp]),
    "wg_lhe_scratch_bytes": (_sz, [_i64, _i64, _i64, _i64, _i64, _i64]),
    "wg_local_lhe_f64": (_i, [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _d, _vp, _sz, _vp]),
    "wg_tonemap_local_f64": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _d, _d, _i64, _i64, _i64, _d, _vp, _sz,
                                  _vp]),
    "wg_decolor_tone_local_u8": (_i, [_vp, _vp, _vp, _i64, _i64, _i64, _d, _d, _i64, _i64, _i64, _d, _vp, _sz,
                                      _vp]),
    "wg_host_local_lhe_f64": (_i, [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _d, _i]),
    "wg_host_tonemap_local_f64": (_i, [_vp, _vp, _vp, _i64, _i64, _d, _d, _i64, _i64, _i64, _d, _i]),
    "wg_host_decolor_tone_local_u8": (_i, [_vp, _vp, _vp, _i64, _i64, _i64, _d, _d, _i64, _i64, _i64, _d, _i]),
    "wg_host_luma_rows_f64": (_i, [_vp, _vp, _i64, _i64, _i, _i64, _i64, _i]),
    "wg_host_lab_rows_f64": (_i, [_vp, _vp, _i64, _i64, _i64, _i64, _i]),
    "wg_host_luma_u8": (_i, [_vp, _vp, _i64, _i, _i]),
    "wg_host_decolor_rows_f64": (_i, [_vp, _vp, _i64, _i64, _d, _d, _i64, _i64, _i]),
    "wg_host_decolor_u8": (_i, [_vp, _vp, _i64, _d, _d, _i]),
    "wg_host_decolor_u8_exact": (_i, [_vp, _vp, _i64, _d, _d, _i]),
    "wg_host_decolor_f32": (_i, [_vp, _vp, _i64, _f, _f, _i]),
    "wg_host_decolor_tone_u8": (_i, [_vp, _vp, _vp, _i64, _f, _f, _f, _f, _i]),
    "wg_host_sigmoid_f64": (_i, [_vp, _vp, _i64, _d, _d, _i]),
    "wg_host_reinstate_f64": (_i, [_vp, _vp, _vp, _vp, _i64, _i]),
    "wg_host_tonemap_global_f64": (_i, [_vp, _vp, _vp, _i64, _d, _d, _d, _d, _i]),
    "wg_host_quantize_u8_f64": (_i, [_vp, _vp, _i64, _i]),
    "wg_host_dequantize_u8_f64": (_i, [_vp, _vp, _i64, _i]),
    "wg_host_hdr_tonemap_u8": (_i, [_vp, _vp, _i64, _i64, _f, _f, _f, _f, _i]),
    "wg_metric_scratch_bytes": (_sz, [_i64]),
    "wg_metric_hist_f64": (_i, [_vp, _vp, _i64, _vp, _i, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "wg_metric_counts_from_hist": (_i, [_vp, _i, _vp]),
    "wg_host_metric_counts_f64": (_i, [_vp, _vp, _i64, _vp, _i, _vp, _vp, _i64, _vp, _i]),
    "wg_pnm_probe": (_i, [ctypes.c_char_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                          ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_i64)]),
    "wg_pnm_read_batch": (_i, [ctypes.POINTER(ctypes.c_char_p), _i64, _vp, _i64, _i64, ctypes.c_int32,
                               ctypes.c_int32]),
    "wg_pnm_write_batch": (_i, [ctypes.POINTER(ctypes.c_char_p), _i64, _vp, _i64, _i64, ctypes.c_int32,
                                ctypes.c_int32]),
    "wg_synth_uniform_u8": (_i, [_vp, _i64, _i64, _u32, _i64, _vp]),
    "wg_synth_voronoi_u8": (_i, [_vp, _i64, ctypes.c_int32, ctypes.c_int32, _vp, _vp,
                                 ctypes.c_int32, _u32, _i64, _vp]),
    "wg_synth_blobs_f32": (_i, [_vp, _i64, ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32,
                                _vp, _f, _u32, _i64, _vp]),
    "wg_synth_hdr_f32": (_i, [_vp, _i64, _i64, _f, _f, _u32, _i64, _vp]),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load the library once and attach the C signatures."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ExtensionMissing(
                    f"{path} not found: the sm_100a library is not built "
                    "(python -c 'import __graft_entry__ as g; g.build()')")
            handle = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def available() -> bool:
    try:
        load()
    except (ExtensionMissing, OSError):
        return False
    return True


def last_error() -> str:
    return load().wg_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    """Raise the Python exception matching a C-ABI status code."""
    if status == 0:
        return
    msg = last_error() or f"status {status}"
    if status == WG_ECODEC:  # file errors carry the reference's message as is
        raise CodecError(msg)
    if status == WG_EIO:
        raise OSError(msg)
    if what:
        msg = f"{what}: {msg}"
    if status == ENODEV:
        raise CudaError(msg)
    if status < 0:
        raise ValueError(msg)
    raise CudaError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def device_count() -> int:
    return int(load().wg_device_count())
