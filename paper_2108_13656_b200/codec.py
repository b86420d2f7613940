"""Image codec: the reference's file API plus a uint8 batch path.

Drop-in for /root/reference/pkg/src/warmgray/codec.py:

* ``quantize_u8`` (floor(clip(v, 0, 1) * 255 + 0.5), round half up) and
  ``dequantize_u8`` (k / 255.0), codec.py:22-29 -- device kernels;
* ``load_image`` / ``save_image`` / ``CodecError`` (codec.py:85-140): binary
  PGM / PPM natively (header grammar and errors of the reference, parsed by
  the library, csrc/wg_io.cu), 8-bit PNG through Pillow as in the reference.

The reference turns every file into float64 (dequantize + clip + validation,
~16 ns/px) before any kernel runs. The batch path keeps bytes as uint8 from
the file to the device and back: ``read_pnm_batch`` reads many same-size
files into one (pinned) uint8 batch with one host thread per file,
``write_pnm_batch`` writes one back, and ``decolor_files`` chains them with
the pipelined device path (gray / global tone / local tone).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from ._lib import CodecError
from .backend import get_device
from .core import PlanarImage

__all__ = ["CodecError", "quantize_u8", "dequantize_u8", "load_image", "save_image", "load_u8", "save_u8",
           "read_pnm_batch", "write_pnm_batch", "decolor_files"]


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


def _threads(threads: int | None) -> int:
    return threads if threads else min(32, len(os.sched_getaffinity(0)))


def _paths(paths) -> ctypes.Array:
    enc = [os.fsencode(os.fspath(p)) for p in paths]
    return (ctypes.c_char_p * max(1, len(enc)))(*enc)


def _is_pnm(path: str) -> bool:
    with open(path, "rb") as f:
        head = f.read(2)
    return head[:1] == b"P" and head[1:2] in b"123456"  # (b"" in b"123456": a lone "P" is PNM too)


def pnm_info(path) -> tuple[int, int, int]:
    """(height, width, channels) of a binary PGM/PPM file."""
    w, h, c, off = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64()
    _lib.check(_lib.load().wg_pnm_probe(os.fsencode(os.fspath(path)), ctypes.byref(w), ctypes.byref(h),
                                        ctypes.byref(c), ctypes.byref(off)), "wg_pnm_probe")
    return h.value, w.value, c.value


def _load_png_u8(path: str) -> np.ndarray:
    from PIL import Image, UnidentifiedImageError

    try:
        with Image.open(path) as im:
            if im.format != "PNG":
                raise CodecError(f"{path}: unsupported format {im.format!r} (need PNG or binary PPM/PGM)")
            mode = im.mode
            if mode == "L":
                return np.asarray(im)
            if mode == "LA":
                return np.asarray(im.convert("L"))
            if mode in ("RGB", "RGBA", "P"):
                return np.asarray(im.convert("RGB"))
            raise CodecError(f"{path}: unsupported PNG mode {mode!r} (need 8-bit gray/RGB)")
    except UnidentifiedImageError:
        raise CodecError(f"{path}: not a decodable image") from None


def load_u8(path) -> np.ndarray:
    """Decode a PNG/PPM/PGM file to uint8 (H, W, 3) or (H, W), without the float64 detour."""
    path = os.fspath(path)
    if _is_pnm(path):
        h, w, c = pnm_info(path)
        out = np.empty((h, w, 3) if c == 3 else (h, w), dtype=np.uint8)
        _lib.check(_lib.load().wg_pnm_read_batch(_paths([path]), 1, out.ctypes.data, w, h, c, 1),
                   "wg_pnm_read_batch")
        return out
    return np.ascontiguousarray(_load_png_u8(path))


def load_image(path) -> PlanarImage:
    """Decode a PNG/PPM/PGM file into a PlanarImage (codec.py:85-95)."""
    return PlanarImage._from_kernel(dequantize_u8(load_u8(path)))


def save_u8(path, u8: np.ndarray) -> None:
    """Encode uint8 (H, W, 3) / (H, W) by extension: .png, .ppm (rgb only), .pgm (gray only)."""
    path = os.fspath(path)
    u8 = np.ascontiguousarray(u8, dtype=np.uint8)
    rgb = u8.ndim == 3
    ext = os.path.splitext(path)[1].lower()
    if ext == ".png":
        from PIL import Image

        Image.fromarray(u8, mode="RGB" if rgb else "L").save(path, format="PNG")
    elif ext in (".ppm", ".pgm"):
        if ext == ".ppm" and not rgb:
            raise CodecError("PPM stores rgb images; use .pgm or .png for luminance")
        if ext == ".pgm" and rgb:
            raise CodecError("PGM stores luminance images; use .ppm or .png for rgb")
        write_pnm_batch([path], u8[None])
    else:
        raise CodecError(f"unsupported output extension {ext!r} (use .png/.ppm/.pgm)")


def save_image(path, img: PlanarImage) -> None:
    """Encode to PNG/PPM/PGM chosen by file extension (codec.py:98-132)."""
    path = os.fspath(path)
    ext = os.path.splitext(path)[1].lower()
    if ext == ".ppm" and img.kind != "rgb":
        raise CodecError("PPM stores rgb images; use .pgm or .png for luminance")
    if ext == ".pgm" and img.kind != "luminance":
        raise CodecError("PGM stores luminance images; use .ppm or .png for rgb")
    if ext not in (".png", ".ppm", ".pgm"):
        raise CodecError(f"unsupported output extension {ext!r} (use .png/.ppm/.pgm)")
    save_u8(path, quantize_u8(img.data))


def _empty_batch(shape, pinned: bool) -> np.ndarray:
    if pinned:
        import torch

        # the ndarray's base is the tensor, which keeps the pinned allocation alive
        return torch.empty(shape, dtype=torch.uint8, pin_memory=True).numpy()
    return np.empty(shape, dtype=np.uint8)


def read_pnm_batch(paths, threads: int | None = None, pinned: bool = True, out=None) -> np.ndarray:
    """Read same-size binary PGM/PPM files into one uint8 batch (N, H, W[, 3]).

    The batch lives in pinned host memory by default (the device path copies
    it with DMA), or in ``out`` (C-contiguous uint8 of the batch's shape) when
    given; one host thread per file up to ``threads``.
    """
    paths = [os.fspath(p) for p in paths]
    if not paths:
        raise ValueError("read_pnm_batch needs at least one path")
    h, w, c = pnm_info(paths[0])
    shape = (len(paths), h, w, 3) if c == 3 else (len(paths), h, w)
    if out is None:
        out = _empty_batch(shape, pinned)
    elif out.shape != shape or out.dtype != np.uint8 or not out.flags["C_CONTIGUOUS"]:
        raise ValueError(f"out must be C-contiguous uint8 of shape {shape}")
    _lib.check(_lib.load().wg_pnm_read_batch(_paths(paths), len(paths), out.ctypes.data, w, h, c,
                                             _threads(threads)), "wg_pnm_read_batch")
    return out


def write_pnm_batch(paths, batch: np.ndarray, threads: int | None = None) -> None:
    """Write a uint8 batch (N, H, W) -> PGM or (N, H, W, 3) -> PPM, one file per image."""
    paths = [os.fspath(p) for p in paths]
    batch = np.ascontiguousarray(batch, dtype=np.uint8)
    if batch.ndim not in (3, 4) or (batch.ndim == 4 and batch.shape[-1] != 3):
        raise ValueError(f"expected (N, H, W) or (N, H, W, 3), got shape {batch.shape}")
    if len(paths) != batch.shape[0]:
        raise ValueError(f"{len(paths)} paths for {batch.shape[0]} images")
    c = 3 if batch.ndim == 4 else 1
    _lib.check(_lib.load().wg_pnm_write_batch(_paths(paths), len(paths), batch.ctypes.data, batch.shape[2],
                                              batch.shape[1], c, _threads(threads)), "wg_pnm_write_batch")


def _image_shape(path: str) -> tuple:
    """(H, W, 3) or (H, W) of a PNM or PNG file, from its header."""
    if _is_pnm(path):
        h, w, c = pnm_info(path)
        return (h, w, 3) if c == 3 else (h, w)
    from PIL import Image, UnidentifiedImageError

    try:
        with Image.open(path) as im:
            if im.format != "PNG":
                raise CodecError(f"{path}: unsupported format {im.format!r} (need PNG or binary PPM/PGM)")
            return (im.size[1], im.size[0]) if im.mode in ("L", "LA") else (im.size[1], im.size[0], 3)
    except UnidentifiedImageError:
        raise CodecError(f"{path}: not a decodable image") from None


def read_batch(paths, threads: int | None = None, out=None, pinned: bool = True) -> np.ndarray:
    """Read same-size PNG / PPM / PGM files into one uint8 batch (pinned by default).

    All-PNM batches go through the native reader (:func:`read_pnm_batch`);
    otherwise each file is decoded (Pillow for PNG, as in the reference) on a
    thread pool straight into the batch -- the decoders release the GIL.
    """
    paths = [os.fspath(p) for p in paths]
    if not paths:
        raise ValueError("read_batch needs at least one path")
    if all(_is_pnm(p) for p in paths):
        return read_pnm_batch(paths, threads=threads, pinned=pinned, out=out)
    shape = (len(paths), *_image_shape(paths[0]))
    if out is None:
        out = _empty_batch(shape, pinned)
    elif out.shape != shape or out.dtype != np.uint8 or not out.flags["C_CONTIGUOUS"]:
        raise ValueError(f"out must be C-contiguous uint8 of shape {shape}")

    def one(k):
        img = load_u8(paths[k])
        if img.shape != shape[1:]:
            raise CodecError(f"{paths[k]}: shape {img.shape} differs from the batch's {shape[1:]}")
        out[k] = img

    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(_threads(threads), len(paths))) as pool:
        list(pool.map(one, range(len(paths))))
    return out


def write_batch(paths, batch: np.ndarray, threads: int | None = None) -> None:
    """Write a uint8 batch, one file per image, format by extension (.png / .ppm / .pgm).

    All-PNM targets go through the native writer (:func:`write_pnm_batch`);
    otherwise each file is encoded on a thread pool.
    """
    paths = [os.fspath(p) for p in paths]
    if len(paths) != len(batch):
        raise ValueError(f"{len(paths)} paths for {len(batch)} images")
    if all(os.path.splitext(p)[1].lower() in (".ppm", ".pgm") for p in paths):
        write_pnm_batch(paths, batch, threads=threads)
        return
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(_threads(threads), len(paths))) as pool:
        list(pool.map(lambda k: save_u8(paths[k], batch[k]), range(len(paths))))


def decolor_files(src_paths, dst_paths, mode: str = "gray", params=None, curve=None, grid=None,
                  batch: int = 32, threads: int | None = None, device: int | None = None,
                  exact: bool = False) -> int:
    """uint8 files in, uint8 gray files out, bytes never leave uint8.

    ``mode``: "gray" (decolor), "global" (decolor + sigmoid) or "local"
    (decolor + local tone map); outputs are bit-identical to
    quantize_u8 of the reference's fp64 chain for "local" (and for "gray" /
    "global" with ``exact=True``), else within the north-star bound (+-1 on
    <= 0.01% of pixels).
    Same-size RGB inputs (binary PPM through the native reader, PNG through
    Pillow on a thread pool) go in groups of ``batch``; outputs are written by
    extension (.pgm natively, .png through Pillow). Reading batch i + 1, the
    device pass of batch i and writing batch i - 1 overlap (pinned double
    buffers).
    Returns the number of files.
    """
    from . import batch as _batch
    from .core import DEFAULT_PARAMS
    from .tonemap import SigmoidCurve

    src_paths, dst_paths = list(src_paths), list(dst_paths)
    if len(src_paths) != len(dst_paths):
        raise ValueError("src_paths and dst_paths differ in length")
    params = params or DEFAULT_PARAMS
    if mode not in ("gray", "global", "local"):
        raise ValueError(f"unknown mode {mode!r} (use 'gray', 'global' or 'local')")
    groups = [(src_paths[k:k + batch], dst_paths[k:k + batch]) for k in range(0, len(src_paths), batch)]
    # Three-stage pipeline over the batches: the native reader fills pinned
    # buffer (i + 1) % 2 and the native writer drains output buffer (i - 1) % 2
    # on two worker threads (the C calls release the GIL) while this thread
    # runs batch i through the device.
    bufs = {}

    def buf(slot, kind, shape):
        b = bufs.get((slot, kind))
        if b is None or b.shape != shape:
            b = bufs[(slot, kind)] = _empty_batch(shape, True)
        return b

    def read(i):
        paths = [os.fspath(p) for p in groups[i][0]]
        shape = (len(paths), *_image_shape(paths[0]))
        return read_batch(paths, threads=threads, out=buf(i % 2, "in", shape))

    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=2) as pool:
        nxt = pool.submit(read, 0) if groups else None
        writes = [None, None]
        for i in range(len(groups)):
            rgb = nxt.result()
            if rgb.ndim != 4:
                raise CodecError(f"{groups[i][0][0]}: decolor_files needs rgb (P6) inputs")
            if i + 1 < len(groups):
                nxt = pool.submit(read, i + 1)  # its input slot's last reader (batch i - 1) is done
            if writes[i % 2] is not None:
                writes[i % 2].result()  # output slot free again
            dst = buf(i % 2, "out", rgb.shape[:-1])
            if mode == "gray":
                out = _batch.decolor_host(rgb, params, out=dst, device=device, exact=exact)
            elif mode == "global":
                out = _batch.decolor_tone_host(rgb, curve or SigmoidCurve(), params, device=device, out=dst,
                                               exact=exact)
            else:
                out = _batch.decolor_tone_local_host(rgb, grid, params, device=device, out=dst)
            writes[i % 2] = pool.submit(write_batch, groups[i][1], out, threads)
        for f in writes:
            if f is not None:
                f.result()
    return len(src_paths)
