"""Seeded synthetic workloads of BASELINE.json (SURVEY.md 8 d), generated on the GPU.

The reference benchmarks on ``default_rng(seed).random((H, W, 3))``
(bench.py:72-73) and the paper on photo datasets that are not available
here; BASELINE.json instead names five synthetic configurations, which are
reproduced by seeded generators:

  C1  1 x 512x512 u8, ``default_rng(0).integers(0, 256, ...)`` (host, as specified)
  C2  64 x 1080x1920 f32: mid-gray base + 32 Gaussian colour blobs + U(-0.02, 0.02) noise
  C3  256 x 2160x3840 u8: 200-cell Voronoi (HSV colours, V >= 0.2) + integer noise -4..4
  C4  32 x 2048x2048 f32 HDR radiance: luminance log-uniform in [1e-3, 1e4]
  C5  1024 x 4320x7680 u8 i.i.d. uniform bytes (counter hash; sharded by image)

Per-image tables (Voronoi seeds / colours, blob parameters) come from
``np.random.default_rng([seed, image_index])`` so any image of any shard can
be regenerated independently; per-pixel randomness comes from a counter hash
of (seed, image, index), so the device generators are deterministic and
GPU-count invariant.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class Workload:
    name: str
    dtype: str        # input dtype: "uint8" | "float32"
    output: str       # "gray_u8" | "gray_f32" | "hdr_u8"
    n_images: int
    height: int
    width: int

    @property
    def pix_per_image(self) -> int:
        return self.height * self.width

    @property
    def pixels(self) -> int:
        return self.n_images * self.pix_per_image

    @property
    def in_bytes_per_px(self) -> int:
        return 3 if self.dtype == "uint8" else 12

    @property
    def out_bytes_per_px(self) -> int:
        return 4 if self.output == "gray_f32" else 1

    @property
    def bytes_per_px(self) -> int:
        """Algorithmic (compulsory) HBM bytes per pixel: read input once, write output once."""
        return self.in_bytes_per_px + self.out_bytes_per_px


WORKLOADS = {
    "C1": Workload("C1", "uint8", "gray_u8", 1, 512, 512),
    "C2": Workload("C2", "float32", "gray_f32", 64, 1080, 1920),
    "C3": Workload("C3", "uint8", "gray_u8", 256, 2160, 3840),
    "C4": Workload("C4", "float32", "hdr_u8", 32, 2048, 2048),
    "C5": Workload("C5", "uint8", "gray_u8", 1024, 4320, 7680),
}

# per-GPU size sweep of config C5 at ~2^32 pixels per GPU (SURVEY.md 8 d)
SIZE_SWEEP = [(256, 256, 65536), (512, 512, 16384), (1024, 1024, 4096), (1080, 1920, 2071),
              (2048, 2048, 1024), (2160, 3840, 518), (4320, 7680, 129)]


def hsv_to_rgb(h, s, v):
    """Vectorised HSV -> RGB in [0, 1] (standard hexcone model)."""
    h = np.asarray(h, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    i = np.floor(h * 6.0)
    f = h * 6.0 - i
    i = i.astype(np.int64) % 6
    p = v * (1.0 - s)
    q = v * (1.0 - s * f)
    t = v * (1.0 - s * (1.0 - f))
    r = np.choose(i, [v, q, p, p, t, v])
    g = np.choose(i, [t, v, v, q, p, p])
    b = np.choose(i, [p, p, t, v, v, q])
    return np.stack([r, g, b], axis=-1)


def voronoi_tables(n_images: int, height: int, width: int, n_seeds: int = 200, seed: int = 0,
                   first_image: int = 0):
    """Per-image Voronoi seed points (int32 x, y) and u8 cell colours (C3)."""
    xy = np.empty((n_images, n_seeds, 2), dtype=np.int32)
    col = np.empty((n_images, n_seeds, 3), dtype=np.uint8)
    for i in range(n_images):
        rng = np.random.default_rng([seed, first_image + i])
        xy[i, :, 0] = rng.integers(0, width, n_seeds)
        xy[i, :, 1] = rng.integers(0, height, n_seeds)
        hue, sat, val = rng.random(n_seeds), rng.random(n_seeds), rng.uniform(0.2, 1.0, n_seeds)
        rgb = hsv_to_rgb(hue, sat, val)
        col[i] = np.floor(np.clip(rgb, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    return xy, col


def blob_tables(n_images: int, height: int, width: int, n_blobs: int = 32, seed: int = 0,
                first_image: int = 0):
    """Per-image blob table (n, n_blobs, 8) {cx, cy, 1/(2 sigma^2), amp, r, g, b, 0} and base (C2)."""
    tab = np.zeros((n_images, n_blobs, 8), dtype=np.float32)
    base = np.empty(n_images, dtype=np.float32)
    for i in range(n_images):
        rng = np.random.default_rng([seed, 7919, first_image + i])
        base[i] = rng.uniform(0.35, 0.65)
        sigma = rng.uniform(20.0, 200.0, n_blobs)
        tab[i, :, 0] = rng.uniform(0, width, n_blobs)
        tab[i, :, 1] = rng.uniform(0, height, n_blobs)
        tab[i, :, 2] = 1.0 / (2.0 * sigma * sigma)
        tab[i, :, 3] = rng.uniform(0.3, 0.9, n_blobs)
        tab[i, :, 4:7] = hsv_to_rgb(rng.random(n_blobs), np.ones(n_blobs), np.ones(n_blobs))
    return tab, base


def c1_image() -> np.ndarray:
    """Config C1 exactly as BASELINE.json states it (host RNG)."""
    return np.random.default_rng(0).integers(0, 256, (512, 512, 3), dtype=np.uint8)


# ---------------------------------------------------------------- device generators (torch tensors)

def _stream(t):
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream


def fill_uniform_u8(out, seed: int = 0, first_image: int = 0) -> None:
    """C5-style i.i.d. bytes into a contiguous (N, H, W, 3) uint8 CUDA tensor."""
    n = out.shape[0]
    per = out[0].numel() if n else 0
    _lib.call("wg_synth_uniform_u8", out.data_ptr(), n, per, seed, first_image, _stream(out))


def fill_voronoi_u8(out, seed: int = 0, first_image: int = 0, n_seeds: int = 200) -> None:
    """C3-style Voronoi images into a contiguous (N, H, W, 3) uint8 CUDA tensor."""
    import torch

    n, h, w = out.shape[0], out.shape[1], out.shape[2]
    step = 4096  # table upload granularity
    for i0 in range(0, n, step):
        m = min(step, n - i0)
        xy, col = voronoi_tables(m, h, w, n_seeds, seed, first_image + i0)
        dxy = torch.from_numpy(xy).to(out.device)
        dcol = torch.from_numpy(col).to(out.device)
        _lib.call("wg_synth_voronoi_u8", out[i0].data_ptr(), m, w, h, dxy.data_ptr(),
                  dcol.data_ptr(), n_seeds, seed, first_image + i0, _stream(out))
        torch.cuda.current_stream(out.device).synchronize()


def fill_blobs_f32(out, seed: int = 0, first_image: int = 0, n_blobs: int = 32,
                   noise: float = 0.02) -> None:
    """C2-style blob images into a contiguous (N, H, W, 3) float32 CUDA tensor."""
    import torch

    n, h, w = out.shape[0], out.shape[1], out.shape[2]
    tab, base = blob_tables(n, h, w, n_blobs, seed, first_image)
    dtab = torch.from_numpy(tab).to(out.device)
    dbase = torch.from_numpy(base).to(out.device)
    _lib.call("wg_synth_blobs_f32", out.data_ptr(), n, w, h, dtab.data_ptr(), n_blobs,
              dbase.data_ptr(), noise, seed, first_image, _stream(out))
    torch.cuda.current_stream(out.device).synchronize()


def fill_hdr_f32(out, seed: int = 0, first_image: int = 0, lum_lo: float = 1e-3,
                 lum_hi: float = 1e4) -> None:
    """C4-style HDR radiance into a contiguous (N, H, W, 3) float32 CUDA tensor."""
    n = out.shape[0]
    per = out[0].numel() // 3 if n else 0
    _lib.call("wg_synth_hdr_f32", out.data_ptr(), n, per, lum_lo, lum_hi, seed, first_image,
              _stream(out))


def make_batch(workload: Workload, device, n_images: int | None = None, seed: int = 0,
               first_image: int = 0):
    """Allocate and fill the input batch of ``workload`` on ``device``."""
    import torch

    n = workload.n_images if n_images is None else n_images
    shape = (n, workload.height, workload.width, 3)
    if workload.name == "C1":
        t = torch.from_numpy(np.broadcast_to(c1_image(), shape).copy()).to(device)
        return t
    dtype = torch.uint8 if workload.dtype == "uint8" else torch.float32
    t = torch.empty(shape, dtype=dtype, device=device)
    if workload.name == "C2":
        fill_blobs_f32(t, seed, first_image)
    elif workload.name == "C3":
        fill_voronoi_u8(t, seed, first_image)
    elif workload.name == "C4":
        fill_hdr_f32(t, seed, first_image)
    else:
        fill_uniform_u8(t, seed, first_image)
    return t
