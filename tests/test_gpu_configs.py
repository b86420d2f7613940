"""SURVEY.md 8(d) parity protocol on the bench's own inputs (BASELINE configs).

The oracle runs on the identical input bytes (copied D2H). Coverage: all 64
images of C2, all 32 of C4, and for C5 the first and last image of each GPU
shard at 8 GPUs (16 images of 7680x4320); C1 and >= 16 images of C3 are in
test_gpu_u8.py, the exhaustive colour cube for decolor and decolor + sigmoid
too. Criteria: uint8 identical except +-1 on <= 0.01% of pixels, fp32
max-abs <= 1e-6. Input sha256s and seeds are printed (pytest -s) for the log.
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import F32_TOL, U8_MAX_FRAC, u8_mismatch

pytestmark = pytest.mark.gpu


def _sha(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]


def test_c2_all_images():
    import torch

    import paper_2108_13656_b200 as wg
    from oracle import oracle
    from paper_2108_13656_b200 import synth

    wl = synth.WORKLOADS["C2"]
    worst = 0.0
    for i0 in range(0, wl.n_images, 8):
        rgb = torch.empty((8, wl.height, wl.width, 3), dtype=torch.float32, device="cuda")
        synth.fill_blobs_f32(rgb, seed=0, first_image=i0)  # == synth.make_batch(C2, seed=0) images i0..i0+7
        got = wg.decolor(rgb).cpu().numpy().astype(np.float64)
        err = float(np.abs(got - oracle.decolor_f32in(rgb.cpu().numpy(), threads=oracle.default_threads())).max())
        print(f"C2 seed 0 images {i0}..{i0 + 7} sha {_sha(rgb)} max abs err {err:.3e}")
        worst = max(worst, err)
    assert worst <= F32_TOL


def test_c4_all_images():
    import torch

    import paper_2108_13656_b200 as wg
    from oracle import oracle
    from paper_2108_13656_b200 import synth

    wl = synth.WORKLOADS["C4"]
    bad = total = 0
    for i0 in range(0, wl.n_images, 4):
        rgb = torch.empty((4, wl.height, wl.width, 3), dtype=torch.float32, device="cuda")
        synth.fill_hdr_f32(rgb, seed=0, first_image=i0)
        got = wg.hdr_tonemap(rgb).cpu().numpy()
        want = oracle.hdr_u8(rgb.cpu().numpy(), threads=oracle.default_threads())
        mx, frac = u8_mismatch(got, want)
        print(f"C4 seed 0 images {i0}..{i0 + 3} sha {_sha(rgb)} max {mx} frac {frac:.2e}")
        assert mx <= 1
        bad += int(round(frac * want.size))
        total += want.size
    assert bad <= U8_MAX_FRAC * total


def test_c4_full_batch_scale_invariance():
    """A size-independent property at the full C4 size (32 x 2048^2): the HDR
    adapter depends on radiance only through g / gmin, and the fp32 gray is
    exactly homogeneous under power-of-two scales (every rounding scales with
    the operands; the roots see powers of four), so x * 4 and x / 8 must give
    the very same bytes -- on the tensor-memory kernel and the grouped schedule."""
    import torch

    import paper_2108_13656_b200 as wg
    from paper_2108_13656_b200 import synth

    wl = synth.WORKLOADS["C4"]
    rgb = torch.empty((wl.n_images, wl.height, wl.width, 3), dtype=torch.float32, device="cuda")
    synth.fill_hdr_f32(rgb, seed=0, first_image=0)
    base = wg.hdr_tonemap(rgb)
    assert torch.equal(wg.hdr_tonemap(rgb * 4.0), base)
    assert torch.equal(wg.hdr_tonemap(rgb * 0.125), base)
    os.environ["WG_HDR_SCHEDULE"] = "grouped"
    try:
        assert torch.equal(wg.hdr_tonemap(rgb * 4.0), base)
    finally:
        del os.environ["WG_HDR_SCHEDULE"]


def test_c5_shard_edges():
    import torch

    import paper_2108_13656_b200 as wg
    from oracle import oracle
    from paper_2108_13656_b200 import synth

    wl = synth.WORKLOADS["C5"]
    per = wl.n_images // 8
    edges = sorted({g * per for g in range(8)} | {g * per + per - 1 for g in range(8)})
    assert len(edges) == 16
    rgb = torch.empty((1, wl.height, wl.width, 3), dtype=torch.uint8, device="cuda")
    bad = total = 0
    for k, idx in enumerate(edges):
        synth.fill_uniform_u8(rgb, seed=0, first_image=idx)  # bench: make_batch(C5, seed=0, first_image=rank*n)
        host = rgb.cpu().numpy()
        if k in (0, len(edges) - 1):  # the device generator is the oracle's counter hash
            np.testing.assert_array_equal(host, oracle.synth_uniform_u8(1, wl.height, wl.width, 0, idx))
        got = wg.decolor(rgb).cpu().numpy()
        want = oracle.decolor_u8(host, threads=oracle.default_threads())
        mx, frac = u8_mismatch(got, want)
        print(f"C5 seed 0 image {idx} sha {_sha(rgb)} max {mx} frac {frac:.2e}")
        assert mx <= 1
        bad += int(round(frac * want.size))
        total += want.size
        if k == 0:
            np.testing.assert_array_equal(wg.decolor(rgb, exact=True).cpu().numpy(), want)
    assert bad <= U8_MAX_FRAC * total


def test_run_on_devices_every_visible_gpu():
    """sharder.run_on_devices (one process, one host thread per device) over every
    visible GPU gives the bytes of the single-device call and meets the bar
    against the oracle; with one GPU the shards all land on device 0 (the
    multi-device fan-out is then exercised with repeated ordinals)."""
    import torch

    import paper_2108_13656_b200 as wg
    from oracle import oracle
    from paper_2108_13656_b200 import sharder

    ndev = torch.cuda.device_count()
    batch = oracle.synth_uniform_u8(6, 64, 96, seed=3)
    whole = wg.decolor_host(batch, device=0)
    for devices in (list(range(ndev)), [0] * 3, list(range(ndev)) * 2):
        got = sharder.run_on_devices(lambda shard, d: wg.decolor_host(shard, device=d), batch, devices)
        assert np.array_equal(got, whole), devices
    mx, frac = u8_mismatch(whole, oracle.decolor_u8(batch))
    assert mx <= 1 and frac <= U8_MAX_FRAC
    print(f"run_on_devices over {ndev} visible GPU(s): identical to the single-device call")
