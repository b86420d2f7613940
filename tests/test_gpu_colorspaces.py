"""GPU parity of the baseline colour-to-gray methods and CIELAB.

* BT.601 and HSV V (fp64 plugin rows and device batches): bit-identical to
  the reference's compiled backend (golden vectors from the reference).
* CIELAB (lab_lightness_rows, lab_rows): CUDA pow / cbrt vs glibc differ in
  the last ulp; bound 1e-12 absolute on L*, a*, b* (the reference's own
  backends agree only to 1e-9, test_backend.py:84-101).
* uint8 -> uint8 over all 2^24 colours: sha256 == reference for y, v and lab.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, rand_rgb

import paper_2108_13656_b200 as wg

pytestmark = pytest.mark.gpu

LAB_TOL = 1e-12
ROWS = {"y": "bt601_rows", "weighted": "bt601_rows", "v": "hsv_value_rows", "lab": "lab_lightness_rows"}


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "colorspaces.npz"))


@pytest.fixture(scope="module")
def kat():
    with open(os.path.join(GOLDEN, "colorspaces.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def cube():
    from oracle import oracle

    return oracle.color_cube_u8()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("tag", ["rgb", "edge"])
@pytest.mark.parametrize("method", ["y", "weighted", "v", "lab"])
def test_luminance_image_vs_reference(golden, tag, method):
    out = wg.luminance_image(wg.PlanarImage(golden[tag]), method=method).data
    want = golden[f"{tag}_{ROWS[method]}"]
    if method == "lab":
        assert np.abs(out - want).max() <= LAB_TOL
    else:
        np.testing.assert_array_equal(out, want)


@pytest.mark.parametrize("tag", ["rgb", "edge"])
def test_lab_image_vs_reference(golden, tag):
    out = wg.lab_image(wg.PlanarImage(golden[tag]))
    assert out.shape == golden[tag].shape
    assert np.abs(out - golden[f"{tag}_lab_rows"]).max() <= LAB_TOL


def test_methods_match_scalar_oracles(rng):
    """Port of the reference's TestImageDrivers.test_methods_match_scalar_oracles."""
    img = rand_rgb(rng, 6, 7)
    scalar = {"ours": wg.decolor_pixel, "y": wg.luma_weighted, "weighted": wg.luma_weighted,
              "v": wg.hsv_v, "lab": wg.lab_lightness}
    for method, fn in scalar.items():
        out = wg.luminance_image(img, method=method).data
        ref = np.array([[fn(tuple(img.data[y, x])) for x in range(img.width)] for y in range(img.height)])
        assert np.abs(out - ref).max() <= 1e-6, method
    lab = wg.lab_image(img)
    c = wg.rgb_to_lab(tuple(img.data[2, 3]))
    assert lab[2, 3] == pytest.approx([c.l_star, c.a_star, c.b_star], abs=1e-9)


def test_plugin_rows_partial_range(golden):
    """Row-range contract: only out[row0:row1] is written (_kernels.pyx:59-132)."""
    from paper_2108_13656_b200 import _kernels_cuda as k

    rgb = golden["rgb"]
    out = np.full(rgb.shape[:2], -7.0)
    k.hsv_value_rows(rgb, out, 5, 17)
    np.testing.assert_array_equal(out[5:17], golden["rgb_hsv_value_rows"][5:17])
    assert (out[:5] == -7.0).all() and (out[17:] == -7.0).all()
    lab = np.full(rgb.shape, -7.0)
    k.lab_rows(rgb, lab, 30, 37)
    assert np.abs(lab[30:] - golden["rgb_lab_rows"][30:]).max() <= LAB_TOL
    assert (lab[:30] == -7.0).all()
    k.bt601_rows(rgb, out, 0, 0)  # empty range is a no-op
    with pytest.raises(ValueError):
        k.bt601_rows(rgb, out, 3, 99)


@pytest.mark.parametrize("method", ["y", "v", "lab"])
def test_u8_cube_device_batch(kat, cube, method):
    import torch

    got = wg.luma(torch.from_numpy(cube).cuda(), method).cpu().numpy()
    assert sha(got) == kat[f"cube_{method}_u8_sha256"]


@pytest.mark.parametrize("method", ["y", "v", "lab"])
def test_u8_host_path_and_ragged_sizes(method):
    """luma_host (pipelined H2D/compute/D2H) == device batch, on odd sizes and unaligned views."""
    import torch

    from oracle import oracle

    rng = np.random.default_rng(5)
    for n in (0, 1, 3, 5, 4097, 1 << 20 | 7):
        rgb = rng.integers(0, 256, (n, 3), dtype=np.uint8)
        want = oracle.luma_u8(rgb, method)
        got_host = wg.luma_host(rgb, method)
        np.testing.assert_array_equal(got_host, want)
        if n:
            buf = torch.from_numpy(np.concatenate([np.zeros(1, np.uint8), rgb.ravel()])).cuda()
            view = buf[1:].view(n, 3)  # 1-byte offset -> scalar fallback path
            got_dev = wg.luma(view, method).cpu().numpy()
            np.testing.assert_array_equal(got_dev, got_host)


def test_f64_device_batch_vs_oracle(golden):
    import torch

    from oracle import oracle

    rgb = np.random.default_rng(9).random((3, 333, 517, 3))
    t = torch.from_numpy(rgb).cuda()
    for method in ("y", "v"):
        np.testing.assert_array_equal(wg.luma(t, method).cpu().numpy(), oracle.luma_f64(rgb, method))
    assert np.abs(wg.luma(t, "lab").cpu().numpy() - oracle.luma_f64(rgb, "lab")).max() <= LAB_TOL
    assert np.abs(wg.lab(t).cpu().numpy() - oracle.lab_f64(rgb)).max() <= LAB_TOL


def test_bad_method_raises():
    import torch

    with pytest.raises(ValueError):
        wg.luma(torch.zeros((2, 3), dtype=torch.uint8, device="cuda"), "nope")
    from paper_2108_13656_b200 import _lib

    with pytest.raises(ValueError):
        _lib.call("wg_luma_u8", None, None, 0, 7, None)


def test_run_benchmark_lab_vs_ours():
    """run_benchmark over both methods (test_bench.py:38-42 / test_acceptance.py:170-177 shape)."""
    rows = wg.run_benchmark(["ours", "lab", "y", "v"], 64, 48, repeats=5)
    assert [r.method for r in rows] == ["ours", "lab", "y", "v"]
    assert all(r.backend == "cuda" and r.per_pixel_ns > 0 for r in rows)
