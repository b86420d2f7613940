"""GPU parity of the local tone map.

* fp64 drop-in (apply_local_lhe, tonemap_image(mode="local")): bit-identical
  to the reference on its own outputs (tests/golden/lhe.npz) and to the oracle
  on random grids.
* Fused uint8 batch (decolor_tone_local): bit-identical to
  quantize_u8 of the fp64 reference chain -- on the reference's own u8
  outputs, on full-HD images and on all 2^24 colours in one 4096^2 image.
* The error bound the u8 fast route relies on (fp32 gray within 2.5e-7 of the
  fp64 gray for every byte colour) is checked exhaustively.
"""

import os

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import GOLDEN

import paper_2108_13656_b200 as wg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "lhe.npz"))


def lhe(data, tw, th, nb=256, s=0.7):
    return wg.apply_local_lhe(wg.PlanarImage(data), wg.LocalHistogramGrid(int(tw), int(th), int(nb), float(s))).data


# ---------------------------------------------------------------- fp64 drop-in
def test_cases_bit_identical_to_reference(golden):
    for i, (h, w, tw, th, nb, s) in enumerate(golden["cases"]):
        out = lhe(golden[f"in{i}"], tw, th, nb, s)
        assert out.tobytes() == golden[f"out{i}"].tobytes(), (h, w, tw, th, nb, s)


@pytest.mark.parametrize("name", ["halves", "ramp", "const"])
def test_structured_bit_identical_to_reference(golden, name):
    tw, th, nb, s = golden[f"{name}_grid"]
    out = lhe(golden[f"{name}_in"], tw, th, nb, s)
    assert out.tobytes() == golden[f"{name}_out"].tobytes()


def test_reference_properties(golden, rng):
    """The reference's TestLocalLhe properties, on the product."""
    img = rng.random((16, 16))
    assert lhe(img, 4, 4, s=0.0).tobytes() == img.tobytes()              # strength 0: identity
    const = np.full((12, 10), 0.37)
    assert np.array_equal(lhe(const, 4, 4, s=1.0), const)               # constant unchanged
    assert lhe(rng.random((6, 6)), 10_000, 10_000, s=1.0).shape == (6, 6)  # oversize tiles clamp
    out = lhe(rng.random((20, 24)), 6, 5, s=1.0)
    assert out.min() >= 0.0 and out.max() <= 1.0
    halves = golden["halves_in"]
    out = lhe(halves, 4, 8, 16, 1.0)
    assert out[:, :4].std() > halves[:, :4].std() and out[:, 4:].std() > halves[:, 4:].std()
    smooth = lhe(golden["ramp_in"], 8, 8, s=1.0)
    assert np.abs(np.diff(smooth, axis=1)).max() <= 0.15               # blended curves, no seams
    base = wg.apply_local_lhe(wg.PlanarImage(img), wg.LocalHistogramGrid(6, 7, strength=0.9), threads=1)
    for t in (2, 5, 8):
        again = wg.apply_local_lhe(wg.PlanarImage(img), wg.LocalHistogramGrid(6, 7, strength=0.9), threads=t)
        assert again.data.tobytes() == base.data.tobytes()


def test_tonemap_image_local_bit_identical(golden):
    rgb = wg.PlanarImage(golden["tm_rgb"])
    r1, l1 = wg.tonemap_image(rgb, mode="local")
    assert l1.data.tobytes() == golden["tm_l_out"].tobytes()
    assert r1.data.tobytes() == golden["tm_rgb_out"].tobytes()
    r2, l2 = wg.tonemap_image(rgb, mode="local", params=wg.DecolorParams(0.7, 0.9),
                              grid=wg.LocalHistogramGrid(7, 5, 64, 0.9))
    assert l2.data.tobytes() == golden["tm_l_out2"].tobytes()
    assert r2.data.tobytes() == golden["tm_rgb_out2"].tobytes()


@settings(max_examples=40, deadline=None)
@given(h=st.integers(1, 70), w=st.integers(1, 70), tw=st.integers(1, 80), th=st.integers(1, 80),
       nb=st.sampled_from([2, 3, 16, 255, 256, 1000]), s=st.floats(0.0, 1.0), seed=st.integers(0, 2**31))
def test_random_grids_vs_oracle(h, w, tw, th, nb, s, seed):
    from oracle import oracle

    d = np.random.default_rng(seed).random((h, w))
    if seed % 3 == 0:
        d = np.round(d * 255) / 255
    assert lhe(d, tw, th, nb, s).tobytes() == oracle.local_lhe_f64(d, tw, th, nb, s).tobytes()


def test_device_batch_f64_vs_oracle():
    import torch

    from oracle import oracle
    from paper_2108_13656_b200 import _lib

    lum = np.random.default_rng(3).random((5, 270, 480))
    t = torch.from_numpy(lum).cuda()
    out = torch.empty_like(t)
    need = int(_lib.load().wg_lhe_scratch_bytes(5, 270, 480, 60, 34, 256))
    scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
    _lib.call("wg_local_lhe_f64", t.data_ptr(), out.data_ptr(), 5, 270, 480, 60, 34, 256, 0.7,
              scratch.data_ptr(), need, torch.cuda.current_stream().cuda_stream)
    assert out.cpu().numpy().tobytes() == oracle.local_lhe_f64(lum, 60, 34, 256, 0.7, threads=5).tobytes()
    with pytest.raises(ValueError):  # scratch too small
        _lib.call("wg_local_lhe_f64", t.data_ptr(), out.data_ptr(), 5, 270, 480, 60, 34, 256, 0.7,
                  scratch.data_ptr(), need - 1, torch.cuda.current_stream().cuda_stream)
    with pytest.raises(ValueError):  # bins < 2
        _lib.call("wg_local_lhe_f64", t.data_ptr(), out.data_ptr(), 5, 270, 480, 60, 34, 1, 0.7,
                  scratch.data_ptr(), need, torch.cuda.current_stream().cuda_stream)


# ---------------------------------------------------------------- fused uint8 batch
def test_u8_fast_route_error_bound():
    """fp32 gray of every byte colour within 2.5e-7 of the fp64 reference (the margin the u8 route assumes)."""
    import torch

    from oracle import oracle

    cube = oracle.color_cube_u8()
    f = (cube.astype(np.float32) * np.float32(1.0 / 255.0)).astype(np.float32)
    got = wg.decolor(torch.from_numpy(f).cuda()).cpu().numpy().astype(np.float64)
    want = oracle.decolor_f64(cube.astype(np.float64) / 255.0, threads=oracle.default_threads())
    assert np.abs(got - want).max() < 2.5e-7


def test_u8_golden_bit_identical(golden):
    import torch

    rgb = golden["u8_rgb"]
    toned, gray = wg.decolor_tone_local(torch.from_numpy(rgb).cuda(), return_gray=True)
    np.testing.assert_array_equal(toned.cpu().numpy(), golden["u8_toned"])
    np.testing.assert_array_equal(gray.cpu().numpy(), golden["u8_gray"])
    t2, g2 = wg.decolor_tone_local_host(rgb, return_gray=True)
    np.testing.assert_array_equal(t2, golden["u8_toned"])
    np.testing.assert_array_equal(g2, golden["u8_gray"])


@pytest.mark.parametrize("shape,grid", [((2, 1080, 1920), None), ((3, 97, 131), (17, 13, 64, 0.9)),
                                        ((1, 64, 48), (1, 1, 256, 1.0)), ((4, 33, 35), (5, 7, 1000, 0.3)),
                                        # nb = 512: largest bin count the plane word carries; 513: fp32 plane
                                        ((2, 50, 70), (9, 11, 512, 0.8)), ((2, 50, 70), (9, 11, 513, 0.8))])
def test_u8_batch_vs_oracle(shape, grid):
    import torch

    from oracle import oracle

    n, h, w = shape
    rng = np.random.default_rng(h * w)
    rgb = rng.integers(0, 256, (n, h, w, 3), dtype=np.uint8)
    rgb[0, : h // 3] = rgb[0, : h // 3] // 16 * 16  # posterised band: many exact bin edges
    g = wg.LocalHistogramGrid(*grid) if grid else wg.LocalHistogramGrid.for_image(w, h)
    toned = wg.decolor_tone_local(torch.from_numpy(rgb).cuda(), grid=g).cpu().numpy()
    want = oracle.tone_local_u8(rgb, g.tile_w, g.tile_h, g.bins, g.strength, threads=n)
    np.testing.assert_array_equal(toned, want)


def test_u8_all_colours_one_image():
    """All 2^24 colours in one 4096^2 image (default 8x8 grid): every margin decision exercised."""
    import torch

    from oracle import oracle

    cube = oracle.color_cube_u8()
    g = wg.LocalHistogramGrid.for_image(4096, 4096)
    toned, gray = wg.decolor_tone_local(torch.from_numpy(cube).cuda(), return_gray=True)
    want_t, want_g = oracle.tone_local_u8(cube, g.tile_w, g.tile_h, g.bins, g.strength, with_gray=True)
    np.testing.assert_array_equal(gray.cpu().numpy(), want_g)
    np.testing.assert_array_equal(toned.cpu().numpy(), want_t)


def test_u8_empty_and_errors():
    import torch

    out = wg.decolor_tone_local(torch.zeros((0, 4, 4, 3), dtype=torch.uint8, device="cuda"),
                                grid=wg.LocalHistogramGrid(2, 2))
    assert out.shape == (0, 4, 4)
    from types import SimpleNamespace

    with pytest.raises(ValueError):  # the C ABI validates beta itself (core.py:33-51)
        wg.decolor_tone_local(torch.zeros((4, 4, 3), dtype=torch.uint8, device="cuda"),
                              params=SimpleNamespace(beta_r=0.4, beta_k=0.8))
