"""CPU-side behaviour of the drop-in API (no GPU needed).

Ports the reference's host-logic tests (pkg/tests/test_core.py:34-159,
test_backend.py:27-60, test_tonemap.py:106-116,146-153) to this package:
parameter / container validation, the scalar model, backend registry,
thread resolution, run_rows, and that image entry points refuse to run
anywhere but the GPU.
"""

import math
import os

import numpy as np
import pytest
from hypothesis import assume, given
from hypothesis import strategies as st

import paper_2108_13656_b200 as wg
from paper_2108_13656_b200 import backend
from conftest import GOLDEN, rand_rgb

INV_SQRT3 = 1.0 / math.sqrt(3.0)
channels = st.floats(0.0, 1.0, allow_nan=False, allow_infinity=False, width=64)
pixels = st.tuples(channels, channels, channels)
betas = st.floats(0.5, 1.0, exclude_min=True, exclude_max=True, width=64)
params_st = st.builds(wg.DecolorParams, beta_r=betas, beta_k=betas)


class TestScalarModel:
    def test_fixtures(self):
        assert wg.white_luminance((1, 1, 1)) == pytest.approx(1.0, abs=1e-12)
        assert wg.white_luminance((0, 0, 0)) == 0.0
        assert wg.white_luminance((0, 0, 1)) == pytest.approx(INV_SQRT3, abs=1e-5)
        assert wg.blue_luminance((0.3, 0.9, 0.4)) == 0.4
        assert wg.red_green_luminance((1, 0, 0)) == pytest.approx(math.sqrt(0.55), abs=1e-5)
        assert wg.red_green_luminance((0, 1, 0)) == pytest.approx(math.sqrt(0.45), abs=1e-5)
        assert wg.warm_luminance((1, 0, 0)) == pytest.approx(math.sqrt(0.55), abs=1e-5)
        assert wg.warm_luminance((0, 1, 0)) == pytest.approx(INV_SQRT3, abs=1e-5)
        assert wg.warm_luminance((0, 0, 0)) == 0.0
        assert wg.cool_luminance((0, 0, 1)) == pytest.approx(INV_SQRT3, abs=1e-5)
        assert wg.cool_luminance((0, 1, 0)) == 0.0
        assert wg.decolor_pixel((1, 0, 0)) == pytest.approx(math.sqrt(0.44), abs=1e-5)
        assert wg.decolor_pixel((0, 0, 1)) == pytest.approx(INV_SQRT3, abs=1e-5)
        assert wg.decolor_pixel((0, 0, 0)) == 0.0

    def test_matches_reference_kats(self):
        import json

        with open(os.path.join(GOLDEN, "kat.json")) as f:
            kat = json.load(f)
        for name in ("decolor_pixel", "white_luminance", "red_green_luminance", "warm_luminance",
                     "cool_luminance"):
            fn = getattr(wg, name)
            for px, want in kat[name]:
                assert fn(tuple(px)) == pytest.approx(want, abs=1e-15), (name, px)
        for px, want in kat["custom_params"]:
            assert wg.decolor_pixel(tuple(px), wg.DecolorParams(0.9, 0.6)) == pytest.approx(want, abs=1e-15)

    @given(v=channels, p=params_st)
    def test_gray_axis_fixpoint(self, v, p):
        assert abs(wg.decolor_pixel((v, v, v), p) - v) <= 1e-9

    @given(pix=pixels, s=channels, p=params_st)
    def test_positive_homogeneity(self, pix, s, p):
        scaled = tuple(s * c for c in pix)
        assert abs(wg.decolor_pixel(scaled, p) - s * wg.decolor_pixel(pix, p)) <= 1e-7

    @given(pix=pixels, p=params_st)
    def test_bounded(self, pix, p):
        assert 0.0 <= wg.decolor_pixel(pix, p) <= 1.0

    @given(pix=pixels, b1=betas, b2=betas)
    def test_beta_k_monotonicity(self, pix, b1, b2):
        assume(abs(b2 - b1) > 1e-6)
        assume(wg.warm_luminance(pix) - wg.cool_luminance(pix) > 1e-3)
        lo, hi = sorted((b1, b2))
        assert wg.decolor_pixel(pix, wg.DecolorParams(beta_k=hi)) > wg.decolor_pixel(
            pix, wg.DecolorParams(beta_k=lo))

    def test_pure_hue_ordering(self):
        assert wg.decolor_pixel((1, 0, 0)) > wg.decolor_pixel((0, 0, 1)) > wg.decolor_pixel((0, 1, 0))


class TestParamsAndContainers:
    def test_defaults(self):
        assert wg.DEFAULT_PARAMS.beta_r == 0.55 and wg.DEFAULT_PARAMS.beta_k == 0.8

    @pytest.mark.parametrize("bad", [0.5, 1.0, 0.0, -0.1, 1.5, float("nan"), float("inf")])
    def test_open_interval_rejected(self, bad):
        with pytest.raises(ValueError):
            wg.DecolorParams(beta_r=bad)
        with pytest.raises(ValueError):
            wg.DecolorParams(beta_k=bad)

    def test_planar_image(self, rng):
        img = rand_rgb(rng, 4, 5)
        assert (img.width, img.height, img.kind, img.pixel_count) == (5, 4, "rgb", 20)
        assert wg.PlanarImage(rng.random((4, 5))).kind == "luminance"
        for bad in (rng.random((4, 5, 2)), rng.random(7), np.array([[1.2]]), np.array([[-0.1]]),
                    np.array([[float("nan")]])):
            with pytest.raises(ValueError):
                wg.PlanarImage(bad)
        assert wg.PlanarImage(np.zeros((0, 0, 3))).pixel_count == 0

    def test_curves_and_grids(self):
        for kw in ({"slope": 0.0}, {"slope": -2.0}, {"slope": float("inf")}, {"midpoint": 1.5}):
            with pytest.raises(ValueError):
                wg.SigmoidCurve(**kw)
        with pytest.raises(ValueError):
            wg.LocalHistogramGrid(tile_w=0, tile_h=4)
        with pytest.raises(ValueError):
            wg.LocalHistogramGrid(tile_w=4, tile_h=4, bins=1)
        with pytest.raises(ValueError):
            wg.LocalHistogramGrid(tile_w=4, tile_h=4, strength=1.2)
        g = wg.LocalHistogramGrid.for_image(100, 50)
        assert (g.tile_w, g.tile_h) == (13, 7)


class TestBackend:
    def test_single_cuda_backend(self):
        assert wg.available_backends() == ("cuda",)
        assert wg.active_backend() == "cuda"
        assert wg.compiled_available()
        k = backend.get_kernels()
        assert k.NAME == "cuda"
        assert backend.get_kernels("compiled") is k  # reference name accepted as alias

    def test_unknown_backend(self):
        with pytest.raises(ValueError):
            backend.get_kernels("fortran")
        with pytest.raises(ValueError):
            backend.get_kernels("python")  # no CPU fallback backend exists

    def test_threads(self, monkeypatch):
        assert backend.resolve_threads(3) == 3
        monkeypatch.delenv(backend.THREADS_ENV, raising=False)
        assert backend.resolve_threads(None) == 1
        monkeypatch.setenv(backend.THREADS_ENV, "5")
        assert backend.resolve_threads(None) == 5
        with pytest.raises(ValueError):
            backend.resolve_threads(0)

    @pytest.mark.parametrize("height,threads", [(1, 1), (7, 2), (8, 3), (5, 16), (0, 4)])
    def test_run_rows_covers_all_rows_once(self, height, threads):
        hits = np.zeros(height, dtype=int)
        backend.run_rows(height, threads, lambda r0, r1: hits.__setitem__(slice(r0, r1), hits[r0:r1] + 1))
        assert (hits == 1).all()

    def test_run_rows_propagates_errors(self):
        def boom(r0, r1):
            raise RuntimeError("worker failure")

        with pytest.raises(RuntimeError):
            backend.run_rows(10, 4, boom)

    def test_device_selection(self, monkeypatch):
        monkeypatch.setattr(backend, "_device", None)
        monkeypatch.setenv(backend.DEVICE_ENV, "3")
        assert backend.get_device() == 3
        backend.set_device(1)
        assert backend.get_device() == 1
        with pytest.raises(ValueError):
            backend.set_device(-1)
        monkeypatch.setattr(backend, "_device", None)


class TestNoCpuFallback:
    """Without a GPU every image entry point must fail loudly (never compute on the CPU)."""

    @pytest.fixture(autouse=True)
    def _skip_with_gpu(self):
        from paper_2108_13656_b200 import _lib

        if _lib.device_count() > 0:
            pytest.skip("a GPU is present")

    def test_decolor_image_raises(self, rng):
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            wg.decolor_image(rand_rgb(rng, 3, 3))

    def test_tone_and_codec_raise(self, rng):
        with pytest.raises(RuntimeError):
            wg.apply_sigmoid(wg.PlanarImage(rng.random((2, 2))))
        with pytest.raises(RuntimeError):
            wg.tonemap_image(rand_rgb(rng, 2, 2))
        with pytest.raises(RuntimeError):
            wg.quantize_u8(np.array([0.5]))
        with pytest.raises(RuntimeError):
            wg.decolor_host(np.zeros((2, 3), dtype=np.uint8))

    def test_argument_errors_still_first(self, rng):
        with pytest.raises(ValueError):
            wg.decolor_image(wg.PlanarImage(rng.random((3, 3))))
        with pytest.raises(ValueError):
            wg.tonemap_image(rand_rgb(rng, 2, 2), mode="fancy")
        with pytest.raises(ValueError):
            wg.luminance_image(rand_rgb(rng, 2, 2), method="nope")


def test_empty_images_need_no_device():
    out = wg.decolor_image(wg.PlanarImage(np.zeros((0, 0, 3))))
    assert out.kind == "luminance" and out.pixel_count == 0
    assert wg.quantize_u8(np.zeros(0)).shape == (0,)
