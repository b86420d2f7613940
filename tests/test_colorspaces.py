"""Baseline colour-to-gray methods and CIELAB, CPU side.

* The scalar host API (luma_weighted, hsv_v, rgb_to_lab, lab_lightness,
  delta_e76) against the reference's own known answers
  (tests/golden/colorspaces.json) and the properties the reference's
  test_colorspaces.py checks.
* The oracle restatement (or_luma_f64 / or_lab_f64 / or_luma_u8) against the
  reference's compiled row kernels on seeded images and branch points, and
  against the sha256 of the reference over all 2^24 uint8 colours.
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest
from hypothesis import assume, given
from hypothesis import strategies as st

from conftest import GOLDEN
from oracle import oracle

import paper_2108_13656_b200 as wg

unit = st.floats(0.0, 1.0, allow_nan=False, allow_infinity=False, width=64)
pixels = st.tuples(unit, unit, unit)
ab = st.floats(-128.0, 128.0, allow_nan=False, allow_infinity=False, width=64)
labs = st.builds(wg.LabColor, l_star=st.floats(0, 100, width=64), a_star=ab, b_star=ab)


@pytest.fixture(scope="module")
def kat():
    with open(os.path.join(GOLDEN, "colorspaces.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "colorspaces.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- scalar API
@pytest.mark.parametrize("name", ["luma_weighted", "hsv_v", "lab_lightness"])
def test_scalar_known_answers(kat, name):
    fn = getattr(wg, name)
    for pix, want in kat[name]:
        assert fn(tuple(pix)) == want, (name, pix)


def test_rgb_to_lab_known_answers(kat):
    for pix, want in kat["rgb_to_lab"]:
        c = wg.rgb_to_lab(tuple(pix))
        assert [c.l_star, c.a_star, c.b_star] == want, pix


def test_delta_e76_known_answers(kat):
    for p, q, want in kat["delta_e76"]:
        assert wg.delta_e76(wg.rgb_to_lab(tuple(p)), wg.rgb_to_lab(tuple(q))) == want


def test_scalar_fixed_points():
    assert wg.luma_weighted((1, 0, 0)) == pytest.approx(0.2989, abs=1e-12)
    assert wg.luma_weighted((1, 1, 1)) == pytest.approx(0.9999, abs=1e-12)
    assert wg.luma_weighted((0, 0, 0)) == 0.0
    assert wg.hsv_v((0.2, 0.5, 0.3)) == 0.5
    white, black = wg.rgb_to_lab((1, 1, 1)), wg.rgb_to_lab((0, 0, 0))
    assert white.l_star == pytest.approx(100.0, abs=1e-4) and abs(white.a_star) < 1e-4 and abs(white.b_star) < 1e-4
    assert (black.l_star, black.a_star, black.b_star) == pytest.approx((0, 0, 0), abs=1e-9)
    assert wg.rgb_to_lab((1, 0, 0)).l_star == pytest.approx(53.2408, abs=1e-3)
    assert wg.delta_e76(wg.LabColor(50, 0, 0), wg.LabColor(60, 0, 0)) == pytest.approx(10.0)
    assert wg.delta_e76(white, black) == pytest.approx(100.0, abs=1e-3)


@given(pix=pixels)
def test_luma_and_lightness_in_unit_range(pix):
    assert 0.0 <= wg.luma_weighted(pix) <= 1.0
    assert 0.0 <= wg.lab_lightness(pix) <= 1.0


@given(v=unit)
def test_hsv_gray_axis(v):
    assert wg.hsv_v((v, v, v)) == v


@given(v1=unit, v2=unit)
def test_lightness_monotone_on_gray_axis(v1, v2):
    assume(abs(v1 - v2) > 1e-6)
    lo, hi = sorted((v1, v2))
    assert wg.lab_lightness((lo, lo, lo)) < wg.lab_lightness((hi, hi, hi))


@given(a=labs, b=labs, c=labs)
def test_delta_e_metric_axioms(a, b, c):
    assert wg.delta_e76(a, b) == wg.delta_e76(b, a) >= 0.0
    assert wg.delta_e76(a, c) <= wg.delta_e76(a, b) + wg.delta_e76(b, c) + 1e-9
    if a == b:
        assert wg.delta_e76(a, b) == 0.0


def test_method_names():
    assert wg.METHOD_NAMES == ("ours", "y", "v", "lab", "weighted")


# ---------------------------------------------------------------- oracle pinning
@pytest.mark.parametrize("tag", ["rgb", "edge"])
@pytest.mark.parametrize("method,row", [("y", "bt601_rows"), ("v", "hsv_value_rows"),
                                        ("lab", "lab_lightness_rows")])
def test_oracle_luma_bit_identical_to_reference(golden, tag, method, row):
    out = oracle.luma_f64(golden[tag], method)
    np.testing.assert_array_equal(out, golden[f"{tag}_{row}"])


@pytest.mark.parametrize("tag", ["rgb", "edge"])
def test_oracle_lab_bit_identical_to_reference(golden, tag):
    np.testing.assert_array_equal(oracle.lab_f64(golden[tag]), golden[f"{tag}_lab_rows"])


@pytest.mark.parametrize("method", ["y", "v", "lab"])
def test_oracle_u8_cube_matches_reference(kat, method):
    """All 2^24 colours: quantize_u8(luminance_image(dequantize_u8(cube), method)) sha256."""
    out = oracle.luma_u8(oracle.color_cube_u8(), method, threads=oracle.default_threads())
    assert np.bincount(out.ravel(), minlength=256).tolist() == kat[f"cube_{method}_u8_histogram"]
    assert sha(out) == kat[f"cube_{method}_u8_sha256"]


def test_oracle_lab_matches_scalar_api(golden):
    """The row restatement against the scalar API (reference tolerance 1e-9, test_colorspaces.py:126-133)."""
    rgb = golden["rgb"][:4, :6]
    lab = oracle.lab_f64(rgb)
    for y in range(rgb.shape[0]):
        for x in range(rgb.shape[1]):
            c = wg.rgb_to_lab(tuple(rgb[y, x]))
            assert lab[y, x] == pytest.approx([c.l_star, c.a_star, c.b_star], abs=1e-9)
            assert math.isclose(oracle.luma_f64(rgb[y:y + 1, x:x + 1], "lab")[0, 0],
                                wg.lab_lightness(tuple(rgb[y, x])), abs_tol=1e-9)


# ---------------------------------------------------------------- host-side validation (no GPU needed)
def test_luminance_image_rejects_gray_and_unknown(rng):
    with pytest.raises(ValueError):
        wg.luminance_image(wg.PlanarImage(rng.random((3, 3))), method="y")
    with pytest.raises(ValueError):
        wg.lab_image(wg.PlanarImage(rng.random((3, 3))))
    with pytest.raises(ValueError):
        wg.luminance_image(wg.PlanarImage(rng.random((2, 2, 3))), method="nope")
