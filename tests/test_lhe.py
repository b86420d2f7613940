"""Local tone map, CPU side: pin the oracle to the reference.

tests/golden/lhe.npz holds the reference's own apply_local_lhe /
tonemap_image(mode="local") outputs (tests/golden/make_golden.py). The oracle
restatement (oracle/warmgray_oracle.c: or_local_lhe_f64, or_tone_local_u8)
must reproduce them bit for bit; the GPU tests then compare against it.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle

import paper_2108_13656_b200 as wg


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "lhe.npz"))


def test_oracle_cases_bit_identical(golden):
    for i, (h, w, tw, th, nb, s) in enumerate(golden["cases"]):
        out = oracle.local_lhe_f64(golden[f"in{i}"], int(tw), int(th), int(nb), float(s))
        assert out.tobytes() == golden[f"out{i}"].tobytes(), (h, w, tw, th, nb, s)


@pytest.mark.parametrize("name", ["halves", "ramp", "const"])
def test_oracle_structured_bit_identical(golden, name):
    tw, th, nb, s = golden[f"{name}_grid"]
    out = oracle.local_lhe_f64(golden[f"{name}_in"], int(tw), int(th), int(nb), float(s))
    assert out.tobytes() == golden[f"{name}_out"].tobytes()


def test_oracle_u8_batch_matches_reference(golden):
    rgb = golden["u8_rgb"]
    g = wg.LocalHistogramGrid.for_image(rgb.shape[2], rgb.shape[1])
    toned, gray = oracle.tone_local_u8(rgb, g.tile_w, g.tile_h, g.bins, g.strength, with_gray=True, threads=3)
    np.testing.assert_array_equal(toned, golden["u8_toned"])
    np.testing.assert_array_equal(gray, golden["u8_gray"])


def test_oracle_batch_equals_per_image(golden):
    lum = np.stack([golden["in2"], golden["in2"][::-1].copy(), golden["in2"] * 0.5])
    batch = oracle.local_lhe_f64(lum, 10, 8, 256, 0.7, threads=3)
    for k in range(3):
        assert batch[k].tobytes() == oracle.local_lhe_f64(lum[k], 10, 8, 256, 0.7).tobytes()


def test_grid_validation_and_for_image():
    with pytest.raises(ValueError):
        wg.LocalHistogramGrid(tile_w=0, tile_h=4)
    with pytest.raises(ValueError):
        wg.LocalHistogramGrid(tile_w=4, tile_h=4, bins=1)
    with pytest.raises(ValueError):
        wg.LocalHistogramGrid(tile_w=4, tile_h=4, strength=1.2)
    g = wg.LocalHistogramGrid.for_image(3840, 2160)
    assert (g.tile_w, g.tile_h, g.bins, g.strength) == (480, 270, 256, 0.7)
    assert wg.LocalHistogramGrid.for_image(5, 3, tiles_x=8, tiles_y=8).tile_w == 1


def test_rejects_rgb_and_unknown_mode(rng):
    with pytest.raises(ValueError):
        wg.apply_local_lhe(wg.PlanarImage(rng.random((4, 4, 3))), wg.LocalHistogramGrid(2, 2))
    with pytest.raises(ValueError):
        wg.tonemap_image(wg.PlanarImage(rng.random((4, 4, 3))), mode="nope")
