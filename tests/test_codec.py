"""uint8 file codec.

CPU: the native PGM/PPM reader/writer (csrc/wg_io.cu) and the PNG route
against what the reference's own load_image returns for files its
save_image wrote, plus hand-made and malformed files
(tests/golden/codec/codec.json, tests/golden/make_golden.py codec_golden).
GPU: the float API (load_image / save_image through the device quantizer)
and decolor_files end to end against the oracle.
"""

import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2108_13656_b200 as wg
from paper_2108_13656_b200 import codec

CODEC = os.path.join(GOLDEN, "codec")


@pytest.fixture(scope="module")
def expect():
    with open(os.path.join(CODEC, "codec.json")) as f:
        return json.load(f)


def test_load_u8_matches_reference(expect):
    for name, e in expect.items():
        path = os.path.join(CODEC, name)
        if "error" in e:
            with pytest.raises(wg.CodecError) as info:
                wg.load_u8(path)
            assert str(info.value).replace(CODEC + os.sep, "") == e["message"], name
        else:
            got = wg.load_u8(path)
            assert list(got.shape) == e["shape"], name
            assert got.ravel().tolist() == e["u8"], name


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(OSError):
        wg.load_u8(tmp_path / "nope.png")
    with pytest.raises(OSError):
        wg.read_pnm_batch([tmp_path / "nope.ppm"], pinned=False)


def test_header_layout_and_round_trip(tmp_path):
    wg.save_u8(tmp_path / "w.ppm", np.full((1, 1, 3), 255, np.uint8))
    assert (tmp_path / "w.ppm").read_bytes() == b"P6\n1 1\n255\n\xff\xff\xff"
    assert (tmp_path / "w.ppm").read_bytes() == open(os.path.join(CODEC, "white.ppm"), "rb").read()
    rng = np.random.default_rng(0)
    for shape, ext in (((6, 9, 3), ".ppm"), ((4, 7), ".pgm"), ((5, 8, 3), ".png"), ((5, 8), ".png")):
        a = rng.integers(0, 256, shape, dtype=np.uint8)
        wg.save_u8(tmp_path / f"a{ext}", a)
        np.testing.assert_array_equal(wg.load_u8(tmp_path / f"a{ext}"), a)
    # the reference's own files re-encode to identical bytes
    for name in ("rgb.ppm", "gray.pgm"):
        a = wg.load_u8(os.path.join(CODEC, name))
        wg.save_u8(tmp_path / name, a)
        assert (tmp_path / name).read_bytes() == open(os.path.join(CODEC, name), "rb").read()


def test_save_u8_kind_and_extension_errors(tmp_path):
    with pytest.raises(wg.CodecError):
        wg.save_u8(tmp_path / "x.pgm", np.zeros((2, 2, 3), np.uint8))
    with pytest.raises(wg.CodecError):
        wg.save_u8(tmp_path / "x.ppm", np.zeros((2, 2), np.uint8))
    with pytest.raises(wg.CodecError):
        wg.save_u8(tmp_path / "x.tiff", np.zeros((2, 2, 3), np.uint8))


def test_batch_read_write(tmp_path):
    rng = np.random.default_rng(1)
    batch = rng.integers(0, 256, (7, 13, 11, 3), dtype=np.uint8)
    paths = [tmp_path / f"{k}.ppm" for k in range(7)]
    wg.write_pnm_batch(paths, batch, threads=3)
    for k, p in enumerate(paths):
        np.testing.assert_array_equal(wg.load_u8(p), batch[k])
    back = wg.read_pnm_batch(paths, threads=4, pinned=False)
    np.testing.assert_array_equal(back, batch)
    gray = batch[..., 0].copy()
    gpaths = [tmp_path / f"{k}.pgm" for k in range(7)]
    wg.write_pnm_batch(gpaths, gray)
    np.testing.assert_array_equal(wg.read_pnm_batch(gpaths, pinned=False), gray)
    # a file of another size in the batch is a CodecError naming it
    wg.save_u8(tmp_path / "odd.ppm", np.zeros((3, 3, 3), np.uint8))
    with pytest.raises(wg.CodecError, match="odd.ppm"):
        wg.read_pnm_batch(paths[:2] + [tmp_path / "odd.ppm"], pinned=False)
    # a malformed member (the reference's error text)
    shutil.copy(os.path.join(CODEC, "short.ppm"), tmp_path / "short.ppm")
    with pytest.raises(wg.CodecError, match="truncated"):
        wg.read_pnm_batch([tmp_path / "short.ppm"], pinned=False)
    with pytest.raises(ValueError):
        wg.write_pnm_batch(paths[:3], batch)


def test_pnm_info_and_trailing_bytes():
    assert codec.pnm_info(os.path.join(CODEC, "rgb.ppm")) == (6, 9, 3)
    assert codec.pnm_info(os.path.join(CODEC, "trailing.pgm")) == (1, 3, 1)
    np.testing.assert_array_equal(wg.load_u8(os.path.join(CODEC, "trailing.pgm")), [[1, 2, 3]])


# ---------------------------------------------------------------- GPU: float API and the batch pipeline
@pytest.mark.gpu
def test_load_image_matches_reference(expect):
    for name, e in expect.items():
        if "error" in e:
            continue
        img = wg.load_image(os.path.join(CODEC, name))
        assert img.kind == e["kind"]
        np.testing.assert_array_equal(wg.quantize_u8(img.data).ravel(), e["u8"])
        np.testing.assert_array_equal(img.data, np.reshape(e["u8"], e["shape"]) / 255.0)


@pytest.mark.gpu
def test_save_image_round_trips(tmp_path, rng):
    """The reference's TestPnm / TestPng round trips (test_codec.py:27-116)."""
    rgb = wg.PlanarImage(rng.integers(0, 256, (6, 9, 3)).astype(np.float64) / 255.0)
    gray = wg.PlanarImage(rng.integers(0, 256, (4, 7)).astype(np.float64) / 255.0)
    for img, name in ((rgb, "a.ppm"), (gray, "g.pgm"), (rgb, "a.png"), (gray, "g.png")):
        wg.save_image(tmp_path / name, img)
        again = wg.load_image(tmp_path / name)
        assert again.kind == img.kind
        assert np.array_equal(again.data, img.data)
    wg.save_image(tmp_path / "b.ppm", wg.load_image(tmp_path / "a.ppm"))
    assert (tmp_path / "a.ppm").read_bytes() == (tmp_path / "b.ppm").read_bytes()
    wg.save_image(tmp_path / "w.ppm", wg.PlanarImage(np.ones((1, 1, 3))))
    assert (tmp_path / "w.ppm").read_bytes() == b"P6\n1 1\n255\n\xff\xff\xff"
    with pytest.raises(wg.CodecError):
        wg.save_image(tmp_path / "x.pgm", rgb)
    with pytest.raises(wg.CodecError):
        wg.save_image(tmp_path / "x.ppm", gray)
    with pytest.raises(wg.CodecError):
        wg.save_image(tmp_path / "a.tiff", rgb)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["gray", "local", "gray_exact", "global_exact", "gray_png"])
def test_decolor_files_vs_oracle(tmp_path, mode):
    from oracle import oracle

    rng = np.random.default_rng(5)
    batch = rng.integers(0, 256, (5, 96, 128, 3), dtype=np.uint8)
    batch[0, :40] = batch[0, :40] // 32 * 32
    ext_in, ext_out = (".png", ".png") if mode == "gray_png" else (".ppm", ".pgm")
    src = [tmp_path / f"in{k}{ext_in}" for k in range(5)]
    dst = [tmp_path / f"out{k}{ext_out}" for k in range(5)]
    wg.write_batch(src, batch)
    exact = mode.endswith("_exact") or mode == "gray_png"
    base = mode.replace("_exact", "").replace("_png", "")
    assert wg.decolor_files(src, dst, mode=base, batch=2, exact=exact) == 5
    got = np.stack([wg.load_u8(p) for p in dst])
    if mode in ("gray_exact", "gray_png"):
        np.testing.assert_array_equal(got, oracle.decolor_u8(batch))
    elif mode == "global_exact":
        np.testing.assert_array_equal(got, oracle.tone_rgb_u8(batch)[1])
    elif mode == "gray":
        want = oracle.decolor_u8(batch)
        d = np.abs(got.astype(int) - want.astype(int))
        assert d.max() <= 1 and (d != 0).mean() <= 1e-4
    else:
        g = wg.LocalHistogramGrid.for_image(128, 96)
        np.testing.assert_array_equal(got, oracle.tone_local_u8(batch, g.tile_w, g.tile_h, g.bins, g.strength))


def test_read_write_batch_png_and_pnm(tmp_path):
    """read_batch / write_batch: PNG through Pillow on a thread pool, PNM natively;
    same bytes either way; mixed sizes rejected."""
    rng = np.random.default_rng(9)
    batch = rng.integers(0, 256, (4, 24, 40, 3), dtype=np.uint8)
    png = [tmp_path / f"a{k}.png" for k in range(4)]
    ppm = [tmp_path / f"a{k}.ppm" for k in range(4)]
    wg.write_batch(png, batch)
    wg.write_batch(ppm, batch)
    np.testing.assert_array_equal(wg.read_batch(png, pinned=False), batch)
    np.testing.assert_array_equal(wg.read_batch(ppm, pinned=False), batch)
    np.testing.assert_array_equal(wg.read_batch([png[0], ppm[1]], pinned=False), batch[:2])  # mixed formats
    wg.save_u8(tmp_path / "small.png", batch[0, :10])
    with pytest.raises(wg.CodecError):
        wg.read_batch([png[0], tmp_path / "small.png"], pinned=False)


@pytest.mark.parametrize("header", [b"P6\n_5 4\n255\n", b"P6\n5_ 4\n255\n", b"P6\n+_5 4\n255\n", b"P5\n5 _\n255\n",
                                    b"P6\n999999999999999999 999999999999999999\n255\n",
                                    b"P5\n4294967296 4294967296\n255\n"])
def test_hostile_headers_are_codec_errors(tmp_path, header):
    """Untrusted headers: a leading / trailing '_' in a number (the reference's
    int() rejects it) and dimensions whose product overflows 64 bits or exceeds
    the file are CodecErrors, never an out-of-bounds read or a wrapped size."""
    p = tmp_path / "h.ppm"
    p.write_bytes(header + b"\x00" * 64)
    with pytest.raises(wg.CodecError):
        wg.load_u8(p)
