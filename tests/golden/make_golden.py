"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory, builds the reference's
own Cython extension there (`python setup.py build_ext --inplace`, the
reference's documented build), imports `warmgray` from that scratch copy and
records the outputs of the reference's public functions on seeded inputs.
Nothing under /root/reference is modified and no reference source is copied
into this repository; only the outputs below are committed:

  kat.json            scalar / image known answers (test_core, test_codec,
                      test_tonemap fixtures) evaluated by the reference
  cube.json           sha256 of the reference's outputs over all 2^24 u8
                      colours (fp64 gray, u8 gray, u8 toned) for both backends
  c1.json             C1 (512x512 u8, default_rng(0)) input/output sha256
  rand_f64.npz        seeded fp64 images and the reference's decolor output
  sigmoid.npz         apply_sigmoid over a grid of inputs and curves
  reinstate.npz       reinstate_color on seeded inputs
  tonemap_global.npz  tonemap_image(mode="global") on a seeded image
  hdr.npz             HDR adapter evaluated with the
                      reference's decolor_image/apply_sigmoid/quantize_u8
  colorspaces.npz     bt601/hsv/lab_lightness/lab rows (compiled backend) on
                      seeded fp64 images incl. sRGB / Lab branch points
  lhe.npz             apply_local_lhe on seeded / structured luminance over
                      grids incl. 1x1 tiles, oversize tiles, 2..1000 bins,
                      strength 0 and 1; tonemap_image(mode="local") on seeded
                      rgb; quantize_u8 of the local tone map of uint8 images
  codec/              PPM/PGM/PNG files written by the reference's save_image
                      (plus hand-made headers and malformed files) and
                      codec.json: what the reference's load_image returns for
                      each (uint8 samples) or which exception it raises
  metrics.npz/json    _sweep_counts / evaluate / ccpr / ccfr / write_sweep_csv of
                      the reference on seeded image pairs (exhaustive and
                      sampled pair sets, several gray methods)
  tone_rgb.npz        quantize_u8 of tonemap_image(mode="global") colour and
                      luminance outputs on uint8 images (default and custom
                      parameters, black and very dark pixels)
  colorspaces.json    scalar known answers (luma_weighted, hsv_v, rgb_to_lab,
                      lab_lightness, delta_e76) and sha256 of the u8 cube
                      through luminance_image for y / v / lab
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"


def build_reference() -> str:
    scratch = os.path.join(tempfile.gettempdir(), "wg_ref_golden")
    if not os.path.exists(os.path.join(scratch, "src", "warmgray")):
        shutil.rmtree(scratch, ignore_errors=True)
        shutil.copytree(REF_PKG, scratch)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=scratch,
                   check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    return os.path.join(scratch, "src")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def color_cube_u8() -> np.ndarray:
    i = np.arange(1 << 24, dtype=np.uint32)
    cube = np.empty((1 << 24, 3), dtype=np.uint8)
    cube[:, 0] = i >> 16
    cube[:, 1] = (i >> 8) & 255
    cube[:, 2] = i & 255
    return cube.reshape(4096, 4096, 3)


def main() -> None:
    sys.path.insert(0, build_reference())
    import warmgray as wg
    from warmgray.backend import get_kernels

    assert wg.compiled_available(), "reference extension did not build"

    # ---------------- known answers ----------------
    fixture_pixels = [(1, 1, 1), (0, 0, 0), (0, 0, 1), (1, 0, 0), (0, 1, 0), (0.3, 0.9, 0.4),
                      (0.5, 0.25, 0.1), (1, 1, 0), (0, 1, 1), (1, 0, 1), (0.2, 0.2, 0.2)]
    kat = {
        "decolor_pixel": [[list(map(float, p)), wg.decolor_pixel(p)] for p in fixture_pixels],
        "white_luminance": [[list(map(float, p)), wg.white_luminance(p)] for p in fixture_pixels],
        "red_green_luminance": [[list(map(float, p)), wg.red_green_luminance(p)]
                                for p in fixture_pixels],
        "warm_luminance": [[list(map(float, p)), wg.warm_luminance(p)] for p in fixture_pixels],
        "cool_luminance": [[list(map(float, p)), wg.cool_luminance(p)] for p in fixture_pixels],
        "custom_params": [[list(map(float, p)), wg.decolor_pixel(p, wg.DecolorParams(0.9, 0.6))]
                          for p in fixture_pixels],
        "two_pixel_image": wg.decolor_image(
            wg.PlanarImage(np.array([[[1, 0, 0], [0, 1, 0]]], dtype=np.float64))).data.tolist(),
        "quantize_in": [0.0, 0.5, 1.0, 0.66332, 0.2989, 127.5 / 255.0, -0.5, 1.5],
    }
    kat["quantize_out"] = wg.quantize_u8(np.array(kat["quantize_in"])).tolist()
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)

    # ---------------- exhaustive u8 cube ----------------
    cube = color_cube_u8()
    x = wg.dequantize_u8(cube)
    cube_info = {}
    for backend in ("compiled", "python"):
        out = np.empty((4096, 4096), dtype=np.float64)
        get_kernels(backend).decolor_rows(x, out, 0.55, 0.8, 0, 4096)
        gray_u8 = wg.quantize_u8(out)
        toned = wg.quantize_u8(wg.apply_sigmoid(wg.PlanarImage(out)).data)
        toned2 = wg.quantize_u8(
            wg.apply_sigmoid(wg.PlanarImage(out), wg.SigmoidCurve(0.3, 12.0)).data)
        cube_info[backend] = {
            "gray_f64_sha256": sha(out),
            "gray_u8_sha256": sha(gray_u8),
            "toned_u8_default_sha256": sha(toned),
            "toned_u8_m0.3_k12_sha256": sha(toned2),
            "gray_u8_histogram": np.bincount(gray_u8.ravel(), minlength=256).tolist(),
        }
        if backend == "compiled":
            ref_compiled = out
    cube_info["python_vs_compiled_f64_max_abs"] = float(np.abs(out - ref_compiled).max())
    cube_info["layout"] = "index i -> (i>>16, (i>>8)&255, i&255), 4096x4096 row-major"
    # custom parameters over the cube (u8 only)
    out = np.empty((4096, 4096), dtype=np.float64)
    get_kernels("compiled").decolor_rows(x, out, 0.9, 0.6, 0, 4096)
    cube_info["compiled_b0.9_0.6_gray_u8_sha256"] = sha(wg.quantize_u8(out))
    with open(os.path.join(HERE, "cube.json"), "w") as f:
        json.dump(cube_info, f, indent=1)

    # ---------------- C1 ----------------
    c1 = np.random.default_rng(0).integers(0, 256, (512, 512, 3), dtype=np.uint8)
    c1_gray = wg.quantize_u8(wg.decolor_image(wg.PlanarImage(wg.dequantize_u8(c1))).data)
    with open(os.path.join(HERE, "c1.json"), "w") as f:
        json.dump({"input_sha256": sha(c1), "gray_u8_sha256": sha(c1_gray),
                   "gray_u8_mean": float(c1_gray.mean()),
                   "generator": "np.random.default_rng(0).integers(0,256,(512,512,3),dtype=np.uint8)"},
                  f, indent=1)

    # ---------------- seeded fp64 images ----------------
    rng = np.random.default_rng(1234)
    rgb_a = rng.random((23, 31, 3))
    rgb_b = rng.random((8, 11, 3))
    edge = np.array([[[0, 0, 0], [1, 1, 1], [1, 0, 0], [0, 1, 0], [0, 0, 1]]], dtype=np.float64)
    np.savez_compressed(
        os.path.join(HERE, "rand_f64.npz"),
        rgb_a=rgb_a, gray_a=wg.decolor_image(wg.PlanarImage(rgb_a)).data,
        gray_a_custom=wg.decolor_image(wg.PlanarImage(rgb_a), wg.DecolorParams(0.9, 0.6)).data,
        rgb_b=rgb_b, gray_b=wg.decolor_image(wg.PlanarImage(rgb_b)).data,
        edge=edge, gray_edge=wg.decolor_image(wg.PlanarImage(edge)).data,
    )

    # ---------------- sigmoid ----------------
    xs = np.concatenate([np.linspace(0.0, 1.0, 1001), [0.5, 0.0, 1.0, 1e-9, 1 - 1e-9, 0.3]])
    curves = [(0.5, 8.0), (0.5, 7.0), (0.3, 5.0), (0.5, 1e-6), (0.8, 50.0), (0.0, 3.0),
              (1.0, 3.0), (0.5, 1e-3), (0.25, 0.1)]
    outs = np.stack([wg.apply_sigmoid(wg.PlanarImage(xs[None, :]), wg.SigmoidCurve(m, k)).data[0]
                     for m, k in curves])
    np.savez_compressed(os.path.join(HERE, "sigmoid.npz"), x=xs, curves=np.array(curves), out=outs)

    # ---------------- reinstate ----------------
    rng = np.random.default_rng(77)
    rgb = rng.random((8, 9, 3))
    l_in = wg.decolor_image(wg.PlanarImage(rgb)).data.copy()
    l_in[0, :3] = 0.0
    l_in[1, :2] = 5e-7
    l_out = rng.random((8, 9))
    np.savez_compressed(os.path.join(HERE, "reinstate.npz"), rgb=rgb, l_in=l_in, l_out=l_out,
                        out=wg.reinstate_color(wg.PlanarImage(rgb), wg.PlanarImage(l_in),
                                               wg.PlanarImage(l_out)).data)

    # ---------------- tonemap global ----------------
    rng = np.random.default_rng(78)
    rgb = rng.random((12, 10, 3))
    rgb[0, 0] = 0.0
    rgb_out, l_out = wg.tonemap_image(wg.PlanarImage(rgb), mode="global")
    rgb_out2, l_out2 = wg.tonemap_image(wg.PlanarImage(rgb), mode="global",
                                        params=wg.DecolorParams(0.7, 0.9),
                                        curve=wg.SigmoidCurve(0.4, 3.0))
    np.savez_compressed(os.path.join(HERE, "tonemap_global.npz"), rgb=rgb, rgb_out=rgb_out.data,
                        l_out=l_out.data, rgb_out2=rgb_out2.data, l_out2=l_out2.data)

    # ---------------- HDR adapter via the reference's own operators ----------------
    rng = np.random.default_rng(79)
    n, h, w = 3, 24, 32
    lum = 10.0 ** rng.uniform(-3, 4, (n, h, w))
    chroma = rng.random((n, h, w, 3))
    chroma[..., rng.integers(0, 3, (n, h, w))[..., None] == np.arange(3)] = 0.0
    y = chroma @ np.array([0.2126, 0.7152, 0.0722])
    hdr = (chroma * (lum / np.maximum(y, 1e-6))[..., None]).astype(np.float32)
    hdr[0, 0, 0] = 0.0                       # a black pixel
    hdr[2] = hdr[2, 0, 0]                    # a constant image (gmax == gmin)
    outs = []
    for im in hdr.astype(np.float64):
        m = im.max()
        gn = wg.decolor_image(wg.PlanarImage(im / m)).data
        pos = gn > 0
        gmin, gmax = gn[pos].min(), gn[pos].max()
        if gmax > gmin:
            t = np.where(pos, np.clip(np.log(np.where(pos, gn, 1.0) / gmin) / np.log(gmax / gmin),
                                      0, 1), 0.0)
        else:
            t = np.where(pos, 1.0, 0.0)
        outs.append(wg.quantize_u8(wg.apply_sigmoid(wg.PlanarImage(t)).data))
    np.savez_compressed(os.path.join(HERE, "hdr.npz"), rgb=hdr, out=np.stack(outs))
    colorspaces_golden(wg, get_kernels)
    lhe_golden(wg)
    codec_golden(wg)
    metrics_golden(wg)
    tone_rgb_golden(wg)
    print("golden fixtures written to", HERE)


def tone_rgb_golden(wg) -> None:
    """uint8 colour output of the global tone map: quantize_u8 of tonemap_image(mode="global")."""
    rng = np.random.default_rng(2112)
    u8 = rng.integers(0, 256, (2, 40, 56, 3), dtype=np.uint8)
    u8[0, 0, :8] = 0      # black pixels (l_in == 0 -> 0)
    u8[1, :4] = 3         # very dark pixels (ratio amplifies)
    out = {"u8": u8}
    for tag, curve, params in (("default", wg.SigmoidCurve(), wg.DEFAULT_PARAMS),
                               ("custom", wg.SigmoidCurve(0.3, 12.0), wg.DecolorParams(0.7, 0.9))):
        rgb_o, toned = [], []
        for im in u8:
            r, lo = wg.tonemap_image(wg.PlanarImage(wg.dequantize_u8(im)), mode="global", params=params, curve=curve)
            rgb_o.append(wg.quantize_u8(r.data))
            toned.append(wg.quantize_u8(lo.data))
        out[f"{tag}_rgb"] = np.stack(rgb_o)
        out[f"{tag}_toned"] = np.stack(toned)
    np.savez_compressed(os.path.join(HERE, "tone_rgb.npz"), **out)


def metrics_golden(wg) -> None:
    """the reference's contrast metrics."""
    import io as _io

    from warmgray import metrics as m

    rng = np.random.default_rng(2111)
    cases = []  # (name, rgb, gray, cfg)
    rgb = rng.random((12, 10, 3))
    cases.append(("exh_ours", rgb, wg.luminance_image(wg.PlanarImage(rgb)).data, m.PairSampleConfig(exhaustive=True)))
    cases.append(("exh_lab", rgb, wg.luminance_image(wg.PlanarImage(rgb), method="lab").data,
                  m.PairSampleConfig(exhaustive=True)))
    u8 = rng.integers(0, 256, (40, 56, 3)).astype(np.float64) / 255.0
    cases.append(("smp_ours", u8, wg.luminance_image(wg.PlanarImage(u8)).data, m.PairSampleConfig()))
    cases.append(("smp_v", u8, wg.luminance_image(wg.PlanarImage(u8), method="v").data,
                  m.PairSampleConfig(pair_count=3000, seed=9)))
    small = rng.random((3, 3, 3))
    cases.append(("cover", small, wg.luminance_image(wg.PlanarImage(small)).data,
                  m.PairSampleConfig(pair_count=100, seed=7)))
    out, js = {}, {}
    taus = list(m.TAU_SWEEP)
    for name, c, g, cfg in cases:
        ci, gi = wg.PlanarImage(c), wg.PlanarImage(g)
        out[f"{name}_rgb"] = c
        out[f"{name}_gray"] = g
        out[f"{name}_counts"] = m._sweep_counts(ci, gi, taus, cfg)
        rep = m.evaluate(ci, gi, cfg)
        js[name] = {"cfg": [cfg.pair_count, cfg.seed, cfg.exhaustive],
                    "per_tau": [[r.tau, r.ccpr, r.ccfr, r.escore] for r in rep.per_tau],
                    "mean_escore": rep.mean_escore,
                    "ccpr_2.5": m.ccpr(ci, gi, 2.5, cfg), "ccfr_7": m.ccfr(ci, gi, 7.0, cfg)}
    buf = _io.StringIO()
    m.write_sweep_csv(buf, [("a", m.evaluate(wg.PlanarImage(cases[0][1]), wg.PlanarImage(cases[0][2]), cases[0][3])),
                            ("b", m.evaluate(wg.PlanarImage(cases[2][1]), wg.PlanarImage(cases[2][2]), cases[2][3]))])
    js["csv"] = buf.getvalue()
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)
    with open(os.path.join(HERE, "metrics.json"), "w") as f:
        json.dump(js, f, indent=1)


def codec_golden(wg) -> None:
    """the reference's file codec on files it writes and on malformed ones."""
    from PIL import Image
    from warmgray.codec import CodecError

    d = os.path.join(HERE, "codec")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(2110)
    rgb = wg.PlanarImage(rng.integers(0, 256, (6, 9, 3)).astype(np.float64) / 255.0)
    gray = wg.PlanarImage(rng.integers(0, 256, (4, 7)).astype(np.float64) / 255.0)
    wg.save_image(os.path.join(d, "rgb.ppm"), rgb)
    wg.save_image(os.path.join(d, "gray.pgm"), gray)
    wg.save_image(os.path.join(d, "rgb.png"), rgb)
    wg.save_image(os.path.join(d, "gray.png"), gray)
    wg.save_image(os.path.join(d, "white.ppm"), wg.PlanarImage(np.ones((1, 1, 3))))
    u8 = rng.integers(0, 256, (5, 4, 4), dtype=np.uint8)
    Image.fromarray(u8, mode="RGBA").save(os.path.join(d, "rgba.png"))
    Image.fromarray(u8[..., :2].copy(), mode="LA").save(os.path.join(d, "la.png"))
    Image.fromarray(u8[..., 0].copy(), mode="L").convert("P").save(os.path.join(d, "pal.png"))
    raw = {
        "comments.ppm": b"P6\n# a comment\n2 1\n# another\n255\n" + bytes([255, 0, 0, 0, 255, 0]),
        "trailing.pgm": b"P5 3 1 255 " + bytes([1, 2, 3]) + b"extra",
        "ascii.ppm": b"P3\n1 1\n255\n255 0 0\n",
        "deep.ppm": b"P6\n1 1\n65535\n" + bytes(6),
        "short.ppm": b"P6\n2 2\n255\n\xff",
        "badtoken.pgm": b"P5\n2 x\n255\n" + bytes(2),
        "zero.pgm": b"P5\n0 1\n255\n",
        "header.pgm": b"P5\n2",
        "lone.pgm": b"P",
        "text.png": b"hello world",
    }
    for name, data in raw.items():
        with open(os.path.join(d, name), "wb") as f:
            f.write(data)
    expect = {}
    for name in sorted(os.listdir(d)):
        if name.endswith(".json"):
            continue
        try:
            img = wg.load_image(os.path.join(d, name))
            expect[name] = {"kind": img.kind, "shape": list(img.data.shape),
                            "u8": wg.quantize_u8(img.data).ravel().tolist()}
        except CodecError as e:
            expect[name] = {"error": "CodecError", "message": str(e).replace(d + os.sep, "")}
    with open(os.path.join(d, "codec.json"), "w") as f:
        json.dump(expect, f, indent=1)


LHE_CASES = [  # (h, w, tile_w, tile_h, bins, strength)
    (11, 13, 5, 4, 32, 0.7), (30, 17, 6, 7, 256, 0.9), (64, 80, 10, 8, 256, 0.7), (1, 1, 4, 4, 16, 1.0),
    (1, 50, 3, 3, 8, 0.5), (50, 1, 3, 3, 8, 0.5), (6, 6, 10000, 10000, 256, 1.0), (40, 33, 1, 1, 7, 0.3),
    (37, 41, 9, 5, 1000, 1.0), (20, 20, 4, 4, 2, 0.7), (16, 16, 4, 4, 256, 0.0), (97, 131, 17, 13, 256, 0.7),
]


def lhe_golden(wg) -> None:
    """the reference's local tone map."""
    rng = np.random.default_rng(2109)
    out = {"cases": np.array(LHE_CASES, dtype=np.float64)}
    for i, (h, w, tw, th, nb, s) in enumerate(LHE_CASES):
        d = rng.random((h, w))
        if i == 2:
            d = np.round(d * 255) / 255  # u8-derived values: many exact bin edges
        out[f"in{i}"] = d
        out[f"out{i}"] = wg.apply_local_lhe(wg.PlanarImage(d), wg.LocalHistogramGrid(tw, th, nb, s)).data
    # structured: two-tile halves, ramp, constant (test_tonemap.py fixtures' shapes)
    xs = np.linspace(0.0, 1.0, 4)
    halves = np.hstack([0.3 * np.tile(xs, (8, 1)), 0.7 + 0.3 * np.tile(xs, (8, 1))])
    ramp = np.tile(np.linspace(0.0, 1.0, 64), (32, 1))
    const = np.full((12, 10), 0.37)
    for name, d, grid in (("halves", halves, wg.LocalHistogramGrid(4, 8, 16, 1.0)),
                          ("ramp", ramp, wg.LocalHistogramGrid(8, 8, strength=1.0)),
                          ("const", const, wg.LocalHistogramGrid(4, 4, strength=1.0))):
        out[f"{name}_in"] = d
        out[f"{name}_grid"] = np.array([grid.tile_w, grid.tile_h, grid.bins, grid.strength])
        out[f"{name}_out"] = wg.apply_local_lhe(wg.PlanarImage(d), grid).data
    # tonemap_image(mode="local")
    rgb = rng.random((24, 36, 3))
    rgb[0, 0] = 0.0
    r1, l1 = wg.tonemap_image(wg.PlanarImage(rgb), mode="local")
    g2 = wg.LocalHistogramGrid(7, 5, 64, 0.9)
    r2, l2 = wg.tonemap_image(wg.PlanarImage(rgb), mode="local", params=wg.DecolorParams(0.7, 0.9), grid=g2)
    out.update(tm_rgb=rgb, tm_rgb_out=r1.data, tm_l_out=l1.data, tm_rgb_out2=r2.data, tm_l_out2=l2.data)
    # uint8 batch: quantize_u8(local tone map) and quantize_u8(gray)
    u8 = rng.integers(0, 256, (3, 48, 64, 3), dtype=np.uint8)
    u8[1, :24] = u8[1, 0, 0]  # a flat region (identity tiles)
    toned, gray = [], []
    for im in u8:
        img = wg.PlanarImage(wg.dequantize_u8(im))
        _, lo = wg.tonemap_image(img, mode="local")
        toned.append(wg.quantize_u8(lo.data))
        gray.append(wg.quantize_u8(wg.decolor_image(img).data))
    out.update(u8_rgb=u8, u8_toned=np.stack(toned), u8_gray=np.stack(gray))
    np.savez_compressed(os.path.join(HERE, "lhe.npz"), **out)


def colorspaces_golden(wg, get_kernels) -> None:
    """the reference's baseline extractors."""
    comp = get_kernels("compiled")
    rng = np.random.default_rng(2108)
    rgb = rng.random((37, 53, 3))
    # exact branch points of the sRGB linearisation and the Lab compander
    special = np.array([0.0, 1.0, 0.04045, np.nextafter(0.04045, 1), np.nextafter(0.04045, 0),
                        0.5, 1e-300, 0.01, 0.2, 0.99999999])
    edge = np.stack(np.meshgrid(special, special, special, indexing="ij"), -1).reshape(-1, 1, 3)
    edge = np.ascontiguousarray(edge.reshape(len(special), -1, 3))
    out = {"rgb": rgb, "edge": edge}
    for tag, img in (("rgb", rgb), ("edge", edge)):
        h = img.shape[0]
        for name in ("bt601_rows", "hsv_value_rows", "lab_lightness_rows"):
            o = np.empty(img.shape[:2])
            getattr(comp, name)(img, o, 0, h)
            out[f"{tag}_{name}"] = o
        o3 = np.empty(img.shape)
        comp.lab_rows(img, o3, 0, h)
        out[f"{tag}_lab_rows"] = o3
    np.savez_compressed(os.path.join(HERE, "colorspaces.npz"), **out)

    pix = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1), (0, 0, 0), (0.3, 0.7, 0.2), (0.2, 0.5, 0.3),
           (0.04045, 0.5, 0.9), (0.01, 0.02, 0.03)]
    kat = {
        "luma_weighted": [[list(map(float, p)), wg.luma_weighted(p)] for p in pix],
        "hsv_v": [[list(map(float, p)), wg.hsv_v(p)] for p in pix],
        "lab_lightness": [[list(map(float, p)), wg.lab_lightness(p)] for p in pix],
        "rgb_to_lab": [[list(map(float, p)), list(map(float, (lambda c: (c.l_star, c.a_star, c.b_star))(
            wg.rgb_to_lab(p))))] for p in pix],
        "delta_e76": [[list(map(float, p)), list(map(float, q)),
                       wg.delta_e76(wg.rgb_to_lab(p), wg.rgb_to_lab(q))] for p, q in zip(pix, pix[1:])],
    }
    cube = wg.PlanarImage(wg.dequantize_u8(color_cube_u8()))
    for method in ("y", "v", "lab"):
        g = wg.quantize_u8(wg.luminance_image(cube, method=method, backend="compiled").data)
        kat[f"cube_{method}_u8_sha256"] = sha(g)
        kat[f"cube_{method}_u8_histogram"] = np.bincount(g.ravel(), minlength=256).tolist()
    with open(os.path.join(HERE, "colorspaces.json"), "w") as f:
        json.dump(kat, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1:] == ["tone_rgb"]:
        sys.path.insert(0, build_reference())
        import warmgray as _wg

        tone_rgb_golden(_wg)
        sys.exit(0)
    if sys.argv[1:] == ["metrics"]:
        sys.path.insert(0, build_reference())
        import warmgray as _wg

        metrics_golden(_wg)
        sys.exit(0)
    if sys.argv[1:] == ["codec"]:
        sys.path.insert(0, build_reference())
        import warmgray as _wg

        codec_golden(_wg)
        sys.exit(0)
    if sys.argv[1:] == ["lhe"]:
        sys.path.insert(0, build_reference())
        import warmgray as _wg

        lhe_golden(_wg)
        sys.exit(0)
    if sys.argv[1:] == ["colorspaces"]:
        sys.path.insert(0, build_reference())
        import warmgray as _wg
        from warmgray.backend import get_kernels as _gk
        colorspaces_golden(_wg, _gk)
        sys.exit(0)
    main()
