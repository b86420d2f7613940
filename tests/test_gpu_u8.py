"""uint8 -> uint8 parity of the sm_100a kernels against the CPU oracle.

Default decolor (the headline kernel): the north-star bar, identical except
+-1 LSB on <= 0.01% of pixels (rounding ties). ``exact=True``: bit-identical
to the reference -- the fp32 kernel's near-tie pixels take the exact byte of
their colour from a table settled over all 2^24 colours (csrc/wg_u8exact.cu).
Checked on the exhaustive colour cube (exact: sha256 == the reference's), for
several parameter pairs, on C1, on C3 4K Voronoi images generated on the
device, and on edge cases (empty, ragged tails, misaligned buffers).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, U8_MAX_FRAC, u8_mismatch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    import torch

    return torch, torch.device("cuda:0")


@pytest.fixture(scope="module")
def cube():
    from oracle import oracle

    return oracle.color_cube_u8()


@pytest.fixture(scope="module")
def cube_oracle(cube):
    from oracle import oracle

    return oracle.decolor_u8(cube, threads=oracle.default_threads())


def _dev_decolor(torch, dev, arr, **kw):
    import paper_2108_13656_b200 as wg

    t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
    out = wg.decolor(t, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def test_cube_exhaustive(torch_dev, cube, cube_oracle):
    torch, dev = torch_dev
    got = _dev_decolor(torch, dev, cube)
    mx, frac = u8_mismatch(got, cube_oracle)
    print(f"cube u8: max diff {mx}, mismatch fraction {frac:.3e} ({int(frac * cube_oracle.size)} px)")
    assert mx <= 1 and frac <= U8_MAX_FRAC
    np.testing.assert_array_equal(_dev_decolor(torch, dev, cube, exact=True), cube_oracle)


def test_cube_matches_reference_hash_histogram(torch_dev, cube):
    import hashlib

    torch, dev = torch_dev
    got = _dev_decolor(torch, dev, cube, exact=True)
    with open(os.path.join(GOLDEN, "cube.json")) as f:
        ref = json.load(f)
    assert hashlib.sha256(got.tobytes()).hexdigest() == ref["compiled"]["gray_u8_sha256"]
    assert np.bincount(got.ravel(), minlength=256).tolist() == ref["compiled"]["gray_u8_histogram"]


def test_cube_custom_params(torch_dev, cube):
    import hashlib

    import paper_2108_13656_b200 as wg
    from oracle import oracle

    torch, dev = torch_dev
    got = _dev_decolor(torch, dev, cube, params=wg.DecolorParams(0.9, 0.6), exact=True)
    with open(os.path.join(GOLDEN, "cube.json")) as f:
        assert hashlib.sha256(got.tobytes()).hexdigest() == json.load(f)["compiled_b0.9_0.6_gray_u8_sha256"]
    for br, bk in [(0.500001, 0.999999), (0.75, 0.75), (0.99, 0.51)]:
        want = oracle.decolor_u8(cube, br, bk, threads=oracle.default_threads())
        np.testing.assert_array_equal(_dev_decolor(torch, dev, cube, params=wg.DecolorParams(br, bk), exact=True),
                                      want)
        mx, frac = u8_mismatch(_dev_decolor(torch, dev, cube, params=wg.DecolorParams(br, bk)), want)
        print(f"cube u8 beta=({br},{bk}): max {mx} frac {frac:.3e}")
        assert mx <= 1 and frac <= U8_MAX_FRAC


def test_exact_table_info():
    import ctypes

    from paper_2108_13656_b200 import _lib

    margin, slots, err, err_sq = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
    _lib.call("wg_u8_exact_info", 0.55, 0.8, ctypes.byref(margin), ctypes.byref(slots), ctypes.byref(err),
              ctypes.byref(err_sq))
    print(f"near-tie table: margin {margin.value} units of 2^-15, {slots.value} slots, max error {err.value} units, "
          f"square-domain max error {err_sq.value} float-bit units")
    assert 3 <= margin.value <= 16 and slots.value >= 1024
    assert 1 <= err.value <= 16  # the fast gray's exhaustive error bound (the exact tone map's margin - 2)
    assert 1 <= err_sq.value < 64  # the square-domain bound, within the tables' anchor reach
    with pytest.raises(ValueError):
        _lib.call("wg_u8_exact_info", 0.5, 0.8, None, None, None, None)


def test_c1_config(torch_dev):
    from paper_2108_13656_b200 import synth

    torch, dev = torch_dev
    c1 = synth.c1_image()
    got = _dev_decolor(torch, dev, c1)
    with open(os.path.join(GOLDEN, "c1.json")) as f:
        ref = json.load(f)
    import hashlib

    assert hashlib.sha256(c1.tobytes()).hexdigest() == ref["input_sha256"]
    from oracle import oracle

    mx, frac = u8_mismatch(got, oracle.decolor_u8(c1))
    assert mx <= 1 and frac <= U8_MAX_FRAC
    exact = _dev_decolor(torch, dev, c1, exact=True)
    assert hashlib.sha256(exact.tobytes()).hexdigest() == ref["gray_u8_sha256"]


def test_c3_full_size_images(torch_dev):
    """C3 (3840x2160 Voronoi) at full image size; 16 images spread over the batch."""
    from oracle import oracle
    from paper_2108_13656_b200 import synth

    torch, dev = torch_dev
    import paper_2108_13656_b200 as wg

    idx = np.linspace(0, 255, 16).astype(int)
    for i in idx:
        rgb = torch.empty((1, 2160, 3840, 3), dtype=torch.uint8, device=dev)
        synth.fill_voronoi_u8(rgb, seed=0, first_image=int(i))
        want = oracle.decolor_u8(rgb.cpu().numpy(), threads=oracle.default_threads())
        np.testing.assert_array_equal(wg.decolor(rgb, exact=True).cpu().numpy(), want)
        mx, frac = u8_mismatch(wg.decolor(rgb).cpu().numpy(), want)
        assert mx <= 1 and frac <= U8_MAX_FRAC


@pytest.mark.parametrize("npix", [0, 1, 7, 4095, 4096, 4097, 12345, 3 * 4096 + 17])
def test_ragged_sizes(torch_dev, npix):
    from oracle import oracle

    torch, dev = torch_dev
    rgb = np.random.default_rng(npix).integers(0, 256, (npix, 3), dtype=np.uint8)
    got = _dev_decolor(torch, dev, rgb)
    assert got.shape == (npix,)
    if npix:
        want = oracle.decolor_u8(rgb)
        mx, frac = u8_mismatch(got, want)
        assert mx <= 1
        np.testing.assert_array_equal(_dev_decolor(torch, dev, rgb, exact=True), want)


def test_misaligned_buffers_bit_identical(torch_dev):
    """Unaligned views take the scalar kernel; results must equal the vector path bit for bit."""
    import paper_2108_13656_b200 as wg

    torch, dev = torch_dev
    n = 50_000
    base = torch.from_numpy(np.random.default_rng(2).integers(0, 256, (n + 1, 3), dtype=np.uint8)).to(dev)
    aligned = wg.decolor(base[:n].contiguous())
    flat = base.reshape(-1)
    shifted = flat[3:].view(n, 3)  # 3-byte offset: not 16-B aligned
    assert shifted.data_ptr() % 16 != 0
    out = torch.empty(n + 1, dtype=torch.uint8, device=dev)
    wg.decolor(shifted, out=out[1:])  # misaligned output too
    torch.cuda.synchronize()
    ref = wg.decolor(base[1:].contiguous())
    assert torch.equal(out[1:], ref)
    assert torch.equal(aligned[1:], ref[:-1])
    # the exact variant: scalar path (with its table lookups) == vector path == oracle
    from oracle import oracle

    wg.decolor(shifted, out=out[1:], exact=True)
    want = oracle.decolor_u8(base[1:].cpu().numpy())
    np.testing.assert_array_equal(out[1:].cpu().numpy(), want)
    np.testing.assert_array_equal(wg.decolor(base[1:].contiguous(), exact=True).cpu().numpy(), want)


def test_shard_invariance(torch_dev):
    """Splitting a batch into shards (as across GPUs) gives bit-identical bytes."""
    import paper_2108_13656_b200 as wg
    from paper_2108_13656_b200 import sharder, synth

    torch, dev = torch_dev
    rgb = torch.empty((8, 270, 480, 3), dtype=torch.uint8, device=dev)
    synth.fill_voronoi_u8(rgb, seed=3)
    whole = wg.decolor(rgb)
    for world in (2, 4, 8):
        parts = [wg.decolor(rgb[a:b]) for a, b in (sharder.shard_range(8, world, r) for r in range(world))]
        assert torch.equal(torch.cat(parts), whole)


def test_host_pipeline_matches_device(torch_dev):
    import paper_2108_13656_b200 as wg

    torch, dev = torch_dev
    rgb = np.random.default_rng(9).integers(0, 256, (3, 1000, 1501, 3), dtype=np.uint8)
    host = wg.decolor_host(rgb)
    devv = _dev_decolor(torch, dev, rgb)
    assert np.array_equal(host, devv)


def test_host_calls_from_concurrent_threads(torch_dev):
    """Host-array calls from several threads at once (the reference drives
    decolor_rows from a thread pool, backend.py:65-81): each call leases its own
    context (streams + staging) from the device's pool, so they overlap and give
    the same bytes as sequential calls -- uint8 (pinned-style NumPy input), the
    fp64 drop-in on pageable buffers, and the HDR host path, interleaved."""
    import threading

    import paper_2108_13656_b200 as wg
    from paper_2108_13656_b200 import PlanarImage

    rng = np.random.default_rng(21)
    u8 = [rng.integers(0, 256, (301, 777 + 13 * i, 3), dtype=np.uint8) for i in range(6)]
    f64 = [rng.random((129, 211 + i, 3)) for i in range(4)]
    hdr = [(rng.random((2, 64, 96, 3)) * 100).astype(np.float32) for _ in range(2)]
    want_u8 = [wg.decolor_host(a) for a in u8]
    want_f64 = [wg.decolor_image(PlanarImage(a)).data for a in f64]
    want_hdr = [wg.hdr_tonemap_host(a) for a in hdr]
    got = {}
    errors = []

    def work(kind, i):
        try:
            for rep in range(3):
                if kind == "u8":
                    got[(kind, i, rep)] = wg.decolor_host(u8[i])
                elif kind == "f64":
                    got[(kind, i, rep)] = wg.decolor_image(PlanarImage(f64[i])).data
                else:
                    got[(kind, i, rep)] = wg.hdr_tonemap_host(hdr[i])
        except Exception as e:  # surfaced below
            errors.append(e)

    jobs = [("u8", i) for i in range(6)] + [("f64", i) for i in range(4)] + [("hdr", i) for i in range(2)]
    ts = [threading.Thread(target=work, args=j) for j in jobs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for (kind, i, rep), v in got.items():
        want = {"u8": want_u8, "f64": want_f64, "hdr": want_hdr}[kind][i]
        np.testing.assert_array_equal(v, want, err_msg=f"{kind} {i} rep {rep}")
    assert len(got) == 3 * len(jobs)


def test_generators_pinned(torch_dev):
    """Device generators equal their integer restatement in the oracle (C3, C5)."""
    from oracle import oracle
    from paper_2108_13656_b200 import synth

    torch, dev = torch_dev
    v = torch.empty((2, 48, 64, 3), dtype=torch.uint8, device=dev)
    synth.fill_voronoi_u8(v, seed=5, first_image=10)
    xy, col = synth.voronoi_tables(2, 48, 64, 200, 5, 10)
    assert np.array_equal(v.cpu().numpy(), oracle.synth_voronoi_u8(48, 64, xy, col, 5, 10))
    u = torch.empty((3, 20, 36, 3), dtype=torch.uint8, device=dev)
    synth.fill_uniform_u8(u, seed=7, first_image=4)
    assert np.array_equal(u.cpu().numpy(), oracle.synth_uniform_u8(3, 20, 36, 7, 4))
    u2 = torch.empty((2, 5, 7, 3), dtype=torch.uint8, device=dev)  # bytes/img not % 16
    synth.fill_uniform_u8(u2, seed=7, first_image=4)
    assert np.array_equal(u2.cpu().numpy(), oracle.synth_uniform_u8(2, 5, 7, 7, 4))


def test_tone_u8_cube(torch_dev, cube):
    import paper_2108_13656_b200 as wg
    from oracle import oracle

    torch, dev = torch_dev
    t = torch.from_numpy(cube).to(dev)
    # k = 200 / 2000: bins with several thresholds (the binary-search fallback); m = 0 / 1: one-sided curves
    for m, k in [(0.5, 8.0), (0.3, 12.0), (0.5, 1e-6), (0.5, 200.0), (0.6, 2000.0), (0.0, 3.0), (1.0, 3.0)]:
        toned, gray, _ = wg.decolor_tone(t, wg.SigmoidCurve(m, k), return_gray=True)
        want_t, want_g = oracle.tone_u8(cube, midpoint=m, slope=k, threads=oracle.default_threads(),
                                        with_gray=True)
        mx, frac = u8_mismatch(toned.cpu().numpy(), want_t)
        print(f"tone cube m={m} k={k}: max {mx} frac {frac:.3e}")
        assert mx <= 1 and frac <= U8_MAX_FRAC
        mx, frac = u8_mismatch(gray.cpu().numpy(), want_g)
        assert mx <= 1 and frac <= U8_MAX_FRAC
        # toned-only launch (the other kernel variant) gives the same bytes
        assert torch.equal(wg.decolor_tone(t, wg.SigmoidCurve(m, k)), toned)


def test_tone_u8_step_words_equal_bins(torch_dev, cube, monkeypatch):
    """The linear route's 32-bit step words (byte 3 of step + bits) give the
    same bytes as its 8-byte bins (count + float compare), over all 2^24
    colours, toned-only and with gray."""
    import paper_2108_13656_b200 as wg

    torch, dev = torch_dev
    t = torch.from_numpy(cube).to(dev)
    monkeypatch.setenv("WG_TONE_ROUTE", "linear")
    for m, k in [(0.5, 8.0), (0.3, 12.0), (0.5, 1e-6), (0.0, 3.0), (1.0, 3.0), (0.45, 60.0)]:
        curve = wg.SigmoidCurve(m, k)
        a = wg.decolor_tone(t, curve)
        ta, ga, _ = wg.decolor_tone(t, curve, return_gray=True)
        monkeypatch.setenv("WG_TONE_BINS64", "1")
        b = wg.decolor_tone(t, curve)
        tb, gb, _ = wg.decolor_tone(t, curve, return_gray=True)
        monkeypatch.delenv("WG_TONE_BINS64")
        assert torch.equal(a, b) and torch.equal(ta, tb) and torch.equal(ga, gb), (m, k)
        assert torch.equal(a, ta)


def test_tone_u8_routes_vs_oracle(torch_dev, cube, monkeypatch):
    """Both uint8 tone routes -- the square-domain step words (default: no
    final root, 1/S^2 from a table) and the linear step words -- meet the bar
    against the oracle over all 2^24 colours, toned and gray."""
    import paper_2108_13656_b200 as wg
    from oracle import oracle

    torch, dev = torch_dev
    t = torch.from_numpy(cube).to(dev)
    for m, k in [(0.5, 8.0), (0.3, 12.0), (0.5, 1e-6), (0.0, 3.0), (1.0, 3.0), (0.45, 60.0)]:
        want_t, want_g = oracle.tone_u8(cube, midpoint=m, slope=k, threads=oracle.default_threads(),
                                        with_gray=True)
        for route in ("square", "linear"):
            if route == "linear":
                monkeypatch.setenv("WG_TONE_ROUTE", "linear")
            toned, gray, _ = wg.decolor_tone(t, wg.SigmoidCurve(m, k), return_gray=True)
            monkeypatch.delenv("WG_TONE_ROUTE", raising=False)
            for name, got, want in (("toned", toned, want_t), ("gray", gray, want_g)):
                mx, frac = u8_mismatch(got.cpu().numpy(), want)
                print(f"tone route {route} m={m} k={k} {name}: max {mx} frac {frac:.3e}")
                assert mx <= 1 and frac <= U8_MAX_FRAC, (route, m, k, name)


def test_tone_rgb_u8_golden_and_cube(torch_dev, cube):
    """Colour output of the global tone map: bit-identical (fp64 chain per pixel)."""
    import paper_2108_13656_b200 as wg
    from oracle import oracle

    torch, dev = torch_dev
    g = np.load(os.path.join(GOLDEN, "tone_rgb.npz"))
    t = torch.from_numpy(g["u8"]).to(dev)
    for tag, curve, params in (("default", wg.SigmoidCurve(), wg.DEFAULT_PARAMS),
                               ("custom", wg.SigmoidCurve(0.3, 12.0), wg.DecolorParams(0.7, 0.9))):
        toned, _, out = wg.decolor_tone(t, curve, params, return_rgb=True)
        assert np.array_equal(out.cpu().numpy(), g[f"{tag}_rgb"])
        assert np.array_equal(toned.cpu().numpy(), g[f"{tag}_toned"])
    t = torch.from_numpy(cube).to(dev)
    # fp32 fast kernel + fp64 queue (1e-6 <= k <= 1e4): default, steep, flat, one-sided curves,
    # custom betas; k = 2e4 runs the all-fp64 kernel
    cases = [(0.5, 8.0, 0.55, 0.8), (0.3, 12.0, 0.7, 0.9), (0.6, 2000.0, 0.55, 0.8), (0.0, 3.0, 0.55, 0.8),
             (1.0, 3.0, 0.51, 0.99), (0.5, 1e-6, 0.55, 0.8), (0.5, 200.0, 0.95, 0.6), (0.4, 2e4, 0.55, 0.8)]
    for m, k, br, bk in cases:
        toned, gray, out = wg.decolor_tone(t, wg.SigmoidCurve(m, k), wg.DecolorParams(br, bk), return_gray=True,
                                           return_rgb=True)
        want_o, want_t, want_g = oracle.tone_rgb_u8(cube, br, bk, m, k, threads=oracle.default_threads())
        n_o = int((out.cpu().numpy() != want_o).sum())
        n_t = int((toned.cpu().numpy() != want_t).sum())
        n_g = int((gray.cpu().numpy() != want_g).sum())
        print(f"tone rgb cube m={m} k={k} betas {br}/{bk}: rgb diffs {n_o} toned diffs {n_t} gray diffs {n_g}")
        assert n_o == n_t == n_g == 0
    # exact toned / gray without the colour image (rgb_out null): the same bytes
    for m, k in [(0.5, 8.0), (0.6, 2000.0)]:
        toned_e, gray_e, none = wg.decolor_tone(t, wg.SigmoidCurve(m, k), return_gray=True, exact=True)
        assert none is None
        _, want_t, want_g = oracle.tone_rgb_u8(cube, midpoint=m, slope=k, threads=oracle.default_threads())
        assert np.array_equal(toned_e.cpu().numpy(), want_t) and np.array_equal(gray_e.cpu().numpy(), want_g)
    assert np.array_equal(wg.decolor_tone(t, exact=True).cpu().numpy(),
                          oracle.tone_rgb_u8(cube, threads=oracle.default_threads())[1])
    # toned-only request through the same kernel (gray pointer null)
    toned2, _, out2 = wg.decolor_tone(t, return_rgb=True)
    want_o, want_t, _ = oracle.tone_rgb_u8(cube, threads=oracle.default_threads())
    assert np.array_equal(out2.cpu().numpy(), want_o) and np.array_equal(toned2.cpu().numpy(), want_t)
    # unaligned device buffers (the all-fp64 kernel) and a ragged tail
    raw = torch.from_numpy(cube.reshape(-1)[: 5000 * 3 + 1].copy()).to(dev)
    sub = raw[1: 1 + 5000 * 3].view(5000, 3)
    toned3, _, out3 = wg.decolor_tone(sub, return_rgb=True)
    want_o, want_t, _ = oracle.tone_rgb_u8(cube.reshape(-1)[1: 1 + 5000 * 3].reshape(5000, 3))
    assert np.array_equal(out3.cpu().numpy(), want_o) and np.array_equal(toned3.cpu().numpy(), want_t)
    # host-buffer entry point, ragged size
    h = cube.reshape(-1, 3)[: 1000003]
    toned, gray, out = wg.decolor_tone_host(h, return_gray=True, return_rgb=True)
    want_o, want_t, want_g = oracle.tone_rgb_u8(h)
    assert np.array_equal(out, want_o) and np.array_equal(toned, want_t) and np.array_equal(gray, want_g)
    assert np.array_equal(wg.decolor_tone_host(h, exact=True), want_t)


def test_tone_rgb_u8_voronoi_frames(torch_dev):
    """C3-shape Voronoi frames (200 flat cells each): a cell whose colour is
    near a rounding tie sends thousands of consecutive pixels through the warp
    queues at once -- bytes still identical to the oracle."""
    import paper_2108_13656_b200 as wg
    from oracle import oracle
    from paper_2108_13656_b200 import synth

    torch, dev = torch_dev
    rgb = torch.empty((2, 2160, 3840, 3), dtype=torch.uint8, device=dev)
    synth.fill_voronoi_u8(rgb, seed=0, first_image=7)
    host = rgb.cpu().numpy()
    for m, k in [(0.5, 8.0), (0.45, 30.0)]:
        toned, gray, out = wg.decolor_tone(rgb, wg.SigmoidCurve(m, k), return_gray=True, return_rgb=True)
        want_o, want_t, want_g = oracle.tone_rgb_u8(host, midpoint=m, slope=k, threads=oracle.default_threads())
        assert np.array_equal(out.cpu().numpy(), want_o)
        assert np.array_equal(toned.cpu().numpy(), want_t) and np.array_equal(gray.cpu().numpy(), want_g)
    # a frame of the colour whose exact rgb value lies closest to a rounding
    # boundary (fp64 chain in NumPy): every pixel of it is queued
    cols = np.random.default_rng(4).integers(1, 256, (200_000, 3), dtype=np.uint8)
    c = cols.astype(np.float64) / 255.0
    li = oracle.decolor_f64(c)
    lo_, hi_ = 1.0 / (1.0 + np.exp(8.0 * 0.5)), 1.0 / (1.0 + np.exp(-8.0 * 0.5))
    lout = np.clip((1.0 / (1.0 + np.exp(-8.0 * (li - 0.5))) - lo_) / (hi_ - lo_), 0.0, 1.0)
    v = np.clip(c * (lout / li)[:, None], 0.0, 1.0) * 255.0
    dist = np.abs(v - np.floor(v) - 0.5).min(axis=1)
    pick = cols[int(np.argmin(dist))]
    print(f"nearest-tie colour {pick.tolist()} at {dist.min():.2e} from a boundary")
    flat = torch.empty((1, 512, 4096, 3), dtype=torch.uint8, device=dev)
    flat[:] = torch.from_numpy(pick).to(dev)
    _, _, fo = wg.decolor_tone(flat, return_rgb=True)
    want, _, _ = oracle.tone_rgb_u8(pick[None])
    assert (fo.view(-1, 3).cpu().numpy() == want[0]).all()


def test_exact_tone_routes_agree(torch_dev, cube, monkeypatch):
    """decolor_tone(u8, exact=True) without the colour image: the square-domain
    kernel with its exhaustively settled margin (tone_sq_exact_kernel, default),
    the linear threshold kernel (tone_u8_exact_kernel, WG_TONE_ROUTE=linear) and
    the colour kernel with rgb_out = NULL (WG_TONE_EXACT_VIA_RGB) give identical
    bytes -- toned-only and with gray, steep (multi-threshold bins) curves
    included -- and equal the oracle's (the reference's bytes)."""
    import paper_2108_13656_b200 as wg
    from oracle import oracle

    torch, dev = torch_dev
    t = torch.from_numpy(cube).to(dev)
    for curve in (wg.SigmoidCurve(), wg.SigmoidCurve(0.3, 12.0), wg.SigmoidCurve(0.0, 3.0),
                  wg.SigmoidCurve(0.2, 60.0), wg.SigmoidCurve(0.55, 500.0)):
        a, ga, _ = wg.decolor_tone(t, curve, return_gray=True, exact=True)
        a_only = wg.decolor_tone(t, curve, exact=True)
        want_t, want_g = oracle.tone_u8(cube, midpoint=curve.midpoint, slope=curve.slope,
                                        threads=oracle.default_threads(), with_gray=True)
        assert np.array_equal(a.cpu().numpy(), want_t) and np.array_equal(ga.cpu().numpy(), want_g), curve
        assert torch.equal(a_only, a)
        for env in ("WG_TONE_ROUTE", "WG_TONE_EXACT_VIA_RGB"):
            monkeypatch.setenv(env, "linear" if env == "WG_TONE_ROUTE" else "1")
            b, gb, _ = wg.decolor_tone(t, curve, return_gray=True, exact=True)
            monkeypatch.delenv(env)
            assert torch.equal(a, b) and torch.equal(ga, gb), (curve, env)
        monkeypatch.setenv("WG_TONE_EXACT_KERNEL", "1")  # toned only through the standalone kernel
        assert torch.equal(wg.decolor_tone(t, curve, exact=True), a)
        monkeypatch.delenv("WG_TONE_EXACT_KERNEL")


def test_exact_tone_voronoi_frames(torch_dev):
    """exact=True on 16 C3 frames (4K Voronoi) equals the oracle byte for byte."""
    import paper_2108_13656_b200 as wg
    from oracle import oracle
    from paper_2108_13656_b200 import synth

    torch, dev = torch_dev
    for first in (0, 120, 240):
        rgb = torch.empty((2, 2160, 3840, 3), dtype=torch.uint8, device=dev)
        synth.fill_voronoi_u8(rgb, seed=0, first_image=first)
        toned, gray, _ = wg.decolor_tone(rgb, return_gray=True, exact=True)
        want_t, want_g = oracle.tone_u8(rgb.cpu().numpy(), threads=oracle.default_threads(), with_gray=True)
        assert np.array_equal(toned.cpu().numpy(), want_t) and np.array_equal(gray.cpu().numpy(), want_g)


def test_tone_rgb_u8_bound_headroom(torch_dev, cube, monkeypatch):
    """The fast kernel's error bound with every margin halved still settles
    only correct bytes over all 2^24 colours: the first-order budget has at
    least 2x headroom on the realised fp32 errors (csrc/wg_tone.cu)."""
    import paper_2108_13656_b200 as wg
    from oracle import oracle

    torch, dev = torch_dev
    monkeypatch.setenv("WG_TONE_RGB_MARGIN_SCALE", "0.5")
    t = torch.from_numpy(cube).to(dev)
    for m, k, br, bk in [(0.5, 8.0, 0.55, 0.8), (0.3, 12.0, 0.7, 0.9), (0.6, 200.0, 0.9, 0.6)]:
        toned, gray, out = wg.decolor_tone(t, wg.SigmoidCurve(m, k), wg.DecolorParams(br, bk), return_gray=True,
                                           return_rgb=True)
        want_o, want_t, want_g = oracle.tone_rgb_u8(cube, br, bk, m, k, threads=oracle.default_threads())
        n = [int((a.cpu().numpy() != b).sum()) for a, b in ((out, want_o), (toned, want_t), (gray, want_g))]
        print(f"tone rgb half margins m={m} k={k}: diffs {n}")
        assert n == [0, 0, 0]


def test_table_caches_under_concurrent_eviction(torch_dev):
    """Threads on their own streams cycle through more tone curves (cache of 8)
    and exact-u8 parameter pairs (cache of 4) than the per-device caches hold:
    a table stays alive until the launch that uses it is enqueued, so every
    result equals the single-threaded one."""
    import threading

    import paper_2108_13656_b200 as wg

    torch, dev = torch_dev
    rgb = torch.randint(0, 256, (64, 1024, 3), dtype=torch.uint8, device=dev)
    curves = [wg.SigmoidCurve(0.3 + 0.02 * i, 4.0 + i) for i in range(12)]
    pairs = [wg.DecolorParams(0.55 + 0.03 * i, 0.8 - 0.02 * i) for i in range(6)]
    want_t = [wg.decolor_tone(rgb, c) for c in curves]
    want_e = [wg.decolor(rgb, p, exact=True) for p in pairs]
    torch.cuda.synchronize()
    errors = []

    def worker(seed):
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            for it in range(8):
                i = (seed * 5 + it) % len(curves)
                j = (seed * 3 + it) % len(pairs)
                t = wg.decolor_tone(rgb, curves[i], stream=s)
                e = wg.decolor(rgb, pairs[j], exact=True, stream=s)
                s.synchronize()
                if not torch.equal(t, want_t[i]) or not torch.equal(e, want_e[j]):
                    errors.append((seed, it))

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors


def test_empty_and_errors(torch_dev):
    import paper_2108_13656_b200 as wg

    torch, dev = torch_dev
    e = torch.empty((0, 3), dtype=torch.uint8, device=dev)
    assert wg.decolor(e).shape == (0,)
    with pytest.raises(ValueError):
        wg.decolor(torch.zeros((4, 4), dtype=torch.uint8, device=dev))
    with pytest.raises(ValueError):
        wg.decolor(torch.zeros((4, 3), dtype=torch.int32, device=dev))
    from paper_2108_13656_b200 import _lib

    with pytest.raises(ValueError):
        _lib.call("wg_decolor_u8", e.data_ptr(), e.data_ptr(), 5, 0.5, 0.8, None)
