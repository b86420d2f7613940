"""Localise u8 local-tone mismatches: u8 fused path vs the fp64 device chain vs the oracle."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_13656_b200 as wg  # noqa: E402
from oracle import oracle  # noqa: E402

n, h, w = 2, 1080, 1920
rng = np.random.default_rng(h * w)
rgb = rng.integers(0, 256, (n, h, w, 3), dtype=np.uint8)
rgb[0, : h // 3] = rgb[0, : h // 3] // 16 * 16
g = wg.LocalHistogramGrid.for_image(w, h)
for strength in (0.0, 0.7):
    gg = wg.LocalHistogramGrid(g.tile_w, g.tile_h, g.bins, strength)
    toned, gray = wg.decolor_tone_local(torch.from_numpy(rgb).cuda(), grid=gg, return_gray=True)
    toned, gray = toned.cpu().numpy(), gray.cpu().numpy()
    want_t, want_g = oracle.tone_local_u8(rgb, gg.tile_w, gg.tile_h, gg.bins, gg.strength, threads=2, with_gray=True)
    # fp64 device chain
    chain = []
    for k in range(n):
        x = wg.dequantize_u8(rgb[k])
        l_in = wg.decolor_image(wg.PlanarImage(x))
        lo = wg.apply_local_lhe(l_in, gg)
        chain.append(wg.quantize_u8(lo.data))
    chain = np.stack(chain)
    for name, a, b in (("gray u8 vs oracle", gray, want_g), ("toned u8 vs oracle", toned, want_t),
                       ("f64 chain vs oracle", chain, want_t), ("toned u8 vs chain", toned, chain)):
        d = np.abs(a.astype(int) - b.astype(int))
        idx = np.argwhere(d > 0)
        print(f"s={strength} {name}: mismatches {len(idx)} max {d.max()}", idx[:5].tolist())
    bad = np.argwhere(toned != want_t)
    if len(bad):
        imgs, ys, xs = bad[:, 0], bad[:, 1], bad[:, 2]
        print("images", np.bincount(imgs), "tiles y", np.bincount(ys // gg.tile_h), "tiles x",
              np.bincount(xs // gg.tile_w))
        for k, y, x in bad[:8]:
            p = rgb[k, y, x]
            v = oracle.decolor_f64(p[None].astype(np.float64) / 255.0)[0]
            print("px", k, y, x, "rgb", p.tolist(), "v", repr(v), "v*256", v * 256, "got", toned[k, y, x],
                  "want", want_t[k, y, x])
