"""Locate mismatches between the tiled and the grid-stride HDR tone kernels."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CODE = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2108_13656_b200 as wg
from paper_2108_13656_b200 import synth
rgb = torch.empty((4, 2048, 2048, 3), dtype=torch.float32, device='cuda')
synth.fill_hdr_f32(rgb, seed=0)
out = wg.hdr_tonemap(rgb).cpu().numpy()
np.save(sys.argv[1], out)
""" % ROOT

a, b = "/tmp/hdr_tiled.npy", "/tmp/hdr_plain.npy"
subprocess.run([sys.executable, "-c", CODE, a], check=True)
subprocess.run([sys.executable, "-c", CODE, b], check=True, env={**os.environ, "WG_HDR_NO_TILED": "1"})
x, y = np.load(a).reshape(4, -1), np.load(b).reshape(4, -1)
bad = np.argwhere(x != y)
print("mismatches", len(bad))
for img, p in bad[:40]:
    print(f"img {img} px {p} tile {p // 4096} off {p % 4096} (float4 {p % 4096 // 4}) tiled {x[img, p]} plain {y[img, p]}")
tiles = sorted(set((int(i), int(p // 4096)) for i, p in bad))
print("distinct (img, tile):", tiles[:40], len(tiles))
