"""Device-resident per-method throughput (the paper's Table 1 comparison on B200).

Times wg_decolor_u8 ("ours") against the baseline extractors (wg_luma_u8:
y / v / lab), the tone maps and the colour tone map (tone_rgb: 3 B in,
3 B rgb + 1 B toned out per pixel) on the same uint8 batch already in HBM, CUDA events on the
launching stream, inputs larger than L2. Prints one JSON line per method.

    python scripts/bench_methods.py [--mpix 512] [--iters 50]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2108_13656_b200 as wg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mpix", type=int, default=512)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--methods", default="ours,tone,y,v,lab,local")
    args = ap.parse_args()
    # 4K frames (C3 shape) so the tiled local tone map sees real images
    nimg = max(1, (args.mpix << 20) // (2160 * 3840))
    n = nimg * 2160 * 3840
    rgb4 = torch.randint(0, 256, (nimg, 2160, 3840, 3), dtype=torch.uint8, device="cuda")
    rgb = rgb4.view(n, 3)
    scratch = torch.empty(int(wg._lib.load().wg_lhe_scratch_bytes(nimg, 2160, 3840, 480, 270, 256)),
                          dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.uint8, device="cuda")
    peaks = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
    hbm = peaks.get("hbm_gbs", 6545.3)
    fns = {
        "ours": lambda: wg.decolor(rgb, out=out.view(n)),
        "tone": lambda: wg.decolor_tone(rgb),
        "tone_rgb": lambda: wg.decolor_tone(rgb, return_rgb=True),
        "tone_exact": lambda: wg.decolor_tone(rgb, exact=True),
        "y": lambda: wg.luma(rgb, "y"),
        "v": lambda: wg.luma(rgb, "v"),
        "lab": lambda: wg.luma(rgb, "lab"),
        "local": lambda: wg.decolor_tone_local(rgb4, scratch=scratch),
    }
    for name in args.methods.split(","):
        fn = fns[name]
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.iters
        gbps = (7 if name == "tone_rgb" else 4) * n / ms / 1e6  # algorithmic bytes per pixel
        print(json.dumps({"method": name, "npix": n, "ms": round(ms, 4), "gpix_s": round(n / ms / 1e6, 1),
                          "per_pixel_ps": round(ms * 1e9 / n, 3), "gbps": round(gbps, 1),
                          "frac_hbm": round(gbps / hbm, 3)}))


if __name__ == "__main__":
    main()
