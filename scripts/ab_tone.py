"""A/B of uint8 kernel variants (tuning knobs set through the environment)
against the default decolor kernel on the C3 batch (256 Voronoi 4K frames,
device-generated), CUDA events.

    python scripts/ab_tone.py [--op tone|decolor|tone_exact|local] [--images 256] [--iters 20] [--rounds 3]
        [--sleep 2] [--configs "ROUTE=linear;GRID=20"]

Each config sets WG_TONE_ROUTE / WG_LDG_GRID_PER_SM for
the library calls; rounds interleave the default decolor and every config
(with --sleep seconds between measurements so the board's power average
recovers); the median is printed, and each config's output is compared
with the default call's bytes.
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2108_13656_b200 as wg  # noqa: E402
from paper_2108_13656_b200 import synth  # noqa: E402

KEYS = {"GRID": "WG_LDG_GRID_PER_SM", "ROUTE": "WG_TONE_ROUTE", "XK": "WG_TONE_EXACT_KERNEL",
        "LP": "WG_LHE_PLANE", "PF": "WG_HDR_PF", "SCHED": "WG_HDR_SCHEDULE", "RING": "WG_HDR_RING_MB", "TM": "WG_HDR_TMEM", "TMDBG": "WG_HDR_TMDBG", "RING3": "WG_HDR_TMRING", "PACKED": "WG_HDR_PACKED"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=256)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--configs", default="ROUTE=linear")
    ap.add_argument("--op", default="tone", choices=("tone", "decolor", "tone_exact", "local", "hdr", "rgb"))
    ap.add_argument("--sleep", type=float, default=0.0)
    ap.add_argument("--lib", default=None, help="load this build of the library (cross-build A/B)")
    args = ap.parse_args()
    if args.lib:
        wg._lib.load(args.lib)
    dev = torch.device("cuda", 0)
    if args.op == "hdr":
        args.workload = "C4"
    wl = synth.WORKLOADS[args.workload]
    rgb = synth.make_batch(wl, dev, n_images=args.images)
    out = torch.empty(rgb.shape[:-1], dtype=torch.uint8, device=dev)
    img4 = rgb.view(args.images, wl.height, wl.width, 3)
    grid = wg.LocalHistogramGrid.for_image(wl.width, wl.height)
    scratch = None
    if args.op == "local":
        scratch = torch.empty(int(wg._lib.load().wg_lhe_scratch_bytes(args.images, wl.height, wl.width, grid.tile_w,
                                                                      grid.tile_h, grid.bins)),
                              dtype=torch.uint8, device=dev)
    op = {"tone": lambda: wg.decolor_tone(rgb, out=out), "decolor": lambda: wg.decolor(rgb, out=out),
          "tone_exact": lambda: wg.decolor_tone(rgb, out=out, exact=True),
          "hdr": lambda: wg.hdr_tonemap(rgb, out=out),
          "rgb": lambda: wg.decolor_tone(rgb, return_rgb=True, out=out)[0],
          "local": lambda: wg.decolor_tone_local(img4, grid=grid, scratch=scratch,
                                                 out=out.view(args.images, wl.height, wl.width))}[args.op]
    tone_ref = op().clone()
    npx = out.numel()
    configs = [dict(kv.split("=") for kv in c.split(",") if kv) for c in args.configs.split(";")]

    def timed(fn):
        if args.sleep:
            torch.cuda.synchronize()
            time.sleep(args.sleep)
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return npx / (e0.elapsed_time(e1) / args.iters) / 1e6

    def setenv(cfg):
        for k, v in KEYS.items():
            os.environ.pop(v, None)
        for k, v in cfg.items():
            os.environ[KEYS[k]] = v

    res = {"decolor": []}
    gray = torch.empty(rgb.shape[:-1], dtype=rgb.dtype, device=dev) if args.op == "hdr" else out
    for r in range(args.rounds):
        setenv({})
        res["decolor"].append(timed(lambda: wg.decolor(rgb, out=gray)))
        for cfg in configs:
            setenv(cfg)
            name = ",".join(f"{k}={v}" for k, v in cfg.items()) or "default"
            res.setdefault(name, []).append(timed(op))
            if r == 0:
                diff = (out.view(-1).int() - tone_ref.view(-1).int()).abs()
                print(json.dumps({"config": name, "vs_default_max": int(diff.max()),
                                  "vs_default_frac": float((diff > 0).float().mean())}))
    setenv({})
    base = statistics.median(res["decolor"])
    for name, v in res.items():
        m = statistics.median(v)
        print(json.dumps({"kernel": name, "gpix_s": round(m, 1), "vs_decolor": round(m / base, 3),
                          "frac": round(m * {"hdr": 13, "rgb": 7}.get(args.op, 4) / 6454.6, 3), "all": [round(x, 1) for x in v]}))


if __name__ == "__main__":
    main()
