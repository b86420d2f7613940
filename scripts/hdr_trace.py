"""Timeline of the HDR tensor-memory kernel on C4 (diagnostic).

Runs wg.hdr_tonemap with WG_HDR_TMDBG=4 (the kernel records, per image and
CTA, globaltimer at producer start / publish and consumer start / done) and
prints per-image summaries: producer duration spread over CTAs, the skew of
the publish times, the consumer wait and tone times.

    python scripts/hdr_trace.py [--images 32] [--runs 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_13656_b200 as wg  # noqa: E402
from paper_2108_13656_b200 import _lib, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=32)
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--mode", default="4", help="WG_HDR_TMDBG value (4 = trace; +8 stat by one thread, +16 fp32 thresholds)")
    ap.add_argument("--ring", default="2", help="WG_HDR_TMRING (2 or 3 slots)")
    ap.add_argument("--summary", action="store_true", help="print only the summary line and image 1")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    wl = synth.WORKLOADS["C4"]
    rgb = synth.make_batch(wl, dev, n_images=args.images)
    out = torch.empty(rgb.shape[:-1], dtype=torch.uint8, device=dev)
    os.environ["WG_HDR_TMDBG"] = args.mode
    os.environ["WG_HDR_TMRING"] = args.ring
    lib = _lib.load()
    n = lib.wg_hdr_debug_trace(None)
    buf = np.zeros(n, dtype=np.uint64)
    for _ in range(args.runs):
        wg.hdr_tonemap(rgb, out=out)
    torch.cuda.synchronize()
    lib.wg_hdr_debug_trace(buf.ctypes.data)
    tr = buf.reshape(64, 1024, 7)[: args.images].astype(np.int64)
    ncta = int((tr[0, :, 0] > 0).sum())
    tr = tr[:, :ncta, :]
    t0 = tr[0, :, 0].min()
    tr = tr - t0
    for i in range(args.images):
        if args.summary and i != 1:
            continue
        ps, pp, cs, cd, ct, cf, cl = (tr[i, :, k] for k in range(7))
        dur = pp - ps
        print(json.dumps({
            "img": i, "prod_start_us": [round(ps.min() / 1e3, 2), round(ps.max() / 1e3, 2)],
            "prod_dur_us": [round(dur.min() / 1e3, 2), round(np.median(dur) / 1e3, 2), round(dur.max() / 1e3, 2)],
            "publish_skew_us": round((pp.max() - pp.min()) / 1e3, 2),
            "cons_start_after_last_publish_us": round((cs.min() - pp.max()) / 1e3, 2),
            "cons_dur_us": [round((cd - cs).min() / 1e3, 2), round(np.median(cd - cs) / 1e3, 2),
                            round((cd - cs).max() / 1e3, 2)],
            "cons_fold_us": round(float(np.median(cf - cs)) / 1e3, 2),
            "cons_stat_us": round(float(np.median(cl - cf)) / 1e3, 2),
            "cons_table_us": round(float(np.median(ct - cl)) / 1e3, 2),
            "cons_tone_us": round(float(np.median(cd - ct)) / 1e3, 2),
            "slowest_cta": int(dur.argmax()),
        }))
    total = (tr[args.images - 1, :, 3].max() - tr[0, :, 0].min()) / 1e3
    dur_all = tr[:, :, 1] - tr[:, :, 0]
    slow = np.bincount(dur_all.argmax(axis=1), minlength=ncta)
    print(json.dumps({"mode": args.mode, "ring": args.ring, "total_us": round(total, 1), "gpix_s": round(args.images * wl.height * wl.width / total / 1e3, 1),
                      "ctas": ncta, "most_often_slowest": [int(x) for x in np.argsort(-slow)[:8]],
                      "per_cta_mean_prod_us_minmax": [round(dur_all.mean(0).min() / 1e3, 2),
                                                      round(dur_all.mean(0).max() / 1e3, 2)]}))


if __name__ == "__main__":
    main()
