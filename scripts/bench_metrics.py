"""Pair-count throughput of the contrast metrics.

Exhaustive CCPR/CCFR counting (all n(n-1)/2 pairs, 15 taus) on the device via
the C ABI (device buffers, CUDA events), against the CPU oracle (all host
cores) on a smaller image, in pairs per second.

    python scripts/bench_metrics.py [--side 256] [--cpu-side 64]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--cpu-side", type=int, default=64)
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()

    import paper_2108_13656_b200 as wg
    from paper_2108_13656_b200 import _lib
    from oracle import oracle

    n = args.side * args.side
    rng = np.random.default_rng(0)
    rgb = rng.integers(0, 256, (n, 3)).astype(np.float64) / 255.0
    gray = wg.luminance_image(wg.PlanarImage(rgb.reshape(args.side, args.side, 3))).data.reshape(n)
    taus = np.arange(1, 16, dtype=np.float64)
    d_rgb = torch.from_numpy(rgb).cuda()
    d_gray = torch.from_numpy(gray).cuda()
    hist = torch.zeros(16 * 16, dtype=torch.int64, device="cuda")
    sb = int(_lib.load().wg_metric_scratch_bytes(n))
    scratch = torch.empty(sb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def run():
        _lib.call("wg_metric_hist_f64", d_rgb.data_ptr(), d_gray.data_ptr(), n, taus.ctypes.data, 15, None, None, 0,
                  hist.data_ptr(), scratch.data_ptr(), sb, st)

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    pairs = n * (n - 1) // 2
    print(json.dumps({"variant": "gpu_exhaustive", "pixels": n, "pairs": pairs, "ms": round(ms, 3),
                      "gpairs_s": round(pairs / ms / 1e6, 2)}))

    m = args.cpu_side * args.cpu_side
    crgb = rgb[:m]
    cgray = gray[:m]
    threads = oracle.default_threads()
    t0 = time.perf_counter()
    oracle.metric_counts(crgb, cgray, taus, None, threads=threads)
    secs = time.perf_counter() - t0
    cp = m * (m - 1) // 2
    print(json.dumps({"variant": "cpu_oracle_exhaustive", "pixels": m, "pairs": cp, "seconds": round(secs, 3),
                      "gpairs_s": round(cp / secs / 1e9, 4), "cores": threads}))


if __name__ == "__main__":
    main()
