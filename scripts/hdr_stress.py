"""Stress the HDR persistent kernels against the grouped schedule (an
independent implementation of the same bytes): random batch shapes, repeated
calls on one scratch buffer, the TMEM kernel, its shared-memory third slot and
the L2-ring variant. Any byte difference is a race or a slot-handoff bug.

    python scripts/hdr_stress.py [--iters 100] [--seed 0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_13656_b200 as wg  # noqa: E402
from paper_2108_13656_b200 import synth  # noqa: E402


def run(rgb, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return wg.hdr_tonemap(rgb)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    dev = torch.device("cuda", 0)
    variants = {"tmem": {}, "tmem+smem": {"WG_HDR_TMRING": "3"}, "ring": {"WG_HDR_TMEM": "0"}}
    bad = 0
    for it in range(args.iters):
        nimg = int(rng.integers(1, 13))
        w = 32 * int(rng.integers(1, 65))
        h = int(rng.integers(1, max(2, 4_900_000 // w)))  # up to just over one TMEM slot per SM
        rgb = torch.empty((nimg, h, w, 3), dtype=torch.float32, device=dev)
        synth.fill_hdr_f32(rgb, seed=int(rng.integers(0, 1 << 30)))
        if rng.random() < 0.2:
            rgb[int(rng.integers(0, nimg))] = float(rng.random())  # a constant image
        ref = run(rgb, {"WG_HDR_SCHEDULE": "grouped"})
        for name, env in variants.items():
            got = run(rgb, env)
            if not torch.equal(got, ref):
                bad += 1
                n = int((got != ref).sum())
                print(f"iter {it}: {name} differs on {n} px (nimg {nimg}, {h}x{w})", flush=True)
    torch.cuda.synchronize()
    print(f"hdr_stress: {args.iters} batches x {len(variants)} variants, {bad} mismatching", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
