#!/usr/bin/env python
"""Benchmark: decolorized Gpixels/s on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3] [--impl ours|reference]

A "step" is one pass of the hot path over one batch resident in HBM:
workload C3 (BASELINE.json configs[2], the graded 4K batch) = 256 RGB u8
images of 3840x2160 -> u8 gray per GPU, one kernel launch per step. Under
torchrun (N > 1) every rank decolorizes its own 256-image shard (images are
independent: weak scaling, no collective on the data path); the step time is
the max over ranks of the CUDA-event time.

Keys beyond the base contract:
  roofline      algorithmic bytes per launch (4 B/px for u8->u8) / mean launch
                duration from CUDA events on the launching stream, against
                MEASURED_PEAKS.json hbm_gbs; traffic = ncu dram bytes / launch
                from profiles/ when a capture for this workload is committed.
  cpu_baseline  the reference's own CPU path on all host cores, rank 0 at N=1,
                over a bounded sample of the same workload: its _kernels.pyx
                compiled into oracle/_ref by oracle/build_ref.py, driven as
                decolor_image / dequantize_u8 / quantize_u8 do (kind
                "reference", plus kernel_only_gpix_s); the oracle port
                (oracle/warmgray_oracle.c, bit-identical) where that is not
                built or for the HDR adapter, which the reference lacks.
  e2e           the same metric through the public host-array API
                (paper_2108_13656_b200.decolor_host -> wg_host_decolor_u8):
                pinned host input -> H2D -> kernel -> D2H every step.
  clocks        NVML SM clock / throttle reasons sampled during the timed region.

--impl reference: the same reference CPU path (kind "reference" when
oracle/_ref is built -- it travels to the GPU box with the snapshot --, else
the bit-identical oracle port) on every host core, timed on the same
workload/metric; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "decolorized Gpixels/s (device-timed) at 1/2/4/8 B200; % of HBM roofline"
L2_BYTES = 126 * 2 ** 20


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------------ clocks (NVML, during timed region)
_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
            0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz, self.ok = [], 0, None, False
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _reasons(self):
        nv = self.nv
        for name in ("nvmlDeviceGetCurrentClocksEventReasons", "nvmlDeviceGetCurrentClocksThrottleReasons"):
            fn = getattr(nv, name, None)
            if fn is not None:
                try:
                    return fn(self.h)
                except Exception:
                    continue
        return 0

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self._reasons())
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        names = [n for bit, n in _REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU legs
def reference_fns(workload, threads: int):
    """The reference's own CPU path for this workload, when its compiled kernels
    are present (oracle/_ref, built from /root/reference by oracle/build_ref.py):
    returns (end-to-end fn, kernel-only fn, label) or None.

    End to end is what the reference's public API does for the metric: codec.py's
    dequantize_u8 (u8 workloads), PlanarImage's validation (core.py:69-80),
    core.decolor_image -- _kernels.decolor_rows over contiguous row chunks on a
    thread pool of `threads` workers created per call (backend.run_rows) -- the
    validation of the result, and quantize_u8 (or the fp32 cast). Kernel only
    is decolor_rows over the same row chunks on pre-converted fp64 input.
    The HDR adapter (C4) has no reference implementation: None.
    """
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from oracle import build_ref

    if workload.output not in ("gray_u8", "gray_f32"):
        return None
    try:
        k = build_ref.load()
    except ImportError:
        return None

    def validate(a):  # PlanarImage.__init__
        if a.size and (not np.isfinite(a).all() or a.min() < 0.0 or a.max() > 1.0):
            raise ValueError("image samples must lie in [0, 1]")

    def run_rows(f, out):  # backend.run_rows: contiguous chunks, one pool per call
        h = f.shape[0]
        workers = max(1, min(threads, h))
        chunk = -(-h // workers)
        spans = [(r0, min(r0 + chunk, h)) for r0 in range(0, h, chunk)]
        with ThreadPoolExecutor(max_workers=len(spans)) as pool:
            list(pool.map(lambda sp: k.decolor_rows(f, out, 0.55, 0.8, sp[0], sp[1]), spans))

    def decolor_image(f):
        out = np.empty(f.shape[:2], dtype=np.float64)
        run_rows(f, out)
        validate(out)  # the returned PlanarImage
        return out

    if workload.output == "gray_u8":
        def e2e(batch):
            for img in batch:
                f = img.astype(np.float64) / 255.0  # dequantize_u8
                validate(f)
                np.floor(np.clip(decolor_image(f), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)  # quantize_u8
    else:
        def e2e(batch):
            for img in batch:
                f = np.ascontiguousarray(img, dtype=np.float64)
                validate(f)
                decolor_image(f).astype(np.float32)
    cache = {}

    def kernel(batch):
        f = cache.get(id(batch))
        if f is None:
            f = cache[id(batch)] = [np.ascontiguousarray(img, dtype=np.float64) / (255.0 if img.dtype == np.uint8 else 1.0)
                                    for img in batch]
        for x in f:
            run_rows(x, np.empty(x.shape[:2], dtype=np.float64))
    return e2e, kernel, ("the reference's _kernels.pyx compiled by oracle/build_ref.py (cython + gcc -O3 as "
                         "setup.py), driven as decolor_image / dequantize_u8 / quantize_u8 do")


def _rate(fn, rgb, seconds):
    fn(rgb[:1])  # warm-up
    px = 0
    t0 = time.perf_counter()
    while True:
        fn(rgb)
        px += rgb.size // 3
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return px / el / 1e9, el, px


def cpu_port_rate(workload, seconds: float = 10.0, max_images: int = 4):
    """Gpix/s of the reference's CPU path on all host cores: its compiled kernels
    (oracle/_ref) when built, else the oracle port (fp64 scalar, bit-identical).
    Returns (rate, threads, sample description, kind, extra)."""
    from oracle import oracle

    threads = oracle.default_threads()
    rgb, desc = cpu_sample(workload, max_images)
    ref = reference_fns(workload, threads)
    if ref is not None:
        e2e, kernel, label = ref
        rate, el, px = _rate(e2e, rgb, seconds)
        krate, _, _ = _rate(kernel, rgb, min(seconds, 5.0))
        return (rate, threads, f"{desc}, repeated for {el:.1f} s ({px / 1e6:.0f} Mpx); {label}", "reference",
                {"kernel_only_gpix_s": round(krate, 4)})
    fn = {"gray_u8": lambda x: oracle.decolor_u8(x, threads=threads),
          "gray_f32": lambda x: oracle.decolor_f32in(x, threads=threads),
          "hdr_u8": lambda x: oracle.hdr_u8(x, threads=threads)}[workload.output]
    rate, el, px = _rate(fn, rgb, seconds)
    return rate, threads, f"{desc}, repeated for {el:.1f} s ({px / 1e6:.0f} Mpx)", "port", {}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample(workload, n: int):
    """A bounded sample of the workload's input, generated on the host."""
    import numpy as np

    from oracle import oracle
    from paper_2108_13656_b200 import synth

    h, w = workload.height, workload.width
    n = min(n, workload.n_images)
    if workload.name == "C1":
        return synth.c1_image()[None], "C1 512x512 u8"
    if workload.name == "C3":
        xy, col = synth.voronoi_tables(n, h, w)
        return oracle.synth_voronoi_u8(h, w, xy, col, 0), f"{n} C3 images {w}x{h} u8 (host Voronoi)"
    if workload.name == "C5":
        return oracle.synth_uniform_u8(n, h, w, 0), f"{n} C5 images {w}x{h} u8"
    rng = np.random.default_rng(0)
    if workload.name == "C4":
        lum = 10.0 ** rng.uniform(-3, 4, (n, h, w))
        chroma = rng.random((n, h, w, 3))
        y = chroma @ np.array([0.2126, 0.7152, 0.0722])
        return (chroma * (lum / np.maximum(y, 1e-6))[..., None]).astype(np.float32), \
            f"{n} C4-like HDR images {w}x{h} f32"
    return rng.random((n, h, w, 3), dtype=np.float32), f"{n} C2-size images {w}x{h} f32 (uniform)"


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="C3", choices=("C1", "C2", "C3", "C4", "C5"))
    ap.add_argument("--images", type=int, default=None, help="images per GPU (default: workload's)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="C5: skip the per-GPU size sweep (256x256 .. 8K at fixed total pixels)")
    ap.add_argument("--no-methods", action="store_true",
                    help="skip the per-method side table (paper Table 1 on the GPU + local tone map)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()

    from paper_2108_13656_b200.synth import WORKLOADS

    wl = WORKLOADS[args.workload]
    rank, world, local = dist_env()
    warmup = max(args.warmup, 3)
    steps = max(args.steps, 1)

    if args.impl == "reference":
        if rank != 0:
            return
        run_reference(args, wl, steps, warmup, world)
        return

    import numpy as np
    import torch

    import paper_2108_13656_b200 as wg
    from paper_2108_13656_b200 import synth

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    wg.set_device(local)
    group = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    n_img = args.images or wl.n_images
    rgb = synth.make_batch(wl, dev, n_images=n_img, seed=0, first_image=rank * n_img)
    torch.cuda.synchronize()
    out_dtype = torch.float32 if wl.output == "gray_f32" else torch.uint8
    out = torch.empty(rgb.shape[:-1], dtype=out_dtype, device=dev)
    scratch = wg.HdrScratch(n_img, wl.pix_per_image, device=dev) if wl.output == "hdr_u8" else None

    def step():
        if wl.output == "hdr_u8":
            wg.hdr_tonemap(rgb, scratch=scratch, out=out)
        else:
            wg.decolor(rgb, out=out)

    if wl.output == "hdr_u8":
        # wg_hdr.cu: gray + stats + tone per group of images whose gray plane fits 128 MiB
        group = max(1, min(32, n_img))
        launches_per_step = 3 * (-(-n_img // group))
    else:
        launches_per_step = 1
    in_bytes = rgb.numel() * rgb.element_size()
    flush = None
    if in_bytes < 4 * L2_BYTES:  # small batches: flush L2 between timed steps
        flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    stream = torch.cuda.current_stream(dev)
    if flush is None:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            ev0.record(stream)
            for _ in range(steps):
                step()
            ev1.record(stream)
            torch.cuda.synchronize()
        barrier()
        elapsed_ms = ev0.elapsed_time(ev1)
    else:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            for a, b in evs:
                flush.zero_()
                a.record(stream)
                step()
                b.record(stream)
            torch.cuda.synchronize()
        barrier()
        elapsed_ms = sum(a.elapsed_time(b) for a, b in evs)

    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    per_rank = [elapsed_ms]
    if world > 1:
        allt = torch.zeros(world, dtype=torch.float64, device=dev)
        torch.distributed.all_gather_into_tensor(allt, t)
        per_rank = allt.cpu().tolist()
    max_ms = max(per_rank)
    px_step = n_img * wl.pix_per_image
    value = world * px_step * steps / (max_ms / 1e3) / 1e9
    ms_per_step = max_ms / steps

    peak, peak_src = peaks()
    achieved = wl.bytes_per_px * px_step / (elapsed_ms / steps / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": committed_traffic(wl.name),
                "bytes_per_px": wl.bytes_per_px, "peak_source": peak_src,
                # the measured peak is a 1:1 copy; read-dominant streams (3:1 for the fp32
                # path) can exceed it, so the fraction of the 8 TB/s HBM3e spec is given too
                "frac_vs_spec_8000": round(achieved / 8000.0, 4),
                "kernel": "ldg_stream_kernel<OpDecolorU8>" if wl.dtype == "uint8" and wl.output == "gray_u8"
                else ("ldg_stream_kernel<OpDecolorF32>" if wl.output == "gray_f32"
                      else "hdr_gray_kernel + hdr_stats_kernel + hdr_tone_kernel")}

    # ---- side table (not the metric): the paper's Table 1 comparison on this batch
    methods = None
    if not args.no_methods and wl.dtype == "uint8" and wl.output == "gray_u8":
        methods = run_methods(wg, torch, rgb, out, n_img, wl, stream)

    # ---- end to end through the public host-array API (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(wg, torch, wl, rgb, n_img, steps, dev, world)
    del out, rgb
    torch.cuda.empty_cache()

    sweep = None
    if wl.name == "C5" and not args.no_sweep:
        sweep = run_size_sweep(wg, torch, dev, stream, rank)
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, sample, kind, extra = cpu_port_rate(wl, seconds=args.cpu_seconds)
        cpu = {"value": round(v, 4), "unit": "Gpix/s", "cores": cores, "kind": kind, "sample": sample,
               "cpu_model": cpu_model(), **extra}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "Gpix/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32",  # arithmetic type of the kernels (I/O type is in config.io)
            "data": "synthetic, seeded, generated on device (%s)" % wl.name,
            "config": {"workload": f"{wl.name}: {n_img} x {wl.width}x{wl.height} RGB {wl.dtype} -> {wl.output} per GPU",
                       "images_per_gpu": n_img, "height": wl.height, "width": wl.width,
                       "io": f"{wl.dtype}->{wl.output}", "parallelism": f"image-sharded x{world}, no collective",
                       "l2": "inputs larger than L2, no flush" if flush is None else "L2 flushed between steps"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": steps * launches_per_step, "clocks": clk.summary(),
            # each GPU's own rate next to the aggregate (SURVEY 8 e)
            "per_gpu_gpix_s": [round(px_step * steps / (ms / 1e3) / 1e9, 2) for ms in per_rank],
        }
        if wl.name == "C1":  # a single 512^2 image is latency-bound: report the latency (SURVEY 8 d)
            line["latency_us_per_image"] = round(ms_per_step * 1e3 / n_img, 2)
        if methods:
            line["methods"] = methods
        if sweep:
            line["size_sweep"] = sweep
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def run_size_sweep(wg, torch, dev, stream, rank, iters: int = 5):
    """C5's per-GPU size sweep: 256x256 .. 8K uint8 images at fixed total pixels.

    BASELINE.json configs[4]: the same ~4.3 Gpx per GPU cut into images of each
    size (synth.SIZE_SWEEP), i.i.d. uniform bytes generated on the device; one
    decolor launch per step over the whole batch, device-timed. Shows the
    throughput does not depend on the image size (the kernels see a flat
    pixel stream).
    """
    from paper_2108_13656_b200 import synth

    total = max(n * h * w for h, w, n in synth.SIZE_SWEEP)
    buf = torch.empty(total * 3, dtype=torch.uint8, device=dev)
    gout = torch.empty(total, dtype=torch.uint8, device=dev)
    res = {}
    for h, w, n in synth.SIZE_SWEEP:
        px = n * h * w
        rgb = buf[: px * 3].view(n, h, w, 3)
        synth.fill_uniform_u8(rgb, seed=5, first_image=rank * n)
        out = gout[:px].view(n, h, w)
        wg.decolor(rgb, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            wg.decolor(rgb, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        res[f"{w}x{h}"] = {"images": n, "gpix": round(px / 1e9, 3), "gpix_s": round(px / ms / 1e6, 1)}
    del buf, gout
    res["note"] = (f"{iters} device-resident passes per size in this order, uint8 i.i.d. input, fixed total pixels "
                   "per GPU; sw_power_cap engages over the sweep, so later sizes run at lower SM clocks")
    return res


def run_methods(wg, torch, rgb, out, n_img, wl, stream, iters: int = 5):
    """Device-resident Gpix/s of each colour-to-gray method on the bench batch.

    The paper's Table 1 compares its method's per-pixel time with the CIE Lab
    lightness baseline; BT.601 ("y") and HSV value ("v") are the reference's
    other extractors (colorspaces.py:87-112), all uint8 -> uint8 and
    bit-identical to quantize_u8 of the reference. "global_tone" is the fused
    decolor + global sigmoid (tonemap_image(mode="global"), north-star bar),
    "global_tone_exact" its bit-identical route, "global_tone_rgb" the same
    with the reinstated colour image as uint8 (bit-identical), and "local_tone" the fused decolor + local tone map (mode="local",
    SURVEY 8 f1, bit-identical).
    """
    grid = wg.LocalHistogramGrid.for_image(wl.width, wl.height)
    # at most ~2.2 Gpx (all of C3; 66 frames of C5): the local tone map's scratch
    # holds a 4 B/px gray plane and the extractors allocate their outputs
    n_img = min(n_img, max(1, 2_200_000_000 // wl.pix_per_image))
    rgb = rgb[:n_img]
    out = out[:n_img]
    img4 = rgb.view(n_img, wl.height, wl.width, 3)
    scratch = torch.empty(int(wg._lib.load().wg_lhe_scratch_bytes(n_img, wl.height, wl.width, grid.tile_w,
                                                                  grid.tile_h, grid.bins)),
                          dtype=torch.uint8, device=rgb.device)
    fns = {
        "ours": lambda: wg.decolor(rgb, out=out),
        "global_tone": lambda: wg.decolor_tone(rgb),
        "global_tone_exact": lambda: wg.decolor_tone(rgb, exact=True),
        "global_tone_rgb": lambda: wg.decolor_tone(rgb, return_rgb=True),
        "y_bt601": lambda: wg.luma(rgb, "y"),
        "v_hsv": lambda: wg.luma(rgb, "v"),
        "lab_lightness": lambda: wg.luma(rgb, "lab"),
        "local_tone": lambda: wg.decolor_tone_local(img4, grid=grid, scratch=scratch),
    }
    npx = n_img * wl.pix_per_image
    res = {}
    for name, fn in fns.items():
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        res[name] = {"gpix_s": round(npx / ms / 1e6, 1), "ps_per_px": round(ms * 1e9 / npx, 3)}
    res["note"] = (f"{iters} device-resident passes each over this batch, uint8 in/out, bit-identical to the "
                   "reference; ours/lab_lightness is the paper's Table 1 ratio")
    return res


def run_e2e(wg, torch, wl, rgb, n_img, steps, dev, world):
    """Same metric through decolor_host / hdr_tonemap_host with pinned host buffers."""
    n_e2e = min(n_img, 32)
    host_in = torch.empty(tuple(rgb[:n_e2e].shape), dtype=rgb.dtype, pin_memory=True)
    host_in.copy_(rgb[:n_e2e])
    out_dtype = torch.float32 if wl.output == "gray_f32" else torch.uint8
    host_out = torch.empty((n_e2e, *rgb.shape[1:-1]), dtype=out_dtype, pin_memory=True)
    xin, xout = host_in.numpy(), host_out.numpy()

    def call():
        if wl.output == "hdr_u8":
            wg.hdr_tonemap_host(xin, out=xout)
        else:
            wg.decolor_host(xin, out=xout)

    k = max(1, min(steps, 5))
    call()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(k):
        call()
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    el = float(t.item())
    px = n_e2e * wl.pix_per_image
    return {"value": round(world * px * k / el / 1e9, 3), "unit": "Gpix/s",
            "h2d_bytes_per_step": int(host_in.numel() * host_in.element_size()),
            "d2h_bytes_per_step": int(host_out.numel() * host_out.element_size()),
            "images_per_step": n_e2e, "steps": k, "api": "decolor_host -> wg_host_decolor_u8"
            if wl.output != "hdr_u8" else "hdr_tonemap_host -> wg_host_hdr_tonemap_u8"}


def committed_traffic(workload: str):
    """dram bytes per launch of the dominant kernel from a committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


def run_reference(args, wl, steps, warmup, world):
    """--impl reference: the reference's CPU path on this workload, all host cores --
    its own compiled kernels (oracle/_ref) driven as its public API does when
    built, else the oracle port."""
    import numpy as np

    from oracle import oracle

    threads = oracle.default_threads()
    rgb, desc = cpu_sample(wl, 1)
    ref = reference_fns(wl, threads)
    kind, extra = "port", {}
    if ref is not None:
        fn, kernel, label = ref
        kind = "reference"
        krate, _, _ = _rate(kernel, rgb, 3.0)
        extra = {"kernel_only_gpix_s": round(krate, 4)}
        desc = f"{desc}; {label}"
    else:
        fn = {"gray_u8": lambda x: oracle.decolor_u8(x, threads=threads),
              "gray_f32": lambda x: oracle.decolor_f32in(x, threads=threads),
              "hdr_u8": lambda x: oracle.hdr_u8(x, threads=threads)}[wl.output]
    for _ in range(min(warmup, 3)):
        fn(rgb)
    # bound the whole run to ~150 s: a step over more than that share of the
    # image runs on its leading rows instead (same per-pixel work)
    t1 = time.perf_counter()
    fn(rgb)
    per_step = time.perf_counter() - t1
    if per_step * steps > 150.0:
        rows = max(1, int(rgb.shape[1] * 150.0 / (per_step * steps)))
        rgb = np.ascontiguousarray(rgb[:, :rows])
        desc = f"{desc}; rows 0..{rows - 1} of each image so {steps} steps fit in ~150 s"
    t0 = time.perf_counter()
    for _ in range(steps):
        fn(rgb)
    el = time.perf_counter() - t0
    px = rgb.size // 3
    value = px * steps / el / 1e9
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "Gpix/s", "n_gpus": world, "steps": steps,
        "warmup": min(warmup, 3), "ms_per_step": round(el / steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic, seeded (%s)" % wl.name,
        "config": {"workload": f"{wl.name}: 1 x {wl.width}x{wl.height} RGB {wl.dtype} -> {wl.output} per step (bounded sample)",
                   "images_per_gpu": wl.n_images, "height": wl.height, "width": wl.width,
                   "io": f"{wl.dtype}->{wl.output}"},
        "cpu_baseline": {"value": round(value, 4), "unit": "Gpix/s", "cores": threads, "kind": kind,
                         "sample": desc + " per step", "cpu_model": cpu_model(), **extra},
        "e2e": {"value": round(value, 4), "unit": "Gpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
