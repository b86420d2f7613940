#!/usr/bin/env python
"""Benchmark: decolorized Gpixels/s on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3] [--op decolor|tone]
                    [--scaling weak|strong] [--impl ours|reference]

A "step" is one pass of the hot path over one batch resident in HBM. Default:
workload C3 (BASELINE.json configs[2], the graded 4K batch) = 256 RGB u8
images of 3840x2160 -> u8 gray per GPU, one kernel launch per step. Under
torchrun (N > 1) every rank runs its own shard; the step time is the max over
ranks of the CUDA-event time. Images are independent, so there is no
collective on the data path:
  * weak scaling (default for C1-C4): every rank owns a full batch of the
    workload (first image = rank x batch, so ranks see different images);
  * strong scaling (default for C5, BASELINE configs[4]: "1024 ... images
    sharded by image across 1/2/4/8 GPUs"): rank r takes
    sharder.shard_range(1024, N, r) of the fixed batch, and the optional
    final gather of the gray shards to rank 0 is timed separately (gather_ms).

--op tone times the fused decolor + global sigmoid tone map
(decolor_tone, wg_decolor_tone_u8; tonemap_image(mode="global")'s toned
gray as uint8) instead of the plain decolor; the default decolor line of a
uint8 workload also carries a "tone" object with the same fields measured
in the same run.

Keys beyond the base contract:
  roofline      algorithmic bytes per launch (input read once + output written
                once: 4 B/px for u8->u8) / mean launch duration from CUDA events
                on the launching stream, against MEASURED_PEAKS.json hbm_gbs
                (burst, the kernel timed alone); traffic = ncu dram bytes per
                launch of that kernel from a committed capture
                (profiles/traffic.json, stamped with the capture and kernel).
  sustained     >= 2 s of back-to-back steps right after the timed region,
                with its own clocks (the power-capped rate next to the burst one).
  cpu_baseline  the reference's own CPU path on all host cores, rank 0 at N=1,
                over a bounded sample of the same input bytes: its _kernels.pyx
                compiled into oracle/_ref by oracle/build_ref.py, driven as
                decolor_image / dequantize_u8 / quantize_u8 (and apply_sigmoid
                for --op tone) do (kind "reference", plus kernel_only_gpix_s);
                the oracle port (oracle/warmgray_oracle.c, bit-identical) for
                the HDR adapter, which the reference lacks.
  e2e           the same metric through the public host-array API
                (decolor_host / decolor_tone_host / hdr_tonemap_host): pinned
                host input -> H2D -> kernel -> D2H every step (3-stream chunked
                pipeline in the library), plus h2d_ms / kernel_ms / d2h_ms of
                the same step timed separately on the device.
  e2e_dropin    the reference-facing drop-in on one image: PlanarImage(fp64)
                -> decolor_image -> quantize_u8, as a user of the reference calls it.
  clocks        NVML SM clock / throttle reasons sampled during the timed region.

--impl reference: the reference's CPU path (kind "reference" when
oracle/_ref is built -- it travels to the GPU box with the snapshot --, else
the bit-identical oracle port) on every host core, timed on the same
workload / op / metric; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
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
SUSTAINED_S = 2.0
COOLDOWN_S = 2.0


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


# ------------------------------------------------------------------ ops
def op_spec(wl, op: str) -> dict:
    """Kernel, algorithmic bytes per pixel and public entry points of (workload, op)."""
    if op == "tone":
        if wl.output != "gray_u8":
            raise SystemExit(f"--op tone needs a uint8 workload (C1, C3, C5), not {wl.name}")
        return {"kernel": "ldg_stream_kernel<OpToneSqU8>", "bytes_per_px": 4, "launches": 1,
                "api": "decolor_tone (wg_decolor_tone_u8)",
                "e2e_api": "decolor_tone_host -> wg_host_decolor_tone_u8",
                "io": "uint8->toned uint8 (tonemap_image(mode='global') l_out, quantize_u8)"}
    if wl.output == "gray_u8":
        return {"kernel": "ldg_stream_kernel<OpDecolorU8>", "bytes_per_px": 4, "launches": 1,
                "api": "decolor (wg_decolor_u8)", "e2e_api": "decolor_host -> wg_host_decolor_u8",
                "io": "uint8->gray uint8"}
    if wl.output == "gray_f32":
        return {"kernel": "ldg_stream_kernel<OpDecolorF32>", "bytes_per_px": 16, "launches": 1,
                "api": "decolor (wg_decolor_f32)", "e2e_api": "decolor_host -> wg_host_decolor_f32",
                "io": "float32->gray float32"}
    return {"kernel": "hdr_tm_kernel", "bytes_per_px": wl.bytes_per_px,
            "launches": 1, "api": "hdr_tonemap (wg_hdr_tonemap_u8)",
            "e2e_api": "hdr_tonemap_host -> wg_host_hdr_tonemap_u8", "io": "float32 radiance->uint8 (HDR adapter)"}


# ------------------------------------------------------------------ CPU legs
def reference_fns(workload, threads: int, op: str = "decolor"):
    """The reference's own CPU path for this workload / op, when its compiled
    kernels are present (oracle/_ref, built from /root/reference by
    oracle/build_ref.py): returns (end-to-end fn, kernel-only fn, label) or None.

    End to end is what the reference's public API does for the metric: codec.py's
    dequantize_u8 (u8 workloads), PlanarImage's validation (core.py:69-80),
    core.decolor_image -- _kernels.decolor_rows over contiguous row chunks on a
    thread pool of `threads` workers created per call (backend.run_rows) -- the
    validation of the result, for --op tone tonemap.py:72-83's apply_sigmoid
    (NumPy, as the reference evaluates it), and quantize_u8 (or the fp32 cast).
    Kernel only is decolor_rows over the same row chunks on pre-converted fp64
    input. The HDR adapter (C4) has no reference implementation: None.
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

    def apply_sigmoid(x, m=0.5, s=8.0):  # tonemap.py:72-83 (SigmoidCurve() defaults)
        lo = 1.0 / (1.0 + np.exp(s * m))
        hi = 1.0 / (1.0 + np.exp(-s * (1.0 - m)))
        y = 1.0 / (1.0 + np.exp(-s * (x - m)))
        out = np.clip((y - lo) / (hi - lo), 0.0, 1.0)
        validate(out)
        return out

    def quantize(x):  # codec.py:22-25
        return np.floor(np.clip(x, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)

    if workload.output == "gray_u8":
        def e2e(batch):
            for img in batch:
                f = img.astype(np.float64) / 255.0  # dequantize_u8
                validate(f)
                g = decolor_image(f)
                quantize(apply_sigmoid(g) if op == "tone" else g)
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
    path = "decolor_image / dequantize_u8 / quantize_u8" + (" / apply_sigmoid" if op == "tone" else "")
    return e2e, kernel, (f"the reference's _kernels.pyx compiled by oracle/build_ref.py (cython + gcc -O3 as "
                         f"setup.py), driven as {path} do")


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


def _port_fn(wl, op, threads):
    from oracle import oracle

    if wl.output == "gray_u8":
        if op == "tone":
            return lambda x: oracle.tone_u8(x, threads=threads)
        return lambda x: oracle.decolor_u8(x, threads=threads)
    if wl.output == "gray_f32":
        return lambda x: oracle.decolor_f32in(x, threads=threads)
    return lambda x: oracle.hdr_u8(x, threads=threads)


def cpu_port_rate(workload, sample, desc, op: str = "decolor", seconds: float = 10.0):
    """Gpix/s of the reference's CPU path on all host cores over `sample`: its
    compiled kernels (oracle/_ref) when built, else the oracle port (fp64
    scalar, bit-identical). Returns (rate, threads, sample description, kind, extra)."""
    from oracle import oracle

    threads = oracle.default_threads()
    ref = reference_fns(workload, threads, op)
    if ref is not None:
        e2e, kernel, label = ref
        rate, el, px = _rate(e2e, sample, seconds)
        krate, _, _ = _rate(kernel, sample, min(seconds, 5.0))
        return (rate, threads, f"{desc}, repeated for {el:.1f} s ({px / 1e6:.0f} Mpx); {label}", "reference",
                {"kernel_only_gpix_s": round(krate, 4)})
    rate, el, px = _rate(_port_fn(workload, op, threads), sample, seconds)
    return rate, threads, f"{desc}, repeated for {el:.1f} s ({px / 1e6:.0f} Mpx); oracle port", "port", {}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_sample(workload, n: int, rgb=None, first_image: int = 0):
    """A bounded sample of the workload's input: the first n images of the
    device batch copied to the host (the bytes the GPU arm processes), or,
    without a device batch (the reference arm), the same images regenerated
    on the host (C1 / C3 / C5: the oracle's generators, identical bytes) or
    same-shape seeded stand-ins (C2 / C4, whose generators are device-only)."""
    import numpy as np

    from oracle import oracle
    from paper_2108_13656_b200 import synth

    h, w = workload.height, workload.width
    n = min(n, workload.n_images)
    if rgb is not None:
        return (rgb[:n].cpu().numpy(),
                f"images {first_image}..{first_image + n - 1} of this run's {workload.name} batch "
                f"({w}x{h} {workload.dtype}), copied D2H")
    if workload.name == "C1":
        return synth.c1_image()[None], "C1 512x512 u8"
    if workload.name == "C3":
        xy, col = synth.voronoi_tables(n, h, w)
        return oracle.synth_voronoi_u8(h, w, xy, col, 0), f"{n} C3 images {w}x{h} u8 (host Voronoi, same bytes)"
    if workload.name == "C5":
        return oracle.synth_uniform_u8(n, h, w, 0), f"{n} C5 images {w}x{h} u8 (same bytes)"
    rng = np.random.default_rng(0)
    if workload.name == "C4":
        lum = 10.0 ** rng.uniform(-3, 4, (n, h, w))
        chroma = rng.random((n, h, w, 3))
        y = chroma @ np.array([0.2126, 0.7152, 0.0722])
        return (chroma * (lum / np.maximum(y, 1e-6))[..., None]).astype(np.float32), \
            f"{n} C4-like HDR images {w}x{h} f32 (host stand-in)"
    return rng.random((n, h, w, 3), dtype=np.float32), f"{n} C2-size images {w}x{h} f32 (host uniform stand-in)"


# ------------------------------------------------------------------ device timing
def time_steps(torch, step, steps, stream, flush, clock_index):
    """CUDA-event time of `steps` steps on `stream` (L2 flushed before each step
    when `flush` is given; then only the steps are timed), with NVML clocks."""
    if flush is None:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with ClockSampler(clock_index) as clk:
            ev0.record(stream)
            for _ in range(steps):
                step()
            ev1.record(stream)
            torch.cuda.synchronize()
        return ev0.elapsed_time(ev1), clk.summary()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    with ClockSampler(clock_index) as clk:
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs), clk.summary()


def roofline_obj(spec, px_step, ms_per_step, workload: str):
    peak, peak_src = peaks()
    achieved = spec["bytes_per_px"] * px_step / (ms_per_step / 1e3) / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": committed_traffic(workload, spec["kernel"]),
            "bytes_per_px": spec["bytes_per_px"], "peak_source": peak_src + ", burst: the kernel timed alone",
            # the measured peak is a 1:1 copy; read-dominant streams (3:1 for the fp32
            # path) can exceed it, so the fraction of the 8 TB/s HBM3e spec is given too
            "frac_vs_spec_8000": round(achieved / 8000.0, 4), "kernel": spec["kernel"]}


def sustained_obj(torch, step, stream, ms_per_step, px_step, spec, clock_index, seconds=SUSTAINED_S):
    """>= `seconds` of back-to-back steps (no flush) with their own clocks."""
    n = max(3, math.ceil(seconds * 1e3 / max(ms_per_step, 1e-3)))
    ms, clk = time_steps(torch, step, n, stream, None, clock_index)
    peak, _ = peaks()
    gpix = px_step * n / (ms / 1e3) / 1e9
    return {"seconds": round(ms / 1e3, 3), "steps": n, "value": round(gpix, 2), "unit": "Gpix/s",
            "frac": round(gpix * spec["bytes_per_px"] / peak, 4), "clocks": clk}


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="C3", choices=("C1", "C2", "C3", "C4", "C5"))
    ap.add_argument("--op", default="decolor", choices=("decolor", "tone"))
    ap.add_argument("--scaling", default=None, choices=("weak", "strong"),
                    help="weak: a full batch per rank; strong: the workload's batch sharded over the ranks "
                         "(default: strong for C5, weak otherwise)")
    ap.add_argument("--images", type=int, default=None,
                    help="images per GPU (weak) / in total (strong); default: the workload's batch")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tone", action="store_true", help="skip the tone object of the default decolor line")
    ap.add_argument("--no-sustained", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="C5: skip the per-GPU size sweep (256x256 .. 8K at fixed total pixels)")
    ap.add_argument("--no-methods", action="store_true",
                    help="skip the per-method side table (paper Table 1 on the GPU + local tone map)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--plan", action="store_true",
                    help="print the sharding plan (one JSON line from rank 0) and exit: no GPU needed; under "
                         "torchrun on CPU it runs over gloo")
    args = ap.parse_args()

    from paper_2108_13656_b200.synth import WORKLOADS

    wl = WORKLOADS[args.workload]
    rank, world, local = dist_env()
    warmup = max(args.warmup, 3)
    steps = max(args.steps, 1)
    scaling = args.scaling or ("strong" if wl.name == "C5" else "weak")
    spec = op_spec(wl, args.op)

    if args.impl == "reference":
        if rank != 0:
            return
        run_reference(args, wl, steps, warmup, world, scaling)
        return
    if args.plan:
        run_plan(args, wl, world, rank, scaling, spec)
        return

    import torch

    import paper_2108_13656_b200 as wg
    from paper_2108_13656_b200 import sharder, synth

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    wg.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    n_total, first, n_img = shard_plan(args, wl, world, rank, scaling)
    rgb = synth.make_batch(wl, dev, n_images=n_img, seed=0, first_image=first)
    torch.cuda.synchronize()
    out_dtype = torch.float32 if wl.output == "gray_f32" else torch.uint8
    out = torch.empty(rgb.shape[:-1], dtype=out_dtype, device=dev)
    scratch = wg.HdrScratch(n_img, wl.pix_per_image, device=dev) if wl.output == "hdr_u8" else None

    def make_step(op):
        if wl.output == "hdr_u8":
            return lambda: wg.hdr_tonemap(rgb, scratch=scratch, out=out)
        if op == "tone":
            return lambda: wg.decolor_tone(rgb, out=out)
        return lambda: wg.decolor(rgb, out=out)

    launches_per_step = spec["launches"]  # hdr: one persistent kernel (+ a memset of its completion counts)
    in_bytes = rgb.numel() * rgb.element_size()
    flush = None
    if in_bytes < 4 * L2_BYTES:  # small batches: flush L2 between timed steps
        flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> list[float]:
        """x of every rank (all-gather), rank order."""
        if world == 1:
            return [x]
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        allt = torch.zeros(world, dtype=torch.float64, device=dev)
        torch.distributed.all_gather_into_tensor(allt, t)
        return allt.cpu().tolist()

    px_step = n_img * wl.pix_per_image

    def measure(op):
        step = make_step(op)
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        barrier()
        ms, clocks = time_steps(torch, step, steps, stream, flush, local)
        barrier()
        per_rank = max_over_ranks(ms)
        max_ms = max(per_rank)
        total_px = sum(px_per_rank)
        sp = op_spec(wl, op)
        res = {"value": round(total_px * steps / (max_ms / 1e3) / 1e9, 2), "ms_per_step": round(max_ms / steps, 4),
               "roofline": roofline_obj(sp, px_step, ms / steps, wl.name), "clocks": clocks,
               "per_gpu_gpix_s": [round(px * steps / (m / 1e3) / 1e9, 2)
                                  for px, m in zip(px_per_rank, per_rank)]}
        return res, step, ms / steps, sp

    def settle():
        # let the board's power average recover between measured ops, so the
        # second op is not timed in the first one's power-capped tail
        torch.cuda.synchronize()
        time.sleep(COOLDOWN_S)

    px_per_rank = [int(p) for p in max_over_ranks(float(px_step))]  # every rank's pixels per step (all-gather)
    main_res, main_step, main_ms, main_sp = measure(args.op)
    tone_res = None
    if args.op == "decolor" and wl.output == "gray_u8" and not args.no_tone:
        settle()
        tone_res, tone_step, tone_ms, tone_sp = measure("tone")
        tone_res["api"] = op_spec(wl, "tone")["api"]
    if not args.no_sustained:  # after every burst measurement
        settle()
        main_res["sustained"] = sustained_obj(torch, main_step, stream, main_ms, px_step, main_sp, local)
        if tone_res is not None:
            settle()
            tone_res["sustained"] = sustained_obj(torch, tone_step, stream, tone_ms, px_step, tone_sp, local)

    # host sample for the CPU baseline: the same input bytes (before e2e reuses the buffers)
    cpu_sample = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_sample = host_sample(wl, 1 if wl.pix_per_image > 4_000_000 else 4, rgb, first)

    # ---- side table (not the metric): the paper's Table 1 comparison on this batch
    methods = None
    if not args.no_methods and wl.dtype == "uint8" and wl.output == "gray_u8":
        methods = run_methods(wg, torch, rgb, out, n_img, wl, stream)

    # ---- end to end through the public host-array API (pinned host buffers)
    e2e = e2e_tone = dropin = None
    if not args.no_e2e:
        e2e = run_e2e(wg, torch, wl, rgb, out, n_img, steps, dev, world, args.op, stream)
        if tone_res is not None:
            e2e_tone = run_e2e(wg, torch, wl, rgb, out, n_img, steps, dev, world, "tone", stream)
        if rank == 0 and wl.output != "hdr_u8":
            dropin = run_dropin(wg, wl, rgb[:1].cpu().numpy())

    # ---- optional final gather of the gray shards (strong scaling, N > 1): timed apart from the metric
    gather = None
    if scaling == "strong" and world > 1:
        step_into = None
        if args.op == "decolor" and wl.output == "gray_u8":
            from paper_2108_13656_b200 import _lib as wg_lib

            def step_into(ptr, _n=rgb.numel() // 3):  # the C ABI with the root's address as out
                wg_lib.call("wg_decolor_u8", rgb.data_ptr(), ptr, _n, wg.DEFAULT_PARAMS.beta_r,
                            wg.DEFAULT_PARAMS.beta_k, stream.cuda_stream)
        gather = run_gather(torch, sharder, out, n_total, world, step_into, first, stream)
    del out, rgb
    torch.cuda.empty_cache()

    sweep = None
    if wl.name == "C5" and not args.no_sweep:
        sweep = run_size_sweep(wg, torch, dev, stream, rank)
        torch.cuda.empty_cache()

    cpu = cpu_tone = None
    if cpu_sample is not None:
        sample, desc = cpu_sample
        v, cores, sdesc, kind, extra = cpu_port_rate(wl, sample, desc, args.op, seconds=args.cpu_seconds)
        cpu = {"value": round(v, 4), "unit": "Gpix/s", "cores": cores, "kind": kind, "sample": sdesc,
               "cpu_model": cpu_model(), **extra}
        if tone_res is not None:
            v, cores, sdesc, kind, extra = cpu_port_rate(wl, sample, desc, "tone", seconds=args.cpu_seconds / 2)
            cpu_tone = {"value": round(v, 4), "unit": "Gpix/s", "cores": cores, "kind": kind, "sample": sdesc,
                        "cpu_model": cpu_model(), **extra}

    if rank == 0:
        per_gpu = "per GPU" if scaling == "weak" else f"in total, {n_img} on rank 0"
        line = {
            "metric": METRIC, "value": main_res["value"], "unit": "Gpix/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": main_res["ms_per_step"],
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f32",  # arithmetic type of the kernels (I/O types are in config.io)
            "data": "synthetic, seeded, generated on device (%s)" % wl.name,
            "config": {"workload": f"{wl.name}: {n_total if scaling == 'strong' else n_img} x "
                                   f"{wl.width}x{wl.height} RGB {wl.dtype} -> {spec['io']} {per_gpu}",
                       "op": args.op, "api": spec["api"], "images_total": n_total,
                       "images_per_gpu": n_img, "height": wl.height, "width": wl.width,
                       "io": spec["io"], "parallelism": f"image-sharded x{world} ({scaling}), no collective",
                       "l2": "inputs larger than L2, no flush" if flush is None else "L2 flushed between steps"},
            "roofline": main_res["roofline"], "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": steps * launches_per_step, "clocks": main_res["clocks"],
            # each GPU's own rate next to the aggregate (SURVEY 8 e)
            "per_gpu_gpix_s": main_res["per_gpu_gpix_s"],
        }
        if "sustained" in main_res:
            line["sustained"] = main_res["sustained"]
        if dropin:
            line["e2e_dropin"] = dropin
        if wl.name == "C1":  # a single 512^2 image is latency-bound: report the latency (SURVEY 8 d)
            line["latency_us_per_image"] = round(main_res["ms_per_step"] * 1e3 / n_img, 2)
        if tone_res is not None:
            tone_res["e2e"] = e2e_tone
            tone_res["cpu_baseline"] = cpu_tone
            tone_res["gpu_launches"] = steps
            line["tone"] = tone_res
        if gather:
            line["gather"] = gather
        if methods:
            line["methods"] = methods
        if sweep:
            line["size_sweep"] = sweep
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def shard_plan(args, wl, world, rank, scaling):
    """(images in the whole job, this rank's first image, this rank's image count)."""
    from paper_2108_13656_b200 import sharder

    if scaling == "strong":
        n_total = args.images or wl.n_images
        first, stop = sharder.shard_range(n_total, world, rank)
        return n_total, first, stop - first
    n_img = args.images or wl.n_images
    return n_img * world, rank * n_img, n_img


def run_plan(args, wl, world, rank, scaling, spec):
    """--plan: every rank's image range (gathered over gloo / NCCL) and the config
    the full run would report, without touching a GPU."""
    n_total, first, n_img = shard_plan(args, wl, world, rank, scaling)
    shards = [[first, first + n_img]]
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        shards = [None] * world
        dist.all_gather_object(shards, [first, first + n_img])
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"plan": True, "n_gpus": world, "scaling": scaling, "op": args.op,
                          "config": {"workload": f"{wl.name}: {n_total} x {wl.width}x{wl.height} RGB {wl.dtype} -> "
                                                 f"{spec['io']} in total",
                                     "images_total": n_total, "shards": shards,
                                     "pixels_per_rank": [(b - a) * wl.pix_per_image for a, b in shards]}}))


def run_gather(torch, sharder, out, n_total, world, step_into=None, first=0, stream=None):
    """sharder.gather_to_root of every rank's gray shard to rank 0, timed on its own;
    with ``step_into`` (the rank's decolor launch with an ``out=`` tensor) also the
    gather fused into the launch: the kernel stores the shard straight into the
    root's buffer mapped over CUDA IPC / NVLink (sharder.PeerBuffer)."""
    torch.cuda.synchronize()
    torch.distributed.barrier()
    t0 = time.perf_counter()
    full = sharder.gather_to_root(out, n_total)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64, device=out.device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    nbytes = n_total * out[0].numel() * out.element_size()
    del full
    res = {"gather_ms": round(float(t.item()) * 1e3, 3), "bytes": int(nbytes),
           "note": "sharder.gather_to_root (NCCL gather to rank 0), outside the device-timed metric; "
                   "max over ranks of the wall time"}
    if step_into is not None and out.dtype == torch.uint8:
        torch.cuda.empty_cache()  # the gather's buffers back to the device for the peer buffer
        try:
            peer = sharder.PeerBuffer(n_total, tuple(out.shape[1:]), out.device.index)
        except Exception as e:  # (no IPC between these processes)
            res["fused"] = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
            return res
        try:
            ptr = peer.ptr_at(first)
            step_into(ptr)  # warm (peer mapping, TLB)
            torch.cuda.synchronize()
            torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            step_into(ptr)
            e1.record(stream)
            torch.cuda.synchronize()
            torch.distributed.barrier()
            wall = time.perf_counter() - t0
            t = torch.tensor([e0.elapsed_time(e1), wall * 1e3], dtype=torch.float64, device=out.device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ok = None
            if torch.distributed.get_rank() == 0:
                ok = bool(torch.equal(peer.full()[first: first + out.shape[0]], out))  # the root's own shard
        except Exception as e:
            peer.close()
            res["fused"] = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
            return res
        peer.close()
        res["fused"] = {"step_ms": round(float(t[0].item()), 3), "wall_ms": round(float(t[1].item()), 3),
                        "root_shard_equal": ok,
                        "note": "decolor launch whose out= is the root's buffer (CUDA IPC, NVLink stores): "
                                "the gather fused into the kernel; device time max over ranks, then wall "
                                "time including the barrier"}
    return res


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


# parity of each side-table method against the reference (tests/test_gpu_*.py measure these)
METHOD_PARITY = {
    "ours": "north-star bar: +-1 on 5.2e-6 of all 2^24 colours (exact=True: bit-identical)",
    "ours_exact": "bit-identical",
    "global_tone": "north-star bar: +-1 on <= 3e-5 of all 2^24 colours (square-domain step words)",
    "global_tone_exact": "bit-identical",
    "global_tone_rgb": "bit-identical (reinstated colour + toned)",
    "y_bt601": "bit-identical",
    "v_hsv": "bit-identical",
    "lab_lightness": "bit-identical",
    "local_tone": "bit-identical",
}


def run_methods(wg, torch, rgb, out, n_img, wl, stream, iters: int = 5):
    """Device-resident Gpix/s of each colour-to-gray method on the bench batch.

    The paper's Table 1 compares its method's per-pixel time with the CIE Lab
    lightness baseline; BT.601 ("y") and HSV value ("v") are the reference's
    other extractors (colorspaces.py:87-112), all uint8 -> uint8. "global_tone"
    is the fused decolor + global sigmoid (tonemap_image(mode="global")),
    "global_tone_exact" its bit-identical route, "global_tone_rgb" the same
    with the reinstated colour image as uint8, and "local_tone" the fused
    decolor + local tone map (mode="local"). Each entry names its
    parity against the reference.
    """
    grid = wg.LocalHistogramGrid.for_image(wl.width, wl.height)
    # at most ~2.2 Gpx (all of C3; 66 frames of C5): the local tone map's scratch
    # holds a 2 B/px plane and the extractors allocate their outputs
    n_img = min(n_img, max(1, 2_200_000_000 // wl.pix_per_image))
    rgb = rgb[:n_img]
    out = out[:n_img]
    img4 = rgb.view(n_img, wl.height, wl.width, 3)
    scratch = torch.empty(int(wg._lib.load().wg_lhe_scratch_bytes(n_img, wl.height, wl.width, grid.tile_w,
                                                                  grid.tile_h, grid.bins)),
                          dtype=torch.uint8, device=rgb.device)
    fns = {
        "ours": lambda: wg.decolor(rgb, out=out),
        "ours_exact": lambda: wg.decolor(rgb, out=out, exact=True),
        "global_tone": lambda: wg.decolor_tone(rgb, out=out),
        "global_tone_exact": lambda: wg.decolor_tone(rgb, exact=True, out=out),
        "global_tone_rgb": lambda: wg.decolor_tone(rgb, return_rgb=True, out=out),
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
        res[name] = {"gpix_s": round(npx / ms / 1e6, 1), "ps_per_px": round(ms * 1e9 / npx, 3),
                     "parity": METHOD_PARITY[name]}
    res["note"] = (f"{iters} device-resident passes each over this batch, uint8 in/out; "
                   "ours / lab_lightness is the paper's Table 1 ratio")
    return res


def run_e2e(wg, torch, wl, rgb, out, n_img, steps, dev, world, op, stream):
    """Same metric through the host-array API with pinned host buffers, plus the
    step's H2D copy, kernel and D2H copy each timed on the device."""
    spec = op_spec(wl, op)
    n_e2e = min(n_img, 32)
    host_in = torch.empty(tuple(rgb[:n_e2e].shape), dtype=rgb.dtype, pin_memory=True)
    host_in.copy_(rgb[:n_e2e])
    out_dtype = torch.float32 if wl.output == "gray_f32" else torch.uint8
    host_out = torch.empty((n_e2e, *rgb.shape[1:-1]), dtype=out_dtype, pin_memory=True)
    xin, xout = host_in.numpy(), host_out.numpy()

    def call():
        if wl.output == "hdr_u8":
            wg.hdr_tonemap_host(xin, out=xout)
        elif op == "tone":
            wg.decolor_tone_host(xin, out=xout)
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

    # the components of one step, each on the device (unpipelined): H2D of the
    # input, the kernel on the device copy, D2H of the result
    din, dout = rgb[:n_e2e], out[:n_e2e]
    scratch = wg.HdrScratch(n_e2e, wl.pix_per_image, device=dev) if wl.output == "hdr_u8" else None

    def kernel():
        if wl.output == "hdr_u8":
            wg.hdr_tonemap(din, scratch=scratch, out=dout)
        elif op == "tone":
            wg.decolor_tone(din, out=dout)
        else:
            wg.decolor(din, out=dout)

    def dev_ms(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    h2d_ms = dev_ms(lambda: din.copy_(host_in, non_blocking=True))
    kernel_ms = dev_ms(kernel)
    d2h_ms = dev_ms(lambda: host_out.copy_(dout, non_blocking=True))
    bi = int(host_in.numel() * host_in.element_size())
    bo = int(host_out.numel() * host_out.element_size())
    return {"value": round(world * px * k / el / 1e9, 3), "unit": "Gpix/s",
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
            "ms_per_step": round(el / k * 1e3, 3), "h2d_ms": round(h2d_ms, 3), "kernel_ms": round(kernel_ms, 3),
            "d2h_ms": round(d2h_ms, 3), "h2d_gbs": round(bi / h2d_ms / 1e6, 1), "d2h_gbs": round(bo / d2h_ms / 1e6, 1),
            "images_per_step": n_e2e, "steps": k, "api": spec["e2e_api"],
            "note": "value: wall time of the host-array call (the library pipelines H2D / kernel / D2H in chunks "
                    "over 3 streams); h2d/kernel/d2h_ms: the same step's parts, each timed alone on the device"}


def run_dropin(wg, wl, img):
    """The reference-facing drop-in on one image, as a user of the reference
    calls it: PlanarImage(fp64 rgb) -> decolor_image (wg_host_decolor_rows_f64:
    24 B/px H2D, 8 B/px D2H) -> quantize_u8 for uint8 workloads."""
    import numpy as np

    img = img[0]
    f = wg.dequantize_u8(img) if img.dtype == np.uint8 else np.ascontiguousarray(img, dtype=np.float64)
    px = f.shape[0] * f.shape[1]

    def full():
        p = wg.PlanarImage(wg.dequantize_u8(img) if img.dtype == np.uint8 else img.astype(np.float64))
        g = wg.decolor_image(p)
        if img.dtype == np.uint8:
            wg.quantize_u8(g.data)

    pl = wg.PlanarImage(f)
    wg.decolor_image(pl)
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        wg.decolor_image(pl)
    t_img = (time.perf_counter() - t0) / reps
    full()
    t0 = time.perf_counter()
    for _ in range(reps):
        full()
    t_full = (time.perf_counter() - t0) / reps
    return {"value": round(px / t_full / 1e9, 3), "unit": "Gpix/s",
            "decolor_image_gpix_s": round(px / t_img / 1e9, 3),
            "h2d_bytes_per_step": px * 24, "d2h_bytes_per_step": px * 8,
            "api": "PlanarImage -> decolor_image -> wg_host_decolor_rows_f64"
                   + (" (+ dequantize_u8 / quantize_u8)" if img.dtype == np.uint8 else ""),
            "sample": f"1 image {wl.width}x{wl.height}, {reps} calls",
            "note": "fp64 drop-in, bit-identical to the reference; PCIe-bound (32 B/px of fp64 through pinned "
                    "staging) plus the host-side dequantize / validate / quantize of PlanarImage's fp64 layout"}


def committed_traffic(workload: str, kernel: str):
    """ncu dram bytes per launch of `kernel` on `workload` from a committed capture
    (profiles/traffic.json: {workload: {kernel: {"bytes": B, "capture": path, ...}}})."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f).get(workload, {}).get(kernel)
        return ent if ent else None
    except Exception:
        return None


def run_reference(args, wl, steps, warmup, world, scaling):
    """--impl reference: the reference's CPU path on this workload / op, all host
    cores -- its own compiled kernels (oracle/_ref) driven as its public API does
    when built, else the oracle port. Each step is a bounded sample (leading
    rows of one image) so warm-up + steps end in about `budget` seconds."""
    import numpy as np

    from oracle import oracle

    threads = oracle.default_threads()
    rgb, desc = host_sample(wl, 1)
    ref = reference_fns(wl, threads, args.op)
    kind, extra = "port", {}
    if ref is not None:
        fn, kernel, label = ref
        kind = "reference"
        krate, _, _ = _rate(kernel, rgb, 3.0)
        extra = {"kernel_only_gpix_s": round(krate, 4)}
        desc = f"{desc}; {label}"
    else:
        fn = _port_fn(wl, args.op, threads)
    budget = 150.0
    t1 = time.perf_counter()
    fn(rgb)
    per_step = time.perf_counter() - t1
    if per_step * (steps + warmup) > budget:
        rows = max(1, int(rgb.shape[1] * budget / (per_step * (steps + warmup))))
        rgb = np.ascontiguousarray(rgb[:, :rows])
        desc = f"{desc}; rows 0..{rows - 1} of the image so {warmup} + {steps} steps fit in ~{budget:.0f} s"
    for _ in range(warmup):
        fn(rgb)
    t0 = time.perf_counter()
    for _ in range(steps):
        fn(rgb)
    el = time.perf_counter() - t0
    px = rgb.size // 3
    value = px * steps / el / 1e9
    spec = op_spec(wl, args.op)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "Gpix/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": round(el / steps * 1e3, 3), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic, seeded (%s)" % wl.name,
        "config": {"workload": f"{wl.name}: 1 x {wl.width}x{wl.height} RGB {wl.dtype} -> {spec['io']} per step "
                               "(bounded sample)",
                   "op": args.op, "images_per_gpu": wl.n_images, "height": wl.height, "width": wl.width,
                   "io": spec["io"]},
        "cpu_baseline": {"value": round(value, 4), "unit": "Gpix/s", "cores": threads, "kind": kind,
                         "sample": desc + " per step", "cpu_model": cpu_model(), **extra},
        "e2e": {"value": round(value, 4), "unit": "Gpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
