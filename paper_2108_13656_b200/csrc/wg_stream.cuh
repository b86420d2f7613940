// wg_stream.cuh -- the streaming skeleton shared by every per-pixel op:
// interleaved input is cut into tiles of 256 threads x 48 bytes; an Op turns
// one thread's 48 bytes (3 x uint4 in registers) into its outputs. Three
// kernels move the tiles:
//  * ldg_stream_kernel: register prefetch of tile t + grid while tile t
//    computes (compute-heavy ops: the uint8 paths);
//  * stream_kernel: a 4-stage cp.async.bulk (TMA engine) ring into shared
//    memory with mbarrier completion (fp32 paths);
//  * scalar_kernel: one pixel per thread for unaligned buffers.
// An Op may define `prologue()` (per-block setup, e.g. staging lookup tables
// in shared memory); it runs once per block before any pixel, followed by a
// block barrier.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "wg_device.cuh"
#include "wg_internal.h"

namespace wg {

constexpr int kThreads = 256;
constexpr int kStages = 4;
constexpr int kTileBytes = kThreads * 48;  // 12288 B: 48 input bytes per thread
constexpr int kSmemBytes = kStages * kTileBytes + kStages * 8;

template <class T, class = void>
struct HasPrologue : std::false_type {};
template <class T>
struct HasPrologue<T, std::void_t<decltype(&T::prologue)>> : std::true_type {};

// An Op with `static constexpr bool kPingPong = true` gets ldg_stream_kernel's
// loop unrolled twice over two register buffers (no copies of the prefetched
// tile); ops whose math already fills the register budget keep one buffer.
template <class T, class = void>
struct PingPong : std::false_type {};
template <class T>
struct PingPong<T, std::void_t<decltype(T::kPingPong)>> : std::bool_constant<T::kPingPong> {};

// Optional Op traits of ldg_stream_kernel's 256-thread shape: kMinBlocks
// (resident CTAs per SM the register budget is cut for; default 5) and
// kGridPerSm (CTAs launched per SM; default 40).
template <class T, class = void>
struct MinBlocks : std::integral_constant<int, 5> {};
template <class T>
struct MinBlocks<T, std::void_t<decltype(T::kMinBlocks)>> : std::integral_constant<int, T::kMinBlocks> {};
template <class T, class = void>
struct GridPerSm : std::integral_constant<int, 40> {};
template <class T>
struct GridPerSm<T, std::void_t<decltype(T::kGridPerSm)>> : std::integral_constant<int, T::kGridPerSm> {};

// An Op may define `epilogue()`: it runs in every thread of ldg_stream_kernel
// after its last tile, before the tail (e.g. draining per-warp queues).
template <class T, class = void>
struct HasEpilogue : std::false_type {};
template <class T>
struct HasEpilogue<T, std::void_t<decltype(&T::epilogue)>> : std::true_type {};

template <class Op>
__device__ __forceinline__ void run_prologue(const Op& op) {
    if constexpr (HasPrologue<Op>::value) {
        op.prologue();
        __syncthreads();
    }
}

// ------------------------------------------------------------------ streaming kernels
template <class Op>
__global__ void __launch_bounds__(kThreads) stream_kernel(Op op, const uint8_t* __restrict__ in,
                                                          int64_t ntiles, int64_t npix) {
    extern __shared__ __align__(128) uint8_t smem[];
    run_prologue(op);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kTileBytes);
    constexpr int kTilePx = kThreads * Op::kPx;
    const int tid = threadIdx.x;
    const int64_t stride = gridDim.x;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();

    uint64_t policy = 0;
    if (tid == 0) {
        policy = l2_policy_evict_first();
#pragma unroll
        for (int s = 0; s < kStages; ++s) {
            const int64_t t = blockIdx.x + s * stride;
            if (t < ntiles) {
                mbar_arrive_expect_tx(&bars[s], kTileBytes);
                bulk_g2s(smem + s * kTileBytes, in + t * kTileBytes, kTileBytes, &bars[s], policy);
            }
        }
    }

    int s = 0;
    uint32_t phase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += stride) {
        mbar_wait(&bars[s], phase);
        uint4 v[3];
        const uint4* src = reinterpret_cast<const uint4*>(smem + s * kTileBytes) + tid * 3;
        v[0] = src[0];
        v[1] = src[1];
        v[2] = src[2];
        fence_proxy_async_smem();  // reads of slot s ordered before its TMA refill
        __syncthreads();           // every thread has drained slot s
        if (tid == 0) {
            const int64_t tn = t + kStages * stride;
            if (tn < ntiles) {
                mbar_arrive_expect_tx(&bars[s], kTileBytes);
                bulk_g2s(smem + s * kTileBytes, in + tn * kTileBytes, kTileBytes, &bars[s], policy);
            }
        }
        op.vec(v, t * kTilePx + static_cast<int64_t>(tid) * Op::kPx);
        if (++s == kStages) {
            s = 0;
            phase ^= 1u;
        }
    }

    // tail (< one tile) by the last CTA
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t p = ntiles * kTilePx + tid; p < npix; p += kThreads) op.scalar(p);
    }
}

// Register-prefetch variant: each thread loads its 48 bytes of tile t + grid
// with three 128-bit loads (evict-first) before computing tile t, so the
// next tile's HBM latency hides under this tile's math. No shared memory and
// no barriers; used where the per-pixel math, not the memory pipe, is the
// limiter (the uint8 path: scripts/tune_u8.cu measured it ahead of the
// bulk-copy ring at equal parity).
// Occupancy 5 CTAs/SM (<= 51 registers, no spills) and a 40 x SM grid measured
// best on C3 (scripts/tune_u8.cu: 74.7% of the HBM roofline vs 70.9% at 4 CTAs/SM).
// kBlock = 256 is the throughput shape; small inputs (fewer tiles than a
// couple of waves) use 64-thread CTAs so a single image still spreads over
// every SM (C1: 256 CTAs instead of 64).
template <class Op, int kBlock = kThreads>
__global__ void __launch_bounds__(kBlock, kBlock == kThreads ? MinBlocks<Op>::value : 20)
    ldg_stream_kernel(Op op, const uint8_t* __restrict__ in, int64_t ntiles, int64_t npix) {
    constexpr int kTilePx = kBlock * Op::kPx;
    constexpr int64_t kBlockBytes = kBlock * 48;
    run_prologue(op);
    const int tid = threadIdx.x;
    const int64_t stride = gridDim.x;
    int64_t t = blockIdx.x;
    const auto load = [&](int64_t tt, uint4 (&d)[3]) {
        const uint4* q = reinterpret_cast<const uint4*>(in + tt * kBlockBytes) + tid * 3;
        d[0] = __ldcs(q);
        d[1] = __ldcs(q + 1);
        d[2] = __ldcs(q + 2);
    };
    if (t < ntiles && !PingPong<Op>::value) {
        uint4 v[3];
        load(t, v);
        for (; t < ntiles; t += stride) {
            uint4 n[3] = {v[0], v[1], v[2]};
            if (t + stride < ntiles) load(t + stride, n);
            op.vec(v, t * kTilePx + static_cast<int64_t>(tid) * Op::kPx);
            v[0] = n[0];
            v[1] = n[1];
            v[2] = n[2];
        }
    } else if (t < ntiles) {
        // two register buffers used in turn (the loop body is unrolled twice),
        // so the prefetched tile is never copied between registers
        uint4 a[3], b[3];
        load(t, a);
        for (;;) {
            if (t + stride < ntiles) load(t + stride, b);
            op.vec(a, t * kTilePx + static_cast<int64_t>(tid) * Op::kPx);
            t += stride;
            if (t >= ntiles) break;
            if (t + stride < ntiles) load(t + stride, a);
            op.vec(b, t * kTilePx + static_cast<int64_t>(tid) * Op::kPx);
            t += stride;
            if (t >= ntiles) break;
        }
    }
    if constexpr (HasEpilogue<Op>::value) op.epilogue();
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t p = ntiles * kTilePx + tid; p < npix; p += kBlock) op.scalar(p);
    }
}

template <class Op>
__global__ void __launch_bounds__(kThreads) scalar_kernel(Op op, int64_t npix) {
    run_prologue(op);
    for (int64_t p = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; p < npix;
         p += static_cast<int64_t>(gridDim.x) * kThreads)
        op.scalar(p);
}

// ------------------------------------------------------------------ launch helpers
template <class Op>
static int stream_grid(int device) {
    // idempotent lazy caches; relaxed atomics keep concurrent first calls race-free
    static std::atomic<int> occ_cache[kMaxDevices];
    static std::atomic<int> attr_set[kMaxDevices];
    if (!attr_set[device].load(std::memory_order_relaxed)) {
        cudaFuncSetAttribute(stream_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemBytes);
        attr_set[device].store(1, std::memory_order_relaxed);
    }
    int occ = occ_cache[device].load(std::memory_order_relaxed);
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stream_kernel<Op>, kThreads,
                                                      kSmemBytes);
        occ = std::max(occ, 1);
        occ_cache[device].store(occ, std::memory_order_relaxed);
    }
    return occ * sm_count(device);
}

template <class Op>
static int launch_stream(const Op& op, const void* in, const void* const* outs, int nouts,
                         int64_t npix, cudaStream_t stream) {
    if (npix == 0) return WG_OK;
    int device = 0;
    cudaGetDevice(&device);
    if (device < 0 || device >= kMaxDevices) return set_error(WG_ENODEV, "device ordinal out of range");
    bool aligned = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    for (int i = 0; i < nouts; ++i)
        if (outs[i] && (reinterpret_cast<uintptr_t>(outs[i]) & 15) != 0) aligned = false;
    constexpr int64_t kTilePx = kThreads * Op::kPx;
    const int64_t ntiles = npix / kTilePx;
    constexpr int kSmall = 64;
    if (aligned && Op::kLdg && ntiles < 2LL * sm_count(device)) {
        const int64_t st = npix / (kSmall * Op::kPx);
        const int64_t grid = std::max<int64_t>(1, st);
        ldg_stream_kernel<Op, kSmall><<<static_cast<unsigned>(grid), kSmall, 0, stream>>>(
            op, static_cast<const uint8_t*>(in), st, npix);
    } else if (aligned && Op::kLdg) {
        int64_t per_sm = GridPerSm<Op>::value;
        if (const char* e = std::getenv("WG_LDG_GRID_PER_SM")) per_sm = std::max(1, std::atoi(e));  // tuning knob
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, per_sm * sm_count(device)));
        ldg_stream_kernel<Op><<<static_cast<unsigned>(grid), kThreads, 0, stream>>>(
            op, static_cast<const uint8_t*>(in), ntiles, npix);
    } else if (aligned) {
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, stream_grid<Op>(device)));
        stream_kernel<Op><<<static_cast<unsigned>(grid), kThreads, kSmemBytes, stream>>>(
            op, static_cast<const uint8_t*>(in), ntiles, npix);
    } else {
        const int64_t blocks = std::min<int64_t>((npix + kThreads - 1) / kThreads, 148LL * 32);
        scalar_kernel<Op><<<static_cast<unsigned>(blocks), kThreads, 0, stream>>>(op, npix);
    }
    return check_launch("stream kernel");
}

}  // namespace wg
