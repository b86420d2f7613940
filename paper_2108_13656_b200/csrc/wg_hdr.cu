// wg_hdr.cu -- HDR adapter: fp32 linear radiance -> uint8.
//
// The reference cannot ingest HDR (PlanarImage rejects samples > 1,
// core.py:76-79), so the adapter is builder-defined and restated
// in the oracle (oracle/warmgray_oracle.c, or_hdr_u8):
//   g  = decolor(x)                          (raw radiance; homogeneous, so the
//                                            image scale cancels below)
//   t  = log(g / gmin) / log(gmax / gmin)    over g > 0 (per image);
//   t  = 0 for g == 0, t = 1 if gmax == gmin
//   out = quantize_u8(apply_sigmoid(t))      (tonemap.py:72-83, codec.py:22-25)
//
// Default schedule (images a multiple of 32 px): ONE warp-specialised
// persistent kernel, one 1024-thread CTA per SM: producer warps compute the
// fp32 gray of the CTA's range of every image and publish exact per-CTA
// (min over g > 0, max) partials; consumer warps of the same CTA fold the
// image's partials once all CTAs have published, build the threshold table
// and tone the CTA's own range. hdr_tm_kernel keeps the gray in the SM's
// tensor memory (two image slots; C4: 429 Gpix/s, 0.99 x the 13 B/px of
// algorithmic traffic); hdr_ws_kernel, for images whose per-SM share exceeds
// a slot, keeps it in an L2-resident ring (C4: 320).
//
// Grouped schedule (WG_HDR_SCHEDULE=grouped, and other image sizes): three
// kernels per group of images:
//   hdr_gray_kernel   unclamped gray (packed-f32x2 MUFU formulation, relative
//                     error ~2e-7) -> scratch; every warp keeps a running
//                     (min over g > 0, max) and writes it to its own slot. No
//                     atomics touch the statistic: min/max are exact, so the
//                     result is independent of grid size and GPU sharding.
//   hdr_stats_kernel  one block per image folds the slots and builds a
//                     threshold table (below).
//   hdr_tone_kernel   blocks are image-uniform: stage the image's table in
//                     shared memory, then one table lookup + one compare per
//                     pixel; the gray lines are dropped from L2 afterwards
//                     (discard.global.L2) so they are not written back.
// Both give the same bytes.
//
// Tone without transcendentals: t, the sigmoid and the rounding are monotone
// in r = g / gmin, so out = #{ j : r >= gamma_j } with 255 per-image
// thresholds gamma_j = 2^(theta_j * log2(gmax/gmin)); theta_j is the t at
// which the reference's logistic curve crosses (j - 0.5)/255 (host, fp64,
// passed as a kernel parameter). The table has 64 bins per octave of r over
// 32 octaves (bin = float bit pattern >> 17), storing per bin the number of
// thresholds below it and the threshold inside it. Exact up to the fp32
// error of g. If a bin would hold two thresholds (very steep curves) or the
// range exceeds 31 octaves, per-pixel log2 + tanh arithmetic is used.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"

namespace wg {
namespace {

constexpr int kT = 256;
constexpr int kWarps = kT / 32;
constexpr int kSlots = 8192;  // (min, max) slots per image (>= warps of one image's gray grid)
constexpr int kLutPerOct = 64, kLutOct = 32, kLutBins = kLutPerOct * kLutOct;
constexpr int kMaxGroup = 32;
// Grouping images so the gray plane stays L2-resident measured slower than one
// group (launch/ramp overheads exceed the saved 8 B/px): default = whole batch
// up to kMaxGroup images; WG_HDR_L2_BUDGET_MB overrides for experiments.
constexpr size_t kL2Budget = size_t(1) << 40;

struct HdrStat {
    float inv_gmin;
    float inv_lrange;
    int mode;  // 0: no positive pixel, 1: log range, 2: gmax == gmin (t = 1)
    int lut;   // 1: the threshold table of this image is valid
};
struct Theta {
    double v[255];
};

// Programmatic dependent launch (stats and tone grids are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): the dependent grid's
// launch overlaps its predecessor's completion, and griddepcontrol.wait blocks
// until the predecessor has completed and its writes are visible (a no-op for
// a grid launched without the attribute). C4: 293.7 -> 296.3 Gpix/s. An early
// griddepcontrol.launch_dependents in the gray / stats grids measured slower
// (291.7): the stats CTAs then sit on SM slots during the gray pass's last wave.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void discard_l2_line(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void warp_minmax(float& lo, float& hi) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
}
__device__ __forceinline__ void track(float v, float& lo, float& hi) {
    if (v > 0.0f) lo = fminf(lo, v);
    hi = fmaxf(hi, v);
}
// bin of r >= 1 over 64 bins per octave: exponent * 64 + top 6 mantissa bits
__device__ __forceinline__ int lut_bin(float r) {
    const int b = static_cast<int>(__float_as_uint(r) >> 17) - (127 << 6);
    return min(max(b, 0), kLutBins - 1);
}

// 32-bit step word per bin (since r02): W[b] = 2^24 count + 2^24 - L - bits(b0)
// (mod 2^32), b0 the first float of bin b, count the thresholds below the bin
// and L the in-bin offset of the bin's one threshold (2^17 = none). For r in
// bin b, W[b] + bits(r) = 2^24 count + 2^24 + (offset - L): the offset minus L
// borrows from or carries into bit 24, so byte 3 is the toned byte -- one LDS
// and one IADD per pixel, no compare. r < 1 happens only for g <= 0 (t = 0) or
// g = gmin rounding below 1: clamped to 1.0 (t = 0).
constexpr uint32_t kOneBits = 0x3F800000u, kLutLastBits = ((kOneBits >> 17) + kLutBins) * (1u << 17) - 1u;
__device__ __forceinline__ uint32_t lut_step_sum(float v, float inv, const uint32_t* s_lut) {
    const uint32_t rb = static_cast<uint32_t>(
        min(max(__float_as_int(__fmul_rn(v, inv)), static_cast<int>(kOneBits)), static_cast<int>(kLutLastBits)));
    return s_lut[(rb >> 17) - (kOneBits >> 17)] + rb;
}
__device__ __forceinline__ uint32_t lut_px32(float v, float inv, const uint32_t* s_lut) {
    return lut_step_sum(v, inv, s_lut) >> 24;
}
// step word of bin b; cb = index of the first threshold whose bin is >= b
// (advanced past bin b's thresholds). s_b[255] is a sentinel.
__device__ __forceinline__ uint32_t step_word(int b, int& cb, const int* s_b, const uint32_t* s_gb) {
    const uint32_t b0 = static_cast<uint32_t>(b + static_cast<int>(kOneBits >> 17)) << 17;
    uint32_t cnt = static_cast<uint32_t>(cb), L = 0x20000u;
    if (s_b[cb] == b) {
        const int64_t d = static_cast<int64_t>(s_gb[cb]) - static_cast<int64_t>(b0);
        if (d <= 0) cnt += 1u;  // threshold at or below the bin start (gamma <= 1 in bin 0): always reached
        else L = static_cast<uint32_t>(d);
        while (s_b[cb] == b) ++cb;  // (two in one bin: conflict, the table is not used)
    }
    return (cnt << 24) + 0x1000000u - L - b0;
}
// Per-image table build by 256 threads (t = 0..255) of a block / named-barrier
// group: thread j < 255 computes threshold j (fp64 exp2, as the host theta),
// then each thread fills 8 consecutive bins from a binary search over the
// sorted threshold bins. Two barriers (bar, then bar_or, which also returns
// whether any two thresholds share a bin or are out of order -> no table).
template <bool kF32 = false, class Bar, class BarOr>
__device__ __forceinline__ int build_step_table(int t, const Theta& theta, double lr, int* s_b, uint32_t* s_gb,
                                                uint32_t* s_lut, Bar bar, BarOr bar_or) {
    if (t < 255) {
        const float gam = kF32 ? exp2f(static_cast<float>(theta.v[t]) * static_cast<float>(lr))
                               : static_cast<float>(exp2(theta.v[t] * lr));
        s_b[t] = lut_bin(gam);
        s_gb[t] = __float_as_uint(gam);
    } else if (t == 255) {
        s_b[255] = 1 << 30;
    }
    bar();
    const int bad = t < 254 && s_b[t] >= s_b[t + 1];
    if (t < 256) {  // (groups of more than 256 threads: the rest only take the barriers)
        const int b0 = t * (kLutBins / 256);
        int cb = 0;
#pragma unroll
        for (int step = 128; step > 0; step >>= 1)
            if (s_b[cb + step - 1] < b0) cb += step;
#pragma unroll
        for (int j = 0; j < kLutBins / 256; ++j) s_lut[b0 + j] = step_word(b0 + j, cb, s_b, s_gb);
    }
    return bar_or(bad);
}
__device__ __forceinline__ int named_bar_or(int id, int nthreads, int pred) {
    int r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\tbarrier.red.or.pred q, %2, %3, p;\n\tselp.s32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"(pred), "r"(id), "r"(nthreads)
        : "memory");
    return r;
}

// ---------------------------------------------------------------- per-pixel tone
struct ToneU8 {
    float m, hk, t0, inv_den;
};
__device__ __forceinline__ ToneU8 make_tone_u8(float m, float slope) {
    ToneU8 c;
    c.m = m;
    c.hk = 0.5f * slope;
    c.t0 = tanhf(__fmul_rn(c.hk, m));
    c.inv_den = __frcp_rn(__fadd_rn(tanhf(__fmul_rn(c.hk, __fsub_rn(1.0f, m))), c.t0));
    return c;
}
// log2 with absolute error ~2^-22 over the whole range: exact exponent plus
// lg2.approx of the mantissa in [1, 2).
__device__ __forceinline__ float log2_split(float x) {
    const uint32_t b = __float_as_uint(x);
    const int e = static_cast<int>(b >> 23) - 127;
    const float mant = __uint_as_float((b & 0x7FFFFFu) | 0x3F800000u);
    float l;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(mant));
    return __fadd_rn(static_cast<float>(e), l);
}
// arithmetic path (no table): tanh-form sigmoid of the log-range t
__device__ __forceinline__ uint32_t tone_arith(float g, const HdrStat& st, const ToneU8& c) {
    float t;
    if (!(g > 0.0f)) t = 0.0f;
    else if (st.mode == 1) t = fminf(fmaxf(__fmul_rn(log2_split(__fmul_rn(g, st.inv_gmin)), st.inv_lrange), 0.0f), 1.0f);
    else t = 1.0f;
    const float v = fminf(fmaxf(__fmul_rn(__fadd_rn(tanhf(__fmul_rn(c.hk, __fsub_rn(t, c.m))), c.t0), c.inv_den), 0.0f), 1.0f);
    return __float_as_uint(__fadd_rz(__fmaf_rn(v, 255.0f, 0.5f), kMagic)) & 0xFFu;
}

// ---------------------------------------------------------------- pass 1: gray + per-warp (min, max)
__global__ void __launch_bounds__(kT) hdr_gray_kernel(const float* __restrict__ rgb, float* __restrict__ gray,
                                                      float2* __restrict__ parts, int64_t ppi, U8Consts k) {
    const int img = blockIdx.y, lane = threadIdx.x & 31;
    const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const float* in = rgb + static_cast<int64_t>(img) * ppi * 3;
    float* g = gray + static_cast<int64_t>(img) * ppi;
    float lo = INFINITY, hi = 0.0f;
    const bool vec = (ppi & 3) == 0 && (reinterpret_cast<uintptr_t>(rgb) & 15) == 0;
    if (vec) {  // 4 px per thread: 3 x 16 B in (evict-first), 16 B out; next quad prefetched into registers
        const int64_t nq = ppi >> 2, step = static_cast<int64_t>(gridDim.x) * kT;
        int64_t q = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
        float4 n0, n1, n2;
        if (q < nq) {
            const float4* src = reinterpret_cast<const float4*>(in + 12 * q);
            n0 = __ldcs(src);
            n1 = __ldcs(src + 1);
            n2 = __ldcs(src + 2);
        }
        for (; q < nq; q += step) {
            const float4 v0 = n0, v1 = n1, v2 = n2;
            if (q + step < nq) {
                const float4* src = reinterpret_cast<const float4*>(in + 12 * (q + step));
                n0 = __ldcs(src);
                n1 = __ldcs(src + 1);
                n2 = __ldcs(src + 2);
            }
            // the scalar twin of decolor_fast_x2 (same bits; no pair moves, see hdr_tm_kernel)
            const float2 a = make_float2(decolor_fast_x1(v0.x, v0.y, v0.z, k), decolor_fast_x1(v0.w, v1.x, v1.y, k));
            const float2 b = make_float2(decolor_fast_x1(v1.z, v1.w, v2.x, k), decolor_fast_x1(v2.y, v2.z, v2.w, k));
            track(a.x, lo, hi);
            track(a.y, lo, hi);
            track(b.x, lo, hi);
            track(b.y, lo, hi);
            reinterpret_cast<float4*>(g)[q] = make_float4(a.x, a.y, b.x, b.y);
        }
    } else {
        for (int64_t p = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; p < ppi;
             p += static_cast<int64_t>(gridDim.x) * kT) {
            const float v = decolor_fast_x1(in[3 * p], in[3 * p + 1], in[3 * p + 2], k);
            g[p] = v;
            track(v, lo, hi);
        }
    }
    warp_minmax(lo, hi);
    if (lane == 0) parts[static_cast<int64_t>(img) * kSlots + gwarp] = make_float2(lo, hi);
}

// ---------------------------------------------------------------- pass 2: statistic + threshold table
// per-image statistic from the folded (min over g > 0, max)
__device__ __forceinline__ HdrStat hdr_stat_of(float lo, float hi, double* lr) {
    HdrStat st{0.0f, 0.0f, 0, 0};
    *lr = 0.0;
    if (hi > 0.0f && lo <= hi) {
        st.inv_gmin = static_cast<float>(1.0 / static_cast<double>(lo));
        if (hi > lo) {
            st.mode = 1;
            *lr = log2(static_cast<double>(hi) / static_cast<double>(lo));
            st.inv_lrange = static_cast<float>(1.0 / *lr);
        } else {
            st.mode = 2;
        }
    }
    return st;
}

__global__ void __launch_bounds__(kT) hdr_stats_kernel(const float2* __restrict__ parts, int nslots,
                                                       HdrStat* __restrict__ stats, float2* __restrict__ luts,
                                                       Theta theta) {
    static_assert(kT == 256, "build_step_table takes 256 threads");
    __shared__ float s_lo[kWarps], s_hi[kWarps];
    __shared__ int s_b[256];
    __shared__ uint32_t s_gb[256];
    __shared__ uint32_t s_lut[kLutBins];
    const int img = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_wait();  // the gray pass's slots are complete and visible
    const float2* slots = parts + static_cast<int64_t>(img) * kSlots;
    float lo = INFINITY, hi = 0.0f;
    for (int q = tid; q < nslots; q += kT) {
        const float2 pr = slots[q];
        lo = fminf(lo, pr.x);
        hi = fmaxf(hi, pr.y);
    }
    warp_minmax(lo, hi);
    if (lane == 0) {
        s_lo[warp] = lo;
        s_hi[warp] = hi;
    }
    __syncthreads();
    lo = s_lo[0];
    hi = s_hi[0];
    for (int w = 1; w < kWarps; ++w) {
        lo = fminf(lo, s_lo[w]);
        hi = fmaxf(hi, s_hi[w]);
    }
    double lr;
    HdrStat st = hdr_stat_of(lo, hi, &lr);
    if (st.mode == 1 && lr < kLutOct - 1) {  // block-uniform
        const int bad = build_step_table(
            tid, theta, lr, s_b, s_gb, s_lut, [] { __syncthreads(); }, [](int p) { return __syncthreads_or(p); });
        uint32_t* lut = reinterpret_cast<uint32_t*>(luts) + static_cast<int64_t>(img) * kLutBins;
        for (int b = tid; b < kLutBins; b += kT) lut[b] = s_lut[b];
        st.lut = bad ? 0 : 1;
    }
    if (tid == 0) stats[img] = st;
}

// ---------------------------------------------------------------- pass 3: tone (image-uniform blocks)
// One 16-px chunk (4 x 16 B loads, one 16 B store) per thread per iteration;
// the per-image mode is hoisted out of the loop.
// Table path for images of a multiple of 4096 px: gray tiles of 16 KiB stream
// through a 3-stage cp.async.bulk ring; thread t takes float4 t + 256 j
// (conflict-free LDS.128) and stores 4 coalesced 32-bit words.
constexpr int kToneTilePx = 4096;
constexpr int kToneStages = 3;
constexpr int kToneSmem = kToneStages * kToneTilePx * 4 + kToneStages * 8;

template <class Px>
__device__ __forceinline__ void tone_loop(const float* __restrict__ g, uint8_t* __restrict__ o, int64_t ppi,
                                          bool discard, Px px) {
    if (ppi % kToneTilePx == 0) {
        // 4096-px tiles, thread t takes float4 t + 256 j (coalesced 128-bit loads,
        // coalesced 32-bit stores), next tile prefetched into registers
        const int64_t ntiles = ppi / kToneTilePx;
        const int tid = threadIdx.x;
        int64_t t = blockIdx.x;
        float4 nx[4];
        if (t < ntiles) {
#pragma unroll
            for (int j = 0; j < 4; ++j) nx[j] = __ldcs(reinterpret_cast<const float4*>(g + t * kToneTilePx) + tid + 256 * j);
        }
        for (; t < ntiles; t += gridDim.x) {
            float4 v[4] = {nx[0], nx[1], nx[2], nx[3]};
            if (t + gridDim.x < ntiles) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    nx[j] = __ldcs(reinterpret_cast<const float4*>(g + (t + gridDim.x) * kToneTilePx) + tid + 256 * j);
            }
            uint32_t* dst = reinterpret_cast<uint32_t*>(o + t * kToneTilePx);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                __stcs(dst + tid + 256 * j, px(v[j].x) | (px(v[j].y) << 8) | (px(v[j].z) << 16) | (px(v[j].w) << 24));
            // this thread's loads of tile t are consumed: one 128 B gray line per 8 threads' float4s
            if (discard && (tid & 7) == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j) discard_l2_line(g + t * kToneTilePx + 4 * (tid + 256 * j));
            }
        }
    } else if ((ppi & 15) == 0) {
        // register prefetch: chunk ch + step is in flight while chunk ch is toned
        const int64_t nchunks = ppi >> 4;
        const int64_t step = static_cast<int64_t>(gridDim.x) * kT;
        int64_t ch = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
        float4 nx[4];
        if (ch < nchunks) {
#pragma unroll
            for (int j = 0; j < 4; ++j) nx[j] = __ldcs(reinterpret_cast<const float4*>(g + (ch << 4)) + j);
        }
        for (; ch < nchunks; ch += step) {
            float v[16];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                v[4 * j] = nx[j].x;
                v[4 * j + 1] = nx[j].y;
                v[4 * j + 2] = nx[j].z;
                v[4 * j + 3] = nx[j].w;
            }
            if (ch + step < nchunks) {
#pragma unroll
                for (int j = 0; j < 4; ++j) nx[j] = __ldcs(reinterpret_cast<const float4*>(g + ((ch + step) << 4)) + j);
            }
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                w[j] = px(v[4 * j]) | (px(v[4 * j + 1]) << 8) | (px(v[4 * j + 2]) << 16) | (px(v[4 * j + 3]) << 24);
            st_global_cs_v4(o + (ch << 4), make_uint4(w[0], w[1], w[2], w[3]));
            // chunks (even, even + 1) are held by lanes (l, l + 1) of one warp, whose
            // loads this lane's results already waited on: one 128 B gray line --
            // only where that line is exactly these two chunks (an image whose
            // plane starts 64 B into a line shares its first / last line with
            // the neighbouring image, which another block may not have read yet)
            if (discard && (ch & 1) == 0 && ch + 1 < nchunks &&
                (reinterpret_cast<uintptr_t>(g + (ch << 4)) & 127) == 0)
                discard_l2_line(g + (ch << 4));
        }
    } else {
        for (int64_t p = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; p < ppi;
             p += static_cast<int64_t>(gridDim.x) * kT)
            o[p] = static_cast<uint8_t>(px(g[p]));
    }
}

// table lookup of one pixel; r = 0 (black) falls in bin 0 whose count is 0



template <class Px>
__device__ __forceinline__ void tone_tiles(const float* __restrict__ g, uint8_t* __restrict__ o, int64_t ppi,
                                           bool discard, uint8_t* smem, Px px) {
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kToneStages * kToneTilePx * 4);
    const int tid = threadIdx.x;
    const int64_t ntiles = ppi / kToneTilePx;
    if (tid == 0) {
        for (int s = 0; s < kToneStages; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    uint64_t pol = 0;
    if (tid == 0) {
        pol = l2_policy_evict_first();
        for (int s = 0; s < kToneStages; ++s) {
            const int64_t t = blockIdx.x + s * static_cast<int64_t>(gridDim.x);
            if (t < ntiles) {
                mbar_arrive_expect_tx(&bars[s], kToneTilePx * 4);
                bulk_g2s(smem + s * kToneTilePx * 4, g + t * kToneTilePx, kToneTilePx * 4, &bars[s], pol);
            }
        }
    }
    int s = 0;
    uint32_t phase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&bars[s], phase);
        const float4* src = reinterpret_cast<const float4*>(smem + s * kToneTilePx * 4);
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = src[tid + 256 * j];
        fence_proxy_async_smem();  // reads of stage s ordered before its TMA refill
        __syncthreads();
        if (tid == 0) {
            const int64_t tn = t + kToneStages * static_cast<int64_t>(gridDim.x);
            if (tn < ntiles) {
                mbar_arrive_expect_tx(&bars[s], kToneTilePx * 4);
                bulk_g2s(smem + s * kToneTilePx * 4, g + tn * kToneTilePx, kToneTilePx * 4, &bars[s], pol);
            }
        }
        if (discard && tid < kToneTilePx * 4 / 128) discard_l2_line(g + t * kToneTilePx + tid * 32);
        uint32_t* dst = reinterpret_cast<uint32_t*>(o + t * kToneTilePx);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            __stcs(dst + tid + 256 * j, px(v[j].x) | (px(v[j].y) << 8) | (px(v[j].z) << 16) | (px(v[j].w) << 24));
        if (++s == kToneStages) {
            s = 0;
            phase ^= 1u;
        }
    }
}

__global__ void __launch_bounds__(kT) hdr_tone_tiled_kernel(const float* __restrict__ gray, uint8_t* __restrict__ out,
                                                            int64_t ppi, const HdrStat* __restrict__ stats,
                                                            const float2* __restrict__ luts, float m, float slope,
                                                            bool discard) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t s_lut[kLutBins];
    const int64_t img = blockIdx.y;
    pdl_wait();  // stats / tables of the previous (stats) grid
    const HdrStat st = stats[img];
    const float* g = gray + img * ppi;
    uint8_t* o = out + img * ppi;
    if (st.mode == 1 && st.lut) {  // block-uniform
        const uint32_t* lut = reinterpret_cast<const uint32_t*>(luts) + img * kLutBins;
        for (int q = threadIdx.x; q < kLutBins; q += kT) s_lut[q] = lut[q];
        // (made visible by the __syncthreads inside tone_tiles before first use)
        const float inv = st.inv_gmin;
        tone_tiles(g, o, ppi, discard, smem, [&](float v) -> uint32_t { return lut_px32(v, inv, s_lut); });
    } else if (st.mode == 2) {
        tone_tiles(g, o, ppi, discard, smem, [](float v) -> uint32_t { return v > 0.0f ? 255u : 0u; });
    } else {
        const ToneU8 c = make_tone_u8(m, slope);
        tone_tiles(g, o, ppi, discard, smem, [&](float v) -> uint32_t { return tone_arith(v, st, c); });
    }
}

__global__ void __launch_bounds__(kT) hdr_tone_kernel(const float* __restrict__ gray, uint8_t* __restrict__ out,
                                                      int64_t ppi, const HdrStat* __restrict__ stats,
                                                      const float2* __restrict__ luts, float m, float slope,
                                                      bool discard) {
    __shared__ uint32_t s_lut[kLutBins];
    const int64_t img = blockIdx.y;
    pdl_wait();  // stats / tables of the previous (stats) grid
    const HdrStat st = stats[img];
    const float* g = gray + img * ppi;
    uint8_t* o = out + img * ppi;
    if (st.mode == 1 && st.lut) {
        const uint32_t* lut = reinterpret_cast<const uint32_t*>(luts) + img * kLutBins;
        for (int q = threadIdx.x; q < kLutBins; q += kT) s_lut[q] = lut[q];
        __syncthreads();
        const float inv = st.inv_gmin;
        tone_loop(g, o, ppi, discard, [&](float v) -> uint32_t { return lut_px32(v, inv, s_lut); });
    } else if (st.mode == 2) {
        tone_loop(g, o, ppi, discard, [](float v) -> uint32_t { return v > 0.0f ? 255u : 0u; });  // t = 1
    } else {
        const ToneU8 c = make_tone_u8(m, slope);
        tone_loop(g, o, ppi, discard, [&](float v) -> uint32_t { return tone_arith(v, st, c); });
    }
}

// ================================================================ warp-specialised persistent schedule (default)
// One cooperative launch for the whole batch; every CTA owns the same
// contiguous range of 128-byte gray lines (32 px) of every image, so the gray
// plane is produced and consumed inside one CTA and only the statistic crosses
// CTAs:
//  * producer warps (12): gray of image i over the CTA's range -> ring slot
//    i % nring (L2 evict_last: the ring is sized to stay in L2), exact
//    (min over g > 0, max); the CTA's partial goes to parts[i][c] and a
//    per-image completion count (release);
//  * consumer warps (4): wait until all CTAs' partials of image i are in
//    (acquire), fold them, build the threshold table in shared memory (the
//    same table as hdr_stats_kernel), tone the CTA's range of image i from the
//    ring and drop the consumed gray lines from L2 (discard: no write-back),
//    then release the ring slot to this CTA's producers.
// Producers never wait on other CTAs (only on their own consumers freeing a
// slot nring images back), so the grid-wide dependency and the table build
// overlap the next images' gray pass. HBM traffic is the compulsory 12 B/px
// in + 1 B/px out (the gray plane stays in L2). Same per-pixel gray, min/max
// and table arithmetic as the grouped schedule: identical bytes.
constexpr int kWsT = 1024;   // one CTA per SM
// warps: kWsT / 32 - kCons producers (the gray pass is bound by the loads in
// flight per SM), kCons consumers (table build + tone from L2, latency-bound)
constexpr int kWsLinePx = 32;    // partition unit: one 128 B gray line
constexpr int kWsMaxGrid = 1024;  // partial slots per image
constexpr int kWsMaxRing = 4;
// gray ring bytes kept L2-resident: 2 slots (C4: 2 slots 322.6, 3 slots 310.8,
// 4 slots 294 Gpix/s -- the ring competes with the RGB stream for L2)
constexpr size_t kWsRingBudget = 0;
// producer L2 prefetch distance in waves of the CTA's range (C4, TMEM kernel
// before the cross-image register prefetch: 0 -> 320.8, 2 -> 339.5, 3 -> 340.1,
// 8 -> 336.7 Gpix/s; after: 2 -> 362.1, 3 -> 359.7, 6 -> 359.6; with the scalar
// producer loop: 1 -> 386.2, 2 -> 408.1, 3 -> 423.5, 4 -> 426.4, 5 -> 425.0;
// L2 ring: 0 -> 296, 3 -> 309)
constexpr int kWsPrefetchWaves = 4;



__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned target) {
    // relaxed polling (an ld.acquire per poll compiles to an L1 invalidate each
    // time, which stalls the SM's shared-memory pipe for the producers), one
    // acquire fence once the count is reached; bounded: a broken co-residency
    // assumption must fail loudly, not hang the GPU
    for (uint32_t spins = 0; ld_relaxed(p) < target; ++spins) {
        __nanosleep(256);
        if (spins > (1u << 25)) __trap();
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_v4_hint(float* p, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
}
// bulk L2 prefetch (no registers, no shared memory): the producers' loads then
// hit L2, so the same registers in flight sustain more HBM bandwidth
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}


// the rare arithmetic path out of line (keeps the unrolled consumer loop's registers)
__device__ __noinline__ uint32_t tone_arith_call(float g, HdrStat st, ToneU8 c) { return tone_arith(g, st, c); }

// The quads / 16-px chunks of an image a CTA owns (the same for every image):
// one contiguous range of 128 B gray lines [l0, l1). (Interleaving blocks of
// 8 lines over the CTAs -- the grid streaming each image as one wave --
// measured the same: 276 vs 265 Gpix/s, producers alone 353 vs 361.)
struct WsMap {
    int64_t l0, l1;
    __device__ __forceinline__ int64_t nquads() const { return (l1 - l0) * 8; }
    __device__ __forceinline__ int64_t nchunks() const { return (l1 - l0) * 2; }
    __device__ __forceinline__ int64_t quad(int64_t u) const { return l0 * 8 + u; }
    __device__ __forceinline__ int64_t chunk(int64_t v) const { return l0 * 2 + v; }
};

// consumer tone of a CTA's chunks: 16-px chunks, chunk pairs (one 128 B gray
// line) on lanes (2l, 2l + 1) of one warp, the line dropped from L2 once both
// are read
template <int kU, int kConsT, class Px>
__device__ __forceinline__ void ws_tone_range(const float* __restrict__ gsl, uint8_t* __restrict__ o,
                                              const WsMap& mp, int ct, Px px) {
    // warp-uniform trip count (the __syncwarp below needs every lane); lanes past
    // the range idle. CTA-local chunks 2j, 2j + 1 are one 128 B gray line and sit
    // on lanes (2l, 2l + 1); kU chunks per lane per iteration, all loads issued
    // before any use (L2 latency, not bandwidth, bounds these few warps).
    const int lane = ct & 31;
    const int64_t nch = mp.nchunks();
    for (int64_t base = ct - lane; base < nch; base += kU * kConsT) {
        float4 x[kU][4];
#pragma unroll
        for (int u = 0; u < kU; ++u) {  // unconditional loads (clamped index): no maybe-unset registers
            const int64_t ch = mp.chunk(min(base + lane + u * kConsT, nch - 1));
            const float4* src = reinterpret_cast<const float4*>(gsl + (ch << 4));
#pragma unroll
            for (int j = 0; j < 4; ++j) x[u][j] = __ldcg(src + j);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t v = base + lane + u * kConsT;
            if (v < nch) {
                const int64_t ch = mp.chunk(v);
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    w[j] = px(x[u][j].x) | (px(x[u][j].y) << 8) | (px(x[u][j].z) << 16) | (px(x[u][j].w) << 24);
                st_global_cs_v4(o + (ch << 4), make_uint4(w[0], w[1], w[2], w[3]));
            }
        }
        __syncwarp();  // both chunks of each line are read (their values are used above)
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t v = base + lane + u * kConsT;
            if (v < nch && (lane & 1) == 0) discard_l2_line(gsl + (mp.chunk(v) << 4));
        }
    }
}

template <int kCons_>
__global__ void __launch_bounds__(kWsT, 1)
    hdr_ws_kernel(const float* __restrict__ rgb, uint8_t* __restrict__ out, float* __restrict__ ring,
                  float2* __restrict__ parts, unsigned* __restrict__ counts, int64_t nimg, int64_t ppi, int nring,
                  U8Consts k, float m, float slope, Theta theta, int pf_waves) {
    constexpr int kProd_ = kWsT / 32 - kCons_, kProdT_ = kProd_ * 32, kConsT_ = kCons_ * 32;
    static_assert(kConsT_ == 256, "build_step_table takes 256 consumer threads");
    __shared__ uint32_t s_lut[kLutBins];
    __shared__ int s_b[256];
    __shared__ uint32_t s_gb[256];
    __shared__ float s_plo[kProd_], s_phi[kProd_], s_clo[kCons_], s_chi[kCons_];
    __shared__ volatile int s_toned;  // images this CTA's consumers have finished
    __shared__ int s_pf[2];           // producer thread 0: next (image, wave) to prefetch into L2
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t nlines = ppi / kWsLinePx;
    const WsMap mp{nlines * c / G, nlines * (c + 1) / G};
    if (tid == 0) {
        s_toned = 0;
        s_pf[0] = s_pf[1] = 0;
    }
    __syncthreads();

    if (warp < kProd_) {
        // ---------------- producers: three 128-bit loads per quad, the next quad in flight
        const uint64_t pol_gray = l2_policy_evict_last();
        const int64_t nq = mp.nquads();  // this CTA's quads (4 px) of every image
        // L2 prefetch pf_waves waves (kProdT_ quads, 36 KiB) ahead of the loads,
        // across image boundaries; thread 0 keeps the next (image, wave) in
        // shared memory (no registers in the other threads)
        const int nw = static_cast<int>((nq + kProdT_ - 1) / kProdT_);
        auto prefetch_next = [&]() {
            const int i2 = s_pf[0], w2 = s_pf[1];
            if (i2 >= nimg) return;
            const int64_t q0 = static_cast<int64_t>(w2) * kProdT_, q1 = min(nq, q0 + kProdT_);
            prefetch_l2_bulk(rgb + i2 * ppi * 3 + 12 * mp.quad(q0), static_cast<uint32_t>((q1 - q0) * 48));
            if (w2 + 1 == nw) {
                s_pf[0] = i2 + 1;
                s_pf[1] = 0;
            } else {
                s_pf[1] = w2 + 1;
            }
        };
        if (tid == 0)
            for (int w = 0; w < pf_waves; ++w) prefetch_next();
        // (as hdr_tm_kernel: register prefetch continued across images, two
        // register buffers in turn, one selected-pointer load per quad, an
        // integer minimum over g > 0; lanes past the range load and track a
        // clamped duplicate quad and store nothing)
        const uint32_t nq32 = static_cast<uint32_t>(nq), ulast = nq32 - 1u;
        const float* base0 = rgb + 12 * mp.quad(0);
        const int64_t img_floats = ppi * 3;
        struct Quad {
            float4 a, b, c;
        };
        Quad qa, qb;
        {
            const float4* src = reinterpret_cast<const float4*>(base0) + 3u * min(static_cast<uint32_t>(tid), ulast);
            qa.a = __ldcs(src);
            qa.b = __ldcs(src + 1);
            qa.c = __ldcs(src + 2);
        }
        for (int64_t i = 0; i < nimg; ++i) {
            if (i >= nring) {  // slot i % nring: this CTA's consumers are done with image i - nring
                for (uint32_t spins = 0; s_toned < i - nring + 1; ++spins) {
                    __nanosleep(64);
                    if (spins > (1u << 26)) __trap();
                }
            }
            float* g = ring + (i % nring) * ppi + 4 * mp.quad(0);
            const float* base = base0 + i * img_floats;
            const float* alt = i + 1 < nimg ? base + img_floats + 12u * min(static_cast<uint32_t>(tid), ulast) : base;
            uint32_t lo1 = 0xFFFFFFFFu;
            float hi = 0.0f;
            const auto body = [&](const Quad& cur, Quad& nxt, uint32_t u) {
                if (pf_waves > 0 && tid == 0) prefetch_next();
                {
                    const float* src = u + kProdT_ < nq32 ? base + 12u * (u + kProdT_) : alt;
                    const float4* s4 = reinterpret_cast<const float4*>(src);
                    nxt.a = __ldcs(s4);
                    nxt.b = __ldcs(s4 + 1);
                    nxt.c = __ldcs(s4 + 2);
                }
                const float2 a = make_float2(decolor_fast_x1(cur.a.x, cur.a.y, cur.a.z, k),
                                             decolor_fast_x1(cur.a.w, cur.b.x, cur.b.y, k));
                const float2 b = make_float2(decolor_fast_x1(cur.b.z, cur.b.w, cur.c.x, k),
                                             decolor_fast_x1(cur.c.y, cur.c.z, cur.c.w, k));
                lo1 = min(min(min(lo1, __float_as_uint(a.x) - 1u), min(__float_as_uint(a.y) - 1u, __float_as_uint(b.x) - 1u)),
                          __float_as_uint(b.y) - 1u);
                hi = fmaxf(fmaxf(fmaxf(hi, a.x), fmaxf(a.y, b.x)), b.y);
                st_v4_hint(g + 4 * u, make_float4(a.x, a.y, b.x, b.y), pol_gray);
            };
            for (uint32_t u = tid;;) {
                if (u >= nq32) break;
                body(qa, qb, u);
                u += kProdT_;
                if (u >= nq32) {
                    qa = qb;  // the next image's first quad (once per image)
                    break;
                }
                body(qb, qa, u);
                u += kProdT_;
            }
            if (static_cast<uint32_t>(tid) >= nq32 && i + 1 < nimg) {  // (a range smaller than one wave)
                const float4* src = reinterpret_cast<const float4*>(alt);
                qa.a = __ldcs(src);
                qa.b = __ldcs(src + 1);
                qa.c = __ldcs(src + 2);
            }
            float lo = lo1 >= 0x7F800000u ? INFINITY : __uint_as_float(lo1 + 1u);
            warp_minmax(lo, hi);
            if (lane == 0) {
                s_plo[warp] = lo;
                s_phi[warp] = hi;
            }
            __threadfence();  // this thread's gray stores before the image's completion count
            named_bar(1, kProdT_);
            if (tid == 0) {
                for (int w = 0; w < kProd_; ++w) {
                    lo = fminf(lo, s_plo[w]);
                    hi = fmaxf(hi, s_phi[w]);
                }
                __stcg(parts + i * kWsMaxGrid + c, make_float2(lo, hi));
                __threadfence();
                atomicAdd(counts + i, 1u);
            }
            named_bar(1, kProdT_);  // s_plo / s_phi are rewritten for the next image
        }
        return;
    }

    // ---------------- consumers
    const int ct = tid - kProdT_, cw = ct >> 5;
    const ToneU8 tc = make_tone_u8(m, slope);
    for (int64_t i = 0; i < nimg; ++i) {
        if (ct == 0) wait_geq(counts + i, static_cast<unsigned>(G));
        named_bar(2, kConsT_);
        float lo = INFINITY, hi = 0.0f;
        for (int q = ct; q < G; q += kConsT_) {
            const float2 pr = __ldcg(parts + i * kWsMaxGrid + q);
            lo = fminf(lo, pr.x);
            hi = fmaxf(hi, pr.y);
        }
        warp_minmax(lo, hi);
        if (lane == 0) {
            s_clo[cw] = lo;
            s_chi[cw] = hi;
        }
        named_bar(2, kConsT_);
        lo = s_clo[0];
        hi = s_chi[0];
        for (int w = 1; w < kCons_; ++w) {
            lo = fminf(lo, s_clo[w]);
            hi = fmaxf(hi, s_chi[w]);
        }
        double lr;
        HdrStat st = hdr_stat_of(lo, hi, &lr);
        if (st.mode == 1 && lr < kLutOct - 1) {  // uniform over the consumer warps
            const int bad = build_step_table(
                ct, theta, lr, s_b, s_gb, s_lut, [] { named_bar(2, kConsT_); },
                [](int p) { return named_bar_or(2, kConsT_, p); });
            st.lut = bad ? 0 : 1;
        }
        // tone this CTA's lines (per-image mode hoisted out of the pixel loop)
        const float* gsl = ring + (i % nring) * ppi;
        uint8_t* o = out + i * ppi;
        if (st.mode == 1 && st.lut) {
            const float inv = st.inv_gmin;
            ws_tone_range<2, kConsT_>(gsl, o, mp, ct, [&](float v) -> uint32_t { return lut_px32(v, inv, s_lut); });
        } else if (st.mode == 2) {
            ws_tone_range<2, kConsT_>(gsl, o, mp, ct, [](float v) -> uint32_t { return v > 0.0f ? 255u : 0u; });
        } else {
            ws_tone_range<2, kConsT_>(gsl, o, mp, ct, [&](float v) -> uint32_t { return tone_arith_call(v, st, tc); });
        }
        named_bar(2, kConsT_);  // every consumer is done with the slot and with s_lut
        if (ct == 0) s_toned = static_cast<int>(i + 1);
    }
}

// ---------------------------------------------------------------- TMEM-staged variant
// hdr_tm_kernel: the same warp-specialised schedule, but the gray of the CTA's
// range never leaves the SM: producers tcgen05.st it into tensor memory (256 KiB
// per SM, otherwise unused by this bandwidth-bound map: 2 slots of 128 lanes x
// 256 columns = 32768 px each), consumers tcgen05.ld it back. HBM/L2 traffic is
// the compulsory 12 B/px in + 1 B/px out and no gray line competes with the RGB
// stream for L2. Fits when a CTA's per-image range is <= 8192 quads (C4: 7085).
// Quad u of the range lives at TMEM lane u % 128, columns 4 (u / 128) + 0..3:
// kProdT_ is a multiple of 128, so producer warp w always hits lanes
// 32 (w % 4) .. + 31 -- the lanes its warp may access -- and a consumer warp
// reads whole column groups of its own quadrant.
constexpr int kTmCols = 512, kTmSlotCols = 256, kTmMaxQuads = kTmSlotCols / 4 * 128;
// timing trace of the TMEM kernel (kDbg == 4, scripts/hdr_trace.py): per (image,
// CTA) globaltimer at producer start / publish, consumer start / done / table built
constexpr int kTraceImgs = 64;
__device__ unsigned long long g_hdr_trace[kTraceImgs][kWsMaxGrid][7];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void tm_st4(uint32_t taddr, float a, float b, float c, float d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d))
                 : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// consumer tone of one slot: warp cw of quadrant cw % 4, half cw / 4 of the
// column groups, four groups (16 columns) per tcgen05.ld -- or, for the
// shared-memory slot (sslot != nullptr), four conflict-free LDS.128 of the same
// quads; one 32-bit store per quad (a warp stores 128 contiguous bytes)
template <int kCons_, bool kByte3, class Px>
__device__ __forceinline__ void tm_tone_slot(uint32_t tslot, const float4* sslot, uint8_t* __restrict__ o,
                                             int64_t nq, int cw, int lane, Px px) {
    const int qd = cw & 3, h = cw >> 2;
    constexpr int kHalves = kCons_ / 4;
    const int ncg = static_cast<int>((nq + 127) >> 7);
    const int per = (((ncg + kHalves - 1) / kHalves) + 3) & ~3;  // groups per warp, a multiple of 4
    const int g0 = h * per, g1 = min(ncg, g0 + per);
    const uint32_t tl = tslot + (static_cast<uint32_t>(qd * 32) << 16);
    for (int g = g0; g < g1; g += 4) {
        uint32_t r[16];
        if (sslot) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t u = min((static_cast<int64_t>(g + j) << 7) + qd * 32 + lane, nq - 1);
                const float4 v = sslot[u];
                r[4 * j] = __float_as_uint(v.x);
                r[4 * j + 1] = __float_as_uint(v.y);
                r[4 * j + 2] = __float_as_uint(v.z);
                r[4 * j + 3] = __float_as_uint(v.w);
            }
        } else {
            tm_ld16(tl + 4 * g, r);
            tm_wait_ld();
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t u = (static_cast<int64_t>(g + j) << 7) + qd * 32 + lane;
            if (g + j < g1 && u < nq) {
                uint32_t w;
                if (kByte3) {  // px returns a step sum whose byte 3 is the toned byte: 3 PRMT per quad
                    const uint32_t lo = __byte_perm(px(__uint_as_float(r[4 * j])), px(__uint_as_float(r[4 * j + 1])), 0x0073);
                    const uint32_t hi =
                        __byte_perm(px(__uint_as_float(r[4 * j + 2])), px(__uint_as_float(r[4 * j + 3])), 0x0073);
                    w = __byte_perm(lo, hi, 0x5410);
                } else {
                    w = px(__uint_as_float(r[4 * j])) | (px(__uint_as_float(r[4 * j + 1])) << 8) |
                        (px(__uint_as_float(r[4 * j + 2])) << 16) | (px(__uint_as_float(r[4 * j + 3])) << 24);
                }
                __stcs(reinterpret_cast<unsigned*>(o) + u, w);
            }
        }
    }
}

// kDbg & 4: per-image globaltimer trace (scripts/hdr_trace.py); kRing 3: a third
// slot in shared memory (A/B only: slower); kPackedGray: the producers' packed
// f32x2 gray (A/B only: slower, ~40 register moves per quad)
template <int kCons_, int kDbg = 0, int kRing = 2, bool kPackedGray = false>
__global__ void __launch_bounds__(kWsT, 1)
    hdr_tm_kernel(const float* __restrict__ rgb, uint8_t* __restrict__ out, float2* __restrict__ parts,
                  unsigned* __restrict__ counts, int64_t nimg, int64_t ppi, U8Consts k, float m, float slope,
                  Theta theta, int pf_waves) {
    // (12 consumer warps measured slower: 401 vs 423 Gpix/s, fewer producers)
    static_assert(kCons_ % 4 == 0, "consumer warps come in whole quadrant sets");
    constexpr int kProd_ = kWsT / 32 - kCons_, kProdT_ = kProd_ * 32, kConsT_ = kCons_ * 32;
    static_assert(kProdT_ % 128 == 0, "producer waves must cover whole TMEM column groups");
    static_assert(kRing == 2 || kRing == 3, "2 TMEM slots (+ 1 shared-memory slot)");
    extern __shared__ float4 s_slot[];  // the third slot (kRing == 3): kTmMaxQuads quads
    static_assert(kConsT_ >= 256, "build_step_table takes 256 consumer threads");
    __shared__ uint32_t s_lut[kLutBins];
    __shared__ int s_b[256];
    __shared__ uint32_t s_gb[256];
    __shared__ float s_plo[kProd_], s_phi[kProd_], s_clo[kCons_], s_chi[kCons_];
    __shared__ volatile int s_toned;  // images this CTA's consumers have finished
    __shared__ int s_pf[2];           // producer thread 0: next (image, wave) to prefetch into L2
    __shared__ uint32_t s_tmem;       // TMEM base address (tcgen05.alloc)
    __shared__ HdrStat s_st;
    __shared__ double s_lr;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t nlines = ppi / kWsLinePx;
    const WsMap mp{nlines * c / G, nlines * (c + 1) / G};
    const int64_t nq = mp.nquads();  // <= kTmMaxQuads (host check)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem))),
                     "n"(kTmCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        s_toned = 0;
        s_pf[0] = s_pf[1] = 0;
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const uint32_t tbase = s_tmem;

    if (warp < kProd_) {
        // ---------------- producers: three 128-bit loads per quad, the next quad in flight
        const int nw = static_cast<int>((nq + kProdT_ - 1) / kProdT_);
        auto prefetch_next = [&]() {
            const int i2 = s_pf[0], w2 = s_pf[1];
            if (i2 >= nimg) return;
            const int64_t q0 = static_cast<int64_t>(w2) * kProdT_, q1 = min(nq, q0 + kProdT_);
            prefetch_l2_bulk(rgb + i2 * ppi * 3 + 12 * mp.quad(q0), static_cast<uint32_t>((q1 - q0) * 48));
            if (w2 + 1 == nw) {
                s_pf[0] = i2 + 1;
                s_pf[1] = 0;
            } else {
                s_pf[1] = w2 + 1;
            }
        };
        if (tid == 0)
            for (int w = 0; w < pf_waves; ++w) prefetch_next();
        const uint32_t tq = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16);  // this warp's lane quadrant
        // register prefetch of the next quad, continued across image boundaries
        // (the next image's first quad is in flight during the publish and the
        // slot wait); two register buffers used in turn (no copy of the
        // prefetched quad per iteration); 32-bit quad indices within the CTA's
        // range; lanes past the range load (and track) a clamped duplicate quad
        const uint32_t nq32 = static_cast<uint32_t>(nq), ulast = nq32 - 1u;
        const float* base0 = rgb + 12 * mp.quad(0);
        const int64_t img_floats = ppi * 3;
        struct Quad {
            float4 a, b, c;
        };
        auto load = [&](Quad& d, const float* base, uint32_t uq) {
            const float4* src = reinterpret_cast<const float4*>(base) + 3u * min(uq, ulast);
            d.a = __ldcs(src);
            d.b = __ldcs(src + 1);
            d.c = __ldcs(src + 2);
        };
        Quad qa, qb;
        load(qa, base0, tid);
        for (int64_t i = 0; i < nimg; ++i) {
            if (i >= kRing) {  // slot i % kRing: this CTA's consumers are done with image i - kRing
                for (uint32_t spins = 0; s_toned < i - kRing + 1; ++spins) {
                    __nanosleep(64);
                    if (spins > (1u << 26)) __trap();
                }
                tm_fence_after();
            }
            if ((kDbg & 4) && tid == 0 && i < kTraceImgs) g_hdr_trace[i][c][0] = gtimer();
            const int slot = static_cast<int>(i % kRing);
            const uint32_t ts = tq + static_cast<uint32_t>(slot * kTmSlotCols);
            const float* base = base0 + i * img_floats;
            // the quad loaded in the warp's last iteration: the next image's first
            // (a harmless reload of this image's after the last image)
            const float* alt = i + 1 < nimg ? base + img_floats + 12u * min(static_cast<uint32_t>(tid), ulast) : base;
            // min over g > 0 as the unsigned minimum of bits(g) - 1 (0 and negative
            // values wrap above every positive float), max as fmaxf
            uint32_t lo1 = 0xFFFFFFFFu;
            float hi = 0.0f;
            const auto body = [&](const Quad& cur, Quad& nxt, uint32_t u) {
                if (pf_waves > 0 && tid == 0) prefetch_next();
                {  // unconditional load (one selected pointer): no register merges
                    const float* src = u + kProdT_ - lane < nq32 ? base + 12u * min(u + kProdT_, ulast) : alt;
                    const float4* s4 = reinterpret_cast<const float4*>(src);
                    nxt.a = __ldcs(s4);
                    nxt.b = __ldcs(s4 + 1);
                    nxt.c = __ldcs(s4 + 2);
                }
                // scalar twin of decolor_fast_x2 (same per-lane operations, same
                // bits): the packed form needs ~40 register moves per quad to pair
                // same-channel values of the interleaved fp32 RGB
                float2 a, b;
                if (kPackedGray) {
                    a = decolor_fast_x2(make_float2(cur.a.x, cur.a.w), make_float2(cur.a.y, cur.b.x),
                                        make_float2(cur.a.z, cur.b.y), k);
                    b = decolor_fast_x2(make_float2(cur.b.z, cur.c.y), make_float2(cur.b.w, cur.c.z),
                                        make_float2(cur.c.x, cur.c.w), k);
                } else {
                    a.x = decolor_fast_x1(cur.a.x, cur.a.y, cur.a.z, k);
                    a.y = decolor_fast_x1(cur.a.w, cur.b.x, cur.b.y, k);
                    b.x = decolor_fast_x1(cur.b.z, cur.b.w, cur.c.x, k);
                    b.y = decolor_fast_x1(cur.c.y, cur.c.z, cur.c.w, k);
                }
                lo1 = min(min(min(lo1, __float_as_uint(a.x) - 1u), min(__float_as_uint(a.y) - 1u, __float_as_uint(b.x) - 1u)),
                          __float_as_uint(b.y) - 1u);
                hi = fmaxf(fmaxf(fmaxf(hi, a.x), fmaxf(a.y, b.x)), b.y);
                if (slot < 2) tm_st4(ts + 4u * (u >> 7), a.x, a.y, b.x, b.y);
                else if (u < nq32) s_slot[u] = make_float4(a.x, a.y, b.x, b.y);
            };
            // warp-uniform trip count (tcgen05.st is .aligned)
            for (uint32_t u = tid;;) {
                if (u - lane >= nq32) break;
                body(qa, qb, u);
                u += kProdT_;
                if (u - lane >= nq32) {
                    qa = qb;  // the next image's first quad (once per image)
                    break;
                }
                body(qb, qa, u);
                u += kProdT_;
            }
            float lo = lo1 >= 0x7F800000u ? INFINITY : __uint_as_float(lo1 + 1u);  // none (or NaN / negative only)
            tm_wait_st();
            tm_fence_before();
            warp_minmax(lo, hi);
            if (lane == 0) {
                s_plo[warp] = lo;
                s_phi[warp] = hi;
            }
            named_bar(1, kProdT_);
            if (tid == 0) {
                for (int w = 0; w < kProd_; ++w) {
                    lo = fminf(lo, s_plo[w]);
                    hi = fmaxf(hi, s_phi[w]);
                }
                __stcg(parts + i * kWsMaxGrid + c, make_float2(lo, hi));
                __threadfence();
                atomicAdd(counts + i, 1u);
                if ((kDbg & 4) && i < kTraceImgs) g_hdr_trace[i][c][1] = gtimer();
            }
            named_bar(1, kProdT_);  // s_plo / s_phi are rewritten for the next image
        }
    } else {
        // ---------------- consumers
        const int ct = tid - kProdT_, cw = ct >> 5;
        const ToneU8 tc = make_tone_u8(m, slope);
        for (int64_t i = 0; i < nimg; ++i) {
            if (ct == 0) {
                wait_geq(counts + i, static_cast<unsigned>(G));
                if ((kDbg & 4) && i < kTraceImgs) g_hdr_trace[i][c][2] = gtimer();
            }
            named_bar(2, kConsT_);
            tm_fence_after();
            float lo = INFINITY, hi = 0.0f;
            for (int q = ct; q < G; q += kConsT_) {
                const float2 pr = __ldcg(parts + i * kWsMaxGrid + q);
                lo = fminf(lo, pr.x);
                hi = fmaxf(hi, pr.y);
            }
            warp_minmax(lo, hi);
            if (lane == 0) {
                s_clo[cw] = lo;
                s_chi[cw] = hi;
            }
            named_bar(2, kConsT_);
            if ((kDbg & 4) && ct == 0 && i < kTraceImgs) g_hdr_trace[i][c][5] = gtimer();
            lo = s_clo[0];
            hi = s_chi[0];
            for (int w = 1; w < kCons_; ++w) {
                lo = fminf(lo, s_clo[w]);
                hi = fmaxf(hi, s_chi[w]);
            }
            double lr;
            // the statistic (fp64 log2 and divisions) by one thread, broadcast
            // (C4: +0.7% over every consumer thread computing it)
            if (ct == 0) {
                s_st = hdr_stat_of(lo, hi, &lr);
                s_lr = lr;
            }
            named_bar(2, kConsT_);
            HdrStat st = s_st;
            lr = s_lr;
            if ((kDbg & 4) && ct == 0 && i < kTraceImgs) g_hdr_trace[i][c][6] = gtimer();
            if (st.mode == 1 && lr < kLutOct - 1) {  // uniform over the consumer warps
                const int bad = build_step_table<(kDbg & 16) != 0>(
                    ct, theta, lr, s_b, s_gb, s_lut, [] { named_bar(2, kConsT_); },
                    [](int p) { return named_bar_or(2, kConsT_, p); });
                st.lut = bad ? 0 : 1;
            }
            if ((kDbg & 4) && ct == 0 && i < kTraceImgs) g_hdr_trace[i][c][4] = gtimer();
            const int slot = static_cast<int>(i % kRing);
            const uint32_t ts = tbase + static_cast<uint32_t>(slot * kTmSlotCols);
            const float4* ss = slot < 2 ? nullptr : s_slot;
            uint8_t* o = out + i * ppi + mp.quad(0) * 4;
            if (st.mode == 1 && st.lut) {
                const float inv = st.inv_gmin;
                tm_tone_slot<kCons_, true>(ts, ss, o, nq, cw, lane,
                                           [&](float v) -> uint32_t { return lut_step_sum(v, inv, s_lut); });
            } else if (st.mode == 2) {
                tm_tone_slot<kCons_, false>(ts, ss, o, nq, cw, lane, [](float v) -> uint32_t { return v > 0.0f ? 255u : 0u; });
            } else {
                tm_tone_slot<kCons_, false>(ts, ss, o, nq, cw, lane,
                                     [&](float v) -> uint32_t { return tone_arith_call(v, st, tc); });
            }
            tm_fence_before();
            named_bar(2, kConsT_);  // every consumer is done with the slot and with s_lut
            if (ct == 0) {
                s_toned = static_cast<int>(i + 1);
                if ((kDbg & 4) && i < kTraceImgs) g_hdr_trace[i][c][3] = gtimer();
            }
        }
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmCols) : "memory");
}

// ---------------------------------------------------------------- host helpers
// opt-in knobs are read per call (tests switch them within one process)
bool ws_enabled() {
    // WG_HDR_SCHEDULE=grouped: the three-kernel grouped schedule (A/B tests);
    // C4: 308 vs 288 Gpix/s
    const char* e = getenv("WG_HDR_SCHEDULE");
    return !(e && std::strcmp(e, "grouped") == 0);
}
size_t l2_budget() {
    const char* e = getenv("WG_HDR_L2_BUDGET_MB");  // tuning knob (scripts/), default kL2Budget
    return e ? static_cast<size_t>(atoll(e)) << 20 : kL2Budget;
}
// launch with programmatic stream serialization (PDL) when `pdl`, else a plain launch
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, cudaStream_t s, bool pdl, Args... args) {
    if (!pdl || getenv("WG_HDR_NO_PDL")) {
        kern<<<grid, kT, 0, s>>>(args...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

int group_size(int64_t nimg, int64_t ppi) {
    const int64_t fit = static_cast<int64_t>(l2_budget() / (static_cast<size_t>(ppi) * sizeof(float)));
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({fit, nimg, kMaxGroup})));
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
int ws_ring(int64_t ppi) {
    size_t budget = kWsRingBudget;
    if (const char* e = getenv("WG_HDR_RING_MB")) budget = static_cast<size_t>(atoll(e)) << 20;  // tuning knob
    const int64_t fit = static_cast<int64_t>(budget / (static_cast<size_t>(ppi) * sizeof(float)));
    return static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(fit, kWsMaxRing)));
}
size_t ws_bytes(int64_t nimg, int64_t ppi) {
    // gray ring | partials [nimg][kWsMaxGrid] | completion counts [nimg]
    return align256(static_cast<size_t>(ws_ring(ppi)) * ppi * sizeof(float)) +
           align256(static_cast<size_t>(nimg) * kWsMaxGrid * sizeof(float2)) +
           align256(static_cast<size_t>(nimg) * sizeof(unsigned));
}
// two scratch sets (double buffering across the two streams) when there is more than one group
int scratch_sets(int64_t nimg, int64_t ppi) {
    const int g = group_size(nimg, ppi);
    return (nimg + g - 1) / g > 1 ? 2 : 1;
}
size_t grouped_bytes(int64_t nimg, int64_t ppi) {
    // per set: G gray planes | G slot arrays | G tables | stats[G]
    const size_t g = static_cast<size_t>(group_size(nimg, ppi));
    return scratch_sets(nimg, ppi) * (align256(g * ppi * sizeof(float)) + align256(g * kSlots * sizeof(float2)) +
                                      align256(g * kLutBins * sizeof(float2)) + align256(g * sizeof(HdrStat)));
}

// per-device auxiliary stream + events of the pipelined grouped schedule
struct HdrStreams {
    std::mutex mu;
    cudaStream_t aux = nullptr;
    cudaEvent_t start = nullptr, gray_done[2] = {nullptr, nullptr}, tone_done[2] = {nullptr, nullptr};
};
HdrStreams* hdr_streams(int device) {
    static HdrStreams hs[kMaxDevices];
    static std::mutex init_mu;
    if (device < 0 || device >= kMaxDevices) return nullptr;
    std::lock_guard<std::mutex> g(init_mu);
    HdrStreams& h = hs[device];
    if (!h.aux) {
        if (cudaStreamCreateWithFlags(&h.aux, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        cudaEventCreateWithFlags(&h.start, cudaEventDisableTiming);
        for (int q = 0; q < 2; ++q) {
            cudaEventCreateWithFlags(&h.gray_done[q], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&h.tone_done[q], cudaEventDisableTiming);
        }
    }
    return &h;
}

Theta make_theta(double m, double k) {
    // theta_j: t where the reference's logistic (tonemap.py:76-81) reaches (j - 0.5) / 255
    Theta th;
    const double slo = 1.0 / (1.0 + std::exp(k * m)), shi = 1.0 / (1.0 + std::exp(-k * (1.0 - m)));
    for (int j = 0; j < 255; ++j) {
        const double y = (j + 0.5) / 255.0;
        const double p = slo + y * (shi - slo);
        th.v[j] = m + std::log(p / (1.0 - p)) / k;
    }
    return th;
}

}  // namespace
}  // namespace wg

using namespace wg;

// diagnostic: copy the TMEM kernel's timing trace (WG_HDR_TMDBG=4) to host memory
// (kTraceImgs x kWsMaxGrid x 7 uint64); returns the element count
extern "C" WG_API int64_t wg_hdr_debug_trace(uint64_t* host) {
    const size_t n = sizeof(g_hdr_trace) / sizeof(unsigned long long);
    if (host && cudaMemcpyFromSymbol(host, g_hdr_trace, sizeof(g_hdr_trace)) != cudaSuccess) return -1;
    return static_cast<int64_t>(n);
}

extern "C" size_t wg_hdr_scratch_bytes(int64_t nimg, int64_t pix_per_img) {
    if (nimg <= 0 || pix_per_img <= 0) return 0;
    return std::max(ws_bytes(nimg, pix_per_img), grouped_bytes(nimg, pix_per_img));
}

extern "C" int wg_hdr_tonemap_u8(const float* rgb, uint8_t* out, int64_t nimg, int64_t pix_per_img,
                                 float beta_r, float beta_k, float midpoint, float slope, void* scratch,
                                 size_t scratch_bytes, void* stream) {
    WG_CHECK_ARGS(check_npix(nimg) || check_npix(pix_per_img) || check_params(beta_r, beta_k) ||
                  check_curve(midpoint, slope));
    if (nimg == 0 || pix_per_img == 0) return WG_OK;
    if (!rgb || !out || !scratch) return set_error(WG_EINVAL, "hdr: null pointer");
    // the tone passes store 16 (grouped: 4) bytes at a time at pixel offsets that are
    // multiples of 16 when pix_per_img allows it: out must be 16-byte aligned
    if ((reinterpret_cast<uintptr_t>(out) & 15) != 0)
        return set_error(WG_EALIGN, "hdr: out must be 16-byte aligned");
    if ((reinterpret_cast<uintptr_t>(scratch) & 255) != 0)
        return set_error(WG_EALIGN, "hdr: scratch must be 256-byte aligned");
    if (scratch_bytes < wg_hdr_scratch_bytes(nimg, pix_per_img))
        return set_error(WG_ESCRATCH, "hdr: scratch buffer smaller than wg_hdr_scratch_bytes()");
    if (nimg > 65535) return set_error(WG_EINVAL, "hdr: at most 65535 images per call");
    int device = 0;
    cudaGetDevice(&device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const U8Consts k = make_u8_consts(beta_r, beta_k);
    const Theta theta = make_theta(midpoint, slope);
    const int sms = sm_count(device);
    // ---- default: the warp-specialised persistent kernel (cooperative launch:
    // its CTAs wait on each other's partials, so all must be co-resident)
    const bool ws_ok = (pix_per_img % kWsLinePx) == 0 && (reinterpret_cast<uintptr_t>(rgb) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(out) & 15) == 0 && device >= 0 && device < kMaxDevices;
    // 8 consumer warps of 32 (C4: 4 -> 274, 12 -> 261, 16 -> 270 vs 308 Gpix/s)
    static std::atomic<int> ws_occ[1][kMaxDevices];  // idempotent lazy cache
    const int var = 0;
    const auto ws_kern = hdr_ws_kernel<8>;
    if (ws_ok && ws_enabled()) {
        if (!ws_occ[var][device]) {
            int coop = 0, occ = 0;
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
                        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ws_kern, kWsT, 0);
            cudaGetLastError();
            ws_occ[var][device] = coop && occ > 0 ? occ : -1;
        }
        if (ws_occ[var][device] > 0) {
            uint8_t* fb = static_cast<uint8_t*>(scratch);
            int nring = ws_ring(pix_per_img);
            float* wring = reinterpret_cast<float*>(fb);
            fb += align256(static_cast<size_t>(nring) * pix_per_img * sizeof(float));
            float2* wparts = reinterpret_cast<float2*>(fb);
            fb += align256(static_cast<size_t>(nimg) * kWsMaxGrid * sizeof(float2));
            unsigned* wcounts = reinterpret_cast<unsigned*>(fb);
            cudaError_t e = cudaMemsetAsync(wcounts, 0, static_cast<size_t>(nimg) * sizeof(unsigned), st);
            if (e != cudaSuccess) return set_error(static_cast<int>(e), "hdr: memset: %s", cudaGetErrorString(e));
            const int64_t lines = pix_per_img / kWsLinePx;
            const unsigned grid = static_cast<unsigned>(
                std::max<int64_t>(1, std::min<int64_t>({static_cast<int64_t>(ws_occ[var][device]) * sms, kWsMaxGrid, lines})));
            int64_t n = nimg, ppi = pix_per_img;
            U8Consts kk = k;
            float mm = midpoint, ss = slope;
            Theta th = theta;
            int pf = kWsPrefetchWaves;
            if (const char* e = getenv("WG_HDR_PF")) pf = atoi(e);  // tuning knob (scripts/ab_tone.py)
            // TMEM staging when a CTA's per-image range fits one TMEM slot
            const int64_t max_quads = (lines + grid - 1) / grid * (kWsLinePx / 4);
            const char* tm_env = getenv("WG_HDR_TMEM");
            const bool tm = max_quads <= kTmMaxQuads && !(tm_env && std::strcmp(tm_env, "0") == 0);
            if (tm) {
                void* targs[] = {&rgb, &out, &wparts, &wcounts, &n, &ppi, &kk, &mm, &ss, &th, &pf};
                // 8 consumer warps (4: 293 vs 340 Gpix/s, the tone falls behind)
                const char* de = getenv("WG_HDR_TMDBG");  // timing experiments only (4: trace)
                // WG_HDR_TMRING=3 adds a third slot in shared memory: slower (C4 341.6 vs
                // 352.2 Gpix/s -- 128 KiB of shared memory shrink the L1 that holds the
                // producers' loads in flight)
                const char* re = getenv("WG_HDR_TMRING");
                const int tdbg = de ? atoi(de) : 0, ring = re ? atoi(re) : 2;
                using TmK = void (*)(const float*, uint8_t*, float2*, unsigned*, int64_t, int64_t, U8Consts, float,
                                     float, Theta, int);
                const char* pe = getenv("WG_HDR_PACKED");  // A/B: packed-pair gray in the producers
                TmK tk = ring == 3                 ? (tdbg == 4 ? hdr_tm_kernel<8, 4, 3> : hdr_tm_kernel<8, 0, 3>)
                         : (pe && atoi(pe) == 1) ? hdr_tm_kernel<8, 0, 2, true>
                                                 : (tdbg == 4 ? hdr_tm_kernel<8, 4, 2> : hdr_tm_kernel<8, 0, 2>);
                const size_t dsm = ring == 2 ? 0 : static_cast<size_t>(kTmMaxQuads) * sizeof(float4);
                if (dsm) {
                    e = cudaFuncSetAttribute(reinterpret_cast<const void*>(tk),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsm));
                    if (e != cudaSuccess) return set_error(static_cast<int>(e), "hdr: smem attribute: %s", cudaGetErrorString(e));
                }
                e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(tk), dim3(grid), dim3(kWsT), targs, dsm, st);
            } else {
                void* args[] = {&rgb, &out, &wring, &wparts, &wcounts, &n, &ppi, &nring, &kk, &mm, &ss, &th, &pf};
                e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(ws_kern), dim3(grid), dim3(kWsT),
                                                args, 0, st);
            }
            if (e != cudaSuccess) {
                cudaGetLastError();
                return set_error(static_cast<int>(e), "hdr: cooperative launch: %s", cudaGetErrorString(e));
            }
            return check_launch("hdr_ws_kernel");
        }
    }
    // ---- grouped schedule. Consecutive groups alternate between two scratch
    // sets so the HBM-bound gray pass of group n+1 (caller's stream) overlaps
    // the L2-bound stats + tone of group n (an internal stream); events order
    // the reuse of each set and join the internal stream back into `stream`.
    const int G = group_size(nimg, pix_per_img);
    const int64_t ngroups = (nimg + G - 1) / G;
    const int nsets = scratch_sets(nimg, pix_per_img);
    struct Set {
        float* gray;
        float2* parts;
        float2* luts;
        HdrStat* stats;
    } sets[2];
    uint8_t* base = static_cast<uint8_t*>(scratch);
    for (int q = 0; q < nsets; ++q) {
        sets[q].gray = reinterpret_cast<float*>(base);
        base += align256(static_cast<size_t>(G) * pix_per_img * sizeof(float));
        sets[q].parts = reinterpret_cast<float2*>(base);
        base += align256(static_cast<size_t>(G) * kSlots * sizeof(float2));
        sets[q].luts = reinterpret_cast<float2*>(base);
        base += align256(static_cast<size_t>(G) * kLutBins * sizeof(float2));
        sets[q].stats = reinterpret_cast<HdrStat*>(base);
        base += align256(static_cast<size_t>(G) * sizeof(HdrStat));
    }
    HdrStreams* hs = nullptr;
    std::unique_lock<std::mutex> lock;
    if (nsets == 2) {
        hs = hdr_streams(device);
        if (!hs) return set_error(WG_ENODEV, "hdr: could not create the auxiliary stream");
        lock = std::unique_lock<std::mutex>(hs->mu);
        cudaEventRecord(hs->start, st);
        cudaStreamWaitEvent(hs->aux, hs->start, 0);
    }
    for (int64_t gi = 0; gi < ngroups; ++gi) {
        const int64_t i0 = gi * G;
        const int g = static_cast<int>(std::min<int64_t>(G, nimg - i0));
        const Set& S = sets[gi % nsets];
        float* gray = S.gray;
        float2* parts = S.parts;
        float2* luts = S.luts;
        HdrStat* stats = S.stats;
        cudaStream_t sb = st;
        if (nsets == 2) {
            if (gi >= 2) cudaStreamWaitEvent(st, hs->tone_done[gi % 2], 0);  // set free again
            sb = hs->aux;
        }
        // gray: ~8 waves of blocks over the group, at most kSlots warps per image
        const int64_t work = (pix_per_img & 3) == 0 ? pix_per_img / 4 : pix_per_img;
        const int64_t bx = std::max<int64_t>(
            1, std::min<int64_t>({(work + kT - 1) / kT, std::max<int64_t>(1, 8LL * sms / g), kSlots / kWarps}));
        hdr_gray_kernel<<<dim3(static_cast<unsigned>(bx), static_cast<unsigned>(g)), kT, 0, st>>>(
            rgb + i0 * pix_per_img * 3, gray, parts, pix_per_img, k);
        if (nsets == 2) {
            cudaEventRecord(hs->gray_done[gi % 2], st);
            cudaStreamWaitEvent(sb, hs->gray_done[gi % 2], 0);
        }
        launch_pdl(hdr_stats_kernel, dim3(static_cast<unsigned>(g)), sb, sb == st, parts, static_cast<int>(bx) * kWarps,
                   stats, luts, theta);
        const int64_t twork = (pix_per_img & 15) == 0 ? pix_per_img / 16 : pix_per_img;
        const int64_t bt = std::max<int64_t>(1, std::min<int64_t>((twork + kT - 1) / kT, std::max<int64_t>(1, 8LL * sms / g)));
        // drop the gray lines from L2 only when the group's plane can actually be resident there
        const bool discard = static_cast<size_t>(g) * pix_per_img * sizeof(float) <= (size_t(96) << 20) &&
                             !getenv("WG_HDR_NO_DISCARD");
        if (pix_per_img % kToneTilePx == 0 && getenv("WG_HDR_TILED")) {
            static std::atomic<int> tone_occ[kMaxDevices];  // idempotent lazy cache
            if (device >= 0 && device < kMaxDevices && !tone_occ[device]) {
                cudaFuncSetAttribute(hdr_tone_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kToneSmem);
                int occ = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hdr_tone_tiled_kernel, kT, kToneSmem);
                tone_occ[device] = std::max(occ, 1);
            }
            const int occ = device >= 0 && device < kMaxDevices ? tone_occ[device].load() : 1;
            const int64_t ntiles = pix_per_img / kToneTilePx;
            const int64_t bt2 = std::max<int64_t>(1, std::min<int64_t>(ntiles, (static_cast<int64_t>(occ) * sms + g - 1) / g));
            hdr_tone_tiled_kernel<<<dim3(static_cast<unsigned>(bt2), static_cast<unsigned>(g)), kT, kToneSmem, sb>>>(
                gray, out + i0 * pix_per_img, pix_per_img, stats, luts, midpoint, slope, discard);
        } else {
            launch_pdl(hdr_tone_kernel, dim3(static_cast<unsigned>(bt), static_cast<unsigned>(g)), sb, true,
                       static_cast<const float*>(gray), out + i0 * pix_per_img, pix_per_img,
                       static_cast<const HdrStat*>(stats), static_cast<const float2*>(luts), midpoint, slope, discard);
        }
        if (nsets == 2) cudaEventRecord(hs->tone_done[gi % 2], sb);
        const int rc = check_launch("hdr_tonemap_u8");
        if (rc != WG_OK) {
            if (nsets == 2) cudaStreamWaitEvent(st, hs->tone_done[gi % 2], 0);
            return rc;
        }
    }
    if (nsets == 2) cudaStreamWaitEvent(st, hs->tone_done[(ngroups - 1) % 2], 0);  // join
    return check_launch("hdr_tonemap_u8");
}
