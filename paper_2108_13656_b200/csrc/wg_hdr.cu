// wg_hdr.cu -- HDR adapter: fp32 linear radiance -> uint8.
//
// The reference cannot ingest HDR (PlanarImage rejects samples > 1,
// core.py:76-79), so the adapter is builder-defined and restated
// in the oracle (oracle/warmgray_oracle.c, or_hdr_u8):
//   g  = decolor(x)                          (raw radiance; homogeneous, so the
//                                            image scale cancels below)
//   t  = log(g / gmin) / log(gmax / gmin)    over g > 0 (per image);
//   t  = 0 for g == 0, t = 1 if gmax == gmin
//   out = quantize_u8(apply_sigmoid(t))
//
// Per group of images whose fp32 gray plane fits in L2 (kL2Budget):
//   1. hdr_gray_kernel   cp.async.bulk ring over 12 KiB rgb tiles (1024 px),
//                        packed-f32x2 MUFU formulation, gray stored with an
//                        L2 evict_last policy; every warp keeps a running
//                        (min over g > 0, max) per image and writes it to its
//                        own slot: no atomics, exact and order-independent,
//                        so results are identical for any grid / GPU count.
//   2. hdr_stats_kernel  folds the slots of each image into the per-image
//                        constants (fp64 log of the range).
//   3. hdr_tone_kernel   reads the gray back from L2 (16 px per thread),
//                        log-range normalisation + tanh-form sigmoid + round,
//                        writes uint8 and drops the gray lines from L2 with
//                        discard.global.L2 so they are never written to HBM.
// HBM traffic is therefore ~ the algorithmic 12 B in + 1 B out per pixel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"

namespace wg {
namespace {

constexpr int kT = 256;
constexpr int kWarps = kT / 32;
constexpr int kTilePx = 1024;                // fp32 rgb tile = 12 KiB
constexpr int kTileB = kTilePx * 12;
constexpr int kStagesH = 4;
constexpr int kSmemH = kStagesH * kTileB + kStagesH * 8;
constexpr int kSlots = 4096;                 // (min, max) slots per image
constexpr int kMaxGroup = 32;                // images per group (visited-image bitmask)
constexpr size_t kL2Budget = size_t(128) << 20;

struct HdrStat {
    float inv_gmin;
    float inv_lrange;
    int mode;  // 0: no positive pixel, 1: log range, 2: gmax == gmin (t = 1)
    int pad;
};

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

// ---------------------------------------------------------------- pass 1 (ppi % 1024 == 0)
__global__ void __launch_bounds__(kT) hdr_gray_kernel(const float* __restrict__ rgb, float* __restrict__ gray,
                                                      float2* __restrict__ parts, int64_t ntiles,
                                                      int64_t tiles_per_img, int nimg, U8Consts k) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStagesH * kTileB);
    const int tid = threadIdx.x, lane = tid & 31;
    const int gwarp = blockIdx.x * kWarps + (tid >> 5);
    const int64_t stride = gridDim.x;
    const uint8_t* in = reinterpret_cast<const uint8_t*>(rgb);
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < kStagesH; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    uint64_t pol_in = 0;
    if (tid == 0) {
        pol_in = l2_policy_evict_first();
        for (int s = 0; s < kStagesH; ++s) {
            const int64_t t = blockIdx.x + s * stride;
            if (t < ntiles) {
                mbar_arrive_expect_tx(&bars[s], kTileB);
                bulk_g2s(smem + s * kTileB, in + t * kTileB, kTileB, &bars[s], pol_in);
            }
        }
    }
    const uint64_t pol_gray = l2_policy_evict_last();
    int cur = -1;
    uint32_t seen = 0;
    float lo = INFINITY, hi = 0.0f;
    int s = 0;
    uint32_t phase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += stride) {
        const int img = static_cast<int>(t / tiles_per_img);  // CTA-uniform
        if (img != cur) {
            if (cur >= 0) {
                warp_minmax(lo, hi);
                if (lane == 0) parts[static_cast<int64_t>(cur) * kSlots + gwarp] = make_float2(lo, hi);
            }
            cur = img;
            seen |= 1u << img;
            lo = INFINITY;
            hi = 0.0f;
        }
        mbar_wait(&bars[s], phase);
        const uint4* src = reinterpret_cast<const uint4*>(smem + s * kTileB) + tid * 3;
        const uint4 v0 = src[0], v1 = src[1], v2 = src[2];
        __syncthreads();
        if (tid == 0) {
            const int64_t tn = t + kStagesH * stride;
            if (tn < ntiles) {
                mbar_arrive_expect_tx(&bars[s], kTileB);
                bulk_g2s(smem + s * kTileB, in + tn * kTileB, kTileB, &bars[s], pol_in);
            }
        }
        const float f[12] = {__uint_as_float(v0.x), __uint_as_float(v0.y), __uint_as_float(v0.z),
                             __uint_as_float(v0.w), __uint_as_float(v1.x), __uint_as_float(v1.y),
                             __uint_as_float(v1.z), __uint_as_float(v1.w), __uint_as_float(v2.x),
                             __uint_as_float(v2.y), __uint_as_float(v2.z), __uint_as_float(v2.w)};
        // pixels (0,1) and (2,3) as packed pairs
        const float2 a = decolor_fast_x2(make_float2(f[0], f[3]), make_float2(f[1], f[4]),
                                         make_float2(f[2], f[5]), k);
        const float2 b = decolor_fast_x2(make_float2(f[6], f[9]), make_float2(f[7], f[10]),
                                         make_float2(f[8], f[11]), k);
        track(a.x, lo, hi);
        track(a.y, lo, hi);
        track(b.x, lo, hi);
        track(b.y, lo, hi);
        st_v4_hint(gray + t * kTilePx + tid * 4, make_float4(a.x, a.y, b.x, b.y), pol_gray);
        if (++s == kStagesH) {
            s = 0;
            phase ^= 1u;
        }
    }
    if (cur >= 0) {
        warp_minmax(lo, hi);
        if (lane == 0) parts[static_cast<int64_t>(cur) * kSlots + gwarp] = make_float2(lo, hi);
    }
    if (lane == 0)
        for (int i = 0; i < nimg; ++i)
            if (!(seen >> i & 1u)) parts[static_cast<int64_t>(i) * kSlots + gwarp] = make_float2(INFINITY, 0.0f);
}

// ---------------------------------------------------------------- pass 1, any image size
__global__ void __launch_bounds__(kT) hdr_gray_generic_kernel(const float* __restrict__ rgb,
                                                              float* __restrict__ gray,
                                                              float2* __restrict__ parts, int64_t ppi,
                                                              U8Consts k) {
    const int img = blockIdx.y, lane = threadIdx.x & 31;
    const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const float* in = rgb + static_cast<int64_t>(img) * ppi * 3;
    float* g = gray + static_cast<int64_t>(img) * ppi;
    float lo = INFINITY, hi = 0.0f;
    for (int64_t p = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; p < ppi;
         p += static_cast<int64_t>(gridDim.x) * kT) {
        const float v = decolor_fast_x1(in[3 * p], in[3 * p + 1], in[3 * p + 2], k);
        g[p] = v;
        track(v, lo, hi);
    }
    warp_minmax(lo, hi);
    if (lane == 0) parts[static_cast<int64_t>(img) * kSlots + gwarp] = make_float2(lo, hi);
}

// ---------------------------------------------------------------- per-image constants
__global__ void __launch_bounds__(kT) hdr_stats_kernel(const float2* __restrict__ parts, int nslots,
                                                       HdrStat* __restrict__ stats) {
    const int img = blockIdx.x;
    float lo = INFINITY, hi = 0.0f;
    for (int i = threadIdx.x; i < nslots; i += kT) {
        const float2 pr = parts[static_cast<int64_t>(img) * kSlots + i];
        lo = fminf(lo, pr.x);
        hi = fmaxf(hi, pr.y);
    }
    warp_minmax(lo, hi);
    __shared__ float s_lo[kWarps], s_hi[kWarps];
    if ((threadIdx.x & 31) == 0) {
        s_lo[threadIdx.x >> 5] = lo;
        s_hi[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kWarps; ++w) {
            lo = fminf(lo, s_lo[w]);
            hi = fmaxf(hi, s_hi[w]);
        }
        HdrStat st{0.0f, 0.0f, 0, 0};
        if (hi > 0.0f && lo <= hi) {
            st.inv_gmin = static_cast<float>(1.0 / static_cast<double>(lo));
            if (hi > lo) {
                st.mode = 1;
                st.inv_lrange = static_cast<float>(1.0 / log2(static_cast<double>(hi) / static_cast<double>(lo)));
            } else {
                st.mode = 2;
            }
        }
        stats[img] = st;
    }
}

// ---------------------------------------------------------------- pass 2
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
    const float m = __uint_as_float((b & 0x7FFFFFu) | 0x3F800000u);
    float l;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(m));
    return __fadd_rn(static_cast<float>(e), l);
}

__device__ __forceinline__ uint32_t tone_px(float g, const HdrStat& st, const ToneU8& c) {
    float t;
    if (!(g > 0.0f)) t = 0.0f;
    else if (st.mode == 1) t = fminf(fmaxf(__fmul_rn(log2_split(__fmul_rn(g, st.inv_gmin)), st.inv_lrange), 0.0f), 1.0f);
    else t = 1.0f;
    const float v = fminf(fmaxf(__fmul_rn(__fadd_rn(tanhf(__fmul_rn(c.hk, __fsub_rn(t, c.m))), c.t0), c.inv_den), 0.0f), 1.0f);
    return __float_as_uint(__fadd_rz(__fmaf_rn(v, 255.0f, 0.5f), kMagic)) & 0xFFu;
}

__global__ void __launch_bounds__(kT) hdr_tone_kernel(const float* __restrict__ gray, uint8_t* __restrict__ out,
                                                      int64_t npx, int64_t ppi, const HdrStat* __restrict__ stats,
                                                      float m, float slope) {
    const ToneU8 c = make_tone_u8(m, slope);
    if ((ppi & 15) == 0) {
        const int64_t nchunks = npx >> 4;
        for (int64_t ch = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; ch < nchunks;
             ch += static_cast<int64_t>(gridDim.x) * kT) {
            const int64_t p0 = ch << 4;
            const HdrStat st = stats[p0 / ppi];
            const float4* src = reinterpret_cast<const float4*>(gray + p0);
            float g[16];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float4 v = __ldcs(src + j);
                g[4 * j] = v.x;
                g[4 * j + 1] = v.y;
                g[4 * j + 2] = v.z;
                g[4 * j + 3] = v.w;
            }
            uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int j = 0; j < 16; ++j) w[j >> 2] |= tone_px(g[j], st, c) << (8 * (j & 3));
            st_global_cs_v4(out + p0, make_uint4(w[0], w[1], w[2], w[3]));
            // this chunk and the next (lane + 1, same warp, already consumed: the
            // results above depend on the whole warp's load) form one 128 B line
            if ((ch & 1) == 0 && ch + 1 < nchunks) discard_l2_line(gray + p0);
        }
    } else {
        for (int64_t p = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; p < npx;
             p += static_cast<int64_t>(gridDim.x) * kT)
            out[p] = static_cast<uint8_t>(tone_px(gray[p], stats[p / ppi], c));
    }
}

size_t l2_budget() {
    static size_t b = [] {
        const char* e = getenv("WG_HDR_L2_BUDGET_MB");  // tuning knob (scripts/), default kL2Budget
        return e ? static_cast<size_t>(atoll(e)) << 20 : kL2Budget;
    }();
    return b;
}

int group_size(int64_t nimg, int64_t ppi) {
    const int64_t fit = static_cast<int64_t>(l2_budget() / (static_cast<size_t>(ppi) * sizeof(float)));
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({fit, nimg, kMaxGroup})));
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace
}  // namespace wg

using namespace wg;

extern "C" size_t wg_hdr_scratch_bytes(int64_t nimg, int64_t pix_per_img) {
    if (nimg <= 0 || pix_per_img <= 0) return 0;
    const int g = group_size(nimg, pix_per_img);
    return align256(static_cast<size_t>(g) * pix_per_img * sizeof(float)) +
           align256(static_cast<size_t>(g) * kSlots * sizeof(float2)) + align256(g * sizeof(HdrStat));
}

extern "C" int wg_hdr_tonemap_u8(const float* rgb, uint8_t* out, int64_t nimg, int64_t pix_per_img,
                                 float beta_r, float beta_k, float midpoint, float slope, void* scratch,
                                 size_t scratch_bytes, void* stream) {
    WG_CHECK_ARGS(check_npix(nimg) || check_npix(pix_per_img) || check_params(beta_r, beta_k) ||
                  check_curve(midpoint, slope));
    if (nimg == 0 || pix_per_img == 0) return WG_OK;
    if (!rgb || !out || !scratch) return set_error(WG_EINVAL, "hdr: null pointer");
    if ((reinterpret_cast<uintptr_t>(scratch) & 255) != 0)
        return set_error(WG_EALIGN, "hdr: scratch must be 256-byte aligned");
    if (scratch_bytes < wg_hdr_scratch_bytes(nimg, pix_per_img))
        return set_error(WG_ESCRATCH, "hdr: scratch buffer smaller than wg_hdr_scratch_bytes()");
    int device = 0;
    cudaGetDevice(&device);
    const int G = group_size(nimg, pix_per_img);
    float* gray = static_cast<float*>(scratch);
    float2* parts = reinterpret_cast<float2*>(static_cast<uint8_t*>(scratch) +
                                              align256(static_cast<size_t>(G) * pix_per_img * sizeof(float)));
    HdrStat* stats = reinterpret_cast<HdrStat*>(reinterpret_cast<uint8_t*>(parts) +
                                                align256(static_cast<size_t>(G) * kSlots * sizeof(float2)));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const U8Consts k = make_u8_consts(beta_r, beta_k);
    const bool tiled = (pix_per_img % kTilePx) == 0 && (reinterpret_cast<uintptr_t>(rgb) & 15) == 0;
    static int occ_cache[kMaxDevices] = {0};
    if (tiled && !occ_cache[device]) {
        cudaFuncSetAttribute(hdr_gray_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemH);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hdr_gray_kernel, kT, kSmemH);
        occ_cache[device] = std::max(occ, 1);
    }
    const int sms = sm_count(device);
    for (int64_t i0 = 0; i0 < nimg; i0 += G) {
        const int g = static_cast<int>(std::min<int64_t>(G, nimg - i0));
        const float* in = rgb + i0 * pix_per_img * 3;
        int nslots;
        if (tiled) {
            const int64_t tiles_per_img = pix_per_img / kTilePx, ntiles = g * tiles_per_img;
            const int64_t grid = std::max<int64_t>(
                1, std::min<int64_t>({ntiles, static_cast<int64_t>(occ_cache[device]) * sms, kSlots / kWarps}));
            hdr_gray_kernel<<<static_cast<unsigned>(grid), kT, kSmemH, st>>>(in, gray, parts, ntiles,
                                                                             tiles_per_img, g, k);
            nslots = static_cast<int>(grid) * kWarps;
        } else {
            const int64_t bx = std::max<int64_t>(1, std::min<int64_t>((pix_per_img + kT - 1) / kT,
                                                                      std::max<int64_t>(1, 4LL * sms / g)));
            const dim3 grid(static_cast<unsigned>(std::min<int64_t>(bx, kSlots / kWarps)), static_cast<unsigned>(g));
            hdr_gray_generic_kernel<<<grid, kT, 0, st>>>(in, gray, parts, pix_per_img, k);
            nslots = static_cast<int>(grid.x) * kWarps;
        }
        hdr_stats_kernel<<<g, kT, 0, st>>>(parts, nslots, stats);
        const int64_t npx = g * pix_per_img;
        const int64_t work = (pix_per_img & 15) == 0 ? npx / 16 : npx;
        const unsigned tb = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((work + kT - 1) / kT, 8LL * sms)));
        hdr_tone_kernel<<<tb, kT, 0, st>>>(gray, out + i0 * pix_per_img, npx, pix_per_img, stats, midpoint, slope);
        const int rc = check_launch("hdr_tonemap_u8");
        if (rc != WG_OK) return rc;
    }
    return WG_OK;
}
