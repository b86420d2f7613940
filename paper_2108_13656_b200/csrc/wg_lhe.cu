// wg_lhe.cu -- local tone map by tile-histogram equalisation:
// LocalHistogramGrid / apply_local_lhe / tonemap_image(mode="local")
// (/root/reference/pkg/src/warmgray/tonemap.py:36-69, 86-169, 195-216).
//
// Per image, ny x nx tiles of (clamped) tile_h x tile_w pixels:
//   1. hist    per-tile nb-bin counts of bin(v) = min(int(v * nb), nb - 1).
//              One CTA per (image, tile row, row chunk) accumulates the nx
//              tiles of its rows in shared memory (integer atomics, so the
//              counts are exact and order-independent) and flushes them to
//              the global histogram with one atomic per non-empty bin.
//   2. curves  one CTA per tile: block scan of the counts into the CDF,
//              low = CDF at the first occupied bin, and
//              curve[k] = clip((cdf[k] - low) / (total - low), 0, 1) with the
//              integer -> double conversion and IEEE division NumPy performs;
//              low == total marks an identity tile.
//   3. axes    per column / row the two neighbouring tile centres and the
//              blend fraction (_axis_weights, tonemap.py:90-100).
//   4. apply   per pixel the four neighbouring tile curves at the pixel's bin,
//              blended bilinearly and mixed with the identity by `strength`.
//
// The fused uint8 route (bins <= 65536) runs five kernels per batch:
// lhe_axis_kernel, lhe_hist16_kernel (RGB -> per-tile counts + a 16-bit plane
// word per pixel, 3 + 2 B/px), lhe_curve_kernel, lhe_table_kernel (one blend
// table per image x row band: the four tile curves each pixel of the band
// blends, pre-scaled) and lhe_apply16_kernel (plane -> toned byte, 2 + 1 B/px):
// 8 B/px of HBM traffic. Both per-pixel kernels work on 16-pixel groups inside
// one row (128-bit loads when rows are 16-byte aligned); the hist uses the
// packed MUFU gray estimate of the decolor kernel (decolor_fast_x2, |error| <=
// 2.4e-7 over all byte colours: scripts/margin_probe.cu) and merges runs of
// equal cells before its shared-memory adds; the apply stages its band's table
// with bulk copies (TMA) and does one 128-bit shared load per pixel.
//
// The fp64 drop-in evaluates every step with the reference's operations and
// order (no contraction), so it is bit-identical to the NumPy code. The fused
// uint8 batch path (decolor -> local equalisation -> quantize) computes the
// gray, the bin and the blended value in fp32 and re-evaluates in fp64 -- the
// reference's own chain -- only the pixels whose fp32 value lies within a
// proven error margin of a bin edge or of a quantization boundary; its output
// is therefore bit-identical to quantize_u8 of the fp64 reference as well.
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

constexpr int kBlock = 256;
// |decolor_acc(k/255) - decolor_f64(k/255)| over all 2^24 byte colours is
// < 2.5e-7 (tests/test_gpu_lhe.py pins it); margins below leave >= 4x headroom.
constexpr float kGrayMargin = 1e-6f;  // bin edges (gray domain)
// (bins of the uint8 route need margin_t = kGrayMargin * nb < 0.5, i.e. nb < 500000)
constexpr int kGrp = 16;                                // pixels per thread group (48 input bytes)
// quantization margin in the x = 255 v + 0.5 domain. Error budget of the uint8
// route's fp32 x: gray estimate <= 255 * 2.4e-7 = 6.1e-5 (+ 1.5e-5 when the
// plane stores it with ulp 2^-15, kPacked), fp32 curves (255 domain) <= 7.6e-6,
// fp32 blend fractions <= 2 * 255 * 6e-8, the six roundings of the blend
// <= 6e-5: < 1.8e-4, so 4e-4 leaves 2.2x headroom.
constexpr float kQuantMargin = 4e-4f;
constexpr size_t kHistSmemCap = 96 * 1024;
constexpr size_t kApplySmemCap = 200 * 1024;

struct LheGeom {
    int64_t h, w, nimg;
    int tw, th, nx, ny, nb;
    int64_t ntile;
    double strength;
};

struct LheBufs {
    uint32_t* hist;  // [nimg][ntile][nb]
    double* curve;   // [nimg][ntile][nb]
    float* curvef;   // [nimg][ntile][nb]: 255 * curve, NaN for identity tiles (uint8 route)
    uint8_t* ident;  // [nimg][ntile]
    int32_t* xi;     // [w] left neighbour tile column
    double* xf;      // [w] blend fraction
    float* xff;
    int32_t* yi;  // [h]
    double* yf;
    float* yff;
    uint16_t* plane;  // [nimg][h][w] uint8 route: the hist pass's 16-bit plane words (plane_u16), read by apply
    // uint8 route (bins <= 65536), built once per call for the apply blocks:
    float4* qtab;    // [nimg][nband][nx * nb] blend table of each row band (lhe_table_kernel)
    uint8_t* qident; // [nimg][nband] the band's table holds an identity tile (raw curves)
    float* colf;     // [wpad] per-column blend fraction, apply's interleaved order
    uint32_t* colo;  // [wpad] per-column byte offset of the left tile's table, same order
};

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// byte layout of the scratch buffer; base == nullptr only sizes it
size_t layout(const LheGeom& g, uint8_t* base, LheBufs* b) {
    const size_t cells = static_cast<size_t>(g.nimg) * g.ntile * g.nb;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* p = base ? base + off : nullptr;
        off += al(bytes);
        return p;
    };
    LheBufs t;
    t.hist = reinterpret_cast<uint32_t*>(take(cells * 4));
    t.curve = reinterpret_cast<double*>(take(cells * 8));
    t.curvef = reinterpret_cast<float*>(take(cells * 4));
    t.ident = take(static_cast<size_t>(g.nimg) * g.ntile);
    t.xi = reinterpret_cast<int32_t*>(take(g.w * 4));
    t.xf = reinterpret_cast<double*>(take(g.w * 8));
    t.xff = reinterpret_cast<float*>(take(g.w * 4));
    t.yi = reinterpret_cast<int32_t*>(take(g.h * 4));
    t.yf = reinterpret_cast<double*>(take(g.h * 8));
    t.yff = reinterpret_cast<float*>(take(g.h * 4));
    const bool u8 = g.nb <= 65536;
    t.plane = reinterpret_cast<uint16_t*>(take(u8 ? static_cast<size_t>(g.nimg) * g.h * g.w * 2 : 0));
    const size_t nband = g.ny > 1 ? g.ny - 1 : 1, wpad = (g.w + 15) / 16 * 16;
    t.qtab = reinterpret_cast<float4*>(take(u8 ? static_cast<size_t>(g.nimg) * nband * g.nx * g.nb * 16 : 0));
    t.qident = take(u8 ? static_cast<size_t>(g.nimg) * nband : 0);
    t.colf = reinterpret_cast<float*>(take(u8 ? wpad * 4 : 0));
    t.colo = reinterpret_cast<uint32_t*>(take(u8 ? wpad * 4 : 0));
    if (b) *b = t;
    return off;
}

int make_geom(int64_t nimg, int64_t h, int64_t w, int64_t tile_w, int64_t tile_h, int64_t bins, double strength,
              LheGeom* g) {
    if (nimg < 0 || h < 0 || w < 0)
        return set_error(WG_EINVAL, "image count and size must be >= 0");
    if (tile_w < 1 || tile_h < 1)
        return set_error(WG_EINVAL, "tile size must be >= 1, got %lldx%lld", static_cast<long long>(tile_w),
                         static_cast<long long>(tile_h));
    if (bins < 2 || bins > (1 << 24)) return set_error(WG_EINVAL, "bins must lie in [2, 2^24], got %lld",
                                                      static_cast<long long>(bins));
    if (!(strength >= 0.0 && strength <= 1.0))
        return set_error(WG_EINVAL, "strength must lie in [0, 1], got %.17g", strength);
    if (h > INT32_MAX || w > INT32_MAX) return set_error(WG_EINVAL, "image side exceeds 2^31 - 1");
    g->h = h;
    g->w = w;
    g->nimg = nimg;
    // tiles larger than the image are clamped to it (tonemap.py:128-129)
    g->tw = static_cast<int>(std::max<int64_t>(1, std::min(tile_w, w)));
    g->th = static_cast<int>(std::max<int64_t>(1, std::min(tile_h, h)));
    g->nx = static_cast<int>((w + g->tw - 1) / g->tw);
    g->ny = static_cast<int>((h + g->th - 1) / g->th);
    g->nb = static_cast<int>(bins);
    g->ntile = static_cast<int64_t>(g->nx) * g->ny;
    g->strength = strength;
    return WG_OK;
}

// ------------------------------------------------------------------ pixel sources
// Each source yields the bin of a pixel exactly as the reference computes it
// from its fp64 luminance, plus what the apply pass needs.

__device__ __forceinline__ int bin_d(double v, int nb) {
    // (data * nb).astype(intp), then min(., nb - 1) (tonemap.py:136)
    return min(static_cast<int>(__dmul_rn(v, static_cast<double>(nb))), nb - 1);
}

struct SrcF64 {
    const double* lum;
    void advance(int64_t px) { lum += px; }
    __device__ __forceinline__ int bin(int64_t p, int nb) const { return bin_d(lum[p], nb); }
};

// the reference's fp64 gray of a byte colour; out of line: it is the rare route
__device__ __noinline__ double exact_gray(uint32_t r, uint32_t g, uint32_t b, double br, double bk) {
    return decolor_f64(deq_byte(r), deq_byte(g), deq_byte(b), br, bk);
}

// uint8 RGB: gray = decolor_image(dequantize_u8(rgb)) (core.py:147-169).
struct SrcU8 {
    const uint8_t* rgb;
    AccConsts k;
    double br, bk;
    float fnb, inv_nb;  // bins and fl(1 / bins)

    void advance(int64_t px) { rgb += 3 * px; }
    __device__ __forceinline__ void load(int64_t p, uint32_t& r, uint32_t& g, uint32_t& b) const {
        r = __ldg(rgb + 3 * p);
        g = __ldg(rgb + 3 * p + 1);
        b = __ldg(rgb + 3 * p + 2);
    }
    __device__ __forceinline__ float gray_f(uint32_t r, uint32_t g, uint32_t b) const {
        const float s = 1.0f / 255.0f;
        return decolor_acc(__fmul_rn(static_cast<float>(r), s), __fmul_rn(static_cast<float>(g), s),
                           __fmul_rn(static_cast<float>(b), s), k);
    }
    __device__ __forceinline__ double gray_d(uint32_t r, uint32_t g, uint32_t b) const {
        return exact_gray(r, g, b, br, bk);
    }
    // exact bin from the fp32 gray; fp64 only within kGrayMargin of an edge
    __device__ __forceinline__ int bin_of(float vf, uint32_t r, uint32_t g, uint32_t b, int nb) const {
        const float inv = inv_nb;
        const int k = min(static_cast<int>(__fmul_rn(vf, fnb)), nb - 1);
        const bool lo_ok = k == 0 || __fsub_rn(vf, __fmul_rn(static_cast<float>(k), inv)) > kGrayMargin;
        const bool hi_ok = k == nb - 1 || __fsub_rn(__fmul_rn(static_cast<float>(k + 1), inv), vf) > kGrayMargin;
        if (lo_ok && hi_ok) return k;
        return bin_d(gray_d(r, g, b), nb);
    }
    __device__ __forceinline__ int bin(int64_t p, int nb) const {
        uint32_t r, g, b;
        load(p, r, g, b);
        return bin_of(gray_f(r, g, b), r, g, b, nb);
    }
};

// ------------------------------------------------------------------ 1. histograms
template <class Src, bool kSmem>
__global__ void __launch_bounds__(kBlock) lhe_hist_kernel(Src src, LheGeom g, uint32_t* __restrict__ hist,
                                                          int rows_per_chunk) {
    extern __shared__ uint32_t sh[];
    const int64_t img = blockIdx.z;
    const int ty = blockIdx.y;
    const int64_t y0 = static_cast<int64_t>(ty) * g.th + static_cast<int64_t>(blockIdx.x) * rows_per_chunk;
    const int64_t y1 = imin64(imin64(y0 + rows_per_chunk, static_cast<int64_t>(ty + 1) * g.th), g.h);
    if (y0 >= y1) return;  // uniform per block
    const int cells = g.nx * g.nb;
    uint32_t* gh = hist + (img * g.ntile + static_cast<int64_t>(ty) * g.nx) * g.nb;
    if constexpr (kSmem) {
        for (int i = threadIdx.x; i < cells; i += blockDim.x) sh[i] = 0;
        __syncthreads();
    }
    for (int64_t y = y0; y < y1; ++y) {
        const int64_t row = (img * g.h + y) * g.w;
        for (int64_t x = threadIdx.x; x < g.w; x += blockDim.x) {
            const int cell = (static_cast<int>(x) / g.tw) * g.nb + src.bin(row + x, g.nb);
            if constexpr (kSmem) atomicAdd(&sh[cell], 1u);
            else atomicAdd(&gh[cell], 1u);
        }
    }
    if constexpr (kSmem) {
        __syncthreads();
        for (int i = threadIdx.x; i < cells; i += blockDim.x)
            if (sh[i]) atomicAdd(&gh[i], sh[i]);
    }
}

// ------------------------------------------------------------------ 2. curves
__global__ void __launch_bounds__(kBlock) lhe_curve_kernel(LheGeom g, LheBufs s) {
    __shared__ unsigned long long warp_sum[kBlock / 32];
    __shared__ int first_sh;
    __shared__ unsigned long long low_sh, total_sh;
    const int64_t cell0 = (static_cast<int64_t>(blockIdx.y) * g.ntile + blockIdx.x) * g.nb;
    const uint32_t* h = s.hist + cell0;
    const int per = (g.nb + kBlock - 1) / kBlock;
    const int k0 = min(static_cast<int>(threadIdx.x) * per, g.nb), k1 = min(k0 + per, g.nb);
    if (threadIdx.x == 0) first_sh = g.nb;
    unsigned long long sum = 0;
    int first = g.nb;
    for (int k = k0; k < k1; ++k) {
        sum += h[k];
        if (h[k] && first == g.nb) first = k;
    }
    // block exclusive scan of the per-thread sums
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long inc = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) warp_sum[wid] = inc;
    __syncthreads();
    if (first < g.nb) atomicMin(&first_sh, first);
    unsigned long long base = 0, total = 0;
    for (int w = 0; w < kBlock / 32; ++w) {
        if (w < wid) base += warp_sum[w];
        total += warp_sum[w];
    }
    const unsigned long long excl = base + inc - sum;
    __syncthreads();
    const int f = first_sh;
    if (f >= k0 && f < k1) {  // owner of the first occupied bin: low = cdf[f]
        unsigned long long c = excl;
        for (int k = k0; k <= f; ++k) c += h[k];
        low_sh = c;
        total_sh = total;
    }
    __syncthreads();
    const unsigned long long low = low_sh;
    const bool ident = low == total_sh;
    if (threadIdx.x == 0) s.ident[static_cast<int64_t>(blockIdx.y) * g.ntile + blockIdx.x] = ident;
    const double den = static_cast<double>(static_cast<long long>(total_sh - low));
    unsigned long long c = excl;
    for (int k = k0; k < k1; ++k) {
        c += h[k];
        double v = 0.0;
        if (!ident) {
            // np.clip((cdf - low) / (total - low), 0, 1) with int64 numerator
            v = __ddiv_rn(static_cast<double>(static_cast<long long>(c) - static_cast<long long>(low)), den);
            v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        }
        s.curve[cell0 + k] = v;
        // fp32 table in the 0..255 domain of the uint8 route; NaN marks an identity tile
        s.curvef[cell0 + k] = ident ? __int_as_float(0x7fc00000) : static_cast<float>(__dmul_rn(v, 255.0));
    }
}

// ------------------------------------------------------------------ 3. axis tables
// _axis_weights (tonemap.py:90-100): centres c_k = (s0 + s1 - 1) / 2;
// idx = clip(#{c_k <= pos} - 1, 0, n - 2); frac = clip((pos - c_idx) / (c_idx+1 - c_idx), 0, 1)
__device__ __forceinline__ double centre(int k, int step, int64_t len) {
    const int64_t s0 = static_cast<int64_t>(k) * step, s1 = imin64(s0 + step, len);
    return __ddiv_rn(static_cast<double>(s0 + s1 - 1), 2.0);
}

__global__ void lhe_axis_kernel(LheGeom g, LheBufs s) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= g.w + g.h) return;
    const bool is_x = i < g.w;
    const int64_t pos = is_x ? i : i - g.w, len = is_x ? g.w : g.h;
    const int n = is_x ? g.nx : g.ny, step = is_x ? g.tw : g.th;
    int idx = 0;
    double f = 0.0;
    if (n > 1) {
        const double p = static_cast<double>(pos);
        int lo = 0, hi = n;  // count of centres <= p
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (centre(mid, step, len) <= p) lo = mid + 1;
            else hi = mid;
        }
        idx = min(max(lo - 1, 0), n - 2);
        const double c0 = centre(idx, step, len), c1 = centre(idx + 1, step, len);
        f = __ddiv_rn(__dsub_rn(p, c0), __dsub_rn(c1, c0));
        f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
    }
    if (is_x) {
        s.xi[pos] = idx;
        s.xf[pos] = f;
        s.xff[pos] = static_cast<float>(f);
    } else {
        s.yi[pos] = idx;
        s.yf[pos] = f;
        s.yff[pos] = static_cast<float>(f);
    }
}

// ------------------------------------------------------------------ 4. apply
struct Corner {
    int64_t c00, c01, c10, c11;  // tile indices (image-relative)
};

__device__ __forceinline__ double blend_d(double v, double c00, double c01, double c10, double c11, double wx,
                                          double wy, double strength) {
    // tonemap.py:156-163, operation for operation
    const double top = __dadd_rn(c00, __dmul_rn(wx, __dsub_rn(c01, c00)));
    const double bottom = __dadd_rn(c10, __dmul_rn(wx, __dsub_rn(c11, c10)));
    const double eq = __dadd_rn(top, __dmul_rn(wy, __dsub_rn(bottom, top)));
    return clamp01_d(__dadd_rn(v, __dmul_rn(strength, __dsub_rn(eq, v))));
}

__device__ __forceinline__ double curve_d(const LheBufs& s, const LheGeom& g, int64_t img, int64_t tile, int bin,
                                          double v) {
    const int64_t t = img * g.ntile + tile;
    return s.ident[t] ? v : s.curve[t * g.nb + bin];
}

__global__ void __launch_bounds__(kBlock) lhe_apply_f64_kernel(const double* __restrict__ lum,
                                                               double* __restrict__ out, LheGeom g, LheBufs s) {
    const int64_t rows = g.nimg * g.h;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int64_t img = r / g.h, y = r - img * g.h;
        const int j0 = s.yi[y], j1 = g.ny > 1 ? j0 + 1 : 0;
        const double wy = s.yf[y];
        for (int64_t x = threadIdx.x; x < g.w; x += blockDim.x) {
            const int64_t p = r * g.w + x;
            const double v = lum[p];
            const int b = bin_d(v, g.nb);
            const int i0 = s.xi[x], i1 = g.nx > 1 ? i0 + 1 : 0;
            const double c00 = curve_d(s, g, img, static_cast<int64_t>(j0) * g.nx + i0, b, v);
            const double c01 = curve_d(s, g, img, static_cast<int64_t>(j0) * g.nx + i1, b, v);
            const double c10 = curve_d(s, g, img, static_cast<int64_t>(j1) * g.nx + i0, b, v);
            const double c11 = curve_d(s, g, img, static_cast<int64_t>(j1) * g.nx + i1, b, v);
            out[p] = blend_d(v, c00, c01, c10, c11, s.xf[x], wy, g.strength);
        }
    }
}

// uint8 RGB -> toned uint8 (+ gray uint8): fp32 fast route, fp64 near boundaries
__global__ void __launch_bounds__(kBlock) lhe_apply_u8_kernel(SrcU8 src, uint8_t* __restrict__ toned,
                                                              uint8_t* __restrict__ gray, LheGeom g, LheBufs s) {
    const int64_t rows = g.nimg * g.h;
    const float sf = static_cast<float>(g.strength);
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int64_t img = r / g.h, y = r - img * g.h;
        const int j0 = s.yi[y], j1 = g.ny > 1 ? j0 + 1 : 0;
        const float wyf = s.yff[y];
        const int64_t tbase = img * g.ntile;
        for (int64_t x = threadIdx.x; x < g.w; x += blockDim.x) {
            const int64_t p = r * g.w + x;
            uint32_t cr, cg, cb;
            src.load(p, cr, cg, cb);
            const float vf = src.gray_f(cr, cg, cb);
            const int b = src.bin_of(vf, cr, cg, cb, g.nb);
            const int i0 = s.xi[x], i1 = g.nx > 1 ? i0 + 1 : 0;
            const int64_t t00 = tbase + static_cast<int64_t>(j0) * g.nx + i0, t01 = t00 - i0 + i1;
            const int64_t t10 = tbase + static_cast<int64_t>(j1) * g.nx + i0, t11 = t10 - i0 + i1;
            constexpr float k255 = 1.0f / 255.0f;  // curvef is in the 0..255 domain
            const float c00 = s.ident[t00] ? vf : __fmul_rn(s.curvef[t00 * g.nb + b], k255);
            const float c01 = s.ident[t01] ? vf : __fmul_rn(s.curvef[t01 * g.nb + b], k255);
            const float c10 = s.ident[t10] ? vf : __fmul_rn(s.curvef[t10 * g.nb + b], k255);
            const float c11 = s.ident[t11] ? vf : __fmul_rn(s.curvef[t11 * g.nb + b], k255);
            const float wxf = s.xff[x];
            const float top = __fmaf_rn(wxf, __fsub_rn(c01, c00), c00);
            const float bottom = __fmaf_rn(wxf, __fsub_rn(c11, c10), c10);
            const float eq = __fmaf_rn(wyf, __fsub_rn(bottom, top), top);
            const float res = fminf(fmaxf(__fmaf_rn(sf, __fsub_rn(eq, vf), vf), 0.0f), 1.0f);
            const float xq = __fmaf_rn(res, 255.0f, 0.5f);
            const float fl = floorf(xq);
            uint32_t q = static_cast<uint32_t>(fl);
            // res is clipped to [0, 1]: the ends 0.5 and 255.5 are not boundaries
            const bool sure = fabsf(__fsub_rn(__fsub_rn(xq, fl), 0.5f)) < 0.5f - kQuantMargin || xq >= 255.5f ||
                              xq <= 0.5f;
            double vd = -1.0;
            if (!sure) {
                vd = src.gray_d(cr, cg, cb);
                const double c00d = s.ident[t00] ? vd : s.curve[t00 * g.nb + b];
                const double c01d = s.ident[t01] ? vd : s.curve[t01 * g.nb + b];
                const double c10d = s.ident[t10] ? vd : s.curve[t10 * g.nb + b];
                const double c11d = s.ident[t11] ? vd : s.curve[t11 * g.nb + b];
                q = quantize_d(blend_d(vd, c00d, c01d, c10d, c11d, s.xf[x], s.yf[y], g.strength));
            }
            toned[p] = static_cast<uint8_t>(q);
            if (gray) {
                const float xg = __fmaf_rn(vf, 255.0f, 0.5f);
                const float fg = floorf(xg);
                uint32_t qg = static_cast<uint32_t>(fg);
                if (!(fabsf(__fsub_rn(__fsub_rn(xg, fg), 0.5f)) < 0.5f - kQuantMargin || xg >= 255.5f))
                    qg = quantize_d(vd >= 0.0 ? vd : src.gray_d(cr, cg, cb));
                gray[p] = static_cast<uint8_t>(qg);
            }
        }
    }
}

// ------------------------------------------------------------------ uint8 group kernels
// One thread handles kGrp consecutive pixels of one row.
struct U8Group {
    uint32_t w[12];  // 48 bytes, zero-padded past the row end
    int npx;

    __device__ __forceinline__ void load(const uint8_t* rgb, int64_t p0, int n, bool vec) {
        npx = n;
        if (vec && n == kGrp) {
            const uint4* q = reinterpret_cast<const uint4*>(rgb + 3 * p0);
            const uint4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
            w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
            w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
            w[8] = c.x; w[9] = c.y; w[10] = c.z; w[11] = c.w;
        } else {
#pragma unroll
            for (int i = 0; i < 12; ++i) w[i] = 0;
            const uint8_t* src = rgb + 3 * p0;
#pragma unroll
            for (int i = 0; i < 3 * kGrp; ++i)  // static indices keep w[] in registers
                if (i < 3 * n) w[i >> 2] |= static_cast<uint32_t>(__ldg(src + i)) << (8 * (i & 3));
        }
    }
    // 255 * gray estimates (decolor_fast_x2 on pixel pairs)
    __device__ __forceinline__ void gray255(const U8Consts& k, float (&g)[kGrp]) const {
#pragma unroll
        for (int j = 0; j < kGrp / 2; ++j) {
            float2 ch[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int b0 = 3 * (2 * j) + c, b1 = 3 * (2 * j + 1) + c;
                ch[c] = add2(make_float2(byte_biased(w[b0 >> 2], b0 & 3), byte_biased(w[b1 >> 2], b1 & 3)),
                             bc2(-kMagic));
            }
            const float2 f = decolor_fast_x2(ch[0], ch[1], ch[2], k);
            g[2 * j] = f.x;
            g[2 * j + 1] = f.y;
        }
    }
};

struct U8Lhe {
    SrcU8 src;
    U8Consts k8;
    U8Consts kt;  // k8 with inv_c4sq scaled by (255 / nb)^2: the same estimate times nb / 255, i.e. t = v nb
    float nb_over_255;  // fl(nb / 255)
    float half_m;       // 0.5 - m, m = 1e-6 nb the margin in t = v * nb
    float t_hi;         // nb - 0.5
    // 16-bit plane word u = floor(t * 2^F) (t = v nb unclamped, F = 16 - ceil(log2 nb)):
    // bin = u >> F, v = (u + 1/2) 2^-F / nb to within qhalf = 2^-F / (2 nb)
    float u_magic;  // 2^(7 + ceil(log2 nb)): fl_rd(t + u_magic) holds floor(t 2^F) in its low bits
    int ufrac;      // F
    uint32_t umax;  // nb 2^F - 1

    // bin from the 0..255-domain estimate g255: t = g255 * nb/255 with
    // |t - v nb| <= (2.4e-7 + 6e-8 + 6e-8) nb < m. t is clamped to [0.5, nb - 0.5]
    // (0 and nb are not bin edges), floor(t) taken as the low bits of
    // fl_rd(t + 2^23) (no F2I); `sure` is false within m of an inner edge.
    __device__ __forceinline__ int bin_fast_t(float tu, bool& sure) const {
        const float t = fminf(fmaxf(tu, 0.5f), t_hi);
        const float tf = __fadd_rd(t, 8388608.0f);
        sure = fabsf(__fsub_rn(__fsub_rn(t, __fsub_rn(tf, 8388608.0f)), 0.5f)) < half_m;
        return static_cast<int>(__float_as_uint(tf) & 0x7fffffu);
    }
};

// Per-warp queue of the rare pixels that need the reference's fp64 chain
// (entry = group index * 16 + pixel): each round every lane with flagged pixels
// appends one at its ballot rank, and once 32 are queued the warp drains them
// through `fix` with all lanes busy (instead of each flagged lane running the
// long fp64 chain while its warp waits). Capacity: < 32 carried + 32 appended.
constexpr int kWq = 64;
constexpr size_t kWqBytes = static_cast<size_t>(kBlock / 32) * kWq * 4;
template <class F>
__device__ __forceinline__ void wq_push(uint32_t* q, int& qn, uint32_t mask, uint32_t gi, F&& fix) {
    const uint32_t lane = threadIdx.x & 31u;
    for (;;) {
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, mask != 0u);
        if (!bal) return;
        if (mask) {
            q[qn + __popc(bal & ((1u << lane) - 1u))] = gi * kGrp + static_cast<uint32_t>(__ffs(mask) - 1);
            mask &= mask - 1u;
        }
        qn += __popc(bal);
        __syncwarp();  // appends (and the callers' provisional stores) before the drain
        if (qn >= 32) {
            const uint32_t e = q[lane];
            const uint32_t rest = static_cast<int>(lane) + 32 < qn ? q[lane + 32] : 0u;
            __syncwarp();
            if (static_cast<int>(lane) + 32 < qn) q[lane] = rest;
            qn -= 32;
            fix(e);
            __syncwarp();  // queue moves before the next appends
        }
    }
}
template <class F>
__device__ __forceinline__ void wq_flush(const uint32_t* q, int qn, F&& fix) {
    __syncwarp();
    if (static_cast<int>(threadIdx.x & 31u) < qn) fix(q[threadIdx.x & 31u]);
}

// the 16-bit plane word of t = v nb (unclamped, t >= 0): floor(t 2^F), capped
// at nb 2^F - 1 (v = 1 gives t = nb, bin nb - 1). For a pixel whose bin is sure,
// u >> F is that bin (the same fp32 t floored); the others are patched by the fix.
__device__ __forceinline__ uint32_t plane_u16(const U8Lhe& L, float tu) {
    return min(__float_as_uint(__fadd_rd(tu, L.u_magic)) & 0x7FFFFFu, L.umax);
}
// a plane word whose bin (u >> F) must be b: the nearest word of bin b
__device__ __forceinline__ uint32_t plane_u16_fix(uint32_t u, int b, int F) {
    const int cb = static_cast<int>(u >> F);
    return cb == b ? u : (b < cb ? ((static_cast<uint32_t>(b) << F) | ((1u << F) - 1u)) : (static_cast<uint32_t>(b) << F));
}

// shared-memory add at a shared-window address (unconditional: the caller
// points the adds it does not want at a per-lane scratch cell, which costs less
// than the branch ptxas builds around a predicated atomic)
__device__ __forceinline__ void red_shared_at(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Histogram pass of the 16-bit plane route. Per pixel: t = v nb from the gray
// estimate, the bin test on t clamped to [1/2, nb - 1/2] (0 and nb are not bin
// edges), the plane word from the unclamped t, and the run-merged count: the
// cell's shared-memory address is formed straight from the bits of
// fl_rd(t + 2^23) (one LEA; an unsure pixel is counted in its fp32 bin and
// queued: the fix moves the count if the fp64 bin differs), a run is flushed
// with one red.shared when the address changes (otherwise the add goes to a
// per-lane scratch cell). Group coordinates advance incrementally and a per-column-group table
// (tile column, "group inside one tile") replaces the divisions per group.
__global__ void __launch_bounds__(kBlock, 4) lhe_hist16_kernel(U8Lhe L, LheGeom g, uint32_t* __restrict__ hist,
                                                            uint16_t* __restrict__ plane, int rows_per_chunk,
                                                            bool vec) {
    // [nx * nb] + one dummy cell, the warp queues, the column-group table, 32 per-lane scratch cells
    extern __shared__ uint32_t sh[];
    const int64_t img = blockIdx.z;
    const int ty = blockIdx.y;
    const int64_t y0 = static_cast<int64_t>(ty) * g.th + static_cast<int64_t>(blockIdx.x) * rows_per_chunk;
    const int64_t y1 = imin64(imin64(y0 + rows_per_chunk, static_cast<int64_t>(ty + 1) * g.th), g.h);
    if (y0 >= y1) return;
    const int cells = g.nx * g.nb;
    const uint32_t gpr = static_cast<uint32_t>((g.w + kGrp - 1) / kGrp);
    uint32_t* wq = sh + cells + 1 + (threadIdx.x >> 5) * kWq;
    uint32_t* ctab = sh + cells + 1 + (kBlock / 32) * kWq;  // [gpr]: tile column | whole-group flag << 31
    const uint32_t lane_cell = smem_addr(ctab + gpr + (threadIdx.x & 31u));
    for (int i = threadIdx.x; i <= cells; i += blockDim.x) sh[i] = 0;
    for (uint32_t c = threadIdx.x; c < gpr; c += blockDim.x) {
        const int64_t x0 = static_cast<int64_t>(c) * kGrp;
        const int64_t tx = x0 / g.tw;
        ctab[c] = static_cast<uint32_t>(tx) | (x0 + kGrp <= (tx + 1) * g.tw ? 0x80000000u : 0u);
    }
    int qn = 0;
    __syncthreads();
    const uint32_t ngroups = static_cast<uint32_t>(y1 - y0) * gpr;  // < 2^31: rows of one tile row
    const int64_t row0 = (img * g.h + y0) * g.w;
    const uint32_t sh_base = smem_addr(sh);
    const uint32_t dummy = sh_base + 4u * static_cast<uint32_t>(cells);
    // address of cell (tx, bin) from bits(fl_rd(t + 2^23)) = 0x4B000000 + bin: LEA(bits, base, 2)
    const uint32_t nb4 = 4u * static_cast<uint32_t>(g.nb);
    const uint32_t lea_base = sh_base - (0x4B000000u << 2);
    // the reference's fp64 bin for a pixel next to a bin edge (rare); the pixel
    // was counted in its fp32 bin, which is moved if the two differ
    const auto fix = [&](uint32_t e) {
        const uint32_t gi = e / kGrp, gy = gi / gpr;
        const int x = static_cast<int>(gi - gy * gpr) * kGrp + static_cast<int>(e % kGrp);
        const int64_t pp = row0 + static_cast<int64_t>(gy) * g.w + x;
        uint32_t cr, cg, cb;
        L.src.load(pp, cr, cg, cb);
        const int b = bin_d(L.src.gray_d(cr, cg, cb), g.nb);
        bool sure;
        const int b32 = L.bin_fast_t(decolor_fast_x1(static_cast<float>(cr), static_cast<float>(cg),
                                                     static_cast<float>(cb), L.kt), sure);
        if (b32 != b) {
            const int c0 = (x / g.tw) * g.nb;
            atomicSub(&sh[c0 + b32], 1u);
            atomicAdd(&sh[c0 + b], 1u);
        }
        plane[pp] = static_cast<uint16_t>(plane_u16_fix(plane[pp], b, L.ufrac));  // after the warp's stores
    };
    const uint32_t dq = blockDim.x / gpr, dr = blockDim.x - dq * gpr;
    uint32_t ny_ = threadIdx.x / gpr, nx_ = threadIdx.x - ny_ * gpr;  // the next group
    const uint32_t lane = threadIdx.x & 31u;
    U8Group nxt;
    if (threadIdx.x < ngroups)
        nxt.load(L.src.rgb, row0 + static_cast<int64_t>(ny_) * g.w + nx_ * kGrp,
                 static_cast<int>(imin64(kGrp, g.w - static_cast<int64_t>(nx_) * kGrp)), vec);
    // warp-uniform trip count (the queue uses warp collectives)
    for (uint32_t gb = threadIdx.x - lane; gb < ngroups; gb += blockDim.x) {
        const uint32_t gi = gb + lane;
        uint32_t slow = 0;
        if (gi < ngroups) {
        const U8Group grp = nxt;
        const uint32_t gy = ny_, gx = nx_;
        nx_ += dr;
        ny_ += dq;
        if (nx_ >= gpr) {
            nx_ -= gpr;
            ++ny_;
        }
        if (gi + blockDim.x < ngroups)  // register prefetch of this thread's next group
            nxt.load(L.src.rgb, row0 + static_cast<int64_t>(ny_) * g.w + nx_ * kGrp,
                     static_cast<int>(imin64(kGrp, g.w - static_cast<int64_t>(nx_) * kGrp)), vec);
        const int x0 = static_cast<int>(gx) * kGrp;
        const int n = static_cast<int>(imin64(kGrp, g.w - x0));
        const int64_t p0 = row0 + static_cast<int64_t>(gy) * g.w + x0;
        const uint32_t ct = ctab[gx];
        uint32_t tx = ct & 0x7FFFFFFFu;
        if (n == kGrp) {
            float tv[kGrp];
            grp.gray255(L.kt, tv);  // t = v nb directly (the scale folded into the constants)
            uint32_t words[kGrp];
            uint32_t run_addr = dummy, run = 0;
            const auto px = [&](int p, uint32_t base) {
                const float tu = tv[p];
                const float t = fminf(fmaxf(tu, 0.5f), L.t_hi);
                const float tf = __fadd_rd(t, 8388608.0f);
                const bool sure = fabsf(__fsub_rn(__fsub_rn(t, __fsub_rn(tf, 8388608.0f)), 0.5f)) < L.half_m;
                words[p] = plane_u16(L, tu);  // unsure bins are patched by the fix
                slow |= static_cast<uint32_t>(!sure) << p;
                const uint32_t addr = base + (__float_as_uint(tf) << 2);  // unsure: moved by the fix
                const bool flush = addr != run_addr;
                red_shared_at(flush ? run_addr : lane_cell, run);
                run = flush ? 1u : run + 1u;
                run_addr = addr;
            };
            if (ct & 0x80000000u) {  // the whole group inside one tile column
                const uint32_t base = lea_base + tx * nb4;
#pragma unroll
                for (int p = 0; p < kGrp; ++p) px(p, base);
            } else {
                int next = static_cast<int>(tx + 1) * g.tw;
#pragma unroll
                for (int p = 0; p < kGrp; ++p) {
                    const bool stp = x0 + p >= next;
                    tx += stp;
                    next += stp ? g.tw : 0;
                    px(p, lea_base + tx * nb4);
                }
            }
            red_shared_at(run_addr, run);
            if (vec) {
#pragma unroll
                for (int q = 0; q < kGrp / 8; ++q)
                    reinterpret_cast<uint4*>(plane + p0)[q] =
                        make_uint4(__byte_perm(words[8 * q], words[8 * q + 1], 0x5410),
                                   __byte_perm(words[8 * q + 2], words[8 * q + 3], 0x5410),
                                   __byte_perm(words[8 * q + 4], words[8 * q + 5], 0x5410),
                                   __byte_perm(words[8 * q + 6], words[8 * q + 7], 0x5410));
            } else {
#pragma unroll
                for (int q = 0; q < kGrp; ++q) plane[p0 + q] = static_cast<uint16_t>(words[q]);
            }
        } else {  // row tail of a width that is not a multiple of 16
            int next = static_cast<int>(tx + 1) * g.tw;
#pragma unroll 1
            for (int p = 0; p < n; ++p) {
                if (x0 + p >= next) {
                    ++tx;
                    next += g.tw;
                }
                uint32_t cr, cg, cb;  // (a dynamic index into grp.w would spill it to local memory)
                L.src.load(p0 + p, cr, cg, cb);
                // (decolor_fast_x1 with kt: the same t as a lane of the group path, and as the fix)
                const float tu = decolor_fast_x1(static_cast<float>(cr), static_cast<float>(cg),
                                                 static_cast<float>(cb), L.kt);
                bool sure;
                const int b = L.bin_fast_t(tu, sure);
                plane[p0 + p] = static_cast<uint16_t>(plane_u16(L, tu));
                atomicAdd(&sh[tx * g.nb + b], 1u);  // unsure: moved by the fix
                if (!sure) slow |= 1u << p;
            }
        }
        }
        wq_push(wq, qn, slow, gi, fix);  // rare: pixels next to a bin edge
    }
    wq_flush(wq, qn, fix);
    __syncthreads();
    uint32_t* gh = hist + (img * g.ntile + static_cast<int64_t>(ty) * g.nx) * g.nb;
    for (int i = threadIdx.x; i < cells; i += blockDim.x)
        if (sh[i]) atomicAdd(&gh[i], sh[i]);
}

// row width padded to whole 16-pixel groups (the per-column tables)
__host__ __device__ inline int64_t wpad16(int64_t w) { return (w + kGrp - 1) / kGrp * kGrp; }

// ------------------------------------------------------------------ apply on the 16-bit plane
// The hist pass writes u = floor(v nb 2^F) per pixel (2 B/px, plane_u16); the
// apply pass reads it back instead of 4 B/px of fp32 estimates: 3 + 2 + 2 + 1 =
// 8 B/px of traffic. v is known to within uhalf = 2^-F / (2 nb) (255 domain:
// <= 255 / 2^16), which the quantization margins below absorb; the pixels inside
// them take the fp64 queue. Bands without identity tiles get a blend table
// pre-scaled by the strength s, offset by 256.5 + (1 - s) uhalf, with the
// column differences: (s c00 + off, s c01 - s c00, s c10 + off, s c11 - s c10),
// so per pixel T = fma(wx, d0, a0), B = fma(wx, d1, a1), E = fma(wy, B - T, T)
// and r' = fma((1 - s) uscale, u, E) = 256.5 + v + s (eq - v): the rounded byte and
// its distance to the rounding boundary are integer fields of r''s bits.
struct Apply16 {
    float uscale, uhalf;  // v255 = (u + 1/2) uscale
    float oms_us;         // fl((1 - s) uscale)
    float off;            // 256.5 + (1 - s) uhalf
    uint32_t mq, mq_ident, mg;  // margins of the toned / identity-tile / gray byte, units of 2^-15
};

// shared memory of the apply kernel: the band's blend table [nx][nb] (16 B
// entries), the per-column blend fractions and table offsets (interleaved, see
// lhe_table_kernel), the per-warp fp64 queues, one mbarrier
struct Apply16Smem {
    static __host__ __device__ size_t bytes(int nx, int nb, int64_t w) {
        return static_cast<size_t>(nx) * nb * 16 + static_cast<size_t>(wpad16(w)) * 8 + kWqBytes + 16;
    }
};

// per (image, row band) the table of the band's tile-row pair (j0, j1) = (band,
// band + 1), or (0, 0) for a single tile row: entry [i0][b] covers the tiles
// (j0, i0), (j0, i1), (j1, i0), (j1, i1), i1 = min(i0 + 1, nx - 1). One block
// per (tile column i0, band, image).
__global__ void __launch_bounds__(kBlock) lhe_table_kernel(LheGeom g, LheBufs s, Apply16 A) {
    const int col = blockIdx.x, band = blockIdx.y, nband = g.ny > 1 ? g.ny - 1 : 1;
    const int64_t img = blockIdx.z;
    const int jrow = g.ny > 1 ? 1 : 0;
    const float* cf = s.curvef + (img * g.ntile + static_cast<int64_t>(g.ny > 1 ? band : 0) * g.nx) * g.nb;
    const int rowoff = jrow * g.nx * g.nb;
    bool any_ident = false;
    for (int i = threadIdx.x; i < (1 + jrow) * g.nx; i += blockDim.x) any_ident |= cf[i * g.nb] != cf[i * g.nb];
    const bool ident = __syncthreads_or(any_ident);
    float4* qt = s.qtab + (img * nband + band) * static_cast<int64_t>(g.nx) * g.nb;
    const float sf = static_cast<float>(g.strength);
    const int i0 = col, i1 = g.nx > 1 ? min(i0 + 1, g.nx - 1) : i0;
    for (int b = threadIdx.x; b < g.nb; b += blockDim.x) {
        const int i = i0 * g.nb + b;
        const float c00 = cf[i0 * g.nb + b], c01 = cf[i1 * g.nb + b];
        const float c10 = cf[rowoff + i0 * g.nb + b], c11 = cf[rowoff + i1 * g.nb + b];
        if (ident) {
            qt[i] = make_float4(c00, c01, c10, c11);
        } else {
            const float a0 = __fmul_rn(sf, c00), a1 = __fmul_rn(sf, c01);
            const float b0 = __fmul_rn(sf, c10), b1 = __fmul_rn(sf, c11);
            qt[i] = make_float4(__fadd_rn(a0, A.off), __fsub_rn(a1, a0), __fadd_rn(b0, A.off), __fsub_rn(b1, b0));
        }
    }
    if (threadIdx.x == 0 && col == 0) s.qident[img * nband + band] = ident;
    // the per-column tables (image-independent): column x = 16 gc + 4 q + r is
    // stored at ((q * G + gc) * 4 + r), G = wpad / 16, so the lanes of a warp
    // (consecutive groups gc) read consecutive 16-byte vectors
    if (band == 0 && img == 0) {  // split over the nx blocks of (band 0, image 0)
        const int64_t wp = wpad16(g.w), G = wp / kGrp;
        for (int64_t x = threadIdx.x + static_cast<int64_t>(col) * blockDim.x; x < wp;
             x += static_cast<int64_t>(blockDim.x) * g.nx) {
            const int64_t xc = imin64(x, g.w - 1);
            const int64_t gc = x / kGrp, q = (x % kGrp) >> 2, r = x & 3;
            const int64_t at = (q * G + gc) * 4 + r;
            s.colf[at] = s.xff[xc];
            s.colo[at] = static_cast<uint32_t>(s.xi[xc]) * static_cast<uint32_t>(g.nb) * 16u;
        }
    }
}

__device__ __forceinline__ uint64_t l2_policy_evict_last_lhe() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// byte of r' (in [256, 512): mantissa bits 22..15 = floor(r + 1/2)) and the
// flag "within m of a rounding boundary", from e = bits(r') + m
__device__ __forceinline__ uint32_t q_byte(uint32_t e) { return (e >> 15) & 255u; }
__device__ __forceinline__ bool q_unsure(uint32_t e, uint32_t m) { return (e & 0x7FFFu) < 2u * m; }

// kF: the plane's fraction bits when fixed at compile time (8: bins 129..256), else -1
template <bool kGray, bool kIdent, int kF>
__device__ __forceinline__ void apply16_groups(const U8Lhe& L, const Apply16& A, uint8_t* __restrict__ toned,
                                               uint8_t* __restrict__ gray, const LheGeom& g, const LheBufs& s,
                                               int64_t y0, int64_t y1, int64_t img, const uint8_t* quadb,
                                               const float* sxf, const uint32_t* sxo, int64_t G, bool vec,
                                               uint32_t* wq) {
    const float sf = static_cast<float>(g.strength);
    const uint32_t gpr = static_cast<uint32_t>((g.w + kGrp - 1) / kGrp);
    const uint32_t ngroups = static_cast<uint32_t>(y1 - y0) * gpr;  // < 2^31: rows of one tile row
    const uint16_t* plane = s.plane;
    const int F = kF >= 0 ? kF : L.ufrac;
    const int64_t rowbase = (img * g.h + y0) * g.w;
    // group gi = (row gy, column group gx); the thread's groups advance by
    // blockDim.x: gx += dr, gy += dq (+1 on wrap) instead of a division per group
    const uint32_t dq = blockDim.x / gpr, dr = blockDim.x - dq * gpr;
    const auto step = [&](uint32_t& gy, uint32_t& gx) {
        gx += dr;
        gy += dq;
        if (gx >= gpr) {
            gx -= gpr;
            ++gy;
        }
    };
    auto load_w = [&](uint32_t gy, uint32_t gx, uint4 (&e)[2]) {
        const int x0 = static_cast<int>(gx) * kGrp;
        const uint16_t* src = plane + rowbase + static_cast<int64_t>(gy) * g.w + x0;
        if (vec) {  // (w % 16 == 0: every group is whole)
            e[0] = __ldcs(reinterpret_cast<const uint4*>(src));
            e[1] = __ldcs(reinterpret_cast<const uint4*>(src) + 1);
        } else {
            const int n = static_cast<int>(imin64(kGrp, g.w - x0));
            uint32_t t[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                t[q] = (2 * q < n ? static_cast<uint32_t>(src[2 * q]) : 0u) |
                       (2 * q + 1 < n ? static_cast<uint32_t>(src[2 * q + 1]) << 16 : 0u);
            e[0] = make_uint4(t[0], t[1], t[2], t[3]);
            e[1] = make_uint4(t[4], t[5], t[6], t[7]);
        }
    };
    // the reference's fp64 chain for a pixel within a margin (queued, rare):
    // overwrites the provisional bytes the warp stored
    const auto fix = [&](uint32_t e) {
        const uint32_t gi = e / kGrp, gy = gi / gpr;
        const int p = static_cast<int>(e % kGrp);
        const int64_t y = y0 + gy;
        const int x = static_cast<int>(gi - gy * gpr) * kGrp + p;
        const int64_t pp = (img * g.h + y) * g.w + x;
        const int j0 = s.yi[y], j1 = g.ny > 1 ? j0 + 1 : 0;
        uint32_t cr, cg, cb;
        L.src.load(pp, cr, cg, cb);
        const double vd = L.src.gray_d(cr, cg, cb);
        const int b = bin_d(vd, g.nb);
        const int i0 = s.xi[x], i1 = g.nx > 1 ? i0 + 1 : 0;
        const int64_t t00 = img * g.ntile + static_cast<int64_t>(j0) * g.nx + i0, t01 = t00 - i0 + i1;
        const int64_t t10 = img * g.ntile + static_cast<int64_t>(j1) * g.nx + i0, t11 = t10 - i0 + i1;
        const double c00 = s.ident[t00] ? vd : s.curve[t00 * g.nb + b];
        const double c01 = s.ident[t01] ? vd : s.curve[t01 * g.nb + b];
        const double c10 = s.ident[t10] ? vd : s.curve[t10 * g.nb + b];
        const double c11 = s.ident[t11] ? vd : s.curve[t11 * g.nb + b];
        toned[pp] = static_cast<uint8_t>(quantize_d(blend_d(vd, c00, c01, c10, c11, s.xf[x], s.yf[y], g.strength)));
        if constexpr (kGray) gray[pp] = static_cast<uint8_t>(quantize_d(vd));
    };
    const uint32_t lane = threadIdx.x & 31u;
    int qn = 0;
    uint4 nxt[2];
    float wyn = 0.0f;  // the next group's row weight
    uint32_t ny_ = threadIdx.x / gpr, nx_ = threadIdx.x - ny_ * gpr;  // the next group
    if (threadIdx.x < ngroups) {
        load_w(ny_, nx_, nxt);
        wyn = s.yff[y0 + ny_];
    }
    // warp-uniform trip count (the queue uses warp collectives)
    for (uint32_t gb = threadIdx.x - lane; gb < ngroups; gb += blockDim.x) {
        const uint32_t gi = gb + lane;
        uint32_t slow = 0;
        if (gi < ngroups) {
        const uint32_t gy = ny_, gx = nx_;
        const uint32_t wd[8] = {nxt[0].x, nxt[0].y, nxt[0].z, nxt[0].w, nxt[1].x, nxt[1].y, nxt[1].z, nxt[1].w};
        const float wy = wyn;  // every row of the block blends the same tile-row pair
        step(ny_, nx_);
        if (gi + blockDim.x < ngroups) {
            load_w(ny_, nx_, nxt);
            wyn = s.yff[y0 + ny_];
        }
        const int x0 = static_cast<int>(gx) * kGrp;
        const int64_t p0 = rowbase + static_cast<int64_t>(gy) * g.w + x0;
        uint32_t ot[4] = {0u, 0u, 0u, 0u}, og[4] = {0u, 0u, 0u, 0u};
        float4 f;
        uint4 o;
#pragma unroll
        for (int p = 0; p < kGrp; ++p) {
            if ((p & 3) == 0) {  // the quad's blend fractions and table offsets, loaded where used
                f = reinterpret_cast<const float4*>(sxf)[(p >> 2) * G + gx];
                o = reinterpret_cast<const uint4*>(sxo)[(p >> 2) * G + gx];
            }
            const uint32_t xo = (p & 3) == 0 ? o.x : (p & 3) == 1 ? o.y : (p & 3) == 2 ? o.z : o.w;
            const float wx = (p & 3) == 0 ? f.x : (p & 3) == 1 ? f.y : (p & 3) == 2 ? f.z : f.w;
            const uint32_t w = wd[p >> 1];
            // 2^23 + u as a float (u exactly after one FADD) and the table entry's address
            uint32_t fb, boff;
            if constexpr (kF == 8) {
                fb = (p & 1) ? (w >> 16) | 0x4B000000u : (w & 0xFFFFu) | 0x4B000000u;
                boff = xo + ((p & 1) ? ((w >> 20) & 0xFF0u) : ((w & 0xFF00u) >> 4));
            } else {
                const uint32_t u = (p & 1) ? w >> 16 : w & 0xFFFFu;
                fb = u | 0x4B000000u;
                boff = xo + ((u >> F) << 4);
            }
            const float uf = __fsub_rn(__uint_as_float(fb), 8388608.0f);
            const float4 cq = *reinterpret_cast<const float4*>(quadb + boff);
            uint32_t e;
            bool uns;
            if constexpr (kIdent) {  // raw curves, NaN = identity tile (the pixel's own value)
                const float v = __fmaf_rn(uf, A.uscale, A.uhalf);
                const float c00 = cq.x != cq.x ? v : cq.x, c01 = cq.y != cq.y ? v : cq.y;
                const float c10 = cq.z != cq.z ? v : cq.z, c11 = cq.w != cq.w ? v : cq.w;
                const float top = __fmaf_rn(wx, __fsub_rn(c01, c00), c00);
                const float bottom = __fmaf_rn(wx, __fsub_rn(c11, c10), c10);
                const float eq = __fmaf_rn(wy, __fsub_rn(bottom, top), top);
                e = __float_as_uint(__fadd_rn(__fmaf_rn(sf, __fsub_rn(eq, v), v), 256.5f)) + A.mq_ident;
                uns = q_unsure(e, A.mq_ident);
            } else {
                const float T = __fmaf_rn(wx, cq.y, cq.x), B = __fmaf_rn(wx, cq.w, cq.z);
                const float E = __fmaf_rn(wy, __fsub_rn(B, T), T);
                e = __float_as_uint(__fmaf_rn(A.oms_us, uf, E)) + A.mq;
                uns = q_unsure(e, A.mq);
            }
            ot[p >> 2] |= q_byte(e) << (8 * (p & 3));
            if constexpr (kGray) {
                const uint32_t eg = __float_as_uint(__fadd_rn(__fmaf_rn(uf, A.uscale, A.uhalf), 256.5f)) + A.mg;
                uns = uns || q_unsure(eg, A.mg);
                og[p >> 2] |= q_byte(eg) << (8 * (p & 3));
            }
            slow |= static_cast<uint32_t>(uns) << p;
        }
        if (vec) {
            st_global_cs_v4(toned + p0, make_uint4(ot[0], ot[1], ot[2], ot[3]));
            if constexpr (kGray) st_global_cs_v4(gray + p0, make_uint4(og[0], og[1], og[2], og[3]));
        } else {
            const int n = static_cast<int>(imin64(kGrp, g.w - x0));
            slow &= (1u << n) - 1u;
#pragma unroll
            for (int p = 0; p < kGrp; ++p) {
                if (p < n) {
                    toned[p0 + p] = static_cast<uint8_t>(ot[p >> 2] >> (8 * (p & 3)));
                    if constexpr (kGray) gray[p0 + p] = static_cast<uint8_t>(og[p >> 2] >> (8 * (p & 3)));
                }
            }
        }
        }
        wq_push(wq, qn, slow, gi, fix);
    }
    wq_flush(wq, qn, fix);
}

template <bool kGray, int kF>
__global__ void __launch_bounds__(kBlock, 3) lhe_apply16_kernel(U8Lhe L, Apply16 A, uint8_t* __restrict__ toned,
                                                             uint8_t* __restrict__ gray, LheGeom g, LheBufs s,
                                                             int rows_per_chunk, bool vec) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int64_t img = blockIdx.z;
    // row bands between tile-row centres, as lhe_apply_u8g_kernel
    const int band = blockIdx.y, nband = g.ny > 1 ? g.ny - 1 : 1;
    const int64_t lo = band == 0 ? 0 : static_cast<int64_t>(ceil(centre(band, g.th, g.h)));
    const int64_t hi = band == nband - 1 ? g.h : static_cast<int64_t>(ceil(centre(band + 1, g.th, g.h)));
    const int64_t y0 = lo + static_cast<int64_t>(blockIdx.x) * rows_per_chunk;
    const int64_t y1 = imin64(y0 + rows_per_chunk, hi);
    if (y0 >= y1) return;
    const int64_t wp = wpad16(g.w);
    const int nq = g.nx * g.nb;
    uint4* quad = reinterpret_cast<uint4*>(smem);                              // [nx][nb] (lhe_table_kernel)
    float* sxf = reinterpret_cast<float*>(quad + nq);                          // [wp]
    uint32_t* sxo = reinterpret_cast<uint32_t*>(sxf + wp);                     // [wp] byte offsets
    uint32_t* wq = sxo + wp + (threadIdx.x >> 5) * kWq;                        // per-warp queues
    uint64_t* bar = reinterpret_cast<uint64_t*>(sxo + wp + (kBlock / 32) * kWq);
    // the band's blend table and the column tables: three bulk copies (TMA), no
    // register round trip (the register-staged copy was ~11% of the kernel's stalls)
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
        const uint32_t tb = static_cast<uint32_t>(nq) * 16u, cb = static_cast<uint32_t>(wp) * 4u;
        const uint64_t pol = l2_policy_evict_last_lhe();
        mbar_arrive_expect_tx(bar, tb + 2u * cb);
        bulk_g2s(quad, s.qtab + (img * nband + band) * static_cast<int64_t>(nq), tb, bar, pol);
        bulk_g2s(sxf, s.colf, cb, bar, pol);
        bulk_g2s(sxo, s.colo, cb, bar, pol);
    }
    const bool ident = s.qident[img * nband + band] != 0;
    __syncthreads();  // the barrier's initialisation before anyone waits on it
    mbar_wait(bar, 0);
    const uint8_t* quadb = reinterpret_cast<const uint8_t*>(quad);
    const int64_t G = wp / kGrp;
    if (ident)
        apply16_groups<kGray, true, kF>(L, A, toned, gray, g, s, y0, y1, img, quadb, sxf, sxo, G, vec, wq);
    else
        apply16_groups<kGray, false, kF>(L, A, toned, gray, g, s, y0, y1, img, quadb, sxf, sxo, G, vec, wq);
}

// ------------------------------------------------------------------ driver

Apply16 make_apply16(int nb, int F, double strength) {
    Apply16 a;
    const double us = 255.0 / (static_cast<double>(nb) * static_cast<double>(1u << F)), uh = 0.5 * us;
    a.uscale = static_cast<float>(us);
    a.uhalf = static_cast<float>(uh);
    a.oms_us = static_cast<float>((1.0 - strength) * us);
    a.off = static_cast<float>(256.5 + (1.0 - strength) * uh);
    // |v_recon - v| <= uh + 1.5e-4 (estimate <= 255 * 3.6e-7 = 9.2e-5 with the t scale
    // folded into its constants, reconstruction 1.5e-5); the blend's own fp32
    // roundings, curve and weight errors < 4e-4 (255 domain)
    const double ev = uh + 1.5e-4;
    a.mq = static_cast<uint32_t>(std::ceil((4e-4 + (1.0 - strength) * ev) * 32768.0)) + 1;
    a.mq_ident = static_cast<uint32_t>(std::ceil((4.2e-4 + ev) * 32768.0)) + 1;
    a.mg = static_cast<uint32_t>(std::ceil((ev + 3e-5) * 32768.0)) + 1;
    return a;
}

struct Chunking {
    int rows_per_chunk, chunks;
};
// enough (image, tile row, row chunk) blocks to cover the SMs a few times
Chunking chunking(const LheGeom& g) {
    int device = 0;
    cudaGetDevice(&device);
    const int64_t bands = std::max<int64_t>(1, std::min<int64_t>(g.nimg, 65535) * g.ny);
    // ~16 blocks per SM: several waves, so the last one is a small tail
    const int64_t want = std::max<int64_t>(1, (16LL * sm_count(device) + bands - 1) / bands);
    Chunking c;
    c.rows_per_chunk = static_cast<int>(std::max<int64_t>(1, (g.th + want - 1) / want));
    c.chunks = (g.th + c.rows_per_chunk - 1) / c.rows_per_chunk;
    return c;
}

// hist memset + axis tables
int lhe_begin(const LheGeom& g, const LheBufs& b, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(b.hist, 0, static_cast<size_t>(g.nimg) * g.ntile * g.nb * 4, st);
    if (e != cudaSuccess) return set_error(static_cast<int>(e), "lhe: hist memset: %s", cudaGetErrorString(e));
    const int64_t na = g.w + g.h;
    lhe_axis_kernel<<<static_cast<unsigned>((na + kBlock - 1) / kBlock), kBlock, 0, st>>>(g, b);
    return WG_OK;
}

// images are processed in slices of at most 65535 (grid z)
template <class F>
void per_image_slice(const LheGeom& g, F f) {
    for (int64_t i0 = 0; i0 < g.nimg; i0 += 65535) {
        LheGeom gi = g;
        gi.nimg = std::min<int64_t>(65535, g.nimg - i0);
        f(i0, gi);
    }
}

template <class Src>
void lhe_hist(const Src& src, const LheGeom& g, const LheBufs& b, cudaStream_t st) {
    const Chunking c = chunking(g);
    const size_t smem = static_cast<size_t>(g.nx) * g.nb * 4;
    per_image_slice(g, [&](int64_t i0, const LheGeom& gi) {
        Src si = src;
        si.advance(i0 * g.h * g.w);
        uint32_t* hist = b.hist + i0 * g.ntile * g.nb;
        const dim3 grid(c.chunks, g.ny, static_cast<unsigned>(gi.nimg));
        if (smem <= kHistSmemCap) {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(lhe_hist_kernel<Src, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem));
            lhe_hist_kernel<Src, true><<<grid, kBlock, smem, st>>>(si, gi, hist, c.rows_per_chunk);
        } else {
            lhe_hist_kernel<Src, false><<<grid, kBlock, 0, st>>>(si, gi, hist, c.rows_per_chunk);
        }
    });
}

void lhe_curves(const LheGeom& g, const LheBufs& b, cudaStream_t st) {
    per_image_slice(g, [&](int64_t i0, const LheGeom& gi) {
        LheBufs bi = b;
        bi.hist += i0 * g.ntile * g.nb;
        bi.curve += i0 * g.ntile * g.nb;
        bi.curvef += i0 * g.ntile * g.nb;
        bi.ident += i0 * g.ntile;
        lhe_curve_kernel<<<dim3(static_cast<unsigned>(g.ntile), static_cast<unsigned>(gi.nimg)), kBlock, 0, st>>>(
            gi, bi);
    });
}

template <class Src>
int run_lhe(const Src& src, const LheGeom& g, const LheBufs& b, cudaStream_t st) {
    int rc = lhe_begin(g, b, st);
    if (rc != WG_OK) return rc;
    lhe_hist(src, g, b, st);
    lhe_curves(g, b, st);
    return check_launch("local lhe (hist/curves)");
}

unsigned apply_grid(const LheGeom& g) {
    int device = 0;
    cudaGetDevice(&device);
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(g.nimg * g.h, 8LL * sm_count(device))));
}

}  // namespace
}  // namespace wg

using namespace wg;

extern "C" size_t wg_lhe_scratch_bytes(int64_t nimg, int64_t height, int64_t width, int64_t tile_w, int64_t tile_h,
                                       int64_t bins) {
    LheGeom g;
    if (make_geom(nimg, height, width, tile_w, tile_h, bins, 0.0, &g) != WG_OK) return 0;
    return std::max<size_t>(256, layout(g, nullptr, nullptr));
}

static int lhe_prepare(int64_t nimg, int64_t h, int64_t w, int64_t tile_w, int64_t tile_h, int64_t bins,
                       double strength, void* scratch, size_t scratch_bytes, LheGeom* g, LheBufs* b) {
    const int rc = make_geom(nimg, h, w, tile_w, tile_h, bins, strength, g);
    if (rc != WG_OK) return rc;
    const size_t need = layout(*g, nullptr, nullptr);
    if (nimg * h * w > 0 && (scratch == nullptr || scratch_bytes < need))
        return set_error(WG_ESCRATCH, "local lhe scratch too small: need %zu bytes, got %zu", need, scratch_bytes);
    layout(*g, static_cast<uint8_t*>(scratch), b);
    return WG_OK;
}

extern "C" int wg_local_lhe_f64(const double* lum, double* out, int64_t nimg, int64_t height, int64_t width,
                                int64_t tile_w, int64_t tile_h, int64_t bins, double strength, void* scratch,
                                size_t scratch_bytes, void* stream) {
    LheGeom g;
    LheBufs b;
    int rc = lhe_prepare(nimg, height, width, tile_w, tile_h, bins, strength, scratch, scratch_bytes, &g, &b);
    if (rc != WG_OK) return rc;
    const int64_t npix = nimg * height * width;
    WG_CHECK_ARGS(check_ptrs(npix, lum, out));
    if (npix == 0) return WG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    rc = run_lhe(SrcF64{lum}, g, b, st);
    if (rc != WG_OK) return rc;
    lhe_apply_f64_kernel<<<apply_grid(g), kBlock, 0, st>>>(lum, out, g, b);
    return check_launch("local lhe (apply f64)");
}

extern "C" int wg_tonemap_local_f64(const double* rgb, double* gray, double* l_out, double* rgb_out, int64_t nimg,
                                    int64_t height, int64_t width, double beta_r, double beta_k, int64_t tile_w,
                                    int64_t tile_h, int64_t bins, double strength, void* scratch,
                                    size_t scratch_bytes, void* stream) {
    WG_CHECK_ARGS(check_params(beta_r, beta_k));
    LheGeom g;
    LheBufs b;
    int rc = lhe_prepare(nimg, height, width, tile_w, tile_h, bins, strength, scratch, scratch_bytes, &g, &b);
    if (rc != WG_OK) return rc;
    const int64_t npix = nimg * height * width;
    WG_CHECK_ARGS(check_ptrs(npix, rgb, gray) || check_ptrs(npix, l_out, rgb_out));
    if (npix == 0) return WG_OK;
    // tonemap.py:209-216: l_in = decolor_image; l_out = apply_local_lhe(l_in); reinstate_color
    rc = wg_decolor_f64(rgb, gray, npix, beta_r, beta_k, stream);
    if (rc != WG_OK) return rc;
    rc = wg_local_lhe_f64(gray, l_out, nimg, height, width, tile_w, tile_h, bins, strength, scratch, scratch_bytes,
                          stream);
    if (rc != WG_OK) return rc;
    return wg_reinstate_f64(rgb, gray, l_out, rgb_out, npix, stream);
}

extern "C" int wg_decolor_tone_local_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray_or_null, int64_t nimg,
                                        int64_t height, int64_t width, double beta_r, double beta_k, int64_t tile_w,
                                        int64_t tile_h, int64_t bins, double strength, void* scratch,
                                        size_t scratch_bytes, void* stream) {
    WG_CHECK_ARGS(check_params(beta_r, beta_k));
    LheGeom g;
    LheBufs b;
    int rc = lhe_prepare(nimg, height, width, tile_w, tile_h, bins, strength, scratch, scratch_bytes, &g, &b);
    if (rc != WG_OK) return rc;
    const int64_t npix = nimg * height * width;
    WG_CHECK_ARGS(check_ptrs(npix, rgb, toned));
    if (npix == 0) return WG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the exact route needs the caller's fp64 betas (0.55f != 0.55); the fast route rounds them
    const SrcU8 src{rgb,
                    make_acc_consts(static_cast<float>(beta_r), static_cast<float>(beta_k)),
                    beta_r,
                    beta_k,
                    static_cast<float>(bins),
                    1.0f / static_cast<float>(bins)};
    const float m = static_cast<float>(kGrayMargin * static_cast<double>(bins));
    int kb = 1;
    while ((int64_t(1) << kb) < bins) ++kb;  // 2^kb >= bins
    const int F = kb <= 16 ? 16 - kb : 0;
    U8Consts kt = make_u8_consts(static_cast<float>(beta_r), static_cast<float>(beta_k));
    kt.inv_c4sq = static_cast<float>(3.0 / static_cast<double>(static_cast<float>(beta_k)) * (255.0 / bins) *
                                     (255.0 / bins));
    const U8Lhe L{src,
                  make_u8_consts(static_cast<float>(beta_r), static_cast<float>(beta_k)),
                  kt,
                  static_cast<float>(bins) / 255.0f,
                  0.5f - m,
                  static_cast<float>(bins) - 0.5f,
                  std::ldexp(1.0f, 7 + kb),
                  F,
                  static_cast<uint32_t>(bins) * (1u << F) - 1u};
    // 16-pixel groups load/store 16-byte vectors when every row starts aligned
    const bool vec = width % 16 == 0 && (reinterpret_cast<uintptr_t>(rgb) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(toned) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(gray_or_null) & 15) == 0;
    rc = lhe_begin(g, b, st);
    if (rc != WG_OK) return rc;
    const Chunking c = chunking(g);
    // + the dummy cell, warp queues, column-group table
    const size_t hsmem = static_cast<size_t>(g.nx) * g.nb * 4 + 4 + kWqBytes + wpad16(g.w) / kGrp * 4 + 128;
    const size_t asmem = Apply16Smem::bytes(g.nx, g.nb, g.w);
    // the group kernels' t-domain bin test needs nb <= 65536 (t + 2^23 exact, and
    // the 16-bit plane word); the group apply reads the plane the group hist
    // writes, so both or neither (the per-warp queue entries are group * 16 +
    // pixel within one row chunk: < 2^32)
    const bool group_ok = bins <= 65536 && hsmem <= kHistSmemCap && asmem <= kApplySmemCap &&
                          g.ny <= 65535 && g.nx <= 65535 &&  // grid dimensions of the hist / table / apply grids
                          static_cast<int64_t>(c.rows_per_chunk) * wpad16(g.w) < (int64_t(1) << 32);
    if (group_ok) {
        if (hsmem > 48 * 1024)
            cudaFuncSetAttribute(lhe_hist16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(hsmem));
        per_image_slice(g, [&](int64_t i0, const LheGeom& gi) {
            U8Lhe Li = L;
            Li.src.advance(i0 * g.h * g.w);
            lhe_hist16_kernel<<<dim3(c.chunks, g.ny, static_cast<unsigned>(gi.nimg)), kBlock, hsmem, st>>>(
                Li, gi, b.hist + i0 * g.ntile * g.nb, b.plane + i0 * g.h * g.w, c.rows_per_chunk, vec);
        });
    } else {
        lhe_hist(src, g, b, st);
    }
    lhe_curves(g, b, st);
    if (group_ok) {
        auto kern = F == 8 ? (gray_or_null ? lhe_apply16_kernel<true, 8> : lhe_apply16_kernel<false, 8>)
                           : (gray_or_null ? lhe_apply16_kernel<true, -1> : lhe_apply16_kernel<false, -1>);
        const Apply16 A16 = make_apply16(static_cast<int>(bins), F, strength);
        const int nband = g.ny > 1 ? g.ny - 1 : 1;
        if (asmem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(asmem));
        per_image_slice(g, [&](int64_t i0, const LheGeom& gi) {
            U8Lhe Li = L;
            Li.src.advance(i0 * g.h * g.w);
            LheBufs bi = b;  // the kernels index tiles per image slice
            bi.curve += i0 * g.ntile * g.nb;
            bi.curvef += i0 * g.ntile * g.nb;
            bi.ident += i0 * g.ntile;
            const int64_t off = i0 * g.h * g.w;
            bi.plane += off;
            bi.qtab += i0 * nband * static_cast<int64_t>(g.nx) * g.nb;
            bi.qident += i0 * nband;
            lhe_table_kernel<<<dim3(g.nx, nband, static_cast<unsigned>(gi.nimg)), kBlock, 0, st>>>(gi, bi, A16);
            // row bands between tile-row centres are at most ~1.5 tile heights (+2 rows)
            const int achunks = static_cast<int>((2LL * g.th + 2 + c.rows_per_chunk - 1) / c.rows_per_chunk);
            kern<<<dim3(achunks, nband, static_cast<unsigned>(gi.nimg)), kBlock, asmem, st>>>(
                Li, A16, toned + off, gray_or_null ? gray_or_null + off : nullptr, gi, bi, c.rows_per_chunk, vec);
        });
    } else {
        lhe_apply_u8_kernel<<<apply_grid(g), kBlock, 0, st>>>(src, toned, gray_or_null, g, b);
    }
    return check_launch("local lhe (u8)");
}
