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
// The fp64 drop-in evaluates every step with the reference's operations and
// order (no contraction), so it is bit-identical to the NumPy code. The fused
// uint8 batch path (decolor -> local equalisation -> quantize) computes the
// gray, the bin and the blended value in fp32 and re-evaluates in fp64 -- the
// reference's own chain -- only the pixels whose fp32 value lies within a
// proven error margin of a bin edge or of a quantization boundary; its output
// is therefore bit-identical to quantize_u8 of the fp64 reference as well.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"

namespace wg {
namespace {

constexpr int kBlock = 256;
// |decolor_acc(k/255) - decolor_f64(k/255)| over all 2^24 byte colours is
// < 2.5e-7 (tests/test_gpu_lhe.py pins it); margins below leave >= 4x headroom.
constexpr float kGrayMargin = 1e-6f;  // bin edges (gray domain)
constexpr float kQuantMargin = 1e-3f;  // quantization (x = v * 255 + 0.5 domain)
constexpr size_t kHistSmemCap = 96 * 1024;

struct LheGeom {
    int64_t h, w, nimg;
    int tw, th, nx, ny, nb;
    int64_t ntile;
    double strength;
};

struct LheBufs {
    uint32_t* hist;  // [nimg][ntile][nb]
    double* curve;   // [nimg][ntile][nb]
    float* curvef;   // [nimg][ntile][nb]
    uint8_t* ident;  // [nimg][ntile]
    int32_t* xi;     // [w] left neighbour tile column
    double* xf;      // [w] blend fraction
    float* xff;
    int32_t* yi;  // [h]
    double* yf;
    float* yff;
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
        return decolor_f64(deq_byte(r), deq_byte(g), deq_byte(b), br, bk);
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
        s.curvef[cell0 + k] = static_cast<float>(v);
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
            const float c00 = s.ident[t00] ? vf : s.curvef[t00 * g.nb + b];
            const float c01 = s.ident[t01] ? vf : s.curvef[t01 * g.nb + b];
            const float c10 = s.ident[t10] ? vf : s.curvef[t10 * g.nb + b];
            const float c11 = s.ident[t11] ? vf : s.curvef[t11 * g.nb + b];
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

// ------------------------------------------------------------------ driver
template <class Src>
int run_lhe(const Src& src, const LheGeom& g, const LheBufs& b, cudaStream_t st) {
    int device = 0;
    cudaGetDevice(&device);
    const int sms = sm_count(device);
    cudaError_t e = cudaMemsetAsync(b.hist, 0, static_cast<size_t>(g.nimg) * g.ntile * g.nb * 4, st);
    if (e != cudaSuccess) return set_error(static_cast<int>(e), "lhe: hist memset: %s", cudaGetErrorString(e));
    // axis tables
    const int64_t na = g.w + g.h;
    lhe_axis_kernel<<<static_cast<unsigned>((na + kBlock - 1) / kBlock), kBlock, 0, st>>>(g, b);
    // histograms: enough (image, tile row, chunk) blocks to cover the SMs a few times
    const int64_t bands = g.nimg * g.ny;
    const int64_t want_chunks = std::max<int64_t>(1, (4LL * sms + bands - 1) / bands);
    const int rows_per_chunk = static_cast<int>(std::max<int64_t>(1, (g.th + want_chunks - 1) / want_chunks));
    const int chunks = (g.th + rows_per_chunk - 1) / rows_per_chunk;
    const size_t smem = static_cast<size_t>(g.nx) * g.nb * 4;
    for (int64_t i0 = 0; i0 < g.nimg; i0 += 65535) {
        LheGeom gi = g;
        gi.nimg = std::min<int64_t>(65535, g.nimg - i0);
        Src si = src;
        si.advance(i0 * g.h * g.w);
        uint32_t* hist = b.hist + i0 * g.ntile * g.nb;
        const dim3 grid(chunks, g.ny, static_cast<unsigned>(gi.nimg));
        if (smem <= kHistSmemCap) {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(lhe_hist_kernel<Src, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem));
            lhe_hist_kernel<Src, true><<<grid, kBlock, smem, st>>>(si, gi, hist, rows_per_chunk);
        } else {
            lhe_hist_kernel<Src, false><<<grid, kBlock, 0, st>>>(si, gi, hist, rows_per_chunk);
        }
    }
    for (int64_t i0 = 0; i0 < g.nimg; i0 += 65535) {
        LheGeom gi = g;
        gi.nimg = std::min<int64_t>(65535, g.nimg - i0);
        LheBufs bi = b;
        bi.hist += i0 * g.ntile * g.nb;
        bi.curve += i0 * g.ntile * g.nb;
        bi.curvef += i0 * g.ntile * g.nb;
        bi.ident += i0 * g.ntile;
        lhe_curve_kernel<<<dim3(static_cast<unsigned>(g.ntile), static_cast<unsigned>(gi.nimg)), kBlock, 0, st>>>(gi,
                                                                                                              bi);
    }
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
    rc = run_lhe(src, g, b, st);
    if (rc != WG_OK) return rc;
    lhe_apply_u8_kernel<<<apply_grid(g), kBlock, 0, st>>>(src, toned, gray_or_null, g, b);
    return check_launch("local lhe (apply u8)");
}
