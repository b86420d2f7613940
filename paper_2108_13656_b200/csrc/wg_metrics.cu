// wg_metrics.cu -- contrast-preservation pair counts on the GPU:
// the hot loop of CCPR / CCFR / E-score (metrics.py:84-135, _pair_delta_chunks
// and _sweep_counts).
//
// For each evaluated pixel pair (i, j) the reference computes
//   delta_e   = sqrt(((d0*d0 + d1*d1) + d2*d2)),  d = lab[i] - lab[j]
//   gray_diff = |100 g[i] - 100 g[j]|
// and, per threshold tau, counts pairs with delta_e >= tau (color set),
// both >= tau (kept), gray_diff >= tau (gray set), and gray but not colour
// (fabricated). With the taus sorted, a pair is summarised by
//   kc = #{tau : delta_e >= tau},  kg = #{tau : gray_diff >= tau},
// so the four counts per tau follow from the 2D histogram H[kc][kg]:
//   color(k) = #(kc > k), kept(k) = #(min(kc, kg) > k), gray(k) = #(kg > k),
//   fabricated(k) = gray(k) - kept(k).
// delta_e >= tau is decided without a square root: fl(sqrt(s)) is monotone,
// so it equals s >= S_tau with S_tau the least double whose correctly rounded
// square root reaches tau (host bisection). Counts are integers, exact and
// order-independent.
//
// Pair sets: all n(n-1)/2 unordered pairs (triangular grid of 256 x 256 pixel
// tiles, the j tile staged in shared memory), or an explicit (i, j) list -- the
// reference's seeded sample, drawn on the host with its own NumPy generator.
// With the integer thresholds 1..ntau of TAU_SWEEP the exhaustive kernel
// counts in fp32 with a proven margin and an fp64 recheck (metric_all_pairs_int_kernel).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"

namespace wg {
namespace {

constexpr int kMaxTau = 15;  // taus per call (TAU_SWEEP has 15); thresholds padded to 16
constexpr int kBins = (kMaxTau + 1) * (kMaxTau + 1);
constexpr int kTile = 256;

struct Thresholds {
    double s[16];  // S_tau in the squared-distance domain, padded with +inf
    double g[16];  // tau itself for the gray difference, padded with +inf
    int ntau;
};

// count of sorted thresholds t[0..15) <= x (t[15] = +inf): branch-free binary search
__device__ __forceinline__ int count_le(const double* t, double x) {
    int k = 0;
    k += (x >= t[k + 7]) ? 8 : 0;
    k += (x >= t[k + 3]) ? 4 : 0;
    k += (x >= t[k + 1]) ? 2 : 0;
    k += (x >= t[k]) ? 1 : 0;
    return k;
}

// lab (L*, a*, b*) of the pixel and 100 * gray, as in metrics.py:89-90
// (lab_rows order of operations, _kernels.pyx:115-132)
constexpr double MX0 = 0.4124564, MX1 = 0.3575761, MX2 = 0.1804375;
constexpr double MY0 = 0.2126729, MY1 = 0.7151522, MY2 = 0.0721750;
constexpr double MZ0 = 0.0193339, MZ1 = 0.1191920, MZ2 = 0.9503041;
constexpr double WHITE_X = 0.95047, WHITE_Z = 1.08883;
constexpr double LAB_EPS = 216.0 / 24389.0, LAB_KAPPA = 24389.0 / 27.0;

__device__ __forceinline__ double lin_d(double c) {
    if (c <= 0.04045) return __ddiv_rn(c, 12.92);
    return pow(__ddiv_rn(__dadd_rn(c, 0.055), 1.055), 2.4);
}
__device__ __forceinline__ double labf_d(double t) {
    if (t > LAB_EPS) return cbrt(t);
    return __ddiv_rn(__dadd_rn(__dmul_rn(LAB_KAPPA, t), 16.0), 116.0);
}
__device__ __forceinline__ double dot3d(double a0, double a1, double a2, double x, double y, double z) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a0, x), __dmul_rn(a1, y)), __dmul_rn(a2, z));
}

__global__ void metric_prep_kernel(const double* __restrict__ rgb, const double* __restrict__ gray,
                                   double4* __restrict__ labg, float4* __restrict__ lab32, int64_t n) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double lr = lin_d(rgb[3 * p]), lg = lin_d(rgb[3 * p + 1]), lb = lin_d(rgb[3 * p + 2]);
        const double fx = labf_d(__ddiv_rn(dot3d(MX0, MX1, MX2, lr, lg, lb), WHITE_X));
        const double fy = labf_d(dot3d(MY0, MY1, MY2, lr, lg, lb));
        const double fz = labf_d(__ddiv_rn(dot3d(MZ0, MZ1, MZ2, lr, lg, lb), WHITE_Z));
        const double4 v = make_double4(__dsub_rn(__dmul_rn(116.0, fy), 16.0), __dmul_rn(500.0, __dsub_rn(fx, fy)),
                                       __dmul_rn(200.0, __dsub_rn(fy, fz)), __dmul_rn(gray[p], 100.0));
        labg[p] = v;
        lab32[p] = make_float4(__double2float_rn(v.x), __double2float_rn(v.y), __double2float_rn(v.z),
                               __double2float_rn(v.w));
    }
}

// (kc, kg) bin of one pair, reference operation order
__device__ __forceinline__ int pair_bin(const double4& a, const double4& b, const double* ts, const double* tg,
                                        int stride) {
    const double d0 = __dsub_rn(a.x, b.x), d1 = __dsub_rn(a.y, b.y), d2 = __dsub_rn(a.z, b.z);
    const double s = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
    const double gd = fabs(__dsub_rn(a.w, b.w));
    return count_le(ts, s) * stride + count_le(tg, gd);
}

struct WarpHist {
    uint32_t* h;  // this warp's bins in shared memory
    uint32_t full = 0;  // the saturated bin (kc = kg = ntau), counted in a register
    int full_bin;
    __device__ __forceinline__ void add(int bin) {
        const bool f = bin == full_bin;
        full += f;
        if (!f) atomicAdd(&h[bin], 1u);
    }
};

__device__ __forceinline__ void flush_hist(uint32_t* sh, const WarpHist& wh, int nbins, unsigned long long* hist) {
    atomicAdd(&wh.h[wh.full_bin], wh.full);
    __syncthreads();
    const int warps = blockDim.x / 32;
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
        unsigned long long c = 0;
        for (int w = 0; w < warps; ++w) c += sh[w * kBins + b];
        if (c) atomicAdd(&hist[b], c);
    }
}

__global__ void __launch_bounds__(kTile) metric_all_pairs_kernel(const double4* __restrict__ labg, int64_t n,
                                                                 Thresholds th, unsigned long long* hist) {
    const int64_t ti = blockIdx.y, tj = blockIdx.x;
    if (tj < ti) return;  // triangle: tile pairs (ti <= tj)
    __shared__ double4 tile[kTile];
    __shared__ uint32_t sh[(kTile / 32) * kBins];
    __shared__ double ts[16], tg[16];
    const int stride = th.ntau + 1, nbins = stride * stride;
    for (int b = threadIdx.x; b < (kTile / 32) * kBins; b += blockDim.x) sh[b] = 0;
    if (threadIdx.x < 16) {
        ts[threadIdx.x] = th.s[threadIdx.x];
        tg[threadIdx.x] = th.g[threadIdx.x];
    }
    const int64_t j0 = tj * kTile;
    const int64_t jn = imin64(kTile, n - j0);
    if (threadIdx.x < jn) tile[threadIdx.x] = labg[j0 + threadIdx.x];
    __syncthreads();
    WarpHist wh;
    wh.h = sh + (threadIdx.x / 32) * kBins;
    wh.full_bin = th.ntau * stride + th.ntau;
    const int64_t i = ti * kTile + threadIdx.x;
    if (i < n) {
        const double4 a = labg[i];
        // diagonal tile: only j > i
        const int jstart = ti == tj ? static_cast<int>(threadIdx.x) + 1 : 0;
        for (int jj = jstart; jj < jn; ++jj) wh.add(pair_bin(a, tile[jj], ts, tg, stride));
    }
    flush_hist(sh, wh, nbins, hist);
}

// Integer thresholds tau = 1..ntau (TAU_SWEEP): kc = #{k <= ntau : delta_e >= k} =
// min(floor(delta_e), ntau) and kg likewise from gray_diff, evaluated in fp32
// (one MUFU sqrt) from fp32 copies of lab / 100 g. Rigorous margins against
// the reference's fp64 values: each lab component (|.| <= 128) rounds by
// <= 128 u, so |d32 - D| <= 256 u + u|D| and |sqrt(s32) - |D|| <= 2 sqrt(3)
// 1.53e-5 + 5u|D| + 3e-10 / |D|, plus 2.5 u r for sqrt.approx: <= 6.1e-5 for
// r <= 16 (the reference's own fl(sqrt) is within 1e-15); gray_diff (|.| <=
// 100) <= 200 u + u gd <= 1.3e-5. A pair whose fp32 value lies within 8e-5
// (colour) / 2e-5 (gray) of a threshold takes the reference's fp64 route
// (pair_bin); every other count is decided exactly.
constexpr float kMarginDe = 8e-5f, kMarginGd = 2e-5f;
// count of the integer thresholds 1..ntau a value reaches, for two values in
// packed f32x2: each clamped to [1/2, ntau + 1/2] (neither end is a
// threshold, both floor into [0, ntau]); near when within `margin` of an integer
__device__ __forceinline__ void int_count2(float2 v, float margin, float vmax, uint32_t& k0, uint32_t& k1,
                                           bool& near0, bool& near1) {
    const float2 c = make_float2(fminf(fmaxf(v.x, 0.5f), vmax), fminf(fmaxf(v.y, 0.5f), vmax));
    const float2 f = add2_rz(c, bc2(8388608.0f));  // 2^23 + floor(c)
    const float2 e = add2(fma2(add2(f, bc2(-8388608.0f)), bc2(-1.0f), c), bc2(-0.5f));  // frac - 1/2
    near0 = near0 || fabsf(e.x) > 0.5f - margin;
    near1 = near1 || fabsf(e.y) > 0.5f - margin;
    k0 = __float_as_uint(f.x) & 0x7FFFFFu;
    k1 = __float_as_uint(f.y) & 0x7FFFFFu;
}

// shared-memory histogram increment without the compiler's warp-aggregation
// scaffolding: a predicated red.shared
__device__ __forceinline__ void red_shared_inc(uint32_t* p, bool pred) {
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q red.shared.add.u32 [%0], 1;\n}" ::"r"(
                     smem_addr(p)),
                 "r"(static_cast<uint32_t>(pred))
                 : "memory");
}

__global__ void __launch_bounds__(kTile) metric_all_pairs_int_kernel(const float4* __restrict__ lab32,
                                                                     const double4* __restrict__ labg, int64_t n,
                                                                     Thresholds th, float vmax,
                                                                     unsigned long long* hist) {
    const int64_t ti = blockIdx.y, tj = blockIdx.x;
    if (tj < ti) return;  // triangle: tile pairs (ti <= tj)
    // the j tile as structure of arrays: one 64-bit shared load per component
    // fetches two j (a warp-wide broadcast, no bank conflicts)
    __shared__ __align__(16) float soa[4][kTile];
    __shared__ uint32_t sh[(kTile / 32) * kBins];
    __shared__ double ts[16], tg[16];
    const int ntau = th.ntau, stride = ntau + 1, nbins = stride * stride;
    for (int b = threadIdx.x; b < (kTile / 32) * kBins; b += blockDim.x) sh[b] = 0;
    if (threadIdx.x < 16) {
        ts[threadIdx.x] = th.s[threadIdx.x];
        tg[threadIdx.x] = th.g[threadIdx.x];
    }
    const int64_t j0 = tj * kTile;
    const int jn = static_cast<int>(imin64(kTile, n - j0));
    if (static_cast<int>(threadIdx.x) < jn) {
        const float4 v = lab32[j0 + threadIdx.x];
        soa[0][threadIdx.x] = v.x;
        soa[1][threadIdx.x] = v.y;
        soa[2][threadIdx.x] = v.z;
        soa[3][threadIdx.x] = v.w;
    }
    __syncthreads();
    uint32_t* wh = sh + (threadIdx.x / 32) * kBins;
    const int full_bin = ntau * stride + ntau;
    uint32_t full = 0;  // the saturated bin, counted in a register
    const int64_t i = ti * kTile + threadIdx.x;
    const bool active = i < n;
    const float4 a = active ? lab32[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const auto add = [&](int bin, bool valid) {
        const bool f = bin == full_bin;
        full += (f && valid) ? 1u : 0u;
        red_shared_inc(wh + bin, valid && !f);
    };
    const auto exact = [&](int jj) { return pair_bin(labg[i], labg[j0 + jj], ts, tg, stride); };
    // pairs (k, k + 1) over a block-uniform range; each element masked by this
    // lane's lower bound (diagonal tile: j > i only) and the tile end
    const int lo = ti == tj ? static_cast<int>(threadIdx.x) + 1 : 0;
    const float2 ax = bc2(a.x), ay = bc2(a.y), az = bc2(a.z), aw = bc2(a.w);
#pragma unroll 2
    for (int k = 0; k < jn; k += 2) {
        const bool v0 = active && k >= lo, v1 = active && k + 1 >= lo && k + 1 < jn;
        const float2 d0 = fma2(*reinterpret_cast<const float2*>(&soa[0][k]), bc2(-1.0f), ax);  // a - b, one rounding
        const float2 d1 = fma2(*reinterpret_cast<const float2*>(&soa[1][k]), bc2(-1.0f), ay);
        const float2 d2 = fma2(*reinterpret_cast<const float2*>(&soa[2][k]), bc2(-1.0f), az);
        const float2 gd = fma2(*reinterpret_cast<const float2*>(&soa[3][k]), bc2(-1.0f), aw);
        const float2 s2 = fma2(d2, d2, fma2(d1, d1, mul2(d0, d0)));
        const float2 de = make_float2(sqrt_mufu(s2.x), sqrt_mufu(s2.y));
        bool n0 = false, n1 = false;
        uint32_t kc0, kc1, kg0, kg1;
        int_count2(de, kMarginDe, vmax, kc0, kc1, n0, n1);
        int_count2(make_float2(fabsf(gd.x), fabsf(gd.y)), kMarginGd, vmax, kg0, kg1, n0, n1);
        int b0 = static_cast<int>(kc0) * stride + static_cast<int>(kg0);
        int b1 = static_cast<int>(kc1) * stride + static_cast<int>(kg1);
        n0 = n0 && v0;
        n1 = n1 && v1;
        if (__any_sync(0xFFFFFFFFu, n0 || n1)) {  // rare: the reference's fp64 route
            if (n0) b0 = exact(k);
            if (n1) b1 = exact(k + 1);
        }
        add(b0, v0);
        add(b1, v1);
    }
    WarpHist w;
    w.h = wh;
    w.full = full;
    w.full_bin = full_bin;
    flush_hist(sh, w, nbins, hist);
}

__global__ void __launch_bounds__(kTile) metric_pairs_kernel(const double4* __restrict__ labg,
                                                             const int64_t* __restrict__ pi,
                                                             const int64_t* __restrict__ pj, int64_t npairs,
                                                             Thresholds th, unsigned long long* hist) {
    __shared__ uint32_t sh[(kTile / 32) * kBins];
    __shared__ double ts[16], tg[16];
    const int stride = th.ntau + 1, nbins = stride * stride;
    for (int b = threadIdx.x; b < (kTile / 32) * kBins; b += blockDim.x) sh[b] = 0;
    if (threadIdx.x < 16) {
        ts[threadIdx.x] = th.s[threadIdx.x];
        tg[threadIdx.x] = th.g[threadIdx.x];
    }
    __syncthreads();
    WarpHist wh;
    wh.h = sh + (threadIdx.x / 32) * kBins;
    wh.full_bin = th.ntau * stride + th.ntau;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < npairs;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x)
        wh.add(pair_bin(labg[pi[q]], labg[pj[q]], ts, tg, stride));
    flush_hist(sh, wh, nbins, hist);
}

// least double s >= 0 with fl(sqrt(s)) >= tau (host libm sqrt is correctly rounded)
double sqrt_threshold(double tau) {
    uint64_t lo = 0, hi;
    const double top = tau * tau * 4.0 + 4.0;
    std::memcpy(&hi, &top, 8);
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        double m;
        std::memcpy(&m, &mid, 8);
        (std::sqrt(m) >= tau ? hi : lo) = mid;
    }
    double r;
    std::memcpy(&r, &hi, 8);
    return r;
}

int make_thresholds(const double* taus, int ntau, Thresholds* th) {
    if (ntau < 1 || ntau > kMaxTau) return set_error(WG_EINVAL, "need 1..%d thresholds, got %d", kMaxTau, ntau);
    for (int k = 0; k < ntau; ++k) {
        if (!(taus[k] > 0.0) || std::isinf(taus[k]))
            return set_error(WG_EINVAL, "tau must be positive and finite, got %.17g", taus[k]);
        if (k && !(taus[k] > taus[k - 1])) return set_error(WG_EINVAL, "taus must be strictly increasing");
    }
    for (int k = 0; k < 16; ++k) {
        th->s[k] = k < ntau ? sqrt_threshold(taus[k]) : INFINITY;
        th->g[k] = k < ntau ? taus[k] : INFINITY;
    }
    th->ntau = ntau;
    return WG_OK;
}

// taus == 1, 2, ..., ntau (TAU_SWEEP and its prefixes): the fp32 integer-count kernel applies
bool integer_taus(const double* taus, int ntau) {
    for (int k = 0; k < ntau; ++k)
        if (taus[k] != static_cast<double>(k + 1)) return false;
    return true;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

int metric_hist_from_lab(const double4* labg, const float4* lab32, int64_t npix, const double* taus, int ntau,
                         const Thresholds& th, const int64_t* pair_i, const int64_t* pair_j, int64_t npairs,
                         unsigned long long* hist, cudaStream_t st);

// Host Lab: lab_rows (_kernels.pyx:115-132) in the reference's operation order
// with the platform libm's pow / cbrt -- the very functions its compiled
// kernel calls -- so every (L*, a*, b*) and every pair's delta E is the
// reference's to the last bit, and the device pair counts are exact by
// construction. (The device's own pow / cbrt, used by wg_metric_hist_f64 on
// device pointers, agree only to ~1e-12: a pair whose delta E lies that close
// to a threshold could count differently.) Per pixel O(1) on host threads;
// the O(n^2) pair loop stays on the device.
namespace {
double host_lin(double c) { return c <= 0.04045 ? c / 12.92 : std::pow((c + 0.055) / 1.055, 2.4); }
double host_labf(double t) { return t > LAB_EPS ? std::cbrt(t) : (LAB_KAPPA * t + 16.0) / 116.0; }
double host_dot(double a0, double a1, double a2, double x, double y, double z) { return a0 * x + a1 * y + a2 * z; }
}  // namespace

void host_lab(const double* rgb, const double* gray, int64_t n, double4* labg, float4* lab32) {
    const auto span = [&](int64_t p0, int64_t p1) {
        for (int64_t p = p0; p < p1; ++p) {
            const double lr = host_lin(rgb[3 * p]), lg = host_lin(rgb[3 * p + 1]), lb = host_lin(rgb[3 * p + 2]);
            const double fx = host_labf(host_dot(MX0, MX1, MX2, lr, lg, lb) / WHITE_X);
            const double fy = host_labf(host_dot(MY0, MY1, MY2, lr, lg, lb));
            const double fz = host_labf(host_dot(MZ0, MZ1, MZ2, lr, lg, lb) / WHITE_Z);
            const double4 v = make_double4(116.0 * fy - 16.0, 500.0 * (fx - fy), 200.0 * (fy - fz), gray[p] * 100.0);
            labg[p] = v;
            lab32[p] = make_float4(static_cast<float>(v.x), static_cast<float>(v.y), static_cast<float>(v.z),
                                   static_cast<float>(v.w));
        }
    };
    static const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t nt = std::min<int64_t>({16, static_cast<int64_t>(hw), (n + 16383) / 16384});
    if (nt <= 1) {
        span(0, n);
        return;
    }
    const int64_t per = (n + nt - 1) / nt;
    std::vector<std::thread> ts;
    for (int64_t t = 1; t < nt; ++t) ts.emplace_back(span, t * per, std::min(n, (t + 1) * per));
    span(0, std::min(n, per));
    for (std::thread& t : ts) t.join();
}

// exact counts from host arrays: host Lab, then the device pair loop
int metric_hist_host_lab(const double* rgb, const double* gray, int64_t npix, const double* taus, int ntau,
                         const int64_t* pair_i, const int64_t* pair_j, int64_t npairs, unsigned long long* hist,
                         void* scratch, size_t scratch_bytes, cudaStream_t st) {
    Thresholds th;
    int rc = make_thresholds(taus, ntau, &th);
    if (rc != WG_OK) return rc;
    if (scratch_bytes < wg_metric_scratch_bytes(npix) || (npix > 0 && !scratch))
        return set_error(WG_ESCRATCH, "metric scratch too small: need %zu bytes", wg_metric_scratch_bytes(npix));
    const int stride = ntau + 1;
    cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * stride * stride, st);
    if (e != cudaSuccess) return set_error(static_cast<int>(e), "metric: memset: %s", cudaGetErrorString(e));
    if (npix < 2) return WG_OK;
    std::vector<double4> hg(static_cast<size_t>(npix));
    std::vector<float4> h32(static_cast<size_t>(npix));
    host_lab(rgb, gray, npix, hg.data(), h32.data());
    double4* labg = static_cast<double4*>(scratch);
    float4* lab32 = reinterpret_cast<float4*>(static_cast<uint8_t*>(scratch) +
                                              align256(static_cast<size_t>(npix) * sizeof(double4)));
    e = cudaMemcpyAsync(labg, hg.data(), static_cast<size_t>(npix) * sizeof(double4), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(lab32, h32.data(), static_cast<size_t>(npix) * sizeof(float4), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return set_error(static_cast<int>(e), "metric: H2D: %s", cudaGetErrorString(e));
    rc = metric_hist_from_lab(labg, lab32, npix, taus, ntau, th, pair_i, pair_j, npairs, hist, st);
    cudaStreamSynchronize(st);  // the host arrays above are copied before they go out of scope
    return rc;
}
}  // namespace wg

using namespace wg;

extern "C" size_t wg_metric_scratch_bytes(int64_t npix) {
    // fp64 (L*, a*, b*, 100 g) per pixel, then its fp32 copy
    return npix < 0 ? 0
                    : align256(static_cast<size_t>(npix) * sizeof(double4)) +
                          align256(static_cast<size_t>(npix) * sizeof(float4)) + 256;
}

extern "C" int wg_metric_hist_f64(const double* rgb, const double* gray, int64_t npix, const double* taus, int ntau,
                                  const int64_t* pair_i, const int64_t* pair_j, int64_t npairs,
                                  unsigned long long* hist, void* scratch, size_t scratch_bytes, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_npix(npairs) || check_ptrs(npix, rgb, gray));
    Thresholds th;
    int rc = make_thresholds(taus, ntau, &th);
    if (rc != WG_OK) return rc;
    if (!hist) return set_error(WG_EINVAL, "null histogram");
    if ((pair_i == nullptr) != (pair_j == nullptr)) return set_error(WG_EINVAL, "pair_i / pair_j: both or neither");
    if (scratch_bytes < wg_metric_scratch_bytes(npix) || (npix > 0 && !scratch))
        return set_error(WG_ESCRATCH, "metric scratch too small: need %zu bytes", wg_metric_scratch_bytes(npix));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int stride = ntau + 1;
    cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * stride * stride, st);
    if (e != cudaSuccess) return set_error(static_cast<int>(e), "metric: memset: %s", cudaGetErrorString(e));
    if (npix < 2) return WG_OK;
    double4* labg = static_cast<double4*>(scratch);
    float4* lab32 = reinterpret_cast<float4*>(static_cast<uint8_t*>(scratch) +
                                              align256(static_cast<size_t>(npix) * sizeof(double4)));
    int device = 0;
    cudaGetDevice(&device);
    const unsigned prep_blocks =
        static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((npix + 255) / 256, 16LL * sm_count(device))));
    metric_prep_kernel<<<prep_blocks, 256, 0, st>>>(rgb, gray, labg, lab32, npix);
    return metric_hist_from_lab(labg, lab32, npix, taus, ntau, th, pair_i, pair_j, npairs, hist, st);
}

namespace wg {
// the pair loops on (L*, a*, b*, 100 g) already in device memory (labg, and its fp32 copy lab32)
int metric_hist_from_lab(const double4* labg, const float4* lab32, int64_t npix, const double* taus, int ntau,
                         const Thresholds& th, const int64_t* pair_i, const int64_t* pair_j, int64_t npairs,
                         unsigned long long* hist, cudaStream_t st) {
    int device = 0;
    cudaGetDevice(&device);
    if (pair_i) {
        if (npairs) {
            const unsigned blocks = static_cast<unsigned>(
                std::max<int64_t>(1, std::min<int64_t>((npairs + kTile - 1) / kTile, 8LL * sm_count(device))));
            metric_pairs_kernel<<<blocks, kTile, 0, st>>>(labg, pair_i, pair_j, npairs, th, hist);
        }
    } else {
        const int64_t nt = (npix + kTile - 1) / kTile;
        if (nt > 65535) return set_error(WG_EINVAL, "exhaustive pairs support up to %d pixels", 65535 * kTile);
        const dim3 grid(static_cast<unsigned>(nt), static_cast<unsigned>(nt));
        if (integer_taus(taus, ntau))
            metric_all_pairs_int_kernel<<<grid, kTile, 0, st>>>(lab32, labg, npix, th,
                                                                 static_cast<float>(ntau) + 0.5f, hist);
        else
            metric_all_pairs_kernel<<<grid, kTile, 0, st>>>(labg, npix, th, hist);
    }
    return check_launch("metric pair counts");
}
}  // namespace wg

// counts[k][0..3] = (color set, kept, gray set, fabricated) for tau k, from H[kc][kg]
extern "C" int wg_metric_counts_from_hist(const unsigned long long* hist, int ntau, int64_t* counts) {
    if (ntau < 1 || ntau > kMaxTau || !hist || !counts) return set_error(WG_EINVAL, "bad histogram arguments");
    const int stride = ntau + 1;
    for (int k = 0; k < ntau; ++k) {
        int64_t color = 0, kept = 0, grayc = 0;
        for (int kc = 0; kc <= ntau; ++kc)
            for (int kg = 0; kg <= ntau; ++kg) {
                const int64_t c = static_cast<int64_t>(hist[kc * stride + kg]);
                color += kc > k ? c : 0;
                grayc += kg > k ? c : 0;
                kept += (kc > k && kg > k) ? c : 0;
            }
        counts[4 * k] = color;
        counts[4 * k + 1] = kept;
        counts[4 * k + 2] = grayc;
        counts[4 * k + 3] = grayc - kept;
    }
    return WG_OK;
}
