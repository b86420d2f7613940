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
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
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
                                   double4* __restrict__ labg, int64_t n) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double lr = lin_d(rgb[3 * p]), lg = lin_d(rgb[3 * p + 1]), lb = lin_d(rgb[3 * p + 2]);
        const double fx = labf_d(__ddiv_rn(dot3d(MX0, MX1, MX2, lr, lg, lb), WHITE_X));
        const double fy = labf_d(dot3d(MY0, MY1, MY2, lr, lg, lb));
        const double fz = labf_d(__ddiv_rn(dot3d(MZ0, MZ1, MZ2, lr, lg, lb), WHITE_Z));
        labg[p] = make_double4(__dsub_rn(__dmul_rn(116.0, fy), 16.0), __dmul_rn(500.0, __dsub_rn(fx, fy)),
                               __dmul_rn(200.0, __dsub_rn(fy, fz)), __dmul_rn(gray[p], 100.0));
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
        if (bin == full_bin) ++full;
        else atomicAdd(&h[bin], 1u);
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

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace
}  // namespace wg

using namespace wg;

extern "C" size_t wg_metric_scratch_bytes(int64_t npix) {
    return npix < 0 ? 0 : align256(static_cast<size_t>(npix) * sizeof(double4)) + 256;
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
    int device = 0;
    cudaGetDevice(&device);
    const unsigned prep_blocks =
        static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((npix + 255) / 256, 16LL * sm_count(device))));
    metric_prep_kernel<<<prep_blocks, 256, 0, st>>>(rgb, gray, labg, npix);
    if (pair_i) {
        if (npairs) {
            const unsigned blocks = static_cast<unsigned>(
                std::max<int64_t>(1, std::min<int64_t>((npairs + kTile - 1) / kTile, 8LL * sm_count(device))));
            metric_pairs_kernel<<<blocks, kTile, 0, st>>>(labg, pair_i, pair_j, npairs, th, hist);
        }
    } else {
        const int64_t nt = (npix + kTile - 1) / kTile;
        if (nt > 65535) return set_error(WG_EINVAL, "exhaustive pairs support up to %d pixels", 65535 * kTile);
        metric_all_pairs_kernel<<<dim3(static_cast<unsigned>(nt), static_cast<unsigned>(nt)), kTile, 0, st>>>(
            labg, npix, th, hist);
    }
    return check_launch("metric pair counts");
}

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
