// wg_colorspaces.cu -- baseline luminance extractors:
// BT.601 luma, HSV value, CIELAB lightness and full CIELAB, restating the
// reference kernels _kernels.pyx:59-132 (and the scalar oracles
// colorspaces.py:38-84). The paper compares its method against these
// (Table 1: "ours" vs "L of CIE Lab" per-pixel time).
//
// fp64 kernels follow the reference's operation order with explicit rn
// intrinsics, so BT.601 and HSV V are bit-identical to the compiled backend;
// CIELAB goes through pow / cbrt, which CUDA and glibc round differently in
// the last ulp (the reference's own backends agree only to 1e-9,
// test_backend.py:84-101). The uint8 -> uint8 variants (also fp64, see
// luma_u8_kernel) serve the GPU-side Table-1 comparison.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"

namespace wg {
namespace {

// sRGB (D65, 2 degree observer) -> XYZ rows (_kernels.pyx:14-20)
constexpr double MX0 = 0.4124564, MX1 = 0.3575761, MX2 = 0.1804375;
constexpr double MY0 = 0.2126729, MY1 = 0.7151522, MY2 = 0.0721750;
constexpr double MZ0 = 0.0193339, MZ1 = 0.1191920, MZ2 = 0.9503041;
constexpr double WHITE_X = 0.95047, WHITE_Z = 1.08883;
constexpr double LAB_EPS = 216.0 / 24389.0, LAB_KAPPA = 24389.0 / 27.0;

__device__ __forceinline__ double bt601_d(double r, double g, double b) {
    return clamp01_d(__dadd_rn(__dadd_rn(__dmul_rn(0.2989, r), __dmul_rn(0.5870, g)), __dmul_rn(0.1140, b)));
}
__device__ __forceinline__ double hsv_v_d(double r, double g, double b) {
    double v = r;
    if (g > v) v = g;
    if (b > v) v = b;
    return v;
}
__device__ __forceinline__ double srgb_to_linear_d(double c) {
    if (c <= 0.04045) return __ddiv_rn(c, 12.92);
    return pow(__ddiv_rn(__dadd_rn(c, 0.055), 1.055), 2.4);
}
__device__ __forceinline__ double lab_f_d(double t) {
    if (t > LAB_EPS) return cbrt(t);
    return __ddiv_rn(__dadd_rn(__dmul_rn(LAB_KAPPA, t), 16.0), 116.0);
}
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double x, double y, double z) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a0, x), __dmul_rn(a1, y)), __dmul_rn(a2, z));
}
__device__ __forceinline__ double lab_l_d(double r, double g, double b) {
    const double lr = srgb_to_linear_d(r), lg = srgb_to_linear_d(g), lb = srgb_to_linear_d(b);
    const double lum = __dsub_rn(__dmul_rn(116.0, lab_f_d(dot3(MY0, MY1, MY2, lr, lg, lb))), 16.0);
    return clamp01_d(__ddiv_rn(lum, 100.0));
}

template <int METHOD>
__global__ void luma_f64_kernel(const double* __restrict__ rgb, double* __restrict__ out, int64_t npix) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npix;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double r = rgb[3 * p], g = rgb[3 * p + 1], b = rgb[3 * p + 2];
        out[p] = METHOD == 0 ? bt601_d(r, g, b) : METHOD == 1 ? hsv_v_d(r, g, b) : lab_l_d(r, g, b);
    }
}

__global__ void lab_f64_kernel(const double* __restrict__ rgb, double* __restrict__ out, int64_t npix) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npix;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double lr = srgb_to_linear_d(rgb[3 * p]), lg = srgb_to_linear_d(rgb[3 * p + 1]),
                     lb = srgb_to_linear_d(rgb[3 * p + 2]);
        const double fx = lab_f_d(__ddiv_rn(dot3(MX0, MX1, MX2, lr, lg, lb), WHITE_X));
        const double fy = lab_f_d(dot3(MY0, MY1, MY2, lr, lg, lb));
        const double fz = lab_f_d(__ddiv_rn(dot3(MZ0, MZ1, MZ2, lr, lg, lb), WHITE_Z));
        out[3 * p] = __dsub_rn(__dmul_rn(116.0, fy), 16.0);
        out[3 * p + 1] = __dmul_rn(500.0, __dsub_rn(fx, fy));
        out[3 * p + 2] = __dmul_rn(200.0, __dsub_rn(fy, fz));
    }
}

// uint8 -> uint8 = quantize_u8(<method>_rows(dequantize_u8(rgb))) evaluated in
// fp64 with the reference's operation order, so the result is bit-identical
// (BT.601 of integer bytes hits exact .5 ties for ~1e-4 of all colours; fp32
// would round those either way). The dequantized channel k/255 comes from an
// exact shared table; for Lab the sRGB linearisation of the 256 byte values
// is tabulated on the host with the same libm pow the reference links
// (_kernels.pyx:87-90), leaving one cbrt per pixel on the device. B200 runs
// fp64 at half the fp32 rate, far above what a 4 B/px stream needs.
struct ByteTable {
    double v[256];
};

__device__ __forceinline__ uint32_t quantize_d(double v) {
    // codec.py:22-25: floor(clip(v, 0, 1) * 255 + 0.5)
    return static_cast<uint32_t>(__dadd_rn(__dmul_rn(clamp01_d(v), 255.0), 0.5));
}

template <int METHOD>
__device__ __forceinline__ uint32_t luma_u8_px(const double* deq, const double* lin, uint32_t r, uint32_t g,
                                               uint32_t b) {
    if (METHOD == 1) return max(r, max(g, b));  // dequantize / quantize are monotone and exact on bytes
    if (METHOD == 0) return quantize_d(bt601_d(deq[r], deq[g], deq[b]));
    const double lum = __dsub_rn(__dmul_rn(116.0, lab_f_d(dot3(MY0, MY1, MY2, lin[r], lin[g], lin[b]))), 16.0);
    return quantize_d(__ddiv_rn(lum, 100.0));
}

// 4 px per thread (12 B in as 3 words, 4 B out); tails and unaligned buffers scalar
template <int METHOD>
__global__ void __launch_bounds__(256) luma_u8_kernel(const uint8_t* __restrict__ rgb, uint8_t* __restrict__ out,
                                                      int64_t npix, ByteTable lin_tab) {
    __shared__ double deq[256], lin[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        deq[i] = __ddiv_rn(static_cast<double>(i), 255.0);  // == dequantize_u8 (codec.py:28-29)
        lin[i] = lin_tab.v[i];
    }
    __syncthreads();
    const int64_t nq = npix >> 2;
    const bool vec = (reinterpret_cast<uintptr_t>(rgb) & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (vec) {
        for (int64_t q = t0; q < nq; q += stride) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(rgb + 12 * q);
            const uint32_t w0 = __ldcs(src), w1 = __ldcs(src + 1), w2 = __ldcs(src + 2);
            const uint32_t by[12] = {w0 & 255, w0 >> 8 & 255, w0 >> 16 & 255, w0 >> 24, w1 & 255, w1 >> 8 & 255,
                                     w1 >> 16 & 255, w1 >> 24, w2 & 255, w2 >> 8 & 255, w2 >> 16 & 255, w2 >> 24};
            uint32_t o = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                o |= luma_u8_px<METHOD>(deq, lin, by[3 * j], by[3 * j + 1], by[3 * j + 2]) << (8 * j);
            __stcs(reinterpret_cast<uint32_t*>(out) + q, o);
        }
    }
    for (int64_t p = (vec ? 4 * nq : 0) + t0; p < npix; p += stride)
        out[p] = static_cast<uint8_t>(luma_u8_px<METHOD>(deq, lin, rgb[3 * p], rgb[3 * p + 1], rgb[3 * p + 2]));
}

// host libm pow, exactly the reference's _srgb_to_linear on k / 255.0
const ByteTable& srgb_byte_table() {
    static const ByteTable tab = [] {
        ByteTable t{};
        for (int k = 0; k < 256; ++k) {
            const volatile double c = static_cast<double>(k) / 255.0;
            t.v[k] = c <= 0.04045 ? c / 12.92 : std::pow((c + 0.055) / 1.055, 2.4);
        }
        return t;
    }();
    return tab;
}

unsigned blocks_for(int64_t n) {
    int device = 0;
    cudaGetDevice(&device);
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 16LL * sm_count(device))));
}

}  // namespace
}  // namespace wg

using namespace wg;

extern "C" int wg_luma_f64(const double* rgb, double* out, int64_t npix, int method, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, out));
    if (method < 0 || method > 2) return set_error(WG_EINVAL, "luma method must be 0 (bt601), 1 (hsv v) or 2 (lab L*)");
    if (npix == 0) return WG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned b = blocks_for(npix);
    if (method == 0) luma_f64_kernel<0><<<b, 256, 0, st>>>(rgb, out, npix);
    else if (method == 1) luma_f64_kernel<1><<<b, 256, 0, st>>>(rgb, out, npix);
    else luma_f64_kernel<2><<<b, 256, 0, st>>>(rgb, out, npix);
    return check_launch("luma_f64");
}

extern "C" int wg_lab_f64(const double* rgb, double* lab, int64_t npix, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, lab));
    if (npix == 0) return WG_OK;
    lab_f64_kernel<<<blocks_for(npix), 256, 0, static_cast<cudaStream_t>(stream)>>>(rgb, lab, npix);
    return check_launch("lab_f64");
}

extern "C" int wg_luma_u8(const uint8_t* rgb, uint8_t* out, int64_t npix, int method, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, out));
    if (method < 0 || method > 2) return set_error(WG_EINVAL, "luma method must be 0 (bt601), 1 (hsv v) or 2 (lab L*)");
    if (npix == 0) return WG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned b = blocks_for((npix + 3) / 4);
    const ByteTable& lin = srgb_byte_table();
    if (method == 0) luma_u8_kernel<0><<<b, 256, 0, st>>>(rgb, out, npix, lin);
    else if (method == 1) luma_u8_kernel<1><<<b, 256, 0, st>>>(rgb, out, npix, lin);
    else luma_u8_kernel<2><<<b, 256, 0, st>>>(rgb, out, npix, lin);
    return check_launch("luma_u8");
}
