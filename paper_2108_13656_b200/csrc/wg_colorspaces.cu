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
// test_backend.py:84-101). The uint8 -> uint8 variants are bit-identical for
// all three methods (see OpLumaU8) and serve the GPU-side Table-1
// comparison.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <cstdint>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"
#include "wg_stream.cuh"

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

// uint8 -> uint8 = quantize_u8(<method>_rows(dequantize_u8(rgb))), bit-identical
// to the reference (codec.py:22-29 around _kernels.pyx:59-112) without
// evaluating its fp64 chain per pixel. These run as Ops on the shared
// streaming skeleton (wg_stream.cuh, register-prefetch LDG kernel, 16 px per
// thread per tile).
//  * BT.601: v*255 is S/10000 for the exact integer S = 2989r + 5870g + 1140b
//    up to fp64 rounding (< 1e-12), so round-half-up of S/10000 is the
//    reference's result except at exact ties (S mod 10000 == 5000, ~1e-4 of
//    colours), where fp64 rounding decides: those pixels evaluate the
//    reference expression as written (out of line).
//  * HSV V: dequantize / quantize are monotone and exact on bytes -> byte max.
//  * Lab L*: x = L*/100 * 255 + 0.5 is formed in fp32 from per-byte fp32
//    tables of M_Y[c] * lin(k/255) (shared memory) and a MUFU y^(-1/3) with
//    one division-free Newton step; |x_f32 - x| < 5e-5. Pixels whose x lies within kLabMargin
//    of a rounding boundary take the exact route: Y in fp64 from the host's
//    M_Y[c] * lin(k/255) products (libm pow, the reference's own rounding) and
//    the 255 Y thresholds where the quantized output steps, found on the host
//    by bisection over the reference's fp64 chain (libm cbrt).
constexpr float kLabMargin = 2e-4f;

struct LabTables {
    double prod[3][256];  // fl(M_Y[c] * _srgb_to_linear(k / 255.0)), exact reference products
    double step[257];     // step[j] = least Y with quantized L* >= j; step[0] = -inf, step[256] = +inf
    float prodf[3][256];  // the same products rounded to fp32 (hot path)
};

// the reference's fp64 expression, for the exact-tie pixels
__device__ __forceinline__ uint32_t bt601_u8_tie(uint32_t r, uint32_t g, uint32_t b) {
    return quantize_d(bt601_d(deq_byte(r), deq_byte(g), deq_byte(b)));
}

// (rounded S/10000, tie flag)
__device__ __forceinline__ uint32_t bt601_u8_fast(uint32_t r, uint32_t g, uint32_t b, bool& tie) {
    const uint32_t s = 2989u * r + 5870u * g + 1140u * b + 5000u;
    const uint32_t q = s / 10000u;
    tie = s == q * 10000u;
    return q;
}

__device__ __forceinline__ float log2f_mufu(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float exp2f_mufu(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// x = L*/100 * 255 + 0.5 in fp32 (explicit FMAs: the build is -fmad=false for
// the fp64 paths), clamped to the mid-bin 255.25 (the reference clamps L*/100 at
// 1, so everything past 254.5 is 255). Returns t = fl_rd(x + 2^23), whose low
// byte is floor(x), and whether x is farther than kLabMargin from an integer.
__device__ __forceinline__ float lab_u8_fast(float y, bool& sure, float& x_out) {
    // cube-root branch: r ~ y^(-1/3) from MUFU, one division-free Newton step,
    // cbrt(y) = y * r^2 -> x = 295.8 * cbrt(y) - 40.3
    const float r0 = exp2f_mufu(__fmul_rn(log2f_mufu(y), -1.0f / 3.0f));
    const float u = __fmaf_rn(-y, __fmul_rn(__fmul_rn(r0, r0), r0), 4.0f);
    const float ru = __fmul_rn(r0, u);  // 3 * r1
    const float f = __fmul_rn(__fmul_rn(y, 1.0f / 9.0f), __fmul_rn(ru, ru));
    const float x_cbrt = __fmaf_rn(f, 116.0f * 2.55f, 0.5f - 16.0f * 2.55f);
    // linear toe: L* = kappa * y
    const float x_toe = __fmaf_rn(y, static_cast<float>(LAB_KAPPA) * 2.55f, 0.5f);
    const float x = fminf(y > static_cast<float>(LAB_EPS) ? x_cbrt : x_toe, 255.25f);
    const float t = __fadd_rd(x, 8388608.0f);
    const float d = __fsub_rn(x, __fsub_rn(t, 8388608.0f));  // x - floor(x)
    sure = fabsf(__fsub_rn(d, 0.5f)) < 0.5f - kLabMargin;
    x_out = x;
    return t;
}

// Near a rounding boundary j (|x - j| <= margin) the result is j - 1 or j;
// Y in fp64 (the reference's products, L1-cached) against step[j] decides.
__device__ __forceinline__ uint32_t lab_u8_exact(const LabTables* tab, float x, uint32_t r, uint32_t g,
                                                 uint32_t b) {
    const double y = __dadd_rn(__dadd_rn(__ldg(&tab->prod[0][r]), __ldg(&tab->prod[1][g])), __ldg(&tab->prod[2][b]));
    const int j = min(max(__float2int_rn(x), 1), 255);
    return static_cast<uint32_t>(y >= __ldg(&tab->step[j]) ? j : j - 1);
}

__device__ __forceinline__ float* lab_prodf_smem() {
    __shared__ float s[3 * 256];
    return s;
}

template <int METHOD>
struct OpLumaU8 {
    static constexpr bool kLdg = true;
    static constexpr int kPx = 16;
    const uint8_t* in;
    uint8_t* out;
    const LabTables* tab;  // device copy (method 2 only)

    __device__ __forceinline__ void prologue() const {
        if constexpr (METHOD == 2) {
            float* s = lab_prodf_smem();
            const float* src = &tab->prodf[0][0];
            for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) s[i] = src[i];
        }
    }
    // fast route for one pixel; `slow` flags a pixel the exact route must redo
    // (BT.601 exact tie, Lab near a rounding boundary)
    __device__ __forceinline__ uint32_t fast(uint32_t r, uint32_t g, uint32_t b, bool& slow) const {
        if constexpr (METHOD == 0) {
            return bt601_u8_fast(r, g, b, slow);
        } else if constexpr (METHOD == 1) {
            slow = false;
            return max(r, max(g, b));
        } else {
            const float* s = lab_prodf_smem();
            bool sure;
            float x;
            const float t = lab_u8_fast(__fadd_rn(__fadd_rn(s[r], s[256 + g]), s[512 + b]), sure, x);
            slow = !sure;
            return __float_as_uint(t) & 255u;
        }
    }
    // exact route for pixel p, straight from global memory
    __device__ __forceinline__ uint32_t exact(int64_t p) const {
        const uint32_t r = __ldg(in + 3 * p), g = __ldg(in + 3 * p + 1), b = __ldg(in + 3 * p + 2);
        if constexpr (METHOD == 0) {
            return bt601_u8_tie(r, g, b);
        } else {
            const float* s = lab_prodf_smem();
            bool sure;
            float x;
            lab_u8_fast(__fadd_rn(__fadd_rn(s[r], s[256 + g]), s[512 + b]), sure, x);
            return lab_u8_exact(tab, x, r, g, b);
        }
    }
    __device__ __forceinline__ void vec(const uint4 (&v)[3], int64_t px0) const {
        const uint32_t w[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                                v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
        uint32_t o[4] = {0u, 0u, 0u, 0u};
        uint32_t slow_mask = 0;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            uint32_t c[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int bi = 3 * p + k;
                c[k] = __byte_perm(w[bi >> 2], 0u, 0x4440u | (bi & 3));
            }
            bool slow;
            o[p >> 2] |= fast(c[0], c[1], c[2], slow) << (8 * (p & 3));
            slow_mask |= static_cast<uint32_t>(slow) << p;
        }
        if constexpr (METHOD != 1) {
            if (slow_mask) {  // rare; a real branch, so the exact route costs nothing when not taken
#pragma unroll 1
                for (int p = 0; p < 16; ++p) {
                    if (slow_mask >> p & 1u) {
                        const uint32_t q = exact(px0 + p), sh = 8 * (p & 3), k = p >> 2;
                        // o[k] with a dynamic k would go to local memory: select instead
                        const uint32_t m = ~(255u << sh), qs = q << sh;
                        o[0] = k == 0 ? (o[0] & m) | qs : o[0];
                        o[1] = k == 1 ? (o[1] & m) | qs : o[1];
                        o[2] = k == 2 ? (o[2] & m) | qs : o[2];
                        o[3] = k == 3 ? (o[3] & m) | qs : o[3];
                    }
                }
            }
        }
        st_global_cs_v4(out + px0, make_uint4(o[0], o[1], o[2], o[3]));
    }
    __device__ __forceinline__ void scalar(int64_t p) const {
        bool slow;
        const uint32_t q = fast(in[3 * p], in[3 * p + 1], in[3 * p + 2], slow);
        out[p] = static_cast<uint8_t>(slow ? exact(p) : q);
    }
};

// ---- host side of the Lab tables: the reference's fp64 chain on the host libm
double host_srgb_to_linear(double c) { return c <= 0.04045 ? c / 12.92 : std::pow((c + 0.055) / 1.055, 2.4); }
double host_lab_f(double t) { return t > LAB_EPS ? std::cbrt(t) : (LAB_KAPPA * t + 16.0) / 116.0; }
int host_lab_q(double y) {
    double v = (116.0 * host_lab_f(y) - 16.0) / 100.0;
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    return static_cast<int>(std::floor(v * 255.0 + 0.5));
}

LabTables make_lab_tables() {
    LabTables t{};
    const double my[3] = {MY0, MY1, MY2};
    for (int k = 0; k < 256; ++k) {
        const double lin = host_srgb_to_linear(static_cast<double>(k) / 255.0);
        for (int c = 0; c < 3; ++c) {
            t.prod[c][k] = my[c] * lin;
            t.prodf[c][k] = static_cast<float>(t.prod[c][k]);
        }
    }
    t.step[0] = -INFINITY;
    t.step[256] = INFINITY;
    for (int j = 1; j < 256; ++j) {
        // least double y in [0, 2] with host_lab_q(y) >= j; positive doubles order like their bits
        uint64_t lo, hi;
        double d0 = 0.0, d1 = 2.0;
        std::memcpy(&lo, &d0, 8);
        std::memcpy(&hi, &d1, 8);
        while (hi - lo > 1) {
            const uint64_t mid = lo + (hi - lo) / 2;
            double m;
            std::memcpy(&m, &mid, 8);
            (host_lab_q(m) >= j ? hi : lo) = mid;
        }
        std::memcpy(&t.step[j], &hi, 8);
    }
    return t;
}

// one device-resident copy per device, uploaded on first use
const LabTables* device_lab_tables(int device) {
    static std::mutex mu;
    static const LabTables* tabs[kMaxDevices] = {nullptr};
    std::lock_guard<std::mutex> lock(mu);
    if (!tabs[device]) {
        static const LabTables host = make_lab_tables();
        void* d = nullptr;
        if (cudaMalloc(&d, sizeof(LabTables)) != cudaSuccess) return nullptr;
        if (cudaMemcpy(d, &host, sizeof(LabTables), cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(d);
            return nullptr;
        }
        tabs[device] = static_cast<const LabTables*>(d);
    }
    return tabs[device];
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
    const void* outs[1] = {out};
    if (method == 0) return launch_stream(OpLumaU8<0>{rgb, out, nullptr}, rgb, outs, 1, npix, st);
    if (method == 1) return launch_stream(OpLumaU8<1>{rgb, out, nullptr}, rgb, outs, 1, npix, st);
    int device = 0;
    cudaGetDevice(&device);
    if (device < 0 || device >= kMaxDevices) return set_error(WG_ENODEV, "device ordinal out of range");
    const LabTables* tab = device_lab_tables(device);
    if (!tab) return set_error(static_cast<int>(cudaErrorMemoryAllocation), "lab tables: device allocation failed");
    return launch_stream(OpLumaU8<2>{rgb, out, tab}, rgb, outs, 1, npix, st);
}
