// wg_kernels.cu -- the decolor / sigmoid / quantize Ops and their stream-ordered
// C-ABI launchers.
//
// Hot path: the per-pixel Ops (OpDecolorU8, OpDecolorU8Exact, OpDecolorF32,
// OpToneF32) run on the streaming skeleton of wg_stream.cuh, all of them on
// ldg_stream_kernel: each thread takes 48 contiguous input bytes (three
// 128-bit coalesced loads) of a 256-thread tile with the next tile already in
// flight in registers, de-interleaves the RGB bytes with PRMT into packed
// f32x2 pairs (uint8), computes in registers and writes its output with one
// 128-bit store; the grid is a multiple of the SM count. The cp.async.bulk
// (TMA) shared-memory ring of the same skeleton (stream_kernel) measured
// slower (uint8: issue-bound ops; fp32: 80-89% vs 105% of the copy peak) and
// serves ops without kLdg; the fp64 row
// kernels below (decolor_f64_kernel & co.) are the bit-identical drop-in path.
//
// Reference correspondence: _kernels.pyx:47-56 (decolor_rows),
// tonemap.py:72-83 (apply_sigmoid), :172-192 (reinstate_color),
// :195-216 (tonemap_image global), codec.py:22-29 (quantize / dequantize).
#include <cuda_runtime.h>

#include <mutex>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"
#include "wg_stream.cuh"

namespace wg {

// ------------------------------------------------------------------ ops
// An Op consumes the 48 input bytes of one thread (3 x uint4, already in
// registers) for pixels [px0, px0 + kPx) and stores its outputs; scalar()
// handles one pixel straight from global memory (tails, unaligned buffers)
// with bit-identical arithmetic.

// Default uint8 op: round-to-nearest of 255*gray in fp32 (the north-star bar:
// identical except +-1 on <= 0.01% of pixels; measured 5e-6 over all colours).
struct OpDecolorU8 {
    static constexpr bool kLdg = true;
    static constexpr int kInBpp = 3;
    static constexpr int kPx = 16;
    const uint8_t* in;
    uint8_t* gray;
    U8Consts k;

    __device__ __forceinline__ void vec(const uint4 (&v)[3], int64_t px0) const {
        const uint32_t w[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                                v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
        float2 f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            // pixels 2j and 2j+1 share one packed lane pair
            float2 ch[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int b0 = 3 * (2 * j) + c, b1 = 3 * (2 * j + 1) + c;
                ch[c] = make_float2(byte_biased(w[b0 >> 2], b0 & 3), byte_biased(w[b1 >> 2], b1 & 3));
                ch[c] = add2(ch[c], bc2(-kMagic));
            }
            f[j] = decolor255_x2(ch[0], ch[1], ch[2], k);
        }
        uint4 o;
        o.x = __byte_perm(pack_lo2(f[0].x, f[0].y), pack_lo2(f[1].x, f[1].y), 0x5410u);
        o.y = __byte_perm(pack_lo2(f[2].x, f[2].y), pack_lo2(f[3].x, f[3].y), 0x5410u);
        o.z = __byte_perm(pack_lo2(f[4].x, f[4].y), pack_lo2(f[5].x, f[5].y), 0x5410u);
        o.w = __byte_perm(pack_lo2(f[6].x, f[6].y), pack_lo2(f[7].x, f[7].y), 0x5410u);
        st_global_cs_v4(gray + px0, o);
    }
    __device__ __forceinline__ void scalar(int64_t p) const {
        gray[p] = decolor255_x1(static_cast<float>(in[3 * p]), static_cast<float>(in[3 * p + 1]),
                                static_cast<float>(in[3 * p + 2]), k);
    }
};


// Bit-exact variant (opt-in, wg_decolor_u8_exact): the final FMA keeps 15
// fraction bits (decolor255_bits_x2); groups with a pixel within the table's
// margin of a rounding boundary take the exact byte of that colour from the
// near-tie table (csrc/wg_u8exact.cu). ~10% slower than OpDecolorU8 on C3:
// the shift, shift-add and compare per pixel compete for issue slots with the
// saturated FMA and MUFU pipes.
struct OpDecolorU8Exact {
    static constexpr bool kLdg = true;
    static constexpr int kInBpp = 3;
    static constexpr int kPx = 16;
    const uint8_t* in;
    uint8_t* gray;
    U8Consts k;
    U8Exact ex;  // exact bytes of the near-tie colours (csrc/wg_u8exact.cu)

    __device__ __forceinline__ void vec(const uint4 (&v)[3], int64_t px0) const {
        const uint32_t w[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                                v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
        uint32_t bits[16];
        // near-tie test: ((bits + margin) << 17) < (2 margin + 1) << 17, i.e. the
        // 15-bit fraction within `margin` of a rounding boundary; one shift-add and
        // one compare per pixel, OR-ed into a per-group flag
        const uint32_t madd = ex.margin << 17, mlim = (2u * ex.margin + 1u) << 17;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            // pixels 2j and 2j+1 share one packed lane pair
            float2 ch[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int b0 = 3 * (2 * j) + c, b1 = 3 * (2 * j + 1) + c;
                ch[c] = make_float2(byte_biased(w[b0 >> 2], b0 & 3), byte_biased(w[b1 >> 2], b1 & 3));
                ch[c] = add2(ch[c], bc2(-kMagic));
            }
            const float2 f = decolor255_bits_x2(ch[0], ch[1], ch[2], k);
            bits[2 * j] = __float_as_uint(f.x);
            bits[2 * j + 1] = __float_as_uint(f.y);
        }
        const uint32_t any_tie = any_near_tie16(bits, madd, mlim);
        // low byte of bits >> 15 = floor(255 gray + 0.5)
        uint4 o;
        o.x = __byte_perm(__byte_perm(bits[0] >> 15, bits[1] >> 15, 0x0040u),
                          __byte_perm(bits[2] >> 15, bits[3] >> 15, 0x0040u), 0x5410u);
        o.y = __byte_perm(__byte_perm(bits[4] >> 15, bits[5] >> 15, 0x0040u),
                          __byte_perm(bits[6] >> 15, bits[7] >> 15, 0x0040u), 0x5410u);
        o.z = __byte_perm(__byte_perm(bits[8] >> 15, bits[9] >> 15, 0x0040u),
                          __byte_perm(bits[10] >> 15, bits[11] >> 15, 0x0040u), 0x5410u);
        o.w = __byte_perm(__byte_perm(bits[12] >> 15, bits[13] >> 15, 0x0040u),
                          __byte_perm(bits[14] >> 15, bits[15] >> 15, 0x0040u), 0x5410u);
        if (any_tie) fix_ties(bits, o, px0);  // ~0.4% of groups
        st_global_cs_v4(gray + px0, o);
    }
    // pixels next to a rounding boundary take the exact byte of their colour
    __device__ __forceinline__ void fix_ties(const uint32_t (&bits)[16], uint4& o, int64_t px0) const {
        uint32_t slow = 0;
#pragma unroll
        for (int p = 0; p < 16; ++p) slow |= static_cast<uint32_t>(bits_near_tie(bits[p], ex.margin)) << p;
        while (slow) {
            const int p = __ffs(slow) - 1;
            slow &= slow - 1;
            const uint8_t* src = in + 3 * (px0 + p);
            const uint32_t key = (static_cast<uint32_t>(__ldg(src)) << 16) | (static_cast<uint32_t>(__ldg(src + 1)) << 8) |
                                 __ldg(src + 2);
            const uint32_t sh = 8 * (p & 3), q = p >> 2;
            const uint32_t word = q == 0 ? o.x : q == 1 ? o.y : q == 2 ? o.z : o.w;
            const uint32_t e = u8exact_lookup(ex, key, (word >> sh) & 255u);
            const uint32_t nw = (word & ~(255u << sh)) | (e << sh);
            // o.{x,y,z,w} with a dynamic index would go to local memory: select instead
            o.x = q == 0 ? nw : o.x;
            o.y = q == 1 ? nw : o.y;
            o.z = q == 2 ? nw : o.z;
            o.w = q == 3 ? nw : o.w;
        }
    }
    __device__ __forceinline__ void scalar(int64_t p) const {
        const uint32_t r = in[3 * p], g = in[3 * p + 1], bl = in[3 * p + 2];
        const uint32_t bits = decolor255_bits_x1(static_cast<float>(r), static_cast<float>(g), static_cast<float>(bl), k);
        uint32_t q = bits_byte(bits);
        if (bits_near_tie(bits, ex.margin)) q = u8exact_lookup(ex, (r << 16) | (g << 8) | bl, q);
        gray[p] = static_cast<uint8_t>(q);
    }
};

struct OpDecolorF32 {
    static constexpr bool kLdg = true;
    static constexpr int kInBpp = 12;
    static constexpr int kPx = 4;
    const float* in;
    float* gray;
    AccConsts k;

    __device__ __forceinline__ void vec(const uint4 (&v)[3], int64_t px0) const {
        const float* f = reinterpret_cast<const float*>(&v[0]);
        float4 o;
        o.x = decolor_acc(f[0], f[1], f[2], k);
        o.y = decolor_acc(f[3], f[4], f[5], k);
        o.z = decolor_acc(f[6], f[7], f[8], k);
        o.w = decolor_acc(f[9], f[10], f[11], k);
        st_global_cs_v4(gray + px0, make_uint4(__float_as_uint(o.x), __float_as_uint(o.y),
                                              __float_as_uint(o.z), __float_as_uint(o.w)));
    }
    __device__ __forceinline__ void scalar(int64_t p) const {
        gray[p] = decolor_acc(in[3 * p], in[3 * p + 1], in[3 * p + 2], k);
    }
};

// decolor + global sigmoid (+ reinstate) on fp32 input
struct OpToneF32 {
    static constexpr bool kLdg = true;
    static constexpr int kInBpp = 12;
    static constexpr int kPx = 4;
    const float* in;
    float* toned;
    float* gray;     // may be null
    float* rgb_out;  // may be null
    AccConsts k;
    float m, slope;

    __device__ __forceinline__ void one(const float* px, const SigF& s, int64_t p) const {
        float l = decolor_acc(px[0], px[1], px[2], k);
        float lo = sigmoid_f(l, s);
        toned[p] = lo;
        if (gray) gray[p] = l;
        if (rgb_out) {
            // reinstate_color (tonemap.py:187-191)
            float ratio = __fdiv_rn(lo, fmaxf(l, 1e-6f));
#pragma unroll
            for (int c = 0; c < 3; ++c)
                rgb_out[3 * p + c] = l == 0.0f ? 0.0f : fminf(fmaxf(__fmul_rn(px[c], ratio), 0.0f), 1.0f);
        }
    }
    __device__ __forceinline__ void vec(const uint4 (&v)[3], int64_t px0) const {
        const SigF s = make_sig_f(m, slope);
        const float* f = reinterpret_cast<const float*>(&v[0]);
#pragma unroll
        for (int p = 0; p < 4; ++p) one(f + 3 * p, s, px0 + p);
    }
    __device__ __forceinline__ void scalar(int64_t p) const {
        const SigF s = make_sig_f(m, slope);
        one(in + 3 * p, s, p);
    }
};

// ------------------------------------------------------------------ elementwise fp64 kernels
// Two pixels per thread per iteration (p and p + stride: independent dependency
// chains of IEEE divisions and roots the scheduler interleaves), so an image of
// up to two grids' worth of pixels finishes in one chain latency instead of
// two waves (800x600: 9.6 -> ~5 us).
__global__ void decolor_f64_kernel(const double* __restrict__ rgb, double* __restrict__ out,
                                   int64_t npix, double br, double bk) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npix; p += 2 * stride) {
        const int64_t q = p + stride;
        const bool two = q < npix;
        const double r0 = rgb[3 * p], g0 = rgb[3 * p + 1], b0 = rgb[3 * p + 2];
        const double r1 = two ? rgb[3 * q] : 0.0, g1 = two ? rgb[3 * q + 1] : 0.0, b1 = two ? rgb[3 * q + 2] : 0.0;
        const double v0 = decolor_f64(r0, g0, b0, br, bk);
        const double v1 = decolor_f64(r1, g1, b1, br, bk);
        out[p] = v0;
        if (two) out[q] = v1;
    }
}

__global__ void sigmoid_f64_kernel(const double* __restrict__ in, double* __restrict__ out,
                                   int64_t n, double m, double k) {
    const SigD s = make_sig_d(m, k);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = sigmoid_d(in[i], s);
}

__global__ void sigmoid_f32_kernel(const float* __restrict__ in, float* __restrict__ out,
                                   int64_t n, float m, float k) {
    const SigF s = make_sig_f(m, k);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = sigmoid_f(in[i], s);
}

// reinstate_color, tonemap.py:187-191
__device__ __forceinline__ void reinstate_px_d(const double* c, double li, double lo, double* o) {
    const double ratio = lo / (li > 1e-6 ? li : 1e-6);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) o[ch] = li == 0.0 ? 0.0 : clamp01_d(c[ch] * ratio);
}

__global__ void reinstate_f64_kernel(const double* __restrict__ rgb, const double* __restrict__ l_in,
                                     const double* __restrict__ l_out, double* __restrict__ out,
                                     int64_t npix) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npix;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        reinstate_px_d(rgb + 3 * p, l_in[p], l_out[p], out + 3 * p);
}

__global__ void tonemap_global_f64_kernel(const double* __restrict__ rgb, double* __restrict__ l_out,
                                          double* __restrict__ rgb_out, int64_t npix, double br,
                                          double bk, double m, double k) {
    const SigD s = make_sig_d(m, k);
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npix;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double* c = rgb + 3 * p;
        const double li = decolor_f64(c[0], c[1], c[2], br, bk);
        const double lo = sigmoid_d(li, s);
        l_out[p] = lo;
        reinstate_px_d(c, li, lo, rgb_out + 3 * p);
    }
}

__global__ void quantize_u8_f64_kernel(const double* __restrict__ in, uint8_t* __restrict__ out,
                                       int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double v = clamp01_d(in[i]);
        if (v != v) v = 0.0;  // np.clip keeps NaN; astype(uint8) of NaN is 0 on x86
        out[i] = static_cast<uint8_t>(floor(__dadd_rn(__dmul_rn(v, 255.0), 0.5)));
    }
}

__global__ void dequantize_u8_f64_kernel(const uint8_t* __restrict__ in, double* __restrict__ out,
                                         int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __ddiv_rn(static_cast<double>(in[i]), 255.0);
}

static unsigned ew_blocks(int64_t n) {
    int device = 0;
    cudaGetDevice(&device);
    const int64_t want = (n + 255) / 256;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 8LL * sm_count(device))));
}

}  // namespace wg

using namespace wg;

// ====================================================================== C ABI (device pointers)

extern "C" int wg_decolor_u8(const uint8_t* rgb, uint8_t* gray, int64_t npix, double beta_r,
                             double beta_k, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, gray) || check_params(beta_r, beta_k));
    if (npix == 0) return WG_OK;
    OpDecolorU8 op{rgb, gray, make_u8_consts(beta_r, beta_k)};
    const void* outs[1] = {gray};
    return launch_stream(op, rgb, outs, 1, npix, static_cast<cudaStream_t>(stream));
}

extern "C" int wg_decolor_u8_exact(const uint8_t* rgb, uint8_t* gray, int64_t npix, double beta_r, double beta_k,
                                   void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, gray) || check_params(beta_r, beta_k));
    if (npix == 0) return WG_OK;
    U8Exact ex;
    std::unique_lock<std::mutex> hold;  // keeps the cached table alive until the launch is enqueued
    const int rc = u8exact_get(beta_r, beta_k, &ex, &hold);
    if (rc != WG_OK) return rc;
    OpDecolorU8Exact op{rgb, gray, make_u8_consts(beta_r, beta_k), ex};
    const void* outs[1] = {gray};
    return launch_stream(op, rgb, outs, 1, npix, static_cast<cudaStream_t>(stream));
}

extern "C" int wg_decolor_f32(const float* rgb, float* gray, int64_t npix, float beta_r,
                              float beta_k, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, gray) || check_params(beta_r, beta_k));
    OpDecolorF32 op{rgb, gray, make_acc_consts(beta_r, beta_k)};
    const void* outs[1] = {gray};
    return launch_stream(op, rgb, outs, 1, npix, static_cast<cudaStream_t>(stream));
}

extern "C" int wg_decolor_f64(const double* rgb, double* gray, int64_t npix, double beta_r,
                              double beta_k, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, gray) || check_params(beta_r, beta_k));
    if (npix == 0) return WG_OK;
    decolor_f64_kernel<<<ew_blocks(npix), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        rgb, gray, npix, beta_r, beta_k);
    return check_launch("decolor_f64");
}

extern "C" int wg_sigmoid_f64(const double* lum, double* out, int64_t n, double midpoint,
                              double slope, void* stream) {
    WG_CHECK_ARGS(check_npix(n) || check_ptrs(n, lum, out) || check_curve(midpoint, slope));
    if (n == 0) return WG_OK;
    sigmoid_f64_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(lum, out, n,
                                                                                    midpoint, slope);
    return check_launch("sigmoid_f64");
}

extern "C" int wg_sigmoid_f32(const float* lum, float* out, int64_t n, float midpoint, float slope,
                              void* stream) {
    WG_CHECK_ARGS(check_npix(n) || check_ptrs(n, lum, out) || check_curve(midpoint, slope));
    if (n == 0) return WG_OK;
    sigmoid_f32_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(lum, out, n,
                                                                                    midpoint, slope);
    return check_launch("sigmoid_f32");
}

extern "C" int wg_reinstate_f64(const double* rgb, const double* l_in, const double* l_out,
                                double* rgb_out, int64_t npix, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, rgb_out) || check_ptrs(npix, l_in, l_out));
    if (npix == 0) return WG_OK;
    reinstate_f64_kernel<<<ew_blocks(npix), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        rgb, l_in, l_out, rgb_out, npix);
    return check_launch("reinstate_f64");
}

extern "C" int wg_tonemap_global_f64(const double* rgb, double* l_out, double* rgb_out,
                                     int64_t npix, double beta_r, double beta_k, double midpoint,
                                     double slope, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, l_out) || check_ptrs(npix, rgb_out, rgb) ||
                  check_params(beta_r, beta_k) || check_curve(midpoint, slope));
    if (npix == 0) return WG_OK;
    tonemap_global_f64_kernel<<<ew_blocks(npix), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        rgb, l_out, rgb_out, npix, beta_r, beta_k, midpoint, slope);
    return check_launch("tonemap_global_f64");
}

extern "C" int wg_decolor_tone_f32(const float* rgb, float* toned, float* gray_or_null,
                                   float* rgb_out_or_null, int64_t npix, float beta_r, float beta_k,
                                   float midpoint, float slope, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, toned) || check_params(beta_r, beta_k) ||
                  check_curve(midpoint, slope));
    OpToneF32 op{rgb, toned, gray_or_null, rgb_out_or_null, make_acc_consts(beta_r, beta_k),
                 midpoint, slope};
    const void* outs[3] = {toned, gray_or_null, rgb_out_or_null};
    return launch_stream(op, rgb, outs, 3, npix, static_cast<cudaStream_t>(stream));
}

extern "C" int wg_quantize_u8_f64(const double* in, uint8_t* out, int64_t n, void* stream) {
    WG_CHECK_ARGS(check_npix(n) || check_ptrs(n, in, out));
    if (n == 0) return WG_OK;
    quantize_u8_f64_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(in, out, n);
    return check_launch("quantize_u8_f64");
}

extern "C" int wg_dequantize_u8_f64(const uint8_t* in, double* out, int64_t n, void* stream) {
    WG_CHECK_ARGS(check_npix(n) || check_ptrs(n, in, out));
    if (n == 0) return WG_OK;
    dequantize_u8_f64_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(in, out, n);
    return check_launch("dequantize_u8_f64");
}
