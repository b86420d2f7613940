// wg_device.cuh -- device-side building blocks for the sm_100a decolorization
// kernels: PTX wrappers (mbarrier, cp.async.bulk, packed f32x2 math, MUFU)
// and the three per-pixel formulations of the warm/cool model (Eqs. 1-6,
// reference _kernels.pyx:31-44 / core.py:102-144):
//
//   decolor255_x2   uint8 path: two pixels per packed f32x2 lane pair, in the
//                   0..255 domain (homogeneity), 3 MUFU / px, no divide.
//   decolor_acc     fp32 path: IEEE sqrt / reciprocal, <= ~2e-7 abs error.
//   decolor_f64     fp64 path: the reference's operation order with explicit
//                   round-to-nearest intrinsics (no FMA contraction), hence
//                   bit-identical to the reference's compiled backend.
#pragma once

#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

namespace wg {

// ---------------------------------------------------------------- PTX: smem / mbarrier / bulk copy
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 32-bit load from a shared-memory (CTA window) address; non-volatile, so the
// compiler schedules it like a plain LDS and folds address arithmetic into it
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// Consumers of a cp.async.bulk ring must order their generic-proxy reads of a
// stage before the async-proxy (TMA) write that refills it: bar.sync alone
// does not (measured: LDS still in flight were overwritten by the next tile).
// Every consumer executes this after reading its stage, before the barrier
// that precedes the refill.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// One-thread bulk copy global -> shared (TMA engine, no tensor map needed for a
// contiguous byte range); completion is signalled on `bar` as tx bytes.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void st_global_cs_v4(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// ---------------------------------------------------------------- packed f32x2 (FFMA2 / FMUL2 / FADD2)
__device__ __forceinline__ unsigned long long pk(float2 a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 upk(unsigned long long r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
    return upk(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)));
    return upk(d);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)));
    return upk(d);
}
__device__ __forceinline__ float2 add2_rz(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)));
    return upk(d);
}
__device__ __forceinline__ float2 add2_rm(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)));
    return upk(d);
}
__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

// ---------------------------------------------------------------- MUFU
__device__ __forceinline__ float sqrt_mufu(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_mufu(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---------------------------------------------------------------- byte <-> float
// 0x4B0000bb as float is 2^23 + bb: one PRMT inserts the byte, one packed
// FADD removes the 2^23 bias (exact), instead of a quarter-rate I2F.
constexpr float kMagic = 8388608.0f;  // 2^23
__device__ __forceinline__ float byte_biased(uint32_t w, int k) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7440u | static_cast<uint32_t>(k)));
}
// low bytes of a and b -> bytes 0,1 of the result
__device__ __forceinline__ uint32_t pack_lo2(float a, float b) {
    return __byte_perm(__float_as_uint(a), __float_as_uint(b), 0x0040u);
}

// ---------------------------------------------------------------- uint8 path (0..255 domain)
// With r, g, b the raw byte values and S = r + g + b (homogeneity lets the
// whole model run in the 0..255 domain, so gray*255 comes out directly):
//   W   = sqrt(r^2 + g^2 + b^2)                  (= sqrt(3) * white, Eq. 1)
//   RGq = sqrt(cr r^2 + g^2), cr = br/(1-br)     (= RG / sqrt(1-br), Eq. 3)
//   A   = c1 r RGq + (g+b) W                     (= sqrt(3) * S * warm, Eq. 4)
//   B   = b (sqrt(3)(r+g) + W)                   (= sqrt(3) * S * cool, Eqs. 2, 5)
//   T   = A^2 + c3 B^2, c3 = (1-bk)/bk
//   gray255 = c4 * sqrt(T) / S = T * rsqrt(T S^2 / c4^2 + tiny),  c4 = sqrt(bk/3)   (Eq. 6)
// 3 MUFU (2 sqrt, 1 rsqrt) and no divide per pixel; the tiny bias makes black
// (T = S = 0) come out 0 instead of 0*inf. gray <= max(r,g,b) <= 255, so no
// clamp is needed. The final FMA T*y + 2^23 rounds to nearest: its low byte is
// round(gray255), which equals the reference's floor(v + 0.5) (codec.py:22-25)
// except when the exact product T*y is a half-integer (an exact tie).
// The operation order minimises distinct register operands per packed op:
// on sm_100a the u8 kernel is bound by register-file reads / FMA-pipe issue,
// not by HBM (scripts/ubench_mix.cu, scripts/tune_u8.cu).
struct U8Consts {
    float cr, c1, sqrt3, c3, inv_c4sq;
};

inline U8Consts make_u8_consts(double beta_r, double beta_k) {
    // derive in double, round once to fp32
    const double br = beta_r, bk = beta_k;
    U8Consts k;
    k.cr = static_cast<float>(br / (1.0 - br));
    k.c1 = static_cast<float>(1.7320508075688772 * std::sqrt(1.0 - br));
    k.sqrt3 = 1.7320508075688772f;
    k.c3 = static_cast<float>((1.0 - bk) / bk);
    k.inv_c4sq = static_cast<float>(3.0 / bk);  // 1 / c4^2, c4 = sqrt(bk / 3)
    return k;
}

// Unclamped gray of two non-negative pixels of ANY scale (homogeneous of
// degree 1), same operation sequence as decolor255_x2 minus the rounding:
// used on raw HDR radiance, where only relative accuracy (~2e-7) matters.
__device__ __forceinline__ float2 decolor_fast_x2(float2 R, float2 G, float2 B, const U8Consts& k) {
    float2 R2 = mul2(R, R);
    float2 G2 = mul2(G, G);
    float2 RG2 = add2(R2, G2);
    float2 q = fma2(B, B, RG2);
    float2 p = fma2(R2, bc2(k.cr), G2);
    float2 Rc1 = mul2(R, bc2(k.c1));
    float2 W = make_float2(sqrt_mufu(q.x), sqrt_mufu(q.y));
    float2 RGq = make_float2(sqrt_mufu(p.x), sqrt_mufu(p.y));
    float2 RG = add2(R, G);
    float2 S = add2(RG, B);
    float2 GB = add2(G, B);
    float2 t1 = mul2(GB, W);
    float2 A = fma2(Rc1, RGq, t1);
    float2 u = fma2(RG, bc2(k.sqrt3), W);
    float2 Bp = mul2(B, u);
    float2 B2 = mul2(Bp, Bp);
    float2 A2 = mul2(A, A);
    float2 T = fma2(B2, bc2(k.c3), A2);
    float2 S2 = mul2(S, S);
    float2 S2k = mul2(S2, bc2(k.inv_c4sq));
    float2 X = fma2(T, S2k, bc2(1e-36f));
    float2 y = make_float2(rsqrt_mufu(X.x), rsqrt_mufu(X.y));
    return mul2(T, y);
}

// Scalar twin of decolor_fast_x2 (identical per-lane operation sequence).
__device__ __forceinline__ float decolor_fast_x1(float r, float g, float b, const U8Consts& k) {
    float R2 = __fmul_rn(r, r);
    float G2 = __fmul_rn(g, g);
    float RG2 = __fadd_rn(R2, G2);
    float q = __fmaf_rn(b, b, RG2);
    float p = __fmaf_rn(R2, k.cr, G2);
    float Rc1 = __fmul_rn(r, k.c1);
    float W = sqrt_mufu(q);
    float RGq = sqrt_mufu(p);
    float RG = __fadd_rn(r, g);
    float S = __fadd_rn(RG, b);
    float GB = __fadd_rn(g, b);
    float t1 = __fmul_rn(GB, W);
    float A = __fmaf_rn(Rc1, RGq, t1);
    float u = __fmaf_rn(RG, k.sqrt3, W);
    float Bp = __fmul_rn(b, u);
    float B2 = __fmul_rn(Bp, Bp);
    float A2 = __fmul_rn(A, A);
    float T = __fmaf_rn(B2, k.c3, A2);
    float S2 = __fmul_rn(S, S);
    float S2k = __fmul_rn(S2, k.inv_c4sq);
    float X = __fmaf_rn(T, S2k, 1e-36f);
    return __fmul_rn(T, rsqrt_mufu(X));
}

// Two pixels per packed lane pair. Returns 2^23 + round(gray255) per lane
// (the low byte is the uint8 gray).
__device__ __forceinline__ float2 decolor255_x2(float2 R, float2 G, float2 B, const U8Consts& k) {
    float2 R2 = mul2(R, R);
    float2 G2 = mul2(G, G);
    float2 RG2 = add2(R2, G2);
    float2 q = fma2(B, B, RG2);                 // r^2 + g^2 + b^2
    float2 p = fma2(R2, bc2(k.cr), G2);         // cr r^2 + g^2
    float2 Rc1 = mul2(R, bc2(k.c1));
    float2 W = make_float2(sqrt_mufu(q.x), sqrt_mufu(q.y));
    float2 RGq = make_float2(sqrt_mufu(p.x), sqrt_mufu(p.y));
    float2 RG = add2(R, G);
    float2 S = add2(RG, B);
    float2 GB = add2(G, B);
    float2 t1 = mul2(GB, W);
    float2 A = fma2(Rc1, RGq, t1);              // sqrt(3) S warm
    float2 u = fma2(RG, bc2(k.sqrt3), W);
    float2 Bp = mul2(B, u);                     // sqrt(3) S cool
    float2 B2 = mul2(Bp, Bp);
    float2 A2 = mul2(A, A);
    float2 T = fma2(B2, bc2(k.c3), A2);
    float2 S2 = mul2(S, S);
    float2 S2k = mul2(S2, bc2(k.inv_c4sq));
    float2 X = fma2(T, S2k, bc2(1e-30f));
    float2 y = make_float2(rsqrt_mufu(X.x), rsqrt_mufu(X.y));
    return fma2(T, y, bc2(kMagic));
}

// Scalar twin of decolor255_x2 with the identical per-lane operation
// sequence (IEEE rn ops are lane-exact), so tails / unaligned buffers give
// bit-identical bytes to the vector path.
__device__ __forceinline__ uint8_t decolor255_x1(float r, float g, float b, const U8Consts& k) {
    float R2 = __fmul_rn(r, r);
    float G2 = __fmul_rn(g, g);
    float RG2 = __fadd_rn(R2, G2);
    float q = __fmaf_rn(b, b, RG2);
    float p = __fmaf_rn(R2, k.cr, G2);
    float Rc1 = __fmul_rn(r, k.c1);
    float W = sqrt_mufu(q);
    float RGq = sqrt_mufu(p);
    float RG = __fadd_rn(r, g);
    float S = __fadd_rn(RG, b);
    float GB = __fadd_rn(g, b);
    float t1 = __fmul_rn(GB, W);
    float A = __fmaf_rn(Rc1, RGq, t1);
    float u = __fmaf_rn(RG, k.sqrt3, W);
    float Bp = __fmul_rn(b, u);
    float B2 = __fmul_rn(Bp, Bp);
    float A2 = __fmul_rn(A, A);
    float T = __fmaf_rn(B2, k.c3, A2);
    float S2 = __fmul_rn(S, S);
    float S2k = __fmul_rn(S2, k.inv_c4sq);
    float X = __fmaf_rn(T, S2k, 1e-30f);
    float y = rsqrt_mufu(X);
    return static_cast<uint8_t>(__float_as_uint(__fmaf_rn(T, y, kMagic)) & 0xFFu);
}

// Exact-rounding variants: the final FMA adds 256.5 instead of 2^23, so the
// float's bits hold floor(T*y + 0.5) in bits 15..22 and the next 15 bits of
// its fraction below them (value in [256.5, 512): exponent fixed, ulp 2^-15).
// The integer part is the fast byte; the fraction tells how close T*y came to
// a rounding boundary (csrc/wg_u8exact.cu settles those against the fp64
// reference). Same FMA-pipe work as decolor255_x2.
constexpr float kMagicFrac = 256.5f;
__device__ __forceinline__ float2 decolor255_bits_x2(float2 R, float2 G, float2 B, const U8Consts& k) {
    float2 R2 = mul2(R, R);
    float2 G2 = mul2(G, G);
    float2 RG2 = add2(R2, G2);
    float2 q = fma2(B, B, RG2);
    float2 p = fma2(R2, bc2(k.cr), G2);
    float2 Rc1 = mul2(R, bc2(k.c1));
    float2 W = make_float2(sqrt_mufu(q.x), sqrt_mufu(q.y));
    float2 RGq = make_float2(sqrt_mufu(p.x), sqrt_mufu(p.y));
    float2 RG = add2(R, G);
    float2 S = add2(RG, B);
    float2 GB = add2(G, B);
    float2 t1 = mul2(GB, W);
    float2 A = fma2(Rc1, RGq, t1);
    float2 u = fma2(RG, bc2(k.sqrt3), W);
    float2 Bp = mul2(B, u);
    float2 B2 = mul2(Bp, Bp);
    float2 A2 = mul2(A, A);
    float2 T = fma2(B2, bc2(k.c3), A2);
    float2 S2 = mul2(S, S);
    float2 S2k = mul2(S2, bc2(k.inv_c4sq));
    float2 X = fma2(T, S2k, bc2(1e-30f));
    float2 y = make_float2(rsqrt_mufu(X.x), rsqrt_mufu(X.y));
    return fma2(T, y, bc2(kMagicFrac));
}
// The model's T and S of a pixel pair, T as in decolor255_bits_x2 and S
// returned biased by 2^23 (Sb = (R + G) + (B + 2^23), exact: its float bits
// are 0x4B000000 + S), for the square-domain routes that never take the
// final root: (gray255)^2 = T c4^2 / S^2 (csrc/wg_tone.cu OpToneSqU8).
__device__ __forceinline__ void decolor255_T_x2(float2 R, float2 G, float2 B, float2 Bb, const U8Consts& k,
                                                float2& T, float2& Sb) {
    float2 R2 = mul2(R, R);
    float2 G2 = mul2(G, G);
    float2 RG2 = add2(R2, G2);
    float2 q = fma2(B, B, RG2);
    float2 p = fma2(R2, bc2(k.cr), G2);
    float2 Rc1 = mul2(R, bc2(k.c1));
    float2 W = make_float2(sqrt_mufu(q.x), sqrt_mufu(q.y));
    float2 RGq = make_float2(sqrt_mufu(p.x), sqrt_mufu(p.y));
    float2 RG = add2(R, G);
    Sb = add2(RG, Bb);
    float2 GB = add2(G, B);
    float2 t1 = mul2(GB, W);
    float2 A = fma2(Rc1, RGq, t1);
    float2 u = fma2(RG, bc2(k.sqrt3), W);
    float2 Bp = mul2(B, u);
    float2 B2 = mul2(Bp, Bp);
    float2 A2 = mul2(A, A);
    T = fma2(B2, bc2(k.c3), A2);
}
__device__ __forceinline__ void decolor255_T_x1(float r, float g, float b, const U8Consts& k, float& T, float& S) {
    float R2 = __fmul_rn(r, r);
    float G2 = __fmul_rn(g, g);
    float RG2 = __fadd_rn(R2, G2);
    float q = __fmaf_rn(b, b, RG2);
    float p = __fmaf_rn(R2, k.cr, G2);
    float Rc1 = __fmul_rn(r, k.c1);
    float W = sqrt_mufu(q);
    float RGq = sqrt_mufu(p);
    float RG = __fadd_rn(r, g);
    S = __fadd_rn(RG, b);
    float GB = __fadd_rn(g, b);
    float t1 = __fmul_rn(GB, W);
    float A = __fmaf_rn(Rc1, RGq, t1);
    float u = __fmaf_rn(RG, k.sqrt3, W);
    float Bp = __fmul_rn(b, u);
    float B2 = __fmul_rn(Bp, Bp);
    float A2 = __fmul_rn(A, A);
    T = __fmaf_rn(B2, k.c3, A2);
}
// scalar twin (lane-exact: identical IEEE rn operation sequence)
__device__ __forceinline__ uint32_t decolor255_bits_x1(float r, float g, float b, const U8Consts& k) {
    float R2 = __fmul_rn(r, r);
    float G2 = __fmul_rn(g, g);
    float RG2 = __fadd_rn(R2, G2);
    float q = __fmaf_rn(b, b, RG2);
    float p = __fmaf_rn(R2, k.cr, G2);
    float Rc1 = __fmul_rn(r, k.c1);
    float W = sqrt_mufu(q);
    float RGq = sqrt_mufu(p);
    float RG = __fadd_rn(r, g);
    float S = __fadd_rn(RG, b);
    float GB = __fadd_rn(g, b);
    float t1 = __fmul_rn(GB, W);
    float A = __fmaf_rn(Rc1, RGq, t1);
    float u = __fmaf_rn(RG, k.sqrt3, W);
    float Bp = __fmul_rn(b, u);
    float B2 = __fmul_rn(Bp, Bp);
    float A2 = __fmul_rn(A, A);
    float T = __fmaf_rn(B2, k.c3, A2);
    float S2 = __fmul_rn(S, S);
    float S2k = __fmul_rn(S2, k.inv_c4sq);
    float X = __fmaf_rn(T, S2k, 1e-30f);
    return __float_as_uint(__fmaf_rn(T, rsqrt_mufu(X), kMagicFrac));
}
// byte and boundary distance (in 2^-15 units) of decolor255_bits_* results
__device__ __forceinline__ uint32_t bits_byte(uint32_t bits) { return (bits >> 15) & 0xFFu; }
__device__ __forceinline__ bool bits_near_tie(uint32_t bits, uint32_t margin) {
    return ((bits + margin) & 0x7FFFu) <= 2u * margin;
}

// 1 if any of the 16 results lies within `margin` of a rounding boundary:
// ((bits + margin) << 17) < (2 margin + 1) << 17, chained through one
// predicate (a shift-add and an OR-compare per pixel)
__device__ __forceinline__ uint32_t any_near_tie16(const uint32_t (&b)[16], uint32_t madd, uint32_t mlim) {
    uint32_t r;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
        "mad.lo.u32 t, %1, 131072, %17;\n\tsetp.lt.u32 p, t, %18;\n\t"
        "mad.lo.u32 t, %2, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %3, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %4, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %5, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %6, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %7, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %8, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %9, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %10, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %11, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %12, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %13, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %14, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %15, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "mad.lo.u32 t, %16, 131072, %17;\n\tsetp.lt.or.u32 p, t, %18, p;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r)
        : "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]), "r"(b[6]), "r"(b[7]), "r"(b[8]),
          "r"(b[9]), "r"(b[10]), "r"(b[11]), "r"(b[12]), "r"(b[13]), "r"(b[14]), "r"(b[15]), "r"(madd), "r"(mlim));
    return r;
}

// Exact bytes of the near-tie colours (csrc/wg_u8exact.cu): an open-addressing
// table of (rgb << 8 | byte) entries, 0xFFFFFFFF = empty (white is never a
// near-tie colour). A pixel whose fast result lies within `margin` of a
// rounding boundary looks its colour up; absent means the fast byte is exact.
struct U8Exact {
    const uint32_t* tab;
    uint32_t mask;    // slots - 1 (power of two)
    uint32_t margin;  // in 2^-15 units
    uint32_t err;     // max |f_fast - f_exact| over all colours, 2^-15 units, rounded up
    uint32_t err_sq;  // max |bits(u_fast) - bits(F(v_exact))| over all colours (square-domain route)
};
__host__ __device__ __forceinline__ uint32_t u8exact_slot(uint32_t key, uint32_t mask) {
    return (key * 2654435761u >> 8) & mask;
}
static __device__ __noinline__ uint32_t u8exact_lookup(U8Exact t, uint32_t key, uint32_t fast) {
    for (uint32_t s = u8exact_slot(key, t.mask);; s = (s + 1) & t.mask) {
        const uint32_t e = __ldg(t.tab + s);
        if (e == 0xFFFFFFFFu) return fast;
        if ((e >> 8) == key) return e & 0xFFu;
    }
}

// ---------------------------------------------------------------- fp32 path (accurate)
struct AccConsts {
    float br, omr, bk, omk;
};
inline AccConsts make_acc_consts(float beta_r, float beta_k) {
    AccConsts k;
    k.br = beta_r;
    k.omr = static_cast<float>(1.0 - static_cast<double>(beta_r));
    k.bk = beta_k;
    k.omk = static_cast<float>(1.0 - static_cast<double>(beta_k));
    return k;
}

// Unclamped gray of an fp32 pixel (any non-negative scale: used on raw HDR
// radiance too, where homogeneity makes the clamp meaningless).
__device__ __forceinline__ float decolor_acc_raw(float r, float g, float b, const AccConsts& k) {
    float q = __fmaf_rn(r, r, __fmaf_rn(g, g, __fmul_rn(b, b)));
    float white = __fsqrt_rn(__fmul_rn(q, 0.333333343f));               // Eq. 1
    float s = __fadd_rn(__fadd_rn(r, g), b);
    float inv = s > 0.0f ? __frcp_rn(s) : 0.0f;                        // black: shares 0
    float rg = __fsqrt_rn(__fmaf_rn(k.br, __fmul_rn(r, r), __fmul_rn(k.omr, __fmul_rn(g, g))));
    float warm = __fmaf_rn(__fmul_rn(r, inv), __fsub_rn(rg, white), white);   // Eq. 4
    float cool = __fmaf_rn(__fmul_rn(b, inv), __fsub_rn(white, b), b);       // Eq. 5
    return __fsqrt_rn(
        __fmaf_rn(__fmul_rn(k.bk, warm), warm, __fmul_rn(k.omk, __fmul_rn(cool, cool))));  // Eq. 6
}
__device__ __forceinline__ float decolor_acc(float r, float g, float b, const AccConsts& k) {
    return fminf(fmaxf(decolor_acc_raw(r, g, b, k), 0.0f), 1.0f);
}

// quantize_u8 (codec.py:22-25) of a [0,1] fp32 value: floor(clip(v)*255 + 0.5)
__device__ __forceinline__ uint8_t quantize_f32(float v) {
    v = fminf(fmaxf(v, 0.0f), 1.0f);
    return static_cast<uint8_t>(__float2uint_rd(__fmaf_rn(v, 255.0f, 0.5f)));
}

// ---------------------------------------------------------------- global sigmoid, fp32 (tanh form)
// apply_sigmoid (tonemap.py:72-83) computes (y - lo)/(hi - lo) with
// y = logistic(k(x - m)); that difference cancels catastrophically in fp32
// for small slopes. The algebraically equal tanh form
//   (tanh(k(x-m)/2) + tanh(km/2)) / (tanh(k(1-m)/2) + tanh(km/2))
// keeps full relative precision; t0/den are evaluated on the device with the
// same operations as the numerator so x = 0 -> 0 and x = 1 -> 1 exactly.
struct SigF {
    float m, hk, t0, den;
};
__device__ __forceinline__ SigF make_sig_f(float midpoint, float slope) {
    SigF s;
    s.m = midpoint;
    s.hk = 0.5f * slope;
    s.t0 = tanhf(__fmul_rn(s.hk, midpoint));
    s.den = __fadd_rn(tanhf(__fmul_rn(s.hk, __fsub_rn(1.0f, midpoint))), s.t0);
    return s;
}
__device__ __forceinline__ float sigmoid_f(float x, const SigF& s) {
    float num = __fadd_rn(tanhf(__fmul_rn(s.hk, __fsub_rn(x, s.m))), s.t0);
    return fminf(fmaxf(__fdiv_rn(num, s.den), 0.0f), 1.0f);
}

// ---------------------------------------------------------------- fp64 path (reference-exact)
__device__ __forceinline__ double clamp01_d(double v) {
    if (v < 0.0) return 0.0;   // _kernels.pyx:23-28
    if (v > 1.0) return 1.0;
    return v;
}
__device__ __forceinline__ double decolor_f64(double r, double g, double b, double br, double bk) {
    double white = __dsqrt_rn(__ddiv_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(r, r), __dmul_rn(g, g)), __dmul_rn(b, b)), 3.0));
    double s = __dadd_rn(__dadd_rn(r, g), b);
    double wr = 0.0, wb = 0.0;
    if (s > 0.0) {
        wr = __ddiv_rn(r, s);
        wb = __ddiv_rn(b, s);
    }
    double redgreen = __dsqrt_rn(__dadd_rn(__dmul_rn(__dmul_rn(br, r), r),
                                           __dmul_rn(__dmul_rn(__dsub_rn(1.0, br), g), g)));
    double warm = __dadd_rn(__dmul_rn(wr, redgreen), __dmul_rn(__dsub_rn(1.0, wr), white));
    double cool = __dadd_rn(__dmul_rn(__dsub_rn(1.0, wb), b), __dmul_rn(wb, white));
    return clamp01_d(__dsqrt_rn(__dadd_rn(__dmul_rn(__dmul_rn(bk, warm), warm),
                                          __dmul_rn(__dmul_rn(__dsub_rn(1.0, bk), cool), cool))));
}

// dequantize_u8 (codec.py:28-29): k / 255.0 correctly rounded for every byte k,
// as one FMA correction of k * fl(1/255) (checked exhaustively against IEEE
// division over k = 0..255).
__device__ __forceinline__ double deq_byte(uint32_t k) {
    // (double)k exactly, as 2^52 + k minus 2^52 (a DADD instead of an XU-pipe I2F.F64)
    const double inv = 1.0 / 255.0, x = __hiloint2double(0x43300000, static_cast<int>(k)) - 4503599627370496.0;
    const double q0 = __dmul_rn(x, inv);
    return __fma_rn(__fma_rn(-q0, 255.0, x), inv, q0);
}

// quantize_u8 (codec.py:22-25) in fp64: floor(clip(v, 0, 1) * 255 + 0.5)
__device__ __forceinline__ uint32_t quantize_d(double v) {
    return static_cast<uint32_t>(__dadd_rn(__dmul_rn(clamp01_d(v), 255.0), 0.5));
}

// apply_sigmoid in fp64, logistic form exactly as tonemap.py:76-83.
struct SigD {
    double m, k, lo, hi;
};
__device__ __forceinline__ SigD make_sig_d(double midpoint, double slope) {
    SigD s;
    s.m = midpoint;
    s.k = slope;
    s.lo = 1.0 / (1.0 + exp(slope * midpoint));
    s.hi = 1.0 / (1.0 + exp(-slope * (1.0 - midpoint)));
    return s;
}
__device__ __forceinline__ double sigmoid_d(double x, const SigD& s) {
    double y = 1.0 / (1.0 + exp(-s.k * (x - s.m)));
    return clamp01_d((y - s.lo) / (s.hi - s.lo));
}

// ---------------------------------------------------------------- counter hash (synthetic inputs)
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}
__host__ __device__ __forceinline__ uint32_t hash3(uint32_t seed, uint32_t image, uint32_t ctr) {
    return mix32(ctr ^ mix32(image ^ mix32(seed ^ 0x9e3779b9U)));
}
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ float u01(uint32_t h) { return (h >> 8) * (1.0f / 16777216.0f); }

}  // namespace wg
