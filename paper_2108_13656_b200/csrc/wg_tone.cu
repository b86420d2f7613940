// wg_tone.cu -- fused decolor + global tone map on uint8 (decolor_tone u8):
// toned = quantize_u8(apply_sigmoid(decolor_image(rgb / 255)))
// (tonemap.py:72-83 after core.py:147-169, codec.py:22-25).
//
// The toned byte is a monotone step function of the gray v: it is the number
// of the 255 thresholds theta_j (least v whose toned byte reaches j) that v
// reaches. The host finds them by bisection over the reference's fp64
// logistic + clip + round-half-up (once per curve, cached per device), and
// the kernels replace exp / tanh / division by one shared-memory "step word"
// per pixel whose byte 3, after adding the pixel's float bits, is the toned
// byte. Two routes:
//  * square domain (default, OpToneSqU8): the step words are indexed by
//    u = (255 v)^2 + 1/8 = T W[S] + 1/8, so the decolor's final rsqrt is never
//    taken (W[S] = c4^2 / S^2 comes from a 768-entry shared table, S = r+g+b
//    being an integer) -- 2 MUFU per pixel instead of 3, the MUFU (XU) pipe
//    being what binds the decolor kernel;
//  * linear (OpToneU8): the decolor kernel's packed MUFU sequence keeping 15
//    fraction bits of f = 256 + (255 v + 0.5) and 4096 bins of 255 v + 0.5;
//    used when a square-domain bin would hold several thresholds, with 8-byte
//    bins and a binary search when even linear bins do (k >~ 100).
// The optional gray output is the rounded gray of the same computation.
// Parity: the north-star bar (+-1 on <= 0.01%; only pixels whose gray lies
// within the fp32 error of a threshold or a rounding boundary can differ).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"
#include "wg_square.cuh"
#include "wg_stream.cuh"

namespace wg {
namespace {

constexpr int kToneBins = 4096;  // bins of x = 255 v + 0.5 over [0, 256), width 1/16
constexpr float kBinAdd = 130816.0f;  // 2^17 - 256: fl_rm(f + kBinAdd) = 2^17 + floor(64 x) / 64


struct ToneTable {
    float2 bins[kToneBins];  // {count of thresholds below the bin (as bits), f-domain threshold inside or NaN}
    float thr[256];          // f-domain thresholds 256 + x_j (j = 1..255 at [j-1]), +inf padded
    int multi;               // any bin with several thresholds (host-side flag)
    int pad[3];
    // exact route only (not staged by OpToneU8): 1 where a neighbouring bin's
    // threshold lies within kEdgeUnits (2^-15 units) of the shared edge
    uint8_t edge[kToneBins];
    // single-threshold curves (multi == 0), staged by OpToneU8<.., false>:
    // step[b] = 2^24 count + (2^24 - L) - (bits of the bin's first f), mod
    // 2^32, L = the low 11 bits of the bin's threshold (2048 without one), so
    // that for f in bin b byte 3 of step[b] + bits(f) is the toned byte: the
    // in-bin offset minus L borrows from (or carries into) bit 24 exactly when
    // f is below (at or above) the threshold -- one LDS.32 and an IADD per
    // pixel, and the pack's PRMT picks byte 3 directly (no shift)
    uint32_t step[kToneBins];
    // square-domain route (OpToneSqU8): u = (255 v)^2 + 1/8 in [2^-3, 2^16),
    // 256 log-spaced bins per octave (bin = float bits >> 15), step words as
    // above with a 15-bit in-bin offset: step[b] = 2^24 count + (2^24 - L) -
    // (bits of the bin's first u), L = the low 15 bits of the bin's threshold
    // (2^15 without one). sq_gray holds the rounding thresholds (j - 1/2)^2 + 1/8
    // of quantize_u8 (the gray byte), sq_multi flags bins with several toned
    // thresholds (then the linear route above runs).
    uint32_t sq_step[kSqBins];
    uint32_t sq_gray[kSqBins];
    int sq_multi;
    int sq_exact_ok;  // every bin's anchor is its only threshold within kSqReach (both tables)
    int sq_pad[2];
};
constexpr uint32_t kEdgeUnits = 64;
constexpr size_t kToneStaged = offsetof(ToneTable, edge);  // bytes OpToneU8 stages

__device__ __forceinline__ uint32_t* step_smem() {
    __shared__ __align__(16) uint32_t t[kToneBins];
    return t;
}
__device__ __forceinline__ ToneTable* tone_smem() {
    __shared__ __align__(16) uint8_t t[kToneStaged];  // bins + thr (+ multi); edge is not staged here
    return reinterpret_cast<ToneTable*>(t);
}

// Linear route (WG_TONE_ROUTE=linear, and curves whose square-domain table
// has a bin with several thresholds). kMulti: the curve's linear table has
// such bins too (steep curves): 8-byte bins and a binary search.
// (r02 A/B on C3, toned only: one register buffer, 4 or 6 CTAs/SM and 10/20
// CTAs per SM all lost to two buffers at 5 CTAs/SM and 40 per SM.)
template <bool kGray, bool kMulti>
struct OpToneU8 {
    static constexpr bool kLdg = true;
    static constexpr bool kPingPong = !kGray && !kMulti;  // the others would spill
    static constexpr int kPx = 16;
    const uint8_t* in;
    uint8_t* toned;
    uint8_t* gray;
    U8Consts k;
    const ToneTable* tab;

    __device__ __forceinline__ void prologue() const {
        if constexpr (kMulti) {
            ToneTable* s = tone_smem();
            const float4* src = reinterpret_cast<const float4*>(tab);
            float4* dst = reinterpret_cast<float4*>(s);
            for (int i = threadIdx.x; i < static_cast<int>(kToneStaged / 16); i += blockDim.x) dst[i] = src[i];
        } else {
            const uint4* src = reinterpret_cast<const uint4*>(tab->step);
            uint4* dst = reinterpret_cast<uint4*>(step_smem());
            for (int i = threadIdx.x; i < kToneBins / 4; i += blockDim.x) dst[i] = src[i];
        }
    }
    // step route: the word whose byte 3 is the toned byte of f. gbits = bits
    // of g = fl_rm(f + (2^17 - 256)) = 2^17 + floor(64 x) / 64 (exact floor:
    // f - 256 = x is exact and the ulp of g is 2^-6), so gbits & 0x3FFC =
    // 4 floor(16 x) is the byte offset of f's bin (bits(f) >> 11) & 4095 --
    // one FADD2.RM per pixel pair and a LOP3 instead of a shift and a mask
    __device__ __forceinline__ uint32_t step_word(uint32_t gbits, uint32_t bits) const {
        const uint32_t e =
            *reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(step_smem()) + (gbits & 0x3FFCu));
        return e + bits;
    }
    // toned byte from the f-domain bits of one pixel (kMulti tables)
    __device__ __forceinline__ uint32_t tone(uint32_t bits) const {
        const ToneTable* s = tone_smem();
        const float f = __uint_as_float(bits);
        const float2 e = s->bins[(bits >> 11) & (kToneBins - 1)];
        if constexpr (kMulti)
            if (e.y != e.y) return count_all(f);  // NaN: several thresholds in this bin
        return __float_as_uint(e.x) + (f >= e.y ? 1u : 0u);
    }
    __device__ __noinline__ uint32_t count_all(float f) const {
        const float* t = tone_smem()->thr;
        uint32_t c = 0;  // number of thresholds <= f (binary search over 256 padded entries)
#pragma unroll
        for (uint32_t step = 128; step; step >>= 1) c += (f >= t[c + step - 1]) ? step : 0;
        return c;
    }
    __device__ __forceinline__ void vec(const uint4 (&v)[3], int64_t px0) const {
        const uint32_t w[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                                v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
        // pack each 4-pixel word as soon as its two pairs are done (keeps registers low)
        uint32_t tw[4], gw[4];
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            uint32_t t[4], q[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = 2 * qd + h;
                float2 ch[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int b0 = 3 * (2 * j) + c, b1 = 3 * (2 * j + 1) + c;
                    ch[c] = add2(make_float2(byte_biased(w[b0 >> 2], b0 & 3), byte_biased(w[b1 >> 2], b1 & 3)),
                                 bc2(-kMagic));
                }
                const float2 f = decolor255_bits_x2(ch[0], ch[1], ch[2], k);
                const uint32_t x = __float_as_uint(f.x), y = __float_as_uint(f.y);
                if constexpr (kMulti) {
                    t[2 * h] = tone(x);
                    t[2 * h + 1] = tone(y);
                } else {
                    const float2 g = add2_rm(f, bc2(kBinAdd));
                    t[2 * h] = step_word(__float_as_uint(g.x), x);
                    t[2 * h + 1] = step_word(__float_as_uint(g.y), y);
                }
                q[2 * h] = x >> 15;
                q[2 * h + 1] = y >> 15;
            }
            constexpr uint32_t sel = kMulti ? 0x0040u : 0x0073u;  // low byte / byte 3 of each word
            tw[qd] = __byte_perm(__byte_perm(t[0], t[1], sel), __byte_perm(t[2], t[3], sel), 0x5410u);
            if constexpr (kGray)
                gw[qd] = __byte_perm(__byte_perm(q[0], q[1], 0x0040u), __byte_perm(q[2], q[3], 0x0040u), 0x5410u);
        }
        st_global_cs_v4(toned + px0, make_uint4(tw[0], tw[1], tw[2], tw[3]));
        if constexpr (kGray) st_global_cs_v4(gray + px0, make_uint4(gw[0], gw[1], gw[2], gw[3]));
    }
    __device__ __forceinline__ void scalar(int64_t p) const {
        const uint32_t bits = decolor255_bits_x1(static_cast<float>(in[3 * p]), static_cast<float>(in[3 * p + 1]),
                                                 static_cast<float>(in[3 * p + 2]), k);
        if constexpr (kMulti)
            toned[p] = static_cast<uint8_t>(tone(bits));
        else
            toned[p] = static_cast<uint8_t>(
                step_word(__float_as_uint(__fadd_rd(__uint_as_float(bits), kBinAdd)), bits) >> 24);
        if constexpr (kGray) gray[p] = static_cast<uint8_t>(bits >> 15);
    }
};

// Square-domain route: toned (and gray) bytes without the final root.
// (gray255)^2 = c4^2 T / S^2 (decolor255_T_x2), S = r + g + b an integer in
// [0, 765], so 1 / S^2 is a shared-memory table W[S] (indexed by the bits of
// the 2^23-biased S, one LEA) instead of the MUFU rsqrt of the linear route:
// u = T W[S] + 1/8 = (255 v)^2 + 1/8 (one FFMA per pixel), and the toned byte
// is the number of the curve's thresholds U_j = (255 theta_j)^2 + 1/8 that u
// reaches, read from log-spaced step words (SHF + LOP3 for the bin address,
// LDS, IADD; byte 3). Two MUFU per pixel instead of three: the decolor
// kernel is bound by the MUFU (XU) pipe at 3 per pixel (16 per clock per SM),
// the tone map's extra lookup work then fits in the issue slots the XU left.
// Parity: the north-star bar, as the linear route (u carries ~10 u of
// relative error, half of that in v: only pixels within ~5e-7 relative of a
// threshold can differ).
__device__ __forceinline__ uint32_t* sq_step_smem() {
    __shared__ __align__(16) uint32_t t[kSqBins];
    return t;
}
__device__ __forceinline__ uint32_t* sq_gray_smem() {
    __shared__ __align__(16) uint32_t t[kSqBins];
    return t;
}
__device__ __forceinline__ float* sq_w_smem() {
    __shared__ __align__(16) float t[kSqW];
    return t;
}
template <bool kGray>
struct OpToneSqU8 {
    static constexpr bool kLdg = true;
    static constexpr bool kPingPong = !kGray;
    static constexpr int kPx = 16;
    const uint8_t* in;
    uint8_t* toned;
    uint8_t* gray;
    U8Consts k;
    const ToneTable* tab;
    uint32_t wofs;  // -(0x4B000000 << 2) mod 2^32
    float w[kSqW];  // W[S] = c4^2 / S^2 (host fp64, rounded once), W[0] = 0

    __device__ __forceinline__ void prologue() const {
        const uint4* src = reinterpret_cast<const uint4*>(tab->sq_step);
        uint4* dst = reinterpret_cast<uint4*>(sq_step_smem());
        for (int i = threadIdx.x; i < kSqBins / 4; i += blockDim.x) dst[i] = src[i];
        if constexpr (kGray) {
            const uint4* sg = reinterpret_cast<const uint4*>(tab->sq_gray);
            uint4* dg = reinterpret_cast<uint4*>(sq_gray_smem());
            for (int i = threadIdx.x; i < kSqBins / 4; i += blockDim.x) dg[i] = sg[i];
        }
        float* ws = sq_w_smem();
        for (int i = threadIdx.x; i < kSqW; i += blockDim.x) ws[i] = w[i];
    }
    // W[S] from the bits of Sb = S + 2^23: shared address (bits << 2) + (W - (0x4B000000 << 2)) = W + 4 S
    // (mod 2^32: one LEA)
    // (the bias offset comes in as a kernel parameter, wofs = -(0x4B000000 << 2),
    // so the compiler folds table address + offset into one uniform register and
    // keeps a single LEA per pixel instead of LEA + IADD with an immediate)
    __device__ __forceinline__ uint32_t w_base() const { return smem_addr(sq_w_smem()) + wofs; }
    __device__ __forceinline__ static float w_at(uint32_t sb, uint32_t wb) {
        return __uint_as_float(lds_u32((sb << 2) + wb));
    }
    __device__ __forceinline__ static uint32_t bin_off(uint32_t ub) { return sq_bin_off(ub); }
    __device__ __forceinline__ static uint32_t word(const uint32_t* t, uint32_t off, uint32_t ub) {
        return sq_word(t, off, ub);
    }
    __device__ __forceinline__ void vec(const uint4 (&v)[3], int64_t px0) const {
        const uint32_t w[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                                v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
        uint32_t tw[4], gw[4];
        const uint32_t wb = w_base();
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            uint32_t t[4], q[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = 2 * qd + h;
                float2 cb[3], ch[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int b0 = 3 * (2 * j) + c, b1 = 3 * (2 * j + 1) + c;
                    cb[c] = make_float2(byte_biased(w[b0 >> 2], b0 & 3), byte_biased(w[b1 >> 2], b1 & 3));
                    ch[c] = add2(cb[c], bc2(-kMagic));
                }
                float2 T, Sb;
                decolor255_T_x2(ch[0], ch[1], ch[2], cb[2], k, T, Sb);
                const float2 W = make_float2(w_at(__float_as_uint(Sb.x), wb), w_at(__float_as_uint(Sb.y), wb));
                const float2 u = fma2(T, W, bc2(kSqBias));
                const uint32_t ux = __float_as_uint(u.x), uy = __float_as_uint(u.y);
                const uint32_t ox = bin_off(ux), oy = bin_off(uy);
                t[2 * h] = word(sq_step_smem(), ox, ux);
                t[2 * h + 1] = word(sq_step_smem(), oy, uy);
                if constexpr (kGray) {
                    q[2 * h] = word(sq_gray_smem(), ox, ux);
                    q[2 * h + 1] = word(sq_gray_smem(), oy, uy);
                }
            }
            tw[qd] = __byte_perm(__byte_perm(t[0], t[1], 0x0073u), __byte_perm(t[2], t[3], 0x0073u), 0x5410u);
            if constexpr (kGray)
                gw[qd] = __byte_perm(__byte_perm(q[0], q[1], 0x0073u), __byte_perm(q[2], q[3], 0x0073u), 0x5410u);
        }
        st_global_cs_v4(toned + px0, make_uint4(tw[0], tw[1], tw[2], tw[3]));
        if constexpr (kGray) st_global_cs_v4(gray + px0, make_uint4(gw[0], gw[1], gw[2], gw[3]));
    }
    __device__ __forceinline__ void scalar(int64_t p) const {
        float T, S;
        decolor255_T_x1(static_cast<float>(in[3 * p]), static_cast<float>(in[3 * p + 1]),
                        static_cast<float>(in[3 * p + 2]), k, T, S);
        const uint32_t ub = __float_as_uint(__fmaf_rn(T, sq_w_smem()[static_cast<int>(S)], kSqBias));
        const uint32_t o = bin_off(ub);
        toned[p] = static_cast<uint8_t>(word(sq_step_smem(), o, ub) >> 24);
        if constexpr (kGray) gray[p] = static_cast<uint8_t>(word(sq_gray_smem(), o, ub) >> 24);
    }
};

// ---- host: the reference's curve and its thresholds
struct HostSig {
    double m, k, lo, hi;
};
HostSig host_sig(double m, double k) {
    // tonemap.py:76-80
    return {m, k, 1.0 / (1.0 + std::exp(k * m)), 1.0 / (1.0 + std::exp(-k * (1.0 - m)))};
}
int host_toned(const HostSig& s, double v) {
    const double y = 1.0 / (1.0 + std::exp(-s.k * (v - s.m)));
    double o = (y - s.lo) / (s.hi - s.lo);
    o = o < 0.0 ? 0.0 : (o > 1.0 ? 1.0 : o);
    return static_cast<int>(std::floor(o * 255.0 + 0.5));
}

}  // namespace

// Anchored step words over sorted float thresholds uf[0..n) for nbins bins of
// `shift` low bits starting at float bits `lo_bits` (csrc/wg_square.cuh). The
// anchor A of bin b is its threshold, else the one within `reach` units of
// the bin, else a virtual one 2^23 units below it; step[b] = (c0 << 24) +
// 2^24 - bits(A), c0 = #{thresholds below A} (for the virtual anchor: the
// count below the bin, minus one). Byte 3 of step[b] + bits(u) is the number
// of thresholds <= u for every u of the bin, and its low 24 bits are bits(u) -
// bits(A) mod 2^24, the exact route's distance to the nearest threshold.
// Returns kSqMulti if a bin holds two thresholds (the route cannot decide
// it), kSqCrowded if a bin has two thresholds within reach (the exact
// route's distance test would miss one).
int sq_step_words(const float* uf, int n, uint32_t* step, int nbins, uint32_t lo_bits, int shift, uint32_t reach) {
    const auto bits_of = [&](int j) {
        uint32_t x;
        std::memcpy(&x, &uf[j], 4);
        return x;
    };
    int flags = 0;
    int below = 0, near_lo = 0;
    for (int b = 0; b < nbins; ++b) {
        const uint32_t first = lo_bits + (static_cast<uint32_t>(b) << shift), next = first + (1u << shift);
        while (below < n && bits_of(below) < first) ++below;
        while (near_lo < n && bits_of(near_lo) + reach < first) ++near_lo;  // first threshold >= first - reach
        int inside = below;
        while (inside < n && bits_of(inside) < next) ++inside;
        int near_hi = inside;
        while (near_hi < n && bits_of(near_hi) < next + reach) ++near_hi;
        if (inside - below > 1) flags |= kSqMulti;
        if (near_hi - near_lo > 1) flags |= kSqCrowded;
        int a = -1;  // anchor index
        if (inside > below) {
            a = below;
        } else if (near_hi > near_lo) {  // the nearest threshold within reach
            a = near_lo;
            for (int j = near_lo + 1; j < near_hi; ++j) {
                const uint32_t dj = bits_of(j) < first ? first - bits_of(j) : bits_of(j) - next + 1;
                const uint32_t da = bits_of(a) < first ? first - bits_of(a) : bits_of(a) - next + 1;
                if (dj < da) a = j;
            }
        }
        if (a >= 0)
            step[b] = (static_cast<uint32_t>(a) << 24) + 0x1000000u - bits_of(a);
        else  // virtual anchor first - 2^23: byte 3 = (below - 1) + 1
            step[b] = (static_cast<uint32_t>(below - 1) << 24) + 0x1000000u - (first - 0x800000u);
    }
    return flags;
}

void sq_weights(double c4sq, float* w) {
    w[0] = 0.0f;  // black: T = 0
    for (int i = 1; i < kSqW; ++i) w[i] = static_cast<float>(c4sq / (static_cast<double>(i) * i));
}

namespace {

// least double v in [0, 1] with pred(v) true, pred monotone (false ... true);
// non-negative doubles order like their bits
template <class Pred>
double least_double(Pred pred) {
    double v0 = 0.0, v1 = 1.0;
    uint64_t lo, hi;
    std::memcpy(&lo, &v0, 8);
    std::memcpy(&hi, &v1, 8);
    if (pred(0.0)) return 0.0;
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        double mv;
        std::memcpy(&mv, &mid, 8);
        (pred(mv) ? hi : lo) = mid;
    }
    double th;
    std::memcpy(&th, &hi, 8);
    return th;
}

void build_tone_table(double m, double k, ToneTable* t) {
    const HostSig s = host_sig(m, k);
    t->multi = 0;
    float xf[255];  // f-domain thresholds
    float uf[255];  // square-domain thresholds (255 theta)^2 + 1/8
    for (int j = 1; j <= 255; ++j) {
        const double th = least_double([&](double v) { return host_toned(s, v) >= j; });  // theta_j
        xf[j - 1] = static_cast<float>(256.0 + (th * 255.0 + 0.5));  // f = 256 + 255 v + 0.5
        uf[j - 1] = static_cast<float>((th * 255.0) * (th * 255.0) + 0.125);
    }
    const int tf = sq_step_words(uf, 255, t->sq_step, kSqBins, kSqLoBits, 15, kSqReach);
    // quantize_u8's boundaries g_j (least v with floor(v * 255 + 0.5) >= j, by bisection
    // over the reference's fp64 expression) through the same map u = (255 v)^2 + 1/8
    float gf[255];
    for (int j = 1; j <= 255; ++j) {
        const double g = least_double([&](double v) { return std::floor(v * 255.0 + 0.5) >= j; });
        gf[j - 1] = static_cast<float>((g * 255.0) * (g * 255.0) + 0.125);
    }
    const int gfl = sq_step_words(gf, 255, t->sq_gray, kSqBins, kSqLoBits, 15, kSqReach);
    t->sq_multi = (tf & kSqMulti) ? 1 : 0;
    t->sq_exact_ok = ((tf | gfl) & (kSqMulti | kSqCrowded)) ? 0 : 1;
    for (int j = 0; j < 256; ++j) t->thr[j] = j < 255 ? xf[j] : INFINITY;
    int below = 0;
    for (int b = 0; b < kToneBins; ++b) {
        const double lo_f = 256.0 + b / 16.0, hi_f = 256.0 + (b + 1) / 16.0;
        while (below < 255 && xf[below] < lo_f) ++below;
        int inside = below;
        while (inside < 255 && xf[inside] < hi_f) ++inside;
        uint32_t cnt = static_cast<uint32_t>(below);
        float tin = INFINITY;
        if (inside - below == 1) tin = xf[below];
        if (inside - below > 1) {
            tin = NAN;
            t->multi = 1;
        }
        float base;
        std::memcpy(&base, &cnt, 4);
        t->bins[b] = make_float2(base, tin);
        uint32_t L = 0x800u;  // no threshold in the bin: never reached
        if (inside - below == 1) {
            uint32_t tb;
            std::memcpy(&tb, &xf[below], 4);
            L = tb & 0x7FFu;  // 0: the whole bin counts it
        }
        t->step[b] = (cnt << 24) + (0x1000000u - L) - (0x43800000u + (static_cast<uint32_t>(b) << 11));  // bits(256 + b/16)
    }
    std::memset(t->edge, 0, sizeof(t->edge));
    for (int j = 0; j < 255; ++j) {
        uint32_t bits;
        std::memcpy(&bits, &xf[j], 4);
        const int b = static_cast<int>((bits >> 11) & (kToneBins - 1));
        const uint32_t low = bits & 0x7FFu;
        if (low < kEdgeUnits && b > 0) t->edge[b - 1] = 1;
        if (0x800u - low <= kEdgeUnits && b + 1 < kToneBins) t->edge[b + 1] = 1;
    }
}

struct Entry {
    bool used = false;
    double m = 0, k = 0;
    ToneTable* dev = nullptr;
    bool multi = false;
    bool sq_multi = false;
    bool sq_exact_ok = false;
};
constexpr int kCache = 8;
Entry g_cache[kMaxDevices][kCache];
int g_next[kMaxDevices];
std::mutex g_mu;

// The table stays valid while *hold is locked: the caller enqueues its kernel
// before releasing it, so an eviction by another thread (cudaFree, which waits
// for the device's queued work) cannot free a table a pending launch uses.
int tone_table(double m, double k, const ToneTable** out, bool* multi, std::unique_lock<std::mutex>* hold,
               bool* sq_multi = nullptr, bool* sq_exact_ok = nullptr) {
    int device = 0;
    cudaGetDevice(&device);
    if (device < 0 || device >= kMaxDevices) return set_error(WG_ENODEV, "device ordinal out of range");
    *hold = std::unique_lock<std::mutex>(g_mu);
    for (Entry& e : g_cache[device])
        if (e.used && e.m == m && e.k == k) {
            *out = e.dev;
            *multi = e.multi;
            if (sq_multi) *sq_multi = e.sq_multi;
            if (sq_exact_ok) *sq_exact_ok = e.sq_exact_ok;
            return WG_OK;
        }
    static ToneTable host;  // under g_mu
    build_tone_table(m, k, &host);
    ToneTable* d = nullptr;
    cudaError_t err = cudaMalloc(&d, sizeof(ToneTable));
    if (err == cudaSuccess) err = cudaMemcpy(d, &host, sizeof(ToneTable), cudaMemcpyHostToDevice);
    if (err != cudaSuccess) {
        if (d) cudaFree(d);
        return set_error(static_cast<int>(err), "tone table: %s", cudaGetErrorString(err));
    }
    Entry& slot = g_cache[device][g_next[device]];
    g_next[device] = (g_next[device] + 1) % kCache;
    if (slot.used) cudaFree(slot.dev);
    slot = {true, m, k, d, host.multi != 0, host.sq_multi != 0, host.sq_exact_ok != 0};
    *out = d;
    *multi = host.multi != 0;
    if (sq_multi) *sq_multi = host.sq_multi != 0;
    if (sq_exact_ok) *sq_exact_ok = host.sq_exact_ok != 0;
    return WG_OK;
}

// ---------------------------------------------------------------- colour output
// tonemap_image(mode="global")'s rgb_out on uint8 (tonemap.py:172-216):
// rgb_out_c = quantize_u8(clip(c * l_out / max(l_in, 1e-6))), 0 where l_in == 0;
// toned = quantize_u8(l_out), gray = quantize_u8(l_in).
//
// The ratio l_out / l_in amplifies fp32 error into the rounding of every
// channel, so bit-identity needs the reference's fp64 chain wherever an output
// byte is in doubt -- and only there. The fast kernel evaluates the chain in
// packed fp32 (two pixels per f32x2 op) on MUFU approximations, together with
// a per-pixel bound `rel` on the relative error of the output values. Each
// byte is settled by two FFMAs, lo = RN(v (1 - rel) + 2^23) and
// hi = RN(v (1 + rel) + 2^23): if they agree, every value within the bound
// rounds to the same byte (the low byte of lo). A pixel with any
// disagreement (sum of hi - lo over its outputs != 0) is queued in shared
// memory, one queue per warp (pixel index; lanes append at a shuffle prefix
// sum; the queue holds a whole warp-tile on top of the drain threshold, so it
// cannot overflow), and the warp drains it through the fp64 chain
// (tone_rgb_px) once 32 are waiting -- all lanes busy, and no block barrier
// anywhere in the loop. ~1% of pixels take the fp64 route at the default
// curve. Bit-identical to the reference by construction.
//
// fp32 chain, in the 0..255 domain (decolor is homogeneous of degree 1) and
// pre-scaled by sqrt(3) (white' = sqrt(3) white etc.), with bytes R, G, B:
//   white' = sqrt(R^2+G^2+B^2), rg' = sqrt(3 br R^2 + 3 (1-br) G^2),
//   W' = R rg' + (G+B) white', C' = B (sqrt(3) (R+G) + white'), s = R+G+B
//   Qn = (bk/3) W'^2 + ((1-bk)/3) C'^2, q = rsqrt(Qn s^2),
//   L = 255 l_in = Qn q = sqrt(Qn)/s, 1/L = s^2 q   (one MUFU for both)
//   (warm = W'/(sqrt(3) s), cool = C'/(sqrt(3) s))
// (black: Qn gets +1e-30 and s is floored at 1, so L = 1e-15 and every
// output value is 0 without a branch; l_in == 0 only for black with betas in
// (0.5, 1)). Logistic difference in product form (no cancellation at small k):
//   N(x) = (sig(k(x-m)) - sig(-km)) / (sig(k(1-m)) - sig(-km))
//        = sig(t) (1 - e^{-kx}) / (sig(k(1-m)) (1 - e^{-k})),  t = k(x-m)
//   e^{-kx} = 2^y, y = -kx log2(e); e^{-t} = 2^y e^{km} (one ex2) for k <= 80,
//   2^{y + km log2 e} (a second ex2) beyond; 1 - 2^y by a degree-6 series in
//   y for kx < 1/4 (evaluated only by warps that hold such a pixel).
// Error bound (u = 2^-24; MUFU ex2/rsqrt/sqrt/rcp <= 2.45 u measured
// exhaustively on the B200 by scripts/mufu_error.cu, budgeted at e = 3 u each;
// first-order sums along the chain, each budget rounded up):
//   white' 3u, rg' 4.5u, W' 5.5u, C' 5u, Qn 14u (bytes, R^2+G^2+B^2 and s^2
//   exact); L = Qn rsqrt(Qn s^2) and 1/L: Qn enters as delta/2 -> 11.5 u
//   (budget relL = 13 u);
//   rel(e^{-t}) <= 5u + kx (relL + 2u)            (one-ex2 form)
//              <= 3u + 2 km u + kx (relL + 3u)    (two-ex2 form)
//   rel(1 - e^{-kx}) <= 3.52 e + relL + 3u (1 - E, kx >= 1/4) or
//     relL + 9u (series) -> 28 u;
//   rel(N) <= omS rel(e^{-t}) + 4u (1 + e^{-t}, rcp) + 28u + 3u (products,
//     cn255) + ref, omS = 1 - sig(t) (the logistic's own conditioning), ref
//     the reference's fp64 error (1e-13 + 4e-16 / D + 1e-15 k, D = hi - lo);
//   rgb v_c = R N 255 / L: rel(N) + rel(1/L) + 2u (+2u for the scale
//     constants) -> relRgb 17 u, + the reference's absolute y - lo error
//     folded in relative form (v >= 0.4 where it matters: 1.1e-10 / (0.4 D));
//     the toned value 255 N shares the rgb scales (a wider margin than it
//     needs).
// A wide margin is never wrong, only slower (more pairs take the fp64 chain).
// Curves with k < 1e-3 or k > 1e4 run the fp64 kernel for every pixel.
struct ToneRgbF {
    float br3, br13, bk3, bk13;  // 3 br, 3 (1-br), bk/3, (1-bk)/3
    float nak;      // -k log2(e) / 255: y = L nak, e^{-kx} = 2^y
    float ekm;      // e^{km} (one-ex2 form)
    float tc;       // k m log2(e): e^{-t} = 2^{y + tc} (two-ex2 form)
    float ycut;     // -0.25 log2(e): the series below |y| < |ycut| (kx < 1/4)
    float cn255;    // 255 / (sig(k(1-m)) (1 - e^{-k}))
    float cA, cC, cD;  // rel(N) <= omS (L cA + cC) + cD
    float relRgb;      // rel(v_rgb) = rel(N) + relRgb (toned shares it when rgb is produced)
    float relT;        // rel(v_toned) = rel(N) + relT when only toned / gray are produced
    float glo, ghi;    // gray scales 1 -/+ rel(L)
};

__device__ __forceinline__ float ex2_mufu(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_mufu(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 sqrt2_mufu(float2 x) { return make_float2(sqrt_mufu(x.x), sqrt_mufu(x.y)); }
__device__ __forceinline__ float2 rsqrt2_mufu(float2 x) { return make_float2(rsqrt_mufu(x.x), rsqrt_mufu(x.y)); }
__device__ __forceinline__ float2 rcp2_mufu(float2 x) { return make_float2(rcp_mufu(x.x), rcp_mufu(x.y)); }
__device__ __forceinline__ float2 ex22_mufu(float2 x) { return make_float2(ex2_mufu(x.x), ex2_mufu(x.y)); }
// the low bytes of a, b, c, d as one word
__device__ __forceinline__ uint32_t pack4(float a, float b, float c, float d) {
    return __byte_perm(__byte_perm(__float_as_uint(a), __float_as_uint(b), 0x0040u),
                       __byte_perm(__float_as_uint(c), __float_as_uint(d), 0x0040u), 0x5410u);
}
// hi - lo as integers: 0 when both round to the same byte, else the count of crossed boundaries
__device__ __forceinline__ void crossed(float2 lo, float2 hi, uint32_t& x0, uint32_t& x1) {
    x0 += __float_as_uint(hi.x) - __float_as_uint(lo.x);
    x1 += __float_as_uint(hi.y) - __float_as_uint(lo.y);
}

// the reference's fp64 chain for one pixel (also the unaligned / tail path)
static __device__ __noinline__ void tone_rgb_px(const uint8_t* __restrict__ rgb, uint8_t* __restrict__ rgb_out,
                                                uint8_t* __restrict__ toned, uint8_t* __restrict__ gray, int64_t p,
                                                double br, double bk, double m, double k, double lo, double hi) {
    SigD sig;
    sig.m = m;
    sig.k = k;
    sig.lo = lo;
    sig.hi = hi;
    const double r = deq_byte(rgb[3 * p]), g = deq_byte(rgb[3 * p + 1]), b = deq_byte(rgb[3 * p + 2]);
    const double li = decolor_f64(r, g, b, br, bk);
    const double lout = sigmoid_d(li, sig);
    const double ratio = __ddiv_rn(lout, li > 1e-6 ? li : 1e-6);
    const bool black = li == 0.0;
    if (rgb_out) {
        rgb_out[3 * p] = black ? 0 : static_cast<uint8_t>(quantize_d(__dmul_rn(r, ratio)));
        rgb_out[3 * p + 1] = black ? 0 : static_cast<uint8_t>(quantize_d(__dmul_rn(g, ratio)));
        rgb_out[3 * p + 2] = black ? 0 : static_cast<uint8_t>(quantize_d(__dmul_rn(b, ratio)));
    }
    if (toned) toned[p] = static_cast<uint8_t>(quantize_d(lout));
    if (gray) gray[p] = static_cast<uint8_t>(quantize_d(li));
}

__global__ void __launch_bounds__(256) tone_rgb_u8_kernel(const uint8_t* __restrict__ rgb, uint8_t* __restrict__ rgb_out,
                                                          uint8_t* __restrict__ toned, uint8_t* __restrict__ gray,
                                                          int64_t npix, double br, double bk, SigD sig) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npix;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        tone_rgb_px(rgb, rgb_out, toned, gray, p, br, bk, sig.m, sig.k, sig.lo, sig.hi);
}

constexpr int kRgbPx = 16;                            // pixels per thread per tile (48 input bytes)
constexpr int kRgbTile = 256 * kRgbPx;                // 4096 pixels per tile
constexpr int kQueueDrain = 32;                       // a warp drains once a warp's worth is queued
constexpr int kQueueCap = kQueueDrain + 32 * kRgbPx;  // < kQueueDrain carried + one tile of the warp

// One pixel pair through the fp32 chain: settled bytes (lo values) and each
// pixel's crossed-boundary count (0: all its bytes settled).
struct PairOut {
    float2 r, g, b, t, y;
    uint32_t crossed0, crossed1;
};
template <bool kTwoEx2, bool kRgb, bool kToned, bool kGray>
__device__ __forceinline__ PairOut tone_rgb_pair(float2 R, float2 G, float2 B, const ToneRgbF& c) {
    const float2 M2 = bc2(kMagic), one2 = bc2(1.0f);
    // decolor
    const float2 R2 = mul2(R, R), G2 = mul2(G, G);
    const float2 white = sqrt2_mufu(fma2(B, B, add2(R2, G2)));
    const float2 rg = sqrt2_mufu(fma2(R2, bc2(c.br3), mul2(G2, bc2(c.br13))));
    const float2 RG = add2(R, G);
    const float2 s = add2(RG, B);
    const float2 W = fma2(R, rg, mul2(add2(G, B), white));
    const float2 C = mul2(B, fma2(RG, bc2(1.7320508075688772f), white));
    const float2 Qn = fma2(mul2(W, bc2(c.bk3)), W, fma2(mul2(C, bc2(c.bk13)), C, bc2(1e-30f)));
    const float2 s1 = make_float2(fmaxf(s.x, 1.0f), fmaxf(s.y, 1.0f));
    const float2 ss = mul2(s1, s1);                     // exact (s <= 765)
    const float2 q = rsqrt2_mufu(mul2(Qn, ss));         // 1 / (s sqrt(Qn))
    const float2 L = mul2(Qn, q);                       // sqrt(Qn) / s
    const float2 invL = mul2(ss, q);                    // s / sqrt(Qn)
    // logistic difference
    const float2 y = mul2(L, bc2(c.nak));  // -kx log2(e)
    const float2 E = ex22_mufu(y);
    const float2 eT = kTwoEx2 ? ex22_mufu(add2(y, bc2(c.tc))) : mul2(E, bc2(c.ekm));
    const float2 sg = rcp2_mufu(add2(eT, one2));
    float2 omS = mul2(eT, sg);
    if constexpr (kTwoEx2) omS = make_float2(fminf(omS.x, 1.0f), fminf(omS.y, 1.0f));  // inf * 0
    float2 omE = fma2(E, bc2(-1.0f), one2);
    if (__any_sync(0xFFFFFFFFu, fminf(y.x, y.y) > c.ycut)) {
        // 1 - 2^y = sum_n -(y ln2)^n / n!, n = 1..6
        constexpr float l1 = 0.6931471805599453f, l2 = 0.2402265069591007f, l3 = 0.0555041086648216f,
                        l4 = 0.0096181291076285f, l5 = 0.0013333558146428f, l6 = 0.0001540353039338f;
        const float2 ser =
            mul2(y, fma2(y, fma2(y, fma2(y, fma2(y, fma2(y, bc2(-l6), bc2(-l5)), bc2(-l4)), bc2(-l3)), bc2(-l2)),
                         bc2(-l1)));
        omE.x = y.x > c.ycut ? ser.x : omE.x;
        omE.y = y.y > c.ycut ? ser.y : omE.y;
    }
    const float2 N255 = mul2(mul2(sg, omE), bc2(c.cn255));
    // error bound -> one scale pair for the rgb and toned values
    const float2 relC = fma2(omS, fma2(L, bc2(c.cA), bc2(c.cC)), bc2(c.cD + (kRgb ? c.relRgb : c.relT)));
    const float2 cl = fma2(relC, bc2(-1.0f), one2), ch = add2(relC, one2);
    // outputs
    PairOut o;
    uint32_t x0 = 0, x1 = 0;
    if constexpr (kRgb) {
        const float2 rs = mul2(N255, invL);
        const float2 vR = mul2(R, rs), vG = mul2(G, rs), vB = mul2(B, rs);
        const float2 vr = make_float2(fminf(vR.x, 255.0f), fminf(vR.y, 255.0f));
        const float2 vg = make_float2(fminf(vG.x, 255.0f), fminf(vG.y, 255.0f));
        const float2 vb = make_float2(fminf(vB.x, 255.0f), fminf(vB.y, 255.0f));
        o.r = fma2(vr, cl, M2);
        o.g = fma2(vg, cl, M2);
        o.b = fma2(vb, cl, M2);
        crossed(o.r, fma2(vr, ch, M2), x0, x1);
        crossed(o.g, fma2(vg, ch, M2), x0, x1);
        crossed(o.b, fma2(vb, ch, M2), x0, x1);
    }
    if constexpr (kToned) {
        o.t = fma2(N255, cl, M2);
        crossed(o.t, fma2(N255, ch, M2), x0, x1);
    }
    if constexpr (kGray) {
        o.y = fma2(L, bc2(c.glo), M2);
        crossed(o.y, fma2(L, bc2(c.ghi), M2), x0, x1);
    }
    o.crossed0 = x0;
    o.crossed1 = x1;
    return o;
}

template <bool kTwoEx2, bool kRgb, bool kToned, bool kGray>
__global__ void __launch_bounds__(256, 3)
    tone_rgb_fast_kernel(const uint8_t* __restrict__ rgb, uint8_t* __restrict__ rgb_out,
                         uint8_t* __restrict__ toned, uint8_t* __restrict__ gray, int64_t ntiles, int64_t npix,
                         ToneRgbF c, double br, double bk, SigD sig) {
    __shared__ int64_t queues[8][kQueueCap];  // one per warp: appends and drains need only __syncwarp
    const int tid = threadIdx.x, lane = tid & 31;
    int64_t* queue = queues[tid >> 5];
    int qn = 0;  // warp-uniform queue length
    const int64_t stride = gridDim.x;
    int64_t t = blockIdx.x;
    uint4 v[3];
    if (t < ntiles) {
        const uint4* p = reinterpret_cast<const uint4*>(rgb + t * (kRgbTile * 3)) + tid * 3;
        v[0] = __ldcs(p);
        v[1] = __ldcs(p + 1);
        v[2] = __ldcs(p + 2);
    }
    for (; t < ntiles; t += stride) {
        uint4 nx[3] = {v[0], v[1], v[2]};
        if (t + stride < ntiles) {
            const uint4* q = reinterpret_cast<const uint4*>(rgb + (t + stride) * (kRgbTile * 3)) + tid * 3;
            nx[0] = __ldcs(q);
            nx[1] = __ldcs(q + 1);
            nx[2] = __ldcs(q + 2);
        }
        const uint32_t w[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                                v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
        uint32_t o[12], ot[4], og[4];
        uint32_t mask = 0;  // bit i: pixel i needs the fp64 chain
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // pixels 4q..4q+3 = words 3q..3q+2: R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3
            const uint32_t w0 = w[3 * q], w1 = w[3 * q + 1], w2 = w[3 * q + 2];
            const float2 mM = bc2(-kMagic);
            const float2 RA = add2(make_float2(byte_biased(w0, 0), byte_biased(w0, 3)), mM);
            const float2 GA = add2(make_float2(byte_biased(w0, 1), byte_biased(w1, 0)), mM);
            const float2 BA = add2(make_float2(byte_biased(w0, 2), byte_biased(w1, 1)), mM);
            const float2 RB = add2(make_float2(byte_biased(w1, 2), byte_biased(w2, 1)), mM);
            const float2 GB = add2(make_float2(byte_biased(w1, 3), byte_biased(w2, 2)), mM);
            const float2 BB = add2(make_float2(byte_biased(w2, 0), byte_biased(w2, 3)), mM);
            const PairOut a = tone_rgb_pair<kTwoEx2, kRgb, kToned, kGray>(RA, GA, BA, c);
            const PairOut b = tone_rgb_pair<kTwoEx2, kRgb, kToned, kGray>(RB, GB, BB, c);
            if constexpr (kRgb) {
                o[3 * q] = pack4(a.r.x, a.g.x, a.b.x, a.r.y);
                o[3 * q + 1] = pack4(a.g.y, a.b.y, b.r.x, b.g.x);
                o[3 * q + 2] = pack4(b.b.x, b.r.y, b.g.y, b.b.y);
            }
            if constexpr (kToned) ot[q] = pack4(a.t.x, a.t.y, b.t.x, b.t.y);
            if constexpr (kGray) og[q] = pack4(a.y.x, a.y.y, b.y.x, b.y.y);
            mask |= (a.crossed0 ? 1u : 0u) << (4 * q);
            mask |= (a.crossed1 ? 1u : 0u) << (4 * q + 1);
            mask |= (b.crossed0 ? 1u : 0u) << (4 * q + 2);
            mask |= (b.crossed1 ? 1u : 0u) << (4 * q + 3);
        }
        const int64_t p0 = t * kRgbTile + static_cast<int64_t>(tid) * kRgbPx;
        if constexpr (kRgb) {
            uint4* orgb = reinterpret_cast<uint4*>(rgb_out + p0 * 3);
            __stcs(orgb, make_uint4(o[0], o[1], o[2], o[3]));
            __stcs(orgb + 1, make_uint4(o[4], o[5], o[6], o[7]));
            __stcs(orgb + 2, make_uint4(o[8], o[9], o[10], o[11]));
        }
        if constexpr (kToned) __stcs(reinterpret_cast<uint4*>(toned + p0), make_uint4(ot[0], ot[1], ot[2], ot[3]));
        if constexpr (kGray) __stcs(reinterpret_cast<uint4*>(gray + p0), make_uint4(og[0], og[1], og[2], og[3]));
        if (__any_sync(0xFFFFFFFFu, mask != 0u)) {
            // exclusive prefix of the lanes' pixel counts -> each lane's slots
            const int cnt = __popc(mask);
            int pre = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int x = __shfl_up_sync(0xFFFFFFFFu, pre, d);
                if (lane >= d) pre += x;
            }
            int slot = qn + pre - cnt;
            for (uint32_t mm = mask; mm; mm &= mm - 1) queue[slot++] = p0 + (__ffs(mm) - 1);
            qn += __shfl_sync(0xFFFFFFFFu, pre, 31);
            __syncwarp();  // appends and this tile's provisional stores before the drain
            if (qn >= kQueueDrain) {
                for (int j = lane; j < qn; j += 32)
                    tone_rgb_px(rgb, rgb_out, toned, gray, queue[j], br, bk, sig.m, sig.k, sig.lo, sig.hi);
                qn = 0;
                __syncwarp();  // queue reads before the next appends
            }
        }
        v[0] = nx[0];
        v[1] = nx[1];
        v[2] = nx[2];
    }
    for (int j = lane; j < qn; j += 32)
        tone_rgb_px(rgb, rgb_out, toned, gray, queue[j], br, bk, sig.m, sig.k, sig.lo, sig.hi);
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t p = ntiles * kRgbTile + tid; p < npix; p += 256)
            tone_rgb_px(rgb, rgb_out, toned, gray, p, br, bk, sig.m, sig.k, sig.lo, sig.hi);
    }
}

// ---------------------------------------------------------------- exact toned-only route
// decolor_tone(u8, exact=True) without the colour image: the threshold-table
// kernel's arithmetic (decolor255_bits_x2, one table lookup per pixel) plus a
// proof that the fast toned byte is the reference's: err = max |f_fast -
// f_exact| over all 2^24 colours for (beta_r, beta_k), settled exhaustively
// with the exact-u8 table (wg_u8exact.cu), and M = err + 2 units of 2^-15 (the
// float rounding of the thresholds, one of slack). A pixel whose f lies
// within M of the threshold of its bin -- or of an edge of a bin flagged with
// a neighbour's threshold at that edge, or (gray requested) of a rounding
// boundary -- goes through the per-warp queue to the reference's fp64 chain.
constexpr int kExactQueue = 32 + 32 * kRgbPx;  // < 32 carried + one warp-tile
template <bool kGray, bool kMulti>
__global__ void __launch_bounds__(256, 4)
    tone_u8_exact_kernel(const uint8_t* __restrict__ rgb, uint8_t* __restrict__ toned, uint8_t* __restrict__ gray,
                         int64_t ntiles, int64_t npix, const ToneTable* __restrict__ tab, U8Consts k, uint32_t M,
                         double br, double bk, SigD sig) {
    extern __shared__ __align__(16) uint8_t dsm[];
    ToneTable* T = reinterpret_cast<ToneTable*>(dsm);  // bins + thr staged; edge folded into bins[].x
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t* queue = reinterpret_cast<uint32_t*>(dsm + kToneStaged) + wid * kExactQueue;
    {
        const float4* src = reinterpret_cast<const float4*>(tab);
        float4* dst = reinterpret_cast<float4*>(T);
        for (int i = tid; i < static_cast<int>(kToneStaged / 16); i += 256) dst[i] = src[i];
        __syncthreads();
        // the edge flag rides in bit 16 of each bin's count word: one LDS.64 per pixel
        for (int b = tid; b < kToneBins; b += 256)
            if (tab->edge[b])
                T->bins[b].x = __uint_as_float(__float_as_uint(T->bins[b].x) | 0x10000u);
    }
    __syncthreads();
    int qn = 0;
    const int64_t stride = gridDim.x;
    const auto pix = [&](uint32_t e) {  // (tile iteration << 9) | pixel offset in the warp's slice
        return (static_cast<int64_t>(blockIdx.x) + static_cast<int64_t>(e >> 9) * stride) * kRgbTile + wid * 512 +
               (e & 511u);
    };
    const auto fix = [&](int64_t p) {
        tone_rgb_px(rgb, nullptr, toned, gray, p, br, bk, sig.m, sig.k, sig.lo, sig.hi);
    };
    // toned byte of one pixel's f-domain bits; near |= f within M of a threshold
    const auto tone = [&](uint32_t bits, bool& near) -> uint32_t {
        const uint32_t b = (bits >> 11) & (kToneBins - 1);
        const float2 e = T->bins[b];
        const float f = __uint_as_float(bits);
        const uint32_t low = bits & 0x7FFu, cw = __float_as_uint(e.x);
        near = near || ((cw >> 16) != 0u && (low < M || low >= 0x800u - M));
        if constexpr (kMulti) {
            if (e.y != e.y) {  // several thresholds in this bin: binary search, both neighbours checked
                uint32_t c = 0;
#pragma unroll
                for (uint32_t st = 128; st; st >>= 1) c += (f >= T->thr[c + st - 1]) ? st : 0;
                const uint32_t lo_b = c ? __float_as_uint(T->thr[c - 1]) : 0u;
                const uint32_t hi_b = __float_as_uint(T->thr[c]);  // +inf pad: far away
                near = near || bits - lo_b <= M || hi_b - bits <= M;
                return c;
            }
        }
        near = near || bits - __float_as_uint(e.y) + M <= 2u * M;  // |bits - thr| <= M (inf: no)
        return (cw & 0xFFFFu) + (f >= e.y ? 1u : 0u);
    };
    int64_t t = blockIdx.x;
    uint4 v[3];
    if (t < ntiles) {
        const uint4* p = reinterpret_cast<const uint4*>(rgb + t * (kRgbTile * 3)) + tid * 3;
        v[0] = __ldcs(p);
        v[1] = __ldcs(p + 1);
        v[2] = __ldcs(p + 2);
    }
    for (int64_t it = 0; t < ntiles; t += stride, ++it) {
        uint4 nx[3] = {v[0], v[1], v[2]};
        if (t + stride < ntiles) {
            const uint4* q = reinterpret_cast<const uint4*>(rgb + (t + stride) * (kRgbTile * 3)) + tid * 3;
            nx[0] = __ldcs(q);
            nx[1] = __ldcs(q + 1);
            nx[2] = __ldcs(q + 2);
        }
        const uint32_t w[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                                v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
        uint32_t ot[4], og[4];
        uint32_t mask = 0;  // bit i: pixel i needs the fp64 chain
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            uint32_t tt[4], gg[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = 2 * qd + h;
                float2 ch[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int b0 = 3 * (2 * j) + c, b1 = 3 * (2 * j + 1) + c;
                    ch[c] = add2(make_float2(byte_biased(w[b0 >> 2], b0 & 3), byte_biased(w[b1 >> 2], b1 & 3)),
                                 bc2(-kMagic));
                }
                const float2 f = decolor255_bits_x2(ch[0], ch[1], ch[2], k);
                const uint32_t x = __float_as_uint(f.x), y = __float_as_uint(f.y);
                bool n0 = false, n1 = false;
                tt[2 * h] = tone(x, n0);
                tt[2 * h + 1] = tone(y, n1);
                if constexpr (kGray) {
                    gg[2 * h] = x >> 15;
                    gg[2 * h + 1] = y >> 15;
                    n0 = n0 || bits_near_tie(x, M);
                    n1 = n1 || bits_near_tie(y, M);
                }
                mask |= (n0 ? 1u : 0u) << (2 * j);
                mask |= (n1 ? 1u : 0u) << (2 * j + 1);
            }
            ot[qd] = __byte_perm(__byte_perm(tt[0], tt[1], 0x0040u), __byte_perm(tt[2], tt[3], 0x0040u), 0x5410u);
            if constexpr (kGray)
                og[qd] = __byte_perm(__byte_perm(gg[0], gg[1], 0x0040u), __byte_perm(gg[2], gg[3], 0x0040u), 0x5410u);
        }
        const int64_t p0 = t * kRgbTile + static_cast<int64_t>(tid) * kRgbPx;
        __stcs(reinterpret_cast<uint4*>(toned + p0), make_uint4(ot[0], ot[1], ot[2], ot[3]));
        if constexpr (kGray) __stcs(reinterpret_cast<uint4*>(gray + p0), make_uint4(og[0], og[1], og[2], og[3]));
        if (__any_sync(0xFFFFFFFFu, mask != 0u)) {
            const int cnt = __popc(mask);
            int pre = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int x = __shfl_up_sync(0xFFFFFFFFu, pre, d);
                if (lane >= d) pre += x;
            }
            int slot = qn + pre - cnt;
            const uint32_t e0 = (static_cast<uint32_t>(it) << 9) | static_cast<uint32_t>(lane * kRgbPx);
            for (uint32_t mm = mask; mm; mm &= mm - 1) queue[slot++] = e0 + (__ffs(mm) - 1);
            qn += __shfl_sync(0xFFFFFFFFu, pre, 31);
            __syncwarp();  // appends and this tile's provisional stores before the drain
            if (qn >= kQueueDrain) {
                for (int jj = lane; jj < qn; jj += 32) fix(pix(queue[jj]));
                qn = 0;
                __syncwarp();
            }
        }
        v[0] = nx[0];
        v[1] = nx[1];
        v[2] = nx[2];
    }
    __syncwarp();
    for (int jj = lane; jj < qn; jj += 32) fix(pix(queue[jj]));
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t p = ntiles * kRgbTile + tid; p < npix; p += 256) fix(p);
    }
}

// ---------------------------------------------------------------- exact square-domain route
// decolor_tone(u8, exact=True) without the colour image, on the square-domain
// step words (OpToneSqU8's arithmetic) plus a proof per pixel: err_sq = max
// |bits(u_fast) - bits(F(v))| over all 2^24 colours for (beta_r, beta_k),
// F(v) = float((255 v)^2 + 1/8) the monotone map the thresholds went through
// (wg_u8exact.cu settles it exhaustively), and M = err_sq + 1. A threshold
// U_j = F(theta_j) more than M float-bit units from bits(u_fast) is decided
// exactly: F(v) lies on the same side of U_j, and F is monotone, so v lies on
// the same side of theta_j. Each bin's step word is anchored at the only
// threshold within kSqReach >= M units of the bin (tables with two are not
// used here: ToneTable::sq_exact_ok), so the low 24 bits of word + bits(u) -- the
// signed distance to that anchor -- settle the pixel with two ALU ops; a
// pixel within M of its anchor (for the toned byte, or the gray's boundary
// table when gray is requested) goes through the per-warp queue to the
// reference's fp64 chain. Bit-identical to the reference by construction.
// the square-domain words (toned, gray) of pixel pair j of a thread's 16
// pixels (12 input words): exactly OpToneSqU8's arithmetic
template <bool kGray>
__device__ __forceinline__ void sq_pair_words(const uint32_t (&wd)[12], int j, const U8Consts& k,
                                              const uint32_t* s_step, const uint32_t* s_gray, uint32_t wb,
                                              uint32_t (&t)[2], uint32_t (&g)[2]) {
    float2 cb[3], ch[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int b0 = 3 * (2 * j) + c, b1 = 3 * (2 * j + 1) + c;
        cb[c] = make_float2(byte_biased(wd[b0 >> 2], b0 & 3), byte_biased(wd[b1 >> 2], b1 & 3));
        ch[c] = add2(cb[c], bc2(-kMagic));
    }
    float2 T, Sb;
    decolor255_T_x2(ch[0], ch[1], ch[2], cb[2], k, T, Sb);
    const float2 W = make_float2(__uint_as_float(lds_u32((__float_as_uint(Sb.x) << 2) + wb)),
                                 __uint_as_float(lds_u32((__float_as_uint(Sb.y) << 2) + wb)));
    const float2 u = fma2(T, W, bc2(kSqBias));
    const uint32_t ux = __float_as_uint(u.x), uy = __float_as_uint(u.y);
    const uint32_t ox = sq_bin_off(ux), oy = sq_bin_off(uy);
    t[0] = sq_word(s_step, ox, ux);
    t[1] = sq_word(s_step, oy, uy);
    if constexpr (kGray) {
        g[0] = sq_word(s_gray, ox, ux);
        g[1] = sq_word(s_gray, oy, uy);
    }
}

template <bool kGray>
__global__ void __launch_bounds__(256, kGray ? 3 : 4)
    tone_sq_exact_kernel(const uint8_t* __restrict__ rgb, uint8_t* __restrict__ toned, uint8_t* __restrict__ gray,
                         int64_t ntiles, int64_t npix, const ToneTable* __restrict__ tab, U8Consts k, SqWeights w,
                         uint32_t M, double br, double bk, SigD sig) {
    extern __shared__ __align__(16) uint8_t dsm[];
    uint32_t* s_step = reinterpret_cast<uint32_t*>(dsm);
    uint32_t* s_gray = s_step + kSqBins;
    float* s_w = reinterpret_cast<float*>(s_step + (kGray ? 2 : 1) * kSqBins);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t* queue = reinterpret_cast<uint32_t*>(s_w + kSqW) + wid * kExactQueue;
    {
        const uint4* src = reinterpret_cast<const uint4*>(tab->sq_step);
        for (int i = tid; i < kSqBins / 4; i += 256) reinterpret_cast<uint4*>(s_step)[i] = src[i];
        if constexpr (kGray) {
            const uint4* sg = reinterpret_cast<const uint4*>(tab->sq_gray);
            for (int i = tid; i < kSqBins / 4; i += 256) reinterpret_cast<uint4*>(s_gray)[i] = sg[i];
        }
        for (int i = tid; i < kSqW; i += 256) s_w[i] = w.w[i];
    }
    __syncthreads();
    const uint32_t wb = smem_addr(s_w) + w.ofs;  // shared address of W[S] = (bits(S + 2^23) << 2) + wb
    const uint32_t twoM = 2 * M;
    int qn = 0;
    const int64_t stride = gridDim.x;
    const auto pix = [&](uint32_t e) {  // (tile iteration << 9) | pixel offset in the warp's slice
        return (static_cast<int64_t>(blockIdx.x) + static_cast<int64_t>(e >> 9) * stride) * kRgbTile + wid * 512 +
               (e & 511u);
    };
    const auto fix = [&](int64_t p) {
        tone_rgb_px(rgb, nullptr, toned, gray, p, br, bk, sig.m, sig.k, sig.lo, sig.hi);
    };
    int64_t t = blockIdx.x;
    uint4 v[3];
    if (t < ntiles) {
        const uint4* p = reinterpret_cast<const uint4*>(rgb + t * (kRgbTile * 3)) + tid * 3;
        v[0] = __ldcs(p);
        v[1] = __ldcs(p + 1);
        v[2] = __ldcs(p + 2);
    }
    for (int64_t it = 0; t < ntiles; t += stride, ++it) {
        uint4 nx[3] = {v[0], v[1], v[2]};
        if (t + stride < ntiles) {
            const uint4* q = reinterpret_cast<const uint4*>(rgb + (t + stride) * (kRgbTile * 3)) + tid * 3;
            nx[0] = __ldcs(q);
            nx[1] = __ldcs(q + 1);
            nx[2] = __ldcs(q + 2);
        }
        const uint32_t wd[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                                 v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
        uint32_t ot[4], og[4];
        uint32_t mask = 0;  // bit i: pixel i needs the fp64 chain
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            uint32_t tt[4], gg[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t t2[2], g2[2];
                sq_pair_words<kGray>(wd, 2 * qd + h, k, s_step, s_gray, wb, t2, g2);
                tt[2 * h] = t2[0];
                tt[2 * h + 1] = t2[1];
                // |bits(u) - bits(anchor)| <= M  <=>  ((word + M) mod 2^24) <= 2M
                const int j = 2 * qd + h;
                mask |= ((((t2[0] + M) & 0xFFFFFFu) <= twoM) ? 1u : 0u) << (2 * j);
                mask |= ((((t2[1] + M) & 0xFFFFFFu) <= twoM) ? 1u : 0u) << (2 * j + 1);
                if constexpr (kGray) {
                    gg[2 * h] = g2[0];
                    gg[2 * h + 1] = g2[1];
                    mask |= ((((g2[0] + M) & 0xFFFFFFu) <= twoM) ? 1u : 0u) << (2 * j);
                    mask |= ((((g2[1] + M) & 0xFFFFFFu) <= twoM) ? 1u : 0u) << (2 * j + 1);
                }
            }
            ot[qd] = __byte_perm(__byte_perm(tt[0], tt[1], 0x0073u), __byte_perm(tt[2], tt[3], 0x0073u), 0x5410u);
            if constexpr (kGray)
                og[qd] = __byte_perm(__byte_perm(gg[0], gg[1], 0x0073u), __byte_perm(gg[2], gg[3], 0x0073u), 0x5410u);
        }
        const int64_t p0 = t * kRgbTile + static_cast<int64_t>(tid) * kRgbPx;
        __stcs(reinterpret_cast<uint4*>(toned + p0), make_uint4(ot[0], ot[1], ot[2], ot[3]));
        if constexpr (kGray) __stcs(reinterpret_cast<uint4*>(gray + p0), make_uint4(og[0], og[1], og[2], og[3]));
        if (__any_sync(0xFFFFFFFFu, mask != 0u)) {
            const int cnt = __popc(mask);
            int pre = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int x = __shfl_up_sync(0xFFFFFFFFu, pre, d);
                if (lane >= d) pre += x;
            }
            int slot = qn + pre - cnt;
            const uint32_t e0 = (static_cast<uint32_t>(it) << 9) | static_cast<uint32_t>(lane * kRgbPx);
            for (uint32_t mm = mask; mm; mm &= mm - 1) queue[slot++] = e0 + (__ffs(mm) - 1);
            qn += __shfl_sync(0xFFFFFFFFu, pre, 31);
            __syncwarp();  // appends and this tile's provisional stores before the drain
            if (qn >= kQueueDrain) {
                for (int jj = lane; jj < qn; jj += 32) fix(pix(queue[jj]));
                qn = 0;
                __syncwarp();
            }
        }
        v[0] = nx[0];
        v[1] = nx[1];
        v[2] = nx[2];
    }
    __syncwarp();
    for (int jj = lane; jj < qn; jj += 32) fix(pix(queue[jj]));
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t p = ntiles * kRgbTile + tid; p < npix; p += 256) fix(p);
    }
}

// The toned-only exact route as an Op of the streaming skeleton (default;
// WG_TONE_EXACT_KERNEL=1 selects tone_sq_exact_kernel, which also serves the
// gray output): the same arithmetic and proof as tone_sq_exact_kernel, 955
// vs 897 Gpix/s on C3; the per-warp queues live in
// shared memory with their length (warp-uniform), the skeleton's epilogue
// drains what is left. An entry is (tile iteration << 12 | pixel in tile).
struct OpToneSqExactU8 {
    static constexpr bool kLdg = true;
    static constexpr bool kPingPong = false;  // one register buffer ...
    static constexpr int kMinBlocks = 4;      // ... at 4 CTAs/SM (64 registers): 955 Gpix/s on C3;
    // two buffers spill at 48 or 64 registers (624 / 875), one buffer at 48 spills too (559)
    static constexpr int kPx = 16;
    const uint8_t* in;
    uint8_t* toned;
    U8Consts k;
    const ToneTable* tab;
    uint32_t M;
    double br, bk;
    SigD sig;
    SqWeights w;

    __device__ __forceinline__ static uint32_t* s_step() {
        __shared__ __align__(16) uint32_t t[kSqBins];
        return t;
    }
    __device__ __forceinline__ static float* s_w() {
        __shared__ __align__(16) float t[kSqW];
        return t;
    }
    __device__ __forceinline__ static uint32_t* s_queue() {
        __shared__ uint32_t q[8 * kExactQueue];
        return q;
    }
    __device__ __forceinline__ static int* s_qn() {
        __shared__ int n[8];
        return n;
    }
    // the staged step words carry + M: word' = word + M, so the flag test is
    // (word' mod 2^24) <= 2M without a per-pixel add; byte 3 of word' differs from
    // byte 3 of word only when the low 24 bits wrap, i.e. for flagged pixels,
    // whose bytes the fp64 queue rewrites
    __device__ __forceinline__ void prologue() const {
        const uint4* src = reinterpret_cast<const uint4*>(tab->sq_step);
        for (int i = threadIdx.x; i < kSqBins / 4; i += blockDim.x) {
            const uint4 v = src[i];
            reinterpret_cast<uint4*>(s_step())[i] = make_uint4(v.x + M, v.y + M, v.z + M, v.w + M);
        }
        for (int i = threadIdx.x; i < kSqW; i += blockDim.x) s_w()[i] = w.w[i];
        if (threadIdx.x < 8) s_qn()[threadIdx.x] = 0;
    }
    __device__ __forceinline__ void fix(int64_t p) const {
        tone_rgb_px(in, nullptr, toned, nullptr, p, br, bk, sig.m, sig.k, sig.lo, sig.hi);
    }
    __device__ __forceinline__ int64_t entry_px(uint32_t e) const {
        const int64_t tpx = static_cast<int64_t>(blockDim.x) * kPx;
        return (static_cast<int64_t>(blockIdx.x) + static_cast<int64_t>(e >> 12) * gridDim.x) * tpx + (e & 4095u);
    }
    __device__ __forceinline__ void drain(uint32_t* q, int qn) const {
        for (int j = threadIdx.x & 31; j < qn; j += 32) fix(entry_px(q[j]));
    }
    __device__ __forceinline__ void vec(const uint4 (&v)[3], int64_t px0) const {
        const uint32_t wd[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                                 v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
        const uint32_t wb = smem_addr(s_w()) + w.ofs;
        const uint32_t twoM = 2 * M;
        // |bits(u) - bits(anchor)| <= M  <=>  ((word + M) mod 2^24) <= 2M (+ M staged):
        // the group keeps only the minimum of the low 24 bits (one VIMNMX per pixel);
        // the rare group with a flagged pixel recomputes its words for the mask
        uint32_t ot[4], lo24 = 0xFFFFFFFFu;
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            uint32_t tt[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = 2 * qd + h;
                uint32_t t2[2], g2[2];
                sq_pair_words<false>(wd, j, k, s_step(), nullptr, wb, t2, g2);
                tt[2 * h] = t2[0];
                tt[2 * h + 1] = t2[1];
                lo24 = min(lo24, min(t2[0] & 0xFFFFFFu, t2[1] & 0xFFFFFFu));
            }
            ot[qd] = __byte_perm(__byte_perm(tt[0], tt[1], 0x0073u), __byte_perm(tt[2], tt[3], 0x0073u), 0x5410u);
        }
        st_global_cs_v4(toned + px0, make_uint4(ot[0], ot[1], ot[2], ot[3]));
        if (__any_sync(0xFFFFFFFFu, lo24 <= twoM)) {  // rare: queue the pixels for the fp64 chain
            uint32_t mask = 0;
            if (lo24 <= twoM) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {  // (static indices keep wd[] in registers)
                    uint32_t t2[2], g2[2];
                    sq_pair_words<false>(wd, j, k, s_step(), nullptr, wb, t2, g2);
                    mask |= (((t2[0] & 0xFFFFFFu) <= twoM) ? 1u : 0u) << (2 * j);
                    mask |= (((t2[1] & 0xFFFFFFu) <= twoM) ? 1u : 0u) << (2 * j + 1);
                }
            }
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            uint32_t* q = s_queue() + wid * kExactQueue;
            int qn = s_qn()[wid];
            const int cnt = __popc(mask);
            int pre = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int x = __shfl_up_sync(0xFFFFFFFFu, pre, d);
                if (lane >= d) pre += x;
            }
            int slot = qn + pre - cnt;
            const int64_t tpx = static_cast<int64_t>(blockDim.x) * kPx;
            const int64_t tile = px0 / tpx;
            const uint32_t e0 = (static_cast<uint32_t>((tile - blockIdx.x) / gridDim.x) << 12) |
                                static_cast<uint32_t>(px0 - tile * tpx);
            for (uint32_t mm = mask; mm; mm &= mm - 1) q[slot++] = e0 + (__ffs(mm) - 1);
            qn += __shfl_sync(0xFFFFFFFFu, pre, 31);
            __syncwarp();  // appends and this tile's provisional stores before the drain
            if (qn >= kQueueDrain) {
                drain(q, qn);
                qn = 0;
                __syncwarp();
            }
            if (lane == 0) s_qn()[wid] = qn;
            __syncwarp();
        }
    }
    __device__ __forceinline__ void epilogue() const {
        const int wid = threadIdx.x >> 5;
        __syncwarp();
        drain(s_queue() + wid * kExactQueue, s_qn()[wid]);
    }
    __device__ __forceinline__ void scalar(int64_t p) const { fix(p); }
};

// fp32 constants and error budget of the fast kernel; false if the curve is
// outside its range (then the fp64 kernel runs every pixel)
bool make_tone_rgb_consts(double br, double bk, double m, double k, ToneRgbF* c, bool* two_ex2) {
    const double u = std::ldexp(1.0, -24), log2e = 1.4426950408889634;
    if (!(k >= 1e-3 && k <= 1e4)) return false;
    const double sig1 = 1.0 / (1.0 + std::exp(-k * (1.0 - m)));  // sig(k(1-m))
    const double D = sig1 - 1.0 / (1.0 + std::exp(k * m));       // hi - lo as the reference forms it
    const double cn = 1.0 / (sig1 * -std::expm1(-k));
    if (!(D > 0.0) || !std::isfinite(cn)) return false;
    *two_ex2 = k > 80.0;
    const double relL = 13 * u;
    const double ref = 1e-13 + 4e-16 / D + 1e-15 * k;
    c->br3 = static_cast<float>(3.0 * br);
    c->br13 = static_cast<float>(3.0 * (1.0 - br));
    c->bk3 = static_cast<float>(bk / 3.0);
    c->bk13 = static_cast<float>((1.0 - bk) / 3.0);
    c->nak = static_cast<float>(-k * log2e / 255.0);
    c->ekm = *two_ex2 ? 0.0f : static_cast<float>(std::exp(k * m));
    c->tc = static_cast<float>(k * m * log2e);
    c->ycut = static_cast<float>(-0.25 * log2e);
    c->cn255 = static_cast<float>(255.0 * cn);
    const double cA = k / 255.0 * (relL + 3 * u);
    const double cC = *two_ex2 ? 3 * u + 2 * k * m * u : 5 * u;
    const double cD = 36 * u + ref;
    const double relRgb = 17 * u + 1.1e-10 / (0.4 * D);
    // test knob: WG_TONE_RGB_MARGIN_SCALE in (0, 1] shrinks every margin, so the
    // GPU tests can show the bound holds with headroom (bit-identical at 0.5)
    double sc = 1.0;
    if (const char* e = std::getenv("WG_TONE_RGB_MARGIN_SCALE")) {
        const double v = std::atof(e);
        if (v > 0.0 && v <= 1.0) sc = v;
    }
    c->cA = static_cast<float>(sc * cA);
    c->cC = static_cast<float>(sc * cC);
    c->cD = static_cast<float>(sc * cD);
    c->relRgb = static_cast<float>(sc * relRgb);
    c->relT = static_cast<float>(sc * 3 * u);  // cn255 and the scale constants
    c->glo = static_cast<float>(1.0 - sc * (relL + 2 * u));
    c->ghi = static_cast<float>(1.0 + sc * (relL + 2 * u));
    return true;
}

template <bool kTwoEx2, bool kRgb>
void launch_tone_rgb_fast(unsigned grid, cudaStream_t st, const uint8_t* rgb, uint8_t* rgb_out, uint8_t* toned,
                          uint8_t* gray, int64_t ntiles, int64_t npix, const ToneRgbF& c, double br, double bk,
                          const SigD& sig) {
    if (toned && gray)
        tone_rgb_fast_kernel<kTwoEx2, kRgb, true, true><<<grid, 256, 0, st>>>(rgb, rgb_out, toned, gray, ntiles,
                                                                              npix, c, br, bk, sig);
    else if (toned)
        tone_rgb_fast_kernel<kTwoEx2, kRgb, true, false><<<grid, 256, 0, st>>>(rgb, rgb_out, toned, gray, ntiles,
                                                                               npix, c, br, bk, sig);
    else if (gray)
        tone_rgb_fast_kernel<kTwoEx2, kRgb, false, true><<<grid, 256, 0, st>>>(rgb, rgb_out, toned, gray, ntiles,
                                                                               npix, c, br, bk, sig);
    else
        tone_rgb_fast_kernel<kTwoEx2, kRgb, false, false><<<grid, 256, 0, st>>>(rgb, rgb_out, toned, gray, ntiles,
                                                                                npix, c, br, bk, sig);
}

}  // namespace
}  // namespace wg

using namespace wg;

extern "C" int wg_decolor_tone_rgb_u8(const uint8_t* rgb, uint8_t* rgb_out, uint8_t* toned_or_null,
                                      uint8_t* gray_or_null, int64_t npix, double beta_r, double beta_k,
                                      double midpoint, double slope, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, rgb) || check_params(beta_r, beta_k) ||
                  check_curve(midpoint, slope));
    if (npix > 0 && !rgb_out && !toned_or_null && !gray_or_null)
        return set_error(WG_EINVAL, "decolor_tone_rgb_u8: no output requested");
    if (npix == 0) return WG_OK;
    int device = 0;
    cudaGetDevice(&device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the curve's constants, as apply_sigmoid forms them (tonemap.py:76-80)
    SigD sig;
    sig.m = midpoint;
    sig.k = slope;
    sig.lo = 1.0 / (1.0 + std::exp(slope * midpoint));
    sig.hi = 1.0 / (1.0 + std::exp(-slope * (1.0 - midpoint)));
    ToneRgbF c;
    bool two_ex2 = false;
    const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const bool aligned = al(rgb) && (!rgb_out || al(rgb_out)) && (!toned_or_null || al(toned_or_null)) &&
                         (!gray_or_null || al(gray_or_null));
    const int64_t ntiles = npix / kRgbTile;
    if (!rgb_out && toned_or_null && aligned && ntiles > 0 && !std::getenv("WG_TONE_EXACT_VIA_RGB")) {
        // toned (+ gray) only: the threshold-table kernel with a proven margin
        // (locks: tone cache, then exact-u8 cache, both held until the launch is enqueued)
        const ToneTable* tab = nullptr;
        bool multi = false, sq_multi = false, sq_exact_ok = false;
        std::unique_lock<std::mutex> hold_t, hold_e;
        int rc = tone_table(midpoint, slope, &tab, &multi, &hold_t, &sq_multi, &sq_exact_ok);
        if (rc != WG_OK) return rc;
        U8Exact ex;
        rc = u8exact_get(beta_r, beta_k, &ex, &hold_e);
        if (rc != WG_OK) return rc;
        const char* route = std::getenv("WG_TONE_ROUTE");
        const uint32_t Msq = ex.err_sq + 1;
        if (sq_exact_ok && Msq <= kSqReach && !(route && std::strcmp(route, "linear") == 0)) {
            // square-domain route with its proven margin
            const U8Consts k = make_u8_consts(beta_r, beta_k);
            SqWeights w;
            w.ofs = 0u - (0x4B000000u << 2);
            sq_weights(beta_k / 3.0, w.w);
            const size_t smem = ((gray_or_null ? 2 : 1) * kSqBins + kSqW + 8 * kExactQueue) * sizeof(uint32_t);
            const unsigned grid =
                static_cast<unsigned>(std::min<int64_t>(ntiles, (gray_or_null ? 3LL : 4LL) * sm_count(device)));
            if (!gray_or_null && !std::getenv("WG_TONE_EXACT_KERNEL")) {
                // toned only: the Op on the streaming skeleton (pingpong, 5 CTAs/SM)
                const void* outs[1] = {toned_or_null};
                return launch_stream(OpToneSqExactU8{rgb, toned_or_null, k, tab, Msq, beta_r, beta_k, sig, w}, rgb,
                                     outs, 1, npix, st);
            }
            auto kern = gray_or_null ? tone_sq_exact_kernel<true> : tone_sq_exact_kernel<false>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            kern<<<grid, 256, smem, st>>>(rgb, toned_or_null, gray_or_null, ntiles, npix, tab, k, w, Msq, beta_r,
                                          beta_k, sig);
            return check_launch("tone_sq_exact");
        }
        const uint32_t M = ex.err + 2;
        if (M <= kEdgeUnits) {
            const U8Consts k = make_u8_consts(beta_r, beta_k);
            const size_t smem = kToneStaged + 8 * kExactQueue * sizeof(uint32_t);
            const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ntiles, 4LL * sm_count(device)));
            auto kern = gray_or_null ? (multi ? tone_u8_exact_kernel<true, true> : tone_u8_exact_kernel<true, false>)
                                     : (multi ? tone_u8_exact_kernel<false, true> : tone_u8_exact_kernel<false, false>);
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            kern<<<grid, 256, smem, st>>>(rgb, toned_or_null, gray_or_null, ntiles, npix, tab, k, M, beta_r, beta_k,
                                         sig);
            return check_launch("tone_u8_exact");
        }
    }
    if (aligned && ntiles > 0 && make_tone_rgb_consts(beta_r, beta_k, midpoint, slope, &c, &two_ex2)) {
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ntiles, 3LL * sm_count(device)));
        auto launch = two_ex2 ? (rgb_out ? launch_tone_rgb_fast<true, true> : launch_tone_rgb_fast<true, false>)
                              : (rgb_out ? launch_tone_rgb_fast<false, true> : launch_tone_rgb_fast<false, false>);
        launch(grid, st, rgb, rgb_out, toned_or_null, gray_or_null, ntiles, npix, c, beta_r, beta_k, sig);
        return check_launch("tone_rgb_fast");
    }
    const unsigned blocks = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>((npix + 255) / 256, 16LL * sm_count(device))));
    tone_rgb_u8_kernel<<<blocks, 256, 0, st>>>(rgb, rgb_out, toned_or_null, gray_or_null, npix, beta_r, beta_k, sig);
    return check_launch("tone_rgb_u8");
}

extern "C" int wg_decolor_tone_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray_or_null, int64_t npix,
                                  float beta_r, float beta_k, float midpoint, float slope, void* stream) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, toned) || check_params(beta_r, beta_k) ||
                  check_curve(midpoint, slope));
    if (npix == 0) return WG_OK;
    const ToneTable* tab = nullptr;
    bool multi = false, sq_multi = false;
    std::unique_lock<std::mutex> hold;  // keeps the cached table alive until the launch is enqueued
    const int rc = tone_table(midpoint, slope, &tab, &multi, &hold, &sq_multi);
    if (rc != WG_OK) return rc;
    const U8Consts k = make_u8_consts(beta_r, beta_k);
    const void* outs[2] = {toned, gray_or_null};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // square-domain route unless a bin holds several thresholds (steep curves)
    // or WG_TONE_ROUTE=linear (A/B tests of the linear step words)
    const char* route = std::getenv("WG_TONE_ROUTE");
    if (!sq_multi && !(route && std::strcmp(route, "linear") == 0) && !std::getenv("WG_TONE_BINS64")) {
        const double c4sq = static_cast<double>(beta_k) / 3.0;
        if (gray_or_null)
        if (gray_or_null) {
            OpToneSqU8<true> op{rgb, toned, gray_or_null, k, tab, 0u - (0x4B000000u << 2), {}};
            sq_weights(c4sq, op.w);
            return launch_stream(op, rgb, outs, 2, npix, st);
        }
        OpToneSqU8<false> op{rgb, toned, nullptr, k, tab, 0u - (0x4B000000u << 2), {}};
        sq_weights(c4sq, op.w);
        return launch_stream(op, rgb, outs, 2, npix, st);
    }
    // WG_TONE_BINS64=1: the 8-byte-bin variant for every curve (A/B tests of the step words)
    if (multi || std::getenv("WG_TONE_BINS64")) {
        if (gray_or_null)
            return launch_stream(OpToneU8<true, true>{rgb, toned, gray_or_null, k, tab}, rgb, outs, 2, npix, st);
        return launch_stream(OpToneU8<false, true>{rgb, toned, nullptr, k, tab}, rgb, outs, 2, npix, st);
    }
    if (gray_or_null)
        return launch_stream(OpToneU8<true, false>{rgb, toned, gray_or_null, k, tab}, rgb, outs, 2, npix, st);
    return launch_stream(OpToneU8<false, false>{rgb, toned, nullptr, k, tab}, rgb, outs, 2, npix, st);
}
