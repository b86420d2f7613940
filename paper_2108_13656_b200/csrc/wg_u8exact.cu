// wg_u8exact.cu -- bit-exact uint8 decolor: the table of near-tie colours.
//
// The uint8 kernel computes 255*gray in fp32 (decolor255_bits_x2, |error| <=
// 6e-5 in the 0..255 domain) and rounds it; the reference rounds its fp64 gray
// (floor(v * 255 + 0.5), codec.py:22-25). The two bytes can differ only where
// 255*gray + 0.5 lies next to an integer. Because a uint8 pixel is one of 2^24
// colours, the set of such colours is settled once per (beta_r, beta_k) by
// exhaustion: a setup pass runs every colour through both the kernel's fp32
// sequence and the reference's fp64 chain, finds the margin (distance from
// the boundary, in 2^-15 units) that covers every colour where they differ,
// and stores the exact byte of every colour within that margin in a small
// open-addressing table (a few thousand entries). The kernel flags pixels
// within the margin (three ALU ops) and looks only those up, so its output is
// bit-identical to the reference for every input, by construction.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"

namespace wg {
namespace {

constexpr uint32_t kColours = 1u << 24;
constexpr uint32_t kMinMargin = 3;  // >= the estimate's error (6e-5 ~ 2 units) + 1

__device__ __forceinline__ uint32_t exact_byte(uint32_t c, double br, double bk) {
    return quantize_d(decolor_f64(deq_byte(c >> 16), deq_byte((c >> 8) & 255u), deq_byte(c & 255u), br, bk));
}

__device__ __forceinline__ uint32_t fast_bits(uint32_t c, const U8Consts& k) {
    return decolor255_bits_x1(static_cast<float>(c >> 16), static_cast<float>((c >> 8) & 255u),
                              static_cast<float>(c & 255u), k);
}

__device__ __forceinline__ uint32_t tie_distance(uint32_t bits) {
    const uint32_t f = bits & 0x7FFFu;
    return f < 0x4000u ? f : 0x8000u - f;
}

// need[0]: largest boundary distance among colours whose fast byte is wrong;
// need[1]: the largest |f_fast - f_exact| over all colours in 2^-15 units,
// rounded up (f = 255 gray + 0.5 in the bits' fixed-point form) -- a true
// error bound of the fast gray for this (beta_r, beta_k), which the exact
// tone map compares against its thresholds;
// need[2]: the same for the square-domain route (csrc/wg_square.cuh): the
// largest |bits(u_fast) - bits(F(v))| with u_fast = T W[S] + 1/8 exactly as
// the tone kernel forms it and F(v) = float((255 v)^2 + 1/8) of the
// reference's fp64 gray v (the map its thresholds go through)
__global__ void u8exact_need_kernel(U8Consts k, double br, double bk, uint32_t* need) {
    uint32_t worst = 0, err = 0, err_sq = 0;
    const double c4sq = bk / 3.0;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < kColours; c += gridDim.x * blockDim.x) {
        const uint32_t bits = fast_bits(c, k);
        if (bits_byte(bits) != exact_byte(c, br, bk)) worst = max(worst, tie_distance(bits) + 1);
        const double v = decolor_f64(deq_byte(c >> 16), deq_byte((c >> 8) & 255u), deq_byte(c & 255u), br, bk);
        const double exact_units = (v * 255.0 + 0.5) * 32768.0;  // bits & 0x7FFFFF = (f - 256) * 2^15
        const double d = fabs(static_cast<double>(bits & 0x7FFFFFu) - exact_units);
        err = max(err, static_cast<uint32_t>(ceil(d)));
        float T, S;
        decolor255_T_x1(static_cast<float>(c >> 16), static_cast<float>((c >> 8) & 255u),
                        static_cast<float>(c & 255u), k, T, S);
        const float W = S > 0.0f ? static_cast<float>(__ddiv_rn(c4sq, __dmul_rn(S, S))) : 0.0f;  // sq_weights
        const float uf = __fmaf_rn(T, W, 0.125f);
        const double v255 = __dmul_rn(v, 255.0);
        const float ue = static_cast<float>(__dadd_rn(__dmul_rn(v255, v255), 0.125));
        const int64_t du = static_cast<int64_t>(__float_as_uint(uf)) - static_cast<int64_t>(__float_as_uint(ue));
        err_sq = max(err_sq, static_cast<uint32_t>(du < 0 ? -du : du));
    }
    if (worst) atomicMax(need, worst);
    if (err) atomicMax(need + 1, err);
    if (err_sq) atomicMax(need + 2, err_sq);
}

// every colour within the margin goes into the table with its exact byte
__global__ void u8exact_fill_kernel(U8Consts k, double br, double bk, uint32_t margin, uint32_t* tab, uint32_t mask,
                                    uint32_t* count) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < kColours; c += gridDim.x * blockDim.x) {
        const uint32_t bits = fast_bits(c, k);
        if (!bits_near_tie(bits, margin)) continue;
        const uint32_t e = (c << 8) | exact_byte(c, br, bk);
        atomicAdd(count, 1u);
        for (uint32_t s = u8exact_slot(c, mask);; s = (s + 1) & mask) {
            const uint32_t prev = atomicCAS(tab + s, 0xFFFFFFFFu, e);
            if (prev == 0xFFFFFFFFu || prev == e) break;
        }
    }
}

struct Entry {
    bool used = false;
    double br = 0, bk = 0;
    U8Exact t{};
};
constexpr int kCache = 4;
Entry g_cache[kMaxDevices][kCache];
int g_next[kMaxDevices];
std::mutex g_mu;

int build(int device, double br, double bk, U8Exact* out) {
    const U8Consts k = make_u8_consts(br, bk);  // exactly the constants the kernels use
    cudaStream_t st;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e != cudaSuccess) return set_error(static_cast<int>(e), "u8 exact table: stream: %s", cudaGetErrorString(e));
    uint32_t* scratch = nullptr;  // need, error bound, square-domain error bound, count
    uint32_t* tab = nullptr;
    int rc = WG_OK;
    const int blocks = 8 * sm_count(device);
    uint32_t host[4] = {0, 0, 0, 0};
    uint32_t slots = 1u << 15;
    do {
        if ((e = cudaMalloc(&scratch, 16)) != cudaSuccess) break;
        if ((e = cudaMemsetAsync(scratch, 0, 16, st)) != cudaSuccess) break;
        u8exact_need_kernel<<<blocks, 256, 0, st>>>(k, br, bk, scratch);
        if ((e = cudaMemcpyAsync(host, scratch, 12, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
        const uint32_t margin = host[0] > kMinMargin ? host[0] : kMinMargin;
        for (;;) {  // grow until the table is at most half full
            if ((e = cudaMalloc(&tab, slots * 4ull)) != cudaSuccess) break;
            if ((e = cudaMemsetAsync(tab, 0xFF, slots * 4ull, st)) != cudaSuccess) break;
            if ((e = cudaMemsetAsync(scratch + 3, 0, 4, st)) != cudaSuccess) break;
            u8exact_fill_kernel<<<blocks, 256, 0, st>>>(k, br, bk, margin, tab, slots - 1, scratch + 3);
            if ((e = cudaMemcpyAsync(host + 3, scratch + 3, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
            if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
            if (host[3] * 2 <= slots) break;
            cudaFree(tab);
            tab = nullptr;
            slots <<= 2;
        }
        if (e != cudaSuccess) break;
        out->tab = tab;
        out->mask = slots - 1;
        out->margin = margin;
        out->err = host[1];
        out->err_sq = host[2];
    } while (false);
    if (e != cudaSuccess) {
        rc = set_error(static_cast<int>(e), "u8 exact table: %s", cudaGetErrorString(e));
        if (tab) cudaFree(tab);
    }
    if (scratch) cudaFree(scratch);
    cudaStreamDestroy(st);
    return rc;
}

}  // namespace

// The table for (beta_r, beta_k) on the current device, built on first use.
// *hold stays locked: the caller enqueues its kernel before releasing it, so an
// eviction by another thread (cudaFree waits for queued work) cannot free a
// table that a pending launch uses.
int u8exact_get(double beta_r, double beta_k, U8Exact* out, std::unique_lock<std::mutex>* hold) {
    int device = 0;
    cudaGetDevice(&device);
    if (device < 0 || device >= kMaxDevices) return set_error(WG_ENODEV, "device ordinal out of range");
    *hold = std::unique_lock<std::mutex>(g_mu);
    for (Entry& en : g_cache[device])
        if (en.used && en.br == beta_r && en.bk == beta_k) {
            *out = en.t;
            return WG_OK;
        }
    U8Exact t;
    const int rc = build(device, beta_r, beta_k, &t);
    if (rc != WG_OK) return rc;
    Entry& slot = g_cache[device][g_next[device]];
    g_next[device] = (g_next[device] + 1) % kCache;
    if (slot.used) cudaFree(const_cast<uint32_t*>(slot.t.tab));
    slot.used = true;
    slot.br = beta_r;
    slot.bk = beta_k;
    slot.t = t;
    *out = t;
    return WG_OK;
}

}  // namespace wg

using namespace wg;

// diagnostics: the margin and entry count of the table for (beta_r, beta_k)
extern "C" int wg_u8_exact_info(double beta_r, double beta_k, uint32_t* margin, uint32_t* slots, uint32_t* err,
                                uint32_t* err_sq) {
    WG_CHECK_ARGS(check_params(beta_r, beta_k));
    U8Exact t;
    std::unique_lock<std::mutex> hold;
    const int rc = u8exact_get(beta_r, beta_k, &t, &hold);
    if (rc != WG_OK) return rc;
    if (margin) *margin = t.margin;
    if (slots) *slots = t.mask + 1;
    if (err) *err = t.err;
    if (err_sq) *err_sq = t.err_sq;
    return WG_OK;
}
