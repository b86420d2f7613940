// wg_square.cuh -- the square-domain uint8 route of the tone map
// (csrc/wg_tone.cu, OpToneSqU8):
// (255 gray)^2 = c4^2 T / S^2 for the model's T (decolor255_T_x2) and the byte
// sum S = r + g + b, so with W[S] = c4^2 / S^2 from a 768-entry shared table
// u = T W[S] + 1/8 = (255 v)^2 + 1/8 needs no root. A monotone byte function of
// v (quantize_u8 itself, or a tone curve) is then the number of its
// thresholds U_j <= u, read from log-spaced "step words": 256 bins per octave
// of u over [2^-3, 2^16) (bin = float bits >> 15), step[b] = 2^24 count +
// (2^24 - L) - (bits of the bin's first u), L the low 15 bits of the bin's
// threshold (2^15 without one), so that byte 3 of step[b] + bits(u) is the
// byte (the in-bin offset minus L borrows from / carries into bit 24).
#pragma once

#include <cstdint>

namespace wg {

constexpr int kSqBins = 19 * 256;            // 19 octaves [2^-3, 2^16), 256 per octave
constexpr uint32_t kSqLoBits = 0x3E000000u;  // bits of 2^-3, the first bin
constexpr float kSqBias = 0.125f;            // u >= 2^-3 for every pixel (black too)
constexpr int kSqW = 768;                    // W[S] for S = r + g + b in [0, 765]

// byte offset of u's bin in a step table: ((bits >> 15) - (kSqLoBits >> 15)) * 4
__device__ __forceinline__ uint32_t sq_bin_off(uint32_t ub) { return ((ub >> 13) & 0xFFFFCu) - (kSqLoBits >> 13); }
// the step word of u's bin plus bits(u): byte 3 is the byte
__device__ __forceinline__ uint32_t sq_word(const uint32_t* t, uint32_t off, uint32_t ub) {
    return *reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(t) + off) + ub;
}

constexpr uint32_t kSqReach = 64;  // anchor reach (float-bit units of u): the exact route's margin limit
constexpr int kSqMulti = 1, kSqCrowded = 2;

// W[S] as a kernel parameter, with the bias offset of its shared-memory lookup
// (ofs = -(0x4B000000 << 2) mod 2^32: W + 4 S = (bits(S + 2^23) << 2) + W + ofs)
struct SqWeights {
    uint32_t ofs;
    float w[kSqW];
};

// host side (csrc/wg_tone.cu)
void sq_weights(double c4sq, float* w);  // W[S] = c4^2 / S^2 (fp64, rounded once), W[0] = 0
int sq_step_words(const float* uf, int n, uint32_t* step, int nbins, uint32_t lo_bits, int shift, uint32_t reach);

}  // namespace wg

// (r02: the same route for a share of the plain decolor kernel's pixel pairs,
// to offload its MUFU-bound rsqrt, measured slower on C3 -- 1 / 2 / 3 / 8 of 8
// pairs: 1203 / 1171 / 1166 / 1152 vs 1206 Gpix/s: the decolor kernel is
// bound by issue as much as by the XU pipe, so extra instructions cost more
// than the MUFU they save.)
