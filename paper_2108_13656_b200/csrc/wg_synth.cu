// wg_synth.cu -- on-device generators for the seeded synthetic workloads of
// BASELINE.json configs C2-C5 (SURVEY.md 8 d). Large batches (C5 is 102 GB of
// input) are generated in HBM instead of being staged from the host. The
// integer generators (C3 Voronoi, C5 uniform) are restated bit-exactly in
// oracle/warmgray_oracle.c so tests can pin them.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/warmgray_b200.h"
#include "wg_device.cuh"
#include "wg_internal.h"

namespace wg {

// C5: word w of image i = hash3(seed, first_image + i, w); bytes little-endian.
__global__ void synth_uniform_kernel(uint8_t* __restrict__ out, int64_t nimg, int64_t bytes_per_img,
                                     uint32_t seed, int64_t first_image) {
    const int64_t words = (bytes_per_img + 3) / 4;
    const bool vec = (bytes_per_img % 16) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    for (int64_t img = blockIdx.y; img < nimg; img += gridDim.y) {
        uint8_t* o = out + img * bytes_per_img;
        const uint32_t im = static_cast<uint32_t>(first_image + img);
        if (vec) {
            for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < words / 4;
                 q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
                const uint32_t w0 = static_cast<uint32_t>(4 * q);
                uint4 v = make_uint4(hash3(seed, im, w0), hash3(seed, im, w0 + 1), hash3(seed, im, w0 + 2),
                                     hash3(seed, im, w0 + 3));
                __stcs(reinterpret_cast<uint4*>(o) + q, v);
            }
        } else {
            for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < bytes_per_img;
                 j += static_cast<int64_t>(gridDim.x) * blockDim.x)
                o[j] = static_cast<uint8_t>(hash3(seed, im, static_cast<uint32_t>(j >> 2)) >> (8 * (j & 3)));
        }
    }
}

// C3: Voronoi cells (exact int distances, ties -> lowest index) + noise.
constexpr int kMaxSeeds = 1024;
__global__ void synth_voronoi_kernel(uint8_t* __restrict__ out, int32_t width, int32_t height,
                                     const int32_t* __restrict__ seeds_xy,
                                     const uint8_t* __restrict__ colors, int32_t nseeds,
                                     uint32_t seed, int64_t first_image) {
    __shared__ int32_t sx[kMaxSeeds], sy[kMaxSeeds];
    const int64_t img = blockIdx.y;
    for (int k = threadIdx.x; k < nseeds; k += blockDim.x) {
        sx[k] = seeds_xy[(img * nseeds + k) * 2];
        sy[k] = seeds_xy[(img * nseeds + k) * 2 + 1];
    }
    __syncthreads();
    const int64_t npx = static_cast<int64_t>(width) * height;
    const uint8_t* col = colors + img * nseeds * 3;
    uint8_t* o = out + img * npx * 3;
    const uint32_t im = static_cast<uint32_t>(first_image + img);
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npx;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t x = static_cast<int32_t>(p % width), y = static_cast<int32_t>(p / width);
        int32_t best = 0;
        int64_t bd = INT64_MAX;
        for (int k = 0; k < nseeds; ++k) {
            const int64_t dx = x - sx[k], dy = y - sy[k];
            const int64_t d = dx * dx + dy * dy;
            if (d < bd) {
                bd = d;
                best = k;
            }
        }
        const uint32_t h = hash3(seed ^ 0x5bd1e995U, im, static_cast<uint32_t>(p));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int n = static_cast<int>((h >> (10 * c)) & 1023U) % 9 - 4;
            const int v = static_cast<int>(col[3 * best + c]) + n;
            o[3 * p + c] = static_cast<uint8_t>(v < 0 ? 0 : (v > 255 ? 255 : v));
        }
    }
}

// C2: mid-gray base + Gaussian colour blobs + uniform noise, clipped to [0,1].
constexpr int kMaxBlobs = 256;
__global__ void synth_blobs_kernel(float* __restrict__ out, int32_t width, int32_t height,
                                   const float* __restrict__ blobs, int32_t nblobs,
                                   const float* __restrict__ base, float noise, uint32_t seed,
                                   int64_t first_image) {
    __shared__ float sb[kMaxBlobs * 8];
    const int64_t img = blockIdx.y;
    for (int k = threadIdx.x; k < nblobs * 8; k += blockDim.x) sb[k] = blobs[img * nblobs * 8 + k];
    __syncthreads();
    const float b0 = base[img];
    const int64_t npx = static_cast<int64_t>(width) * height;
    float* o = out + img * npx * 3;
    const uint32_t im = static_cast<uint32_t>(first_image + img);
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npx;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float x = static_cast<float>(p % width), y = static_cast<float>(p / width);
        float c[3] = {b0, b0, b0};
        for (int k = 0; k < nblobs; ++k) {
            const float* bl = sb + 8 * k;
            const float dx = x - bl[0], dy = y - bl[1];
            const float g = bl[3] * __expf(-(dx * dx + dy * dy) * bl[2]);
            c[0] += g * (bl[4] - b0);
            c[1] += g * (bl[5] - b0);
            c[2] += g * (bl[6] - b0);
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const uint32_t h = hash3(seed ^ 0x27d4eb2fU, im, static_cast<uint32_t>(3 * p + ch));
            const float v = c[ch] + noise * (2.0f * u01(h) - 1.0f);
            o[3 * p + ch] = fminf(fmaxf(v, 0.0f), 1.0f);
        }
    }
}

// C4: per-pixel i.i.d. HDR radiance.
__global__ void synth_hdr_kernel(float* __restrict__ out, int64_t nimg, int64_t ppi, float log_lo,
                                 float log_hi, uint32_t seed, int64_t first_image) {
    const int64_t total = nimg * ppi;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t img = q / ppi, p = q - img * ppi;
        const uint32_t im = static_cast<uint32_t>(first_image + img);
        const uint32_t h1 = hash3(seed ^ 0x165667b1U, im, static_cast<uint32_t>(3 * p));
        const uint32_t h2 = hash3(seed ^ 0x165667b1U, im, static_cast<uint32_t>(3 * p + 1));
        const uint32_t h3 = hash3(seed ^ 0x165667b1U, im, static_cast<uint32_t>(3 * p + 2));
        const float lum = exp10f(log_lo + (log_hi - log_lo) * u01(h1));
        const float hue = 6.0f * u01(h2), mixw = u01(h3);
        const int sector = min(static_cast<int>(hue), 5);
        const float f = hue - sector;
        float r, g, b;
        switch (sector) {
            case 0: r = 1.f; g = f; b = 0.f; break;
            case 1: r = 1.f - f; g = 1.f; b = 0.f; break;
            case 2: r = 0.f; g = 1.f; b = f; break;
            case 3: r = 0.f; g = 1.f - f; b = 1.f; break;
            case 4: r = f; g = 0.f; b = 1.f; break;
            default: r = 1.f; g = 0.f; b = 1.f - f; break;
        }
        r = r + mixw * (1.f - r);
        g = g + mixw * (1.f - g);
        b = b + mixw * (1.f - b);
        const float y = 0.2126f * r + 0.7152f * g + 0.0722f * b;
        const float s = lum / y;
        float* o = out + 3 * q;
        o[0] = r * s;
        o[1] = g * s;
        o[2] = b * s;
    }
}

static unsigned blocks_for(int64_t n, int per_image_cap) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, per_image_cap)));
}

}  // namespace wg

using namespace wg;

extern "C" int wg_synth_uniform_u8(uint8_t* out, int64_t nimg, int64_t bytes_per_img, uint32_t seed,
                                   int64_t first_image, void* stream) {
    WG_CHECK_ARGS(check_npix(nimg) || check_npix(bytes_per_img) || check_ptrs(nimg * bytes_per_img, out, out));
    if (nimg == 0 || bytes_per_img == 0) return WG_OK;
    const dim3 grid(blocks_for(bytes_per_img / 16 + 1, 2048),
                    static_cast<unsigned>(std::min<int64_t>(nimg, 65535)));
    synth_uniform_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, nimg, bytes_per_img,
                                                                              seed, first_image);
    return check_launch("synth_uniform_u8");
}

extern "C" int wg_synth_voronoi_u8(uint8_t* out, int64_t nimg, int32_t width, int32_t height,
                                   const int32_t* seeds_xy, const uint8_t* colors, int32_t nseeds,
                                   uint32_t seed, int64_t first_image, void* stream) {
    WG_CHECK_ARGS(check_npix(nimg) || width < 0 || height < 0);
    if (nseeds < 1 || nseeds > kMaxSeeds) return set_error(WG_EINVAL, "nseeds must be in [1, %d]", kMaxSeeds);
    if (nimg > 65535) return set_error(WG_EINVAL, "at most 65535 images per call");
    const int64_t npx = static_cast<int64_t>(width) * height;
    if (nimg == 0 || npx == 0) return WG_OK;
    WG_CHECK_ARGS(check_ptrs(1, out, seeds_xy) || check_ptrs(1, colors, colors));
    const dim3 grid(blocks_for(npx, 4096), static_cast<unsigned>(nimg));
    synth_voronoi_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        out, width, height, seeds_xy, colors, nseeds, seed, first_image);
    return check_launch("synth_voronoi_u8");
}

extern "C" int wg_synth_blobs_f32(float* out, int64_t nimg, int32_t width, int32_t height,
                                  const float* blobs, int32_t nblobs, const float* base, float noise,
                                  uint32_t seed, int64_t first_image, void* stream) {
    WG_CHECK_ARGS(check_npix(nimg) || width < 0 || height < 0);
    if (nblobs < 0 || nblobs > kMaxBlobs) return set_error(WG_EINVAL, "nblobs must be in [0, %d]", kMaxBlobs);
    if (nimg > 65535) return set_error(WG_EINVAL, "at most 65535 images per call");
    const int64_t npx = static_cast<int64_t>(width) * height;
    if (nimg == 0 || npx == 0) return WG_OK;
    WG_CHECK_ARGS(check_ptrs(1, out, base) || (nblobs > 0 && blobs == nullptr));
    const dim3 grid(blocks_for(npx, 4096), static_cast<unsigned>(nimg));
    synth_blobs_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        out, width, height, blobs, nblobs, base, noise, seed, first_image);
    return check_launch("synth_blobs_f32");
}

extern "C" int wg_synth_hdr_f32(float* out, int64_t nimg, int64_t pix_per_img, float lum_lo,
                                float lum_hi, uint32_t seed, int64_t first_image, void* stream) {
    WG_CHECK_ARGS(check_npix(nimg) || check_npix(pix_per_img) || !(lum_lo > 0.0f) || !(lum_hi >= lum_lo));
    if (nimg == 0 || pix_per_img == 0) return WG_OK;
    WG_CHECK_ARGS(check_ptrs(1, out, out));
    int device = 0;
    cudaGetDevice(&device);
    const unsigned blocks = blocks_for(nimg * pix_per_img, 32 * sm_count(device));
    synth_hdr_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        out, nimg, pix_per_img, log10f(lum_lo), log10f(lum_hi), seed, first_image);
    return check_launch("synth_hdr_f32");
}
