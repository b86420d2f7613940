// mufu_error.cu -- exhaustive max relative error of the MUFU approximations
// the fp32 colour tone-map path (wg_tone.cu, tone_rgb_fast_kernel) bounds
// its error with: ex2.approx.ftz.f32 over every float in [-126, 0],
// rsqrt.approx / sqrt.approx over [1, 4) (exponent-periodic), rcp.approx over
// [1, 2). Reference values in fp64 (exp2 / rsqrt / sqrt / 1/x correctly
// rounded to ~1e-16). Prints the max relative error in units of u = 2^-24.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_error scripts/mufu_error.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2a(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rsqa(float x) { float y; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sqa(float x) { float y; asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcpa(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__device__ unsigned long long g_max[5];

__device__ __forceinline__ void upd(int i, double rel) {
    // rel >= 0: the bit pattern of a non-negative double orders like an integer
    atomicMax(&g_max[i], static_cast<unsigned long long>(__double_as_longlong(rel)));
}

__global__ void probe(uint32_t lo_bits, uint32_t n, int which, int slot) {
    double worst = 0.0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float x = __uint_as_float(lo_bits + i);
        double ref, got;
        if (which == 0) { got = ex2a(x); ref = exp2(static_cast<double>(x)); }
        else if (which == 1) { got = rsqa(x); ref = rsqrt(static_cast<double>(x)); }
        else if (which == 2) { got = sqa(x); ref = sqrt(static_cast<double>(x)); }
        else { got = rcpa(x); ref = 1.0 / static_cast<double>(x); }
        const double rel = fabs(got - ref) / ref;
        worst = rel > worst ? rel : worst;
    }
    upd(slot, worst);
}

int main() {
    const float u = 5.9604644775390625e-08f;  // 2^-24
    struct R { const char* name; float lo, hi; int which; } rs[] = {
        {"ex2.approx.ftz  [-126, 0]", -126.0f, -0.0f, 0},
        {"rsqrt.approx.ftz [1, 4)", 1.0f, 4.0f, 1},
        {"sqrt.approx.ftz  [1, 4)", 1.0f, 4.0f, 2},
        {"rcp.approx.ftz   [1, 2)", 1.0f, 2.0f, 3},
        {"ex2.approx.ftz  [0, 127]", 0.0f, 127.0f, 0},
    };
    unsigned long long zero[5] = {0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_max, zero, sizeof(zero));
    int slot = 0;
    for (auto& r : rs) {
        uint32_t a, b;
        if (slot == 0) {  // negative floats: bits grow with magnitude; [-0, -126]
            a = 0x80000000u;
            b = 0xC2FC0000u;  // -126.0f
        } else {
            memcpy(&a, &r.lo, 4);
            memcpy(&b, &r.hi, 4);
        }
        probe<<<148 * 16, 256>>>(a, b - a + 1, r.which, slot);
        ++slot;
    }
    cudaDeviceSynchronize();
    unsigned long long got[5];
    cudaMemcpyFromSymbol(got, g_max, sizeof(got));
    slot = 0;
    for (auto& r : rs) {
        double rel;
        memcpy(&rel, &got[slot++], 8);
        printf("%s  max rel err %.3e = %.2f u\n", r.name, rel, rel / u);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
