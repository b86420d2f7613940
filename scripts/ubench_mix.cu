// ubench_mix.cu -- do MUFU and packed-FMA instructions overlap on sm_100a?
// Each variant runs CH independent chains per thread; per chain step it issues
// the listed mix. Reported: chain-steps per clock per SM and the implied
// cycles per step per SMSP (issue model check for the u8 decolor kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubmix scripts/ubench_mix.cu && /tmp/ubmix
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int CH = 4;

__device__ __forceinline__ unsigned long long pk(float2 a) { unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y)); return r; }
__device__ __forceinline__ float2 upk(unsigned long long r) { float2 a; asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r)); return a; }
#define FFMA2(d, a, b, c) { unsigned long long r_; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r_) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c))); d = upk(r_); }
#define FMUL2(d, a, b) { unsigned long long r_; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r_) : "l"(pk(a)), "l"(pk(b))); d = upk(r_); }
#define SQRT(x) asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(x))

template <int V>
__global__ void mix(float* out) {
    float2 a[CH], b[CH], c[CH], d[CH], e[CH];
    float s[CH], t[CH];
    uint32_t w[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        float f = 1.0f + 1e-3f * (threadIdx.x + i);
        a[i] = make_float2(f, f + 1); b[i] = make_float2(f + 2, f + 3); c[i] = make_float2(f + 4, f + 5);
        d[i] = make_float2(f + 6, f + 7); e[i] = make_float2(f + 8, f + 9); s[i] = f + 10; t[i] = f + 11;
        w[i] = threadIdx.x * 7 + i;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (V == 0) { SQRT(s[i]); }                                  // MUFU only
            if (V == 1) { FFMA2(a[i], a[i], b[i], c[i]); FFMA2(d[i], d[i], b[i], e[i]); FFMA2(c[i], c[i], e[i], b[i]); FFMA2(e[i], e[i], a[i], d[i]); }  // 4 FFMA2 3-distinct
            if (V == 2) { SQRT(s[i]); FFMA2(a[i], a[i], b[i], c[i]); FFMA2(d[i], d[i], b[i], e[i]); FFMA2(c[i], c[i], e[i], b[i]); FFMA2(e[i], e[i], a[i], d[i]); }
            if (V == 3) { SQRT(s[i]); SQRT(t[i]); FFMA2(a[i], a[i], b[i], c[i]); FFMA2(d[i], d[i], b[i], e[i]); FFMA2(c[i], c[i], e[i], b[i]); FFMA2(e[i], e[i], a[i], d[i]); }
            if (V == 4) { FFMA2(a[i], a[i], a[i], a[i]); FFMA2(d[i], d[i], d[i], d[i]); FFMA2(c[i], c[i], c[i], c[i]); FFMA2(e[i], e[i], e[i], e[i]); }  // 1-distinct
            if (V == 5) { SQRT(s[i]); FFMA2(a[i], a[i], a[i], a[i]); FFMA2(d[i], d[i], d[i], d[i]); FFMA2(c[i], c[i], c[i], c[i]); FFMA2(e[i], e[i], e[i], e[i]); }
            if (V == 6) { FMUL2(a[i], a[i], b[i]); FMUL2(d[i], d[i], b[i]); FMUL2(c[i], c[i], e[i]); FMUL2(e[i], e[i], a[i]); }  // 4 FMUL2 2-distinct
            if (V == 7) { SQRT(s[i]); FMUL2(a[i], a[i], b[i]); FMUL2(d[i], d[i], b[i]); FMUL2(c[i], c[i], e[i]); FMUL2(e[i], e[i], a[i]); }
            if (V == 8) { uint32_t x; asm volatile("prmt.b32 %0, %1, %2, 0x7440;" : "=r"(x) : "r"(w[i]), "r"(w[(i + 1) % CH])); w[i] = x;
                          asm volatile("prmt.b32 %0, %1, %2, 0x7441;" : "=r"(x) : "r"(w[i]), "r"(w[(i + 2) % CH])); w[i] ^= x; }  // 2 PRMT
            if (V == 9) { SQRT(s[i]); uint32_t x; asm volatile("prmt.b32 %0, %1, %2, 0x7440;" : "=r"(x) : "r"(w[i]), "r"(w[(i + 1) % CH])); w[i] = x;
                          asm volatile("prmt.b32 %0, %1, %2, 0x7441;" : "=r"(x) : "r"(w[i]), "r"(w[(i + 2) % CH])); w[i] ^= x;
                          FFMA2(a[i], a[i], b[i], c[i]); FFMA2(d[i], d[i], b[i], e[i]); }
            if (V == 10) { float y; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(s[i]), "f"(t[i]), "f"(s[(i + 1) % CH])); s[i] = y;
                           asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(t[i]), "f"(s[i]), "f"(t[(i + 1) % CH])); t[i] = y; }  // 2 scalar FFMA
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) acc += a[i].x + b[i].y + c[i].x + d[i].y + e[i].x + s[i] + t[i] + __uint_as_float(w[i]);
    if (acc == 1234.5f) out[0] = acc;
}

template <int V>
void run(const char* name, int sms, double mhz, float* buf, int warps_per_sm) {
    const int threads = 256, blocks = sms * warps_per_sm / 8;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    mix<V><<<blocks, threads>>>(buf);
    cudaEventRecord(a);
    mix<V><<<blocks, threads>>>(buf);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double steps = double(blocks) * threads / 32 * ITERS * CH;  // warp chain-steps
    double cyc = ms * 1e-3 * mhz * 1e6;
    double per_smsp = cyc * sms * 4 / steps;
    printf("%-46s warps/SM=%2d  %7.3f ms  %6.2f cycles per warp-step per SMSP\n", name, warps_per_sm, ms, per_smsp);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double mhz = 1965.0;
    float* buf; cudaMalloc(&buf, 64);
    for (int wps : {16, 32, 48}) {
        run<0>("1 MUFU", sms, mhz, buf, wps);
        run<1>("4 FFMA2 (3 distinct)", sms, mhz, buf, wps);
        run<2>("1 MUFU + 4 FFMA2 (3 distinct)", sms, mhz, buf, wps);
        run<3>("2 MUFU + 4 FFMA2 (3 distinct)", sms, mhz, buf, wps);
        run<4>("4 FFMA2 (1 distinct)", sms, mhz, buf, wps);
        run<5>("1 MUFU + 4 FFMA2 (1 distinct)", sms, mhz, buf, wps);
        run<6>("4 FMUL2 (2 distinct)", sms, mhz, buf, wps);
        run<7>("1 MUFU + 4 FMUL2 (2 distinct)", sms, mhz, buf, wps);
        run<8>("2 PRMT", sms, mhz, buf, wps);
        run<9>("1 MUFU + 2 PRMT + 2 FFMA2", sms, mhz, buf, wps);
        run<10>("2 scalar FFMA (3 regs)", sms, mhz, buf, wps);
    }
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
