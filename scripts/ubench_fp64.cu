// ubench_fp64.cu -- can the FP64 pipe take work off the saturated FMA / XU
// pipes of the u8 decolor kernel? Measures per-SM throughput of DFMA / DADD,
// the f32 <-> f64 conversions, and mixes (DFMA + FFMA2, F2F + MUFU) to see
// which pipes overlap on the B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubf scripts/ubench_fp64.cu && /tmp/ubf
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int CH = 8;

__device__ __forceinline__ unsigned long long pk(float2 a) { unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y)); return r; }
__device__ __forceinline__ float2 upk(unsigned long long r) { float2 a; asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r)); return a; }

// OP bit set: 1 DFMA, 2 FFMA2, 4 MUFU.SQRT, 8 F2F.F32.F64, 16 F2F.F64.F32, 32 DADD
template <int OP>
__global__ void bench(float* out, uint32_t seed) {
    float x[CH]; float2 v[CH]; double d[CH], e[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        x[c] = 1.0f + (threadIdx.x + c + seed) * 1e-3f; v[c] = make_float2(x[c], x[c] + 0.5f);
        d[c] = x[c]; e[c] = x[c] * 0.5;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP & 1) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(d[(c + 1) % CH]), "d"(d[(c + 2) % CH]));
            if (OP & 2) {
                unsigned long long r;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(v[c])), "l"(pk(v[(c + 1) % CH])), "l"(pk(v[(c + 2) % CH])));
                v[c] = upk(r);
            }
            if (OP & 4) asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
            if (OP & 8) { float f; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(e[c])); e[c] += (double)0 * f; x[c] += f * 0.0f; asm volatile("" :: "f"(f)); }
            if (OP & 16) { double t; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(x[(c + 3) % CH])); asm volatile("" :: "d"(t)); }
            if (OP & 32) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(e[c]) : "d"(e[(c + 1) % CH]));
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) acc += x[c] + v[c].x + v[c].y + (float)d[c] + (float)e[c];
    if (acc == 12345.678f) out[0] = acc;
}

template <int OP>
void run(const char* name, int sms, float* buf) {
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    bench<OP><<<blocks, threads>>>(buf, 3);
    cudaEventRecord(a);
    bench<OP><<<blocks, threads>>>(buf, 5);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    // per-SM rate of "one iteration of the mix" per thread, and the clock seen by clock64 is not needed:
    // report ns per 1M thread-iterations-per-SM so mixes compare to their parts directly
    double iters = double(blocks) * threads * ITERS * CH / sms;
    printf("%-28s %8.3f ms   %7.2f thread-iters/ns/SM\n", name, ms, iters / (ms * 1e6));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* buf; cudaMalloc(&buf, 1024);
    run<1>("DFMA", sms, buf);
    run<32>("DADD", sms, buf);
    run<2>("FFMA2", sms, buf);
    run<4>("MUFU.SQRT", sms, buf);
    run<8>("F2F.F32.F64", sms, buf);
    run<16>("F2F.F64.F32", sms, buf);
    run<1 | 2>("DFMA + FFMA2", sms, buf);
    run<4 | 8>("MUFU.SQRT + F2F.F32.F64", sms, buf);
    run<4 | 16>("MUFU.SQRT + F2F.F64.F32", sms, buf);
    run<2 | 8>("FFMA2 + F2F.F32.F64", sms, buf);
    run<1 | 4>("DFMA + MUFU.SQRT", sms, buf);
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
