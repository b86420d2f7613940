// ubench_pipes.cu -- per-SM issue throughput of the instruction classes the
// u8 decolor kernel is built from (FFMA2/FMUL2/FADD2, MUFU sqrt/rsqrt,
// PRMT, I2F/I2FP conversions, FP64), measured on the B200 itself.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench scripts/ubench_pipes.cu && /tmp/ubench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__device__ __forceinline__ unsigned long long pk(float2 a) { unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y)); return r; }
__device__ __forceinline__ float2 upk(unsigned long long r) { float2 a; asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r)); return a; }

template <int OP>
__global__ void bench(float* out, uint32_t seed) {
    float x[CH]; float2 v[CH]; uint32_t w[CH]; double d[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        x[c] = 1.0f + (threadIdx.x + c) * 1e-3f; v[c] = make_float2(x[c], x[c] + 0.5f);
        w[c] = seed * (threadIdx.x + 17 * c + 1); d[c] = x[c];
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP == 0) {  // FFMA2
                unsigned long long r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(v[c])), "l"(pk(v[c])), "l"(pk(v[c]))); v[c] = upk(r);
            } else if (OP == 1) {  // FFMA scalar 3-reg
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(x[(c + 1) % CH]), "f"(x[(c + 2) % CH]));
            } else if (OP == 2) {  // MUFU.SQRT
                asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
            } else if (OP == 3) {  // MUFU.RSQ
                asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
            } else if (OP == 4) {  // PRMT
                asm volatile("prmt.b32 %0, %0, %1, 0x7440;" : "+r"(w[c]) : "r"(w[(c + 1) % CH]));
            } else if (OP == 5) {  // I2F.U8 byte-select (cvt.rn.f32.u8 on a register)
                float f; asm volatile("{ .reg .u8 b; cvt.u8.u32 b, %1; cvt.rn.f32.u8 %0, b; }" : "=f"(f) : "r"(w[c])); w[c] += __float_as_uint(f);
            } else if (OP == 6) {  // I2FP.F32.U32
                float f; asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(f) : "r"(w[c])); w[c] ^= __float_as_uint(f);
            } else if (OP == 7) {  // FADD2
                unsigned long long r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(v[c])), "l"(pk(v[(c + 1) % CH]))); v[c] = upk(r);
            } else if (OP == 8) {  // DFMA
                asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(d[(c + 1) % CH]), "d"(d[(c + 2) % CH]));
            } else if (OP == 9) {  // FFMA with immediate
                asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A83126F;" : "+f"(x[c]));
            } else if (OP == 10) {  // IADD3-ish integer add
                asm volatile("add.u32 %0, %0, %1;" : "+r"(w[c]) : "r"(w[(c + 3) % CH]));
            } else if (OP == 11) {  // HFMA2
                uint32_t r; asm volatile("fma.rn.f16x2 %0, %1, %1, %1;" : "=r"(r) : "r"(w[c])); w[c] = r;
            } else if (OP == 12) {  // FMNMX
                asm volatile("max.f32 %0, %0, %1;" : "+f"(x[c]) : "f"(x[(c + 1) % CH]));
            }
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) acc += x[c] + v[c].x + v[c].y + __uint_as_float(w[c]) + (float)d[c];
    if (acc == 12345.678f) out[0] = acc;
}

template <int OP>
void run(const char* name, int sms, int clk_khz, float* buf) {
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    bench<OP><<<blocks, threads>>>(buf, 3);
    cudaEventRecord(a);
    bench<OP><<<blocks, threads>>>(buf, 5);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = double(blocks) * threads * ITERS * CH;
    double cycles = ms * 1e-3 * clk_khz * 1e3;
    printf("%-22s %8.2f thread-ops/clk/SM  (%.3f ms @ %d MHz assumed)\n", name, ops / cycles / sms, ms, clk_khz / 1000);
}

int main() {
    int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* buf; cudaMalloc(&buf, 1024);
    run<0>("FFMA2 (x2 lanes)", sms, clk, buf);
    run<1>("FFMA 3-reg", sms, clk, buf);
    run<9>("FFMA imm", sms, clk, buf);
    run<7>("FADD2 (x2 lanes)", sms, clk, buf);
    run<2>("MUFU.SQRT", sms, clk, buf);
    run<3>("MUFU.RSQ", sms, clk, buf);
    run<4>("PRMT", sms, clk, buf);
    run<5>("I2F.U8", sms, clk, buf);
    run<6>("I2FP.F32.U32", sms, clk, buf);
    run<8>("DFMA", sms, clk, buf);
    run<10>("IADD", sms, clk, buf);
    run<11>("HFMA2", sms, clk, buf);
    run<12>("FMNMX", sms, clk, buf);
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
