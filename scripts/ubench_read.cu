// ubench_read.cu -- HBM bandwidth by read:write mix on the B200: streams a
// 4 GiB buffer with 128-bit loads (evict-first) and writes 1/k of the bytes
// (k = 0: reads only), three 128-bit loads per thread per iteration with the
// next three in flight (the kernels' pattern), grid = 8 CTAs of 256 threads per SM. Tells how far the read-dominant kernels (C2 f32: 3:1,
// C4 HDR: 12:1) can go above the 1:1 copy peak of MEASURED_PEAKS.json.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubr scripts/ubench_read.cu && /tmp/ubr
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// U vectors (16 B) per thread per iteration, the next U in flight (register prefetch)
template <int U>
__global__ void __launch_bounds__(256) mix_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t n,
                                                  int wk, uint32_t* sink) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * U;
    uint32_t acc = 0;
    int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * U;
    uint4 nx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) nx[u] = i + u < n ? __ldcs(in + i + u) : make_uint4(0, 0, 0, 0);
    for (; i < n; i += stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = nx[u];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + stride + u < n) nx[u] = __ldcs(in + i + stride + u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (i + u >= n) break;
            acc ^= v[u].x + v[u].y + v[u].z + v[u].w;
            if (wk && ((i + u) % wk) == 0) __stcs(out + (i + u) / wk, v[u]);
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;  // keeps the loads alive
}

int main() {
    const size_t bytes = size_t(4) << 30;
    const int64_t n = bytes / 16;
    uint4 *in, *out;
    uint32_t* sink;
    cudaMalloc(&in, bytes);
    cudaMalloc(&out, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(in, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int wk : {0, 12, 4, 1}) {
        for (int rep = 0; rep < 2; ++rep) mix_kernel<3><<<8 * sms, 256>>>(in, out, n, wk, sink);
        cudaEventRecord(a);
        const int iters = 10;
        for (int rep = 0; rep < iters; ++rep) mix_kernel<3><<<8 * sms, 256>>>(in, out, n, wk, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); return 1; }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double rd = double(bytes) * iters, wr = wk ? rd / wk : 0.0;
        printf("{\"read_write_ratio\": \"%s\", \"read_gbs\": %.1f, \"write_gbs\": %.1f, \"total_gbs\": %.1f}\n",
               wk ? (wk == 1 ? "1:1" : (wk == 4 ? "4:1" : "12:1")) : "read only", rd / ms / 1e6, wr / ms / 1e6,
               (rd + wr) / ms / 1e6);
    }
    return 0;
}
