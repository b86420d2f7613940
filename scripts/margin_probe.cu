// margin_probe.cu -- worst-case error of the fp32 gray estimates over all 2^24
// byte colours against the reference's fp64 chain (decolor_f64 of k/255):
//   fast : decolor_fast_x1(r, g, b) / 255     (MUFU sqrt / rsqrt, 0..255 domain)
//   acc  : decolor_acc(r/255, g/255, b/255)   (IEEE sqrt / rcp)
// The exact-fallback margins in csrc/wg_lhe.cu are set from these numbers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -o margin_probe scripts/margin_probe.cu
#include <cstdio>

#include "../paper_2108_13656_b200/csrc/wg_device.cuh"

using namespace wg;

__global__ void probe(U8Consts k8, AccConsts ka, double br, double bk, unsigned long long* out) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= (1u << 24)) return;
    const uint32_t r = c >> 16, g = (c >> 8) & 255, b = c & 255;
    const double v = decolor_f64(deq_byte(r), deq_byte(g), deq_byte(b), br, bk);
    const double fast = static_cast<double>(decolor_fast_x1(static_cast<float>(r), static_cast<float>(g),
                                                            static_cast<float>(b), k8)) / 255.0;
    const float s = 1.0f / 255.0f;
    const double acc = static_cast<double>(decolor_acc(__fmul_rn(static_cast<float>(r), s),
                                                       __fmul_rn(static_cast<float>(g), s),
                                                       __fmul_rn(static_cast<float>(b), s), ka));
    // max of non-negative doubles via their bit patterns
    atomicMax(&out[0], static_cast<unsigned long long>(__double_as_longlong(fabs(fast - v))));
    atomicMax(&out[1], static_cast<unsigned long long>(__double_as_longlong(fabs(acc - v))));
    if (v > 0) atomicMax(&out[2], static_cast<unsigned long long>(__double_as_longlong(fabs(fast - v) / v)));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 3 * sizeof(unsigned long long));
    const float brs[3] = {0.55f, 0.9f, 0.51f}, bks[3] = {0.8f, 0.6f, 0.99f};
    for (int i = 0; i < 3; ++i) {
        cudaMemset(d, 0, 3 * sizeof(unsigned long long));
        const double br = i == 0 ? 0.55 : (i == 1 ? 0.9 : 0.51), bk = i == 0 ? 0.8 : (i == 1 ? 0.6 : 0.99);
        probe<<<(1 << 24) / 256, 256>>>(make_u8_consts(brs[i], bks[i]), make_acc_consts(brs[i], bks[i]), br, bk, d);
        unsigned long long h[3];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double e[3];
        for (int j = 0; j < 3; ++j) e[j] = __builtin_bit_cast(double, h[j]);
        std::printf("beta (%.2f, %.2f): max|fast-v| %.3e  max|acc-v| %.3e  max rel fast %.3e\n", br, bk, e[0], e[1],
                    e[2]);
    }
    return 0;
}
