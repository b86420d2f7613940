// wg_internal.h -- host-side helpers shared by the translation units of
// libwarmgray_b200.so (error reporting, argument checks, device info).
#pragma once

#include <mutex>

#include <cstdint>
#include <cuda_runtime.h>

namespace wg {

constexpr int kMaxDevices = 64;

// Records a thread-local message for wg_last_error() and returns `code`.
int set_error(int code, const char* fmt, ...);
// cudaGetLastError() after a launch: 0, or the (positive) cudaError_t with a message.
int check_launch(const char* what);
// Cached multiprocessor count of `device` (148 on B200).
int sm_count(int device);

// Argument checks: return nonzero (after recording a message) on failure.
int check_npix(int64_t n);
int check_ptrs(int64_t n, const void* a, const void* b);
int check_params(double beta_r, double beta_k);   // core.py:33-51: 0.5 < beta < 1
int check_curve(double midpoint, double slope);   // tonemap.py:22-33

struct U8Exact;
// Near-tie table of the bit-exact uint8 decolor for (beta_r, beta_k) on the
// current device (csrc/wg_u8exact.cu); built on first use, then cached.
// `hold` returns locked; keep it until the kernel using the table is enqueued.
int u8exact_get(double beta_r, double beta_k, U8Exact* out, std::unique_lock<std::mutex>* hold);

// Contrast-metric pair counts of host arrays (csrc/wg_metrics.cu): (L*, a*, b*,
// 100 g) on host threads with the platform libm (bit-identical to the
// reference's lab_rows), the pair loop on the device; `hist` and `scratch` are
// device buffers, pair_i / pair_j device arrays or null (all pairs).
int metric_hist_host_lab(const double* rgb, const double* gray, int64_t npix, const double* taus, int ntau,
                         const int64_t* pair_i, const int64_t* pair_j, int64_t npairs, unsigned long long* hist,
                         void* scratch, size_t scratch_bytes, cudaStream_t st);

}  // namespace wg

#define WG_CHECK_ARGS(failed) \
    do {                      \
        if (failed) return WG_EINVAL; \
    } while (0)
