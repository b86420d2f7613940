// wg_host.cu -- host runtime of libwarmgray_b200.so: error reporting, device
// info, and the host-buffer entry points (wg_host_*).
//
// The reference's plugin call `_kernels.decolor_rows(rgb, out, ...)`
// (_kernels.pyx:47-56) consumes host buffers. The wg_host_* entry points keep
// that contract: they stream the caller's host arrays through per-device
// staging buffers in chunks, rotating over kSlots CUDA streams so the
// host->device copy of chunk i+1, the kernel on chunk i and the device->host
// copy of chunk i-1 overlap (PCIe is full duplex), then return when the
// output is complete. Staging buffers are allocated once per context and
// grown on demand (the device-buffer manager); each device keeps a small pool
// of such contexts (streams + staging), and a call leases one for its
// duration, so concurrent host calls on one device (the reference drives
// decolor_rows from a thread pool, backend.py:65-81) overlap instead of
// serialising on a device lock.
// Pageable caller buffers (a NumPy array, the reference's PlanarImage data)
// are staged through per-slot pinned host buffers filled / drained by host
// threads, so their copies overlap the device work like pinned ones.
#include <cuda_runtime.h>

#include <atomic>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/warmgray_b200.h"
#include "wg_internal.h"

namespace wg {

static thread_local std::string t_err;

int set_error(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return code;
}

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(static_cast<int>(e), "%s: %s (%s)", what, cudaGetErrorString(e),
                         cudaGetErrorName(e));
    return WG_OK;
}

static int cuda_fail(cudaError_t e, const char* what) {
    return set_error(static_cast<int>(e), "%s: %s (%s)", what, cudaGetErrorString(e),
                     cudaGetErrorName(e));
}

int sm_count(int device) {
    // idempotent lazy cache; relaxed atomics keep concurrent first calls race-free
    static std::atomic<int> cache[kMaxDevices];
    if (device < 0 || device >= kMaxDevices) return 148;
    if (!cache[device].load(std::memory_order_relaxed)) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = 148;
        }
        cache[device].store(n, std::memory_order_relaxed);
    }
    return cache[device].load(std::memory_order_relaxed);
}

int check_npix(int64_t n) {
    return n < 0 ? set_error(WG_EINVAL, "size must be >= 0, got %lld", static_cast<long long>(n)) : 0;
}

int check_ptrs(int64_t n, const void* a, const void* b) {
    return (n > 0 && (a == nullptr || b == nullptr)) ? set_error(WG_EINVAL, "null buffer pointer") : 0;
}

int check_params(double beta_r, double beta_k) {
    if (!(beta_r > 0.5 && beta_r < 1.0))
        return set_error(WG_EINVAL, "beta_r must lie strictly between 0.5 and 1, got %.17g", beta_r);
    if (!(beta_k > 0.5 && beta_k < 1.0))
        return set_error(WG_EINVAL, "beta_k must lie strictly between 0.5 and 1, got %.17g", beta_k);
    return 0;
}

int check_curve(double midpoint, double slope) {
    if (!(midpoint >= 0.0 && midpoint <= 1.0))
        return set_error(WG_EINVAL, "midpoint must lie in [0, 1], got %.17g", midpoint);
    if (!(slope > 0.0) || std::isinf(slope))
        return set_error(WG_EINVAL, "slope must be a positive finite value, got %.17g", slope);
    return 0;
}

// ---------------------------------------------------------------- device-buffer manager
constexpr int kSlots = 3;
constexpr size_t kChunkBytes = size_t(64) << 20;  // staging bytes per slot (in + out + scratch)

struct Slot {
    cudaStream_t stream = nullptr;
    void* dbuf = nullptr;
    size_t cap = 0;
    void* hbuf = nullptr;  // pinned staging for pageable host buffers (cudaHostAlloc)
    size_t hcap = 0;
};
struct DevCtx {
    bool init = false;
    Slot slots[kSlots];
};
// per-device pool of contexts: a call leases one (creating up to kMaxCtx),
// waiting only when all are in use
constexpr int kMaxCtx = 4;
struct DevPool {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<DevCtx*> free;
    int created = 0;
};
static DevPool g_pool[kMaxDevices];

class CtxLease {
  public:
    explicit CtxLease(int device) : pool_(g_pool[device]) {
        std::unique_lock<std::mutex> lk(pool_.mu);
        pool_.cv.wait(lk, [&] { return !pool_.free.empty() || pool_.created < kMaxCtx; });
        if (!pool_.free.empty()) {
            ctx_ = pool_.free.back();
            pool_.free.pop_back();
        } else {
            ctx_ = new DevCtx();  // lives for the process (like the streams and staging it owns)
            ++pool_.created;
        }
    }
    ~CtxLease() {
        {
            std::lock_guard<std::mutex> lk(pool_.mu);
            pool_.free.push_back(ctx_);
        }
        pool_.cv.notify_one();
    }
    DevCtx& ctx() { return *ctx_; }

  private:
    DevPool& pool_;
    DevCtx* ctx_ = nullptr;
};

class DeviceGuard {
  public:
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev_);
        ok_ = cudaSetDevice(dev);
    }
    ~DeviceGuard() { cudaSetDevice(prev_); }
    cudaError_t status() const { return ok_; }

  private:
    int prev_ = 0;
    cudaError_t ok_ = cudaSuccess;
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct HostIn {
    const void* p;
    size_t bpu;  // bytes per unit
};
struct HostOut {
    void* p;  // may be null (optional output)
    size_t bpu;
};

// Pageable (not page-locked) host memory: a cudaMemcpyAsync from it is staged
// by the driver through its own small bounce buffer and blocks the calling
// thread (~8 GB/s, no overlap). Such buffers go through the slots' pinned
// staging instead, filled and drained by host threads in parallel.
static bool is_pageable(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// memcpy split over up to 8 host threads (the calling thread takes one part):
// one thread copies pageable <-> pinned at ~8-10 GB/s
static void parallel_copy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kPart = size_t(4) << 20;
    static const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>({8, hw, (bytes + kPart - 1) / kPart});
    if (nt <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t per = (bytes + nt - 1) / nt;
    std::vector<std::thread> ts;
    ts.reserve(nt - 1);
    for (size_t t = 1; t < nt; ++t) {
        const size_t a = t * per, b = std::min(bytes, a + per);
        if (a < b)
            ts.emplace_back([=] { std::memcpy(static_cast<uint8_t*>(dst) + a, static_cast<const uint8_t*>(src) + a, b - a); });
    }
    std::memcpy(dst, src, std::min(per, bytes));
    for (std::thread& t : ts) t.join();
}

// Streams `nunits` units (pixels or images) through the device in chunks.
// launch(dev_in[], dev_out[], dev_scratch, n_units, stream) -> WG status.
template <class Launch, class ScratchFn>
static int host_pipeline(int device, int64_t nunits, const HostIn* ins, int nin, const HostOut* outs,
                         int nout, int64_t quantum, ScratchFn scratch_bytes, Launch launch) {
    if (nunits == 0) return WG_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_error(WG_ENODEV, "no CUDA device available (this library has no CPU fallback)");
    }
    if (device < 0 || device >= ndev || device >= kMaxDevices)
        return set_error(WG_ENODEV, "device ordinal %d out of range (have %d)", device, ndev);
    DeviceGuard guard(device);
    if (guard.status() != cudaSuccess) return cuda_fail(guard.status(), "cudaSetDevice");

    size_t bpu = 0;
    for (int i = 0; i < nin; ++i) bpu += ins[i].bpu;
    for (int i = 0; i < nout; ++i) bpu += outs[i].bpu;
    int64_t chunk = static_cast<int64_t>(kChunkBytes / std::max<size_t>(bpu, 1));
    chunk = std::max<int64_t>(quantum, chunk / quantum * quantum);
    chunk = std::min<int64_t>(chunk, (nunits + quantum - 1) / quantum * quantum);

    size_t need = 0;
    for (int i = 0; i < nin; ++i) need += align256(chunk * ins[i].bpu);
    for (int i = 0; i < nout; ++i) need += align256(chunk * outs[i].bpu);
    const size_t scratch = align256(scratch_bytes(chunk));
    need += scratch;
    // pinned staging for the pageable buffers: per slot, their chunks in order
    bool pg_in[4] = {false, false, false, false}, pg_out[4] = {false, false, false, false};
    size_t hneed = 0;
    for (int i = 0; i < nin; ++i)
        if ((pg_in[i] = is_pageable(ins[i].p))) hneed += align256(chunk * ins[i].bpu);
    for (int i = 0; i < nout; ++i)
        if ((pg_out[i] = is_pageable(outs[i].p))) hneed += align256(chunk * outs[i].bpu);

    CtxLease lease(device);
    DevCtx& ctx = lease.ctx();
    if (!ctx.init) {
        for (Slot& s : ctx.slots) {
            cudaError_t e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        }
        ctx.init = true;
    }
    for (Slot& s : ctx.slots) {
        if (s.cap < need) {
            if (s.dbuf) cudaFree(s.dbuf);
            s.dbuf = nullptr;
            s.cap = 0;
            cudaError_t e = cudaMalloc(&s.dbuf, need);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
            s.cap = need;
        }
        if (s.hcap < hneed) {
            if (s.hbuf) cudaFreeHost(s.hbuf);
            s.hbuf = nullptr;
            s.hcap = 0;
            cudaError_t e = cudaHostAlloc(&s.hbuf, hneed, cudaHostAllocDefault);
            if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc(staging)");
            s.hcap = hneed;
        }
    }

    // a slot's pending pageable outputs: (chunk, unit offset, unit count), drained
    // into the caller's buffers once the slot's stream has delivered them
    struct Pending {
        bool active = false;
        int64_t u0 = 0, n = 0;
    } pend[kSlots];
    const auto drain = [&](int si) -> int {
        Slot& s = ctx.slots[si];
        if (!pend[si].active) return WG_OK;
        cudaError_t e = cudaStreamSynchronize(s.stream);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
        uint8_t* h = static_cast<uint8_t*>(s.hbuf);
        for (int i = 0; i < nin; ++i)
            if (pg_in[i]) h += align256(chunk * ins[i].bpu);
        for (int i = 0; i < nout; ++i) {
            if (!pg_out[i]) continue;
            if (outs[i].p)
                parallel_copy(static_cast<uint8_t*>(outs[i].p) + pend[si].u0 * outs[i].bpu, h,
                              pend[si].n * outs[i].bpu);
            h += align256(chunk * outs[i].bpu);
        }
        pend[si].active = false;
        return WG_OK;
    };

    int rc = WG_OK;
    const int64_t nchunks = (nunits + chunk - 1) / chunk;
    for (int64_t c = 0; c < nchunks && rc == WG_OK; ++c) {
        const int si = static_cast<int>(c % kSlots);
        Slot& s = ctx.slots[si];
        if (hneed) {  // the slot's staging is reused: its previous chunk must be complete and drained
            rc = drain(si);
            if (rc != WG_OK) break;
            if (c >= kSlots && !pend[si].active) {
                cudaError_t e = cudaStreamSynchronize(s.stream);
                if (e != cudaSuccess) { rc = cuda_fail(e, "cudaStreamSynchronize"); break; }
            }
        }
        const int64_t u0 = c * chunk;
        const int64_t n = std::min<int64_t>(chunk, nunits - u0);
        uint8_t* cur = static_cast<uint8_t*>(s.dbuf);
        uint8_t* hcur = static_cast<uint8_t*>(s.hbuf);
        const void* din[4] = {nullptr, nullptr, nullptr, nullptr};
        void* dout[4] = {nullptr, nullptr, nullptr, nullptr};
        uint8_t* hout[4] = {nullptr, nullptr, nullptr, nullptr};
        for (int i = 0; i < nin; ++i) {
            din[i] = cur;
            const uint8_t* src = static_cast<const uint8_t*>(ins[i].p) + u0 * ins[i].bpu;
            if (pg_in[i]) {  // pageable: host threads fill the pinned stage, the DMA engine takes it from there
                parallel_copy(hcur, src, n * ins[i].bpu);
                src = hcur;
                hcur += align256(chunk * ins[i].bpu);
            }
            cudaError_t e = cudaMemcpyAsync(cur, src, n * ins[i].bpu, cudaMemcpyHostToDevice, s.stream);
            if (e != cudaSuccess) { rc = cuda_fail(e, "cudaMemcpyAsync H2D"); break; }
            cur += align256(chunk * ins[i].bpu);
        }
        if (rc != WG_OK) break;
        for (int i = 0; i < nout; ++i) {
            dout[i] = outs[i].p ? cur : nullptr;
            cur += align256(chunk * outs[i].bpu);
            if (pg_out[i]) {
                hout[i] = hcur;
                hcur += align256(chunk * outs[i].bpu);
            }
        }
        rc = launch(din, dout, scratch ? static_cast<void*>(cur) : nullptr, n, s.stream);
        if (rc != WG_OK) break;
        for (int i = 0; i < nout; ++i) {
            if (!outs[i].p) continue;
            void* dst = pg_out[i] ? static_cast<void*>(hout[i])
                                  : static_cast<void*>(static_cast<uint8_t*>(outs[i].p) + u0 * outs[i].bpu);
            cudaError_t e = cudaMemcpyAsync(dst, dout[i], n * outs[i].bpu, cudaMemcpyDeviceToHost, s.stream);
            if (e != cudaSuccess) { rc = cuda_fail(e, "cudaMemcpyAsync D2H"); break; }
        }
        if (hneed) pend[si] = {true, u0, n};
    }
    for (int si = 0; si < kSlots; ++si) {
        const int r = hneed ? drain(si) : WG_OK;
        if (r != WG_OK && rc == WG_OK) rc = r;
        cudaError_t e = cudaStreamSynchronize(ctx.slots[si].stream);
        if (e != cudaSuccess && rc == WG_OK) rc = cuda_fail(e, "cudaStreamSynchronize");
    }
    return rc;
}

static size_t no_scratch(int64_t) { return 0; }

// Runs fn(stream) on `device` with a stream of a leased context (device
// checks, lazy stream creation), then synchronises.
template <class F>
static int on_device(int device, F fn) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_error(WG_ENODEV, "no CUDA device available (this library has no CPU fallback)");
    }
    if (device < 0 || device >= ndev || device >= kMaxDevices)
        return set_error(WG_ENODEV, "device ordinal %d out of range (have %d)", device, ndev);
    DeviceGuard guard(device);
    if (guard.status() != cudaSuccess) return cuda_fail(guard.status(), "cudaSetDevice");
    CtxLease lease(device);
    DevCtx& ctx = lease.ctx();
    if (!ctx.init) {
        for (Slot& sl : ctx.slots) {
            cudaError_t e = cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        }
        ctx.init = true;
    }
    cudaStream_t st = ctx.slots[0].stream;
    int rc = fn(st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess && rc == WG_OK) rc = cuda_fail(e, "cudaStreamSynchronize");
    return rc;
}

}  // namespace wg

using namespace wg;

// ====================================================================== info
extern "C" int wg_version(void) { return 100; }

extern "C" const char* wg_last_error(void) { return t_err.c_str(); }

extern "C" int wg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

extern "C" int wg_sm_count(int device) { return sm_count(device); }

// ====================================================================== peer buffers (SURVEY.md 8 e)
// The optional final gather as part of the decolor launch: the root allocates
// the whole batch's output here and shares a CUDA IPC handle (64 bytes, sent
// over torch.distributed); every other rank maps it (peer access over NVLink
// enabled by the open) and its decolor kernel stores its shard straight into
// the root's HBM -- no staging copy and no separate collective.
static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");

extern "C" int wg_ipc_alloc(size_t bytes, int device, void** dptr, uint8_t* handle) {
    if (!dptr || !handle || bytes == 0) return set_error(WG_EINVAL, "ipc_alloc: null pointer or zero size");
    DeviceGuard guard(device);
    if (guard.status() != cudaSuccess) return cuda_fail(guard.status(), "cudaSetDevice");
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);  // its own allocation: the handle's base is the pointer
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(ipc)");
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    std::memcpy(handle, &h, sizeof h);
    *dptr = p;
    return WG_OK;
}

extern "C" int wg_ipc_open(const uint8_t* handle, int device, void** dptr) {
    if (!dptr || !handle) return set_error(WG_EINVAL, "ipc_open: null pointer");
    DeviceGuard guard(device);
    if (guard.status() != cudaSuccess) return cuda_fail(guard.status(), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    return WG_OK;
}

extern "C" int wg_ipc_close(void* dptr) {
    cudaError_t e = cudaIpcCloseMemHandle(dptr);
    return e == cudaSuccess ? WG_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

extern "C" int wg_ipc_free(void* dptr, int device) {
    DeviceGuard guard(device);
    cudaError_t e = cudaFree(dptr);
    return e == cudaSuccess ? WG_OK : cuda_fail(e, "cudaFree(ipc)");
}

// ====================================================================== host-side container check
// PlanarImage's validation (core.py:69-80: finite, then inside [0, 1]) over a
// host float64 array, split over host threads: 0 ok, 1 a non-finite sample,
// 2 a sample outside [0, 1]. The reference's NumPy checks make three passes
// over the samples on one core; this is one pass on up to 16.
extern "C" int wg_host_check_unit_f64(const double* p, int64_t n, int* result) {
    WG_CHECK_ARGS(check_npix(n) || (n > 0 && (!p || !result)) || !result);
    constexpr int64_t kPart = int64_t(1) << 20;
    static const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t nt = std::min<int64_t>({16, static_cast<int64_t>(hw), (n + kPart - 1) / kPart});
    std::vector<int> bad(static_cast<size_t>(std::max<int64_t>(nt, 1)), 0);  // bit 0 non-finite, bit 1 out of range
    const auto scan = [&](int64_t t) {
        const int64_t per = (n + nt - 1) / nt, a = t * per, b = std::min(n, a + per);
        int f = 0;
        for (int64_t i = a; i < b; ++i) {
            const double v = p[i];
            if (!(v - v == 0.0)) f |= 1;         // NaN or +-inf
            else if (v < 0.0 || v > 1.0) f |= 2;  // -0.0 passes, as in NumPy
        }
        bad[static_cast<size_t>(t)] = f;
    };
    if (nt <= 1) {
        if (n > 0) scan(0);
    } else {
        std::vector<std::thread> ts;
        for (int64_t t = 1; t < nt; ++t) ts.emplace_back(scan, t);
        scan(0);
        for (std::thread& t : ts) t.join();
    }
    int f = 0;
    for (int x : bad) f |= x;
    *result = (f & 1) ? 1 : ((f & 2) ? 2 : 0);
    return WG_OK;
}

// ====================================================================== host-buffer entry points
extern "C" int wg_host_decolor_rows_f64(const double* rgb, double* out, int64_t height, int64_t width,
                                        double beta_r, double beta_k, int64_t row0, int64_t row1,
                                        int device) {
    WG_CHECK_ARGS(check_npix(height) || check_npix(width) || check_params(beta_r, beta_k));
    if (row0 < 0 || row1 > height || row0 > row1)
        return set_error(WG_EINVAL, "row range [%lld, %lld) outside [0, %lld]", (long long)row0,
                         (long long)row1, (long long)height);
    const int64_t npix = (row1 - row0) * width;
    WG_CHECK_ARGS(check_ptrs(npix, rgb, out));
    HostIn in[1] = {{rgb + row0 * width * 3, 24}};
    HostOut o[1] = {{out + row0 * width, 8}};
    return host_pipeline(device, npix, in, 1, o, 1, 256, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_decolor_f64(static_cast<const double*>(di[0]),
                                                   static_cast<double*>(dout[0]), n, beta_r, beta_k, st);
                         });
}

extern "C" int wg_host_luma_rows_f64(const double* rgb, double* out, int64_t height, int64_t width, int method,
                                     int64_t row0, int64_t row1, int device) {
    WG_CHECK_ARGS(check_npix(height) || check_npix(width));
    if (row0 < 0 || row1 > height || row0 > row1)
        return set_error(WG_EINVAL, "row range [%lld, %lld) outside [0, %lld]", (long long)row0,
                         (long long)row1, (long long)height);
    if (method < 0 || method > 2) return set_error(WG_EINVAL, "luma method must be 0, 1 or 2");
    const int64_t npix = (row1 - row0) * width;
    WG_CHECK_ARGS(check_ptrs(npix, rgb, out));
    HostIn in[1] = {{rgb + row0 * width * 3, 24}};
    HostOut o[1] = {{out + row0 * width, 8}};
    return host_pipeline(device, npix, in, 1, o, 1, 256, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_luma_f64(static_cast<const double*>(di[0]), static_cast<double*>(dout[0]), n,
                                                method, st);
                         });
}

extern "C" int wg_host_lab_rows_f64(const double* rgb, double* lab, int64_t height, int64_t width, int64_t row0,
                                    int64_t row1, int device) {
    WG_CHECK_ARGS(check_npix(height) || check_npix(width));
    if (row0 < 0 || row1 > height || row0 > row1)
        return set_error(WG_EINVAL, "row range [%lld, %lld) outside [0, %lld]", (long long)row0,
                         (long long)row1, (long long)height);
    const int64_t npix = (row1 - row0) * width;
    WG_CHECK_ARGS(check_ptrs(npix, rgb, lab));
    HostIn in[1] = {{rgb + row0 * width * 3, 24}};
    HostOut o[1] = {{lab + row0 * width * 3, 24}};
    return host_pipeline(device, npix, in, 1, o, 1, 256, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_lab_f64(static_cast<const double*>(di[0]), static_cast<double*>(dout[0]), n, st);
                         });
}

extern "C" int wg_host_luma_u8(const uint8_t* rgb, uint8_t* out, int64_t npix, int method, int device) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, out));
    if (method < 0 || method > 2) return set_error(WG_EINVAL, "luma method must be 0, 1 or 2");
    HostIn in[1] = {{rgb, 3}};
    HostOut o[1] = {{out, 1}};
    return host_pipeline(device, npix, in, 1, o, 1, 4096, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_luma_u8(static_cast<const uint8_t*>(di[0]), static_cast<uint8_t*>(dout[0]), n,
                                               method, st);
                         });
}

extern "C" int wg_host_decolor_u8(const uint8_t* rgb, uint8_t* gray, int64_t npix, double beta_r,
                                  double beta_k, int device) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, gray) || check_params(beta_r, beta_k));
    HostIn in[1] = {{rgb, 3}};
    HostOut o[1] = {{gray, 1}};
    return host_pipeline(device, npix, in, 1, o, 1, 4096, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_decolor_u8(static_cast<const uint8_t*>(di[0]),
                                                  static_cast<uint8_t*>(dout[0]), n, beta_r, beta_k, st);
                         });
}

extern "C" int wg_host_decolor_u8_exact(const uint8_t* rgb, uint8_t* gray, int64_t npix, double beta_r,
                                        double beta_k, int device) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, gray) || check_params(beta_r, beta_k));
    HostIn in[1] = {{rgb, 3}};
    HostOut o[1] = {{gray, 1}};
    return host_pipeline(device, npix, in, 1, o, 1, 4096, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_decolor_u8_exact(static_cast<const uint8_t*>(di[0]),
                                                        static_cast<uint8_t*>(dout[0]), n, beta_r, beta_k, st);
                         });
}

extern "C" int wg_host_decolor_f32(const float* rgb, float* gray, int64_t npix, float beta_r,
                                   float beta_k, int device) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, gray) || check_params(beta_r, beta_k));
    HostIn in[1] = {{rgb, 12}};
    HostOut o[1] = {{gray, 4}};
    return host_pipeline(device, npix, in, 1, o, 1, 1024, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_decolor_f32(static_cast<const float*>(di[0]),
                                                   static_cast<float*>(dout[0]), n, beta_r, beta_k, st);
                         });
}

extern "C" int wg_host_decolor_tone_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray_or_null,
                                       int64_t npix, float beta_r, float beta_k, float midpoint,
                                       float slope, int device) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, toned) || check_params(beta_r, beta_k) ||
                  check_curve(midpoint, slope));
    HostIn in[1] = {{rgb, 3}};
    HostOut o[2] = {{toned, 1}, {gray_or_null, 1}};
    return host_pipeline(device, npix, in, 1, o, 2, 4096, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_decolor_tone_u8(static_cast<const uint8_t*>(di[0]),
                                                       static_cast<uint8_t*>(dout[0]),
                                                       static_cast<uint8_t*>(dout[1]), n, beta_r,
                                                       beta_k, midpoint, slope, st);
                         });
}

extern "C" int wg_host_decolor_tone_rgb_u8(const uint8_t* rgb, uint8_t* rgb_out, uint8_t* toned_or_null,
                                           uint8_t* gray_or_null, int64_t npix, double beta_r, double beta_k,
                                           double midpoint, double slope, int device) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, rgb) || check_params(beta_r, beta_k) ||
                  check_curve(midpoint, slope));
    if (npix > 0 && !rgb_out && !toned_or_null && !gray_or_null)
        return set_error(WG_EINVAL, "decolor_tone_rgb_u8: no output requested");
    HostIn in[1] = {{rgb, 3}};
    HostOut o[3] = {{rgb_out, 3}, {toned_or_null, 1}, {gray_or_null, 1}};
    return host_pipeline(device, npix, in, 1, o, 3, 256, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_decolor_tone_rgb_u8(static_cast<const uint8_t*>(di[0]),
                                                           static_cast<uint8_t*>(dout[0]),
                                                           static_cast<uint8_t*>(dout[1]),
                                                           static_cast<uint8_t*>(dout[2]), n, beta_r, beta_k,
                                                           midpoint, slope, st);
                         });
}

extern "C" int wg_host_sigmoid_f64(const double* lum, double* out, int64_t n, double midpoint,
                                   double slope, int device) {
    WG_CHECK_ARGS(check_npix(n) || check_ptrs(n, lum, out) || check_curve(midpoint, slope));
    HostIn in[1] = {{lum, 8}};
    HostOut o[1] = {{out, 8}};
    return host_pipeline(device, n, in, 1, o, 1, 256, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t k, cudaStream_t st) {
                             return wg_sigmoid_f64(static_cast<const double*>(di[0]),
                                                   static_cast<double*>(dout[0]), k, midpoint, slope, st);
                         });
}

extern "C" int wg_host_reinstate_f64(const double* rgb, const double* l_in, const double* l_out,
                                     double* rgb_out, int64_t npix, int device) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, rgb_out) || check_ptrs(npix, l_in, l_out));
    HostIn in[3] = {{rgb, 24}, {l_in, 8}, {l_out, 8}};
    HostOut o[1] = {{rgb_out, 24}};
    return host_pipeline(device, npix, in, 3, o, 1, 256, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_reinstate_f64(static_cast<const double*>(di[0]),
                                                     static_cast<const double*>(di[1]),
                                                     static_cast<const double*>(di[2]),
                                                     static_cast<double*>(dout[0]), n, st);
                         });
}

extern "C" int wg_host_tonemap_global_f64(const double* rgb, double* l_out, double* rgb_out,
                                          int64_t npix, double beta_r, double beta_k, double midpoint,
                                          double slope, int device) {
    WG_CHECK_ARGS(check_npix(npix) || check_ptrs(npix, rgb, l_out) || check_ptrs(npix, rgb_out, rgb) ||
                  check_params(beta_r, beta_k) || check_curve(midpoint, slope));
    HostIn in[1] = {{rgb, 24}};
    HostOut o[2] = {{l_out, 8}, {rgb_out, 24}};
    return host_pipeline(device, npix, in, 1, o, 2, 256, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t n, cudaStream_t st) {
                             return wg_tonemap_global_f64(static_cast<const double*>(di[0]),
                                                          static_cast<double*>(dout[0]),
                                                          static_cast<double*>(dout[1]), n, beta_r,
                                                          beta_k, midpoint, slope, st);
                         });
}

extern "C" int wg_host_quantize_u8_f64(const double* in_, uint8_t* out, int64_t n, int device) {
    WG_CHECK_ARGS(check_npix(n) || check_ptrs(n, in_, out));
    HostIn in[1] = {{in_, 8}};
    HostOut o[1] = {{out, 1}};
    return host_pipeline(device, n, in, 1, o, 1, 256, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t k, cudaStream_t st) {
                             return wg_quantize_u8_f64(static_cast<const double*>(di[0]),
                                                       static_cast<uint8_t*>(dout[0]), k, st);
                         });
}

extern "C" int wg_host_dequantize_u8_f64(const uint8_t* in_, double* out, int64_t n, int device) {
    WG_CHECK_ARGS(check_npix(n) || check_ptrs(n, in_, out));
    HostIn in[1] = {{in_, 1}};
    HostOut o[1] = {{out, 8}};
    return host_pipeline(device, n, in, 1, o, 1, 256, no_scratch,
                         [&](const void** di, void** dout, void*, int64_t k, cudaStream_t st) {
                             return wg_dequantize_u8_f64(static_cast<const uint8_t*>(di[0]),
                                                         static_cast<double*>(dout[0]), k, st);
                         });
}

// CCPR / CCFR pair counts (metrics.py:84-135) for one (rgb, gray) image pair
extern "C" int wg_host_metric_counts_f64(const double* rgb, const double* gray, int64_t npix, const double* taus,
                                         int ntau, const int64_t* pair_i, const int64_t* pair_j, int64_t npairs,
                                         int64_t* counts, int device) {
    WG_CHECK_ARGS(check_npix(npix) || check_npix(npairs) || check_ptrs(npix, rgb, gray));
    if (!taus || !counts || ntau < 1 || ntau > 15) return set_error(WG_EINVAL, "need 1..15 thresholds and counts");
    if ((pair_i == nullptr) != (pair_j == nullptr)) return set_error(WG_EINVAL, "pair_i / pair_j: both or neither");
    if (pair_i) {
        for (int64_t q = 0; q < npairs; ++q)
            if (pair_i[q] < 0 || pair_i[q] >= npix || pair_j[q] < 0 || pair_j[q] >= npix)
                return set_error(WG_EINVAL, "pair index out of range at %lld", static_cast<long long>(q));
    }
    const int stride = ntau + 1;
    std::vector<unsigned long long> hist(static_cast<size_t>(stride * stride), 0ull);
    int rc = on_device(device, [&](cudaStream_t st) {
        // (the host computes (L*, a*, b*, 100 g) itself: metric_hist_host_lab)
        const size_t b_pairs = pair_i ? align256(static_cast<size_t>(npairs) * 8) : 0;
        const size_t b_hist = align256(hist.size() * 8);
        const size_t b_scratch = wg_metric_scratch_bytes(npix);
        const size_t b_taus = 256;
        uint8_t* d = nullptr;
        const size_t total = 2 * b_pairs + b_hist + b_scratch + b_taus;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), total, st);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(metric)");
        uint8_t* p = d;
        int64_t* d_pi = pair_i ? reinterpret_cast<int64_t*>(p) : nullptr; p += b_pairs;
        int64_t* d_pj = pair_i ? reinterpret_cast<int64_t*>(p) : nullptr; p += b_pairs;
        unsigned long long* d_hist = reinterpret_cast<unsigned long long*>(p); p += b_hist;
        void* d_scratch = p;
        int r = WG_OK;
        auto h2d = [&](void* dst, const void* src, size_t bytes) {
            if (r == WG_OK && bytes) {
                cudaError_t ee = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
                if (ee != cudaSuccess) r = cuda_fail(ee, "cudaMemcpyAsync H2D");
            }
        };
        if (pair_i) {
            h2d(d_pi, pair_i, static_cast<size_t>(npairs) * 8);
            h2d(d_pj, pair_j, static_cast<size_t>(npairs) * 8);
        }
        if (r == WG_OK)  // Lab on the host with the reference's libm, pair loop on the device: exact counts
            r = metric_hist_host_lab(rgb, gray, npix, taus, ntau, d_pi, d_pj, npairs, d_hist, d_scratch, b_scratch,
                                     st);
        if (r == WG_OK) {
            e = cudaMemcpyAsync(hist.data(), d_hist, hist.size() * 8, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) r = cuda_fail(e, "cudaMemcpyAsync D2H");
        }
        cudaFreeAsync(d, st);
        return r;
    });
    if (rc != WG_OK) return rc;
    return wg_metric_counts_from_hist(hist.data(), ntau, counts);
}

// LocalHistogramGrid validation (tonemap.py:45-51), also for empty images
static int check_lhe(int64_t tile_w, int64_t tile_h, int64_t bins, double strength) {
    if (tile_w < 1 || tile_h < 1)
        return set_error(WG_EINVAL, "tile size must be >= 1, got %lldx%lld", static_cast<long long>(tile_w),
                         static_cast<long long>(tile_h));
    if (bins < 2 || bins > (1 << 24))
        return set_error(WG_EINVAL, "bins must lie in [2, 2^24], got %lld", static_cast<long long>(bins));
    if (!(strength >= 0.0 && strength <= 1.0))
        return set_error(WG_EINVAL, "strength must lie in [0, 1], got %.17g", strength);
    return 0;
}

extern "C" int wg_host_local_lhe_f64(const double* lum, double* out, int64_t height, int64_t width, int64_t tile_w,
                                     int64_t tile_h, int64_t bins, double strength, int device) {
    WG_CHECK_ARGS(check_npix(height) || check_npix(width) || check_lhe(tile_w, tile_h, bins, strength));
    const int64_t npix = height * width;
    if (npix == 0) return WG_OK;
    WG_CHECK_ARGS(check_ptrs(1, lum, out));
    HostIn in[1] = {{lum, static_cast<size_t>(npix) * 8}};
    HostOut o[1] = {{out, static_cast<size_t>(npix) * 8}};
    auto scratch = [&](int64_t n) { return wg_lhe_scratch_bytes(n, height, width, tile_w, tile_h, bins); };
    return host_pipeline(device, 1, in, 1, o, 1, 1, scratch,
                         [&](const void** di, void** dout, void* sc, int64_t n, cudaStream_t st) {
                             return wg_local_lhe_f64(static_cast<const double*>(di[0]), static_cast<double*>(dout[0]),
                                                     n, height, width, tile_w, tile_h, bins, strength, sc,
                                                     scratch(n), st);
                         });
}

extern "C" int wg_host_tonemap_local_f64(const double* rgb, double* l_out, double* rgb_out, int64_t height,
                                         int64_t width, double beta_r, double beta_k, int64_t tile_w, int64_t tile_h,
                                         int64_t bins, double strength, int device) {
    WG_CHECK_ARGS(check_npix(height) || check_npix(width) || check_params(beta_r, beta_k) ||
                  check_lhe(tile_w, tile_h, bins, strength));
    const int64_t npix = height * width;
    if (npix == 0) return WG_OK;
    WG_CHECK_ARGS(check_ptrs(1, rgb, l_out) || check_ptrs(1, rgb_out, rgb_out));
    HostIn in[1] = {{rgb, static_cast<size_t>(npix) * 24}};
    HostOut o[2] = {{l_out, static_cast<size_t>(npix) * 8}, {rgb_out, static_cast<size_t>(npix) * 24}};
    // scratch = the decolor gray (l_in) followed by the lhe tables
    const size_t gray_bytes = align256(static_cast<size_t>(npix) * 8);
    auto lhe_bytes = [&](int64_t n) { return wg_lhe_scratch_bytes(n, height, width, tile_w, tile_h, bins); };
    return host_pipeline(device, 1, in, 1, o, 2, 1, [&](int64_t n) { return gray_bytes + lhe_bytes(n); },
                         [&](const void** di, void** dout, void* sc, int64_t n, cudaStream_t st) {
                             uint8_t* base = static_cast<uint8_t*>(sc);
                             return wg_tonemap_local_f64(static_cast<const double*>(di[0]),
                                                         reinterpret_cast<double*>(base),
                                                         static_cast<double*>(dout[0]), static_cast<double*>(dout[1]),
                                                         n, height, width, beta_r, beta_k, tile_w, tile_h, bins,
                                                         strength, base + gray_bytes, lhe_bytes(n), st);
                         });
}

extern "C" int wg_host_decolor_tone_local_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray_or_null, int64_t nimg,
                                             int64_t height, int64_t width, double beta_r, double beta_k,
                                             int64_t tile_w, int64_t tile_h, int64_t bins, double strength,
                                             int device) {
    WG_CHECK_ARGS(check_npix(nimg) || check_npix(height) || check_npix(width) || check_params(beta_r, beta_k) ||
                  check_lhe(tile_w, tile_h, bins, strength));
    const int64_t ppi = height * width;
    if (nimg == 0 || ppi == 0) return WG_OK;
    WG_CHECK_ARGS(check_ptrs(1, rgb, toned));
    HostIn in[1] = {{rgb, static_cast<size_t>(ppi) * 3}};
    HostOut o[2] = {{toned, static_cast<size_t>(ppi)}, {gray_or_null, static_cast<size_t>(ppi)}};
    auto scratch = [&](int64_t n) { return wg_lhe_scratch_bytes(n, height, width, tile_w, tile_h, bins); };
    return host_pipeline(device, nimg, in, 1, o, 2, 1, scratch,
                         [&](const void** di, void** dout, void* sc, int64_t n, cudaStream_t st) {
                             return wg_decolor_tone_local_u8(static_cast<const uint8_t*>(di[0]),
                                                             static_cast<uint8_t*>(dout[0]),
                                                             static_cast<uint8_t*>(dout[1]), n, height, width,
                                                             beta_r, beta_k, tile_w, tile_h, bins, strength, sc,
                                                             scratch(n), st);
                         });
}

extern "C" int wg_host_hdr_tonemap_u8(const float* rgb, uint8_t* out, int64_t nimg, int64_t pix_per_img,
                                      float beta_r, float beta_k, float midpoint, float slope,
                                      int device) {
    WG_CHECK_ARGS(check_npix(nimg) || check_npix(pix_per_img) || check_params(beta_r, beta_k) ||
                  check_curve(midpoint, slope));
    if (nimg == 0 || pix_per_img == 0) return WG_OK;
    WG_CHECK_ARGS(check_ptrs(1, rgb, out));
    HostIn in[1] = {{rgb, static_cast<size_t>(pix_per_img) * 12}};
    HostOut o[1] = {{out, static_cast<size_t>(pix_per_img)}};
    return host_pipeline(device, nimg, in, 1, o, 1, 1,
                         [&](int64_t chunk) { return wg_hdr_scratch_bytes(chunk, pix_per_img); },
                         [&](const void** di, void** dout, void* scratch, int64_t n, cudaStream_t st) {
                             return wg_hdr_tonemap_u8(static_cast<const float*>(di[0]),
                                                      static_cast<uint8_t*>(dout[0]), n, pix_per_img,
                                                      beta_r, beta_k, midpoint, slope, scratch,
                                                      wg_hdr_scratch_bytes(n, pix_per_img), st);
                         });
}
