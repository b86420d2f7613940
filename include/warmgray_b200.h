/*
 * warmgray_b200.h -- C ABI of the B200-native warm/cool decolorization path.
 *
 * This is the drop-in boundary that replaces the reference's kernel-module
 * plugin API (`backend.get_kernels(name)` -> module with `NAME` and
 * `decolor_rows(rgb, out, beta_r, beta_k, row0, row1)`,
 * /root/reference/pkg/src/warmgray/backend.py:44-52, _kernels.pyx:47-56) and
 * the NumPy-only stages the reference runs after it (apply_sigmoid,
 * reinstate_color, quantize_u8 / dequantize_u8; tonemap.py:72-83,172-192,
 * codec.py:22-29).
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch / Python types.
 *  - Return value: 0 = OK; negative = argument error (the Python layer raises
 *    ValueError, like the reference's memoryview / validation errors);
 *    positive = a cudaError_t (raised as RuntimeError). wg_last_error()
 *    returns a thread-local message for the last failing call.
 *  - `wg_*` device entry points take DEVICE pointers and a cudaStream_t
 *    (passed as void*; NULL = legacy default stream). They are asynchronous,
 *    stream-ordered, allocate nothing and are safe to call concurrently on
 *    disjoint outputs (the analogue of decolor_rows being re-entrant over
 *    disjoint row ranges with the GIL released, _kernels.pyx:52).
 *  - `wg_host_*` entry points take HOST pointers (pinned or pageable) plus a
 *    device ordinal; they stream chunks host->device->host through
 *    per-device staging buffers on several CUDA streams and return when the
 *    output is complete (synchronous, like the reference call).
 *  - RGB is interleaved (H, W, 3) row-major (C-contiguous), exactly the
 *    reference's PlanarImage layout (core.py:57-99); a batch of N images is
 *    (N, H, W, 3). Gray is (H, W) / (N, H, W).
 *  - beta_r / beta_k must satisfy 0.5 < beta < 1 (core.py:33-51),
 *    midpoint in [0, 1] and slope > 0 finite (tonemap.py:22-33); violations
 *    return WG_EINVAL.
 *  - There is no CPU fallback: every entry point runs on the GPU or fails.
 */
#ifndef WARMGRAY_B200_H
#define WARMGRAY_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define WG_API __attribute__((visibility("default")))
#else
#define WG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define WG_OK 0
#define WG_EINVAL (-1)      /* bad argument (size, parameter range, null pointer) */
#define WG_EALIGN (-2)      /* misaligned buffer where alignment is mandatory (hdr out / scratch) */
#define WG_ESCRATCH (-3)    /* scratch buffer too small */
#define WG_ENODEV (-4)      /* no CUDA device / bad ordinal */
#define WG_ECODEC (-5)      /* unsupported or malformed image file (reference: CodecError) */
#define WG_EIO (-6)         /* file could not be opened / written (reference: OSError) */

/* ---- host-side container check ---------------------------------------------
 * PlanarImage's validation (core.py:69-80) of n host float64 samples, on host
 * threads: *result = 0 ok, 1 a non-finite sample (checked first, as the
 * reference does), 2 a sample outside [0, 1]. No device work. */
WG_API int wg_host_check_unit_f64(const double* p, int64_t n, int* result);

/* ---- library / device info ------------------------------------------------ */
WG_API int wg_version(void);                              /* 100 * major + minor */
WG_API const char* wg_last_error(void);                   /* thread-local; "" when none */
WG_API int wg_device_count(void);
WG_API int wg_sm_count(int device);

/* ---- peer buffers: the optional final gather fused into the launch (SURVEY.md 8 e) ----
 * The root rank allocates the whole batch's output with wg_ipc_alloc and
 * sends the 64-byte CUDA IPC handle to the other ranks (torch.distributed);
 * each maps it with wg_ipc_open (peer access over NVLink) and passes
 * root_ptr + its shard offset as the `out` of its decolor call, so the shard
 * is stored straight into the root's memory by the kernel. Replaces
 * decolor-then-gather (sharder.gather_to_root); the reference has no
 * collective at all (single process). */
WG_API int wg_ipc_alloc(size_t bytes, int device, void** dptr, uint8_t* handle64);
WG_API int wg_ipc_open(const uint8_t* handle64, int device, void** dptr);
WG_API int wg_ipc_close(void* dptr);
WG_API int wg_ipc_free(void* dptr, int device);

/* ---- device-pointer, stream-ordered hot path ------------------------------ */

/* uint8 RGB -> uint8 gray, i.e. quantize_u8(decolor_image(dequantize_u8(rgb)))
 * (codec.py:22-29 around core.py:147-169 / _kernels.pyx:31-56), fused in one
 * pass over a flat batch of npix pixels: 3 B in, 1 B out per pixel. Identical
 * to the reference except +-1 on rounding ties (5e-6 of all colours; the
 * north-star bar is 1e-4). */
WG_API int wg_decolor_u8(const uint8_t* rgb, uint8_t* gray, int64_t npix, double beta_r, double beta_k,
                  void* stream);
/* Same, bit-identical to the reference for every input (~10% slower): pixels
 * whose fp32 result lies next to a rounding boundary take the exact byte of
 * their colour from a per-(beta_r, beta_k) table settled once over all 2^24
 * colours against the fp64 chain (built on the first call, cached per device). */
WG_API int wg_decolor_u8_exact(const uint8_t* rgb, uint8_t* gray, int64_t npix, double beta_r, double beta_k,
                               void* stream);
/* Diagnostics of that table: boundary margin (2^-15 units), slot count,
 * err, the max |fast - exact| of 255 * gray + 0.5 over all 2^24 colours
 * (2^-15 units, rounded up; the linear exact tone route's margin is err + 2),
 * and err_sq, the max |bits(u_fast) - bits(float((255 v)^2 + 1/8))| of the
 * square-domain route (its exact tone route's margin is err_sq + 1). Any
 * output pointer may be NULL. */
WG_API int wg_u8_exact_info(double beta_r, double beta_k, uint32_t* margin, uint32_t* slots, uint32_t* err,
                            uint32_t* err_sq);

/* fp32 RGB in [0,1] -> fp32 gray (decolor_image on float data; core.py:147-169). */
WG_API int wg_decolor_f32(const float* rgb, float* gray, int64_t npix, float beta_r, float beta_k,
                   void* stream);

/* fp64 RGB -> fp64 gray: replaces _kernels.decolor_rows (_kernels.pyx:47-56)
 * operation for operation in IEEE fp64 without contraction, so the result is
 * bit-identical to the reference's compiled backend. */
WG_API int wg_decolor_f64(const double* rgb, double* gray, int64_t npix, double beta_r, double beta_k,
                   void* stream);

/* apply_sigmoid (tonemap.py:72-83) on fp64 / fp32 luminance. */
WG_API int wg_sigmoid_f64(const double* lum, double* out, int64_t n, double midpoint, double slope,
                   void* stream);
WG_API int wg_sigmoid_f32(const float* lum, float* out, int64_t n, float midpoint, float slope,
                   void* stream);

/* reinstate_color (tonemap.py:172-192) on fp64 data. */
WG_API int wg_reinstate_f64(const double* rgb, const double* l_in, const double* l_out, double* rgb_out,
                     int64_t npix, void* stream);

/* tonemap_image(mode="global") (tonemap.py:195-216) fused in one fp64 pass:
 * decolor -> sigmoid -> reinstate; writes l_out (toned luminance) and rgb_out. */
WG_API int wg_tonemap_global_f64(const double* rgb, double* l_out, double* rgb_out, int64_t npix,
                          double beta_r, double beta_k, double midpoint, double slope,
                          void* stream);

/* Fused decolor + global tone map on uint8 RGB (tonemap.py:72-83 after
 * core.py:147-169, codec.py:22-29):
 * toned = quantize_u8(apply_sigmoid(decolor(rgb/255))); gray_or_null receives
 * quantize_u8(decolor(rgb/255)) when non-NULL. North-star bar (+-1 on rounding
 * ties); wg_decolor_tone_rgb_u8 with rgb_out = NULL is the bit-identical route. */
WG_API int wg_decolor_tone_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray_or_null, int64_t npix,
                       float beta_r, float beta_k, float midpoint, float slope, void* stream);

/* Exact global tone map on uint8, bit-identical to the reference: rgb_out =
 * quantize_u8 of tonemap_image(mode="global")'s reinstated RGB
 * (tonemap.py:172-216), toned = quantize_u8 of its l_out, gray = quantize_u8
 * of l_in; each output may be null (at least one requested). fp32 with a
 * rigorous per-pixel error bound; pixels in doubt take the reference's fp64
 * chain. */
WG_API int wg_decolor_tone_rgb_u8(const uint8_t* rgb, uint8_t* rgb_out, uint8_t* toned_or_null,
                                  uint8_t* gray_or_null, int64_t npix, double beta_r, double beta_k,
                                  double midpoint, double slope, void* stream);

/* Fused decolor + global tone map on fp32 RGB; gray_or_null gets the
 * untoned gray, rgb_out_or_null the reinstated colour (tonemap.py:172-192). */
WG_API int wg_decolor_tone_f32(const float* rgb, float* toned, float* gray_or_null,
                        float* rgb_out_or_null, int64_t npix, float beta_r, float beta_k,
                        float midpoint, float slope, void* stream);

/* codec.py:22-29 on device buffers. */
WG_API int wg_quantize_u8_f64(const double* in, uint8_t* out, int64_t n, void* stream);
WG_API int wg_dequantize_u8_f64(const uint8_t* in, double* out, int64_t n, void* stream);

/* HDR adapter (no reference counterpart):
 * nimg fp32 linear-radiance images of pix_per_img pixels -> uint8 via
 * per-image log-range normalisation of the gray channel, then the global
 * sigmoid. Exact per-CTA min/max partials (no atomics on the statistic); one
 * warp-specialised persistent kernel (cooperative launch) when pix_per_img is
 * a multiple of 32 (the gray of each SM's range staged in tensor memory when
 * it fits, else in an L2-resident ring), else gray / stats / tone kernels.
 * `out` must be 16-byte aligned (WG_EALIGN), `scratch` 256-byte aligned and at
 * least wg_hdr_scratch_bytes() long (WG_ESCRATCH). */
WG_API size_t wg_hdr_scratch_bytes(int64_t nimg, int64_t pix_per_img);
WG_API int wg_hdr_tonemap_u8(const float* rgb, uint8_t* out, int64_t nimg, int64_t pix_per_img,
                      float beta_r, float beta_k, float midpoint, float slope, void* scratch,
                      size_t scratch_bytes, void* stream);
/* Diagnostic (scripts/hdr_trace.py): the tensor-memory kernel's per (image,
 * CTA) globaltimer trace of the last call made with WG_HDR_TMDBG=4, copied to
 * `host` (NULL: only the element count); returns the uint64 count or -1. */
WG_API int64_t wg_hdr_debug_trace(uint64_t* host);

/* ---- baseline luminance extractors (_kernels.pyx:59-132) ----
 * method: 0 = BT.601 luma (bt601_rows, also "weighted"), 1 = HSV V
 * (hsv_value_rows), 2 = CIELAB lightness / 100 (lab_lightness_rows). fp64
 * follows the reference's operation order (BT.601 and V bit-identical; Lab to
 * the last ulp of pow/cbrt). wg_lab_f64 = lab_rows: (L*, a*, b*) per pixel. */
WG_API int wg_luma_f64(const double* rgb, double* out, int64_t npix, int method, void* stream);
WG_API int wg_lab_f64(const double* rgb, double* lab, int64_t npix, void* stream);
WG_API int wg_luma_u8(const uint8_t* rgb, uint8_t* out, int64_t npix, int method, void* stream);

/* ---- local tone map (tonemap.py:36-69, 86-169, 195-216) ----
 * nimg images of height x width, tile-histogram equalisation with tiles of
 * tile_w x tile_h (clamped to the image), `bins` >= 2 histogram bins and
 * blend `strength` in [0, 1] (LocalHistogramGrid). Scratch from
 * wg_lhe_scratch_bytes (0 = invalid arguments). */
WG_API size_t wg_lhe_scratch_bytes(int64_t nimg, int64_t height, int64_t width, int64_t tile_w, int64_t tile_h,
                                   int64_t bins);
/* apply_local_lhe on fp64 luminance: bit-identical to the reference. */
WG_API int wg_local_lhe_f64(const double* lum, double* out, int64_t nimg, int64_t height, int64_t width,
                            int64_t tile_w, int64_t tile_h, int64_t bins, double strength, void* scratch,
                            size_t scratch_bytes, void* stream);
/* tonemap_image(mode="local") on fp64 rgb: gray = decolor, l_out = local lhe of gray,
 * rgb_out = reinstate_color(rgb, gray, l_out). */
WG_API int wg_tonemap_local_f64(const double* rgb, double* gray, double* l_out, double* rgb_out, int64_t nimg,
                                int64_t height, int64_t width, double beta_r, double beta_k, int64_t tile_w,
                                int64_t tile_h, int64_t bins, double strength, void* scratch, size_t scratch_bytes,
                                void* stream);
/* Fused uint8 batch: toned = quantize_u8(apply_local_lhe(decolor(rgb / 255))) and
 * gray_or_null = quantize_u8(decolor(rgb / 255)); bit-identical to the fp64 reference
 * (hence fp64 beta / strength: the exact route evaluates the reference chain with them). */
WG_API int wg_decolor_tone_local_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray_or_null, int64_t nimg,
                                    int64_t height, int64_t width, double beta_r, double beta_k, int64_t tile_w,
                                    int64_t tile_h, int64_t bins, double strength, void* scratch,
                                    size_t scratch_bytes, void* stream);

/* ---- host-buffer entry points (synchronous; pipelined H2D/compute/D2H) ----
 * Each wg_host_X takes host arrays and a device ordinal and replaces the same
 * reference interface as the device entry wg_X above (cited there); results
 * are identical to wg_X's. */

/* bt601_rows / hsv_value_rows / lab_lightness_rows and lab_rows on host fp64
 * buffers, with the plugin's (rgb, out, ..., row0, row1) contract. */
WG_API int wg_host_luma_rows_f64(const double* rgb, double* out, int64_t height, int64_t width, int method,
                                 int64_t row0, int64_t row1, int device);
WG_API int wg_host_lab_rows_f64(const double* rgb, double* lab, int64_t height, int64_t width, int64_t row0,
                                int64_t row1, int device);
WG_API int wg_host_luma_u8(const uint8_t* rgb, uint8_t* out, int64_t npix, int method, int device);

/* The plugin call itself: fills out[row0:row1] of an (height, width) fp64
 * gray image from rgb (height, width, 3) fp64, like
 * _kernels.decolor_rows(rgb, out, beta_r, beta_k, row0, row1). */
WG_API int wg_host_decolor_rows_f64(const double* rgb, double* out, int64_t height, int64_t width,
                             double beta_r, double beta_k, int64_t row0, int64_t row1,
                             int device);
WG_API int wg_host_decolor_u8(const uint8_t* rgb, uint8_t* gray, int64_t npix, double beta_r,
                       double beta_k, int device);
WG_API int wg_host_decolor_u8_exact(const uint8_t* rgb, uint8_t* gray, int64_t npix, double beta_r,
                                    double beta_k, int device);
WG_API int wg_host_decolor_f32(const float* rgb, float* gray, int64_t npix, float beta_r, float beta_k,
                        int device);
WG_API int wg_host_decolor_tone_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray_or_null,
                            int64_t npix, float beta_r, float beta_k, float midpoint,
                            float slope, int device);
WG_API int wg_host_decolor_tone_rgb_u8(const uint8_t* rgb, uint8_t* rgb_out, uint8_t* toned_or_null,
                                       uint8_t* gray_or_null, int64_t npix, double beta_r, double beta_k,
                                       double midpoint, double slope, int device);
WG_API int wg_host_sigmoid_f64(const double* lum, double* out, int64_t n, double midpoint, double slope,
                        int device);
WG_API int wg_host_reinstate_f64(const double* rgb, const double* l_in, const double* l_out,
                          double* rgb_out, int64_t npix, int device);
WG_API int wg_host_tonemap_global_f64(const double* rgb, double* l_out, double* rgb_out, int64_t npix,
                               double beta_r, double beta_k, double midpoint, double slope,
                               int device);
WG_API int wg_host_quantize_u8_f64(const double* in, uint8_t* out, int64_t n, int device);
WG_API int wg_host_dequantize_u8_f64(const uint8_t* in, double* out, int64_t n, int device);
WG_API int wg_host_local_lhe_f64(const double* lum, double* out, int64_t height, int64_t width, int64_t tile_w,
                                 int64_t tile_h, int64_t bins, double strength, int device);
WG_API int wg_host_tonemap_local_f64(const double* rgb, double* l_out, double* rgb_out, int64_t height,
                                     int64_t width, double beta_r, double beta_k, int64_t tile_w, int64_t tile_h,
                                     int64_t bins, double strength, int device);
WG_API int wg_host_decolor_tone_local_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray_or_null, int64_t nimg,
                                         int64_t height, int64_t width, double beta_r, double beta_k, int64_t tile_w,
                                         int64_t tile_h, int64_t bins, double strength, int device);
WG_API int wg_host_hdr_tonemap_u8(const float* rgb, uint8_t* out, int64_t nimg, int64_t pix_per_img,
                           float beta_r, float beta_k, float midpoint, float slope, int device);

/* ---- contrast metrics (metrics.py:84-135) -----------------
 * Pair counts behind CCPR / CCFR / E-score for one (rgb, gray) fp64 image pair
 * of npix pixels: per threshold tau_k (1..15 strictly increasing, positive)
 * the numbers of pairs with delta_e >= tau (colour set), with both >= tau
 * (kept), with gray_diff >= tau (gray set) and gray-but-not-colour
 * (fabricated), delta_e being the CIE76 distance of the pixels' Lab colours
 * and gray_diff |100 g_i - 100 g_j|. pair_i / pair_j (both NULL = all
 * n(n-1)/2 unordered pairs) list the sampled pairs. The device entry writes
 * the (ntau+1)^2 histogram of (#tau <= delta_e, #tau <= gray_diff);
 * wg_metric_counts_from_hist turns it into counts[ntau][4]. */
WG_API size_t wg_metric_scratch_bytes(int64_t npix);
WG_API int wg_metric_hist_f64(const double* rgb, const double* gray, int64_t npix, const double* taus, int ntau,
                              const int64_t* pair_i, const int64_t* pair_j, int64_t npairs,
                              unsigned long long* hist, void* scratch, size_t scratch_bytes, void* stream);
WG_API int wg_metric_counts_from_hist(const unsigned long long* hist, int ntau, int64_t* counts);
WG_API int wg_host_metric_counts_f64(const double* rgb, const double* gray, int64_t npix, const double* taus,
                                     int ntau, const int64_t* pair_i, const int64_t* pair_j, int64_t npairs,
                                     int64_t* counts, int device);

/* ---- uint8 file ingest / egress (codec.py:37-82, 135-140) -----
 * Binary PGM (P5, 1 channel) / PPM (P6, 3 channels), maxval 255, with the
 * reference's header grammar and errors. Host-only; files are read straight
 * into / written from the caller's batch buffer (pinned for the device path),
 * one host thread per file up to `threads`. The batch is n images of
 * height x width x channels uint8. */
WG_API int wg_pnm_probe(const char* path, int64_t* width, int64_t* height, int32_t* channels,
                        int64_t* data_offset);
WG_API int wg_pnm_read_batch(const char* const* paths, int64_t n, uint8_t* dst, int64_t width, int64_t height,
                             int32_t channels, int32_t threads);
WG_API int wg_pnm_write_batch(const char* const* paths, int64_t n, const uint8_t* src, int64_t width,
                              int64_t height, int32_t channels, int32_t threads);

/* ---- synthetic workload generators (bench / test inputs, on device) ------- */

/* C5: i.i.d. uniform bytes from a counter hash of (seed, image, 32-bit word). */
WG_API int wg_synth_uniform_u8(uint8_t* out, int64_t nimg, int64_t bytes_per_img, uint32_t seed,
                        int64_t first_image, void* stream);
/* C3: Voronoi partition (exact int distances, ties -> lowest index) coloured
 * from a per-image table, plus integer noise -4..4, clipped. seeds_xy
 * (nimg, nseeds, 2) int32 and colors (nimg, nseeds, 3) u8 are DEVICE arrays. */
WG_API int wg_synth_voronoi_u8(uint8_t* out, int64_t nimg, int32_t width, int32_t height,
                        const int32_t* seeds_xy, const uint8_t* colors, int32_t nseeds,
                        uint32_t seed, int64_t first_image, void* stream);
/* C2: Gaussian colour blobs over a mid-gray base plus uniform noise, clipped
 * to [0,1]. blobs: (nimg, nblobs, 8) fp32 device table
 * {cx, cy, inv_two_sigma2, amp, r, g, b, 0}; base: (nimg,) fp32. */
WG_API int wg_synth_blobs_f32(float* out, int64_t nimg, int32_t width, int32_t height,
                       const float* blobs, int32_t nblobs, const float* base, float noise,
                       uint32_t seed, int64_t first_image, void* stream);
/* C4: i.i.d. HDR radiance: luminance log-uniform in [lum_lo, lum_hi],
 * saturated hue mixed with white, scaled so BT.709 Y equals the luminance. */
WG_API int wg_synth_hdr_f32(float* out, int64_t nimg, int64_t pix_per_img, float lum_lo, float lum_hi,
                     uint32_t seed, int64_t first_image, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* WARMGRAY_B200_H */
