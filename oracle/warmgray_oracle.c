/*
 * warmgray_oracle.c -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, fp64, scalar restatement of the reference's per-pixel hot path
 * (package `warmgray`, /root/reference/pkg/src/warmgray). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the CHECKER or as the timed CPU
 * baseline -- never as the product path (the product is the CUDA library in
 * paper_2108_13656_b200/, which has no CPU fallback).
 *
 * Pinning: tests/test_oracle_golden.py checks this restatement against the
 * golden vectors produced by the reference itself (tests/golden/, generated
 * by tests/golden/make_golden.py from both reference backends), including
 * the sha256 of the reference's fp64 output over all 2^24 uint8 colours.
 *
 * Arithmetic provenance: the reference kernel is Cython compiled with
 * `gcc -O3` and no -march (setup.py:9), i.e. SSE2 fp64 without FMA
 * contraction; libm sqrt is correctly rounded. This file is compiled with
 * -O3 -ffp-contract=off and evaluates every expression in the same order,
 * so it is bit-identical to `_kernels.decolor_rows`.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_API __attribute__((visibility("default")))

/* _kernels.pyx:23-28 (_clamp01); core.py:144 */
static inline double clamp01(double v) {
    if (v < 0.0) return 0.0;
    if (v > 1.0) return 1.0;
    return v;
}

/* Eqs. 1-6, following _kernels.pyx:31-44 (_decolor_px) operation for
 * operation; scalar oracle in core.py:102-144 states the same model. */
static inline double decolor_px(double r, double g, double b, double beta_r, double beta_k) {
    double white = sqrt((r * r + g * g + b * b) / 3.0);        /* Eq. 1 */
    double s = r + g + b;
    double wr = 0.0, wb = 0.0;
    if (s > 0.0) {                                              /* black: shares 0 */
        wr = r / s;
        wb = b / s;
    }
    double redgreen = sqrt(beta_r * r * r + (1.0 - beta_r) * g * g);   /* Eq. 3 */
    double warm = wr * redgreen + (1.0 - wr) * white;                 /* Eq. 4 */
    double cool = (1.0 - wb) * b + wb * white;                        /* Eq. 5 (L_B = b, Eq. 2) */
    return clamp01(sqrt(beta_k * warm * warm + (1.0 - beta_k) * cool * cool)); /* Eq. 6 */
}

/* codec.py:22-25: floor(clip(v, 0, 1) * 255 + 0.5) */
static inline uint8_t quantize(double v) {
    double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    return (uint8_t)floor(c * 255.0 + 0.5);
}

/* codec.py:28-29: k / 255.0 */
static inline double dequantize(uint8_t k) { return (double)k / 255.0; }

/* tonemap.py:72-83 (apply_sigmoid): logistic curve renormalised so 0->0, 1->1. */
typedef struct { double m, k, lo, hi; } sig_t;
static inline sig_t sig_make(double m, double k) {
    sig_t s;
    s.m = m;
    s.k = k;
    s.lo = 1.0 / (1.0 + exp(k * m));
    s.hi = 1.0 / (1.0 + exp(-k * (1.0 - m)));
    return s;
}
static inline double sig_apply(const sig_t* s, double x) {
    double y = 1.0 / (1.0 + exp(-s->k * (x - s->m)));
    double out = (y - s->lo) / (s->hi - s->lo);
    return clamp01(out);
}

/* ------------------------------------------------------------------ */
/* row-span thread pool, the analogue of backend.run_rows (backend.py:65-81) */

typedef void (*span_fn)(void* ctx, int64_t p0, int64_t p1);
typedef struct { span_fn fn; void* ctx; int64_t p0, p1; } span_job;

static void* span_thread(void* arg) {
    span_job* j = (span_job*)arg;
    j->fn(j->ctx, j->p0, j->p1);
    return NULL;
}

static void run_spans(int64_t n, int threads, span_fn fn, void* ctx) {
    if (n <= 0) return;
    if (threads < 1) threads = 1;
    if (threads > n) threads = (int)n;
    if (threads == 1) {
        fn(ctx, 0, n);
        return;
    }
    int64_t chunk = (n + threads - 1) / threads;
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    span_job* jobs = (span_job*)calloc((size_t)threads, sizeof(span_job));
    int started = 0;
    for (int t = 0; t < threads; ++t) {
        int64_t p0 = (int64_t)t * chunk, p1 = p0 + chunk > n ? n : p0 + chunk;
        if (p0 >= p1) break;
        jobs[t].fn = fn; jobs[t].ctx = ctx; jobs[t].p0 = p0; jobs[t].p1 = p1;
        if (pthread_create(&tid[t], NULL, span_thread, &jobs[t]) != 0) {
            span_thread(&jobs[t]);  /* degrade to inline on failure */
            tid[t] = 0;
        }
        ++started;
    }
    for (int t = 0; t < started; ++t)
        if (tid[t]) pthread_join(tid[t], NULL);
    free(tid);
    free(jobs);
}

/* ------------------------------------------------------------------ */
/* decolor, fp64 in -> fp64 out (the reference kernel's own representation) */

typedef struct { const double* rgb; double* out; double br, bk; } dec64_ctx;
static void dec64_span(void* c, int64_t p0, int64_t p1) {
    dec64_ctx* x = (dec64_ctx*)c;
    for (int64_t i = p0; i < p1; ++i)
        x->out[i] = decolor_px(x->rgb[3 * i], x->rgb[3 * i + 1], x->rgb[3 * i + 2], x->br, x->bk);
}
OR_API void or_decolor_f64(const double* rgb, double* out, int64_t npix, double beta_r,
                           double beta_k, int threads) {
    dec64_ctx c = {rgb, out, beta_r, beta_k};
    run_spans(npix, threads, dec64_span, &c);
}

/* fp32 samples promoted exactly to fp64 (PlanarImage stores float64; core.py:68) */
typedef struct { const float* rgb; double* out; double br, bk; } dec32_ctx;
static void dec32_span(void* c, int64_t p0, int64_t p1) {
    dec32_ctx* x = (dec32_ctx*)c;
    for (int64_t i = p0; i < p1; ++i)
        x->out[i] = decolor_px((double)x->rgb[3 * i], (double)x->rgb[3 * i + 1],
                               (double)x->rgb[3 * i + 2], x->br, x->bk);
}
OR_API void or_decolor_f32in(const float* rgb, double* out, int64_t npix, double beta_r,
                             double beta_k, int threads) {
    dec32_ctx c = {rgb, out, beta_r, beta_k};
    run_spans(npix, threads, dec32_span, &c);
}

/* uint8 -> uint8: quantize_u8(decolor_image(PlanarImage(dequantize_u8(u8))).data) */
typedef struct { const uint8_t* rgb; uint8_t* out; double br, bk; } dec8_ctx;
static void dec8_span(void* c, int64_t p0, int64_t p1) {
    dec8_ctx* x = (dec8_ctx*)c;
    for (int64_t i = p0; i < p1; ++i)
        x->out[i] = quantize(decolor_px(dequantize(x->rgb[3 * i]), dequantize(x->rgb[3 * i + 1]),
                                        dequantize(x->rgb[3 * i + 2]), x->br, x->bk));
}
OR_API void or_decolor_u8(const uint8_t* rgb, uint8_t* out, int64_t npix, double beta_r,
                          double beta_k, int threads) {
    dec8_ctx c = {rgb, out, beta_r, beta_k};
    run_spans(npix, threads, dec8_span, &c);
}

/* ------------------------------------------------------------------ */
/* baseline luminance extractors, _kernels.pyx:59-132 */

/* D65 sRGB -> XYZ rows and white point, _kernels.pyx:14-20 */
static const double CS_M[3][3] = {{0.4124564, 0.3575761, 0.1804375},
                                  {0.2126729, 0.7151522, 0.0721750},
                                  {0.0193339, 0.1191920, 0.9503041}};
static const double CS_WX = 0.95047, CS_WZ = 1.08883;
#define CS_EPS (216.0 / 24389.0)
#define CS_KAPPA (24389.0 / 27.0)

/* bt601_rows (_kernels.pyx:59-68): weighted sum then clamp */
static inline double cs_bt601(double r, double g, double b) {
    return clamp01(0.2989 * r + 0.5870 * g + 0.1140 * b);
}
/* hsv_value_rows (_kernels.pyx:71-84): strict-greater max, r first */
static inline double cs_hsv_v(double r, double g, double b) {
    double v = r;
    if (g > v) v = g;
    if (b > v) v = b;
    return v;
}
/* _srgb_to_linear / _lab_f (_kernels.pyx:87-96): glibc pow / cbrt */
static inline double cs_lin(double c) { return c <= 0.04045 ? c / 12.92 : pow((c + 0.055) / 1.055, 2.4); }
static inline double cs_f(double t) { return t > CS_EPS ? cbrt(t) : (CS_KAPPA * t + 16.0) / 116.0; }
static inline double cs_row(int k, double lr, double lg, double lb) {
    return CS_M[k][0] * lr + CS_M[k][1] * lg + CS_M[k][2] * lb;
}
/* lab_lightness_rows (_kernels.pyx:99-112) */
static inline double cs_lab_l(double r, double g, double b) {
    double l = 116.0 * cs_f(cs_row(1, cs_lin(r), cs_lin(g), cs_lin(b))) - 16.0;
    return clamp01(l / 100.0);
}
static inline double cs_luma(int method, double r, double g, double b) {
    return method == 0 ? cs_bt601(r, g, b) : method == 1 ? cs_hsv_v(r, g, b) : cs_lab_l(r, g, b);
}

typedef struct { const double* rgb; double* out; int method; } luma64_ctx;
static void luma64_span(void* c, int64_t p0, int64_t p1) {
    luma64_ctx* x = (luma64_ctx*)c;
    for (int64_t i = p0; i < p1; ++i)
        x->out[i] = cs_luma(x->method, x->rgb[3 * i], x->rgb[3 * i + 1], x->rgb[3 * i + 2]);
}
/* method 0 = bt601_rows, 1 = hsv_value_rows, 2 = lab_lightness_rows */
OR_API void or_luma_f64(const double* rgb, double* out, int64_t npix, int method, int threads) {
    luma64_ctx c = {rgb, out, method};
    run_spans(npix, threads, luma64_span, &c);
}

typedef struct { const double* rgb; double* lab; } lab64_ctx;
static void lab64_span(void* c, int64_t p0, int64_t p1) {
    lab64_ctx* x = (lab64_ctx*)c;
    for (int64_t i = p0; i < p1; ++i) {
        const double* p = x->rgb + 3 * i;
        double lr = cs_lin(p[0]), lg = cs_lin(p[1]), lb = cs_lin(p[2]);
        double fx = cs_f(cs_row(0, lr, lg, lb) / CS_WX);
        double fy = cs_f(cs_row(1, lr, lg, lb));
        double fz = cs_f(cs_row(2, lr, lg, lb) / CS_WZ);
        x->lab[3 * i] = 116.0 * fy - 16.0;
        x->lab[3 * i + 1] = 500.0 * (fx - fy);
        x->lab[3 * i + 2] = 200.0 * (fy - fz);
    }
}
/* lab_rows (_kernels.pyx:115-132) */
OR_API void or_lab_f64(const double* rgb, double* lab, int64_t npix, int threads) {
    lab64_ctx c = {rgb, lab};
    run_spans(npix, threads, lab64_span, &c);
}

/* uint8 -> uint8: quantize_u8(luminance_image(dequantize_u8(u8), method).data) */
typedef struct { const uint8_t* rgb; uint8_t* out; int method; } luma8_ctx;
static void luma8_span(void* c, int64_t p0, int64_t p1) {
    luma8_ctx* x = (luma8_ctx*)c;
    for (int64_t i = p0; i < p1; ++i)
        x->out[i] = quantize(cs_luma(x->method, dequantize(x->rgb[3 * i]), dequantize(x->rgb[3 * i + 1]),
                                     dequantize(x->rgb[3 * i + 2])));
}
OR_API void or_luma_u8(const uint8_t* rgb, uint8_t* out, int64_t npix, int method, int threads) {
    luma8_ctx c = {rgb, out, method};
    run_spans(npix, threads, luma8_span, &c);
}

/* ------------------------------------------------------------------ */
/* Contrast metrics: _sweep_counts (metrics.py:84-135) written out per pair.
 * lab = lab_rows of the colour image, g100 = gray * 100; for each pair
 * de = sqrt((d0*d0 + d1*d1) + d2*d2), gd = |g100_i - g100_j|, and per tau the
 * four counts (colour set, kept, gray set, fabricated). pair_i == NULL means
 * all unordered pairs i < j. Threads split the anchor range. */
typedef struct {
    const double* lab; const double* g; int64_t n; const double* taus; int ntau;
    const int64_t* pi; const int64_t* pj; int64_t npairs; int64_t* counts; /* [threads][ntau][4] */
} met_ctx;
static void met_pair(const met_ctx* x, int64_t i, int64_t j, int64_t* c) {
    const double* a = x->lab + 3 * i;
    const double* b = x->lab + 3 * j;
    double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
    double de = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    double gd = fabs(x->g[i] - x->g[j]);
    for (int k = 0; k < x->ntau; ++k) {
        double t = x->taus[k];
        int in_c = de >= t, in_g = gd >= t;
        c[4 * k] += in_c;
        c[4 * k + 1] += in_c && in_g;
        c[4 * k + 2] += in_g;
        c[4 * k + 3] += in_g && !in_c;
    }
}
typedef struct { const met_ctx* m; int64_t* c; int64_t p0, p1; } met_job;
static void* met_thread(void* arg) {
    met_job* jb = (met_job*)arg;
    const met_ctx* x = jb->m;
    if (x->pi) {
        for (int64_t q = jb->p0; q < jb->p1; ++q) met_pair(x, x->pi[q], x->pj[q], jb->c);
    } else {
        for (int64_t i = jb->p0; i < jb->p1; ++i)
            for (int64_t j = i + 1; j < x->n; ++j) met_pair(x, i, j, jb->c);
    }
    return NULL;
}
OR_API void or_metric_counts_f64(const double* rgb, const double* gray, int64_t npix, const double* taus,
                                 int ntau, const int64_t* pair_i, const int64_t* pair_j, int64_t npairs,
                                 int64_t* counts, int threads) {
    memset(counts, 0, sizeof(int64_t) * 4 * (size_t)ntau);
    if (npix < 2) return;
    double* lab = (double*)malloc(sizeof(double) * 3 * (size_t)npix);
    double* g = (double*)malloc(sizeof(double) * (size_t)npix);
    lab64_ctx lc = {rgb, lab};
    lab64_span(&lc, 0, npix);
    for (int64_t p = 0; p < npix; ++p) g[p] = gray[p] * 100.0;
    met_ctx m = {lab, g, npix, taus, ntau, pair_i, pair_j, npairs, NULL};
    int64_t units = pair_i ? npairs : npix - 1;
    if (threads < 1) threads = 1;
    if (threads > units) threads = units > 0 ? (int)units : 1;
    int64_t* part = (int64_t*)calloc((size_t)threads * 4 * (size_t)ntau, sizeof(int64_t));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    met_job* jobs = (met_job*)calloc((size_t)threads, sizeof(met_job));
    for (int t = 0; t < threads; ++t) {
        /* anchors are interleaved so the triangular work balances */
        jobs[t].m = &m;
        jobs[t].c = part + (size_t)t * 4 * (size_t)ntau;
        jobs[t].p0 = units * t / threads;
        jobs[t].p1 = units * (t + 1) / threads;
        if (pthread_create(&tid[t], NULL, met_thread, &jobs[t]) != 0) {
            met_thread(&jobs[t]);
            tid[t] = 0;
        }
    }
    for (int t = 0; t < threads; ++t) {
        if (tid[t]) pthread_join(tid[t], NULL);
        for (int k = 0; k < 4 * ntau; ++k) counts[k] += part[(size_t)t * 4 * (size_t)ntau + (size_t)k];
    }
    free(part);
    free(tid);
    free(jobs);
    free(lab);
    free(g);
}

/* apply_sigmoid on fp64 luminance (tonemap.py:72-83) */
OR_API void or_sigmoid_f64(const double* in, double* out, int64_t n, double midpoint,
                           double slope) {
    sig_t s = sig_make(midpoint, slope);
    for (int64_t i = 0; i < n; ++i) out[i] = sig_apply(&s, in[i]);
}

/* reinstate_color (tonemap.py:172-192): clip(c * l_out / max(l_in, 1e-6)), l_in == 0 -> 0 */
OR_API void or_reinstate_f64(const double* rgb, const double* l_in, const double* l_out,
                             double* out, int64_t npix) {
    for (int64_t i = 0; i < npix; ++i) {
        double li = l_in[i];
        double ratio = l_out[i] / (li > 1e-6 ? li : 1e-6);
        for (int c = 0; c < 3; ++c) {
            double v = clamp01(rgb[3 * i + c] * ratio);
            out[3 * i + c] = li == 0.0 ? 0.0 : v;
        }
    }
}

/* u8 -> toned u8 via the global tone map:
 * quantize_u8(apply_sigmoid(decolor_image(dequantize_u8(u8))).data); optional
 * gray u8 = quantize_u8(decolor_image(...)). */
typedef struct { const uint8_t* rgb; uint8_t* toned; uint8_t* gray; double br, bk; sig_t s; } tone8_ctx;
static void tone8_span(void* c, int64_t p0, int64_t p1) {
    tone8_ctx* x = (tone8_ctx*)c;
    for (int64_t i = p0; i < p1; ++i) {
        double g = decolor_px(dequantize(x->rgb[3 * i]), dequantize(x->rgb[3 * i + 1]),
                              dequantize(x->rgb[3 * i + 2]), x->br, x->bk);
        x->toned[i] = quantize(sig_apply(&x->s, g));
        if (x->gray) x->gray[i] = quantize(g);
    }
}
OR_API void or_tone_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray, int64_t npix,
                       double beta_r, double beta_k, double midpoint, double slope, int threads) {
    tone8_ctx c = {rgb, toned, gray, beta_r, beta_k, sig_make(midpoint, slope)};
    run_spans(npix, threads, tone8_span, &c);
}

/* u8 rgb -> u8 colour tone map: quantize_u8 of tonemap_image(mode="global")'s
 * (rgb_out, l_out) on dequantize_u8(rgb) (tonemap.py:172-216, codec.py:22-29);
 * toned / gray may be NULL. */
typedef struct { const uint8_t* rgb; uint8_t* rgb_out; uint8_t* toned; uint8_t* gray; double br, bk; sig_t s; } tonergb_ctx;
static void tonergb_span(void* c, int64_t p0, int64_t p1) {
    tonergb_ctx* x = (tonergb_ctx*)c;
    for (int64_t i = p0; i < p1; ++i) {
        double r = dequantize(x->rgb[3 * i]), g = dequantize(x->rgb[3 * i + 1]), b = dequantize(x->rgb[3 * i + 2]);
        double li = decolor_px(r, g, b, x->br, x->bk);
        double lo = sig_apply(&x->s, li);
        double ratio = lo / (li > 1e-6 ? li : 1e-6);
        x->rgb_out[3 * i] = li == 0.0 ? 0 : quantize(clamp01(r * ratio));
        x->rgb_out[3 * i + 1] = li == 0.0 ? 0 : quantize(clamp01(g * ratio));
        x->rgb_out[3 * i + 2] = li == 0.0 ? 0 : quantize(clamp01(b * ratio));
        if (x->toned) x->toned[i] = quantize(lo);
        if (x->gray) x->gray[i] = quantize(li);
    }
}
OR_API void or_tone_rgb_u8(const uint8_t* rgb, uint8_t* rgb_out, uint8_t* toned, uint8_t* gray, int64_t npix,
                           double beta_r, double beta_k, double midpoint, double slope, int threads) {
    tonergb_ctx c = {rgb, rgb_out, toned, gray, beta_r, beta_k, sig_make(midpoint, slope)};
    run_spans(npix, threads, tonergb_span, &c);
}

/* fp64 rgb -> (toned luminance, reinstated rgb): tonemap_image(mode="global")
 * (tonemap.py:195-216) = decolor -> apply_sigmoid -> reinstate_color. */
OR_API void or_tonemap_global_f64(const double* rgb, double* l_out, double* rgb_out, int64_t npix,
                                  double beta_r, double beta_k, double midpoint, double slope) {
    sig_t s = sig_make(midpoint, slope);
    for (int64_t i = 0; i < npix; ++i) {
        double li = decolor_px(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], beta_r, beta_k);
        double lo = sig_apply(&s, li);
        l_out[i] = lo;
        double ratio = lo / (li > 1e-6 ? li : 1e-6);
        for (int c = 0; c < 3; ++c) {
            double v = clamp01(rgb[3 * i + c] * ratio);
            rgb_out[3 * i + c] = li == 0.0 ? 0.0 : v;
        }
    }
}

/* ------------------------------------------------------------------ */
/* HDR adapter. No reference counterpart: the
 * reference rejects samples > 1 (core.py:78-79) and lists HDR ingestion as a
 * non-goal. Builder-defined, restated here on top of the
 * reference's own operators:
 *   M  = max over the image's samples;  gn = decolor_image(x / M)  (clamp inactive)
 *   t  = log(gn / gmin) / log(gmax / gmin) over gn > 0, gmin/gmax over gn > 0
 *   t  = 0 where gn == 0;  t = 1 for gn > 0 when gmax == gmin
 *   out = quantize_u8(apply_sigmoid(t, curve))
 * Scale cancels in t, so the device may decolorize the raw radiance. */
typedef struct {
    const float* rgb; uint8_t* out; int64_t ppi; double br, bk; sig_t s;
} hdr_ctx;
static void hdr_span(void* c, int64_t i0, int64_t i1) {
    hdr_ctx* x = (hdr_ctx*)c;
    double* g = (double*)malloc((size_t)x->ppi * sizeof(double));
    for (int64_t im = i0; im < i1; ++im) {
        const float* px = x->rgb + im * x->ppi * 3;
        uint8_t* o = x->out + im * x->ppi;
        double M = 0.0;
        for (int64_t j = 0; j < x->ppi * 3; ++j)
            if ((double)px[j] > M) M = (double)px[j];
        double gmin = INFINITY, gmax = 0.0;
        for (int64_t j = 0; j < x->ppi; ++j) {
            double gv = 0.0;
            if (M > 0.0)
                gv = decolor_px((double)px[3 * j] / M, (double)px[3 * j + 1] / M,
                                (double)px[3 * j + 2] / M, x->br, x->bk);
            g[j] = gv;
            if (gv > 0.0) {
                if (gv < gmin) gmin = gv;
                if (gv > gmax) gmax = gv;
            }
        }
        double lrange = gmax > gmin ? log(gmax / gmin) : 0.0;
        for (int64_t j = 0; j < x->ppi; ++j) {
            double t;
            if (!(g[j] > 0.0)) t = 0.0;
            else if (lrange > 0.0) t = clamp01(log(g[j] / gmin) / lrange);
            else t = 1.0;
            o[j] = quantize(sig_apply(&x->s, t));
        }
    }
    free(g);
}
OR_API void or_hdr_u8(const float* rgb, uint8_t* out, int64_t nimg, int64_t pix_per_img,
                      double beta_r, double beta_k, double midpoint, double slope, int threads) {
    hdr_ctx c = {rgb, out, pix_per_img, beta_r, beta_k, sig_make(midpoint, slope)};
    run_spans(nimg, threads, hdr_span, &c);
}

/* ------------------------------------------------------------------ */
/* Local tone map: apply_local_lhe (tonemap.py:103-169) on one fp64
 * luminance image, written as plain loops in the reference's operation
 * order. Tiles of min(tile, side) pixels (:128-129); bin = min(int(v*nb),
 * nb-1) (:136); per-tile CDF curves clip((cdf-low)/(total-low), 0, 1) with
 * identity tiles where low == total (:139-148); neighbour tiles and blend
 * fractions from the tile centres (_axis_weights, :90-100); bilinear blend
 * and identity mix (:150-166). */

static inline int lhe_bin(double v, int nb) {
    int k = (int)(v * (double)nb);
    return k < nb - 1 ? k : nb - 1;
}

static inline double lhe_centre(int64_t k, int64_t step, int64_t len) {
    int64_t s0 = k * step, s1 = s0 + step < len ? s0 + step : len;
    return (double)(s0 + s1 - 1) / 2.0;
}

/* idx[pos], frac[pos] for one axis of `len` positions split into n spans of `step` */
static void lhe_axis(int64_t len, int64_t step, int n, int* idx, double* frac) {
    for (int64_t pos = 0; pos < len; ++pos) {
        if (n == 1) {
            idx[pos] = 0;
            frac[pos] = 0.0;
            continue;
        }
        int cnt = 0; /* number of centres <= pos (searchsorted side="right") */
        while (cnt < n && lhe_centre(cnt, step, len) <= (double)pos) ++cnt;
        int i = cnt - 1;
        if (i < 0) i = 0;
        if (i > n - 2) i = n - 2;
        double c0 = lhe_centre(i, step, len), c1 = lhe_centre(i + 1, step, len);
        double f = ((double)pos - c0) / (c1 - c0);
        idx[pos] = i;
        frac[pos] = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
    }
}

static void lhe_image(const double* data, double* out, int64_t h, int64_t w, int64_t tile_w, int64_t tile_h,
                      int nb, double strength) {
    if (h == 0 || w == 0) return;
    int64_t tw = tile_w < w ? tile_w : w, th = tile_h < h ? tile_h : h;
    int nx = (int)((w + tw - 1) / tw), ny = (int)((h + th - 1) / th);
    int64_t ntile = (int64_t)nx * ny;
    double* curves = (double*)calloc((size_t)(ntile * nb), sizeof(double));
    char* ident = (char*)calloc((size_t)ntile, 1);
    int64_t* hist = (int64_t*)malloc(sizeof(int64_t) * (size_t)nb);
    for (int ty = 0; ty < ny; ++ty) {
        for (int tx = 0; tx < nx; ++tx) {
            memset(hist, 0, sizeof(int64_t) * (size_t)nb);
            int64_t y1 = (ty + 1) * th < h ? (ty + 1) * th : h, x1 = (tx + 1) * tw < w ? (tx + 1) * tw : w;
            for (int64_t y = ty * th; y < y1; ++y)
                for (int64_t x = tx * tw; x < x1; ++x) hist[lhe_bin(data[y * w + x], nb)]++;
            int64_t total = 0, low = -1;
            for (int k = 0; k < nb; ++k) {
                total += hist[k];
                if (low < 0 && hist[k]) low = total;
            }
            double* c = curves + ((int64_t)ty * nx + tx) * nb;
            if (low == total) {
                ident[(int64_t)ty * nx + tx] = 1;
            } else {
                int64_t cdf = 0;
                for (int k = 0; k < nb; ++k) {
                    cdf += hist[k];
                    double v = (double)(cdf - low) / (double)(total - low);
                    c[k] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                }
            }
        }
    }
    int* xi = (int*)malloc(sizeof(int) * (size_t)w);
    int* yi = (int*)malloc(sizeof(int) * (size_t)h);
    double* xf = (double*)malloc(sizeof(double) * (size_t)w);
    double* yf = (double*)malloc(sizeof(double) * (size_t)h);
    lhe_axis(w, tw, nx, xi, xf);
    lhe_axis(h, th, ny, yi, yf);
    for (int64_t y = 0; y < h; ++y) {
        int j0 = yi[y], j1 = ny > 1 ? j0 + 1 : 0;
        double wy = yf[y];
        for (int64_t x = 0; x < w; ++x) {
            int i0 = xi[x], i1 = nx > 1 ? i0 + 1 : 0;
            double wx = xf[x], v = data[y * w + x];
            int b = lhe_bin(v, nb);
            int64_t t00 = (int64_t)j0 * nx + i0, t01 = (int64_t)j0 * nx + i1;
            int64_t t10 = (int64_t)j1 * nx + i0, t11 = (int64_t)j1 * nx + i1;
            double c00 = ident[t00] ? v : curves[t00 * nb + b];
            double c01 = ident[t01] ? v : curves[t01 * nb + b];
            double c10 = ident[t10] ? v : curves[t10 * nb + b];
            double c11 = ident[t11] ? v : curves[t11 * nb + b];
            double top = c00 + wx * (c01 - c00);
            double bottom = c10 + wx * (c11 - c10);
            double eq = top + wy * (bottom - top);
            out[y * w + x] = clamp01(v + strength * (eq - v));
        }
    }
    free(curves);
    free(ident);
    free(hist);
    free(xi);
    free(yi);
    free(xf);
    free(yf);
}

typedef struct { const double* lum; double* out; int64_t h, w, tw, th; int nb; double s; } lhe_ctx;
static void lhe_span(void* c, int64_t i0, int64_t i1) {
    lhe_ctx* x = (lhe_ctx*)c;
    for (int64_t i = i0; i < i1; ++i)
        lhe_image(x->lum + i * x->h * x->w, x->out + i * x->h * x->w, x->h, x->w, x->tw, x->th, x->nb, x->s);
}
/* nimg images of h x w fp64 luminance, one image per thread */
OR_API void or_local_lhe_f64(const double* lum, double* out, int64_t nimg, int64_t h, int64_t w, int64_t tile_w,
                             int64_t tile_h, int nb, double strength, int threads) {
    lhe_ctx c = {lum, out, h, w, tile_w, tile_h, nb, strength};
    run_spans(nimg, threads, lhe_span, &c);
}

/* uint8 batch: toned = quantize_u8(apply_local_lhe(decolor_image(dequantize_u8(rgb)))),
 * gray = quantize_u8(decolor_image(...)) (gray may be NULL) */
typedef struct {
    const uint8_t* rgb; uint8_t* toned; uint8_t* gray; int64_t h, w, tw, th; int nb; double s, br, bk;
} tonel_ctx;
static void tonel_span(void* c, int64_t i0, int64_t i1) {
    tonel_ctx* x = (tonel_ctx*)c;
    int64_t n = x->h * x->w;
    double* g = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* o = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = i0; i < i1; ++i) {
        const uint8_t* p = x->rgb + i * n * 3;
        for (int64_t k = 0; k < n; ++k)
            g[k] = decolor_px(dequantize(p[3 * k]), dequantize(p[3 * k + 1]), dequantize(p[3 * k + 2]), x->br, x->bk);
        lhe_image(g, o, x->h, x->w, x->tw, x->th, x->nb, x->s);
        for (int64_t k = 0; k < n; ++k) {
            x->toned[i * n + k] = quantize(o[k]);
            if (x->gray) x->gray[i * n + k] = quantize(g[k]);
        }
    }
    free(g);
    free(o);
}
OR_API void or_tone_local_u8(const uint8_t* rgb, uint8_t* toned, uint8_t* gray, int64_t nimg, int64_t h, int64_t w,
                             double beta_r, double beta_k, int64_t tile_w, int64_t tile_h, int nb, double strength,
                             int threads) {
    tonel_ctx c = {rgb, toned, gray, h, w, tile_w, tile_h, nb, strength, beta_r, beta_k};
    run_spans(nimg, threads, tonel_span, &c);
}

/* ------------------------------------------------------------------ */
/* Synthetic-workload restatements (integer-exact, so the device generators
 * in paper_2108_13656_b200/csrc/wg_synth.cu can be checked bit for bit). */

/* lowbias32 integer hash (public-domain mixer by C. Wellons) */
static inline uint32_t mix32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU;
    x ^= x >> 15; x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}
static inline uint32_t hash3(uint32_t seed, uint32_t image, uint32_t ctr) {
    return mix32(ctr ^ mix32(image ^ mix32(seed ^ 0x9e3779b9U)));
}

/* C5: i.i.d. uniform bytes; 32-bit word w of image i holds bytes 4w..4w+3 */
OR_API void or_synth_uniform_u8(uint8_t* out, int64_t nimg, int64_t bytes_per_img,
                                uint32_t seed, int64_t first_image) {
    for (int64_t im = 0; im < nimg; ++im) {
        uint8_t* o = out + im * bytes_per_img;
        for (int64_t j = 0; j < bytes_per_img; ++j) {
            uint32_t h = hash3(seed, (uint32_t)(first_image + im), (uint32_t)(j >> 2));
            o[j] = (uint8_t)(h >> (8 * (j & 3)));
        }
    }
}

/* C3: Voronoi cells, exact integer squared distance, ties -> lowest index;
 * cell colour + per-channel integer noise in -4..4, clipped to 0..255.
 * seeds_xy: (nimg, nseeds, 2) int32; colors: (nimg, nseeds, 3) uint8. */
OR_API void or_synth_voronoi_u8(uint8_t* out, int64_t nimg, int32_t width, int32_t height,
                                const int32_t* seeds_xy, const uint8_t* colors, int32_t nseeds,
                                uint32_t seed, int64_t first_image) {
    for (int64_t im = 0; im < nimg; ++im) {
        const int32_t* sxy = seeds_xy + im * nseeds * 2;
        const uint8_t* col = colors + im * nseeds * 3;
        uint8_t* o = out + im * (int64_t)width * height * 3;
        for (int32_t y = 0; y < height; ++y)
            for (int32_t x = 0; x < width; ++x) {
                int32_t best = 0;
                int64_t bd = INT64_MAX;
                for (int32_t k = 0; k < nseeds; ++k) {
                    int64_t dx = x - sxy[2 * k], dy = y - sxy[2 * k + 1];
                    int64_t d = dx * dx + dy * dy;
                    if (d < bd) { bd = d; best = k; }
                }
                int64_t p = (int64_t)y * width + x;
                uint32_t h = hash3(seed ^ 0x5bd1e995U, (uint32_t)(first_image + im), (uint32_t)p);
                for (int c = 0; c < 3; ++c) {
                    int n = (int)((h >> (10 * c)) & 1023U) % 9 - 4;
                    int v = (int)col[3 * best + c] + n;
                    o[3 * p + c] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
                }
            }
    }
}
