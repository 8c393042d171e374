/* skoracle.c — CPU restatement of the spectralkit transform path. TEST INFRASTRUCTURE ONLY
 * (see skoracle.h). Every function cites the reference lines it restates
 * (paths relative to /root/reference/proj/src). fp64, same operation order as the
 * reference's std::complex<double> arithmetic: (a+ib)(c+id) = (ac-bd) + i(ad+bc).
 */
#define _GNU_SOURCE
#include "skoracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static const double kPi = 3.141592653589793238462643383279502884; /* std::numbers::pi */
#define TWO_PI (2.0 * kPi)

static __thread char g_err[256];
const char* sko_last_error(void) { return g_err; }
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return 1;
}

typedef struct { double re, im; } cx;
static inline cx cmul(cx a, cx b) {
    cx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    return r;
}
static inline cx cadd(cx a, cx b) { cx r = {a.re + b.re, a.im + b.im}; return r; }
static inline cx csub(cx a, cx b) { cx r = {a.re - b.re, a.im - b.im}; return r; }
static inline cx cscale(cx a, double s) { cx r = {a.re * s, a.im * s}; return r; }

/* numerics.cpp:14 */
int sko_is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }

/* numerics.cpp:16-24 */
size_t sko_next_pow2(size_t n) {
    if (n == 0) { fail("next_pow2: n must be >= 1"); return 0; }
    size_t p = 1;
    while (p < n) {
        if (p > ((size_t)1 << 62)) { fail("next_pow2: overflow"); return 0; }
        p <<= 1;
    }
    return p;
}

/* numerics.cpp:122-128: fma split of q*t, reduced to [-1/2, 1/2] cycles */
static cx cis_cycles(double q, double t) {
    const double hi = q * t;
    const double lo = fma(q, t, -hi);
    const double frac = (hi - nearbyint(hi)) + lo;
    const double ang = TWO_PI * frac;
    cx r = {cos(ang), sin(ang)};
    return r;
}
void sko_cis_cycles(double q, double t, double out[2]) {
    cx v = cis_cycles(q, t);
    out[0] = v.re;
    out[1] = v.im;
}

/* ---- FftPlan: numerics.cpp:52-100 ------------------------------------------------ */
struct sko_fft_plan {
    size_t n;
    unsigned log2n;
    cx* tw;   /* exp(-i 2 pi k / n), k < n/2 */
    cx* itw;  /* conjugates */
    uint32_t* bitrev;
};

sko_fft_plan* sko_fft_plan_create(size_t n) {
    if (!sko_is_pow2(n)) { fail("FftPlan: size must be a power of two"); return NULL; }
    sko_fft_plan* p = (sko_fft_plan*)calloc(1, sizeof *p);
    p->n = n;
    while (((size_t)1 << p->log2n) < n) ++p->log2n;
    size_t h = n / 2 ? n / 2 : 1;
    p->tw = (cx*)malloc(h * sizeof(cx));
    p->itw = (cx*)malloc(h * sizeof(cx));
    for (size_t k = 0; k < n / 2; ++k) {
        const double ang = -TWO_PI * (double)k / (double)n;   /* numerics.cpp:60 */
        p->tw[k].re = cos(ang);
        p->tw[k].im = sin(ang);
        p->itw[k].re = p->tw[k].re;
        p->itw[k].im = -p->tw[k].im;
    }
    p->bitrev = (uint32_t*)malloc(n * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) {
        uint32_t r = 0;
        for (unsigned b = 0; b < p->log2n; ++b)
            if (i & ((size_t)1 << b)) r |= (uint32_t)1 << (p->log2n - 1 - b);
        p->bitrev[i] = r;
    }
    return p;
}

void sko_fft_plan_free(sko_fft_plan* p) {
    if (!p) return;
    free(p->tw);
    free(p->itw);
    free(p->bitrev);
    free(p);
}

/* numerics.cpp:73-97 — bit-reversal swaps, log2 n radix-2 DIT stages, 1/n on inverse */
int sko_fft_plan_run(const sko_fft_plan* p, double* data, size_t n, int invert) {
    if (n != p->n) return fail("FftPlan: buffer size does not match plan");
    cx* a = (cx*)data;
    for (size_t i = 0; i < n; ++i) {
        const size_t j = p->bitrev[i];
        if (i < j) { cx t = a[i]; a[i] = a[j]; a[j] = t; }
    }
    const cx* tw = invert ? p->itw : p->tw;
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len >> 1;
        const size_t stride = n / len;
        for (size_t base = 0; base < n; base += len) {
            for (size_t j = 0; j < half; ++j) {
                const cx w = tw[j * stride];
                const cx t = cmul(w, a[base + half + j]);
                const cx u = a[base + j];
                a[base + j] = cadd(u, t);
                a[base + half + j] = csub(u, t);
            }
        }
    }
    if (invert) {
        const double s = 1.0 / (double)n;
        for (size_t i = 0; i < n; ++i) a[i] = cscale(a[i], s);
    }
    return 0;
}

/* numerics.cpp:102-120 */
int sko_fft(const double* x, size_t n, int invert, double* out) {
    if (n == 0) return fail("fft: empty input");
    if (!sko_is_pow2(n)) {
        snprintf(g_err, sizeof g_err, "fft: length %zu is not a power of two; zero_pad to %zu first",
                 n, sko_next_pow2(n));
        return 1;
    }
    memmove(out, x, n * 2 * sizeof(double));
    sko_fft_plan* p = sko_fft_plan_create(n);
    int rc = sko_fft_plan_run(p, out, n, invert);
    sko_fft_plan_free(p);
    return rc;
}

/* numerics.cpp:35-50 — exact integer phase index (k*m) mod n */
int sko_dft_naive(const double* xin, size_t n, double* out) {
    if (n == 0) return fail("dft_naive: empty input");
    const cx* x = (const cx*)xin;
    cx* tw = (cx*)malloc(n * sizeof(cx));
    for (size_t r = 0; r < n; ++r) {
        const double ang = -TWO_PI * (double)r / (double)n;
        tw[r].re = cos(ang);
        tw[r].im = sin(ang);
    }
    cx* o = (cx*)out;
    for (size_t k = 0; k < n; ++k) {
        cx acc = {0.0, 0.0};
        for (size_t m = 0; m < n; ++m) acc = cadd(acc, cmul(x[m], tw[(k * m) % n]));
        o[k] = acc;
    }
    free(tw);
    return 0;
}

/* ---- CZT: czt.cpp ------------------------------------------------------------------ */
/* czt.cpp:15-32 PolarPow: z^t = |z|^t exp(i 2 pi q t), |log|z|| < 1e-14 snapped to 0 */
typedef struct { double log_mag, q; } polar_pow;
static int polar_init(polar_pow* pp, const double z[2]) {
    const double mag = hypot(z[0], z[1]);
    if (!(mag > 0.0)) return fail("czt: parameter magnitude is zero");
    pp->log_mag = log(mag);
    if (fabs(pp->log_mag) < 1e-14) pp->log_mag = 0.0;
    pp->q = atan2(z[1], z[0]) / (2.0 * kPi);
    return 0;
}
static cx polar_pow_at(const polar_pow* pp, double t) {
    cx u = cis_cycles(pp->q, t);
    if (pp->log_mag != 0.0) u = cscale(u, exp(pp->log_mag * t));
    return u;
}

/* czt.cpp:36-40 */
static int validate_params(const double a[2], const double w[2], size_t m) {
    if (m == 0) return fail("czt: m must be >= 1");
    if (!(hypot(a[0], a[1]) > 0.0) || !(hypot(w[0], w[1]) > 0.0))
        return fail("czt: a and w must be nonzero");
    return 0;
}

/* czt.cpp:42-56 */
int sko_czt_params_for_band(double f1, double f2, double fs, size_t m, double a[2], double w[2]) {
    if (!(fs > 0.0)) return fail("czt_params_for_band: sample rate must be positive");
    if (!(f1 >= 0.0) || !(f1 < f2)) return fail("czt_params_for_band: need 0 <= f1 < f2");
    if (f2 > fs * (1.0 + 1e-12)) return fail("czt_params_for_band: f2 exceeds the sample rate");
    if (m < 2) return fail("czt_params_for_band: m must be >= 2");
    sko_cis_cycles(f1 / fs, 1.0, a);
    sko_cis_cycles(-(f2 - f1) / ((double)m * fs), 1.0, w);
    return 0;
}

/* czt.cpp:58-75 — literal O(n m) sum */
int sko_czt_direct(const double* xin, size_t n, const double a[2], const double w[2], size_t m,
                   double* out) {
    if (validate_params(a, w, m)) return 1;
    if (n == 0) return fail("czt_direct: empty input");
    polar_pow A, W;
    if (polar_init(&A, a) || polar_init(&W, w)) return 1;
    const cx* x = (const cx*)xin;
    cx* xa = (cx*)malloc(n * sizeof(cx));
    for (size_t i = 0; i < n; ++i) xa[i] = cmul(x[i], polar_pow_at(&A, -(double)i));
    cx* o = (cx*)out;
    for (size_t k = 0; k < m; ++k) {
        cx acc = {0.0, 0.0};
        for (size_t i = 0; i < n; ++i)
            acc = cadd(acc, cmul(xa[i], polar_pow_at(&W, (double)k * (double)i)));
        o[k] = acc;
    }
    free(xa);
    return 0;
}

struct sko_czt_plan {
    size_t n, m, L;
    sko_fft_plan* fft;
    cx* in_chirp;   /* a^-i w^(i^2/2) */
    cx* out_chirp;  /* w^(k^2/2) */
    cx* kernel;     /* FFT of circular w^(-j^2/2) */
};

/* czt.cpp:78-114 */
sko_czt_plan* sko_czt_plan_create(size_t n, const double a[2], const double w[2], size_t m) {
    if (validate_params(a, w, m)) return NULL;
    if (n == 0) { fail("CztPlan: empty input length"); return NULL; }
    polar_pow A, W;
    if (polar_init(&A, a) || polar_init(&W, w)) return NULL;
    sko_czt_plan* p = (sko_czt_plan*)calloc(1, sizeof *p);
    p->n = n;
    p->m = m;
    p->L = sko_next_pow2(n + m - 1);
    p->fft = sko_fft_plan_create(p->L);
    p->in_chirp = (cx*)malloc(n * sizeof(cx));
    for (size_t i = 0; i < n; ++i) {
        const double t = (double)i;
        p->in_chirp[i] = cmul(polar_pow_at(&A, -t), polar_pow_at(&W, 0.5 * t * t));
    }
    p->out_chirp = (cx*)malloc(m * sizeof(cx));
    for (size_t k = 0; k < m; ++k) {
        const double t = (double)k;
        p->out_chirp[k] = polar_pow_at(&W, 0.5 * t * t);
    }
    p->kernel = (cx*)calloc(p->L, sizeof(cx));
    for (size_t k = 0; k < m; ++k) {
        const double t = (double)k;
        p->kernel[k] = polar_pow_at(&W, -0.5 * t * t);
    }
    for (size_t i = 1; i < n; ++i) {
        const double t = (double)i;
        p->kernel[p->L - i] = polar_pow_at(&W, -0.5 * t * t);
    }
    sko_fft_plan_run(p->fft, (double*)p->kernel, p->L, 0);
    return p;
}

void sko_czt_plan_free(sko_czt_plan* p) {
    if (!p) return;
    sko_fft_plan_free(p->fft);
    free(p->in_chirp);
    free(p->out_chirp);
    free(p->kernel);
    free(p);
}

size_t sko_czt_plan_conv_size(const sko_czt_plan* p) { return p->L; }

/* czt.cpp:116-130 */
int sko_czt_execute(const sko_czt_plan* p, const double* xin, double* scratch, double* out) {
    const cx* x = (const cx*)xin;
    cx* s = (cx*)scratch;
    int own = 0;
    if (!s) { s = (cx*)malloc(p->L * sizeof(cx)); own = 1; }
    for (size_t i = 0; i < p->n; ++i) s[i] = cmul(x[i], p->in_chirp[i]);
    for (size_t i = p->n; i < p->L; ++i) { s[i].re = 0.0; s[i].im = 0.0; }
    sko_fft_plan_run(p->fft, (double*)s, p->L, 0);
    for (size_t j = 0; j < p->L; ++j) s[j] = cmul(s[j], p->kernel[j]);
    sko_fft_plan_run(p->fft, (double*)s, p->L, 1);
    cx* o = (cx*)out;
    for (size_t k = 0; k < p->m; ++k) o[k] = cmul(s[k], p->out_chirp[k]);
    if (own) free(s);
    return 0;
}

/* czt.cpp:139-142 */
int sko_czt(const double* x, size_t n, const double a[2], const double w[2], size_t m, double* out) {
    if (n == 0) return fail("czt: empty input");
    sko_czt_plan* p = sko_czt_plan_create(n, a, w, m);
    if (!p) return 1;
    sko_czt_execute(p, x, NULL, out);
    sko_czt_plan_free(p);
    return 0;
}

/* czt.cpp:144-153 */
int sko_dft_any(const double* x, size_t n, double* out) {
    if (n == 0) return fail("dft_any: empty input");
    if (sko_is_pow2(n)) return sko_fft(x, n, 0, out);
    double a[2] = {1.0, 0.0}, w[2];
    sko_cis_cycles(-1.0 / (double)n, 1.0, w);
    return sko_czt(x, n, a, w, n, out);
}

/* ---- spectra.cpp:21-61 --------------------------------------------------------------- */
static int validate_trace(const double* s, size_t n, double fs) {   /* types.cpp:20-27 */
    if (n == 0) return fail("trace: no samples");
    if (!(fs > 0.0) || !isfinite(fs)) return fail("trace: sample rate must be positive and finite");
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(s[i])) return fail("trace: non-finite sample");
    return 0;
}

int sko_fft_spectrum(const double* samples, size_t n, double fs, size_t transform_len,
                     size_t* out_len, double* out) {
    if (validate_trace(samples, n, fs)) return 1;
    const size_t len = transform_len == 0 ? sko_next_pow2(n) : transform_len;
    if (len < n) return fail("fft_spectrum: transform length shorter than the trace");
    *out_len = len;
    if (!out) return 0;
    double* x = (double*)calloc(2 * len, sizeof(double));
    for (size_t i = 0; i < n; ++i) x[2 * i] = samples[i];
    int rc = sko_dft_any(x, len, out);
    free(x);
    return rc;
}

int sko_slice_band(size_t n_bins, double f_start, double f_step, double f_lo, double f_hi,
                   size_t* k_first, size_t* k_count) {
    if (n_bins == 0) return fail("slice_band: empty spectrum");
    if (!(f_step > 0.0)) return fail("slice_band: non-positive step");
    if (!(f_lo <= f_hi)) return fail("slice_band: inverted band");
    const double eps = 0.5 * f_step * 1e-9;
    const double lo = (f_lo - f_start) / f_step;
    const double hi = (f_hi - f_start) / f_step;
    const long k_lo = (long)ceil(lo - eps);
    const long k_hi = (long)floor(hi + eps);
    const long last = (long)n_bins - 1;
    const long a = k_lo > 0 ? k_lo : 0;
    const long b = k_hi < last ? k_hi : last;
    if (a > b) return fail("slice_band: no bins fall inside the requested band");
    *k_first = (size_t)a;
    *k_count = (size_t)(b - a + 1);
    return 0;
}

/* magnitude_db (types.cpp:13-18): 20 log10 |v| (|v| = hypot, as std::abs of std::complex), -300 dB
 * floor at |v| <= 1e-15; interleaved complex in, n reals out */
void sko_magnitude_db(const double* v, size_t n, double* out) {
    for (size_t k = 0; k < n; ++k) {
        const double mag = hypot(v[2 * k], v[2 * k + 1]);
        out[k] = mag > 1e-15 ? 20.0 * log10(mag) : -300.0;
    }
}

/* ---- zoomfft.cpp ----------------------------------------------------------------------- */
void sko_zoom_options_defaults(sko_zoom_options* o) {   /* zoomfft.hpp:17-26 */
    memset(o, 0, sizeof *o);
    o->circular = 1;
    o->pad_pow2 = 1;
}

/* zoomfft.cpp:15-42 */
int sko_design_lowpass(double cutoff, double fs, size_t num_taps, double* taps) {
    if (!(fs > 0.0)) return fail("design_lowpass: sample rate must be positive");
    if (!(cutoff > 0.0) || cutoff > fs / 2.0) return fail("design_lowpass: cutoff must lie in (0, fs/2]");
    if (num_taps == 0 || num_taps % 2 == 0) return fail("design_lowpass: tap count must be odd");
    if (num_taps == 1) { taps[0] = 1.0; return 0; }
    const double fc = cutoff / fs;
    const size_t mid = (num_taps - 1) / 2;
    double sum = 0.0;
    for (size_t t = 0; t < num_taps; ++t) {
        const double k = (double)t - (double)mid;
        const double arg = 2.0 * fc * k;
        double sinc = 1.0;
        if (k != 0.0) sinc = sin(kPi * arg) / (kPi * arg);
        const double window = 0.54 - 0.46 * cos(2.0 * kPi * (double)t / (double)(num_taps - 1));
        taps[t] = 2.0 * fc * sinc * window;
        sum += taps[t];
    }
    for (size_t t = 0; t < num_taps; ++t) taps[t] /= sum;
    return 0;
}

struct sko_zoom_plan {
    double f1, f2, center, fs, cutoff;
    size_t decimation;
    double* taps;
    size_t n_taps;
    double group_delay;
    int circular, trim, pad_pow2;
    size_t input_len, usable_len, trim_samples, decimated_len, n_fft;
    cx* shift;
    sko_fft_plan* fft;   /* set when n_fft is a power of two */
};

/* zoomfft.cpp:106-181 */
sko_zoom_plan* sko_zoom_plan_create(size_t input_len, double f1, double f2, double fs,
                                    const sko_zoom_options* opts) {
    sko_zoom_options d;
    if (!opts) { sko_zoom_options_defaults(&d); opts = &d; }
    if (input_len < 2) { fail("make_zoom_plan: need at least 2 input samples"); return NULL; }
    if (!(fs > 0.0)) { fail("make_zoom_plan: sample rate must be positive"); return NULL; }
    if (!(f1 >= 0.0) || !(f2 > f1)) { fail("make_zoom_plan: band must satisfy 0 <= f1 < f2"); return NULL; }
    if (f2 > fs / 2.0 * (1.0 + 1e-12)) { fail("make_zoom_plan: band exceeds the Nyquist frequency"); return NULL; }
    sko_zoom_plan* p = (sko_zoom_plan*)calloc(1, sizeof *p);
    p->f1 = f1; p->f2 = f2; p->fs = fs;
    p->circular = opts->circular != 0;
    p->trim = opts->trim_transient != 0;
    p->pad_pow2 = opts->pad_pow2 != 0;
    p->input_len = input_len;
    const double band = f2 - f1;
    p->center = opts->center_set ? opts->center_hz : 0.5 * (f1 + f2);
    if (!isfinite(p->center)) { fail("make_zoom_plan: non-finite center frequency"); goto bad; }
    {
        const int auto_decim = opts->decimation == 0;
        if (auto_decim) {
            size_t dd = (size_t)floor(fs / (2.0 * band));
            p->decimation = dd > 1 ? dd : 1;
        } else {
            p->decimation = opts->decimation;
        }
        const double dnyq = fs / (2.0 * (double)p->decimation);
        const double r1 = f2 - p->center, r2 = p->center - f1;
        const double reach = r1 > r2 ? r1 : r2;
        if (reach > dnyq * (1.0 + 1e-12)) { fail("make_zoom_plan: decimation too large for the requested band"); goto bad; }
        const int auto_filter = opts->num_taps == 0 && !(opts->cutoff_hz > 0.0);
        if (p->decimation == 1 && auto_filter) {
            p->n_taps = 1;
            p->taps = (double*)malloc(sizeof(double));
            p->taps[0] = 1.0;
            p->cutoff = fs / 2.0;
        } else {
            p->cutoff = opts->cutoff_hz > 0.0 ? opts->cutoff_hz : 0.5 * (0.5 * band + dnyq);
            p->n_taps = opts->num_taps == 0 ? 101 : opts->num_taps;
            p->taps = (double*)malloc(p->n_taps * sizeof(double));
            if (sko_design_lowpass(p->cutoff, fs, p->n_taps, p->taps)) goto bad;
        }
    }
    p->group_delay = 0.5 * (double)(p->n_taps - 1);
    p->usable_len = p->circular ? (input_len / p->decimation) * p->decimation : input_len;
    if (p->usable_len / p->decimation < 2) { fail("make_zoom_plan: record too short for this decimation factor"); goto bad; }
    if (p->circular && p->n_taps > p->usable_len) { fail("make_zoom_plan: filter longer than the usable record"); goto bad; }
    {
        size_t block = p->usable_len / p->decimation;
        if (!p->circular && p->trim) {
            p->trim_samples = (p->n_taps - 1 + p->decimation - 1) / p->decimation;
            if (p->trim_samples >= block) { fail("make_zoom_plan: transient trim would consume the whole record"); goto bad; }
            block -= p->trim_samples;
        }
        p->decimated_len = block;
        p->n_fft = p->pad_pow2 ? sko_next_pow2(block) : block;
    }
    {
        const double q = -p->center / fs;
        p->shift = (cx*)malloc(p->usable_len * sizeof(cx));
        for (size_t n = 0; n < p->usable_len; ++n) p->shift[n] = cis_cycles(q, (double)n);
    }
    if (sko_is_pow2(p->n_fft)) p->fft = sko_fft_plan_create(p->n_fft);
    return p;
bad:
    sko_zoom_plan_free(p);
    return NULL;
}

void sko_zoom_plan_free(sko_zoom_plan* p) {
    if (!p) return;
    free(p->taps);
    free(p->shift);
    sko_fft_plan_free(p->fft);
    free(p);
}

void sko_zoom_plan_info(const sko_zoom_plan* p, size_t info[6], double dinfo[4]) {
    info[0] = p->decimation;
    info[1] = p->n_taps;
    info[2] = p->usable_len;
    info[3] = p->decimated_len;
    info[4] = p->n_fft;
    info[5] = p->trim_samples;
    dinfo[0] = p->center;
    dinfo[1] = p->cutoff;
    dinfo[2] = p->group_delay;
    dinfo[3] = p->fs / ((double)p->decimation * (double)p->n_fft);   /* zoomfft.cpp:11-13 */
}

int sko_zoom_plan_set_taps(sko_zoom_plan* p, const double* taps, size_t count) {
    if (count == 0) return fail("zoom: empty filter");
    free(p->taps);
    p->taps = (double*)malloc(count * sizeof(double));
    memcpy(p->taps, taps, count * sizeof(double));
    p->n_taps = count;
    p->group_delay = 0.5 * (double)(count - 1);
    return 0;
}

int sko_zoom_plan_set_n_fft(sko_zoom_plan* p, size_t n_fft) {
    if (n_fft < p->decimated_len) return fail("zoom: n_fft shorter than the decimated block");
    p->n_fft = n_fft;
    sko_fft_plan_free(p->fft);
    p->fft = sko_is_pow2(n_fft) ? sko_fft_plan_create(n_fft) : NULL;
    return 0;
}

/* zoomfft.cpp:66-80 */
static void filter_decimate(const cx* x, size_t n, const double* taps, size_t nt, size_t d, cx* out) {
    const size_t no = n / d;
    for (size_t m = 0; m < no; ++m) {
        cx acc = {0.0, 0.0};
        const size_t base = m * d;
        const size_t t_end = nt < base + 1 ? nt : base + 1;
        for (size_t t = 0; t < t_end; ++t) acc = cadd(acc, cscale(x[base - t], taps[t]));
        out[m] = acc;
    }
}

/* zoomfft.cpp:82-104 */
static void filter_decimate_circular(const cx* x, size_t n, const double* taps, size_t nt, size_t d,
                                     cx* out) {
    const size_t no = n / d;
    for (size_t m = 0; m < no; ++m) {
        cx acc = {0.0, 0.0};
        const size_t base = m * d;
        for (size_t t = 0; t < nt; ++t) {
            const size_t j = base >= t ? base - t : base + n - t;
            acc = cadd(acc, cscale(x[j], taps[t]));
        }
        out[m] = acc;
    }
}

/* zoomfft.cpp:183-239 */
int sko_zoom_fft(const sko_zoom_plan* p, const double* samples, size_t n, double fs,
                 size_t* out_bins, double* f_start, double* f_step, double* out) {
    if (validate_trace(samples, n, fs)) return 1;
    if (n != p->input_len) return fail("zoom_fft: trace length does not match the plan");
    if (fabs(fs - p->fs) > 1e-9 * p->fs) return fail("zoom_fft: trace sample rate does not match the plan");

    const double step = p->fs / ((double)p->decimation * (double)p->n_fft);
    const long nn = (long)p->n_fft;
    const double lo_idx = (p->f1 - p->center) / step;
    const double hi_idx = (p->f2 - p->center) / step;
    const double mx = fabs(lo_idx) > fabs(hi_idx) ? fabs(lo_idx) : fabs(hi_idx);
    const double eps = 1e-9 * (1.0 + mx);
    long k_lo = (long)ceil(lo_idx - eps);
    long k_hi = (long)floor(hi_idx + eps);
    if (k_lo < -(nn / 2)) k_lo = -(nn / 2);
    if (k_hi > nn - 1 - nn / 2) k_hi = nn - 1 - nn / 2;
    if (k_lo > k_hi) return fail("zoom_fft: no transform bins fall inside the band");
    *out_bins = (size_t)(k_hi - k_lo + 1);
    *f_start = p->center + (double)k_lo * step;
    *f_step = step;
    if (!out) return 0;

    cx* y = (cx*)malloc(p->usable_len * sizeof(cx));
    for (size_t i = 0; i < p->usable_len; ++i) y[i] = cscale(p->shift[i], samples[i]);
    const size_t zlen = p->n_fft > p->usable_len / p->decimation ? p->n_fft : p->usable_len / p->decimation;
    cx* z = (cx*)calloc(zlen, sizeof(cx));
    if (p->circular) {
        filter_decimate_circular(y, p->usable_len, p->taps, p->n_taps, p->decimation, z);
    } else {
        filter_decimate(y, p->usable_len, p->taps, p->n_taps, p->decimation, z);
        if (p->trim_samples > 0) {
            const size_t cnt = p->usable_len / p->decimation;
            memmove(z, z + p->trim_samples, (cnt - p->trim_samples) * sizeof(cx));
            for (size_t i = cnt - p->trim_samples; i < cnt; ++i) { z[i].re = 0.0; z[i].im = 0.0; }
        }
    }
    for (size_t i = p->decimated_len; i < p->n_fft; ++i) { z[i].re = 0.0; z[i].im = 0.0; }
    cx* Z = (cx*)malloc(p->n_fft * sizeof(cx));
    if (p->fft) {
        memcpy(Z, z, p->n_fft * sizeof(cx));
        sko_fft_plan_run(p->fft, (double*)Z, p->n_fft, 0);
    } else {
        sko_dft_any((const double*)z, p->n_fft, (double*)Z);
    }
    const double scale = (double)p->decimation;
    const double delay = p->group_delay + (double)(p->trim_samples * p->decimation);
    const double q = delay / ((double)p->decimation * (double)p->n_fft);
    cx* o = (cx*)out;
    size_t w = 0;
    for (long k = k_lo; k <= k_hi; ++k) {
        const size_t idx = (size_t)(((k % nn) + nn) % nn);
        o[w++] = cmul(cscale(Z[idx], scale), cis_cycles(q, (double)k));
    }
    free(y);
    free(z);
    free(Z);
    return 0;
}

/* ---- H(f) — restated division (no reference code) ------------------------ */
void sko_transfer(const double* xs, const double* xr, size_t bins, double* h, double* mag,
                  double* phase) {
    for (size_t k = 0; k < bins; ++k) {
        const double a = xs[2 * k], b = xs[2 * k + 1], c = xr[2 * k], d = xr[2 * k + 1];
        const double den = c * c + d * d;
        const double re = (a * c + b * d) / den;
        const double im = (b * c - a * d) / den;
        if (h) { h[2 * k] = re; h[2 * k + 1] = im; }
        if (mag) mag[k] = hypot(re, im);
        if (phase) phase[k] = atan2(im, re);
    }
}

/* ---- threaded batch helpers for the CPU baseline ------------------------------------- */
static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct {
    int kind;
    const void* plan;
    size_t L;
    const double* x;
    size_t n;
    double fs;
    size_t begin, end;
    double* out;
} job_t;

static void* run_job(void* arg) {
    job_t* j = (job_t*)arg;
    if (j->kind == 0) {   /* czt: plan reuse, per-thread scratch (bench.cpp:194-204) */
        const sko_czt_plan* p = (const sko_czt_plan*)j->plan;
        cx* s = (cx*)malloc(p->L * sizeof(cx));
        cx* xc = (cx*)malloc(p->n * sizeof(cx));
        cx* o = (cx*)malloc(p->m * sizeof(cx));
        for (size_t t = j->begin; t < j->end; ++t) {
            for (size_t i = 0; i < p->n; ++i) { xc[i].re = j->x[t * j->n + i]; xc[i].im = 0.0; }
            sko_czt_execute(p, (const double*)xc, (double*)s, j->out ? j->out + 2 * t * p->m : (double*)o);
        }
        free(s); free(xc); free(o);
    } else if (j->kind == 1) {   /* fft spectrum: FftPlan(L).forward on a padded buffer */
        const sko_fft_plan* p = (const sko_fft_plan*)j->plan;
        cx* b = (cx*)malloc(j->L * sizeof(cx));
        for (size_t t = j->begin; t < j->end; ++t) {
            cx* dst = j->out ? (cx*)(j->out + 2 * t * j->L) : b;
            memset(dst, 0, j->L * sizeof(cx));
            for (size_t i = 0; i < j->n; ++i) dst[i].re = j->x[t * j->n + i];
            sko_fft_plan_run(p, (double*)dst, j->L, 0);
        }
        free(b);
    } else {   /* zoom: prebuilt plan */
        const sko_zoom_plan* p = (const sko_zoom_plan*)j->plan;
        size_t nb; double fst, fsp;
        sko_zoom_fft(p, j->x, j->n, j->fs, &nb, &fst, &fsp, NULL);
        double* o = (double*)malloc(2 * nb * sizeof(double));
        for (size_t t = j->begin; t < j->end; ++t)
            sko_zoom_fft(p, j->x + t * j->n, j->n, j->fs, &nb, &fst, &fsp, j->out ? j->out + 2 * t * nb : o);
        free(o);
    }
    return NULL;
}

static double run_threads(job_t proto, size_t count, int threads) {
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
    job_t* jobs = (job_t*)malloc((size_t)threads * sizeof(job_t));
    const double t0 = now_s();
    for (int i = 0; i < threads; ++i) {
        jobs[i] = proto;
        jobs[i].begin = count * (size_t)i / (size_t)threads;
        jobs[i].end = count * (size_t)(i + 1) / (size_t)threads;
        pthread_create(&th[i], NULL, run_job, &jobs[i]);
    }
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    const double dt = now_s() - t0;
    free(th);
    free(jobs);
    return dt;
}

double sko_bench_czt(const sko_czt_plan* p, const double* x_real, size_t n, size_t count,
                     int threads, double* out) {
    job_t j = {0, p, p->L, x_real, n, 0.0, 0, 0, out};
    return run_threads(j, count, threads);
}

double sko_bench_fft_spectrum(size_t L, const double* x_real, size_t n, size_t count, int threads,
                              double* out) {
    sko_fft_plan* p = sko_fft_plan_create(L);
    if (!p) return -1.0;   /* not a power of two: the caller uses the per-trace route */
    job_t j = {1, p, L, x_real, n, 0.0, 0, 0, out};
    double dt = run_threads(j, count, threads);
    sko_fft_plan_free(p);
    return dt;
}

double sko_bench_zoom(const sko_zoom_plan* p, const double* x_real, size_t n, double fs, size_t count,
                      int threads) {
    job_t j = {2, p, 0, x_real, n, fs, 0, 0, NULL};
    return run_threads(j, count, threads);
}

/* the same, keeping every trace's band bins (count x bins interleaved complex) for parity checks */
double sko_batch_zoom(const sko_zoom_plan* p, const double* x_real, size_t n, double fs, size_t count,
                      int threads, double* out) {
    job_t j = {2, p, 0, x_real, n, fs, 0, 0, out};
    return run_threads(j, count, threads);
}
