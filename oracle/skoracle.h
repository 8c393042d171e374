/* skoracle — CPU restatement of the spectralkit transform path (TEST INFRASTRUCTURE).
 *
 * This is the parity CHECKER for the B200 library, not a product path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 * Each function restates the reference algorithm (paths relative to
 * /root/reference/proj) in plain C99, fp64 only, single-threaded per call, with the
 * same operation order as the reference so results agree to the last few ulps.
 * Pinned by tests/test_oracle.py against (a) the reference's own KATs and
 * (b) golden vectors produced by the reference itself (oracle/_ref, tests/golden/).
 *
 * Complex buffers are interleaved (re, im) doubles, i.e. the memory layout of
 * std::complex<double> (reference types.hpp:9-10).
 */
#ifndef SKORACLE_H
#define SKORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status: 0 ok, 1 invalid argument (message in sko_last_error) */
const char* sko_last_error(void);

int sko_is_pow2(size_t n);                                /* numerics.cpp:14 */
size_t sko_next_pow2(size_t n);                           /* numerics.cpp:16-24; 0 on error */
void sko_cis_cycles(double q, double t, double out[2]);   /* numerics.cpp:122-128 */

/* FftPlan (numerics.hpp:27-43, numerics.cpp:52-100) */
typedef struct sko_fft_plan sko_fft_plan;
sko_fft_plan* sko_fft_plan_create(size_t n);
void sko_fft_plan_free(sko_fft_plan* p);
int sko_fft_plan_run(const sko_fft_plan* p, double* data, size_t n, int invert);

int sko_fft(const double* x, size_t n, int invert, double* out);      /* numerics.cpp:102-120 */
int sko_dft_naive(const double* x, size_t n, double* out);            /* numerics.cpp:35-50 */

/* CZT (czt.hpp:13-68, czt.cpp:15-175) */
int sko_czt_params_for_band(double f1, double f2, double fs, size_t m, double a[2], double w[2]);
typedef struct sko_czt_plan sko_czt_plan;
sko_czt_plan* sko_czt_plan_create(size_t n, const double a[2], const double w[2], size_t m);
void sko_czt_plan_free(sko_czt_plan* p);
size_t sko_czt_plan_conv_size(const sko_czt_plan* p);
/* scratch: conv_size complex entries (may be NULL -> allocated per call) */
int sko_czt_execute(const sko_czt_plan* p, const double* x, double* scratch, double* out);
int sko_czt(const double* x, size_t n, const double a[2], const double w[2], size_t m, double* out);
int sko_czt_direct(const double* x, size_t n, const double a[2], const double w[2], size_t m,
                   double* out);
int sko_dft_any(const double* x, size_t n, double* out);              /* czt.cpp:144-153 */

/* Spectra (spectra.cpp:21-61). out holds len complex bins. */
int sko_fft_spectrum(const double* samples, size_t n, double fs, size_t transform_len,
                     size_t* out_len, double* out /* may be NULL to query */);
int sko_slice_band(size_t n_bins, double f_start, double f_step, double f_lo, double f_hi,
                   size_t* k_first, size_t* k_count);
void sko_magnitude_db(const double* v, size_t n, double* out);

/* Zoom (zoomfft.hpp:17-86, zoomfft.cpp:11-239) */
typedef struct sko_zoom_options {
    double center_hz;
    int center_set;
    size_t decimation;
    double cutoff_hz;
    size_t num_taps;
    int circular;
    int trim_transient;
    int pad_pow2;
} sko_zoom_options;
void sko_zoom_options_defaults(sko_zoom_options* o);
int sko_design_lowpass(double cutoff, double fs, size_t taps, double* out);
typedef struct sko_zoom_plan sko_zoom_plan;
sko_zoom_plan* sko_zoom_plan_create(size_t n, double f1, double f2, double fs,
                                    const sko_zoom_options* o);
void sko_zoom_plan_free(sko_zoom_plan* p);
/* info: decimation, taps, usable_len, decimated_len, n_fft, trim_samples */
void sko_zoom_plan_info(const sko_zoom_plan* p, size_t info[6], double dinfo[4]);
/* overwrite the filter (extension: even-tap designs, used for the 64-tap cfg3 variant) */
int sko_zoom_plan_set_taps(sko_zoom_plan* p, const double* taps, size_t count);
/* overwrite n_fft (extension: 2048-point cfg3 variant; zoomfft.hpp:50-53 public fields) */
int sko_zoom_plan_set_n_fft(sko_zoom_plan* p, size_t n_fft);
/* band bins: query size with out == NULL */
int sko_zoom_fft(const sko_zoom_plan* p, const double* samples, size_t n, double fs,
                 size_t* out_bins, double* f_start, double* f_step, double* out);

/* Transfer function H = Xs / Xr (not in the reference; SURVEY 8c "H(f) oracle"):
 * per bin complex divide, |H| = hypot, arg H = atan2. */
void sko_transfer(const double* xs, const double* xr, size_t bins, double* h, double* mag,
                  double* phase);

/* Batched helpers used only by bench.py's cpu_baseline leg: run `count` traces on
 * `threads` POSIX threads with one shared immutable plan (numerics.hpp:24-26). */
double sko_bench_czt(const sko_czt_plan* p, const double* x_real, size_t n, size_t count,
                     int threads, double* out /* count*m complex, may be NULL */);
double sko_bench_fft_spectrum(size_t L, const double* x_real, size_t n, size_t count,
                              int threads, double* out);
double sko_bench_zoom(const sko_zoom_plan* p, const double* x_real, size_t n, double fs,
                      size_t count, int threads);
double sko_batch_zoom(const sko_zoom_plan* p, const double* x_real, size_t n, double fs, size_t count,
                      int threads, double* out);

#ifdef __cplusplus
}
#endif
#endif
