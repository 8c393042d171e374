/* spectralkit.h — drop-in C ABI of the B200 spectral library (libspectralkit_b200.so).
 *
 * This header declares the hot-path subset of the reference's C interface
 * (/root/reference/proj/include/spectralkit.h) with identical names, argument order, argument
 * meaning, ownership rules and status codes, so a reference client recompiles and relinks
 * against this library unchanged. Every transform executes on the GPU (sm_100a); host buffers
 * are copied to and from device memory inside the call. The batched, device-resident extension
 * lives in spectralkit_gpu.h.
 *
 * Conventions kept from the reference (capi.cpp:44-83):
 *   - every sk_status-returning call reports SK_OK or an error code; the message is stored in
 *     thread-local storage and returned by sk_last_error() until the next failing call on the
 *     same thread;
 *   - null pointers are rejected with SK_ERR_INVALID_ARGUMENT before any work;
 *   - handles created by sk_*_create / transform calls are released with the matching sk_*_free
 *     (null-safe); getters on a null handle return 0 / NaN-free defaults;
 *   - raw transforms take caller-owned split re[] / im[] arrays.
 * A CUDA failure (no device, launch error) is reported as SK_ERR_INTERNAL.
 */
#ifndef SPECTRALKIT_B200_H
#define SPECTRALKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#define SK_API __attribute__((visibility("default")))

#ifdef __cplusplus
extern "C" {
#endif

/* reference spectralkit.h:30-38 */
typedef enum sk_status {
    SK_OK = 0,
    SK_ERR_INVALID_ARGUMENT = 1,
    SK_ERR_IO = 2,
    SK_ERR_PARSE = 3,
    SK_ERR_FORMAT = 4,
    SK_ERR_INSUFFICIENT_RESOLUTION = 5,
    SK_ERR_INTERNAL = 6
} sk_status;

SK_API const char* sk_status_name(sk_status status);   /* ref spectralkit.h:40, capi.cpp:152-164 */
SK_API const char* sk_last_error(void);                /* ref spectralkit.h:41 */
SK_API const char* sk_version(void);                   /* ref spectralkit.h:42 */

/* Raw transforms on split arrays. */
/* ref spectralkit.h:47 / capi.cpp:170-177: in place, n a power of two, forward unnormalised */
SK_API sk_status sk_fft(double* re, double* im, size_t n);
/* ref spectralkit.h:48 / capi.cpp:179-186: in place, applies 1/n */
SK_API sk_status sk_ifft(double* re, double* im, size_t n);
/* ref spectralkit.h:51-52 / capi.cpp:188-195: O(n^2) direct sum with exact (k*m) mod n phases */
SK_API sk_status sk_dft_naive(const double* re, const double* im, size_t n, double* out_re,
                              double* out_im);
/* ref spectralkit.h:56-58 / capi.cpp:197-205: m bins X[k] = sum x[n] a^-n w^(kn) via Bluestein */
SK_API sk_status sk_czt(const double* re, const double* im, size_t n, double a_re, double a_im,
                        double w_re, double w_im, size_t m, double* out_re, double* out_im);
/* ref spectralkit.h:59-61 / capi.cpp:207-216: the O(n m) defining sum */
SK_API sk_status sk_czt_direct(const double* re, const double* im, size_t n, double a_re,
                               double a_im, double w_re, double w_im, size_t m, double* out_re,
                               double* out_im);
/* ref spectralkit.h:64-66 / czt.cpp:42-56: a = e^{i2pi f1/fs}, w = e^{-i2pi (f2-f1)/(m fs)} */
SK_API sk_status sk_czt_params_for_band(double f1_hz, double f2_hz, double sample_rate_hz,
                                        size_t m, double* a_re, double* a_im, double* w_re,
                                        double* w_im);

/* ref spectralkit.h:70: smallest power of two >= max(n, 1) */
SK_API size_t sk_next_pow2(size_t n);
/* sizing helpers (ref spectralkit.h:71-78, resolution.cpp:18-63) */
SK_API sk_status sk_fft_resolution(double sample_rate_hz, size_t n, double* out_hz);
SK_API sk_status sk_record_len_for_step(double sample_rate_hz, double target_step_hz, size_t* out_len);
SK_API sk_status sk_zeros_for_resolution(double sample_rate_hz, size_t n, double target_step_hz,
                                         size_t* out_zeros);
SK_API sk_status sk_czt_len_for_matched_resolution(double f1_hz, double f2_hz, double sample_rate_hz,
                                                   size_t n_fft, size_t* out_m);

/* Traces (ref spectralkit.h:82-90, capi.cpp:264-297). */
typedef struct sk_trace sk_trace;
SK_API sk_status sk_trace_create(const double* samples, size_t n, double sample_rate_hz,
                                 double t0_s, sk_trace** out);
SK_API void sk_trace_free(sk_trace* t);
SK_API size_t sk_trace_size(const sk_trace* t);
SK_API double sk_trace_sample_rate(const sk_trace* t);
SK_API double sk_trace_t0(const sk_trace* t);
SK_API const double* sk_trace_samples(const sk_trace* t);
/* CSV "time_s,amplitude" (ref spectralkit.h:133-134, signals.cpp:125-189): optional header row,
 * median-step sample rate with a 1e-6 uniformity check, SK_ERR_PARSE with the line number for a
 * malformed row, SK_ERR_FORMAT for < 2 samples / non-increasing / non-uniform time, SK_ERR_IO for
 * unopenable files; "-" = stdin / stdout. Rows written as %.17g. */
SK_API sk_status sk_trace_read_csv(const char* path, sk_trace** out);
SK_API sk_status sk_trace_write_csv(const sk_trace* t, const char* path);

/* Spectra (ref spectralkit.h:138-161, capi.cpp:412-481). */
typedef struct sk_spectrum sk_spectrum;
/* full [0, fs) spectrum; transform_len 0 = next power of two, otherwise exact (Bluestein when
 * not a power of two); spectra.cpp:21-38 */
SK_API sk_status sk_fft_spectrum(const sk_trace* t, size_t transform_len, sk_spectrum** out);
/* m bins on [f1, f2] with step (f2-f1)/m; czt.cpp:155-175 */
SK_API sk_status sk_czt_spectrum(const sk_trace* t, double f1_hz, double f2_hz, size_t m,
                                 sk_spectrum** out);
SK_API sk_status sk_spectrum_create(const double* re, const double* im, size_t n,
                                    double f_start_hz, double f_step_hz, sk_spectrum** out);
SK_API void sk_spectrum_free(sk_spectrum* s);
SK_API size_t sk_spectrum_size(const sk_spectrum* s);
SK_API double sk_spectrum_f_start(const sk_spectrum* s);
SK_API double sk_spectrum_f_step(const sk_spectrum* s);
SK_API double sk_spectrum_frequency(const sk_spectrum* s, size_t k);
SK_API size_t sk_spectrum_source_n(const sk_spectrum* s);
SK_API sk_status sk_spectrum_bin(const sk_spectrum* s, size_t k, double* re, double* im);
SK_API sk_status sk_spectrum_magnitude_db(const sk_spectrum* s, size_t k, double* out_db);
SK_API sk_status sk_spectrum_copy_data(const sk_spectrum* s, double* re, double* im);
SK_API sk_status sk_spectrum_slice_band(const sk_spectrum* s, double f_lo_hz, double f_hi_hz,
                                        sk_spectrum** out);
/* CSV "frequency_hz,re,im,magnitude_db", %.17g rows (ref spectralkit.h:163-165, spectra.cpp:63-78);
 * byte-identical to the reference's writer */
SK_API sk_status sk_spectrum_write_csv(const sk_spectrum* s, const char* path);
/* ref spectralkit.h:166, spectra.cpp:161-183: {f_start_hz, f_step_hz, im[], magnitude_db[], re[],
 * source_n}, two-space indentation, numbers in the reference JSON library's shortest form (Grisu2);
 * byte-identical to the reference's writer */
SK_API sk_status sk_spectrum_write_json(const sk_spectrum* s, const char* path);
/* ref spectralkit.h:164, spectra.cpp:94-156: four fields per row, optional header, uniform axis
 * (1e-6 step tolerance); SK_ERR_PARSE / SK_ERR_FORMAT / SK_ERR_IO as the reference */
SK_API sk_status sk_spectrum_read_csv(const char* path, sk_spectrum** out);

/* Two-tone analysis (ref spectralkit.h:197-243, analysis.cpp:30-195). The resolvability sweep runs
 * every separation's padded-FFT route and band-CZT route as two batched GPU launches; the valley
 * test (dip_metric) runs on host threads. SK_ERR_INSUFFICIENT_RESOLUTION from sk_dip_metric_compute
 * when fewer than 3 bins lie between the tones. */
typedef struct sk_dip_metric {
    int resolved;
    double dip_db;
    double f_peak_a_hz;
    double peak_a_db;
    double f_peak_b_hz;
    double peak_b_db;
    double f_valley_hz;
    double valley_db;
} sk_dip_metric;
SK_API sk_status sk_dip_metric_compute(const sk_spectrum* s, double f_a_hz, double f_b_hz,
                                       sk_dip_metric* out);
typedef struct sk_scan_config {
    double sample_rate_hz;
    size_t n;
    double f1_hz;
    double f2_hz;
    size_t m;
    double center_hz; /* 0 = band midpoint */
    double sep_start_hz;
    double sep_stop_hz;
    double sep_step_hz;
} sk_scan_config;
SK_API void sk_scan_config_defaults(sk_scan_config* cfg);
typedef struct sk_resolvability_curve sk_resolvability_curve;
SK_API sk_status sk_resolvability_scan(const sk_scan_config* cfg, sk_resolvability_curve** out);
SK_API void sk_resolvability_curve_free(sk_resolvability_curve* c);
SK_API size_t sk_resolvability_curve_size(const sk_resolvability_curve* c);
SK_API sk_status sk_resolvability_curve_point(const sk_resolvability_curve* c, size_t i,
                                              double* separation_hz, sk_dip_metric* fft_m,
                                              sk_dip_metric* czt_m);
/* NaN when no separation resolved on that route */
SK_API double sk_resolvability_min_fft(const sk_resolvability_curve* c);
SK_API double sk_resolvability_min_czt(const sk_resolvability_curve* c);
/* ref spectralkit.h:239, serialize.cpp:141-154: byte-identical CSV of the curve */
SK_API sk_status sk_resolvability_write_csv(const sk_resolvability_curve* c, const char* path);
/* ref spectralkit.h:241, serialize.cpp:113-135 */
SK_API sk_status sk_resolvability_write_json(const sk_resolvability_curve* c, const char* path);

/* Zoom pipeline (ref spectralkit.h:170-195, capi.cpp:515-564). Same struct layout. */
typedef struct sk_zoom_options {
    double center_hz;     /* used only when center_set */
    int center_set;
    size_t decimation;    /* 0: floor(fs / (2 (f2 - f1))) */
    double cutoff_hz;     /* 0: derived */
    size_t num_taps;      /* 0: 101; must be odd */
    int circular;         /* default 1 */
    int trim_transient;   /* linear mode only */
    int pad_pow2;         /* default 1 */
} sk_zoom_options;

SK_API void sk_zoom_options_defaults(sk_zoom_options* opts);
typedef struct sk_zoom_plan sk_zoom_plan;
SK_API sk_status sk_zoom_plan_create(size_t input_len, double f1_hz, double f2_hz,
                                     double sample_rate_hz, const sk_zoom_options* opts,
                                     sk_zoom_plan** out);
SK_API void sk_zoom_plan_free(sk_zoom_plan* p);
SK_API size_t sk_zoom_plan_decimation(const sk_zoom_plan* p);
SK_API size_t sk_zoom_plan_n_fft(const sk_zoom_plan* p);
SK_API size_t sk_zoom_plan_filter_len(const sk_zoom_plan* p);
SK_API double sk_zoom_plan_f_step(const sk_zoom_plan* p);
SK_API sk_status sk_zoom_spectrum(const sk_zoom_plan* p, const sk_trace* t, sk_spectrum** out);

#ifdef __cplusplus
}
#endif

#endif /* SPECTRALKIT_B200_H */
