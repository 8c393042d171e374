/* spectralkit_gpu.h — batched, device-resident extension of the spectralkit C ABI.
 *
 * The reference has no batch interface: every sk_* call transforms one trace held in host
 * memory. These entry points run the same transforms on a batch of traces that
 * already lives in GPU memory (device pointers from cudaMalloc, torch, CuPy, ...), enqueue on
 * the caller's CUDA stream and return without synchronising. Plans hold the precomputed
 * twiddle / chirp / filter tables on the device and are immutable after creation, so one plan
 * may be shared by concurrent streams (the reference's plan rule, numerics.hpp:24-26).
 *
 * Layouts: traces are real rows of `n` samples, row stride `x_stride` elements; complex outputs
 * are interleaved (re, im) — the std::complex layout of the reference's ComplexBuffer —
 * with row stride in complex elements. precision: SKG_F64 (double / complex128 buffers) or
 * SKG_F32 (float / complex64 buffers; tables are rounded from fp64).
 */
#ifndef SPECTRALKIT_GPU_H
#define SPECTRALKIT_GPU_H

#include "spectralkit.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum skg_precision { SKG_F64 = 0, SKG_F32 = 1 } skg_precision;

/* device facts of the current CUDA device */
SK_API sk_status skg_device_info(int* device, int* sm_count, size_t* smem_optin, size_t* l2_bytes);
/* number of kernels this library has launched in the process (evidence counter) */
SK_API uint64_t skg_launch_count(void);
/* Test hook: cap every persistent kernel grid at `cap` CTAs (0 = off, the default). The kernels
 * loop over their units; a small cap drives every CTA through many units so parity tests cover
 * the later waves (next-unit prefetch, workspace-slot reuse) at batch sizes an oracle checks fast. */
SK_API void skg_debug_set_grid_cap(unsigned cap);
/* cudaStreamSynchronize(stream) with the library's error reporting */
SK_API sk_status skg_synchronize(void* stream);

/* Complex-to-complex FFT of `batch` rows of n points (power of two); inverse applies 1/n
 * (numerics.cpp:73-100). d_in == d_out is allowed. */
SK_API sk_status skg_fft_batch(size_t n, int inverse, int precision, const void* d_in,
                               size_t in_stride, void* d_out, size_t out_stride, size_t batch,
                               void* stream);

/* Zero-padded spectrum of real traces (fft_spectrum, spectra.cpp:21-38). transform_len 0 =
 * next_pow2(n). layout SKG_FULL: transform_len bins on [0, fs) (the reference layout);
 * SKG_HALF: transform_len/2 + 1 bins on [0, fs/2]. Non-power-of-two transform_len runs the
 * chirp route (dft_any, czt.cpp:144-153) and supports SKG_FULL only. */
#define SKG_FULL 0
#define SKG_HALF 1
SK_API sk_status skg_fft_spectrum_batch(size_t n, size_t transform_len, int precision, int layout,
                                        const void* d_x, size_t x_stride, size_t batch,
                                        void* d_out, size_t out_stride, void* stream);

/* Band slice + dB column. skg_band_bins restates slice_band's bin selection
 * (spectra.cpp:40-61: 1e-9-step slack, clipped to the spectrum, same errors) for a spectrum of
 * spectrum_size bins at f_start + k f_step. skg_fft_spectrum_band_batch writes only bins
 * [k_lo, k_lo + count) of the full zero-padded spectrum (the sk_spectrum_slice_band result) as
 * complex (d_bins, may be NULL) and/or magnitude_db (d_db, may be NULL; types.cpp:13-18:
 * 20 log10|X|, -300 dB at |X| <= 1e-15), fused into the FFT store. skg_band_db_batch does the same
 * slice/dB pass over complex rows already on the device (CZT and zoom outputs, full spectra). */
SK_API sk_status skg_band_bins(size_t spectrum_size, double f_start_hz, double f_step_hz, double f_lo_hz,
                               double f_hi_hz, size_t* k_lo, size_t* count, double* band_f_start_hz);
SK_API sk_status skg_fft_spectrum_band_batch(size_t n, size_t transform_len, int precision, size_t k_lo,
                                             size_t count, const void* d_x, size_t x_stride, size_t batch,
                                             void* d_bins, size_t bins_stride, void* d_db, size_t db_stride,
                                             void* stream);
SK_API sk_status skg_band_db_batch(int precision, const void* d_in, size_t in_stride, size_t k_lo, size_t count,
                                   size_t batch, void* d_bins, size_t bins_stride, void* d_db, size_t db_stride,
                                   void* stream);

/* Batched trace ingest and spectrum output. skg_traces_read_csv runs
 * sk_trace_read_csv's parser and checks (signals.cpp:125-170) on `count` files in parallel host
 * threads (threads 0 = all cores); every file must hold n samples (else SK_ERR_FORMAT). The rows land
 * in pinned staging and go to d_out (row stride out_stride elements; SKG_F32 rounds) with one copy
 * on `stream`; per-file sample rate / t0 go to fs_out / t0_out (host, may be NULL). On failure the
 * lowest-index failing file's status and message are reported and nothing is copied.
 * skg_spectra_write_csv copies `count` rows of nbins complex bins from the device and writes one
 * reference-format CSV per path in parallel (f_start_hz: per-row start frequency, NULL = 0). Both
 * calls return after the transfer completed. */
SK_API sk_status skg_traces_read_csv(const char* const* paths, size_t count, size_t n, int precision,
                                     void* d_out, size_t out_stride, double* fs_out, double* t0_out,
                                     int threads, void* stream);
SK_API sk_status skg_spectra_write_csv(const char* const* paths, size_t count, int precision,
                                       const void* d_bins, size_t bins_stride, size_t nbins,
                                       const double* f_start_hz, double f_step_hz, int threads,
                                       void* stream);

/* padded full-range transform length of a resolvability curve (ResolvabilityCurve::fft_len) */
SK_API size_t skg_resolvability_fft_len(const sk_resolvability_curve* c);

/* Chirp-z transform plan (CztPlan, czt.cpp:85-137). */
typedef struct skg_czt_plan skg_czt_plan;
SK_API sk_status skg_czt_plan_create(size_t n, double a_re, double a_im, double w_re, double w_im,
                                     size_t m, int precision, skg_czt_plan** out);
SK_API void skg_czt_plan_free(skg_czt_plan* p);
SK_API size_t skg_czt_plan_conv_size(const skg_czt_plan* p);
/* x: real (x_complex = 0) or interleaved complex rows of n; out: rows of m complex bins */
SK_API sk_status skg_czt_execute(const skg_czt_plan* p, const void* d_x, int x_complex,
                                 size_t x_stride, size_t batch, void* d_out, size_t out_stride,
                                 void* stream);

/* Transfer function H(f) = X_sample(f) / X_ref(f) against one shared reference trace, fused
 * into the FFT store epilogue: per trace, transform_len/2 + 1 bins of |H| and arg H (radians,
 * atan2 convention) and optionally the complex H. */
typedef struct skg_transfer_plan skg_transfer_plan;
SK_API sk_status skg_transfer_plan_create(const double* ref_samples, size_t n, size_t transform_len,
                                          int precision, skg_transfer_plan** out);
SK_API void skg_transfer_plan_free(skg_transfer_plan* p);
SK_API size_t skg_transfer_plan_bins(const skg_transfer_plan* p);
/* copies X_ref (bins complex, fp64) to host */
SK_API sk_status skg_transfer_plan_reference(const skg_transfer_plan* p, double* xr_interleaved);
SK_API sk_status skg_transfer_execute(const skg_transfer_plan* p, const void* d_x, size_t x_stride,
                                      size_t batch, void* d_mag, void* d_phase, size_t mp_stride,
                                      void* d_h, size_t h_stride, void* stream);

/* Zoom FFT plan (make_zoom_plan + zoom_fft, zoomfft.cpp:106-239). `ext` (may be NULL) carries
 * knobs the reference struct lacks: an explicit short-FFT length n_fft (>= decimated block;
 * the reference derives next_pow2(block)) and an explicit filter (any length, including the
 * even 64-tap design of the cfg3 text; the reference designs odd Hamming-sinc filters only). */
typedef struct skg_zoom_ext {
    size_t n_fft;          /* 0 = reference sizing */
    const double* taps;    /* NULL = reference design */
    size_t num_taps;
} skg_zoom_ext;
typedef struct skg_zoom_plan skg_zoom_plan;
SK_API sk_status skg_zoom_plan_create(size_t input_len, double f1_hz, double f2_hz,
                                      double sample_rate_hz, const sk_zoom_options* opts,
                                      const skg_zoom_ext* ext, int precision, skg_zoom_plan** out);
SK_API void skg_zoom_plan_free(skg_zoom_plan* p);
SK_API sk_status skg_zoom_plan_info(const skg_zoom_plan* p, size_t* bins, double* f_start_hz,
                                    double* f_step_hz, size_t* n_fft, size_t* decimation,
                                    size_t* num_taps);
SK_API sk_status skg_zoom_execute(const skg_zoom_plan* p, const void* d_x, size_t x_stride,
                                  size_t batch, void* d_out, size_t out_stride, void* stream);

/* ---- host-buffer batched calls -----------------------------------------------------------------
 * The batched counterparts of the reference's host-buffer one-shot calls (sk_czt, capi.cpp:197-205;
 * sk_fft_spectrum; sk_zoom_spectrum): rows in host memory in, rows in host memory out. The library
 * moves `chunk` rows at a time (0 = automatic, about 8 chunks) on its own streams so the H2D copy of
 * one chunk, the kernel of the next and the D2H copy of a third overlap. Pinned caller buffers
 * (cudaHostAlloc / cudaHostRegister) are copied directly; pageable ones through library-owned pinned
 * staging. Strides are in elements as in the device calls. The calls return when every output row is
 * in host memory. */
SK_API sk_status skg_czt_execute_host(const skg_czt_plan* p, const void* h_x, int x_complex, size_t x_stride,
                                      size_t batch, void* h_out, size_t out_stride, size_t chunk);
SK_API sk_status skg_fft_spectrum_host(size_t n, size_t transform_len, int precision, int layout, const void* h_x,
                                       size_t x_stride, size_t batch, void* h_out, size_t out_stride, size_t chunk);
SK_API sk_status skg_zoom_execute_host(const skg_zoom_plan* p, const void* h_x, size_t x_stride, size_t batch,
                                       void* h_out, size_t out_stride, size_t chunk);
SK_API sk_status skg_transfer_execute_host(const skg_transfer_plan* p, const void* h_x, size_t x_stride,
                                           size_t batch, void* h_mag, void* h_phase, size_t mp_stride,
                                           size_t chunk);

#ifdef __cplusplus
}
#endif

#endif /* SPECTRALKIT_GPU_H */
