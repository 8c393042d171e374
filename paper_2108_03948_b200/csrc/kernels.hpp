// kernels.hpp — host-callable launchers for the B200 spectral kernels (no torch types).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace skg {

// Test hook (skg_debug_set_grid_cap): upper bound on every persistent grid, 0 = none. Lets the
// parity tests drive the persistent loops (later units, L2 prefetch, workspace-slot reuse) through
// many waves at batch sizes the CPU oracle checks in seconds.
unsigned grid_cap();

// One row of the launch table: which single-CTA sizes exist.
constexpr int kMaxLog2F64 = 13;   // 8192 complex fp64 = 136 KB padded SMEM
constexpr int kMaxLog2F32 = 14;   // 16384 complex fp32

template <typename T> constexpr int max_log2() { return sizeof(T) == 8 ? kMaxLog2F64 : kMaxLog2F32; }

// complex -> complex, natural order in and out; scale applied on store (1/L for inverse).
// in == out allowed.
template <typename T>
cudaError_t launch_fft_c2c(int log2L, bool inverse, const void* in, long long in_stride, void* out,
                           long long out_stride, long long batch, const void* tw, T scale,
                           cudaStream_t st);

// real trace (N samples, zero padded to L = 2^(log2M+1)) -> spectrum via an M-point complex FFT
// of packed sample pairs. mode 0: full L-bin spectrum (reference layout, spectra.cpp:21-38);
// mode 1: half spectrum, M+1 bins; mode 2: H = X * rtab (rtab = 1/X_ref), |H| and arg H on M+1
// bins (h optional, M+1 complex); mode 3: bins klo..khi of the full spectrum (slice_band,
// spectra.cpp:40-61) as complex (out, optional) and/or magnitude_db (mag, optional; types.cpp:13-18).
template <typename T>
cudaError_t launch_fft_r2c(int log2M, long long N, const T* x, long long x_stride, long long batch,
                           const void* tw, const void* post, int mode, void* out, long long out_stride,
                           const void* rtab, T* mag, T* phase, long long mp_stride, long long klo, long long khi,
                           cudaStream_t st);

// fused Bluestein CZT (czt.cpp:116-130): x * chirp_in -> FFT_L -> * khat (pre-scaled by 1/L)
// -> IFFT_L -> * chirp_out, first M bins stored. x real (T) or complex (cx<T>). The M outputs are
// split into nseg segments of seg_len bins (segment s uses input chirp cin + s*N, shared khat and
// output chirp); L is the convolution length of ONE segment.
template <typename T>
cudaError_t launch_czt(int log2L, long long N, long long M, bool complex_in, const void* x,
                       long long x_stride, long long batch, int nseg, long long seg_len, long long cin_stride,
                       void* out, long long out_stride, const void* tw, const void* cin, const void* khat,
                       const void* cout, cudaStream_t st);

// shared-forward segmented CZT: one forward FFT of x*cin (cin = segment 0's chirp) serves all nseg
// blocks; khat = nseg x L kernel spectra (block s: g[j] = W^{-(s seg + j)^2/2}, prescaled 1/L),
// cout = nseg x seg_len output chirps W^{(s seg + k)^2/2}. cudaErrorNotSupported when the
// geometry has no instantiation or the per-CTA shared memory does not fit (caller falls back).
// ywork (optional): ywork_slots x L complex scratch that lets more transform groups share an SM.
// twl (optional): (L/16) x 16 table W_L^{j k}, the last radix-16 pass's twiddles, which the TMEM
// variant keeps per thread (kernels_czt_tm.cuh).
template <typename T>
cudaError_t launch_czt_sf(int log2L, long long N, long long M, bool complex_in, const void* x, long long x_stride,
                          long long batch, int nseg, long long seg_len, void* out, long long out_stride,
                          const void* tw, const void* cin, const void* khat, const void* cout, void* ywork,
                          long long ywork_slots, const void* twl, cudaStream_t st);

// ---- four-step passes for L = R * C beyond one CTA (kernels_4step.cuh) ----------------------
// in_kind: 0 complex x, 1 real x, 2 real x * chirp, 3 complex x * chirp, 4 work buffer Y
// out_kind: 0 Y with the W_L twiddle, 1 out * chirp_out (n < M), 2 out * scale (conj optional)
template <typename T>
cudaError_t launch_4step_col(int log2R, bool inverse, int in_kind, int conj_in, const void* x, long long x_stride,
                             long long N, const void* cin, void* Y, int log2C, long long batch, const void* tw,
                             const void* twL, int out_kind, void* out, long long out_stride, long long M,
                             const void* cout, T scale, int conj_out, cudaStream_t st);
// mode 0: FFT_C per row, natural-order store to out (scale/conj); mode 1: Bluestein middle in place
template <typename T>
cudaError_t launch_4step_row(int log2C, int mode, void* Y, int log2R, long long batch, const void* tw,
                             const void* twL, const void* khat_p, void* out, long long out_stride, T scale,
                             int conj_out, cudaStream_t st);

// real traces, Hermitian half (kernels_4step_real.cuh): column pass into (R/2 + 1) x C work rows, row pass with
// the mirrored conjugate store; half != 0 writes the L/2 + 1 bin layout
template <typename T>
cudaError_t launch_4step_colr(int log2R, const void* x, long long x_stride, long long N, void* Y, int log2C,
                              long long batch, const void* tw, const void* twL, cudaStream_t st);
template <typename T>
cudaError_t launch_4step_rowh(int log2C, const void* Y, int log2R, long long batch, const void* tw, void* out,
                              long long out_stride, int half, cudaStream_t st);

// both passes in one cooperative persistent launch, work rows in a ring of `slots` traces (square R = C = 2^lg);
// grid_out / ups_out != nullptr: only report the grid the launch would use and the units per trace step.
template <typename T>
cudaError_t launch_4step_rfused(int lg, const void* x, long long x_stride, long long N, void* Yring, int slots, int delta,
                                long long batch, const void* tw, const void* twL, void* out, long long out_stride,
                                int half, unsigned* col_done, unsigned* row_done, int* grid_out, int* ups_out,
                                cudaStream_t st);

// multi-pass CZT in one cooperative persistent launch (kernels_4step_czt.cuh): forward column, row (Bluestein
// middle) and inverse column units interleaved, work rows in a ring of `slots` traces; counters = 3 * batch
// zeroed words; grid_out/ups_out != nullptr: only report the grid and the units per trace step.
template <typename T>
cudaError_t launch_4step_czt_fused(int lR, int lC, const void* x, int complex_in, long long x_stride, long long N,
                                   const void* cin, void* Yring, int slots, int delta, long long batch, const void* twR,
                                   const void* twC, const void* twL, const void* khat_p, void* out, long long out_stride,
                                   long long M, const void* cout, unsigned* counters, int* grid_out, int* ups_out,
                                   cudaStream_t st);

// ---- fused Zoom FFT (kernels_zoom.cu) --------------------------------------------------
constexpr int kZoomK = 4;   // FIR outputs per thread
struct ZoomArgs {
    long long n;       // samples per trace
    long long U;       // usable length (circular) or n (linear)
    int D;             // decimation
    int T;             // taps
    int nout;          // FIR outputs fed to the FFT (decimated_len)
    int trim;          // first FIR output kept (linear trim mode)
    int rowlen;        // polyphase row length (elements, unpadded, incl. margin)
    int pre;           // zero prefix per row (lh + kZoomK)
    int rs;            // padded row stride (odd)
    int lh;            // taps per phase row, rounded up to kZoomK
    int k_lo;          // first signed band bin
    int nbins;         // band bins
    int mwrap;         // outputs needing the circular wrap correction
    int circular;
    double wre, wim;   // wrap factor e^{-i2pi fc U/fs}
};
cudaError_t launch_zoom_f64(const ZoomArgs& a, int log2n, const double* x, long long xs, long long batch,
                            const void* g, const void* S, const void* tw, const void* band, void* out,
                            long long os, cudaStream_t st);
cudaError_t launch_zoom_f32(const ZoomArgs& a, int log2n, const float* x, long long xs, long long batch,
                            const void* g, const void* S, const void* tw, const void* band, void* out,
                            long long os, cudaStream_t st);
// unfused path: FIR/decimate into zb (rows of z_stride complex, first nout written), band gather
cudaError_t launch_zoom_fir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch, const void* g,
                            const void* S, void* zb, long long z_stride, cudaStream_t st);
cudaError_t launch_zoom_band(bool f32, const void* Z, long long z_stride, long long n_fft, int k_lo, int nbins,
                             const void* band, void* out, long long out_stride, long long batch, cudaStream_t st);
int zoom_chunk_rowlen(const ZoomArgs& a);
// split zoom: warp-chunk FIR into work rows (z_stride >= nout), then FFT + band gather per row
bool zoom_wfir_fits(const ZoomArgs& a, bool f32, const void* x, long long x_stride);
cudaError_t launch_zoom_wfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch, const void* g,
                             const void* S, void* zb, long long z_stride, cudaStream_t st);
cudaError_t launch_zoom_fftband(int log2n, bool f32, const void* zb, long long z_stride, int nout, long long batch,
                                int k_lo, int nbins, const void* tw, const void* band, void* out, long long out_stride,
                                cudaStream_t st);
// phase-lane FIR (power-of-two D <= 16, short phase rows): zoom_pfir_lh(a) > 0 when available;
// gnat = the taps in natural order g[t] (wrap terms)
int zoom_pfir_lh(const ZoomArgs& a);
cudaError_t launch_zoom_pfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                             const void* gph, const void* gnat, const void* S, void* zb, long long z_stride,
                             cudaStream_t st);
// the phase-lane FIR fed by a TMA pipeline of whole records (kernels_zoom_tfir.cu): circular,
// untrimmed, power-of-two U, D in {4, 8, 16}, 16-byte aligned rows
bool zoom_tfir_fits(const ZoomArgs& a, bool f32, const void* x, long long x_stride);
cudaError_t launch_zoom_tfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                             const void* gph, const void* gnat, const void* S, void* zb, long long z_stride,
                             cudaStream_t st);
// whole-output FIR with constant-bank taps and cp.async-filled polyphase rows (kernels_zoom_pcfir.cu):
// circular, untrimmed, nout a multiple of 256, (D, T) in {(8, 65), (8, 101)}; gnat_host = the plan's
// natural-order taps as interleaved fp64 complex
// fuse: the n_fft = 512 transform + band gather in the same launch (zoom_pcfir_fused_fits), output
// straight to out; else the decimated rows to zb
// raw-window whole-output FIR (kernels_zoom_rfir.cu): D in {4, 16}, 101 taps, untrimmed
bool zoom_rfir_fits(const ZoomArgs& a, bool f32, const void* x, long long x_stride);
cudaError_t launch_zoom_rfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                             const void* gnat_host, const void* gnat, const void* S, void* zb, long long z_stride,
                             cudaStream_t st);
bool zoom_rfir_fft_fits(const ZoomArgs& a, bool f32, int log2n);
cudaError_t launch_zoom_rfir_fft(const ZoomArgs& a, bool f32, int log2n, const void* x, long long xs, long long batch,
                                 const void* gnat_host, const void* S, const void* tw, const void* band, void* out,
                                 long long out_stride, cudaStream_t st);
bool zoom_pcfir_fits(const ZoomArgs& a, bool f32);
bool zoom_pcfir_fused_fits(const ZoomArgs& a, bool f32, int log2n);
cudaError_t launch_zoom_pcfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                              const void* gnat_host, const void* S, void* zb, long long z_stride, bool fuse,
                              const void* tw, const void* band, void* out, long long out_stride, cudaStream_t st);
// the phase-lane FIR and the short FFT + band gather in one kernel (kernels_zoom_fused.cu); returns
// cudaErrorNotSupported outside its instantiated geometry (the caller then runs the split route)
cudaError_t launch_zoom_pfir_fft(const ZoomArgs& a, int lh, int log2n, bool f32, const void* x, long long xs,
                                 long long batch, const void* gph, const void* gnat, const void* S, const void* tw,
                                 int k_lo, int nbins, const void* band, void* out, long long out_stride,
                                 cudaStream_t st);
// circular zoom with n_fft = U / D in the frequency domain (kernels_zoom_spec.cu): one U-point FFT of
// the shifted trace, x DFT_U(h), D-term alias sum per band bin; U = 2^log2u (2^8 .. single-CTA max)
cudaError_t launch_zoom_spec(int log2u, bool f32, const void* x, long long xs, long long batch, const void* tw,
                             const void* shift, const void* hf, int nf, int D, int k_lo, int nbins, const void* band,
                             void* out, long long os, cudaStream_t st);
// constant-bank FIR specialised on (D, T) (kernels_zoom_cfir.cu); gph_host = the plan's phase-row
// taps as interleaved fp64 complex (D x lh)
bool zoom_cfir_available(const ZoomArgs& a);
cudaError_t launch_zoom_cfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                             const void* gph_host, const void* gnat, const void* S, void* zb, long long z_stride,
                             cudaStream_t st);
// shared bytes the fused zoom kernel needs for this geometry
size_t zoom_smem_bytes(const ZoomArgs& a, int log2n, bool f32);

// ---- cluster FFT (kernels_cluster.cu): one L-point transform per 8-CTA cluster, DSMEM exchange ----
// log2 of the per-CTA length Q = L / 8 when L has a cluster instantiation (fp64 2^15..2^16,
// fp32 2^16..2^17), else 0
int cluster_fft_log2q(int log2L, bool f32);
// in_kind 0 complex rows / 1 real rows; mode 0 all L bins, 1 bins 0..L/2; tw_q = Stockham tables of
// the Q-point transform, twc = W_L^{r k2} (r < 8, k2 < Q) row-major
cudaError_t launch_fft_cluster(int log2L, bool f32, bool inverse, int mode, const void* x, int in_kind,
                               long long x_stride, long long N, long long batch, const void* tw_q, const void* twc,
                               void* out, long long out_stride, double scale, cudaStream_t st);

// band slice + magnitude_db of complex rows (slice_band spectra.cpp:40-61, magnitude_db types.cpp:13-18):
// bins [klo, klo + nb) of each input row -> out (optional) and dB (optional)
cudaError_t launch_band_db(bool f32, const void* in, long long in_stride, long long klo, long long nb,
                           long long batch, void* out, long long out_stride, void* db, long long db_stride,
                           cudaStream_t st);

// elementwise helpers
cudaError_t launch_c64_to_c32(const void* in, void* out, long long n, cudaStream_t st);
cudaError_t launch_scale_c64(void* data, long long n, double s, cudaStream_t st);

}  // namespace skg
