// host.hpp — host-side runtime of the B200 spectral library: errors, device memory, fp64 table
// builders (restating the reference's phase arithmetic) and the plan objects that own device
// tables. No torch types anywhere; the C ABI in capi.cpp is a thin layer over this.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.hpp"

namespace skg {

using cd = std::complex<double>;

// CUDA failures (reported as SK_ERR_INTERNAL by the C ABI)
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
void check(cudaError_t e, const char* what);
void require_device();          // throws CudaError when no usable CUDA device exists
int current_device();
// stream-ordered work buffer from the default pool (kept cached across synchronisations); free with cudaFreeAsync
void* stream_alloc(size_t bytes, cudaStream_t st);
std::atomic<uint64_t>& launch_counter();
std::atomic<unsigned>& grid_cap_ref();   // skg_debug_set_grid_cap
inline void count_launch(int n = 1) { launch_counter().fetch_add((uint64_t)n, std::memory_order_relaxed); }

// ---- numerics restated from the reference (fp64, host) ----------------------------------
bool is_pow2(size_t n);                         // numerics.cpp:14
size_t next_pow2(size_t n);                     // numerics.cpp:16-24 (throws invalid_argument)
int ilog2(size_t n);
cd cis_cycles(double q, double t);              // numerics.cpp:122-128
struct PolarPow {                               // czt.cpp:15-32
    double log_mag = 0.0, q = 0.0;
    explicit PolarPow(cd z);
    cd pow(double t) const;
};
std::vector<double> design_lowpass(double cutoff_hz, double fs, size_t taps);   // zoomfft.cpp:15-42

// ---- device memory -------------------------------------------------------------------------
struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    DevMem() = default;
    explicit DevMem(size_t n);
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    DevMem(DevMem&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DevMem& operator=(DevMem&& o) noexcept;
    ~DevMem();
    void upload(const void* host, size_t n, cudaStream_t st = nullptr);
};
// fp64 complex host table -> device table in the requested precision
DevMem to_device(const std::vector<cd>& h, bool f32);

// Plan tables keyed by (device, precision): a plan shared by threads bound to different GPUs
// builds one set of device tables per GPU on first use there (the Stockham twiddles are keyed the
// same way), so no kernel is ever handed another device's pointers.
template <typename D> class PerDevice {
  public:
    template <typename F> const D& get(bool f32, F&& build) const {
        const int key = current_device() * 2 + (f32 ? 1 : 0);
        std::lock_guard<std::mutex> lk(mu_);
        for (const auto& e : sets_)
            if (e.first == key) return *e.second;
        auto d = std::make_unique<D>();
        build(*d);
        sets_.emplace_back(key, std::move(d));
        return *sets_.back().second;
    }

  private:
    mutable std::mutex mu_;
    mutable std::vector<std::pair<int, std::unique_ptr<D>>> sets_;
};

// cached per-device twiddle tables for the Stockham engine (FftGeom<log2L>)
const void* stockham_twiddles(int log2L, bool f32);
// W_{2M}^k / 2, k < M: post-processing twiddles of the real-input transform (1/2 of the split folded in)
const void* r2c_post_twiddles(int log2M, bool f32);
// four-step tables: W_L^{r c} for the (R x C) split of L = R*C
const void* fourstep_twiddles(int log2R, int log2C, bool f32);

int single_cta_max_log2(bool f32);

// ---- transforms ----------------------------------------------------------------------------
// complex FFT of `batch` rows (device pointers); any power of two n
void fft_c2c(size_t n, bool inverse, bool f32, const void* in, long long in_stride, void* out,
             long long out_stride, long long batch, cudaStream_t st);

struct FourStepRef { const void* p; };   // host.cpp's four-step geometry, opaque here

// Bluestein chirp-z plan (CztPlan, czt.cpp:85-137) with device tables
class CztPlanG {
  public:
    CztPlanG(size_t n, cd a, cd w, size_t m);
    size_t input_size() const { return n_; }
    size_t output_size() const { return m_; }
    size_t conv_size() const { return L_; }          // the reference's next_pow2(n + m - 1), czt.hpp:46
    size_t segments() const { return nseg_; }        // output segments executed independently
    size_t segment_len() const { return seg_; }
    size_t segment_conv_size() const { return Ls_; } // transform length actually run per segment
    // x rows of n real (complex_in = false) or complex values; `load_n` <= n leading samples are
    // read (the rest are zeros — used by dft_any on zero-padded traces)
    void execute(const void* x, bool complex_in, long long x_stride, long long batch, void* out,
                 long long out_stride, bool f32, cudaStream_t st, size_t load_n = 0) const;

  private:
    struct Dev {
        DevMem cin, cout, khat;
        DevMem khat_sf, cout_sf;   // shared-forward tables (nseg > 1): per-block kernel spectra / out chirps
    };
    const Dev& dev(bool f32) const;
    // multi-pass plans: the one-launch pipeline (kernels_4step_czt.cuh); false = not applicable
    bool czt_4step_fused(const FourStepRef& f, bool f32, const void* x, bool complex_in, long long x_stride, long long N,
                         const Dev& d, long long batch, void* out, long long out_stride, cudaStream_t st) const;
    size_t n_, m_, L_;
    size_t nseg_ = 1, seg_ = 0, Ls_ = 0;
    int log2L_;   // of Ls_
    std::vector<cd> cin_, cout_, kern_;
    std::vector<cd> kern_sf_, cout_sf_;   // nseg x Ls kernel segments, nseg x seg output chirps
    PerDevice<Dev> devs_;
};

// zero-padded spectrum of real traces; layout 0 full, 1 half (pow2 only)
void fft_spectrum_batch(size_t n, size_t len, bool f32, int layout, const void* x, long long x_stride,
                        long long batch, void* out, long long out_stride, cudaStream_t st);
// slice_band (spectra.cpp:40-61) on a spectrum of `size` bins at f_start + k f_step: first bin and
// count of the band [f_lo, f_hi], with the reference's 1e-9 step slack and its errors
struct BandBins {
    long long k_lo = 0, count = 0;
    double f_start = 0.0;
};
BandBins slice_band_bins(size_t size, double f_start, double f_step, double f_lo, double f_hi);
// zero-padded spectrum restricted to bins [k_lo, k_lo + count) of the full [0, fs) layout, as complex
// (out, optional) and magnitude_db (db, optional); fused into the FFT store when the FFT is one CTA
void fft_spectrum_band_batch(size_t n, size_t len, bool f32, long long k_lo, long long count, const void* x,
                             long long x_stride, long long batch, void* out, long long out_stride, void* db,
                             long long db_stride, cudaStream_t st);
void band_db_batch(bool f32, const void* in, long long in_stride, long long k_lo, long long count, long long batch,
                   void* out, long long out_stride, void* db, long long db_stride, cudaStream_t st);

class TransferPlanG {
  public:
    TransferPlanG(const double* ref, size_t n, size_t len, bool f32);
    size_t bins() const { return len_ / 2 + 1; }
    size_t input_size() const { return n_; }
    bool f32() const { return f32_; }
    const std::vector<cd>& reference_spectrum() const { return xref_; }
    const void* rtab(bool f32) const;   // device 1 / X_ref on the current device
    void execute(const void* x, long long x_stride, long long batch, void* mag, void* phase,
                 long long mp_stride, void* h, long long h_stride, cudaStream_t st) const;

  private:
    size_t n_, len_;
    bool f32_;
    std::vector<cd> xref_;
    std::vector<cd> rtab_h_;   // 1 / X_ref, fp64
    PerDevice<DevMem> rtab_;
};

struct ZoomOptionsG {                 // ZoomOptions, zoomfft.hpp:17-26
    double center_hz = 0.0;
    bool center_set = false;
    size_t decimation = 0;
    double cutoff_hz = 0.0;
    size_t num_taps = 0;
    bool circular = true;
    bool trim_transient = false;
    bool pad_pow2 = true;
};

struct ZoomFields {                   // the public fields of ZoomFftPlan (zoomfft.hpp:34-50)
    double f1_hz = 0, f2_hz = 0, center_hz = 0, sample_rate_hz = 0, cutoff_hz = 0;
    size_t decimation = 1;
    std::vector<double> filter_taps;
    double group_delay_samples = 0;
    bool circular = true, trim_transient = false, pad_pow2 = true;
    size_t input_len = 0, usable_len = 0, trim_samples = 0, decimated_len = 0, n_fft = 0;
};

class ZoomPlanG {                     // ZoomFftPlan + make_zoom_plan, zoomfft.hpp:33-56
  public:
    ZoomPlanG(size_t input_len, double f1, double f2, double fs, const ZoomOptionsG& o,
              size_t n_fft_override = 0, const double* taps = nullptr, size_t num_taps = 0);
    // a plan whose public fields were set (or edited) directly, as the reference's ZoomFftPlan allows
    // (zoomfft.hpp:33-56): band window and chirp-route plan are derived from the fields
    static std::unique_ptr<ZoomPlanG> from_fields(const ZoomFields& fields);
    double f1_hz, f2_hz, center_hz, sample_rate_hz, cutoff_hz;
    size_t decimation = 1;
    std::vector<double> filter_taps;
    double group_delay_samples = 0.0;
    bool circular = true, trim_transient = false, pad_pow2 = true;
    size_t input_len = 0, usable_len = 0, trim_samples = 0, decimated_len = 0, n_fft = 0;
    long k_lo = 0, k_hi = -1;         // signed band window (zoomfft.cpp:209-219)
    double f_step_hz() const;
    size_t bins() const { return (size_t)(k_hi - k_lo + 1); }
    double f_start_hz() const;
    void execute(const void* x, long long x_stride, long long batch, void* out, long long out_stride,
                 bool f32, cudaStream_t st) const;

  private:
    ZoomPlanG() = default;
    struct Dev {
        DevMem g, gn, sdec, wrap, band;
        DevMem shift, hf;     // frequency-domain route: e^{-i2pi fc n/fs} (n < U), DFT_U of the taps
        std::vector<cd> gh;   // host copy of g (phase rows, fp64) for the constant-bank FIR
        std::vector<cd> gnh;  // host copy of g in natural order (fp64) for the whole-output FIR
    };
    const Dev& dev(bool f32) const;
    void compute_band();
    bool spectral_route_ok() const;
    PerDevice<Dev> devs_;
    std::unique_ptr<CztPlanG> bluestein_;   // n_fft not a power of two (dft_any route)
};

}  // namespace skg
