// spectral_b200.hpp — the reference's C++ transform API (namespace spectral, /root/reference/proj/src
// numerics.hpp, czt.hpp, spectra.hpp, zoomfft.hpp, types.hpp) re-declared over the B200 library.
//
// Same class names, member functions, argument meaning, output layout and exceptions
// (std::invalid_argument for every validation, as in the reference), so code written against
// spectralkit's C++ headers recompiles against this one and links libspectralkit_b200.so. Every
// transform runs on the GPU: host spans are copied to device memory inside the call (use
// spectralkit_gpu.h for device-resident batches). Plans keep their tables on the device and are
// immutable after construction (numerics.hpp:24-26).
#pragma once

#include <complex>
#include <cstddef>
#include <iosfwd>
#include <stdexcept>
#include <string>
#include <memory>
#include <optional>
#include <span>
#include <vector>

#pragma GCC visibility push(default)

namespace spectral {

using cplx = std::complex<double>;                  // types.hpp:9
using ComplexBuffer = std::vector<cplx>;            // types.hpp:10

struct Trace {                                      // types.hpp:13-19
    std::vector<double> samples;
    double sample_rate_hz = 0.0;
    double t0_s = 0.0;
    std::size_t size() const { return samples.size(); }
};

struct Spectrum {                                   // types.hpp:23-36
    ComplexBuffer bins;
    double f_start_hz = 0.0;
    double f_step_hz = 0.0;
    std::size_t source_n = 0;
    std::size_t size() const { return bins.size(); }
    double frequency(std::size_t k) const { return f_start_hz + static_cast<double>(k) * f_step_hz; }
    double f_end_hz() const { return bins.empty() ? f_start_hz : frequency(bins.size() - 1); }
};

double magnitude_db(const cplx& v);                 // types.cpp:13-18
double magnitude_db(double mag);
void validate_trace(const Trace& t);                // types.cpp:20-27

bool is_pow2(std::size_t n);                        // numerics.hpp:11-14
std::size_t next_pow2(std::size_t n);
ComplexBuffer zero_pad(std::span<const cplx> x, std::size_t target_len);   // numerics.hpp:17
ComplexBuffer dft_naive(std::span<const cplx> x);                         // numerics.hpp:22
cplx cis_cycles(double q, double t);                                       // numerics.hpp:52

class FftPlan {                                     // numerics.hpp:27-43
  public:
    explicit FftPlan(std::size_t n);                // n must be a power of two
    void forward(std::span<cplx> data) const;
    void inverse(std::span<cplx> data) const;       // applies 1/n
    std::size_t size() const { return n_; }

  private:
    void run(std::span<cplx> data, bool invert) const;
    std::size_t n_ = 0;
};

ComplexBuffer fft(std::span<const cplx> x);         // numerics.hpp:47-48
ComplexBuffer ifft(std::span<const cplx> x);

struct CztParams {                                  // czt.hpp:13-17
    cplx a{1.0, 0.0};
    cplx w{1.0, 0.0};
    std::size_t m = 0;
};
void validate(const CztParams& p);
CztParams czt_params_for_band(double f1_hz, double f2_hz, double sample_rate_hz, std::size_t m);
ComplexBuffer czt_direct(std::span<const cplx> x, const CztParams& p);

class CztPlan {                                     // czt.hpp:34-56
  public:
    CztPlan(std::size_t input_len, const CztParams& p);
    ComplexBuffer execute(std::span<const cplx> x) const;
    void execute(std::span<const cplx> x, std::span<cplx> conv_scratch, std::span<cplx> out) const;
    std::size_t input_size() const;
    std::size_t output_size() const;
    std::size_t conv_size() const;

  private:
    std::shared_ptr<const void> impl_;
};

ComplexBuffer czt(std::span<const cplx> x, const CztParams& p);            // czt.hpp:59
ComplexBuffer dft_any(std::span<const cplx> x);                           // czt.hpp:63
Spectrum czt_spectrum(const Trace& trace, double f1_hz, double f2_hz, std::size_t m);

Spectrum fft_spectrum(const Trace& t, std::size_t transform_len = 0);     // spectra.hpp:14
Spectrum slice_band(const Spectrum& s, double f_lo_hz, double f_hi_hz);   // spectra.hpp:19

struct ZoomOptions {                                // zoomfft.hpp:17-26
    double center_hz = 0.0;
    bool center_set = false;
    std::size_t decimation = 0;
    double cutoff_hz = 0.0;
    std::size_t num_taps = 0;
    bool circular = true;
    bool trim_transient = false;
    bool pad_pow2 = true;
};

struct ZoomFftPlan {                                // zoomfft.hpp:33-56 (public fields kept)
    double f1_hz = 0.0;
    double f2_hz = 0.0;
    double center_hz = 0.0;
    double sample_rate_hz = 0.0;
    double cutoff_hz = 0.0;
    std::size_t decimation = 1;
    std::vector<double> filter_taps;
    double group_delay_samples = 0.0;
    bool circular = true;
    bool trim_transient = false;
    bool pad_pow2 = true;
    std::size_t input_len = 0;
    std::size_t usable_len = 0;
    std::size_t trim_samples = 0;
    std::size_t decimated_len = 0;
    std::size_t n_fft = 0;
    double f_step_hz() const;
    // device plan, built from the fields above on first use (and rebuilt if they are edited)
    mutable std::shared_ptr<void> device;
};

std::vector<double> design_lowpass(double cutoff_hz, double sample_rate_hz, std::size_t num_taps);
ComplexBuffer frequency_shift(std::span<const double> x, double f_shift_hz, double sample_rate_hz);
ComplexBuffer frequency_shift(std::span<const cplx> x, double f_shift_hz, double sample_rate_hz);
ComplexBuffer filter_decimate(std::span<const cplx> x, std::span<const double> taps, std::size_t d);
ComplexBuffer filter_decimate_circular(std::span<const cplx> x, std::span<const double> taps, std::size_t d);
ZoomFftPlan make_zoom_plan(std::size_t input_len, double f1_hz, double f2_hz, double sample_rate_hz,
                           const ZoomOptions& opts = {});
Spectrum zoom_fft(const ZoomFftPlan& plan, const Trace& t);


// ---- errors.hpp:9-30 ---------------------------------------------------------------------------
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
    ParseError(const std::string& msg, std::size_t line_no) : std::runtime_error(msg), line(line_no) {}
    std::size_t line = 0;
};
struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InsufficientResolutionError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- trace / spectrum CSV (signals.hpp, spectra.hpp; byte-identical formats) -------------------
Trace read_trace_csv(std::istream& in, const std::string& origin);      // signals.cpp:125-170
Trace read_trace_csv_file(const std::string& path);
void write_trace_csv(const Trace& t, std::ostream& out);                // signals.cpp:178-189
void write_trace_csv_file(const Trace& t, const std::string& path);
Spectrum read_spectrum_csv(std::istream& in, const std::string& origin);    // spectra.cpp:94-150
Spectrum read_spectrum_csv_file(const std::string& path);
void write_spectrum_csv(const Spectrum& s, std::ostream& out);              // spectra.cpp:63-72
void write_spectrum_csv_file(const Spectrum& s, const std::string& path);
void write_spectrum_json(const Spectrum& s, std::ostream& out);             // spectra.cpp:161-176
void write_spectrum_json_file(const Spectrum& s, const std::string& path);

// ---- resolution.hpp sizing helpers --------------------------------------------------------------
std::size_t record_len_for_step(double sample_rate_hz, double target_step_hz);
double fft_resolution(double sample_rate_hz, std::size_t n);
std::size_t zeros_for_resolution(double sample_rate_hz, std::size_t n, double target_step_hz);
std::size_t czt_len_for_matched_resolution(double f1_hz, double f2_hz, double sample_rate_hz, std::size_t n_fft);

// ---- analysis.hpp: two-tone valley test and the resolvability sweep (both routes batched on the GPU)
struct DipMetric {
    bool resolved = false;
    double dip_db = 0.0;
    double f_peak_a_hz = 0.0;
    double peak_a_db = 0.0;
    double f_peak_b_hz = 0.0;
    double peak_b_db = 0.0;
    double f_valley_hz = 0.0;
    double valley_db = 0.0;
};
DipMetric dip_metric(const Spectrum& s, double f_a_hz, double f_b_hz);
struct ScanConfig {
    double sample_rate_hz = 8000.0;
    std::size_t n = 128;
    double f1_hz = 100.0;
    double f2_hz = 1000.0;
    std::size_t m = 128;
    double center_hz = 0.0;
    double sep_start_hz = 10.0;
    double sep_stop_hz = 200.0;
    double sep_step_hz = 5.0;
};
struct ResolvabilityCurve {
    ScanConfig config;
    std::vector<double> separations_hz;
    std::vector<DipMetric> fft_metrics;
    std::vector<DipMetric> czt_metrics;
    double min_resolved_fft_hz = 0.0;
    double min_resolved_czt_hz = 0.0;
    std::size_t fft_len = 0;
};
ResolvabilityCurve resolvability_scan(const ScanConfig& cfg);
void write_resolvability_csv(const ResolvabilityCurve& c, std::ostream& out);   // serialize.cpp:141-154
void write_resolvability_json(const ResolvabilityCurve& c, std::ostream& out);  // serialize.cpp:113-135

}  // namespace spectral

#pragma GCC visibility pop
