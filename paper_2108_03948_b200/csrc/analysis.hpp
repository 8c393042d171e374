// analysis.hpp — the reference's two-tone resolvability sweep (analysis.cpp:30-195) as a batched
// caller of the GPU transforms: every separation's trace is generated on the host,
// both routes (padded full-range FFT sliced to the band, band CZT) run as ONE batched launch each,
// and the valley test runs per separation on host threads.
#pragma once

#include <complex>
#include <cstddef>
#include <stdexcept>
#include <vector>

namespace skg {

struct InsufficientResolution : std::runtime_error {   // errors.hpp:27-30
    using std::runtime_error::runtime_error;
};

struct DipMetricH {   // analysis.hpp:15-24
    bool resolved = false;
    double dip_db = 0.0, f_peak_a_hz = 0.0, peak_a_db = 0.0, f_peak_b_hz = 0.0, peak_b_db = 0.0;
    double f_valley_hz = 0.0, valley_db = 0.0;
};
DipMetricH dip_metric(const std::complex<double>* bins, size_t n, double f_start, double f_step, double f_a,
                      double f_b);

struct ScanConfigH {   // analysis.hpp:31-41 (defaults)
    double sample_rate_hz = 8000.0;
    size_t n = 128;
    double f1_hz = 100.0, f2_hz = 1000.0;
    size_t m = 128;
    double center_hz = 0.0, sep_start_hz = 10.0, sep_stop_hz = 200.0, sep_step_hz = 5.0;
};
struct CurveH {   // analysis.hpp:46-54
    ScanConfigH config;
    std::vector<double> separations_hz;
    std::vector<DipMetricH> fft_metrics, czt_metrics;
    double min_resolved_fft_hz = 0.0, min_resolved_czt_hz = 0.0;
    size_t fft_len = 0;
};
CurveH resolvability_scan(const ScanConfigH& cfg, int threads = 0);

// write_resolvability_csv (serialize.cpp:39-45, 141-154): two rows per separation, %.17g fields
std::string format_resolvability_csv(const CurveH& c);
// write_resolvability_json (serialize.cpp:113-135): the reference JSON library's object layout
std::string format_resolvability_json(const CurveH& c);

double fft_resolution(double fs, size_t n);                   // resolution.cpp:28-32
size_t czt_len_for_matched_resolution(double f1, double f2, double fs, size_t n_fft);   // resolution.cpp:49-63
size_t record_len_for_step(double fs, double step);           // resolution.cpp:18-26
size_t zeros_for_resolution(double fs, size_t n, double step);   // resolution.cpp:34-47

}  // namespace skg
