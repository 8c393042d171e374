// analysis.cpp — see analysis.hpp. Restates analysis.cpp:19-195, resolution.cpp:11-47 and
// gen_two_tone (signals.cpp:24-44) of the reference; the transforms are the batched GPU kernels.
#include "analysis.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <numbers>
#include <string>

#include "host.hpp"
#include "io.hpp"

namespace skg {

namespace {

void check_rate(double fs) {
    if (!(fs > 0.0) || !std::isfinite(fs)) throw std::invalid_argument("sample rate must be positive and finite");
}

double mag_db(double mag) { return mag > 1e-15 ? 20.0 * std::log10(mag) : -300.0; }   // types.cpp:13-16

bool is_local_max(const std::vector<double>& m, size_t k) {   // analysis.cpp:20-26
    const size_t last = m.size() - 1;
    if (k == 0) return m[0] > m[1];
    if (k == last) return m[last] > m[last - 1];
    if (m[k] < m[k - 1] || m[k] < m[k + 1]) return false;
    return m[k] > m[k - 1] || m[k] > m[k + 1];
}

}  // namespace

size_t record_len_for_step(double fs, double step) {
    check_rate(fs);
    if (!(step > 0.0)) throw std::invalid_argument("record_len_for_step: target step must be positive");
    const double q = fs / step;
    const double qr = std::round(q);
    if (std::abs(q - qr) <= 1e-9 * q) return static_cast<size_t>(qr);
    return static_cast<size_t>(std::ceil(q));
}

double fft_resolution(double fs, size_t n) {
    check_rate(fs);
    if (n == 0) throw std::invalid_argument("fft_resolution: n must be >= 1");
    return fs / static_cast<double>(n);
}

size_t czt_len_for_matched_resolution(double f1, double f2, double fs, size_t n_fft) {
    check_rate(fs);
    if (n_fft == 0) throw std::invalid_argument("czt_len_for_matched_resolution: n_fft must be >= 1");
    if (!(f1 >= 0.0) || !(f1 < f2)) throw std::invalid_argument("czt_len_for_matched_resolution: need 0 <= f1 < f2");
    if (f2 > fs / 2.0 * (1.0 + 1e-12))
        throw std::invalid_argument("czt_len_for_matched_resolution: band edge exceeds the usable half rate");
    const double m = std::round((f2 - f1) / fs * static_cast<double>(n_fft));
    return m < 1.0 ? 1 : static_cast<size_t>(m);
}

std::string format_resolvability_csv(const CurveH& c) {
    std::string out = "separation_hz,method,resolved,dip_db,f_peak_a_hz,peak_a_db,f_peak_b_hz,peak_b_db,"
                      "f_valley_hz,valley_db\n";
    auto fields = [&](const DipMetricH& m) {
        out += m.resolved ? "1" : "0";
        for (double v : {m.dip_db, m.f_peak_a_hz, m.peak_a_db, m.f_peak_b_hz, m.peak_b_db, m.f_valley_hz, m.valley_db}) {
            out += ',';
            append_g17(out, v);
        }
    };
    for (size_t i = 0; i < c.separations_hz.size(); ++i) {
        std::string sep;
        append_g17(sep, c.separations_hz[i]);
        out += sep + ",fft,";
        fields(c.fft_metrics[i]);
        out += "\n" + sep + ",czt,";
        fields(c.czt_metrics[i]);
        out += '\n';
    }
    return out;
}

std::string format_resolvability_json(const CurveH& c) {
    // keys in sorted order at every level (the library's object is an ordered map), two-space indent
    std::string o = "{\n  \"config\": {\n";
    auto num = [&](const char* ind, const char* key, double v, bool last) {
        o += ind;
        o += '"';
        o += key;
        o += "\": ";
        json_number(o, v);
        o += last ? "\n" : ",\n";
    };
    auto uint = [&](const char* ind, const char* key, size_t v, bool last) {
        o += ind;
        o += '"';
        o += key;
        o += "\": " + std::to_string(v) + (last ? "\n" : ",\n");
    };
    const char* i4 = "    ";
    num(i4, "center_hz", c.config.center_hz, false);
    num(i4, "f1_hz", c.config.f1_hz, false);
    num(i4, "f2_hz", c.config.f2_hz, false);
    uint(i4, "m", c.config.m, false);
    uint(i4, "n", c.config.n, false);
    num(i4, "sample_rate_hz", c.config.sample_rate_hz, false);
    num(i4, "sep_start_hz", c.config.sep_start_hz, false);
    num(i4, "sep_step_hz", c.config.sep_step_hz, false);
    num(i4, "sep_stop_hz", c.config.sep_stop_hz, true);
    o += "  },\n";
    auto metrics = [&](const char* key, const std::vector<DipMetricH>& ms) {
        o += "  \"";
        o += key;
        o += "\": ";
        if (ms.empty()) {
            o += "[],\n";
            return;
        }
        o += "[\n";
        const char* i6 = "      ";
        for (size_t i = 0; i < ms.size(); ++i) {
            const DipMetricH& m = ms[i];
            o += "    {\n";
            num(i6, "dip_db", m.dip_db, false);
            num(i6, "f_peak_a_hz", m.f_peak_a_hz, false);
            num(i6, "f_peak_b_hz", m.f_peak_b_hz, false);
            num(i6, "f_valley_hz", m.f_valley_hz, false);
            num(i6, "peak_a_db", m.peak_a_db, false);
            num(i6, "peak_b_db", m.peak_b_db, false);
            o += i6;
            o += m.resolved ? "\"resolved\": true,\n" : "\"resolved\": false,\n";
            num(i6, "valley_db", m.valley_db, true);
            o += i + 1 < ms.size() ? "    },\n" : "    }\n";
        }
        o += "  ],\n";
    };
    metrics("czt", c.czt_metrics);
    metrics("fft", c.fft_metrics);
    uint("  ", "fft_len", c.fft_len, false);
    num("  ", "min_resolved_czt_hz", c.min_resolved_czt_hz, false);
    num("  ", "min_resolved_fft_hz", c.min_resolved_fft_hz, false);
    o += "  \"separations_hz\": ";
    if (c.separations_hz.empty()) {
        o += "[],\n";
    } else {
        o += "[\n";
        for (size_t i = 0; i < c.separations_hz.size(); ++i) {
            o += "    ";
            json_number(o, c.separations_hz[i]);
            o += i + 1 < c.separations_hz.size() ? ",\n" : "\n";
        }
        o += "  ],\n";
    }
    o += "  \"v\": 1\n}\n";
    return o;
}

size_t zeros_for_resolution(double fs, size_t n, double step) {
    check_rate(fs);
    if (n == 0) throw std::invalid_argument("zeros_for_resolution: n must be >= 1");
    if (!(step > 0.0)) throw std::invalid_argument("zeros_for_resolution: target step must be positive");
    const double natural = fs / static_cast<double>(n);
    if (step > natural * (1.0 + 1e-12))
        throw std::invalid_argument("zeros_for_resolution: target step " + std::to_string(step) +
                                    " Hz is coarser than the unpadded spacing " + std::to_string(natural) + " Hz");
    const size_t total = record_len_for_step(fs, step);
    return total <= n ? 0 : total - n;
}

DipMetricH dip_metric(const std::complex<double>* bins, size_t n, double f_start, double f_step, double f_a,
                      double f_b) {
    if (n < 2 || !(f_step > 0.0)) throw std::invalid_argument("dip_metric: need a spectrum with a real axis");
    if (!(f_a < f_b)) throw std::invalid_argument("dip_metric: need f_a < f_b");
    const double half = 0.5 * f_step;
    const double f_end = f_start + static_cast<double>(n - 1) * f_step;
    if (f_a < f_start - half || f_b > f_end + half)
        throw std::invalid_argument("dip_metric: tone frequencies fall off the axis");
    const double tiny = 1e-9;
    const long k_a = static_cast<long>(std::ceil((f_a - f_start) / f_step - tiny));
    const long k_b = static_cast<long>(std::floor((f_b - f_start) / f_step + tiny));
    if (k_b - k_a + 1 < 3)
        throw InsufficientResolution(
            "dip_metric: fewer than 3 bins between the tones; the axis cannot hold a valley at this separation");
    std::vector<double> mags(n);
    for (size_t k = 0; k < n; ++k) mags[k] = std::abs(bins[k]);
    std::vector<size_t> maxima;
    for (size_t k = 0; k < n; ++k)
        if (is_local_max(mags, k)) maxima.push_back(k);
    DipMetricH m;
    if (maxima.empty()) return m;
    auto freq = [&](size_t k) { return f_start + static_cast<double>(k) * f_step; };
    auto nearest = [&](double f) {
        size_t best = maxima.front();
        double best_d = std::abs(freq(best) - f);
        for (size_t k : maxima) {
            const double d = std::abs(freq(k) - f);
            if (d < best_d) {
                best_d = d;
                best = k;
            }
        }
        return best;
    };
    const size_t pa = nearest(f_a), pb = nearest(f_b);
    m.f_peak_a_hz = freq(pa);
    m.peak_a_db = mag_db(mags[pa]);
    m.f_peak_b_hz = freq(pb);
    m.peak_b_db = mag_db(mags[pb]);
    const size_t lo = std::min(pa, pb), hi = std::max(pa, pb);
    if (hi - lo <= 1) {
        const size_t weaker = mags[pa] <= mags[pb] ? pa : pb;
        m.f_valley_hz = freq(weaker);
        m.valley_db = mag_db(mags[weaker]);
        return m;
    }
    size_t v = lo + 1;
    for (size_t k = lo + 2; k < hi; ++k)
        if (mags[k] < mags[v]) v = k;
    m.f_valley_hz = freq(v);
    m.valley_db = mag_db(mags[v]);
    const double weaker = std::min(mags[pa], mags[pb]);
    m.resolved = mags[v] < weaker;
    m.dip_db = mags[v] == 0.0 ? std::numeric_limits<double>::infinity() : 20.0 * std::log10(weaker / mags[v]);
    return m;
}

CurveH resolvability_scan(const ScanConfigH& cfg, int threads) {
    // analysis.cpp:99-114: the same checks in the same order
    if (!(cfg.sample_rate_hz > 0.0)) throw std::invalid_argument("resolvability_scan: sample rate must be positive");
    if (cfg.n < 2) throw std::invalid_argument("resolvability_scan: record too short");
    if (!(cfg.f1_hz >= 0.0) || !(cfg.f2_hz > cfg.f1_hz) || cfg.f2_hz > cfg.sample_rate_hz / 2.0 * (1.0 + 1e-12))
        throw std::invalid_argument("resolvability_scan: band must satisfy 0 <= f1 < f2 <= fs/2");
    if (cfg.m < 2) throw std::invalid_argument("resolvability_scan: need at least 2 band bins");
    if (!(cfg.sep_start_hz > 0.0) || !(cfg.sep_step_hz > 0.0) || cfg.sep_stop_hz < cfg.sep_start_hz)
        throw std::invalid_argument("resolvability_scan: bad separation sweep");
    const double center = cfg.center_hz > 0.0 ? cfg.center_hz : 0.5 * (cfg.f1_hz + cfg.f2_hz);
    if (center - cfg.sep_stop_hz / 2.0 < cfg.f1_hz || center + cfg.sep_stop_hz / 2.0 > cfg.f2_hz)
        throw std::invalid_argument("resolvability_scan: tone pair leaves the band at the widest separation");
    const double fs = cfg.sample_rate_hz;
    const double czt_step = (cfg.f2_hz - cfg.f1_hz) / static_cast<double>(cfg.m);
    const size_t fft_len = cfg.n + zeros_for_resolution(fs, cfg.n, czt_step);

    CurveH curve;
    curve.config = cfg;
    curve.config.center_hz = center;
    curve.fft_len = fft_len;
    curve.min_resolved_fft_hz = std::numeric_limits<double>::quiet_NaN();
    curve.min_resolved_czt_hz = std::numeric_limits<double>::quiet_NaN();
    for (size_t i = 0;; ++i) {   // analysis.cpp:134-137
        const double sep = cfg.sep_start_hz + static_cast<double>(i) * cfg.sep_step_hz;
        if (sep > cfg.sep_stop_hz * (1.0 + 1e-12)) break;
        curve.separations_hz.push_back(sep);
    }
    const size_t S = curve.separations_hz.size(), n = cfg.n;
    // gen_two_tone (signals.cpp:24-44) for every separation: unit amplitudes, zero phases
    std::vector<double> x(S * n);
    constexpr double two_pi = 2.0 * std::numbers::pi;
    parallel_for(S, threads, [&](size_t s) {
        const double sep = curve.separations_hz[s];
        const double fa = center - sep / 2.0, fb = center + sep / 2.0;
        const double nyq = fs / 2.0;
        if (!(fa >= 0.0) || !(fb >= 0.0) || fa >= nyq || fb >= nyq)
            throw std::invalid_argument("gen_two_tone: tone frequencies must lie in [0, fs/2)");
        for (size_t i = 0; i < n; ++i) {
            const double ti = static_cast<double>(i) / fs;
            x[s * n + i] = 1.0 * std::sin(two_pi * fa * ti + 0.0) + 1.0 * std::sin(two_pi * fb * ti + 0.0);
        }
    });
    // the two routes as batched GPU launches (fp64)
    require_device();
    const BandBins bb = slice_band_bins(fft_len, 0.0, fs / static_cast<double>(fft_len), cfg.f1_hz, cfg.f2_hz);
    const cd a = cis_cycles(cfg.f1_hz / fs, 1.0);   // czt_params_for_band (czt.cpp:42-56)
    const cd w = cis_cycles(-(cfg.f2_hz - cfg.f1_hz) / (static_cast<double>(cfg.m) * fs), 1.0);
    CztPlanG band_plan(n, a, w, cfg.m);
    cudaStream_t st = cudaStreamPerThread;
    DevMem dx(S * n * sizeof(double)), dfft((size_t)S * bb.count * sizeof(cd)), dczt(S * cfg.m * sizeof(cd));
    dx.upload(x.data(), x.size() * sizeof(double), st);
    fft_spectrum_band_batch(n, fft_len, false, bb.k_lo, bb.count, dx.p, (long long)n, (long long)S, dfft.p,
                            bb.count, nullptr, 0, st);
    band_plan.execute(dx.p, false, (long long)n, (long long)S, dczt.p, (long long)cfg.m, false, st);
    std::vector<cd> hfft((size_t)S * bb.count), hczt(S * cfg.m);
    check(cudaMemcpyAsync(hfft.data(), dfft.p, hfft.size() * sizeof(cd), cudaMemcpyDeviceToHost, st), "D2H");
    check(cudaMemcpyAsync(hczt.data(), dczt.p, hczt.size() * sizeof(cd), cudaMemcpyDeviceToHost, st), "D2H");
    check(cudaStreamSynchronize(st), "sync");
    // the valley test per separation; a separation too tight for the axis is unresolved, not an error
    curve.fft_metrics.resize(S);
    curve.czt_metrics.resize(S);
    const double fstep = fs / static_cast<double>(fft_len);
    parallel_for(S, threads, [&](size_t s) {
        const double sep = curve.separations_hz[s];
        const double fa = center - sep / 2.0, fb = center + sep / 2.0;
        auto metric = [&](const cd* b, size_t nb, double f0, double df) {
            try {
                return dip_metric(b, nb, f0, df, fa, fb);
            } catch (const InsufficientResolution&) {
                return DipMetricH{};
            }
        };
        curve.fft_metrics[s] = metric(hfft.data() + s * bb.count, (size_t)bb.count, bb.f_start, fstep);
        curve.czt_metrics[s] = metric(hczt.data() + s * cfg.m, cfg.m, cfg.f1_hz, czt_step);
    });
    for (size_t i = 0; i < S; ++i) {
        if (curve.fft_metrics[i].resolved && std::isnan(curve.min_resolved_fft_hz))
            curve.min_resolved_fft_hz = curve.separations_hz[i];
        if (curve.czt_metrics[i].resolved && std::isnan(curve.min_resolved_czt_hz))
            curve.min_resolved_czt_hz = curve.separations_hz[i];
    }
    return curve;
}

}  // namespace skg
