// C++ API drop-in check: reference-style unit tests (test_numerics.cpp, test_czt.cpp, test_spectra.cpp,
// test_zoomfft.cpp) written against include/spectral_b200.hpp and linked to libspectralkit_b200.so.
// Built and run by tests/test_cpp_api.py (compile+link on CPU, run on the GPU).
#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>

#include "spectral_b200.hpp"

using namespace spectral;

static int failures = 0;
#define CHECK(c)                                                             \
    do {                                                                     \
        if (!(c)) {                                                          \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);         \
            ++failures;                                                      \
        }                                                                    \
    } while (0)
template <typename F> static bool throws_invalid(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static double rel_error(const ComplexBuffer& got, const ComplexBuffer& want) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < got.size(); ++i) {
        num = std::max(num, std::abs(got[i] - want[i]));
        den = std::max(den, std::abs(want[i]));
    }
    return den > 0 ? num / den : num;
}

static ComplexBuffer random_buf(size_t n, std::mt19937_64& rng) {
    std::uniform_real_distribution<double> d(-1.0, 1.0);
    ComplexBuffer x(n);
    for (auto& v : x) v = cplx(d(rng), d(rng));
    return x;
}

int main() {
    // numerics: KAT, errors, plan reuse, round trip
    const ComplexBuffer k4{{1, 0}, {2, 0}, {3, 0}, {4, 0}};
    const ComplexBuffer X4 = fft(k4);
    CHECK(std::abs(X4[1] - cplx(-2, 2)) < 1e-12 && std::abs(X4[3] - cplx(-2, -2)) < 1e-12);
    CHECK(rel_error(dft_naive(k4), X4) < 1e-12);
    try {
        fft(ComplexBuffer(6, cplx(1, 0)));
        CHECK(false);
    } catch (const std::invalid_argument& e) {
        const std::string m = e.what();
        CHECK(m.find("pad") != std::string::npos && m.find('8') != std::string::npos);
    }
    CHECK(throws_invalid([] { FftPlan p(12); }));
    std::mt19937_64 rng(4);
    FftPlan plan(64);
    for (int r = 0; r < 3; ++r) {
        ComplexBuffer x = random_buf(64, rng);
        const ComplexBuffer want = dft_naive(x);
        plan.forward(x);
        CHECK(rel_error(x, want) < 1e-10);
    }
    ComplexBuffer bad(4);
    CHECK(throws_invalid([&] { plan.forward(bad); }));
    const ComplexBuffer x512 = random_buf(512, rng);
    CHECK(rel_error(ifft(fft(x512)), x512) < 1e-12);
    // czt: band params, full circle, plan reuse, alloc-free path, dft_any
    const CztParams bp = czt_params_for_band(100.0, 1000.0, 8000.0, 64);
    CHECK(std::abs(bp.a - std::polar(1.0, 2 * M_PI * 100 / 8000)) < 1e-15);
    const ComplexBuffer x48 = random_buf(48, rng);
    CztPlan cp(48, bp);
    CHECK(cp.input_size() == 48 && cp.output_size() == 64 && cp.conv_size() == next_pow2(48 + 64 - 1));
    ComplexBuffer scratch(cp.conv_size()), out(cp.output_size());
    cp.execute(x48, scratch, out);
    CHECK(rel_error(out, czt_direct(x48, bp)) < 1e-9);
    CHECK(rel_error(cp.execute(x48), out) < 1e-12);
    CHECK(throws_invalid([&] { cp.execute(ComplexBuffer(12)); }));
    const ComplexBuffer x100 = random_buf(100, rng);
    CHECK(rel_error(dft_any(x100), dft_naive(x100)) < 1e-9);
    CztParams spiral;
    spiral.a = std::polar(1.05, 0.3);
    spiral.w = std::polar(0.995, -0.11);
    spiral.m = 24;
    const ComplexBuffer x20 = random_buf(20, rng);
    CHECK(rel_error(czt(x20, spiral), czt_direct(x20, spiral)) < 1e-9);
    // spectra: default pad, exact non-pow2 length, slice_band
    Trace imp;
    imp.sample_rate_hz = 10e12;
    imp.samples.assign(500, 0.0);
    imp.samples[0] = 1.0;
    const Spectrum s512 = fft_spectrum(imp);
    CHECK(s512.size() == 512 && s512.source_n == 512 && std::abs(s512.f_step_hz - 10e12 / 512) < 1e-3);
    const Spectrum s500 = fft_spectrum(imp, 500);
    CHECK(s500.size() == 500);
    for (const auto& v : s500.bins) CHECK(std::abs(std::abs(v) - 1.0) < 1e-9);
    CHECK(throws_invalid([&] { fft_spectrum(imp, 499); }));
    // slice_band keeps inclusive edges (test_spectra.cpp:61-80). Note the reference's edge slack is
    // 0.5 * f_step * 1e-9 in BIN units (spectra.cpp:44), i.e. many bins for THz steps; we keep it.
    Spectrum lin11;
    lin11.f_step_hz = 10.0;
    lin11.source_n = 64;
    for (int k = 0; k < 11; ++k) lin11.bins.push_back(cplx(k, 0));
    const Spectrum cut = slice_band(lin11, 20.0, 50.0);
    CHECK(cut.size() == 4 && cut.f_start_hz == 20.0 && cut.bins[3].real() == 5.0 && cut.source_n == 64);
    CHECK(throws_invalid([&] { slice_band(lin11, 500.0, 600.0); }));
    const Spectrum cs = czt_spectrum(imp, 0.0, 2.5e12, 125);
    CHECK(cs.size() == 125 && std::abs(cs.f_step_hz - 2e10) < 1e-3);
    // zoom: default plan sizing, helpers, degenerate zoom, edited public fields
    const ZoomFftPlan zp = make_zoom_plan(500, 0.5e12, 2.0e12, 10e12);
    CHECK(zp.decimation == 3 && zp.filter_taps.size() == 101 && zp.usable_len == 498 && zp.n_fft == 256);
    CHECK(throws_invalid([] { design_lowpass(1000.0, 8000.0, 30); }));
    const ComplexBuffer xs{{1, 0}, {2, 0}, {3, 0}, {4, 0}, {5, 0}, {6, 0}};
    const std::vector<double> taps{1.0, 1.0, 1.0};
    const ComplexBuffer lin = filter_decimate(xs, taps, 2), circ = filter_decimate_circular(xs, taps, 2);
    CHECK(std::abs(lin[1].real() - 6) < 1e-12 && std::abs(lin[2].real() - 12) < 1e-12);
    CHECK(std::abs(circ[0].real() - 12) < 1e-12 && std::abs(circ[1].real() - 6) < 1e-12);
    std::vector<double> ones(8, 1.0);
    const ComplexBuffer sh = frequency_shift(ones, 1000.0, 8000.0);
    CHECK(std::abs(sh[3] - std::polar(1.0, -2 * M_PI * 3 / 8)) < 1e-12);
    Trace pulse;
    pulse.sample_rate_hz = 10e12;
    for (int i = 0; i < 500; ++i) {
        const double u = (i / 10e12 - 10e-12) / 300e-15;
        pulse.samples.push_back(-std::exp(0.5) * u * std::exp(-0.5 * u * u));
    }
    const Spectrum z = zoom_fft(zp, pulse);
    CHECK(z.size() == 115);
    ZoomOptions d1;
    d1.decimation = 1;
    Trace rnd;
    rnd.sample_rate_hz = 256.0;
    std::uniform_real_distribution<double> u(-1, 1);
    for (int i = 0; i < 256; ++i) rnd.samples.push_back(u(rng));
    const Spectrum zd = zoom_fft(make_zoom_plan(256, 32.0, 96.0, 256.0, d1), rnd);
    const Spectrum fd = slice_band(fft_spectrum(rnd, 256), 32.0, 96.0);
    CHECK(zd.size() == fd.size() && rel_error(zd.bins, fd.bins) < 1e-10);
    ZoomFftPlan edited = make_zoom_plan(500, 0.5e12, 2.0e12, 10e12);
    edited.n_fft = 512;   // public field edit (zoomfft.hpp:50), like the oracle's 2048-point variant
    const Spectrum ze = zoom_fft(edited, pulse);
    CHECK(ze.source_n == 512 && std::abs(ze.f_step_hz - 10e12 / (3.0 * 512)) < 1e-3);
    Trace wrong = pulse;
    wrong.samples.resize(400);
    CHECK(throws_invalid([&] { zoom_fft(zp, wrong); }));
    // CSV formats (signals.cpp:125-189, spectra.cpp:63-150): stream round trips and the error classes
    std::stringstream ts;
    write_trace_csv(pulse, ts);
    const Trace back = read_trace_csv(ts, "mem");
    CHECK(back.samples == pulse.samples && back.size() == 500 && std::abs(back.sample_rate_hz - 10e12) < 1e-9 * 10e12);
    std::stringstream bad_trace("t,x\n0,1\n1;2\n");
    try {
        read_trace_csv(bad_trace, "mem");
        CHECK(false);
    } catch (const ParseError& e) {
        CHECK(e.line == 3 && std::string(e.what()) == "mem: malformed row at line 3");
    }
    std::stringstream one("0,1\n");
    bool fmt = false;
    try {
        read_trace_csv(one, "mem");
    } catch (const FormatError&) {
        fmt = true;
    }
    CHECK(fmt);
    std::stringstream ss;
    write_spectrum_csv(s512, ss);
    const Spectrum sback = read_spectrum_csv(ss, "mem");
    CHECK(sback.size() == 512 && sback.bins == s512.bins && sback.f_start_hz == 0.0);
    CHECK(std::abs(sback.f_step_hz - s512.f_step_hz) < 1e-6 * s512.f_step_hz);
    std::stringstream js;
    write_spectrum_json(s512, js);
    const std::string jtxt = js.str();
    CHECK(jtxt.rfind("{\n  \"f_start_hz\": 0.0,\n", 0) == 0 && jtxt.find("\"source_n\": 512\n}\n") != std::string::npos);
    bool io = false;
    try {
        read_trace_csv_file("/nonexistent/dir/trace.csv");
    } catch (const IoError& e) {
        io = std::string(e.what()) == "cannot open trace file: /nonexistent/dir/trace.csv";
    }
    CHECK(io);
    // sizing helpers and the resolvability sweep (resolution.cpp, analysis.cpp:99-195): the reference's
    // default sweep resolves both routes first at 45 Hz (tests/golden/scan.npz)
    CHECK(record_len_for_step(10e12, 20e9) == 500 && zeros_for_resolution(8000.0, 128, 62.5) == 0);
    const ResolvabilityCurve rc = resolvability_scan(ScanConfig{});
    CHECK(rc.separations_hz.size() == 39 && rc.fft_len == 1138);
    CHECK(rc.min_resolved_fft_hz == 45.0 && rc.min_resolved_czt_hz == 45.0);
    std::stringstream cs2;
    write_resolvability_csv(rc, cs2);
    std::string first;
    std::getline(cs2, first);
    CHECK(first == "separation_hz,method,resolved,dip_db,f_peak_a_hz,peak_a_db,f_peak_b_hz,peak_b_db,f_valley_hz,valley_db");
    bool ins = false;
    try {
        dip_metric(s512, 1e9, 2e9);
    } catch (const InsufficientResolutionError&) {
        ins = true;
    }
    CHECK(ins);
    std::printf("%s: %d failures\n", failures ? "FAILED" : "ok", failures);
    return failures ? 1 : 0;
}
