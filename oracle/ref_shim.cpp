// ref_shim.cpp — TEST INFRASTRUCTURE. A thin C shim over the UNMODIFIED reference C++ core
// (compiled from /root/reference/proj/src by oracle/Makefile into oracle/_ref/libskref.so).
// It exposes the reference's plan-reuse entry points — the ones its own bench harness
// times (bench.cpp:167-226) — to Python via ctypes, plus a std::thread pool over one shared
// immutable plan (legal per numerics.hpp:24-26, czt.hpp:30-33). The reference's own sk_*
// C ABI (capi.cpp) is linked into the same .so and is used directly for the one-shot paths.
#include <chrono>
#include <cmath>
#include <string>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#include "bench.hpp"
#include "czt.hpp"
#include "numerics.hpp"
#include "spectra.hpp"
#include "types.hpp"
#include "zoomfft.hpp"

using namespace spectral;

namespace {
double run_pool(std::size_t count, int threads, const std::function<void(std::size_t, std::size_t)>& fn) {
    if (threads < 1) threads = 1;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) {
        const std::size_t b = count * i / threads, e = count * (i + 1) / threads;
        pool.emplace_back([&, b, e] { fn(b, e); });
    }
    for (auto& t : pool) t.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

extern "C" {

void* skr_czt_plan_create(std::size_t n, double a_re, double a_im, double w_re, double w_im,
                          std::size_t m) {
    try {
        CztParams p;
        p.a = cplx(a_re, a_im);
        p.w = cplx(w_re, w_im);
        p.m = m;
        return new CztPlan(n, p);
    } catch (...) {
        return nullptr;
    }
}
void skr_czt_plan_free(void* p) { delete static_cast<CztPlan*>(p); }

// CztPlan::execute(x, scratch, out) on `count` real traces (bench.cpp:194-204 alloc-free path)
double skr_czt_batch(void* plan, const double* x_real, std::size_t n, std::size_t count, int threads,
                     double* out) {
    const CztPlan& p = *static_cast<CztPlan*>(plan);
    return run_pool(count, threads, [&](std::size_t b, std::size_t e) {
        ComplexBuffer x(n), scratch(p.conv_size()), o(p.output_size());
        for (std::size_t t = b; t < e; ++t) {
            for (std::size_t i = 0; i < n; ++i) x[i] = cplx(x_real[t * n + i], 0.0);
            p.execute(x, scratch, o);
            if (out) std::memcpy(out + 2 * t * p.output_size(), o.data(), o.size() * sizeof(cplx));
        }
    });
}

// FftPlan(L).forward on a zero-padded copy of each real trace (bench.cpp:176-186)
double skr_fft_batch(std::size_t L, const double* x_real, std::size_t n, std::size_t count, int threads,
                     double* out) {
    FftPlan plan(L);
    return run_pool(count, threads, [&](std::size_t b, std::size_t e) {
        ComplexBuffer buf(L);
        for (std::size_t t = b; t < e; ++t) {
            std::fill(buf.begin(), buf.end(), cplx(0.0, 0.0));
            for (std::size_t i = 0; i < n; ++i) buf[i] = cplx(x_real[t * n + i], 0.0);
            plan.forward(buf);
            if (out) std::memcpy(out + 2 * t * L, buf.data(), L * sizeof(cplx));
        }
    });
}

void* skr_zoom_plan_create(std::size_t n, double f1, double f2, double fs, double center_hz,
                           int center_set, std::size_t decimation, double cutoff_hz,
                           std::size_t num_taps, int circular, int trim, int pad_pow2) {
    try {
        ZoomOptions o;
        o.center_hz = center_hz;
        o.center_set = center_set != 0;
        o.decimation = decimation;
        o.cutoff_hz = cutoff_hz;
        o.num_taps = num_taps;
        o.circular = circular != 0;
        o.trim_transient = trim != 0;
        o.pad_pow2 = pad_pow2 != 0;
        return new ZoomFftPlan(make_zoom_plan(n, f1, f2, fs, o));
    } catch (...) {
        return nullptr;
    }
}
void skr_zoom_plan_free(void* p) { delete static_cast<ZoomFftPlan*>(p); }

// public plan fields (zoomfft.hpp:33-56): override n_fft (cfg3 "2048-point" variant) and taps
// (cfg3 "64-tap" variant), as SURVEY §9 D1/D2 prescribe for the oracle.
int skr_zoom_plan_set_n_fft(void* plan, std::size_t n_fft) {
    auto& p = *static_cast<ZoomFftPlan*>(plan);
    if (n_fft < p.decimated_len) return 1;
    p.n_fft = n_fft;
    if (is_pow2(n_fft)) p.fft.emplace(n_fft); else p.fft.reset();
    return 0;
}
int skr_zoom_plan_set_taps(void* plan, const double* taps, std::size_t count) {
    auto& p = *static_cast<ZoomFftPlan*>(plan);
    p.filter_taps.assign(taps, taps + count);
    p.group_delay_samples = 0.5 * static_cast<double>(count - 1);
    return 0;
}
void skr_zoom_plan_taps(void* plan, double* out) {
    auto& p = *static_cast<ZoomFftPlan*>(plan);
    std::memcpy(out, p.filter_taps.data(), p.filter_taps.size() * sizeof(double));
}

// zoom_fft(plan, trace) per trace; returns seconds, bins per trace through *nbins
double skr_zoom_batch(void* plan, const double* x_real, std::size_t n, double fs, std::size_t count,
                      int threads, double* out, std::size_t* nbins, double* f_start, double* f_step) {
    const ZoomFftPlan& p = *static_cast<ZoomFftPlan*>(plan);
    {
        Trace t;
        t.samples.assign(x_real, x_real + n);
        t.sample_rate_hz = fs;
        const Spectrum s = zoom_fft(p, t);
        if (nbins) *nbins = s.size();
        if (f_start) *f_start = s.f_start_hz;
        if (f_step) *f_step = s.f_step_hz;
    }
    return run_pool(count, threads, [&](std::size_t b, std::size_t e) {
        Trace t;
        t.sample_rate_hz = fs;
        for (std::size_t i = b; i < e; ++i) {
            t.samples.assign(x_real + i * n, x_real + (i + 1) * n);
            const Spectrum s = zoom_fft(p, t);
            if (out) std::memcpy(out + 2 * i * s.size(), s.bins.data(), s.size() * sizeof(cplx));
        }
    });
}

// bench_environment() (bench.cpp:100-129): the CPU model / kernel / compiler line the reference's
// own bench reports print beside their numbers
const char* skr_bench_environment() {
    static const std::string env = bench_environment();
    return env.c_str();
}

// H(f) of `count` real traces against one reference trace on the reference's FFT: FftPlan(L).forward
// of each zero-padded trace (bench.cpp:176-186) and of the reference once, then the restated
// per-bin division H = X_s / X_ref, |H| = hypot, arg H = atan2 on the L/2 + 1 bins (
// the reference has no H). mag / phase may be NULL (timing only).
double skr_transfer_batch(std::size_t L, const double* ref, const double* x_real, std::size_t n, std::size_t count,
                          int threads, double* mag, double* phase) {
    FftPlan plan(L);
    const std::size_t nb = L / 2 + 1;
    ComplexBuffer xr(L, cplx(0.0, 0.0));
    for (std::size_t i = 0; i < n; ++i) xr[i] = cplx(ref[i], 0.0);
    plan.forward(xr);
    return run_pool(count, threads, [&](std::size_t b, std::size_t e) {
        ComplexBuffer buf(L);
        std::vector<double> m(nb), p(nb);
        for (std::size_t t = b; t < e; ++t) {
            std::fill(buf.begin(), buf.end(), cplx(0.0, 0.0));
            for (std::size_t i = 0; i < n; ++i) buf[i] = cplx(x_real[t * n + i], 0.0);
            plan.forward(buf);
            for (std::size_t k = 0; k < nb; ++k) {
                const cplx h = buf[k] / xr[k];
                m[k] = std::hypot(h.real(), h.imag());
                p[k] = std::atan2(h.imag(), h.real());
            }
            if (mag) std::memcpy(mag + t * nb, m.data(), nb * sizeof(double));
            if (phase) std::memcpy(phase + t * nb, p.data(), nb * sizeof(double));
        }
    });
}

}  // extern "C"
