// capi.cpp — the drop-in sk_* C ABI (include/spectralkit.h) and the batched skg_* extension
// (include/spectralkit_gpu.h). Error convention follows the reference's capi.cpp:44-83:
// exceptions are mapped to status codes, the message goes to a thread-local string.
#include <algorithm>
#include <cmath>
#include <limits>
#include <memory>
#include <mutex>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "analysis.hpp"
#include "host.hpp"
#include "staging.hpp"
#include "io.hpp"
#include "spectralkit.h"
#include "spectralkit_gpu.h"

namespace skg {
cudaError_t launch_dft_naive(const void* x, long long n, const void* tw, void* out, cudaStream_t st);
cudaError_t launch_czt_direct(const void* x, long long n, double a_logm, double a_q, double w_logm, double w_q,
                              long long m, void* xa_scratch, void* out, cudaStream_t st);
}  // namespace skg

using skg::cd;

struct sk_trace {
    std::vector<double> samples;
    double fs = 0.0, t0 = 0.0;
};
struct sk_spectrum {
    std::vector<cd> bins;
    double f_start = 0.0, f_step = 0.0;
    size_t source_n = 0;
};
struct sk_zoom_plan {
    std::unique_ptr<skg::ZoomPlanG> p;
};
struct sk_resolvability_curve {
    skg::CurveH c;
};
struct skg_czt_plan {
    std::unique_ptr<skg::CztPlanG> p;
    bool f32 = false;
};
struct skg_transfer_plan {
    std::unique_ptr<skg::TransferPlanG> p;
};
struct skg_zoom_plan {
    std::unique_ptr<skg::ZoomPlanG> p;
    bool f32 = false;
};

namespace {

thread_local std::string g_err;

template <typename Fn> sk_status guarded(Fn&& fn) {
    try {
        fn();
        return SK_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SK_ERR_INVALID_ARGUMENT;
    } catch (const skg::InsufficientResolution& e) {   // capi.cpp:56-67 of the reference
        g_err = e.what();
        return SK_ERR_INSUFFICIENT_RESOLUTION;
    } catch (const skg::ParseError& e) {
        g_err = e.what();
        return SK_ERR_PARSE;
    } catch (const skg::FormatError& e) {
        g_err = e.what();
        return SK_ERR_FORMAT;
    } catch (const skg::IoError& e) {
        g_err = e.what();
        return SK_ERR_IO;
    } catch (const std::bad_alloc&) {
        g_err = "out of memory";
        return SK_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SK_ERR_INTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return SK_ERR_INTERNAL;
    }
}

sk_status bad_arg(const char* msg) {
    g_err = msg;
    return SK_ERR_INVALID_ARGUMENT;
}

// Row-stride and precision checks of the batched entry points: with more than one row, a stride
// shorter than the row would make rows overlap (reads past the end of a caller's buffer, writes
// over the next row).
void need_stride(const char* fn, const char* what, size_t batch, size_t stride, size_t row) {
    if (batch > 1 && stride < row)
        throw std::invalid_argument(std::string(fn) + ": " + what + " stride " + std::to_string(stride) +
                                    " is shorter than the row (" + std::to_string(row) + ")");
}
void need_precision(const char* fn, int precision) {
    if (precision != SKG_F64 && precision != SKG_F32)
        throw std::invalid_argument(std::string(fn) + ": precision must be SKG_F64 or SKG_F32");
}

// types.cpp:20-27
void validate_trace(const sk_trace& t) {
    if (t.samples.empty()) throw std::invalid_argument("trace: no samples");
    if (!(t.fs > 0.0) || !std::isfinite(t.fs))
        throw std::invalid_argument("trace: sample rate must be positive and finite");
    for (double v : t.samples)
        if (!std::isfinite(v)) throw std::invalid_argument("trace: non-finite sample");
    if (!std::isfinite(t.t0)) throw std::invalid_argument("trace: non-finite start time");
}

std::vector<cd> join(const double* re, const double* im, size_t n) {
    std::vector<cd> x(n);
    for (size_t i = 0; i < n; ++i) x[i] = cd(re[i], im ? im[i] : 0.0);
    return x;
}

void split(const std::vector<cd>& x, double* re, double* im) {
    for (size_t i = 0; i < x.size(); ++i) {
        re[i] = x[i].real();
        im[i] = x[i].imag();
    }
}

// one-shot staging: host -> device -> host on the per-thread default stream, through the
// per-thread grow-only pinned / device slots of skg::CallStage (no cudaMalloc / cudaFree per call)
struct Stage {
    struct Ptr {
        void* p = nullptr;
    };
    skg::CallStage cs;
    cudaStream_t st = cs.stream();
    Ptr in, out;
    void put(const void* h, size_t bytes) { in.p = cs.up(h, bytes); }
    void alloc_out(size_t bytes) { out.p = cs.out(bytes); }
    void get(void* h, size_t bytes) { cs.down(h, out.p, bytes); }
};

void fft_inplace(double* re, double* im, size_t n, bool inverse) {   // numerics.cpp:102-120
    if (n == 0) throw std::invalid_argument("fft: empty input");
    if (!skg::is_pow2(n))
        throw std::invalid_argument("fft: length " + std::to_string(n) + " is not a power of two; zero_pad to " +
                                    std::to_string(skg::next_pow2(n)) + " first");
    std::vector<cd> x = join(re, im, n);
    Stage s;
    s.put(x.data(), n * sizeof(cd));
    skg::fft_c2c(n, inverse, false, s.in.p, 0, s.in.p, 0, 1, s.st);
    s.out = s.in;
    s.get(x.data(), n * sizeof(cd));
    split(x, re, im);
}

// The one-shot calls (sk_czt, sk_czt_spectrum) build a plan per call in the reference
// (czt.cpp:139-142, 155-175); here the last few plans are kept, keyed on the exact bits of
// (n, a, w, m), so a repeated call skips the O(L log L) table build and the uploads.
const skg::CztPlanG& czt_plan_cached(size_t n, cd a, cd w, size_t m) {
    struct Key {
        size_t n, m;
        double ar, ai, wr, wi;
        bool operator==(const Key& o) const { return std::memcmp(this, &o, sizeof(Key)) == 0; }
    };
    static std::mutex mu;
    static std::vector<std::pair<Key, std::shared_ptr<skg::CztPlanG>>> lru;   // front = most recent
    thread_local std::shared_ptr<skg::CztPlanG> hold;   // keeps the returned plan alive for this call
    Key k{};
    k.n = n, k.m = m, k.ar = a.real(), k.ai = a.imag(), k.wr = w.real(), k.wi = w.imag();
    {
        std::lock_guard<std::mutex> lk(mu);
        for (size_t i = 0; i < lru.size(); ++i)
            if (lru[i].first == k) {
                std::rotate(lru.begin(), lru.begin() + i, lru.begin() + i + 1);
                hold = lru.front().second;
                return *hold;
            }
    }
    auto plan = std::make_shared<skg::CztPlanG>(n, a, w, m);   // validates; may throw
    std::lock_guard<std::mutex> lk(mu);
    lru.insert(lru.begin(), {k, plan});
    if (lru.size() > 8) lru.pop_back();
    hold = plan;
    return *hold;
}

std::vector<cd> czt_gpu(const std::vector<cd>& x, cd a, cd w, size_t m) {   // czt.cpp:139-142
    if (x.empty()) throw std::invalid_argument("czt: empty input");
    const skg::CztPlanG& plan = czt_plan_cached(x.size(), a, w, m);
    Stage s;
    s.put(x.data(), x.size() * sizeof(cd));
    s.alloc_out(m * sizeof(cd));
    plan.execute(s.in.p, true, 0, 1, s.out.p, 0, false, s.st);
    std::vector<cd> y(m);
    s.get(y.data(), m * sizeof(cd));
    return y;
}

sk_spectrum* fft_spectrum_gpu(const sk_trace& t, size_t transform_len) {   // spectra.cpp:21-38
    validate_trace(t);
    const size_t n = t.samples.size();
    const size_t len = transform_len == 0 ? skg::next_pow2(n) : transform_len;
    if (len < n) throw std::invalid_argument("fft_spectrum: transform length shorter than the trace");
    Stage s;
    s.put(t.samples.data(), n * sizeof(double));
    s.alloc_out(len * sizeof(cd));
    skg::fft_spectrum_batch(n, len, false, 0, s.in.p, 0, 1, s.out.p, 0, s.st);
    auto* out = new sk_spectrum;
    out->bins.resize(len);
    s.get(out->bins.data(), len * sizeof(cd));
    out->f_start = 0.0;
    out->f_step = t.fs / static_cast<double>(len);
    out->source_n = len;
    return out;
}

}  // namespace

extern "C" {

const char* sk_status_name(sk_status status) {
    switch (status) {
        case SK_OK: return "ok";
        case SK_ERR_INVALID_ARGUMENT: return "invalid argument";
        case SK_ERR_IO: return "io error";
        case SK_ERR_PARSE: return "parse error";
        case SK_ERR_FORMAT: return "format error";
        case SK_ERR_INSUFFICIENT_RESOLUTION: return "insufficient resolution";
        case SK_ERR_INTERNAL: return "internal error";
    }
    return "unknown status";
}

const char* sk_last_error(void) { return g_err.c_str(); }
const char* sk_version(void) { return "0.1.0-b200"; }

sk_status sk_fft(double* re, double* im, size_t n) {
    if (!re || !im) return bad_arg("sk_fft: null buffer");
    return guarded([&] { fft_inplace(re, im, n, false); });
}

sk_status sk_ifft(double* re, double* im, size_t n) {
    if (!re || !im) return bad_arg("sk_ifft: null buffer");
    return guarded([&] { fft_inplace(re, im, n, true); });
}

sk_status sk_dft_naive(const double* re, const double* im, size_t n, double* out_re, double* out_im) {
    if (!re || !im || !out_re || !out_im) return bad_arg("sk_dft_naive: null buffer");
    return guarded([&] {
        if (n == 0) throw std::invalid_argument("dft_naive: empty input");
        std::vector<cd> x = join(re, im, n), tw(n);
        for (size_t r = 0; r < n; ++r) {   // numerics.cpp:38-42
            const double ang = -2.0 * M_PI * static_cast<double>(r) / static_cast<double>(n);
            tw[r] = cd(std::cos(ang), std::sin(ang));
        }
        Stage s;
        s.put(x.data(), n * sizeof(cd));
        void* dtw = s.cs.up(tw.data(), n * sizeof(cd));
        s.alloc_out(n * sizeof(cd));
        skg::check(skg::launch_dft_naive(s.in.p, (long long)n, dtw, s.out.p, s.st), "dft_naive");
        skg::count_launch();
        s.get(x.data(), n * sizeof(cd));
        split(x, out_re, out_im);
    });
}

sk_status sk_czt(const double* re, const double* im, size_t n, double a_re, double a_im, double w_re, double w_im,
                 size_t m, double* out_re, double* out_im) {
    if (!re || !im || !out_re || !out_im) return bad_arg("sk_czt: null buffer");
    return guarded([&] { split(czt_gpu(join(re, im, n), cd(a_re, a_im), cd(w_re, w_im), m), out_re, out_im); });
}

sk_status sk_czt_direct(const double* re, const double* im, size_t n, double a_re, double a_im, double w_re,
                        double w_im, size_t m, double* out_re, double* out_im) {
    if (!re || !im || !out_re || !out_im) return bad_arg("sk_czt_direct: null buffer");
    return guarded([&] {
        if (m == 0) throw std::invalid_argument("czt: m must be >= 1");
        const cd a(a_re, a_im), w(w_re, w_im);
        if (!(std::abs(a) > 0.0) || !(std::abs(w) > 0.0)) throw std::invalid_argument("czt: a and w must be nonzero");
        if (n == 0) throw std::invalid_argument("czt_direct: empty input");
        const skg::PolarPow A(a), W(w);
        std::vector<cd> x = join(re, im, n);
        Stage s;
        s.put(x.data(), n * sizeof(cd));
        void* xa = s.cs.scratch(n * sizeof(cd));
        s.alloc_out(m * sizeof(cd));
        skg::check(skg::launch_czt_direct(s.in.p, (long long)n, A.log_mag, A.q, W.log_mag, W.q, (long long)m, xa,
                                          s.out.p, s.st),
                   "czt_direct");
        skg::count_launch(2);
        std::vector<cd> y(m);
        s.get(y.data(), m * sizeof(cd));
        split(y, out_re, out_im);
    });
}

sk_status sk_czt_params_for_band(double f1, double f2, double fs, size_t m, double* a_re, double* a_im,
                                 double* w_re, double* w_im) {
    if (!a_re || !a_im || !w_re || !w_im) return bad_arg("sk_czt_params_for_band: null output");
    return guarded([&] {   // czt.cpp:42-56
        if (!(fs > 0.0)) throw std::invalid_argument("czt_params_for_band: sample rate must be positive");
        if (!(f1 >= 0.0) || !(f1 < f2)) throw std::invalid_argument("czt_params_for_band: need 0 <= f1 < f2");
        if (f2 > fs * (1.0 + 1e-12)) throw std::invalid_argument("czt_params_for_band: f2 exceeds the sample rate");
        if (m < 2) throw std::invalid_argument("czt_params_for_band: m must be >= 2");
        const cd a = skg::cis_cycles(f1 / fs, 1.0);
        const cd w = skg::cis_cycles(-(f2 - f1) / (static_cast<double>(m) * fs), 1.0);
        *a_re = a.real();
        *a_im = a.imag();
        *w_re = w.real();
        *w_im = w.imag();
    });
}

size_t sk_next_pow2(size_t n) {
    try {
        return skg::next_pow2(n == 0 ? 1 : n);
    } catch (...) {
        return 0;
    }
}

// ---- traces ------------------------------------------------------------------------------------
sk_status sk_trace_create(const double* samples, size_t n, double fs, double t0, sk_trace** out) {
    if (!samples || !out) return bad_arg("sk_trace_create: null argument");
    return guarded([&] {
        auto* t = new sk_trace;
        t->samples.assign(samples, samples + n);
        t->fs = fs;
        t->t0 = t0;
        try {
            validate_trace(*t);
        } catch (...) {
            delete t;
            throw;
        }
        *out = t;
    });
}
void sk_trace_free(sk_trace* t) { delete t; }
size_t sk_trace_size(const sk_trace* t) { return t ? t->samples.size() : 0; }
double sk_trace_sample_rate(const sk_trace* t) { return t ? t->fs : 0.0; }
double sk_trace_t0(const sk_trace* t) { return t ? t->t0 : 0.0; }
const double* sk_trace_samples(const sk_trace* t) { return t ? t->samples.data() : nullptr; }

// trace / spectrum CSV files (signals.cpp:125-189, spectra.cpp:63-78; capi.cpp:391-408, 483-501)
sk_status sk_trace_read_csv(const char* path, sk_trace** out) {
    if (!path || !out) return bad_arg("sk_trace_read_csv: null argument");
    return guarded([&] {
        skg::HostTrace h = skg::read_trace_csv_file(path);
        auto* t = new sk_trace;
        t->samples = std::move(h.samples);
        t->fs = h.fs;
        t->t0 = h.t0;
        *out = t;
    });
}

sk_status sk_trace_write_csv(const sk_trace* t, const char* path) {
    if (!t || !path) return bad_arg("sk_trace_write_csv: null argument");
    return guarded([&] { skg::write_trace_csv_file(t->samples.data(), t->samples.size(), t->fs, t->t0, path); });
}

sk_status sk_spectrum_write_json(const sk_spectrum* s, const char* path) {
    if (!s || !path) return bad_arg("sk_spectrum_write_json: null argument");
    return guarded([&] {
        skg::write_spectrum_json_file(reinterpret_cast<const double*>(s->bins.data()), s->bins.size(), s->f_start,
                                      s->f_step, s->source_n, path);
    });
}

sk_status sk_spectrum_read_csv(const char* path, sk_spectrum** out) {
    if (!path || !out) return bad_arg("sk_spectrum_read_csv: null argument");
    return guarded([&] {
        skg::HostSpectrum h = skg::read_spectrum_csv_file(path);
        auto* s = new sk_spectrum;
        s->bins.resize(h.bins.size() / 2);
        for (size_t k = 0; k < s->bins.size(); ++k) s->bins[k] = cd(h.bins[2 * k], h.bins[2 * k + 1]);
        s->f_start = h.f_start;
        s->f_step = h.f_step;
        s->source_n = h.source_n;
        *out = s;
    });
}

sk_status sk_spectrum_write_csv(const sk_spectrum* s, const char* path) {
    if (!s || !path) return bad_arg("sk_spectrum_write_csv: null argument");
    return guarded([&] {
        skg::write_spectrum_csv_file(reinterpret_cast<const double*>(s->bins.data()), s->bins.size(), s->f_start,
                                     s->f_step, path);
    });
}

namespace {
// grow-only pinned staging for the batched file paths (one batch in flight per process)
std::mutex g_io_mu;
void* g_io_pin = nullptr;
size_t g_io_cap = 0;
void* io_pinned(size_t bytes) {
    if (bytes > g_io_cap) {
        if (g_io_pin) cudaFreeHost(g_io_pin);
        g_io_pin = nullptr;
        g_io_cap = 0;
        skg::check(cudaHostAlloc(&g_io_pin, bytes, cudaHostAllocDefault), "cudaHostAlloc");
        g_io_cap = bytes;
    }
    return g_io_pin;
}
}  // namespace

sk_status skg_traces_read_csv(const char* const* paths, size_t count, size_t n, int precision, void* d_out,
                              size_t out_stride, double* fs_out, double* t0_out, int threads, void* stream) {
    if (!paths || !d_out) return bad_arg("skg_traces_read_csv: null argument");
    if (n == 0) return bad_arg("skg_traces_read_csv: n must be the per-trace sample count");
    if (out_stride < n) return bad_arg("skg_traces_read_csv: row stride shorter than the trace");
    for (size_t i = 0; i < count; ++i)
        if (!paths[i]) return bad_arg("skg_traces_read_csv: null path");
    return guarded([&] {
        if (count == 0) return;
        skg::require_device();
        std::lock_guard<std::mutex> lk(g_io_mu);
        const bool f32 = precision == SKG_F32;
        const size_t es = f32 ? sizeof(float) : sizeof(double);
        unsigned char* pin = static_cast<unsigned char*>(io_pinned(count * n * es));
        skg::parallel_for(count, threads, [&](size_t i) {
            skg::HostTrace h = skg::read_trace_csv_file(paths[i]);
            if (h.samples.size() != n)
                throw skg::FormatError(std::string(paths[i]) + ": expected " + std::to_string(n) + " samples, got " +
                                       std::to_string(h.samples.size()));
            if (f32) {
                float* dst = reinterpret_cast<float*>(pin) + i * n;
                for (size_t k = 0; k < n; ++k) dst[k] = (float)h.samples[k];
            } else {
                std::memcpy(reinterpret_cast<double*>(pin) + i * n, h.samples.data(), n * sizeof(double));
            }
            if (fs_out) fs_out[i] = h.fs;
            if (t0_out) t0_out[i] = h.t0;
        });
        const cudaStream_t st = (cudaStream_t)stream;
        skg::check(cudaMemcpy2DAsync(d_out, out_stride * es, pin, n * es, n * es, count, cudaMemcpyHostToDevice, st),
                   "H2D");
        skg::check(cudaStreamSynchronize(st), "sync");
    });
}

sk_status skg_spectra_write_csv(const char* const* paths, size_t count, int precision, const void* d_bins,
                                size_t bins_stride, size_t nbins, const double* f_start_hz, double f_step_hz,
                                int threads, void* stream) {
    if (!paths || !d_bins) return bad_arg("skg_spectra_write_csv: null argument");
    if (bins_stride < nbins) return bad_arg("skg_spectra_write_csv: row stride shorter than the spectrum");
    for (size_t i = 0; i < count; ++i)
        if (!paths[i]) return bad_arg("skg_spectra_write_csv: null path");
    return guarded([&] {
        if (count == 0 || nbins == 0) return;
        skg::require_device();
        std::lock_guard<std::mutex> lk(g_io_mu);
        const bool f32 = precision == SKG_F32;
        const size_t cs = f32 ? 2 * sizeof(float) : 2 * sizeof(double);
        unsigned char* pin = static_cast<unsigned char*>(io_pinned(count * nbins * cs));
        const cudaStream_t st = (cudaStream_t)stream;
        skg::check(cudaMemcpy2DAsync(pin, nbins * cs, d_bins, bins_stride * cs, nbins * cs, count,
                                     cudaMemcpyDeviceToHost, st),
                   "D2H");
        skg::check(cudaStreamSynchronize(st), "sync");
        skg::parallel_for(count, threads, [&](size_t i) {
            const double f0 = f_start_hz ? f_start_hz[i] : 0.0;
            if (f32) {   // the reference's writer prints doubles: promote
                std::vector<double> b(2 * nbins);
                const float* src = reinterpret_cast<const float*>(pin) + 2 * i * nbins;
                for (size_t k = 0; k < 2 * nbins; ++k) b[k] = src[k];
                skg::write_spectrum_csv_file(b.data(), nbins, f0, f_step_hz, paths[i]);
            } else {
                skg::write_spectrum_csv_file(reinterpret_cast<const double*>(pin) + 2 * i * nbins, nbins, f0,
                                             f_step_hz, paths[i]);
            }
        });
    });
}

// ---- two-tone analysis (analysis.cpp:30-195; capi.cpp:568-629 of the reference) ----------------
namespace {
void copy_metric(const skg::DipMetricH& m, sk_dip_metric* o) {
    o->resolved = m.resolved ? 1 : 0;
    o->dip_db = m.dip_db;
    o->f_peak_a_hz = m.f_peak_a_hz;
    o->peak_a_db = m.peak_a_db;
    o->f_peak_b_hz = m.f_peak_b_hz;
    o->peak_b_db = m.peak_b_db;
    o->f_valley_hz = m.f_valley_hz;
    o->valley_db = m.valley_db;
}
}  // namespace

sk_status sk_dip_metric_compute(const sk_spectrum* s, double f_a, double f_b, sk_dip_metric* out) {
    if (!s || !out) return bad_arg("sk_dip_metric_compute: null argument");
    return guarded([&] {
        copy_metric(skg::dip_metric(s->bins.data(), s->bins.size(), s->f_start, s->f_step, f_a, f_b), out);
    });
}

void sk_scan_config_defaults(sk_scan_config* cfg) {
    if (!cfg) return;
    const skg::ScanConfigH d;
    cfg->sample_rate_hz = d.sample_rate_hz;
    cfg->n = d.n;
    cfg->f1_hz = d.f1_hz;
    cfg->f2_hz = d.f2_hz;
    cfg->m = d.m;
    cfg->center_hz = d.center_hz;
    cfg->sep_start_hz = d.sep_start_hz;
    cfg->sep_stop_hz = d.sep_stop_hz;
    cfg->sep_step_hz = d.sep_step_hz;
}

sk_status sk_resolvability_scan(const sk_scan_config* cfg, sk_resolvability_curve** out) {
    if (!cfg || !out) return bad_arg("sk_resolvability_scan: null argument");
    return guarded([&] {
        skg::ScanConfigH c;
        c.sample_rate_hz = cfg->sample_rate_hz;
        c.n = cfg->n;
        c.f1_hz = cfg->f1_hz;
        c.f2_hz = cfg->f2_hz;
        c.m = cfg->m;
        c.center_hz = cfg->center_hz;
        c.sep_start_hz = cfg->sep_start_hz;
        c.sep_stop_hz = cfg->sep_stop_hz;
        c.sep_step_hz = cfg->sep_step_hz;
        *out = new sk_resolvability_curve{skg::resolvability_scan(c)};
    });
}
void sk_resolvability_curve_free(sk_resolvability_curve* c) { delete c; }
size_t sk_resolvability_curve_size(const sk_resolvability_curve* c) { return c ? c->c.separations_hz.size() : 0; }
sk_status sk_resolvability_curve_point(const sk_resolvability_curve* c, size_t i, double* sep, sk_dip_metric* fm,
                                       sk_dip_metric* cm) {
    if (!c) return bad_arg("sk_resolvability_curve_point: null curve");
    if (i >= c->c.separations_hz.size()) return bad_arg("sk_resolvability_curve_point: index out of range");
    if (sep) *sep = c->c.separations_hz[i];
    if (fm) copy_metric(c->c.fft_metrics[i], fm);
    if (cm) copy_metric(c->c.czt_metrics[i], cm);
    return SK_OK;
}
double sk_resolvability_min_fft(const sk_resolvability_curve* c) {
    return c ? c->c.min_resolved_fft_hz : std::numeric_limits<double>::quiet_NaN();
}
double sk_resolvability_min_czt(const sk_resolvability_curve* c) {
    return c ? c->c.min_resolved_czt_hz : std::numeric_limits<double>::quiet_NaN();
}
size_t skg_resolvability_fft_len(const sk_resolvability_curve* c) { return c ? c->c.fft_len : 0; }
sk_status sk_resolvability_write_csv(const sk_resolvability_curve* c, const char* path) {
    if (!c || !path) return bad_arg("sk_resolvability_write_csv: null argument");
    return guarded([&] {
        skg::write_text_file(skg::format_resolvability_csv(c->c), path, "cannot open for writing: ", "resolvability csv");
    });
}

sk_status sk_resolvability_write_json(const sk_resolvability_curve* c, const char* path) {
    if (!c || !path) return bad_arg("sk_resolvability_write_json: null argument");
    return guarded([&] {
        skg::write_text_file(skg::format_resolvability_json(c->c), path, "cannot open for writing: ",
                             "resolvability json");
    });
}

// sizing helpers (resolution.cpp:18-63; capi.cpp:237-265 of the reference)
sk_status sk_fft_resolution(double fs, size_t n, double* out) {
    if (!out) return bad_arg("sk_fft_resolution: null output");
    return guarded([&] { *out = skg::fft_resolution(fs, n); });
}
sk_status sk_record_len_for_step(double fs, double step, size_t* out) {
    if (!out) return bad_arg("sk_record_len_for_step: null output");
    return guarded([&] { *out = skg::record_len_for_step(fs, step); });
}
sk_status sk_zeros_for_resolution(double fs, size_t n, double step, size_t* out) {
    if (!out) return bad_arg("sk_zeros_for_resolution: null output");
    return guarded([&] { *out = skg::zeros_for_resolution(fs, n, step); });
}
sk_status sk_czt_len_for_matched_resolution(double f1, double f2, double fs, size_t n_fft, size_t* out) {
    if (!out) return bad_arg("sk_czt_len_for_matched_resolution: null output");
    return guarded([&] { *out = skg::czt_len_for_matched_resolution(f1, f2, fs, n_fft); });
}

// ---- spectra -----------------------------------------------------------------------------------
sk_status sk_fft_spectrum(const sk_trace* t, size_t transform_len, sk_spectrum** out) {
    if (!t || !out) return bad_arg("sk_fft_spectrum: null argument");
    return guarded([&] { *out = fft_spectrum_gpu(*t, transform_len); });
}

sk_status sk_czt_spectrum(const sk_trace* t, double f1, double f2, size_t m, sk_spectrum** out) {
    if (!t || !out) return bad_arg("sk_czt_spectrum: null argument");
    return guarded([&] {   // czt.cpp:155-175
        validate_trace(*t);
        const double nyquist = t->fs / 2.0;
        if (!(f1 >= 0.0) || !(f1 < f2)) throw std::invalid_argument("czt_spectrum: need 0 <= f1 < f2");
        if (f2 > nyquist * (1.0 + 1e-12))
            throw std::invalid_argument("czt_spectrum: band edge " + std::to_string(f2) +
                                        " Hz exceeds the Nyquist rate " + std::to_string(nyquist) + " Hz");
        double ar, ai, wr, wi;
        if (sk_czt_params_for_band(f1, f2, t->fs, m, &ar, &ai, &wr, &wi) != SK_OK)
            throw std::invalid_argument(g_err);
        const size_t n = t->samples.size();
        const skg::CztPlanG& plan = czt_plan_cached(n, cd(ar, ai), cd(wr, wi), m);
        Stage s;
        s.put(t->samples.data(), n * sizeof(double));
        s.alloc_out(m * sizeof(cd));
        plan.execute(s.in.p, false, 0, 1, s.out.p, 0, false, s.st);
        auto* sp = new sk_spectrum;
        sp->bins.resize(m);
        s.get(sp->bins.data(), m * sizeof(cd));
        sp->f_start = f1;
        sp->f_step = (f2 - f1) / static_cast<double>(m);
        sp->source_n = n;
        *out = sp;
    });
}

sk_status sk_spectrum_create(const double* re, const double* im, size_t n, double f_start, double f_step,
                             sk_spectrum** out) {
    if (!re || !out) return bad_arg("sk_spectrum_create: null argument");
    return guarded([&] {
        if (n == 0) throw std::invalid_argument("sk_spectrum_create: empty spectrum");
        if (!(f_step >= 0.0)) throw std::invalid_argument("sk_spectrum_create: negative step");
        auto* s = new sk_spectrum;
        s->bins = join(re, im, n);
        s->f_start = f_start;
        s->f_step = f_step;
        s->source_n = n;
        *out = s;
    });
}
void sk_spectrum_free(sk_spectrum* s) { delete s; }
size_t sk_spectrum_size(const sk_spectrum* s) { return s ? s->bins.size() : 0; }
double sk_spectrum_f_start(const sk_spectrum* s) { return s ? s->f_start : 0.0; }
double sk_spectrum_f_step(const sk_spectrum* s) { return s ? s->f_step : 0.0; }
double sk_spectrum_frequency(const sk_spectrum* s, size_t k) {
    return s ? s->f_start + static_cast<double>(k) * s->f_step : 0.0;
}
size_t sk_spectrum_source_n(const sk_spectrum* s) { return s ? s->source_n : 0; }

sk_status sk_spectrum_bin(const sk_spectrum* s, size_t k, double* re, double* im) {
    if (!s || !re || !im) return bad_arg("sk_spectrum_bin: null argument");
    if (k >= s->bins.size()) return bad_arg("sk_spectrum_bin: index out of range");
    *re = s->bins[k].real();
    *im = s->bins[k].imag();
    return SK_OK;
}

sk_status sk_spectrum_magnitude_db(const sk_spectrum* s, size_t k, double* out_db) {
    if (!s || !out_db) return bad_arg("sk_spectrum_magnitude_db: null argument");
    if (k >= s->bins.size()) return bad_arg("sk_spectrum_magnitude_db: index out of range");
    const double mag = std::abs(s->bins[k]);   // types.cpp:13-18
    *out_db = mag > 1e-15 ? 20.0 * std::log10(mag) : -300.0;
    return SK_OK;
}

sk_status sk_spectrum_copy_data(const sk_spectrum* s, double* re, double* im) {
    if (!s || !re || !im) return bad_arg("sk_spectrum_copy_data: null argument");
    split(s->bins, re, im);
    return SK_OK;
}

sk_status sk_spectrum_slice_band(const sk_spectrum* s, double f_lo, double f_hi, sk_spectrum** out) {
    if (!s || !out) return bad_arg("sk_spectrum_slice_band: null argument");
    return guarded([&] {   // spectra.cpp:40-61
        if (s->bins.empty()) throw std::invalid_argument("slice_band: empty spectrum");
        if (!(s->f_step > 0.0)) throw std::invalid_argument("slice_band: non-positive step");
        if (!(f_lo <= f_hi)) throw std::invalid_argument("slice_band: inverted band");
        const double eps = 0.5 * s->f_step * 1e-9;
        const double lo = (f_lo - s->f_start) / s->f_step;
        const double hi = (f_hi - s->f_start) / s->f_step;
        const long k_lo = static_cast<long>(std::ceil(lo - eps));
        const long k_hi = static_cast<long>(std::floor(hi + eps));
        const long last = static_cast<long>(s->bins.size()) - 1;
        const long a = std::max(k_lo, 0L), b = std::min(k_hi, last);
        if (a > b) throw std::invalid_argument("slice_band: no bins fall inside the requested band");
        auto* o = new sk_spectrum;
        o->bins.assign(s->bins.begin() + a, s->bins.begin() + b + 1);
        o->f_start = s->f_start + static_cast<double>(a) * s->f_step;
        o->f_step = s->f_step;
        o->source_n = s->source_n;
        *out = o;
    });
}

// ---- zoom --------------------------------------------------------------------------------------
void sk_zoom_options_defaults(sk_zoom_options* o) {
    if (!o) return;
    o->center_hz = 0.0;
    o->center_set = 0;
    o->decimation = 0;
    o->cutoff_hz = 0.0;
    o->num_taps = 0;
    o->circular = 1;
    o->trim_transient = 0;
    o->pad_pow2 = 1;
}

static skg::ZoomOptionsG to_opts(const sk_zoom_options* o) {
    skg::ZoomOptionsG g;
    if (o) {
        g.center_hz = o->center_hz;
        g.center_set = o->center_set != 0;
        g.decimation = o->decimation;
        g.cutoff_hz = o->cutoff_hz;
        g.num_taps = o->num_taps;
        g.circular = o->circular != 0;
        g.trim_transient = o->trim_transient != 0;
        g.pad_pow2 = o->pad_pow2 != 0;
    }
    return g;
}

sk_status sk_zoom_plan_create(size_t input_len, double f1, double f2, double fs, const sk_zoom_options* opts,
                              sk_zoom_plan** out) {
    if (!out) return bad_arg("sk_zoom_plan_create: null output");
    return guarded([&] {
        auto p = std::make_unique<skg::ZoomPlanG>(input_len, f1, f2, fs, to_opts(opts));
        *out = new sk_zoom_plan{std::move(p)};
    });
}
void sk_zoom_plan_free(sk_zoom_plan* p) { delete p; }
size_t sk_zoom_plan_decimation(const sk_zoom_plan* p) { return p ? p->p->decimation : 0; }
size_t sk_zoom_plan_n_fft(const sk_zoom_plan* p) { return p ? p->p->n_fft : 0; }
size_t sk_zoom_plan_filter_len(const sk_zoom_plan* p) { return p ? p->p->filter_taps.size() : 0; }
double sk_zoom_plan_f_step(const sk_zoom_plan* p) { return p ? p->p->f_step_hz() : 0.0; }

sk_status sk_zoom_spectrum(const sk_zoom_plan* p, const sk_trace* t, sk_spectrum** out) {
    if (!p || !t || !out) return bad_arg("sk_zoom_spectrum: null argument");
    return guarded([&] {   // zoomfft.cpp:183-189 checks, then the fused kernel
        validate_trace(*t);
        const skg::ZoomPlanG& z = *p->p;
        if (t->samples.size() != z.input_len)
            throw std::invalid_argument("zoom_fft: trace length does not match the plan");
        if (std::abs(t->fs - z.sample_rate_hz) > 1e-9 * z.sample_rate_hz)
            throw std::invalid_argument("zoom_fft: trace sample rate does not match the plan");
        if (z.k_lo > z.k_hi) throw std::invalid_argument("zoom_fft: no transform bins fall inside the band");
        Stage s;
        s.put(t->samples.data(), t->samples.size() * sizeof(double));
        const size_t nb = z.bins();
        s.alloc_out(nb * sizeof(cd));
        z.execute(s.in.p, 0, 1, s.out.p, 0, false, s.st);
        auto* sp = new sk_spectrum;
        sp->bins.resize(nb);
        s.get(sp->bins.data(), nb * sizeof(cd));
        sp->f_start = z.f_start_hz();
        sp->f_step = z.f_step_hz();
        sp->source_n = z.n_fft;
        *out = sp;
    });
}

// ---- batched extension -------------------------------------------------------------------------
sk_status skg_device_info(int* device, int* sm_count, size_t* smem_optin, size_t* l2_bytes) {
    return guarded([&] {
        skg::require_device();
        const int d = skg::current_device();
        cudaDeviceProp pr;
        skg::check(cudaGetDeviceProperties(&pr, d), "cudaGetDeviceProperties");
        if (device) *device = d;
        if (sm_count) *sm_count = pr.multiProcessorCount;
        if (smem_optin) *smem_optin = pr.sharedMemPerBlockOptin;
        if (l2_bytes) *l2_bytes = pr.l2CacheSize;
    });
}

uint64_t skg_launch_count(void) { return skg::launch_counter().load(); }

void skg_debug_set_grid_cap(unsigned cap) { skg::grid_cap_ref().store(cap); }

sk_status skg_synchronize(void* stream) {
    return guarded([&] { skg::check(cudaStreamSynchronize((cudaStream_t)stream), "cudaStreamSynchronize"); });
}

sk_status skg_fft_batch(size_t n, int inverse, int precision, const void* d_in, size_t in_stride, void* d_out,
                        size_t out_stride, size_t batch, void* stream) {
    if (!d_in || !d_out) return bad_arg("skg_fft_batch: null buffer");
    return guarded([&] {
        if (n == 0) throw std::invalid_argument("fft: empty input");
        if (!skg::is_pow2(n))
            throw std::invalid_argument("fft: length " + std::to_string(n) + " is not a power of two; zero_pad to " +
                                        std::to_string(skg::next_pow2(n)) + " first");
        need_precision("skg_fft_batch", precision);
        need_stride("skg_fft_batch", "input", batch, in_stride, n);
        need_stride("skg_fft_batch", "output", batch, out_stride, n);
        skg::fft_c2c(n, inverse != 0, precision == SKG_F32, d_in, (long long)in_stride, d_out, (long long)out_stride,
                     (long long)batch, (cudaStream_t)stream);
    });
}

sk_status skg_fft_spectrum_batch(size_t n, size_t transform_len, int precision, int layout, const void* d_x,
                                 size_t x_stride, size_t batch, void* d_out, size_t out_stride, void* stream) {
    if (!d_x || !d_out) return bad_arg("skg_fft_spectrum_batch: null buffer");
    return guarded([&] {
        if (n == 0) throw std::invalid_argument("trace: no samples");
        need_precision("skg_fft_spectrum_batch", precision);
        const size_t len = transform_len ? transform_len : skg::next_pow2(n);
        need_stride("skg_fft_spectrum_batch", "trace", batch, x_stride, n);
        need_stride("skg_fft_spectrum_batch", "output", batch, out_stride, layout == SKG_HALF ? len / 2 + 1 : len);
        skg::fft_spectrum_batch(n, transform_len, precision == SKG_F32, layout, d_x, (long long)x_stride,
                                (long long)batch, d_out, (long long)out_stride, (cudaStream_t)stream);
    });
}

sk_status skg_band_bins(size_t size, double f_start, double f_step, double f_lo, double f_hi, size_t* k_lo,
                        size_t* count, double* band_f_start) {
    if (!k_lo || !count) return bad_arg("skg_band_bins: null output");
    return guarded([&] {
        const skg::BandBins r = skg::slice_band_bins(size, f_start, f_step, f_lo, f_hi);
        *k_lo = (size_t)r.k_lo;
        *count = (size_t)r.count;
        if (band_f_start) *band_f_start = r.f_start;
    });
}

sk_status skg_fft_spectrum_band_batch(size_t n, size_t transform_len, int precision, size_t k_lo, size_t count,
                                      const void* d_x, size_t x_stride, size_t batch, void* d_bins, size_t bins_stride,
                                      void* d_db, size_t db_stride, void* stream) {
    if (!d_x || (!d_bins && !d_db)) return bad_arg("skg_fft_spectrum_band_batch: null buffer");
    return guarded([&] {
        if (n == 0) throw std::invalid_argument("trace: no samples");
        need_precision("skg_fft_spectrum_band_batch", precision);
        need_stride("skg_fft_spectrum_band_batch", "trace", batch, x_stride, n);
        if (d_bins) need_stride("skg_fft_spectrum_band_batch", "bins", batch, bins_stride, count);
        if (d_db) need_stride("skg_fft_spectrum_band_batch", "dB", batch, db_stride, count);
        skg::fft_spectrum_band_batch(n, transform_len, precision == SKG_F32, (long long)k_lo, (long long)count, d_x,
                                     (long long)x_stride, (long long)batch, d_bins, (long long)bins_stride, d_db,
                                     (long long)db_stride, (cudaStream_t)stream);
    });
}

sk_status skg_band_db_batch(int precision, const void* d_in, size_t in_stride, size_t k_lo, size_t count, size_t batch,
                            void* d_bins, size_t bins_stride, void* d_db, size_t db_stride, void* stream) {
    if (!d_in || (!d_bins && !d_db)) return bad_arg("skg_band_db_batch: null buffer");
    if (count == 0) return bad_arg("slice_band: no bins fall inside the requested band");
    return guarded([&] {
        need_precision("skg_band_db_batch", precision);
        need_stride("skg_band_db_batch", "input", batch, in_stride, k_lo + count);
        if (d_bins) need_stride("skg_band_db_batch", "bins", batch, bins_stride, count);
        if (d_db) need_stride("skg_band_db_batch", "dB", batch, db_stride, count);
        skg::band_db_batch(precision == SKG_F32, d_in, (long long)in_stride, (long long)k_lo, (long long)count,
                           (long long)batch, d_bins, (long long)bins_stride, d_db, (long long)db_stride,
                           (cudaStream_t)stream);
    });
}

sk_status skg_czt_plan_create(size_t n, double a_re, double a_im, double w_re, double w_im, size_t m, int precision,
                              skg_czt_plan** out) {
    if (!out) return bad_arg("skg_czt_plan_create: null output");
    return guarded([&] {
        need_precision("skg_czt_plan_create", precision);
        auto p = std::make_unique<skg::CztPlanG>(n, cd(a_re, a_im), cd(w_re, w_im), m);
        *out = new skg_czt_plan{std::move(p), precision == SKG_F32};
    });
}
void skg_czt_plan_free(skg_czt_plan* p) { delete p; }
size_t skg_czt_plan_conv_size(const skg_czt_plan* p) { return p ? p->p->conv_size() : 0; }

sk_status skg_czt_execute(const skg_czt_plan* p, const void* d_x, int x_complex, size_t x_stride, size_t batch,
                          void* d_out, size_t out_stride, void* stream) {
    if (!p || !d_x || !d_out) return bad_arg("skg_czt_execute: null argument");
    return guarded([&] {
        need_stride("skg_czt_execute", "trace", batch, x_stride, p->p->input_size());
        need_stride("skg_czt_execute", "output", batch, out_stride, p->p->output_size());
        p->p->execute(d_x, x_complex != 0, (long long)x_stride, (long long)batch, d_out, (long long)out_stride, p->f32,
                      (cudaStream_t)stream);
    });
}

sk_status skg_transfer_plan_create(const double* ref, size_t n, size_t transform_len, int precision,
                                   skg_transfer_plan** out) {
    if (!ref || !out) return bad_arg("skg_transfer_plan_create: null argument");
    return guarded([&] {
        need_precision("skg_transfer_plan_create", precision);
        auto p = std::make_unique<skg::TransferPlanG>(ref, n, transform_len, precision == SKG_F32);
        *out = new skg_transfer_plan{std::move(p)};
    });
}
void skg_transfer_plan_free(skg_transfer_plan* p) { delete p; }
size_t skg_transfer_plan_bins(const skg_transfer_plan* p) { return p ? p->p->bins() : 0; }
sk_status skg_transfer_plan_reference(const skg_transfer_plan* p, double* xr) {
    if (!p || !xr) return bad_arg("skg_transfer_plan_reference: null argument");
    const auto& v = p->p->reference_spectrum();
    std::memcpy(xr, v.data(), v.size() * sizeof(cd));
    return SK_OK;
}
sk_status skg_transfer_execute(const skg_transfer_plan* p, const void* d_x, size_t x_stride, size_t batch,
                               void* d_mag, void* d_phase, size_t mp_stride, void* d_h, size_t h_stride,
                               void* stream) {
    if (!p || !d_x || !d_mag || !d_phase) return bad_arg("skg_transfer_execute: null argument");
    return guarded([&] {
        need_stride("skg_transfer_execute", "trace", batch, x_stride, p->p->input_size());
        need_stride("skg_transfer_execute", "|H| / arg H", batch, mp_stride, p->p->bins());
        if (d_h) need_stride("skg_transfer_execute", "H", batch, h_stride, p->p->bins());
        p->p->execute(d_x, (long long)x_stride, (long long)batch, d_mag, d_phase, (long long)mp_stride, d_h,
                      (long long)h_stride, (cudaStream_t)stream);
    });
}

sk_status skg_zoom_plan_create(size_t input_len, double f1, double f2, double fs, const sk_zoom_options* opts,
                               const skg_zoom_ext* ext, int precision, skg_zoom_plan** out) {
    if (!out) return bad_arg("skg_zoom_plan_create: null output");
    return guarded([&] {
        need_precision("skg_zoom_plan_create", precision);
        auto p = std::make_unique<skg::ZoomPlanG>(input_len, f1, f2, fs, to_opts(opts), ext ? ext->n_fft : 0,
                                                  ext ? ext->taps : nullptr, ext ? ext->num_taps : 0);
        *out = new skg_zoom_plan{std::move(p), precision == SKG_F32};
    });
}
void skg_zoom_plan_free(skg_zoom_plan* p) { delete p; }
sk_status skg_zoom_plan_info(const skg_zoom_plan* p, size_t* bins, double* f_start, double* f_step, size_t* n_fft,
                             size_t* decimation, size_t* num_taps) {
    if (!p) return bad_arg("skg_zoom_plan_info: null plan");
    const skg::ZoomPlanG& z = *p->p;
    if (bins) *bins = z.k_hi >= z.k_lo ? z.bins() : 0;
    if (f_start) *f_start = z.f_start_hz();
    if (f_step) *f_step = z.f_step_hz();
    if (n_fft) *n_fft = z.n_fft;
    if (decimation) *decimation = z.decimation;
    if (num_taps) *num_taps = z.filter_taps.size();
    return SK_OK;
}
sk_status skg_zoom_execute(const skg_zoom_plan* p, const void* d_x, size_t x_stride, size_t batch, void* d_out,
                           size_t out_stride, void* stream) {
    if (!p || !d_x || !d_out) return bad_arg("skg_zoom_execute: null argument");
    return guarded([&] {
        need_stride("skg_zoom_execute", "trace", batch, x_stride, p->p->input_len);
        if (p->p->k_hi >= p->p->k_lo) need_stride("skg_zoom_execute", "output", batch, out_stride, p->p->bins());
        p->p->execute(d_x, (long long)x_stride, (long long)batch, d_out, (long long)out_stride, p->f32,
                      (cudaStream_t)stream);
    });
}


// ---- host-buffer batched calls (staging.hpp pipeline) ---------------------------------------------
sk_status skg_czt_execute_host(const skg_czt_plan* p, const void* h_x, int x_complex, size_t x_stride, size_t batch,
                               void* h_out, size_t out_stride, size_t chunk) {
    if (!p || !h_x || !h_out) return bad_arg("skg_czt_execute_host: null argument");
    return guarded([&] {
        const skg::CztPlanG& g = *p->p;
        const size_t n = g.input_size(), m = g.output_size();
        need_stride("skg_czt_execute_host", "trace", batch, x_stride, n);
        need_stride("skg_czt_execute_host", "output", batch, out_stride, m);
        const size_t rs = p->f32 ? 4 : 8, es = x_complex ? 2 * rs : rs;
        skg::HostPlane in{const_cast<void*>(h_x), x_stride * es, n * es};
        skg::HostPlane out{h_out, out_stride * 2 * rs, m * 2 * rs};
        skg::run_host_batched(in, {out}, (long long)batch, (long long)chunk,
                              [&](const void* dx, void* const* dout, long long rows, cudaStream_t st) {
                                  g.execute(dx, x_complex != 0, (long long)n, rows, dout[0], (long long)m, p->f32, st);
                              });
    });
}

sk_status skg_fft_spectrum_host(size_t n, size_t transform_len, int precision, int layout, const void* h_x,
                                size_t x_stride, size_t batch, void* h_out, size_t out_stride, size_t chunk) {
    if (!h_x || !h_out) return bad_arg("skg_fft_spectrum_host: null buffer");
    return guarded([&] {
        if (n == 0) throw std::invalid_argument("trace: no samples");
        need_precision("skg_fft_spectrum_host", precision);
        const size_t len = transform_len ? transform_len : skg::next_pow2(n);
        const size_t nb = layout == SKG_HALF ? len / 2 + 1 : len;
        need_stride("skg_fft_spectrum_host", "trace", batch, x_stride, n);
        need_stride("skg_fft_spectrum_host", "output", batch, out_stride, nb);
        const bool f32 = precision == SKG_F32;
        const size_t rs = f32 ? 4 : 8;
        skg::HostPlane in{const_cast<void*>(h_x), x_stride * rs, n * rs};
        skg::HostPlane out{h_out, out_stride * 2 * rs, nb * 2 * rs};
        skg::run_host_batched(in, {out}, (long long)batch, (long long)chunk,
                              [&](const void* dx, void* const* dout, long long rows, cudaStream_t st) {
                                  skg::fft_spectrum_batch(n, len, f32, layout, dx, (long long)n, rows, dout[0],
                                                          (long long)nb, st);
                              });
    });
}

sk_status skg_zoom_execute_host(const skg_zoom_plan* p, const void* h_x, size_t x_stride, size_t batch, void* h_out,
                                size_t out_stride, size_t chunk) {
    if (!p || !h_x || !h_out) return bad_arg("skg_zoom_execute_host: null argument");
    return guarded([&] {
        const skg::ZoomPlanG& z = *p->p;
        if (z.k_lo > z.k_hi) throw std::invalid_argument("zoom_fft: no transform bins fall inside the band");
        const size_t n = z.input_len, nb = z.bins();
        need_stride("skg_zoom_execute_host", "trace", batch, x_stride, n);
        need_stride("skg_zoom_execute_host", "output", batch, out_stride, nb);
        const size_t rs = p->f32 ? 4 : 8;
        skg::HostPlane in{const_cast<void*>(h_x), x_stride * rs, n * rs};
        skg::HostPlane out{h_out, out_stride * 2 * rs, nb * 2 * rs};
        skg::run_host_batched(in, {out}, (long long)batch, (long long)chunk,
                              [&](const void* dx, void* const* dout, long long rows, cudaStream_t st) {
                                  z.execute(dx, (long long)n, rows, dout[0], (long long)nb, p->f32, st);
                              });
    });
}

sk_status skg_transfer_execute_host(const skg_transfer_plan* p, const void* h_x, size_t x_stride, size_t batch,
                                    void* h_mag, void* h_phase, size_t mp_stride, size_t chunk) {
    if (!p || !h_x || !h_mag || !h_phase) return bad_arg("skg_transfer_execute_host: null argument");
    return guarded([&] {
        const skg::TransferPlanG& t = *p->p;
        const size_t n = t.input_size(), nb = t.bins();
        need_stride("skg_transfer_execute_host", "trace", batch, x_stride, n);
        need_stride("skg_transfer_execute_host", "|H| / arg H", batch, mp_stride, nb);
        const size_t rs = t.f32() ? 4 : 8;
        skg::HostPlane in{const_cast<void*>(h_x), x_stride * rs, n * rs};
        skg::HostPlane mag{h_mag, mp_stride * rs, nb * rs}, ph{h_phase, mp_stride * rs, nb * rs};
        skg::run_host_batched(in, {mag, ph}, (long long)batch, (long long)chunk,
                              [&](const void* dx, void* const* dout, long long rows, cudaStream_t st) {
                                  t.execute(dx, (long long)n, rows, dout[0], dout[1], (long long)nb, nullptr, 0, st);
                              });
    });
}

}  // extern "C"
