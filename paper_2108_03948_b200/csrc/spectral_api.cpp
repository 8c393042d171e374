// spectral_api.cpp — the reference's C++ API (include/spectral_b200.hpp) over the GPU runtime.
// Transforms run on the device; sizing, validation and fp64 table building stay on the host exactly
// as in the reference (they are scalar plan-time work there too).
#include "spectral_b200.hpp"

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include <istream>
#include <iterator>
#include <ostream>

#include "analysis.hpp"
#include "host.hpp"
#include "io.hpp"
#include "staging.hpp"

namespace skg {
cudaError_t launch_dft_naive(const void* x, long long n, const void* tw, void* out, cudaStream_t st);
cudaError_t launch_czt_direct(const void* x, long long n, double a_logm, double a_q, double w_logm, double w_q,
                              long long m, void* xa_scratch, void* out, cudaStream_t st);
cudaError_t launch_freq_shift(const double* xr, const void* xc, long long n, double q, void* y, cudaStream_t st);
cudaError_t launch_filter_decimate(const void* x, long long n, const double* taps, int T, int d, int circular,
                                   void* out, long long nout, cudaStream_t st);
}  // namespace skg

namespace spectral {

namespace {
#define kStream cudaStreamPerThread

// host span -> device slot -> kernel -> host vector: every call stages through the calling thread's
// grow-only pinned / device slots (skg::CallStage), never a cudaMalloc / cudaFree per call
}  // namespace

// ---- types.cpp ---------------------------------------------------------------------------------
double magnitude_db(double mag) { return mag > 1e-15 ? 20.0 * std::log10(mag) : -300.0; }
double magnitude_db(const cplx& v) { return magnitude_db(std::abs(v)); }

void validate_trace(const Trace& t) {
    if (t.samples.empty()) throw std::invalid_argument("trace: no samples");
    if (!(t.sample_rate_hz > 0.0) || !std::isfinite(t.sample_rate_hz))
        throw std::invalid_argument("trace: sample rate must be positive and finite");
    for (double v : t.samples)
        if (!std::isfinite(v)) throw std::invalid_argument("trace: non-finite sample");
    if (!std::isfinite(t.t0_s)) throw std::invalid_argument("trace: non-finite start time");
}

// ---- numerics.cpp -------------------------------------------------------------------------------
bool is_pow2(std::size_t n) { return skg::is_pow2(n); }
std::size_t next_pow2(std::size_t n) { return skg::next_pow2(n); }
cplx cis_cycles(double q, double t) { return skg::cis_cycles(q, t); }

ComplexBuffer zero_pad(std::span<const cplx> x, std::size_t target_len) {
    if (target_len < x.size())
        throw std::invalid_argument("zero_pad: target length " + std::to_string(target_len) +
                                    " is shorter than the input (" + std::to_string(x.size()) + ")");
    ComplexBuffer out(target_len, cplx(0.0, 0.0));
    std::copy(x.begin(), x.end(), out.begin());
    return out;
}

ComplexBuffer dft_naive(std::span<const cplx> x) {
    if (x.empty()) throw std::invalid_argument("dft_naive: empty input");
    const size_t n = x.size();
    std::vector<cplx> tw(n);
    for (size_t r = 0; r < n; ++r) {
        const double ang = -2.0 * M_PI * static_cast<double>(r) / static_cast<double>(n);
        tw[r] = cplx(std::cos(ang), std::sin(ang));
    }
    skg::CallStage cs;
    void* dx = cs.up(x.data(), n * sizeof(cplx));
    void* dt = cs.up(tw.data(), n * sizeof(cplx));
    void* dy = cs.out(n * sizeof(cplx));
    skg::check(skg::launch_dft_naive(dx, (long long)n, dt, dy, kStream), "dft_naive");
    skg::count_launch();
    ComplexBuffer y(n);
    cs.down(y.data(), dy, n * sizeof(cplx));
    return y;
}

FftPlan::FftPlan(std::size_t n) : n_(n) {
    if (!skg::is_pow2(n)) throw std::invalid_argument("FftPlan: size must be a power of two");
}

void FftPlan::run(std::span<cplx> a, bool invert) const {
    if (a.size() != n_) throw std::invalid_argument("FftPlan: buffer size does not match plan");
    skg::CallStage cs;
    void* d = cs.up(a.data(), n_ * sizeof(cplx));
    skg::fft_c2c(n_, invert, false, d, 0, d, 0, 1, kStream);
    cs.down(a.data(), d, n_ * sizeof(cplx));
}
void FftPlan::forward(std::span<cplx> data) const { run(data, false); }
void FftPlan::inverse(std::span<cplx> data) const { run(data, true); }

static ComplexBuffer run_pow2(std::span<const cplx> x, bool invert) {   // numerics.cpp:102-117
    if (x.empty()) throw std::invalid_argument("fft: empty input");
    if (!skg::is_pow2(x.size()))
        throw std::invalid_argument("fft: length " + std::to_string(x.size()) + " is not a power of two; zero_pad to " +
                                    std::to_string(skg::next_pow2(x.size())) + " first");
    ComplexBuffer buf(x.begin(), x.end());
    FftPlan plan(buf.size());
    if (invert) plan.inverse(buf);
    else plan.forward(buf);
    return buf;
}
ComplexBuffer fft(std::span<const cplx> x) { return run_pow2(x, false); }
ComplexBuffer ifft(std::span<const cplx> x) { return run_pow2(x, true); }

// ---- czt.cpp -----------------------------------------------------------------------------------
void validate(const CztParams& p) {
    if (p.m == 0) throw std::invalid_argument("czt: m must be >= 1");
    if (!(std::abs(p.a) > 0.0) || !(std::abs(p.w) > 0.0))
        throw std::invalid_argument("czt: a and w must be nonzero");
}

CztParams czt_params_for_band(double f1, double f2, double fs, std::size_t m) {
    if (!(fs > 0.0)) throw std::invalid_argument("czt_params_for_band: sample rate must be positive");
    if (!(f1 >= 0.0) || !(f1 < f2)) throw std::invalid_argument("czt_params_for_band: need 0 <= f1 < f2");
    if (f2 > fs * (1.0 + 1e-12)) throw std::invalid_argument("czt_params_for_band: f2 exceeds the sample rate");
    if (m < 2) throw std::invalid_argument("czt_params_for_band: m must be >= 2");
    CztParams p;
    p.a = skg::cis_cycles(f1 / fs, 1.0);
    p.w = skg::cis_cycles(-(f2 - f1) / (static_cast<double>(m) * fs), 1.0);
    p.m = m;
    return p;
}

ComplexBuffer czt_direct(std::span<const cplx> x, const CztParams& p) {
    validate(p);
    if (x.empty()) throw std::invalid_argument("czt_direct: empty input");
    const skg::PolarPow A(p.a), W(p.w);
    const size_t n = x.size();
    skg::CallStage cs;
    void* dx = cs.up(x.data(), n * sizeof(cplx));
    void* xa = cs.scratch(n * sizeof(cplx));
    void* dy = cs.out(p.m * sizeof(cplx));
    skg::check(skg::launch_czt_direct(dx, (long long)n, A.log_mag, A.q, W.log_mag, W.q, (long long)p.m, xa,
                                      dy, kStream),
               "czt_direct");
    skg::count_launch(2);
    ComplexBuffer y(p.m);
    cs.down(y.data(), dy, p.m * sizeof(cplx));
    return y;
}

CztPlan::CztPlan(std::size_t input_len, const CztParams& p) {
    validate(p);
    impl_ = std::make_shared<skg::CztPlanG>(input_len, p.a, p.w, p.m);
}
static const skg::CztPlanG& G(const std::shared_ptr<const void>& p) { return *static_cast<const skg::CztPlanG*>(p.get()); }
std::size_t CztPlan::input_size() const { return G(impl_).input_size(); }
std::size_t CztPlan::output_size() const { return G(impl_).output_size(); }
std::size_t CztPlan::conv_size() const { return G(impl_).conv_size(); }

void CztPlan::execute(std::span<const cplx> x, std::span<cplx> conv_scratch, std::span<cplx> out) const {
    if (x.size() != input_size()) throw std::invalid_argument("CztPlan: input length does not match plan");
    if (conv_scratch.size() != conv_size() || out.size() != output_size())
        throw std::invalid_argument("CztPlan: scratch/output size mismatch");
    skg::CallStage cs;
    void* dx = cs.up(x.data(), x.size() * sizeof(cplx));
    void* dy = cs.out(out.size() * sizeof(cplx));
    G(impl_).execute(dx, true, 0, 1, dy, 0, false, kStream);
    cs.down(out.data(), dy, out.size() * sizeof(cplx));
}

ComplexBuffer CztPlan::execute(std::span<const cplx> x) const {
    if (x.size() != input_size()) throw std::invalid_argument("CztPlan: input length does not match plan");
    ComplexBuffer out(output_size());
    skg::CallStage cs;
    void* dx = cs.up(x.data(), x.size() * sizeof(cplx));
    void* dy = cs.out(out.size() * sizeof(cplx));
    G(impl_).execute(dx, true, 0, 1, dy, 0, false, kStream);
    cs.down(out.data(), dy, out.size() * sizeof(cplx));
    return out;
}

ComplexBuffer czt(std::span<const cplx> x, const CztParams& p) {
    if (x.empty()) throw std::invalid_argument("czt: empty input");
    return CztPlan(x.size(), p).execute(x);
}

ComplexBuffer dft_any(std::span<const cplx> x) {
    if (x.empty()) throw std::invalid_argument("dft_any: empty input");
    if (skg::is_pow2(x.size())) return fft(x);
    CztParams p;
    p.a = cplx(1.0, 0.0);
    p.w = skg::cis_cycles(-1.0 / static_cast<double>(x.size()), 1.0);
    p.m = x.size();
    return czt(x, p);
}

Spectrum czt_spectrum(const Trace& trace, double f1, double f2, std::size_t m) {
    validate_trace(trace);
    const double nyquist = trace.sample_rate_hz / 2.0;
    if (!(f1 >= 0.0) || !(f1 < f2)) throw std::invalid_argument("czt_spectrum: need 0 <= f1 < f2");
    if (f2 > nyquist * (1.0 + 1e-12))
        throw std::invalid_argument("czt_spectrum: band edge " + std::to_string(f2) + " Hz exceeds the Nyquist rate " +
                                    std::to_string(nyquist) + " Hz");
    const CztParams p = czt_params_for_band(f1, f2, trace.sample_rate_hz, m);
    const size_t n = trace.samples.size();
    skg::CztPlanG plan(n, p.a, p.w, p.m);
    skg::CallStage cs;
    void* dx = cs.up(trace.samples.data(), n * sizeof(double));
    void* dy = cs.out(m * sizeof(cplx));
    plan.execute(dx, false, 0, 1, dy, 0, false, kStream);
    Spectrum s;
    s.bins.resize(m);
    cs.down(s.bins.data(), dy, m * sizeof(cplx));
    s.f_start_hz = f1;
    s.f_step_hz = (f2 - f1) / static_cast<double>(m);
    s.source_n = n;
    return s;
}

// ---- spectra.cpp -------------------------------------------------------------------------------
Spectrum fft_spectrum(const Trace& t, std::size_t transform_len) {
    validate_trace(t);
    const size_t n = t.size();
    const size_t len = transform_len == 0 ? skg::next_pow2(n) : transform_len;
    if (len < n) throw std::invalid_argument("fft_spectrum: transform length shorter than the trace");
    skg::CallStage cs;
    void* dx = cs.up(t.samples.data(), n * sizeof(double));
    void* dy = cs.out(len * sizeof(cplx));
    skg::fft_spectrum_batch(n, len, false, 0, dx, 0, 1, dy, 0, kStream);
    Spectrum s;
    s.bins.resize(len);
    cs.down(s.bins.data(), dy, len * sizeof(cplx));
    s.f_start_hz = 0.0;
    s.f_step_hz = t.sample_rate_hz / static_cast<double>(len);
    s.source_n = len;
    return s;
}

Spectrum slice_band(const Spectrum& s, double f_lo, double f_hi) {
    if (s.bins.empty()) throw std::invalid_argument("slice_band: empty spectrum");
    if (!(s.f_step_hz > 0.0)) throw std::invalid_argument("slice_band: non-positive step");
    if (!(f_lo <= f_hi)) throw std::invalid_argument("slice_band: inverted band");
    const double eps = 0.5 * s.f_step_hz * 1e-9;
    const long k_lo = static_cast<long>(std::ceil((f_lo - s.f_start_hz) / s.f_step_hz - eps));
    const long k_hi = static_cast<long>(std::floor((f_hi - s.f_start_hz) / s.f_step_hz + eps));
    const long a = std::max(k_lo, 0L), b = std::min(k_hi, static_cast<long>(s.bins.size()) - 1);
    if (a > b) throw std::invalid_argument("slice_band: no bins fall inside the requested band");
    Spectrum out;
    out.bins.assign(s.bins.begin() + a, s.bins.begin() + b + 1);
    out.f_start_hz = s.frequency(static_cast<size_t>(a));
    out.f_step_hz = s.f_step_hz;
    out.source_n = s.source_n;
    return out;
}

// ---- zoomfft.cpp -------------------------------------------------------------------------------
double ZoomFftPlan::f_step_hz() const {
    return sample_rate_hz / (static_cast<double>(decimation) * static_cast<double>(n_fft));
}

std::vector<double> design_lowpass(double cutoff, double fs, std::size_t taps) {
    return skg::design_lowpass(cutoff, fs, taps);
}

static ComplexBuffer shift_impl(const double* xr, const cplx* xc, size_t n, double f, double fs) {
    if (!(fs > 0.0)) throw std::invalid_argument("frequency_shift: sample rate must be positive");
    ComplexBuffer y(n);
    if (n == 0) return y;
    skg::CallStage cs;
    void* dx = xr ? cs.up(xr, n * sizeof(double)) : cs.up(xc, n * sizeof(cplx));
    void* dy = cs.out(n * sizeof(cplx));
    skg::check(skg::launch_freq_shift(xr ? (const double*)dx : nullptr, xr ? nullptr : dx, (long long)n,
                                      -f / fs, dy, kStream),
               "frequency_shift");
    skg::count_launch();
    cs.down(y.data(), dy, n * sizeof(cplx));
    return y;
}
ComplexBuffer frequency_shift(std::span<const double> x, double f, double fs) {
    return shift_impl(x.data(), nullptr, x.size(), f, fs);
}
ComplexBuffer frequency_shift(std::span<const cplx> x, double f, double fs) {
    return shift_impl(nullptr, x.data(), x.size(), f, fs);
}

static ComplexBuffer fd_impl(std::span<const cplx> x, std::span<const double> taps, std::size_t d, bool circular) {
    const size_t n = x.size();
    ComplexBuffer out(n / (d ? d : 1));
    if (out.empty()) return out;
    skg::CallStage cs;
    void* dx = cs.up(x.data(), n * sizeof(cplx));
    void* dt = cs.up(taps.data(), taps.size() * sizeof(double));
    void* dy = cs.out(out.size() * sizeof(cplx));
    skg::check(skg::launch_filter_decimate(dx, (long long)n, (const double*)dt, (int)taps.size(), (int)d,
                                           circular ? 1 : 0, dy, (long long)out.size(), kStream),
               "filter_decimate");
    skg::count_launch();
    cs.down(out.data(), dy, out.size() * sizeof(cplx));
    return out;
}
ComplexBuffer filter_decimate(std::span<const cplx> x, std::span<const double> taps, std::size_t d) {
    if (d == 0) throw std::invalid_argument("filter_decimate: decimation must be >= 1");
    if (taps.empty()) throw std::invalid_argument("filter_decimate: empty filter");
    return fd_impl(x, taps, d, false);
}
ComplexBuffer filter_decimate_circular(std::span<const cplx> x, std::span<const double> taps, std::size_t d) {
    if (d == 0) throw std::invalid_argument("filter_decimate_circular: decimation must be >= 1");
    if (taps.empty()) throw std::invalid_argument("filter_decimate_circular: empty filter");
    if (x.empty() || x.size() % d != 0)
        throw std::invalid_argument("filter_decimate_circular: decimation must divide the record length");
    if (taps.size() > x.size()) throw std::invalid_argument("filter_decimate_circular: filter longer than record");
    return fd_impl(x, taps, d, true);
}

namespace {
struct ZoomDevice {
    ZoomFftPlan fields;   // snapshot the device plan was built from
    std::unique_ptr<skg::ZoomPlanG> plan;
};
bool same_fields(const ZoomFftPlan& a, const ZoomFftPlan& b) {
    return a.f1_hz == b.f1_hz && a.f2_hz == b.f2_hz && a.center_hz == b.center_hz &&
           a.sample_rate_hz == b.sample_rate_hz && a.decimation == b.decimation && a.filter_taps == b.filter_taps &&
           a.group_delay_samples == b.group_delay_samples && a.circular == b.circular &&
           a.trim_transient == b.trim_transient && a.input_len == b.input_len && a.usable_len == b.usable_len &&
           a.trim_samples == b.trim_samples && a.decimated_len == b.decimated_len && a.n_fft == b.n_fft;
}
}  // namespace

ZoomFftPlan make_zoom_plan(std::size_t input_len, double f1, double f2, double fs, const ZoomOptions& o) {
    skg::ZoomOptionsG g;
    g.center_hz = o.center_hz;
    g.center_set = o.center_set;
    g.decimation = o.decimation;
    g.cutoff_hz = o.cutoff_hz;
    g.num_taps = o.num_taps;
    g.circular = o.circular;
    g.trim_transient = o.trim_transient;
    g.pad_pow2 = o.pad_pow2;
    auto plan = std::make_unique<skg::ZoomPlanG>(input_len, f1, f2, fs, g);
    ZoomFftPlan p;
    p.f1_hz = plan->f1_hz;
    p.f2_hz = plan->f2_hz;
    p.center_hz = plan->center_hz;
    p.sample_rate_hz = plan->sample_rate_hz;
    p.cutoff_hz = plan->cutoff_hz;
    p.decimation = plan->decimation;
    p.filter_taps = plan->filter_taps;
    p.group_delay_samples = plan->group_delay_samples;
    p.circular = plan->circular;
    p.trim_transient = plan->trim_transient;
    p.pad_pow2 = plan->pad_pow2;
    p.input_len = plan->input_len;
    p.usable_len = plan->usable_len;
    p.trim_samples = plan->trim_samples;
    p.decimated_len = plan->decimated_len;
    p.n_fft = plan->n_fft;
    auto dev = std::make_shared<ZoomDevice>();
    dev->fields = p;
    dev->plan = std::move(plan);
    p.device = dev;
    return p;
}

Spectrum zoom_fft(const ZoomFftPlan& plan, const Trace& t) {   // zoomfft.cpp:183-239
    validate_trace(t);
    if (t.size() != plan.input_len) throw std::invalid_argument("zoom_fft: trace length does not match the plan");
    if (std::abs(t.sample_rate_hz - plan.sample_rate_hz) > 1e-9 * plan.sample_rate_hz)
        throw std::invalid_argument("zoom_fft: trace sample rate does not match the plan");
    auto dev = std::static_pointer_cast<ZoomDevice>(plan.device);
    if (!dev || !same_fields(dev->fields, plan)) {
        // the public fields were edited (or the plan was built by hand): rebuild the device plan
        auto nd = std::make_shared<ZoomDevice>();
        nd->fields = plan;
        skg::ZoomFields f;
        f.f1_hz = plan.f1_hz;
        f.f2_hz = plan.f2_hz;
        f.sample_rate_hz = plan.sample_rate_hz;
        f.center_hz = plan.center_hz;
        f.cutoff_hz = plan.cutoff_hz;
        f.decimation = plan.decimation;
        f.filter_taps = plan.filter_taps;
        f.group_delay_samples = plan.group_delay_samples;
        f.circular = plan.circular;
        f.trim_transient = plan.trim_transient;
        f.pad_pow2 = plan.pad_pow2;
        f.input_len = plan.input_len;
        f.usable_len = plan.usable_len;
        f.trim_samples = plan.trim_samples;
        f.decimated_len = plan.decimated_len;
        f.n_fft = plan.n_fft;
        nd->plan = skg::ZoomPlanG::from_fields(f);
        plan.device = nd;
        dev = nd;
    }
    const skg::ZoomPlanG& z = *dev->plan;
    if (z.k_lo > z.k_hi) throw std::invalid_argument("zoom_fft: no transform bins fall inside the band");
    skg::CallStage cs;
    void* dx = cs.up(t.samples.data(), t.size() * sizeof(double));
    void* dy = cs.out(z.bins() * sizeof(cplx));
    z.execute(dx, 0, 1, dy, 0, false, kStream);
    Spectrum s;
    s.bins.resize(z.bins());
    cs.down(s.bins.data(), dy, z.bins() * sizeof(cplx));
    s.f_start_hz = z.f_start_hz();
    s.f_step_hz = z.f_step_hz();
    s.source_n = z.n_fft;
    return s;
}

// ---- file formats and analysis (io.cpp / analysis.cpp), the runtime's errors mapped to the
// reference's exception classes ------------------------------------------------------------------
namespace {
template <typename F> auto mapped(F&& f) -> decltype(f()) {
    try {
        return f();
    } catch (const skg::ParseError& e) {
        throw ParseError(e.what(), e.line);
    } catch (const skg::FormatError& e) {
        throw FormatError(e.what());
    } catch (const skg::IoError& e) {
        throw IoError(e.what());
    } catch (const skg::InsufficientResolution& e) {
        throw InsufficientResolutionError(e.what());
    }
}
std::string slurp(std::istream& in) { return std::string(std::istreambuf_iterator<char>(in), {}); }
Trace to_trace(skg::HostTrace&& h) {
    Trace t;
    t.samples = std::move(h.samples);
    t.sample_rate_hz = h.fs;
    t.t0_s = h.t0;
    return t;
}
Spectrum to_spectrum(const skg::HostSpectrum& h) {
    Spectrum s;
    s.bins.resize(h.bins.size() / 2);
    for (std::size_t k = 0; k < s.bins.size(); ++k) s.bins[k] = cplx(h.bins[2 * k], h.bins[2 * k + 1]);
    s.f_start_hz = h.f_start;
    s.f_step_hz = h.f_step;
    s.source_n = h.source_n;
    return s;
}
std::string trace_csv(const Trace& t) {
    validate_trace(t);
    std::string out = "time_s,amplitude\n";
    const double dt = 1.0 / t.sample_rate_hz;
    for (std::size_t i = 0; i < t.samples.size(); ++i) {
        skg::append_g17(out, t.t0_s + static_cast<double>(i) * dt);
        out += ',';
        skg::append_g17(out, t.samples[i]);
        out += '\n';
    }
    return out;
}
skg::DipMetricH to_h(const DipMetric& m) {
    skg::DipMetricH h;
    h.resolved = m.resolved;
    h.dip_db = m.dip_db;
    h.f_peak_a_hz = m.f_peak_a_hz;
    h.peak_a_db = m.peak_a_db;
    h.f_peak_b_hz = m.f_peak_b_hz;
    h.peak_b_db = m.peak_b_db;
    h.f_valley_hz = m.f_valley_hz;
    h.valley_db = m.valley_db;
    return h;
}
DipMetric from_h(const skg::DipMetricH& h) {
    DipMetric m;
    m.resolved = h.resolved;
    m.dip_db = h.dip_db;
    m.f_peak_a_hz = h.f_peak_a_hz;
    m.peak_a_db = h.peak_a_db;
    m.f_peak_b_hz = h.f_peak_b_hz;
    m.peak_b_db = h.peak_b_db;
    m.f_valley_hz = h.f_valley_hz;
    m.valley_db = h.valley_db;
    return m;
}
}  // namespace

Trace read_trace_csv(std::istream& in, const std::string& origin) {
    const std::string s = slurp(in);
    return mapped([&] { return to_trace(skg::parse_trace_csv(s.data(), s.size(), origin)); });
}
Trace read_trace_csv_file(const std::string& path) {
    return mapped([&] { return to_trace(skg::read_trace_csv_file(path)); });
}
void write_trace_csv(const Trace& t, std::ostream& out) {
    out << trace_csv(t);
    if (!out) throw IoError("trace csv: write failed");
}
void write_trace_csv_file(const Trace& t, const std::string& path) {
    mapped([&] { skg::write_trace_csv_file(t.samples.data(), t.samples.size(), t.sample_rate_hz, t.t0_s, path); });
}
Spectrum read_spectrum_csv(std::istream& in, const std::string& origin) {
    const std::string s = slurp(in);
    return mapped([&] { return to_spectrum(skg::parse_spectrum_csv(s.data(), s.size(), origin)); });
}
Spectrum read_spectrum_csv_file(const std::string& path) {
    return mapped([&] { return to_spectrum(skg::read_spectrum_csv_file(path)); });
}
void write_spectrum_csv(const Spectrum& s, std::ostream& out) {
    out << skg::format_spectrum_csv(reinterpret_cast<const double*>(s.bins.data()), s.bins.size(), s.f_start_hz,
                                    s.f_step_hz);
    if (!out) throw IoError("spectrum csv: write failed");
}
void write_spectrum_csv_file(const Spectrum& s, const std::string& path) {
    mapped([&] {
        skg::write_spectrum_csv_file(reinterpret_cast<const double*>(s.bins.data()), s.bins.size(), s.f_start_hz,
                                     s.f_step_hz, path);
    });
}

void write_spectrum_json(const Spectrum& s, std::ostream& out) {
    out << skg::format_spectrum_json(reinterpret_cast<const double*>(s.bins.data()), s.bins.size(), s.f_start_hz,
                                     s.f_step_hz, s.source_n);
    if (!out) throw IoError("spectrum json: write failed");
}
void write_spectrum_json_file(const Spectrum& s, const std::string& path) {
    mapped([&] {
        skg::write_spectrum_json_file(reinterpret_cast<const double*>(s.bins.data()), s.bins.size(), s.f_start_hz,
                                      s.f_step_hz, s.source_n, path);
    });
}

std::size_t record_len_for_step(double fs, double step) { return skg::record_len_for_step(fs, step); }
double fft_resolution(double fs, std::size_t n) { return skg::fft_resolution(fs, n); }
std::size_t zeros_for_resolution(double fs, std::size_t n, double step) { return skg::zeros_for_resolution(fs, n, step); }
std::size_t czt_len_for_matched_resolution(double f1, double f2, double fs, std::size_t n_fft) {
    return skg::czt_len_for_matched_resolution(f1, f2, fs, n_fft);
}

DipMetric dip_metric(const Spectrum& s, double f_a, double f_b) {
    return mapped([&] { return from_h(skg::dip_metric(s.bins.data(), s.bins.size(), s.f_start_hz, s.f_step_hz, f_a, f_b)); });
}

ResolvabilityCurve resolvability_scan(const ScanConfig& cfg) {
    skg::ScanConfigH c;
    c.sample_rate_hz = cfg.sample_rate_hz;
    c.n = cfg.n;
    c.f1_hz = cfg.f1_hz;
    c.f2_hz = cfg.f2_hz;
    c.m = cfg.m;
    c.center_hz = cfg.center_hz;
    c.sep_start_hz = cfg.sep_start_hz;
    c.sep_stop_hz = cfg.sep_stop_hz;
    c.sep_step_hz = cfg.sep_step_hz;
    const skg::CurveH h = mapped([&] { return skg::resolvability_scan(c); });
    ResolvabilityCurve r;
    r.config = cfg;
    r.config.center_hz = h.config.center_hz;
    r.separations_hz = h.separations_hz;
    for (const auto& m : h.fft_metrics) r.fft_metrics.push_back(from_h(m));
    for (const auto& m : h.czt_metrics) r.czt_metrics.push_back(from_h(m));
    r.min_resolved_fft_hz = h.min_resolved_fft_hz;
    r.min_resolved_czt_hz = h.min_resolved_czt_hz;
    r.fft_len = h.fft_len;
    return r;
}

namespace {
skg::CurveH to_curve_h(const ResolvabilityCurve& c) {
    skg::CurveH h;
    h.config.sample_rate_hz = c.config.sample_rate_hz;
    h.config.n = c.config.n;
    h.config.f1_hz = c.config.f1_hz;
    h.config.f2_hz = c.config.f2_hz;
    h.config.m = c.config.m;
    h.config.center_hz = c.config.center_hz;
    h.config.sep_start_hz = c.config.sep_start_hz;
    h.config.sep_stop_hz = c.config.sep_stop_hz;
    h.config.sep_step_hz = c.config.sep_step_hz;
    h.separations_hz = c.separations_hz;
    for (const auto& m : c.fft_metrics) h.fft_metrics.push_back(to_h(m));
    for (const auto& m : c.czt_metrics) h.czt_metrics.push_back(to_h(m));
    h.min_resolved_fft_hz = c.min_resolved_fft_hz;
    h.min_resolved_czt_hz = c.min_resolved_czt_hz;
    h.fft_len = c.fft_len;
    return h;
}
}  // namespace

void write_resolvability_json(const ResolvabilityCurve& c, std::ostream& out) {
    out << skg::format_resolvability_json(to_curve_h(c));
    if (!out) throw IoError("resolvability json: write failed");
}

void write_resolvability_csv(const ResolvabilityCurve& c, std::ostream& out) {
    skg::CurveH h;
    h.separations_hz = c.separations_hz;
    for (const auto& m : c.fft_metrics) h.fft_metrics.push_back(to_h(m));
    for (const auto& m : c.czt_metrics) h.czt_metrics.push_back(to_h(m));
    out << skg::format_resolvability_csv(h);
    if (!out) throw IoError("resolvability csv: write failed");
}

}  // namespace spectral
