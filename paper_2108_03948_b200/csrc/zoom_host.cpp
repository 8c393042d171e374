// zoom_host.cpp — ZoomFftPlan restated (make_zoom_plan, zoomfft.cpp:106-181) plus the device
// tables of the fused zoom kernel.
#include <algorithm>
#include <cmath>

#include "host.hpp"

#include <cstdlib>
#include <string>

namespace skg {

ZoomPlanG::ZoomPlanG(size_t in_len, double f1, double f2, double fs, const ZoomOptionsG& opts,
                     size_t n_fft_override, const double* taps, size_t num_taps) {
    // validation order and messages follow zoomfft.cpp:108-115
    if (in_len < 2) throw std::invalid_argument("make_zoom_plan: need at least 2 input samples");
    if (!(fs > 0.0)) throw std::invalid_argument("make_zoom_plan: sample rate must be positive");
    if (!(f1 >= 0.0) || !(f2 > f1)) throw std::invalid_argument("make_zoom_plan: band must satisfy 0 <= f1 < f2");
    if (f2 > fs / 2.0 * (1.0 + 1e-12))
        throw std::invalid_argument("make_zoom_plan: band exceeds the Nyquist frequency");
    f1_hz = f1;
    f2_hz = f2;
    sample_rate_hz = fs;
    circular = opts.circular;
    trim_transient = opts.trim_transient;
    pad_pow2 = opts.pad_pow2;
    input_len = in_len;
    const double band = f2 - f1;
    center_hz = opts.center_set ? opts.center_hz : 0.5 * (f1 + f2);
    if (!std::isfinite(center_hz)) throw std::invalid_argument("make_zoom_plan: non-finite center frequency");
    decimation = opts.decimation == 0
                     ? std::max<size_t>(1, static_cast<size_t>(std::floor(fs / (2.0 * band))))
                     : opts.decimation;
    const double dnyq = fs / (2.0 * static_cast<double>(decimation));
    const double reach = std::max(f2 - center_hz, center_hz - f1);
    if (reach > dnyq * (1.0 + 1e-12))
        throw std::invalid_argument("make_zoom_plan: decimation too large for the requested band");
    const bool auto_filter = opts.num_taps == 0 && !(opts.cutoff_hz > 0.0);
    if (decimation == 1 && auto_filter) {
        filter_taps = {1.0};
        cutoff_hz = fs / 2.0;
    } else {
        cutoff_hz = opts.cutoff_hz > 0.0 ? opts.cutoff_hz : 0.5 * (0.5 * band + dnyq);
        filter_taps = design_lowpass(cutoff_hz, fs, opts.num_taps == 0 ? 101 : opts.num_taps);
    }
    if (taps) {   // extension: explicit filter (e.g. the even 64-tap design of the cfg3 text)
        if (num_taps == 0) throw std::invalid_argument("zoom: empty filter");
        filter_taps.assign(taps, taps + num_taps);
    }
    group_delay_samples = 0.5 * static_cast<double>(filter_taps.size() - 1);
    usable_len = circular ? (in_len / decimation) * decimation : in_len;
    if (usable_len / decimation < 2)
        throw std::invalid_argument("make_zoom_plan: record too short for this decimation factor");
    if (circular && filter_taps.size() > usable_len)
        throw std::invalid_argument("make_zoom_plan: filter longer than the usable record");
    size_t block = usable_len / decimation;
    if (!circular && trim_transient) {
        trim_samples = (filter_taps.size() - 1 + decimation - 1) / decimation;
        if (trim_samples >= block)
            throw std::invalid_argument("make_zoom_plan: transient trim would consume the whole record");
        block -= trim_samples;
    }
    decimated_len = block;
    n_fft = pad_pow2 ? next_pow2(block) : block;
    if (n_fft_override) {
        if (n_fft_override < block) throw std::invalid_argument("zoom: n_fft shorter than the decimated block");
        n_fft = n_fft_override;
    }
    compute_band();
    if (!is_pow2(n_fft))   // dft_any's chirp route for the short transform (zoomfft.cpp:204-207)
        bluestein_ = std::make_unique<CztPlanG>(n_fft, cd(1.0, 0.0),
                                                cis_cycles(-1.0 / static_cast<double>(n_fft), 1.0), n_fft);
}

std::unique_ptr<ZoomPlanG> ZoomPlanG::from_fields(const ZoomFields& f) {
    std::unique_ptr<ZoomPlanG> p(new ZoomPlanG());
    p->f1_hz = f.f1_hz;
    p->f2_hz = f.f2_hz;
    p->center_hz = f.center_hz;
    p->sample_rate_hz = f.sample_rate_hz;
    p->cutoff_hz = f.cutoff_hz;
    p->decimation = f.decimation;
    p->filter_taps = f.filter_taps;
    p->group_delay_samples = f.group_delay_samples;
    p->circular = f.circular;
    p->trim_transient = f.trim_transient;
    p->pad_pow2 = f.pad_pow2;
    p->input_len = f.input_len;
    p->usable_len = f.usable_len;
    p->trim_samples = f.trim_samples;
    p->decimated_len = f.decimated_len;
    p->n_fft = f.n_fft;
    if (p->decimation == 0 || p->filter_taps.empty() || p->n_fft < p->decimated_len || p->decimated_len == 0)
        throw std::invalid_argument("zoom_fft: inconsistent plan fields");
    p->compute_band();
    if (!is_pow2(p->n_fft))
        p->bluestein_ = std::make_unique<CztPlanG>(p->n_fft, cd(1.0, 0.0),
                                                   cis_cycles(-1.0 / static_cast<double>(p->n_fft), 1.0), p->n_fft);
    return p;
}

// the frequency-domain route's conditions: circular, no trim, the whole record used, a power-of-two
// record, and the short FFT exactly the decimated length (no zero padding of u)
bool ZoomPlanG::spectral_route_ok() const {
    return circular && trim_samples == 0 && usable_len == input_len && is_pow2(usable_len) && decimation >= 1 &&
           is_pow2(n_fft) && n_fft * decimation == usable_len;
}

double ZoomPlanG::f_step_hz() const {   // zoomfft.cpp:11-13
    return sample_rate_hz / (static_cast<double>(decimation) * static_cast<double>(n_fft));
}

double ZoomPlanG::f_start_hz() const { return center_hz + static_cast<double>(k_lo) * f_step_hz(); }

void ZoomPlanG::compute_band() {   // zoomfft.cpp:209-219
    const double step = f_step_hz();
    const long n = static_cast<long>(n_fft);
    const double lo_idx = (f1_hz - center_hz) / step;
    const double hi_idx = (f2_hz - center_hz) / step;
    const double eps = 1e-9 * (1.0 + std::max(std::abs(lo_idx), std::abs(hi_idx)));
    k_lo = static_cast<long>(std::ceil(lo_idx - eps));
    k_hi = static_cast<long>(std::floor(hi_idx + eps));
    k_lo = std::max(k_lo, -(n / 2));
    k_hi = std::min(k_hi, n - 1 - n / 2);
    // an empty window is reported by execute, like zoom_fft (zoomfft.cpp:218-219)
}

namespace {
ZoomArgs make_args(const ZoomPlanG& p) {
    ZoomArgs a{};
    const int D = static_cast<int>(p.decimation);
    const int T = static_cast<int>(p.filter_taps.size());
    a.n = static_cast<long long>(p.input_len);
    a.U = static_cast<long long>(p.usable_len);
    a.D = D;
    a.T = T;
    a.nout = static_cast<int>(p.decimated_len);
    a.trim = static_cast<int>(p.trim_samples);
    const int per_row = (T + D - 1) / D;
    a.lh = (per_row + kZoomK - 1) / kZoomK * kZoomK;
    a.pre = a.lh + kZoomK;
    a.rowlen = static_cast<int>((p.usable_len + p.decimation - 1) / p.decimation) + 2 * kZoomK;
    int rs = (a.pre + a.rowlen) + (a.pre + a.rowlen) / kZoomK + 1;
    if ((rs & 1) == 0) ++rs;
    a.rs = rs;
    a.k_lo = static_cast<int>(p.k_lo);
    a.nbins = static_cast<int>(p.k_hi - p.k_lo + 1);
    a.mwrap = (p.circular && T >= 2) ? (T - 2) / D + 1 : 0;
    a.circular = p.circular ? 1 : 0;
    const cd w = cis_cycles(-p.center_hz / p.sample_rate_hz, static_cast<double>(p.usable_len));
    a.wre = w.real();
    a.wim = w.imag();
    return a;
}
}  // namespace

const ZoomPlanG::Dev& ZoomPlanG::dev(bool f32) const {
    require_device();
    return devs_.get(f32, [&](Dev& d) {
        const ZoomArgs a = make_args(*this);
        const double qc = -center_hz / sample_rate_hz;   // zoomfft.cpp:174
        const int D = a.D, T = a.T;
        // taps by phase row: g[t] = h[t] e^{-i 2pi qc t}, row ph holds t = l D + (D - ph) % D
        std::vector<cd> g(static_cast<size_t>(D) * a.lh, cd(0.0, 0.0));
        for (int ph = 0; ph < D; ++ph) {
            const int t0 = (D - ph) % D;
            for (int l = 0; l < a.lh; ++l) {
                const int t = l * D + t0;
                if (t < T) g[static_cast<size_t>(ph) * a.lh + l] = filter_taps[t] * cis_cycles(-qc, static_cast<double>(t));
            }
        }
        d.g = to_device(g, f32);
        d.gh = g;
        std::vector<cd> gn(static_cast<size_t>(std::max(T, 1)), cd(0.0, 0.0));   // natural order (wrap terms)
        for (int t = 0; t < T; ++t) gn[static_cast<size_t>(t)] = filter_taps[t] * cis_cycles(-qc, static_cast<double>(t));
        d.gn = to_device(gn, f32);
        d.gnh = gn;
        // S[m] = e^{i 2pi qc (m + trim) D} (the shift table sampled at the decimation points)
        std::vector<cd> S(decimated_len);
        for (size_t m = 0; m < decimated_len; ++m)
            S[m] = cis_cycles(qc, static_cast<double>((m + trim_samples) * decimation));
        d.sdec = to_device(S, f32);
        // band: D e^{i 2pi k delay / (D n_fft)} (zoomfft.cpp:223-234)
        const double delay = group_delay_samples + static_cast<double>(trim_samples * decimation);
        const double q = delay / (static_cast<double>(decimation) * static_cast<double>(n_fft));
        std::vector<cd> band(static_cast<size_t>(std::max<long>(0, k_hi - k_lo + 1)));
        for (long k = k_lo; k <= k_hi; ++k)
            band[static_cast<size_t>(k - k_lo)] = static_cast<double>(decimation) * cis_cycles(q, static_cast<double>(k));
        d.band = to_device(band.empty() ? std::vector<cd>{cd(0, 0)} : band, f32);
        // frequency-domain route tables (circular, untrimmed, n_fft = U / D, U a power of two)
        if (spectral_route_ok()) {
            const size_t U = usable_len;
            std::vector<cd> sh(U), hf(U, cd(0.0, 0.0));
            for (size_t n = 0; n < U; ++n) sh[n] = cis_cycles(qc, static_cast<double>(n));   // zoomfft.cpp:174-177
            // H[k] = sum_t h[t] e^{-i 2pi t k / U}, the exponent reduced exactly mod U
            for (size_t k = 0; k < U; ++k) {
                cd acc(0.0, 0.0);
                for (int t = 0; t < T; ++t)
                    acc += filter_taps[t] * cis_cycles(-1.0 / static_cast<double>(U),
                                                       static_cast<double>((static_cast<size_t>(t) * k) % U));
                hf[k] = acc;
            }
            d.shift = to_device(sh, f32);
            d.hf = to_device(hf, f32);
        }
    });
}

void ZoomPlanG::execute(const void* x, long long x_stride, long long batch, void* out, long long out_stride,
                        bool f32, cudaStream_t st) const {
    if (k_lo > k_hi) throw std::invalid_argument("zoom_fft: no transform bins fall inside the band");
    if (batch <= 0) return;
    const Dev& d = dev(f32);
    const ZoomArgs a = make_args(*this);
    const int lg = ilog2(n_fft);
    int dev_id = current_device();
    int smem_max = 0;
    check(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev_id), "attr");
    // SKG_ZOOM_PATH=fused|unfused forces a route (A/B measurements); the default is the split route
    static const char* force = getenv("SKG_ZOOM_PATH");
    const bool single = is_pow2(n_fft) && lg <= single_cta_max_log2(f32);
    const bool wfir = zoom_wfir_fits(a, f32, x, x_stride);
    static const bool no_pfir = getenv("SKG_ZOOM_NO_PFIR") != nullptr;
    const bool pfir = !no_pfir && zoom_pfir_lh(a) > 0;
    static const bool no_cfir = getenv("SKG_ZOOM_NO_CFIR") != nullptr;
    const bool cfir = !no_cfir && zoom_cfir_available(a);
    static const bool split_only = getenv("SKG_ZOOM_SPLIT") != nullptr;   // A/B: the two-kernel route
    static const bool no_spec = getenv("SKG_ZOOM_NO_SPEC") != nullptr;
    // circular, n_fft = U / D, long phase rows: FIR + decimation + short FFT as ONE U-point transform
    // (an exact rewrite, kernels_zoom_spec.cu). Measured against the FIR routes: 2x faster at 101 taps,
    // D = 4 (26 taps per phase row: fp64 0.40 -> 0.19-0.22 ms, fp32 0.50 -> 0.21-0.31 ms per 256 MiB),
    // slower with short rows (cfg3, 9 taps per row: 0.095 -> 0.119 ms; D = 16, 7 per row: 0.14 -> 0.23
    // ms), so it takes over above 12 taps per phase row (SKG_ZOOM_NO_SPEC=1: never)
    const size_t taps_per_row = (filter_taps.size() + decimation - 1) / decimation;
    if (!force && !split_only && !no_pfir && !no_cfir && !no_spec && spectral_route_ok() && taps_per_row > 12 &&
        ilog2(usable_len) <= single_cta_max_log2(f32) && ilog2(usable_len) >= 8) {
        check(launch_zoom_spec(ilog2(usable_len), f32, x, x_stride, batch, stockham_twiddles(ilog2(usable_len), f32),
                               d.shift.p, d.hf.p, (int)n_fft, (int)decimation, (int)k_lo, (int)bins(), d.band.p, out,
                               out_stride, st),
              "zoom spectral");
        count_launch();
        return;
    }
    // split route FIR: the TMA-fed phase-lane FIR where it fits (fp64 cfg3 n_fft 2048: 0.111 ms against
    // 0.120 for the whole-output FIR + separate transform), else the whole-output FIR
    // D in {4, 16} with 101 taps: whole outputs per lane from a raw shared-memory window (kernels_zoom_rfir.cu)
    const bool rfir = zoom_rfir_fits(a, f32, x, x_stride);
    const bool tfir = !rfir && zoom_tfir_fits(a, f32, x, x_stride);
    const bool pcfir = !rfir && !tfir && zoom_pcfir_fits(a, f32);
    if (!force && !split_only && zoom_pcfir_fused_fits(a, f32, lg)) {
        // whole-output FIR + 512-point transform + band in one launch (kernels_zoom_pcfir.cu)
        check(launch_zoom_pcfir(a, f32, x, x_stride, batch, d.gnh.data(), d.sdec.p, nullptr, 0, true,
                                stockham_twiddles(lg, f32), d.band.p, out, out_stride, st),
              "zoom fir+fft");
        count_launch();
        return;
    }
    if (!force && !split_only && rfir && zoom_rfir_fft_fits(a, f32, lg)) {
        // raw-window FIR + n_fft 2048 transform + band in one launch (kernels_zoom_rfir.cu)
        check(launch_zoom_rfir_fft(a, f32, lg, x, x_stride, batch, d.gnh.data(), d.sdec.p, stockham_twiddles(lg, f32),
                                   d.band.p, out, out_stride, st),
              "zoom fir+fft");
        count_launch();
        return;
    }
    if (single && pfir && !rfir && !tfir && !pcfir && !force && !split_only) {
        // FIR and short FFT in one kernel where instantiated (configs[2] geometry)
        const cudaError_t e = launch_zoom_pfir_fft(a, zoom_pfir_lh(a), lg, f32, x, x_stride, batch, d.g.p, d.gn.p,
                                                   d.sdec.p, stockham_twiddles(lg, f32), (int)k_lo, (int)bins(),
                                                   d.band.p, out, out_stride, st);
        if (e != cudaErrorNotSupported) {
            check(e, "zoom fir+fft");
            count_launch();
            return;
        }
    }
    if (single && (rfir || pcfir || tfir || wfir || pfir || cfir) && !force) {
        // warp-chunk FIR -> work rows (L2-resident chunk of records) -> FFT + band gather
        const size_t cs = f32 ? 8 : 16, es = f32 ? 4 : 8;
        const long long zrow = a.nout;
        const long long chunk = std::max<long long>(1, (48ll << 20) / (zrow * (long long)cs));
        const long long nb0 = std::min(chunk, batch);
        void* zb = nullptr;
        zb = stream_alloc((size_t)nb0 * zrow * cs, st);
        const void* tw = stockham_twiddles(lg, f32);
        for (long long b0 = 0; b0 < batch; b0 += chunk) {
            const long long nb = std::min(chunk, batch - b0);
            const void* xb = static_cast<const char*>(x) + b0 * x_stride * (long long)es;
            // phase-lane FIR where it exists (power-of-two D <= 16), else the constant-bank FIR for the
            // specialised (D, T) pairs, else the warp-window FIR (all three measured within a few
            // percent of each other on cfg3)
            if (rfir)
                check(launch_zoom_rfir(a, f32, xb, x_stride, nb, d.gnh.data(), d.gn.p, d.sdec.p, zb, zrow, st), "zoom fir");
            else if (pcfir)
                check(launch_zoom_pcfir(a, f32, xb, x_stride, nb, d.gnh.data(), d.sdec.p, zb, zrow, false, nullptr,
                                        nullptr, nullptr, 0, st),
                      "zoom fir");
            else if (tfir)
                check(launch_zoom_tfir(a, f32, xb, x_stride, nb, d.g.p, d.gn.p, d.sdec.p, zb, zrow, st), "zoom fir");
            else if (pfir)
                check(launch_zoom_pfir(a, f32, xb, x_stride, nb, d.g.p, d.gn.p, d.sdec.p, zb, zrow, st), "zoom fir");
            else if (cfir)
                check(launch_zoom_cfir(a, f32, xb, x_stride, nb, d.gh.data(), d.gn.p, d.sdec.p, zb, zrow, st),
                      "zoom fir");
            else
                check(launch_zoom_wfir(a, f32, xb, x_stride, nb, d.g.p, d.sdec.p, zb, zrow, st), "zoom fir");
            check(launch_zoom_fftband(lg, f32, zb, zrow, a.nout, nb, (int)k_lo, (int)bins(), tw, d.band.p,
                                      static_cast<char*>(out) + b0 * out_stride * (long long)cs, out_stride, st),
                  "zoom fft+band");
            count_launch(2);
        }
        check(cudaFreeAsync(zb, st), "free");
        return;
    }
    const bool fused = !(force && std::string(force) == "unfused") && single &&
                       zoom_smem_bytes(a, lg, f32) <= static_cast<size_t>(smem_max);
    if (!fused) {
        // FIR/decimate by output chunks -> work buffer (zero padded to n_fft) -> FFT -> band gather
        ZoomArgs c = a;
        c.rowlen = zoom_chunk_rowlen(a);
        int rs = c.rowlen + c.rowlen / kZoomK + 1;
        if ((rs & 1) == 0) ++rs;
        c.rs = rs;
        const size_t cs = f32 ? 8 : 16;
        void* zb = nullptr;
        zb = stream_alloc((size_t)batch * n_fft * cs, st);
        // the FIR writes the first nout values of every row: only the zero padding behind them is cleared
        if ((size_t)a.nout < n_fft)
            check(cudaMemset2DAsync(static_cast<char*>(zb) + (size_t)a.nout * cs, n_fft * cs, 0,
                                    (n_fft - (size_t)a.nout) * cs, (size_t)batch, st),
                  "memset");
        if (rfir)
            check(launch_zoom_rfir(a, f32, x, x_stride, batch, d.gnh.data(), d.gn.p, d.sdec.p, zb, (long long)n_fft, st),
                  "zoom fir");
        else if (wfir)
            check(launch_zoom_wfir(a, f32, x, x_stride, batch, d.g.p, d.sdec.p, zb, (long long)n_fft, st), "zoom fir");
        else
            check(launch_zoom_fir(c, f32, x, x_stride, batch, d.g.p, d.sdec.p, zb, (long long)n_fft, st), "zoom fir");
        count_launch();
        if (is_pow2(n_fft)) {
            fft_c2c(n_fft, false, f32, zb, (long long)n_fft, zb, (long long)n_fft, batch, st);
        } else {   // dft_any's chirp route (zoomfft.cpp:204-207)
            void* zf = nullptr;
            zf = stream_alloc((size_t)batch * n_fft * cs, st);
            bluestein_->execute(zb, true, (long long)n_fft, batch, zf, (long long)n_fft, f32, st);
            check(cudaFreeAsync(zb, st), "free");
            zb = zf;
        }
        check(launch_zoom_band(f32, zb, (long long)n_fft, (long long)n_fft, (int)k_lo, (int)bins(), d.band.p, out,
                               out_stride, batch, st),
              "zoom band");
        count_launch();
        check(cudaFreeAsync(zb, st), "free");
        return;
    }
    const void* tw = stockham_twiddles(lg, f32);
    cudaError_t e = f32 ? launch_zoom_f32(a, lg, (const float*)x, x_stride, batch, d.g.p, d.sdec.p, tw, d.band.p,
                                          out, out_stride, st)
                        : launch_zoom_f64(a, lg, (const double*)x, x_stride, batch, d.g.p, d.sdec.p, tw, d.band.p,
                                          out, out_stride, st);
    check(e, "zoom launch");
    count_launch();
}

}  // namespace skg
