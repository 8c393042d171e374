// host.cpp — runtime, table builders and plan objects of the B200 spectral library.
#include "host.hpp"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <numbers>

#include "fft_device.cuh"

namespace skg {

// ---- errors / device -----------------------------------------------------------------------
void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();   // clear sticky-free errors so the next call can proceed
        throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    }
}

void require_device() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw CudaError(std::string("no CUDA device available (") +
                        (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                        "); the B200 spectral library has no CPU fallback");
    }
}

// Stream-ordered work buffers come from the device's default memory pool. Its release threshold is
// raised once per device so freed blocks stay cached in the pool: without it every synchronisation
// returns the memory to the driver and the next cudaMallocAsync re-maps it (hundreds of us).
void* stream_alloc(size_t bytes, cudaStream_t st) {
    static std::once_flag once[64];
    int dev = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    std::call_once(once[dev & 63], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = 8ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    });
    void* p = nullptr;
    check(cudaMallocAsync(&p, bytes, st), "cudaMallocAsync");
    return p;
}

int current_device() {
    int d = 0;
    check(cudaGetDevice(&d), "cudaGetDevice");
    return d;
}

std::atomic<unsigned>& grid_cap_ref() {
    static std::atomic<unsigned> c{0};
    return c;
}
unsigned grid_cap() { return grid_cap_ref().load(std::memory_order_relaxed); }

std::atomic<uint64_t>& launch_counter() {
    static std::atomic<uint64_t> c{0};
    return c;
}

// ---- numerics ---------------------------------------------------------------------------------
bool is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }

size_t next_pow2(size_t n) {
    if (n == 0) throw std::invalid_argument("next_pow2: n must be >= 1");
    size_t p = 1;
    while (p < n) {
        if (p > (size_t{1} << 62)) throw std::invalid_argument("next_pow2: overflow");
        p <<= 1;
    }
    return p;
}

int ilog2(size_t n) {
    int l = 0;
    while ((size_t{1} << l) < n) ++l;
    return l;
}

// exp(i 2 pi q t) with q*t reduced by an fma split (numerics.cpp:122-128)
cd cis_cycles(double q, double t) {
    const double hi = q * t;
    const double lo = std::fma(q, t, -hi);
    const double frac = (hi - std::nearbyint(hi)) + lo;
    const double ang = 2.0 * std::numbers::pi * frac;
    return {std::cos(ang), std::sin(ang)};
}

PolarPow::PolarPow(cd z) {
    const double mag = std::abs(z);
    if (!(mag > 0.0)) throw std::invalid_argument("czt: parameter magnitude is zero");
    log_mag = std::log(mag);
    if (std::abs(log_mag) < 1e-14) log_mag = 0.0;
    q = std::arg(z) / (2.0 * std::numbers::pi);
}

cd PolarPow::pow(double t) const {
    cd u = cis_cycles(q, t);
    if (log_mag != 0.0) u *= std::exp(log_mag * t);
    return u;
}

std::vector<double> design_lowpass(double cutoff_hz, double fs, size_t num_taps) {
    if (!(fs > 0.0)) throw std::invalid_argument("design_lowpass: sample rate must be positive");
    if (!(cutoff_hz > 0.0) || cutoff_hz > fs / 2.0)
        throw std::invalid_argument("design_lowpass: cutoff must lie in (0, fs/2]");
    if (num_taps == 0 || num_taps % 2 == 0)
        throw std::invalid_argument("design_lowpass: tap count must be odd");
    if (num_taps == 1) return {1.0};
    const double fc = cutoff_hz / fs;
    const size_t mid = (num_taps - 1) / 2;
    std::vector<double> taps(num_taps);
    double sum = 0.0;
    for (size_t t = 0; t < num_taps; ++t) {
        const double k = static_cast<double>(t) - static_cast<double>(mid);
        const double arg = 2.0 * fc * k;
        const double sinc = k != 0.0 ? std::sin(std::numbers::pi * arg) / (std::numbers::pi * arg) : 1.0;
        const double win = 0.54 - 0.46 * std::cos(2.0 * std::numbers::pi * static_cast<double>(t) /
                                                   static_cast<double>(num_taps - 1));
        taps[t] = 2.0 * fc * sinc * win;
        sum += taps[t];
    }
    for (double& v : taps) v /= sum;
    return taps;
}

// ---- device memory ----------------------------------------------------------------------------
DevMem::DevMem(size_t n) : bytes(n) {
    if (n) check(cudaMalloc(&p, n), "cudaMalloc");
}
DevMem& DevMem::operator=(DevMem&& o) noexcept {
    if (this != &o) {
        if (p) cudaFree(p);
        p = o.p;
        bytes = o.bytes;
        o.p = nullptr;
        o.bytes = 0;
    }
    return *this;
}
DevMem::~DevMem() {
    if (p) cudaFree(p);
}
void DevMem::upload(const void* host, size_t n, cudaStream_t st) {
    check(cudaMemcpyAsync(p, host, n, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync H2D");
    check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
}

DevMem to_device(const std::vector<cd>& h, bool f32) {
    if (!f32) {
        DevMem d(h.size() * sizeof(cd));
        d.upload(h.data(), d.bytes);
        return d;
    }
    std::vector<float> f(2 * h.size());
    for (size_t i = 0; i < h.size(); ++i) {
        f[2 * i] = static_cast<float>(h[i].real());
        f[2 * i + 1] = static_cast<float>(h[i].imag());
    }
    DevMem d(f.size() * sizeof(float));
    d.upload(f.data(), d.bytes);
    return d;
}

namespace {
std::mutex g_tab_mu;
std::map<std::tuple<int, int, int, int>, DevMem>& tab_cache() {
    static std::map<std::tuple<int, int, int, int>, DevMem> m;
    return m;
}

template <int LG> void stockham_host(std::vector<cd>& out) {
    using G = FftGeom<LG>;
    out.assign(G::TW_ALLOC, cd(1.0, 0.0));
    if constexpr (G::L >= 16) {
        for (int s = 1; s < G::P; ++s) {
            const int R = G::radix(s);
            for (int d = 0; d < G::digits(s); ++d) {
                // digit d of k carries weight 16^d: W_{pR}^{kd 16^d} = W_{M}^{kd}, M = p R / 16^d
                const double M = static_cast<double>(G::pval(s)) * R / static_cast<double>(1 << (4 * d));
                const double q = -1.0 / M;   // exact power of two
                for (int jj = 0; jj < 4; ++jj)
                    for (int kd = 0; kd < 16; ++kd)
                        out[G::tw_off(s, d) + jj * 16 + kd] = cis_cycles(q, static_cast<double>((1 << jj) * kd));
            }
        }
    }
}

template <int LO, int HI> void stockham_dispatch(int lg, std::vector<cd>& out) {
    if constexpr (LO <= HI) {
        if (lg == LO) return stockham_host<LO>(out);
        stockham_dispatch<LO + 1, HI>(lg, out);
    }
}

const void* cached(int kind, int a, int b, bool f32, const std::function<std::vector<cd>()>& build) {
    std::lock_guard<std::mutex> lk(g_tab_mu);
    const auto key = std::make_tuple(current_device(), kind * 4096 + a * 64 + b, f32 ? 1 : 0, 0);
    auto it = tab_cache().find(key);
    if (it != tab_cache().end()) return it->second.p;
    DevMem d = to_device(build(), f32);
    const void* p = d.p;
    tab_cache().emplace(key, std::move(d));
    return p;
}
}  // namespace

int single_cta_max_log2(bool f32) { return f32 ? kMaxLog2F32 : kMaxLog2F64; }

// W_L^{j k}, k < L/16, j < 16 (row k): the last radix-16 Stockham pass's twiddles per butterfly,
// with the reference's phase reduction (numerics.cpp:122-128); read once per CTA into TMEM
const void* last_pass_twiddles(int log2L, bool f32) {
    require_device();
    return cached(5, log2L, 0, f32, [&] {
        const size_t L = size_t{1} << log2L, P = L / 16;
        std::vector<cd> v(L);
        const double q = -1.0 / static_cast<double>(L);
        for (size_t k = 0; k < P; ++k)
            for (size_t j = 0; j < 16; ++j) v[k * 16 + j] = cis_cycles(q, static_cast<double>(j * k));
        return v;
    });
}

namespace {
// W_L^{r k2}, r < 8, k2 < L/8: the cluster FFT's inter-CTA twiddles (fp64 phase reduction)
const void* cluster_twiddles(int log2L, bool f32) {
    require_device();
    return cached(4, log2L, 0, f32, [&] {
        const size_t L = size_t{1} << log2L, Q = L / 8;
        std::vector<cd> v(L);
        const double q = -1.0 / static_cast<double>(L);
        for (size_t r = 0; r < 8; ++r)
            for (size_t k = 0; k < Q; ++k) v[r * Q + k] = cis_cycles(q, static_cast<double>(r * k));
        return v;
    });
}
// opt-in (SKG_CLUSTER=1): measured slower than the four-step passes on B200 (fp64 L = 2^15: 7.5 vs
// 6.7 ms, 2^16: 10.6 vs 6.9 ms per 1 GiB batch; fp32 2^16 equal) — the per-SM Q-point FFTs run at
// 1-2 CTAs per SM and stall on the exchange; kept, tested, for the packed / multi-trace follow-up
bool cluster_enabled(int log2L, bool f32) {
    const char* e = getenv("SKG_CLUSTER");   // read per call so tests can switch paths in-process
    return e && e[0] == '1' && cluster_fft_log2q(log2L, f32) > 0;
}
// one L-point transform per 8-CTA cluster (kernels_cluster.cu); in_kind 0 complex, 1 real rows
void fft_cluster(int lg, bool f32, bool inverse, int mode, const void* x, int in_kind, long long x_stride,
                 long long N, long long batch, void* out, long long out_stride, cudaStream_t st) {
    const int lq = cluster_fft_log2q(lg, f32);
    check(launch_fft_cluster(lg, f32, inverse, mode, x, in_kind, x_stride, N, batch, stockham_twiddles(lq, f32),
                             cluster_twiddles(lg, f32), out, out_stride,
                             inverse ? 1.0 / static_cast<double>(size_t{1} << lg) : 1.0, st),
          "cluster fft launch");
    count_launch();
}
}  // namespace

const void* stockham_twiddles(int log2L, bool f32) {
    require_device();
    return cached(1, log2L, 0, f32, [&] {
        std::vector<cd> v;
        stockham_dispatch<0, kMaxLog2F32>(log2L, v);
        return v;
    });
}

const void* r2c_post_twiddles(int log2M, bool f32) {
    require_device();
    return cached(2, log2M, 0, f32, [&] {
        const size_t M = size_t{1} << log2M;
        std::vector<cd> v(M);
        const double q = -1.0 / (2.0 * static_cast<double>(M));
        // stored as W^k / 2: the split's 1/2 rides on the table (a power-of-two scale, exact)
        for (size_t k = 0; k < M; ++k) v[k] = 0.5 * cis_cycles(q, static_cast<double>(k));
        return v;
    });
}

const void* fourstep_twiddles(int log2R, int log2C, bool f32) {
    require_device();
    return cached(3, log2R, log2C, f32, [&] {
        const size_t R = size_t{1} << log2R, C = size_t{1} << log2C;
        std::vector<cd> v(R * C);
        const double q = -1.0 / static_cast<double>(R * C);
        for (size_t r = 0; r < R; ++r)
            for (size_t c = 0; c < C; ++c) v[r * C + c] = cis_cycles(q, static_cast<double>(r * c));
        return v;
    });
}

// ---- four-step plumbing -------------------------------------------------------------------------
namespace {
struct FourStep {
    int lR, lC;
    long long L;
    const void *twR, *twC, *twL;
    FourStep(int log2L, bool f32) {
        lR = log2L / 2;
        lC = log2L - lR;
        if (lC > 10 || lR < 4)
            throw std::invalid_argument("fft: length 2^" + std::to_string(log2L) + " exceeds the supported maximum 2^20");
        L = 1LL << log2L;
        twR = stockham_twiddles(lR, f32);
        twC = stockham_twiddles(lC, f32);
        twL = fourstep_twiddles(lR, lC, f32);
    }
    // traces per launch pair. Chunking to keep the work buffer L2 resident was measured SLOWER at every
    // size (configs[4] rows, 4 MB .. 4 GB chunks: the pass kernels are latency bound and a bigger grid
    // amortises their ramp/tail better than L2 residency saves), so the chunk only caps the work
    // buffer at 2 GB.
    long long chunk(bool f32) const {
        const long long bytes = L * (f32 ? 8 : 16);
        const char* e = std::getenv("SKG_4STEP_CHUNK_MB");
        const long long mb = e ? std::atoll(e) : 2048;
        return std::max<long long>(1, (mb << 20) / bytes);
    }
};

struct Scratch {   // stream-ordered work buffer
    void* p = nullptr;
    cudaStream_t st;
    Scratch(size_t bytes, cudaStream_t s) : st(s) { p = stream_alloc(bytes, s); }
    ~Scratch() {
        if (p) cudaFreeAsync(p, st);
    }
};

template <typename T>
void c2c_4step(const FourStep& f, bool inverse, int in_kind, const void* in, long long in_stride, long long N, void* out,
               long long out_stride, long long batch, cudaStream_t st) {
    const long long ch = f.chunk(sizeof(T) == 4);
    Scratch Y((size_t)std::min(ch, batch) * f.L * 2 * sizeof(T), st);
    const T scale = inverse ? (T)(1.0 / (double)f.L) : (T)1;
    for (long long b0 = 0; b0 < batch; b0 += ch) {
        const long long nb = std::min(ch, batch - b0);
        const size_t es = in_kind == 1 ? sizeof(T) : 2 * sizeof(T);
        const void* src = static_cast<const char*>(in) + (size_t)b0 * in_stride * es;
        void* dst = static_cast<char*>(out) + (size_t)b0 * out_stride * 2 * sizeof(T);
        check(launch_4step_col<T>(f.lR, false, in_kind, inverse ? 1 : 0, src, in_stride, N, nullptr, Y.p, f.lC, nb,
                                  f.twR, f.twL, 0, nullptr, 0, 0, nullptr, (T)1, 0, st),
              "4step col");
        check(launch_4step_row<T>(f.lC, 0, Y.p, f.lR, nb, f.twC, f.twL, nullptr, dst, out_stride, scale,
                                  inverse ? 1 : 0, st),
              "4step row");
        count_launch(2);
    }
}

// Real traces: Hermitian-half four-step (kernels_4step_real.cuh) — column pairs ride one complex column
// transform, only the work rows k1 <= R/2 exist, the row pass stores each bin and its mirror.
// layout 0: L bins, 1: L/2 + 1 bins. SKG_4STEP_REAL=0 selects the complex four-step (A/B).
bool r2c_4step_enabled(const FourStep& f, bool f32) {
    const char* e = std::getenv("SKG_4STEP_REAL");
    if (e && e[0] == '0') return false;
    return (1LL << f.lC) >= 2 * (f32 ? 16 : 8);
}
// One cooperative persistent launch for both passes with the work rows in an L2-resident ring (square
// factorisations R = C, batches of at least a few grids of units; same arithmetic as the two launches, so
// the results are identical bit for bit). SKG_4STEP_FUSED=0 disables it; SKG_4STEP_DELTA_X10 scales the
// look-ahead (tenths of a grid of units, default 25).
template <typename T>
bool r2c_4step_fused(const FourStep& f, const void* in, long long in_stride, long long N, void* out,
                     long long out_stride, int layout, long long batch, cudaStream_t st) {
    const char* e = std::getenv("SKG_4STEP_FUSED");
    if (e && e[0] == '0') return false;
    if (f.lR != f.lC || f.lR < 8 || f.lR > 9) return false;
    int grid = 0, ups = 0;
    if (launch_4step_rfused<T>(f.lR, in, in_stride, N, nullptr, 1, 1, batch, f.twR, f.twL, out, out_stride, layout,
                               nullptr, nullptr, &grid, &ups, st) != cudaSuccess || grid <= 0 || ups <= 0) {
        cudaGetLastError();
        return false;
    }
    const char* dx = std::getenv("SKG_4STEP_DELTA_X10");
    const long long x10 = dx ? std::max(1, std::atoi(dx)) : 25;
    const long long delta = std::max<long long>(2, (grid * x10 / 10 + ups - 1) / ups);
    // column start .. row units read; a ring twice as long measured slower (it spills from L2):
    // FFT 2^16 fp64 3.28 -> 3.53 ms
    const long long slots = delta + (grid + ups - 1) / ups + 2;
    if (batch < slots) return false;   // short batches: the two launches
    const long long rows = (1LL << f.lR) / 2 + 1, Cn = 1LL << f.lC;
    Scratch Y((size_t)slots * rows * Cn * 2 * sizeof(T), st);
    Scratch cnt((size_t)batch * 2 * sizeof(unsigned), st);
    check(cudaMemsetAsync(cnt.p, 0, (size_t)batch * 2 * sizeof(unsigned), st), "4step fused counters");
    unsigned* col_done = static_cast<unsigned*>(cnt.p);
    if (launch_4step_rfused<T>(f.lR, in, in_stride, N, Y.p, (int)slots, (int)delta, batch, f.twR, f.twL, out, out_stride,
                               layout, col_done, col_done + batch, nullptr, nullptr, st) != cudaSuccess) {
        cudaGetLastError();   // no cooperative launch here (e.g. the grid cannot be co-resident): the two launches
        return false;
    }
    count_launch();
    return true;
}
template <typename T>
void r2c_4step(const FourStep& f, const void* in, long long in_stride, long long N, void* out, long long out_stride,
               int layout, long long batch, cudaStream_t st) {
    if (r2c_4step_fused<T>(f, in, in_stride, N, out, out_stride, layout, batch, st)) return;
    const long long rows = (1LL << f.lR) / 2 + 1, Cn = 1LL << f.lC;
    const long long per = rows * Cn * 2 * (long long)sizeof(T);
    const long long ch = std::max<long long>(1, std::min<long long>(batch, (2048LL << 20) / per));
    Scratch Y((size_t)ch * per, st);
    for (long long b0 = 0; b0 < batch; b0 += ch) {
        const long long nb = std::min(ch, batch - b0);
        const void* src = static_cast<const char*>(in) + (size_t)b0 * in_stride * sizeof(T);
        void* dst = static_cast<char*>(out) + (size_t)b0 * out_stride * 2 * sizeof(T);
        check(launch_4step_colr<T>(f.lR, src, in_stride, N, Y.p, f.lC, nb, f.twR, f.twL, st), "4step real col");
        check(launch_4step_rowh<T>(f.lC, Y.p, f.lR, nb, f.twC, dst, out_stride, layout, st), "4step real row");
        count_launch(2);
    }
}
}  // namespace

// ---- transforms -------------------------------------------------------------------------------
void fft_c2c(size_t n, bool inverse, bool f32, const void* in, long long in_stride, void* out,
             long long out_stride, long long batch, cudaStream_t st) {
    if (batch <= 0) return;
    const int lg = ilog2(n);
    if (lg > single_cta_max_log2(f32) && cluster_enabled(lg, f32)) {   // in place is safe: a trace is
        fft_cluster(lg, f32, inverse, 0, in, 0, in_stride, (long long)n, batch, out, out_stride, st);   // read before it is written
        return;
    }
    if (lg > single_cta_max_log2(f32)) {
        FourStep f(lg, f32);
        if (in == out) {   // the row pass scatters: stage through a copy for in-place calls
            Scratch tmp((size_t)batch * n * (f32 ? 8 : 16), st);
            check(cudaMemcpy2DAsync(tmp.p, n * (f32 ? 8 : 16), in, in_stride * (f32 ? 8 : 16), n * (f32 ? 8 : 16),
                                    batch, cudaMemcpyDeviceToDevice, st),
                  "copy");
            if (f32) c2c_4step<float>(f, inverse, 0, tmp.p, (long long)n, (long long)n, out, out_stride, batch, st);
            else c2c_4step<double>(f, inverse, 0, tmp.p, (long long)n, (long long)n, out, out_stride, batch, st);
            return;
        }
        if (f32) c2c_4step<float>(f, inverse, 0, in, in_stride, (long long)n, out, out_stride, batch, st);
        else c2c_4step<double>(f, inverse, 0, in, in_stride, (long long)n, out, out_stride, batch, st);
        return;
    }
    const void* tw = stockham_twiddles(lg, f32);
    cudaError_t e;
    if (f32)
        e = launch_fft_c2c<float>(lg, inverse, in, in_stride, out, out_stride, batch, tw,
                                  inverse ? 1.0f / static_cast<float>(n) : 1.0f, st);
    else
        e = launch_fft_c2c<double>(lg, inverse, in, in_stride, out, out_stride, batch, tw,
                                   inverse ? 1.0 / static_cast<double>(n) : 1.0, st);
    check(e, "fft_c2c launch");
    count_launch();
}

// ---- CZT ---------------------------------------------------------------------------------------
CztPlanG::CztPlanG(size_t n, cd a, cd w, size_t m) : n_(n), m_(m) {
    // czt.cpp:36-40, 78-82
    if (m == 0) throw std::invalid_argument("czt: m must be >= 1");
    if (!(std::abs(a) > 0.0) || !(std::abs(w) > 0.0))
        throw std::invalid_argument("czt: a and w must be nonzero");
    if (n == 0) throw std::invalid_argument("CztPlan: empty input length");
    L_ = next_pow2(n + m - 1);
    // Output segmentation: X[s M' + k'] for k' < M' is the chirp-z transform with start
    // A_s = A W^{-s M'} and the same W, so the m bins can run as S independent transforms of
    // length Ls = next_pow2(n + M' - 1) that share the kernel spectrum and the output chirp. Pick S
    // minimising S Ls log2 Ls (transforms that fit one CTA preferred): for configs[1]
    // (n=1024, m=2048) this is S=2, Ls=2048 — slightly less arithmetic than one 4096-point pair
    // and half the shared memory per CTA, i.e. twice the resident CTAs per SM.
    double best = 0.0;
    // SKG_CZT_SEGMENTS=<S> pins the segment count (tuning / A-B experiments)
    const char* env = std::getenv("SKG_CZT_SEGMENTS");
    const size_t forced = env ? static_cast<size_t>(std::strtoul(env, nullptr, 10)) : 0;
    for (size_t S = 1; S <= m; S *= 2) {
        if (forced && S != forced) {
            if (S > forced) break;
            continue;
        }
        const size_t seg = (m + S - 1) / S;
        const size_t Ls = next_pow2(n + seg - 1);
        double cost = static_cast<double>((m + seg - 1) / seg) * static_cast<double>(Ls) * ilog2(Ls);
        if (ilog2(Ls) > single_cta_max_log2(false)) cost *= 1.5;   // multi-pass: work buffer round trips
        if (S == 1 || forced || cost < best * 0.999) {
            best = cost;
            nseg_ = (m + seg - 1) / seg;
            seg_ = seg;
            Ls_ = Ls;
        }
        if (seg == 1) break;
    }
    log2L_ = ilog2(Ls_);
    if (log2L_ > 20)
        throw std::invalid_argument("czt: convolution length " + std::to_string(Ls_) +
                                    " exceeds the supported maximum 2^20");
    const PolarPow A(a), W(w);
    // czt.cpp:90-112, per segment: input chirp A^{-i} W^{i^2/2 + s M' i} (one fma-split phase)
    cin_.resize(nseg_ * n);
    for (size_t sg = 0; sg < nseg_; ++sg)
        for (size_t i = 0; i < n; ++i) {
            const double t = static_cast<double>(i);
            cin_[sg * n + i] = A.pow(-t) * W.pow(0.5 * t * t + static_cast<double>(sg * seg_) * t);
        }
    cout_.resize(seg_);
    for (size_t k = 0; k < seg_; ++k) {
        const double t = static_cast<double>(k);
        cout_[k] = W.pow(0.5 * t * t);
    }
    kern_.assign(Ls_, cd(0.0, 0.0));
    for (size_t k = 0; k < seg_; ++k) {
        const double t = static_cast<double>(k);
        kern_[k] = W.pow(-0.5 * t * t);
    }
    for (size_t i = 1; i < n; ++i) {
        const double t = static_cast<double>(i);
        kern_[Ls_ - i] = W.pow(-0.5 * t * t);
    }
    if (nseg_ > 1 && log2L_ <= single_cta_max_log2(false)) {
        // shared-forward form (kernels_impl.cuh k_czt_sf): block s convolves the segment-0 chirped
        // input with g_s[j] = W^{-(s M' + j)^2/2}, j in (-n, M'), and finishes with W^{(s M' + k)^2/2}
        kern_sf_.assign(nseg_ * Ls_, cd(0.0, 0.0));
        cout_sf_.assign(nseg_ * seg_, cd(0.0, 0.0));
        for (size_t sg = 0; sg < nseg_; ++sg) {
            const double k0 = static_cast<double>(sg * seg_);
            cd* kr = kern_sf_.data() + sg * Ls_;
            for (size_t j = 0; j < seg_; ++j) {
                const double t = k0 + static_cast<double>(j);
                kr[j] = W.pow(-0.5 * t * t);
                cout_sf_[sg * seg_ + j] = W.pow(0.5 * t * t);
            }
            for (size_t i = 1; i < n; ++i) {
                const double t = k0 - static_cast<double>(i);
                kr[Ls_ - i] = W.pow(-0.5 * t * t);
            }
        }
    }
}

const CztPlanG::Dev& CztPlanG::dev(bool f32) const {
    require_device();
    return devs_.get(f32, [&](Dev& d) {
        d.cin = to_device(cin_, f32);
        d.cout = to_device(cout_, f32);
        // kernel spectrum: forward FFT of the circular chirp on the GPU in fp64, scaled by 1/L so the
        // inverse transform of the fused kernel needs no extra pass (czt.cpp:113, numerics.cpp:93-96)
        DevMem k64 = to_device(kern_, false);
        fft_c2c(Ls_, false, false, k64.p, 0, k64.p, 0, 1, nullptr);
        check(launch_scale_c64(k64.p, (long long)Ls_, 1.0 / static_cast<double>(Ls_), nullptr), "scale");
        count_launch();
        if (log2L_ > single_cta_max_log2(f32)) {
            // four-step layout: khat_p[k1][k2] = khat[k1 + R k2]
            const int lR = log2L_ / 2, lC = log2L_ - lR;
            const size_t R = size_t{1} << lR, Cn = size_t{1} << lC;
            std::vector<cd> h(Ls_), p(Ls_);
            check(cudaMemcpy(h.data(), k64.p, Ls_ * sizeof(cd), cudaMemcpyDeviceToHost), "D2H khat");
            for (size_t k1 = 0; k1 < R; ++k1)
                for (size_t k2 = 0; k2 < Cn; ++k2) p[k1 * Cn + k2] = h[k1 + R * k2];
            k64.upload(p.data(), Ls_ * sizeof(cd));
        }
        if (f32) {
            DevMem k32(Ls_ * 2 * sizeof(float));
            check(launch_c64_to_c32(k64.p, k32.p, (long long)Ls_, nullptr), "convert");
            count_launch();
            d.khat = std::move(k32);
        } else {
            d.khat = std::move(k64);
        }
        if (!kern_sf_.empty()) {   // the per-block kernel spectra, same fp64 FFT + 1/L scale
            DevMem ks = to_device(kern_sf_, false);
            fft_c2c(Ls_, false, false, ks.p, (long long)Ls_, ks.p, (long long)Ls_, (long long)nseg_, nullptr);
            check(launch_scale_c64(ks.p, (long long)(nseg_ * Ls_), 1.0 / static_cast<double>(Ls_), nullptr), "scale");
            count_launch();
            if (f32) {
                DevMem k32(nseg_ * Ls_ * 2 * sizeof(float));
                check(launch_c64_to_c32(ks.p, k32.p, (long long)(nseg_ * Ls_), nullptr), "convert");
                count_launch();
                d.khat_sf = std::move(k32);
            } else {
                d.khat_sf = std::move(ks);
            }
            d.cout_sf = to_device(cout_sf_, f32);
        }
        check(cudaStreamSynchronize(nullptr), "czt plan upload");
    });
}

bool CztPlanG::czt_4step_fused(const FourStepRef& fr, bool f32, const void* x, bool complex_in, long long x_stride,
                               long long N, const Dev& d, long long batch, void* out, long long out_stride,
                               cudaStream_t st) const {
    const FourStep& f = *static_cast<const FourStep*>(fr.p);
    const char* e = std::getenv("SKG_4STEP_FUSED");
    if (e && e[0] == '0') return false;
    const size_t cs = f32 ? 8 : 16;
    auto call = [&](const void* cinp, void* yring, int slots, int delta, void* dst, long long mh, unsigned* cnt,
                    int* grid, int* ups) {
        return f32 ? launch_4step_czt_fused<float>(f.lR, f.lC, x, complex_in ? 1 : 0, x_stride, N, cinp, yring, slots,
                                                   delta, batch, f.twR, f.twC, f.twL, d.khat.p, dst, out_stride, mh,
                                                   d.cout.p, cnt, grid, ups, st)
                   : launch_4step_czt_fused<double>(f.lR, f.lC, x, complex_in ? 1 : 0, x_stride, N, cinp, yring, slots,
                                                    delta, batch, f.twR, f.twC, f.twL, d.khat.p, dst, out_stride, mh,
                                                    d.cout.p, cnt, grid, ups, st);
    };
    int grid = 0, ups = 0;
    if (call(nullptr, nullptr, 1, 1, nullptr, 0, nullptr, &grid, &ups) != cudaSuccess || grid <= 0 || ups <= 0) {
        cudaGetLastError();
        return false;
    }
    const char* dx = std::getenv("SKG_4STEP_DELTA_X10");
    const long long x10 = dx ? std::max(1, std::atoi(dx)) : 25;
    const long long delta = std::max<long long>(1, (grid * x10 / 10 + ups - 1) / ups);
    const long long slots = 2 * delta + (grid + ups - 1) / ups + 2;   // forward column start .. inverse column read
    const size_t ring = (size_t)slots * (size_t)f.L * cs;
    if (batch < slots || ring > (size_t{72} << 20)) return false;   // the ring has to stay L2 resident
    Scratch Y(ring, st);
    Scratch cnt((size_t)batch * 3 * sizeof(unsigned), st);
    for (size_t sg = 0; sg < nseg_; ++sg) {
        check(cudaMemsetAsync(cnt.p, 0, (size_t)batch * 3 * sizeof(unsigned), st), "czt fused counters");
        void* dst = static_cast<char*>(out) + sg * seg_ * cs;
        const void* cinp = static_cast<const char*>(d.cin.p) + sg * n_ * cs;
        const long long mh = (long long)std::min(seg_, m_ - sg * seg_);
        if (call(cinp, Y.p, (int)slots, (int)delta, dst, mh, static_cast<unsigned*>(cnt.p), nullptr, nullptr) !=
            cudaSuccess) {
            cudaGetLastError();
            if (sg == 0) return false;   // no cooperative launch here: the three launches
            throw std::runtime_error("czt 4step fused: launch failed");
        }
        count_launch();
    }
    return true;
}

void CztPlanG::execute(const void* x, bool complex_in, long long x_stride, long long batch, void* out,
                       long long out_stride, bool f32, cudaStream_t st, size_t load_n) const {
    if (batch <= 0) return;
    const Dev& d = dev(f32);
    const long long N = static_cast<long long>(load_n ? std::min(load_n, n_) : n_);
    if (log2L_ > single_cta_max_log2(f32)) {
        FourStep f(log2L_, f32);
        const long long ch = f.chunk(f32);
        const size_t cs = f32 ? 8 : 16, es = complex_in ? cs : cs / 2;
        Scratch Y((size_t)std::min(ch, batch) * f.L * cs, st);
        const int kind = complex_in ? 3 : 2;
        // one cooperative launch per segment with the work rows in an L2-resident ring (kernels_4step_czt.cuh);
        // same unit arithmetic as the three launches below, which serve short batches, rings that would not
        // fit in L2 and SKG_4STEP_FUSED=0
        if (czt_4step_fused(FourStepRef{&f}, f32, x, complex_in, x_stride, N, d, batch, out, out_stride, st)) return;
        for (long long b0 = 0; b0 < batch; b0 += ch) {
            const long long nb = std::min(ch, batch - b0);
            const void* src = static_cast<const char*>(x) + (size_t)b0 * x_stride * es;
            for (size_t sg = 0; sg < nseg_; ++sg) {
                void* dst = static_cast<char*>(out) + ((size_t)b0 * out_stride + sg * seg_) * cs;
                const void* cs_ = static_cast<const char*>(d.cin.p) + sg * n_ * cs;
                const long long mh = (long long)std::min(seg_, m_ - sg * seg_);
                cudaError_t e1, e2, e3;
                if (f32) {
                    e1 = launch_4step_col<float>(f.lR, false, kind, 0, src, x_stride, N, cs_, Y.p, f.lC, nb, f.twR,
                                                 f.twL, 0, nullptr, 0, 0, nullptr, 1.0f, 0, st);
                    e2 = launch_4step_row<float>(f.lC, 1, Y.p, f.lR, nb, f.twC, f.twL, d.khat.p, nullptr, 0, 1.0f, 0,
                                                 st);
                    e3 = launch_4step_col<float>(f.lR, true, 4, 0, nullptr, 0, 0, nullptr, Y.p, f.lC, nb, f.twR, f.twL,
                                                 1, dst, out_stride, mh, d.cout.p, 1.0f, 0, st);
                } else {
                    e1 = launch_4step_col<double>(f.lR, false, kind, 0, src, x_stride, N, cs_, Y.p, f.lC, nb, f.twR,
                                                  f.twL, 0, nullptr, 0, 0, nullptr, 1.0, 0, st);
                    e2 = launch_4step_row<double>(f.lC, 1, Y.p, f.lR, nb, f.twC, f.twL, d.khat.p, nullptr, 0, 1.0, 0,
                                                  st);
                    e3 = launch_4step_col<double>(f.lR, true, 4, 0, nullptr, 0, 0, nullptr, Y.p, f.lC, nb, f.twR, f.twL,
                                                  1, dst, out_stride, mh, d.cout.p, 1.0, 0, st);
                }
                check(e1, "czt 4step col");
                check(e2, "czt 4step row");
                check(e3, "czt 4step col inv");
                count_launch(3);
            }
        }
        return;
    }
    const void* tw = stockham_twiddles(log2L_, f32);
    cudaError_t e;
    static const bool no_sf = std::getenv("SKG_CZT_NO_SF") != nullptr;
    if (!kern_sf_.empty() && !no_sf) {
        // spectrum parking slots: one per transform group that can be resident (4 per SM)
        int sms = 0;
        check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device()), "attr");
        const long long slots = 4LL * sms;
        void* yw = stream_alloc((size_t)slots * Ls_ * (f32 ? 8 : 16), st);
        e = f32 ? launch_czt_sf<float>(log2L_, N, (long long)m_, complex_in, x, x_stride, batch, (int)nseg_,
                                       (long long)seg_, out, out_stride, tw, d.cin.p, d.khat_sf.p, d.cout_sf.p, yw,
                                       slots, last_pass_twiddles(log2L_, f32), st)
                : launch_czt_sf<double>(log2L_, N, (long long)m_, complex_in, x, x_stride, batch, (int)nseg_,
                                        (long long)seg_, out, out_stride, tw, d.cin.p, d.khat_sf.p, d.cout_sf.p, yw,
                                        slots, last_pass_twiddles(log2L_, f32), st);
        cudaFreeAsync(yw, st);
        if (e != cudaErrorNotSupported) {
            check(e, "czt launch");
            count_launch();
            return;
        }
        cudaGetLastError();
    }
    if (f32)
        e = launch_czt<float>(log2L_, N, (long long)m_, complex_in, x, x_stride, batch, (int)nseg_, (long long)seg_,
                              (long long)n_, out, out_stride, tw,
                              d.cin.p, d.khat.p, d.cout.p, st);
    else
        e = launch_czt<double>(log2L_, N, (long long)m_, complex_in, x, x_stride, batch, (int)nseg_,
                               (long long)seg_, (long long)n_, out, out_stride, tw,
                               d.cin.p, d.khat.p, d.cout.p, st);
    check(e, "czt launch");
    count_launch();
}

// ---- FFT spectrum -------------------------------------------------------------------------------
namespace {
std::mutex g_bluestein_mu;
std::map<size_t, std::unique_ptr<CztPlanG>>& bluestein_cache() {
    static std::map<size_t, std::unique_ptr<CztPlanG>> m;
    return m;
}
}  // namespace

// dft_any's chirp route for a non-power-of-two length (czt.cpp:144-153)
static const CztPlanG& bluestein_plan(size_t len) {
    std::lock_guard<std::mutex> lk(g_bluestein_mu);
    auto& m = bluestein_cache();
    auto it = m.find(len);
    if (it == m.end())
        it = m.emplace(len, std::make_unique<CztPlanG>(len, cd(1.0, 0.0),
                                                       cis_cycles(-1.0 / static_cast<double>(len), 1.0), len))
                 .first;
    return *it->second;
}

void fft_spectrum_batch(size_t n, size_t len, bool f32, int layout, const void* x, long long x_stride,
                        long long batch, void* out, long long out_stride, cudaStream_t st) {
    if (len == 0) len = next_pow2(n);
    if (len < n) throw std::invalid_argument("fft_spectrum: transform length shorter than the trace");
    if (batch <= 0) return;
    if (!is_pow2(len)) {
        if (layout != 0) throw std::invalid_argument("fft_spectrum: half layout needs a power-of-two length");
        bluestein_plan(len).execute(x, false, x_stride, batch, out, out_stride, f32, st, n);
        return;
    }
    if (len == 1) {
        // one bin: X[0] = x[0]
        const size_t es = f32 ? sizeof(float) : sizeof(double);
        check(cudaMemset2DAsync(out, out_stride * 2 * es, 0, 2 * es, batch, st), "memset");
        check(cudaMemcpy2DAsync(out, out_stride * 2 * es, x, x_stride * es, es, batch, cudaMemcpyDeviceToDevice, st),
              "copy");
        return;
    }
    const int lgM = ilog2(len) - 1;
    if (lgM > single_cta_max_log2(f32) && cluster_enabled(lgM + 1, f32)) {
        // one cluster per transform: complex FFT of the zero-padded real rows, full or half layout
        fft_cluster(lgM + 1, f32, false, layout == 0 ? 0 : 1, x, 1, x_stride, (long long)n, batch, out, out_stride, st);
        return;
    }
    if (lgM > single_cta_max_log2(f32)) {
        // multi-pass: complex FFT of the zero-padded real rows (imaginary part synthesised as 0)
        FourStep f(lgM + 1, f32);
        const size_t cs = f32 ? 8 : 16;
        if (r2c_4step_enabled(f, f32)) {
            if (f32) r2c_4step<float>(f, x, x_stride, (long long)n, out, out_stride, layout, batch, st);
            else r2c_4step<double>(f, x, x_stride, (long long)n, out, out_stride, layout, batch, st);
            return;
        }
        if (layout == 0) {
            if (f32) c2c_4step<float>(f, false, 1, x, x_stride, (long long)n, out, out_stride, batch, st);
            else c2c_4step<double>(f, false, 1, x, x_stride, (long long)n, out, out_stride, batch, st);
        } else {
            Scratch full((size_t)batch * len * cs, st);
            if (f32) c2c_4step<float>(f, false, 1, x, x_stride, (long long)n, full.p, (long long)len, batch, st);
            else c2c_4step<double>(f, false, 1, x, x_stride, (long long)n, full.p, (long long)len, batch, st);
            check(cudaMemcpy2DAsync(out, out_stride * cs, full.p, len * cs, (len / 2 + 1) * cs, batch,
                                    cudaMemcpyDeviceToDevice, st),
                  "half copy");
        }
        return;
    }
    const void* tw = stockham_twiddles(lgM, f32);
    const void* post = r2c_post_twiddles(lgM, f32);
    cudaError_t e;
    if (f32)
        e = launch_fft_r2c<float>(lgM, (long long)n, (const float*)x, x_stride, batch, tw, post, layout, out,
                                  out_stride, nullptr, nullptr, nullptr, 0, 0, 0, st);
    else
        e = launch_fft_r2c<double>(lgM, (long long)n, (const double*)x, x_stride, batch, tw, post, layout, out,
                                   out_stride, nullptr, nullptr, nullptr, 0, 0, 0, st);
    check(e, "fft_spectrum launch");
    count_launch();
}

// ---- band slice + magnitude_db ---------------------------------------------------------------------
BandBins slice_band_bins(size_t size, double f_start, double f_step, double f_lo, double f_hi) {
    // spectra.cpp:40-61, same checks in the same order
    if (size == 0) throw std::invalid_argument("slice_band: empty spectrum");
    if (!(f_step > 0.0)) throw std::invalid_argument("slice_band: non-positive step");
    if (!(f_lo <= f_hi)) throw std::invalid_argument("slice_band: inverted band");
    const double eps = 0.5 * f_step * 1e-9;
    const double lo = (f_lo - f_start) / f_step;
    const double hi = (f_hi - f_start) / f_step;
    const long k_lo = static_cast<long>(std::ceil(lo - eps));
    const long k_hi = static_cast<long>(std::floor(hi + eps));
    const long last = static_cast<long>(size) - 1;
    const long a = std::max(k_lo, 0L), b = std::min(k_hi, last);
    if (a > b) throw std::invalid_argument("slice_band: no bins fall inside the requested band");
    BandBins r;
    r.k_lo = a;
    r.count = b - a + 1;
    r.f_start = f_start + static_cast<double>(a) * f_step;   // Spectrum::frequency(a)
    return r;
}

void band_db_batch(bool f32, const void* in, long long in_stride, long long k_lo, long long count, long long batch,
                   void* out, long long out_stride, void* db, long long db_stride, cudaStream_t st) {
    if (batch <= 0 || count <= 0 || (!out && !db)) return;
    check(launch_band_db(f32, in, in_stride, k_lo, count, batch, out, out_stride, db, db_stride, st), "band launch");
    count_launch();
}

void fft_spectrum_band_batch(size_t n, size_t len, bool f32, long long k_lo, long long count, const void* x,
                             long long x_stride, long long batch, void* out, long long out_stride, void* db,
                             long long db_stride, cudaStream_t st) {
    if (len == 0) len = next_pow2(n);
    if (len < n) throw std::invalid_argument("fft_spectrum: transform length shorter than the trace");
    if (k_lo < 0 || count <= 0 || (size_t)(k_lo + count) > len)
        throw std::invalid_argument("fft_spectrum_band: band outside the spectrum");
    if (batch <= 0 || (!out && !db)) return;
    const int lgM = is_pow2(len) && len >= 2 ? ilog2(len) - 1 : -1;
    if (lgM >= 0 && lgM <= single_cta_max_log2(f32)) {
        // fused: the FFT store epilogue writes only the band (and its dB column)
        const void* tw = stockham_twiddles(lgM, f32);
        const void* post = r2c_post_twiddles(lgM, f32);
        cudaError_t e;
        if (f32)
            e = launch_fft_r2c<float>(lgM, (long long)n, (const float*)x, x_stride, batch, tw, post, 3, out,
                                      out_stride, nullptr, (float*)db, nullptr, db_stride, k_lo, k_lo + count - 1, st);
        else
            e = launch_fft_r2c<double>(lgM, (long long)n, (const double*)x, x_stride, batch, tw, post, 3, out,
                                       out_stride, nullptr, (double*)db, nullptr, db_stride, k_lo, k_lo + count - 1,
                                       st);
        check(e, "fft_spectrum_band launch");
        count_launch();
        return;
    }
    // multi-pass / chirp routes: full spectrum into a work buffer, then the band pass
    const size_t cs = f32 ? 8 : 16;
    Scratch full((size_t)batch * len * cs, st);
    fft_spectrum_batch(n, len, f32, 0, x, x_stride, batch, full.p, (long long)len, st);
    band_db_batch(f32, full.p, (long long)len, k_lo, count, batch, out, out_stride, db, db_stride, st);
}

// ---- transfer function ---------------------------------------------------------------------------
TransferPlanG::TransferPlanG(const double* ref, size_t n, size_t len, bool f32) : n_(n), f32_(f32) {
    if (n == 0) throw std::invalid_argument("transfer: empty reference trace");
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(ref[i])) throw std::invalid_argument("trace: non-finite sample");
    len_ = len == 0 ? next_pow2(n) : len;
    if (len_ < n) throw std::invalid_argument("fft_spectrum: transform length shorter than the trace");
    if (!is_pow2(len_) || len_ < 2)
        throw std::invalid_argument("transfer: transform length must be a power of two >= 2");
    require_device();
    // X_ref on the GPU in fp64 (the fused epilogue multiplies by 1/X_ref)
    DevMem dref(n * sizeof(double));
    dref.upload(ref, n * sizeof(double));
    DevMem dx(bins() * sizeof(cd));
    fft_spectrum_batch(n, len_, false, 1, dref.p, 0, 1, dx.p, 0, nullptr);
    xref_.resize(bins());
    check(cudaMemcpy(xref_.data(), dx.p, bins() * sizeof(cd), cudaMemcpyDeviceToHost), "D2H");
    // 1 / X_ref = conj(v) / |v| / |v|: no |v|^2 underflow for tiny bins (the oracle divides directly;
    // its quotient is inf / NaN only where X_ref is exactly 0, and there H is reported as 0)
    rtab_h_.resize(bins());
    for (size_t k = 0; k < bins(); ++k) {
        const cd v = xref_[k];
        const double mag = std::hypot(v.real(), v.imag());
        if (mag > 0.0) {
            const double s = 1.0 / mag;
            rtab_h_[k] = cd(v.real() * s * s, -v.imag() * s * s);
        } else {
            rtab_h_[k] = cd(0.0, 0.0);
        }
    }
    rtab(f32);
}

const void* TransferPlanG::rtab(bool f32) const {
    return rtab_.get(f32, [&](DevMem& d) { d = to_device(rtab_h_, f32); }).p;
}

void TransferPlanG::execute(const void* x, long long x_stride, long long batch, void* mag, void* phase,
                            long long mp_stride, void* h, long long h_stride, cudaStream_t st) const {
    if (batch <= 0) return;
    const int lgM = ilog2(len_) - 1;
    if (lgM > single_cta_max_log2(f32_))
        throw std::invalid_argument("transfer: length needs the multi-pass path (not available in this build)");
    const void* tw = stockham_twiddles(lgM, f32_);
    const void* post = r2c_post_twiddles(lgM, f32_);
    cudaError_t e;
    if (f32_)
        e = launch_fft_r2c<float>(lgM, (long long)n_, (const float*)x, x_stride, batch, tw, post, 2, h, h_stride,
                                  rtab(true), (float*)mag, (float*)phase, mp_stride, 0, 0, st);
    else
        e = launch_fft_r2c<double>(lgM, (long long)n_, (const double*)x, x_stride, batch, tw, post, 2, h, h_stride,
                                   rtab(false), (double*)mag, (double*)phase, mp_stride, 0, 0, st);
    check(e, "transfer launch");
    count_launch();
}

}  // namespace skg
