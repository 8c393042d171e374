// kernels_zoom_tfir.cu — Zoom FFT FIR (zoom_fft's filter_decimate_circular, zoomfft.cpp:82-104,
// 183-207) fed by a TMA pipeline of whole records.
//
// The phase-lane FIR (kernels_zoom_fir.cuh) loads each sample from global memory into registers a
// few mini-batches ahead; ncu on configs[2] fp64 showed it stalled on those loads (long scoreboard
// 1.87 per issue, the hottest instruction a register move waiting on an LDG, 21% warps active at
// 128 registers) with the FP64 pipe 40% busy. Here the record streams into shared memory ahead of
// the compute instead:
//   * a CTA runs NTEAM teams of 4 warps; a team owns one record at a time and a ring of STAGES
//     record buffers; its leader thread keeps STAGES-1 records in flight with 1-D TMA bulk copies
//     (cp.async.bulk, completion on an mbarrier per stage), re-arming a stage as soon as the team
//     has left it — HBM streams under the FIR with no registers spent on loads in flight;
//   * the record lands as 128/D chunks of CH = U/128 polyphase rows (row r = x[rD .. rD+D-1]) with
//     one padding row after each chunk, so the D-lane groups of a warp (each on its own chunk) read
//     disjoint bank windows: conflict-free LDS;
//   * lanes are (group, phase) exactly as in the phase-lane FIR: a lane convolves its phase row with
//     that row's taps held in registers; the window is re-read from shared memory each mini-batch
//     (no register window moves), and the D phase partials are summed by an xor-shuffle
//     transpose-reduce instead of a shared-memory round trip.
// Same sum and the same wrap correction as the phase-lane FIR: u[m] = S[m] sum_t g[t] x[mD - t],
// complex taps g, real samples, the wrapped terms of the first outputs times e^{-i2pi fc U/fs}.
// Geometry: circular, untrimmed, U a power of two with U / 128 a multiple of the mini-batch, D a
// power of two 4..16; anything else runs the other FIR routes.
#include "bulk_copy.cuh"
#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"

namespace skg {

namespace {

constexpr int TF_TEAM_WARPS = 4;
constexpr int TF_TEAMS = 2;

struct TfirGeom {
    int stages;
    int cr;            // rows per chunk region: LH margin + CH rows (+1 to make it odd)
    int stage_elems;
    size_t red_off, s_off, ring_off, smem;
};

// shared layout: [full | empty mbarriers][per-warp wrap terms][per-warp phase partials][S table][rings]
inline TfirGeom tfir_geom(const ZoomArgs& a, int lh, bool f32, int optin) {
    TfirGeom g{};
    const int D = a.D, ch = (int)(a.U >> 7), MB = D > 8 ? D : 8, G = 32 / D;
    const size_t es = f32 ? 4 : 8, cs = 2 * es;
    g.cr = lh + ch;
    if ((g.cr & 1) == 0) ++g.cr;   // odd region stride: the lane groups of a wavefront hit disjoint banks
    g.stage_elems = (128 / D) * g.cr * D;
    const size_t stage_bytes = (size_t)g.stage_elems * es;
    const int nw = TF_TEAMS * TF_TEAM_WARPS;
    g.red_off = (2 * TF_TEAMS * 8 * 8 + (size_t)nw * (a.mwrap + 1) * cs + 127) / 128 * 128;
    g.s_off = (g.red_off + (size_t)nw * G * MB * (D + 1) * cs + 127) / 128 * 128;
    g.ring_off = (g.s_off + (size_t)a.nout * cs + 127) / 128 * 128;
    g.stages = 0;
    for (int st = 4; st >= 2; --st)
        if (g.ring_off + (size_t)TF_TEAMS * st * stage_bytes <= (size_t)optin) {
            g.stages = st;
            break;
        }
    g.smem = g.ring_off + (size_t)TF_TEAMS * g.stages * stage_bytes;
    return g;
}

template <typename T, int D, int LH>
__global__ void __launch_bounds__(32 * (TF_TEAM_WARPS * TF_TEAMS + 1), 1)
k_zoom_tfir(const T* __restrict__ x, long long x_stride, long long batch, ZoomArgs a, int tma, int stages, int cr,
            int stage_elems, int red_off, int s_off, int ring_off, const cx_t<T>* __restrict__ gph,
            const cx_t<T>* __restrict__ gnat, const cx_t<T>* __restrict__ S, cx_t<T>* __restrict__ zb,
            long long z_stride) {
    using C = cx_t<T>;
    constexpr int G = 32 / D;              // lane groups per warp
    constexpr int MB = D > 8 ? D : 8;      // outputs per mini-batch
    constexpr int K = MB / D;              // finished outputs per lane per mini-batch
    constexpr int W = LH - 1 + MB;         // window samples per mini-batch
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int U = (int)a.U;
    const int ch = U >> 7;                 // rows per chunk = outputs per lane group task
    const int nchunk = 128 / D;
    extern __shared__ __align__(128) unsigned char smraw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw);            // [team][8]
    uint64_t* empty = full + TF_TEAMS * 8;                          // [team][8]
    C* cwall = reinterpret_cast<C*>(smraw + 2 * TF_TEAMS * 8 * 8);   // [warp][mwrap + 1]
    T* ring0 = reinterpret_cast<T*>(smraw + ring_off);
    const long long tstride = (long long)gridDim.x * TF_TEAMS;
    if (threadIdx.x == 0) {
        for (int i = 0; i < TF_TEAMS * stages; ++i) {
            mbar_init(full + (i / stages) * 8 + i % stages, 1);
            mbar_init(empty + (i / stages) * 8 + i % stages, TF_TEAM_WARPS);
        }
        mbar_fence_init();
    }
    C* s_S = reinterpret_cast<C*>(smraw + s_off);   // the output phase table S[m], m < nout
    for (int i = threadIdx.x; i < a.nout; i += blockDim.x) s_S[i] = __ldg(S + i);
    // chunk 0's margin rows (before the record) are never written by the copies: zero them once
    for (int i = threadIdx.x; i < TF_TEAMS * stages * LH * D; i += blockDim.x)
        ring0[(size_t)(i / (LH * D)) * stage_elems + i % (LH * D)] = (T)0;
    fence_proxy_async_smem();
    __syncthreads();
    if (warp == TF_TEAMS * TF_TEAM_WARPS && !tma) {
        // rows not 16-byte aligned (no bulk copies): the producer warp copies each record itself, same
        // layout, then one arrive completes the stage (same route, so the same results bit for bit)
        for (int k = 0;; ++k) {
            bool any = false;
            for (int t = 0; t < TF_TEAMS; ++t) {
                const long long b = (long long)blockIdx.x * TF_TEAMS + t + k * tstride;
                if (b >= batch) continue;
                any = true;
                const int s = k % stages;
                if (k >= stages) mbar_wait(empty + t * 8 + s, (uint32_t)((k / stages - 1) & 1));
                const T* src = x + b * x_stride;
                T* dst = ring0 + ((size_t)t * stages + s) * stage_elems;
                for (int n = lane; n < U; n += 32) {
                    const int r = n / D, c = r / ch;
                    const T v = __ldg(src + n);
                    dst[((size_t)c * cr + LH + (r - c * ch)) * D + n % D] = v;
                    if (c + 1 < nchunk && r >= (c + 1) * ch - LH)   // also the next chunk's margin
                        dst[((size_t)(c + 1) * cr + (r - ((c + 1) * ch - LH))) * D + n % D] = v;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(full + t * 8 + s);
            }
            if (!any) break;
        }
        return;
    }
    if (warp == TF_TEAMS * TF_TEAM_WARPS) {   // producer warp: one thread keeps every team's ring full
        if (lane == 0) {
            const uint32_t row_b = (uint32_t)(D * sizeof(T));
            for (int k = 0;; ++k) {
                bool any = false;
                for (int t = 0; t < TF_TEAMS; ++t) {
                    const long long b = (long long)blockIdx.x * TF_TEAMS + t + k * tstride;
                    if (b >= batch) continue;
                    any = true;
                    const int s = k % stages;
                    if (k >= stages) mbar_wait_sleep(empty + t * 8 + s, (uint32_t)((k / stages - 1) & 1));
                    const T* src = x + b * x_stride;
                    T* dst = ring0 + ((size_t)t * stages + s) * stage_elems;
                    mbar_arrive_expect_tx(full + t * 8 + s, row_b * (uint32_t)(nchunk * (ch + LH) - LH));
                    // chunk c: rows [c ch - LH, (c + 1) ch) -> region rows [0, LH + ch) (chunk 0: no margin)
                    bulk_g2s(dst + LH * D, src, row_b * ch, full + t * 8 + s);
                    for (int c = 1; c < nchunk; ++c)
                        bulk_g2s(dst + (size_t)c * cr * D, src + (size_t)(c * ch - LH) * D, row_b * (ch + LH),
                                 full + t * 8 + s);
                }
                if (!any) break;
            }
        }
        return;
    }
    const int team = warp / TF_TEAM_WARPS, tw = warp % TF_TEAM_WARPS;
    const int ph = lane % D, g = lane / D;
    const int delta = ph != 0;
    C* cw = cwall + warp * (a.mwrap + 1);
    C* red = reinterpret_cast<C*>(smraw + red_off) + warp * (G * MB * (D + 1)) + g * MB * (D + 1);
    // this lane's phase-row taps, loaded once
    C tp[LH];
#pragma unroll
    for (int l = 0; l < LH; ++l) tp[l] = l < a.lh ? __ldg(gph + ph * a.lh + l) : czero<C>();
    int k = 0;
    for (long long b = (long long)blockIdx.x * TF_TEAMS + team; b < batch; b += tstride, ++k) {
        const int s = k % stages;
        const T* stage = ring0 + ((size_t)team * stages + s) * stage_elems;
        // output block of this warp: rotated per record so the block with the wrap terms (0) moves
        // round the team's warps and no warp carries it every time
        const int blk = (tw + TF_TEAM_WARPS - (k % TF_TEAM_WARPS)) % TF_TEAM_WARPS;
        const int cg = blk * G + g;   // this lane group's chunk
        const int m0 = cg * ch;       // its first output (= row)
        const bool wraps = a.circular && blk == 0 && a.mwrap > 0;
        mbar_wait(full + team * 8 + s, (uint32_t)((k / stages) & 1));
        if (wraps) {   // wrapped terms of the first mwrap outputs, from the staged record
            const int lch = 31 - __clz(ch);
            auto at = [&](int n) -> T {   // sample n of the record (row r = n / D in chunk c = r / ch)
                const int r = n / D, c = r >> lch;
                return stage[(c * cr + LH + (r - (c << lch))) * D + (n & (D - 1))];
            };
            const int h = lane >> 4, hl = lane & 15;
            for (int mm = 0; mm < a.mwrap; mm += 2) {
                const int m = mm + h;
                C acc = czero<C>();
                if (m < a.mwrap)
                    for (int s1 = 1 + hl; s1 <= a.T - 1 - m * D; s1 += 16)
                        acc = cadd(acc, rmul(at(U - s1), __ldg(gnat + m * D + s1)));
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                }
                if (hl == 0 && m < a.mwrap) cw[m] = cmul(acc, mk<C>((T)a.wre, (T)a.wim));
            }
            __syncwarp();
        }
        // window of the mini-batch at output mf: rows mf - (LH - 1) - delta + i, i < W; region row =
        // LH + (row - m0): compile-time offsets from one pointer that advances by MB rows
        const T* wp = stage + ((size_t)cg * cr + 1 - delta) * D + ph;
        for (int mb = 0; mb < ch; mb += MB, wp += MB * D) {
            T buf[W];
#pragma unroll
            for (int i = 0; i < W; ++i) buf[i] = wp[i * D];
            C P[MB];
#pragma unroll
            for (int j = 0; j < MB; ++j) {
                C e = czero<C>(), o = czero<C>();
#pragma unroll
                for (int l = 0; l < LH; l += 2) {
                    e.x = fma(tp[l].x, buf[LH - 1 + j - l], e.x);
                    e.y = fma(tp[l].y, buf[LH - 1 + j - l], e.y);
                    if (l + 1 < LH) {
                        o.x = fma(tp[l + 1].x, buf[LH - 2 + j - l], o.x);
                        o.y = fma(tp[l + 1].y, buf[LH - 2 + j - l], o.y);
                    }
                }
                P[j] = cadd(e, o);
            }
            // sum over the D phase-lanes of the group through a padded shared-memory transpose
            // (conflict free): lane (g, ph) posts its MB partials, then finishes outputs ph K + kk
#pragma unroll
            for (int j = 0; j < MB; ++j) red[j * (D + 1) + ph] = P[j];
            __syncwarp();
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                const int jj = ph * K + kk;
                // pairwise (tree) sum of the D phase partials: depth log2 D instead of a D-long chain
                C r[D];
#pragma unroll
                for (int q = 0; q < D; ++q) r[q] = red[jj * (D + 1) + q];
#pragma unroll
                for (int w = 1; w < D; w *= 2)
#pragma unroll
                    for (int q = 0; q + w < D; q += 2 * w) r[q] = cadd(r[q], r[q + w]);
                C v = r[0];
                const int m = m0 + mb + jj;
                if (m < a.nout) {
                    if (wraps && m < a.mwrap) v = cadd(v, cw[m]);
                    zb[b * z_stride + m] = cmul(v, s_S[m]);
                }
            }
            __syncwarp();
        }
        if (lane == 0) mbar_arrive(empty + team * 8 + s);   // this warp is done with the stage
    }
}

template <typename T, int D, int LH>
cudaError_t run_tfir(const ZoomArgs& a, const T* x, long long xs, long long batch, const void* gph, const void* gnat,
                     const void* S, void* zb, long long z_stride, cudaStream_t st) {
    using C = cx_t<T>;
    int dev = 0, optin = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const TfirGeom geo = tfir_geom(a, LH, sizeof(T) == 4, optin);
    if (geo.stages < 2) return cudaErrorNotSupported;
    const int tma = ((uintptr_t)x % 16) == 0 && ((size_t)xs * sizeof(T)) % 16 == 0;
    auto kern = k_zoom_tfir<T, D, LH>;
    cudaError_t e = prep_smem(kern, geo.smem);
    if (e != cudaSuccess) return e;
    long long grid = (batch + TF_TEAMS - 1) / TF_TEAMS;
    if (grid > sms) grid = sms;
    if (const unsigned gc = grid_cap(); gc && gc < grid) grid = gc;
    kern<<<(unsigned)grid, 32 * (TF_TEAM_WARPS * TF_TEAMS + 1), geo.smem, st>>>(
        x, xs, batch, a, tma, geo.stages, geo.cr, geo.stage_elems, (int)geo.red_off, (int)geo.s_off, (int)geo.ring_off, (const C*)gph,
        (const C*)gnat, (const C*)S, (C*)zb, z_stride);
    return cudaGetLastError();
}

template <typename T, int D>
cudaError_t tfir_lh(int lh, const ZoomArgs& a, const T* x, long long xs, long long batch, const void* gph,
                    const void* gnat, const void* S, void* zb, long long z_stride, cudaStream_t st) {
    switch (lh) {
        case 5: return run_tfir<T, D, 5>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 7: return run_tfir<T, D, 7>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 9: return run_tfir<T, D, 9>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace

bool zoom_tfir_fits(const ZoomArgs& a, bool f32, const void* x, long long x_stride) {
    static const bool off = std::getenv("SKG_ZOOM_NO_TFIR") != nullptr;
    if (off || !a.circular || a.trim != 0) return false;
    const int D = a.D;
    if (D != 4 && D != 8 && D != 16) return false;
    const long long U = a.U;
    if (U < 1024 || (U & (U - 1)) || (long long)a.nout * D != U || a.n < U) return false;
    const int ch = (int)(U >> 7), MB = D > 8 ? D : 8;
    if (ch % MB || ch < a.mwrap || ch < (a.T + D - 1) / D) return false;
    (void)x;
    (void)x_stride;   // unaligned rows run the same kernel with a copy loop instead of bulk copies
    const int lh = zoom_pfir_lh(a);
    if (lh != 5 && lh != 7 && lh != 9) return false;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return tfir_geom(a, lh, f32, optin).stages >= 2;
}

cudaError_t launch_zoom_tfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                             const void* gph, const void* gnat, const void* S, void* zb, long long z_stride,
                             cudaStream_t st) {
    const int lh = zoom_pfir_lh(a);
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        const T* xt = static_cast<const T*>(x);
        switch (a.D) {
            case 4: return tfir_lh<T, 4>(lh, a, xt, xs, batch, gph, gnat, S, zb, z_stride, st);
            case 8: return tfir_lh<T, 8>(lh, a, xt, xs, batch, gph, gnat, S, zb, z_stride, st);
            case 16: return tfir_lh<T, 16>(lh, a, xt, xs, batch, gph, gnat, S, zb, z_stride, st);
            default: return cudaErrorNotSupported;
        }
    };
    return f32 ? go(float{}) : go(double{});
}

}  // namespace skg
