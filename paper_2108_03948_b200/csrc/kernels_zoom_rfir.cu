// kernels_zoom_rfir.cu — Zoom FFT FIR (filter_decimate / filter_decimate_circular, zoomfft.cpp:82-104)
// for large decimations and ragged lengths: whole outputs per lane straight from a RAW (not polyphase)
// window of the trace in shared memory.
//
// Same sum as the other FIR routes: u[m] = S[m] (sum_t g[t] x[mD - t] + wrap_m), complex taps
// g[t] = h[t] e^{+i2pi fc t/fs} on real samples, samples outside [0, U) zero, the circular wrap terms of the
// first outputs times e^{-i2pi fc U/fs}. The phase-lane FIR (kernels_zoom_fir.cuh) gives every lane one
// polyphase row and sums the D partials of each output through shared memory: at D = 16 with 101 taps that
// is 7 taps per lane per output against a 16-term cross-lane reduction — about 30 instructions per lane
// per output for 14 useful FMAs (ncu: the fp32 FIR issue-bound at 62% issue / 23% warps, 2 TB/s on rows
// the survey counts as HBM bound). Here:
//   * a lane owns K consecutive outputs and sums ALL their taps (no partial sums cross lanes) from one
//     contiguous window of (K - 1) D + T samples, read as 16-byte units; the window's units and the tap of
//     every (sample, output) pair are compile-time, taps are constant-bank operands of the FMA
//     (__grid_constant__ parameter block): ~2 K T FMAs + ((K - 1) D + T) / EU loads per lane per item;
//   * a warp item = 32 K outputs of one record; its samples are copied global -> shared with 16-byte
//     cp.async into the raw order plus one pad unit per lane stride K D (the lanes' window bases then sit
//     an odd number of units apart: conflict-free LDS.128), double-buffered per warp where it fits; no
//     barriers beyond the warp, any nout (ragged last item), any U (units straddling the record's ends are
//     filled per element).
// Geometry: trim = 0; (D, T, K) specialised below (the configs[4] sweep: D in {4, 16},
// 101 taps). Output: decimated rows zb for k_zoom_fftband.
#include "bulk_copy.cuh"
#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"

#include <utility>

namespace skg {

namespace {

template <typename T, int NTAPS> struct RfTaps {
    cx_t<T> g[NTAPS];   // natural order g[t]
};

template <typename T, int D, int NTAPS, int K> struct RfGeom {
    static constexpr int EU = 16 / (int)sizeof(T);                 // elements per 16-byte unit
    static constexpr int LS = K * D;                                 // lane stride (samples)
    static constexpr int PART = 32 * K;                              // outputs per warp item
    static constexpr int PADL = (NTAPS - 1 + LS - 1) / LS * LS;      // samples before the item's first output sample
    static constexpr int SPAN = PADL + PART * D;                     // samples per item buffer (raw)
    static constexpr int UNITS = SPAN / EU;                          // 16-byte units per item
    static constexpr int LSP = LS + EU;                              // padded lane stride
    static constexpr int BUF = (SPAN / LS) * LSP;                    // padded elements per item buffer
    static constexpr int W0 = (PADL - (NTAPS - 1)) / EU * EU;        // window start relative to the lane base
    static constexpr int W1 = PADL + (K - 1) * D + 1;                // window end (exclusive)
    static constexpr int WU = (W1 - W0 + EU - 1) / EU;               // window units
    static_assert(LS % EU == 0 && (LS / EU) % 2 == 0, "lane stride: an even number of units (odd once padded)");
    __host__ __device__ static constexpr int pidx(int j) { return j + (j / LS) * EU; }
};

__device__ __forceinline__ void unit_elems(const float4& v, float (&e)[4]) {
    e[0] = v.x, e[1] = v.y, e[2] = v.z, e[3] = v.w;
}
__device__ __forceinline__ void unit_elems(const double2& v, double (&e)[2]) { e[0] = v.x, e[1] = v.y; }

#ifndef SKG_RFIR_WARPS
#define SKG_RFIR_WARPS 4
#endif
#ifndef SKG_RFIR_NBUF_F64
#define SKG_RFIR_NBUF_F64 1
#endif
#ifndef SKG_RFIR_WARPS_F64
#define SKG_RFIR_WARPS_F64 SKG_RFIR_WARPS
#endif
#ifndef SKG_RFIR_NBUF_F32
#define SKG_RFIR_NBUF_F32 2
#endif
template <typename T> __host__ __device__ constexpr int rf_nbuf() { return sizeof(T) == 8 ? SKG_RFIR_NBUF_F64 : SKG_RFIR_NBUF_F32; }
template <typename T> __host__ __device__ constexpr int rf_warps() { return sizeof(T) == 8 ? SKG_RFIR_WARPS_F64 : SKG_RFIR_WARPS; }

template <typename T, int D, int NTAPS, int K>
__global__ void __launch_bounds__(rf_warps<T>() * 32)
k_zoom_rfir(const T* __restrict__ x, long long x_stride, unsigned batch, int aligned, ZoomArgs a,
            const __grid_constant__ RfTaps<T, NTAPS> tp, const cx_t<T>* __restrict__ S, cx_t<T>* __restrict__ zb,
            long long z_stride) {
    using C = cx_t<T>;
    using RG = RfGeom<T, D, NTAPS, K>;
    constexpr int EU = RG::EU;
    constexpr int NBUF = rf_nbuf<T>();
    constexpr int WT = NTAPS - 1;                 // wrap samples x[U - s], s = 1..T-1
    constexpr int WTU = (WT + EU - 1) / EU;       // as 16-byte units (the tail starts unit aligned: U, T - 1 are)
    static_assert(WT % EU == 0, "tail of whole units");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    extern __shared__ __align__(16) unsigned char smraw[];
    // [taps g[t] (wrap terms' lane-varying reads)][per warp: NBUF x (item buffer + tail)]
    C* s_g = reinterpret_cast<C*>(smraw);
    constexpr int GB = (NTAPS * (int)sizeof(C) + 15) / 16 * 16;
    constexpr int SLOT = RG::BUF + WTU * EU;      // elements per buffer slot
    T* bufs = reinterpret_cast<T*>(smraw + GB) + (size_t)warp * NBUF * SLOT;
    for (int i = threadIdx.x; i < NTAPS; i += blockDim.x) s_g[i] = tp.g[i];
    __syncthreads();
    const int U = (int)a.U;
    const unsigned parts = (unsigned)(a.nout + RG::PART - 1) / RG::PART;
    const unsigned nitem = batch * parts;   // < 2^31 (checked by the launcher)
    const unsigned w0 = blockIdx.x * rf_warps<T>() + warp, wstride = gridDim.x * rf_warps<T>();
    const bool wrap = a.circular && a.mwrap > 0;
    // fill: unit un of the item covers samples i0 + un EU .. + EU - 1, i0 = p PART D - PADL
    auto fill = [&](unsigned item, int slot) {
        const unsigned b = item / parts;
        const int p = (int)(item - b * parts);
        const int i0 = p * RG::PART * D - RG::PADL;
        const T* xr = x + (long long)b * x_stride;
        T* dst = bufs + slot * SLOT;
#pragma unroll
        for (int uu = 0; uu < (RG::UNITS + 31) / 32; ++uu) {
            const int un = lane + 32 * uu;
            if (RG::UNITS % 32 == 0 || un < RG::UNITS) {
                const int j = un * EU, i = i0 + j;
                T* d = dst + RG::pidx(j);
                if (aligned && i >= 0 && i + EU <= U) {
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d)), "l"(xr + i) : "memory");
                } else {   // the record's ends, or rows that are not 16-byte aligned: element copies
#pragma unroll
                    for (int e = 0; e < EU; ++e) {
                        if (i + e >= 0 && i + e < U) cp_async_el(d + e, xr + i + e, true);
                        else d[e] = (T)0;
                    }
                }
            }
        }
        if (p == 0 && wrap) {   // the record's last T - 1 samples, for the wrapped terms
#pragma unroll
            for (int k = lane; k < WTU; k += 32) {
                if (aligned) {
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + RG::BUF + k * EU)),
                                 "l"(xr + U - WT + k * EU)
                                 : "memory");
                } else {
#pragma unroll
                    for (int e = 0; e < EU; ++e) cp_async_el(dst + RG::BUF + k * EU + e, xr + U - WT + k * EU + e, true);
                }
            }
        }
        cp_async_commit();
    };
    static_assert(WTU <= 64, "tail units");
    if (NBUF == 2 && w0 < nitem) fill(w0, 0);
    int slot = 0;
    for (unsigned item = w0; item < nitem; item += wstride) {
        if (NBUF == 1) {
            fill(item, 0);
            if (item + wstride < nitem) {   // single-buffered: at least pull the next item's samples into L2
                const unsigned bn = (item + wstride) / parts;
                const int i0n = (int)((item + wstride) - bn * parts) * RG::PART * D - RG::PADL;
                const T* xn = x + (long long)bn * x_stride + i0n;
                constexpr int per = 128 / (int)sizeof(T);
                for (int i = lane * per; i < RG::SPAN; i += 32 * per)
                    if (i0n + i >= 0 && i0n + i < U) prefetch_l2(xn + i);
            }
            cp_async_wait_all();
        } else if (item + wstride < nitem) {
            fill(item + wstride, slot ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            cp_async_wait_all();
        }
        __syncwarp();
        const unsigned b = item / parts;
        const int p = (int)(item - b * parts);
        const T* wl = bufs + slot * SLOT + lane * RG::LSP;
        C acc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = czero<C>();
        using VT = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
        // the lane's window, unit by unit: sample at relative position r = W0 + u EU + e feeds output c
        // with tap t = PADL + c D - r (when 0 <= t < T); everything but the lane base is compile-time
#pragma unroll
        for (int u = 0; u < RG::WU; ++u) {
            const int r0 = RG::W0 + u * EU;
            const VT v = *reinterpret_cast<const VT*>(wl + RG::pidx(r0));
            T e[EU];   // registers (no address taken)
            unit_elems(v, e);
#pragma unroll
            for (int k2 = 0; k2 < EU; ++k2) {
                const int r = r0 + k2;
#pragma unroll
                for (int c = 0; c < K; ++c) {
                    const int t = RG::PADL + c * D - r;
                    if (t >= 0 && t < NTAPS) {
                        const C g = tp.g[t];
                        acc[c].x = fma(g.x, e[k2], acc[c].x);
                        acc[c].y = fma(g.y, e[k2], acc[c].y);
                    }
                }
            }
        }
        const int mb = p * RG::PART + lane * K;
        if (p == 0 && wrap) {
            // wrapped terms cw[m] = w sum_{s=1}^{T-1-mD} g[mD + s] x[U - s], m < mwrap, from the staged tail
            // (x[U - s] = tail[T - 1 - s]): lane i sums a quarter of output mw + i / 4, then the owner lane
            // (m / K) collects them
            const T* tail = bufs + slot * SLOT + RG::BUF;
            for (int mw = 0; mw < a.mwrap; mw += 8) {
                const int m = mw + (lane >> 2), q = lane & 3;
                C v = czero<C>();
                if (m < a.mwrap) {
                    C v2 = czero<C>();   // two chains
                    int s1 = 1 + q;
                    for (; s1 + 4 <= WT - m * D; s1 += 8) {
                        v = cadd(v, rmul(tail[WT - s1], s_g[m * D + s1]));
                        v2 = cadd(v2, rmul(tail[WT - s1 - 4], s_g[m * D + s1 + 4]));
                    }
                    if (s1 <= WT - m * D) v = cadd(v, rmul(tail[WT - s1], s_g[m * D + s1]));
                    v = cadd(v, v2);
                }
                v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
                v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
                v.x += __shfl_xor_sync(0xffffffffu, v.x, 2);
                v.y += __shfl_xor_sync(0xffffffffu, v.y, 2);
                v = cmul(v, mk<C>((T)a.wre, (T)a.wim));
#pragma unroll
                for (int c = 0; c < K; ++c) {
                    // output mb + c of this lane takes lane 4 (mb + c - mw) when that is in range
                    const int src = 4 * (mb + c - mw);
                    C got;
                    got.x = __shfl_sync(0xffffffffu, v.x, src & 31);
                    got.y = __shfl_sync(0xffffffffu, v.y, src & 31);
                    const T f = (T)(src >= 0 && src < 32 && mb + c < a.mwrap);   // arithmetic select: acc stays in registers
                    acc[c].x = fma(f, got.x, acc[c].x);
                    acc[c].y = fma(f, got.y, acc[c].y);
                }
            }
        }
        C* zr = zb + (long long)b * z_stride + mb;
#pragma unroll
        for (int c = 0; c < K; ++c)
            if (mb + c < a.nout) zr[c] = cmul(acc[c], __ldg(S + mb + c));
        __syncwarp();   // the buffer is refilled by a later item
        if (NBUF == 2) slot ^= 1;
    }
}

// ---- FIR + short FFT + band in ONE launch (the north_star's single zoom kernel for n_fft <= 2048) ------
// A CTA of 4 warps owns a record: warp p filters part p (32 K outputs) exactly as k_zoom_rfir does, the
// decimated values go to a shared row instead of the L2 work rows, then the CTA's 128 threads run the
// n_fft-point transform (zero padding pruned from its first pass) and store the signed band bins x D x
// group-delay phase (zoomfft.cpp:204-234) straight from registers — no work rows, no second launch (whose
// 4096 single-record CTAs ran as 7 latency-bound waves). The transform's exchange region aliases the part
// buffers the FIR has just consumed (buffers are laid out by parity: [slot 0 of warps 0..3][slot 1 ..], so
// a parity is one contiguous region and the prefetched next record, in the other parity, is untouched).
// Geometry: nout <= 4 x 32 K, n_fft = 2^LOG2N in [512, 2048] >= nout.
template <typename T, int D, int NTAPS, int K, int LOG2N, int NZ>
__global__ void __launch_bounds__(128, 4)
k_zoom_rfir_fft(const T* __restrict__ x, long long x_stride, unsigned batch, int aligned, ZoomArgs a,
                const __grid_constant__ RfTaps<T, NTAPS> tp, const cx_t<T>* __restrict__ S,
                const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ band, cx_t<T>* __restrict__ out,
                long long out_stride) {
    using C = cx_t<T>;
    using RG = RfGeom<T, D, NTAPS, K>;
    using G = FftGeom<LOG2N>;
    constexpr int EU = RG::EU;
    constexpr int NBUF = rf_nbuf<T>();
    constexpr int WT = NTAPS - 1;
    constexpr int WTU = (WT + EU - 1) / EU;
    constexpr int SLOT = RG::BUF + WTU * EU;
    constexpr int GB = (NTAPS * (int)sizeof(C) + 15) / 16 * 16;
    static_assert(4 * SLOT * sizeof(T) >= G::SMEM * sizeof(C), "the exchange region fits in one buffer parity");
    static_assert(G::NT <= 128, "transform threads");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    extern __shared__ __align__(16) unsigned char smraw[];
    // [taps][NBUF parities x 4 warps x slot][decimated row: 4 x 32 K complex][twiddle tables]
    C* s_g = reinterpret_cast<C*>(smraw);
    T* bufs = reinterpret_cast<T*>(smraw + GB);
    C* zrow = reinterpret_cast<C*>(bufs + (size_t)NBUF * 4 * SLOT);
    C* tws = zrow + 4 * RG::PART;
    for (int i = threadIdx.x; i < NTAPS; i += blockDim.x) s_g[i] = tp.g[i];
    load_twiddles<LOG2N>(tws, tw);
    __syncthreads();
    const int U = (int)a.U;
    const int parts = (a.nout + RG::PART - 1) / RG::PART;   // <= 4
    const bool wrap = a.circular && a.mwrap > 0;
    const bool mine = warp < parts;
    auto fill = [&](unsigned b, int par) {
        const int p = warp;
        const int i0 = p * RG::PART * D - RG::PADL;
        const T* xr = x + (long long)b * x_stride;
        T* dst = bufs + ((size_t)par * 4 + warp) * SLOT;
#pragma unroll
        for (int uu = 0; uu < (RG::UNITS + 31) / 32; ++uu) {
            const int un = lane + 32 * uu;
            if (RG::UNITS % 32 == 0 || un < RG::UNITS) {
                const int j = un * EU, i = i0 + j;
                T* d = dst + RG::pidx(j);
                if (aligned && i >= 0 && i + EU <= U) {
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d)), "l"(xr + i) : "memory");
                } else {
#pragma unroll
                    for (int e = 0; e < EU; ++e) {
                        if (i + e >= 0 && i + e < U) cp_async_el(d + e, xr + i + e, true);
                        else d[e] = (T)0;
                    }
                }
            }
        }
        if (p == 0 && wrap) {
#pragma unroll
            for (int k = lane; k < WTU; k += 32) {
                if (aligned) {
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + RG::BUF + k * EU)),
                                 "l"(xr + U - WT + k * EU)
                                 : "memory");
                } else {
#pragma unroll
                    for (int e = 0; e < EU; ++e) cp_async_el(dst + RG::BUF + k * EU + e, xr + U - WT + k * EU + e, true);
                }
            }
        }
        cp_async_commit();
    };
    if (NBUF == 2 && mine && blockIdx.x < batch) fill(blockIdx.x, 0);
    int par = 0;
    for (unsigned b = blockIdx.x; b < batch; b += gridDim.x) {
        if (mine) {
            if (NBUF == 1) {
                fill(b, 0);
                if (b + gridDim.x < batch) {   // single-buffered: at least pull the next record's part into L2
                    const T* xn = x + (long long)(b + gridDim.x) * x_stride + warp * RG::PART * D - RG::PADL;
                    constexpr int per = 128 / (int)sizeof(T);
                    for (int i = lane * per; i < RG::SPAN; i += 32 * per)
                        if (warp * RG::PART * D - RG::PADL + i >= 0 && warp * RG::PART * D - RG::PADL + i < U) prefetch_l2(xn + i);
                }
                cp_async_wait_all();
            } else if (b + gridDim.x < batch) {
                fill(b + gridDim.x, par ^ 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                cp_async_wait_all();
            }
            __syncwarp();
            const T* slot = bufs + ((size_t)par * 4 + warp) * SLOT;
            const T* wl = slot + lane * RG::LSP;
            C acc[K];
#pragma unroll
            for (int c = 0; c < K; ++c) acc[c] = czero<C>();
            using VT = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
#pragma unroll
            for (int u = 0; u < RG::WU; ++u) {
                const int r0 = RG::W0 + u * EU;
                const VT v = *reinterpret_cast<const VT*>(wl + RG::pidx(r0));
                T e[EU];
                unit_elems(v, e);
#pragma unroll
                for (int k2 = 0; k2 < EU; ++k2) {
                    const int r = r0 + k2;
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        const int t = RG::PADL + c * D - r;
                        if (t >= 0 && t < NTAPS) {
                            const C g = tp.g[t];
                            acc[c].x = fma(g.x, e[k2], acc[c].x);
                            acc[c].y = fma(g.y, e[k2], acc[c].y);
                        }
                    }
                }
            }
            const int mb = warp * RG::PART + lane * K;
            if (warp == 0 && wrap) {
                const T* tail = slot + RG::BUF;
                for (int mw = 0; mw < a.mwrap; mw += 8) {
                    const int m = mw + (lane >> 2), q = lane & 3;
                    C v = czero<C>();
                    if (m < a.mwrap) {
                        C v2 = czero<C>();
                        int s1 = 1 + q;
                        for (; s1 + 4 <= WT - m * D; s1 += 8) {
                            v = cadd(v, rmul(tail[WT - s1], s_g[m * D + s1]));
                            v2 = cadd(v2, rmul(tail[WT - s1 - 4], s_g[m * D + s1 + 4]));
                        }
                        if (s1 <= WT - m * D) v = cadd(v, rmul(tail[WT - s1], s_g[m * D + s1]));
                        v = cadd(v, v2);
                    }
                    v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
                    v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
                    v.x += __shfl_xor_sync(0xffffffffu, v.x, 2);
                    v.y += __shfl_xor_sync(0xffffffffu, v.y, 2);
                    v = cmul(v, mk<C>((T)a.wre, (T)a.wim));
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        const int src = 4 * (mb + c - mw);
                        C got;
                        got.x = __shfl_sync(0xffffffffu, v.x, src & 31);
                        got.y = __shfl_sync(0xffffffffu, v.y, src & 31);
                        const T f = (T)(src >= 0 && src < 32 && mb + c < a.mwrap);
                        acc[c].x = fma(f, got.x, acc[c].x);
                        acc[c].y = fma(f, got.y, acc[c].y);
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < K; ++c)
                if (mb + c < a.nout) zrow[mb + c] = cmul(acc[c], __ldg(S + mb + c));
        }
        __syncthreads();   // the decimated row is complete; every part buffer of this parity is consumed
        // n_fft-point transform of the zero-padded row by the CTA, exchange region = this parity's buffers
        C* fsm = reinterpret_cast<C*>(bufs + (size_t)par * 4 * SLOT);
        const bool act = tid < G::NT;
        C v[G::EPT];
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            const int pos = tid + G::NT * q;
            v[q] = (act && q < NZ && pos < a.nout) ? zrow[pos] : czero<C>();
        }
        block_fft<false, LOG2N, NZ>(v, fsm, tws, tid, act);
        if (act) {
            C* o = out + (long long)b * out_stride;
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) {   // bin k = tid + NT q of [0, n_fft) is signed bin k_lo + i
                const int i = (tid + G::NT * q - a.k_lo) & (G::L - 1);
                if (i < a.nbins) o[i] = cmul(v[q], __ldg(band + i));
            }
        }
        __syncthreads();   // zrow and the exchange region are free for the next record
        if (NBUF == 2) par ^= 1;
    }
}

template <typename T, int D, int NTAPS, int K, int LOG2N>
cudaError_t run_rfir_fft(const ZoomArgs& a, const T* x, long long xs, long long batch, const void* gnat_host,
                         const void* S, const void* tw, const void* band, void* out, long long out_stride,
                         cudaStream_t st) {
    using C = cx_t<T>;
    using RG = RfGeom<T, D, NTAPS, K>;
    using G = FftGeom<LOG2N>;
    constexpr int EU = RG::EU;
    RfTaps<T, NTAPS> tp;
    const double* gh = static_cast<const double*>(gnat_host);
    for (int t = 0; t < NTAPS; ++t) {
        tp.g[t].x = (T)gh[2 * t];
        tp.g[t].y = (T)gh[2 * t + 1];
    }
    const size_t smem = (NTAPS * sizeof(C) + 15) / 16 * 16 +
                        (size_t)4 * rf_nbuf<T>() * (RG::BUF + (NTAPS - 1 + EU - 1) / EU * EU) * sizeof(T) +
                        ((size_t)4 * RG::PART + G::TW_ALLOC) * sizeof(C);
    if (batch >= (1LL << 31)) return cudaErrorNotSupported;
    const int aligned = reinterpret_cast<uintptr_t>(x) % 16 == 0 && xs % EU == 0 && a.U % EU == 0;
    auto launch = [&](auto kern) -> cudaError_t {
        cudaError_t e = prep_smem(kern, smem);
        if (e != cudaSuccess) return e;
        const unsigned grid = persistent_grid(kern, 128, smem, batch);
        kern<<<grid, 128, smem, st>>>(x, xs, (unsigned)batch, aligned, a, tp, (const C*)S, (const C*)tw, (const C*)band,
                                      (C*)out, out_stride);
        return cudaGetLastError();
    };
    const int nz = nz_class(a.nout, G::NT);
    if (nz == 4) return launch(k_zoom_rfir_fft<T, D, NTAPS, K, LOG2N, 4>);
    if (nz == 8) return launch(k_zoom_rfir_fft<T, D, NTAPS, K, LOG2N, 8>);
    return launch(k_zoom_rfir_fft<T, D, NTAPS, K, LOG2N, 16>);
}

template <typename T, int D, int NTAPS, int K>
cudaError_t run_rfir(const ZoomArgs& a, const T* x, long long xs, long long batch, const void* gnat_host,
                     const void* S, void* zb, long long z_stride, cudaStream_t st) {
    using C = cx_t<T>;
    using RG = RfGeom<T, D, NTAPS, K>;
    RfTaps<T, NTAPS> tp;
    const double* gh = static_cast<const double*>(gnat_host);   // fp64 natural-order taps (re, im pairs)
    for (int t = 0; t < NTAPS; ++t) {
        tp.g[t].x = (T)gh[2 * t];
        tp.g[t].y = (T)gh[2 * t + 1];
    }
    constexpr int EU = RG::EU;
    const size_t smem = (NTAPS * sizeof(C) + 15) / 16 * 16 +
                        (size_t)rf_warps<T>() * rf_nbuf<T>() * (RG::BUF + (NTAPS - 1 + EU - 1) / EU * EU) * sizeof(T);
    auto kern = k_zoom_rfir<T, D, NTAPS, K>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long long parts = (a.nout + RG::PART - 1) / RG::PART;
    if (batch * parts >= (1LL << 31)) return cudaErrorNotSupported;
    // 16-byte copies need aligned rows (and, for the wrap tail, U a whole number of units); otherwise the
    // same kernel copies element by element — the route, and so the bits, do not depend on the alignment
    const int aligned = reinterpret_cast<uintptr_t>(x) % 16 == 0 && xs % EU == 0 && a.U % EU == 0;
    constexpr int NW = rf_warps<T>();
    const unsigned grid = persistent_grid(kern, NW * 32, smem, (batch * parts + NW - 1) / NW);
    kern<<<grid, NW * 32, smem, st>>>(x, xs, (unsigned)batch, aligned, a, tp, (const C*)S, (C*)zb, z_stride);
    return cudaGetLastError();
}

}  // namespace

// raw-window whole-output FIR: specialised (D, T)
bool zoom_rfir_fits(const ZoomArgs& a, bool f32, const void* x, long long x_stride) {
    const bool off = std::getenv("SKG_ZOOM_NO_RFIR") != nullptr;   // read per call: tests switch routes in-process
    if (off || a.trim != 0) return false;
    const int key = a.D * 1000 + a.T;
    if (key != 16101 && key != 4101 && key != 8065 && key != 8101) return false;
    (void)f32, (void)x, (void)x_stride;
    return a.U <= a.n && a.U >= a.T;
}

cudaError_t launch_zoom_rfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                             const void* gnat_host, const void* gnat, const void* S, void* zb, long long z_stride,
                             cudaStream_t st) {
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        const T* xt = static_cast<const T*>(x);
        switch (a.D * 1000 + a.T) {
            case 16101: return run_rfir<T, 16, 101, 2>(a, xt, xs, batch, gnat_host, S, zb, z_stride, st);
            case 4101: return run_rfir<T, 4, 101, 8>(a, xt, xs, batch, gnat_host, S, zb, z_stride, st);
            case 8065: return run_rfir<T, 8, 65, 4>(a, xt, xs, batch, gnat_host, S, zb, z_stride, st);
            case 8101: return run_rfir<T, 8, 101, 4>(a, xt, xs, batch, gnat_host, S, zb, z_stride, st);
            default: return cudaErrorNotSupported;
        }
    };
    return f32 ? go(float{}) : go(double{});
}

// FIR + n_fft-point transform + band in one launch: configs[2] geometry (D = 8, 65 taps, nout <= 512) with
// n_fft = 2048 (SKG_ZOOM_NO_FUSE=1 or SKG_ZOOM_NO_RFIR_FFT=1: the two launches)
bool zoom_rfir_fft_fits(const ZoomArgs& a, bool f32, int log2n) {
    (void)f32;
    if (std::getenv("SKG_ZOOM_NO_FUSE") || std::getenv("SKG_ZOOM_NO_RFIR_FFT") || std::getenv("SKG_ZOOM_NO_RFIR"))
        return false;
    if (a.trim != 0 || a.D != 8 || a.T != 65 || log2n != 11) return false;
    return a.nout <= 4 * 32 * 4 && a.nout <= (1 << log2n) && a.U <= a.n && a.U >= a.T;
}

cudaError_t launch_zoom_rfir_fft(const ZoomArgs& a, bool f32, int log2n, const void* x, long long xs, long long batch,
                                 const void* gnat_host, const void* S, const void* tw, const void* band, void* out,
                                 long long out_stride, cudaStream_t st) {
    if (log2n != 11 || a.D != 8 || a.T != 65) return cudaErrorNotSupported;
    if (f32)
        return run_rfir_fft<float, 8, 65, 4, 11>(a, static_cast<const float*>(x), xs, batch, gnat_host, S, tw, band, out,
                                                 out_stride, st);
    return run_rfir_fft<double, 8, 65, 4, 11>(a, static_cast<const double*>(x), xs, batch, gnat_host, S, tw, band, out,
                                              out_stride, st);
}

}  // namespace skg
