// kernels_zoom_pcfir.cu — Zoom FFT FIR (zoom_fft's filter_decimate_circular, zoomfft.cpp:82-104,
// 183-207): every lane sums whole outputs, taps in the constant bank, polyphase rows filled by
// asynchronous copies.
//
// Same sum as the other FIR routes (kernels_zoom.cu): u[m] = S[m] sum_t g[t] x[mD - t], complex taps
// g[t] = h[t] e^{+i2pi fc t/fs} on real samples, the wrapped terms of the first outputs times
// e^{-i2pi fc U/fs}. What changes is the work split:
//   * a lane owns K = 8 consecutive outputs and sums ALL their taps, so no partial sums cross lanes
//     (the phase-lane FIR spends a shared-memory transpose and D - 1 adds per output on that);
//   * the kernel is specialised on (D, T): with the tap loop fully unrolled every tap is a
//     compile-time offset into the launch's parameter block, so the DFMA / FFMA takes it as a
//     constant-bank operand — no tap registers, no tap loads, and two register operands per FMA
//     (tools/micro/fp64_regs.cu: 31.8 TF/s fp64 that way against 22-26 with three);
//   * a warp works through parts of 256 outputs; the rows a part needs (256 + 16 margin per phase)
//     are copied global -> shared with cp.async into a polyphase layout (row block of 8 + one pad
//     unit: the K-row lane stride lands on distinct banks) while the warp filters the previous part
//     from the other buffer — one coalesced 8-byte copy per sample, both addresses a per-lane base
//     plus compile-time offsets; no barriers beyond the warp.
// Geometry: circular, untrimmed, nout a multiple of 256, U = nout D; (D, T) specialised below.
#include "bulk_copy.cuh"
#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"

#include <utility>

namespace skg {

namespace {

constexpr int PC_K = 8;        // outputs per lane
constexpr int PC_PART = 256;   // outputs per warp task (32 lanes x K)
constexpr int PC_PRE = 16;     // margin rows before a part (>= the window reach)

template <typename T, int NTAPS> struct PcTaps {
    cx_t<T> g[NTAPS];   // natural order g[t]
};

template <typename T> struct PcGeom {
    static constexpr int EU = 16 / (int)sizeof(T);         // elements per 16-byte unit
    static constexpr int BS = 8 + EU;                        // row block of 8 + one pad unit
    static constexpr int NB = (PC_PRE + PC_PART) / 8;        // row blocks per phase
    // phase stride (elements, a 16-byte multiple): fp64 = 2 (mod 16), fp32 = 4 (mod 32), so the 32 lanes of
    // a copy instruction (8 phases x 4 rows) write distinct banks
    static constexpr int PSE = sizeof(T) == 8 ? (NB * BS + 15) / 16 * 16 + 2 : (NB * BS + 31) / 32 * 32 + 4;
    __host__ __device__ static constexpr int pidx(int i) { return (i >> 3) * BS + (i & 7); }
};

// buffers per warp: fp32 double-buffers its parts; fp64 parts are twice the size, so a warp fills
// its one buffer and waits, and the other warps of the SM filter meanwhile (8 warps either way)
#ifndef SKG_PC_F32_WARPS
#define SKG_PC_F32_WARPS 12
#endif
#ifndef SKG_PC_F32_NBUF
#define SKG_PC_F32_NBUF 1
#endif
template <typename T> __host__ __device__ constexpr int pc_nbuf() { return sizeof(T) == 8 ? 1 : SKG_PC_F32_NBUF; }
template <typename T> __host__ __device__ constexpr int pc_warps() { return sizeof(T) == 8 ? 8 : SKG_PC_F32_WARPS; }

struct WarpSync {
    __device__ __forceinline__ void operator()() const { __syncwarp(); }
};

// FUSE: the warp also runs the record's 512-point transform (nout = 2 parts = n_fft) and the signed
// band gather x band factor straight from the part buffer it has just consumed — one launch per
// batch, no work rows (else the decimated rows go to zb for k_zoom_fftband)
template <typename T, int D, int NTAPS, bool FUSE>
__global__ void __launch_bounds__(pc_warps<T>() * 32, 1)
k_zoom_pcfir(const T* __restrict__ x, long long x_stride, long long batch, ZoomArgs a,
             const __grid_constant__ PcTaps<T, NTAPS> tp, const cx_t<T>* __restrict__ S, cx_t<T>* __restrict__ zb,
             long long z_stride, const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ band,
             cx_t<T>* __restrict__ out, long long out_stride) {
    using C = cx_t<T>;
    using PG = PcGeom<T>;
    constexpr int LH = (NTAPS + D - 1) / D;                        // taps per phase row
    constexpr int WB = (LH + PG::EU - 1) / PG::EU * PG::EU;          // window rows before the block
    static_assert(WB <= PC_PRE, "margin");
    constexpr int WROWS = WB + PC_K;                                 // window rows per phase
    constexpr int LQ = 32 / D;                                       // rows per 32-lane copy
    constexpr int NCP = (PC_PRE + PC_PART) * D / 32;                 // copies per lane per part
    constexpr int BUF = D * PG::PSE;                                 // elements per part buffer
    constexpr int WT = NTAPS - 1;                                    // wrap samples x[U - s], s = 1..T-1
    constexpr int NBUF = pc_nbuf<T>();
    constexpr int WTP = (WT + 3) / 4 * 4;
    constexpr int JP = PC_PRE * D / 32;                              // copies covering the margin rows
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const int U = (int)a.U;
    const int parts = a.nout / PC_PART;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* s_S = reinterpret_cast<C*>(smraw);                            // S[m], m < nout
    C* s_g = s_S + a.nout;                                           // taps g[t] (the wrap terms' lane-varying reads)
    T* wbuf = reinterpret_cast<T*>(s_g + NTAPS) + warp * NBUF * WTP;
    // part buffers 16-byte aligned (window loads are LDS.128)
    const size_t boff = ((size_t)(a.nout + NTAPS) * sizeof(C) + (size_t)nw * NBUF * WTP * sizeof(T) + 15) / 16 * 16;
    T* bufs = reinterpret_cast<T*>(smraw + boff) + (size_t)warp * NBUF * BUF;
    C* tws = reinterpret_cast<C*>(smraw + boff + (size_t)nw * NBUF * BUF * sizeof(T));   // FUSE: n_fft twiddles
    for (int i = threadIdx.x; i < a.nout; i += blockDim.x) s_S[i] = __ldg(S + i);
    for (int i = threadIdx.x; i < NTAPS; i += blockDim.x) s_g[i] = tp.g[i];
    if constexpr (FUSE) load_twiddles<9>(tws, tw);
    __syncthreads();
    // this warp's records b0 + k rstride, all parts in order: item i = (record k = i / parts, part i % parts)
    const long long b0 = (long long)blockIdx.x * nw + warp, rstride = (long long)gridDim.x * nw;
    const long long nrec = b0 < batch ? (batch - 1 - b0) / rstride + 1 : 0;
    const long long nitem = nrec * parts;
    // copy geometry of this lane: phase ph, row-in-copy lq; destination base in a part buffer
    const int cph = lane % D, clq = lane / D;
    const int cdst = cph * PG::PSE + clq;
    auto fill = [&](long long item, int slot) {
        const long long b = b0 + (item / parts) * rstride;
        const int p = (int)(item % parts);
        const int r0 = p * PC_PART - PC_PRE;   // first row copied
        const T* src = x + b * x_stride + (long long)r0 * D + lane;
        T* dst = bufs + slot * BUF + cdst;
        const uint32_t dsa = smem_u32(dst);
        // one 8- / 4-byte copy per sample: shared and global addresses are this lane's bases plus
        // compile-time offsets (immediates in the instruction)
        auto copy = [&]<int J>(std::integral_constant<int, J>) {
            constexpr int ES = (int)sizeof(T);
            constexpr int doff = (((LQ * J) >> 3) * PG::BS + ((LQ * J) & 7)) * ES;
            if (J < JP && p == 0) {   // rows before the record (the linear part of the wrap)
                dst[doff / ES] = (T)0;
            } else {
                asm volatile("cp.async.ca.shared.global [%0+%2], [%1+%3], %4;" ::"r"(dsa), "l"(src), "n"(doff),
                             "n"(32 * J * ES), "n"(ES)
                             : "memory");
            }
        };
        [&]<int... J>(std::integer_sequence<int, J...>) {
            (copy(std::integral_constant<int, J>{}), ...);
        }(std::make_integer_sequence<int, NCP>{});
        if (p == 0 && a.circular) {   // the record's last T-1 samples, for the wrapped terms
            const T* xr = x + b * x_stride;
            for (int s1 = lane; s1 < WT; s1 += 32) cp_async_el(wbuf + slot * WTP + s1, xr + U - 1 - s1, true);
        }
        cp_async_commit();
    };
    if (NBUF == 2 && nitem > 0) fill(0, 0);
    C keep[PC_K];   // FUSE: part 0's outputs while part 1 is filtered
    for (long long item = 0; item < nitem; ++item) {
        const int slot = NBUF == 2 ? (int)(item & 1) : 0;
        if (NBUF == 1) {
            fill(item, 0);
            cp_async_wait_all();
        } else if (item + 1 < nitem) {
            fill(item + 1, slot ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            cp_async_wait_all();
        }
        __syncwarp();
        const long long b = b0 + (item / parts) * rstride;
        const int p = (int)(item % parts);
        const T* xb = bufs + slot * BUF;
        // this lane's outputs m = p * 256 + 8 lane + c; window of phase ph = part rows
        // [8 lane + PRE - WB, 8 lane + PRE + K): block `lane`, offset PRE - WB, then compile-time
        C acc[PC_K];
#pragma unroll
        for (int c = 0; c < PC_K; ++c) acc[c] = czero<C>();
        const T* wl = xb + lane * PG::BS;
        // the window as whole 16-byte units (LDS.128: the odd unit stride of the lanes keeps a quarter
        // warp on distinct banks; narrower loads would conflict)
        using VT = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
        static_assert(WB % PG::EU == 0 && (PC_PRE - WB) % PG::EU == 0 && WROWS % PG::EU == 0, "unit window");
        auto load_window = [&](int ph, T (&w)[WROWS]) {
#pragma unroll
            for (int u = 0; u < WROWS / PG::EU; ++u) {
                const VT v = *reinterpret_cast<const VT*>(wl + ph * PG::PSE + PG::pidx(PC_PRE - WB + u * PG::EU));
                const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
                for (int k2 = 0; k2 < PG::EU; ++k2) w[u * PG::EU + k2] = e[k2];
            }
        };
#pragma unroll
        for (int ph = 0; ph < D; ++ph) {
            T w[WROWS];
            load_window(ph, w);
            const int t0 = ph ? D - ph : 0, dl = ph ? 1 : 0;
#pragma unroll
            for (int l = 0; l < LH; ++l) {
                const int t = l * D + t0;
                if (t < NTAPS) {
                    const C g = tp.g[t];
#pragma unroll
                    for (int c = 0; c < PC_K; ++c) {
                        // row m - l - dl = (m_l - WB) + (WB + c - l - dl)
                        const T s = w[WB + c - l - dl];
                        acc[c].x = fma(g.x, s, acc[c].x);
                        acc[c].y = fma(g.y, s, acc[c].y);
                    }
                }
            }
        }
        const int mb = p * PC_PART + lane * PC_K;
        if (p == 0 && a.circular && a.mwrap > 0) {
            // wrapped terms cw[m] = w sum_{s=1}^{T-1-mD} g[mD + s] x[U - s], m < mwrap (<= 32 lanes x K):
            // lane i sums a quarter of output mw + i / 4, then the owner lane (m / K) collects them
            const T* wx = wbuf + slot * WTP;
            for (int mw = 0; mw < a.mwrap; mw += 8) {
                const int m = mw + (lane >> 2), q = lane & 3;
                C v = czero<C>();
                if (m < a.mwrap) {
                    C v2 = czero<C>();   // two chains
                    int s1 = 1 + q;
                    for (; s1 + 4 <= NTAPS - 1 - m * D; s1 += 8) {
                        v = cadd(v, rmul(wx[s1 - 1], s_g[m * D + s1]));
                        v2 = cadd(v2, rmul(wx[s1 + 3], s_g[m * D + s1 + 4]));
                    }
                    if (s1 <= NTAPS - 1 - m * D) v = cadd(v, rmul(wx[s1 - 1], s_g[m * D + s1]));
                    v = cadd(v, v2);
                }
                v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
                v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
                v.x += __shfl_xor_sync(0xffffffffu, v.x, 2);
                v.y += __shfl_xor_sync(0xffffffffu, v.y, 2);
                v = cmul(v, mk<C>((T)a.wre, (T)a.wim));
#pragma unroll
                for (int c = 0; c < PC_K; ++c) {
                    // output mb + c of this lane takes lane 4 (mb + c - mw) when that is in range
                    const int src = 4 * (mb + c - mw);
                    C got;
                    got.x = __shfl_sync(0xffffffffu, v.x, src & 31);
                    got.y = __shfl_sync(0xffffffffu, v.y, src & 31);
                    if (src >= 0 && src < 32 && mb + c < a.mwrap) acc[c] = cadd(acc[c], got);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < PC_K; ++c) acc[c] = cmul(acc[c], s_S[mb + c]);
        if constexpr (!FUSE) {
            C* zr = zb + b * z_stride + mb;
#pragma unroll
            for (int c = 0; c < PC_K; ++c) zr[c] = acc[c];
        } else if (p == 0) {
#pragma unroll
            for (int c = 0; c < PC_K; ++c) keep[c] = acc[c];
        } else {
            // the whole decimated record is in registers (keep: part 0, acc: part 1): through the part
            // buffer it was filtered from (now dead) into natural order, the 512-point transform by this
            // warp (32 threads x 16), then the signed band bins x the band factor (zoomfft.cpp:208-235)
            using G = FftGeom<9>;
            C* fsm = reinterpret_cast<C*>(bufs + slot * BUF);
            __syncwarp();
#pragma unroll
            for (int c = 0; c < PC_K; ++c) {
                fsm[pad16(lane * PC_K + c)] = keep[c];
                fsm[pad16(PC_PART + lane * PC_K + c)] = acc[c];
            }
            __syncwarp();
            C v[G::EPT];
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) v[q] = fsm[pad16(lane + G::NT * q)];
            __syncwarp();
            block_fft<false, 9, 16, 16, C, WarpSync>(v, fsm, tws, lane, true, WarpSync{});
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) fsm[pad16(lane + G::NT * q)] = v[q];
            __syncwarp();
            C* o = out + b * out_stride;
            for (int i = lane; i < a.nbins; i += 32) {
                const int kb = a.k_lo + i;
                const int idx = ((kb % G::L) + G::L) % G::L;
                o[i] = cmul(fsm[pad16(idx)], __ldg(band + i));
            }
        }
        __syncwarp();   // the buffer is refilled by a later item
    }
}

template <typename T, int D, int NTAPS>
size_t pc_smem(const ZoomArgs& a, int nw, bool fuse) {
    constexpr int WTP = (NTAPS - 1 + 3) / 4 * 4;
    return ((size_t)(a.nout + NTAPS) * sizeof(cx_t<T>) + (size_t)nw * pc_nbuf<T>() * WTP * sizeof(T) + 15) / 16 * 16 +
           (size_t)nw * pc_nbuf<T>() * D * PcGeom<T>::PSE * sizeof(T) +
           (fuse ? (size_t)FftGeom<9>::TW_ALLOC * sizeof(cx_t<T>) : 0);
}

template <typename T, int D, int NTAPS>
cudaError_t run_pcfir(const ZoomArgs& a, const T* x, long long xs, long long batch, const void* gnat_host,
                      const void* S, void* zb, long long z_stride, bool fuse, const void* tw, const void* band,
                      void* out, long long out_stride, cudaStream_t st) {
    using C = cx_t<T>;
    PcTaps<T, NTAPS> tp;
    const double* gh = static_cast<const double*>(gnat_host);   // fp64 natural-order taps
    for (int t = 0; t < NTAPS; ++t) {
        tp.g[t].x = (T)gh[2 * t];
        tp.g[t].y = (T)gh[2 * t + 1];
    }
    const int nw = pc_warps<T>();
    const size_t smem = pc_smem<T, D, NTAPS>(a, nw, fuse);
    int dev = 0, optin = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (smem > (size_t)optin) return cudaErrorNotSupported;
    auto launch = [&](auto kern) -> cudaError_t {
        cudaError_t e = prep_smem(kern, smem);
        if (e != cudaSuccess) return e;
        long long grid = std::min<long long>((batch + nw - 1) / nw, sms);
        if (const unsigned gc = grid_cap(); gc && gc < grid) grid = gc;
        kern<<<(unsigned)grid, nw * 32, smem, st>>>(x, xs, batch, a, tp, (const C*)S, (C*)zb, z_stride, (const C*)tw,
                                                     (const C*)band, (C*)out, out_stride);
        return cudaGetLastError();
    };
    return fuse ? launch(k_zoom_pcfir<T, D, NTAPS, true>) : launch(k_zoom_pcfir<T, D, NTAPS, false>);
}

}  // namespace

bool zoom_pcfir_fits(const ZoomArgs& a, bool f32) {
    static const bool off = std::getenv("SKG_ZOOM_NO_PCFIR") != nullptr;
    if (off || !a.circular || a.trim != 0 || a.nout % PC_PART || (long long)a.nout * a.D != a.U || a.n < a.U) return false;
    if (a.mwrap > PC_PART) return false;
    (void)f32;
    switch (a.D * 1000 + a.T) {
        case 8065: case 8101: return true;   // D = 16 part buffers do not fit twice per warp
        default: return false;
    }
}

// the FIR and the n_fft = 512 transform + band in one launch: nout = 512 (two parts)
bool zoom_pcfir_fused_fits(const ZoomArgs& a, bool f32, int log2n) {
    static const bool off = std::getenv("SKG_ZOOM_NO_FUSE") != nullptr;
    return !off && log2n == 9 && a.nout == 2 * PC_PART && zoom_pcfir_fits(a, f32);
}

cudaError_t launch_zoom_pcfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                              const void* gnat_host, const void* S, void* zb, long long z_stride, bool fuse,
                              const void* tw, const void* band, void* out, long long out_stride, cudaStream_t st) {
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        const T* xt = static_cast<const T*>(x);
        switch (a.D * 1000 + a.T) {
            case 8065:
                return run_pcfir<T, 8, 65>(a, xt, xs, batch, gnat_host, S, zb, z_stride, fuse, tw, band, out, out_stride, st);
            case 8101:
                return run_pcfir<T, 8, 101>(a, xt, xs, batch, gnat_host, S, zb, z_stride, fuse, tw, band, out, out_stride,
                                            st);
            default: return cudaErrorNotSupported;
        }
    };
    return f32 ? go(float{}) : go(double{});
}

}  // namespace skg
