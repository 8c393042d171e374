// kernels_zoom_cfir.cu — Zoom FIR with the taps in the constant bank (zoom_fft's
// filter_decimate_circular, zoomfft.cpp:82-104, refactored as in kernels_zoom.cu:
// u[m] = S[m] * sum_t g[t] x[mD - t], complex taps g, real samples).
//
// For the tap counts that matter (the reference default 101 and cfg3's 65) the kernel is
// specialised on (D, T): the whole polyphase loop is unrolled, so every tap is a compile-time
// offset into the kernel-parameter constant bank and feeds the DFMA/FFMA directly as a constant
// operand — no tap loads at all, and the FMA pipe runs at its constant-operand rate (a
// microbenchmark, tools/micro/fp64_regs.cu, measures 31.8 TF/s fp64 this way against 22-26 TF/s
// with three register operands). Each warp owns 32*WZK consecutive outputs of one record and its
// own polyphase window in shared memory (swizzled rows, no padding); lanes slide a WZK-sample
// register window along each phase row: one shared load per tap feeds 2*WZK FMAs.
#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"
#include "bulk_copy.cuh"

namespace skg {

namespace {

constexpr int CF_WARPS = 4;
constexpr int CZK = 4;   // window refill granularity (the row prefix is a multiple of it)

template <int D> __host__ __device__ constexpr int cf_wzk() { return D >= 16 ? 4 : 8; }   // outputs per lane

__device__ __forceinline__ int csw(int p) { return p ^ ((p >> 4) & 7); }

template <typename T, int D, int NTAPS> struct CTaps {
    static constexpr int LH = (NTAPS + D - 1) / D;   // longest phase row
    cx_t<T> g[D * LH];                              // g[ph * LH + l] = tap l D + (D - ph) % D (0 past T)
};

template <int D> int cf_rs(const ZoomArgs& a) {
    // positions 0..span are written; the swizzle permutes within aligned groups of 8, so a row needs
    // (span | 7) + 1 slots; the stride is then kept = 2 (mod 16) (the pair scatter stays conflict free)
    const int need = ((a.pre + 32 * cf_wzk<D>() + 2 * CZK) | 7) + 1;
    int rs = (need + 15) / 16 * 16 + 2;
    if (rs - 16 >= need) rs -= 16;
    return rs;
}

template <typename T, int D, int NTAPS>
__global__ void __launch_bounds__(CF_WARPS * 32, 3)
k_zoom_cfir(const T* __restrict__ x, long long x_stride, long long batch, ZoomArgs a, int wchunks, int wrs, int wbytes,
            const __grid_constant__ CTaps<T, D, NTAPS> tp, const cx_t<T>* __restrict__ gnat,
            const cx_t<T>* __restrict__ S, cx_t<T>* __restrict__ zb, long long z_stride) {
    using C = cx_t<T>;
    constexpr int LH = CTaps<T, D, NTAPS>::LH;
    constexpr int WZK = cf_wzk<D>();
    constexpr int WOUT = 32 * WZK;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int U = (int)a.U;
    unsigned char* wr = smraw + (size_t)warp * wbytes;
    C* cw = reinterpret_cast<C*>(wr);
    T* xs = reinterpret_cast<T*>(cw + (a.mwrap + 1));
    const long long ntasks = batch * wchunks;
    const long long tstride = (long long)gridDim.x * CF_WARPS;
    const int span = a.pre + WOUT + 2 * CZK;
    const int ntot = span * D;
    for (long long task = (long long)blockIdx.x * CF_WARPS + warp; task < ntasks; task += tstride) {
        const long long b = task / wchunks;
        const int ck = (int)(task % wchunks);
        const T* xr = x + b * x_stride;
        const int m_lo = ck * WOUT;
        const int mf_lo = m_lo + a.trim;
        const int r_lo = mf_lo - a.pre;
        const int n0 = r_lo * D;
        // the next task's window is pulled into L2 while this one is filtered
        {
            const long long tn = task + tstride;
            if (tn < ntasks) {
                const T* xn = x + (tn / wchunks) * x_stride;
                const int nn0 = max(((int)(tn % wchunks) * WOUT + a.trim - a.pre) * D, 0);
                const int nn1 = min(nn0 + ntot, U);
                for (int n = nn0 + lane * (128 / (int)sizeof(T)); n < nn1; n += 32 * (128 / (int)sizeof(T)))
                    prefetch_l2(xn + n);
            }
        }
        C sv[WZK];
#pragma unroll
        for (int c = 0; c < WZK; ++c) {
            const int m = m_lo + lane * WZK + c;
            sv[c] = m < a.nout ? __ldg(S + m) : czero<C>();
        }
        // record -> polyphase window: xs[ph wrs + csw(r - r_lo + (ph != 0))] = x[r D + ph], 0 outside [0, U)
        {
            constexpr int V = 16 / (int)sizeof(T);
            // loads in flight per lane before the first store: a window is ~34 (fp64) / ~17 (fp32)
            // 16-byte loads per lane, so this takes three rounds of memory latency, not nine
            constexpr int UNR = sizeof(T) == 8 ? 12 : 8;
            using VT = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
            const bool vec = (D % V) == 0 && ((uintptr_t)xr % 16) == 0;   // n0 is a multiple of D
            if (vec) {
                const int nv = ntot / V;
                for (int i0 = lane; i0 < nv; i0 += 32 * UNR) {
                    VT buf[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int n = n0 + (i0 + 32 * u) * V;
                        T* e = reinterpret_cast<T*>(&buf[u]);
                        if (i0 + 32 * u < nv && n >= 0 && n + V <= U) {
#ifdef SKG_CFIR_NOLOAD   // microbenchmark: the kernel without its record loads
#pragma unroll
                            for (int k = 0; k < V; ++k) e[k] = (T)((n + k) * 1e-3);
#else
                            buf[u] = __ldg(reinterpret_cast<const VT*>(xr + n));
#endif
                        } else {
#pragma unroll
                            for (int k = 0; k < V; ++k) e[k] = (n + k >= 0 && n + k < U) ? __ldg(xr + n + k) : (T)0;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int i = i0 + 32 * u;
                        if (i < nv) {
                            const T* e = reinterpret_cast<const T*>(&buf[u]);
                            const int n = n0 + i * V;
                            const int ph = (n - n0) % D;   // n0 = r_lo D
                            const int r = r_lo + (n - n0) / D;
#pragma unroll
                            for (int k = 0; k < V; ++k)
                                xs[(ph + k) * wrs + csw(r - r_lo + ((ph + k) != 0))] = e[k];
                        }
                    }
                }
            } else {
                for (int i0 = lane; i0 < ntot; i0 += 32 * UNR) {
                    T buf[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int n = n0 + i0 + 32 * u;
                        buf[u] = (i0 + 32 * u < ntot && n >= 0 && n < U) ? __ldg(xr + n) : (T)0;
                    }
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int i = i0 + 32 * u;
                        if (i < ntot) {
                            const int ph = i % D, rr = i / D;
                            xs[ph * wrs + csw(rr + (ph != 0))] = buf[u];
                        }
                    }
                }
            }
        }
        // wrap correction (circular): cw[m] = w * sum_{s=1}^{T-1-mD} g[mD + s] x[U - s], m < mwrap
        const bool wraps = a.circular && mf_lo < a.mwrap;
        if (wraps) {
            const int h = lane >> 4, hl = lane & 15;
            for (int m0 = mf_lo; m0 < min(a.mwrap, mf_lo + WOUT); m0 += 2) {
                const int m = m0 + h;
                C acc = czero<C>();
                if (m < a.mwrap)
                    for (int s1 = 1 + hl; s1 <= NTAPS - 1 - m * D; s1 += 16)
                        acc = cadd(acc, rmul(__ldg(xr + U - s1), __ldg(gnat + m * D + s1)));
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                }
                if (hl == 0 && m < a.mwrap) cw[m - mf_lo] = cmul(acc, mk<C>((T)a.wre, (T)a.wim));
            }
        }
        __syncwarp();
        // FIR, fully unrolled over (phase row, tap): taps are constant-bank operands
        C acc[WZK];
#pragma unroll
        for (int c = 0; c < WZK; ++c) acc[c] = czero<C>();
        const int base = a.pre + lane * WZK;   // a multiple of 4 (pre = lh + 4, lh a multiple of 4)
#pragma unroll
        for (int ph = 0; ph < D; ++ph) {
            const int t0 = ph ? D - ph : 0;
            const int cnt = t0 < NTAPS ? (NTAPS - t0 + D - 1) / D : 0;   // compile time after unrolling
            const T* row = xs + ph * wrs;
            T wv[WZK];
#pragma unroll
            for (int c = 0; c < WZK; ++c) wv[c] = row[csw(base + c)];
#pragma unroll
            for (int l = 0; l < LH; ++l) {
                if (l < cnt) {
                    const C g = tp.g[ph * LH + l];
#pragma unroll
                    for (int c = 0; c < WZK; ++c) {
                        acc[c].x = fma(g.x, wv[c], acc[c].x);
                        acc[c].y = fma(g.y, wv[c], acc[c].y);
                    }
                    if (l + 1 < cnt) {
#pragma unroll
                        for (int c = WZK - 1; c > 0; --c) wv[c] = wv[c - 1];
                        wv[0] = row[csw(base - l - 1)];
                    }
                }
            }
        }
        C* zr = zb + b * z_stride;
#pragma unroll
        for (int c = 0; c < WZK; ++c) {
            const int m = m_lo + lane * WZK + c;
            if (m < a.nout) {
                C v = acc[c];
                const int mf = m + a.trim;
                if (wraps && mf < a.mwrap) v = cadd(v, cw[mf - mf_lo]);
                zr[m] = cmul(v, sv[c]);
            }
        }
        __syncwarp();   // window / wrap-term reuse by the next task
    }
}

template <typename T, int D, int NTAPS>
cudaError_t run_cfir(const ZoomArgs& a, const T* x, long long xs, long long batch, const void* gph_host, const void* gnat,
                     const void* S, void* zb, long long z_stride, cudaStream_t st) {
    using C = cx_t<T>;
    using TP = CTaps<T, D, NTAPS>;
    constexpr int WOUT = 32 * cf_wzk<D>();
    // taps by phase row (host fp64 copy of the plan table, row stride a.lh) -> the constant-bank
    // parameter block of this launch
    TP tp;
    const double* gh = static_cast<const double*>(gph_host);
    for (int ph = 0; ph < D; ++ph)
        for (int l = 0; l < TP::LH; ++l) {
            const size_t i = (size_t)ph * a.lh + l;
            C v{};   // (host code: no device helpers here)
            if (l < a.lh) {
                v.x = (T)gh[2 * i];
                v.y = (T)gh[2 * i + 1];
            }
            tp.g[ph * TP::LH + l] = v;
        }
    const int wchunks = (a.nout + WOUT - 1) / WOUT;
    const int wrs = cf_rs<D>(a);
    const size_t wbytes = ((size_t)(a.mwrap + 1) * sizeof(C) + (size_t)D * wrs * sizeof(T) + 15) / 16 * 16;
    const size_t smem = wbytes * CF_WARPS;
    auto kern = k_zoom_cfir<T, D, NTAPS>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long long tasks = batch * wchunks;
    const unsigned grid = persistent_grid(kern, CF_WARPS * 32, smem, (tasks + CF_WARPS - 1) / CF_WARPS);
    kern<<<grid, CF_WARPS * 32, smem, st>>>(x, xs, batch, a, wchunks, wrs, (int)wbytes, tp, (const C*)gnat, (const C*)S,
                                           (C*)zb, z_stride);
    return cudaGetLastError();
}

}  // namespace

// the specialised (D, T) pairs: the reference's default 101 taps at the usual decimations and cfg3's 65
bool zoom_cfir_available(const ZoomArgs& a) {
    switch (a.D * 1000 + a.T) {
        case 8065: case 4065: case 16065: case 2101: case 3101: case 4101: case 5101: case 8101: case 16101:
            return a.trim >= 0;
        default: return false;
    }
}

cudaError_t launch_zoom_cfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                             const void* gph_host, const void* gnat, const void* S, void* zb, long long z_stride,
                             cudaStream_t st) {
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        const T* xt = static_cast<const T*>(x);
        switch (a.D * 1000 + a.T) {
            case 8065: return run_cfir<T, 8, 65>(a, xt, xs, batch, gph_host, gnat, S, zb, z_stride, st);
            case 4065: return run_cfir<T, 4, 65>(a, xt, xs, batch, gph_host, gnat, S, zb, z_stride, st);
            case 16065: return run_cfir<T, 16, 65>(a, xt, xs, batch, gph_host, gnat, S, zb, z_stride, st);
            case 2101: return run_cfir<T, 2, 101>(a, xt, xs, batch, gph_host, gnat, S, zb, z_stride, st);
            case 3101: return run_cfir<T, 3, 101>(a, xt, xs, batch, gph_host, gnat, S, zb, z_stride, st);
            case 4101: return run_cfir<T, 4, 101>(a, xt, xs, batch, gph_host, gnat, S, zb, z_stride, st);
            case 5101: return run_cfir<T, 5, 101>(a, xt, xs, batch, gph_host, gnat, S, zb, z_stride, st);
            case 8101: return run_cfir<T, 8, 101>(a, xt, xs, batch, gph_host, gnat, S, zb, z_stride, st);
            case 16101: return run_cfir<T, 16, 101>(a, xt, xs, batch, gph_host, gnat, S, zb, z_stride, st);
            default: return cudaErrorInvalidValue;
        }
    };
    return f32 ? go(float{}) : go(double{});
}

}  // namespace skg
