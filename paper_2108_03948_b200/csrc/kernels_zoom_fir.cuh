// kernels_zoom_fir.cuh — the phase-lane polyphase FIR task shared by the zoom split route
// (kernels_zoom.cu) and the fused FIR + FFT kernel (kernels_zoom_fused.cu).
#pragma once

#include "fft_device.cuh"
#include "kernels.hpp"

namespace skg {

#ifndef SKG_PFIR_MINB64
// fp64 CTAs per SM the register cap targets: 4 (128 registers) where that spills nothing — D <= 8
// with <= 10-tap phase rows, cfg3: 0.102 -> 0.097 ms per call — else 3
#define SKG_PFIR_MINB64(D, LH) ((D) <= 8 && (LH) <= 10 ? 4 : 3)
#endif
#ifndef SKG_PFIR_MINB32
#define SKG_PFIR_MINB32 4
#endif
// One warp task of the phase-lane FIR: outputs [mw0, mw0 + G gchunk) of record task / tasks_per_rec,
// each finished output handed to store(record, m, value). Shared by the split route's FIR kernel
// (store -> L2 work rows) and the fused FIR + FFT kernel (store -> shared-memory record slot).
template <typename T, int D, int LH, typename Store>
__device__ __forceinline__ void pfir_task(const T* __restrict__ x, long long x_stride, const ZoomArgs& a, int gchunk,
                                          int tasks_per_rec, long long task, long long ntasks, long long tstride,
                                          const cx_t<T> (&tp)[LH], const cx_t<T>* __restrict__ gnat,
                                          const cx_t<T>* __restrict__ S, cx_t<T>* cw, cx_t<T>* red, Store&& store) {
    using C = cx_t<T>;
    constexpr int G = 32 / D;              // groups per warp
    constexpr int MB = D > 8 ? D : 8;      // outputs per mini-batch
    constexpr int K = MB / D;              // finished outputs per lane per mini-batch
    const int lane = threadIdx.x & 31;
    const int ph = lane % D, g = lane / D;
    const int delta = ph != 0;
    const int U = (int)a.U;
    const int nout = a.nout, trim = a.trim, mwrap = a.mwrap;
        const long long b = task / tasks_per_rec;
        const int tk = (int)(task % tasks_per_rec);
        const T* xr = x + b * x_stride;
        const int mw0 = tk * G * gchunk;               // first decimated output of the warp task
        const int m0 = mw0 + g * gchunk;               // of this lane's group
        const int mf0 = m0 + a.trim;
        // wrap correction (circular) for task outputs below mwrap (half-warps own outputs)
        const bool wraps = a.circular && mw0 + a.trim < a.mwrap;
        // the warp's next task input is pulled into L2 while this one runs
        {
            const long long tn = task + tstride;
            if (tn < ntasks) {
                const T* xn = x + (tn / tasks_per_rec) * x_stride;
                const int mwn = (int)(tn % tasks_per_rec) * G * gchunk + a.trim;
                const int n_lo = max((mwn - LH) * D, 0), n_hi = min((mwn + G * gchunk) * D, U);
                for (int n = n_lo + lane * (128 / (int)sizeof(T)); n < n_hi; n += 32 * (128 / (int)sizeof(T)))
                    prefetch_l2(xn + n);
            }
        }
        if (wraps) {
            const int h = lane >> 4, hl = lane & 15;
            for (int mm = mw0 + a.trim; mm < min(a.mwrap, mw0 + a.trim + G * gchunk); mm += 2) {
                const int m = mm + h;
                C acc = czero<C>();
                if (m < a.mwrap)
                    for (int s1 = 1 + hl; s1 <= a.T - 1 - m * D; s1 += 16)
                        acc = cadd(acc, rmul(__ldg(xr + U - s1), __ldg(gnat + m * D + s1)));
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                }
                if (hl == 0 && m < a.mwrap) cw[m] = cmul(acc, mk<C>((T)a.wre, (T)a.wim));
            }
            __syncwarp();
        }
        // samples of this lane's phase row: x[r D + ph] = xp[r D], zero outside the record
        const T* xp = xr + ph;
        const int r_end = (U - ph + D - 1) / D;   // rows r < r_end exist (r D + ph < U)
#ifdef SKG_PFIR_NOLOAD   // microbenchmark: the FIR / reduction without the sample loads
        auto sample = [&](int r) -> T { return (r >= 0 && r < r_end) ? (T)(r * 1e-3) : (T)0; };
#else
        auto sample = [&](int r) -> T { return (r >= 0 && r < r_end) ? __ldg(xp + r * D) : (T)0; };
#endif
        // window buf[i] <-> row mf - (LH - 1) - delta + i for the mini-batch starting at output mf;
        // the next two mini-batches' samples are in flight (nx1, nx2)
        T buf[LH - 1 + MB];
#pragma unroll
        for (int i = 0; i < LH - 1; ++i) buf[i] = sample(mf0 - (LH - 1) - delta + i);
        T nx1[MB], nx2[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) nx1[j] = sample(mf0 - delta + j);
#pragma unroll
        for (int j = 0; j < MB; ++j) nx2[j] = sample(mf0 + MB - delta + j);
        for (int mb = 0; mb < gchunk; mb += MB) {
            const int mf = mf0 + mb;
#pragma unroll
            for (int j = 0; j < MB; ++j) {
                buf[LH - 1 + j] = nx1[j];
                nx1[j] = nx2[j];
            }
            if (mb + 2 * MB < gchunk) {
#pragma unroll
                for (int j = 0; j < MB; ++j) nx2[j] = sample(mf + 2 * MB - delta + j);
            }
            // even and odd taps accumulate separately: four FMA chains per output, so the
            // compiler's two-outputs-at-a-time schedule still has eight chains in flight
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
            // sum over the D phase-lanes of the group through shared memory: lane (g, ph) posts its
            // MB partials, then finishes outputs ph K + j (j < K) from the D phase partials
            C* rg = red + g * MB * (D + 1);
#pragma unroll
            for (int j = 0; j < MB; ++j) rg[j * (D + 1) + ph] = P[j];
            __syncwarp();
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const int jj = ph * K + j;
                C v = rg[jj * (D + 1)];
#pragma unroll
                for (int q = 1; q < D; ++q) v = cadd(v, rg[jj * (D + 1) + q]);
                const int m = m0 + mb + jj;   // decimated index
                if (m < nout) {
                    const int mfo = m + trim;
                    if (wraps && mfo < mwrap) v = cadd(v, cw[mfo]);
                    store(b, m, cmul(v, __ldg(S + m)));
                }
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < LH - 1; ++i) buf[i] = buf[i + MB];
        }
        __syncwarp();   // cw reuse by the next task
}

}  // namespace skg
