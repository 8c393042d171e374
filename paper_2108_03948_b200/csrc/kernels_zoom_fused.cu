// kernels_zoom_fused.cu — the zoom split route's FIR and short FFT in ONE kernel:
// the phase-lane FIR of kernels_zoom.cu writes each record's decimated block into a shared-memory
// record slot instead of the L2 work rows, and the CTA — whose four warps cover whole records —
// then runs the n_fft-point Stockham transform on those slots and stores the signed band window
// (x D x group-delay phase). One launch, no work-row round trip; the FIR is the same code.
#include <cstdlib>

#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"

#ifndef SKG_PFIR_MINB64
#define SKG_PFIR_MINB64(D, LH) ((D) <= 8 && (LH) <= 10 ? 4 : 3)
#endif
#ifndef SKG_PFIR_MINB32
#define SKG_PFIR_MINB32 4
#endif
#ifndef SKG_ZF_MINB64
#define SKG_ZF_MINB64 4
#endif

namespace skg {

// a tap load the compiler may not hoist out of the task loop (volatile asm): keeps the taps' live
// range inside the FIR phase, so the FFT phase gets their registers
__device__ __forceinline__ double2 ld_tap(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ float2 ld_tap(const float2* p) {
    float2 v;
    asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

template <typename T, int D, int LH, int LOG2N>
__global__ void __launch_bounds__(128, sizeof(T) == 8 ? SKG_ZF_MINB64 : SKG_PFIR_MINB32)
k_zoom_pfir_fft(const T* __restrict__ x, long long x_stride, long long batch, ZoomArgs a, int gchunk, int tasks_per_rec,
            const cx_t<T>* __restrict__ gph, const cx_t<T>* __restrict__ gnat, const cx_t<T>* __restrict__ S,
            const cx_t<T>* __restrict__ tw, int k_lo, int nbins, const cx_t<T>* __restrict__ band,
            cx_t<T>* __restrict__ out, long long out_stride) {
    using C = cx_t<T>;
    constexpr int G = 32 / D;              // groups per warp
    constexpr int MB = D > 8 ? D : 8;      // outputs per mini-batch
    constexpr int K = MB / D;              // finished outputs per lane per mini-batch
    extern __shared__ __align__(16) unsigned char smraw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ph = lane % D, g = lane / D;
    const int delta = ph != 0;
    const int U = (int)a.U;
    // per warp: [wrap terms (mwrap + 1)][phase partials G x MB x (D + 1) (padded: conflict-free reads)]
    using FG = FftGeom<LOG2N>;
    constexpr int RSM = FG::L >= 16 ? FG::SMEM : FG::L;   // record buffer (padded Stockham layout)
    C* cw = reinterpret_cast<C*>(smraw) + warp * (a.mwrap + 1 + G * MB * (D + 1));
    C* red = cw + (a.mwrap + 1);
    C* recs = reinterpret_cast<C*>(smraw) + 4 * (a.mwrap + 1 + G * MB * (D + 1));   // RPC record buffers
    C* tws = recs + 4 * RSM;
    if constexpr (FG::L >= 16) load_twiddles<LOG2N>(tws, tw);
    __syncthreads();
    const int rpc = 4 / tasks_per_rec;          // records per CTA iteration
    const int slot = warp / tasks_per_rec;      // this warp's record slot
    auto ridx = [&](int m) { return FG::L >= 16 ? pad16(m) : m; };
    const int nout = a.nout, trim = a.trim, mwrap = a.mwrap;
    // this phase row's taps (rows are zero padded to a.lh >= LH entries... or shorter: guard)
    const long long ntasks = batch * tasks_per_rec;
    const long long tstride = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long tbase = (long long)blockIdx.x * (blockDim.x >> 5); tbase < ntasks; tbase += tstride) {
      const long long task = tbase + warp;
      const bool has_task = task < ntasks;
      if (has_task) {
        // this phase row's taps, re-read (L1) every task so they are not live across the FFT phase
        C tp[LH];
#pragma unroll
        for (int l = 0; l < LH; ++l) {
            tp[l] = czero<C>();
            if (l < a.lh) tp[l] = ld_tap(gph + ph * a.lh + l);
        }
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
                    recs[slot * RSM + ridx(m)] = cmul(v, __ldg(S + m));
                }
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < LH - 1; ++i) buf[i] = buf[i + MB];
        }
        __syncwarp();   // cw reuse by the next task
      }
        // every warp's decimated block is in its record slot: the short FFT (zero padded to n_fft),
        // GROUPS_F records at a time, then the signed band gather x D x group-delay phase
        __syncthreads();
        constexpr int GF = FG::NT >= 128 ? 1 : 128 / FG::NT;
        const int fg = threadIdx.x / FG::NT, ftid = threadIdx.x % FG::NT;
        const int nvalid = nout < FG::L ? nout : FG::L;
        for (int r0 = 0; r0 < rpc; r0 += GF) {
            const int r = r0 + fg;
            const long long rb = tbase / tasks_per_rec + r;   // record of this slot
            const bool act = fg < GF && r < rpc && rb < batch;
            C* rs = recs + (act ? r : 0) * RSM;
            C v[FG::EPT];
#pragma unroll
            for (int q = 0; q < FG::EPT; ++q) {
                const int pos = ftid + FG::NT * q;
                v[q] = (act && pos < nvalid) ? rs[ridx(pos)] : czero<C>();
            }
            __syncthreads();   // the record buffers double as the transforms' exchange buffers
            block_fft<false, LOG2N>(v, rs, tws, ftid, act);
            if (act) {
#pragma unroll
                for (int q = 0; q < FG::EPT; ++q) rs[ridx(ftid + FG::NT * q)] = v[q];
            }
            __syncthreads();
            if (act) {
                C* o = out + rb * out_stride;
                for (int i = ftid; i < nbins; i += FG::NT) {
                    const int kk = k_lo + i;
                    const int idx = ((kk % FG::L) + FG::L) % FG::L;
                    o[i] = cmul(rs[ridx(idx)], __ldg(band + i));
                }
            }
            __syncthreads();
        }
    }
}


namespace {
template <typename T, int D, int LH, int LOG2N>
cudaError_t run_pfir_fft(const ZoomArgs& a, const T* x, long long xs, long long batch, const void* gph, const void* gnat,
                         const void* S, const void* tw, int k_lo, int nbins, const void* band, void* out,
                         long long out_stride, cudaStream_t st) {
    using C = cx_t<T>;
    using FG = FftGeom<LOG2N>;
    constexpr int G = 32 / D;
    constexpr int MB = D > 8 ? D : 8;
    const int gchunk = std::max(MB, (std::min(64, (a.nout + G - 1) / G) + MB - 1) / MB * MB);
    const int tasks_per_rec = (a.nout + G * gchunk - 1) / (G * gchunk);
    if (4 % tasks_per_rec != 0) return cudaErrorNotSupported;
    constexpr int RSM = FG::L >= 16 ? FG::SMEM : FG::L;
    const size_t smem = (size_t)4 * (a.mwrap + 1 + G * MB * (D + 1)) * sizeof(C) + (size_t)4 * RSM * sizeof(C) +
                       (size_t)(FG::L >= 16 ? FG::TW_ALLOC : 0) * sizeof(C);
    if (smem > (size_t)smem_optin()) return cudaErrorNotSupported;
    auto kern = k_zoom_pfir_fft<T, D, LH, LOG2N>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long long ctas = (batch * tasks_per_rec + 3) / 4;
    kern<<<persistent_grid(kern, 128, smem, ctas), 128, smem, st>>>(x, xs, batch, a, gchunk, tasks_per_rec, (const C*)gph,
                                                                   (const C*)gnat, (const C*)S, (const C*)tw, k_lo,
                                                                   nbins, (const C*)band, (C*)out, out_stride);
    return cudaGetLastError();
}
}  // namespace

// Measured against the split route (tools/zoom_time.py, cfg3, 4096 records): fp32 n_fft 512 0.065 ->
// 0.062 ms; fp64 n_fft 512 0.094 -> 0.100 ms with the taps live across the FFT phase (168-register cap),
// 0.094 -> 0.096 ms with them re-read per task (128 registers; SKG_ZF_F64=1 enables it), n_fft 2048
// slower in both precisions (one 2048-point record at a time per CTA: fp64 0.124 -> 0.207 ms). So it is
// used for fp32 D = 8 with 9 / 10-tap rows and n_fft 512; everything else runs the split route.
cudaError_t launch_zoom_pfir_fft(const ZoomArgs& a, int lh, int log2n, bool f32, const void* x, long long xs,
                                 long long batch, const void* gph, const void* gnat, const void* S, const void* tw,
                                 int k_lo, int nbins, const void* band, void* out, long long out_stride,
                                 cudaStream_t st) {
    if (a.D != 8 || (lh != 9 && lh != 10) || log2n != 9) return cudaErrorNotSupported;
    static const bool f64_on = std::getenv("SKG_ZF_F64") != nullptr;
    if (!f32 && !f64_on) return cudaErrorNotSupported;
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        const T* xt = static_cast<const T*>(x);
        if (lh == 9)
            return run_pfir_fft<T, 8, 9, 9>(a, xt, xs, batch, gph, gnat, S, tw, k_lo, nbins, band, out, out_stride, st);
        return run_pfir_fft<T, 8, 10, 9>(a, xt, xs, batch, gph, gnat, S, tw, k_lo, nbins, band, out, out_stride, st);
    };
    return f32 ? go(float{}) : go(double{});
}

}  // namespace skg
