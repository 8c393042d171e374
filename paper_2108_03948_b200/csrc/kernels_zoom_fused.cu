// kernels_zoom_fused.cu — the zoom split route's FIR and short FFT in ONE kernel:
// the phase-lane FIR of kernels_zoom.cu writes each record's decimated block into a shared-memory
// record slot instead of the L2 work rows, and the CTA — whose four warps cover whole records —
// then runs the n_fft-point Stockham transform on those slots and stores the signed band window
// (x D x group-delay phase). One launch, no work-row round trip; the FIR is the same code.
#include <cstdlib>

#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"
#include "kernels_zoom_fir.cuh"

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
    using FG = FftGeom<LOG2N>;
    constexpr int G = 32 / D;
    constexpr int MB = D > 8 ? D : 8;
    constexpr int RSM = FG::L >= 16 ? FG::SMEM : FG::L;   // record slot (padded Stockham layout)
    extern __shared__ __align__(16) unsigned char smraw[];
    const int warp = threadIdx.x >> 5, ph = (threadIdx.x & 31) % D;
    // per warp: [wrap terms (mwrap + 1)][phase partials G x MB x (D + 1)]; then 4 record slots, twiddles
    C* cw = reinterpret_cast<C*>(smraw) + warp * (a.mwrap + 1 + G * MB * (D + 1));
    C* red = cw + (a.mwrap + 1);
    C* recs = reinterpret_cast<C*>(smraw) + 4 * (a.mwrap + 1 + G * MB * (D + 1));
    C* tws = recs + 4 * RSM;
    if constexpr (FG::L >= 16) load_twiddles<LOG2N>(tws, tw);
    __syncthreads();
    const int rpc = 4 / tasks_per_rec;          // records per CTA iteration
    const int slot = warp / tasks_per_rec;      // this warp's record slot
    auto ridx = [&](int m) { return FG::L >= 16 ? pad16(m) : m; };
    const long long ntasks = batch * tasks_per_rec;
    const long long tstride = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long tbase = (long long)blockIdx.x * (blockDim.x >> 5); tbase < ntasks; tbase += tstride) {
        const long long task = tbase + warp;
        if (task < ntasks) {
            // this phase row's taps, re-read (L1) every task so they are not live across the FFT phase
            C tp[LH];
#pragma unroll
            for (int l = 0; l < LH; ++l) {
                tp[l] = czero<C>();
                if (l < a.lh) tp[l] = ld_tap(gph + ph * a.lh + l);
            }
            pfir_task<T, D, LH>(x, x_stride, a, gchunk, tasks_per_rec, task, ntasks, tstride, tp, gnat, S, cw, red,
                                [&](long long, int m, C v) { recs[slot * RSM + ridx(m)] = v; });
        }
        // every warp's decimated block is in its record slot: the short FFT (zero padded to n_fft),
        // GROUPS_F records at a time, then the signed band gather x D x group-delay phase
        __syncthreads();
        constexpr int GF = FG::NT >= 128 ? 1 : 128 / FG::NT;
        const int fg = threadIdx.x / FG::NT, ftid = threadIdx.x % FG::NT;
        const int nvalid = a.nout < FG::L ? a.nout : FG::L;
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
