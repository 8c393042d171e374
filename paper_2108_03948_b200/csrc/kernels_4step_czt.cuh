// kernels_4step_czt.cuh — the multi-pass Bluestein CZT (CztPlan::execute, czt.cpp:116-130, convolution
// lengths beyond one CTA) as ONE persistent cooperative launch with the work rows in an L2-resident ring.
//
// The three-launch path (kernels_4step.cuh: column pass, row kernel with the Bluestein middle, inverse
// column pass) moves a trace's L-point work buffer through HBM four times (written, read + written, read):
// 4 L 2s bytes against N s + M 2s of algorithmic traffic. Here the units of the three passes form one
// sequence — step s holds the forward column units of trace s, the row units of trace s - delta and the
// inverse column units of trace s - 2 delta — walked by a grid of co-resident CTAs with stride gridDim.x
// (see kernels_4step_real.cuh for the scheme and its deadlock argument). A trace's work rows live in slot
// (trace mod slots) of a ring that stays in L2; release/acquire counters order the passes:
//   row unit of t            waits for a_done[t]  (all forward column units of t stored)
//   inverse column unit of t waits for b_done[t]  (all row units of t stored)
//   forward column unit of t waits for c_done[t - slots] (the slot's previous trace fully read)
// Unit bodies = the bodies of k4_col / k4_row<MODE 1>, with ld.cg reads of the ring (an L1 line could be
// a stale copy of the slot's previous trace) and streaming stores of the result.
#pragma once

#include "kernels_4step_real.cuh"

namespace skg {

#ifndef SKG_CZTF_THREADS_F64
#define SKG_CZTF_THREADS_F64 512   // resident threads per SM the fp64 register cap targets
#endif
#ifndef SKG_CZTF_MINB_F32
#define SKG_CZTF_MINB_F32 4   // 64 registers, 4 CTAs of 256 threads per SM: L = 2^15 rows 5.9 -> 5.2 ms (3: 80 registers; 2: 7.0 ms)
#endif
// exchange barrier of a row transform under the row-major mapping: the NT threads of a row are a warp or
// part of one (NT <= 32: __syncwarp), else a named barrier per row (ids 1.., 0 is __syncthreads)
struct RowWarpSync {
    __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
template <typename T, int LR, int LC> struct CztFusedCfg {
    using GR = FftGeom<LR>;
    using GC = FftGeom<LC>;
    static constexpr int BMIN = sizeof(T) == 8 ? 128 : 256;
    static constexpr int WA0 = BMIN / GR::NT > Tile<T>::W ? BMIN / GR::NT : Tile<T>::W;   // columns per column unit
    static constexpr int BLOCK = GR::NT * WA0 > GC::NT * 4 ? GR::NT * WA0 : GC::NT * 4;
    static constexpr int WA = BLOCK / GR::NT;
    static constexpr int WB = BLOCK / GC::NT;             // rows per row unit
    static constexpr int WARPS = BLOCK / 32;
    static constexpr int NA = GC::L / WA;                 // column units per trace (each direction)
    static constexpr int NB = GR::L / WB;                 // row units per trace
    static constexpr int UPS = 2 * NA + NB;
    static constexpr size_t REG_A = (size_t)WA * (GR::SMEM + 1), REG_B = (size_t)WB * (GC::SMEM + 1);
    static constexpr size_t SMEM = ((REG_A > REG_B ? REG_A : REG_B) + GR::TW_ALLOC + GC::TW_ALLOC) * sizeof(cx_t<T>);
    static constexpr bool OK = GR::EPT == 16 && GC::EPT == 16 && BLOCK <= 1024 && GC::L % WA == 0 && GR::L % WB == 0 &&
                               SMEM <= 220 * 1024;
    static constexpr int MINB = sizeof(T) == 8 ? (SKG_CZTF_THREADS_F64 / BLOCK > 0 ? SKG_CZTF_THREADS_F64 / BLOCK : 1)
                                               : (BLOCK >= 512 ? 1 : SKG_CZTF_MINB_F32);
};

template <typename T, int LR, int LC, int NZ>
__global__ void __launch_bounds__(CztFusedCfg<T, LR, LC>::BLOCK, CztFusedCfg<T, LR, LC>::MINB)
k4_czt_fused(const void* __restrict__ xin, int complex_in, long long x_stride, long long N,
             const cx_t<T>* __restrict__ cin, cx_t<T>* Yring, int slots, int delta, long long batch,
             const cx_t<T>* __restrict__ twR, const cx_t<T>* __restrict__ twC, const cx_t<T>* __restrict__ twL,
             const cx_t<T>* __restrict__ khat_p, cx_t<T>* __restrict__ out, long long out_stride, long long M,
             const cx_t<T>* __restrict__ cout, unsigned* a_done, unsigned* b_done, unsigned* c_done) {
    using C = cx_t<T>;
    using F = CztFusedCfg<T, LR, LC>;
    using GR = typename F::GR;
    using GC = typename F::GC;
    constexpr long long Rn = GR::L, Cn = GC::L, L = Rn * Cn;
    extern __shared__ __align__(16) unsigned char smraw[];
    // column units: lane-interleaved (adjacent lanes = adjacent columns)
    const int g = threadIdx.x % F::WA, tid = threadIdx.x / F::WA;
    // row units: row-major (adjacent lanes = adjacent positions of one row)
    const int gb = threadIdx.x / GC::NT, tb = threadIdx.x % GC::NT;
    C* sm = reinterpret_cast<C*>(smraw) + g * (GR::SMEM + 1);
    C* smb = reinterpret_cast<C*>(smraw) + gb * (GC::SMEM + 1);
    C* twsR = reinterpret_cast<C*>(smraw) + (F::REG_A > F::REG_B ? F::REG_A : F::REG_B);
    C* twsC = twsR + GR::TW_ALLOC;
    load_twiddles<LR>(twsR, twR);
    load_twiddles<LC>(twsC, twC);
    const long long units = (batch + 2LL * delta) * F::UPS;
    // kind of a unit: 0 forward column, 1 row, 2 inverse column; its trace; -1: no work
    auto decode = [&](long long uu, long long& t, int& idx) -> int {
        if (uu >= units) return -1;
        const long long s = uu / F::UPS;
        const int j = (int)(uu % F::UPS);
        int kind;
        if (j < F::NA) {
            kind = 0, t = s, idx = j;
        } else if (j < F::NA + F::NB) {
            kind = 1, t = s - delta, idx = j - F::NA;
        } else {
            kind = 2, t = s - 2LL * delta, idx = j - F::NA - F::NB;
        }
        return t >= 0 && t < batch ? kind : -1;
    };
    auto dep = [&](int kind, long long t, unsigned& target) -> const unsigned* {
        if (kind == 0) {
            target = (unsigned)(F::NA * F::WARPS);
            return t >= slots ? c_done + (t - slots) : nullptr;
        }
        if (kind == 1) {
            target = (unsigned)(F::NA * F::WARPS);
            return a_done + t;
        }
        target = (unsigned)(F::NB * F::WARPS);
        return b_done + t;
    };
    bool ready = false;   // thread 0: this unit's dependency was seen satisfied during the previous unit
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        long long t;
        int idx;
        const int kind = decode(u, t, idx);
        if (kind < 0) {
            ready = false;
            continue;
        }
        if (threadIdx.x == 0) {
            unsigned target;
            const unsigned* d = dep(kind, t, target);
            if (d && !ready) wait_count(d, target);
        }
        __syncthreads();   // dependency satisfied; every thread has left the previous unit's shared memory
        if (threadIdx.x == 0) {   // peek at the next unit's dependency: the load is in flight during this unit
            long long tn;
            int in;
            const int kn = decode(u + gridDim.x, tn, in);
            ready = true;
            if (kn >= 0) {
                unsigned target;
                const unsigned* d = dep(kn, tn, target);
                if (d) ready = ld_acquire_u32(d) >= target;
            }
        }
        C* Yt = Yring + (t % slots) * L;
        C v[16];
        if (kind == 0) {
            // ---- forward column unit: x * chirp -> R-point transforms -> x W_L^{n2 k1} -> Y[k1][n2]
            const long long n2 = (long long)idx * F::WA + g;
            const C tw_a = __ldg(twL + (long long)tid * Cn + n2);
            const C tw_s = __ldg(twL + (long long)GR::NT * Cn + n2);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const long long n = (tid + (long long)GR::NT * q) * Cn + n2;
                C val = czero<C>();
                if (q < NZ && n < N) {
                    if (complex_in) val = __ldg(reinterpret_cast<const C*>(xin) + t * x_stride + n);
                    else val = mk<C>(__ldg(reinterpret_cast<const T*>(xin) + t * x_stride + n), (T)0);
                    val = cmul(val, __ldg(cin + n));
                }
                v[q] = val;
            }
            block_fft<false, LR, NZ>(v, sm, twsR, tid);
            twiddle_series(tw_a, tw_s, [&](int q, C w) { Yt[(tid + (long long)GR::NT * q) * Cn + n2] = cmul(v[q], w); });
            __syncwarp();
            if ((threadIdx.x & 31) == 0) red_release_inc(a_done + t);
        } else if (kind == 1) {
            // ---- row unit: FFT_C, x khat, IFFT_C, x conj W_L^{n2 k1}, in place
            const long long k1 = (long long)idx * F::WB + gb;
            C* row = Yt + k1 * Cn;
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = __ldcg(row + tb + GC::NT * q);
            const C* tl = twL + k1 * Cn;
            const C tw_a = __ldg(tl + tb), tw_s = __ldg(tl + GC::NT);
            const C* kp = khat_p + k1 * Cn;
            // the kernel-spectrum row into L1 while the forward transform runs (an L2 round trip otherwise
            // waited for between the two transforms)
#pragma unroll
            for (int q = 0; q < 16; ++q) prefetch_l1(kp + tb + GC::NT * q);
            if constexpr (GC::NT <= 32) {
                block_fft<false, LC, 16, 16, C, RowWarpSync>(v, smb, twsC, tb, true, RowWarpSync());
            } else {
                block_fft<false, LC, 16, 16, C, GroupSync>(v, smb, twsC, tb, true, GroupSync{1 + gb, GC::NT});
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = cmul(v[q], __ldg(kp + tb + GC::NT * q));
            if constexpr (GC::NT <= 32) {
                block_fft<true, LC, 16, 16, C, RowWarpSync>(v, smb, twsC, tb, true, RowWarpSync());
            } else {
                block_fft<true, LC, 16, 16, C, GroupSync>(v, smb, twsC, tb, true, GroupSync{1 + gb, GC::NT});
            }
            twiddle_series(tw_a, tw_s, [&](int q, C w) { row[tb + GC::NT * q] = cmulc(v[q], w); });
            __syncwarp();
            if ((threadIdx.x & 31) == 0) red_release_inc(b_done + t);
        } else {
            // ---- inverse column unit: IFFT_R over k1 -> x output chirp -> out[n], n = C n1 + n2 < M
            const long long n2 = (long long)idx * F::WA + g;
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = __ldcg(Yt + (tid + (long long)GR::NT * q) * Cn + n2);
#pragma unroll
            for (int q = 0; q < 16; ++q) {   // the output chirp into L1 while the transform runs
                const long long n = (tid + (long long)GR::NT * q) * Cn + n2;
                if (n < M && g % (128 / (int)sizeof(C)) == 0) prefetch_l1(cout + n);
            }
            block_fft<true, LR>(v, sm, twsR, tid);
            // the first exchange of the transform consumed every load: the slot is free
            __syncwarp();
            if ((threadIdx.x & 31) == 0) red_release_inc(c_done + t);
            C* o = out + t * out_stride;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const long long n = (tid + (long long)GR::NT * q) * Cn + n2;
                if (n < M) __stcs(o + n, cmul(v[q], __ldg(cout + n)));
            }
        }
    }
}

template <typename T>
cudaError_t launch_4step_czt_fused_impl(int lR, int lC, const void* x, int complex_in, long long x_stride, long long N,
                                        const void* cin, void* Yring, int slots, int delta, long long batch,
                                        const void* twR, const void* twC, const void* twL, const void* khat_p, void* out,
                                        long long out_stride, long long M, const void* cout, unsigned* counters,
                                        int* grid_out, int* ups_out, cudaStream_t st) {
    using C = cx_t<T>;
    auto run = [&](auto lr, auto lc) -> cudaError_t {
        constexpr int LR = decltype(lr)::value, LC = decltype(lc)::value;
        using F = CztFusedCfg<T, LR, LC>;
        if constexpr (!F::OK) {
            return cudaErrorInvalidValue;
        } else {
            auto launch = [&](auto kern) {
                cudaError_t e = prep_smem(kern, F::SMEM);
                if (e != cudaSuccess) return e;
                const unsigned grid = persistent_grid(kern, F::BLOCK, F::SMEM, 1LL << 40);
                if (grid_out) {
                    *grid_out = (int)grid;
                    *ups_out = F::UPS;
                    return cudaSuccess;
                }
                const C* cinp = (const C*)cin;
                C* yp = (C*)Yring;
                const C *twr = (const C*)twR, *twc = (const C*)twC, *twl = (const C*)twL, *kp = (const C*)khat_p;
                C* op = (C*)out;
                const C* coutp = (const C*)cout;
                unsigned *a = counters, *b = counters + batch, *c = counters + 2 * batch;
                void* args[] = {&x, &complex_in, &x_stride, &N, &cinp, &yp, &slots, &delta, &batch, &twr, &twc,
                                &twl, &kp, &op, &out_stride, &M, &coutp, &a, &b, &c};
                return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(F::BLOCK), args, F::SMEM, st);
            };
            const int nz = LR >= 8 ? nz_class((N + (1LL << LC) - 1) >> LC, F::GR::NT) : 16;
            if (nz == 4) return launch(k4_czt_fused<T, LR, LC, 4>);
            if (nz == 8) return launch(k4_czt_fused<T, LR, LC, 8>);
            return launch(k4_czt_fused<T, LR, LC, 16>);
        }
    };
    if (lC == lR) return dispatch_log2<7, 9>(lR, [&](auto lr) { return run(lr, lr); });
    if (lC == lR + 1)
        return dispatch_log2<7, 9>(lR, [&](auto lr) { return run(lr, IC<decltype(lr)::value + 1>{}); });
    return cudaErrorInvalidValue;
}

}  // namespace skg
