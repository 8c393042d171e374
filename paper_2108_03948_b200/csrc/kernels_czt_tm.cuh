// kernels_czt_tm.cuh — the shared-forward segmented Bluestein CZT (CztPlan::execute, czt.cpp:116-130)
// with its per-record tables and the parked spectrum in tensor memory.
//
// Same algorithm and operation order as k_czt_sf (kernels_impl.cuh): one forward FFT of the chirped
// record y = x·cin, then per output block s the product with K̂_s, the inverse FFT and the output
// chirp cout_s. What moves: k_czt_sf keeps K̂ (and, fp32, cout and Y) in shared memory and parks
// the fp64 spectrum Y in an L2 workspace slot, so every record re-reads ~180 KB of tables and parked
// data through the same L1 / shared-memory path the FFT exchanges need (the kernel was co-limited
// by that path and the FP64 pipe, each ~55% busy). Here every thread keeps its own slice of
// cin, K̂_s and cout_s, and its group's parked Y, in its TMEM lane (tmem.cuh: 32x32b accesses,
// measured 3.5x the LDS bandwidth and running beside it), so shared memory carries only the
// exchanges and the twiddle tables.
//
// TMEM layout (32-bit columns of lane t, t = thread index within the 128-thread group; every group's
// thread t sees the same lane, so the trace-independent tables are stored once per CTA):
//   [0, KH)            K̂_s[t + NT q], s < nseg, q < EPT        (nseg * EPT * W columns)
//   [KH, KH + CO)      cout_s[t + NT q], q < NO (zero past m)   (nseg * NOC * W)
//   TWT: [.., + 16 W)  the last pass's twiddles W_L^{j t}, j < 16 (cin is read through L1)
//   else [.., + CI)    cin[t + NT q], q < NXC (zero past N)     (NXC * W; twiddles formed by products)
//   [.., + Y)          Y of group g, g < RG                      (RG * EPT * W)
// W = 32-bit words per complex (4 fp64, 2 fp32); NOC / NXC round NO / NX up to whole 16-word chunks.
// fp64 configs[1] (nseg 2, NO 8): 128 + 64 + 64 + 256 = 512 columns with TWT.
#pragma once

#include "fft_device.cuh"
#include "tmem.cuh"

namespace skg {

template <typename T, int LOG2L, int NZ, int NO, int RG, bool TWT> struct TmCfg {
    using C = cx_t<T>;
    using G = FftGeom<LOG2L>;
    static constexpr int W = CxWords<C>::W;
    static constexpr int K4 = 16 / W;   // complex values per 16-word chunk
    static constexpr int NX = NZ < G::EPT ? NZ : G::EPT;
    static constexpr int NXC = (NX + K4 - 1) / K4 * K4;
    static constexpr int NOC = (NO + K4 - 1) / K4 * K4;
    static constexpr int BLOCK = G::NT * RG;
    __host__ __device__ static constexpr int col_co(int nseg) { return nseg * G::EPT * W; }
    __host__ __device__ static constexpr int col_ci(int nseg) { return col_co(nseg) + nseg * NOC * W; }
    __host__ __device__ static constexpr int col_y(int nseg) { return col_ci(nseg) + (TWT ? 16 : NXC) * W; }
    __host__ __device__ static constexpr int cols(int nseg) { return col_y(nseg) + RG * G::EPT * W; }
    static constexpr size_t smem_bytes() { return ((size_t)RG * G::SMEM + G::TW_ALLOC) * sizeof(C) + 16; }
};

template <typename T, int LOG2L, int NZ, int NO, bool CPLX, int RG, bool TWT>
__global__ void __launch_bounds__(TmCfg<T, LOG2L, NZ, NO, RG, TWT>::BLOCK, 1)
k_czt_tm(const void* __restrict__ xin, long long x_stride, long long N, long long M, long long batch, int nseg,
         long long seg_len, cx_t<T>* __restrict__ out, long long out_stride, const cx_t<T>* __restrict__ tw,
         const cx_t<T>* __restrict__ cin, const cx_t<T>* __restrict__ khat, const cx_t<T>* __restrict__ cout,
         const cx_t<T>* __restrict__ twl) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2L>;
    using K = TmCfg<T, LOG2L, NZ, NO, RG, TWT>;
    static_assert(!TWT || (G::radix(G::P - 1) == 16 && G::NT == G::pval(G::P - 1)), "one last-pass butterfly per thread");
    static_assert(G::NT == 128, "TMEM lane = thread index within a 128-thread transform group");
    constexpr int K4 = K::K4, W = K::W, EPT = G::EPT;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int gid = threadIdx.x / G::NT;
    const int tid = threadIdx.x % G::NT;
    C* sm = reinterpret_cast<C*>(smraw) + gid * G::SMEM;
    C* tws = reinterpret_cast<C*>(smraw) + RG * G::SMEM;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tws + G::TW_ALLOC);
    load_twiddles<LOG2L>(tws, tw);
    const uint32_t tb = tmem_alloc_cta<512>(tslot);   // includes the barrier that publishes the twiddles
    const uint32_t tl = tmem_lane_addr(tb, 0);         // this thread's lane, column 0
    const uint32_t c_co = K::col_co(nseg), c_ci = K::col_ci(nseg), c_y = K::col_y(nseg) + gid * EPT * W;
    if (gid == 0) {   // group 0 writes the CTA's tables into lanes 0..127
        C t[K4];
        for (int s = 0; s < nseg; ++s) {
#pragma unroll
            for (int c = 0; c < EPT / K4; ++c) {
#pragma unroll
                for (int i = 0; i < K4; ++i) t[i] = __ldg(khat + (long long)s * G::L + tid + G::NT * (c * K4 + i));
                tmem_put<C, K4>(tl + (s * EPT + c * K4) * W, t);
            }
            const long long m_here = min(seg_len, M - s * seg_len);
#pragma unroll
            for (int c = 0; c < K::NOC / K4; ++c) {
#pragma unroll
                for (int i = 0; i < K4; ++i) {
                    const long long pos = tid + G::NT * (c * K4 + i);
                    t[i] = pos < m_here ? __ldg(cout + s * seg_len + pos) : czero<C>();
                }
                tmem_put<C, K4>(tl + c_co + (s * K::NOC + c * K4) * W, t);
            }
        }
        if constexpr (TWT) {
#pragma unroll
            for (int c = 0; c < 16 / K4; ++c) {
#pragma unroll
                for (int i = 0; i < K4; ++i) t[i] = __ldg(twl + tid * 16 + c * K4 + i);
                tmem_put<C, K4>(tl + c_ci + c * K4 * W, t);
            }
        } else {
#pragma unroll
            for (int c = 0; c < K::NXC / K4; ++c) {
#pragma unroll
                for (int i = 0; i < K4; ++i) {
                    const long long pos = tid + G::NT * (c * K4 + i);
                    t[i] = pos < N ? __ldg(cin + pos) : czero<C>();
                }
                tmem_put<C, K4>(tl + c_ci + c * K4 * W, t);
            }
        }
        tmem_wait_st();
    }
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    const GroupSync gsync{1 + gid, G::NT};
    using XT = typename std::conditional<CPLX, C, T>::type;
    const int n32 = (int)N;   // N <= L and the segment bounds fit 32 bits (L = 2048)
    for (long long b = (long long)blockIdx.x * RG + gid; b < batch; b += (long long)gridDim.x * RG) {
        const XT* xb = reinterpret_cast<const XT*>(xin) + b * x_stride;
        XT xr[K::NX];
#pragma unroll
        for (int q = 0; q < K::NX; ++q) {
            const int pos = tid + G::NT * q;
            if constexpr (CPLX) xr[q] = czero<C>();
            else xr[q] = (T)0;
            if (pos < n32) xr[q] = __ldg(xb + pos);
        }
        if (b + (long long)gridDim.x * RG < batch) {   // the group's next trace into L2
            const XT* xn = xb + (long long)gridDim.x * RG * x_stride;
#pragma unroll
            for (int q = 0; q < K::NX; ++q) {
                const int pos = tid + G::NT * q;
                if (pos < n32) prefetch_l2(xn + pos);
            }
        }
        C v[EPT];
#pragma unroll
        for (int q = K::NX; q < EPT; ++q) v[q] = czero<C>();
        if constexpr (TWT) {
#pragma unroll
            for (int q = 0; q < K::NX; ++q) {
                const int pos = tid + G::NT * q;
                v[q] = czero<C>();
                if (pos < n32) {
                    const C ch = __ldg(cin + pos);
                    if constexpr (CPLX) v[q] = cmul(xr[q], ch);
                    else v[q] = rmul(xr[q], ch);
                }
            }
        } else {
#pragma unroll
            for (int c = 0; c < K::NXC / K4; ++c) {
                C ch[K4];
                tmem_get<C, K4>(tl + c_ci + c * K4 * W, ch);
#pragma unroll
                for (int i = 0; i < K4; ++i) {
                    const int q = c * K4 + i;
                    if (q < K::NX) {   // cin is zero past N, so the padded samples stay zero
                        if constexpr (CPLX) v[q] = cmul(xr[q], ch[i]);
                        else v[q] = rmul(xr[q], ch[i]);
                    }
                }
            }
        }
        const uint32_t tmt = tl + c_ci;   // TWT: the last pass's twiddles
        block_fft<false, LOG2L, NZ, 16, C, GroupSync, TWT>(v, sm, tws, tid, true, gsync, tmt);
        if (nseg > 1) {
#pragma unroll
            for (int c = 0; c < EPT / K4; ++c) {
                C t[K4];
#pragma unroll
                for (int i = 0; i < K4; ++i) t[i] = v[c * K4 + i];
                tmem_put<C, K4>(tl + c_y + c * K4 * W, t);
            }
        }
        for (int sg = 0; sg < nseg; ++sg) {
            if (sg > 0) {
                tmem_wait_st();
#pragma unroll
                for (int c = 0; c < EPT / K4; ++c) {
                    C t[K4];
                    tmem_get<C, K4>(tl + c_y + c * K4 * W, t);
#pragma unroll
                    for (int i = 0; i < K4; ++i) v[c * K4 + i] = t[i];
                }
            }
#pragma unroll
            for (int c = 0; c < EPT / K4; ++c) {
                C kh[K4];
                tmem_get<C, K4>(tl + (sg * EPT + c * K4) * W, kh);
#pragma unroll
                for (int i = 0; i < K4; ++i) v[c * K4 + i] = cmul(v[c * K4 + i], kh[i]);
            }
            block_fft<true, LOG2L, 16, NO, C, GroupSync, TWT>(v, sm, tws, tid, true, gsync, tmt);
            const int m_here = (int)min(seg_len, M - sg * seg_len);
            C* o = out + b * out_stride + sg * seg_len;
#pragma unroll
            for (int c = 0; c < K::NOC / K4; ++c) {
                C co[K4];
                tmem_get<C, K4>(tl + c_co + (sg * K::NOC + c * K4) * W, co);
#pragma unroll
                for (int i = 0; i < K4; ++i) {
                    const int q = c * K4 + i;
                    const int pos = tid + G::NT * q;
                    if (q < NO && pos < m_here) o[pos] = cmul(v[q], co[i]);
                }
            }
            gsync();   // the next transform's first exchange must not overwrite this one's last reads
        }
    }
    tmem_free_cta<512>(tb);
}

}  // namespace skg
