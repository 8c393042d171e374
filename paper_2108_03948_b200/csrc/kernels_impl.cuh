// kernels_impl.cuh — batched single-CTA FFT / real-input FFT / fused Bluestein CZT kernels.
// Instantiated per scalar type in kernels_f64.cu / kernels_f32.cu.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "bulk_copy.cuh"
#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_czt_tm.cuh"

namespace skg {

template <typename T, int LOG2L> struct KCfg {
    using G = FftGeom<LOG2L>;
    static constexpr int GROUPS = G::NT >= 128 ? 1 : 128 / G::NT;   // transforms per CTA
    static constexpr int BLOCK = G::NT * GROUPS;
    // [GROUPS padded data regions][factorised twiddle tables]
    static constexpr size_t SMEM_BYTES = ((size_t)GROUPS * G::SMEM + (G::L >= 16 ? G::TW_ALLOC : 0)) * sizeof(cx_t<T>);
    // cap registers at 128/thread (>= 2 CTAs of 256 threads per SM) unless the block is wider
    static constexpr int MINB = BLOCK >= 512 ? 1 : 512 / BLOCK;
};

template <typename K> inline cudaError_t prep_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return cudaSuccess;
}

inline unsigned grid_for(long long batch, int groups) { return (unsigned)((batch + groups - 1) / groups); }

// persistent grid: as many CTAs as fit on the device at once (capped by the work)
template <typename K> inline unsigned persistent_grid(K kernel, int block, size_t smem, long long units) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    long long cap = (long long)per_sm * sms;
    if (const unsigned gc = grid_cap(); gc && gc < cap) cap = gc;
    return (unsigned)(units < cap ? (units > 0 ? units : 1) : cap);
}

// common prologue: shared-memory carve-up and the twiddle tables
#define SKG_PROLOGUE(T, LG)                                                                        \
    using C = cx_t<T>;                                                                             \
    using G = FftGeom<LG>;                                                                         \
    using K = KCfg<T, LG>;                                                                         \
    extern __shared__ __align__(16) unsigned char smraw[];                                         \
    C* sm = reinterpret_cast<C*>(smraw) + (threadIdx.x / G::NT) * G::SMEM;                         \
    C* tws = reinterpret_cast<C*>(smraw) + K::GROUPS * G::SMEM;                                    \
    if constexpr (G::L >= 16) load_twiddles<LG>(tws, tw);                                          \
    __syncthreads();                                                                               \
    const int tid = threadIdx.x % G::NT;                                                           \
    const int gid = threadIdx.x / G::NT;

// ---------------------------------------------------------------------------------------
// complex -> complex (FftPlan::forward/inverse, numerics.cpp:73-100; fft/ifft 102-120)
template <typename T, int LOG2L, bool INV>
__global__ void __launch_bounds__(KCfg<T, LOG2L>::BLOCK, KCfg<T, LOG2L>::MINB)
k_fft_c2c(const cx_t<T>* in, long long in_stride, cx_t<T>* out, long long out_stride, long long batch,
          const cx_t<T>* __restrict__ tw, T scale) {
    SKG_PROLOGUE(T, LOG2L)
    for (long long base = (long long)blockIdx.x * K::GROUPS; base < batch; base += (long long)gridDim.x * K::GROUPS) {
        const long long b = base + gid;
        const bool active = b < batch;
        C v[G::EPT];
        const C* src = in + b * in_stride;
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) v[q] = active ? src[tid + G::NT * q] : czero<C>();
        block_fft<INV, LOG2L>(v, sm, tws, tid);
        if (active) {
            C* dst = out + b * out_stride;
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) dst[tid + G::NT * q] = cscale(v[q], scale);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// real input, zero padded to L = 2M: M-point complex FFT of z[n] = x[2n] + i x[2n+1], then
// X[k] = E[k] + W_L^k O[k] with E/O split from Z[k], conj Z[M-k]. Replaces fft_spectrum's
// zero_pad + dft_any (spectra.cpp:21-38) without ever materialising the zeros.
#ifndef SKG_R2C_MINB_F32
#define SKG_R2C_MINB_F32 3   // measured on configs[3]: 2 -> 1.269 ms, 3 -> 1.192 ms, 4 -> 1.215 ms
#endif
#ifndef SKG_R2C_MINB_F32_512
#define SKG_R2C_MINB_F32_512 2   // 64 registers, 2 CTAs per SM: fp32 L = 16384 spectra 2.94 -> 2.69 ms per 256 MiB batch
#endif
template <typename T, int LOG2M> struct R2cCfg {
    // fp32 256-thread transforms: CTAs per SM the register cap targets (2 = 128 registers)
    static constexpr int MINB = (sizeof(T) == 4 && KCfg<T, LOG2M>::BLOCK == 256) ? SKG_R2C_MINB_F32
                                : (sizeof(T) == 4 && KCfg<T, LOG2M>::BLOCK == 512) ? SKG_R2C_MINB_F32_512
                                                                                   : KCfg<T, LOG2M>::MINB;
};
constexpr size_t kR2cTmaBytes = 8192;   // longest trace staged by TMA in k_fft_r2c
template <typename T, int LOG2M, int NZ, int MODE>
__global__ void __launch_bounds__(KCfg<T, LOG2M>::BLOCK, R2cCfg<T, LOG2M>::MINB)
k_fft_r2c(const T* __restrict__ x, long long x_stride, long long N, int vec, long long batch,
          const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ post, cx_t<T>* __restrict__ out,
          long long out_stride, const cx_t<T>* __restrict__ rtab, T* __restrict__ mag, T* __restrict__ phase,
          long long mp_stride, long long klo, long long khi) {
    SKG_PROLOGUE(T, LOG2M)
    constexpr int M = G::L;
    constexpr long long L = 2LL * M;
    const long long half = N >> 1;
#ifndef SKG_R2C_NO_TMA
    // One transform per CTA, rows of whole 16-byte units, traces of at most 8 KB: the NEXT unit's trace
    // arrives by one TMA bulk copy (cp.async.bulk + mbarrier) while this one is transformed, and the first
    // pass reads its samples from shared memory instead of global memory. Measured against the L2-prefetch +
    // LDG path (-DSKG_R2C_NO_TMA): cube 1.068 -> 1.034 ms, 1024 -> 4096 fp32 0.217 -> 0.214 ms, fp64
    // at par; 16 KB traces (L = 16384 fp32) measured 1% slower, so they keep the LDG path.
    __shared__ __align__(8) uint64_t stg_bar;
    const bool tma = K::GROUPS == 1 && vec && (N * sizeof(T)) % 16 == 0 && N * sizeof(T) <= kR2cTmaBytes &&
                     (x_stride * sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(x) % 16) == 0;
    T* stg = reinterpret_cast<T*>((reinterpret_cast<uintptr_t>(tws + G::TW_ALLOC) + 15) & ~static_cast<uintptr_t>(15));
    uint32_t parity = 0;
    auto issue = [&](long long bb) {
        if (threadIdx.x != 0 || bb >= batch) return;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&stg_bar, (uint32_t)(N * sizeof(T)));
        bulk_g2s(stg, x + bb * x_stride, (uint32_t)(N * sizeof(T)), &stg_bar);
    };
    if (tma) {
        if (threadIdx.x == 0) {
            mbar_init(&stg_bar, 1);
            mbar_fence_init();
        }
        __syncthreads();
        issue((long long)blockIdx.x);
    }
#endif
    for (long long base = (long long)blockIdx.x * K::GROUPS; base < batch; base += (long long)gridDim.x * K::GROUPS) {
        const long long b = base + gid;
        const bool active = b < batch;
        C v[G::EPT];
        const T* xs = x + b * x_stride;
#ifndef SKG_R2C_NO_TMA
        if (tma) {
            mbar_wait(&stg_bar, parity);
            parity ^= 1u;
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) {
                v[q] = czero<C>();
                const long long pos = tid + (long long)G::NT * q;
                if (q < NZ && pos < half) v[q] = reinterpret_cast<const C*>(stg)[pos];
            }
            __syncthreads();                          // every sample read out of the staging buffer
            issue(base + (long long)gridDim.x);       // the next trace streams in during this transform
        } else
#endif
        {
        {
            const long long bn = b + (long long)gridDim.x * K::GROUPS;
            if (bn < batch) {
                const T* xn = x + bn * x_stride;
#pragma unroll
                for (int q = 0; q < G::EPT; ++q) {
                    const long long pos = tid + (long long)G::NT * q;
                    if (q < NZ && 2 * pos < N) prefetch_l2(xn + 2 * pos);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            v[q] = czero<C>();
            if (q < NZ && active) {
                const long long pos = tid + (long long)G::NT * q;
                if (vec) {
                    if (pos < half) v[q] = __ldg(reinterpret_cast<const C*>(xs) + pos);
                    else if (2 * pos < N) v[q] = mk<C>(xs[2 * pos], (T)0);
                } else {
                    if (2 * pos < N) v[q].x = xs[2 * pos];
                    if (2 * pos + 1 < N) v[q].y = xs[2 * pos + 1];
                }
            }
        }
        }
        block_fft<false, LOG2M, NZ>(v, sm, tws, tid);
        // pair Z[k] with Z[M-k]
        if constexpr (G::NT > 1) {
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) sm[pad16(tid + G::NT * q)] = v[q];
            __syncthreads();
        }
        if (active) {
            C* o = out ? out + b * out_stride : nullptr;
            T* mg = (MODE == 2 || MODE == 3) && mag ? mag + b * mp_stride : nullptr;
            T* ph = MODE == 2 ? phase + b * mp_stride : nullptr;
            // one bin of the band [klo, khi] of the full [0, L) spectrum: complex and/or dB
            auto put = [&](long long k, C X) {
                if (k >= klo && k <= khi) {
                    if (o) o[k - klo] = X;
                    if (mg) mg[k - klo] = magnitude_db_t(X.x, X.y);
                }
            };
            // store one output bin (full / half spectrum, band slice, or H = X / X_ref as |H|, arg H)
            auto emit = [&](long long k, C X) {
                if constexpr (MODE == 0) {
                    o[k] = X;
                    if (k && k < M) o[L - k] = cconj(X);
                } else if constexpr (MODE == 1) {
                    o[k] = X;
                } else if constexpr (MODE == 3) {
                    put(k, X);
                    if (k && k < M) put(L - k, cconj(X));
                } else {
                    const C H = cmul(X, __ldg(rtab + k));
                    mg[k] = abs_t(H.x, H.y);
                    ph[k] = atan2_t(H.y, H.x);
                    if (o) o[k] = H;
                }
            };
            // bins in conjugate pairs (k, M - k), k < M/2: from Z[k], Z[M-k]
            //   E = (Z[k] + conj Z[M-k]) / 2, O = (Z[k] - conj Z[M-k]) / 2i,
            //   X[k] = E + W^k O,  X[M-k] = conj(E - W^k O)   (W = e^{-2 pi i / 2M})
            // k = 0 pairs with the Nyquist bin M; k = M/2 is its own partner.
#pragma unroll
            for (int q = 0; q < (G::EPT > 1 ? G::EPT / 2 : 1); ++q) {
                const int k = tid + G::NT * q;
                C c;
                if constexpr (G::NT == 1) c = v[(M - q) & (M - 1)];
                else c = sm[pad16((M - k) & (M - 1))];
                const C z = v[q];
                // E' = 2E, O' = 2O; post = W^k / 2, so X = E'/2 + post O' (exact rescaling of the
                // textbook split: same rounding, two multiplies fewer per bin)
                const C E2 = mk<C>(z.x + c.x, z.y - c.y);
                const C WO = cmul(mk<C>(z.y + c.y, c.x - z.x), __ldg(post + k));
                emit(k, mk<C>(fma((T)0.5, E2.x, WO.x), fma((T)0.5, E2.y, WO.y)));
                emit(M - k, mk<C>(fma((T)0.5, E2.x, -WO.x), fma((T)-0.5, E2.y, WO.y)));
            }
            if constexpr (G::EPT > 1) {
                if (tid == 0) {   // k = M/2 (its own partner)
                    const int k = M / 2;
                    const C z = v[G::EPT / 2];
                    C c;
                    if constexpr (G::NT == 1) c = v[G::EPT / 2];
                    else c = z;
                    const C E2 = mk<C>(z.x + c.x, z.y - c.y);
                    const C WO = cmul(mk<C>(z.y + c.y, c.x - z.x), __ldg(post + k));
                    emit(k, mk<C>(fma((T)0.5, E2.x, WO.x), fma((T)0.5, E2.y, WO.y)));
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// fused Bluestein CZT (CztPlan::execute, czt.cpp:116-130)
#ifndef SKG_CZT_MINB_F32_512
#define SKG_CZT_MINB_F32_512 1
#endif
template <typename T, int LOG2L> struct CztCfg {
    // fp32 512-thread transforms (L = 8192): CTAs per SM the register cap targets
    static constexpr int MINB = (sizeof(T) == 4 && KCfg<T, LOG2L>::BLOCK == 512) ? SKG_CZT_MINB_F32_512
                                                                                 : KCfg<T, LOG2L>::MINB;
};
template <typename T, int LOG2L, int NZ, int NO>
__global__ void __launch_bounds__(KCfg<T, LOG2L>::BLOCK, CztCfg<T, LOG2L>::MINB)
k_czt(const void* __restrict__ xin, int complex_in, long long x_stride, long long N, long long M, long long batch,
      int nseg, long long seg_len, long long cin_stride, cx_t<T>* __restrict__ out, long long out_stride, const cx_t<T>* __restrict__ tw,
      const cx_t<T>* __restrict__ cin, const cx_t<T>* __restrict__ khat, const cx_t<T>* __restrict__ cout) {
    SKG_PROLOGUE(T, LOG2L)
    // work unit u = trace * nseg + segment; segment s covers outputs [s seg_len, (s+1) seg_len)
    const long long units = batch * nseg;
    for (long long base = (long long)blockIdx.x * K::GROUPS; base < units; base += (long long)gridDim.x * K::GROUPS) {
        const long long u = base + gid;
        const bool active = u < units;
        const long long b = active ? u / nseg : 0;
        const long long sg = active ? u - b * nseg : 0;
        const C* cs = cin + sg * cin_stride;
        const long long m_here = min(seg_len, M - sg * seg_len);
        if (active) {
            // the kernel spectrum is needed after the forward transform: pull this thread's lines
            // into L1 now (every CTA on the SM reads the same table)
#pragma unroll
            for (int q = 0; q < G::EPT; q += (G::NT >= 8 ? 1 : G::EPT)) prefetch_l1(khat + tid + G::NT * q);
            // next unit of this CTA: its trace row into L2 while we work on this one
            const long long un = u + (long long)gridDim.x * K::GROUPS;
            if (un < units) {
                const long long bn = un / nseg;
                const char* xn = reinterpret_cast<const char*>(xin) +
                                 (size_t)(bn * x_stride) * (complex_in ? sizeof(C) : sizeof(T));
#pragma unroll
                for (int q = 0; q < G::EPT; ++q) {
                    const long long pos = tid + (long long)G::NT * q;
                    if (q < NZ && pos < N) prefetch_l2(xn + pos * (complex_in ? sizeof(C) : sizeof(T)));
                }
            }
        }
        C v[G::EPT];
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            v[q] = czero<C>();
            const long long pos = tid + (long long)G::NT * q;
            if (q < NZ && active && pos < N) {
                const C ch = __ldg(cs + pos);
                if (complex_in) v[q] = cmul(__ldg(reinterpret_cast<const C*>(xin) + b * x_stride + pos), ch);
                else v[q] = rmul(__ldg(reinterpret_cast<const T*>(xin) + b * x_stride + pos), ch);
            }
        }
        block_fft<false, LOG2L, NZ>(v, sm, tws, tid);
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) v[q] = cmul(v[q], __ldg(khat + tid + G::NT * q));
        block_fft<true, LOG2L, 16, NO>(v, sm, tws, tid);
        if (active) {
            C* o = out + b * out_stride + sg * seg_len;
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) {
                const long long pos = tid + (long long)G::NT * q;
                if (q < NO && pos < m_here) o[pos] = cmul(v[q], __ldg(cout + pos));
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// Resident-table Bluestein CZT: one CTA per SM, RG independent trace groups of NT threads (each
// group syncs on its own named barrier), and every table the segment needs — factorised twiddles,
// the segment's input chirp, the kernel spectrum K̂ and the output chirp — resident in shared
// memory for the whole launch. The only global traffic left is the trace in and the bins out.
template <typename T, int LOG2L> struct RtCfg {
    using G = FftGeom<LOG2L>;
    static constexpr int RG = G::NT >= 128 ? 4 : 512 / G::NT;   // trace groups per CTA (512 threads)
    static constexpr int BLOCK = G::NT * RG;
};

template <typename T, int LOG2L, int NZ, int NO, bool CPLX>
__global__ void __launch_bounds__(RtCfg<T, LOG2L>::BLOCK, 1)
k_czt_rt(const void* __restrict__ xin, long long x_stride, long long N, long long M, long long batch,
         int nseg, long long seg_len, long long cin_stride, cx_t<T>* __restrict__ out, long long out_stride,
         const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ cin, const cx_t<T>* __restrict__ khat,
         const cx_t<T>* __restrict__ cout) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2L>;
    constexpr int RG = RtCfg<T, LOG2L>::RG;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int gid = threadIdx.x / G::NT;
    const int tid = threadIdx.x % G::NT;
    C* sm = reinterpret_cast<C*>(smraw) + gid * G::SMEM;
    C* tws = reinterpret_cast<C*>(smraw) + RG * G::SMEM;
    C* s_cin = tws + G::TW_ALLOC;
    C* s_kh = s_cin + N;
    C* s_co = s_kh + G::L;
    // this CTA serves one output segment; its traces are strided over the CTAs of that segment
    const int sg = blockIdx.x % nseg;
    const long long team = gridDim.x / nseg;           // CTAs per segment
    const long long first = blockIdx.x / nseg;
    const long long m_here = min(seg_len, M - sg * seg_len);
    load_twiddles<LOG2L>(tws, tw);
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_cin[i] = __ldg(cin + sg * cin_stride + i);
    for (int i = threadIdx.x; i < G::L; i += blockDim.x) s_kh[i] = __ldg(khat + i);
    for (int i = threadIdx.x; i < m_here; i += blockDim.x) s_co[i] = __ldg(cout + i);
    __syncthreads();
    const GroupSync gsync{1 + gid, G::NT};
    // raw samples of the group's current trace, loaded one trace ahead (register double buffer)
    constexpr int NX = NZ < G::EPT ? NZ : G::EPT;
    using XT = typename std::conditional<CPLX, C, T>::type;
    XT xr[NX];
    auto load_x = [&](long long bb) {
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const long long pos = tid + (long long)G::NT * q;
            if constexpr (CPLX) xr[q] = czero<C>();
            else xr[q] = (T)0;
            if (bb < batch && pos < N) xr[q] = __ldg(reinterpret_cast<const XT*>(xin) + bb * x_stride + pos);
        }
    };
#ifndef SKG_RT_XPREFETCH
#define SKG_RT_XPREFETCH 0   // register double buffer measured slower (spills) than an L2 prefetch
#endif
    if (SKG_RT_XPREFETCH) load_x(first * RG + gid);
    for (long long b = first * RG + gid; b < batch; b += team * RG) {
        if (!SKG_RT_XPREFETCH) {
            load_x(b);
            const long long bn = b + team * RG;   // and the group's next trace into L2
            if (bn < batch) {
#pragma unroll
                for (int q = 0; q < NX; ++q) {
                    const long long pos = tid + (long long)G::NT * q;
                    if (pos < N) prefetch_l2(reinterpret_cast<const XT*>(xin) + bn * x_stride + pos);
                }
            }
        }
        C v[G::EPT];
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            v[q] = czero<C>();
            const long long pos = tid + (long long)G::NT * q;
            if (q < NX && pos < N) {
                if constexpr (CPLX) v[q] = cmul(xr[q], s_cin[pos]);
                else v[q] = rmul(xr[q], s_cin[pos]);
            }
        }
        if (SKG_RT_XPREFETCH) load_x(b + team * RG);   // in flight during this trace's two transforms
        block_fft<false, LOG2L, NZ>(v, sm, tws, tid, true, gsync);
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            v[q] = cmul(v[q], s_kh[tid + G::NT * q]);
            if ((q & 3) == 3) asm volatile("" ::: "memory");   // bound the K̂ loads in flight (registers)
        }
        block_fft<true, LOG2L, 16, NO>(v, sm, tws, tid, true, gsync);
        C* o = out + b * out_stride + sg * seg_len;
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            const long long pos = tid + (long long)G::NT * q;
            if (q < NO && pos < m_here) o[pos] = cmul(v[q], s_co[pos]);
            if ((q & 3) == 3) asm volatile("" ::: "memory");
        }
        gsync();   // the next trace's first exchange must not overwrite this one's last reads
    }
}

// ---------------------------------------------------------------------------------------
// Shared-forward segmented Bluestein CZT. The M bins run as S blocks of M' = seg_len; block s is
// the linear convolution of the SAME chirped input y = x·cin (cin = A^{-n} W^{n^2/2}) with the
// kernel segment g_s[j] = W^{-(sM' + j)^2/2}, j in (-N, M'), so ONE forward FFT serves all S
// blocks:  X[sM' + k'] = cout_s[k'] · IFFT(FFT(y) · K̂_s)[k'],  cout_s[k'] = W^{(sM'+k')^2/2}.
// Against per-segment start points (A_s = A W^{-sM'}: S forward + S inverse transforms) this does
// 1 + S transforms per trace (configs[1]: 3 instead of 4). The spectrum Y is parked in a private
// per-group shared buffer (each thread re-reads only its own positions: no barrier) while the
// blocks' inverse transforms run. RG trace groups per CTA, named barriers per group.
template <int LOG2L, int RG> struct SfCfg {
    static constexpr int BLOCK = FftGeom<LOG2L>::NT * RG;
};

// TS (bits): 0 kernel spectra and output chirps read through L1/L2, 1 kernel spectra in shared
// memory, 2 both in shared memory; +4: the parked spectrum Y lives in a global (L2-resident)
// workspace slot per group instead of shared memory (frees 32 KB per group for more groups)
template <typename T, int LOG2L, int NZ, int NO, bool CPLX, int RG, int TS>
__global__ void __launch_bounds__(SfCfg<LOG2L, RG>::BLOCK, 1)
k_czt_sf(const void* __restrict__ xin, long long x_stride, long long N, long long M, long long batch, int nseg,
         long long seg_len, cx_t<T>* __restrict__ out, long long out_stride, const cx_t<T>* __restrict__ tw,
         const cx_t<T>* __restrict__ cin, const cx_t<T>* __restrict__ khat, const cx_t<T>* __restrict__ cout,
         cx_t<T>* __restrict__ ywork) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2L>;
    constexpr bool KS = (TS & 3) >= 1, CS = (TS & 3) >= 2, YG = (TS & 4) != 0;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int gid = threadIdx.x / G::NT;
    const int tid = threadIdx.x % G::NT;
    C* sm = reinterpret_cast<C*>(smraw) + gid * G::SMEM;
    C* yb = YG ? ywork + ((long long)blockIdx.x * RG + gid) * G::L
               : reinterpret_cast<C*>(smraw) + RG * G::SMEM + gid * G::L;
    C* tws = reinterpret_cast<C*>(smraw) + RG * (G::SMEM + (YG ? 0 : G::L));
    C* s_cin = tws + G::TW_ALLOC;
    C* s_kh = s_cin + N;                       // KS: nseg x L
    C* s_co = s_kh + (KS ? nseg * G::L : 0);   // CS: nseg x seg_len
    load_twiddles<LOG2L>(tws, tw);
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_cin[i] = __ldg(cin + i);
    if constexpr (KS)
        for (int i = threadIdx.x; i < nseg * G::L; i += blockDim.x) s_kh[i] = __ldg(khat + i);
    if constexpr (CS)
        for (long long i = threadIdx.x; i < nseg * seg_len; i += blockDim.x) s_co[i] = __ldg(cout + i);
    __syncthreads();
    const C* kh_all = KS ? s_kh : khat;
    const C* co_all = CS ? s_co : cout;
    const GroupSync gsync{1 + gid, G::NT};
    constexpr int NX = NZ < G::EPT ? NZ : G::EPT;
    using XT = typename std::conditional<CPLX, C, T>::type;
    for (long long b = (long long)blockIdx.x * RG + gid; b < batch; b += (long long)gridDim.x * RG) {
        XT xr[NX];
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const long long pos = tid + (long long)G::NT * q;
            if constexpr (CPLX) xr[q] = czero<C>();
            else xr[q] = (T)0;
            if (pos < N) xr[q] = __ldg(reinterpret_cast<const XT*>(xin) + b * x_stride + pos);
        }
        {   // the group's next trace into L2
            const long long bn = b + (long long)gridDim.x * RG;
            if (bn < batch) {
#pragma unroll
                for (int q = 0; q < NX; ++q) {
                    const long long pos = tid + (long long)G::NT * q;
                    if (pos < N) prefetch_l2(reinterpret_cast<const XT*>(xin) + bn * x_stride + pos);
                }
            }
        }
        C v[G::EPT];
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            v[q] = czero<C>();
            const long long pos = tid + (long long)G::NT * q;
            if (q < NX && pos < N) {
                if constexpr (CPLX) v[q] = cmul(xr[q], s_cin[pos]);
                else v[q] = rmul(xr[q], s_cin[pos]);
            }
        }
        block_fft<false, LOG2L, NZ>(v, sm, tws, tid, true, gsync);
        for (int sg = 0; sg < nseg; ++sg) {
            if (sg == 0) {
                if (nseg > 1) {
#pragma unroll
                    for (int q = 0; q < G::EPT; ++q) yb[q * G::NT + tid] = v[q];
                }
            } else {
#pragma unroll
                for (int q = 0; q < G::EPT; ++q) v[q] = yb[q * G::NT + tid];
            }
            const C* kh = kh_all + (long long)sg * G::L;
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) {
                v[q] = cmul(v[q], KS ? kh[tid + G::NT * q] : __ldg(kh + tid + G::NT * q));
                if ((q & 3) == 3) asm volatile("" ::: "memory");
            }
            block_fft<true, LOG2L, 16, NO>(v, sm, tws, tid, true, gsync);
            const long long m_here = min(seg_len, M - sg * seg_len);
            const C* co = co_all + sg * seg_len;
            C* o = out + b * out_stride + sg * seg_len;
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) {
                const long long pos = tid + (long long)G::NT * q;
                if (q < NO && pos < m_here) o[pos] = cmul(v[q], CS ? co[pos] : __ldg(co + pos));
                if ((q & 3) == 3) asm volatile("" ::: "memory");
            }
            gsync();   // the next transform's first exchange must not overwrite this one's last reads
        }
    }
}

template <typename T, int LOG2L>
inline size_t sf_smem_bytes(int rg, int ts, long long N, int nseg, long long seg_len) {
    using G = FftGeom<LOG2L>;
    return ((size_t)rg * (G::SMEM + ((ts & 4) ? 0 : G::L)) + G::TW_ALLOC + (size_t)N +
            ((ts & 3) >= 1 ? (size_t)nseg * G::L : 0) + ((ts & 3) >= 2 ? (size_t)nseg * seg_len : 0)) *
           sizeof(cx_t<T>);
}

template <typename T, int LOG2L>
inline size_t rt_smem_bytes(long long N, long long seg_len) {
    using G = FftGeom<LOG2L>;
    return ((size_t)RtCfg<T, LOG2L>::RG * G::SMEM + G::TW_ALLOC + (size_t)N + G::L + (size_t)seg_len) * sizeof(cx_t<T>);
}

// ---------------------------------------------------------------------------------------
// launch plumbing

template <typename T, int LOG2L, bool INV>
cudaError_t run_c2c(const void* in, long long in_stride, void* out, long long out_stride, long long batch,
                    const void* tw, T scale, cudaStream_t st) {
    using K = KCfg<T, LOG2L>;
    using C = cx_t<T>;
    auto kern = k_fft_c2c<T, LOG2L, INV>;
    cudaError_t e = prep_smem(kern, K::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<persistent_grid(kern, K::BLOCK, K::SMEM_BYTES, grid_for(batch, K::GROUPS)), K::BLOCK, K::SMEM_BYTES, st>>>(
        (const C*)in, in_stride, (C*)out, out_stride, batch, (const C*)tw, scale);
    return cudaGetLastError();
}

template <typename T, int LOG2M, int NZ, int MODE>
cudaError_t run_r2c(long long N, const T* x, long long x_stride, long long batch, const void* tw,
                    const void* post, void* out, long long out_stride, const void* rtab, T* mag,
                    T* phase, long long mp_stride, long long klo, long long khi, cudaStream_t st) {
    using K = KCfg<T, LOG2M>;
    using C = cx_t<T>;
    auto kern = k_fft_r2c<T, LOG2M, NZ, MODE>;
#ifndef SKG_R2C_NO_TMA
    const size_t smem_bytes =
        K::SMEM_BYTES + (K::GROUPS == 1 && (size_t)N * sizeof(T) <= kR2cTmaBytes ? 16 + (size_t)N * sizeof(T) : 0);
#else
    const size_t smem_bytes = K::SMEM_BYTES;
#endif
    cudaError_t e = prep_smem(kern, smem_bytes);
    if (e != cudaSuccess) return e;
    const int vec = ((N & 1) == 0 && (x_stride & 1) == 0 && ((uintptr_t)x % (2 * sizeof(T))) == 0) ? 1 : 0;
    kern<<<persistent_grid(kern, K::BLOCK, smem_bytes, grid_for(batch, K::GROUPS)), K::BLOCK, smem_bytes, st>>>(
        x, x_stride, N, vec, batch, (const C*)tw, (const C*)post, (C*)out, out_stride, (const C*)rtab,
        mag, phase, mp_stride, klo, khi);
    return cudaGetLastError();
}

inline int smem_optin() {
    static int v = 0;
    if (!v) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    return v;
}

template <typename T, int LOG2L, int NZ, int NO>
cudaError_t run_czt(long long N, long long M, bool complex_in, const void* x, long long x_stride, long long batch,
                    int nseg, long long seg_len, long long cin_stride, void* out, long long out_stride,
                    const void* tw, const void* cin, const void* khat, const void* cout, cudaStream_t st) {
    using K = KCfg<T, LOG2L>;
    using C = cx_t<T>;
    if constexpr (FftGeom<LOG2L>::NT >= 32) {
        const size_t rts = rt_smem_bytes<T, LOG2L>(N, seg_len);
        static const bool rt_off = getenv("SKG_CZT_NO_RT") != nullptr;
        // the route depends on the plan only, never on the batch size, so a batch split into chunks
        // (skg_*_host) gives bit-identical rows
        if (!rt_off && rts <= (size_t)smem_optin()) {
            auto launch = [&](auto kern) {
                cudaError_t e = prep_smem(kern, rts);
                if (e != cudaSuccess) return e;
                constexpr int RG = RtCfg<T, LOG2L>::RG;
                // grid: resident CTAs, a multiple of nseg so every CTA owns one segment
                long long g = persistent_grid(kern, RtCfg<T, LOG2L>::BLOCK, rts, (batch + RG - 1) / RG * nseg);
                g = std::max<long long>(nseg, g / nseg * nseg);
                kern<<<(unsigned)g, RtCfg<T, LOG2L>::BLOCK, rts, st>>>(
                    x, x_stride, N, M, batch, nseg, seg_len, cin_stride, (C*)out, out_stride, (const C*)tw,
                    (const C*)cin, (const C*)khat, (const C*)cout);
                return cudaGetLastError();
            };
            return complex_in ? launch(k_czt_rt<T, LOG2L, NZ, NO, true>) : launch(k_czt_rt<T, LOG2L, NZ, NO, false>);
        }
    }
    auto kern = k_czt<T, LOG2L, NZ, NO>;
    cudaError_t e = prep_smem(kern, K::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<persistent_grid(kern, K::BLOCK, K::SMEM_BYTES, grid_for(batch * nseg, K::GROUPS)), K::BLOCK, K::SMEM_BYTES,
           st>>>(x, complex_in ? 1 : 0, x_stride, N, M, batch, nseg, seg_len, cin_stride, (C*)out, out_stride, (const C*)tw,
                 (const C*)cin, (const C*)khat, (const C*)cout);
    return cudaGetLastError();
}

// leading nonzero count of the first radix-16 pass, rounded up to {4,8,16} (pruned variants
// are only instantiated for L >= 256; smaller transforms always run the full pass)
inline int nz_class(long long nonzero, int nt) {
    const long long per = (nonzero + nt - 1) / nt;
    if (per <= 4) return 4;
    if (per <= 8) return 8;
    return 16;
}
inline int no_class(long long needed, int nt) {
    const long long per = (needed + nt - 1) / nt;
    return per <= 8 ? 8 : 16;
}

template <int V> struct IC { static constexpr int value = V; };

template <int LO, int HI, typename F> cudaError_t dispatch_log2(int lg, F&& f) {
    if constexpr (LO > HI) {
        return cudaErrorInvalidValue;
    } else {
        if (lg == LO) return f(IC<LO>{});
        return dispatch_log2<LO + 1, HI>(lg, f);
    }
}

template <int LG, typename F> cudaError_t dispatch_nz(int nz, F&& f) {
    if constexpr (LG < 8) {
        return f(IC<16>{});
    } else {
        if (nz == 4) return f(IC<4>{});
        if (nz == 8) return f(IC<8>{});
        return f(IC<16>{});
    }
}

template <typename T>
cudaError_t launch_fft_c2c_impl(int log2L, bool inverse, const void* in, long long in_stride, void* out,
                                long long out_stride, long long batch, const void* tw, T scale, cudaStream_t st) {
    return dispatch_log2<0, max_log2<T>()>(log2L, [&](auto lg) {
        constexpr int LG = decltype(lg)::value;
        return inverse ? run_c2c<T, LG, true>(in, in_stride, out, out_stride, batch, tw, scale, st)
                       : run_c2c<T, LG, false>(in, in_stride, out, out_stride, batch, tw, scale, st);
    });
}

template <typename T>
cudaError_t launch_fft_r2c_impl(int log2M, long long N, const T* x, long long x_stride, long long batch,
                                const void* tw, const void* post, int mode, void* out, long long out_stride,
                                const void* rtab, T* mag, T* phase, long long mp_stride, long long klo,
                                long long khi, cudaStream_t st) {
    return dispatch_log2<0, max_log2<T>()>(log2M, [&](auto lg) {
        constexpr int LG = decltype(lg)::value;
        const int nz = nz_class((N + 1) / 2, FftGeom<LG>::NT);
        return dispatch_nz<LG>(nz, [&](auto z) {
            constexpr int NZ = decltype(z)::value;
            if (mode == 0)
                return run_r2c<T, LG, NZ, 0>(N, x, x_stride, batch, tw, post, out, out_stride, rtab, mag, phase,
                                             mp_stride, klo, khi, st);
            if (mode == 1)
                return run_r2c<T, LG, NZ, 1>(N, x, x_stride, batch, tw, post, out, out_stride, rtab, mag, phase,
                                             mp_stride, klo, khi, st);
            if (mode == 3)
                return run_r2c<T, LG, NZ, 3>(N, x, x_stride, batch, tw, post, out, out_stride, rtab, mag, phase,
                                             mp_stride, klo, khi, st);
            return run_r2c<T, LG, NZ, 2>(N, x, x_stride, batch, tw, post, out, out_stride, rtab, mag, phase,
                                         mp_stride, klo, khi, st);
        });
    });
}

template <typename T, int LOG2L, int NZ, int NO>
cudaError_t run_czt_sf(long long N, long long M, bool complex_in, const void* x, long long x_stride, long long batch,
                       int nseg, long long seg_len, void* out, long long out_stride, const void* tw, const void* cin,
                       const void* khat, const void* cout, void* ywork, long long ywork_slots, const void* twl,
                       cudaStream_t st) {
    using C = cx_t<T>;
    if constexpr (FftGeom<LOG2L>::NT < 32) {
        return cudaErrorNotSupported;
    } else {
        const size_t lim = (size_t)smem_optin();
        // configurations in preference order (measured on configs[1]); SKG_CZT_SF_CFG="rg,ts" pins one
        static const char* env = getenv("SKG_CZT_SF_CFG");
        int want_rg = 0, want_ts = -1;
        if (env) sscanf(env, "%d,%d", &want_rg, &want_ts);
        // tensor-memory variant first (kernels_czt_tm.cuh): 128-thread transforms (L = 2048) whose
        // tables + parked spectra fit the 512 TMEM columns; SKG_CZT_NO_TM=1 for the A/B
        static const bool no_tm = getenv("SKG_CZT_NO_TM") != nullptr;
        static const int tm_rg = getenv("SKG_CZT_TM_RG") ? atoi(getenv("SKG_CZT_TM_RG")) : 0;
        static const bool no_twt = getenv("SKG_CZT_NO_TWT") != nullptr;
        auto go_tm = [&](auto rgc, auto twc) -> cudaError_t {
            constexpr int RG = decltype(rgc)::value;
            constexpr bool TWT = decltype(twc)::value != 0;
            using TK = TmCfg<T, LOG2L, NZ, NO, RG, TWT>;
            if (no_tm || want_rg || (tm_rg && tm_rg != RG) || (TWT && (no_twt || !twl)) || TK::cols(nseg) > 512 ||
                TK::smem_bytes() > lim)
                return cudaErrorNotSupported;
            auto launch = [&](auto kern) {
                cudaError_t e = prep_smem(kern, TK::smem_bytes());
                if (e != cudaSuccess) return e;
                const unsigned g = persistent_grid(kern, TK::BLOCK, TK::smem_bytes(), (batch + RG - 1) / RG);
                kern<<<g, TK::BLOCK, TK::smem_bytes(), st>>>(x, x_stride, N, M, batch, nseg, seg_len, (C*)out,
                                                             out_stride, (const C*)tw, (const C*)cin, (const C*)khat,
                                                             (const C*)cout, (const C*)twl);
                return cudaGetLastError();
            };
            return complex_in ? launch(k_czt_tm<T, LOG2L, NZ, NO, true, RG, TWT>)
                              : launch(k_czt_tm<T, LOG2L, NZ, NO, false, RG, TWT>);
        };
        if constexpr (FftGeom<LOG2L>::NT == 128) {
            cudaError_t e0;
            // 4 groups measured best for both precisions (fp32 cfg2: 6 groups 0.137 ms, 8 groups 0.155 ms
            // against 0.136 ms — fewer registers per thread spill)
            if ((e0 = go_tm(IC<4>{}, IC<1>{})) != cudaErrorNotSupported) return e0;
            if ((e0 = go_tm(IC<4>{}, IC<0>{})) != cudaErrorNotSupported) return e0;
        }
        auto go = [&](auto rgc, auto tsc) -> cudaError_t {
            constexpr int RG = decltype(rgc)::value, TS = decltype(tsc)::value;
            if (want_rg && (want_rg != RG || want_ts != TS)) return cudaErrorNotSupported;
            const size_t smem = sf_smem_bytes<T, LOG2L>(RG, TS, N, nseg, seg_len);
            if (smem > lim) return cudaErrorNotSupported;
            if ((TS & 4) && (!ywork || nseg < 2)) return cudaErrorNotSupported;
            auto launch = [&](auto kern) {
                cudaError_t e = prep_smem(kern, smem);
                if (e != cudaSuccess) return e;
                unsigned g = persistent_grid(kern, SfCfg<LOG2L, RG>::BLOCK, smem, (batch + RG - 1) / RG);
                if (TS & 4) g = (unsigned)std::min<long long>(g, ywork_slots / RG);   // one workspace slot per group
                kern<<<g, SfCfg<LOG2L, RG>::BLOCK, smem, st>>>(x, x_stride, N, M, batch, nseg, seg_len, (C*)out,
                                                               out_stride, (const C*)tw, (const C*)cin, (const C*)khat,
                                                               (const C*)cout, (C*)ywork);
                return cudaGetLastError();
            };
            return complex_in ? launch(k_czt_sf<T, LOG2L, NZ, NO, true, RG, TS>)
                              : launch(k_czt_sf<T, LOG2L, NZ, NO, false, RG, TS>);
        };
        // measured on configs[1] (B200): fp32 4 groups with every table in shared memory; fp64 4 groups
        // with the spectrum parked in L2 (0.246 ms) ahead of 3 groups in shared memory (0.256 ms)
        cudaError_t e;
        if constexpr (sizeof(T) == 4) {
            if ((e = go(IC<4>{}, IC<2>{})) != cudaErrorNotSupported) return e;
        }
        if ((e = go(IC<4>{}, IC<5>{})) != cudaErrorNotSupported) return e;
        if ((e = go(IC<3>{}, IC<0>{})) != cudaErrorNotSupported) return e;
        if ((e = go(IC<2>{}, IC<0>{})) != cudaErrorNotSupported) return e;
        return cudaErrorNotSupported;
    }
}

template <typename T>
cudaError_t launch_czt_sf_impl(int log2L, long long N, long long M, bool complex_in, const void* x, long long x_stride,
                               long long batch, int nseg, long long seg_len, void* out, long long out_stride,
                               const void* tw, const void* cin, const void* khat, const void* cout, void* ywork,
                               long long ywork_slots, const void* twl, cudaStream_t st) {
    if (log2L < 9 || log2L > 12) return cudaErrorNotSupported;   // instantiated for 512..4096
    return dispatch_log2<9, 12>(log2L, [&](auto lg) {
        constexpr int LG = decltype(lg)::value;
        if constexpr (LG > max_log2<T>()) {
            return cudaErrorNotSupported;
        } else {
            const int nz = nz_class(N, FftGeom<LG>::NT);
            const int no = no_class(seg_len, FftGeom<LG>::NT);
            return dispatch_nz<LG>(nz, [&](auto z) {
                constexpr int NZ = decltype(z)::value;
                if (no == 8)
                    return run_czt_sf<T, LG, NZ, 8>(N, M, complex_in, x, x_stride, batch, nseg, seg_len, out,
                                                    out_stride, tw, cin, khat, cout, ywork, ywork_slots, twl, st);
                return run_czt_sf<T, LG, NZ, 16>(N, M, complex_in, x, x_stride, batch, nseg, seg_len, out, out_stride,
                                                 tw, cin, khat, cout, ywork, ywork_slots, twl, st);
            });
        }
    });
}

template <typename T>
cudaError_t launch_czt_impl(int log2L, long long N, long long M, bool complex_in, const void* x, long long x_stride,
                            long long batch, int nseg, long long seg_len, long long cin_stride, void* out,
                            long long out_stride, const void* tw, const void* cin, const void* khat, const void* cout,
                            cudaStream_t st) {
    return dispatch_log2<0, max_log2<T>()>(log2L, [&](auto lg) {
        constexpr int LG = decltype(lg)::value;
        const int nz = nz_class(N, FftGeom<LG>::NT);
        const int no = no_class(seg_len, FftGeom<LG>::NT);
        return dispatch_nz<LG>(nz, [&](auto z) {
            constexpr int NZ = decltype(z)::value;
            if (LG >= 8 && no == 8)
                return run_czt<T, LG, NZ, (LG >= 8 ? 8 : 16)>(N, M, complex_in, x, x_stride, batch, nseg, seg_len,
                                                              cin_stride, out, out_stride, tw, cin, khat, cout, st);
            return run_czt<T, LG, NZ, 16>(N, M, complex_in, x, x_stride, batch, nseg, seg_len, cin_stride, out,
                                          out_stride, tw, cin, khat, cout, st);
        });
    });
}

}  // namespace skg
