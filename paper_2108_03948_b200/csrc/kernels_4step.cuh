// kernels_4step.cuh — transforms longer than one CTA's shared memory (L = R * C, up to 2^20).
//
// Four-step factorisation with n = C n1 + n2, k = k1 + R k2:
//   X[k1 + R k2] = sum_n2 W_C^{n2 k2} [ W_L^{n2 k1} sum_n1 x[C n1 + n2] W_R^{n1 k1} ]
// Column pass (k4_col): for a tile of TC adjacent columns n2 (lane-interleaved so every load and
// store moves 128-byte segments) an R-point Stockham FFT per column, the W_L twiddle applied on
// the store into the work buffer Y[k1][n2]. Row pass (k4_row): a C-point FFT per row k1 of Y, then
//   mode 0: natural-order store X[k1 + R k2] (rows lane-interleaved so the stride-R scatter is
//           written as 128-byte segments) — complex FFT / zero-padded spectrum;
//   mode 1: the whole Bluestein middle in shared memory: FFT_C, x khat (stored permuted as
//           khat_p[k1][k2]), IFFT_C, x conj twiddle, back into Y — one read and one write of Y;
// then an inverse column pass (input Y) finishes the CZT with the output chirp on the store.
// Both passes are persistent (grid = resident CTAs) and pull the next tile into L2 while transforming.
#pragma once

#include "bulk_copy.cuh"
#include "kernels_impl.cuh"

namespace skg {

// W^{e0 + d q}, q < 16, from two table entries a = W^{e0}, s = W^{d}: products of depth <= 6
// (s^2, s^4, then a s^{4j} s^i), so no per-element table load waits on L2 after the transform
template <typename C, typename F> __device__ __forceinline__ void twiddle_series(C a, C s, F&& use) {
    const C s2 = cmul(s, s), s3 = cmul(s2, s), s4 = cmul(s2, s2);
    C b = a;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        use(4 * j, b);
        use(4 * j + 1, cmul(b, s));
        use(4 * j + 2, cmul(b, s2));
        use(4 * j + 3, cmul(b, s3));
        if (j < 3) b = cmul(b, s4);
    }
}

template <typename T> struct Tile {
    static constexpr int W = 128 / (int)sizeof(cx_t<T>);   // columns per CTA: 8 (fp64) / 16 (fp32)
};

// column pass kinds
enum : int { IN_CPLX = 0, IN_REAL = 1, IN_REAL_CHIRP = 2, IN_CPLX_CHIRP = 3, IN_WORK = 4 };
enum : int { OUT_WORK_TW = 0, OUT_CHIRP = 1, OUT_SCALE = 2 };

#ifndef SKG_4STEP_COL_THREADS
#define SKG_4STEP_COL_THREADS 512   // resident threads per SM the column pass's register cap targets
#endif
// NZ: leading nonzero rows n1 of the column transforms (zero padding: x[C n1 + n2] = 0 for
// C n1 + n2 >= N), which prunes the first radix-16 pass; the forward pass only.
template <typename T, int LOG2R, bool INV, int NZ = 16>
__global__ void __launch_bounds__(FftGeom<LOG2R>::NT * Tile<T>::W,
                                  (FftGeom<LOG2R>::NT * Tile<T>::W) >= SKG_4STEP_COL_THREADS ? 1
                                  : SKG_4STEP_COL_THREADS / ((FftGeom<LOG2R>::NT * Tile<T>::W) < 32 ? 32 : (FftGeom<LOG2R>::NT * Tile<T>::W)))
k4_col(const void* __restrict__ xin, int in_kind, int conj_in, long long x_stride, long long N,
       const cx_t<T>* __restrict__ cin, cx_t<T>* __restrict__ Y, int log2C, long long batch,
       const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ twL, int out_kind, void* __restrict__ out,
       long long out_stride, long long M, const cx_t<T>* __restrict__ cout, T scale, int conj_out) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2R>;
    constexpr int TC = Tile<T>::W;
    constexpr int REG = G::SMEM + 1;   // odd-ish region stride keeps the 8/16 groups on distinct banks
    extern __shared__ __align__(16) unsigned char smraw[];
    const int g = threadIdx.x % TC;
    const int tid = threadIdx.x / TC;
    C* sm = reinterpret_cast<C*>(smraw) + g * REG;
    C* tws = reinterpret_cast<C*>(smraw) + TC * REG;
    load_twiddles<LOG2R>(tws, tw);
    __syncthreads();
    const long long Cn = 1LL << log2C;
    const long long tiles = Cn / TC;
    const long long L = Cn << LOG2R;
    const long long units = tiles * batch;
    // persistent: the CTA walks tiles with stride gridDim.x; the next tile's column segments are
    // pulled into L2 while this one is transformed (the pass is latency bound, not bandwidth bound)
    auto prefetch = [&](long long u) {
        if (u >= units || g != 0) return;   // one lane per 8/16-column segment
        const long long bb = u / tiles, nn2 = (u % tiles) * TC;
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            const long long n = (tid + (long long)G::NT * q) * Cn + nn2;
            if (in_kind == IN_WORK) prefetch_l2(Y + bb * L + n);
            else if (n < N) {
                if (in_kind == IN_REAL || in_kind == IN_REAL_CHIRP)
                    prefetch_l2(reinterpret_cast<const T*>(xin) + bb * x_stride + n);
                else
                    prefetch_l2(reinterpret_cast<const C*>(xin) + bb * x_stride + n);
            }
        }
    };
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const long long b = u / tiles;
        const long long n2 = (u % tiles) * TC + g;
        prefetch(u + gridDim.x);
        // the store's W_L^{n2 k1}, k1 = tid + NT q: two table entries loaded now (in flight during the
        // transform), the sixteen twiddles formed from them after it
        C tw_a = czero<C>(), tw_s = czero<C>();
        if (out_kind == OUT_WORK_TW) {
            tw_a = __ldg(twL + (long long)tid * Cn + n2);
            tw_s = __ldg(twL + (long long)G::NT * Cn + n2);
        }
        C v[G::EPT];
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            const long long n1 = tid + (long long)G::NT * q;
            const long long n = n1 * Cn + n2;
            C val = czero<C>();
            if (q >= NZ && in_kind != IN_WORK) {
                // rows past the data: zero (the caller guarantees C n1 >= N here)
            } else if (in_kind == IN_WORK) {
                val = Y[b * L + n];   // Y[k1][n2] with k1 = n1
            } else if (n < N) {
                if (in_kind == IN_REAL || in_kind == IN_REAL_CHIRP)
                    val = mk<C>(__ldg(reinterpret_cast<const T*>(xin) + b * x_stride + n), (T)0);
                else
                    val = __ldg(reinterpret_cast<const C*>(xin) + b * x_stride + n);
                if (conj_in) val = cconj(val);
                if (in_kind == IN_REAL_CHIRP || in_kind == IN_CPLX_CHIRP) val = cmul(val, __ldg(cin + n));
            }
            v[q] = val;
        }
        block_fft<INV, LOG2R, NZ>(v, sm, tws, tid);
        if (out_kind == OUT_WORK_TW) {
            // Y[k1][n2] = v * W_L^{n2 k1} (forward twiddle of the four-step split)
            if constexpr (G::EPT == 16) {
                twiddle_series(tw_a, tw_s, [&](int q, C w) {
                    Y[b * L + (tid + (long long)G::NT * q) * Cn + n2] = cmul(v[q], w);
                });
            } else {
#pragma unroll
                for (int q = 0; q < G::EPT; ++q) {
                    const long long k1 = tid + (long long)G::NT * q;
                    Y[b * L + k1 * Cn + n2] = cmul(v[q], __ldg(twL + k1 * Cn + n2));
                }
            }
        }
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            const long long k1 = tid + (long long)G::NT * q;
            if (out_kind == OUT_WORK_TW) {
            } else {
                const long long n = k1 * Cn + n2;   // output sample index C n1 + n2
                if (out_kind == OUT_CHIRP) {
                    if (n < M) reinterpret_cast<C*>(out)[b * out_stride + n] = cmul(v[q], __ldg(cout + n));
                } else {
                    C r = cscale(v[q], scale);
                    if (conj_out) r = cconj(r);
                    reinterpret_cast<C*>(out)[b * out_stride + n] = r;
                }
            }
        }
    }
}

// mode 0: rows lane-interleaved (TR = Tile::W rows per CTA), natural-order scatter store.
// mode 1: rows contiguous per group, Bluestein middle in place.
// Rows are staged one unit ahead by TMA bulk copies when the staging buffer fits beside the exchange
// buffers (everything but mode 0 at C = 1024).
template <typename T, int LOG2C, int MODE> struct RowCfg {
    using G = FftGeom<LOG2C>;
    static constexpr int ROWS = MODE == 0 ? Tile<T>::W : KCfg<T, LOG2C>::GROUPS;
    static constexpr size_t BASE = ((size_t)ROWS * (G::SMEM + 1) + G::TW_ALLOC) * sizeof(cx_t<T>);
    static constexpr size_t STAGE = 16 + (size_t)ROWS * (G::L + 16 / sizeof(cx_t<T>)) * sizeof(cx_t<T>);
    static constexpr bool STG = BASE + STAGE <= 200 * 1024;
    static constexpr size_t SMEM = BASE + (STG ? STAGE : 0);
};
template <typename T, int LOG2C, int MODE>
__global__ void __launch_bounds__(MODE == 0 ? FftGeom<LOG2C>::NT * Tile<T>::W : KCfg<T, LOG2C>::BLOCK)
k4_row(cx_t<T>* __restrict__ Y, int log2R, long long batch, const cx_t<T>* __restrict__ tw,
       const cx_t<T>* __restrict__ twL, const cx_t<T>* __restrict__ khat_p, cx_t<T>* __restrict__ out,
       long long out_stride, T scale, int conj_out) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2C>;
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ __align__(8) uint64_t stg_bar;
    const long long R = 1LL << log2R;
    const long long Cn = G::L;
    const long long L = R * Cn;
    int g, tid, rows_per_cta;
    if constexpr (MODE == 0) {
        rows_per_cta = Tile<T>::W;
        g = threadIdx.x % rows_per_cta;
        tid = threadIdx.x / rows_per_cta;
    } else {
        rows_per_cta = KCfg<T, LOG2C>::GROUPS;
        g = threadIdx.x / G::NT;
        tid = threadIdx.x % G::NT;
    }
    C* sm = reinterpret_cast<C*>(smraw) + g * (G::SMEM + 1);
    C* tws = reinterpret_cast<C*>(smraw) + rows_per_cta * (G::SMEM + 1);
    // staging for the NEXT unit's rows (one TMA bulk copy per row, rows padded by 16 bytes so the
    // strided register loads below are conflict free), 16-byte aligned after the twiddle tables
    constexpr int RS = (int)G::L + 16 / (int)sizeof(C);
    C* stg = reinterpret_cast<C*>(
        (reinterpret_cast<uintptr_t>(tws + G::TW_ALLOC) + 15) & ~static_cast<uintptr_t>(15));
    load_twiddles<LOG2C>(tws, tw);
    if (threadIdx.x == 0) {
        mbar_init(&stg_bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    const long long tiles = R / rows_per_cta;
    const long long units = tiles * batch;
    // the unit's rows k1 = k1_0 .. k1_0 + rows - 1 are consecutive rows of Y: rows copies of Cn complex
    auto issue = [&](long long un) {
        if (threadIdx.x != 0 || un >= units) return;
        fence_proxy_async_smem();   // earlier generic reads of stg before the async-proxy writes
        const uint32_t row_bytes = (uint32_t)(Cn * sizeof(C));
        mbar_arrive_expect_tx(&stg_bar, row_bytes * (uint32_t)rows_per_cta);
        const C* src = Y + (un / tiles) * L + ((un % tiles) * rows_per_cta) * Cn;
        for (int r = 0; r < rows_per_cta; ++r) bulk_g2s(stg + r * RS, src + r * Cn, row_bytes, &stg_bar);
    };
    constexpr bool STG = RowCfg<T, LOG2C, MODE>::STG;
    if constexpr (STG) issue(blockIdx.x);
    uint32_t parity = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x, parity ^= 1u) {
        const long long b = u / tiles;
        const long long k1 = (u % tiles) * rows_per_cta + g;
        C* row = Y + b * L + k1 * Cn;
        C v[G::EPT];
        if constexpr (STG) {
            mbar_wait(&stg_bar, parity);
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) v[q] = stg[g * RS + tid + G::NT * q];
            __syncthreads();            // every row read out of the staging buffer
            issue(u + gridDim.x);       // the next unit streams in while this one is transformed
        } else {
            const long long un = u + gridDim.x;   // the next unit's rows into L2
            if (un < units) {
                const C* rn = Y + (un / tiles) * L + ((un % tiles) * rows_per_cta + g) * Cn;
                constexpr int per_line = 128 / (int)sizeof(C);
                for (int i = tid * per_line; i < G::L; i += G::NT * per_line) prefetch_l2(rn + i);
            }
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) v[q] = row[tid + G::NT * q];
        }
        block_fft<false, LOG2C>(v, sm, tws, tid);
        if constexpr (MODE == 0) {
            C* o = out + b * out_stride;
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) {
                const long long k2 = tid + (long long)G::NT * q;
                C r = cscale(v[q], scale);
                if (conj_out) r = cconj(r);
                o[k1 + R * k2] = r;
            }
        } else {
            const C* kp = khat_p + k1 * Cn;
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) v[q] = cmul(v[q], __ldg(kp + tid + G::NT * q));
            const C* t = twL + k1 * Cn;
            const C tw_a = __ldg(t + tid), tw_s = __ldg(t + G::NT);   // in flight during the inverse FFT
            block_fft<true, LOG2C>(v, sm, tws, tid);
            // x conj(W_L^{n2 k1}), n2 = tid + NT q, the twiddles formed from two table entries
            twiddle_series(tw_a, tw_s, [&](int q, C w) { row[tid + G::NT * q] = cmulc(v[q], w); });
        }
    }
}

}  // namespace skg

namespace skg {

// SKG_4STEP_PERSIST=0: one CTA per tile (A/B against the persistent grid)
template <typename K> inline unsigned grid_4step(K kern, int block, size_t smem, long long units) {
    static const char* e = std::getenv("SKG_4STEP_PERSIST");
    if (e && e[0] == '0') return (unsigned)units;
    return persistent_grid(kern, block, smem, units);
}

template <typename T>
cudaError_t launch_4step_col_impl(int log2R, bool inverse, int in_kind, int conj_in, const void* x, long long x_stride,
                                  long long N, const void* cin, void* Y, int log2C, long long batch, const void* tw,
                                  const void* twL, int out_kind, void* out, long long out_stride, long long M,
                                  const void* cout, T scale, int conj_out, cudaStream_t st) {
    using C = cx_t<T>;
    return dispatch_log2<4, 10>(log2R, [&](auto lg) {
        constexpr int LG = decltype(lg)::value;
        using G = FftGeom<LG>;
        constexpr int TC = Tile<T>::W;
        const size_t smem = ((size_t)TC * (G::SMEM + 1) + G::TW_ALLOC) * sizeof(C);
        const long long tiles = (1LL << log2C) / TC;
        auto launch = [&](auto kern) {
            cudaError_t e = prep_smem(kern, smem);
            if (e != cudaSuccess) return e;
            kern<<<grid_4step(kern, G::NT * TC, smem, tiles * batch), G::NT * TC, smem, st>>>(
                x, in_kind, conj_in, x_stride, N, (const C*)cin, (C*)Y, log2C, batch, (const C*)tw, (const C*)twL,
                out_kind, out, out_stride, M, (const C*)cout, scale, conj_out);
            return cudaGetLastError();
        };
        if (inverse || in_kind == IN_WORK) return inverse ? launch(k4_col<T, LG, true>) : launch(k4_col<T, LG, false>);
        // rows n1 holding data: C n1 < N  ->  n1 < ceil(N / C)
        const int nz = LG >= 8 ? nz_class((N + (1LL << log2C) - 1) >> log2C, G::NT) : 16;
        if (nz == 4) return launch(k4_col<T, LG, false, 4>);
        if (nz == 8) return launch(k4_col<T, LG, false, 8>);
        return launch(k4_col<T, LG, false>);
    });
}

template <typename T>
cudaError_t launch_4step_row_impl(int log2C, int mode, void* Y, int log2R, long long batch, const void* tw,
                                  const void* twL, const void* khat_p, void* out, long long out_stride, T scale,
                                  int conj_out, cudaStream_t st) {
    using C = cx_t<T>;
    return dispatch_log2<4, 10>(log2C, [&](auto lg) {
        constexpr int LG = decltype(lg)::value;
        using G = FftGeom<LG>;
        const long long R = 1LL << log2R;
        if (mode == 0) {
            constexpr int TR = Tile<T>::W;
            const size_t smem = RowCfg<T, LG, 0>::SMEM;
            auto kern = k4_row<T, LG, 0>;
            cudaError_t e = prep_smem(kern, smem);
            if (e != cudaSuccess) return e;
            kern<<<grid_4step(kern, G::NT * TR, smem, R / TR * batch), G::NT * TR, smem, st>>>((C*)Y, log2R, batch, (const C*)tw,
                                                                       (const C*)twL, (const C*)khat_p, (C*)out,
                                                                       out_stride, scale, conj_out);
        } else {
            using K = KCfg<T, LG>;
            const size_t smem = RowCfg<T, LG, 1>::SMEM;
            auto kern = k4_row<T, LG, 1>;
            cudaError_t e = prep_smem(kern, smem);
            if (e != cudaSuccess) return e;
            kern<<<grid_4step(kern, K::BLOCK, smem, R / K::GROUPS * batch), K::BLOCK, smem, st>>>((C*)Y, log2R, batch, (const C*)tw,
                                                                           (const C*)twL, (const C*)khat_p, (C*)out,
                                                                           out_stride, scale, conj_out);
        }
        return cudaGetLastError();
    });
}

}  // namespace skg
