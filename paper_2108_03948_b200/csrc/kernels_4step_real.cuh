// kernels_4step_real.cuh — the four-step spectrum of REAL traces (fft_spectrum, spectra.cpp:21-38, for
// lengths beyond one CTA) with the Hermitian symmetry of the column transforms.
//
// With n = C n1 + n2, k = k1 + R k2 (kernels_4step.cuh) the column transform of a real trace,
//   Ycol[n2][k1] = sum_n1 x[C n1 + n2] W_R^{n1 k1},
// satisfies Ycol[n2][R - k1] = conj Ycol[n2][k1], and the output satisfies X[L - k] = conj X[k] with
//   L - (k1 + R k2) = (R - k1) + R (C - 1 - k2).
// So only the rows k1 = 0 .. R/2 of the work buffer are formed and transformed:
//   * column unit (colr_unit): two adjacent real columns ride one complex R-point transform
//     z = x[., n2] + i x[., n2 + 1]; the split A = (Z[k1] + conj Z[R-k1]) / 2, B = (Z[k1] - conj Z[R-k1]) / 2i
//     reads the partner through shared memory; A W_L^{n2 k1}, B W_L^{(n2+1) k1} go to Y[k1][n2], Y[k1][n2+1]
//     for k1 <= R/2 as one 16 / 32-byte store — half the column transforms, half the work rows;
//   * row unit (k4_rowh, the row branch of k4_rfused; store: rowh_store): a C-point transform per row k1 <= R/2;
//     each result is stored at
//     k1 + R k2 and, conjugated, at the mirror (R - k1) + R (C - 1 - k2) (rows 0 and R/2 mirror onto
//     themselves and skip it); the half layout (L/2 + 1 bins) keeps whichever of the two is <= L/2.
// HBM traffic per trace: N s + 2 L 2s (work rows written and read once at half size, output once)
// against N s + 3 L 2s for the complex four-step, and half its flops.
#pragma once

#include "kernels_4step.cuh"

namespace skg {

// two twiddle series at once: W0^{e0 + d q}, W1^{e0 + d q}, q < NQ, each from its seed a = W^{e0} and
// step s = W^{d} (products of depth <= 6, as twiddle_series)
template <int NQ, typename C, typename F>
__device__ __forceinline__ void twiddle_series2(C a0, C s0, C a1, C s1, F&& use) {
    const C p2 = cmul(s0, s0), p3 = cmul(p2, s0), p4 = cmul(p2, p2);
    const C r2 = cmul(s1, s1), r3 = cmul(r2, s1), r4 = cmul(r2, r2);
    C b0 = a0, b1 = a1;
#pragma unroll
    for (int j = 0; j < (NQ + 3) / 4; ++j) {
        use(4 * j, b0, b1);
        if (4 * j + 1 < NQ) use(4 * j + 1, cmul(b0, s0), cmul(b1, s1));
        if (4 * j + 2 < NQ) use(4 * j + 2, cmul(b0, p2), cmul(b1, r2));
        if (4 * j + 3 < NQ) use(4 * j + 3, cmul(b0, p3), cmul(b1, r3));
        if (4 * j + 4 < NQ) {
            b0 = cmul(b0, p4);
            b1 = cmul(b1, r4);
        }
    }
}

template <typename T> struct Vec2;   // two adjacent complex values as one store
template <> struct Vec2<float> {
    static __device__ __forceinline__ void st(float2* p, float2 a, float2 b) {
        *reinterpret_cast<float4*>(p) = make_float4(a.x, a.y, b.x, b.y);
    }
};
template <> struct Vec2<double> {
    static __device__ __forceinline__ void st(double2* p, double2 a, double2 b) {
        p[0] = a;
        p[1] = b;
    }
};

// One column unit: the lane's column pair (n2, n2 + 1), n2 even, of one trace. `x` is the trace,
// `Yt` its (R/2 + 1) x C work rows, `sm` the lane group's exchange region, `vec` whether x + n2 may
// be read as aligned pairs. Ends with a CTA barrier (the exchange region is free on return).
template <int S, int NZ, int LOG2L, typename C>
__device__ __forceinline__ void pass_write(C (&v)[16], C* sm, const C* __restrict__ tw, int tid);
template <int LOG2L, typename C> __device__ __forceinline__ void pass_read(C (&v)[16], const C* sm, int tid);

// FUSED (k4_rfused): the passes are spelled out so that the partner exchange can use its own area `smp`
// (no barrier between the last exchange's reads and the partner writes) and the unit ends WITHOUT a
// barrier — the caller's next unit starts with one.
template <typename T, int LOG2R, int NZ, bool FUSED = false>
__device__ __forceinline__ void colr_unit(const T* __restrict__ x, long long N, bool vec, cx_t<T>* __restrict__ Yt,
                                          long long Cn, long long n2, int tid, cx_t<T>* sm,
                                          const cx_t<T>* __restrict__ tws, const cx_t<T>* __restrict__ twL,
                                          cx_t<T>* smp = nullptr) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2R>;
    static_assert(G::EPT == 16, "column transforms of at least 16 points");
    constexpr int R = G::L, NT = G::NT;
    // the store's twiddles W_L^{n2 k1}, k1 = tid + NT q, for both columns: seeds in flight during the transform
    const C* t0 = twL + (long long)tid * Cn + n2;
    const C* t1 = twL + (long long)NT * Cn + n2;
    C a0 = __ldg(t0), a1 = __ldg(t0 + 1);
    const C s0 = __ldg(t1), s1 = __ldg(t1 + 1);
    C v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        C val = czero<C>();
        if (q < NZ) {
            const long long n = (tid + (long long)NT * q) * Cn + n2;
            if (n + 1 < N) {
                if (vec) {
                    val = __ldg(reinterpret_cast<const C*>(x + n));
                } else {
                    val = mk<C>(__ldg(x + n), __ldg(x + n + 1));
                }
            } else if (n < N) {
                val = mk<C>(__ldg(x + n), (T)0);
            }
        }
        v[q] = val;
    }
    if constexpr (FUSED) {
        pass_write<0, NZ, LOG2R>(v, sm, tws, tid);
        __syncthreads();
        pass_read<LOG2R>(v, sm, tid);
        if constexpr (G::P == 3) {
            __syncthreads();
            pass_write<1, 16, LOG2R>(v, sm, tws, tid);
            __syncthreads();
            pass_read<LOG2R>(v, sm, tid);
        }
        stockham_pass<false, G::P - 1, 16, 16, LOG2R>(v, sm, tws, tid);   // last pass: registers only
        sm = smp;
    } else {
        block_fft<false, LOG2R, NZ>(v, sm, tws, tid);
    }
    // partners: Z[R - k1] for k1 = tid + NT q, q < 8, is held in a slot q' >= 8 of another thread;
    // park the upper half at index k - R/2 and read index R/2 - k1
#pragma unroll
    for (int q = 8; q < 16; ++q) sm[tid + NT * (q - 8)] = v[q];
    __syncthreads();
    a0 = cscale(a0, (T)0.5);   // the split's 1/2 rides on the twiddle (exact)
    a1 = cscale(a1, (T)0.5);
    twiddle_series2<9>(a0, s0, a1, s1, [&](int q, C w0, C w1) {
        if (q < 8) {
            const int k1 = tid + NT * q;
            const C z = v[q];
            const C p = k1 == 0 ? z : sm[R / 2 - k1];
            const C sa = mk<C>(z.x + p.x, z.y - p.y);   // Z + conj P
            const C sb = mk<C>(z.y + p.y, p.x - z.x);   // -i (Z - conj P)
            Vec2<T>::st(Yt + (long long)k1 * Cn + n2, cmul(sa, w0), cmul(sb, w1));
        } else if (tid == 0) {   // k1 = R/2: its own partner, both columns real
            const C z = v[8];
            Vec2<T>::st(Yt + (long long)(R / 2) * Cn + n2, cmul(mk<C>(z.x + z.x, (T)0), w0),
                        cmul(mk<C>(z.y + z.y, (T)0), w1));
        }
    });
    if constexpr (!FUSED) __syncthreads();
}

// Row unit's store: v[q] = FFT_C(row k1)[k2 = tid + NT q] -> X[k1 + R k2] and its mirror
template <bool CS, typename C> __device__ __forceinline__ void st_out(C* p, C v) {
    if constexpr (CS) __stcs(p, v);   // written once, never re-read: evict first (the ring should stay in L2)
    else *p = v;
}
template <typename T, int LOG2C, bool CS = false>
__device__ __forceinline__ void rowh_store(const cx_t<T> (&v)[FftGeom<LOG2C>::EPT], cx_t<T>* __restrict__ o,
                                           long long k1, long long R, int tid, bool half) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2C>;
    const long long L = R * G::L;
    const bool self = k1 == 0 || 2 * k1 == R;
#pragma unroll
    for (int q = 0; q < G::EPT; ++q) {
        const long long idx = k1 + R * (tid + (long long)G::NT * q);
        if (!half) {
            st_out<CS>(o + idx, v[q]);
            if (!self) st_out<CS>(o + (L - idx), cconj(v[q]));
        } else if (2 * idx <= L) {
            st_out<CS>(o + idx, v[q]);
        } else if (!self) {
            st_out<CS>(o + (L - idx), cconj(v[q]));
        }
    }
}

#ifndef SKG_4STEP_COLR_THREADS
#define SKG_4STEP_COLR_THREADS 512
#endif
template <typename T, int LOG2R> struct ColrCfg {
    using G = FftGeom<LOG2R>;
    static constexpr int TC = Tile<T>::W;
    static constexpr int BLOCK = G::NT * TC;
    static constexpr int MINB = BLOCK >= SKG_4STEP_COLR_THREADS ? 1 : SKG_4STEP_COLR_THREADS / (BLOCK < 32 ? 32 : BLOCK);
    static constexpr size_t SMEM = ((size_t)TC * (G::SMEM + 1) + G::TW_ALLOC) * sizeof(cx_t<T>);
};

// column pass over real traces: unit = (trace, tile of 2 TC columns); persistent
template <typename T, int LOG2R, int NZ>
__global__ void __launch_bounds__(ColrCfg<T, LOG2R>::BLOCK, ColrCfg<T, LOG2R>::MINB)
k4_colr(const T* __restrict__ x, long long x_stride, long long N, int vec, cx_t<T>* __restrict__ Y, int log2C,
        long long batch, const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ twL) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2R>;
    constexpr int TC = Tile<T>::W;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int g = threadIdx.x % TC, tid = threadIdx.x / TC;
    C* sm = reinterpret_cast<C*>(smraw) + g * (G::SMEM + 1);
    C* tws = reinterpret_cast<C*>(smraw) + TC * (G::SMEM + 1);
    load_twiddles<LOG2R>(tws, tw);
    __syncthreads();
    const long long Cn = 1LL << log2C;
    const long long tiles = Cn / (2 * TC);
    const long long LY = (G::L / 2 + 1) * Cn;
    const long long units = tiles * batch;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const long long b = u / tiles, n2 = ((u % tiles) * TC + g) * 2;
        const long long un = u + gridDim.x;
        if (un < units) {   // the next unit's sample segments into L2 (one lane per 128-byte segment)
            const long long bn = un / tiles, nn2 = (un % tiles) * TC * 2;
            constexpr int per = 128 / (int)sizeof(T);
            if (g * per < 2 * TC) {
#pragma unroll
                for (int q = 0; q < NZ; ++q) {
                    const long long n = (tid + (long long)G::NT * q) * Cn + nn2 + g * per;
                    if (n < N) prefetch_l2(x + bn * x_stride + n);
                }
            }
        }
        colr_unit<T, LOG2R, NZ>(x + b * x_stride, N, vec != 0, Y + b * LY, Cn, n2, tid, sm, tws, twL);
    }
}

// row pass over the half work buffer: unit = (trace, tile of TR rows k1 <= R/2), rows staged one unit
// ahead by TMA bulk copies when the staging buffer fits (as k4_row)
template <typename T, int LOG2C>
__global__ void __launch_bounds__(FftGeom<LOG2C>::NT * Tile<T>::W)
k4_rowh(const cx_t<T>* __restrict__ Y, int log2R, long long batch, const cx_t<T>* __restrict__ tw,
        cx_t<T>* __restrict__ out, long long out_stride, int half) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2C>;
    constexpr int TR = Tile<T>::W;
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ __align__(8) uint64_t stg_bar;
    const long long R = 1LL << log2R;
    const long long Cn = G::L;
    const long long rows = R / 2 + 1;
    const long long LY = rows * Cn;
    const int g = threadIdx.x % TR, tid = threadIdx.x / TR;
    C* sm = reinterpret_cast<C*>(smraw) + g * (G::SMEM + 1);
    C* tws = reinterpret_cast<C*>(smraw) + TR * (G::SMEM + 1);
    constexpr int RS = (int)G::L + 16 / (int)sizeof(C);
    C* stg = reinterpret_cast<C*>((reinterpret_cast<uintptr_t>(tws + G::TW_ALLOC) + 15) & ~static_cast<uintptr_t>(15));
    load_twiddles<LOG2C>(tws, tw);
    if (threadIdx.x == 0) {
        mbar_init(&stg_bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    const long long tiles = (rows + TR - 1) / TR;
    const long long units = tiles * batch;
    constexpr bool STG = RowCfg<T, LOG2C, 0>::STG;
    auto issue = [&](long long un) {
        if (threadIdx.x != 0 || un >= units) return;
        fence_proxy_async_smem();
        const long long r0 = (un % tiles) * TR;
        const int nr = (int)(rows - r0 < TR ? rows - r0 : TR);
        const uint32_t row_bytes = (uint32_t)(Cn * sizeof(C));
        mbar_arrive_expect_tx(&stg_bar, row_bytes * (uint32_t)nr);
        const C* src = Y + (un / tiles) * LY + r0 * Cn;
        for (int r = 0; r < nr; ++r) bulk_g2s(stg + r * RS, src + r * Cn, row_bytes, &stg_bar);
    };
    if constexpr (STG) issue(blockIdx.x);
    uint32_t parity = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x, parity ^= 1u) {
        const long long b = u / tiles;
        const long long k1 = (u % tiles) * TR + g;
        const bool valid = k1 < rows;
        C v[G::EPT];
        if constexpr (STG) {
            mbar_wait(&stg_bar, parity);
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) v[q] = valid ? stg[g * RS + tid + G::NT * q] : czero<C>();
            __syncthreads();
            issue(u + gridDim.x);
        } else {
            const C* row = Y + b * LY + k1 * Cn;
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) v[q] = valid ? row[tid + G::NT * q] : czero<C>();
        }
        block_fft<false, LOG2C>(v, sm, tws, tid);
        if (valid) rowh_store<T, LOG2C>(v, out + b * out_stride, k1, R, tid, half != 0);
    }
}

template <typename T>
cudaError_t launch_4step_colr_impl(int log2R, const void* x, long long x_stride, long long N, void* Y, int log2C,
                                   long long batch, const void* tw, const void* twL, cudaStream_t st) {
    using C = cx_t<T>;
    return dispatch_log2<4, 10>(log2R, [&](auto lg) {
        constexpr int LG = decltype(lg)::value;
        using K = ColrCfg<T, LG>;
        const long long Cn = 1LL << log2C;
        if (Cn < 2 * K::TC) return cudaErrorInvalidValue;
        const long long tiles = Cn / (2 * K::TC);
        const int vec = (reinterpret_cast<uintptr_t>(x) % (2 * sizeof(T)) == 0 && x_stride % 2 == 0) ? 1 : 0;
        auto launch = [&](auto kern) {
            cudaError_t e = prep_smem(kern, K::SMEM);
            if (e != cudaSuccess) return e;
            kern<<<grid_4step(kern, K::BLOCK, K::SMEM, tiles * batch), K::BLOCK, K::SMEM, st>>>(
                (const T*)x, x_stride, N, vec, (C*)Y, log2C, batch, (const C*)tw, (const C*)twL);
            return cudaGetLastError();
        };
        const int nz = LG >= 8 ? nz_class((N + Cn - 1) >> log2C, K::G::NT) : 16;
        if (nz == 4) return launch(k4_colr<T, LG, 4>);
        if (nz == 8) return launch(k4_colr<T, LG, 8>);
        return launch(k4_colr<T, LG, 16>);
    });
}

template <typename T>
cudaError_t launch_4step_rowh_impl(int log2C, const void* Y, int log2R, long long batch, const void* tw, void* out,
                                   long long out_stride, int half, cudaStream_t st) {
    using C = cx_t<T>;
    return dispatch_log2<4, 10>(log2C, [&](auto lg) {
        constexpr int LG = decltype(lg)::value;
        using G = FftGeom<LG>;
        constexpr int TR = Tile<T>::W;
        const size_t smem = RowCfg<T, LG, 0>::SMEM;
        auto kern = k4_rowh<T, LG>;
        cudaError_t e = prep_smem(kern, smem);
        if (e != cudaSuccess) return e;
        const long long rows = (1LL << log2R) / 2 + 1;
        const long long tiles = (rows + TR - 1) / TR;
        kern<<<grid_4step(kern, G::NT * TR, smem, tiles * batch), G::NT * TR, smem, st>>>(
            (const C*)Y, log2R, batch, (const C*)tw, (C*)out, out_stride, half);
        return cudaGetLastError();
    });
}


// ---- both passes in ONE persistent launch, the work rows in an L2-resident ring -------------------------
// The two-launch path writes every trace's work rows to HBM and reads them back (the batch is far larger
// than L2). Here the units of both passes are interleaved in one sequence — step s holds the column units
// of trace s followed by the row units of trace s - delta — and a persistent grid of co-resident CTAs
// (cooperative launch) walks it with stride gridDim.x. A trace's work rows live in slot (trace mod slots)
// of a ring sized to the traces in flight (tens of MB: it stays in the 126 MB L2, rewritten in place), so
// HBM sees the trace once and the spectrum once (ncu: DRAM reads = the traces, writes = 1.1 x the spectra).
// Dependencies point backwards in the sequence only:
//   row unit of trace t   waits for col_done[t] == column units per trace (release/acquire counters);
//   column unit of trace t waits for row_done[t - slots] == row units per trace before reusing the slot;
// every CTA finishes its units in increasing order and blocks only at the start of its own unit, so the
// lowest unfinished unit can always run: no deadlock. With delta ~ 2-3 grids of units the waits are
// already satisfied when reached.
// The row unit needs no staging buffer: its rows are L2 hits, read coalesced under a row-major thread
// mapping (thread = row * NT + position) for the first pass; the pass's shared-memory exchange is read
// back under the lane-interleaved mapping (thread = position * W + row), so the last pass leaves each
// thread with one row's bins k2 and the W rows of a store are adjacent bins k1 — the transposition the
// TMA staging buffer did rides on the exchange the transform needs anyway. Half the shared memory of
// k4_rowh: twice the CTAs per SM.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_inc(unsigned* p) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
    while (ld_acquire_u32(p) < target) __nanosleep(64);
}

// butterflies of a non-final pass S and the exchange's write side (stockham_pass without its barrier / read)
template <int S, int NZ, int LOG2L, typename C>
__device__ __forceinline__ void pass_write(C (&v)[16], C* sm, const C* __restrict__ tw, int tid) {
    using G = FftGeom<LOG2L>;
    constexpr int R = G::radix(S);
    constexpr int p = G::pval(S);
    constexpr int B = G::EPT / R;
    static_assert(S < G::P - 1 && G::EPT == 16, "non-final pass");
#pragma unroll
    for (int b = 0; b < B; ++b) {
        C u[R];
#pragma unroll
        for (int j = 0; j < R; ++j) u[j] = v[b + B * j];
        const int i = tid + G::NT * b;
        const int k = i & (p - 1);
        if constexpr (p > 1) {
            constexpr int ND = G::digits(S);
            constexpr int TO0 = G::tw_off(S, 0), TO1 = G::tw_off(S, 1), TO2 = G::tw_off(S, 2);
            static_assert(ND <= 3, "digits");
            auto wj = [&](int jj) {
                C w = tw[TO0 + jj * 16 + (k & 15)];
                if constexpr (ND > 1) w = cmul(w, tw[TO1 + jj * 16 + ((k >> 4) & 15)]);
                if constexpr (ND > 2) w = cmul(w, tw[TO2 + jj * 16 + ((k >> 8) & 15)]);
                return w;
            };
            if constexpr (sizeof(sc_t<C>) == 8) {
                apply_twiddles<false, R>(u, wj(0));
            } else {
                apply_twiddles<false, R>(u, wj(0), R >= 4 ? wj(1) : czero<C>(), R >= 8 ? wj(2) : czero<C>(),
                                         R >= 16 ? wj(3) : czero<C>());
            }
        }
        dft_r<R, false, (S == 0 ? NZ : 16), 16>(u);
        const int base = (i / p) * p * R + k;
#pragma unroll
        for (int j = 0; j < R; ++j) sm[pad16(base + j * p)] = u[j];
    }
}
template <int LOG2L, typename C> __device__ __forceinline__ void pass_read(C (&v)[16], const C* sm, int tid) {
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = sm[pad16(tid + FftGeom<LOG2L>::NT * q)];
}

#ifndef SKG_RFUSED_W_F32
#define SKG_RFUSED_W_F32 16
#endif
#ifndef SKG_RFUSED_W_F64
#define SKG_RFUSED_W_F64 8
#endif
#ifndef SKG_RFUSED_MINB_F32_256
#define SKG_RFUSED_MINB_F32_256 4   // 64 registers, 4 CTAs per SM: 2^16 fp32 3.20 -> 3.14 ms (3: 85 registers)
#endif
#ifndef SKG_RFUSED_THREADS_F64
#define SKG_RFUSED_THREADS_F64 512   // resident threads per SM the fp64 register cap targets
#endif
#ifndef SKG_RFUSED_MINB_F32_512
#define SKG_RFUSED_MINB_F32_512 2   // 64 registers, 2 CTAs per SM: 2^18 fp32 4.76 -> 4.00 ms
#endif
template <typename T, int LG> struct FusedCfg {
    using G = FftGeom<LG>;
    static constexpr int W = sizeof(T) == 8 ? SKG_RFUSED_W_F64 : SKG_RFUSED_W_F32;   // rows / column pairs per unit
    static constexpr int BLOCK = G::NT * W;
    static constexpr int NCOL = G::L / (2 * W);        // column units per trace
    static constexpr int ROWS = G::L / 2 + 1;          // work rows per trace
    static constexpr int NROW = (ROWS + W - 1) / W;    // row units per trace
    static constexpr int UPS = NCOL + NROW;            // units per step
    static constexpr long long LY = (long long)ROWS * G::L;
    static constexpr int WARPS = BLOCK / 32;
    // [W exchange regions][twiddle tables][W partner areas of R/2 + 1 (the column unit's split)]
    static constexpr size_t SMEM = ((size_t)W * (G::SMEM + 1) + G::TW_ALLOC + (size_t)W * (G::L / 2 + 1)) * sizeof(cx_t<T>);
    static constexpr bool OK = G::L >= 2 * W && G::P >= 2 && G::P <= 3 && BLOCK % 32 == 0;
    // registers: fp64 holds 16 complex = 64 registers of data (128 per thread); fp32 runs at 85 / 128
    // fp32: 768 resident threads (85 registers) for 256-point transforms, 1024 (64 registers) for 512-point ones
    static constexpr int MINB = sizeof(T) == 8 ? SKG_RFUSED_THREADS_F64 / BLOCK
                                               : (LG >= 9 ? SKG_RFUSED_MINB_F32_512 * 512 : SKG_RFUSED_MINB_F32_256 * 256) / BLOCK;
};

#ifndef SKG_RFUSED_CS
#define SKG_RFUSED_CS 1
#endif
template <typename T, int LG, int NZ>
__global__ void __launch_bounds__(FusedCfg<T, LG>::BLOCK, FusedCfg<T, LG>::MINB)
k4_rfused(const T* __restrict__ x, long long x_stride, long long N, int vec, cx_t<T>* Yring, int slots, int delta,
          long long batch, const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ twL, cx_t<T>* __restrict__ out,
          long long out_stride, int half, unsigned* col_done, unsigned* row_done) {
    using C = cx_t<T>;
    using G = FftGeom<LG>;
    using F = FusedCfg<T, LG>;
    constexpr int W = F::W;
    constexpr long long Cn = G::L, R = G::L;
    extern __shared__ __align__(16) unsigned char smraw[];
    // lane-interleaved mapping (column units; the row unit's last pass and stores)
    const int g = threadIdx.x % W, tid = threadIdx.x / W;
    // row-major mapping (the row unit's loads and first passes)
    const int ga = threadIdx.x / G::NT, ta = threadIdx.x % G::NT;
    C* sm = reinterpret_cast<C*>(smraw) + g * (G::SMEM + 1);
    C* sma = reinterpret_cast<C*>(smraw) + ga * (G::SMEM + 1);
    C* tws = reinterpret_cast<C*>(smraw) + W * (G::SMEM + 1);
    C* smp = tws + G::TW_ALLOC + g * (G::L / 2 + 1);   // odd stride: the W lanes on distinct banks
    load_twiddles<LG>(tws, tw);
    const long long units = (batch + delta) * F::UPS;
    // the counter a unit waits on before it starts (nullptr: none) and its target
    auto dep = [&](long long uu, unsigned& target) -> const unsigned* {
        if (uu >= units) return nullptr;
        const long long ss = uu / F::UPS;
        const int jj = (int)(uu % F::UPS);
        if (jj < F::NCOL) {   // column unit: the slot's previous trace fully read
            target = (unsigned)F::NROW;
            return ss < batch && ss >= slots ? row_done + (ss - slots) : nullptr;
        }
        target = (unsigned)(F::NCOL * F::WARPS);   // row unit: every warp of every column unit released
        return ss >= delta ? col_done + (ss - delta) : nullptr;
    };
    bool ready = false;   // thread 0: this unit's dependency was seen satisfied during the previous unit
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const long long s = u / F::UPS;
        const int j = (int)(u % F::UPS);
        const bool is_col = j < F::NCOL;
        if (is_col ? s >= batch : s < delta) {   // no work in this unit
            ready = false;
            continue;
        }
        if (threadIdx.x == 0) {
            unsigned target;
            const unsigned* d = dep(u, target);
            if (d && !ready) wait_count(d, target);
        }
        __syncthreads();   // dependency satisfied; every thread has left the previous unit's shared memory
        if (threadIdx.x == 0) {   // peek at the next unit's dependency: the load is in flight during this unit
            unsigned target;
            const unsigned* d = dep(u + gridDim.x, target);
            ready = d ? ld_acquire_u32(d) >= target : true;
        }
        if (is_col) {
            {   // the next column unit's sample segments into L2 (one lane per 128-byte segment)
                const long long un = u + gridDim.x;
                const long long sn = un / F::UPS;
                const int jn = (int)(un % F::UPS);
                if (g == 0 && jn < F::NCOL && sn < batch) {
                    const long long nn2 = (long long)jn * W * 2;
#pragma unroll
                    for (int q = 0; q < NZ; ++q) {
                        const long long n = (tid + (long long)G::NT * q) * Cn + nn2;
                        if (n < N) prefetch_l2(x + sn * x_stride + n);
                    }
                }
            }
            const long long n2 = ((long long)j * W + g) * 2;
            colr_unit<T, LG, NZ, true>(x + s * x_stride, N, vec != 0, Yring + (s % slots) * F::LY, Cn, n2, tid, sm,
                                       tws, twL, smp);
            __syncwarp();   // the warp's work-row stores, then one release per warp
            if ((threadIdx.x & 31) == 0) red_release_inc(col_done + s);
        } else {
            const long long t = s - delta;
            const int r0 = (j - F::NCOL) * W;
            // the rows are L2 hits written by other SMs in this launch: ld.cg (an L1 line could be a stale
            // copy of the slot's previous trace)
            const C* row = Yring + (t % slots) * F::LY + (long long)(r0 + ga) * Cn + ta;
            const bool valid_a = r0 + ga < F::ROWS;
            C v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = valid_a ? __ldcg(row + G::NT * q) : czero<C>();
            pass_write<0, 16, LG>(v, sma, tws, ta);
            if constexpr (G::P == 3) {   // the middle pass stays row-major: its exchange is warp-local when NT <= 32
                if constexpr (G::NT <= 32) __syncwarp(); else __syncthreads();
                pass_read<LG>(v, sma, ta);
                if constexpr (G::NT <= 32) __syncwarp(); else __syncthreads();
                pass_write<1, 16, LG>(v, sma, tws, ta);
            }
            __syncthreads();   // every row of the unit has been read out of the slot
            if (threadIdx.x == 0) red_release_inc(row_done + t);
            pass_read<LG>(v, sm, tid);
            stockham_pass<false, G::P - 1, 16, 16, LG>(v, sm, tws, tid);   // last pass: registers only
            const long long k1 = r0 + g;
            if (k1 < F::ROWS)
                rowh_store<T, LG, SKG_RFUSED_CS != 0>(v, out + t * out_stride, k1, R, tid, half != 0);
        }
    }
}

template <typename T>
cudaError_t launch_4step_rfused_impl(int lg, const void* x, long long x_stride, long long N, void* Yring, int slots,
                                     int delta, long long batch, const void* tw, const void* twL, void* out,
                                     long long out_stride, int half, unsigned* col_done, unsigned* row_done,
                                     int* grid_out, int* ups_out, cudaStream_t st) {
    using C = cx_t<T>;
    return dispatch_log2<8, 9>(lg, [&](auto lgc) {
        constexpr int LG = decltype(lgc)::value;
        using F = FusedCfg<T, LG>;
        if constexpr (!F::OK) {
            return cudaErrorInvalidValue;
        } else {
            const long long Cn = 1LL << LG;
            const int vec = (reinterpret_cast<uintptr_t>(x) % (2 * sizeof(T)) == 0 && x_stride % 2 == 0) ? 1 : 0;
            auto launch = [&](auto kern) {
                cudaError_t e = prep_smem(kern, F::SMEM);
                if (e != cudaSuccess) return e;
                const unsigned grid = persistent_grid(kern, F::BLOCK, F::SMEM, 1LL << 40);
                if (grid_out) {   // sizing query: the grid the launch will use
                    *grid_out = (int)grid;
                    if (ups_out) *ups_out = F::UPS;
                    return cudaSuccess;
                }
                const T* xp = (const T*)x;
                C* yp = (C*)Yring;
                const C* twp = (const C*)tw;
                const C* twlp = (const C*)twL;
                C* op = (C*)out;
                void* args[] = {&xp, &x_stride, &N, (void*)&vec, &yp, &slots, &delta, &batch, &twp, &twlp, &op,
                                &out_stride, &half, &col_done, &row_done};
                return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(F::BLOCK), args, F::SMEM, st);
            };
            const int nz = LG >= 8 ? nz_class((N + Cn - 1) >> LG, F::G::NT) : 16;
            if (nz == 4) return launch(k4_rfused<T, LG, 4>);
            if (nz == 8) return launch(k4_rfused<T, LG, 8>);
            return launch(k4_rfused<T, LG, 16>);
        }
    });
}

}  // namespace skg
