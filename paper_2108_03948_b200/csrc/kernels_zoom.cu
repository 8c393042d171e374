// kernels_zoom.cu — fused Zoom FFT (zoom_fft, zoomfft.cpp:183-239) for sm_100a.
//
// One CTA per trace:
//   1. the real trace is pulled into shared memory in a polyphase layout xp[ph][r] = x[rD + ph]
//      (rows padded so the FIR's per-thread sliding windows are bank-conflict free);
//   2. frequency shift + FIR + decimation in one pass. The reference forms y[j] = x[j] e^{-i2pi fc j/fs}
//      and then u[m] = sum_t h[t] y[(mD - t) mod U] (zoomfft.cpp:191-193, 82-104). We use the same sum
//      refactored as u[m] = S[m] * sum_t g[t] x[mD - t], with complex taps g[t] = h[t] e^{+i2pi fc t/fs}
//      and S[m] = e^{-i2pi fc mD/fs} (host fp64 tables), so the inner loop multiplies REAL samples by
//      complex taps (2 FMAs per tap, half the shared-memory traffic of the complex y). The few
//      outputs whose window wraps the record end (circular mode) get the exact wrap factor
//      e^{-i2pi fc U/fs} on the wrapped terms;
//   3. each thread owns K = 8 consecutive outputs and slides an 8-sample register window along
//      each polyphase row: 8 loads feed 8x8 complex-by-real MACs (fp64/fp32 pipe bound);
//   4. the decimated block, zero padded to n_fft, runs through the shared Stockham engine;
//   5. the signed band window is gathered and multiplied by D e^{i2pi k delay/(D n_fft)}
//      (table) on the store.
#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"

namespace skg {

constexpr int ZK = kZoomK;   // outputs per thread (register window)

__host__ __device__ inline int zpad(int r) { return r + r / ZK; }

template <int LOG2N> struct ZoomCfg {
    static constexpr int NT = FftGeom<LOG2N>::NT;
    static constexpr int NTH = NT > 128 ? NT : 128;   // CTA width
    // register cap: 4 CTAs of 128 threads per SM for fp32, 3 for fp64 (the FFT-512 stage would spill at 128)
    template <typename T> static constexpr int minb() { return NTH >= 512 ? 1 : (sizeof(T) == 8 ? 384 : 512) / NTH; }
};

template <typename T, int LOG2N>
__global__ void __launch_bounds__(ZoomCfg<LOG2N>::NTH, ZoomCfg<LOG2N>::template minb<T>())
k_zoom(const T* __restrict__ x, long long x_stride, long long batch, ZoomArgs a,
       const cx_t<T>* __restrict__ gph,     // taps by phase row: gph[ph * lh + l] = g[l D + (D - ph) % D]
       const cx_t<T>* __restrict__ S,       // S[m], m < nout (already offset by trim)
       const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ band, cx_t<T>* __restrict__ out,
       long long out_stride, int groups, int gbytes) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2N>;
    // the CTA carries `groups` traces, one per group of GT threads (small records: several per CTA)
    const int GT = ZoomCfg<LOG2N>::NTH / groups;
    const int gi = threadIdx.x / GT;
    extern __shared__ __align__(16) unsigned char smraw[];
    // shared layout: [twiddles][per group: FFT buffer | wrap terms (mwrap complex) | polyphase rows]
    C* tws = reinterpret_cast<C*>(smraw);
    C* fb = reinterpret_cast<C*>(smraw + ((G::TW_ALLOC * sizeof(C) + 15) / 16 * 16) + (size_t)gi * gbytes);
    C* cw = fb + (G::L + (G::L >> 4) + 1);
    T* xs = reinterpret_cast<T*>(cw + (a.mwrap + 1));
    const long long b_raw = (long long)blockIdx.x * groups + gi;
    const bool active = b_raw < batch;
    const long long b = active ? b_raw : batch - 1;   // inactive groups recompute the last trace, store nothing
    const int tid = threadIdx.x % GT;
    const int lane = tid & 31, warp = tid >> 5;
    const T* xr = x + b * x_stride;
    const int D = a.D;
    const int U = (int)a.U;
    const bool dpow2 = (D & (D - 1)) == 0;
    const int ld = 31 - __clz(D);
    const int NTH = GT;

    // 1. trace -> polyphase rows (zero prefix and tail); clear the FFT buffer; twiddles
    if constexpr (G::L >= 16) load_twiddles<LOG2N>(tws, tw);
    const int total = D * a.rs;
    for (int i = tid; i < total; i += NTH) xs[i] = (T)0;
    for (int i = tid; i < G::L; i += NTH) fb[pad16(i)] = czero<C>();
    __syncthreads();
    // the CTA that takes the next trace (blockIdx + gridDim) gets its row pulled into L2 now
    if (b_raw + (long long)gridDim.x * groups < batch) {
        const T* xn = x + (b_raw + (long long)gridDim.x * groups) * x_stride;
        for (int n = tid * (128 / (int)sizeof(T)); n < U; n += NTH * (128 / (int)sizeof(T))) prefetch_l2(xn + n);
    }
    {
        // 16-byte loads, several in flight per thread, scattered into the polyphase rows
        constexpr int V = 16 / (int)sizeof(T);
        const bool vec = ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
        const int nv = vec ? U / V : 0;
        constexpr int UNR = 4;
        for (int i0 = tid; i0 < nv; i0 += NTH * UNR) {
            T buf[UNR][V];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int i = i0 + u * NTH;
                if (i < nv) {
                    if constexpr (sizeof(T) == 8) {
                        const double2 t = __ldg(reinterpret_cast<const double2*>(xr) + i);
                        buf[u][0] = t.x;
                        buf[u][1] = t.y;
                    } else {
                        const float4 t = __ldg(reinterpret_cast<const float4*>(xr) + i);
                        buf[u][0] = t.x;
                        buf[u][1] = t.y;
                        buf[u][2 % V] = t.z;
                        buf[u][3 % V] = t.w;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int i = i0 + u * NTH;
                if (i < nv) {
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        const int n = i * V + e;
                        const int ph = dpow2 ? (n & (D - 1)) : n % D;
                        const int r = dpow2 ? (n >> ld) : n / D;
                        xs[ph * a.rs + zpad(r + a.pre + (ph != 0))] = buf[u][e];
                    }
                }
            }
        }
        for (int n = nv * V + tid; n < U; n += NTH) {   // tail (or the whole row when unaligned)
            const int ph = dpow2 ? (n & (D - 1)) : n % D;
            const int r = dpow2 ? (n >> ld) : n / D;
            xs[ph * a.rs + zpad(r + a.pre + (ph != 0))] = __ldg(xr + n);
        }
    }
    __syncthreads();

    // wrap correction (circular): cw[m] = w * sum_{t > mD} g[t] x[U + mD - t], m < mwrap;
    // one warp per output, lanes stride the taps, shuffle reduction
    if (a.circular) {
        for (int m = warp; m < a.mwrap; m += NTH / 32) {
            C acc = czero<C>();
            for (int t = m * D + 1 + lane; t < a.T; t += 32) {
                const int j = U + m * D - t;
                const int ph = dpow2 ? (j & (D - 1)) : j % D;
                const int r = dpow2 ? (j >> ld) : j / D;
                const int tm = dpow2 ? (t & (D - 1)) : t % D;
                const int trow = tm ? D - tm : 0;   // phase row holding tap t
                const C g = __ldg(gph + trow * a.lh + (dpow2 ? (t >> ld) : t / D));
                acc = cadd(acc, rmul(xs[ph * a.rs + zpad(r + a.pre + (ph != 0))], g));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
            }
            if (lane == 0) cw[m] = cmul(acc, mk<C>((T)a.wre, (T)a.wim));
        }
        __syncthreads();
    }

    // 2-3. FIR over the polyphase rows; a thread owns outputs [m0, m0 + ZK) per chunk
    const int nchunks = (a.nout + ZK - 1) / ZK;
    for (int chunk = tid; chunk < nchunks; chunk += NTH) {
        C acc[ZK];
#pragma unroll
        for (int c = 0; c < ZK; ++c) acc[c] = czero<C>();
        const int m0 = chunk * ZK + a.trim;
        // rows with ph != 0 are stored one slot later, so every row is read at m - l (+ pre); when
        // m0 + pre is a multiple of ZK the window is one padded group: a single address per ZK taps
        const int base = m0 + a.pre;
        if ((base & (ZK - 1)) == 0) {
            const int gb = zpad(base);
            for (int ph = 0; ph < D; ++ph) {
                const T* row = xs + ph * a.rs + gb;
                const C* gr = gph + ph * a.lh;
                T w[ZK];
#pragma unroll
                for (int c = 0; c < ZK; ++c) w[c] = row[c];
                for (int l0 = 0; l0 < a.lh; l0 += ZK) {
                    const T* nr = row - (ZK + 1) * (l0 / ZK + 1);
                    T nw[ZK];
#pragma unroll
                    for (int c = 0; c < ZK; ++c) nw[c] = nr[c];
#pragma unroll
                    for (int s2 = 0; s2 < ZK; ++s2) {
                        const C g = __ldg(gr + l0 + s2);
#pragma unroll
                        for (int c = 0; c < ZK; ++c) {
                            acc[c].x = fma(g.x, w[c], acc[c].x);
                            acc[c].y = fma(g.y, w[c], acc[c].y);
                        }
#pragma unroll
                        for (int c = ZK - 1; c > 0; --c) w[c] = w[c - 1];
                        w[0] = nw[ZK - 1 - s2];
                    }
                }
            }
        } else {
            for (int ph = 0; ph < D; ++ph) {
                const T* row = xs + ph * a.rs;
                const C* gr = gph + ph * a.lh;
                T w[ZK];
#pragma unroll
                for (int c = 0; c < ZK; ++c) w[c] = row[zpad(base + c)];
                for (int l0 = 0; l0 < a.lh; l0 += ZK) {
                    T nw[ZK];
#pragma unroll
                    for (int c = 0; c < ZK; ++c) nw[c] = row[zpad(base - l0 - ZK + c)];
#pragma unroll
                    for (int s2 = 0; s2 < ZK; ++s2) {
                        const C g = __ldg(gr + l0 + s2);
#pragma unroll
                        for (int c = 0; c < ZK; ++c) {
                            acc[c].x = fma(g.x, w[c], acc[c].x);
                            acc[c].y = fma(g.y, w[c], acc[c].y);
                        }
#pragma unroll
                        for (int c = ZK - 1; c > 0; --c) w[c] = w[c - 1];
                        w[0] = nw[ZK - 1 - s2];
                    }
                }
            }
        }
#pragma unroll
        for (int c = 0; c < ZK; ++c) {
            const int m = chunk * ZK + c;   // index in the decimated block
            const int mf = m + a.trim;      // FIR output index
            if (m < a.nout && m < G::L) {
                C v = acc[c];
                if (a.circular && mf < a.mwrap) v = cadd(v, cw[mf]);
                fb[pad16(m)] = cmul(v, __ldg(S + m));
            }
        }
    }
    __syncthreads();

    // 4. FFT of the zero-padded decimated block
    const bool act = tid < G::NT;
    C v[G::EPT];
#pragma unroll
    for (int q = 0; q < G::EPT; ++q) v[q] = act ? fb[pad16(tid + G::NT * q)] : czero<C>();
    __syncthreads();
    block_fft<false, LOG2N>(v, fb, tws, act ? tid : 0, act);
    if (act) {
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) fb[pad16(tid + G::NT * q)] = v[q];
    }
    __syncthreads();

    // 5. signed band window x D x group-delay phase (zoomfft.cpp:209-234)
    C* o = out + b * out_stride;
    if (active)
    for (int i = tid; i < a.nbins; i += NTH) {
        const int k = a.k_lo + i;
        const int idx = ((k % G::L) + G::L) % G::L;
        o[i] = cmul(fb[pad16(idx)], __ldg(band + i));
    }
}

template <typename T, int LOG2N>
static cudaError_t run_zoom(const ZoomArgs& a, const T* x, long long x_stride, long long batch, const void* g,
                            const void* S, const void* tw, const void* band, void* out, long long out_stride,
                            cudaStream_t st) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2N>;
    constexpr int NTH = ZoomCfg<LOG2N>::NTH;
    const size_t twb = (G::TW_ALLOC * sizeof(C) + 15) / 16 * 16;
    const size_t per = ((size_t)(G::L + (G::L >> 4) + 1 + a.mwrap + 1) * sizeof(C) + (size_t)a.D * a.rs * sizeof(T) +
                        15) / 16 * 16;
    // several small records per CTA (one per >= 32-thread group) while a CTA stays <= ~56 KB
    int groups = 1;
    while (groups < 4 && NTH / (groups * 2) >= 32 && NTH / (groups * 2) >= G::NT &&
           twb + per * groups * 2 <= 56 * 1024 && (long long)groups * 2 * 32 <= batch * 32)
        groups *= 2;
    const size_t smem = twb + per * groups;
    auto kern = k_zoom<T, LOG2N>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)((batch + groups - 1) / groups), NTH, smem, st>>>(x, x_stride, batch, a, (const C*)g, (const C*)S,
                                                                       (const C*)tw, (const C*)band, (C*)out,
                                                                       out_stride, groups, (int)per);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t zoom_dispatch(const ZoomArgs& a, int log2n, const T* x, long long x_stride, long long batch,
                                 const void* g, const void* S, const void* tw, const void* band, void* out,
                                 long long out_stride, cudaStream_t st) {
    return dispatch_log2<1, 14>(log2n, [&](auto lg) {
        constexpr int LG = decltype(lg)::value;
        if constexpr (LG > max_log2<T>()) return cudaErrorInvalidValue;
        else return run_zoom<T, LG>(a, x, x_stride, batch, g, S, tw, band, out, out_stride, st);
    });
}

cudaError_t launch_zoom_f64(const ZoomArgs& a, int log2n, const double* x, long long xs, long long batch,
                            const void* g, const void* S, const void* tw, const void* band, void* out,
                            long long os, cudaStream_t st) {
    return zoom_dispatch<double>(a, log2n, x, xs, batch, g, S, tw, band, out, os, st);
}
cudaError_t launch_zoom_f32(const ZoomArgs& a, int log2n, const float* x, long long xs, long long batch,
                            const void* g, const void* S, const void* tw, const void* band, void* out,
                            long long os, cudaStream_t st) {
    return zoom_dispatch<float>(a, log2n, x, xs, batch, g, S, tw, band, out, os, st);
}

// ---- small elementwise helpers -----------------------------------------------------------------
__global__ void k_c64_to_c32(const double2* __restrict__ in, float2* __restrict__ out, long long n) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) out[i] = make_float2((float)in[i].x, (float)in[i].y);
}
__global__ void k_scale_c64(double2* d, long long n, double s) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) d[i] = make_double2(d[i].x * s, d[i].y * s);
}
cudaError_t launch_c64_to_c32(const void* in, void* out, long long n, cudaStream_t st) {
    k_c64_to_c32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((const double2*)in, (float2*)out, n);
    return cudaGetLastError();
}
cudaError_t launch_scale_c64(void* data, long long n, double s, cudaStream_t st) {
    k_scale_c64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((double2*)data, n, s);
    return cudaGetLastError();
}

}  // namespace skg

namespace skg {
size_t zoom_smem_bytes(const ZoomArgs& a, int log2n, bool f32) {
    const size_t L = size_t{1} << log2n;
    const size_t cs = f32 ? 8 : 16, rs = f32 ? 4 : 8;
    int tw = 1;
    dispatch_log2<1, 14>(log2n, [&](auto lg) {
        tw = FftGeom<decltype(lg)::value>::TW_ALLOC;
        return cudaSuccess;
    });
    return ((size_t)tw * cs + 15) / 16 * 16 + ((L + (L >> 4) + 1 + a.mwrap + 1) * cs + (size_t)a.D * a.rs * rs + 15) / 16 * 16;
}
}  // namespace skg

// ---- unfused zoom: FIR/decimate by output chunks into a work buffer, then the FFT (any length, incl.
// multi-pass and the chirp route for non-power-of-two n_fft) and a band-gather kernel. Used when the
// record or the short transform does not fit one CTA's shared memory (cfg5 N = 65536) and for the
// natural-length mode (pad_pow2 = 0, zoomfft.cpp:172).
namespace skg {

constexpr int ZCH_THREADS = 128;
constexpr int ZCH = ZCH_THREADS * ZK;   // outputs per CTA

template <typename T>
__global__ void __launch_bounds__(ZCH_THREADS)
k_zoom_fir(const T* __restrict__ x, long long x_stride, ZoomArgs a, int chunks, const cx_t<T>* __restrict__ gph,
           const cx_t<T>* __restrict__ S, cx_t<T>* __restrict__ zb, long long z_stride) {
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const long long b = blockIdx.x / chunks;
    const int ck = blockIdx.x % chunks;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = a.D, U = (int)a.U;
    const T* xr = x + b * x_stride;
    // rows hold samples n with n/D in [r0 - pre, r0 - pre + rowlen)
    const int m_first = ck * ZCH + a.trim;                 // first FIR output of this chunk
    const int r0 = m_first;                                 // row index of the chunk's first output
    const int rs = a.rs;                                    // padded row stride for ZCH + pre + margin
    C* cw = reinterpret_cast<C*>(smraw);
    T* xs = reinterpret_cast<T*>(cw + (a.mwrap + 1));
    const int span = a.rowlen;                              // unpadded row entries (pre + ZCH + margin)
    for (int i = tid; i < D * rs; i += ZCH_THREADS) xs[i] = (T)0;
    __syncthreads();
    // samples n in [ (r0 - pre) D, (r0 - pre + span) D ) intersect [0, U)
    const long long n_lo = (long long)(r0 - a.pre) * D;
    const long long n_hi = (long long)(r0 - a.pre + span) * D;
    for (long long n = (n_lo < 0 ? 0 : n_lo) + tid; n < n_hi && n < U; n += ZCH_THREADS) {
        const int ph = (int)(n % D);
        const int rr = (int)(n / D) - (r0 - a.pre);
        xs[ph * rs + zpad(rr)] = __ldg(xr + n);
    }
    if (a.circular && ck == 0) {   // wrap terms, read straight from global memory
        for (int m = warp; m < a.mwrap; m += ZCH_THREADS / 32) {
            C acc = czero<C>();
            for (int t = m * D + 1 + lane; t < a.T; t += 32) {
                const int tm = t % D;
                const int trow = tm ? D - tm : 0;
                acc = cadd(acc, rmul(__ldg(xr + (U + m * D - t)), __ldg(gph + trow * a.lh + t / D)));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
            }
            if (lane == 0) cw[m] = cmul(acc, mk<C>((T)a.wre, (T)a.wim));
        }
    }
    __syncthreads();
    const int m_local0 = tid * ZK;                     // within the chunk
    C acc[ZK];
#pragma unroll
    for (int c = 0; c < ZK; ++c) acc[c] = czero<C>();
    for (int ph = 0; ph < D; ++ph) {
        const T* row = xs + ph * rs;
        const int delta = ph != 0 ? 1 : 0;
        const C* gr = gph + ph * a.lh;
        T w[ZK];
        const int base = m_local0 - delta + a.pre;
#pragma unroll
        for (int c = 0; c < ZK; ++c) w[c] = row[zpad(base + c)];
        for (int l0 = 0; l0 < a.lh; l0 += ZK) {
            T nw[ZK];
#pragma unroll
            for (int c = 0; c < ZK; ++c) nw[c] = row[zpad(base - l0 - ZK + c)];
#pragma unroll
            for (int s = 0; s < ZK; ++s) {
                const C g = __ldg(gr + l0 + s);
#pragma unroll
                for (int c = 0; c < ZK; ++c) {
                    acc[c].x = fma(g.x, w[c], acc[c].x);
                    acc[c].y = fma(g.y, w[c], acc[c].y);
                }
#pragma unroll
                for (int c = ZK - 1; c > 0; --c) w[c] = w[c - 1];
                w[0] = nw[ZK - 1 - s];
            }
        }
    }
    C* zr = zb + b * z_stride;
#pragma unroll
    for (int c = 0; c < ZK; ++c) {
        const int m = ck * ZCH + m_local0 + c;   // index in the decimated block
        const int mf = m + a.trim;
        if (m < a.nout) {
            C v = acc[c];
            if (a.circular && mf < a.mwrap) v = cadd(v, cw[mf]);
            zr[m] = cmul(v, __ldg(S + m));
        }
    }
}

template <typename T>
__global__ void k_zoom_band(const cx_t<T>* __restrict__ Z, long long z_stride, long long n_fft, int k_lo, int nbins,
                            const cx_t<T>* __restrict__ band, cx_t<T>* __restrict__ out, long long out_stride) {
    const long long b = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nbins) return;
    const long long k = k_lo + i;
    const long long idx = ((k % n_fft) + n_fft) % n_fft;
    out[b * out_stride + i] = cmul(Z[b * z_stride + idx], __ldg(band + i));
}

// rows needed per chunk: ZCH outputs + pre + margin
int zoom_chunk_rowlen(const ZoomArgs& a) { return a.pre + ZCH + 2 * ZK; }

template <typename T>
static cudaError_t zoom_fir_impl(const ZoomArgs& a, const T* x, long long xs, long long batch, const void* g,
                                 const void* S, void* zb, long long z_stride, cudaStream_t st) {
    using C = cx_t<T>;
    const int chunks = (a.nout + ZCH - 1) / ZCH;
    const size_t smem = (size_t)(a.mwrap + 1) * sizeof(C) + (size_t)a.D * a.rs * sizeof(T);
    auto kern = k_zoom_fir<T>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)(batch * chunks), ZCH_THREADS, smem, st>>>(x, xs, a, chunks, (const C*)g, (const C*)S, (C*)zb,
                                                                 z_stride);
    return cudaGetLastError();
}

cudaError_t launch_zoom_fir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch, const void* g,
                            const void* S, void* zb, long long z_stride, cudaStream_t st) {
    return f32 ? zoom_fir_impl<float>(a, (const float*)x, xs, batch, g, S, zb, z_stride, st)
               : zoom_fir_impl<double>(a, (const double*)x, xs, batch, g, S, zb, z_stride, st);
}

cudaError_t launch_zoom_band(bool f32, const void* Z, long long z_stride, long long n_fft, int k_lo, int nbins,
                             const void* band, void* out, long long out_stride, long long batch, cudaStream_t st) {
    const dim3 grid((unsigned)((nbins + 255) / 256), (unsigned)batch);
    if (f32)
        k_zoom_band<float><<<grid, 256, 0, st>>>((const float2*)Z, z_stride, n_fft, k_lo, nbins, (const float2*)band,
                                                 (float2*)out, out_stride);
    else
        k_zoom_band<double><<<grid, 256, 0, st>>>((const double2*)Z, z_stride, n_fft, k_lo, nbins,
                                                  (const double2*)band, (double2*)out, out_stride);
    return cudaGetLastError();
}

}  // namespace skg
