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
};

template <typename T, int LOG2N>
__global__ void __launch_bounds__(ZoomCfg<LOG2N>::NTH)
k_zoom(const T* __restrict__ x, long long x_stride, long long batch, ZoomArgs a,
       const cx_t<T>* __restrict__ gph,     // taps by phase row: gph[ph * lh + l] = g[l D + (D - ph) % D]
       const cx_t<T>* __restrict__ S,       // S[m], m < nout (already offset by trim)
       const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ band, cx_t<T>* __restrict__ out,
       long long out_stride) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2N>;
    constexpr int NTH = ZoomCfg<LOG2N>::NTH;
    extern __shared__ __align__(16) unsigned char smraw[];
    // shared layout: [FFT buffer][twiddles][wrap terms: mwrap complex][polyphase rows]
    C* fb = reinterpret_cast<C*>(smraw);
    C* tws = fb + (G::L + (G::L >> 4) + 1);
    C* cw = tws + G::TW_ALLOC;
    T* xs = reinterpret_cast<T*>(cw + (a.mwrap + 1));
    const long long b = blockIdx.x;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const T* xr = x + b * x_stride;
    const int D = a.D;
    const int U = (int)a.U;
    const bool dpow2 = (D & (D - 1)) == 0;
    const int ld = 31 - __clz(D);

    // 1. trace -> polyphase rows (zero prefix and tail); clear the FFT buffer; twiddles
    if constexpr (G::L >= 16) load_twiddles<LOG2N>(tws, tw);
    const int total = D * a.rs;
    for (int i = tid; i < total; i += NTH) xs[i] = (T)0;
    for (int i = tid; i < G::L; i += NTH) fb[pad16(i)] = czero<C>();
    __syncthreads();
    for (int n = tid; n < U; n += NTH) {
        const int ph = dpow2 ? (n & (D - 1)) : n % D;
        const int r = dpow2 ? (n >> ld) : n / D;
        xs[ph * a.rs + zpad(r + a.pre)] = __ldg(xr + n);
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
                acc = cadd(acc, rmul(xs[ph * a.rs + zpad(r + a.pre)], g));
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
        for (int ph = 0; ph < D; ++ph) {
            const T* row = xs + ph * a.rs;
            const int delta = ph != 0 ? 1 : 0;
            const C* gr = gph + ph * a.lh;
            // window w[c] = row[m0 + c - l - delta] at tap l, slid by one sample per tap
            T w[ZK];
            const int base = m0 - delta + a.pre;
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
    constexpr int kFb = G::L + (G::L >> 4) + 1 + G::TW_ALLOC;
    const size_t smem = (size_t)(kFb + a.mwrap + 1) * sizeof(C) + (size_t)a.D * a.rs * sizeof(T);
    auto kern = k_zoom<T, LOG2N>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)batch, NTH, smem, st>>>(x, x_stride, batch, a, (const C*)g, (const C*)S, (const C*)tw,
                                             (const C*)band, (C*)out, out_stride);
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
    return (L + (L >> 4) + 1 + tw + a.mwrap + 1) * cs + (size_t)a.D * a.rs * rs;
}
}  // namespace skg
