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
#include "bulk_copy.cuh"
#include "kernels_zoom_fir.cuh"

namespace skg {

constexpr int ZK = kZoomK;   // outputs per thread (register window)

__host__ __device__ inline int zpad(int r) { return r + r / ZK; }

template <int LOG2N> struct ZoomCfg {
    static constexpr int NT = FftGeom<LOG2N>::NT;
    static constexpr int NTH = NT > 128 ? NT : 128;   // CTA width
    // register cap: 4 CTAs of 128 threads per SM for fp32, 3 for fp64 (its FFT stage spills at 128)
#ifndef SKG_ZOOM_F64_CTAS
#define SKG_ZOOM_F64_CTAS 3
#endif
    template <typename T> static constexpr int minb() {
        return NTH >= 512 ? 1 : (sizeof(T) == 8 ? SKG_ZOOM_F64_CTAS * 128 : 512) / NTH;
    }
};

template <typename T, int LOG2N>
__global__ void __launch_bounds__(ZoomCfg<LOG2N>::NTH, ZoomCfg<LOG2N>::template minb<T>())
k_zoom(const T* __restrict__ x, long long x_stride, long long batch, ZoomArgs a,
       const cx_t<T>* __restrict__ gph,     // taps by phase row: gph[ph * lh + l] = g[l D + (D - ph) % D]
       const cx_t<T>* __restrict__ S,       // S[m], m < nout (already offset by trim)
       const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ band, cx_t<T>* __restrict__ out,
       long long out_stride, int groups, int gbytes, int stage_off) {
    using C = cx_t<T>;
    using G = FftGeom<LOG2N>;
    // persistent: the CTA carries `groups` traces at a time (one per group of GT threads; several
    // only for small records) and walks the batch with stride gridDim.x * groups. With staging
    // (stage_off > 0) the group's next raw record is TMA-bulk-copied into shared memory while the
    // current one is filtered and transformed, so HBM streams under the compute.
    const int GT = ZoomCfg<LOG2N>::NTH / groups;
    const int gi = threadIdx.x / GT;
    extern __shared__ __align__(16) unsigned char smraw[];
    // shared layout: [twiddles][taps D x lh][mbarriers][per group: FFT buffer | wrap terms | polyphase rows | stage]
    C* tws = reinterpret_cast<C*>(smraw);
    const size_t twb = (G::TW_ALLOC * sizeof(C) + 15) / 16 * 16;
    C* s_g = reinterpret_cast<C*>(smraw + twb);
    C* s_gn = s_g + a.D * a.lh;   // the same taps in natural order g[t], t < T (wrap correction)
    const size_t gb = ((size_t)(a.D * a.lh + a.T) * sizeof(C) + 15) / 16 * 16;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smraw + twb + gb);
    unsigned char* grp = smraw + twb + gb + ((size_t)groups * 8 + 15) / 16 * 16 + (size_t)gi * gbytes;
    C* fb = reinterpret_cast<C*>(grp);
    C* cw = fb + (G::L + (G::L >> 4) + 1);
    T* xs = reinterpret_cast<T*>(cw + (a.mwrap + 1));
    T* stage = stage_off ? reinterpret_cast<T*>(grp + stage_off) : nullptr;
    uint64_t* bar = bars + gi;
    const int tid = threadIdx.x % GT;
    const int lane = tid & 31, warp = tid >> 5;
    const int D = a.D;
    const int U = (int)a.U;
    const bool dpow2 = (D & (D - 1)) == 0;
    const int ld = 31 - __clz(D);
    const int NTH = GT;
    // bytes of each record the bulk copy moves (a multiple of 16); the tail comes from global
    const uint32_t nbulk = (uint32_t)((size_t)U * sizeof(T)) & ~15u;
    const int nbulk_el = (int)(nbulk / sizeof(T));
    const long long nslots = (batch + groups - 1) / groups;
    auto trace_of = [&](long long slot) {
        const long long br = slot * groups + gi;
        return br < batch ? br : batch - 1;   // inactive groups recompute the last trace, store nothing
    };

    // once per CTA: twiddles, taps, zero polyphase rows (prefix/tail margins stay zero), barriers
    if constexpr (G::L >= 16) load_twiddles<LOG2N>(tws, tw);
    for (int i = threadIdx.x; i < a.D * a.lh; i += blockDim.x) s_g[i] = __ldg(gph + i);
    for (int t = threadIdx.x; t < a.T; t += blockDim.x) {
        const int tm = t % D;
        s_gn[t] = __ldg(gph + (tm ? D - tm : 0) * a.lh + t / D);
    }
    for (int i = tid; i < D * a.rs; i += NTH) xs[i] = (T)0;
    if (stage && tid == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (stage && tid == 0 && blockIdx.x < nslots && nbulk) {
        mbar_arrive_expect_tx(bar, nbulk);
        bulk_g2s(stage, x + trace_of(blockIdx.x) * x_stride, nbulk, bar);
    }
    uint32_t parity = 0;
    for (long long slot = blockIdx.x; slot < nslots; slot += gridDim.x) {
        const long long b = trace_of(slot);
        const bool active = slot * groups + gi < batch;
        const T* xr = x + b * x_stride;
        auto put = [&](int n, T v) {   // sample n -> its polyphase row
            const int ph = dpow2 ? (n & (D - 1)) : n % D;
            const int r = dpow2 ? (n >> ld) : n / D;
            xs[ph * a.rs + zpad(r + a.pre + (ph != 0))] = v;
        };
        // 1. record -> polyphase rows
        constexpr int V = 16 / (int)sizeof(T);
        // with D a power of two dividing NTH*V (and the row step a multiple of ZK), a thread's samples
        // keep their phase rows from one sweep to the next: precompute the V destinations, then step
        const int rstep = dpow2 ? (NTH * V) >> ld : 0;
        const bool incr = dpow2 && ((NTH * V) & (D - 1)) == 0 && (rstep % ZK) == 0;
        int dst0[V];
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const int n = tid * V + k;
            const int ph = n & (D - 1);
            dst0[k] = ph * a.rs + zpad((n >> ld) + a.pre + (ph != 0));
        }
        const int dstep = rstep + rstep / ZK;
        if (stage) {
            if (nbulk) mbar_wait(bar, parity);
            parity ^= 1;
            using VT = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
            const int nv = nbulk_el / V;
            if (incr) {
                int it = 0;
                for (int i = tid; i < nv; i += NTH, ++it) {
                    const VT t = reinterpret_cast<const VT*>(stage)[i];
                    const T* e = reinterpret_cast<const T*>(&t);
#pragma unroll
                    for (int k = 0; k < V; ++k) xs[dst0[k] + it * dstep] = e[k];
                }
            } else {
                for (int i = tid; i < nv; i += NTH) {
                    const VT t = reinterpret_cast<const VT*>(stage)[i];
                    const T* e = reinterpret_cast<const T*>(&t);
#pragma unroll
                    for (int k = 0; k < V; ++k) put(i * V + k, e[k]);
                }
            }
            for (int n = nv * V + tid; n < U; n += NTH) put(n, __ldg(xr + n));
        } else {
            // the CTA's next record is pulled into L2 while this one is loaded and filtered
            if (slot + gridDim.x < nslots) {
                const T* xn = x + trace_of(slot + gridDim.x) * x_stride;
                for (int n = tid * (128 / (int)sizeof(T)); n < U; n += NTH * (128 / (int)sizeof(T))) prefetch_l2(xn + n);
            }
            // 16-byte loads, several in flight per thread, scattered into the polyphase rows
            const bool vec = ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
            const int nv = vec ? U / V : 0;
            constexpr int UNR = 4;
            for (int i0 = tid, it0 = 0; i0 < nv; i0 += NTH * UNR, it0 += UNR) {
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
                            if (incr) xs[dst0[e] + (it0 + u) * dstep] = buf[u][e];
                            else put(i * V + e, buf[u][e]);
                        }
                    }
                }
            }
            for (int n = nv * V + tid; n < U; n += NTH) put(n, __ldg(xr + n));   // tail / unaligned row
        }
        // wrap correction (circular): cw[m] = w * sum_{s=1}^{T-1-mD} g[mD + s] x[U - s], m < mwrap — the
        // terms whose window wraps the record end; one warp per output, lanes stride s, shuffle sum.
        // Reads only global samples and the natural-order taps, so it needs no barrier of its own.
        if (a.circular) {
            // half-warps own outputs (two per warp per sweep), lanes stride s; 4-level shuffle sums
            const int h = lane >> 4, hl = lane & 15;
            for (int m0 = 2 * warp; m0 < a.mwrap; m0 += 2 * (NTH / 32)) {
                const int m = m0 + h;
                C acc = czero<C>();
                if (m < a.mwrap)
                    for (int s1 = 1 + hl; s1 <= a.T - 1 - m * D; s1 += 16) {
                        const int j = U - s1;   // staged records are read from shared memory, others via L1
                        const T xv = (stage && j < nbulk_el) ? stage[j] : __ldg(xr + j);
                        acc = cadd(acc, rmul(xv, s_gn[m * D + s1]));
                    }
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                }
                if (hl == 0 && m < a.mwrap) cw[m] = cmul(acc, mk<C>((T)a.wre, (T)a.wim));
            }
        }
        __syncthreads();
        // the stage is free again: start the group's next record
        if (stage && tid == 0 && slot + gridDim.x < nslots && nbulk) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(bar, nbulk);
            bulk_g2s(stage, x + trace_of(slot + gridDim.x) * x_stride, nbulk, bar);
        }

        // 2-3. FIR over the polyphase rows; a thread owns outputs [m0, m0 + ZK) per chunk. Row ph
        // holds the taps t = l D + (D - ph) % D: only ceil(count / ZK) blocks of ZK are run per row
        const int nchunks = (a.nout + ZK - 1) / ZK;
        for (int chunk = tid; chunk < nchunks; chunk += NTH) {
            C acc[ZK];
#pragma unroll
            for (int c = 0; c < ZK; ++c) acc[c] = czero<C>();
            const int m0 = chunk * ZK + a.trim;
            // rows with ph != 0 are stored one slot later, so every row is read at m - l (+ pre); when
            // m0 + pre is a multiple of ZK the window is one padded group: a single address per ZK taps
            const int base = m0 + a.pre;
            const bool aligned = (base & (ZK - 1)) == 0;
            for (int ph = 0; ph < D; ++ph) {
                const int t0 = ph ? D - ph : 0;
                const int cnt = t0 < a.T ? (a.T - t0 + D - 1) / D : 0;
                const int lend = (cnt + ZK - 1) / ZK * ZK;
                const T* rowp = xs + ph * a.rs;
                const C* gr = s_g + ph * a.lh;
                T w[ZK];
                if (aligned) {
                    const T* row = rowp + zpad(base);
#pragma unroll
                    for (int c = 0; c < ZK; ++c) w[c] = row[c];
                } else {
#pragma unroll
                    for (int c = 0; c < ZK; ++c) w[c] = rowp[zpad(base + c)];
                }
                for (int l0 = 0; l0 < lend; l0 += ZK) {
                    T nw[ZK];
                    if (aligned) {
                        const T* nr = rowp + zpad(base) - (ZK + 1) * (l0 / ZK + 1);
#pragma unroll
                        for (int c = 0; c < ZK; ++c) nw[c] = nr[c];
                    } else {
#pragma unroll
                        for (int c = 0; c < ZK; ++c) nw[c] = rowp[zpad(base - l0 - ZK + c)];
                    }
#pragma unroll
                    for (int s2 = 0; s2 < ZK; ++s2) {
                        const C g = gr[l0 + s2];
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

        // 4. FFT of the zero-padded decimated block (positions >= nout read as zero)
        const bool act = tid < G::NT;
        const int nvalid = a.nout < G::L ? a.nout : G::L;
        C v[G::EPT];
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            const int pos = tid + G::NT * q;
            v[q] = (act && pos < nvalid) ? fb[pad16(pos)] : czero<C>();
        }
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
}

inline size_t zoom_head_bytes(const ZoomArgs& a, size_t twb, size_t cs, int groups) {
    return twb + ((size_t)(a.D * a.lh + a.T) * cs + 15) / 16 * 16 + ((size_t)groups * 8 + 15) / 16 * 16;
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
    // staging for the TMA record stream when rows are 16-byte aligned and it fits next to the rest
    const size_t stage_b = ((size_t)a.U * sizeof(T) + 15) / 16 * 16;
    const bool aligned = ((uintptr_t)x % 16 == 0) && ((x_stride * (long long)sizeof(T)) % 16 == 0);
    static const bool no_stage = getenv("SKG_ZOOM_NO_STAGE") != nullptr;
    const bool stage = !no_stage && aligned && a.U * (long long)sizeof(T) >= 16 &&
                       zoom_head_bytes(a, twb, sizeof(C), groups) + (per + stage_b) * groups <= (size_t)smem_optin();
    const size_t gbytes = per + (stage ? stage_b : 0);
    const size_t smem = zoom_head_bytes(a, twb, sizeof(C), groups) + gbytes * groups;
    auto kern = k_zoom<T, LOG2N>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long long slots = (batch + groups - 1) / groups;
    kern<<<persistent_grid(kern, NTH, smem, slots), NTH, smem, st>>>(x, x_stride, batch, a, (const C*)g, (const C*)S,
                                                                      (const C*)tw, (const C*)band, (C*)out,
                                                                      out_stride, groups, (int)gbytes,
                                                                      stage ? (int)per : 0);
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
    return ((size_t)tw * cs + 15) / 16 * 16 + ((size_t)(a.D * a.lh + a.T) * cs + 15) / 16 * 16 + 16 +
           ((L + (L >> 4) + 1 + a.mwrap + 1) * cs + (size_t)a.D * a.rs * rs + 15) / 16 * 16;
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

// ---- split zoom (default): warp-chunk FIR -> L2-resident work rows -> batched FFT + band gather ----
// The FIR is the dominant cost (T complex taps per output) and needs occupancy to keep the FP pipe
// fed; a fused one-CTA-per-record kernel is held to ~2 CTAs per SM by its record-sized shared rows
// and leaves three of four warps idle in the short FFT. Here every warp owns 32*ZK consecutive
// outputs of one record and its own small polyphase window (no CTA barriers), and the transform
// runs as a separate batched kernel with several records per CTA. The work rows (nout complex per
// record) are sized by the host to stay in L2 between the two launches.
namespace skg {

constexpr int WF_WARPS = 4;
constexpr int WZK = 8;            // FIR outputs per lane (16 independent FMA chains)
constexpr int WF_OUT = 32 * WZK;  // outputs per warp task

// A warp's polyphase window keeps each phase row contiguous (no padding): the FIR's lane reads
// (position 8*lane + c, same row for all lanes) are made conflict free by an XOR swizzle of the
// low three bits with bits 4-6, which spreads every 16 consecutive lanes over 16 distinct 8-byte
// bank pairs. The row stride is kept = 2 (mod 16) so the pair-wise scatter (two consecutive samples
// -> two phase rows) is conflict free too.
__device__ __forceinline__ int wsw(int p) { return p ^ ((p >> 4) & 7); }

int zoom_wfir_rs(const ZoomArgs& a) {
    // positions 0..span are written and the swizzle permutes within aligned groups of 8
    const int need = ((a.pre + WF_OUT + 2 * ZK) | 7) + 1;
    int rs = (need + 15) / 16 * 16 + 2;
    if (rs - 16 >= need) rs -= 16;
    return rs;
}

template <typename T>
__global__ void __launch_bounds__(WF_WARPS * 32, 4)
k_zoom_wfir(const T* __restrict__ x, long long x_stride, long long batch, ZoomArgs a, int wchunks, int wrs,
            int wbytes, const cx_t<T>* __restrict__ gph, const cx_t<T>* __restrict__ S, cx_t<T>* __restrict__ zb,
            long long z_stride) {
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int D = a.D, U = (int)a.U;
    const bool dpow2 = (D & (D - 1)) == 0;
    const int ld = 31 - __clz(D);
    // [taps by phase row D x lh][taps in natural order T][row tap counts D][per warp: wrap terms | window]
    C* s_g = reinterpret_cast<C*>(smraw);
    C* s_gn = s_g + a.D * a.lh;
    int* s_lend = reinterpret_cast<int*>(s_gn + a.T);
    for (int i = threadIdx.x; i < a.D * a.lh; i += blockDim.x) s_g[i] = __ldg(gph + i);
    for (int t = threadIdx.x; t < a.T; t += blockDim.x) {
        const int tm = t % D;
        s_gn[t] = __ldg(gph + (tm ? D - tm : 0) * a.lh + t / D);
    }
    for (int ph = threadIdx.x; ph < D; ph += blockDim.x) {   // taps in row ph, rounded up to ZK
        const int t0 = ph ? D - ph : 0;
        const int cnt = t0 < a.T ? (a.T - t0 + D - 1) / D : 0;
        s_lend[ph] = (cnt + ZK - 1) / ZK * ZK;
    }
    unsigned char* wr = smraw + ((size_t)(a.D * a.lh + a.T) * sizeof(C) + (size_t)D * 4 + 15) / 16 * 16 +
                        (size_t)warp * wbytes;
    C* cw = reinterpret_cast<C*>(wr);
    T* xs = reinterpret_cast<T*>(cw + (a.mwrap + 1));
    __syncthreads();   // the only CTA-wide barrier: warps are independent from here on
    const long long ntasks = batch * wchunks;
    const long long tstride = (long long)gridDim.x * WF_WARPS;
    const int span = a.pre + WF_OUT + 2 * ZK;
    const int ntot = span * D;   // window samples n in [r_lo D, r_lo D + ntot)
    // sample n -> (phase row, swizzled position); position p = r - r_lo + (ph != 0)
    auto slot = [&](int n, int r_lo) {
        int ph, r;
        if (dpow2) {
            ph = n & (D - 1);
            r = n >> ld;
        } else {
            r = n >= 0 ? n / D : -((-n + D - 1) / D);
            ph = n - r * D;
        }
        return ph * wrs + wsw(r - r_lo + (ph != 0));
    };
    for (long long task = (long long)blockIdx.x * WF_WARPS + warp; task < ntasks; task += tstride) {
        const long long b = task / wchunks;
        const int ck = (int)(task % wchunks);
        const T* xr = x + b * x_stride;
        const int m_lo = ck * WF_OUT;
        const int mf_lo = m_lo + a.trim;
        const int r_lo = mf_lo - a.pre;
        const int n0 = r_lo * D;
        // the warp's next window is pulled into L2 while this one is filtered
        {
            const long long tn = task + tstride;
            if (tn < ntasks) {
                const long long bn = tn / wchunks;
                const int nn0 = max(((int)(tn % wchunks) * WF_OUT + a.trim - a.pre) * D, 0);
                const int nn1 = min(nn0 + ntot, U);
                const T* xn = x + bn * x_stride;
                for (int n = nn0 + lane * (128 / (int)sizeof(T)); n < nn1; n += 32 * (128 / (int)sizeof(T)))
                    prefetch_l2(xn + n);
            }
        }
        // the output chirp S for this lane's outputs, in flight during the FIR
        C sv[WZK];
#pragma unroll
        for (int c = 0; c < WZK; ++c) {
            const int m = m_lo + lane * WZK + c;
            sv[c] = m < a.nout ? __ldg(S + m) : czero<C>();
        }
        // record -> polyphase window (zeros outside the record)
        // record -> polyphase window with asynchronous per-sample copies (cp.async, no registers
        // held, every copy of the window in flight at once); zero fill outside [0, U)
        if (dpow2 && D <= 32) {
            // a lane keeps its phase row across the sweep; the row position advances by 32 / D
            const int ph = (n0 + lane) & (D - 1);
            int p = ((n0 + lane) >> ld) - r_lo + (ph != 0);
            T* rowp = xs + ph * wrs;
            const int dp = 32 >> ld;
            for (int n = n0 + lane; n < n0 + ntot; n += 32, p += dp) {
                const bool ok = n >= 0 && n < U;
                cp_async_el(rowp + wsw(p), xr + (ok ? n : 0), ok);
            }
        } else {
            for (int i = lane; i < ntot; i += 32) {
                const int n = n0 + i;
                const bool ok = n >= 0 && n < U;
                cp_async_el(xs + slot(n, r_lo), xr + (ok ? n : 0), ok);
            }
        }
        cp_async_commit();
        // wrap correction (circular) for the outputs this task owns below mwrap:
        // cw[m] = w * sum_{s=1}^{T-1-mD} g[mD + s] x[U - s]; half-warps own outputs, 4-level shuffle sums
        const bool wraps = a.circular && mf_lo < a.mwrap;
        if (wraps) {
            const int h = lane >> 4, hl = lane & 15;
            for (int m0 = mf_lo; m0 < min(a.mwrap, mf_lo + WF_OUT); m0 += 2) {
                const int m = m0 + h;
                C acc = czero<C>();
                if (m < a.mwrap)
                    for (int s1 = 1 + hl; s1 <= a.T - 1 - m * D; s1 += 16)
                        acc = cadd(acc, rmul(__ldg(xr + U - s1), s_gn[m * D + s1]));
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                }
                if (hl == 0 && m < a.mwrap) cw[m - mf_lo] = cmul(acc, mk<C>((T)a.wre, (T)a.wim));
            }
        }
        cp_async_wait_all();
        __syncwarp();
        // FIR: lane owns outputs mf_lo + lane WZK + [0, WZK); window position a.pre + lane WZK + c - l,
        // new samples fetched four at a time (rows hold ceil(count / 4) * 4 taps)
        C acc[WZK];
#pragma unroll
        for (int c = 0; c < WZK; ++c) acc[c] = czero<C>();
        const int base = a.pre + lane * WZK;   // a multiple of 4
        for (int ph = 0; ph < D; ++ph) {
            const int lend = s_lend[ph];
            const T* row = xs + ph * wrs;
            const C* gr = s_g + ph * a.lh;
            T wv[WZK];
#pragma unroll
            for (int c = 0; c < WZK; ++c) wv[c] = row[wsw(base + c)];
            for (int l0 = 0; l0 < lend; l0 += ZK) {
                const int p = base - l0 - ZK, sw = (p >> 4) & 7;
                T nw[ZK];
#pragma unroll
                for (int c = 0; c < ZK; ++c) nw[c] = row[(p + c) ^ sw];
#pragma unroll
                for (int s2 = 0; s2 < ZK; ++s2) {
                    const C g = gr[l0 + s2];
#pragma unroll
                    for (int c = 0; c < WZK; ++c) {
                        acc[c].x = fma(g.x, wv[c], acc[c].x);
                        acc[c].y = fma(g.y, wv[c], acc[c].y);
                    }
#pragma unroll
                    for (int c = WZK - 1; c > 0; --c) wv[c] = wv[c - 1];
                    wv[0] = nw[ZK - 1 - s2];
                }
            }
        }
        C* zr = zb + b * z_stride;
#pragma unroll
        for (int c = 0; c < WZK; ++c) {
            const int m = m_lo + lane * WZK + c;
            if (m < a.nout) {
                C v = acc[c];
                const int mf = m + a.trim;
                if (wraps && mf < a.mwrap) v = cadd(v, cw[mf - mf_lo]);
                zr[m] = cmul(v, sv[c]);
            }
        }
        __syncwarp();   // cw / window reuse by the next task
    }
}

size_t zoom_wfir_warp_bytes(const ZoomArgs& a, bool f32) {
    const size_t cs = f32 ? 8 : 16, rs = f32 ? 4 : 8;
    return ((size_t)(a.mwrap + 1) * cs + (size_t)a.D * zoom_wfir_rs(a) * rs + 15) / 16 * 16;
}
size_t zoom_wfir_head_bytes(const ZoomArgs& a, bool f32) {
    const size_t cs = f32 ? 8 : 16;
    return ((size_t)(a.D * a.lh + a.T) * cs + (size_t)a.D * 4 + 15) / 16 * 16;
}

template <typename T>
static cudaError_t zoom_wfir_impl(const ZoomArgs& a, const T* x, long long xs, long long batch, const void* g,
                                  const void* S, void* zb, long long z_stride, cudaStream_t st) {
    using C = cx_t<T>;
    const bool f32 = sizeof(T) == 4;
    const int wchunks = (a.nout + WF_OUT - 1) / WF_OUT;
    const size_t wbytes = zoom_wfir_warp_bytes(a, f32);
    const size_t smem = zoom_wfir_head_bytes(a, f32) + wbytes * WF_WARPS;
    auto kern = k_zoom_wfir<T>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long long tasks = batch * wchunks;
    kern<<<persistent_grid(kern, WF_WARPS * 32, smem, (tasks + WF_WARPS - 1) / WF_WARPS), WF_WARPS * 32, smem, st>>>(
        x, xs, batch, a, wchunks, zoom_wfir_rs(a), (int)wbytes, (const C*)g, (const C*)S, (C*)zb, z_stride);
    return cudaGetLastError();
}

bool zoom_wfir_fits(const ZoomArgs& a, bool f32, const void*, long long) {
    return zoom_wfir_head_bytes(a, f32) + zoom_wfir_warp_bytes(a, f32) * WF_WARPS <= (size_t)smem_optin();
}

cudaError_t launch_zoom_wfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch, const void* g,
                             const void* S, void* zb, long long z_stride, cudaStream_t st) {
    return f32 ? zoom_wfir_impl<float>(a, (const float*)x, xs, batch, g, S, zb, z_stride, st)
               : zoom_wfir_impl<double>(a, (const double*)x, xs, batch, g, S, zb, z_stride, st);
}

// FFT of each work row (first nout entries, zero padded to L) and the signed band gather
// x D x group-delay phase (zoomfft.cpp:204-234); several records per CTA for short transforms
template <typename T, int LOG2N, int NZ>
__global__ void __launch_bounds__(KCfg<T, LOG2N>::BLOCK, KCfg<T, LOG2N>::MINB)
k_zoom_fftband(const cx_t<T>* __restrict__ zb, long long z_stride, int nout, long long batch, int k_lo, int nbins,
               const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ band, cx_t<T>* __restrict__ out,
               long long out_stride) {
    SKG_PROLOGUE(T, LOG2N)
    const int nvalid = nout < G::L ? nout : G::L;
    for (long long base = (long long)blockIdx.x * K::GROUPS; base < batch; base += (long long)gridDim.x * K::GROUPS) {
        const long long b = base + gid;
        const bool active = b < batch;
        const C* src = zb + (active ? b : 0) * z_stride;
        C v[G::EPT];
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            const int pos = tid + G::NT * q;
            v[q] = (active && pos < nvalid) ? src[pos] : czero<C>();
        }
        block_fft<false, LOG2N, NZ>(v, sm, tws, tid);   // NZ: the block is zero padded to n_fft
        if constexpr (G::L >= 16) {
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) sm[pad16(tid + G::NT * q)] = v[q];
        } else {
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) sm[tid + G::NT * q] = v[q];
        }
        __syncthreads();
        if (active) {
            C* o = out + b * out_stride;
            for (int i = tid; i < nbins; i += G::NT) {
                const int k = k_lo + i;
                const int idx = ((k % G::L) + G::L) % G::L;
                o[i] = cmul(sm[G::L >= 16 ? pad16(idx) : idx], __ldg(band + i));
            }
        }
        __syncthreads();
    }
}

template <typename T, int LOG2N, int NZ>
static cudaError_t run_zoom_fftband(const void* zb, long long z_stride, int nout, long long batch, int k_lo,
                                    int nbins, const void* tw, const void* band, void* out, long long out_stride,
                                    cudaStream_t st) {
    using K = KCfg<T, LOG2N>;
    using C = cx_t<T>;
    // small transforms (L < 16) still need L entries of exchange space
    constexpr size_t smem = K::SMEM_BYTES > 0 ? K::SMEM_BYTES : (size_t)K::GROUPS * 16 * sizeof(C);
    auto kern = k_zoom_fftband<T, LOG2N, NZ>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<persistent_grid(kern, K::BLOCK, smem, grid_for(batch, K::GROUPS)), K::BLOCK, smem, st>>>(
        (const C*)zb, z_stride, nout, batch, k_lo, nbins, (const C*)tw, (const C*)band, (C*)out, out_stride);
    return cudaGetLastError();
}

cudaError_t launch_zoom_fftband(int log2n, bool f32, const void* zb, long long z_stride, int nout, long long batch,
                                int k_lo, int nbins, const void* tw, const void* band, void* out, long long out_stride,
                                cudaStream_t st) {
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        return dispatch_log2<0, max_log2<T>()>(log2n, [&](auto lg) {
            constexpr int LG = decltype(lg)::value;
            const int nz = nz_class(nout < (1 << LG) ? nout : (1 << LG), FftGeom<LG>::NT);
            return dispatch_nz<LG>(nz, [&](auto z) {
                constexpr int NZ = decltype(z)::value;
                return run_zoom_fftband<T, LG, NZ>(zb, z_stride, nout, batch, k_lo, nbins, tw, band, out, out_stride,
                                                   st);
            });
        });
    };
    return f32 ? go(float{}) : go(double{});
}

}  // namespace skg

// ---- phase-lane FIR (default for power-of-two D <= 16 and short phase rows) -----------------------
// Lanes are (group g, phase ph) with D phase-lanes per group. A lane convolves ITS phase row
// x[r D + ph] with that row's taps, which it keeps in registers (loaded once per kernel), over a
// sliding register window: each output costs one sample load and LH complex-by-real MACs — no
// shared-memory staging, no polyphase scatter. The D phase partials of a mini-batch of MB outputs
// are then summed by a transpose-reduce across the phase-lanes (log2 D xor-shuffle levels, each
// halving the outputs a lane carries), which leaves every lane with MB / D finished outputs.
namespace skg {

template <typename T, int D, int LH>
__global__ void __launch_bounds__(128, sizeof(T) == 8 ? SKG_PFIR_MINB64(D, LH) : SKG_PFIR_MINB32)
k_zoom_pfir(const T* __restrict__ x, long long x_stride, long long batch, ZoomArgs a, int gchunk, int tasks_per_rec,
            const cx_t<T>* __restrict__ gph, const cx_t<T>* __restrict__ gnat, const cx_t<T>* __restrict__ S,
            cx_t<T>* __restrict__ zb, long long z_stride) {
    using C = cx_t<T>;
    constexpr int G = 32 / D;
    constexpr int MB = D > 8 ? D : 8;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int warp = threadIdx.x >> 5, ph = (threadIdx.x & 31) % D;
    // per warp: [wrap terms (mwrap + 1)][phase partials G x MB x (D + 1) (padded: conflict-free reads)]
    C* cw = reinterpret_cast<C*>(smraw) + warp * (a.mwrap + 1 + G * MB * (D + 1));
    C* red = cw + (a.mwrap + 1);
    // this phase row's taps (rows are zero padded to a.lh >= LH entries... or shorter: guard)
    C tp[LH];
#pragma unroll
    for (int l = 0; l < LH; ++l) tp[l] = l < a.lh ? __ldg(gph + ph * a.lh + l) : czero<C>();
    const long long ntasks = batch * tasks_per_rec;
    const long long tstride = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long task = (long long)blockIdx.x * (blockDim.x >> 5) + warp; task < ntasks; task += tstride)
        pfir_task<T, D, LH>(x, x_stride, a, gchunk, tasks_per_rec, task, ntasks, tstride, tp, gnat, S, cw, red,
                            [&](long long b, int m, C v) { zb[b * z_stride + m] = v; });
}

// LH instantiated for these phase-row lengths (a row's taps are zero padded up to the next one)
constexpr int kPfirLH[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 16};

template <typename T, int D, int LH>
static cudaError_t run_pfir(const ZoomArgs& a, const T* x, long long xs, long long batch, const void* gph,
                            const void* gnat, const void* S, void* zb, long long z_stride, cudaStream_t st) {
    using C = cx_t<T>;
    constexpr int G = 32 / D;
    constexpr int MB = D > 8 ? D : 8;
    // a group's outputs per task: whole mini-batches, about 64 outputs
    const int gchunk = std::max(MB, (std::min(64, (a.nout + G - 1) / G) + MB - 1) / MB * MB);
    const int tasks_per_rec = (a.nout + G * gchunk - 1) / (G * gchunk);
    const size_t smem = (size_t)4 * (a.mwrap + 1 + G * MB * (D + 1)) * sizeof(C);
    auto kern = k_zoom_pfir<T, D, LH>;
    cudaError_t e = prep_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long long tasks = batch * tasks_per_rec;
    kern<<<persistent_grid(kern, 128, smem, (tasks + 3) / 4), 128, smem, st>>>(
        x, xs, batch, a, gchunk, tasks_per_rec, (const C*)gph, (const C*)gnat, (const C*)S, (C*)zb, z_stride);
    return cudaGetLastError();
}

template <typename T, int D>
static cudaError_t pfir_lh(int lh, const ZoomArgs& a, const T* x, long long xs, long long batch, const void* gph,
                           const void* gnat, const void* S, void* zb, long long z_stride, cudaStream_t st) {
    switch (lh) {
        case 1: return run_pfir<T, D, 1>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 2: return run_pfir<T, D, 2>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 3: return run_pfir<T, D, 3>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 4: return run_pfir<T, D, 4>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 5: return run_pfir<T, D, 5>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 6: return run_pfir<T, D, 6>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 7: return run_pfir<T, D, 7>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 8: return run_pfir<T, D, 8>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 9: return run_pfir<T, D, 9>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 10: return run_pfir<T, D, 10>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 12: return run_pfir<T, D, 12>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        case 16: return run_pfir<T, D, 16>(a, x, xs, batch, gph, gnat, S, zb, z_stride, st);
        default: return cudaErrorInvalidValue;
    }
}

// the instantiated LH for a plan (0: none, use the window kernel)
int zoom_pfir_lh(const ZoomArgs& a) {
    const int D = a.D;
    if (D < 1 || D > 16 || (D & (D - 1))) return 0;
    const int need = (a.T + D - 1) / D;   // longest phase row
    if (D == 1) return need == 1 ? 1 : 0;
    static const bool no_odd = std::getenv("SKG_PFIR_NO_ODD") != nullptr;   // A/B: pad rows to the even sizes
    for (int v : kPfirLH)
        if (v >= need && v > 1 && !(no_odd && (v == 7 || v == 9))) return v;
    return 0;
}

cudaError_t launch_zoom_pfir(const ZoomArgs& a, bool f32, const void* x, long long xs, long long batch,
                             const void* gph, const void* gnat, const void* S, void* zb, long long z_stride,
                             cudaStream_t st) {
    const int lh = zoom_pfir_lh(a);
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        const T* xt = static_cast<const T*>(x);
        switch (a.D) {
            case 1: return pfir_lh<T, 1>(lh, a, xt, xs, batch, gph, gnat, S, zb, z_stride, st);
            case 2: return pfir_lh<T, 2>(lh, a, xt, xs, batch, gph, gnat, S, zb, z_stride, st);
            case 4: return pfir_lh<T, 4>(lh, a, xt, xs, batch, gph, gnat, S, zb, z_stride, st);
            case 8: return pfir_lh<T, 8>(lh, a, xt, xs, batch, gph, gnat, S, zb, z_stride, st);
            case 16: return pfir_lh<T, 16>(lh, a, xt, xs, batch, gph, gnat, S, zb, z_stride, st);
            default: return cudaErrorInvalidValue;
        }
    };
    return f32 ? go(float{}) : go(double{});
}

}  // namespace skg
