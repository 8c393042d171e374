// kernels_zoom_spec.cu — the Zoom FFT's circular FIR + decimation + short FFT evaluated in the
// frequency domain (zoom_fft, zoomfft.cpp:183-239, circular mode, n_fft = U / D):
//   the reference forms y[n] = x[n] e^{-i 2pi fc n / fs}, u[m] = sum_t h[t] y[(m D - t) mod U] and
//   Z = DFT_{U/D}(u). With c = y (*) h (circular, length U) and C = DFT_U(c) = Y . H,
//   Z[k] = (1/D) sum_{r<D} C[k + r U/D]   (decimation in time = aliasing in frequency),
// which is the same sum, not an approximation. Per trace: ONE U-point transform of the shifted trace
// (shift on load), the filter's spectrum H (plan table) on the registers, and for each band bin the
// D-term alias sum x D x group-delay phase (the plan's band table) / D on the store. The FIR's
// T complex-by-real MACs per output become ~log2(U) butterflies per sample, on the FFT engine.
#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"

namespace skg {

template <typename T, int LOG2U>
__global__ void __launch_bounds__(KCfg<T, LOG2U>::BLOCK, KCfg<T, LOG2U>::MINB)
k_zoom_spec(const T* __restrict__ x, long long x_stride, long long batch, const cx_t<T>* __restrict__ tw,
            const cx_t<T>* __restrict__ shift, const cx_t<T>* __restrict__ hf, int nf, int D, int k_lo, int nbins,
            const cx_t<T>* __restrict__ band, T inv_d, cx_t<T>* __restrict__ out, long long out_stride) {
    SKG_PROLOGUE(T, LOG2U)
    for (long long base = (long long)blockIdx.x * K::GROUPS; base < batch; base += (long long)gridDim.x * K::GROUPS) {
        const long long b = base + gid;
        const bool active = b < batch;
        {   // the group's next trace into L2 while this one is transformed
            const long long bn = b + (long long)gridDim.x * K::GROUPS;
            if (bn < batch) {
                constexpr int per_line = 128 / (int)sizeof(T);
                for (int i = tid * per_line; i < G::L; i += G::NT * per_line) prefetch_l2(x + bn * x_stride + i);
            }
        }
        C v[G::EPT];
        const T* xr = x + (active ? b : 0) * x_stride;
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) {
            const int pos = tid + G::NT * q;
            v[q] = active ? rmul(__ldg(xr + pos), __ldg(shift + pos)) : czero<C>();   // y = x e^{-i w n}
        }
        block_fft<false, LOG2U>(v, sm, tws, tid);
#pragma unroll
        for (int q = 0; q < G::EPT; ++q) sm[pad16(tid + G::NT * q)] = cmul(v[q], __ldg(hf + tid + G::NT * q));
        __syncthreads();
        if (active) {
            C* o = out + b * out_stride;
            for (int j = tid; j < nbins; j += G::NT) {
                const int k = k_lo + j;
                const int idx = ((k % nf) + nf) % nf;
                C acc = czero<C>();
                for (int r = 0; r < D; ++r) acc = cadd(acc, sm[pad16(idx + r * nf)]);
                o[j] = cscale(cmul(acc, __ldg(band + j)), inv_d);
            }
        }
        __syncthreads();
    }
}

namespace {
template <typename T, int LG>
cudaError_t run_spec(const T* x, long long xs, long long batch, const void* tw, const void* shift, const void* hf,
                     int nf, int D, int k_lo, int nbins, const void* band, void* out, long long os, cudaStream_t st) {
    using K = KCfg<T, LG>;
    using C = cx_t<T>;
    auto kern = k_zoom_spec<T, LG>;
    cudaError_t e = prep_smem(kern, K::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<persistent_grid(kern, K::BLOCK, K::SMEM_BYTES, grid_for(batch, K::GROUPS)), K::BLOCK, K::SMEM_BYTES, st>>>(
        x, xs, batch, (const C*)tw, (const C*)shift, (const C*)hf, nf, D, k_lo, nbins, (const C*)band,
        (T)(1.0 / (double)D), (C*)out, os);
    return cudaGetLastError();
}
}  // namespace

// U = 2^log2u in 2^8 .. the single-CTA maximum
cudaError_t launch_zoom_spec(int log2u, bool f32, const void* x, long long xs, long long batch, const void* tw,
                             const void* shift, const void* hf, int nf, int D, int k_lo, int nbins, const void* band,
                             void* out, long long os, cudaStream_t st) {
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        return dispatch_log2<8, max_log2<T>()>(log2u, [&](auto lg) {
            constexpr int LG = decltype(lg)::value;
            return run_spec<T, LG>(static_cast<const T*>(x), xs, batch, tw, shift, hf, nf, D, k_lo, nbins, band, out,
                                   os, st);
        });
    };
    return f32 ? go(float{}) : go(double{});
}

}  // namespace skg
