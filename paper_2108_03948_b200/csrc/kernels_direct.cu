// kernels_direct.cu — the reference's O(n^2) / O(n m) "direct" routes on the GPU:
// dft_naive (numerics.cpp:35-50, exact (k*m) mod n twiddle index) and czt_direct
// (czt.cpp:58-75, every power through the fma-split phase reduction of cis_cycles).
// They are part of the reference's public C ABI (sk_dft_naive, sk_czt_direct); here each output
// bin is one warp-strided dot product.
#include <cuda_runtime.h>

#include "fft_device.cuh"

namespace skg {

__device__ __forceinline__ double2 d_cis_cycles(double q, double t) {   // numerics.cpp:122-128
    const double hi = q * t;
    const double lo = fma(q, t, -hi);
    const double frac = (hi - rint(hi)) + lo;
    double s, c;
    sincospi(2.0 * frac, &s, &c);
    return make_double2(c, s);
}

__device__ __forceinline__ double2 d_polar_pow(double log_mag, double q, double t) {   // czt.cpp:27-31
    double2 u = d_cis_cycles(q, t);
    if (log_mag != 0.0) {
        const double s = exp(log_mag * t);
        u.x *= s;
        u.y *= s;
    }
    return u;
}

// one warp per output bin; lanes stride the input, shuffle-reduce at the end
__global__ void k_dft_naive(const double2* __restrict__ x, long long n, const double2* __restrict__ tw,
                            double2* __restrict__ out) {
    const long long k = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (k >= n) return;
    double2 acc = make_double2(0.0, 0.0);
    for (long long m = lane; m < n; m += 32) {
        const long long idx = (k * m) % n;
        acc = cadd(acc, cmul(__ldg(x + m), __ldg(tw + idx)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) out[k] = acc;
}

__global__ void k_czt_premul(const double2* __restrict__ x, long long n, double a_logm, double a_q,
                             double2* __restrict__ xa) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) xa[i] = cmul(x[i], d_polar_pow(a_logm, a_q, -(double)i));
}

__global__ void k_czt_direct(const double2* __restrict__ xa, long long n, long long m, double w_logm, double w_q,
                             double2* __restrict__ out) {
    const long long k = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (k >= m) return;
    double2 acc = make_double2(0.0, 0.0);
    for (long long i = lane; i < n; i += 32)
        acc = cadd(acc, cmul(__ldg(xa + i), d_polar_pow(w_logm, w_q, (double)k * (double)i)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) out[k] = acc;
}

cudaError_t launch_dft_naive(const void* x, long long n, const void* tw, void* out, cudaStream_t st) {
    const long long threads = n * 32;
    k_dft_naive<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>((const double2*)x, n, (const double2*)tw,
                                                                   (double2*)out);
    return cudaGetLastError();
}

cudaError_t launch_czt_direct(const void* x, long long n, double a_logm, double a_q, double w_logm, double w_q,
                              long long m, void* xa_scratch, void* out, cudaStream_t st) {
    k_czt_premul<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((const double2*)x, n, a_logm, a_q, (double2*)xa_scratch);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const long long threads = m * 32;
    k_czt_direct<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>((const double2*)xa_scratch, n, m, w_logm, w_q,
                                                                     (double2*)out);
    return cudaGetLastError();
}

}  // namespace skg

// ---- zoom helper stages exposed by the reference's C++ API (zoomfft.hpp:63-75) --------------
namespace skg {

__global__ void k_freq_shift(const double* __restrict__ xr, const double2* __restrict__ xc, long long n, double q,
                             double2* __restrict__ y) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double2 c = d_cis_cycles(q, (double)i);   // zoomfft.cpp:44-64 per-sample phase
    y[i] = xr ? make_double2(xr[i] * c.x, xr[i] * c.y) : cmul(xc[i], c);
}

__global__ void k_filter_decimate(const double2* __restrict__ x, long long n, const double* __restrict__ taps, int T,
                                  int d, int circular, double2* __restrict__ out, long long nout) {
    const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (m >= nout) return;
    const long long base = m * d;
    double2 acc = make_double2(0.0, 0.0);
    const long long t_end = circular ? T : (T < base + 1 ? T : base + 1);
    for (long long t = 0; t < t_end; ++t) {   // zoomfft.cpp:66-104
        const long long j = base >= t ? base - t : base + n - t;
        const double h = __ldg(taps + t);
        const double2 v = __ldg(x + j);
        acc.x += h * v.x;
        acc.y += h * v.y;
    }
    out[m] = acc;
}

cudaError_t launch_freq_shift(const double* xr, const void* xc, long long n, double q, void* y, cudaStream_t st) {
    k_freq_shift<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(xr, (const double2*)xc, n, q, (double2*)y);
    return cudaGetLastError();
}

cudaError_t launch_filter_decimate(const void* x, long long n, const double* taps, int T, int d, int circular,
                                   void* out, long long nout, cudaStream_t st) {
    k_filter_decimate<<<(unsigned)((nout + 127) / 128), 128, 0, st>>>((const double2*)x, n, taps, T, d, circular,
                                                                      (double2*)out, nout);
    return cudaGetLastError();
}

}  // namespace skg
