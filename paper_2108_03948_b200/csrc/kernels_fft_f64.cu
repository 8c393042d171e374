// Instantiation of the batched FFT / real-input FFT kernels for double (see kernels_impl.cuh).
#include "kernels_impl.cuh"

namespace skg {

template <>
cudaError_t launch_fft_c2c<double>(int log2L, bool inverse, const void* in, long long in_stride, void* out,
                                long long out_stride, long long batch, const void* tw, double scale,
                                cudaStream_t st) {
    return launch_fft_c2c_impl<double>(log2L, inverse, in, in_stride, out, out_stride, batch, tw, scale, st);
}

template <>
cudaError_t launch_fft_r2c<double>(int log2M, long long N, const double* x, long long x_stride, long long batch,
                                const void* tw, const void* post, int mode, void* out, long long out_stride,
                                const void* rtab, double* mag, double* phase, long long mp_stride, long long klo, long long khi,
                                cudaStream_t st) {
    return launch_fft_r2c_impl<double>(log2M, N, x, x_stride, batch, tw, post, mode, out, out_stride, rtab, mag,
                                    phase, mp_stride, klo, khi, st);
}

}  // namespace skg
