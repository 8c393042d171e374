// kernels_band.cu — band slice + magnitude_db over batched complex spectra already in HBM
// (slice_band, spectra.cpp:40-61; magnitude_db, types.cpp:13-18). Used on the outputs of the
// CZT, zoom and multi-pass FFT routes; the single-CTA zero-padded FFT fuses the same epilogue into
// its store (k_fft_r2c MODE 3). One pass over the band: read nb complex, write nb complex and/or
// nb reals per row — HBM bound, grid-stride over (row, bin) with coalesced rows.
#include <cuda_runtime.h>

#include "fft_device.cuh"
#include "kernels.hpp"

namespace skg {

template <typename T>
__global__ void k_band_db(const cx_t<T>* __restrict__ in, long long in_stride, long long klo, long long nb,
                          long long batch, cx_t<T>* __restrict__ out, long long out_stride, T* __restrict__ db,
                          long long db_stride) {
    const long long total = nb * batch;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long b = i / nb, k = i - b * nb;
        const cx_t<T> v = __ldg(in + b * in_stride + klo + k);
        if (out) out[b * out_stride + k] = v;
        if (db) db[b * db_stride + k] = magnitude_db_t(v.x, v.y);
    }
}

cudaError_t launch_band_db(bool f32, const void* in, long long in_stride, long long klo, long long nb,
                           long long batch, void* out, long long out_stride, void* db, long long db_stride,
                           cudaStream_t st) {
    if (nb <= 0 || batch <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long total = nb * batch;
    const long long want = (total + 255) / 256;
    const unsigned grid = (unsigned)(want < (long long)sms * 8 ? want : (long long)sms * 8);
    if (f32)
        k_band_db<float><<<grid, 256, 0, st>>>((const float2*)in, in_stride, klo, nb, batch, (float2*)out, out_stride,
                                               (float*)db, db_stride);
    else
        k_band_db<double><<<grid, 256, 0, st>>>((const double2*)in, in_stride, klo, nb, batch, (double2*)out,
                                                out_stride, (double*)db, db_stride);
    return cudaGetLastError();
}

}  // namespace skg
