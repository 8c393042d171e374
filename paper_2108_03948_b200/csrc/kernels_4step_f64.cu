// Instantiation of the four-step (multi-pass) kernels for double (see kernels_4step.cuh).
#include "kernels_4step_real.cuh"

namespace skg {

template <>
cudaError_t launch_4step_col<double>(int log2R, bool inverse, int in_kind, int conj_in, const void* x,
                                  long long x_stride, long long N, const void* cin, void* Y, int log2C,
                                  long long batch, const void* tw, const void* twL, int out_kind, void* out,
                                  long long out_stride, long long M, const void* cout, double scale, int conj_out,
                                  cudaStream_t st) {
    return launch_4step_col_impl<double>(log2R, inverse, in_kind, conj_in, x, x_stride, N, cin, Y, log2C, batch, tw,
                                      twL, out_kind, out, out_stride, M, cout, scale, conj_out, st);
}

template <>
cudaError_t launch_4step_row<double>(int log2C, int mode, void* Y, int log2R, long long batch, const void* tw,
                                  const void* twL, const void* khat_p, void* out, long long out_stride,
                                  double scale, int conj_out, cudaStream_t st) {
    return launch_4step_row_impl<double>(log2C, mode, Y, log2R, batch, tw, twL, khat_p, out, out_stride, scale,
                                      conj_out, st);
}

template <>
cudaError_t launch_4step_colr<double>(int log2R, const void* x, long long x_stride, long long N, void* Y, int log2C,
                                   long long batch, const void* tw, const void* twL, cudaStream_t st) {
    return launch_4step_colr_impl<double>(log2R, x, x_stride, N, Y, log2C, batch, tw, twL, st);
}

template <>
cudaError_t launch_4step_rowh<double>(int log2C, const void* Y, int log2R, long long batch, const void* tw, void* out,
                                   long long out_stride, int half, cudaStream_t st) {
    return launch_4step_rowh_impl<double>(log2C, Y, log2R, batch, tw, out, out_stride, half, st);
}

template <>
cudaError_t launch_4step_rfused<double>(int lg, const void* x, long long x_stride, long long N, void* Yring, int slots,
                                     int delta, long long batch, const void* tw, const void* twL, void* out,
                                     long long out_stride, int half, unsigned* col_done, unsigned* row_done,
                                     int* grid_out, int* ups_out, cudaStream_t st) {
    return launch_4step_rfused_impl<double>(lg, x, x_stride, N, Yring, slots, delta, batch, tw, twL, out, out_stride, half,
                                         col_done, row_done, grid_out, ups_out, st);
}

}  // namespace skg
