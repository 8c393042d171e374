// Instantiation of the fused Bluestein CZT kernels for float (see kernels_impl.cuh).
#include "kernels_impl.cuh"

namespace skg {

template <>
cudaError_t launch_czt<float>(int log2L, long long N, long long M, bool complex_in, const void* x,
                            long long x_stride, long long batch, int nseg, long long seg_len, long long cin_stride, void* out,
                            long long out_stride, const void* tw, const void* cin, const void* khat,
                            const void* cout, cudaStream_t st) {
    return launch_czt_impl<float>(log2L, N, M, complex_in, x, x_stride, batch, nseg, seg_len, cin_stride, out, out_stride, tw,
                                cin, khat, cout, st);
}

}  // namespace skg
