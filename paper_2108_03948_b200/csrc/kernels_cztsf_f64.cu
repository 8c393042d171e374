// Instantiation of the shared-forward segmented CZT kernels for double (see kernels_impl.cuh); a
// separate translation unit so the CZT kernel families compile in parallel.
#include "kernels_impl.cuh"

namespace skg {

template <>
cudaError_t launch_czt_sf<double>(int log2L, long long N, long long M, bool complex_in, const void* x, long long x_stride,
                              long long batch, int nseg, long long seg_len, void* out, long long out_stride,
                              const void* tw, const void* cin, const void* khat, const void* cout, void* ywork,
                              long long ywork_slots, const void* twl, cudaStream_t st) {
    return launch_czt_sf_impl<double>(log2L, N, M, complex_in, x, x_stride, batch, nseg, seg_len, out, out_stride, tw, cin,
                                   khat, cout, ywork, ywork_slots, twl, st);
}

}  // namespace skg
