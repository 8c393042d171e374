// Instantiation of the one-launch multi-pass CZT for double (see kernels_4step_czt.cuh).
#include "kernels_4step_czt.cuh"

namespace skg {

template <>
cudaError_t launch_4step_czt_fused<double>(int lR, int lC, const void* x, int complex_in, long long x_stride, long long N,
                                        const void* cin, void* Yring, int slots, int delta, long long batch,
                                        const void* twR, const void* twC, const void* twL, const void* khat_p,
                                        void* out, long long out_stride, long long M, const void* cout,
                                        unsigned* counters, int* grid_out, int* ups_out, cudaStream_t st) {
    return launch_4step_czt_fused_impl<double>(lR, lC, x, complex_in, x_stride, N, cin, Yring, slots, delta, batch, twR, twC,
                                            twL, khat_p, out, out_stride, M, cout, counters, grid_out, ups_out, st);
}

}  // namespace skg
