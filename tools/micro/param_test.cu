// Does a large by-value kernel parameter block (with/without __grid_constant__) launch on this box?
#include <cstdio>
#include <cuda_runtime.h>
template <int N> struct P { double2 g[N]; };
template <int N> __global__ void k_plain(const P<N> p, double* out) { out[threadIdx.x] = p.g[threadIdx.x % N].x; }
template <int N> __global__ void k_gc(const __grid_constant__ P<N> p, double* out) { out[threadIdx.x] = p.g[threadIdx.x % N].y; }
template <int N> void run() {
    P<N> p;
    for (int i = 0; i < N; ++i) p.g[i] = make_double2(i, -i);
    double* d;
    cudaMalloc(&d, 1024 * 8);
    k_plain<N><<<1, 128>>>(p, d);
    cudaError_t e1 = cudaDeviceSynchronize();
    printf("N=%d (%zu B) plain: %s\n", N, sizeof(P<N>), cudaGetErrorString(e1));
    fflush(stdout);
    k_gc<N><<<1, 128>>>(p, d);
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("N=%d (%zu B) grid_constant: %s\n", N, sizeof(P<N>), cudaGetErrorString(e2));
    fflush(stdout);
    cudaFree(d);
}
int main() {
    run<8>();
    run<72>();
    run<200>();
    run<1000>();
    return 0;
}
