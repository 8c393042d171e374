// Microbenchmark: sustained DFMA / FFMA issue rate per SM (independent chains, full occupancy).
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void k_fma(T* out, int iters, T a, T b) {
    T acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = (T)(threadIdx.x + c);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
    }
    T s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == (T)12345.678) out[threadIdx.x] = s;
}

template <typename T, int CH> void run(const char* name, int blocks_per_sm, int threads) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    T* out;
    cudaMalloc(&out, 4096 * sizeof(T));
    const int iters = 4096;
    k_fma<T, CH><<<sms * blocks_per_sm, threads>>>(out, 16, (T)0.999, (T)0.001);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_fma<T, CH><<<sms * blocks_per_sm, threads>>>(out, iters, (T)0.999, (T)0.001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double fmas = (double)sms * blocks_per_sm * threads * iters * CH;
    const double tflops = 2 * fmas / (ms * 1e-3) / 1e12;
    const double lanes_per_clk_sm = fmas / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%s chains=%d warps/SM=%d: %.3f ms  %.2f TFLOP/s  %.1f lane-FMA/clk/SM (at %d MHz nominal)\n", name, CH,
           blocks_per_sm * threads / 32, ms, tflops, lanes_per_clk_sm, clk / 1000);
    cudaFree(out);
}

int main() {
    run<double, 8>("DFMA", 4, 256);
    run<double, 16>("DFMA", 4, 256);
    run<double, 8>("DFMA", 1, 256);
    run<double, 8>("DFMA", 2, 128);
    run<double, 16>("DFMA", 1, 128);
    run<float, 8>("FFMA", 4, 256);
    run<float, 16>("FFMA", 4, 256);
    return 0;
}
