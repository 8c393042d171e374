// Microbenchmark: DFMA throughput when all three operands are registers (FIR-like: tap x sample + acc),
// versus one register operand. Prints lane-FMA per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, int MODE>
__global__ void k(double* out, int iters, const double* in) {
    double acc[CH], xs[CH], ts[4];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        acc[c] = threadIdx.x + c;
        xs[c] = in[(threadIdx.x + c) & 255];
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) ts[t] = in[(threadIdx.x * 3 + t) & 255];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (MODE == 0) acc[c] = fma(acc[c], 0.999, 0.001);          // 1 register operand
                else if (MODE == 1) acc[c] = fma(ts[t], xs[c], acc[c]);    // tap reg x sample reg + acc
                else acc[c] = fma(ts[t], xs[(c + t) % CH], acc[c]);        // sliding-window pattern
            }
        }
#pragma unroll
        for (int c = 0; c < CH; ++c) xs[c] = xs[c] * 0.5 + 0.25;   // keep samples live / changing
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH, int MODE> void run(int blocks_per_sm, int threads) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *out, *in;
    cudaMalloc(&out, 4096 * 8);
    cudaMalloc(&in, 4096 * 8);
    cudaMemset(in, 0, 4096 * 8);
    const int iters = 1024;
    k<CH, MODE><<<sms * blocks_per_sm, threads>>>(out, 4, in);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<CH, MODE><<<sms * blocks_per_sm, threads>>>(out, iters, in);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)sms * blocks_per_sm * threads * iters * CH * 4;
    printf("mode %d chains %2d warps/SM %2d: %.2f TFLOP/s  %.1f lane-DFMA/clk/SM\n", MODE, CH,
           blocks_per_sm * threads / 32, 2 * fmas / (ms * 1e-3) / 1e12, fmas / (ms * 1e-3) / sms / (clk * 1e3));
}

int main() {
    run<8, 0>(4, 128);
    run<8, 1>(4, 128);
    run<8, 2>(4, 128);
    run<16, 1>(4, 128);
    run<16, 2>(4, 128);
    run<8, 1>(2, 128);
    run<16, 2>(2, 128);
    return 0;
}
