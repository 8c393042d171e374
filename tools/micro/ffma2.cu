// Microbenchmark: packed fp32 (FFMA2, fma.rn.f32x2, sm_100a) against scalar FFMA — flops per clock
// per SM at full occupancy, independent chains. Decides whether the fp32 transforms (issue bound on
// the cube) should carry complex arithmetic as float2 pairs.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(float a, float b) {
    return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}

template <int MODE, int CH>
__global__ void k(float* out, int iters, float a, float b) {
    float acc[2 * CH];
    unsigned long long p[CH];
#pragma unroll
    for (int c = 0; c < 2 * CH; ++c) acc[c] = threadIdx.x + c;
#pragma unroll
    for (int c = 0; c < CH; ++c) p[c] = f2(acc[2 * c], acc[2 * c + 1]);
    const unsigned long long A = f2(a, a), B = f2(b, b);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (MODE == 0) {
                acc[2 * c] = fmaf(acc[2 * c], a, b);
                acc[2 * c + 1] = fmaf(acc[2 * c + 1], a, b);
            } else {
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(A), "l"(B));
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[2 * c] + acc[2 * c + 1] + __uint_as_float((unsigned)p[c]) + __uint_as_float((unsigned)(p[c] >> 32));
    if (s == 12345.678f) out[threadIdx.x] = s;
}

template <int MODE, int CH> void run(const char* name) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4096 * 4);
    const int iters = 8192;
    k<MODE, CH><<<sms * 4, 256>>>(out, 16, 0.999f, 0.001f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE, CH><<<sms * 4, 256>>>(out, iters, 0.999f, 0.001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 2 * CH * (double)iters * sms * 4 * 256;   // 2 flops x 2 values x CH chains
    printf("%-6s CH=%d: %.3f ms  %.1f TF/s  %.0f flop/clk/SM (1965 MHz)\n", name, CH, ms, fl / ms / 1e9,
           fl / (ms * 1e-3) / sms / 1.965e9);
    cudaFree(out);
}

int main() {
    run<0, 4>("ffma");
    run<1, 4>("ffma2");
    run<0, 8>("ffma");
    run<1, 8>("ffma2");
    return 0;
}
