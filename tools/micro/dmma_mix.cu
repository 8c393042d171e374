// Microbenchmark: does the FP64 tensor path (mma.sync m8n8k4 f64, DMMA) run beside the DFMA pipe?
// Three kernels at full occupancy: DFMA chains only, DMMA chains only, and both interleaved in every
// warp. If the mixed kernel's DFMA + DMMA flop rate exceeds either alone, the two pipes are separate.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int MODE, int CH>
__global__ void k_mix(double* out, int iters, double a, double b) {
    double acc[CH];
    double m[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        acc[c] = threadIdx.x + c;
        m[c][0] = c;
        m[c][1] = threadIdx.x;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (MODE != 1) acc[c] = fma(acc[c], a, b);
            if (MODE != 0) dmma(m[c], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c] + m[c][0] + m[c][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int MODE, int CH> void run(const char* name, int bps, int threads) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 4096 * sizeof(double));
    const int iters = 2048;
    k_mix<MODE, CH><<<sms * bps, threads>>>(out, 16, 0.999, 0.001);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_mix<MODE, CH><<<sms * bps, threads>>>(out, iters, 0.999, 0.001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)sms * bps * threads / 32;
    // DFMA: 32 lanes x 2 flop; DMMA m8n8k4: 8*8*4*2 = 512 flop per warp instruction
    const double f_fma = MODE != 1 ? warps * iters * CH * 32 * 2 : 0;
    const double f_mma = MODE != 0 ? warps * iters * CH * 512 : 0;
    printf("%-10s CH=%d warps/SM=%2d: %.3f ms  DFMA %.2f TF/s  DMMA %.2f TF/s  total %.2f TF/s\n", name, CH,
           bps * threads / 32, ms, f_fma / ms / 1e9, f_mma / ms / 1e9, (f_fma + f_mma) / ms / 1e9);
    cudaFree(out);
}

int main() {
    run<0, 8>("dfma", 4, 256);
    run<1, 4>("dmma", 4, 256);
    run<1, 8>("dmma", 4, 256);
    run<2, 4>("mixed", 4, 256);
    run<2, 8>("mixed", 4, 256);
    run<0, 8>("dfma", 2, 256);
    run<1, 8>("dmma", 2, 256);
    run<2, 8>("mixed", 2, 256);
    return 0;
}
