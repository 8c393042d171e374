// Microbenchmark: tensor memory (TMEM) as per-thread scratch — tcgen05.ld / tcgen05.st throughput with
// the 32x32b shape (each thread its own lane) from 16 warps per SM, against LDS.128 / STS.128.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define TM_LD16(r, addr)                                                                                        \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),       \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
                 : "r"(addr))
#define TM_ST16(addr, r)                                                                                        \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
                 ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),    \
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]))

// MODE 0: TMEM ld only, 1: TMEM st only, 2: LDS.128 only, 3: TMEM ld + LDS together
template <int MODE>
__global__ void __launch_bounds__(512, 1) k_tm(uint32_t* out, int iters) {
    __shared__ uint32_t taddr_s;
    __shared__ __align__(16) uint4 sm[512 * 4];
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 512 * 4; i += blockDim.x) sm[i] = make_uint4(i, i, i, i);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr_s;
    // warp w: lanes 32*(w%4).., columns 128*(w/4)..
    const uint32_t my = base + ((uint32_t)(32 * (warp % 4)) << 16) + 128 * (warp / 4);
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 16 + i;
    TM_ST16(my, r);
    asm volatile("tcgen05.wait::st.sync.aligned;");
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (MODE == 0 || MODE == 3) {
                TM_LD16(r, my + 16 * c);
                asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
                for (int i = 0; i < 16; ++i) acc ^= r[i];
            }
            if (MODE == 4 && (c & 1) == 0) {   // two loads in flight per wait
                uint32_t r2[16];
                TM_LD16(r, my + 16 * c);
                TM_LD16(r2, my + 16 * c + 16);
                asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
                for (int i = 0; i < 16; ++i) acc ^= r[i] ^ r2[i];
            }
            if (MODE == 1) {
                r[0] += it;
                TM_ST16(my + 16 * c, r);
            }
            if (MODE == 2 || MODE == 3) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    uint4 v = sm[(threadIdx.x + 512 * i + it * 7 + c) & 2047];
                    acc ^= v.x ^ v.y ^ v.z ^ v.w;
                }
            }
        }
    }
    if (MODE == 1) asm volatile("tcgen05.wait::st.sync.aligned;");
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

template <int MODE> void run(const char* name) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, (size_t)sms * 512 * 4);
    const int iters = 4096;
    k_tm<MODE><<<sms, 512>>>(out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_tm<MODE><<<sms, 512>>>(out, iters);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // bytes moved per SM: 512 threads x iters x 8 chunks x 64 B (TMEM) or x 64 B (4 x LDS.128)
    const double bytes = 512.0 * iters * 8 * 64;
    const double clk = 1.965e9;
    printf("%-14s %s: %.3f ms  %.1f B/clk/SM per stream (at 1965 MHz)\n", name, cudaGetErrorString(err), ms,
           bytes / (ms * 1e-3) / clk);
    cudaFree(out);
}

int main() {
    run<0>("tmem ld x16");
    run<1>("tmem st x16");
    run<2>("lds.128");
    run<3>("tmem ld + lds");
    run<4>("tmem ld 2x16");
    return 0;
}
