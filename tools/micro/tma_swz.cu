// Check the shared-memory layout of a 2-D TMA tensor load with a 16-byte inner box and
// CU_TENSOR_MAP_SWIZZLE_128B: hypothesis = row r of the box lands in 16-byte unit r ^ ((r >> 3) & 7)
// (address bits [4:6] ^= bits [7:9], box start 1024-byte aligned), rows packed densely.
// Also checks out-of-bounds rows (negative start coordinate) are zero-filled.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void k_dump(const __grid_constant__ CUtensorMap tm, double* out, int row0) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(dsm);
    const uint32_t pad = (1024 - (base & 1023)) & 1023;
    double* sm = reinterpret_cast<double*>(dsm + pad);
    uint64_t& bar = *reinterpret_cast<uint64_t*>(dsm + pad + 192 * 16);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(192 * 16));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(sm)),
            "l"(&tm), "r"(2), "r"(row0), "r"(1), "r"(sb)
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sb));
    for (int i = threadIdx.x; i < 384; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 3;   // 0 none, 1 32B, 2 64B, 3 128B
    const bool swz = mode == 3;
    const int D = 8, rows = 512, recs = 3;
    double* x;
    cudaMalloc(&x, sizeof(double) * D * rows * recs);
    double h[D * rows * recs];
    for (int i = 0; i < D * rows * recs; ++i) h[i] = i;   // value = flat index
    cudaMemcpy(x, h, sizeof(h), cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(fn);
    CUtensorMap tm;
    cuuint64_t gdim[3] = {(cuuint64_t)D, (cuuint64_t)rows, (cuuint64_t)recs};
    cuuint64_t gstr[2] = {D * 8, (cuuint64_t)D * rows * 8};
    cuuint32_t box[3] = {2, 192, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     (CUtensorMapSwizzle)mode, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    double* out;
    cudaMalloc(&out, 384 * sizeof(double));
    for (int row0 : {0, -64}) {
        k_dump<<<1, 128, 8192>>>(tm, out, row0);
        cudaError_t e = cudaDeviceSynchronize();
        double o[384];
        cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
        int bad = 0, zeros_ok = 1;
        for (int rr = 0; rr < 192; ++rr) {
            const int unit = mode == 3 ? (rr ^ ((rr >> 3) & 7)) : mode == 2 ? (rr ^ ((rr >> 3) & 3)) : mode == 1 ? (rr ^ ((rr >> 3) & 1)) : rr;
            const int grow = row0 + rr;
            for (int c = 0; c < 2; ++c) {
                const double want = grow < 0 ? 0.0 : (double)((1 * rows + grow) * D + 2 + c);
                if (o[unit * 2 + c] != want) {
                    if (bad < 5) printf("row0 %d: box row %d col %d: got %g want %g\n", row0, rr, c, o[unit * 2 + c], want);
                    ++bad;
                }
            }
        }
        printf("row0=%d err=%s mismatches=%d (hypothesis %s)\n", row0, cudaGetErrorString(e), bad, bad ? "WRONG" : "ok");
        (void)zeros_ok;
    }
    return 0;
}
