// tmem.cuh — tensor memory (TMEM) used as per-thread scratch, no tensor-core math.
//
// Each SM has 256 KB of TMEM: 128 lanes x 512 columns of 32 bits. With the 32x32b access shape every
// thread of a warp reads / writes its OWN lane, and warp w may touch lanes 32*(w%4) .. 32*(w%4)+31
// only, so the 128 threads t = 0..127 of any 128-thread slice of the CTA own lanes 0..127 and the
// columns are the free dimension. Measured on B200 (tools/micro/tmem_bw.cu, 16 warps per SM):
// tcgen05.ld 440-460 B/clk/SM, tcgen05.st 734 B/clk/SM, against 127.5 B/clk/SM for LDS.128 — and a
// TMEM read stream beside an LDS stream costs the LDS stream nothing (4.29 vs 4.43 ms). So tables a
// thread re-reads for every record (chirps, kernel spectra) and data it parks between phases move
// off the shared-memory / L1 path, which the FFT exchanges need for themselves.
#pragma once
#include <cstdint>

#include "bulk_copy.cuh"

namespace skg {

// One warp allocates `cols` columns (power of two, 32..512) and publishes the base address through
// shared memory; every thread returns it after the fence / barrier / fence sequence.
template <int COLS> __device__ __forceinline__ uint32_t tmem_alloc_cta(uint32_t* slot) {
    static_assert(COLS >= 32 && COLS <= 512 && (COLS & (COLS - 1)) == 0, "TMEM columns: power of two");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                     "n"(COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    return *reinterpret_cast<volatile uint32_t*>(slot);
}

template <int COLS> __device__ __forceinline__ void tmem_free_cta(uint32_t base) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS) : "memory");
}

// address of this thread's lane, column `col`: lane = 32 * (warp % 4) + lane-in-warp
__device__ __forceinline__ uint32_t tmem_lane_addr(uint32_t base, uint32_t col) {
    return base + ((uint32_t)((threadIdx.x / 32) % 4 * 32) << 16) + col;
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// make TMEM stores of this thread visible to other warps across the next barrier
__device__ __forceinline__ void tmem_fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 4 / 8 / 16 consecutive 32-bit columns of this thread's lane <-> registers (warp-collective)
__device__ __forceinline__ void tmem_ld4(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a)
                 );
}
__device__ __forceinline__ void tmem_ld8(uint32_t a, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(a)
                 );
}
__device__ __forceinline__ void tmem_ld16(uint32_t a, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(a)
        );
}
// load + wait in ONE asm statement: the compiler cannot schedule a use of r[] before the wait
__device__ __forceinline__ void tmem_ld16_wait(uint32_t a, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(a)
        );
}
__device__ __forceinline__ void tmem_st4(uint32_t a, const uint32_t (&r)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3])
                 );
}
__device__ __forceinline__ void tmem_st8(uint32_t a, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 );
}
__device__ __forceinline__ void tmem_st16(uint32_t a, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            a),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        );
}

// complex values <-> 32-bit words (double2: 4 words, float2: 2 words)
template <typename C> struct CxWords;
template <> struct CxWords<double2> {
    static constexpr int W = 4;
    __device__ static __forceinline__ void put(uint32_t* w, double2 v) {
        w[0] = __double2loint(v.x);
        w[1] = __double2hiint(v.x);
        w[2] = __double2loint(v.y);
        w[3] = __double2hiint(v.y);
    }
    __device__ static __forceinline__ double2 get(const uint32_t* w) {
        return make_double2(__hiloint2double(w[1], w[0]), __hiloint2double(w[3], w[2]));
    }
};
template <> struct CxWords<float2> {
    static constexpr int W = 2;
    __device__ static __forceinline__ void put(uint32_t* w, float2 v) {
        w[0] = __float_as_uint(v.x);
        w[1] = __float_as_uint(v.y);
    }
    __device__ static __forceinline__ float2 get(const uint32_t* w) {
        return make_float2(__uint_as_float(w[0]), __uint_as_float(w[1]));
    }
};

// K complex values (K * W == 16 words) at `lane_col` = this thread's lane address (tmem_lane_addr) + column
template <typename C, int K> __device__ __forceinline__ void tmem_get(uint32_t lane_col, C (&v)[K]) {
    static_assert(K * CxWords<C>::W == 16, "16-word chunk");
    uint32_t r[16];
    tmem_ld16_wait(lane_col, r);
#pragma unroll
    for (int i = 0; i < K; ++i) v[i] = CxWords<C>::get(r + i * CxWords<C>::W);
}
template <typename C, int K> __device__ __forceinline__ void tmem_put(uint32_t lane_col, const C (&v)[K]) {
    static_assert(K * CxWords<C>::W == 16, "16-word chunk");
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < K; ++i) CxWords<C>::put(r + i * CxWords<C>::W, v[i]);
    tmem_st16(lane_col, r);
}

}  // namespace skg
