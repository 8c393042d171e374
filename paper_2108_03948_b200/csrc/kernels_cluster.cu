// kernels_cluster.cu — one L-point FFT per thread-block CLUSTER, the exchange through distributed
// shared memory (DSMEM) instead of an HBM work buffer.
//
// For L beyond one CTA's shared memory (fp64 L = 2^15, 2^16; fp32 2^16, 2^17) the four-step path
// (kernels_4step.cuh) writes and re-reads an L-point work row in HBM per transform: 3x the
// algorithm's bytes. Here the CS = 8 CTAs of a cluster (one per SM, same GPC) hold the transform:
//   n = n1 + CS n2, k = k1 Q + k2   (Q = L / CS, n1, k1 < CS; n2, k2 < Q)
//   X[k1 Q + k2] = sum_n1 W_CS^{n1 k1} W_L^{n1 k2} sum_n2 x[n1 + CS n2] W_Q^{n2 k2}
//   1. CTA r = n1 loads x[r + CS n2] (zero padding synthesised: only n < N is read) and runs the
//      Q-point Stockham FFT of fft_device.cuh entirely in its own shared memory / registers;
//   2. twiddle W_L^{r k2} (table row r) and push: the value for k2 goes to the CTA s owning the
//      k2-block [s Q/CS, (s+1) Q/CS) — with NT = Q/16 threads holding k2 = tid + NT q, the owner is
//      q / 2 and the remote write position r (Q/CS) + tid + NT (q & 1): consecutive threads write
//      consecutive DSMEM addresses;
//   3. CTA s finishes a radix-CS DFT over n1 for each of its Q/CS k2 and stores X[k1 Q + k2]:
//      CS runs of Q/CS contiguous bins — coalesced, written once.
// HBM traffic is the algorithmic minimum (trace in, bins out); the exchange crosses the cluster
// once. Per transform: (A) an execution-only cluster barrier — every CTA's Q-FFT is done with its
// shared buffer, which then receives the pushed values — and (B) each CTA waits on its own mbarrier
// until the st.async pushes of all CS CTAs (Q values) have landed. Persistent clusters loop over the
// batch. Opt-in (SKG_CLUSTER=1): measured slower than the four-step passes. Replaces FftPlan::run (numerics.cpp:73-97) at these lengths, as fft_spectrum's full /
// half layout (spectra.cpp:21-38) or the plain complex transform (fft / ifft, numerics.cpp:102-120).
#include <cuda_runtime.h>

#include "fft_device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"


namespace skg {

namespace {

constexpr int CS = 8;   // CTAs per cluster (portable maximum)

// cluster primitives as PTX: explicit shared::cluster stores (no generic-address path, no GPU-scope
// fence) and the split arrive(release) / wait(acquire) cluster barrier
__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_map(const void* smem_ptr, unsigned rank) {
    unsigned a = (unsigned)__cvta_generic_to_shared(smem_ptr), d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(rank));
    return d;
}
// remote store that signals the destination CTA's mbarrier with its byte count (st.async: the
// DSMEM push completes as a transaction on the receiver's barrier — no cluster-wide fence)
__device__ __forceinline__ void cl_st(unsigned addr, double2 v, unsigned rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "d"(v.x), "d"(v.y), "r"(rmbar)
                 : "memory");
}
__device__ __forceinline__ void cl_st(unsigned addr, float2 v, unsigned rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "f"(v.x), "f"(v.y), "r"(rmbar)
                 : "memory");
}
// full cluster barrier (release / acquire: used once at entry and once at exit)
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// execution-only cluster barrier: every CTA has passed this point (its shared reads are done — their
// values are in registers); no memory ordering requested
__device__ __forceinline__ void cl_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(unsigned mbar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned mbar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned mbar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(mbar),
        "r"(parity)
        : "memory");
}
#ifndef SKG_CLUSTER_MINB
#define SKG_CLUSTER_MINB 2   // CTAs per SM the register cap targets (clusters overlap on an SM)
#endif

template <typename T, int LOG2Q> struct ClCfg {
    using G = FftGeom<LOG2Q>;
    static constexpr int Q = G::L;
    static constexpr int NT = G::NT;        // threads per CTA
    static constexpr int DQ = Q / CS;       // k2 per owner CTA (= 2 NT)
    static constexpr size_t SMEM = ((size_t)G::SMEM + G::TW_ALLOC) * sizeof(cx_t<T>);
    static_assert(DQ == 2 * NT, "owner mapping assumes 16 elements per thread and CS = 8");
};

// in_kind: 0 complex rows, 1 real rows (imaginary part 0); MODE 0: all L bins, 1: bins 0..L/2
template <typename T, int LOG2Q, int NZ, bool INV, int MODE>
__global__ void __launch_bounds__(ClCfg<T, LOG2Q>::NT, (ClCfg<T, LOG2Q>::NT <= 256 ? SKG_CLUSTER_MINB : 1))
k_fft_cluster(const void* __restrict__ xin, int in_kind, long long x_stride, long long N, long long batch,
              const cx_t<T>* __restrict__ tw, const cx_t<T>* __restrict__ twc, cx_t<T>* __restrict__ out,
              long long out_stride, T scale) {
    using C = cx_t<T>;
    using K = ClCfg<T, LOG2Q>;
    using G = typename K::G;
    constexpr int Q = K::Q, NT = K::NT, DQ = K::DQ;
    constexpr long long L = (long long)Q * CS;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* sm = reinterpret_cast<C*>(smraw);
    C* tws = sm + G::SMEM;
    __shared__ __align__(8) unsigned long long mbar_store;
    const unsigned mbar = (unsigned)__cvta_generic_to_shared(&mbar_store);
    const int r = (int)cl_rank();
    const int tid = threadIdx.x;
    load_twiddles<LOG2Q>(tws, tw);
    if (tid == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl_sync();   // barriers initialised cluster-wide before any remote signal
    unsigned parity = 0;
    const long long cid = blockIdx.x / CS, ncl = gridDim.x / CS;
    const C* twr = twc + (long long)r * Q;   // W_L^{r k2}
    for (long long b = cid; b < batch; b += ncl) {
        // 1. strided load of this CTA's residue class n = r + CS n2 and the Q-point FFT
        C v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            v[q] = czero<C>();
            const long long n = r + (long long)CS * (tid + NT * q);
            if (q < NZ && n < N) {
                if (in_kind == 0) v[q] = __ldg(reinterpret_cast<const C*>(xin) + b * x_stride + n);
                else v[q].x = __ldg(reinterpret_cast<const T*>(xin) + b * x_stride + n);
            }
        }
        block_fft<INV, LOG2Q, NZ>(v, sm, tws, tid);
        // 2. twiddle, then push k2 = tid + NT q to owner q/2 once every CTA is done with its buffer
        // this CTA's buffer will receive Q values (DQ from each of the CS CTAs, itself included)
        if (tid == 0) mbar_expect_tx(mbar, (unsigned)(Q * sizeof(C)));
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = twmul<INV>(v[q], __ldg(twr + tid + NT * q));
        cl_sync_relaxed();   // (A) every Q-FFT is done with its shared buffer
#pragma unroll
        for (int s2 = 0; s2 < CS; ++s2) {
            const unsigned base = cl_map(sm, (unsigned)s2), rbar = cl_map(&mbar_store, (unsigned)s2);
#pragma unroll
            for (int h = 0; h < 2; ++h)
                cl_st(base + (unsigned)(pad16(r * DQ + tid + NT * h) * sizeof(C)), v[2 * s2 + h], rbar);
        }
        mbar_wait(mbar, parity);   // (B) all Q values of this CTA's k2 block have landed
        parity ^= 1u;
        // 3. radix-CS over n1 for k2 = s DQ + j, j in {tid, tid + NT}; store X[k1 Q + k2]
        C* o = out + b * out_stride;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = tid + NT * h;
            C u[CS];
#pragma unroll
            for (int n1 = 0; n1 < CS; ++n1) u[n1] = sm[pad16(n1 * DQ + j)];
            dft8<INV>(u);
            const long long k2 = (long long)r * DQ + j;
#pragma unroll
            for (int k1 = 0; k1 < CS; ++k1) {
                const long long k = (long long)k1 * Q + k2;
                if (MODE == 0 || k <= L / 2) o[k] = cscale(u[k1], scale);
            }
        }
    }
    cl_sync();   // no CTA leaves while a peer may still address its shared memory
}

template <typename T, int LOG2Q, int NZ, bool INV, int MODE>
cudaError_t run_cluster(const void* x, int in_kind, long long x_stride, long long N, long long batch, const void* tw,
                        const void* twc, void* out, long long out_stride, T scale, cudaStream_t st) {
    using K = ClCfg<T, LOG2Q>;
    using C = cx_t<T>;
    auto kern = k_fft_cluster<T, LOG2Q, NZ, INV, MODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
    if (e != cudaSuccess) return e;
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(K::NT);
    cfg.dynamicSmemBytes = K::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // persistent: as many clusters as can be co-resident, capped by the batch
    int ncl = 0;
    cfg.gridDim = dim3(CS * 64);
    if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl < 1) ncl = std::max(1, sms / CS);
    const long long want = std::min<long long>(ncl, batch > 0 ? batch : 1);
    cfg.gridDim = dim3((unsigned)(want * CS));
    e = cudaLaunchKernelEx(&cfg, kern, x, in_kind, x_stride, N, batch, (const C*)tw, (const C*)twc, (C*)out,
                           out_stride, scale);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename T, int LOG2Q, bool INV, int MODE>
cudaError_t go_nz(const void* x, int in_kind, long long x_stride, long long N, long long batch, const void* tw,
                  const void* twc, void* out, long long out_stride, T scale, cudaStream_t st) {
    // leading nonzero count of the Q-point transforms: n2 < ceil((N - r) / CS) <= ceil(N / CS)
    const int nz = nz_class((N + CS - 1) / CS, ClCfg<T, LOG2Q>::NT);
    if (nz == 4) return run_cluster<T, LOG2Q, 4, INV, MODE>(x, in_kind, x_stride, N, batch, tw, twc, out, out_stride, scale, st);
    if (nz == 8) return run_cluster<T, LOG2Q, 8, INV, MODE>(x, in_kind, x_stride, N, batch, tw, twc, out, out_stride, scale, st);
    return run_cluster<T, LOG2Q, 16, INV, MODE>(x, in_kind, x_stride, N, batch, tw, twc, out, out_stride, scale, st);
}

template <typename T, int LOG2Q>
cudaError_t go_q(bool inverse, int mode, const void* x, int in_kind, long long x_stride, long long N, long long batch,
                 const void* tw, const void* twc, void* out, long long out_stride, T scale, cudaStream_t st) {
    if (inverse)
        return mode == 0 ? go_nz<T, LOG2Q, true, 0>(x, in_kind, x_stride, N, batch, tw, twc, out, out_stride, scale, st)
                         : go_nz<T, LOG2Q, true, 1>(x, in_kind, x_stride, N, batch, tw, twc, out, out_stride, scale, st);
    return mode == 0 ? go_nz<T, LOG2Q, false, 0>(x, in_kind, x_stride, N, batch, tw, twc, out, out_stride, scale, st)
                     : go_nz<T, LOG2Q, false, 1>(x, in_kind, x_stride, N, batch, tw, twc, out, out_stride, scale, st);
}

}  // namespace

int cluster_fft_log2q(int log2L, bool f32) {
    const int lq = log2L - 3;   // CS = 8
    if (f32) return (lq == 13 || lq == 14) ? lq : 0;   // L = 2^16, 2^17
    return (lq == 12 || lq == 13) ? lq : 0;            // L = 2^15, 2^16
}

cudaError_t launch_fft_cluster(int log2L, bool f32, bool inverse, int mode, const void* x, int in_kind,
                               long long x_stride, long long N, long long batch, const void* tw_q, const void* twc,
                               void* out, long long out_stride, double scale, cudaStream_t st) {
    const int lq = cluster_fft_log2q(log2L, f32);
    if (f32) {
        if (lq == 13) return go_q<float, 13>(inverse, mode, x, in_kind, x_stride, N, batch, tw_q, twc, out, out_stride, (float)scale, st);
        if (lq == 14) return go_q<float, 14>(inverse, mode, x, in_kind, x_stride, N, batch, tw_q, twc, out, out_stride, (float)scale, st);
    } else {
        if (lq == 12) return go_q<double, 12>(inverse, mode, x, in_kind, x_stride, N, batch, tw_q, twc, out, out_stride, scale, st);
        if (lq == 13) return go_q<double, 13>(inverse, mode, x, in_kind, x_stride, N, batch, tw_q, twc, out, out_stride, scale, st);
    }
    return cudaErrorNotSupported;
}

}  // namespace skg
