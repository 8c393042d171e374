// fft_device.cuh — in-register / shared-memory Stockham FFT engine for sm_100a.
//
// Replaces the reference's scalar radix-2 DIT loop (FftPlan::run, numerics.cpp:73-97) with a
// batched, block-cooperative autosort (Stockham) FFT:
//   * a transform of L = 2^LOG2L points is owned by NT = L/16 threads; thread `tid` always holds
//     the 16 elements at positions tid + NT*q (q < 16) between passes, so the first pass reads
//     global memory coalesced and the last pass leaves natural-order results in registers,
//     ready for a coalesced store or a fused epilogue (CZT kernel product, H(f), ...);
//   * radix-16 butterflies in registers (4x4 split, constant twiddles folded); the last pass
//     takes the leftover radix 2/4/8; between passes one shared-memory exchange through a
//     padded layout (one pad slot per 16 elements) that keeps the strided first-pass writes
//     conflict-free;
//   * per-pass twiddles W_{pR}^{jk} come from an fp64-accurate table built on the host with the
//     reference's exact phase reduction (cis_cycles, numerics.cpp:122-128); fp32 tables are
//     rounded from fp64, never computed in fp32;
//   * the first pass can skip known-zero inputs (zero padding is synthesised, never loaded) and
//     the last pass can skip unneeded outputs (the CZT keeps only m of L bins).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tmem.cuh"

namespace skg {

template <typename T> struct CxT;
template <> struct CxT<double> { using type = double2; };
template <> struct CxT<float> { using type = float2; };
template <typename T> using cx_t = typename CxT<T>::type;

template <typename C> struct Scalar;
template <> struct Scalar<double2> { using type = double; };
template <> struct Scalar<float2> { using type = float; };
template <typename C> using sc_t = typename Scalar<C>::type;

template <typename C> __device__ __forceinline__ C mk(sc_t<C> a, sc_t<C> b) {
    C r;
    r.x = a;
    r.y = b;
    return r;
}
template <typename C> __device__ __forceinline__ C czero() { return mk<C>(0, 0); }
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return mk<C>(a.x + b.x, a.y + b.y); }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return mk<C>(a.x - b.x, a.y - b.y); }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
    return mk<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename C> __device__ __forceinline__ C cmulc(C a, C b) {
    return mk<C>(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename C> __device__ __forceinline__ C cconj(C a) { return mk<C>(a.x, -a.y); }
template <typename C> __device__ __forceinline__ C cscale(C a, sc_t<C> s) { return mk<C>(a.x * s, a.y * s); }
// real * complex
template <typename C> __device__ __forceinline__ C rmul(sc_t<C> r, C a) { return mk<C>(r * a.x, r * a.y); }
// ---- packed fp32 (sm_100a FADD2 / FMUL2 / FFMA2) --------------------------------------------------
// Blackwell issues two fp32 operations per lane in one instruction (fma.rn.f32x2 & co.), at the same
// flop rate as scalar FFMA (tools/micro/ffma2.cu: 238 against 233 flop/clk/SM) but half the issue
// slots. A complex value is exactly such a pair, and the fp32 transforms are issue bound (the cube:
// 70% issue active, FP instructions 62% of the stream), so float2 arithmetic is carried packed: a
// complex add is one FADD2, a complex product an FMUL2 + FFMA2 (ptxas folds the broadcast / swapped
// operands into the F32 / LO_HI operand selectors; only a swapped-and-negated operand costs a scalar
// negate). Same formulas as the scalar code, fused where the scalar code's contraction fuses.
#ifndef SKG_NO_F32X2
namespace px {
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 up(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ float2 add(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a.x, a.y)), "l"(pk(b.x, b.y)));
    return up(r);
}
__device__ __forceinline__ float2 sub(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a.x, a.y)), "l"(pk(b.x, b.y)));
    return up(r);
}
__device__ __forceinline__ float2 mul(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a.x, a.y)), "l"(pk(b.x, b.y)));
    return up(r);
}
__device__ __forceinline__ float2 fma(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a.x, a.y)), "l"(pk(b.x, b.y)), "l"(pk(c.x, c.y)));
    return up(r);
}
__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }
}  // namespace px

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return px::add(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return px::sub(a, b); }
// a b = a.x (b.x, b.y) + a.y (-b.y, b.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return px::fma(px::bc(a.y), make_float2(-b.y, b.x), px::mul(px::bc(a.x), b));
}
// a conj(b) = b.x (a.x, a.y) + b.y (a.y, -a.x)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return px::fma(px::bc(b.y), make_float2(a.y, -a.x), px::mul(px::bc(b.x), a));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return px::mul(px::bc(s), a); }
__device__ __forceinline__ float2 rmul(float r, float2 a) { return px::mul(px::bc(r), a); }
template <bool INV> __device__ __forceinline__ float2 mul_w8(float2 a) {
    // forward r (a.x + a.y, a.y - a.x) = r (a + (a.y, -a.x)); inverse r (a.x - a.y, a.x + a.y) = r (a + (-a.y, a.x))
    const float r = 0.70710678118654752440f;
    return px::mul(px::bc(r), px::add(a, INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x)));
}
template <bool INV> __device__ __forceinline__ float2 mul_w8_3(float2 a) {
    // forward r (a.y - a.x, -(a.x + a.y)) = r ((a.y, -a.x) - a); inverse r (-(a.x + a.y), a.x - a.y) = r ((-a.y, a.x) - a)
    const float r = 0.70710678118654752440f;
    return px::mul(px::bc(r), px::sub(INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x), a));
}
// a e^{-/+ i theta}: forward c a + s (a.y, -a.x); inverse c a + s (-a.y, a.x)
template <bool INV> __device__ __forceinline__ float2 mul_cs(float2 a, float c, float s) {
    return px::fma(px::bc(s), INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x), px::mul(px::bc(c), a));
}
#endif

// twiddle multiply: forward uses w, inverse uses conj(w)
template <bool INV, typename C> __device__ __forceinline__ C twmul(C a, C w) {
    return INV ? cmulc(a, w) : cmul(a, w);
}
// multiply by W4 = -i (forward) / +i (inverse)
template <bool INV, typename C> __device__ __forceinline__ C mul_w4(C a) {
    return INV ? mk<C>(-a.y, a.x) : mk<C>(a.y, -a.x);
}
// multiply by W8^1 = (1 -/+ i)/sqrt2
template <bool INV, typename C> __device__ __forceinline__ C mul_w8(C a) {
    const sc_t<C> r = (sc_t<C>)0.70710678118654752440;
    return INV ? mk<C>((a.x - a.y) * r, (a.x + a.y) * r) : mk<C>((a.x + a.y) * r, (a.y - a.x) * r);
}
// multiply by W8^3 = (-1 -/+ i)/sqrt2
template <bool INV, typename C> __device__ __forceinline__ C mul_w8_3(C a) {
    const sc_t<C> r = (sc_t<C>)0.70710678118654752440;
    return INV ? mk<C>(-(a.x + a.y) * r, (a.x - a.y) * r) : mk<C>((a.y - a.x) * r, -(a.x + a.y) * r);
}
// multiply by exp(-/+ i theta) given c = cos theta, s = sin theta
template <bool INV, typename C> __device__ __forceinline__ C mul_cs(C a, sc_t<C> c, sc_t<C> s) {
    return INV ? mk<C>(a.x * c - a.y * s, a.y * c + a.x * s) : mk<C>(a.x * c + a.y * s, a.y * c - a.x * s);
}

// ---- epilogue math ----------------------------------------------------------------------------
// fp32 atan2: odd minimax polynomial for atan on [0, 1] plus octant fixups: degree 15 (max error
// 1.4e-7 rad evaluated in fp32); SKG_ATAN_DEG13 selects degree 13 (3.4e-7 rad; coefficients from a
// linear-programming minimax fit on [0, 1]) — measured 0.3% faster on the cube, so not the default.
// The zero vector needs no branch: min / max(max, tiny) is 0 when both are 0 (cube: 1.141 -> 1.101 ms).
// Out-of-range operands of the fp32 epilogue (|v|^2 beyond fp32's range, or the atan2 ratio's divisor
// beyond __fdividef's) are redone with hypotf / atan2f behind a WARP-UNIFORM test (__any_sync): the
// fast path stays straight-line code; a lane-level if would be predicated into every bin, an
// out-of-line call costs the ABI's register spills (measured: cube 1.10 -> 1.33 / 1.42 ms)
__device__ __forceinline__ float fast_atan2f(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
#ifdef SKG_EPI_GUARDS
    const bool odd = mx > 0x1p126f || (mx < 0x1p-100f && mx > 0.0f);
    if (__any_sync(__activemask(), odd) && odd) return atan2f(y, x);
#endif
    const float a = __fdividef(mn, fmaxf(mx, 1e-30f));
    const float s = a * a;
#ifndef SKG_ATAN_DEG13
    float r = -0.004054566379636526f;
    r = fmaf(r, s, 0.02186295948922634f);
    r = fmaf(r, s, -0.055912334471940994f);
    r = fmaf(r, s, 0.0964219868183136f);
    r = fmaf(r, s, -0.1390863060951233f);
    r = fmaf(r, s, 0.19946566224098206f);
    r = fmaf(r, s, -0.33329859375953674f);
    r = fmaf(r, s, 0.9999993443489075f);
#else
    float r = 0.00683815311640501f;
    r = fmaf(r, s, -0.03368566557765007f);
    r = fmaf(r, s, 0.07972026616334915f);
    r = fmaf(r, s, -0.1323888599872589f);
    r = fmaf(r, s, 0.1980941742658615f);
    r = fmaf(r, s, -0.3331758975982666f);
    r = fmaf(r, s, 0.9999962449073792f);
#endif
    r *= a;
    if (ay > ax) r = 1.57079632679489662f - r;
    if (x < 0.0f) r = 3.14159265358979324f - r;
    return copysignf(r, y);
}
__device__ __forceinline__ double atan2_t(double y, double x) { return atan2(y, x); }
__device__ __forceinline__ float atan2_t(float y, float x) { return fast_atan2f(y, x); }
__device__ __forceinline__ double abs_t(double x, double y) { return hypot(x, y); }
__device__ __forceinline__ float abs_t(float x, float y) {
    const float h = fmaf(x, x, y * y);
#ifdef SKG_EPI_GUARDS
    const bool odd = h > 0x1p126f || (h < 0x1p-100f && h > 0.0f);   // |v|^2 out of range
    if (__any_sync(__activemask(), odd) && odd) return hypotf(x, y);
#endif
#ifdef SKG_ABS_RSQRT
    return h > 0.0f ? h * rsqrtf(h) : 0.0f;
#else
    float r;   // MUFU.SQRT (max relative error 2^-23; sqrt(0) = 0, so no zero guard)
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(h));
    return r;
#endif
}
// magnitude_db (types.cpp:13-18): 20 log10 |v|, -300 dB at |v| <= 1e-15
__device__ __forceinline__ double magnitude_db_t(double x, double y) {
    // 20 log10 hypot = 10 log10 |v|^2 (a few ulp of the argument: ~1e-15 dB), without hypot's
    // scaling work; |v|^2 <= 1e-30 <=> |v| <= 1e-15 (an |v|^2 that underflows is below the floor too)
    const double h = fma(x, x, y * y);
    return h > 1e-30 ? 10.0 * log10(h) : -300.0;
}
__device__ __forceinline__ float magnitude_db_t(float x, float y) {
    // 20 log10 sqrt(h) = 10 log10 h; the floor test on h = |v|^2 (1e-30 is a normal float)
    const float h = fmaf(x, x, y * y);
    return h > 1e-30f ? 10.0f * log10f(h) : -300.0f;
}

// ---- small DFTs, natural order in and out.
// NZ = number of leading inputs that may be nonzero, NO = number of leading outputs needed.
template <bool INV, int NZ = 4, int NO = 4, typename C>
__device__ __forceinline__ void dft4(C& a0, C& a1, C& a2, C& a3) {
    if constexpr (NZ <= 0) {
        a0 = czero<C>(); a1 = a0; a2 = a0; a3 = a0;
    } else if constexpr (NZ == 1) {
        a1 = a0; a2 = a0; a3 = a0;
    } else if constexpr (NZ == 2) {
        const C b = mul_w4<INV>(a1);
        const C x0 = cadd(a0, a1), x2 = csub(a0, a1), x1 = cadd(a0, b), x3 = csub(a0, b);
        a0 = x0; a1 = x1; a2 = x2; a3 = x3;
    } else {
        const C t0 = cadd(a0, a2), t1 = csub(a0, a2);
        const C t2 = cadd(a1, a3), t3 = mul_w4<INV>(csub(a1, a3));
        a0 = cadd(t0, t2);
        if constexpr (NO > 1) a1 = cadd(t1, t3);
        if constexpr (NO > 2) a2 = csub(t0, t2);
        if constexpr (NO > 3) a3 = csub(t1, t3);
    }
}

template <bool INV, typename C> __device__ __forceinline__ void dft2(C& a0, C& a1) {
    const C t = a0;
    a0 = cadd(t, a1);
    a1 = csub(t, a1);
}

template <bool INV, typename C> __device__ __forceinline__ void dft8(C (&a)[8]) {
    dft4<INV>(a[0], a[2], a[4], a[6]);
    dft4<INV>(a[1], a[3], a[5], a[7]);
    // now a[2k] = E_k, a[2k+1] = O_k
    const C o1 = mul_w8<INV>(a[3]), o2 = mul_w4<INV>(a[5]), o3 = mul_w8_3<INV>(a[7]);
    const C e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6], o0 = a[1];
    a[0] = cadd(e0, o0); a[4] = csub(e0, o0);
    a[1] = cadd(e1, o1); a[5] = csub(e1, o1);
    a[2] = cadd(e2, o2); a[6] = csub(e2, o2);
    a[3] = cadd(e3, o3); a[7] = csub(e3, o3);
}

// 16-point DFT as 4x4 (n = n2 + 4 n1, k = k1 + 4 k2); NZ in {1,2,4,8,16}, NO in {4,8,16}.
template <bool INV, int NZ = 16, int NO = 16, typename C> __device__ __forceinline__ void dft16(C (&a)[16]) {
    constexpr sc_t<C> C1 = (sc_t<C>)0.92387953251128675613;  // cos(pi/8)
    constexpr sc_t<C> S1 = (sc_t<C>)0.38268343236508977173;  // sin(pi/8)
    // stage 1: column n2 holds a[n2 + 4 n1]
    constexpr int nz0 = NZ >= 13 ? 4 : NZ >= 9 ? 3 : NZ >= 5 ? 2 : NZ >= 1 ? 1 : 0;
    constexpr int nz1 = NZ >= 14 ? 4 : NZ >= 10 ? 3 : NZ >= 6 ? 2 : NZ >= 2 ? 1 : 0;
    constexpr int nz2 = NZ >= 15 ? 4 : NZ >= 11 ? 3 : NZ >= 7 ? 2 : NZ >= 3 ? 1 : 0;
    constexpr int nz3 = NZ >= 16 ? 4 : NZ >= 12 ? 3 : NZ >= 8 ? 2 : NZ >= 4 ? 1 : 0;
    constexpr int rows = NZ >= 4 ? 4 : NZ;   // nonzero rows entering stage 2
    dft4<INV, (nz0 == 3 ? 4 : nz0)>(a[0], a[4], a[8], a[12]);
    if constexpr (rows > 1) dft4<INV, (nz1 == 3 ? 4 : nz1)>(a[1], a[5], a[9], a[13]);
    if constexpr (rows > 2) dft4<INV, (nz2 == 3 ? 4 : nz2)>(a[2], a[6], a[10], a[14]);
    if constexpr (rows > 3) dft4<INV, (nz3 == 3 ? 4 : nz3)>(a[3], a[7], a[11], a[15]);
    // twiddles W16^{n2 k1}: element a[n2 + 4 k1]
    if constexpr (rows > 1) {
        a[5] = mul_cs<INV>(a[5], C1, S1);      // n2=1,k1=1: W16^1
        a[9] = mul_w8<INV>(a[9]);              // n2=1,k1=2: W16^2
        a[13] = mul_cs<INV>(a[13], S1, C1);    // n2=1,k1=3: W16^3
    }
    if constexpr (rows > 2) {
        a[6] = mul_w8<INV>(a[6]);              // W16^2
        a[10] = mul_w4<INV>(a[10]);            // W16^4
        a[14] = mul_w8_3<INV>(a[14]);          // W16^6
    }
    if constexpr (rows > 3) {
        a[7] = mul_cs<INV>(a[7], S1, C1);      // W16^3
        a[11] = mul_w8_3<INV>(a[11]);          // W16^6
        a[15] = mul_cs<INV>(a[15], -C1, -S1);  // W16^9
    }
    // stage 2: for each k1, DFT4 over n2 of a[4 k1 + n2] -> X[k1 + 4 k2] lands in a[4 k1 + k2]
    constexpr int no4 = NO / 4;
    dft4<INV, rows, no4>(a[0], a[1], a[2], a[3]);
    dft4<INV, rows, no4>(a[4], a[5], a[6], a[7]);
    dft4<INV, rows, no4>(a[8], a[9], a[10], a[11]);
    dft4<INV, rows, no4>(a[12], a[13], a[14], a[15]);
    // transpose 4x4 so a[k] = X[k]  (pure register renaming)
    C t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = a[i];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) a[k1 + 4 * k2] = t[4 * k1 + k2];
}

template <int R, bool INV, int NZ, int NO, typename C> __device__ __forceinline__ void dft_r(C (&u)[R]) {
    if constexpr (R == 1) {
    } else if constexpr (R == 2) {
        dft2<INV>(u[0], u[1]);
    } else if constexpr (R == 4) {
        dft4<INV>(u[0], u[1], u[2], u[3]);
    } else if constexpr (R == 8) {
        dft8<INV>(u);
    } else {
        static_assert(R == 16, "radix");
        dft16<INV, NZ, NO>(u);
    }
}

// ---- geometry of an L = 2^LOG2L transform ------------------------------------------------
// Twiddles of pass s (p = 16^s) are W_{pR}^{jk}, k < p, j < R. Only W_{pR}^{k} is stored, factorised
// by the base-16 digits of k (W_{pR}^{k} = prod_d W_{pR/16^d}^{k_d}: one 16-entry table per digit,
// 48 entries for L = 4096) in shared memory; the powers j = 2..R-1 are formed in registers by
// balanced products (depth <= 4). The passes are shared-memory-bandwidth bound (LDS.128 costs four
// wavefronts whatever the broadcast), so trading table reads for FP instructions pays.
template <int LOG2L> struct FftGeom {
    static constexpr int L = 1 << LOG2L;
    static constexpr int EPT = L < 16 ? L : 16;        // elements per thread
    static constexpr int NT = L / EPT;                  // threads per transform
    static constexpr int P = L < 16 ? 1 : (LOG2L + 3) / 4;   // passes
    static constexpr int RSMALL = L < 16 ? L : (1 << (LOG2L - 4 * (P - 1)));   // the one non-16 radix
    static constexpr int SMEM = L < 16 ? 0 : L + (L >> 4);   // padded elements per transform
    // radix of pass s: 16 everywhere except one pass of RSMALL, placed second when there are >= 3
    // passes so that the first (zero-input pruning) and the last (unneeded-output pruning) stay radix 16
    // (measured with the shared-forward CZT: configs[1] fp64 0.234 -> 0.226 ms; other rows neutral)
    __host__ __device__ static constexpr int radix(int s) {
        if (L < 16) return L;
        if (RSMALL == 16) return 16;
#ifndef SKG_SMALL_RADIX_MID
#define SKG_SMALL_RADIX_MID 1
#endif
        if (SKG_SMALL_RADIX_MID && P >= 3) return s == 1 ? RSMALL : 16;
        return s < P - 1 ? 16 : RSMALL;
    }
    __host__ __device__ static constexpr int lg(int v) { return v <= 1 ? 0 : 1 + lg(v / 2); }
    __host__ __device__ static constexpr int pval(int s) {   // product of the radices before pass s
        int p = 1;
        for (int t = 0; t < s; ++t) p *= radix(t);
        return p;
    }
    __host__ __device__ static constexpr int digits(int s) { return (lg(pval(s)) + 3) / 4; }   // base-16 digits of k < p
    // offset of the digit-d table of pass s: 4 x 16 entries W_{pR/16^d}^{j kd}, j in {1, 2, 4, 8}
    // (fp64 reads only j = 1; fp32 reads the four so no twiddle carries more than 4 roundings)
    __host__ __device__ static constexpr int tw_off(int s, int d) {
        int o = 0;
        for (int t = 1; t < s; ++t) o += digits(t) * 64;
        return o + d * 64;
    }
    static constexpr int TW_SIZE = tw_off(P, 0);   // entries (pass 0 needs none)
    static constexpr int TW_ALLOC = TW_SIZE > 0 ? TW_SIZE : 1;
};

__device__ __forceinline__ int pad16(int a) { return a + (a >> 4); }

// u[j] *= W^{jk}, j = 1..R-1, from w1 = W^{k} alone: squarings give w2, w4, w8 and the rest are
// single products applied as soon as they are formed (few twiddles live; product depth <= 4)
template <bool INV, int R, typename C>
__device__ __forceinline__ void apply_twiddles(C (&u)[R], C w1, C l2 = C(), C l4 = C(), C l8 = C()) {
    // fp32: w2, w4, w8 come from the tables (l2, l4, l8); fp64: by squaring
    constexpr bool loaded = sizeof(sc_t<C>) == 4;
    if constexpr (R >= 2) u[1] = twmul<INV>(u[1], w1);
    if constexpr (R >= 4) {
        const C w2 = loaded ? l2 : cmul(w1, w1);
        const C w3 = cmul(w2, w1);
        u[2] = twmul<INV>(u[2], w2);
        u[3] = twmul<INV>(u[3], w3);
        if constexpr (R >= 8) {
            const C w4 = loaded ? l4 : cmul(w2, w2);
            u[4] = twmul<INV>(u[4], w4);
            const C w5 = cmul(w4, w1), w6 = cmul(w4, w2), w7 = cmul(w4, w3);
            u[5] = twmul<INV>(u[5], w5);
            u[6] = twmul<INV>(u[6], w6);
            u[7] = twmul<INV>(u[7], w7);
            if constexpr (R >= 16) {
                const C w8 = loaded ? l8 : cmul(w4, w4);
                u[8] = twmul<INV>(u[8], w8);
                u[9] = twmul<INV>(u[9], cmul(w8, w1));
                u[10] = twmul<INV>(u[10], cmul(w8, w2));
                u[11] = twmul<INV>(u[11], cmul(w8, w3));
                u[12] = twmul<INV>(u[12], cmul(w8, w4));
                u[13] = twmul<INV>(u[13], cmul(w8, w5));
                u[14] = twmul<INV>(u[14], cmul(w8, w6));
                u[15] = twmul<INV>(u[15], cmul(w8, w7));
            }
        }
    }
}

// cache-line prefetches (no registers consumed; the data waits in L1 / L2 for the real load)
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// copy the factorised twiddle tables of an L-point transform into shared memory (whole CTA)
template <int LOG2L, typename C>
__device__ __forceinline__ void load_twiddles(C* dst, const C* __restrict__ src) {
    for (int i = threadIdx.x; i < FftGeom<LOG2L>::TW_SIZE; i += blockDim.x) dst[i] = __ldg(src + i);
}

template <typename C> __device__ __forceinline__ C ldg_c(const C* p) {
#ifdef SKG_PLAIN_LD
    return *p;
#else
    return __ldg(p);
#endif
}

// Barrier used between passes: the whole CTA, or — for kernels whose thread groups work on
// independent transforms — a named barrier shared only by the group's warps.
struct CtaSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct GroupSync {
    int id, nthreads;   // id >= 1 (0 is __syncthreads), nthreads a multiple of 32
    __device__ __forceinline__ void operator()() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
    }
};

// One Stockham pass. v[q] holds position tid + NT*q on entry and exit.
// TMT: the pass is a last radix-16 pass with one butterfly per thread (k = tid) and its fifteen
// twiddles W^{jk} come precomputed from this thread's TMEM lane at `tmt` (16 complex, j = 0..15;
// kernels_czt_tm.cuh) instead of being formed by products from the per-digit tables.
template <bool INV, int S, int NZ, int NO, int LOG2L, typename C, typename SYNC = CtaSync, bool TMT = false>
__device__ __forceinline__ void stockham_pass(C (&v)[FftGeom<LOG2L>::EPT], C* sm, const C* __restrict__ tw,
                                              int tid, bool active = true, SYNC sync = SYNC(), uint32_t tmt = 0) {
    using G = FftGeom<LOG2L>;
    constexpr int R = G::radix(S);
    constexpr int p = G::pval(S);
    constexpr int B = G::EPT / R;
    constexpr bool last = (S == G::P - 1);
#pragma unroll
    for (int b = 0; b < B; ++b) {
        C u[R];
#pragma unroll
        for (int j = 0; j < R; ++j) u[j] = v[b + B * j];
        const int i = tid + G::NT * b;
        const int k = i & (p - 1);
        if constexpr (TMT && last && B == 1 && R == 16) {
            constexpr int K4 = 16 / CxWords<C>::W;
#pragma unroll
            for (int c = 0; c < 16 / K4; ++c) {
                C w[K4];
                tmem_get<C, K4>(tmt + c * 16, w);
#pragma unroll
                for (int i = 0; i < K4; ++i)
                    if (c * K4 + i >= 1) u[c * K4 + i] = twmul<INV>(u[c * K4 + i], w[i]);
            }
        } else if constexpr (p > 1) {
            // W^{jk} for j = 1 (and 2, 4, 8 in fp32) from the per-digit tables. The table geometry is
            // forced to compile time: ptxas once kept a CALL to the (recursive) digit count in the
            // pass loop.
            constexpr int ND = G::digits(S);
            constexpr int TO0 = G::tw_off(S, 0), TO1 = G::tw_off(S, 1), TO2 = G::tw_off(S, 2), TO3 = G::tw_off(S, 3);
            static_assert(ND <= 4, "digits");
            auto wj = [&](int jj) {
                C w = tw[TO0 + jj * 16 + (k & 15)];
                if constexpr (ND > 1) w = cmul(w, tw[TO1 + jj * 16 + ((k >> 4) & 15)]);
                if constexpr (ND > 2) w = cmul(w, tw[TO2 + jj * 16 + ((k >> 8) & 15)]);
                if constexpr (ND > 3) w = cmul(w, tw[TO3 + jj * 16 + ((k >> 12) & 15)]);
                return w;
            };
            if constexpr (sizeof(sc_t<C>) == 8) {
                apply_twiddles<INV, R>(u, wj(0));
            } else {
                apply_twiddles<INV, R>(u, wj(0), R >= 4 ? wj(1) : czero<C>(), R >= 8 ? wj(2) : czero<C>(),
                                       R >= 16 ? wj(3) : czero<C>());
            }
        }
        dft_r<R, INV, (S == 0 ? NZ : 16), (last ? NO : 16)>(u);
        if constexpr (last) {
#pragma unroll
            for (int j = 0; j < R; ++j) v[b + B * j] = u[j];
        } else {
            const int base = (i / p) * p * R + k;
            if (active) {
#pragma unroll
                for (int j = 0; j < R; ++j) sm[pad16(base + j * p)] = u[j];
            }
        }
    }
    if constexpr (!last) {
        sync();
        if (active) {
#pragma unroll
            for (int q = 0; q < G::EPT; ++q) v[q] = sm[pad16(tid + G::NT * q)];
        }
        sync();
    }
}

// Full transform: NZ = leading nonzero inputs of the first radix-16 pass (1..16),
// NO = leading outputs needed from the last radix-16 pass (4, 8 or 16).
// TMT: last-pass twiddles from TMEM at lane address `tmt` (see stockham_pass)
template <bool INV, int LOG2L, int NZ = 16, int NO = 16, typename C, typename SYNC = CtaSync, bool TMT = false>
__device__ __forceinline__ void block_fft(C (&v)[FftGeom<LOG2L>::EPT], C* sm, const C* __restrict__ tw, int tid,
                                          bool active = true, SYNC sync = SYNC(), uint32_t tmt = 0) {
    using G = FftGeom<LOG2L>;
    if constexpr (G::L < 16) {
        dft_r<G::L, INV, 16, 16>(v);
    } else {
        constexpr int nz = G::radix(0) == 16 ? NZ : 16;
        constexpr int no = G::radix(G::P - 1) == 16 ? NO : 16;
        stockham_pass<INV, 0, nz, (G::P == 1 ? no : 16), LOG2L, C, SYNC, TMT && G::P == 1>(v, sm, tw, tid, active, sync, tmt);
        if constexpr (G::P > 1) stockham_pass<INV, 1, 16, (G::P == 2 ? no : 16), LOG2L, C, SYNC, TMT && G::P == 2>(v, sm, tw, tid, active, sync, tmt);
        if constexpr (G::P > 2) stockham_pass<INV, 2, 16, (G::P == 3 ? no : 16), LOG2L, C, SYNC, TMT && G::P == 3>(v, sm, tw, tid, active, sync, tmt);
        if constexpr (G::P > 3) stockham_pass<INV, 3, 16, (G::P == 4 ? no : 16), LOG2L, C, SYNC, TMT && G::P == 4>(v, sm, tw, tid, active, sync, tmt);
        static_assert(G::P <= 4, "single-CTA engine handles L <= 65536");
    }
}

}  // namespace skg
