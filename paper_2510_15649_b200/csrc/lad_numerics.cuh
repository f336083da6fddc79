// lad_numerics.cuh -- device restatement of the reference's floating-point
// evaluation orders (numpy 2.3.5 pairwise sums, OpenBLAS 0.3.30 SkylakeX
// ddot / dgemv_t kernels).  Every add/mul/fma is an explicit round-to-nearest
// intrinsic, so the results are bit-identical to the reference regardless of
// -fmad.  The orders were measured against the reference's numpy in the build
// container (oracle/probe_numerics.py) and are pinned by tests/golden.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lad {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
// binary32 twins (fp32 mode: same operation order, every result rounded to binary32)
__device__ __forceinline__ float dadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float dsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float dmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float ddiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float dfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// Division by a precomputed reciprocal y = RN(1/b): q = RN(a*y) and two
// corrections q += RN(a - q*b)*y.  The first makes q faithful, the second then
// rounds correctly (Markstein), so the result equals a / b in round-to-nearest
// whenever nothing under- or overflows: |a|, |b| within 2^+-450 (binary64) or
// 2^+-50 (binary32); callers route other b to the generic division and the
// rare other a are handled here.
__device__ __forceinline__ bool div_operand_safe(double v)
{
    const unsigned hi = (unsigned)__double2hiint(v) & 0x7fffffffu;
    return hi - (573u << 20) < ((1474u - 573u) << 20);  // 2^-450 <= |v| < 2^451
}
__device__ __forceinline__ bool div_operand_safe(float v)
{
    const unsigned b = (unsigned)__float_as_int(v) & 0x7fffffffu;
    return b - (77u << 23) < ((178u - 77u) << 23);  // 2^-50 <= |v| < 2^51
}
__device__ __forceinline__ double rcp_rn(double v) { return __drcp_rn(v); }
__device__ __forceinline__ float rcp_rn(float v) { return __frcp_rn(v); }

template <typename T>
__device__ __forceinline__ T div_by_rcp(T a, T b, T y)
{
    T q = dmul(a, y);
    T e = dfma(-q, b, a);
    q = dfma(e, y, q);
    e = dfma(-q, b, a);
    q = dfma(e, y, q);
    if (!div_operand_safe(a)) q = (a == T(0)) ? dmul(a, y) : ddiv(a, b);  // rare, divergent
    return q;
}

// a / b (IEEE, round to nearest) for a dividend that is often exactly zero: a
// residual of a row that an accepted coordinate step put on its breakpoint.
// __ddiv_rn sends a zero dividend down its full-range slow path (a call of ~60
// instructions, and in SIMT every lane of the warp waits for it); 0 / b is the
// signed zero 0 * b for finite nonzero b, so zero dividends divide 1 instead
// and take 0 * b.  The dividend select is opaque to the compiler, which would
// otherwise notice that q is unused when a == 0 and divide a itself.
__device__ __forceinline__ double ddiv_zero_fast(double a, double b)
{
    const bool z = (a == 0.0);
    double d = z ? 1.0 : a;
    asm("" : "+d"(d));
    const double q = __ddiv_rn(d, b);
    return z ? __dmul_rn(a, b) : q;
}
__device__ __forceinline__ float ddiv_zero_fast(float a, float b) { return __fdiv_rn(a, b); }

template <typename T>
__device__ __forceinline__ T inf_of();
template <>
__device__ __forceinline__ double inf_of<double>() { return __longlong_as_double(0x7ff0000000000000LL); }
template <>
__device__ __forceinline__ float inf_of<float>() { return __int_as_float(0x7f800000); }

template <typename T>
struct vec2_of;
template <>
struct vec2_of<double> { using type = double2; };
template <>
struct vec2_of<float> { using type = float2; };

// numpy pairwise_sum (loops_utils.h.src) over n <= 128 values produced by f(i).
// n is a compile-time constant in the fast kernels, so the tree unrolls.
template <typename F>
__device__ __forceinline__ auto np_sum(int n, F f) -> decltype(f(0))
{
    using T = decltype(f(0));
    if (n < 8) {
        T res = T(0);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < n) res = dadd(res, f(i));
        return res;
    }
    T r0 = f(0), r1 = f(1), r2 = f(2), r3 = f(3), r4 = f(4), r5 = f(5), r6 = f(6), r7 = f(7);
    int lim = n - (n % 8);
    int i = 8;
#pragma unroll 1
    for (; i < lim; i += 8) {
        r0 = dadd(r0, f(i + 0)); r1 = dadd(r1, f(i + 1)); r2 = dadd(r2, f(i + 2)); r3 = dadd(r3, f(i + 3));
        r4 = dadd(r4, f(i + 4)); r5 = dadd(r5, f(i + 5)); r6 = dadd(r6, f(i + 6)); r7 = dadd(r7, f(i + 7));
    }
    T res = dadd(dadd(dadd(r0, r1), dadd(r2, r3)), dadd(dadd(r4, r5), dadd(r6, r7)));
#pragma unroll 1
    for (; i < n; ++i) res = dadd(res, f(i));
    return res;
}

// numpy pairwise_sum of f(off), ..., f(off + n - 1) (loops_utils.h.src), any n:
// blocked below 129 terms, recursion on halves split at a multiple of 8 above
// (iterative post-order walk of numpy's recursion tree: no device recursion / stack growth)
template <typename F>
__device__ double np_sum_rec(int off, int n, F f)
{
    if (n <= 128) return np_sum(n, [&](int i) { return f(off + i); });
    int fo[12], fn[12], fs[12];
    double fl[12];
    int sp = 0;
    fo[0] = off;
    fn[0] = n;
    fs[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        const int o = fo[sp], m = fn[sp];
        if (m <= 128) {
            ret = np_sum(m, [&](int i) { return f(o + i); });
            --sp;
            continue;
        }
        int m2 = m / 2;
        m2 -= m2 % 8;
        if (fs[sp] == 0) {  // left half first
            fs[sp] = 1;
            ++sp;
            fo[sp] = o;
            fn[sp] = m2;
            fs[sp] = 0;
        } else if (fs[sp] == 1) {  // then the right half
            fl[sp] = ret;
            fs[sp] = 2;
            ++sp;
            fo[sp] = o + m2;
            fn[sp] = m - m2;
            fs[sp] = 0;
        } else {
            ret = dadd(fl[sp], ret);
            --sp;
        }
    }
    return ret;
}

// Same tree with fully unrolled loops for a compile-time length N.
template <int N, typename F>
__device__ __forceinline__ auto np_sum_c(F f) -> decltype(f(0))
{
    using T = decltype(f(0));
    if constexpr (N < 8) {
        T res = T(0);
#pragma unroll
        for (int i = 0; i < N; ++i) res = dadd(res, f(i));
        return res;
    } else {
        T r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = f(j);
        constexpr int lim = N - (N % 8);
#pragma unroll
        for (int i = 8; i < lim; i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], f(i + j));
        T res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
#pragma unroll
        for (int i = lim; i < N; ++i) res = dadd(res, f(i));
        return res;
    }
}

// OpenBLAS ddot_k (SkylakeX) over n <= 47 terms x_i*y_i given by prod(i) (the
// rounded product) and the raw factors fx(i), fy(i) for the FMA tail.
template <typename FX, typename FY>
__device__ __forceinline__ double blas_ddot(int n, FX fx, FY fy)
{
    int n1 = n & -16;
    double dot = 0.0;
    if (n1 == 16) {
        double S[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            double p0 = dmul(fx(l), fy(l)), p4 = dmul(fx(l + 4), fy(l + 4));
            double p8 = dmul(fx(l + 8), fy(l + 8)), p12 = dmul(fx(l + 12), fy(l + 12));
            S[l] = dadd(dadd(dadd(p0, p4), p8), p12);
        }
        dot = dadd(dadd(S[0], S[2]), dadd(S[1], S[3]));
    } else if (n1 == 32) {
        double S[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            double A[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                A[k] = dadd(dmul(fx(8 * k + l), fy(8 * k + l)), dmul(fx(8 * k + l + 4), fy(8 * k + l + 4)));
            S[l] = dadd(dadd(dadd(A[0], A[1]), A[2]), A[3]);
        }
        dot = dadd(dadd(S[0], S[2]), dadd(S[1], S[3]));
    }
#pragma unroll 1
    for (int i = n1; i < n; ++i) dot = dfma(fx(i), fy(i), dot);
    return dot;
}

// Compile-time-length version (all branches resolved, tail unrolled).
template <int N, typename FX, typename FY>
__device__ __forceinline__ double blas_ddot_c(FX fx, FY fy)
{
    constexpr int n1 = N & -16;
    static_assert(n1 <= 32, "ddot model covers n <= 47");
    double dot = 0.0;
    if constexpr (n1 == 16) {
        double S[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            double p0 = dmul(fx(l), fy(l)), p4 = dmul(fx(l + 4), fy(l + 4));
            double p8 = dmul(fx(l + 8), fy(l + 8)), p12 = dmul(fx(l + 12), fy(l + 12));
            S[l] = dadd(dadd(dadd(p0, p4), p8), p12);
        }
        dot = dadd(dadd(S[0], S[2]), dadd(S[1], S[3]));
    } else if constexpr (n1 == 32) {
        double S[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            double A[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                A[k] = dadd(dmul(fx(8 * k + l), fy(8 * k + l)), dmul(fx(8 * k + l + 4), fy(8 * k + l + 4)));
            S[l] = dadd(dadd(dadd(A[0], A[1]), A[2]), A[3]);
        }
        dot = dadd(dadd(S[0], S[2]), dadd(S[1], S[3]));
    }
#pragma unroll
    for (int i = n1; i < N; ++i) dot = dfma(fx(i), fy(i), dot);
    return dot;
}

// One output of x @ b through OpenBLAS dgemv_t (SkylakeX), d <= 8; `row` and
// the row count m pick the 4x4 / 4x2 / 4x1 kernel for d == 8.  xr(j) reads x[row][j].
template <typename FXR, typename FB>
__device__ __forceinline__ auto gemv_row(int d, int row, int m, FXR xr, FB b) -> decltype(xr(0))
{
    using T = decltype(xr(0));
    int nb = d & -4, m3 = d & 3;
    T S = T(0);
    if (nb == 4) {
        T p0 = dmul(xr(0), b(0)), p1 = dmul(xr(1), b(1)), p2 = dmul(xr(2), b(2)), p3 = dmul(xr(3), b(3));
        S = dadd(dadd(p0, p2), dadd(p1, p3));
    } else if (nb == 8) {
        int g4 = 4 * (m >> 2);
        if (row < g4) {
            T q[4];
#pragma unroll
            for (int l = 0; l < 4; ++l) q[l] = dfma(xr(l + 4), b(l + 4), dmul(xr(l), b(l)));
            S = dadd(dadd(q[0], q[2]), dadd(q[1], q[3]));
        } else {
            T p[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = dmul(xr(j), b(j));
            if ((m & 2) && row < g4 + 2) {
                T L0 = dadd(dadd(dadd(p[0], p[2]), p[4]), p[6]);
                T L1 = dadd(dadd(dadd(p[1], p[3]), p[5]), p[7]);
                S = dadd(L0, L1);
            } else {
                S = dadd(dadd(dadd(p[0], p[4]), dadd(p[2], p[6])), dadd(dadd(p[1], p[5]), dadd(p[3], p[7])));
            }
        }
    }
    if (m3 == 1) {
        S = dfma(xr(nb), b(nb), S);
    } else if (m3 == 2) {
        S = dadd(S, dfma(xr(nb), b(nb), dmul(xr(nb + 1), b(nb + 1))));
    } else if (m3 == 3) {
        S = dadd(S, dfma(xr(nb + 2), b(nb + 2), dfma(xr(nb), b(nb), dmul(xr(nb + 1), b(nb + 1)))));
    }
    return S;
}

// ---------------------------------------------------------------------------
// PCG32, XSH-RR, stream 54 (rng.py:25-39); drives the dense-refine start fan.
// ---------------------------------------------------------------------------
struct Pcg32 {
    uint64_t state, inc;
    __host__ __device__ __forceinline__ uint32_t next()
    {
        uint64_t old = state;
        state = old * 6364136223846793005ULL + inc;
        uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
        uint32_t rot = (uint32_t)(old >> 59);
        return (xs >> rot) | (xs << ((32u - rot) & 31u));
    }
    __host__ __device__ __forceinline__ void seed(uint64_t s, uint64_t stream = 54)
    {
        state = 0;
        inc = (stream << 1) | 1u;
        next();
        state += s;
        next();
    }
};

}  // namespace lad
