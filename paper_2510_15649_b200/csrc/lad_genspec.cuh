// lad_genspec.cuh -- the reference's GenSpec generator on the device (datagen.py:63-80, rng.py:25-72).
//
// One thread per problem.  PCG32 (XSH-RR, stream 54, the reference's two-step seeding),
// Box-Muller normals served cos-then-sin with the spare kept across phases, informative
// coefficients U[1, 10] as a + (b - a) u, m noise normals scaled by sigma, outlier rows
// by rejection until distinct, y = x @ beta (OpenBLAS dgemv_t order, gemv_row) + noise.
//
// Python's math.log / math.sin / math.cos are glibc's, not libdevice's.  Here they are
// evaluated in double-double arithmetic (~1e-30 relative) and rounded once: correctly
// rounded (0 of 600,000 Box-Muller inputs differ from mpmath).  glibc 2.39 itself is not
// correctly rounded on ~0.1% of these inputs, so a normal draw (rho * cos) can differ from
// the reference's by up to 2 ulp; most problems are bit-identical.  tests/test_gpu_genspec.py
// measures the agreement with synth.generate and the reference's own generated inputs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lad_numerics.cuh"

namespace lad {
namespace dd {

struct D2 {
    double hi, lo;
};

__device__ __forceinline__ D2 two_sum(double a, double b)
{
    double s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ D2 quick_two_sum(double a, double b)
{
    double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ D2 two_prod(double a, double b)
{
    double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ D2 add(D2 a, D2 b)
{
    D2 s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ D2 neg(D2 a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ D2 mul(D2 a, D2 b)
{
    D2 p = two_prod(a.hi, b.hi);
    p.lo = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ D2 mul_d(D2 a, double b)
{
    D2 p = two_prod(a.hi, b);
    p.lo = __fma_rn(a.lo, b, p.lo);
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ D2 div(D2 a, D2 b)
{
    double q1 = __ddiv_rn(a.hi, b.hi);
    D2 r = add(a, neg(mul_d(b, q1)));
    double q2 = __ddiv_rn(r.hi, b.hi);
    r = add(r, neg(mul_d(b, q2)));
    double q3 = __ddiv_rn(r.hi, b.hi);
    D2 q = quick_two_sum(q1, q2);
    return add(q, D2{q3, 0.0});
}

// natural log of a positive normal double, rounded once from ~1e-30 relative accuracy
__device__ __forceinline__ double log_cr(double x)
{
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    int e = (int)(b >> 52) - 1023;
    double m = __longlong_as_double((long long)((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
    if (m > 0x1.6a09e667f3bcdp+0) {
        m = m * 0.5;
        e += 1;
    }
    const double f = m - 1.0;  // exact
    const D2 s = div(D2{f, 0.0}, two_sum(2.0, f));
    const D2 z = mul(s, s);
    // Q(z) = sum_k z^k / (2k + 3), k = 0..21 (|z| <= 0.0295: remainder < 1e-33)
    static constexpr double C[22][2] = {
        {0x1.5555555555555p-2, 0x1.5555555555555p-56}, {0x1.999999999999ap-3, -0x1.999999999999ap-57},
        {0x1.2492492492492p-3, 0x1.2492492492492p-57}, {0x1.c71c71c71c71cp-4, 0x1.c71c71c71c71cp-58},
        {0x1.745d1745d1746p-4, -0x1.745d1745d1746p-59}, {0x1.3b13b13b13b14p-4, -0x1.3b13b13b13b14p-58},
        {0x1.1111111111111p-4, 0x1.1111111111111p-60}, {0x1.e1e1e1e1e1e1ep-5, 0x1.e1e1e1e1e1e1ep-61},
        {0x1.af286bca1af28p-5, 0x1.af286bca1af28p-59}, {0x1.8618618618618p-5, 0x1.8618618618618p-59},
        {0x1.642c8590b2164p-5, 0x1.642c8590b2164p-60}, {0x1.47ae147ae147bp-5, -0x1.eb851eb851eb8p-61},
        {0x1.2f684bda12f68p-5, 0x1.2f684bda12f68p-59}, {0x1.1a7b9611a7b96p-5, 0x1.1a7b9611a7b96p-61},
        {0x1.0842108421084p-5, 0x1.0842108421084p-60}, {0x1.f07c1f07c1f08p-6, -0x1.f07c1f07c1f08p-61},
        {0x1.d41d41d41d41dp-6, 0x1.0750750750750p-60}, {0x1.bacf914c1bad0p-6, -0x1.bacf914c1bad0p-60},
        {0x1.a41a41a41a41ap-6, 0x1.0690690690690p-60}, {0x1.8f9c18f9c18fap-6, -0x1.f3831f3831f38p-61},
        {0x1.7d05f417d05f4p-6, 0x1.7d05f417d05f4p-62}, {0x1.6c16c16c16c17p-6, -0x1.f49f49f49f49fp-61}};
    D2 q = {C[21][0], C[21][1]};
    for (int k = 20; k >= 0; --k) q = add(mul(q, z), D2{C[k][0], C[k][1]});
    // log m = 2 s (1 + z Q)
    const D2 lm = mul_d(mul(s, add(D2{1.0, 0.0}, mul(z, q))), 2.0);
    // + e ln2 (ln2 in three parts; e ln2 exact to ~1e-33)
    const double de = (double)e;
    D2 el = two_prod(de, 0x1.62e42fefa39efp-1);
    el = add(el, two_prod(de, 0x1.abc9e3b39803fp-56));
    el = add(el, D2{de * 0x1.7b57a079a1934p-111, 0.0});
    const D2 r = add(el, lm);
    return __dadd_rn(r.hi, r.lo);
}

// sin and cos of a double theta in [0, 8) (Box-Muller's 2 pi u), each rounded once
__device__ __forceinline__ void sincos_cr(double th, double &sn, double &cs)
{
    const double k = rint(th * 0x1.45f306dc9c883p-1);  // nearest multiple of pi/2
    // r = th - k pi/2 in double-double (pi/2 in three parts; k <= 5 so each product is exact in D2)
    D2 r = add(D2{th, 0.0}, neg(two_prod(k, 0x1.921fb54442d18p+0)));
    r = add(r, neg(two_prod(k, 0x1.1a62633145c07p-54)));
    r = add(r, D2{-(k * -0x1.f1976b7ed8fbcp-110), 0.0});
    const D2 z = mul(r, r);
    static constexpr double S[14][2] = {
        {0x1.0000000000000p+0, 0.0}, {-0x1.5555555555555p-3, -0x1.5555555555555p-57},
        {0x1.1111111111111p-7, 0x1.1111111111111p-63}, {-0x1.a01a01a01a01ap-13, -0x1.a01a01a01a01ap-73},
        {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73}, {-0x1.ae64567f544e4p-26, 0x1.c062e06d1f209p-80},
        {0x1.6124613a86d09p-33, 0x1.f28e0cc748ebep-87}, {-0x1.ae7f3e733b81fp-41, -0x1.1d8656b0ee8cbp-97},
        {0x1.952c77030ad4ap-49, 0x1.ac981465ddc6cp-103}, {-0x1.2f49b46814157p-57, -0x1.2650f61dbdcb4p-112},
        {0x1.71b8ef6dcf572p-66, -0x1.d043ae40c4647p-120}, {-0x1.761b41316381ap-75, 0x1.3423c7d91404fp-130},
        {0x1.3f3ccdd165fa9p-84, -0x1.58ddadf344487p-139}, {-0x1.d1ab1c2dccea3p-94, -0x1.054d0c78aea14p-149}};
    static constexpr double Cc[14][2] = {
        {0x1.0000000000000p+0, 0.0}, {-0x1.0000000000000p-1, 0.0},
        {0x1.5555555555555p-5, 0x1.5555555555555p-59}, {-0x1.6c16c16c16c17p-10, 0x1.f49f49f49f49fp-65},
        {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76}, {-0x1.27e4fb7789f5cp-22, -0x1.cbbc05b4fa99ap-76},
        {0x1.1eed8eff8d898p-29, -0x1.2aec959e14c06p-83}, {-0x1.93974a8c07c9dp-37, -0x1.05d6f8a2efd1fp-92},
        {0x1.ae7f3e733b81fp-45, 0x1.1d8656b0ee8cbp-101}, {-0x1.6827863b97d97p-53, -0x1.eec01221a8b0bp-107},
        {0x1.e542ba4020225p-62, 0x1.ea72b4afe3c2fp-120}, {-0x1.0ce396db7f853p-70, 0x1.aebcdbd20331cp-124},
        {0x1.f2cf01972f578p-80, -0x1.9ada5fcc1ab14p-135}, {-0x1.88e85fc6a4e5ap-89, 0x1.71c37ebd16540p-143}};
    D2 ps = {S[13][0], S[13][1]}, pc = {Cc[13][0], Cc[13][1]};
    for (int i = 12; i >= 0; --i) {
        ps = add(mul(ps, z), D2{S[i][0], S[i][1]});
        pc = add(mul(pc, z), D2{Cc[i][0], Cc[i][1]});
    }
    const D2 sr = mul(ps, r);
    const double s1 = __dadd_rn(sr.hi, sr.lo), c1 = __dadd_rn(pc.hi, pc.lo);
    switch (((int)k) & 3) {
    case 0: sn = s1; cs = c1; break;
    case 1: sn = c1; cs = -s1; break;
    case 2: sn = -s1; cs = -c1; break;
    default: sn = -c1; cs = s1; break;
    }
}

}  // namespace dd

// PCG32 with the reference's sampling conventions (rng.py:25-72)
struct RefPcg32 {
    uint64_t state, inc;
    double spare;
    bool has_spare;
    __device__ __forceinline__ uint32_t step()
    {
        const uint64_t s = state;
        state = s * 6364136223846793005ull + inc;
        const uint32_t word = (uint32_t)(((s >> 18) ^ s) >> 27);
        const uint32_t rot = (uint32_t)(s >> 59);
        return (word >> rot) | (word << ((32u - rot) & 31u));
    }
    __device__ __forceinline__ void seed(uint64_t sd, uint64_t stream = 54)
    {
        inc = (stream << 1) | 1u;
        state = 0;
        step();
        state += sd;
        step();
        has_spare = false;
    }
    __device__ __forceinline__ double uniform() { return (double)step() * 0x1.0p-32; }
    __device__ __forceinline__ uint32_t below(uint32_t bound)
    {
        const uint32_t reject = (uint32_t)((1ull << 32) % bound);
        uint32_t r = step();
        while (r < reject) r = step();
        return r % bound;
    }
    __device__ __forceinline__ double normal()
    {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        const double u_open = (double)((uint64_t)step() + 1u) * 0x1.0p-32;  // (0, 1]
        const double u_half = (double)step() * 0x1.0p-32;                   // [0, 1)
        const double rho = __dsqrt_rn(__dmul_rn(-2.0, dd::log_cr(u_open)));
        const double theta = __dmul_rn(0x1.921fb54442d18p+2, u_half);    // 2.0 * math.pi * u
        double sn, cs;
        dd::sincos_cr(theta, sn, cs);
        spare = __dmul_rn(rho, sn);
        has_spare = true;
        return __dmul_rn(rho, cs);
    }
};

struct GenSpecArgs {
    int64_t B;
    int m, d, n_informative, n_outliers;
    const double *truth;  // (d,) or null: U[1, 10] on the informative axes
    double noise_sigma, outlier_scale;
    const uint64_t *seeds;
    double *X, *Y, *beta_true;
};

__global__ void genspec_kernel(GenSpecArgs G)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= G.B) return;
    const int m = G.m, d = G.d;
    RefPcg32 R;
    R.seed(G.seeds[t]);
    double *x = G.X + (size_t)t * m * d;
    double *y = G.Y + (size_t)t * m;
    for (int k = 0; k < m * d; ++k) x[k] = R.normal();
    double b[8];
    for (int j = 0; j < d; ++j) b[j] = 0.0;
    if (G.truth) {
        for (int j = 0; j < d; ++j) b[j] = G.truth[j];
    } else {
        for (int j = 0; j < G.n_informative; ++j) b[j] = __dadd_rn(1.0, __dmul_rn(9.0, R.uniform()));
    }
    // noise (drawn even when sigma is 0) into y, scaled; outlier rows by rejection until distinct
    for (int i = 0; i < m; ++i) y[i] = __dmul_rn(R.normal(), G.noise_sigma);
    uint32_t chosen[32];  // m <= 1024
    for (int w = 0; w < 32; ++w) chosen[w] = 0;
    int have = 0;
    while (have < G.n_outliers) {
        const uint32_t r = R.below((uint32_t)m);
        const uint32_t bit = 1u << (r & 31);
        if (!(chosen[r >> 5] & bit)) {
            chosen[r >> 5] |= bit;
            ++have;
            y[r] = __dmul_rn(y[r], G.outlier_scale);
        }
    }
    for (int i = 0; i < m; ++i) {
        const double g = gemv_row(d, i, m, [&](int q) { return x[i * d + q]; }, [&](int q) { return b[q < d ? q : 0]; });
        y[i] = __dadd_rn(g, y[i]);
    }
    if (G.beta_true)
        for (int j = 0; j < d; ++j) G.beta_true[(size_t)t * d + j] = b[j];
}

}  // namespace lad
