// lad_gen.cuh -- on-device generation of the BASELINE.json config problems.
//
// The reference's datagen.py cannot produce these distributions (SURVEY.md
// §8d), and at config 4 scale (64M problems, ~127 GB of fp64 X) the inputs
// must be generated where they are solved.  Problem i of a config draws from a
// counter-based Philox4x32-10 stream keyed by (seed, i), so any index shard is
// reproducible on any GPU without communication.
//
// Host reproducibility: every floating-point operation below is a single IEEE
// operation (+, -, *, /, sqrt, explicit fma; the library builds with
// -fmad=false so nothing is contracted), and the transcendentals (log, sinpi,
// cospi, tan) are this file's own polynomials instead of libdevice's.  A plain
// C restatement (oracle/gen_host.c, built with -ffp-contract=off) therefore
// produces the same bytes on the CPU, which is how the CPU reference arm and
// the reference-held goldens (tests/golden/bench_cfg*.npz) see exactly the
// problems the GPU solves without loading this library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lad {
namespace genmath {

// natural log for finite x > 0 (normal range): x = 2^e m, m in [sqrt(1/2), sqrt(2)),
// log m = 2 atanh(s), s = (m - 1)/(m + 1), atanh series to s^25 (|s| <= 0.1716)
__device__ __forceinline__ double log_pos(double x)
{
    uint64_t b = (uint64_t)__double_as_longlong(x);
    int e = (int)(b >> 52) - 1023;
    double m = __longlong_as_double((long long)((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
    if (m > 0x1.6a09e667f3bcdp+0) {
        m = m * 0.5;
        e += 1;
    }
    double f = m - 1.0;
    double s = f / (2.0 + f);
    double z = s * s;
    double r = 0x1.47ae147ae147bp-5;
    r = fma(r, z, 0x1.642c8590b2164p-5);
    r = fma(r, z, 0x1.8618618618618p-5);
    r = fma(r, z, 0x1.af286bca1af28p-5);
    r = fma(r, z, 0x1.e1e1e1e1e1e1ep-5);
    r = fma(r, z, 0x1.1111111111111p-4);
    r = fma(r, z, 0x1.3b13b13b13b14p-4);
    r = fma(r, z, 0x1.745d1745d1746p-4);
    r = fma(r, z, 0x1.c71c71c71c71cp-4);
    r = fma(r, z, 0x1.2492492492492p-3);
    r = fma(r, z, 0x1.999999999999ap-3);
    r = fma(r, z, 0x1.5555555555555p-2);
    r = r * z;
    double t = 2.0 * s;
    double lm = fma(t, r, t);
    double de = (double)e;
    return de * 0x1.62e42fee00000p-1 + (de * 0x1.a39ef35793c76p-33 + lm);  // ln2 split (hi has 32 bits)
}

// sin(pi r), cos(pi r) for |r| <= 1/4: Taylor polynomials in r^2 (|pi r| <= 0.7854)
__device__ __forceinline__ double sinpi_red(double r)
{
    double z = r * r;
    double q = -0x1.8a404211f9547p-26;
    q = fma(q, z, 0x1.aaec32af93359p-21);
    q = fma(q, z, -0x1.6fadb9f155744p-16);
    q = fma(q, z, 0x1.e8f434d018d63p-12);
    q = fma(q, z, -0x1.e3074fde8871fp-8);
    q = fma(q, z, 0x1.50783487ee782p-4);
    q = fma(q, z, -0x1.32d2cce62bd86p-1);
    q = fma(q, z, 0x1.466bc6775aae2p+1);
    q = fma(q, z, -0x1.4abbce625be53p+2);
    q = fma(q, z, 0x1.921fb54442d18p+1);
    return r * q;
}

__device__ __forceinline__ double cospi_red(double r)
{
    double z = r * r;
    double q = 0x1.ef6e308d6d1c4p-29;
    q = fma(q, z, -0x1.2a0c591af8314p-23);
    q = fma(q, z, 0x1.20c62c2f2d7f5p-18);
    q = fma(q, z, -0x1.b6e24f44b128fp-14);
    q = fma(q, z, 0x1.f9d38a3763cc3p-10);
    q = fma(q, z, -0x1.a6d1f2a204a8cp-6);
    q = fma(q, z, 0x1.e1f506891babbp-3);
    q = fma(q, z, -0x1.55d3c7e3cbffap+0);
    q = fma(q, z, 0x1.03c1f081b5ac4p+2);
    q = fma(q, z, -0x1.3bd3cc9be45dep+2);
    return fma(q, z, 1.0);
}

// cos(pi x) for x in [0, 2): quarter-turn reduction (exact: x is a multiple of 2^-52)
__device__ __forceinline__ double cospi_0_2(double x)
{
    double q = rint(x * 2.0);
    double r = x - q * 0.5;
    switch (((int)q) & 3) {
    case 0: return cospi_red(r);
    case 1: return -sinpi_red(r);
    case 2: return -cospi_red(r);
    default: return sinpi_red(r);
    }
}

// tan(pi w) for w in (-1/2, 1/2), w != +-1/2
__device__ __forceinline__ double tanpi_open(double w)
{
    double a = fabs(w);
    double t;
    if (a <= 0.25) t = sinpi_red(a) / cospi_red(a);
    else {
        double v = 0.5 - a;  // exact (Sterbenz)
        t = cospi_red(v) / sinpi_red(v);
    }
    return w < 0.0 ? -t : t;
}

}  // namespace genmath

struct Philox {
    uint32_t k0, k1;
    uint64_t prob;
    uint32_t ctr;
    uint32_t buf[4];
    int avail;

    __device__ __forceinline__ void init(uint64_t seed, uint64_t problem)
    {
        k0 = (uint32_t)seed;
        k1 = (uint32_t)(seed >> 32);
        prob = problem;
        ctr = 0;
        avail = 0;
    }
    __device__ __forceinline__ void block()
    {
        uint32_t c0 = (uint32_t)prob, c1 = (uint32_t)(prob >> 32), c2 = ctr++, c3 = 0x4C414421u;
        uint32_t a0 = k0, a1 = k1;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
            uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
            uint32_t n0 = hi1 ^ c1 ^ a0, n1 = lo1, n2 = hi0 ^ c3 ^ a1, n3 = lo0;
            c0 = n0; c1 = n1; c2 = n2; c3 = n3;
            a0 += 0x9E3779B9u;
            a1 += 0xBB67AE85u;
        }
        buf[0] = c0; buf[1] = c1; buf[2] = c2; buf[3] = c3;
        avail = 4;
    }
    __device__ __forceinline__ uint32_t u32()
    {
        if (avail == 0) block();
        return buf[4 - avail--];
    }
    // [0, 1) with 53 random bits
    __device__ __forceinline__ double uniform()
    {
        uint64_t hi = u32(), lo = u32();
        uint64_t v = ((hi << 32) | lo) >> 11;
        return (double)v * 0x1.0p-53;
    }
    // (0, 1): an odd 53-bit integer times 2^-53 (exact; never 0, 1/2 or 1)
    __device__ __forceinline__ double uniform_open()
    {
        uint64_t hi = u32(), lo = u32();
        uint64_t v = ((((hi << 32) | lo) >> 12) << 1) | 1u;
        return (double)v * 0x1.0p-53;
    }
    // Box-Muller (cosine branch)
    __device__ __forceinline__ double normal()
    {
        double u1 = uniform_open(), u2 = uniform();
        return sqrt(-2.0 * genmath::log_pos(u1)) * genmath::cospi_0_2(2.0 * u2);
    }
    __device__ __forceinline__ double laplace(double scale)
    {
        double u = uniform_open() - 0.5;  // exact, nonzero
        double s = u < 0 ? -1.0 : 1.0;
        return -scale * s * genmath::log_pos(1.0 - 2.0 * fabs(u));
    }
    __device__ __forceinline__ double cauchy(double scale)
    {
        return scale * genmath::tanpi_open(uniform_open() - 0.5);
    }
    __device__ __forceinline__ double student_t3()
    {
        double z = normal();
        double a = normal(), b = normal(), c = normal();
        return z / sqrt((a * a + b * b + c * c) / 3.0);
    }
    __device__ __forceinline__ uint32_t below(uint32_t bound)
    {
        uint32_t threshold = (0u - bound) % bound;
        for (;;) {
            uint32_t r = u32();
            if (r >= threshold) return r % bound;
        }
    }
};

struct GenArgs {
    int config;
    uint64_t seed;
    int64_t first, B;
    int n, p;
    double *X, *Y, *lam, *beta_true;
};

__global__ void gen_kernel(GenArgs G)
{
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= G.B) return;
    const int n = G.n, p = G.p;
    Philox R;
    R.init(G.seed, (uint64_t)(G.first + t));
    double *x = G.X + (size_t)t * n * p;
    double *y = G.Y + (size_t)t * n;
    double bt[8];
    for (int j = 0; j < 8; ++j) bt[j] = 0.0;
    if (G.config == 1) {
        for (int k = 0; k < n * p; ++k) x[k] = -1.0 + 2.0 * R.uniform();
        for (int j = 0; j < p && j < 8; ++j) bt[j] = R.normal();
    } else {
        bool heavy = G.config == 4;
        for (int k = 0; k < n * p; ++k) x[k] = heavy ? R.student_t3() : R.normal();
        int nz = heavy ? 3 : 2;
        if (nz > p) nz = p;
        int perm[8];
        for (int j = 0; j < p && j < 8; ++j) perm[j] = j;
        for (int q = 0; q < nz; ++q) {  // partial Fisher-Yates: distinct positions
            int r = q + (int)R.below((uint32_t)(p - q));
            int tmp = perm[q];
            perm[q] = perm[r];
            perm[r] = tmp;
            double s = (R.u32() & 1u) ? 1.0 : -1.0;
            bt[perm[q]] = s * (1.0 + 2.0 * R.uniform());
        }
    }
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < p && j < 8; ++j) s += x[i * p + j] * bt[j];
        double e;
        if (G.config == 1) e = R.laplace(0.3);
        else if (G.config == 4) e = R.cauchy(0.2);
        else e = R.laplace(0.5);
        y[i] = s + e;
    }
    if (G.config == 0 || G.config == 2) {  // 10% of rows get y += +-10
        int nout = (n + 5) / 10;
        int rows[64];
        for (int i = 0; i < n && i < 64; ++i) rows[i] = i;
        for (int q = 0; q < nout && q < n; ++q) {
            int r = q + (int)R.below((uint32_t)(n - q));
            int tmp = rows[q];
            rows[q] = rows[r];
            rows[r] = tmp;
            y[rows[q]] += (R.u32() & 1u) ? 10.0 : -10.0;
        }
    }
    if (G.lam) G.lam[t] = G.config == 1 ? 0.1 + 1.9 * R.uniform() : 1.0;
    if (G.beta_true)
        for (int j = 0; j < p && j < 8; ++j) G.beta_true[(size_t)t * p + j] = bt[j];
}

// k-th keep-subset of n0 rows, lexicographic order (itertools.combinations)
__global__ void subsets_kernel(const double *X0, const double *Y0, int n0, int p, int keep, int64_t first, int64_t B,
                               double *X, double *Y)
{
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= B) return;
    int64_t r = first + t;
    int x = 0;
    double *xo = X + (size_t)t * keep * p;
    double *yo = Y + (size_t)t * keep;
    for (int i = 0; i < keep; ++i) {
        for (;;) {
            // number of combinations with element x at position i
            int nn = n0 - 1 - x, kk = keep - 1 - i;
            int64_t cnt = 1;
            if (kk < 0 || kk > nn) cnt = 0;
            else {
                int k2 = kk > nn - kk ? nn - kk : kk;
                for (int q = 1; q <= k2; ++q) cnt = cnt * (nn - k2 + q) / q;
            }
            if (r < cnt) break;
            r -= cnt;
            ++x;
        }
        for (int j = 0; j < p; ++j) xo[i * p + j] = X0[x * p + j];
        yo[i] = Y0[x];
        ++x;
    }
}

}  // namespace lad
