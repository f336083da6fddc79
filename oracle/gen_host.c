/*
 * gen_host.c -- host restatement of the BASELINE config problem generator.
 *
 * TEST INFRASTRUCTURE ONLY (part of liboracle.so).  It restates the device
 * generator of paper_2510_15649_b200/csrc/lad_gen.cuh (Philox4x32-10 keyed by
 * (seed, problem index); Box-Muller / Laplace / Cauchy / Student-t(3)
 * transforms with that file's own log / sinpi / cospi polynomials; config-3
 * lexicographic subset unranking) operation for operation, so that
 *   - bench.py's reference arm (--impl reference) and cpu_baseline solve
 *     exactly the problems the GPU solves without loading the product library;
 *   - tests/golden/bench_cfg*.npz (the unmodified reference run on these
 *     problems, oracle/gen_golden.py) pin the bench's actual inputs.
 * The GPU test tests/test_gpu_generator.py asserts byte equality with
 * lad_generate_f64 / lad_subsets_f64.  The reference has no counterpart: its
 * datagen.py (datagen.py:63-80) cannot produce the BASELINE.json distributions
 * (SURVEY.md §8d).
 *
 * Build with -ffp-contract=off: every a*b+c below is two roundings unless it is
 * an explicit fma(), exactly as the device code (built with -fmad=false).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ---- transcendentals (identical polynomials and operation order to the device) ---- */

static double g_log_pos(double x)
{
    uint64_t b;
    memcpy(&b, &x, 8);
    int e = (int)(b >> 52) - 1023;
    uint64_t mb = (b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
    double m;
    memcpy(&m, &mb, 8);
    if (m > 0x1.6a09e667f3bcdp+0) {
        m = m * 0.5;
        e += 1;
    }
    double f = m - 1.0;
    double s = f / (2.0 + f);
    double z = s * s;
    static const double c[12] = {0x1.47ae147ae147bp-5, 0x1.642c8590b2164p-5, 0x1.8618618618618p-5,
                                 0x1.af286bca1af28p-5, 0x1.e1e1e1e1e1e1ep-5, 0x1.1111111111111p-4,
                                 0x1.3b13b13b13b14p-4, 0x1.745d1745d1746p-4, 0x1.c71c71c71c71cp-4,
                                 0x1.2492492492492p-3, 0x1.999999999999ap-3, 0x1.5555555555555p-2};
    double r = c[0];
    for (int k = 1; k < 12; ++k) r = fma(r, z, c[k]);
    r = r * z;
    double t = 2.0 * s;
    double lm = fma(t, r, t);
    double de = (double)e;
    return de * 0x1.62e42fee00000p-1 + (de * 0x1.a39ef35793c76p-33 + lm);
}

static double g_sinpi_red(double r)
{
    static const double c[10] = {-0x1.8a404211f9547p-26, 0x1.aaec32af93359p-21, -0x1.6fadb9f155744p-16,
                                 0x1.e8f434d018d63p-12,  -0x1.e3074fde8871fp-8, 0x1.50783487ee782p-4,
                                 -0x1.32d2cce62bd86p-1,  0x1.466bc6775aae2p+1,  -0x1.4abbce625be53p+2,
                                 0x1.921fb54442d18p+1};
    double z = r * r;
    double q = c[0];
    for (int k = 1; k < 10; ++k) q = fma(q, z, c[k]);
    return r * q;
}

static double g_cospi_red(double r)
{
    static const double c[10] = {0x1.ef6e308d6d1c4p-29, -0x1.2a0c591af8314p-23, 0x1.20c62c2f2d7f5p-18,
                                 -0x1.b6e24f44b128fp-14, 0x1.f9d38a3763cc3p-10, -0x1.a6d1f2a204a8cp-6,
                                 0x1.e1f506891babbp-3,  -0x1.55d3c7e3cbffap+0, 0x1.03c1f081b5ac4p+2,
                                 -0x1.3bd3cc9be45dep+2};
    double z = r * r;
    double q = c[0];
    for (int k = 1; k < 10; ++k) q = fma(q, z, c[k]);
    return fma(q, z, 1.0);
}

static double g_cospi_0_2(double x)
{
    double q = rint(x * 2.0);
    double r = x - q * 0.5;
    switch (((int)q) & 3) {
    case 0: return g_cospi_red(r);
    case 1: return -g_sinpi_red(r);
    case 2: return -g_cospi_red(r);
    default: return g_sinpi_red(r);
    }
}

static double g_tanpi_open(double w)
{
    double a = fabs(w), t;
    if (a <= 0.25) t = g_sinpi_red(a) / g_cospi_red(a);
    else {
        double v = 0.5 - a;
        t = g_cospi_red(v) / g_sinpi_red(v);
    }
    return w < 0.0 ? -t : t;
}

/* ---- Philox4x32-10 stream keyed by (seed, problem) ---- */

typedef struct {
    uint32_t k0, k1;
    uint64_t prob;
    uint32_t ctr;
    uint32_t buf[4];
    int avail;
} philox;

static void ph_init(philox *R, uint64_t seed, uint64_t problem)
{
    R->k0 = (uint32_t)seed;
    R->k1 = (uint32_t)(seed >> 32);
    R->prob = problem;
    R->ctr = 0;
    R->avail = 0;
}

static void ph_block(philox *R)
{
    uint32_t c0 = (uint32_t)R->prob, c1 = (uint32_t)(R->prob >> 32), c2 = R->ctr++, c3 = 0x4C414421u;
    uint32_t a0 = R->k0, a1 = R->k1;
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ a0, n1 = lo1, n2 = hi0 ^ c3 ^ a1, n3 = lo0;
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
        a0 += 0x9E3779B9u;
        a1 += 0xBB67AE85u;
    }
    R->buf[0] = c0;
    R->buf[1] = c1;
    R->buf[2] = c2;
    R->buf[3] = c3;
    R->avail = 4;
}

static uint32_t ph_u32(philox *R)
{
    if (R->avail == 0) ph_block(R);
    return R->buf[4 - R->avail--];
}

static double ph_uniform(philox *R)
{
    uint64_t hi = ph_u32(R), lo = ph_u32(R);
    uint64_t v = ((hi << 32) | lo) >> 11;
    return (double)v * 0x1.0p-53;
}

static double ph_uniform_open(philox *R)
{
    uint64_t hi = ph_u32(R), lo = ph_u32(R);
    uint64_t v = ((((hi << 32) | lo) >> 12) << 1) | 1u;
    return (double)v * 0x1.0p-53;
}

static double ph_normal(philox *R)
{
    double u1 = ph_uniform_open(R), u2 = ph_uniform(R);
    return sqrt(-2.0 * g_log_pos(u1)) * g_cospi_0_2(2.0 * u2);
}

static double ph_laplace(philox *R, double scale)
{
    double u = ph_uniform_open(R) - 0.5;
    double s = u < 0 ? -1.0 : 1.0;
    return -scale * s * g_log_pos(1.0 - 2.0 * fabs(u));
}

static double ph_cauchy(philox *R, double scale) { return scale * g_tanpi_open(ph_uniform_open(R) - 0.5); }

static double ph_student_t3(philox *R)
{
    double z = ph_normal(R);
    double a = ph_normal(R), b = ph_normal(R), c = ph_normal(R);
    return z / sqrt((a * a + b * b + c * c) / 3.0);
}

static uint32_t ph_below(philox *R, uint32_t bound)
{
    uint32_t threshold = (0u - bound) % bound;
    for (;;) {
        uint32_t r = ph_u32(R);
        if (r >= threshold) return r % bound;
    }
}

/* Problems [first, first + B) of BASELINE config 0, 1, 2 or 4 (lad_generate_f64). */
int orc_generate(int config, uint64_t seed, int64_t first, int64_t B, int n, int p, double *X, double *Y,
                 double *lam, double *beta_true)
{
    if (config < 0 || config > 4 || config == 3 || n < 1 || p < 1 || p > 8 || n > 64 || B < 0) return -1;
    for (int64_t t = 0; t < B; ++t) {
        philox R;
        ph_init(&R, seed, (uint64_t)(first + t));
        double *x = X + (size_t)t * n * p;
        double *y = Y + (size_t)t * n;
        double bt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (config == 1) {
            for (int k = 0; k < n * p; ++k) x[k] = -1.0 + 2.0 * ph_uniform(&R);
            for (int j = 0; j < p; ++j) bt[j] = ph_normal(&R);
        } else {
            int heavy = config == 4;
            for (int k = 0; k < n * p; ++k) x[k] = heavy ? ph_student_t3(&R) : ph_normal(&R);
            int nz = heavy ? 3 : 2;
            if (nz > p) nz = p;
            int perm[8];
            for (int j = 0; j < p; ++j) perm[j] = j;
            for (int q = 0; q < nz; ++q) {
                int r = q + (int)ph_below(&R, (uint32_t)(p - q));
                int tmp = perm[q];
                perm[q] = perm[r];
                perm[r] = tmp;
                double s = (ph_u32(&R) & 1u) ? 1.0 : -1.0;
                bt[perm[q]] = s * (1.0 + 2.0 * ph_uniform(&R));
            }
        }
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int j = 0; j < p; ++j) s += x[i * p + j] * bt[j];
            double e;
            if (config == 1) e = ph_laplace(&R, 0.3);
            else if (config == 4) e = ph_cauchy(&R, 0.2);
            else e = ph_laplace(&R, 0.5);
            y[i] = s + e;
        }
        if (config == 0 || config == 2) {
            int nout = (n + 5) / 10;
            int rows[64];
            for (int i = 0; i < n; ++i) rows[i] = i;
            for (int q = 0; q < nout && q < n; ++q) {
                int r = q + (int)ph_below(&R, (uint32_t)(n - q));
                int tmp = rows[q];
                rows[q] = rows[r];
                rows[r] = tmp;
                y[rows[q]] += (ph_u32(&R) & 1u) ? 10.0 : -10.0;
            }
        }
        if (lam) lam[t] = config == 1 ? 0.1 + 1.9 * ph_uniform(&R) : 1.0;
        if (beta_true)
            for (int j = 0; j < p; ++j) beta_true[(size_t)t * p + j] = bt[j];
    }
    return 0;
}

static int64_t binom(int nn, int kk)
{
    if (kk < 0 || kk > nn) return 0;
    int k2 = kk > nn - kk ? nn - kk : kk;
    int64_t c = 1;
    for (int q = 1; q <= k2; ++q) c = c * (nn - k2 + q) / q;
    return c;
}

/* Config 3: subsets [first, first + B) of `keep` rows out of n0, in
 * itertools.combinations (lexicographic) order (lad_subsets_f64). */
int orc_subsets(const double *X0, const double *Y0, int n0, int p, int keep, int64_t first, int64_t B, double *X,
                double *Y)
{
    if (keep < 1 || keep > n0 || n0 > 64 || p < 1 || B < 0) return -1;
    for (int64_t t = 0; t < B; ++t) {
        int64_t r = first + t;
        int x = 0;
        for (int i = 0; i < keep; ++i) {
            for (;;) {
                int64_t cnt = binom(n0 - 1 - x, keep - 1 - i);
                if (r < cnt) break;
                r -= cnt;
                ++x;
            }
            for (int j = 0; j < p; ++j) X[((size_t)t * keep + i) * p + j] = X0[x * p + j];
            Y[(size_t)t * keep + i] = Y0[x];
            ++x;
        }
    }
    return 0;
}
