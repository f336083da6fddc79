// lad_brute.cuh -- exhaustive vertex evaluation (brute.py:29-145 restated).
//
// Every d-subset of the m+d planes [X; I_d] (lexicographic
// itertools.combinations order) is solved by Gaussian elimination with scaled
// partial pivoting (brute.py:29-59, same operation order, singular when the
// pivot <= 1e-12 * row norm), the objective is evaluated with the reference's
// reduction orders, and the minimum under the key (objective, sum|beta|,
// beta lexicographic) is kept (brute.py:125-133).  That key is a total order,
// so the result is independent of how subsets are partitioned across threads.
//
// Two schedules:
//   brute_thread_kernel   one thread per problem (small C(m+d, d), config 1)
//   brute_chunk_kernel    one block per (problem, subset range), partial keys
//                         reduced by brute_reduce_kernel (configs 0/2/3)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lad_numerics.cuh"

namespace lad {

struct BruteKey {
    double obj, l1;
    double v[8];
    int have;
};

template <int P>
__device__ __forceinline__ bool key_less(const BruteKey &a, const BruteKey &b)
{
    if (!b.have) return a.have;
    if (!a.have) return false;
    if (a.obj < b.obj) return true;
    if (a.obj > b.obj) return false;
    if (a.l1 < b.l1) return true;
    if (a.l1 > b.l1) return false;
#pragma unroll
    for (int c = 0; c < P; ++c) {
        if (a.v[c] < b.v[c]) return true;
        if (a.v[c] > b.v[c]) return false;
    }
    return false;
}

__host__ __device__ inline int64_t binom(int n, int k)
{
    if (k < 0 || k > n) return 0;
    if (k > n - k) k = n - k;
    int64_t r = 1;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

// combination of rank r (lexicographic) of P elements from N
template <int P>
__device__ __forceinline__ void unrank(int64_t r, int N, int (&c)[P])
{
    int x = 0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        for (;;) {
            int64_t cnt = binom(N - 1 - x, P - 1 - i);
            if (r < cnt) break;
            r -= cnt;
            ++x;
        }
        c[i] = x;
        ++x;
    }
}

template <int P>
__device__ __forceinline__ bool next_comb(int N, int (&c)[P])
{
    int i = P - 1;
#pragma unroll
    for (int q = P - 1; q >= 0; --q) {
        if (i == q && c[q] == N - P + q) --i;
    }
    if (i < 0) return false;
    int base = 0;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        if (q == i) {
            c[q] += 1;
            base = c[q];
        } else if (q > i) {
            base += 1;
            c[q] = base;
        }
    }
    return true;
}

// solve_linear_system (brute.py:29-59) on a PxP system held in registers.
template <int P>
__device__ __forceinline__ bool solve_ge(double (&a)[P][P], double (&b)[P], double (&sol)[P])
{
    double rn[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
        double mx = fabs(a[i][0]);
#pragma unroll
        for (int c = 1; c < P; ++c) mx = fabs(a[i][c]) > mx ? fabs(a[i][c]) : mx;
        rn[i] = mx;
    }
    bool ok = true;
#pragma unroll
    for (int i = 0; i < P; ++i) ok = ok && (rn[i] != 0.0);
    if (!ok) return false;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        int pv = k;
        double best = ddiv(fabs(a[k][k]), rn[k]);
#pragma unroll
        for (int i = k + 1; i < P; ++i) {
            double s = ddiv(fabs(a[i][k]), rn[i]);
            if (s > best) {
                best = s;
                pv = i;
            }
        }
        double apk = a[k][k], rnp = rn[k];
#pragma unroll
        for (int i = k + 1; i < P; ++i)
            if (i == pv) {
                apk = a[i][k];
                rnp = rn[i];
            }
        if (fabs(apk) <= dmul(1e-12, rnp)) return false;
        // swap rows k and pv
#pragma unroll
        for (int i = k + 1; i < P; ++i) {
            if (i == pv) {
#pragma unroll
                for (int c = 0; c < P; ++c) {
                    double t = a[k][c];
                    a[k][c] = a[i][c];
                    a[i][c] = t;
                }
                double t = b[k];
                b[k] = b[i];
                b[i] = t;
                t = rn[k];
                rn[k] = rn[i];
                rn[i] = t;
            }
        }
        double f[P];
#pragma unroll
        for (int i = k + 1; i < P; ++i) f[i] = ddiv(a[i][k], a[k][k]);
#pragma unroll
        for (int i = k + 1; i < P; ++i)
#pragma unroll
            for (int c = k; c < P; ++c) a[i][c] = dsub(a[i][c], dmul(f[i], a[k][c]));
#pragma unroll
        for (int i = k + 1; i < P; ++i) b[i] = dsub(b[i], dmul(f[i], b[k]));
    }
#pragma unroll
    for (int k = P - 1; k >= 0; --k) {
        // a[k, k+1:] @ sol[k+1:]: ddot of length < 16 -> FMA chain from 0
        double dot = 0.0;
#pragma unroll
        for (int c = k + 1; c < P; ++c) dot = dfma(a[k][c], sol[c], dot);
        sol[k] = ddiv(dsub(b[k], dot), a[k][k]);
    }
    return true;
}

// evaluate one vertex (subset c of planes) and fold it into `best`
template <int P, typename FX, typename FY>
__device__ __forceinline__ bool eval_vertex(const int (&c)[P], int m, double lam, FX xat, FY yat, BruteKey &best)
{
    double a[P][P], b[P], sol[P];
#pragma unroll
    for (int r = 0; r < P; ++r) {
        int pl = c[r];
#pragma unroll
        for (int q = 0; q < P; ++q) a[r][q] = pl < m ? xat(pl, q) : ((pl - m) == q ? 1.0 : 0.0);
        b[r] = pl < m ? yat(pl) : 0.0;
    }
    if (!solve_ge<P>(a, b, sol)) return false;
    double rs = np_sum(m, [&](int i) {  // m <= 64 here (lad_brute_solve_f64)
        double g = gemv_row(P, i, m, [&](int q) { return xat(i, q); }, [&](int q) { return sol[q < P ? q : P - 1]; });
        return fabs(dsub(yat(i), g));
    });
    double l1 = np_sum_c<P>([&](int q) { return fabs(sol[q]); });
    double obj = dadd(rs, dmul(lam, l1));
    if (best.have && obj > best.obj) return true;
    BruteKey k;
    k.obj = obj;
    k.l1 = l1;
#pragma unroll
    for (int q = 0; q < P; ++q) k.v[q] = sol[q];
    k.have = 1;
    if (key_less<P>(k, best)) best = k;
    return true;
}

struct BruteArgs {
    const double *X, *Y, *lam;
    int64_t B;
    int n;
    double lambda_floor;
    int64_t C;           // candidates per problem
    int64_t chunk;       // candidates per block (chunk kernel)
    int64_t nchunks;     // chunks per problem
    double *beta, *objective;
    int64_t *vertices;
    BruteKey *partial;           // (B * nchunks)
    unsigned long long *pcount;  // (B * nchunks)
};

template <int P>
__global__ void brute_thread_kernel(BruteArgs A)
{
    int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pr >= A.B) return;
    const int m = A.n;
    const double *x = A.X + (size_t)pr * m * P;
    const double *y = A.Y + (size_t)pr * m;
    double lr = A.lam[pr];
    double lam = lr > A.lambda_floor ? lr : A.lambda_floor;
    auto xat = [&](int i, int q) { return __ldg(x + i * P + q); };
    auto yat = [&](int i) { return __ldg(y + i); };
    BruteKey best;
    best.have = 0;
    best.obj = best.l1 = 0.0;
    int c[P];
#pragma unroll
    for (int i = 0; i < P; ++i) c[i] = i;
    int64_t ev = 0;
    const int N = m + P;
    do {
        ev += eval_vertex<P>(c, m, lam, xat, yat, best) ? 1 : 0;
    } while (next_comb<P>(N, c));
#pragma unroll
    for (int q = 0; q < P; ++q) A.beta[(size_t)pr * P + q] = best.v[q];
    A.objective[pr] = best.obj;
    A.vertices[pr] = ev;
}

template <int P>
__global__ void __launch_bounds__(256) brute_chunk_kernel(BruteArgs A)
{
    __shared__ double xs[64 * 8];
    __shared__ double ys[64];
    __shared__ BruteKey wbest[8];
    __shared__ unsigned long long wcnt[8];
    const int64_t pr = blockIdx.y;
    const int64_t ck = blockIdx.x;
    const int m = A.n;
    for (int i = threadIdx.x; i < m * P; i += blockDim.x) xs[i] = A.X[(size_t)pr * m * P + i];
    for (int i = threadIdx.x; i < m; i += blockDim.x) ys[i] = A.Y[(size_t)pr * m + i];
    __syncthreads();
    double lr = A.lam[pr];
    double lam = lr > A.lambda_floor ? lr : A.lambda_floor;
    auto xat = [&](int i, int q) { return xs[i * P + q]; };
    auto yat = [&](int i) { return ys[i]; };
    const int N = m + P;
    int64_t lo = ck * A.chunk, hi = lo + A.chunk < A.C ? lo + A.chunk : A.C;
    int64_t per = (hi - lo + blockDim.x - 1) / blockDim.x;
    int64_t s = lo + threadIdx.x * per, e = s + per < hi ? s + per : hi;
    BruteKey best;
    best.have = 0;
    best.obj = best.l1 = 0.0;
    unsigned long long ev = 0;
    if (s < e) {
        int c[P];
        unrank<P>(s, N, c);
        for (int64_t r = s; r < e; ++r) {
            ev += eval_vertex<P>(c, m, lam, xat, yat, best) ? 1 : 0;
            next_comb<P>(N, c);
        }
    }
    // warp reduce (deterministic: total order)
    for (int off = 16; off > 0; off >>= 1) {
        BruteKey o;
        o.have = __shfl_down_sync(0xffffffffu, best.have, off);
        o.obj = __shfl_down_sync(0xffffffffu, best.obj, off);
        o.l1 = __shfl_down_sync(0xffffffffu, best.l1, off);
#pragma unroll
        for (int q = 0; q < P; ++q) o.v[q] = __shfl_down_sync(0xffffffffu, best.v[q], off);
        unsigned long long oc = __shfl_down_sync(0xffffffffu, ev, off);
        if (key_less<P>(o, best)) best = o;
        ev += oc;
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        wbest[w] = best;
        wcnt[w] = ev;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        BruteKey bb = wbest[0];
        unsigned long long cc = wcnt[0];
        for (int q = 1; q < (int)(blockDim.x >> 5); ++q) {
            if (key_less<P>(wbest[q], bb)) bb = wbest[q];
            cc += wcnt[q];
        }
        A.partial[pr * A.nchunks + ck] = bb;
        A.pcount[pr * A.nchunks + ck] = cc;
    }
}

template <int P>
__global__ void brute_reduce_kernel(BruteArgs A)
{
    int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pr >= A.B) return;
    BruteKey bb = A.partial[pr * A.nchunks];
    unsigned long long cc = A.pcount[pr * A.nchunks];
    for (int64_t q = 1; q < A.nchunks; ++q) {
        const BruteKey &k = A.partial[pr * A.nchunks + q];
        if (key_less<P>(k, bb)) bb = k;
        cc += A.pcount[pr * A.nchunks + q];
    }
#pragma unroll
    for (int q = 0; q < P; ++q) A.beta[(size_t)pr * P + q] = bb.v[q];
    A.objective[pr] = bb.obj;
    A.vertices[pr] = (int64_t)cc;
}

// evaluate_objective for given coefficient vectors (model.py:151-154)
template <int P>
__global__ void objective_kernel(const double *X, const double *Y, const double *lamv, int64_t B, int m,
                                 const double *beta, double lambda_floor, double *out)
{
    int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pr >= B) return;
    const double *x = X + (size_t)pr * m * P;
    const double *y = Y + (size_t)pr * m;
    double b[P];
#pragma unroll
    for (int q = 0; q < P; ++q) b[q] = beta[(size_t)pr * P + q];
    double lr = lamv[pr];
    double lam = lr > lambda_floor ? lr : lambda_floor;
    double rs = np_sum_rec(0, m, [&](int i) {  // numpy pairwise order for any m (model.py:148)
        double g = gemv_row(P, i, m, [&](int q) { return x[i * P + q]; }, [&](int q) { return b[q < P ? q : P - 1]; });
        return fabs(dsub(y[i], g));
    });
    double l1 = np_sum_c<P>([&](int q) { return fabs(b[q]); });
    out[pr] = dadd(rs, dmul(lam, l1));
}

}  // namespace lad
