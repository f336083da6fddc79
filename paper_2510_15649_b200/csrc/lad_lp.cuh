// lad_lp.cuh -- batched dense tableau simplex for the LP recasting (lp.py).
//
// Standard form (lp.formulate, lp.py:82-96): columns bp (d), bn (d), rp (m),
// rn (m); rows x_i.(bp - bn) + rp_i - rn_i = y_i; cost lambda_eff on the
// coefficient parts, 1 on the residual parts.  Primal simplex from the
// sign-split residual basis (lp.py:106-170): Dantzig pricing with a permanent
// switch to Bland's rule after a degenerate streak of n pivots, ratio test
// with 1e-12 relative ties broken by the smallest basic variable index.
//
// One warp per problem, tableau (m+1) x (n+1) in shared memory (sized per
// launch), lanes over columns for row operations and over rows (two per lane,
// m <= 46) for the ratio test.  Bit-exact
// with the reference: the pivot update is numpy's elementwise
// `row /= piv; T -= outer(col, row)` (two roundings per entry), and the
// initial reduced-cost row c - cb @ T and objective cell -(cb @ T[:, n])
// follow OpenBLAS's dgemv_n / strided-ddot orders measured in the build
// container (oracle/orc_lp restates the same; tests pin both to the
// reference).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lad_numerics.cuh"

namespace lad {

constexpr int LP_MMAX = 46, LP_DMAX = 8;
constexpr int LP_NMAX = 2 * LP_DMAX + 2 * LP_MMAX;  // 108 columns
constexpr int LP_WARPS = 4;

struct LpArgs {
    const double *X, *Y, *lam;
    int64_t B;
    int m, d;
    int max_pivots;  // <= 0: 50 * n (lp.py:117)
    int bland;       // pivot_rule == "bland"
    double tol, lambda_floor;
    double *beta, *objective, *xfull;  // xfull (B, 2d+2m) may be null
    int32_t *pivots, *basis;           // basis (B, m) may be null
    uint8_t *converged, *status;       // 0 ok, 1 unbounded, 2 invalid input, 3 objective mismatch
    double *trace;                     // (B, trace_cap) objective after 0, 1, ... pivots; may be null
    int trace_cap;
    int warp_doubles;                  // shared memory per warp: tableau (m+1)(n+1) + pivot column (m+1)
};

// shared memory per warp for an m-row, d-variable problem
__host__ __device__ inline int lp_warp_doubles(int m, int d) { return (m + 1) * (2 * d + 2 * m + 1) + m + 1; }

// c - cb @ T column sum with cb = 1 (every initial basic variable is a residual
// part of cost 1): OpenBLAS dgemv_n folds rows in blocks of 4 ((t0+t1)+t2)+t3
// added to y, then a leftover pair (t0+t1), then a last row; the columns past
// n & -4 take the scalar tail loop (sequential).
__device__ __forceinline__ double lp_colsum(const double *T, int ld, int m, int j, int n)
{
    double y = 0.0;
    if (j >= (n & -4)) {
        for (int i = 0; i < m; ++i) y = dadd(y, T[i * ld + j]);
        return y;
    }
    const int nb = m & -4;
    for (int k = 0; k < nb; k += 4) {
        double t = dadd(dadd(dadd(T[k * ld + j], T[(k + 1) * ld + j]), T[(k + 2) * ld + j]), T[(k + 3) * ld + j]);
        y = dadd(y, t);
    }
    if (m - nb >= 2) y = dadd(y, dadd(T[nb * ld + j], T[(nb + 1) * ld + j]));
    if ((m - nb) & 1) y = dadd(y, T[(m - 1) * ld + j]);
    return y;
}

// cb @ T[:m, n] with cb = 1: OpenBLAS ddot for a non-unit stride (two
// accumulators fed (v0+v2), (v1+v3) per 4 elements, tail into the first).
__device__ __forceinline__ double lp_strided_sum(const double *T, int ld, int m, int j)
{
    double t1 = 0.0, t2 = 0.0;
    const int n1 = m & -4;
    int i = 0;
    for (; i < n1; i += 4) {
        t1 = dadd(t1, dadd(T[i * ld + j], T[(i + 2) * ld + j]));
        t2 = dadd(t2, dadd(T[(i + 1) * ld + j], T[(i + 3) * ld + j]));
    }
    for (; i < m; ++i) t1 = dadd(t1, T[i * ld + j]);
    return dadd(t1, t2);
}

__global__ void __launch_bounds__(32 * LP_WARPS) lp_simplex_kernel(LpArgs A)
{
    extern __shared__ double lp_smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t pr = (int64_t)blockIdx.x * LP_WARPS + w;
    if (pr >= A.B) return;
    const int m = A.m, d = A.d, n = 2 * d + 2 * m, ld = n + 1;
    double *T = lp_smem + (size_t)w * A.warp_doubles;
    double *cv = T + (size_t)(m + 1) * ld;  // pivot column copy (m+1)
    const double *x = A.X + (size_t)pr * m * d, *y = A.Y + (size_t)pr * m;
    const double lraw = A.lam[pr];
    bool ok = isfinite(lraw) && lraw >= 0.0;
    for (int e = lane; e < m * d; e += 32) ok = ok && isfinite(x[e]);
    for (int i = lane; i < m; i += 32) ok = ok && isfinite(y[i]);
    ok = __all_sync(0xffffffffu, ok);
    if (!ok) {
        if (lane == 0) {
            A.status[pr] = 2;
            A.converged[pr] = 0;
            A.pivots[pr] = 0;
            A.objective[pr] = __longlong_as_double(0x7ff8000000000000LL);
        }
        for (int j = lane; j < d; j += 32) A.beta[(size_t)pr * d + j] = __longlong_as_double(0x7ff8000000000000LL);
        return;
    }
    const double lam = lraw > A.lambda_floor ? lraw : A.lambda_floor;
    // rows lane and lane + 32 belong to this lane: their basic variables
    // (lp.initial_basis, lp.py:99-103: rp_i where y_i >= 0, else rn_i)
    int bas[2];
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
        const int i = lane + 32 * sl;
        bas[sl] = i < m ? (y[i] >= 0.0 ? 2 * d + i : 2 * d + m + i) : 0x7fffffff;
    }
    // tableau[:m, :n] = sign * A, tableau[:m, n] = sign * b
    for (int e = lane; e < m * ld; e += 32) {
        const int i = e / ld, j = e - i * ld;
        const double s = y[i] >= 0.0 ? 1.0 : -1.0;
        double a;
        if (j < d) a = x[i * d + j];
        else if (j < 2 * d) a = -x[i * d + (j - d)];
        else if (j < 2 * d + m) a = (j - 2 * d == i) ? 1.0 : 0.0;
        else if (j < n) a = (j - 2 * d - m == i) ? -1.0 : 0.0;
        else a = y[i];
        T[e] = dmul(s, a);
    }
    __syncwarp();
    // reduced costs c - cb @ T and the objective cell -(cb @ T[:, n])
    for (int j = lane; j < n; j += 32) {
        const double c = j < 2 * d ? lam : 1.0;
        T[m * ld + j] = dsub(c, lp_colsum(T, ld, m, j, n));
    }
    if (lane == 0) T[m * ld + n] = -lp_strided_sum(T, ld, m, n);
    __syncwarp();
    double *trace = A.trace ? A.trace + (size_t)pr * A.trace_cap : nullptr;
    if (trace && lane == 0 && A.trace_cap > 0) trace[0] = -T[m * ld + n];

    const double tol = A.tol;
    const int max_piv = A.max_pivots > 0 ? A.max_pivots : 50 * n;
    bool bland = A.bland != 0;
    int streak = 0, pivots = 0;
    bool converged = false, unbounded = false;
    while (pivots < max_piv) {
        // entering column
        int col;
        if (bland) {
            col = 0x7fffffff;
            for (int j0 = 0; j0 < n; j0 += 32) {
                const int j = j0 + lane;
                const unsigned bal = __ballot_sync(0xffffffffu, j < n && T[m * ld + j] < -tol);
                if (bal) {
                    col = j0 + __ffs(bal) - 1;
                    break;
                }
            }
            if (col == 0x7fffffff) {
                converged = true;
                break;
            }
        } else {  // np.argmin: first index of the minimum
            double bv = __longlong_as_double(0x7ff0000000000000LL);
            int bj = 0x7fffffff;
            for (int j = lane; j < n; j += 32) {
                const double v = T[m * ld + j];
                if (v < bv) {
                    bv = v;
                    bj = j;
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
                if (ov < bv || (ov == bv && oj < bj)) {
                    bv = ov;
                    bj = oj;
                }
            }
            col = bj;
            if (bv >= -tol) {
                converged = true;
                break;
            }
        }
        // leaving row: min ratio, ties within 1e-12 relative -> smallest basic index
        double ratio[2];
        bool elig_any = false;
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
            const int i = lane + 32 * sl;
            const double pc = i < m ? T[i * ld + col] : 0.0;
            const bool elig = i < m && pc > tol;
            elig_any = elig_any || elig;
            ratio[sl] = elig ? ddiv(T[i * ld + n], pc) : __longlong_as_double(0x7ff0000000000000LL);
        }
        if (!__any_sync(0xffffffffu, elig_any)) {
            unbounded = true;
            break;
        }
        double best = fmin(ratio[0], ratio[1]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, off));
        const double lim = dadd(best, dmul(1e-12, dadd(1.0, fabs(best))));
        const bool tie0 = lane < m && ratio[0] <= lim, tie1 = lane + 32 < m && ratio[1] <= lim;
        int key = min(tie0 ? bas[0] : 0x7fffffff, tie1 ? bas[1] : 0x7fffffff);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, off));
        const unsigned b0 = __ballot_sync(0xffffffffu, tie0 && bas[0] == key);
        const unsigned b1 = __ballot_sync(0xffffffffu, tie1 && bas[1] == key);
        const int row = b0 ? __ffs(b0) - 1 : 32 + __ffs(b1) - 1;
        // pivot: row /= piv; T -= outer(col_vals, row) with col_vals[row] = 0
        const double piv = T[row * ld + col];
        for (int i = lane; i <= m; i += 32) cv[i] = (i == row) ? 0.0 : T[i * ld + col];
        __syncwarp();
        for (int j = lane; j <= n; j += 32) T[row * ld + j] = ddiv(T[row * ld + j], piv);
        __syncwarp();
        // every other row reads the pivot row, so it is rewritten last (numpy's
        // T[row] - 0 * T[row] still normalises -0 to +0 there)
        for (int e = lane; e < (m + 1) * ld; e += 32) {
            const int i = e / ld, j = e - i * ld;
            if (i != row) T[e] = dsub(T[e], dmul(cv[i], T[row * ld + j]));
        }
        __syncwarp();
        for (int j = lane; j <= n; j += 32) T[row * ld + j] = dsub(T[row * ld + j], dmul(0.0, T[row * ld + j]));
        __syncwarp();
        for (int i = lane; i <= m; i += 32) T[i * ld + col] = (i == row) ? 1.0 : 0.0;
        if (lane == row) bas[0] = col;
        if (lane + 32 == row) bas[1] = col;
        __syncwarp();
        ++pivots;
        if (trace && lane == 0 && pivots < A.trace_cap) trace[pivots] = -T[m * ld + n];
        streak = best <= tol ? streak + 1 : 0;
        if (!bland && streak >= n) bland = true;
    }
    // x[basis] = T[:m, n]; beta = x[:d] - x[d:2d]
    double *xs = T + (size_t)m * ld;  // x over the reduced-cost row, which is no longer needed
    __syncwarp();
    for (int j = lane; j < n; j += 32) xs[j] = 0.0;
    __syncwarp();
#pragma unroll
    for (int sl = 0; sl < 2; ++sl)
        if (lane + 32 * sl < m) xs[bas[sl]] = T[(lane + 32 * sl) * ld + n];
    __syncwarp();
    for (int j = lane; j < d; j += 32) A.beta[(size_t)pr * d + j] = dsub(xs[j], xs[d + j]);
    if (A.xfull)
        for (int j = lane; j < n; j += 32) A.xfull[(size_t)pr * n + j] = xs[j];
    if (A.basis)
#pragma unroll
        for (int sl = 0; sl < 2; ++sl)
            if (lane + 32 * sl < m) A.basis[(size_t)pr * m + lane + 32 * sl] = bas[sl];
    __syncwarp();
    if (lane == 0) {
        // evaluate_objective(beta) (model.py:151) and the consistency check of simplex_solve (lp.py:180-186)
        const double *b = A.beta + (size_t)pr * d;
        const double rs = np_sum(m, [&](int i) {
            return fabs(dsub(y[i], gemv_row(d, i, m, [&](int q) { return x[i * d + q]; }, [&](int q) { return b[q]; })));
        });
        const double obj = dadd(rs, dmul(lam, np_sum(d, [&](int q) { return fabs(b[q]); })));
        double cx = 0.0;  // c @ x, only for the 1e-9 check
        for (int j = 0; j < n; ++j) cx = dfma(j < 2 * d ? lam : 1.0, xs[j], cx);
        const bool mismatch = converged && fabs(dsub(obj, cx)) > dmul(1e-9, fmax(1.0, fabs(obj)));
        A.objective[pr] = obj;
        A.pivots[pr] = pivots;
        A.converged[pr] = converged ? 1 : 0;
        A.status[pr] = unbounded ? 1 : (mismatch ? 3 : 0);
    }
}


}  // namespace lad
