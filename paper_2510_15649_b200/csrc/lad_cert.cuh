// lad_cert.cuh -- batched axis-wise-minimum certificate (ccd.is_axiswise_minimum).
//
// For each problem and each axis j (except `skip`), the axis restriction
// (model.axis_restriction, model.py:157-177) is rebuilt with the reference's
// arithmetic: base = (y - x @ b) + x_j * b_j, breakpoints base_i / x_ij over the
// nonzero rows then 0 (weight lambda_eff); its one-sided slopes at b_j
// (PiecewiseLinear1D.slopes_at, linesearch.py:65-77) use numpy's pairwise sums
// over the masked weight arrays.  The point is certified iff no slope
// descends beyond 1e-12 * (W + 1) (ccd.py:214-237).  One thread per problem:
// this is a check run once per result, not a hot loop.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lad_numerics.cuh"

namespace lad {

struct CertArgs {
    const double *X, *Y, *lam, *beta;
    const int32_t *skip;  // (B,) axis exempt from the test, -1 none; may be null
    int64_t B;
    int n, p;
    double tol, lambda_floor;
    uint8_t *out;  // 1 certified, 0 not, 2 invalid input
};

template <int NMAX, int PMAX>
__global__ void axiswise_minimum_kernel(CertArgs A)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.B) return;
    const int n = A.n, p = A.p;
    const double *x = A.X + (size_t)i * n * p, *y = A.Y + (size_t)i * n, *b = A.beta + (size_t)i * p;
    const double lraw = A.lam[i];
    bool ok = isfinite(lraw) && lraw >= 0.0;
    for (int k = 0; k < n * p; ++k) ok = ok && isfinite(x[k]);
    for (int k = 0; k < n; ++k) ok = ok && isfinite(y[k]);
    for (int k = 0; k < p; ++k) ok = ok && isfinite(b[k]);
    if (!ok) {
        A.out[i] = 2;
        return;
    }
    const double lam = lraw > A.lambda_floor ? lraw : A.lambda_floor;
    const int skip = A.skip ? A.skip[i] : -1;
    double r[NMAX];
    for (int k = 0; k < n; ++k)
        r[k] = dsub(y[k], gemv_row(p, k, n, [&](int q) { return x[k * p + q]; }, [&](int q) { return b[q]; }));
    double loc[NMAX + 1], w[NMAX + 1], sel[NMAX + 1];
    for (int j = 0; j < p; ++j) {
        if (j == skip) continue;
        const double bj = b[j];
        int cnt = 0;
        for (int k = 0; k < n; ++k) {
            const double c = x[k * p + j];
            const double base = dadd(r[k], dmul(c, bj));
            if (c != 0.0) {
                loc[cnt] = ddiv(base, c);
                w[cnt] = fabs(c);
                ++cnt;
            }
        }
        loc[cnt] = 0.0;
        w[cnt] = lam;
        ++cnt;
        const double total = np_sum(cnt, [&](int q) { return w[q]; });
        const double atol = dmul(A.tol, fmax(1.0, fabs(bj)));
        const double lo = dsub(bj, atol), hi = dadd(bj, atol);
        int nb = 0;
        for (int q = 0; q < cnt; ++q)
            if (loc[q] < lo) sel[nb++] = w[q];
        const double w_below = np_sum(nb, [&](int q) { return sel[q]; });
        int na = 0;
        for (int q = 0; q < cnt; ++q)
            if (loc[q] > hi) sel[na++] = w[q];
        const double w_above = np_sum(na, [&](int q) { return sel[q]; });
        const double w_at = dsub(dsub(total, w_below), w_above);
        const double left = dsub(dsub(w_below, w_at), w_above);
        const double right = dsub(dadd(w_below, w_at), w_above);
        const double eps = dmul(1e-12, dadd(total, 1.0));
        if (left > eps || right < -eps) {
            A.out[i] = 0;
            return;
        }
    }
    A.out[i] = 1;
}

}  // namespace lad
