/*
 * ladlasso_oracle.c -- CPU restatement of the reference LAD-LASSO hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path in paper_2510_15649_b200/csrc/.  Only tests/, the smoke() in
 * __graft_entry__.py and bench.py's cpu_baseline / --impl reference legs may
 * load it.  The product never links or calls it.
 *
 * What it restates (reference = /root/reference/pkg/src/ladlasso, pure
 * Python + numpy 2.3.5 + OpenBLAS 0.3.30 SkylakeX kernels):
 *   - model.objective_value            model.py:145-148
 *   - ccd._median_location             ccd.py:81-91
 *   - ccd._AxisWorkspace               ccd.py:94-110
 *   - ccd.ccd_descend                  ccd.py:126-206
 *   - linesearch.expand_bracket        linesearch.py:236-268
 *   - linesearch.ternary_min           linesearch.py:172-203
 *   - linesearch.quadrature_min        linesearch.py:206-233
 *   - locus.axes_by_influence          locus.py:90-93
 *   - locus.default_bracket            locus.py:96-101
 *   - locus.locus_value                locus.py:104-123
 *   - locus._CurveEvaluator            locus.py:150-215
 *   - locus._search_one_axis           locus.py:218-232
 *   - locus._start_fan                 locus.py:235-253
 *   - locus._dense_refine              locus.py:256-297
 *   - locus.solve_locus                locus.py:300-409
 *   - brute.solve_linear_system        brute.py:29-59
 *   - brute.solve_brute                brute.py:106-145
 *   - rng.Pcg32                        rng.py:25-46
 *
 * Floating-point order.  The reference's reductions go through numpy and
 * OpenBLAS; their exact evaluation orders were measured in this container
 * (oracle/probe_numerics.py re-checks them) and are restated below:
 *   np_sum      numpy pairwise_sum: n<8 sequential from 0.0; else 8 lane
 *               accumulators over blocks of 8, tree ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
 *               then the n%8 tail sequentially.
 *   blas_ddot   OpenBLAS ddot_k (SkylakeX): n&-16 == 16 -> per-lane
 *               ((p_l+p_{l+4})+p_{l+8})+p_{l+12}, then (S0+S2)+(S1+S3);
 *               n&-16 == 32 -> 4 zmm accumulators folded 512->256->128;
 *               tail i >= n&-16 is an FMA chain dot = fma(x_i, y_i, dot).
 *   gemv_row    OpenBLAS dgemv_t (SkylakeX) row dot of x @ b, dependent on
 *               the kernel (4x4 / 4x2 / 4x1) the output row falls in and on
 *               the d&3 leftover columns (scalar FMA code).
 * Compile with -ffp-contract=off so that only the fma() calls written here fuse.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_MAX_D 8
#define ORC_MAX_M 1024

/* ------------------------------------------------------------------ */
/* problem + coordinate descent (ccd.py:126-206)                        */
/* ------------------------------------------------------------------ */


typedef struct {
    const double *x; /* (m, d) row-major */
    const double *y; /* (m,) */
    int m, d;
    double lam;      /* lambda_eff = max(lam, floor) */
    const float *xf, *yf; /* fp32 mode: the binary32 data (x, y unused) */
    int f32;
} orc_problem;

typedef struct {
    double beta[ORC_MAX_D];
    double objective;
    int sweeps, steps, converged;
} orc_descent;

typedef struct {
    long long descents;
    long long steps;
} orc_counters;


/* the descent half, once per element type (orc_descent.inc) */
#define REAL double
#define RF(name) name
#define R_FABS fabs
#define R_FMA fma
#define R_X(P) ((P)->x)
#define R_Y(P) ((P)->y)
#include "orc_descent.inc"
#undef REAL
#undef RF
#undef R_FABS
#undef R_FMA
#undef R_X
#undef R_Y
#define REAL float
#define RF(name) name##_f32
#define R_FABS fabsf
#define R_FMA fmaf
#define R_X(P) ((P)->xf)
#define R_Y(P) ((P)->yf)
#include "orc_descent.inc"
#undef REAL
#undef RF
#undef R_FABS
#undef R_FMA
#undef R_X
#undef R_Y

/* precision dispatch: the outer search is binary64 in both modes */
static void ccd_descend(const orc_problem *P, const double *start, int frozen, double sweep_tol, int max_sweeps,
                        orc_descent *out, orc_counters *cnt, double *trace, int *trace_len)
{
    if (P->f32) descend_f32(P, start, frozen, sweep_tol, max_sweeps, out, cnt, trace, trace_len);
    else descend(P, start, frozen, sweep_tol, max_sweeps, out, cnt, trace, trace_len);
}

/* linesearch.weighted_median_min (linesearch.py:133-154): total = weights.sum() */
double orc_weighted_median_min(const double *loc, const double *w, int n, double constant, double *value)
{
    int order[ORC_MAX_M + 1];
    for (int i = 0; i < n; ++i) {
        int k = i;
        while (k > 0 && loc[order[k - 1]] > loc[i]) {
            order[k] = order[k - 1];
            --k;
        }
        order[k] = i;
    }
    double cum[ORC_MAX_M + 1];
    double c = 0.0;
    for (int i = 0; i < n; ++i) {
        c += w[order[i]];
        cum[i] = c;
    }
    double total = orc_np_sum(w, n);
    double half = 0.5 * total;
    int k = 0;
    while (k < n && cum[k] < half) ++k;
    double t;
    if (k + 1 < n && fabs(cum[k] - half) <= 1e-12 * total)
        t = 0.5 * (loc[order[k]] + loc[order[k + 1]]);
    else
        t = loc[order[k < n - 1 ? k : n - 1]];
    double a[ORC_MAX_M + 1];
    for (int i = 0; i < n; ++i) a[i] = fabs(t - loc[i]);
    if (value) *value = constant + orc_ddot(a, w, n);
    return t;
}

/* exported: one ccd_descend; frozen < 0 means None */
int orc_ccd_descend(const double *x, const double *y, int m, int d, double lam, const double *start, int frozen,
                    double sweep_tol, int max_sweeps, double *beta_out, double *obj_out, int *sweeps_out,
                    int *steps_out, int *conv_out, double *trace, int *trace_len)
{
    if (m < 1 || d < 1 || m > ORC_MAX_M || d > ORC_MAX_D) return -1;
    orc_problem P = {x, y, m, d, lam};
    orc_descent D;
    if (trace_len) *trace_len = 0;
    ccd_descend(&P, start, frozen, sweep_tol, max_sweeps, &D, NULL, trace, trace_len);
    memcpy(beta_out, D.beta, sizeof(double) * d);
    *obj_out = D.objective;
    *sweeps_out = D.sweeps;
    *steps_out = D.steps;
    *conv_out = D.converged;
    return 0;
}

/* exported: one ccd_descend in fp32 mode (binary32 data and descent) */
int orc_ccd_descend_f32(const float *x, const float *y, int m, int d, double lam, const double *start, int frozen,
                        double sweep_tol, int max_sweeps, double *beta_out, double *obj_out, int *sweeps_out,
                        int *steps_out, int *conv_out, double *trace, int *trace_len)
{
    if (m < 1 || d < 1 || m > ORC_MAX_M || d > ORC_MAX_D) return -1;
    orc_problem P = {NULL, NULL, m, d, lam, x, y, 1};
    orc_descent D;
    if (trace_len) *trace_len = 0;
    ccd_descend(&P, start, frozen, sweep_tol, max_sweeps, &D, NULL, trace, trace_len);
    memcpy(beta_out, D.beta, sizeof(double) * d);
    *obj_out = D.objective;
    *sweeps_out = D.sweeps;
    *steps_out = D.steps;
    *conv_out = D.converged;
    return 0;
}

/* ccd.is_axiswise_minimum (ccd.py:214-237) through model.axis_restriction
 * (model.py:157-177) and PiecewiseLinear1D.slopes_at (linesearch.py:65-77):
 * masked weight sums are numpy pairwise sums over the compacted arrays. */
int orc_is_axiswise_minimum(const double *x, const double *y, int m, int d, double lam, const double *b, int skip,
                            double tol)
{
    if (m < 1 || d < 1 || m > ORC_MAX_M || d > ORC_MAX_D) return -1;
    double r[ORC_MAX_M];
    residual_init(x, y, m, d, b, r);
    for (int j = 0; j < d; ++j) {
        if (j == skip) continue;
        double loc[ORC_MAX_M + 1], w[ORC_MAX_M + 1], sel[ORC_MAX_M + 1];
        int cnt = 0;
        for (int i = 0; i < m; ++i) {
            double c = x[(size_t)i * d + j];
            double base = r[i] + c * b[j];
            if (c != 0.0) {
                loc[cnt] = base / c;
                w[cnt] = fabs(c);
                ++cnt;
            }
        }
        loc[cnt] = 0.0;
        w[cnt] = lam;
        ++cnt;
        double total = orc_np_sum(w, cnt);
        double atol = tol * fmax(1.0, fabs(b[j]));
        double lo = b[j] - atol, hi = b[j] + atol;
        int nb = 0;
        for (int q = 0; q < cnt; ++q)
            if (loc[q] < lo) sel[nb++] = w[q];
        double w_below = orc_np_sum(sel, nb);
        int na = 0;
        for (int q = 0; q < cnt; ++q)
            if (loc[q] > hi) sel[na++] = w[q];
        double w_above = orc_np_sum(sel, na);
        double w_at = total - w_below - w_above;
        double left = w_below - w_at - w_above;
        double right = w_below + w_at - w_above;
        double eps = 1e-12 * (total + 1.0);
        if (left > eps || right < -eps) return 0;
    }
    return 1;
}

/* ------------------------------------------------------------------ */
/* LP recasting + dense tableau simplex (lp.py:82-215)                  */
/* ------------------------------------------------------------------ */

/* c - cb @ T with cb = 1: OpenBLAS dgemv_n row blocks of 4, pair + odd tail;
 * columns j >= n & -4 use the scalar tail loop (sequential).  Measured with
 * cancellation probes against numpy 2.3.5 / OpenBLAS 0.3.30. */
static double lp_colsum(const double *T, int ld, int m, int j, int n)
{
    double y = 0.0;
    if (j >= (n & -4)) {
        for (int i = 0; i < m; ++i) y += T[i * ld + j];
        return y;
    }
    int nb = m & -4;
    for (int k = 0; k < nb; k += 4) y += ((T[k * ld + j] + T[(k + 1) * ld + j]) + T[(k + 2) * ld + j]) + T[(k + 3) * ld + j];
    if (m - nb >= 2) y += T[nb * ld + j] + T[(nb + 1) * ld + j];
    if ((m - nb) & 1) y += T[(m - 1) * ld + j];
    return y;
}

/* cb @ T[:, j] (strided) with cb = 1: OpenBLAS ddot for non-unit increments */
static double lp_strided_sum(const double *T, int ld, int m, int j)
{
    double t1 = 0.0, t2 = 0.0;
    int i = 0, n1 = m & -4;
    for (; i < n1; i += 4) {
        t1 += T[i * ld + j] + T[(i + 2) * ld + j];
        t2 += T[(i + 1) * ld + j] + T[(i + 3) * ld + j];
    }
    for (; i < m; ++i) t1 += T[i * ld + j];
    return t1 + t2;
}

/* lp.simplex_minimize + simplex_solve.  Returns 0 ok, 1 unbounded, 3 objective mismatch (both
 * SimplexError in the reference), -1 bad shape.
 * x_full (2d+2m) and basis_out (m) may be NULL. */
int orc_lp_solve(const double *x, const double *y, int m, int d, double lam, int max_pivots, int bland_rule,
                 double tol, double *beta, double *objective, int *pivots_out, int *converged_out, double *x_full,
                 int *basis_out)
{
    if (m < 1 || d < 1 || m > ORC_MAX_M || d > ORC_MAX_D) return -1;
    const int n = 2 * d + 2 * m, ld = n + 1;
    double *T = (double *)malloc(sizeof(double) * (size_t)(m + 1) * ld);
    int basis[ORC_MAX_M];
    for (int i = 0; i < m; ++i) {
        double s = y[i] >= 0 ? 1.0 : -1.0;
        basis[i] = y[i] >= 0 ? 2 * d + i : 2 * d + m + i;
        for (int j = 0; j < n; ++j) {
            double a;
            if (j < d) a = x[i * d + j];
            else if (j < 2 * d) a = -x[i * d + (j - d)];
            else if (j < 2 * d + m) a = (j - 2 * d == i) ? 1.0 : 0.0;
            else a = (j - 2 * d - m == i) ? -1.0 : 0.0;
            T[i * ld + j] = s * a;
        }
        T[i * ld + n] = s * y[i];
    }
    for (int j = 0; j < n; ++j) T[m * ld + j] = (j < 2 * d ? lam : 1.0) - lp_colsum(T, ld, m, j, n);
    T[m * ld + n] = -lp_strided_sum(T, ld, m, n);
    int maxp = max_pivots > 0 ? max_pivots : 50 * n;
    int bland = bland_rule, streak = 0, pivots = 0, converged = 0, unbounded = 0;
    double cv[ORC_MAX_M + 1];
    while (pivots < maxp) {
        int col = -1;
        if (bland) {
            for (int j = 0; j < n; ++j)
                if (T[m * ld + j] < -tol) { col = j; break; }
            if (col < 0) { converged = 1; break; }
        } else {
            col = 0;
            for (int j = 1; j < n; ++j)
                if (T[m * ld + j] < T[m * ld + col]) col = j;
            if (T[m * ld + col] >= -tol) { converged = 1; break; }
        }
        double ratios[ORC_MAX_M];
        int any = 0;
        double best = INFINITY;
        for (int i = 0; i < m; ++i) {
            double pc = T[i * ld + col];
            ratios[i] = pc > tol ? T[i * ld + n] / pc : INFINITY;
            if (pc > tol) any = 1;
            if (ratios[i] < best) best = ratios[i];
        }
        if (!any) { unbounded = 1; break; }
        int row = -1;
        double lim = best + 1e-12 * (1.0 + fabs(best));
        for (int i = 0; i < m; ++i)
            if (ratios[i] <= lim && (row < 0 || basis[i] < basis[row])) row = i;
        double piv = T[row * ld + col];
        for (int j = 0; j <= n; ++j) T[row * ld + j] /= piv;
        for (int i = 0; i <= m; ++i) cv[i] = i == row ? 0.0 : T[i * ld + col];
        for (int i = 0; i <= m; ++i) {
            if (i == row) continue;
            for (int j = 0; j <= n; ++j) T[i * ld + j] -= cv[i] * T[row * ld + j];
        }
        for (int j = 0; j <= n; ++j) T[row * ld + j] -= 0.0 * T[row * ld + j];
        for (int i = 0; i <= m; ++i) T[i * ld + col] = 0.0;
        T[row * ld + col] = 1.0;
        basis[row] = col;
        ++pivots;
        streak = best <= tol ? streak + 1 : 0;
        if (!bland && streak >= n) bland = 1;
    }
    double xs[2 * ORC_MAX_D + 2 * ORC_MAX_M];
    for (int j = 0; j < n; ++j) xs[j] = 0.0;
    for (int i = 0; i < m; ++i) xs[basis[i]] = T[i * ld + n];
    free(T);
    for (int j = 0; j < d; ++j) beta[j] = xs[j] - xs[d + j];
    *objective = orc_objective(x, y, m, d, lam, beta);
    double cx = 0.0;
    for (int j = 0; j < n; ++j) cx = fma(j < 2 * d ? lam : 1.0, xs[j], cx);
    int mismatch = converged && fabs(*objective - cx) > 1e-9 * fmax(1.0, fabs(*objective));
    *pivots_out = pivots;
    *converged_out = converged;
    if (x_full) memcpy(x_full, xs, sizeof(double) * n);
    if (basis_out) memcpy(basis_out, basis, sizeof(int) * m);
    return unbounded ? 1 : (mismatch ? 3 : 0);
}

/* ------------------------------------------------------------------ */
/* PCG32 (rng.py:25-46)                                                 */
/* ------------------------------------------------------------------ */

typedef struct { uint64_t state, inc; } orc_pcg32;

static uint32_t pcg_next(orc_pcg32 *g)
{
    uint64_t old = g->state;
    g->state = old * 6364136223846793005ULL + g->inc;
    uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    uint32_t rot = (uint32_t)(old >> 59);
    return (xs >> rot) | (xs << ((32 - rot) & 31));
}

static void pcg_seed(orc_pcg32 *g, uint64_t seed, uint64_t stream)
{
    g->state = 0;
    g->inc = (stream << 1) | 1u;
    pcg_next(g);
    g->state += seed;
    pcg_next(g);
}

void orc_pcg32_sequence(uint64_t seed, uint64_t stream, int n, uint32_t *out)
{
    orc_pcg32 g;
    pcg_seed(&g, seed, stream);
    for (int i = 0; i < n; ++i) out[i] = pcg_next(&g);
}

/* ------------------------------------------------------------------ */
/* locus search (locus.py)                                              */
/* ------------------------------------------------------------------ */

typedef struct {
    int outer_axis;           /* -1 = None (scan axes by influence) */
    int outer_search;         /* 0 ternary, 1 quadrature */
    double outer_tolerance;
    int outer_probes;
    int outer_max_iterations;
    int has_bracket;
    double bracket_lo, bracket_hi;
    double inner_sweep_tol;
    int inner_max_sweeps;
} orc_locus_params;

typedef struct {
    double t;
    double beta[ORC_MAX_D];
    double value;
    int inner_converged;
    int inner_evals;
} orc_point;

typedef struct {
    const orc_problem *P;
    int axis;
    int economy;
    double inner_tol; int inner_sweeps;
    double fast_tol;  int fast_sweeps;
    double margin_scale;
    orc_point *seen; int nseen, cap;
    int calls, failures;
    int has_best;
    orc_point best;
    orc_counters *cnt;
    int error;                /* 1 = unbounded direction */
} orc_curve;

static void curve_init(orc_curve *c, const orc_problem *P, int axis, const orc_locus_params *prm, orc_counters *cnt)
{
    c->P = P;
    c->axis = axis;
    c->economy = P->d > 3;
    c->inner_tol = prm->inner_sweep_tol;
    c->inner_sweeps = c->economy ? (prm->inner_max_sweeps < 150 ? prm->inner_max_sweeps : 150) : prm->inner_max_sweeps;
    c->fast_tol = prm->inner_sweep_tol > 1e-7 ? prm->inner_sweep_tol : 1e-7;
    int cap = c->economy ? 40 : 150;
    c->fast_sweeps = prm->inner_max_sweeps < cap ? prm->inner_max_sweeps : cap;
    c->margin_scale = c->economy ? 1e-4 : 1e-3;
    c->cap = 64;
    c->seen = (orc_point *)malloc(sizeof(orc_point) * c->cap);
    c->nseen = 0;
    c->calls = c->failures = 0;
    c->has_best = 0;
    c->cnt = cnt;
    c->error = 0;
}

static void curve_free(orc_curve *c) { free(c->seen); }

static void curve_append(orc_curve *c, const orc_point *pt)
{
    if (c->nseen == c->cap) {
        c->cap *= 2;
        c->seen = (orc_point *)realloc(c->seen, sizeof(orc_point) * c->cap);
    }
    c->seen[c->nseen++] = *pt;
}

/* locus.locus_value (locus.py:104-123) */
static void locus_value(const orc_problem *P, int axis, double t, double tol, int sweeps, const double *warm,
                        orc_point *pt, orc_counters *cnt)
{
    double start[ORC_MAX_D];
    if (warm) memcpy(start, warm, sizeof(double) * P->d);
    else memset(start, 0, sizeof(double) * P->d);
    start[axis] = t;
    orc_descent D;
    ccd_descend(P, start, axis, tol, sweeps, &D, cnt, NULL, NULL);
    pt->t = t;
    memcpy(pt->beta, D.beta, sizeof(double) * P->d);
    pt->value = D.objective;
    pt->inner_converged = D.converged;
    pt->inner_evals = D.steps;
}

/* optional probe log for debugging parity (set via orc_set_probe_log) */
static double *g_probe_log = NULL;
static int g_probe_cap = 0, g_probe_n = 0;
void orc_set_probe_log(double *buf, int cap) { g_probe_log = buf; g_probe_cap = cap; g_probe_n = 0; }
int orc_probe_log_count(void) { return g_probe_n; }

/* _CurveEvaluator.__call__ (locus.py:193-215) */
static double curve_eval(orc_curve *c, double t)
{
    if (g_probe_log && g_probe_n < g_probe_cap) g_probe_log[g_probe_n++] = t;
    const orc_problem *P = c->P;
    const double *warm = NULL;
    if (c->nseen) { /* _nearest: first minimal |pt.t - t| */
        int bi = 0;
        double bd = fabs(c->seen[0].t - t);
        for (int k = 1; k < c->nseen; ++k) {
            double dd = fabs(c->seen[k].t - t);
            if (dd < bd) { bd = dd; bi = k; }
        }
        warm = c->seen[bi].beta;
    }
    orc_point pt, alt;
    if (c->economy && warm) {
        locus_value(P, c->axis, t, c->fast_tol, c->fast_sweeps, warm, &pt, c->cnt);
    } else {
        locus_value(P, c->axis, t, c->fast_tol, c->fast_sweeps, NULL, &pt, c->cnt);
        if (warm && P->d > 2) {
            locus_value(P, c->axis, t, c->fast_tol, c->fast_sweeps, warm, &alt, c->cnt);
            if (alt.value < pt.value) pt = alt;
        }
    }
    int refine;
    if (!c->has_best) refine = 1;
    else {
        double margin = c->margin_scale * fmax(1.0, fabs(c->best.value));
        refine = pt.value <= c->best.value + margin;
    }
    if (refine) {
        orc_point ref;
        double pb[ORC_MAX_D];
        memcpy(pb, pt.beta, sizeof(double) * P->d);
        locus_value(P, c->axis, t, c->inner_tol, c->inner_sweeps, pb, &ref, c->cnt);
        if (ref.value < pt.value) pt = ref;
    }
    c->calls += 1;
    c->failures += pt.inner_converged ? 0 : 1;
    curve_append(c, &pt);
    if (!c->has_best || pt.value < c->best.value) {
        c->best = pt;
        c->has_best = 1;
    }
    return pt.value;
}

/* linesearch.expand_bracket (linesearch.py:236-268), growth 2, 60 doublings */
static int expand_bracket(orc_curve *c, double *plo, double *phi)
{
    double lo = *plo, hi = *phi;
    double g_lo = curve_eval(c, lo);
    double g_hi = curve_eval(c, hi);
    for (int it = 0; it < 60; ++it) {
        double g_mid = curve_eval(c, 0.5 * (lo + hi));
        if (g_mid < g_lo && g_mid < g_hi) {
            *plo = lo;
            *phi = hi;
            return 0;
        }
        double step = (2.0 - 1.0) * (hi - lo);
        if (g_lo < g_hi) {
            lo -= step;
            g_lo = curve_eval(c, lo);
        } else if (g_hi < g_lo) {
            hi += step;
            g_hi = curve_eval(c, hi);
        } else {
            lo -= step;
            hi += step;
            g_lo = curve_eval(c, lo);
            g_hi = curve_eval(c, hi);
        }
    }
    return 1;
}

/* ternary_min / quadrature_min (linesearch.py:172-233); returns rounds, sets converged */
static int outer_search(orc_curve *c, double lo, double hi, const orc_locus_params *prm, int *converged)
{
    double target = prm->outer_tolerance * (hi - lo);
    curve_eval(c, 0.5 * (lo + hi));
    int rounds = 0;
    if (prm->outer_search == 0) {
        while ((hi - lo) > target && rounds < prm->outer_max_iterations) {
            double third = (hi - lo) / 3.0;
            double m1 = lo + third;
            double m2 = hi - third;
            double v1 = curve_eval(c, m1);
            double v2 = curve_eval(c, m2);
            if (v1 < v2) hi = m2;
            else lo = m1;
            ++rounds;
        }
    } else {
        int np_ = prm->outer_probes;
        while ((hi - lo) > target && rounds < prm->outer_max_iterations) {
            double h = (hi - lo) / (double)(np_ + 1);
            int bi = 0;
            double bv = INFINITY, bt = 0.0;
            for (int k = 1; k <= np_; ++k) {
                double t = lo + h * (double)k;
                double v = curve_eval(c, t);
                if (k == 1 || v < bv) { bv = v; bt = t; bi = k; }
            }
            (void)bi;
            double nlo = bt - h, nhi = bt + h;
            lo = nlo > lo ? nlo : lo; /* max(lo, t - h) */
            hi = nhi < hi ? nhi : hi; /* min(hi, t + h) */
            ++rounds;
        }
    }
    curve_eval(c, 0.5 * (lo + hi));
    *converged = (hi - lo) <= target;
    return rounds;
}

/* np.abs(x).sum(axis=0)[j] (locus.py:92, :97): for d >= 2 numpy reduces the
 * strided axis row by row (sequential); for d == 1 the column is contiguous and
 * numpy uses pairwise_sum.  Measured: oracle/probe_numerics.py. */
static double col_abs_sum(const orc_problem *P, int j)
{
    return P->f32 ? col_abs_sum_t_f32(P, j) : col_abs_sum_t(P, j);
}

static void default_bracket(const orc_problem *P, double *lo, double *hi)
{
    double scale = 0.0;
    for (int j = 0; j < P->d; ++j) {
        double mean = col_abs_sum(P, j) / (double)P->m;
        if (j == 0 || mean > scale) scale = mean;
    }
    double ymax = P->f32 ? y_absmax_t_f32(P) : y_absmax_t(P);
    double radius = scale > 0 ? ymax / scale : INFINITY;
    if (!isfinite(radius) || radius <= 0) radius = 1.0;
    *lo = -radius;
    *hi = radius;
}

static void axes_by_influence(const orc_problem *P, int *axes)
{
    double infl[ORC_MAX_D];
    for (int j = 0; j < P->d; ++j) {
        infl[j] = col_abs_sum(P, j);
        axes[j] = j;
    }
    /* stable insertion sort by -influence (ties keep index order) */
    for (int a = 1; a < P->d; ++a) {
        int v = axes[a], k = a;
        while (k > 0 && -infl[axes[k - 1]] > -infl[v]) {
            axes[k] = axes[k - 1];
            --k;
        }
        axes[k] = v;
    }
}

/* _dense_refine (locus.py:256-297) */
static void dense_refine(const orc_problem *P, int axis, const orc_point *incumbent, const orc_locus_params *prm,
                         double width, int fan, orc_counters *cnt, orc_point *best_out, int *calls_out,
                         int *failures_out)
{
    orc_curve c;
    curve_init(&c, P, axis, prm, cnt);
    curve_append(&c, incumbent);
    c.best = *incumbent;
    c.has_best = 1;
    double margin = c.margin_scale * fmax(1.0, fabs(incumbent->value));
    /* _start_fan (locus.py:235-253) */
    orc_pcg32 g;
    pcg_seed(&g, 0x5EEDULL + (uint64_t)axis, 54);
    for (int s = 0; s < fan; ++s) {
        double start[ORC_MAX_D];
        memcpy(start, incumbent->beta, sizeof(double) * P->d);
        for (int j = 0; j < P->d; ++j) {
            if (j == axis) continue;
            double u = (double)pcg_next(&g) / 4294967296.0;
            double du = -1.0 + (1.0 - -1.0) * u;
            start[j] += du * fmax(1.0, fabs(incumbent->beta[j]));
        }
        orc_point pt;
        locus_value(P, axis, incumbent->t, c.fast_tol, c.fast_sweeps, start, &pt, cnt);
        if (pt.value <= c.best.value + margin) {
            orc_point ref;
            double pb[ORC_MAX_D];
            memcpy(pb, pt.beta, sizeof(double) * P->d);
            locus_value(P, axis, incumbent->t, c.inner_tol, c.inner_sweeps, pb, &ref, cnt);
            if (ref.value < pt.value) pt = ref;
        }
        c.calls += 1;
        curve_append(&c, &pt);
        if (pt.value < c.best.value) c.best = pt;
    }
    double w = width;
    const int probes = 16;
    for (int r = 0; r < 4; ++r) {
        double center = c.best.t;
        double a = center - w, b = center + w;
        double delta = b - a;
        double step = delta / (double)(probes - 1);
        for (int k = 0; k < probes; ++k) {
            double t;
            if (k == probes - 1) t = b;
            else if (step == 0.0) t = ((double)k / (double)(probes - 1)) * delta + a;
            else t = (double)k * step + a;
            curve_eval(&c, t);
        }
        w *= 2.0 / (double)(probes - 1);
    }
    *best_out = c.best;
    *calls_out = c.calls;
    *failures_out = c.failures;
    curve_free(&c);
}

typedef struct {
    double beta[ORC_MAX_D];
    double objective;
    int iterations;
    int objective_evals;
    int converged;
    int status;          /* 0 ok, 1 unbounded direction */
    long long descents;
    long long steps;
} orc_locus_result;

/* locus.solve_locus (locus.py:300-409) */
static void solve_locus(const orc_problem *P, const orc_locus_params *prm, orc_locus_result *res)
{
    orc_counters cnt = {0, 0};
    int axes[ORC_MAX_D], naxes;
    if (prm->outer_axis >= 0) {
        axes[0] = prm->outer_axis;
        naxes = 1;
    } else {
        axes_by_influence(P, axes);
        naxes = P->d;
    }
    orc_point best;
    int has_best = 0, best_axis = axes[0];
    double axis_values[ORC_MAX_D];
    int nvals = 0, rounds = 0, calls = 0, failures = 0, outer_ok = 1, confirmations = 0;
    memset(res, 0, sizeof(*res));
    for (int a = 0; a < naxes; ++a) {
        int axis = axes[a];
        double lo, hi;
        if (prm->has_bracket) { lo = prm->bracket_lo; hi = prm->bracket_hi; }
        else default_bracket(P, &lo, &hi);
        orc_curve c;
        curve_init(&c, P, axis, prm, &cnt);
        if (expand_bracket(&c, &lo, &hi)) {
            curve_free(&c);
            res->status = 1;
            res->descents = cnt.descents;
            res->steps = cnt.steps;
            return;
        }
        int conv;
        int ar = outer_search(&c, lo, hi, prm, &conv);
        orc_point axis_best = c.best;
        axis_values[nvals++] = axis_best.value;
        rounds += ar;
        calls += c.calls;
        failures += c.failures;
        outer_ok = outer_ok && conv;
        curve_free(&c);
        double agree_tol = (P->d > 3 ? 1e-6 : 1e-7) * fmax(1.0, has_best ? fabs(best.value) : 1.0);
        if (!has_best) {
            best = axis_best; best_axis = axis; has_best = 1;
            confirmations = 1;
        } else if (axis_best.value < best.value - agree_tol) {
            best = axis_best; best_axis = axis;
            confirmations = 1;
        } else if (fabs(axis_best.value - best.value) <= agree_tol) {
            confirmations += 1;
        }
        if (P->d > 3 && confirmations >= 2) break;
    }
    if (P->d > 2) {
        double blo, bhi;
        if (prm->has_bracket) { blo = prm->bracket_lo; bhi = prm->bracket_hi; }
        else default_bracket(P, &blo, &bhi);
        double width = 0.01 * (bhi - blo);
        double vmax = axis_values[0], vmin = axis_values[0];
        for (int k = 1; k < nvals; ++k) {
            if (axis_values[k] > vmax) vmax = axis_values[k];
            if (axis_values[k] < vmin) vmin = axis_values[k];
        }
        double spread = vmax - vmin;
        int disagree = spread > 1e-7 * fmax(1.0, fabs(best.value));
        int passes, fan, refine_axes[ORC_MAX_D], nref;
        if (P->d == 3 && disagree) {
            passes = 4; fan = 12; nref = P->d;
            for (int j = 0; j < P->d; ++j) refine_axes[j] = j;
        } else {
            passes = 1; nref = 1; refine_axes[0] = best_axis;
            fan = P->d == 3 ? 0 : 4;
        }
        for (int ps = 0; ps < passes; ++ps) {
            int improved = 0;
            for (int q = 0; q < nref; ++q) {
                int axis = refine_axes[q];
                orc_point seeded = best;
                seeded.t = best.beta[axis];
                seeded.inner_converged = 1;
                seeded.inner_evals = 0;
                orc_point cand;
                int rc, rf;
                dense_refine(P, axis, &seeded, prm, width, fan, &cnt, &cand, &rc, &rf);
                calls += rc;
                failures += rf;
                if (cand.value < best.value - 1e-9 * fmax(1.0, fabs(best.value))) improved = 1;
                if (cand.value < best.value) best = cand;
            }
            if (!improved) break;
        }
    }
    int converged = outer_ok && ((double)failures <= 0.1 * (double)calls);
    orc_descent pol;
    ccd_descend(P, best.beta, -1, prm->inner_sweep_tol, prm->inner_max_sweeps, &pol, &cnt, NULL, NULL);
    const double *beta = pol.objective <= best.value ? pol.beta : best.beta;
    memcpy(res->beta, beta, sizeof(double) * P->d);
    if (P->f32) {
        float bf[ORC_MAX_D];
        for (int j = 0; j < P->d; ++j) bf[j] = (float)res->beta[j];
        res->objective = (double)orc_objective_f32(P->xf, P->yf, P->m, P->d, (float)P->lam, bf);
    } else {
        res->objective = orc_objective(P->x, P->y, P->m, P->d, P->lam, res->beta);
    }
    res->iterations = rounds;
    res->objective_evals = calls;
    res->converged = converged;
    res->status = 0;
    res->descents = cnt.descents;
    res->steps = cnt.steps;
}

/* exported single solve */
int orc_solve_locus(const double *x, const double *y, int m, int d, double lam, const orc_locus_params *prm,
                    double *beta, double *objective, int *iterations, int *objective_evals, int *converged,
                    int *status, long long *descents, long long *steps)
{
    if (m < 1 || d < 1 || m > ORC_MAX_M || d > ORC_MAX_D) return -1;
    orc_problem P = {x, y, m, d, lam};
    orc_locus_result r;
    solve_locus(&P, prm, &r);
    memcpy(beta, r.beta, sizeof(double) * d);
    *objective = r.objective;
    *iterations = r.iterations;
    *objective_evals = r.objective_evals;
    *converged = r.converged;
    *status = r.status;
    if (descents) *descents = r.descents;
    if (steps) *steps = r.steps;
    return 0;
}

/* batched solve across host threads (bench cpu_baseline / --impl reference) */
typedef struct {
    const double *X, *Y, *L;
    const float *Xf, *Yf, *Lf; /* fp32 mode */
    long long B;
    int m, d;
    double lam_floor;
    const orc_locus_params *prm;
    double *beta, *obj;
    int *iters, *evals, *conv, *status;
    long long *descents, *steps;
    long long next;
    pthread_mutex_t mu;
    const double *brackets; /* (B, 2) per-problem initial_bracket or NULL */
} orc_batch;

static void *batch_worker(void *arg)
{
    orc_batch *bt = (orc_batch *)arg;
    for (;;) {
        pthread_mutex_lock(&bt->mu);
        long long b = bt->next++;
        pthread_mutex_unlock(&bt->mu);
        if (b >= bt->B) break;
        orc_problem P;
        memset(&P, 0, sizeof(P));
        P.m = bt->m;
        P.d = bt->d;
        double lraw;
        if (bt->Xf) {
            P.xf = bt->Xf + (size_t)b * bt->m * bt->d;
            P.yf = bt->Yf + (size_t)b * bt->m;
            P.f32 = 1;
            lraw = (double)bt->Lf[b];
        } else {
            P.x = bt->X + (size_t)b * bt->m * bt->d;
            P.y = bt->Y + (size_t)b * bt->m;
            lraw = bt->L[b];
        }
        P.lam = lraw > bt->lam_floor ? lraw : bt->lam_floor;
        orc_locus_result r;
        if (bt->brackets) { /* LocusConfig(initial_bracket=Bracket(lo, hi)) per problem (locus.py:56) */
            orc_locus_params prm = *bt->prm;
            prm.has_bracket = 1;
            prm.bracket_lo = bt->brackets[2 * b];
            prm.bracket_hi = bt->brackets[2 * b + 1];
            if (!(isfinite(prm.bracket_lo) && isfinite(prm.bracket_hi) && prm.bracket_lo < prm.bracket_hi)) {
                /* Bracket() raises InvalidInputError (linesearch.py:85-89): status 2 */
                for (int j = 0; j < bt->d; ++j) bt->beta[(size_t)b * bt->d + j] = NAN;
                bt->obj[b] = NAN;
                bt->iters[b] = bt->evals[b] = bt->conv[b] = 0;
                bt->status[b] = 2;
                if (bt->descents) bt->descents[b] = 0;
                if (bt->steps) bt->steps[b] = 0;
                continue;
            }
            solve_locus(&P, &prm, &r);
        } else {
            solve_locus(&P, bt->prm, &r);
        }
        memcpy(bt->beta + (size_t)b * bt->d, r.beta, sizeof(double) * bt->d);
        bt->obj[b] = r.objective;
        bt->iters[b] = r.iterations;
        bt->evals[b] = r.objective_evals;
        bt->conv[b] = r.converged;
        bt->status[b] = r.status;
        bt->descents[b] = r.descents;
        bt->steps[b] = r.steps;
    }
    return NULL;
}

static int run_batch(orc_batch *bt, int nthreads)
{
    pthread_mutex_init(&bt->mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, batch_worker, bt);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&bt->mu);
    return 0;
}

int orc_solve_locus_batch(const double *X, const double *Y, const double *L, long long B, int m, int d,
                          double lam_floor, const orc_locus_params *prm, int nthreads, double *beta, double *obj,
                          int *iters, int *evals, int *conv, int *status, long long *descents, long long *steps)
{
    if (m < 1 || d < 1 || m > ORC_MAX_M || d > ORC_MAX_D) return -1;
    orc_batch bt = {X, Y, L, NULL, NULL, NULL, B, m, d, lam_floor, prm, beta, obj, iters, evals, conv, status,
                    descents, steps, 0};
    return run_batch(&bt, nthreads);
}

int orc_solve_locus_batch_brackets(const double *X, const double *Y, const double *L, long long B, int m, int d,
                                   double lam_floor, const orc_locus_params *prm, const double *brackets,
                                   int nthreads, double *beta, double *obj, int *iters, int *evals, int *conv,
                                   int *status, long long *descents, long long *steps)
{
    if (m < 1 || d < 1 || m > ORC_MAX_M || d > ORC_MAX_D) return -1;
    orc_batch bt = {X, Y, L, NULL, NULL, NULL, B, m, d, lam_floor, prm, beta, obj, iters, evals, conv, status,
                    descents, steps, 0};
    bt.brackets = brackets;
    return run_batch(&bt, nthreads);
}

/* fp32 mode: binary32 data and descents, binary64 outer search; outputs widened */
int orc_solve_locus_batch_f32(const float *X, const float *Y, const float *L, long long B, int m, int d,
                              double lam_floor, const orc_locus_params *prm, int nthreads, double *beta, double *obj,
                              int *iters, int *evals, int *conv, int *status, long long *descents, long long *steps)
{
    if (m < 1 || d < 1 || m > ORC_MAX_M || d > ORC_MAX_D) return -1;
    orc_batch bt = {NULL, NULL, NULL, X, Y, L, B, m, d, lam_floor, prm, beta, obj, iters, evals, conv, status,
                    descents, steps, 0};
    return run_batch(&bt, nthreads);
}

/* ------------------------------------------------------------------ */
/* brute force (brute.py:29-145)                                        */
/* ------------------------------------------------------------------ */

/* solve_linear_system (brute.py:29-59); returns 0 when singular */
int orc_solve_linear_system(const double *a_in, const double *b_in, int n, double pivot_rtol, double *sol)
{
    double a[ORC_MAX_D][ORC_MAX_D], b[ORC_MAX_D], rn[ORC_MAX_D];
    for (int i = 0; i < n; ++i) {
        b[i] = b_in[i];
        double mx = 0.0;
        for (int c = 0; c < n; ++c) {
            a[i][c] = a_in[i * n + c];
            double v = fabs(a[i][c]);
            if (c == 0 || v > mx) mx = v;
        }
        rn[i] = mx;
    }
    for (int i = 0; i < n; ++i)
        if (rn[i] == 0.0) return 0;
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(a[k][k]) / rn[k];
        for (int i = k + 1; i < n; ++i) {
            double s = fabs(a[i][k]) / rn[i];
            if (s > best) { best = s; p = i; }
        }
        if (fabs(a[p][k]) <= pivot_rtol * rn[p]) return 0;
        if (p != k) {
            for (int c = 0; c < n; ++c) { double t = a[k][c]; a[k][c] = a[p][c]; a[p][c] = t; }
            double t = b[k]; b[k] = b[p]; b[p] = t;
            t = rn[k]; rn[k] = rn[p]; rn[p] = t;
        }
        double f[ORC_MAX_D];
        for (int i = k + 1; i < n; ++i) f[i] = a[i][k] / a[k][k];
        for (int i = k + 1; i < n; ++i)
            for (int c = k; c < n; ++c) a[i][c] = a[i][c] - f[i] * a[k][c];
        for (int i = k + 1; i < n; ++i) b[i] = b[i] - f[i] * b[k];
    }
    for (int k = n - 1; k >= 0; --k) {
        double dot = orc_ddot(&a[k][k + 1], &sol[k + 1], n - 1 - k);
        sol[k] = (b[k] - dot) / a[k][k];
    }
    return 1;
}

static long long comb_count(int n, int k)
{
    if (k < 0 || k > n) return 0;
    long double r = 1;
    if (k > n - k) k = n - k;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return (long long)(r + 0.5);
}

long long orc_candidate_count(int m, int d) { return comb_count(m + d, d); }

/* returns 0 ok, 2 too large (d), 3 too large (count) */
int orc_solve_brute(const double *x, const double *y, int m, int d, double lam, int max_variables,
                    long long max_candidates, double *beta, double *objective, long long *evaluated)
{
    if (d > max_variables) return 2;
    if (comb_count(m + d, d) > max_candidates) return 3;
    if (m > ORC_MAX_M || d > ORC_MAX_D) return -1;
    int N = m + d;
    int idx[ORC_MAX_D];
    for (int i = 0; i < d; ++i) idx[i] = i;
    double best_obj = INFINITY, best_l1 = INFINITY, best_v[ORC_MAX_D];
    int have = 0;
    long long ev = 0;
    for (;;) {
        double a[ORC_MAX_D * ORC_MAX_D], rhs[ORC_MAX_D], sol[ORC_MAX_D];
        for (int r = 0; r < d; ++r) {
            int pl = idx[r];
            for (int c = 0; c < d; ++c)
                a[r * d + c] = pl < m ? x[(size_t)pl * d + c] : (pl - m == c ? 1.0 : 0.0);
            rhs[r] = pl < m ? y[pl] : 0.0;
        }
        if (orc_solve_linear_system(a, rhs, d, 1e-12, sol)) {
            ++ev;
            double obj = orc_objective(x, y, m, d, lam, sol);
            if (!(obj > best_obj)) {
                double l1 = np_sum_abs(sol, d);
                int less = 0;
                if (!have) less = 1;
                else if (obj < best_obj) less = 1;
                else if (obj == best_obj) {
                    if (l1 < best_l1) less = 1;
                    else if (l1 == best_l1) {
                        for (int c = 0; c < d; ++c) {
                            if (sol[c] < best_v[c]) { less = 1; break; }
                            if (sol[c] > best_v[c]) break;
                        }
                    }
                }
                if (less) {
                    best_obj = obj; best_l1 = l1;
                    memcpy(best_v, sol, sizeof(double) * d);
                    have = 1;
                }
            }
        }
        /* next combination (lexicographic) */
        int i = d - 1;
        while (i >= 0 && idx[i] == N - d + i) --i;
        if (i < 0) break;
        ++idx[i];
        for (int k = i + 1; k < d; ++k) idx[k] = idx[k - 1] + 1;
    }
    if (!have) return 4;
    memcpy(beta, best_v, sizeof(double) * d);
    *objective = best_obj;
    *evaluated = ev;
    return 0;
}
