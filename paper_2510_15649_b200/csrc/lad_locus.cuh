// lad_locus.cuh -- batched LAD-LASSO locus solver for sm_100a.
//
// Mapping: one thread per problem (the paper's "one GPU thread per problem",
// north_star), persistent grid, per-lane work stealing through one atomic
// counter.  The reference's nested control flow
//   solve_locus -> axis scan -> expand/ternary/quadrature -> _CurveEvaluator
//   -> locus_value -> ccd_descend -> sweep -> coordinate step
// (locus.py:300-409, :150-297; linesearch.py:172-268; ccd.py:126-206) is
// restated as a resumable state machine (`Ctl`, `controller`) that emits one
// *descent request* at a time.  The kernel's main loop executes exactly one
// coordinate step per iteration for every live lane, so all 32 lanes of a
// warp run the same hot code no matter where each problem is in its solve;
// only the per-descent bookkeeping (residual init, fresh objective, the
// controller) diverges.
//
// Shared memory per warp (interleaved by lane, conflict-free LDS.64):
//   Xs[i][j][lane]  design matrix of the lane's problem
//   Ys[i][lane]     response
//   Ls[i][lane]     unsorted breakpoints of the current step
// Registers: residual r[n], the (key, idx) sort arrays, beta[p].
// Global scratch: per-lane `seen` list of (t, beta) curve points for the
// nearest-point warm start (locus.py:188-191).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lad_numerics.cuh"
#include "lad_sortnet.cuh"

namespace lad {

struct LocusParamsDev {
    int32_t outer_axis;           // -1 = scan all axes by influence
    int32_t outer_search;         // 0 ternary, 1 quadrature
    double outer_tolerance;
    int32_t outer_probes;
    int32_t outer_max_iterations;
    int32_t has_bracket;
    double bracket_lo, bracket_hi;
    double inner_sweep_tol;
    int32_t inner_max_sweeps;
    double lambda_floor;
    int32_t seen_capacity;
};

enum : int { MODE_LOCUS = 0, MODE_DESCENT = 1 };

struct LocusArgs {
    const double *X;        // (Bd, n, p) row-major
    const double *Y;        // (Bd, n)
    const double *lam;      // (B,) raw lambda per problem
    const float *Xf, *Yf, *lamf;  // fp32 mode inputs (warp kernel<float>); X, Y, lam unused then
    const int64_t *data_index;  // (B,) problem -> dataset row, or null (identity)
    int64_t Bd;                 // dataset rows (bounds of data_index; an index outside -> status 2)
    int64_t B;
    int n, p;
    LocusParamsDev prm;
    int mode;
    const double *start;    // MODE_DESCENT: (B, p)
    const int32_t *frozen;  // MODE_DESCENT: (B,) -1 = none
    double desc_tol;        // MODE_DESCENT sweep tolerance
    int desc_sweeps;        // MODE_DESCENT max sweeps
    // outputs
    double *beta;           // (B, p)
    double *objective;      // (B,)
    int32_t *iterations;    // (B,)
    int32_t *objective_evals;
    uint8_t *converged;
    uint8_t *status;        // 0 ok, 1 unbounded direction, 2 invalid input
    int32_t *descents;      // may be null
    int64_t *steps;         // may be null
    // scratch
    double *seen;           // per lane slot: seen_cap * (1 + PMAX) doubles
    int seen_cap;           // curve points kept per evaluator; more -> status 3 (see seen_append)
    const double *brackets; // (B, 2) per-problem initial_bracket (lo, hi), or null (LocusConfig's / default)
    unsigned long long *counter;
    // axis-parallel mode (AXIS_SEARCH: item = problem * p + axis rank)
    int axis_mode;
    double *axis_res;   // (B * p) entries of axis_stride doubles
    int axis_stride;
    unsigned *axis_done;  // (B,) finished axis searches per problem (AXIS_SEARCH); the last one runs the finish
};

template <int PMAX>
struct Point {
    double t;
    double beta[PMAX];
    double value;
    int conv;
};

enum : int {
    PC_FETCH = 0,
    PC_AXIS_START,
    PC_EX_0, PC_EX_1, PC_EX_2, PC_EX_LOOP, PC_EX_MID, PC_EX_NEWLO, PC_EX_NEWHI, PC_EX_BOTH1, PC_EX_BOTH2,
    PC_OT_START, PC_OT_LOOP, PC_OT_V1, PC_OT_V2, PC_OQ_LOOP, PC_OQ_PROBE, PC_OUTER_END,
    PC_AXIS_DONE,
    PC_REFINE_START, PC_REF_AXIS_START, PC_REF_FAN, PC_REF_FAN_AFTER, PC_REF_FAN_REFINED, PC_REF_FAN_FINISH,
    PC_REF_ROUND, PC_REF_GRID_NEXT, PC_REF_AXIS_DONE,
    PC_POLISH, PC_POLISH_AFTER,
    PC_PR_BEGIN, PC_PR_AFTER_COLD, PC_PR_AFTER_WARM, PC_PR_AFTER_FAST_ONLY, PC_PR_REFINE_CHECK,
    PC_PR_AFTER_REFINE, PC_PR_FINISH,
    PC_DESC_AFTER,
    PC_FINISH_AXES,
    PC_AXIS_COUNT,
};

// axis-parallel mode for small batches: the per-axis searches of solve_locus
// share no state (locus.py:223-225), so they run as independent work items;
// a finish pass replays them through the agreement rule in order.
// AXIS_SEARCH: one work item per (problem, axis); the unit that completes a
// problem's last axis search finishes the problem (PC_AXIS_COUNT)
enum : int { AXIS_SERIAL = 0, AXIS_SEARCH = 1 };

// ACT_YIELD (thread kernel, LAD_THREAD_YIELD): the controller stopped at a state every lane passes
// through (the curve evaluator's begin / finish); the caller re-enters it once all lanes of the warp
// that are in the controller have yielded or finished, so those states run converged.
enum : int { ACT_DESCENT = 0, ACT_EXIT = 1, ACT_YIELD = 2 };

template <int PMAX>
struct Ctl {
    // problem
    int64_t prob;
    int arank;  // axis rank of an AXIS_SEARCH item
    int replay; // AXIS_SEARCH: this warp is finishing its problem from the stored axis results
    double lam;
    uint32_t sparse_mask;
    int pc, ret_pc;
    // descent request / result
    double req_start[PMAX];
    int req_frozen;
    double req_tol;
    int req_sweeps;
    double res_beta[PMAX];
    double res_obj;
    int res_conv, res_steps, res_sweeps;
    // probe
    double probe_t, probe_v;
    int warm_idx;
    Point<PMAX> pt;
    // evaluator (_CurveEvaluator)
    int axis, nseen, ev_calls, ev_failures, has_best, seen_over;
    Point<PMAX> ev_best;
    double fast_tol, inner_tol, margin_scale;
    int fast_sweeps, inner_sweeps, economy;
    // solve level
    int axes[PMAX];
    int naxes, a_idx;
    double R_lo, R_hi;
    Point<PMAX> best;
    int best_axis;
    double axis_values[PMAX];
    int nvals, rounds, calls, failures, outer_ok, confirmations;
    // expand / outer
    double lo, hi, g_lo, g_hi, target, m1, m2, v1, h, bt, bv;
    int ex_it, orounds, qk, oconv;
    // refine
    int passes, fan, nref, refine_axes[PMAX], ps, q, improved, fan_i, rr, gk;
    double width, margin, w, ga, gb, gstep, gdelta;
    Point<PMAX> seeded;
    Pcg32 rng;
    // counters
    int D;
    long long S;
    const double *ysrc;  // thread kernel with y read from global memory: the problem's y row
};

// ---------------------------------------------------------------------------
// helpers used by the controller (cold path)
// ---------------------------------------------------------------------------

template <int NMAX, int PMAX>
__device__ __forceinline__ double xs_at(const double *Xs, int i, int j, int lane)
{
    return Xs[(i * PMAX + j) * 32 + lane];
}

// np.abs(x).sum(axis=0)[j]: sequential over rows for d >= 2, pairwise for d == 1
template <int NMAX, int PMAX>
__device__ double col_abs_sum(const double *Xs, int n, int p, int j, int lane)
{
    if (p == 1) return np_sum(n, [&](int i) { return fabs(xs_at<NMAX, PMAX>(Xs, i, 0, lane)); });
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = dadd(s, fabs(xs_at<NMAX, PMAX>(Xs, i, j, lane)));
    return s;
}

template <int NMAX, int PMAX>
__device__ double objective_of(const double *Xs, const double *Yp, int ys, int n, int p, int lane, double lam,
                               const double *b)
{
    double rs = np_sum(n, [&](int i) {
        double g = gemv_row(p, i, n, [&](int jj) { return xs_at<NMAX, PMAX>(Xs, i, jj, lane); },
                            [&](int jj) { return b[jj]; });
        return fabs(dsub(Yp[i * ys], g));
    });
    double bs = np_sum(p, [&](int jj) { return fabs(b[jj]); });
    return dadd(rs, dmul(lam, bs));
}

// The start vector is written through acc.lanes (one element per lane in the
// warp kernel); ISSUE_SEQ writes it sequentially, for starts held in a
// per-thread array (a lane-indexed read of it would go through local memory).
#define ISSUE_TAIL(FROZEN, TOL, SWEEPS, NEXT) \
    C.req_frozen = (FROZEN);                 \
    C.req_tol = (TOL);                       \
    C.req_sweeps = (SWEEPS);                 \
    C.pc = (NEXT);                           \
    return ACT_DESCENT;
#define ISSUE(START_EXPR, FROZEN, TOL, SWEEPS, NEXT)                              \
    do {                                                                          \
        acc.lanes(p, [&](int jj_) { C.req_start[jj_] = (START_EXPR); });          \
        ISSUE_TAIL(FROZEN, TOL, SWEEPS, NEXT)                                     \
    } while (0)
#define ISSUE_SEQ(START_EXPR, FROZEN, TOL, SWEEPS, NEXT)                          \
    do {                                                                          \
        for (int jj_ = 0; jj_ < p; ++jj_) C.req_start[jj_] = (START_EXPR);        \
        ISSUE_TAIL(FROZEN, TOL, SWEEPS, NEXT)                                     \
    } while (0)

#define PROBE(T, RET)                  \
    do {                               \
        C.probe_t = (T);               \
        C.ret_pc = (RET);              \
        if constexpr (AC::kYield) {    \
            C.pc = PC_PR_BEGIN;        \
            return ACT_YIELD;          \
        } else {                       \
            goto L_PC_PR_BEGIN;        \
        }                              \
    } while (0)
#ifndef LAD_THREAD_YIELD_FINISH  // yield before the evaluator's finish state
#define LAD_THREAD_YIELD_FINISH 0
#endif
#ifndef LAD_THREAD_YIELD_RET     // yield after it, before the probe's caller resumes
#define LAD_THREAD_YIELD_RET 1
#endif
#define PROBE_FINISH()                 \
    do {                               \
        if constexpr (AC::kYield && LAD_THREAD_YIELD_FINISH) {    \
            C.pc = PC_PR_FINISH;       \
            return ACT_YIELD;          \
        } else {                       \
            goto L_PC_PR_FINISH;       \
        }                              \
    } while (0)

template <int PMAX, class AC>
__device__ __forceinline__ void set_point_from_result(const AC &acc, Ctl<PMAX> &C, Point<PMAX> &P, double t, int p)
{
    P.t = t;
    P.value = C.res_obj;
    P.conv = C.res_conv;
    acc.lanes(p, [&](int j) { P.beta[j] = C.res_beta[j]; });
}

template <int PMAX, class AC>
__device__ __forceinline__ void seen_append(const AC &acc, const LocusArgs &A, double *seen, Ctl<PMAX> &C,
                                            const Point<PMAX> &P, int p)
{
    if (seen == nullptr) return;
    int k = C.nseen;
    if (k >= A.seen_cap) {  // capacity exceeded: the nearest-point scan would be incomplete, so the
        C.seen_over = 1;    // problem ends with status 3 instead of a silently different warm start
        return;
    }
    double *sb = seen + A.seen_cap + (size_t)k * PMAX;
    acc.lanes_out(1 + p, [&](int q) {
        if (q == 0) seen[k] = P.t;
        else sb[q - 1] = P.beta[q - 1];
    });
    C.nseen = k + 1;
}

template <int PMAX>
__device__ __forceinline__ void evaluator_reset(Ctl<PMAX> &C, int axis, const LocusArgs &A, int p)
{
    C.axis = axis;
    C.nseen = 0;
    C.ev_calls = 0;
    C.ev_failures = 0;
    C.has_best = 0;
    C.economy = p > 3;
    double tol = A.prm.inner_sweep_tol;
    int ms = A.prm.inner_max_sweeps;
    C.inner_tol = tol;
    C.inner_sweeps = C.economy ? (ms < 150 ? ms : 150) : ms;
    C.fast_tol = tol > 1e-7 ? tol : 1e-7;
    int cap = C.economy ? 40 : 150;
    C.fast_sweeps = ms < cap ? ms : cap;
    C.margin_scale = C.economy ? 1e-4 : 1e-3;
}

template <int PMAX>
__device__ __forceinline__ void write_invalid(const LocusArgs &A, int64_t pr, int p)
{
    for (int j = 0; j < p; ++j) A.beta[(size_t)pr * p + j] = __longlong_as_double(0x7ff8000000000000LL);
    A.objective[pr] = __longlong_as_double(0x7ff8000000000000LL);
    A.iterations[pr] = 0;
    A.objective_evals[pr] = 0;
    A.converged[pr] = 0;
    A.status[pr] = 2;
    if (A.descents) A.descents[pr] = 0;
    if (A.steps) A.steps[pr] = 0;
}

// UnboundedDirectionError for the problem in C: counters as of the failing axis
template <int PMAX>
__device__ __forceinline__ void write_unbounded(const LocusArgs &A, const Ctl<PMAX> &C, int p, bool leader)
{
    if (!leader) return;
    const int64_t pr = C.prob;
    for (int j = 0; j < p; ++j) A.beta[(size_t)pr * p + j] = __longlong_as_double(0x7ff8000000000000LL);
    A.objective[pr] = __longlong_as_double(0x7ff8000000000000LL);
    A.iterations[pr] = C.rounds;
    A.objective_evals[pr] = C.calls;
    A.converged[pr] = 0;
    A.status[pr] = 1;
    if (A.descents) A.descents[pr] = C.D;
    if (A.steps) A.steps[pr] = C.S;
}

// first minimal |seen_t[k] - t| (locus.py:188-191), 8 loads in flight
__device__ __forceinline__ int nearest_serial(const double *seen, int lim, double t)
{
    int wi = -1;
    double bd = __longlong_as_double(0x7ff0000000000000LL);
    int k = 0;
    for (; k + 8 <= lim; k += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = seen[k + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            double dd = fabs(dsub(v[q], t));
            if (dd < bd) {
                bd = dd;
                wi = k + q;
            }
        }
    }
    for (; k < lim; ++k) {
        double dd = fabs(dsub(seen[k], t));
        if (dd < bd) {
            bd = dd;
            wi = k;
        }
    }
    return wi;
}

// Access policy of the thread-per-problem kernel: the lane owns its problem;
// data lives in the lane's column of the interleaved shared arrays.
// Thread kernel: the controller yields at the curve evaluator's begin / finish states and is
// re-entered with the warp's controller lanes converged (ACT_YIELD), so those states, which every
// lane passes through on its own path, execute once per round instead of once per diverged group.
#ifndef LAD_THREAD_YIELD
#define LAD_THREAD_YIELD 1
#endif
template <int NMAX, int PMAX>
struct ThreadAccess {
    static constexpr bool kYield = LAD_THREAD_YIELD != 0;
    int n, p, lane;
    double *Xs, *Ys;
    double *Tw;  // per axis: sum of the breakpoint weights (|x_ij| and lambda), any order (median guess test)
    double *RX;  // RN(1 / x_ij), same layout as Xs (division by reciprocal), or null
    float *Sc;   // per axis: 2^30 / (sum of the breakpoint weights), the fixed-point weight scale (rank-sum median), or null
    __device__ __forceinline__ bool leader() const { return true; }
    __device__ __forceinline__ void sync() const {}
    // this slot's curve-point scratch (seen list), null when unused (p <= 2)
    template <int PM>
    __device__ __forceinline__ double *seen_base(const LocusArgs &A, int slot) const
    {
        return (A.seen != nullptr && p > 2) ? A.seen + (size_t)slot * A.seen_cap * (1 + PM) : nullptr;
    }
    // element-wise work on controller vectors: f(k) for k < cnt (Ctl fields / outputs)
    template <class F>
    __device__ __forceinline__ void lanes(int cnt, F f) const
    {
        for (int k = 0; k < cnt; ++k) f(k);
    }
    template <class F>
    __device__ __forceinline__ void lanes_out(int cnt, F f) const
    {
        for (int k = 0; k < cnt; ++k) f(k);
    }
    template <int PM>
    __device__ __forceinline__ void copy_point(Point<PM> &d, const Point<PM> &s) const
    {
        d = s;
    }
    // count one finished unit on *ctr; true for the caller that completes `of` units
    __device__ __forceinline__ bool last_of(unsigned *ctr, unsigned of) const
    {
        __threadfence();
        const bool last = atomicAdd(ctr, 1u) == of - 1u;
        __threadfence();
        return last;
    }
    __device__ __forceinline__ int fetch(Ctl<PMAX> &C, const LocusArgs &A) const
    {
        const int div = A.axis_mode == AXIS_SEARCH ? p : 1;
        unsigned long long item = atomicAdd(A.counter, 1ULL);
        if ((int64_t)item >= A.B * div) return -1;
        const unsigned long long pr = item / div;
        C.prob = (int64_t)pr;
        C.arank = (int)(item % div);
        int64_t src = A.data_index ? A.data_index[pr] : (int64_t)pr;
        if (src < 0 || src >= A.Bd) {  // data_index out of range: invalid input
            C.lam = A.prm.lambda_floor;
            C.sparse_mask = 0;
            write_invalid<PMAX>(A, (int64_t)pr, p);
            return 0;
        }
        const double *xg = A.X + (size_t)src * n * p;
        const double *yg = A.Y + (size_t)src * n;
        bool ok = true;
        uint32_t mask = 0;
        for (int i = 0; i < n; ++i) {
            double yv = yg[i];
            ok = ok && isfinite(yv);
            if (Ys != nullptr) Ys[i * 32 + lane] = yv;
            for (int j = 0; j < p; ++j) {
                double xv = xg[i * p + j];
                ok = ok && isfinite(xv);
                if (xv == 0.0) mask |= 1u << j;
                Xs[(i * PMAX + j) * 32 + lane] = xv;
                if (RX != nullptr) {
                    RX[(i * PMAX + j) * 32 + lane] = rcp_rn(xv);
                    if (!div_operand_safe(xv)) mask |= 1u << j;  // the column takes the generic path (IEEE division)
                }
            }
        }
        double lraw = A.lam[pr];
        ok = ok && isfinite(lraw) && lraw >= 0.0;
        C.lam = lraw > A.prm.lambda_floor ? lraw : A.prm.lambda_floor;
        C.sparse_mask = mask;
        C.ysrc = yg;
        if (Tw != nullptr)
            for (int j = 0; j < p; ++j) {
                double s = C.lam;
                for (int i = 0; i < n; ++i) s += fabs(Xs[(i * PMAX + j) * 32 + lane]);
                Tw[j * 32 + lane] = s;
            }
        if (Sc != nullptr)
            for (int j = 0; j < p; ++j) {  // any summation order and any rounding of the scale will do (step_dense)
                double s = C.lam;
                for (int i = 0; i < n; ++i) s += fabs(Xs[(i * PMAX + j) * 32 + lane]);
                // (a total so small or large that the binary32 scale leaves its finite range accepts
                // nothing: every step of that axis then takes the exact order)
                const float scf = (float)(1073741824.0 / (s * (1.0 + 1e-6)));
                Sc[j * 32 + lane] = (s > 0.0 && s < 1e300 && scf > 0.0f && scf < 3.0e38f) ? scf : 0.0f;
            }
        if (!ok) {
            write_invalid<PMAX>(A, (int64_t)pr, p);
            return 0;
        }
        return 1;
    }
    __device__ double col_abs_sum(int j) const { return lad::col_abs_sum<NMAX, PMAX>(Xs, n, p, j, lane); }
    __device__ double y_absmax(const double *ysrc) const
    {
        double ymax = 0.0;
        for (int i = 0; i < n; ++i) {
            double a = fabs(Ys != nullptr ? Ys[i * 32 + lane] : __ldg(ysrc + i));
            if (i == 0 || a > ymax) ymax = a;
        }
        return ymax;
    }
    __device__ int nearest(const double *seen, int lim, double t) const { return nearest_serial(seen, lim, t); }
};

// ---------------------------------------------------------------------------
// controller: advances the lane's state machine until the next descent
// ---------------------------------------------------------------------------
// AC (access policy) supplies everything that depends on how a problem is
// mapped onto threads: fetching the next problem, column sums, the y range,
// the nearest-seen-point scan, and which thread writes shared results.  The
// controller itself is the same for the thread-per-problem and the
// warp-per-problem kernels (in the latter all 32 lanes run it in lock-step
// on a shared Ctl, with identical values).  C.pc is the state to resume at
// after a descent (set by ISSUE) and after a probe (ret_pc); every other
// transition is a direct jump to the next state's label, not a round trip
// through the state switch.
template <int PMAX, class AC>
__device__ __forceinline__ int controller_body(Ctl<PMAX> &C, const LocusArgs &A, const AC &acc, int slot)
{
    const int n = acc.n;
    const int p = acc.p;
    double *seen = acc.template seen_base<PMAX>(A, slot);
    for (;;) {
        acc.sync();
        if constexpr (AC::kYield) {
            // the states a re-entry usually resumes at, by compare-and-branch: the switch's jump
            // table costs a dependent constant load and an indirect branch per round
            int pc = C.pc;
            asm volatile("" : "+r"(pc));  // opaque: otherwise the compiler folds the chain back into the jump table
            if (pc == PC_PR_BEGIN) goto L_PC_PR_BEGIN;
            if (pc == PC_PR_FINISH) goto L_PC_PR_FINISH;
            if (pc == PC_PR_AFTER_COLD) goto L_PC_PR_AFTER_COLD;
            if (pc == PC_PR_AFTER_REFINE) goto L_PC_PR_AFTER_REFINE;
            if (pc == PC_OT_V1) goto L_PC_OT_V1;
            if (pc == PC_OT_V2) goto L_PC_OT_V2;
            if (pc == PC_OQ_PROBE) goto L_PC_OQ_PROBE;
        }
        switch (C.pc) {
        L_PC_FETCH:
        case PC_FETCH: {
            int got = acc.fetch(C, A);
            if (got < 0) return ACT_EXIT;
            C.D = 0;
            C.S = 0;
            C.replay = 0;
            C.seen_over = 0;
            if (got == 0) goto L_PC_FETCH;  // invalid problem: status written, fetch the next one
            const int64_t pr = C.prob;
            if (A.mode == MODE_DESCENT) {
                const double *st = A.start + (size_t)pr * p;
                int fr = A.frozen ? A.frozen[pr] : -1;
                ISSUE(st[jj_], fr, A.desc_tol, A.desc_sweeps, PC_DESC_AFTER);
            }
            // axes_by_influence (locus.py:90-93) and default_bracket (:96-101)
            double infl[PMAX];
            double scale = 0.0;
            for (int j = 0; j < p; ++j) {
                double s = acc.col_abs_sum(j);
                infl[j] = s;
                double mean = ddiv(s, (double)n);
                if (j == 0 || mean > scale) scale = mean;
            }
            if (A.prm.outer_axis >= 0) {
                C.axes[0] = A.prm.outer_axis;
                C.naxes = 1;
            } else {
                for (int j = 0; j < p; ++j) {
                    int k = j;
                    while (k > 0 && -infl[C.axes[k - 1]] > -infl[j]) {
                        C.axes[k] = C.axes[k - 1];
                        --k;
                    }
                    C.axes[k] = j;
                }
                C.naxes = p;
            }
            if (A.brackets) {  // per-problem initial_bracket (Bracket validation, linesearch.py:85-89)
                const double blo = A.brackets[2 * pr], bhi = A.brackets[2 * pr + 1];
                if (!(isfinite(blo) && isfinite(bhi) && blo < bhi)) {
                    if (acc.leader()) write_invalid<PMAX>(A, pr, p);
                    goto L_PC_FETCH;
                }
                C.R_lo = blo;
                C.R_hi = bhi;
            } else if (A.prm.has_bracket) {
                C.R_lo = A.prm.bracket_lo;
                C.R_hi = A.prm.bracket_hi;
            } else {
                double ymax = acc.y_absmax(C.ysrc);
                double radius = scale > 0.0 ? ddiv(ymax, scale) : __longlong_as_double(0x7ff0000000000000LL);
                if (!isfinite(radius) || radius <= 0.0) radius = 1.0;
                C.R_lo = -radius;
                C.R_hi = radius;
            }
            C.a_idx = 0;
            C.best_axis = C.axes[0];
            C.nvals = C.rounds = C.calls = C.failures = 0;
            C.outer_ok = 1;
            C.confirmations = 0;
            if (A.axis_mode == AXIS_SEARCH) {  // this item is one axis search of the problem
                if (C.arank >= C.naxes) goto L_PC_FETCH;
                C.a_idx = C.arank;
            }
            goto L_PC_AXIS_START;
        }
        // axis-parallel finish: replay the stored per-axis results in influence
        // order through the same agreement rule (locus.py:338-362)
        L_PC_FINISH_AXES:
        case PC_FINISH_AXES: {
            // written by other warps of this launch (fused finish): read through L2
            const double *res = A.axis_res + ((size_t)C.prob * p + C.a_idx) * A.axis_stride;
            C.axis = C.axes[C.a_idx];
            C.ev_best.t = __ldcg(res + 0);
            for (int j = 0; j < p; ++j) C.ev_best.beta[j] = __ldcg(res + 1 + j);
            C.ev_best.value = __ldcg(res + 1 + PMAX);
            C.ev_best.conv = (int)__ldcg(res + 2 + PMAX);
            C.orounds = (int)__ldcg(res + 3 + PMAX);
            C.ev_calls = (int)__ldcg(res + 4 + PMAX);
            C.ev_failures = (int)__ldcg(res + 5 + PMAX);
            C.oconv = (int)__ldcg(res + 6 + PMAX);
            C.seen_over |= (int)__ldcg(res + 9 + PMAX);
            C.D += (int)__ldcg(res + 7 + PMAX);
            C.S += (long long)__ldcg(res + 8 + PMAX);
            if (C.oconv < 0) {  // this axis' bracket expansion failed: raise here, as the serial scan does
                write_unbounded<PMAX>(A, C, p, acc.leader());
                goto L_PC_FETCH;
            }
            goto L_PC_AXIS_DONE;
        }
        // The unit that completes a problem's last axis search replays all of
        // them through the agreement rule, refine and polish right away: the
        // finish of one problem overlaps the other problems' searches, and the
        // problem is still loaded.  Same states as a separate finish pass.
        L_PC_AXIS_COUNT:
        case PC_AXIS_COUNT: {
            const bool last = acc.last_of(A.axis_done + C.prob, (unsigned)C.naxes);
            acc.sync();
            if (!last) {
                goto L_PC_FETCH;
            }
            C.replay = 1;
            C.a_idx = 0;
            C.best_axis = C.axes[0];
            C.nvals = C.rounds = C.calls = C.failures = 0;
            C.outer_ok = 1;
            C.confirmations = 0;
            C.D = 0;  // the replay adds every axis' D and S
            C.S = 0;
            C.seen_over = 0;
            acc.sync();
            goto L_PC_FINISH_AXES;
        }
        case PC_DESC_AFTER: {
            int64_t pr = C.prob;
            if (acc.leader()) {
            for (int j = 0; j < p; ++j) A.beta[(size_t)pr * p + j] = C.res_beta[j];
            A.objective[pr] = C.res_obj;
            A.iterations[pr] = C.res_sweeps;
            A.objective_evals[pr] = C.res_steps;
            A.converged[pr] = (uint8_t)C.res_conv;
            A.status[pr] = 0;
            if (A.descents) A.descents[pr] = C.D;
            if (A.steps) A.steps[pr] = C.S;
            }
            goto L_PC_FETCH;
        }
        // ------------------------------------------------ axis search
        L_PC_AXIS_START:
        case PC_AXIS_START: {
            evaluator_reset(C, C.axes[C.a_idx], A, p);
            C.lo = C.R_lo;
            C.hi = C.R_hi;
            goto L_PC_EX_0;
        }
        // expand_bracket (linesearch.py:247-268)
        L_PC_EX_0:
        case PC_EX_0: PROBE(C.lo, PC_EX_1);
        case PC_EX_1: C.g_lo = C.probe_v; PROBE(C.hi, PC_EX_2);
        case PC_EX_2: C.g_hi = C.probe_v; C.ex_it = 0; goto L_PC_EX_LOOP;
        L_PC_EX_LOOP:
        case PC_EX_LOOP: {
            if (C.ex_it >= 60) {  // UnboundedDirectionError (linesearch.py:266)
                if (A.axis_mode == AXIS_SEARCH && !C.replay) {
                    // record it; the finish raises it when this axis' turn comes
                    if (acc.leader()) {
                        double *res = A.axis_res + ((size_t)C.prob * p + C.a_idx) * A.axis_stride;
                        res[6 + PMAX] = -1.0;
                        res[7 + PMAX] = C.D;
                        res[8 + PMAX] = (double)C.S;
                        res[9 + PMAX] = C.seen_over;
                    }
                    goto L_PC_AXIS_COUNT;
                }
                write_unbounded<PMAX>(A, C, p, acc.leader());
                goto L_PC_FETCH;
            }
            PROBE(dmul(0.5, dadd(C.lo, C.hi)), PC_EX_MID);
        }
        case PC_EX_MID: {
            double g_mid = C.probe_v;
            if (g_mid < C.g_lo && g_mid < C.g_hi) {
                goto L_PC_OT_START;
            }
            double step = dmul(1.0, dsub(C.hi, C.lo));
            if (C.g_lo < C.g_hi) {
                C.lo = dsub(C.lo, step);
                PROBE(C.lo, PC_EX_NEWLO);
            } else if (C.g_hi < C.g_lo) {
                C.hi = dadd(C.hi, step);
                PROBE(C.hi, PC_EX_NEWHI);
            } else {
                C.lo = dsub(C.lo, step);
                C.hi = dadd(C.hi, step);
                PROBE(C.lo, PC_EX_BOTH1);
            }
        }
        case PC_EX_NEWLO: C.g_lo = C.probe_v; C.ex_it++; goto L_PC_EX_LOOP;
        case PC_EX_NEWHI: C.g_hi = C.probe_v; C.ex_it++; goto L_PC_EX_LOOP;
        case PC_EX_BOTH1: C.g_lo = C.probe_v; PROBE(C.hi, PC_EX_BOTH2);
        case PC_EX_BOTH2: C.g_hi = C.probe_v; C.ex_it++; goto L_PC_EX_LOOP;
        // ternary_min / quadrature_min (linesearch.py:172-233)
        L_PC_OT_START:
        case PC_OT_START: {
            C.target = dmul(A.prm.outer_tolerance, dsub(C.hi, C.lo));
            C.orounds = 0;
            PROBE(dmul(0.5, dadd(C.lo, C.hi)), A.prm.outer_search == 0 ? PC_OT_LOOP : PC_OQ_LOOP);
        }
        L_PC_OT_LOOP:
        case PC_OT_LOOP: {
            if (dsub(C.hi, C.lo) > C.target && C.orounds < A.prm.outer_max_iterations) {
                double third = ddiv(dsub(C.hi, C.lo), 3.0);
                C.m1 = dadd(C.lo, third);
                C.m2 = dsub(C.hi, third);
                PROBE(C.m1, PC_OT_V1);
            }
            PROBE(dmul(0.5, dadd(C.lo, C.hi)), PC_OUTER_END);
        }
        L_PC_OT_V1:
        case PC_OT_V1: C.v1 = C.probe_v; PROBE(C.m2, PC_OT_V2);
        L_PC_OT_V2:
        case PC_OT_V2: {
            if (C.v1 < C.probe_v) C.hi = C.m2;
            else C.lo = C.m1;
            C.orounds++;
            goto L_PC_OT_LOOP;
        }
        L_PC_OQ_LOOP:
        case PC_OQ_LOOP: {
            if (dsub(C.hi, C.lo) > C.target && C.orounds < A.prm.outer_max_iterations) {
                C.h = ddiv(dsub(C.hi, C.lo), (double)(A.prm.outer_probes + 1));
                C.qk = 1;
                PROBE(dadd(C.lo, dmul(C.h, 1.0)), PC_OQ_PROBE);
            }
            PROBE(dmul(0.5, dadd(C.lo, C.hi)), PC_OUTER_END);
        }
        L_PC_OQ_PROBE:
        case PC_OQ_PROBE: {
            double t = dadd(C.lo, dmul(C.h, (double)C.qk));
            if (C.qk == 1 || C.probe_v < C.bv) {
                C.bv = C.probe_v;
                C.bt = t;
            }
            C.qk++;
            if (C.qk <= A.prm.outer_probes) PROBE(dadd(C.lo, dmul(C.h, (double)C.qk)), PC_OQ_PROBE);
            double nlo = dsub(C.bt, C.h), nhi = dadd(C.bt, C.h);
            C.lo = nlo > C.lo ? nlo : C.lo;
            C.hi = nhi < C.hi ? nhi : C.hi;
            C.orounds++;
            goto L_PC_OQ_LOOP;
        }
        case PC_OUTER_END: {
            C.oconv = dsub(C.hi, C.lo) <= C.target;
            goto L_PC_AXIS_DONE;
        }
        // axis agreement bookkeeping (locus.py:338-362)
        L_PC_AXIS_DONE:
        case PC_AXIS_DONE: {
            if (A.axis_mode == AXIS_SEARCH && !C.replay) {  // store this axis' result; the finish combines them
                if (acc.leader()) {
                    double *res = A.axis_res + ((size_t)C.prob * p + C.a_idx) * A.axis_stride;
                    res[0] = C.ev_best.t;
                    for (int j = 0; j < p; ++j) res[1 + j] = C.ev_best.beta[j];
                    res[1 + PMAX] = C.ev_best.value;
                    res[2 + PMAX] = C.ev_best.conv;
                    res[3 + PMAX] = C.orounds;
                    res[4 + PMAX] = C.ev_calls;
                    res[5 + PMAX] = C.ev_failures;
                    res[6 + PMAX] = C.oconv;
                    res[7 + PMAX] = C.D;
                    res[8 + PMAX] = (double)C.S;
                    res[9 + PMAX] = C.seen_over;
                }
                goto L_PC_AXIS_COUNT;
            }
            Point<PMAX> &ab = C.ev_best;
            C.axis_values[C.nvals++] = ab.value;
            C.rounds += C.orounds;
            C.calls += C.ev_calls;
            C.failures += C.ev_failures;
            C.outer_ok = C.outer_ok && C.oconv;
            double agree = dmul(p > 3 ? 1e-6 : 1e-7, C.a_idx == 0 ? 1.0 : fmax(1.0, fabs(C.best.value)));
            bool brk = false;
            if (C.a_idx == 0) {
                acc.copy_point(C.best, ab);
                C.best_axis = C.axis;
                C.confirmations = 1;
            } else if (ab.value < dsub(C.best.value, agree)) {
                acc.copy_point(C.best, ab);
                C.best_axis = C.axis;
                C.confirmations = 1;
            } else if (fabs(dsub(ab.value, C.best.value)) <= agree) {
                C.confirmations += 1;
            }
            if (p > 3 && C.confirmations >= 2) brk = true;
            C.a_idx++;
            if (brk || C.a_idx >= C.naxes) goto L_PC_REFINE_START;
            if (A.axis_mode != AXIS_SERIAL) goto L_PC_FINISH_AXES;
            goto L_PC_AXIS_START;
        }
        // dense refinement plan (locus.py:363-395)
        L_PC_REFINE_START:
        case PC_REFINE_START: {
            if (p <= 2) {
                goto L_PC_POLISH;
            }
            C.width = dmul(0.01, dsub(C.R_hi, C.R_lo));
            double vmax = C.axis_values[0], vmin = C.axis_values[0];
            for (int k = 1; k < C.nvals; ++k) {
                if (C.axis_values[k] > vmax) vmax = C.axis_values[k];
                if (C.axis_values[k] < vmin) vmin = C.axis_values[k];
            }
            double spread = dsub(vmax, vmin);
            bool disagree = spread > dmul(1e-7, fmax(1.0, fabs(C.best.value)));
            if (p == 3 && disagree) {
                C.passes = 4;
                C.fan = 12;
                C.nref = p;
                for (int j = 0; j < p; ++j) C.refine_axes[j] = j;
            } else {
                C.passes = 1;
                C.nref = 1;
                C.refine_axes[0] = C.best_axis;
                C.fan = p == 3 ? 0 : 4;
            }
            C.ps = 0;
            C.q = 0;
            C.improved = 0;
            goto L_PC_REF_AXIS_START;
        }
        L_PC_REF_AXIS_START:
        case PC_REF_AXIS_START: {
            int axis = C.refine_axes[C.q];
            evaluator_reset(C, axis, A, p);
            acc.copy_point(C.seeded, C.best);
            C.seeded.t = C.best.beta[axis];
            C.seeded.conv = 1;
            seen_append(acc, A, seen, C, C.seeded, p);
            acc.copy_point(C.ev_best, C.seeded);
            C.has_best = 1;
            C.margin = dmul(C.margin_scale, fmax(1.0, fabs(C.seeded.value)));
            C.rng.seed(0x5EEDULL + (uint64_t)axis, 54);
            C.fan_i = 0;
            goto L_PC_REF_FAN;
        }
        L_PC_REF_FAN:
        case PC_REF_FAN: {
            if (C.fan_i < C.fan) {
                double st[PMAX];
                for (int j = 0; j < p; ++j) {
                    st[j] = C.seeded.beta[j];
                    if (j == C.axis) continue;
                    double u = ddiv((double)C.rng.next(), 4294967296.0);
                    double du = dadd(-1.0, dmul(dsub(1.0, -1.0), u));
                    st[j] = dadd(st[j], dmul(du, fmax(1.0, fabs(C.seeded.beta[j]))));
                }
                st[C.axis] = C.seeded.t;
                ISSUE_SEQ(st[jj_], C.axis, C.fast_tol, C.fast_sweeps, PC_REF_FAN_AFTER);
            }
            C.w = C.width;
            C.rr = 0;
            goto L_PC_REF_ROUND;
        }
        case PC_REF_FAN_AFTER: {
            set_point_from_result(acc, C, C.pt, C.seeded.t, p);
            if (C.pt.value <= dadd(C.ev_best.value, C.margin)) {
                double tt = C.seeded.t;
                ISSUE(jj_ == C.axis ? tt : C.pt.beta[jj_], C.axis, C.inner_tol, C.inner_sweeps, PC_REF_FAN_REFINED);
            }
            goto L_PC_REF_FAN_FINISH;
        }
        case PC_REF_FAN_REFINED: {
            if (C.res_obj < C.pt.value) set_point_from_result(acc, C, C.pt, C.seeded.t, p);
            goto L_PC_REF_FAN_FINISH;
        }
        L_PC_REF_FAN_FINISH:
        case PC_REF_FAN_FINISH: {
            C.ev_calls++;
            seen_append(acc, A, seen, C, C.pt, p);
            if (C.pt.value < C.ev_best.value) acc.copy_point(C.ev_best, C.pt);
            C.fan_i++;
            goto L_PC_REF_FAN;
        }
        L_PC_REF_ROUND:
        case PC_REF_ROUND: {
            if (C.rr < 4) {
                double center = C.ev_best.t;
                C.ga = dsub(center, C.w);
                C.gb = dadd(center, C.w);
                C.gdelta = dsub(C.gb, C.ga);
                C.gstep = ddiv(C.gdelta, 15.0);
                C.gk = 0;
                PROBE(C.gstep == 0.0 ? dadd(dmul(ddiv(0.0, 15.0), C.gdelta), C.ga) : dadd(dmul(0.0, C.gstep), C.ga),
                      PC_REF_GRID_NEXT);
            }
            goto L_PC_REF_AXIS_DONE;
        }
        case PC_REF_GRID_NEXT: {
            C.gk++;
            if (C.gk < 16) {
                double t;
                if (C.gk == 15) t = C.gb;
                else if (C.gstep == 0.0) t = dadd(dmul(ddiv((double)C.gk, 15.0), C.gdelta), C.ga);
                else t = dadd(dmul((double)C.gk, C.gstep), C.ga);
                PROBE(t, PC_REF_GRID_NEXT);
            }
            C.w = dmul(C.w, 2.0 / 15.0);
            C.rr++;
            goto L_PC_REF_ROUND;
        }
        L_PC_REF_AXIS_DONE:
        case PC_REF_AXIS_DONE: {
            Point<PMAX> &cand = C.ev_best;
            C.calls += C.ev_calls;
            C.failures += C.ev_failures;
            if (cand.value < dsub(C.best.value, dmul(1e-9, fmax(1.0, fabs(C.best.value))))) C.improved = 1;
            if (cand.value < C.best.value) acc.copy_point(C.best, cand);
            C.q++;
            if (C.q < C.nref) {
                goto L_PC_REF_AXIS_START;
            }
            C.ps++;
            if (!C.improved || C.ps >= C.passes) {
                goto L_PC_POLISH;
            }
            C.q = 0;
            C.improved = 0;
            goto L_PC_REF_AXIS_START;
        }
        // final snap (locus.py:396-409)
        L_PC_POLISH:
        case PC_POLISH:
            ISSUE(C.best.beta[jj_], -1, A.prm.inner_sweep_tol, A.prm.inner_max_sweeps, PC_POLISH_AFTER);
        case PC_POLISH_AFTER: {
            int64_t pr = C.prob;
            bool use_pol = C.res_obj <= C.best.value;
            if (C.seen_over) {  // scratch capacity exceeded (see seen_append): status 3, counters kept
                if (acc.leader()) {
                    write_invalid<PMAX>(A, pr, p);
                    A.status[pr] = 3;
                    A.iterations[pr] = C.rounds;
                    A.objective_evals[pr] = C.calls;
                    if (A.descents) A.descents[pr] = C.D;
                    if (A.steps) A.steps[pr] = C.S;
                }
                goto L_PC_FETCH;
            }
            if (acc.leader()) {
            for (int j = 0; j < p; ++j) A.beta[(size_t)pr * p + j] = use_pol ? C.res_beta[j] : C.best.beta[j];
            A.objective[pr] = use_pol ? C.res_obj : C.best.value;
            A.iterations[pr] = C.rounds;
            A.objective_evals[pr] = C.calls;
            A.converged[pr] = (uint8_t)(C.outer_ok && ((double)C.failures <= dmul(0.1, (double)C.calls)));
            A.status[pr] = 0;
            if (A.descents) A.descents[pr] = C.D;
            if (A.steps) A.steps[pr] = C.S;
            }
            goto L_PC_FETCH;
        }
        // ------------------------------------------------ curve evaluator call
        L_PC_PR_BEGIN:
        case PC_PR_BEGIN: {
            double t = C.probe_t;
            int wi = -1;
            if (seen != nullptr && C.nseen > 0) wi = acc.nearest(seen, C.nseen < A.seen_cap ? C.nseen : A.seen_cap, t);
            C.warm_idx = wi;
            const double *wb = wi >= 0 ? seen + A.seen_cap + (size_t)wi * PMAX : nullptr;
            if (C.economy && wi >= 0) ISSUE(jj_ == C.axis ? t : wb[jj_], C.axis, C.fast_tol, C.fast_sweeps,
                                            PC_PR_AFTER_FAST_ONLY);
            ISSUE(jj_ == C.axis ? t : 0.0, C.axis, C.fast_tol, C.fast_sweeps, PC_PR_AFTER_COLD);
        }
        L_PC_PR_AFTER_COLD:
        case PC_PR_AFTER_COLD: {
            set_point_from_result(acc, C, C.pt, C.probe_t, p);
            if (C.warm_idx >= 0 && p > 2) {
                const double *wb = seen + A.seen_cap + (size_t)C.warm_idx * PMAX;
                double t = C.probe_t;
                ISSUE(jj_ == C.axis ? t : wb[jj_], C.axis, C.fast_tol, C.fast_sweeps, PC_PR_AFTER_WARM);
            }
            goto L_PC_PR_REFINE_CHECK;
        }
        case PC_PR_AFTER_WARM: {
            if (C.res_obj < C.pt.value) set_point_from_result(acc, C, C.pt, C.probe_t, p);
            goto L_PC_PR_REFINE_CHECK;
        }
        case PC_PR_AFTER_FAST_ONLY: {
            set_point_from_result(acc, C, C.pt, C.probe_t, p);
            goto L_PC_PR_REFINE_CHECK;
        }
        L_PC_PR_REFINE_CHECK:
        case PC_PR_REFINE_CHECK: {
            bool refine = !C.has_best ||
                          C.pt.value <= dadd(C.ev_best.value, dmul(C.margin_scale, fmax(1.0, fabs(C.ev_best.value))));
            if (refine) {
                double t = C.probe_t;
                ISSUE(jj_ == C.axis ? t : C.pt.beta[jj_], C.axis, C.inner_tol, C.inner_sweeps, PC_PR_AFTER_REFINE);
            }
            PROBE_FINISH();
        }
        L_PC_PR_AFTER_REFINE:
        case PC_PR_AFTER_REFINE: {
            if (C.res_obj < C.pt.value) set_point_from_result(acc, C, C.pt, C.probe_t, p);
            PROBE_FINISH();
        }
        L_PC_PR_FINISH:
        case PC_PR_FINISH: {
            C.ev_calls++;
            C.ev_failures += C.pt.conv ? 0 : 1;
            seen_append(acc, A, seen, C, C.pt, p);
            if (!C.has_best || C.pt.value < C.ev_best.value) {
                C.ev_best = C.pt;
                C.has_best = 1;
            }
            C.probe_v = C.pt.value;
            C.pc = C.ret_pc;  // the probe's caller: the one dynamic transition (through the switch)
            if constexpr (AC::kYield && LAD_THREAD_YIELD_RET) return ACT_YIELD;
            break;
        }
        default:
            return ACT_EXIT;
        }
    }
}

#undef ISSUE
#undef PROBE
#undef PROBE_FINISH

// Out-of-line controller (the warp kernels: a cold path next to the step loop).
template <int PMAX, class AC>
__device__ __noinline__ int controller(Ctl<PMAX> &C, const LocusArgs &A, const AC &acc, int slot)
{
    return controller_body<PMAX, AC>(C, A, acc, slot);
}

// Thread kernel: the controller inlined into the main loop (no call ABI: no
// callee-saved register saves and restores in local memory around every
// descent).  Config 1, same-box A/B at B = 262,144: 5.93 M -> 6.19 M solves/s
// at the old 96-register cap, 8.30 M with the cap raised (below).
#ifndef LAD_THREAD_INLINE_CTL
#define LAD_THREAD_INLINE_CTL 1
#endif

// ---------------------------------------------------------------------------
// hot path: one exact coordinate step (ccd.py:160-193)
// ---------------------------------------------------------------------------

// Thread kernel's weighted median: guess the axis' previous median first
// (step_dense_cand) instead of sorting every step (step_dense).
#ifndef LAD_THREAD_CAND
#define LAD_THREAD_CAND 0
#endif
// Thread kernel's weighted median by pairwise rank sums (step_dense) instead of
// the sorting network; the sort stays as the exact fallback for margin cases.
#ifndef LAD_THREAD_RANK
#define LAD_THREAD_RANK 1
#endif
// The rank sums in fixed point (weights scaled to 2^30 per total, as in the warp kernel's median
// test): a pair costs a comparison and two predicated integer adds instead of two FP64 adds and
// four selects, and the 2^14-unit margin makes an accepted element the reference's (see step_dense).
#ifndef LAD_THREAD_QRANK
#define LAD_THREAD_QRANK 1
#endif
constexpr bool thread_qrank_v = LAD_THREAD_RANK && LAD_THREAD_QRANK && !LAD_THREAD_CAND;
// Thread kernel's breakpoint division by a per-problem reciprocal table in
// shared memory (div_by_rcp: Markstein, bit-identical to r / x), columns with
// a divisor outside 2^+-450 on the generic path.
#ifndef LAD_THREAD_RCP
#define LAD_THREAD_RCP 0
#endif
// Thread kernel (compile-time shape): y read from global memory (L1) at the
// per-descent residual and objective instead of a shared-memory copy.
#ifndef LAD_THREAD_YGLOBAL
#define LAD_THREAD_YGLOBAL 0
#endif

// r / x for the thread kernel's breakpoints (LAD_THREAD_ZDIV).  A residual is
// often exactly 0 (the median row of an accepted step), and __ddiv_rn sends a
// zero dividend down its full-range slow path (a call of ~60 instructions,
// divergent: in a thread-per-problem warp some lane hits it at most steps);
// 0 / x is the signed zero 0 * x for finite nonzero x, so a zero dividend
// divides 1 instead and takes 0 * x.
// Config 1, same-box A/B at B = 262,144: 9.67 M -> 11.2 M solves/s (82 -> 67 warp
// instructions per step).  The dividend select must be opaque: otherwise the
// compiler sees that q is unused when z and divides r itself, slow path included.
#ifndef LAD_THREAD_ZDIV
#define LAD_THREAD_ZDIV 1
#endif
__device__ __forceinline__ double div_thread(double r, double x)
{
    if constexpr (LAD_THREAD_ZDIV) {
        return ddiv_zero_fast(r, x);
    } else {
        return ddiv(r, x);
    }
}

// beta register array accessed with a runtime axis index (select chains, no
// local memory)
template <int PMAX>
__device__ __forceinline__ double bget(const double (&b)[PMAX], int j)
{
    double v = b[0];
#pragma unroll
    for (int k = 1; k < PMAX; ++k) v = (j == k) ? b[k] : v;
    return v;
}
template <int PMAX>
__device__ __forceinline__ void bset(double (&b)[PMAX], int j, double v)
{
#pragma unroll
    for (int k = 0; k < PMAX; ++k) b[k] = (j == k) ? v : b[k];
}

constexpr double THREAD_MEDIAN_MARGIN = 1e-9;
constexpr unsigned MEDIAN_MARGIN_QT = 1u << 14;  // fixed-point rank sums: 2^14 units of 2^-30 of the total


// Rows of the per-lane breakpoint staging column Ls: the n data rows; the lambda breakpoint's
// constant 0 has a row only for the median guess (LAD_THREAD_CAND), which reads it by index.
// Without it the config-1 kernel's shared memory is exactly 10 KB per one-warp block, so its 12
// blocks per SM fit the 132 KB carve-out and leave 124 KB of L1 for the controller state in
// local memory (164 KB / 92 KB with the extra row).
// LAD_THREAD_LS = 0: no staging column at all for the rank-sum median (its only reader is the
// rare exact-order fallback, which then takes the breakpoints from a stack array).
#ifndef LAD_THREAD_LS
#define LAD_THREAD_LS 0
#endif
constexpr bool thread_ls_v = LAD_THREAD_LS || LAD_THREAD_CAND || !LAD_THREAD_RANK;
template <int NMAX>
constexpr int thread_ls_rows = !thread_ls_v ? 0 : NMAX + (LAD_THREAD_CAND ? 1 : 0);

struct MedianPick {
    double t;
    int ik;  // index of the element at the median position
};

// The miss path of step_dense_cand, out of line (it keeps the guess path's
// registers free): the breakpoints are re-read from the lane's Ls column and
// ordered by the register sort network, then numpy's cumsum decides
// (ccd.py:83-90), as in step_dense.
template <int NMAX, int PMAX>
__device__ __noinline__ MedianPick median_by_sort(const double *Ls, const double *xc, int lane, double lam, int ls_stride = 32)
{
    constexpr int NE = NMAX + 1;
    constexpr int XS = PMAX * 32;
    double key[NE];
    int idx[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) {
        // Ls: the lane's staging column (stride 32, already offset by the caller when ls_stride == 1:
        // a stack array); the lambda breakpoint sits at 0
        key[i] = (i < NMAX || i < thread_ls_rows<NMAX>) ? Ls[ls_stride == 32 ? i * 32 + lane : i] : 0.0;
        idx[i] = i;
    }
    sort_pairs<NE>(key, idx);
    auto wsorted = [&](int id) -> double {
        int ic = id < NMAX ? id : NMAX - 1;
        double x = xc[ic * XS];
        return id < NMAX ? fabs(x) : lam;
    };
    double c = 0.0;
#pragma unroll
    for (int k = 0; k < NE; ++k) c = dadd(c, wsorted(idx[k]));
    const double tot = c;
    const double hf = dmul(0.5, tot);
    c = 0.0;
    bool found = false;
    int kk = NE;
    double ck = 0.0, tk = key[NE - 1], tk1 = key[NE - 1];
    int ik = idx[NE - 1];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        c = dadd(c, wsorted(idx[k]));
        bool hit = !found && (c >= hf);
        if (hit) {
            kk = k;
            ck = c;
            tk = key[k];
            tk1 = key[k + 1 < NE ? k + 1 : k];
            ik = idx[k];
        }
        found = found || hit;
    }
    MedianPick mp;
    mp.t = (kk + 1 < NE && fabs(dsub(ck, hf)) <= dmul(1e-12, tot)) ? dmul(0.5, dadd(tk, tk1)) : tk;
    mp.ik = ik;
    return mp;
}


// Dense column, compile-time n = NMAX: register sort network.
// Returns true if the step moved beta_j.
template <int NMAX, int PMAX>
__device__ __forceinline__ void step_dense(double (&r)[NMAX], double (&b)[PMAX], const double *Xs, const double *RX,
                                           double *Ls, const float *Sc, int lane, int j, double lam, double &f_cur,
                                           double &sum_abs_b)
{
    constexpr int NE = NMAX + 1;
    constexpr int XS = PMAX * 32;  // row stride of Xs in doubles
    const double *xc = Xs + j * 32 + lane;
    const double *rc = RX + j * 32 + lane;
    const double bj = bget(b, j);
    double t_new;
    if constexpr (thread_qrank_v) {
        // Weighted median by rank sums in fixed point.  qb[i] = weight ordered before element i in
        // the stable (location, index) order (for q < i, q comes first iff loc_q <= loc_i), summed
        // over the weights scaled by s ~ 2^30 / total and truncated: every sum of <= NE terms is an
        // exact integer within NE units below s times the true sum, and so is the total.  Element
        // m is accepted iff qb + 2^14 < tq / 2 and qb + q_m > tq / 2 + 2^14: then the true sums
        // clear half the total by ~1.5e-5 * total on both sides, far beyond numpy's cumsum rounding
        // (NE * 2^-53 * total), so m is numpy's k and not the 1e-12 midpoint tie (ccd.py:83-90).
        // The scale only has to be the same for every term (a float from the problem's fetch; 0
        // for a degenerate total, which accepts nothing).  Otherwise (rare) the exact order decides.
        double loc[NE], w[NE];
        unsigned wq[NE], qb[NE];
        const double sc = (double)Sc[j * 32 + lane];
        unsigned tq = 0u;
#pragma unroll
        for (int i = 0; i < NMAX; ++i) {
            const double x = xc[i * XS];
            // np.divide then += b[j] (ccd.py:165-166)
            loc[i] = dadd(LAD_THREAD_RCP ? div_by_rcp(r[i], x, rc[i * XS]) : div_thread(r[i], x), bj);
            if constexpr (thread_ls_v) Ls[i * 32 + lane] = loc[i];
            w[i] = fabs(x);
            wq[i] = __double2uint_rz(dmul(w[i], sc));
            qb[i] = 0u;
            tq += wq[i];
        }
        loc[NMAX] = 0.0;
        w[NMAX] = lam;
        wq[NMAX] = __double2uint_rz(dmul(lam, sc));
        qb[NMAX] = 0u;
        tq += wq[NMAX];
#pragma unroll
        for (int i = 1; i < NE; ++i)
#pragma unroll
            for (int q = 0; q < i; ++q) {
                // one comparison and two predicated integer adds (written in PTX: the compiler
                // otherwise selects an addend and adds unconditionally, two instructions more per pair)
                asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %2, %3;\n\t@p add.u32 %0, %0, %4;\n\t@!p add.u32 %1, %1, %5;\n\t}"
                    : "+r"(qb[i]), "+r"(qb[q])
                    : "d"(loc[q]), "d"(loc[i]), "r"(wq[q]), "r"(wq[i]));
            }
        const unsigned hq = tq >> 1;
        const unsigned lo_b = hq >= MEDIAN_MARGIN_QT ? hq - MEDIAN_MARGIN_QT : 0u, hi_b = hq + MEDIAN_MARGIN_QT;
        bool found = false;
        t_new = 0.0;
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            const bool c = (qb[i] < lo_b) & (qb[i] + wq[i] > hi_b);
            t_new = c ? loc[i] : t_new;
            found = found | c;
        }
        if (!found) {
            if constexpr (thread_ls_v) {
                t_new = median_by_sort<NMAX, PMAX>(Ls, xc, lane, lam).t;
            } else {
                double tmp[NMAX];
#pragma unroll
                for (int i = 0; i < NMAX; ++i) tmp[i] = loc[i];
                t_new = median_by_sort<NMAX, PMAX>(tmp, xc, lane, lam, 1).t;
            }
        }
        if (fabs(dsub(t_new, bj)) <= dmul(1e-14, dadd(1.0, fabs(bj)))) return;  // ccd.py:172
        const double constant = dmul(lam, dsub(sum_abs_b, fabs(bj)));
        const double dot = blas_ddot_c<NE>([&](int i) { return fabs(dsub(t_new, loc[i])); }, [&](int i) { return w[i]; });
        const double v_new = dadd(constant, dot);
        if (v_new < f_cur) {  // strict accept (ccd.py:187-191)
            const double delta = dsub(t_new, bj);
#pragma unroll
            for (int i = 0; i < NMAX; ++i) r[i] = dsub(r[i], dmul(xc[i * XS], delta));
            sum_abs_b = dadd(sum_abs_b, dsub(fabs(t_new), fabs(bj)));
            bset(b, j, t_new);
            f_cur = v_new;
        }
        return;
    } else if constexpr (LAD_THREAD_RANK) {
        // Weighted median by rank sums: wb[i] = weight ordered before element i in
        // the stable (location, index) order, one comparison per pair (for j < i, j
        // comes first iff loc_j <= loc_i).  Sums in any order are within NE * 2^-53
        // * total of numpy's cumsum, so element m decided beyond a 1e-9 * total
        // margin (wb < half <= wb + w_m) is numpy's k and not the 1e-12 midpoint tie
        // (ccd.py:83-90); otherwise (rare) the sort below decides exactly.  Every
        // lane runs the same straight-line code: no sort, no divergence.
        double loc[NE], w[NE], wb[NE];
        double total = 0.0;
#pragma unroll
        for (int i = 0; i < NMAX; ++i) {
            const double x = xc[i * XS];
            // np.divide then += b[j] (ccd.py:165-166)
            loc[i] = dadd(LAD_THREAD_RCP ? div_by_rcp(r[i], x, rc[i * XS]) : div_thread(r[i], x), bj);
            if constexpr (thread_ls_v) Ls[i * 32 + lane] = loc[i];
            w[i] = fabs(x);
            wb[i] = 0.0;
            total = dadd(total, w[i]);
        }
        loc[NMAX] = 0.0;
        w[NMAX] = lam;
        wb[NMAX] = 0.0;
        total = dadd(total, lam);
#pragma unroll
        for (int i = 1; i < NE; ++i)
#pragma unroll
            for (int q = 0; q < i; ++q) {
                if (loc[q] <= loc[i]) wb[i] = dadd(wb[i], w[q]);
                else wb[q] = dadd(wb[q], w[i]);
            }
        const double hlf = dmul(0.5, total), mg = dmul(THREAD_MEDIAN_MARGIN, total);
        const double lo = dsub(hlf, mg), hi = dadd(hlf, mg);
        bool found = false;
        t_new = 0.0;
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            const bool c = (wb[i] < lo) & (dadd(wb[i], w[i]) > hi);
            t_new = c ? loc[i] : t_new;
            found = found | c;
        }
        if (!found) {
            if constexpr (thread_ls_v) {
                t_new = median_by_sort<NMAX, PMAX>(Ls, xc, lane, lam).t;
            } else {
                double tmp[NMAX];
#pragma unroll
                for (int i = 0; i < NMAX; ++i) tmp[i] = loc[i];
                t_new = median_by_sort<NMAX, PMAX>(tmp, xc, lane, lam, 1).t;
            }
        }
        if (fabs(dsub(t_new, bj)) <= dmul(1e-14, dadd(1.0, fabs(bj)))) return;  // ccd.py:172
        const double constant = dmul(lam, dsub(sum_abs_b, fabs(bj)));
        const double dot = blas_ddot_c<NE>([&](int i) { return fabs(dsub(t_new, loc[i])); }, [&](int i) { return w[i]; });
        const double v_new = dadd(constant, dot);
        if (v_new < f_cur) {  // strict accept (ccd.py:187-191)
            const double delta = dsub(t_new, bj);
#pragma unroll
            for (int i = 0; i < NMAX; ++i) r[i] = dsub(r[i], dmul(xc[i * XS], delta));
            sum_abs_b = dadd(sum_abs_b, dsub(fabs(t_new), fabs(bj)));
            bset(b, j, t_new);
            f_cur = v_new;
        }
        return;
    }
    double key[NE];
    int idx[NE];
#pragma unroll
    for (int i = 0; i < NMAX; ++i) {
        // np.divide then += b[j] (ccd.py:165-166)
        double loc = dadd(LAD_THREAD_RCP ? div_by_rcp(r[i], xc[i * XS], rc[i * XS]) : div_thread(r[i], xc[i * XS]), bj);
        key[i] = loc;
        idx[i] = i;
        Ls[i * 32 + lane] = loc;
    }
    key[NMAX] = 0.0;
    idx[NMAX] = NMAX;
    sort_pairs<NE>(key, idx);
    auto wsorted = [&](int id) -> double {
        int ic = id < NMAX ? id : NMAX - 1;
        double x = xc[ic * XS];
        return id < NMAX ? fabs(x) : lam;
    };
    // cum = sequential cumsum in sorted order; total = cum[-1] (ccd.py:85-86)
    double c = 0.0;
#pragma unroll
    for (int k = 0; k < NE; ++k) c = dadd(c, wsorted(idx[k]));
    const double total = c;
    const double half = dmul(0.5, total);
    // k = searchsorted(cum, half, 'left')
    c = 0.0;
    bool found = false;
    int kk = NE;
    double ck = 0.0, tk = key[NE - 1], tk1 = key[NE - 1];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        c = dadd(c, wsorted(idx[k]));
        bool hit = !found && (c >= half);
        if (hit) {
            kk = k;
            ck = c;
            tk = key[k];
            tk1 = key[k + 1 < NE ? k + 1 : k];
        }
        found = found || hit;
    }
    if (kk + 1 < NE && fabs(dsub(ck, half)) <= dmul(1e-12, total)) t_new = dmul(0.5, dadd(tk, tk1));
    else t_new = tk;
    // skip test (ccd.py:172)
    if (fabs(dsub(t_new, bj)) <= dmul(1e-14, dadd(1.0, fabs(bj)))) return;
    // v_new = lam*(sum|b| - |b_j|) + |t - locs| @ weights  (ccd.py:177-180)
    double constant = dmul(lam, dsub(sum_abs_b, fabs(bj)));
    double dot = blas_ddot_c<NE>([&](int i) { return fabs(dsub(t_new, i < NMAX ? Ls[i * 32 + lane] : 0.0)); },
                                 [&](int i) { return i < NMAX ? fabs(xc[i * XS]) : lam; });
    double v_new = dadd(constant, dot);
    if (v_new < f_cur) {  // strict accept (ccd.py:187-191)
        double delta = dsub(t_new, bj);
#pragma unroll
        for (int i = 0; i < NMAX; ++i) r[i] = dsub(r[i], dmul(xc[i * XS], delta));
        sum_abs_b = dadd(sum_abs_b, dsub(fabs(t_new), fabs(bj)));
        bset(b, j, t_new);
        f_cur = v_new;
    }
}

// Dense column, compile-time n = NMAX, with the median guessed first: the
// element that was this axis' weighted median at its previous step (cand) is
// usually still the median.  Element m is the reference's median iff the
// weight ordered before it in the stable (location, index) order, Wb,
// satisfies Wb < total/2 <= Wb + w_m in numpy's sequential cumsum
// (ccd.py:83-88).  Wb and the total are summed here in index order, and the
// guess is accepted only beyond a margin of 1e-9 * total on both sides: every
// sum of NE <= 33 non-negative terms is within NE * 2^-53 * total of the
// exact one (ours and numpy's), so an accepted guess is numpy's k, and the
// 1e-12 * total midpoint tie (ccd.py:89-90) is excluded.  Otherwise the
// register sort network decides as in step_dense and refreshes the guess.
// Breakpoints stay in registers in index order for v_new (no reload); the
// guess' location is read back through the lane's Ls column.
template <int NMAX, int PMAX>
__device__ __forceinline__ void step_dense_cand(double (&r)[NMAX], double (&b)[PMAX], int (&cand)[PMAX],
                                                const double *Xs, const double *RX, double *Ls, const double *Tw,
                                                int lane, int j, double lam, double &f_cur, double &sum_abs_b)
{
    constexpr int NE = NMAX + 1;
    constexpr int XS = PMAX * 32;
    const double *xc = Xs + j * 32 + lane;
    const double *rc = RX + j * 32 + lane;
    const double bj = bget(b, j);
#pragma unroll
    for (int i = 0; i < NMAX; ++i)
        Ls[i * 32 + lane] = dadd(LAD_THREAD_RCP ? div_by_rcp(r[i], xc[i * XS], rc[i * XS]) : div_thread(r[i], xc[i * XS]),
                                 bj);  // np.divide then += b[j] (ccd.py:165-166)
    // breakpoint i (Ls[NMAX] holds the lambda breakpoint's 0.0 from the kernel start)
    auto loc = [&](int i) { return Ls[i * 32 + lane]; };
    int m = cand[0];
#pragma unroll
    for (int k = 1; k < PMAX; ++k) m = (j == k) ? cand[k] : m;
    const double tm = Ls[m * 32 + lane];
    double wb = 0.0;
#pragma unroll
    for (int i = 0; i < NE; ++i) {
        const double li = loc(i);
        const bool below = (li < tm) | ((li == tm) & (i < m));
        const double wi = i < NMAX ? fabs(xc[i * XS]) : lam;
        if (below) wb = dadd(wb, wi);
    }
    const double wm = m < NMAX ? fabs(xc[(m < NMAX ? m : 0) * XS]) : lam;
    const double total = Tw[j * 32 + lane];
    const double half = dmul(0.5, total), marg = dmul(THREAD_MEDIAN_MARGIN, total);
    double t_new;
    if ((wb < dsub(half, marg)) & (dadd(wb, wm) > dadd(half, marg)) & (tm == tm)) {
        t_new = tm;
    } else {
        const MedianPick mp = median_by_sort<NMAX, PMAX>(Ls, xc, lane, lam);
        t_new = mp.t;
#pragma unroll
        for (int k = 0; k < PMAX; ++k) cand[k] = (j == k) ? mp.ik : cand[k];
    }
    if (fabs(dsub(t_new, bj)) <= dmul(1e-14, dadd(1.0, fabs(bj)))) return;  // ccd.py:172
    const double constant = dmul(lam, dsub(sum_abs_b, fabs(bj)));
    const double dot = blas_ddot_c<NE>([&](int i) { return fabs(dsub(t_new, loc(i))); },
                                       [&](int i) { return i < NMAX ? fabs(xc[(i < NMAX ? i : 0) * XS]) : lam; });
    const double v_new = dadd(constant, dot);
    if (v_new < f_cur) {  // strict accept (ccd.py:187-191)
        const double delta = dsub(t_new, bj);
#pragma unroll
        for (int i = 0; i < NMAX; ++i) r[i] = dsub(r[i], dmul(xc[i * XS], delta));
        sum_abs_b = dadd(sum_abs_b, dsub(fabs(t_new), fabs(bj)));
        bset(b, j, t_new);
        f_cur = v_new;
    }
}

// General column (zero entries, or runtime n): compacted nonzero rows,
// stable insertion sort in local memory.  Rare path.
template <int NMAX, int PMAX>
__device__ __noinline__ void step_general(double *r, double *b, const double *Xs, int lane, int n, int j,
                                          double lam, double *f_cur, double *sum_abs_b)
{
    constexpr int XS = PMAX * 32;
    const double *xc = Xs + j * 32 + lane;
    const double bj = b[j];
    double loc[NMAX + 1], w[NMAX + 1], zr[NMAX];
    int ord[NMAX + 1];
    int k = 0, z = 0;
    bool dense = true;
    for (int i = 0; i < n; ++i)
        if (xc[i * XS] == 0.0) dense = false;
    for (int i = 0; i < n; ++i) {
        double x = xc[i * XS];
        if (x != 0.0) {
            loc[k] = dense ? dadd(ddiv(r[i], x), bj) : ddiv(dadd(r[i], dmul(x, bj)), x);
            w[k] = fabs(x);
            ++k;
        } else {
            zr[z++] = fabs(r[i]);
        }
    }
    loc[k] = 0.0;
    w[k] = lam;
    const int ne = k + 1;
    for (int i = 0; i < ne; ++i) {
        int q = i;
        while (q > 0 && loc[ord[q - 1]] > loc[i]) {
            ord[q] = ord[q - 1];
            --q;
        }
        ord[q] = i;
    }
    double c = 0.0;
    for (int i = 0; i < ne; ++i) c = dadd(c, w[ord[i]]);
    const double total = c;
    const double half = dmul(0.5, total);
    c = 0.0;
    int kk = ne;
    double ck = 0.0;
    for (int i = 0; i < ne; ++i) {
        c = dadd(c, w[ord[i]]);
        if (c >= half) {
            kk = i;
            ck = c;
            break;
        }
    }
    double t_new;
    if (kk + 1 < ne && fabs(dsub(ck, half)) <= dmul(1e-12, total))
        t_new = dmul(0.5, dadd(loc[ord[kk]], loc[ord[kk + 1]]));
    else
        t_new = loc[ord[kk < ne - 1 ? kk : ne - 1]];
    if (fabs(dsub(t_new, bj)) <= dmul(1e-14, dadd(1.0, fabs(bj)))) return;
    double constant = dmul(lam, dsub(*sum_abs_b, fabs(bj)));
    if (z) constant = dadd(constant, np_sum(z, [&](int q) { return zr[q]; }));
    double dot = blas_ddot(ne, [&](int i) { return fabs(dsub(t_new, loc[i])); }, [&](int i) { return w[i]; });
    double v_new = dadd(constant, dot);
    if (v_new < *f_cur) {
        double delta = dsub(t_new, bj);
        for (int i = 0; i < n; ++i) r[i] = dsub(r[i], dmul(xc[i * XS], delta));
        *sum_abs_b = dadd(*sum_abs_b, dsub(fabs(t_new), fabs(bj)));
        b[j] = t_new;
        *f_cur = v_new;
    }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int NMAX, int PMAX, bool EXACT>
__host__ __device__ constexpr size_t smem_doubles_per_warp()
{
    return (size_t)NMAX * PMAX * 32 * (EXACT && LAD_THREAD_RCP ? 2 : 1) +
           (EXACT && LAD_THREAD_YGLOBAL ? 0 : (size_t)NMAX * 32) + (size_t)thread_ls_rows<NMAX> * 32 +
           (EXACT && LAD_THREAD_CAND ? (size_t)PMAX * 32 : 0) + (EXACT && thread_qrank_v ? (size_t)PMAX * 16 : 0);
}



// Occupancy hint for the compile-time-shape kernel (config 1: n = 10, p = 2).
// With the controller inlined, 10 one-warp blocks per SM (168 registers, 12
// resident warps, no spills) beat a higher occupancy with spills: same-box A/B
// at B = 262,144 (solves/s): 96 registers (20 warps) 6.19 M, 128 (16) 7.98 M,
// hint 14 (128 registers) 8.14 M, hint 12 (167) 7.99 M, hint 10 (168) 8.30 M,
// hint 8 (189) 7.18 M.  Also measured and rejected at this shape: the
// reciprocal-table division (LAD_THREAD_RCP: more shared memory, 7.86 M), y
// read from global memory (LAD_THREAD_YGLOBAL: 7.31 M at hint 12), a zero-
// dividend bypass of the division's slow path written as a plain select (7.91 M:
// the compiler undid it, see LAD_THREAD_ZDIV), and the median guess
// (LAD_THREAD_CAND: any lane's miss makes the whole warp sort; 5.2 M vs 5.9 M).
// Re-swept after the direct-jump controller, the zero-dividend division and the rank-sum
// median (B = 262,144): hints 8 / 10 / 12 / 14 / 16 -> 11.08 / 11.75 / 12.00 / 11.37 / 11.37 M.
#ifndef LAD_THREAD_MIN_BLOCKS
#define LAD_THREAD_MIN_BLOCKS 12
#endif
// Warps per block of the compile-time-shape kernel.  Each block pays 1 KB of reserved shared
// memory: with two warps per block the 12 warps of an SM need 6 x (15 + 1) = 96 KB, which fits the
// 100 KB carve-out (156 KB of L1 for the controller state in local memory) where 12 one-warp
// blocks need 102 KB and get the 132 KB one.  The warps of a block are independent (no barrier).
#ifndef LAD_THREAD_WARPS
#define LAD_THREAD_WARPS 2
#endif
template <int NMAX, bool EXACT>
constexpr int thread_warps = (EXACT && NMAX <= 10) ? LAD_THREAD_WARPS : 1;
template <int NMAX, bool EXACT>
constexpr int thread_min_blocks =
    (EXACT && NMAX <= 10) ? (LAD_THREAD_MIN_BLOCKS + LAD_THREAD_WARPS - 1) / LAD_THREAD_WARPS : 1;

template <int NMAX, int PMAX, bool EXACT>
__global__ void __launch_bounds__(32 * thread_warps<NMAX, EXACT>, thread_min_blocks<NMAX, EXACT>) locus_kernel(LocusArgs A)
{
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31;
    constexpr bool ysh = !(EXACT && LAD_THREAD_YGLOBAL);  // y staged in shared memory
    double *Xs = smem + (threadIdx.x >> 5) * smem_doubles_per_warp<NMAX, PMAX, EXACT>();  // this warp's region
    double *Ys = ysh ? Xs + NMAX * PMAX * 32 : nullptr;
    double *Ls = Xs + NMAX * PMAX * 32 + (ysh ? NMAX * 32 : 0);
    double *Tw = Ls + thread_ls_rows<NMAX> * 32;                                // LAD_THREAD_CAND: PMAX * 32 doubles
    double *RX = Tw + (EXACT && LAD_THREAD_CAND ? PMAX * 32 : 0);   // LAD_THREAD_RCP: NMAX * PMAX * 32 doubles
    float *Sc = reinterpret_cast<float *>(RX + (EXACT && LAD_THREAD_RCP ? NMAX * PMAX * 32 : 0));  // thread_qrank_v: PMAX * 32 floats
    if constexpr (thread_ls_rows<NMAX> > NMAX) Ls[NMAX * 32 + lane] = 0.0;  // the lambda breakpoint's location
    const int slot = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = EXACT ? NMAX : A.n;
    const int p = EXACT ? PMAX : A.p;
    constexpr int XS = PMAX * 32;

    Ctl<PMAX> C;
    C.pc = PC_FETCH;
    double r[NMAX];
    double b[PMAX];
    int cand[PMAX];  // per axis: the element that was the weighted median at its last step (a guess)
#pragma unroll
    for (int k = 0; k < PMAX; ++k) {
        b[k] = 0.0;
        cand[k] = NMAX / 2;
    }
#pragma unroll
    for (int i = 0; i < NMAX; ++i) r[i] = 0.0;
    double f_cur = 0.0, f_sweep_start = 0.0, sum_abs_b = 0.0, tol = 0.0, lam = 0.0;
    int j = 0, frozen = -1, sweeps = 0, max_sweeps = 0, steps = 0;
    uint32_t sparse = 0;
    bool need_ctl = true;
    bool alive = true;

    // Every iteration: (1) lanes at a descent boundary run the controller and
    // the descent init, (2) all live lanes execute one coordinate step together.
    // The __syncwarp()s force the lanes back into lock-step after the divergent
    // bookkeeping, so the hot step always runs with every live lane active.
    for (;;) {
        __syncwarp();
        if (!__any_sync(0xffffffffu, alive)) break;
        const unsigned ctl_lanes = __ballot_sync(0xffffffffu, alive && need_ctl);
        if (alive && need_ctl) {
            ThreadAccess<NMAX, PMAX> acc{n, p, lane, Xs, Ys, EXACT && LAD_THREAD_CAND ? Tw : nullptr,
                                         EXACT && LAD_THREAD_RCP ? RX : nullptr, EXACT && thread_qrank_v ? Sc : nullptr};
            int act;
            if constexpr (ThreadAccess<NMAX, PMAX>::kYield) {
                // rounds: every lane still in the controller runs to its next yield point, request or
                // exit; the vote brings the lanes back together before the next round
                act = ACT_YIELD;
                for (;;) {
                    if (act == ACT_YIELD)
                        act = LAD_THREAD_INLINE_CTL ? controller_body<PMAX>(C, A, acc, slot)
                                                    : controller<PMAX>(C, A, acc, slot);
                    if (!__any_sync(ctl_lanes, act == ACT_YIELD)) break;
                }
            } else {
                act = LAD_THREAD_INLINE_CTL ? controller_body<PMAX>(C, A, acc, slot) : controller<PMAX>(C, A, acc, slot);
            }
            if (act == ACT_EXIT) {
                alive = false;
            } else {
                lam = C.lam;
                sparse = C.sparse_mask;
#pragma unroll
                for (int k = 0; k < PMAX; ++k) b[k] = k < p ? C.req_start[k] : 0.0;
                frozen = C.req_frozen;
                tol = C.req_tol;
                max_sweeps = C.req_sweeps;
                // descent init (ccd.py:143-155)
#pragma unroll
                for (int i = 0; i < NMAX; ++i) {
                    if (i < n) {
                        double g = gemv_row(p, i, n, [&](int jj) { return Xs[i * XS + jj * 32 + lane]; },
                                            [&](int jj) { return b[jj < PMAX ? jj : PMAX - 1]; });
                        r[i] = dsub(ysh ? Ys[i * 32 + lane] : __ldg(C.ysrc + i), g);
                    }
                }
                double sb = np_sum(p, [&](int jj) { return fabs(b[jj < PMAX ? jj : PMAX - 1]); });
                double sr = EXACT ? np_sum_c<NMAX>([&](int i) { return fabs(r[i]); })
                                  : np_sum(n, [&](int i) {
                                        double v = 0.0;
#pragma unroll
                                        for (int q = 0; q < NMAX; ++q) v = (q == i) ? r[q] : v;
                                        return fabs(v);
                                    });
                f_cur = dadd(sr, dmul(lam, sb));
                sweeps = 1;
                steps = 0;
                f_sweep_start = f_cur;
                sum_abs_b = sb;
                j = (frozen == 0) ? 1 : 0;
                need_ctl = false;
                if (j >= p) {  // no free axis: one empty sweep, converged (ccd.py:194-196)
                    C.res_conv = 1;
                    C.res_sweeps = 1;
                    C.res_steps = 0;
#pragma unroll
                    for (int k = 0; k < PMAX; ++k)
                        if (k < p) C.res_beta[k] = b[k];
                    C.res_obj = objective_of<NMAX, PMAX>(Xs, ysh ? Ys + lane : C.ysrc, ysh ? 32 : 1, n, p, lane, lam,
                                                         C.res_beta);
                    C.D += 1;
                    need_ctl = true;
                }
            }
        }
        __syncwarp();
        if (!alive || need_ctl) continue;
        // ---- one coordinate step on axis j
        bool dense_step = false;
        if constexpr (EXACT) {
            dense_step = !((sparse >> j) & 1u);
            if (dense_step) {
                if constexpr (LAD_THREAD_CAND)
                    step_dense_cand<NMAX, PMAX>(r, b, cand, Xs, RX, Ls, Tw, lane, j, lam, f_cur, sum_abs_b);
                else
                    step_dense<NMAX, PMAX>(r, b, Xs, RX, Ls, Sc, lane, j, lam, f_cur, sum_abs_b);
            }
        }
        if (!dense_step) {
            // rare path (zero entries in column j, or runtime-shape kernel): work on
            // local copies so the register arrays never have their address taken
            double rl[NMAX], bl[PMAX];
#pragma unroll
            for (int i = 0; i < NMAX; ++i) rl[i] = r[i];
#pragma unroll
            for (int k = 0; k < PMAX; ++k) bl[k] = b[k];
            double fc = f_cur, sa = sum_abs_b;
            step_general<NMAX, PMAX>(rl, bl, Xs, lane, n, j, lam, &fc, &sa);
#pragma unroll
            for (int i = 0; i < NMAX; ++i) r[i] = rl[i];
#pragma unroll
            for (int k = 0; k < PMAX; ++k) b[k] = bl[k];
            f_cur = fc;
            sum_abs_b = sa;
        }
        ++steps;
        // ---- advance (ccd.py:156-196)
        int jn = j + 1;
        if (jn == frozen) ++jn;
        if (jn < p) {
            j = jn;
        } else {
            bool done = false;
            int conv = 0;
            if (dsub(f_sweep_start, f_cur) < tol) {
                done = true;
                conv = 1;
            } else if (sweeps >= max_sweeps) {
                done = true;
            }
            if (!done) {
                ++sweeps;
                f_sweep_start = f_cur;
                sum_abs_b = np_sum(p, [&](int jj) { return fabs(b[jj < PMAX ? jj : PMAX - 1]); });
                j = (frozen == 0) ? 1 : 0;
            } else {
                // ---- descent finished: fresh objective (ccd.py:197)
#pragma unroll
                for (int k = 0; k < PMAX; ++k)
                    if (k < p) C.res_beta[k] = b[k];
                C.res_obj = objective_of<NMAX, PMAX>(Xs, ysh ? Ys + lane : C.ysrc, ysh ? 32 : 1, n, p, lane, lam,
                                                     C.res_beta);
                C.res_conv = conv;
                C.res_sweeps = sweeps;
                C.res_steps = steps;
                C.D += 1;
                C.S += steps;
                need_ctl = true;
            }
        }
    }
}

}  // namespace lad
