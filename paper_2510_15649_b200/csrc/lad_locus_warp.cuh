// lad_locus_warp.cuh -- warp-per-problem locus kernel (n + 1 <= 32 breakpoints).
//
// One warp solves one problem at a time (persistent grid, per-warp work
// stealing).  Lane i owns data row i and its residual r_i; lane n carries the
// lambda breakpoint at 0; lanes > n are +inf pads.  Per coordinate step
// (ccd.py:160-193):
//   * breakpoints r_i / x_ij + b_j: one division per lane;
//   * stable order of (location, index): a 32-lane bitonic network of shuffles;
//   * cumulative weights: Kogge-Stone scan, accepted only when every
//     comparison against half the total is decided by a margin far above the
//     rounding gap to numpy's sequential cumsum; otherwise the exact
//     sequential cumsum is recomputed (so the result is always the
//     reference's);
//   * v_new: OpenBLAS ddot's summation tree mapped onto shuffles, the FMA tail
//     through shared memory.
// Control flow (the controller state machine shared with the thread kernel)
// is warp-uniform: all lanes run it on one shared Ctl.
#pragma once
#include "lad_locus.cuh"

namespace lad {

constexpr unsigned FULLMASK = 0xffffffffu;
constexpr int WARPS_PER_BLOCK = 7;

template <int PMAX>
struct WarpShared {
    Ctl<PMAX> C;
    double X[32 * PMAX];  // row-major [i * p + j]
    double Y[32];
    double B[PMAX];       // beta of the running descent (warp-uniform)
    double sa[32], sw[32], sz[32];
    double2 aw[32];       // (|t - loc_i|, w_i) pairs for the ddot FMA tail
    int perm[PMAX][32];   // per axis: sorted position -> element of the last sort
};

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(FULLMASK, v, src); }
__device__ __forceinline__ double shfl_down_d(double v, int d) { return __shfl_down_sync(FULLMASK, v, d); }
__device__ __forceinline__ double shfl_xor_d(double v, int m) { return __shfl_xor_sync(FULLMASK, v, m); }

// numpy pairwise_sum of cnt values held one per lane (lane i -> element i).
__device__ __forceinline__ double warp_np_sum(double v, int cnt, int lane)
{
    if (cnt < 8) {
        double res = 0.0;
        for (int i = 0; i < cnt; ++i) res = dadd(res, shfl_d(v, i));
        return res;
    }
    const int lim = cnt - (cnt % 8);
    double acc = v;
    for (int blk = 8; blk < lim; blk += 8) acc = dadd(acc, shfl_d(v, (lane + blk) & 31));
    acc = dadd(acc, shfl_xor_d(acc, 1));
    acc = dadd(acc, shfl_xor_d(acc, 2));
    acc = dadd(acc, shfl_xor_d(acc, 4));
    double res = shfl_d(acc, 0);
    for (int i = lim; i < cnt; ++i) res = dadd(res, shfl_d(v, i));
    return res;
}

// OpenBLAS ddot (SkylakeX) over cnt <= 32 terms a_i * w_i held one per lane.
template <int PMAX>
__device__ __forceinline__ double warp_blas_ddot(double a, double w, int cnt, int lane, WarpShared<PMAX> *W)
{
    const int n1 = cnt & -16;
    double dot = 0.0;
    const double pr = dmul(a, w);
    if (n1 == 16) {
        double q4 = shfl_down_d(pr, 4), q8 = shfl_down_d(pr, 8), q12 = shfl_down_d(pr, 12);
        double S = dadd(dadd(dadd(pr, q4), q8), q12);
        double u = dadd(S, shfl_down_d(S, 2));
        double d = dadd(u, shfl_down_d(u, 1));
        dot = shfl_d(d, 0);
    } else if (n1 == 32) {
        double A = dadd(pr, shfl_down_d(pr, 4));
        double a8 = shfl_down_d(A, 8), a16 = shfl_down_d(A, 16), a24 = shfl_down_d(A, 24);
        double S = dadd(dadd(dadd(A, a8), a16), a24);
        double u = dadd(S, shfl_down_d(S, 2));
        double d = dadd(u, shfl_down_d(u, 1));
        dot = shfl_d(d, 0);
    }
    if (n1 < cnt) {  // FMA tail, sequential in index order
        W->sa[lane] = a;
        W->sw[lane] = w;
        __syncwarp();
        for (int i = n1; i < cnt; ++i) dot = dfma(W->sa[i], W->sw[i], dot);
        __syncwarp();
    }
    return dot;
}

// Ascending bitonic sort of (key, idx) over the 32 lanes, lexicographic.
__device__ __forceinline__ void bitonic32(double &key, int &idx, int lane)
{
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            double pk = shfl_xor_d(key, j);
            int pi = __shfl_xor_sync(FULLMASK, idx, j);
            bool plt = (pk < key) | ((pk == key) & (pi < idx));
            bool up = (lane & k) == 0;
            bool lower = (lane & j) == 0;
            bool take = (lower == up) ? plt : !plt;
            key = take ? pk : key;
            idx = take ? pi : idx;
        }
    }
}

// Access policy: the whole warp works on one problem held in WarpShared.
template <int PMAX>
struct WarpAccess {
    int n, p, lane;
    WarpShared<PMAX> *W;
    __device__ __forceinline__ bool leader() const { return lane == 0; }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    __device__ int fetch(Ctl<PMAX> &C, const LocusArgs &A) const
    {
        const int div = A.axis_mode == AXIS_SEARCH ? p : 1;
        unsigned long long item = 0;
        if (lane == 0) item = atomicAdd(A.counter, 1ULL);
        item = __shfl_sync(FULLMASK, item, 0);
        if ((int64_t)item >= A.B * div) return -1;
        const unsigned long long pr = item / div;
        int64_t src = A.data_index ? A.data_index[pr] : (int64_t)pr;
        const double *xg = A.X + (size_t)src * n * p;
        const double *yg = A.Y + (size_t)src * n;
        bool ok = true;
        uint32_t mask = 0;
        for (int e = lane; e < n * p; e += 32) {
            double v = xg[e];
            W->X[e] = v;
            ok = ok && isfinite(v);
            if (v == 0.0) mask |= 1u << (e % p);
        }
        for (int i = lane; i < n; i += 32) {
            double v = yg[i];
            W->Y[i] = v;
            ok = ok && isfinite(v);
        }
        ok = __all_sync(FULLMASK, ok);
        mask = __reduce_or_sync(FULLMASK, mask);
        double lraw = A.lam[pr];
        ok = ok && isfinite(lraw) && lraw >= 0.0;
        __syncwarp();
        C.prob = (int64_t)pr;
        C.arank = (int)(item % div);
        C.lam = lraw > A.prm.lambda_floor ? lraw : A.prm.lambda_floor;
        C.sparse_mask = mask;
        __syncwarp();
        if (!ok) {
            if (lane == 0) write_invalid<PMAX>(A, (int64_t)pr, p);
            return 0;
        }
        return 1;
    }
    __device__ double col_abs_sum(int j) const
    {
        if (p == 1) return np_sum(n, [&](int i) { return fabs(W->X[i]); });
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = dadd(s, fabs(W->X[i * p + j]));
        return s;
    }
    __device__ double y_absmax() const
    {
        double ymax = 0.0;
        for (int i = 0; i < n; ++i) {
            double a = fabs(W->Y[i]);
            if (i == 0 || a > ymax) ymax = a;
        }
        return ymax;
    }
    // first minimal |t_k - t| in insertion order: lane-strided scan + argmin on (dist, k)
    __device__ int nearest(const double *seen, int lim, double t) const
    {
        __syncwarp();
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        int bk = 0x7fffffff;
        for (int k = lane; k < lim; k += 32) {
            double dd = fabs(dsub(seen[k], t));
            if (dd < bd) {
                bd = dd;
                bk = k;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            double od = shfl_xor_d(bd, off);
            int ok = __shfl_xor_sync(FULLMASK, bk, off);
            if (od < bd || (od == bd && ok < bk)) {
                bd = od;
                bk = ok;
            }
        }
        return bk == 0x7fffffff ? -1 : bk;
    }
};

__device__ __forceinline__ uint32_t bitonic_inv_mask(int lane)
{
    uint32_t m = 0;
    int s = 0;
    for (int k = 2; k <= 32; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1, ++s) {
            bool up = (lane & k) == 0;
            bool lower = (lane & j) == 0;
            if (lower != up) m |= 1u << s;
        }
    return m;
}

// Ascending bitonic sort of (key, idx) over 32 lanes, lexicographic, with
// the per-lane direction bits precomputed.
__device__ __forceinline__ void bitonic32m(double &key, int &idx, uint32_t inv_mask)
{
    int s = 0;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1, ++s) {
            double pk = shfl_xor_d(key, j);
            int pi = __shfl_xor_sync(FULLMASK, idx, j);
            bool plt = (pk < key) | ((pk == key) & (pi < idx));
            bool take = plt != (((inv_mask >> s) & 1u) != 0u);
            key = take ? pk : key;
            idx = take ? pi : idx;
        }
    }
}

// (key, idx) ascending across lanes 0..31 (lexicographic)?
__device__ __forceinline__ bool warp_is_sorted(double key, int idx, int lane)
{
    const double nk = shfl_down_d(key, 1);
    const int ni = __shfl_down_sync(FULLMASK, idx, 1);
    const bool ok = (lane == 31) || (key < nk) || ((key == nk) && (idx < ni));
    return __all_sync(FULLMASK, ok);
}

// number of adjacent (key, idx) pairs out of ascending order
__device__ __forceinline__ int warp_order_violations(double key, int idx, int lane)
{
    const double nk = shfl_down_d(key, 1);
    const int ni = __shfl_down_sync(FULLMASK, idx, 1);
    const bool ok = (lane == 31) || (key < nk) || ((key == nk) && (idx < ni));
    return __popc(__ballot_sync(FULLMASK, !ok));
}

// One odd-even transposition phase: pairs (2i, 2i+1) for phase 0, (2i+1, 2i+2)
// for phase 1; the lower lane of a pair keeps the smaller (key, idx).
__device__ __forceinline__ void oddeven_phase(double &key, int &idx, int lane, int phase)
{
    const bool odd = lane & 1;
    const bool lower = (phase == 0) ? !odd : odd;
    int partner = lower ? lane + 1 : lane - 1;
    const bool paired = partner >= 0 && partner < 32;
    partner = paired ? partner : lane;
    const double pk = shfl_d(key, partner);
    const int pi = __shfl_sync(FULLMASK, idx, partner);
    const bool plt = (pk < key) | ((pk == key) & (pi < idx));
    const bool take = paired && (lower ? plt : !plt);
    key = take ? pk : key;
    idx = take ? pi : idx;
}

// numpy's sequential cumsum in sorted order, recomputed exactly (rare path:
// only when the parallel scan leaves a comparison within 1e-13 of a tie).
__device__ __forceinline__ void exact_cumsum_decision(double ws, int lane, int cnt, int &k, double &ck, double &total,
                                                   double &half)
{
    double ce = 0.0;
    for (int i = 0; i < 32; ++i) {
        double wi = shfl_d(ws, i);
        if (i <= lane) ce = dadd(ce, wi);
    }
    total = shfl_d(ce, cnt - 1);
    half = dmul(0.5, total);
    k = __popc(__ballot_sync(FULLMASK, lane < cnt && ce < half));
    ck = shfl_d(ce, k < cnt ? k : cnt - 1);
}

// _AxisWorkspace for a column with zero entries (ccd.py:94-110, :167-169,
// :178-179): nonzero rows compacted to lanes 0..k-1 in row order, the zero
// rows' |r| summed with numpy's pairwise order.  Rare path.
template <int PMAX>
__device__ __forceinline__ void sparse_column(WarpShared<PMAX> *W, int lane, int n, double r, double xij, double bj,
                                           double lam, double &loc, double &w, int &cnt, double &zsum)
{
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    const bool row = lane < n;
    const bool nz = row && xij != 0.0;
    const unsigned nzm = __ballot_sync(FULLMASK, nz);
    const unsigned zm = __ballot_sync(FULLMASK, row && xij == 0.0);
    const unsigned lt = (1u << lane) - 1u;
    const int k = __popc(nzm), z = __popc(zm);
    const bool dense = (k == n);
    __syncwarp();
    if (nz) {
        W->sa[__popc(nzm & lt)] = dense ? dadd(ddiv(r, xij), bj) : ddiv(dadd(r, dmul(xij, bj)), xij);
        W->sw[__popc(nzm & lt)] = fabs(xij);
    }
    if (row && xij == 0.0) W->sz[__popc(zm & lt)] = fabs(r);
    __syncwarp();
    loc = lane < k ? W->sa[lane] : (lane == k ? 0.0 : INF);
    w = lane < k ? W->sw[lane] : (lane == k ? lam : 0.0);
    const double zv = lane < z ? W->sz[lane] : 0.0;
    __syncwarp();
    zsum = z > 0 ? warp_np_sum(zv, z, lane) : 0.0;
    cnt = k + 1;
}

// Weighted median, skip test, v_new and strict accept of one coordinate step
// (ccd.py:81-91, :172-191), given this lane's breakpoint (loc, w).  CNTC > 0:
// compile-time breakpoint count (dense column in a compile-time-n kernel),
// so the reduction trees, tail lengths and bounds are constants.
template <int PMAX, int CNTC>
__device__ __forceinline__ void median_update(WarpShared<PMAX> *W, int lane, uint32_t inv_mask, int j, double lam,
                                              bool cacheable, int cnt_rt, double loc, double w, double zsum,
                                              bool have_zero, bool row, double xij, double bj, double &r,
                                              double &f_cur, double &sum_abs_b, uint32_t &perm_valid)
{
    const int cnt = CNTC > 0 ? CNTC : cnt_rt;
    // stable order by (location, index).  The order is unique, so if this
    // axis' permutation from its previous evaluation is still sorted under the
    // new locations it is the answer; otherwise odd-even transposition rounds
    // repair a nearly sorted permutation, and the 15-stage network runs last.
    double key;
    int idx;
    bool sorted = false;
    if (cacheable && ((perm_valid >> j) & 1u)) {
        idx = W->perm[j][lane];
        key = shfl_d(loc, idx);
        const int violations = warp_order_violations(key, idx, lane);
        sorted = violations == 0;
        // a few adjacent inversions: odd-even rounds; many: straight to the network
#pragma unroll 1
        for (int round = 0; round < 2 && !sorted && violations <= 6; ++round) {
            oddeven_phase(key, idx, lane, 0);
            oddeven_phase(key, idx, lane, 1);
            sorted = warp_is_sorted(key, idx, lane);
        }
        if (sorted) W->perm[j][lane] = idx;
    }
    if (!sorted) {
        key = loc;
        idx = lane;
        bitonic32m(key, idx, inv_mask);
        if (cacheable) W->perm[j][lane] = idx;
    }
    if (cacheable) perm_valid |= 1u << j;
    const double ws = shfl_d(w, idx);
    // Cumulative weights only *locate* k = first cum >= total/2.  An FP32
    // Kogge-Stone scan differs from numpy's sequential FP64 cumsum by at most
    // ~6 * 2^-24 * total (conversion + 5 tree levels); every comparison with
    // total/2 is accepted only beyond a 1e-5 * total margin, which also rules
    // out the 1e-12 * total flat-segment tie.  Otherwise (or on FP32
    // overflow/underflow) the exact FP64 sequential cumsum decides.
    float cf = __double2float_rn(ws);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const float t = __shfl_up_sync(FULLMASK, cf, d);
        if (lane >= d) cf = __fadd_rn(cf, t);
    }
    // pads carry weight 0, so their cumulative weight equals the total (>= half)
    const float totf = __shfl_sync(FULLMASK, cf, cnt - 1);
    const float halff = 0.5f * totf;
    int k = __popc(__ballot_sync(FULLMASK, cf < halff));
    const float ckf = __shfl_sync(FULLMASK, cf, k < cnt ? k : cnt - 1);
    const float margf = 1e-5f * totf;
    const bool risky = !(totf > 0.0f && totf <= 3.0e38f) || fabsf(ckf - halff) <= margf ||
                       __any_sync(FULLMASK, lane < cnt && fabsf(cf - halff) <= margf);
    bool tie = false;
    if (risky) {
        double ck, total, half;
        exact_cumsum_decision(ws, lane, cnt, k, ck, total, half);
        tie = (k + 1 < cnt) && fabs(dsub(ck, half)) <= dmul(1e-12, total);
    }
    const int ks = k < cnt ? k : cnt - 1;
    const double tk = shfl_d(key, ks);
    const double tk1 = shfl_d(key, ks + 1 < 32 ? ks + 1 : 31);
    const double t_new = tie ? dmul(0.5, dadd(tk, tk1)) : tk;
    if (fabs(dsub(t_new, bj)) <= dmul(1e-14, dadd(1.0, fabs(bj)))) return;  // ccd.py:172
    double constant = dmul(lam, dsub(sum_abs_b, fabs(bj)));
    if (have_zero) constant = dadd(constant, zsum);
    // v_new = constant + |t - loc| @ weights, OpenBLAS ddot's order (see warp_blas_ddot)
    const bool in = lane < cnt;
    const double a = in ? fabs(dsub(t_new, loc)) : 0.0;
    const double wv = in ? w : 0.0;
    const int n1 = cnt & -16;
    const double pr = dmul(a, wv);
    double dot = 0.0;
    if (n1 == 16) {
        const double q4 = shfl_down_d(pr, 4), q8 = shfl_down_d(pr, 8), q12 = shfl_down_d(pr, 12);
        const double S = dadd(dadd(dadd(pr, q4), q8), q12);
        const double u = dadd(S, shfl_down_d(S, 2));
        dot = shfl_d(dadd(u, shfl_down_d(u, 1)), 0);
    } else if (n1 == 32) {
        const double A2 = dadd(pr, shfl_down_d(pr, 4));
        const double a8 = shfl_down_d(A2, 8), a16 = shfl_down_d(A2, 16), a24 = shfl_down_d(A2, 24);
        const double S = dadd(dadd(dadd(A2, a8), a16), a24);
        const double u = dadd(S, shfl_down_d(S, 2));
        dot = shfl_d(dadd(u, shfl_down_d(u, 1)), 0);
    }
    if (n1 < cnt) {  // FMA tail in index order, operands as (a, w) pairs from shared memory
        W->aw[lane] = make_double2(a, wv);
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 16; ++t) {  // tail length cnt - n1 < 16
            if (n1 + t < cnt) {
                const double2 q = W->aw[n1 + t];
                dot = dfma(q.x, q.y, dot);
            }
        }
        __syncwarp();
    }
    const double v_new = dadd(constant, dot);
    if (v_new < f_cur) {  // strict accept (ccd.py:187-191)
        const double delta = dsub(t_new, bj);
        r = row ? dsub(r, dmul(xij, delta)) : r;
        sum_abs_b = dadd(sum_abs_b, dsub(fabs(t_new), fabs(bj)));
        f_cur = v_new;
        W->B[j] = t_new;  // every lane stores the same value: no cross-lane hazard
    }
}

// One exact coordinate step on axis j (ccd.py:160-193), all lanes in lock-step.
// NC > 0: compile-time row count (config shapes); NC == 0: runtime n_rt.
template <int PMAX, int NC>
__device__ __forceinline__ void warp_step(WarpShared<PMAX> *W, int lane, uint32_t inv_mask, const double *xrow,
                                          int n_rt, int j, double lam, bool col_sparse, double &r, double &f_cur,
                                          double &sum_abs_b, uint32_t &perm_valid)
{
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    const int n = NC > 0 ? NC : n_rt;
    const bool row = lane < n;
    const double xij = xrow[j];  // lanes >= n read a stale in-bounds slot, never used
    const double bj = W->B[j];
    if (!col_sparse) {
        // np.divide then += b[j] (ccd.py:165-166).  Pad lanes divide 1/1: a zero
        // numerator would send the whole warp through __ddiv_rn's slow path.
        const double q = ddiv(row ? r : 1.0, row ? xij : 1.0);
        const double loc = row ? dadd(q, bj) : (lane == n ? 0.0 : INF);
        const double w = row ? fabs(xij) : (lane == n ? lam : 0.0);
        median_update<PMAX, (NC > 0 ? NC + 1 : 0)>(W, lane, inv_mask, j, lam, true, n + 1, loc, w, 0.0, false, row,
                                                   xij, bj, r, f_cur, sum_abs_b, perm_valid);
    } else {
        double loc, w, zsum;
        int cnt;
        sparse_column<PMAX>(W, lane, n, r, xij, bj, lam, loc, w, cnt, zsum);
        median_update<PMAX, 0>(W, lane, inv_mask, j, lam, false, cnt, loc, w, zsum, true, row, xij, bj, r, f_cur,
                               sum_abs_b, perm_valid);
    }
}

template <int PMAX>
__device__ __forceinline__ double warp_objective(WarpShared<PMAX> *W, int lane, int n, int p, double lam)
{
    double v = 0.0;
    if (lane < n) {
        double g = gemv_row(p, lane, n, [&](int q) { return W->X[lane * p + q]; }, [&](int q) { return W->B[q]; });
        v = fabs(dsub(W->Y[lane], g));
    }
    double rs = warp_np_sum(v, n, lane);
    double bs = np_sum(p, [&](int q) { return fabs(W->B[q]); });
    return dadd(rs, dmul(lam, bs));
}

// ccd_descend (ccd.py:126-206) for the descent request in C, all lanes.
template <int PMAX, int NC>
__device__ __noinline__ void warp_descent(WarpShared<PMAX> *W, Ctl<PMAX> &C, int lane, uint32_t inv_mask, int n_rt,
                                          int p_rt, uint32_t &perm_valid_io)
{
    const int n = NC > 0 ? NC : n_rt;
    const int p = NC > 0 ? PMAX : p_rt;
    uint32_t perm_valid = perm_valid_io;  // register copy for the step loop
    const int frozen = C.req_frozen;
    const double tol = C.req_tol;
    const int max_sweeps = C.req_sweeps;
    const double lam = C.lam;
    const uint32_t sparse = C.sparse_mask;
    if (lane < p) W->B[lane] = C.req_start[lane];
    __syncwarp();
    double r = 0.0;
    if (lane < n) {
        double g = gemv_row(p, lane, n, [&](int q) { return W->X[lane * p + q]; }, [&](int q) { return W->B[q]; });
        r = dsub(W->Y[lane], g);
    }
    const double *xrow = W->X + lane * p;
    const double sb = np_sum(p, [&](int q) { return fabs(W->B[q]); });
    double f_cur = dadd(warp_np_sum(fabs(r), n, lane), dmul(lam, sb));
    double f_sweep_start = f_cur, sum_abs_b = sb;
    int sweeps = 1, steps = 0, conv = 0;
    const int j0 = (frozen == 0) ? 1 : 0;
    int j = j0;
    if (j >= p) {
        conv = 1;
    } else {
        for (;;) {
            warp_step<PMAX, NC>(W, lane, inv_mask, xrow, n, j, lam, (sparse >> j) & 1u, r, f_cur, sum_abs_b,
                                perm_valid);
            ++steps;
            int jn = j + 1;
            jn += (jn == frozen);
            if (jn < p) {
                j = jn;
                continue;
            }
            if (dsub(f_sweep_start, f_cur) < tol) {
                conv = 1;
                break;
            }
            if (sweeps >= max_sweeps) break;
            ++sweeps;
            f_sweep_start = f_cur;
            sum_abs_b = np_sum(p, [&](int q) { return fabs(W->B[q]); });
            j = j0;
        }
    }
    perm_valid_io = perm_valid;
    __syncwarp();
    const double obj = warp_objective<PMAX>(W, lane, n, p, lam);
    const int D = C.D;
    const long long S = C.S;
    __syncwarp();
    if (lane < p) C.res_beta[lane] = W->B[lane];
    if (lane == 0) {
        C.res_obj = obj;
        C.res_conv = conv;
        C.res_sweeps = sweeps;
        C.res_steps = steps;
        C.D = D + 1;
        C.S = S + steps;
    }
    __syncwarp();
}

// PMAX: beta capacity; NC > 0 specialises the row count (and p == PMAX).
template <int PMAX, int NC>
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK, 4) locus_warp_kernel(LocusArgs A)
{
    __shared__ WarpShared<PMAX> WS[WARPS_PER_BLOCK];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpShared<PMAX> *W = &WS[wib];
    const int n = NC > 0 ? NC : A.n, p = NC > 0 ? PMAX : A.p;
    const int slot = blockIdx.x * WARPS_PER_BLOCK + wib;
    WarpAccess<PMAX> acc{n, p, lane, W};
    const uint32_t inv_mask = bitonic_inv_mask(lane);
    // cached breakpoint orders per axis (validated before every use, so they
    // may be carried across descents and problems)
    uint32_t perm_valid = 0;
    Ctl<PMAX> &C = W->C;
    if (lane == 0) C.pc = PC_FETCH;
    __syncwarp();
    for (;;) {
        int act = controller<PMAX>(C, A, acc, slot);
        __syncwarp();
        if (act == ACT_EXIT) break;
        warp_descent<PMAX, NC>(W, C, lane, inv_mask, n, p, perm_valid);
    }
}

}  // namespace lad
