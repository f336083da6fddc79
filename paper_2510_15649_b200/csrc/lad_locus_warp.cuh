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
constexpr int WARPS_PER_BLOCK = 8;

template <int PMAX>
struct WarpShared {
    Ctl<PMAX> C;
    double X[32 * PMAX];  // row-major [i * p + j]
    double Y[32];
    double B[PMAX];       // beta of the running descent (warp-uniform)
    double sa[32], sw[32], sz[32];
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
        unsigned long long pr = 0;
        if (lane == 0) pr = atomicAdd(A.counter, 1ULL);
        pr = __shfl_sync(FULLMASK, pr, 0);
        if ((int64_t)pr >= A.B) return -1;
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

// One exact coordinate step on axis j (ccd.py:160-193), all lanes.
template <int PMAX>
__device__ __forceinline__ void warp_step(WarpShared<PMAX> *W, int lane, int n, int p, int j, double lam,
                                          bool col_sparse, double &r, double &f_cur, double &sum_abs_b)
{
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    const bool row = lane < n;
    const double xij = row ? W->X[lane * p + j] : 0.0;
    const double bj = W->B[j];
    double loc, w, zsum = 0.0;
    int cnt;
    bool have_zero = false;
    if (!col_sparse) {
        loc = row ? dadd(ddiv(r, xij), bj) : (lane == n ? 0.0 : INF);  // np.divide then += b[j]
        w = row ? fabs(xij) : (lane == n ? lam : 0.0);
        cnt = n + 1;
    } else {
        // _AxisWorkspace with zero rows (ccd.py:94-110, :167-169, :178-179)
        const bool nz = row && xij != 0.0;
        const unsigned nzm = __ballot_sync(FULLMASK, nz);
        const unsigned zm = __ballot_sync(FULLMASK, row && xij == 0.0);
        const unsigned lt = (1u << lane) - 1u;
        const int k = __popc(nzm), z = __popc(zm);
        const bool dense = (k == n);
        if (nz) {
            W->sa[__popc(nzm & lt)] = dense ? dadd(ddiv(r, xij), bj) : ddiv(dadd(r, dmul(xij, bj)), xij);
            W->sw[__popc(nzm & lt)] = fabs(xij);
        }
        if (row && xij == 0.0) W->sz[__popc(zm & lt)] = fabs(r);
        __syncwarp();
        loc = lane < k ? W->sa[lane] : (lane == k ? 0.0 : INF);
        w = lane < k ? W->sw[lane] : (lane == k ? lam : 0.0);
        double zv = lane < z ? W->sz[lane] : 0.0;
        __syncwarp();
        have_zero = z > 0;
        zsum = have_zero ? warp_np_sum(zv, z, lane) : 0.0;
        cnt = k + 1;
    }
    // ---- weighted median (ccd.py:81-91)
    double key = loc;
    int idx = lane;
    bitonic32(key, idx, lane);
    const double ws = shfl_d(w, idx);
    double c = ws;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        double t = __shfl_up_sync(FULLMASK, c, d);
        if (lane >= d) c = dadd(c, t);
    }
    const bool in = lane < cnt;
    double total = shfl_d(c, cnt - 1);
    double half = dmul(0.5, total);
    int k = __popc(__ballot_sync(FULLMASK, in && c < half));
    double ck = shfl_d(c, k < cnt ? k : cnt - 1);
    const double marg = dmul(1e-13, total);
    bool risky = __any_sync(FULLMASK, in && fabs(dsub(c, half)) <= marg) ||
                 fabs(dsub(fabs(dsub(ck, half)), dmul(1e-12, total))) <= marg;
    if (risky) {  // exact: numpy's sequential cumsum in sorted order
        double ce = 0.0;
        for (int i = 0; i < 32; ++i) {
            double wi = shfl_d(ws, i);
            if (i <= lane) ce = dadd(ce, wi);
        }
        total = shfl_d(ce, cnt - 1);
        half = dmul(0.5, total);
        k = __popc(__ballot_sync(FULLMASK, in && ce < half));
        ck = shfl_d(ce, k < cnt ? k : cnt - 1);
    }
    const bool tie = (k + 1 < cnt) && fabs(dsub(ck, half)) <= dmul(1e-12, total);
    const int ks = k < cnt ? k : cnt - 1;
    const double tk = shfl_d(key, ks);
    const double tk1 = shfl_d(key, ks + 1 < 32 ? ks + 1 : 31);
    const double t_new = tie ? dmul(0.5, dadd(tk, tk1)) : tk;
    // ---- skip / evaluate / accept (ccd.py:172-191)
    if (fabs(dsub(t_new, bj)) <= dmul(1e-14, dadd(1.0, fabs(bj)))) return;
    double constant = dmul(lam, dsub(sum_abs_b, fabs(bj)));
    if (have_zero) constant = dadd(constant, zsum);
    const double a = lane < cnt ? fabs(dsub(t_new, loc)) : 0.0;
    const double dot = warp_blas_ddot<PMAX>(a, lane < cnt ? w : 0.0, cnt, lane, W);
    const double v_new = dadd(constant, dot);
    if (v_new < f_cur) {
        const double delta = dsub(t_new, bj);
        if (row) r = dsub(r, dmul(xij, delta));
        sum_abs_b = dadd(sum_abs_b, dsub(fabs(t_new), fabs(bj)));
        f_cur = v_new;
        __syncwarp();
        if (lane == 0) W->B[j] = t_new;
        __syncwarp();
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
template <int PMAX>
__device__ __noinline__ void warp_descent(WarpShared<PMAX> *W, Ctl<PMAX> &C, int lane, int n, int p)
{
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
    const double sb = np_sum(p, [&](int q) { return fabs(W->B[q]); });
    double f_cur = dadd(warp_np_sum(fabs(r), n, lane), dmul(lam, sb));
    double f_sweep_start = f_cur, sum_abs_b = sb;
    int sweeps = 1, steps = 0, conv = 0;
    int j = (frozen == 0) ? 1 : 0;
    if (j >= p) {
        conv = 1;
    } else {
        for (;;) {
            warp_step<PMAX>(W, lane, n, p, j, lam, (sparse >> j) & 1u, r, f_cur, sum_abs_b);
            ++steps;
            int jn = j + 1;
            if (jn == frozen) ++jn;
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
            j = (frozen == 0) ? 1 : 0;
        }
    }
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

template <int PMAX>
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK) locus_warp_kernel(LocusArgs A)
{
    __shared__ WarpShared<PMAX> WS[WARPS_PER_BLOCK];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpShared<PMAX> *W = &WS[wib];
    const int n = A.n, p = A.p;
    const int slot = blockIdx.x * WARPS_PER_BLOCK + wib;
    WarpAccess<PMAX> acc{n, p, lane, W};
    Ctl<PMAX> &C = W->C;
    if (lane == 0) C.pc = PC_FETCH;
    __syncwarp();
    for (;;) {
        int act = controller<PMAX>(C, A, acc, slot);
        __syncwarp();
        if (act == ACT_EXIT) break;
        warp_descent<PMAX>(W, C, lane, n, p);
    }
}

}  // namespace lad
