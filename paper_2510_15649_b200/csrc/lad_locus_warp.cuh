// lad_locus_warp.cuh -- warp-per-problem locus kernel (n + 1 <= 32 breakpoints).
//
// One warp solves one problem at a time (persistent grid, per-warp work
// stealing).  Lane i owns data row i and its residual r_i; lane n carries the
// lambda breakpoint at 0; lanes > n are +inf pads.  Per coordinate step
// (ccd.py:160-193):
//   * breakpoints r_i / x_ij + b_j: one division per lane;
//   * weighted median: test the axis' last median element (then the one
//     before it, then its neighbours in order) with two exact fixed-point
//     warp sums against half the total weight, decided only beyond a margin;
//     otherwise order all (location, index) pairs (a 32-lane bitonic
//     network of shuffles) and scan the weights
//     (FP32 Kogge-Stone with a margin, else numpy's exact sequential cumsum),
//     so the result is always the reference's;
//   * v_new: OpenBLAS ddot's summation tree mapped onto shuffles, the FMA tail
//     through shared memory.
// Control flow (the controller state machine shared with the thread kernel)
// is warp-uniform: all lanes run it on one shared Ctl.
//
// Element type T: double is the reference's arithmetic (bit-exact); float is
// the fp32 mode -- data, residuals, breakpoints, medians and objectives in
// binary32 with the same operation order, while the outer search (brackets,
// probe positions, warm starts: the controller) stays binary64.  Probe
// positions and warm starts are rounded to binary32 when a descent starts and
// its results are widened exactly.
#pragma once
#include "lad_locus.cuh"

namespace lad {

constexpr unsigned FULLMASK = 0xffffffffu;
// Launch shape: 4 blocks per SM of 8 warps (32 warps/SM, 64 registers), except
// binary64 p = 8: 5 blocks of 5 warps (25 warps/SM, 72 registers), the most that
// fit with its reciprocal table in shared memory (8.5 KB per warp).  Same-box
// A/B: 32 warps are +3% for config 2, +3.4% for config 4 in fp32; config 4 in
// fp64 (its longer step body spills less at 72 registers): 8 x 4 at 64 registers
// -6% against 7 x 4 at 72; with the table 6 x 4 +2% and 5 x 5 +4% against 7 x 4
// without it; 5 x 6 without the table -7.5%.  36 warps at 56 registers: -3% for
// config 2.
#ifndef LAD_WARP_WARPS_NARROW
#define LAD_WARP_WARPS_NARROW 8
#endif
#ifndef LAD_WARP_WARPS_WIDE
#define LAD_WARP_WARPS_WIDE 5
#endif
#ifndef LAD_WARP_F32_WIDE  // binary32 p = 8 with the binary64 p = 8 shape (72 registers)
#define LAD_WARP_F32_WIDE 0
#endif
#ifndef LAD_WARP_MIN_BLOCKS
#define LAD_WARP_MIN_BLOCKS 4
#endif
constexpr int WARP_MIN_BLOCKS = LAD_WARP_MIN_BLOCKS;
#ifndef LAD_WARP_MIN_BLOCKS_WIDE  // binary64 p = 8
#define LAD_WARP_MIN_BLOCKS_WIDE 5
#endif
template <int PMAX, typename T>
constexpr int warps_per_block = (PMAX <= 5 || (sizeof(T) == 4 && !LAD_WARP_F32_WIDE)) ? LAD_WARP_WARPS_NARROW
                                                                                    : LAD_WARP_WARPS_WIDE;
template <int PMAX, typename T>
constexpr int warp_min_blocks = (PMAX <= 5 || (sizeof(T) == 4 && !LAD_WARP_F32_WIDE)) ? LAD_WARP_MIN_BLOCKS
                                                                                    : LAD_WARP_MIN_BLOCKS_WIDE;

// Division by a precomputed reciprocal: q = RN(r * y), then two corrections
// q += RN(r - q * x) * y with y = RN(1 / x).  The first makes q faithful, the
// second is then correctly rounded (Markstein's theorem), so q == r / x in
// round-to-nearest whenever nothing under- or overflows: |r| and |x| within
// 2^+-450 (binary64) or 2^+-50 (binary32).  Used where shared memory holds the
// reciprocal table.  (For binary64 p = 8 the table lost 13% while the X copy's
// even row stride put a 16-way bank conflict on every x_ij and 1/x_ij load;
// with the odd stride (xs_v) and a launch shape that fits it, it wins 4%.)
#ifndef LAD_WARP_FASTDIV8  // the reciprocal table for binary64 p = 8 too
#define LAD_WARP_FASTDIV8 1
#endif
template <int PMAX, typename T>
constexpr bool fast_div_v = sizeof(T) == 4 || PMAX <= 5 || LAD_WARP_FASTDIV8;

// Pad rows as data (with the reciprocal table): row n of X holds lambda and
// rows > n hold 0, and the pad lanes' residual stays 1, so every lane's
// breakpoint weight is |x_ij| and every lane divides r / x without the pad
// selects (a pad lane's quotient is finite and discarded).
#ifndef LAD_WARP_PADX
#define LAD_WARP_PADX 1
#endif
template <int PMAX, typename T>
constexpr bool padx_v = LAD_WARP_PADX && fast_div_v<PMAX, T>;
// Descent loop specialised for problems without sparse columns (compile-time
// n kernels), optionally with the sweep over the axes unrolled.
#ifndef LAD_WARP_DENSE_LOOP
#define LAD_WARP_DENSE_LOOP 1
#endif
#ifndef LAD_WARP_UNROLL
#define LAD_WARP_UNROLL 0
#endif
// Step micro-variants (same-box A/B): the through-weight of the median guess
// as the below-weight plus its own weight (a shuffle instead of a second
// REDUX); the margin bounds (half -+ margin) precomputed per axis (one
// 64-bit load instead of load + REDUX + two adds); the walk's neighbour from
// the high key word alone when it is unique (one REDUX per hop instead of
// two); the ddot lane tree from products staged in shared memory (no
// shuffles).
#ifndef LAD_WARP_QI_SHFL
#define LAD_WARP_QI_SHFL 0
#endif
#ifndef LAD_WARP_HQ_PAIR
#define LAD_WARP_HQ_PAIR 1
#endif
#ifndef LAD_WARP_WALK_POPC
#define LAD_WARP_WALK_POPC 0
#endif
#ifndef LAD_WARP_DDOT_SMEM
#define LAD_WARP_DDOT_SMEM 0
#endif
// Dense descent loop over a packed list of the free axes (no per-step axis
// bookkeeping); ddot tail operands stored signed with |.| folded into DFMA.
#ifndef LAD_WARP_AXIS_LIST
#define LAD_WARP_AXIS_LIST 0
#endif
#ifndef LAD_WARP_RAW_AW
#define LAD_WARP_RAW_AW 0
#endif
// IEEE division (binary64 p = 8, no reciprocal table) with zero dividends kept
// off its slow path (ddiv_zero_fast).  Neutral here (config 4: -0.6%, same box):
// one lane per warp meets a zero, unlike the thread kernel's 10 rows per lane.
#ifndef LAD_WARP_ZDIV
#define LAD_WARP_ZDIV 0
#endif
// Controller inlined into the warp kernel's outer loop (warp_descent stays out
// of line).
#ifndef LAD_WARP_INLINE_CTL
#define LAD_WARP_INLINE_CTL 1
#endif
// The nearest-seen-point argmin (locus.py:188-191) by REDUX minima on the
// distance's bit pattern and the index instead of a five-round shuffle tree.
#ifndef LAD_WARP_NEAREST_REDUX
#define LAD_WARP_NEAREST_REDUX 1
#endif
// Controller vectors (descent start, result beta, curve points) copied one
// element per lane (WarpAccess::lanes) instead of by every lane in turn.
#ifndef LAD_WARP_CTL_LANES
#define LAD_WARP_CTL_LANES 1
#endif
// The median test's half-total weight by a broadcast load (1 instruction)
// instead of a REDUX into a uniform register.
#ifndef LAD_WARP_HQ_LDS
#define LAD_WARP_HQ_LDS 0
#endif

// Row stride of the per-warp X (and 1/X) copy in elements: p | 1.  Lane i reads x_ij at i * xs + j;
// with an even stride (p = 8: 16 words) lanes two apart hit the same bank pair, a 16-way conflict
// on the step's x_ij load and on every row product of the residual init and the objective.
template <int PMAX>
constexpr int xs_v = PMAX | 1;

template <int PMAX, typename T>
struct WarpShared {
    using T2 = typename vec2_of<T>::type;
    Ctl<PMAX> C;
    T X[32 * xs_v<PMAX>];  // row-major [i * xs + j], xs = p | 1: an odd row stride keeps lane i's row off lane i'+-k's banks
    T RX[fast_div_v<PMAX, T> ? 32 * xs_v<PMAX> : 1];  // RN(1 / x), same layout; 1 for pad lanes
    T Y[32];
    T B[PMAX];       // beta of the running descent (warp-uniform)
    T sa[32], sw[32], sz[32];
    T2 aw[32];       // (|t - loc_i|, w_i) pairs for the ddot FMA tail
    T2 sl[2];        // ddot lane-tree partial sums (S0, S1), (S2, S3)
    int cand[PMAX];      // per axis: element that was the weighted median last time (a guess)
    unsigned wq[PMAX][32];  // per axis: weights in fixed point, floor(w_i * 2^30 / total)
    unsigned halfq[PMAX];   // per axis: (sum of wq) / 2
    uint2 hqb[PMAX];        // per axis: (halfq - margin (0 if below), halfq + margin)
    double *seen;           // this slot's seen-list scratch (null when unused), set at kernel start
    alignas(16) T pp[LAD_WARP_DDOT_SMEM ? 32 : 2];  // ddot lane-tree products (LAD_WARP_DDOT_SMEM), lane l's four at [4 l, 4 l + 4) (n1 = 16) / [8 l, 8 l + 8)
};

// margin of the fixed-point median test, in units of 2^-30 of the total weight
// (1.5e-5 * total; quantisation error <= 32 units, FP64 cumsum error ~1e-14 * total)
constexpr unsigned MEDIAN_MARGIN_Q = 1u << 14;

// Order-preserving unsigned image of a breakpoint location (-0 folded onto +0,
// so equal locations have equal keys), for warp min/max reductions.
template <typename T>
struct OrderKey;

template <>
struct OrderKey<double> {
    unsigned hi, lo;
    __device__ __forceinline__ explicit OrderKey(double v)
    {
        const long long b = __double_as_longlong(__dadd_rn(v, 0.0));
        const unsigned long long k = (unsigned long long)b ^ (b < 0 ? ~0ull : (1ull << 63));
        hi = (unsigned)(k >> 32);
        lo = (unsigned)k;
    }
    // Lane of the first (after = true: smallest key, lowest lane on equal keys)
    // or last (largest key, highest lane) element among the lanes with `side`;
    // -1 if no lane has it.  Warp-uniform.
    __device__ __forceinline__ int nearest(bool side, bool after) const
    {
        const unsigned h = after ? hi : ~hi, l = after ? lo : ~lo;
        const unsigned mh = __reduce_min_sync(FULLMASK, side ? h : ~0u);
        const bool c1 = side && h == mh;
        if constexpr (LAD_WARP_WALK_POPC) {  // a unique high word decides (no side lane has h = ~0)
            const unsigned b1 = __ballot_sync(FULLMASK, c1);
            if (b1 == 0u) return -1;
            if ((b1 & (b1 - 1u)) == 0u) return __ffs(b1) - 1;
        }
        const unsigned ml = __reduce_min_sync(FULLMASK, c1 ? l : ~0u);
        const unsigned bal = __ballot_sync(FULLMASK, c1 && l == ml);
        if (bal == 0u) return -1;
        return after ? __ffs(bal) - 1 : 31 - __clz(bal);
    }
};

template <>
struct OrderKey<float> {
    unsigned k;
    __device__ __forceinline__ explicit OrderKey(float v)
    {
        const unsigned b = __float_as_uint(__fadd_rn(v, 0.0f));
        k = b ^ ((b >> 31) ? ~0u : (1u << 31));
    }
    __device__ __forceinline__ int nearest(bool side, bool after) const
    {
        const unsigned h = after ? k : ~k;
        const unsigned mh = __reduce_min_sync(FULLMASK, side ? h : ~0u);
        const unsigned bal = __ballot_sync(FULLMASK, side && h == mh);
        if (bal == 0u) return -1;
        return after ? __ffs(bal) - 1 : 31 - __clz(bal);
    }
};

template <typename T>
__device__ __forceinline__ T shfl_t(T v, int src) { return __shfl_sync(FULLMASK, v, src); }
template <typename T>
__device__ __forceinline__ T shfl_down_t(T v, int d) { return __shfl_down_sync(FULLMASK, v, d); }
template <typename T>
__device__ __forceinline__ T shfl_xor_t(T v, int m) { return __shfl_xor_sync(FULLMASK, v, m); }
// binary64: shuffle the two 32-bit halves explicitly (keeps the halves in
// their registers; the generic overload lets the compiler swap them back)
template <>
__device__ __forceinline__ double shfl_t<double>(double v, int src)
{
    const int lo = __shfl_sync(FULLMASK, __double2loint(v), src);
    const int hi = __shfl_sync(FULLMASK, __double2hiint(v), src);
    return __hiloint2double(hi, lo);
}
template <>
__device__ __forceinline__ double shfl_down_t<double>(double v, int d)
{
    const int lo = __shfl_down_sync(FULLMASK, __double2loint(v), d);
    const int hi = __shfl_down_sync(FULLMASK, __double2hiint(v), d);
    return __hiloint2double(hi, lo);
}
template <>
__device__ __forceinline__ double shfl_xor_t<double>(double v, int m)
{
    const int lo = __shfl_xor_sync(FULLMASK, __double2loint(v), m);
    const int hi = __shfl_xor_sync(FULLMASK, __double2hiint(v), m);
    return __hiloint2double(hi, lo);
}

// numpy pairwise_sum of cnt values held one per lane (lane i -> element i).
template <typename T>
__device__ __forceinline__ T warp_np_sum(T v, int cnt, int lane)
{
    if (cnt < 8) {
        T res = T(0);
        for (int i = 0; i < cnt; ++i) res = dadd(res, shfl_t(v, i));
        return res;
    }
    const int lim = cnt - (cnt % 8);
    T acc = v;
    for (int blk = 8; blk < lim; blk += 8) acc = dadd(acc, shfl_t(v, (lane + blk) & 31));
    acc = dadd(acc, shfl_xor_t(acc, 1));
    acc = dadd(acc, shfl_xor_t(acc, 2));
    acc = dadd(acc, shfl_xor_t(acc, 4));
    T res = shfl_t(acc, 0);
    for (int i = lim; i < cnt; ++i) res = dadd(res, shfl_t(v, i));
    return res;
}

// Access policy: the whole warp works on one problem held in WarpShared.
template <int PMAX, typename T>
struct WarpAccess {
    static constexpr bool kYield = false;  // controller states jump directly (lad_locus.cuh, ACT_YIELD)
    int n, p, lane;
    WarpShared<PMAX, T> *W;
    int xs;  // row stride of W->X / W->RX (p | 1)
    __device__ __forceinline__ bool leader() const { return lane == 0; }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    // the slot's seen list, computed once per kernel (WarpShared::seen)
    template <int PM>
    __device__ __forceinline__ double *seen_base(const LocusArgs &, int) const
    {
        return W->seen;
    }
    // Controller vectors one element per lane (LAD_WARP_CTL_LANES) instead of
    // every lane repeating the whole loop on the shared Ctl; the warp syncs
    // around the writes (the other lanes read them next).
    template <class F>
    __device__ __forceinline__ void lanes(int cnt, F f) const
    {
        if constexpr (LAD_WARP_CTL_LANES) {
            __syncwarp();
            if (lane < cnt) f(lane);
            __syncwarp();
        } else {
            for (int k = 0; k < cnt; ++k) f(k);
        }
    }
    template <class F>
    __device__ __forceinline__ void lanes_out(int cnt, F f) const
    {
        if constexpr (LAD_WARP_CTL_LANES) {
            if (lane < cnt) f(lane);
        } else if (lane == 0) {
            for (int k = 0; k < cnt; ++k) f(k);
        }
    }
    template <int PM>
    __device__ __forceinline__ void copy_point(Point<PM> &d, const Point<PM> &s) const
    {
        if constexpr (LAD_WARP_CTL_LANES) {
            static_assert(sizeof(Point<PM>) % 8 == 0, "Point is copied in 8-byte words");
            constexpr int nw = sizeof(Point<PM>) / 8;
            __syncwarp();
            if (lane < nw) reinterpret_cast<unsigned long long *>(&d)[lane] =
                               reinterpret_cast<const unsigned long long *>(&s)[lane];
            __syncwarp();
        } else {
            d = s;
        }
    }
    // count one finished unit on *ctr (lane 0, after the warp's global writes are
    // fenced); true in every lane for the warp that completes `of` units
    __device__ __forceinline__ bool last_of(unsigned *ctr, unsigned of) const
    {
        __syncwarp();
        unsigned old = 0;
        if (lane == 0) {
            __threadfence();
            old = atomicAdd(ctr, 1u);
            __threadfence();
        }
        return __shfl_sync(FULLMASK, old, 0) == of - 1u;
    }
    __device__ int fetch(Ctl<PMAX> &C, const LocusArgs &A) const
    {
        const int div = A.axis_mode == AXIS_SEARCH ? p : 1;
        unsigned long long item = 0;
        if (lane == 0) item = atomicAdd(A.counter, 1ULL);
        item = __shfl_sync(FULLMASK, item, 0);
        if ((int64_t)item >= A.B * div) return -1;
        const unsigned long long pr = item / div;
        int64_t src = A.data_index ? A.data_index[pr] : (int64_t)pr;
        if (src < 0 || src >= A.Bd) {  // data_index out of range: invalid input (warp-uniform)
            __syncwarp();
            C.prob = (int64_t)pr;
            C.arank = (int)(item % div);
            __syncwarp();
            if (lane == 0) write_invalid<PMAX>(A, (int64_t)pr, p);
            return 0;
        }
        const T *xsrc, *ysrc;
        if constexpr (sizeof(T) == 4) {
            xsrc = A.Xf;
            ysrc = A.Yf;
        } else {
            xsrc = A.X;
            ysrc = A.Y;
        }
        const T *xg = xsrc + (size_t)src * n * p;
        const T *yg = ysrc + (size_t)src * n;
        bool ok = true;
        uint32_t mask = 0;
        for (int e = lane; e < n * p; e += 32) {
            T v = xg[e];
            const int i = e / p, j = e - i * p;
            W->X[i * xs + j] = v;
            ok = ok && isfinite(v);
            if (v == T(0)) mask |= 1u << j;
            if constexpr (fast_div_v<PMAX, T>) {
                W->RX[i * xs + j] = rcp_rn(v);
                if (!div_operand_safe(v)) mask |= 1u << j;  // column takes the generic path
            }
        }
        if constexpr (fast_div_v<PMAX, T>)
            for (int e = n * p + lane; e < 32 * p; e += 32) {
                const int i = e / p, j = e - i * p;
                W->RX[i * xs + j] = T(1);
            }
        for (int i = lane; i < n; i += 32) {
            T v = yg[i];
            W->Y[i] = v;
            ok = ok && isfinite(v);
        }
        ok = __all_sync(FULLMASK, ok);
        mask = __reduce_or_sync(FULLMASK, mask);
        double lraw;
        if constexpr (sizeof(T) == 4) lraw = (double)A.lamf[pr];
        else lraw = A.lam[pr];
        ok = ok && isfinite(lraw) && lraw >= 0.0;
        const double lam_eff = lraw > A.prm.lambda_floor ? lraw : A.prm.lambda_floor;
        if constexpr (padx_v<PMAX, T>)  // row n: the lambda breakpoint's weight; rows > n: weight 0
            for (int e = n * p + lane; e < 32 * p; e += 32) {
                const int i = e / p, j = e - i * p;
                W->X[i * xs + j] = i == n ? T(lam_eff) : T(0);
            }
        __syncwarp();
        // fixed-point breakpoint weights of each axis (median fast path): any
        // summation order will do, the test keeps a margin of 2^14 units
        for (int j = 0; j < p; ++j) {
            const double wd = lane < n ? (double)fabs(W->X[lane * xs + j]) : (lane == n ? (double)T(lam_eff) : 0.0);
            double tot = wd;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(FULLMASK, tot, off);
            const double scale = 1073741824.0 / (tot * (1.0 + 1e-9));
            // (a finite scale keeps every q below 2^30; a total below ~6e-300 would overflow it)
            const unsigned q = (tot > 0.0 && tot < 1e300 && scale < 1e300) ? __double2uint_rz(wd * scale) : 0u;
            W->wq[j][lane] = q;
            const unsigned sq = __reduce_add_sync(FULLMASK, q);
            if (lane == 0) {
                const unsigned hq = sq / 2u;
                W->halfq[j] = hq;
                W->hqb[j] = make_uint2(hq >= MEDIAN_MARGIN_Q ? hq - MEDIAN_MARGIN_Q : 0u, hq + MEDIAN_MARGIN_Q);
            }
        }
        C.prob = (int64_t)pr;
        C.arank = (int)(item % div);
        C.lam = lam_eff;
        C.sparse_mask = mask;
        __syncwarp();
        if (!ok) {
            if (lane == 0) write_invalid<PMAX>(A, (int64_t)pr, p);
            return 0;
        }
        return 1;
    }
    // np.abs(x).sum(axis=0)[j] in T, widened for the binary64 controller
    __device__ double col_abs_sum(int j) const
    {
        if (p == 1) return (double)np_sum(n, [&](int i) { return fabs(W->X[i]); });
        T s = T(0);
        for (int i = 0; i < n; ++i) s = dadd(s, fabs(W->X[i * xs + j]));
        return (double)s;
    }
    __device__ double y_absmax(const double *) const
    {
        T ymax = T(0);
        for (int i = 0; i < n; ++i) {
            T a = fabs(W->Y[i]);
            if (i == 0 || a > ymax) ymax = a;
        }
        return (double)ymax;
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
        if constexpr (LAD_WARP_NEAREST_REDUX) {
            // (distance, k) lexicographic minimum by three REDUX.MIN: a distance
            // is >= 0, so its bit pattern orders like its value (high word, then
            // low word), and among equal distances the lowest k wins (the
            // reference's first minimum).  Lanes without an entry hold (inf, INT_MAX).
            const unsigned long long bits = (unsigned long long)__double_as_longlong(bd);
            const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
            const unsigned mh = __reduce_min_sync(FULLMASK, hi);
            const bool c1 = hi == mh;
            const unsigned ml = __reduce_min_sync(FULLMASK, c1 ? lo : ~0u);
            const bool c2 = c1 && lo == ml;
            const unsigned mk = __reduce_min_sync(FULLMASK, c2 ? (unsigned)bk : ~0u);
            return mk >= 0x7fffffffu ? -1 : (int)mk;
        } else {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                double od = shfl_xor_t(bd, off);
                int ok = __shfl_xor_sync(FULLMASK, bk, off);
                if (od < bd || (od == bd && ok < bk)) {
                    bd = od;
                    bk = ok;
                }
            }
            return bk == 0x7fffffff ? -1 : bk;
        }
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
template <typename T>
__device__ __forceinline__ void bitonic32m(T &key, int &idx, uint32_t inv_mask)
{
    int s = 0;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1, ++s) {
            T pk = shfl_xor_t(key, j);
            int pi = __shfl_xor_sync(FULLMASK, idx, j);
            bool plt = (pk < key) | ((pk == key) & (pi < idx));
            bool take = plt != (((inv_mask >> s) & 1u) != 0u);
            key = take ? pk : key;
            idx = take ? pi : idx;
        }
    }
}

// numpy's sequential cumsum in sorted order, recomputed exactly (rare path:
// only when the parallel scan leaves a comparison within its error margin).
template <typename T>
__device__ __forceinline__ void exact_cumsum_decision(T ws, int lane, int cnt, int &k, T &ck, T &total, T &half)
{
    T ce = T(0);
    for (int i = 0; i < 32; ++i) {
        T wi = shfl_t(ws, i);
        if (i <= lane) ce = dadd(ce, wi);
    }
    total = shfl_t(ce, cnt - 1);
    half = dmul(T(0.5), total);
    k = __popc(__ballot_sync(FULLMASK, lane < cnt && ce < half));
    ck = shfl_t(ce, k < cnt ? k : cnt - 1);
}

// _AxisWorkspace for a column with zero entries (ccd.py:94-110, :167-169,
// :178-179): nonzero rows compacted to lanes 0..k-1 in row order, the zero
// rows' |r| summed with numpy's pairwise order.  Rare path.
template <int PMAX, typename T>
__device__ __forceinline__ void sparse_column(WarpShared<PMAX, T> *W, int lane, int n, T r, T xij, T bj, T lam,
                                              T &loc, T &w, int &cnt, T &zsum)
{
    const T INF = inf_of<T>();
    const bool row = lane < n;
    const bool nz = row && xij != T(0);
    const unsigned nzm = __ballot_sync(FULLMASK, nz);
    const unsigned zm = __ballot_sync(FULLMASK, row && xij == T(0));
    const unsigned lt = (1u << lane) - 1u;
    const int k = __popc(nzm), z = __popc(zm);
    const bool dense = (k == n);
    __syncwarp();
    if (nz) {
        W->sa[__popc(nzm & lt)] = dense ? dadd(ddiv(r, xij), bj) : ddiv(dadd(r, dmul(xij, bj)), xij);
        W->sw[__popc(nzm & lt)] = fabs(xij);
    }
    if (row && xij == T(0)) W->sz[__popc(zm & lt)] = fabs(r);
    __syncwarp();
    loc = lane < k ? W->sa[lane] : (lane == k ? T(0) : INF);
    w = lane < k ? W->sw[lane] : (lane == k ? lam : T(0));
    const T zv = lane < z ? W->sz[lane] : T(0);
    __syncwarp();
    zsum = z > 0 ? warp_np_sum(zv, z, lane) : T(0);
    cnt = k + 1;
}

// Weighted median by ordering (the walk's rare miss: a margin case, the first
// step of an axis, or a sparse column): stable order of (location, index) by
// the 32-lane bitonic network, then the cumulative-weight decision.
template <int PMAX, int CNTC, typename T>
__device__ __forceinline__ T median_by_order(WarpShared<PMAX, T> *W, int lane, uint32_t inv_mask, int j,
                                             bool cacheable, int cnt_rt, T loc, T w)
{
    const int cnt = CNTC > 0 ? CNTC : cnt_rt;
    T t_new;
    T key = loc;
    int idx = lane;
    bitonic32m(key, idx, inv_mask);
    const T ws = shfl_t(w, idx);
    // Cumulative weights only *locate* k = first cum >= total/2.  An FP32
    // Kogge-Stone scan differs from the sequential cumsum in T by at most
    // ~6 * 2^-24 * total (conversion + 5 tree levels); every comparison with
    // total/2 is accepted only beyond a 1e-5 * total margin, which also rules
    // out the 1e-12 * total flat-segment tie.  Otherwise (or on FP32
    // overflow/underflow) the exact sequential cumsum in T decides.
    float cf = static_cast<float>(ws);
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
        T ck, total, half;
        exact_cumsum_decision(ws, lane, cnt, k, ck, total, half);
        tie = (k + 1 < cnt) && fabs(dsub(ck, half)) <= dmul(T(1e-12), total);
    }
    const int ks = k < cnt ? k : cnt - 1;
    const T tk = shfl_t(key, ks);
    const T tk1 = shfl_t(key, ks + 1 < 32 ? ks + 1 : 31);
    t_new = tie ? dmul(T(0.5), dadd(tk, tk1)) : tk;
    if (cacheable) {  // identical values from every lane
        W->cand[j] = __shfl_sync(FULLMASK, idx, ks);
    }
    return t_new;
}

// Out-of-line copy for p <= 5: the miss path runs on ~10% of steps, and keeping it
// out of the step body keeps the hot path compact in the instruction cache
// (config 2: +5%).  For p = 8 misses are frequent enough that the call costs more.
template <int PMAX, int CNTC, typename T>
__device__ __noinline__ T median_by_order_call(WarpShared<PMAX, T> *W, int lane, uint32_t inv_mask, int j,
                                               bool cacheable, int cnt_rt, T loc, T w)
{
    return median_by_order<PMAX, CNTC, T>(W, lane, inv_mask, j, cacheable, cnt_rt, loc, w);
}

// Weighted median, skip test, v_new and strict accept of one coordinate step
// (ccd.py:81-91, :172-191), given this lane's breakpoint (loc, w).  CNTC > 0:
// compile-time breakpoint count (dense column in a compile-time-n kernel),
// so the reduction trees, tail lengths and bounds are constants.
template <int PMAX, int CNTC, typename T>
__device__ __forceinline__ void median_update(WarpShared<PMAX, T> *W, int lane, uint32_t inv_mask, int j, T lam,
                                              bool cacheable, int cnt_rt, T loc, T w, T zsum, bool have_zero,
                                              bool row, T xij, T bj, T &r, T &f_cur, T &sum_abs_b)
{
    const int cnt = CNTC > 0 ? CNTC : cnt_rt;
    // Fast path (dense columns): the weighted median is usually the same
    // element as at this axis' previous step.  Element m is the median iff the
    // weight of the elements ordered before it, W_below, satisfies
    // W_below < total/2 <= W_below + w_m (in numpy's sequential cumsum).  With
    // the weights in 2^-30-of-total fixed point (floor, <= 32 units of error
    // per sum) both sums are exact warp reductions, and a decision made with
    // a 2^14-unit (1.5e-5 * total) margin on both sides is the reference's
    // decision; it also excludes the 1e-12 * total midpoint tie.  Otherwise
    // the walk below finds the median, and as a last resort (margin cases, an
    // axis' first step, sparse columns) the full order + scan decides.
    T t_new;
    bool hit = false;
    if (cacheable) {
        const unsigned q = W->wq[j][lane];
        // margin bounds: element m is the median iff qb < lo_b and qi > hi_b
        unsigned lo_b, hi_b;
        if constexpr (LAD_WARP_HQ_PAIR) {
            const uint2 hb = W->hqb[j];
            lo_b = hb.x;
            hi_b = hb.y;
        } else {
            const unsigned hq = LAD_WARP_HQ_LDS ? W->halfq[j] : __reduce_max_sync(FULLMASK, W->halfq[j]);
            lo_b = hq >= MEDIAN_MARGIN_Q ? hq - MEDIAN_MARGIN_Q : 0u;
            hi_b = hq + MEDIAN_MARGIN_Q;
        }
        const int m1 = W->cand[j];
        // Where is element m relative to the median, given the fixed-point
        // weight before it (qb) and through it (qi)?  0: m is the median; +1:
        // the median comes after m, -1: before m (decided beyond the margin);
        // 2: undecided.  Exact integer sums: the answer is warp-uniform.
        // (qb < half - margin  <=>  qb + margin < half, for half >= margin;
        // lo_b = 0 otherwise, where nothing is decided below.)
        auto verdict = [&](unsigned qb, unsigned qi) {
            if ((qb < lo_b) & (qi > hi_b)) return 0;
            if (qi < lo_b) return 1;
            if (qb > hi_b) return -1;
            return 2;
        };
        // first candidate (the hit path: ~83% of config-2 steps decide here)
        t_new = shfl_t(loc, m1);
        const bool below1 = (loc < t_new) | ((loc == t_new) & (lane < m1));
        const unsigned qb1 = __reduce_add_sync(FULLMASK, below1 ? q : 0u);
        const unsigned qi1 = LAD_WARP_QI_SHFL ? qb1 + __shfl_sync(FULLMASK, q, m1)
                                              : __reduce_add_sync(FULLMASK, (below1 | (lane == m1)) ? q : 0u);
        hit = (qb1 < lo_b) & (qi1 > hi_b);
        if (!hit) {
            const int v1 = verdict(qb1, qi1);
            // Walk from m1 towards the median through its neighbours in the
            // stable (location, index) order: after a miss the median has
            // usually moved by one element (config 2: 71% of first-candidate
            // misses; the walk also subsumes an earlier test of the median
            // before last: same-box A/B +1.6% without it).  The neighbour nb
            // of the current element is the min/max (location, index) key on
            // its side (two REDUX minima), and since nb is adjacent in the
            // order its fixed-point sums follow exactly from the current ones:
            // walking up, qb(nb) = qi(cur) and qi(nb) = qi(cur) + q(nb);
            // walking down, qi(nb) = qb(cur) and qb(nb) = qb(cur) - q(nb).
            // The walk ends at the median, at a margin case or at the end of
            // the order (<= 31 hops), and a hop's candidate is accepted by the
            // same verdict as the first's, so the walk changes the cost of a
            // step, never its result.
            if (v1 == 1 || v1 == -1) {
                const OrderKey<T> key(loc);
                const bool up = v1 > 0;
                bool side = up ? !(below1 | (lane == m1)) : below1;
                unsigned qb = qb1, qi = qi1;
#pragma unroll 1
                for (int hop = 0; hop < 31; ++hop) {
                    const int nb = key.nearest(side, up);
                    if (nb < 0) break;
                    const unsigned qn = __shfl_sync(FULLMASK, q, nb);
                    if (up) {
                        qb = qi;
                        qi += qn;
                    } else {
                        qi = qb;
                        qb -= qn;
                    }
                    const int vn = verdict(qb, qi);
                    if (vn == 0) {
                        hit = true;
                        t_new = shfl_t(loc, nb);
                        W->cand[j] = nb;  // identical value from every lane
                        break;
                    }
                    if (vn != v1) break;  // undecided
                    side = side & (lane != nb);
                }
            }
        }
    }
    if (!hit) {
        if constexpr (PMAX <= 5)
            t_new = median_by_order_call<PMAX, CNTC, T>(W, lane, inv_mask, j, cacheable, cnt_rt, loc, w);
        else
            t_new = median_by_order<PMAX, CNTC, T>(W, lane, inv_mask, j, cacheable, cnt_rt, loc, w);
    }
    if (fabs(dsub(t_new, bj)) <= dmul(T(1e-14), dadd(T(1), fabs(bj)))) return;  // ccd.py:172
    T constant = dmul(lam, dsub(sum_abs_b, fabs(bj)));
    if (have_zero) constant = dadd(constant, zsum);
    // v_new = constant + |t - loc| @ weights in OpenBLAS ddot's order: n&-16
    // products folded by the SkylakeX lane tree (shuffles), then the FMA tail.
    // Lanes >= cnt (pads) never enter the sum: the lane tree reads lanes 0..15
    // only when cnt >= 16 (lanes 0..31 when cnt = 32) and the tail reads
    // elements < cnt, so their (a, w) need no zeroing.
    const T a = fabs(dsub(t_new, loc));
    const T wv = w;
    const int n1 = cnt & -16;
    const T pr = dmul(a, wv);
    // The four 256-bit lane sums S_0..S_3 come from shuffles into lanes 0..3
    // and go through shared memory, where every lane folds (S0 + S2) + (S1 + S3)
    // itself (one store/load instead of three dependent shuffle rounds).
    T *const sl = reinterpret_cast<T *>(W->sl);
    if constexpr (LAD_WARP_DDOT_SMEM) {
        // products staged so that lane l < 4 finds its partial sum's terms
        // contiguous: n1 = 16: p_{l + 4k} at 4 l + k; n1 = 32: p_{8k + l + 4h} at 8 l + 2 k + h
        if (n1 == 16) {
            if (lane < 16) W->pp[(lane & 3) * 4 + (lane >> 2)] = pr;
        } else if (n1 == 32) {
            W->pp[(lane & 3) * 8 + (lane >> 3) * 2 + ((lane >> 2) & 1)] = pr;
        }
        W->aw[lane] = {a, wv};  // FMA tail operands as (a, w) pairs
        __syncwarp();
        if (lane < 4) {
            using T2 = typename vec2_of<T>::type;
            if (n1 == 16) {
                const T2 *pl = reinterpret_cast<const T2 *>(W->pp) + 2 * lane;
                const T2 u = pl[0], v = pl[1];
                sl[lane] = dadd(dadd(dadd(u.x, u.y), v.x), v.y);
            } else if (n1 == 32) {
                const T2 *pl = reinterpret_cast<const T2 *>(W->pp) + 4 * lane;
                const T2 a0 = pl[0], a1 = pl[1], a2 = pl[2], a3 = pl[3];
                sl[lane] = dadd(dadd(dadd(dadd(a0.x, a0.y), dadd(a1.x, a1.y)), dadd(a2.x, a2.y)), dadd(a3.x, a3.y));
            }
        }
    } else if (n1 == 16) {
        const T q4 = shfl_down_t(pr, 4), q8 = shfl_down_t(pr, 8), q12 = shfl_down_t(pr, 12);
        const T S = dadd(dadd(dadd(pr, q4), q8), q12);
        if (lane < 4) sl[lane] = S;
    } else if (n1 == 32) {
        const T A2 = dadd(pr, shfl_down_t(pr, 4));
        const T a8 = shfl_down_t(A2, 8), a16 = shfl_down_t(A2, 16), a24 = shfl_down_t(A2, 24);
        const T S = dadd(dadd(dadd(A2, a8), a16), a24);
        if (lane < 4) sl[lane] = S;
    }
    if constexpr (!LAD_WARP_DDOT_SMEM) {
        // FMA tail operands as (t - loc_i, x_ij) pairs, signed: the tail's DFMA takes |.| as operand
        // modifiers (exact), so no separate abs instructions
        if constexpr (LAD_WARP_RAW_AW) W->aw[lane] = {dsub(t_new, loc), (padx_v<PMAX, T> && cacheable) ? xij : wv};
        else W->aw[lane] = {a, wv};
    }
    __syncwarp();
    T dot = T(0);
    if (n1 > 0) {
        const auto s01 = W->sl[0], s23 = W->sl[1];
        dot = dadd(dadd(s01.x, s23.x), dadd(s01.y, s23.y));
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {  // FMA tail in index order, length cnt - n1 < 16
        if (n1 + t < cnt) {
            const auto q = W->aw[n1 + t];
            dot = LAD_WARP_RAW_AW ? dfma(fabs(q.x), fabs(q.y), dot) : dfma(q.x, q.y, dot);
        }
    }
    __syncwarp();
    const T v_new = dadd(constant, dot);
    if (v_new < f_cur) {  // strict accept (ccd.py:187-191)
        const T delta = dsub(t_new, bj);
        r = row ? dsub(r, dmul(xij, delta)) : r;
        sum_abs_b = dadd(sum_abs_b, dsub(fabs(t_new), fabs(bj)));
        f_cur = v_new;
        W->B[j] = t_new;  // every lane stores the same value: no cross-lane hazard
    }
}

template <typename T>
struct StepState {
    T r, f_cur, sum_abs_b;
};

// A step on a column with zero entries (compacted breakpoints).  Out of line:
// such columns are rare, and a second inlined copy of the median/update code
// would bloat the hot step body.  State goes in and out by value (registers).
template <int PMAX, typename T>
__device__ __noinline__ StepState<T> sparse_step(WarpShared<PMAX, T> *W, int lane, uint32_t inv_mask, int n, int j,
                                                 T lam, bool row, T xij, T bj, StepState<T> st)
{
    T loc, w, zsum;
    int cnt;
    sparse_column<PMAX, T>(W, lane, n, st.r, xij, bj, lam, loc, w, cnt, zsum);
    median_update<PMAX, 0, T>(W, lane, inv_mask, j, lam, false, cnt, loc, w, zsum, true, row, xij, bj, st.r, st.f_cur,
                              st.sum_abs_b);
    return st;
}

// One exact coordinate step on axis j (ccd.py:160-193), all lanes in lock-step.
// NC > 0: compile-time row count (config shapes); NC == 0: runtime n_rt.
template <int PMAX, int NC, typename T>
__device__ __forceinline__ void warp_step(WarpShared<PMAX, T> *W, int lane, uint32_t inv_mask, const T *xrow,
                                          const T *yrow, int n_rt, int j, T lam, bool col_sparse, T &r, T &f_cur,
                                          T &sum_abs_b)
{
    const T INF = inf_of<T>();
    const int n = NC > 0 ? NC : n_rt;
    const bool row = lane < n;
    const T xij = xrow[j];  // lanes >= n read a stale in-bounds slot, never used
    const T bj = W->B[j];
    if (!col_sparse) {
        // np.divide then += b[j] (ccd.py:165-166).  Pad lanes divide 1/1 (their
        // result is discarded; it keeps them off the division's slow path).
        const T rr = (padx_v<PMAX, T> || row) ? r : T(1), xx = (padx_v<PMAX, T> || row) ? xij : T(1);
        T q;
        if constexpr (fast_div_v<PMAX, T>) {
            q = div_by_rcp(rr, xx, yrow[j]);  // y = 1 on pad lanes
        } else {
            q = LAD_WARP_ZDIV ? ddiv_zero_fast(rr, xx) : ddiv(rr, xx);
        }
        const T loc = row ? dadd(q, bj) : (lane == n ? T(0) : INF);
        const T w = (padx_v<PMAX, T> || row) ? fabs(xij) : (lane == n ? lam : T(0));
        median_update<PMAX, (NC > 0 ? NC + 1 : 0), T>(W, lane, inv_mask, j, lam, true, n + 1, loc, w, T(0), false,
                                                      row, xij, bj, r, f_cur, sum_abs_b);
    } else if constexpr (PMAX <= 5) {
        const StepState<T> st = sparse_step<PMAX, T>(W, lane, inv_mask, n, j, lam, row, xij, bj, {r, f_cur, sum_abs_b});
        r = st.r;
        f_cur = st.f_cur;
        sum_abs_b = st.sum_abs_b;
    } else {  // p = 8: inline (measured faster for the config-4 shape)
        T loc, w, zsum;
        int cnt;
        sparse_column<PMAX, T>(W, lane, n, r, xij, bj, lam, loc, w, cnt, zsum);
        median_update<PMAX, 0, T>(W, lane, inv_mask, j, lam, false, cnt, loc, w, zsum, true, row, xij, bj, r, f_cur,
                                  sum_abs_b);
    }
}

template <int PMAX, typename T>
__device__ __forceinline__ T warp_objective(WarpShared<PMAX, T> *W, int lane, int n, int p, int xs, T lam)
{
    T v = T(0);
    if (lane < n) {
        T g = gemv_row(p, lane, n, [&](int q) { return W->X[lane * xs + q]; }, [&](int q) { return W->B[q]; });
        v = fabs(dsub(W->Y[lane], g));
    }
    T rs = warp_np_sum(v, n, lane);
    T bs = np_sum(p, [&](int q) { return fabs(W->B[q]); });
    return dadd(rs, dmul(lam, bs));
}

// ccd_descend (ccd.py:126-206) for the descent request in C, all lanes.
// The descent and the controller are inlined into the kernel (binary64: +1.6%
// and +2.1% for config 2).  The binary32 p = 8 kernel spills ~690 B per thread
// at its 64-register cap when inlined and is still fastest that way (config 4
// fp32, same box: 157 k inlined, 149 k out of line (no spills), 148 k / 146 k
// with 7 warps at 72 registers (LAD_WARP_F32_WIDE) inlined / out of line).
#ifndef LAD_WARP_INLINE_DESC
#define LAD_WARP_INLINE_DESC 1
#endif
#ifndef LAD_WARP_F32_INLINE
#define LAD_WARP_F32_INLINE 1
#endif
template <typename T>
constexpr bool warp_inline_v = sizeof(T) == 8 || LAD_WARP_F32_INLINE;

template <int PMAX, int NC, typename T>
__device__ __forceinline__ void warp_descent_body(WarpShared<PMAX, T> *W, Ctl<PMAX> &C, int lane, uint32_t inv_mask, int n_rt,
                                          int p_rt)
{
    const int n = NC > 0 ? NC : n_rt;
    const int p = NC > 0 ? PMAX : p_rt;
    const int xs = p | 1;  // row stride of W->X (xs_v)
    const int frozen = C.req_frozen;
    const double tol = C.req_tol;
    const int max_sweeps = C.req_sweeps;
    const T lam = T(C.lam);
    const uint32_t sparse = C.sparse_mask;
    if (lane < p) W->B[lane] = T(C.req_start[lane]);
    __syncwarp();
    T r = padx_v<PMAX, T> ? T(1) : T(0);  // pad lanes (padx: a safe dividend that never changes)
    if (lane < n) {
        T g = gemv_row(p, lane, n, [&](int q) { return W->X[lane * xs + q]; }, [&](int q) { return W->B[q]; });
        r = dsub(W->Y[lane], g);
    }
    const T *xrow = W->X + lane * xs;
    const T *yrow = fast_div_v<PMAX, T> ? W->RX + lane * xs : nullptr;
    const T sb = np_sum(p, [&](int q) { return fabs(W->B[q]); });
    T f_cur = dadd(warp_np_sum(fabs(r), n, lane), dmul(lam, sb));
    T f_sweep_start = f_cur, sum_abs_b = sb;
    int sweeps = 1, steps = 0, conv = 0;
    const int j0 = (frozen == 0) ? 1 : 0;
    int j = j0;
    if (j >= p) {
        conv = 1;
    } else if (LAD_WARP_DENSE_LOOP && NC > 0 && sparse == 0u) {
        uint32_t axis_list = 0u;
        int nfree = 0;
#pragma unroll
        for (int jj = PMAX - 1; jj >= 0; --jj)
            if (jj != frozen) {
                axis_list = (axis_list << 4) | (uint32_t)(jj + 1);
                ++nfree;
            }
        // Every column dense (the common case): no per-step sparse test, and with
        // LAD_WARP_UNROLL the sweep over the PMAX axes is unrolled (compile-time
        // axis offsets, no axis bookkeeping); the frozen axis is skipped in place.
        for (;;) {
            if constexpr (LAD_WARP_UNROLL) {
#pragma unroll
                for (int jj = 0; jj < PMAX; ++jj) {
                    if (jj == frozen) continue;
                    warp_step<PMAX, NC, T>(W, lane, inv_mask, xrow, yrow, n, jj, lam, false, r, f_cur, sum_abs_b);
                    ++steps;
                }
            } else if constexpr (LAD_WARP_AXIS_LIST) {
                // the free axes in sweep order, 4 bits each (axis + 1), consumed low nibble first
#pragma unroll 1
                for (uint32_t lst = axis_list; lst != 0u; lst >>= 4) {
                    const int jj = (int)(lst & 15u) - 1;
                    warp_step<PMAX, NC, T>(W, lane, inv_mask, xrow, yrow, n, jj, lam, false, r, f_cur, sum_abs_b);
                }
                steps += nfree;
            } else {
#pragma unroll 1
                for (int jj = j0; jj < PMAX; jj += 1 + (jj + 1 == frozen)) {
                    warp_step<PMAX, NC, T>(W, lane, inv_mask, xrow, yrow, n, jj, lam, false, r, f_cur, sum_abs_b);
                    ++steps;
                }
            }
            if (dsub(f_sweep_start, f_cur) < tol) {  // gain in T, compared in binary64
                conv = 1;
                break;
            }
            if (sweeps >= max_sweeps) break;
            ++sweeps;
            f_sweep_start = f_cur;
            sum_abs_b = np_sum(p, [&](int q) { return fabs(W->B[q]); });
        }
    } else {
        for (;;) {
            warp_step<PMAX, NC, T>(W, lane, inv_mask, xrow, yrow, n, j, lam, (sparse >> j) & 1u, r, f_cur,
                                   sum_abs_b);
            ++steps;
            int jn = j + 1;
            jn += (jn == frozen);
            if (jn < p) {
                j = jn;
                continue;
            }
            if (dsub(f_sweep_start, f_cur) < tol) {  // gain in T, compared in binary64
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
    __syncwarp();
    const T obj = warp_objective<PMAX, T>(W, lane, n, p, xs, lam);
    const int D = C.D;
    const long long S = C.S;
    __syncwarp();
    if (lane < p) C.res_beta[lane] = (double)W->B[lane];
    if (lane == 0) {
        C.res_obj = (double)obj;
        C.res_conv = conv;
        C.res_sweeps = sweeps;
        C.res_steps = steps;
        C.D = D + 1;
        C.S = S + steps;
    }
    __syncwarp();
}

template <int PMAX, int NC, typename T>
__device__ __noinline__ void warp_descent(WarpShared<PMAX, T> *W, Ctl<PMAX> &C, int lane, uint32_t inv_mask, int n_rt,
                                          int p_rt)
{
    warp_descent_body<PMAX, NC, T>(W, C, lane, inv_mask, n_rt, p_rt);
}

// PMAX: beta capacity; NC > 0 specialises the row count (and p == PMAX).
template <int PMAX, int NC, typename T>
__global__ void __launch_bounds__(32 * warps_per_block<PMAX, T>, warp_min_blocks<PMAX, T>) locus_warp_kernel(LocusArgs A)
{
    extern __shared__ __align__(16) unsigned char warp_smem[];  // warps_per_block x WarpShared
    WarpShared<PMAX, T> *WS = reinterpret_cast<WarpShared<PMAX, T> *>(warp_smem);
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpShared<PMAX, T> *W = &WS[wib];
    const int n = NC > 0 ? NC : A.n, p = NC > 0 ? PMAX : A.p;
    const int slot = blockIdx.x * warps_per_block<PMAX, T> + wib;
    WarpAccess<PMAX, T> acc{n, p, lane, W, p | 1};
    const uint32_t inv_mask = bitonic_inv_mask(lane);
    Ctl<PMAX> &C = W->C;
    if (lane < PMAX) W->cand[lane] = 0;
    if (lane == 0) {
        C.pc = PC_FETCH;
        W->seen = (A.seen != nullptr && p > 2) ? A.seen + (size_t)slot * A.seen_cap * (1 + PMAX) : nullptr;
    }
    __syncwarp();
    for (;;) {
        // inlined: the controller reads LocusArgs straight from the kernel's parameter
        // (constant) bank; out of line it reads every field from a per-lane stack copy
        int act = (LAD_WARP_INLINE_CTL && warp_inline_v<T>) ? controller_body<PMAX>(C, A, acc, slot)
                                                            : controller<PMAX>(C, A, acc, slot);
        __syncwarp();
        if (act == ACT_EXIT) break;
        if constexpr (LAD_WARP_INLINE_DESC && warp_inline_v<T>)
            warp_descent_body<PMAX, NC, T>(W, C, lane, inv_mask, n, p);
        else
            warp_descent<PMAX, NC, T>(W, C, lane, inv_mask, n, p);
    }
}

}  // namespace lad
