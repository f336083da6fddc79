// lad_locus_block.cuh -- block-per-problem locus kernel for 47 <= n <= 1023 rows (binary64).
//
// 32 * ceil((n + 1) / 32) threads per problem (at most 256), persistent grid.
// Thread t owns elements t, t + T, t + 2T, t + 3T of a step (rows, then the
// lambda breakpoint).
// Every warp runs the shared controller (lad_locus.cuh) on its own copy of
// the state: the inputs it sees are identical in every warp, so the copies
// stay identical, and sync() is __syncthreads().  Per coordinate step:
//   * breakpoints r_i / x_ij + b_j (columns with zeros: compacted by a block
//     scan, ccd.py:94-110);
//   * weighted median: the axis' previous median element is verified with two
//     exact fixed-point block sums (as in the warp kernel); otherwise a
//     shared-memory bitonic sort of (location, index), a fixed-point inclusive
//     scan decided with a 2^14-unit margin, and -- inside the margin -- numpy's
//     sequential FP64 cumsum on one thread;
//   * v_new in OpenBLAS ddot's order for any length (lane c of warp 0 runs
//     accumulator chain c over the 32-element blocks, then the 512->256 fold,
//     the 16-element remainder, the lane tree and the FMA tail);
//   * per-descent sums (np.abs(r).sum(), including numpy's pairwise recursion
//     above 128 terms) on one thread.
#pragma once
#include "lad_locus.cuh"
#include "lad_locus_warp.cuh"

namespace lad {

constexpr int BLK_THREADS = 256, BLK_WARPS = 8, BLK_NMAX = 1023, BLK_EPT = 4;  // elements per thread

#ifndef LAD_BLK_WALK_HOPS
#define LAD_BLK_WALK_HOPS 16
#endif
constexpr int BLK_WALK_HOPS = LAD_BLK_WALK_HOPS;

template <int PMAX>
struct BlockHead {
    Ctl<PMAX> C[BLK_WARPS];  // one controller state per warp (identical)
    double B[PMAX];          // beta of the running descent
    double scale[PMAX];      // fixed-point scale per axis (2^30 / total weight)
    unsigned halfq[PMAX];    // (sum of fixed-point weights) / 2 per axis
    int cand[PMAX];          // previous median element per axis
    unsigned long long item;
    double redd[BLK_WARPS];
    unsigned redu[2][BLK_WARPS];
    unsigned long long wkey[BLK_WARPS];  // median walk: per-warp nearest (key, index)
    unsigned widx[BLK_WARPS];
    double bcd[4];
    int bci[4];
    unsigned mask;
};

struct BlockLayout {
    int P2;  // power of two >= n + 1 (sort width)
    size_t off_X, off_Y, off_loc, off_w, off_sk, off_si, off_aw, off_tmp, off_pos, total;
};

template <int PMAX>
__host__ __device__ inline BlockLayout block_layout(int n, int p)
{
    BlockLayout L;
    int P2 = 1;
    while (P2 < n + 1) P2 <<= 1;
    L.P2 = P2;
    size_t o = (sizeof(BlockHead<PMAX>) + 15) & ~(size_t)15;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o = (o + bytes + 15) & ~(size_t)15;
        return r;
    };
    L.off_X = take((size_t)n * (p | 1) * 8);  // row stride p | 1: thread i's row stays off its neighbours' banks
    L.off_Y = take((size_t)n * 8);
    L.off_loc = take((size_t)P2 * 8);
    L.off_w = take((size_t)(n + 1) * 8);
    L.off_sk = take((size_t)P2 * 8);
    L.off_si = take((size_t)P2 * 4);
    L.off_aw = take((size_t)(n + 1) * 16);
    L.off_tmp = take((size_t)(n + 1) * 8);
    L.off_pos = take((size_t)(n + 1) * 4);
    L.total = o;
    return L;
}

template <int PMAX>
struct BlockMem {
    BlockHead<PMAX> *H;
    double *X, *Y, *loc, *w, *sk, *tmp;
    int *si, *pos;
    double2 *aw;
    int P2;
    int xs;  // row stride of X in doubles (p | 1)
};

__device__ __forceinline__ unsigned block_sum_u2(unsigned a, unsigned b, unsigned (*red)[BLK_WARPS], unsigned &sb)
{
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    a = __reduce_add_sync(FULLMASK, a);
    b = __reduce_add_sync(FULLMASK, b);
    if (lane == 0) {
        red[0][wp] = a;
        red[1][wp] = b;
    }
    __syncthreads();
    unsigned sa = 0;
    sb = 0;
    const int nw = (int)(blockDim.x >> 5);
    for (int k = 0; k < nw; ++k) {
        sa += red[0][k];
        sb += red[1][k];
    }
    __syncthreads();
    return sa;
}

// block sum of doubles in a fixed order (identical in every thread; any order is fine for its uses)
__device__ __forceinline__ double block_sum_d(double v, double *red)
{
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULLMASK, v, off);
    if (lane == 0) red[wp] = v;
    __syncthreads();
    double s = 0.0;
    const int nw = (int)(blockDim.x >> 5);
    for (int k = 0; k < nw; ++k) s += red[k];
    __syncthreads();
    return s;
}

// Access policy of the block kernel (see lad_locus.cuh controller()).
template <int PMAX>
struct BlockAccess {
    static constexpr bool kYield = false;  // controller states jump directly (lad_locus.cuh, ACT_YIELD)
    int n, p, lane;
    BlockMem<PMAX> M;
    __device__ __forceinline__ bool leader() const { return threadIdx.x == 0; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    template <int PM>
    __device__ __forceinline__ double *seen_base(const LocusArgs &A, int slot) const
    {
        return (A.seen != nullptr && p > 2) ? A.seen + (size_t)slot * A.seen_cap * (1 + PM) : nullptr;
    }
    // controller vectors: every thread writes the same shared values (lanes), the
    // leader alone writes global outputs (lanes_out)
    template <class F>
    __device__ __forceinline__ void lanes(int cnt, F f) const
    {
        for (int k = 0; k < cnt; ++k) f(k);
    }
    template <class F>
    __device__ __forceinline__ void lanes_out(int cnt, F f) const
    {
        if (threadIdx.x == 0)
            for (int k = 0; k < cnt; ++k) f(k);
    }
    template <int PM>
    __device__ __forceinline__ void copy_point(Point<PM> &d, const Point<PM> &s) const
    {
        d = s;
    }
    __device__ __forceinline__ bool last_of(unsigned *ctr, unsigned of) const
    {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            M.H->bci[3] = (int)(atomicAdd(ctr, 1u) == of - 1u);
            __threadfence();
        }
        __syncthreads();
        const bool last = M.H->bci[3] != 0;
        __syncthreads();
        return last;
    }
    __device__ int fetch(Ctl<PMAX> &C, const LocusArgs &A) const
    {
        BlockHead<PMAX> *H = M.H;
        const int tid = threadIdx.x;
        const int div = A.axis_mode == AXIS_SEARCH ? p : 1;
        __syncthreads();
        if (tid == 0) {
            H->item = atomicAdd(A.counter, 1ULL);
            H->mask = 0;
        }
        __syncthreads();
        const unsigned long long item = H->item;
        if ((int64_t)item >= A.B * div) return -1;
        const unsigned long long pr = item / div;
        const int64_t src = A.data_index ? A.data_index[pr] : (int64_t)pr;
        if (src < 0 || src >= A.Bd) {
            __syncwarp();
            C.prob = (int64_t)pr;
            C.arank = (int)(item % div);
            __syncwarp();
            if (tid == 0) write_invalid<PMAX>(A, (int64_t)pr, p);
            return 0;
        }
        const double *xg = A.X + (size_t)src * n * p, *yg = A.Y + (size_t)src * n;
        bool ok = true;
        unsigned mask = 0;
        for (int e = tid; e < n * p; e += (int)blockDim.x) {
            const double v = xg[e];
            const int i = e / p, j = e - i * p;
            M.X[i * M.xs + j] = v;
            ok = ok && isfinite(v);
            if (v == 0.0) mask |= 1u << j;
        }
        for (int i = tid; i < n; i += (int)blockDim.x) {
            const double v = yg[i];
            M.Y[i] = v;
            ok = ok && isfinite(v);
        }
        mask = __reduce_or_sync(FULLMASK, mask);
        if ((tid & 31) == 0 && mask) atomicOr(&H->mask, mask);
        const double lraw = A.lam[pr];
        ok = __syncthreads_and(ok) && isfinite(lraw) && lraw >= 0.0;
        const double lam_eff = lraw > A.prm.lambda_floor ? lraw : A.prm.lambda_floor;
        // fixed-point weights per axis for the median test (any summation order will do)
        for (int j = 0; j < p; ++j) {
            double s = 0.0;
            for (int e = tid; e <= n; e += (int)blockDim.x) s += e < n ? fabs(M.X[e * M.xs + j]) : lam_eff;
            const double tot = block_sum_d(s, H->redd);
            const double scale = 1073741824.0 / (tot * (1.0 + 1e-9));
            const bool good = tot > 0.0 && tot < 1e300 && scale < 1e300;  // a finite scale keeps every weight below 2^30
            unsigned qs = 0;
            for (int e = tid; e <= n; e += (int)blockDim.x)
                qs += good ? __double2uint_rz((e < n ? fabs(M.X[e * M.xs + j]) : lam_eff) * scale) : 0u;
            unsigned dummy;
            const unsigned sq = block_sum_u2(qs, 0u, H->redu, dummy);
            if (tid == 0) {
                H->scale[j] = good ? scale : 0.0;
                H->halfq[j] = sq / 2u;
            }
        }
        __syncthreads();
        C.prob = (int64_t)pr;
        C.arank = (int)(item % div);
        C.lam = lam_eff;
        C.sparse_mask = H->mask;
        __syncwarp();
        if (!ok) {
            if (tid == 0) write_invalid<PMAX>(A, (int64_t)pr, p);
            return 0;
        }
        return 1;
    }
    __device__ double col_abs_sum(int j) const
    {
        if (p == 1) return np_sum_rec(0, n, [&](int i) { return fabs(M.X[i]); });  // contiguous column: pairwise
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = dadd(s, fabs(M.X[i * M.xs + j]));
        return s;
    }
    __device__ double y_absmax(const double *) const
    {
        double ymax = 0.0;
        for (int i = 0; i < n; ++i) {
            const double a = fabs(M.Y[i]);
            if (i == 0 || a > ymax) ymax = a;
        }
        return ymax;
    }
    __device__ int nearest(const double *seen, int lim, double t) const
    {
        __syncwarp();
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        int bk = 0x7fffffff;
        for (int k = lane; k < lim; k += 32) {
            const double dd = fabs(dsub(seen[k], t));
            if (dd < bd) {
                bd = dd;
                bk = k;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double od = __shfl_xor_sync(FULLMASK, bd, off);
            const int ok = __shfl_xor_sync(FULLMASK, bk, off);
            if (od < bd || (od == bd && ok < bk)) {
                bd = od;
                bk = ok;
            }
        }
        return bk == 0x7fffffff ? -1 : bk;
    }
};


// OpenBLAS ddot (SkylakeX, any length) of the cnt (a, w) pairs in aw, by warp 0;
// the result is returned in every lane of warp 0.
__device__ __forceinline__ double block_blas_ddot(const double2 *aw, int cnt, int lane)
{
    const int n1 = cnt & -16, n32 = n1 & -32;
    double acc = 0.0;  // chain c = lane: 512-bit accumulator k = c / 8, lane l = c % 8
    for (int it = 0; it < n32; it += 32) {
        const double2 q = aw[it + lane];
        acc = dfma(q.x, q.y, acc);
    }
    double a4 = dadd(acc, __shfl_down_sync(FULLMASK, acc, 4));  // 512 -> 256: valid where lane % 8 < 4
    const int k = lane >> 3, l = lane & 7;
    if (n1 > n32 && l < 4) {  // 16-element remainder: one 4-element chunk per 256-bit accumulator
        const double2 q = aw[n32 + 4 * k + l];
        a4 = dfma(q.x, q.y, a4);
    }
    const double a1 = __shfl_sync(FULLMASK, a4, (lane & 3) + 8), a2 = __shfl_sync(FULLMASK, a4, (lane & 3) + 16),
                 a3 = __shfl_sync(FULLMASK, a4, (lane & 3) + 24);
    const double S = dadd(dadd(dadd(a4, a1), a2), a3);  // valid in lanes 0..3
    const double S1 = __shfl_sync(FULLMASK, S, 1), S2 = __shfl_sync(FULLMASK, S, 2), S3 = __shfl_sync(FULLMASK, S, 3);
    double dot = n1 > 0 ? dadd(dadd(S, S2), dadd(S1, S3)) : 0.0;
    dot = __shfl_sync(FULLMASK, dot, 0);
    for (int e = n1; e < cnt; ++e) dot = dfma(aw[e].x, aw[e].y, dot);  // FMA tail in order (uniform)
    return dot;
}

// Ascending bitonic sort of (key, idx) over P2 slots in shared memory (lexicographic).
__device__ __forceinline__ void block_bitonic(double *key, int *idx, int P2)
{
    for (int k = 2; k <= P2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P2; i += (int)blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const double ka = key[i], kb = key[ixj];
                    const int ia = idx[i], ib = idx[ixj];
                    const bool a_gt_b = (ka > kb) | ((ka == kb) & (ia > ib));
                    const bool up = (i & k) == 0;
                    if (up == a_gt_b) {
                        key[i] = kb;
                        key[ixj] = ka;
                        idx[i] = ib;
                        idx[ixj] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// One exact coordinate step on axis j (ccd.py:160-193), block-wide.
template <int PMAX>
__device__ void block_step(const BlockMem<PMAX> &M, int n, int p, int j, double lam, bool col_sparse,
                           double (&r)[BLK_EPT], double &f_cur, double &sum_abs_b)
{
    BlockHead<PMAX> *H = M.H;
    const int tid = threadIdx.x, lane = tid & 31;
    const double bj = H->B[j];
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    // breakpoints (element order: rows with x_ij != 0 in row order, then lambda)
    int cnt;
    double zsum = 0.0;
    if (!col_sparse) {
#pragma unroll
        for (int q = 0; q < BLK_EPT; ++q) {
            const int e = tid + q * (int)blockDim.x;
            if (e < n) {
                const double x = M.X[e * M.xs + j];
                M.loc[e] = dadd(ddiv_zero_fast(r[q], x), bj);
                M.w[e] = fabs(x);
            } else if (e == n) {
                M.loc[e] = 0.0;
                M.w[e] = lam;
            }
        }
        cnt = n + 1;
    } else {  // compact the nonzero rows (block scan of flags); zero rows feed the constant
        int flags[BLK_EPT], nnz = 0;
#pragma unroll
        for (int q = 0; q < BLK_EPT; ++q) {
            const int i = tid * BLK_EPT + q;  // contiguous rows per thread for the scan
            flags[q] = (i < n && M.X[i * M.xs + j] != 0.0) ? 1 : 0;
            nnz += flags[q];
        }
        int incl = nnz;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(FULLMASK, incl, off);
            if (lane >= off) incl += t;
        }
        __syncthreads();
        if (lane == 31) H->redu[0][tid >> 5] = (unsigned)incl;
        __syncthreads();
        int base = 0;
        for (int k = 0; k < (tid >> 5); ++k) base += (int)H->redu[0][k];
        int total = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) total += (int)H->redu[0][k];
        int pnz = base + incl - nnz;
        // rows are spread over threads as i = tid * EPT + q here, but r[q] belongs to row tid + q * 256:
        // stage the residuals in tmp first
        __syncthreads();
#pragma unroll
        for (int q = 0; q < BLK_EPT; ++q) {
            const int i = tid + q * (int)blockDim.x;
            if (i < n) M.tmp[i] = r[q];
        }
        __syncthreads();
        int pz = (tid * BLK_EPT) - (base + incl - nnz);  // zero rows before this thread's first row
#pragma unroll
        for (int q = 0; q < BLK_EPT; ++q) {
            const int i = tid * BLK_EPT + q;
            if (i < n) {
                const double x = M.X[i * M.xs + j];
                if (flags[q]) {
                    M.loc[pnz] = ddiv(dadd(M.tmp[i], dmul(x, bj)), x);
                    M.w[pnz] = fabs(x);
                    ++pnz;
                } else {
                    M.pos[pz++] = i;  // zero rows in order
                }
            }
        }
        if (tid == 0) {
            M.loc[total] = 0.0;
            M.w[total] = lam;
        }
        __syncthreads();
        if (tid == 0) H->bcd[0] = np_sum_rec(0, n - total, [&](int z) { return fabs(M.tmp[M.pos[z]]); });
        __syncthreads();
        zsum = H->bcd[0];
        cnt = total + 1;
    }
    for (int e = cnt + tid; e < M.P2; e += (int)blockDim.x) M.loc[e] = INF;
    __syncthreads();
    // weighted median (ccd.py:81-91)
    const double scale = H->scale[j];
    const unsigned hq = H->halfq[j];
    double t_new;
    bool hit = false;
    if (!col_sparse && scale > 0.0) {
        // Fixed-point weight before element m (qb) and through it (qi): exact
        // block sums, so every decision below is block-uniform.
        auto sums = [&](int m, double lm, unsigned &sqb, unsigned &sqi) {
            unsigned qb = 0, qi = 0;
#pragma unroll
            for (int q = 0; q < BLK_EPT; ++q) {
                const int e = tid + q * (int)blockDim.x;
                if (e < cnt) {
                    const double le = M.loc[e];
                    const unsigned qe = __double2uint_rz(M.w[e] * scale);
                    const bool below = (le < lm) | ((le == lm) & (e < m));
                    qb += below ? qe : 0u;
                    qi += (below | (e == m)) ? qe : 0u;
                }
            }
            sqb = block_sum_u2(qb, qi, H->redu, sqi);
        };
        // 0: the median; +1 / -1: the median comes after / before; 2: undecided
        auto verdict = [&](unsigned qb, unsigned qi) {
            if ((qb + MEDIAN_MARGIN_Q < hq) & (qi > hq + MEDIAN_MARGIN_Q)) return 0;
            if (qi + MEDIAN_MARGIN_Q < hq) return 1;
            if (qb > hq + MEDIAN_MARGIN_Q) return -1;
            return 2;
        };
        const int m1 = H->cand[j];
        const double l1 = M.loc[m1];
        unsigned qb, qi;
        sums(m1, l1, qb, qi);
        const int v1 = verdict(qb, qi);
        if (v1 == 0) {
            hit = true;
            t_new = l1;
        } else if (v1 != 2) {
            // Walk from the last median towards the new one through its
            // neighbours in the stable (location, index) order, as the warp
            // kernel does (lad_locus_warp.cuh): the neighbour is the block-wide
            // min (walking up) or max (down) of the (location key, index) pairs
            // on its side, and its fixed-point sums follow exactly from the
            // current element's.  Each thread keeps its elements' keys
            // (complemented when walking down, so both directions take minima).
            const bool up = v1 > 0;
            unsigned long long key[BLK_EPT];
            unsigned sidebits = 0;
#pragma unroll
            for (int q = 0; q < BLK_EPT; ++q) {
                const int e = tid + q * (int)blockDim.x;
                key[q] = ~0ull;
                if (e < cnt) {
                    const double le = M.loc[e];
                    const bool below = (le < l1) | ((le == l1) & (e < m1));
                    if (up ? !(below | (e == m1)) : below) sidebits |= 1u << q;
                    const long long b = __double_as_longlong(__dadd_rn(le, 0.0));
                    const unsigned long long k = (unsigned long long)b ^ (b < 0 ? ~0ull : (1ull << 63));
                    key[q] = up ? k : ~k;
                }
            }
            // at most BLK_WALK_HOPS hops, then the ordering path: with many
            // breakpoints the median can move far, and a long walk costs more
            // than one sort (n = 1000 without the cap: -7%; caps 8..64 measure
            // within 3% of each other: +17% at n = 40, +30% n = 100, +63% n = 256)
#pragma unroll 1
            for (int hop = 0; hop < BLK_WALK_HOPS; ++hop) {
                unsigned long long bk = ~0ull;
                unsigned bi = ~0u;
#pragma unroll
                for (int q = 0; q < BLK_EPT; ++q) {
                    const unsigned ie = up ? (unsigned)(tid + q * (int)blockDim.x) : ~(unsigned)(tid + q * (int)blockDim.x);
                    if (((sidebits >> q) & 1u) && (key[q] < bk || (key[q] == bk && ie < bi))) {
                        bk = key[q];
                        bi = ie;
                    }
                }
                const unsigned h = (unsigned)(bk >> 32), l = (unsigned)bk;
                const unsigned mh = __reduce_min_sync(FULLMASK, h);
                const unsigned ml = __reduce_min_sync(FULLMASK, h == mh ? l : ~0u);
                const unsigned mi = __reduce_min_sync(FULLMASK, (h == mh && l == ml) ? bi : ~0u);
                if (lane == 0) {
                    H->wkey[tid >> 5] = ((unsigned long long)mh << 32) | ml;
                    H->widx[tid >> 5] = mi;
                }
                __syncthreads();
                unsigned long long gk = ~0ull;
                unsigned gi = ~0u;
                for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
                    const unsigned long long wk = H->wkey[k];
                    const unsigned wi = H->widx[k];
                    if (wk < gk || (wk == gk && wi < gi)) {
                        gk = wk;
                        gi = wi;
                    }
                }
                __syncthreads();
                if (gi == ~0u && gk == ~0ull) break;  // nothing left on this side
                const int nb = up ? (int)gi : (int)~gi;
                const unsigned qn = __double2uint_rz(M.w[nb] * scale);
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
                    t_new = M.loc[nb];
                    if (tid == 0) H->cand[j] = nb;
                    break;
                }
                if (vn != v1) break;  // undecided
                if (nb % (int)blockDim.x == tid) sidebits &= ~(1u << (nb / (int)blockDim.x));
            }
        }
    }
    if (!hit) {
        for (int e = tid; e < M.P2; e += (int)blockDim.x) {
            M.sk[e] = M.loc[e];
            M.si[e] = e;
        }
        __syncthreads();
        block_bitonic(M.sk, M.si, M.P2);
        // k = first sorted position whose cumulative weight reaches half the total:
        // fixed-point counts, decided only when no cumulative sum lies within the margin
        unsigned cq[BLK_EPT];
        unsigned run = 0;
#pragma unroll
        for (int q = 0; q < BLK_EPT; ++q) {
            const int e = tid * BLK_EPT + q;
            run += (e < cnt && scale > 0.0) ? __double2uint_rz(M.w[M.si[e]] * scale) : 0u;
            cq[q] = run;
        }
        unsigned incl = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned t = __shfl_up_sync(FULLMASK, incl, off);
            if (lane >= off) incl += t;
        }
        if (lane == 31) H->redu[0][tid >> 5] = incl;
        __syncthreads();
        unsigned base = 0;
        for (int k = 0; k < (tid >> 5); ++k) base += H->redu[0][k];
        base += incl - run;
        int lo = 0, hi = 0;
#pragma unroll
        for (int q = 0; q < BLK_EPT; ++q) {
            const int e = tid * BLK_EPT + q;
            const unsigned c = base + cq[q];
            if (e < cnt) {
                lo += (c + MEDIAN_MARGIN_Q < hq) ? 1 : 0;
                hi += (c <= hq + MEDIAN_MARGIN_Q) ? 1 : 0;
            }
        }
        __syncthreads();
        unsigned slo2;
        const unsigned shi = block_sum_u2((unsigned)hi, (unsigned)lo, H->redu, slo2);
        int k;
        bool tie = false;
        if (scale > 0.0 && slo2 == shi) {
            k = (int)slo2;
        } else {  // exact: numpy's sequential cumsum in sorted order (ccd.py:84-91), one thread
            if (tid == 0) {
                double c = 0.0, total = 0.0;
                for (int e = 0; e < cnt; ++e) total = dadd(total, M.w[M.si[e]]);
                const double half = dmul(0.5, total);
                int kk = cnt;
                double ck = 0.0;
                for (int e = 0; e < cnt; ++e) {
                    c = dadd(c, M.w[M.si[e]]);
                    if (c >= half) {
                        kk = e;
                        ck = c;
                        break;
                    }
                }
                H->bci[1] = kk;
                H->bci[2] = (kk + 1 < cnt) && fabs(dsub(ck, half)) <= dmul(1e-12, total);
            }
            __syncthreads();
            k = H->bci[1];
            tie = H->bci[2] != 0;
            __syncthreads();
        }
        const int ks = k < cnt ? k : cnt - 1;
        t_new = tie ? dmul(0.5, dadd(M.sk[ks], M.sk[ks + 1])) : M.sk[ks];
        if (!col_sparse && tid == 0) H->cand[j] = M.si[ks];
    }
    __syncthreads();
    if (fabs(dsub(t_new, bj)) <= dmul(1e-14, dadd(1.0, fabs(bj)))) return;  // ccd.py:172
    double constant = dmul(lam, dsub(sum_abs_b, fabs(bj)));
    if (col_sparse) constant = dadd(constant, zsum);
    for (int e = tid; e < cnt; e += (int)blockDim.x) M.aw[e] = make_double2(fabs(dsub(t_new, M.loc[e])), M.w[e]);
    __syncthreads();
    if ((tid >> 5) == 0) {
        const double dot = block_blas_ddot(M.aw, cnt, lane);
        if (lane == 0) H->bcd[1] = dadd(constant, dot);
    }
    __syncthreads();
    const double v_new = H->bcd[1];
    if (v_new < f_cur) {  // strict accept (ccd.py:187-191)
        const double delta = dsub(t_new, bj);
#pragma unroll
        for (int q = 0; q < BLK_EPT; ++q) {
            const int i = tid + q * (int)blockDim.x;
            if (i < n) r[q] = dsub(r[q], dmul(M.X[i * M.xs + j], delta));
        }
        sum_abs_b = dadd(sum_abs_b, dsub(fabs(t_new), fabs(bj)));
        f_cur = v_new;
        if (tid == 0) H->B[j] = t_new;
    }
    __syncthreads();
}

// objective (model.py:145-148) of H->B, identical in every thread
template <int PMAX>
__device__ double block_objective(const BlockMem<PMAX> &M, int n, int p, double lam)
{
    BlockHead<PMAX> *H = M.H;
    for (int i = threadIdx.x; i < n; i += (int)blockDim.x) {
        const double g = gemv_row(p, i, n, [&](int q) { return M.X[i * M.xs + q]; }, [&](int q) { return H->B[q]; });
        M.tmp[i] = fabs(dsub(M.Y[i], g));
    }
    __syncthreads();
    if (threadIdx.x == 0)
        H->bcd[2] = dadd(np_sum_rec(0, n, [&](int i) { return M.tmp[i]; }),
                         dmul(lam, np_sum(p, [&](int q) { return fabs(H->B[q]); })));
    __syncthreads();
    const double v = H->bcd[2];
    __syncthreads();
    return v;
}

// ccd_descend (ccd.py:126-206) for the request in this warp's controller copy, block-wide.
template <int PMAX>
__device__ void block_descent(const BlockMem<PMAX> &M, Ctl<PMAX> &C, int n, int p)
{
    BlockHead<PMAX> *H = M.H;
    const int tid = threadIdx.x, lane = tid & 31;
    const int frozen = C.req_frozen;
    const double tol = C.req_tol;
    const int max_sweeps = C.req_sweeps;
    const double lam = C.lam;
    const uint32_t sparse = C.sparse_mask;
    if (tid < p) H->B[tid] = C.req_start[tid];
    __syncthreads();
    double r[BLK_EPT];
#pragma unroll
    for (int q = 0; q < BLK_EPT; ++q) {
        const int i = tid + q * (int)blockDim.x;
        r[q] = 0.0;
        if (i < n) {
            const double g = gemv_row(p, i, n, [&](int c) { return M.X[i * M.xs + c]; }, [&](int c) { return H->B[c]; });
            r[q] = dsub(M.Y[i], g);
            M.tmp[i] = fabs(r[q]);
        }
    }
    __syncthreads();
    if (tid == 0)
        H->bcd[3] = dadd(np_sum_rec(0, n, [&](int i) { return M.tmp[i]; }),
                         dmul(lam, np_sum(p, [&](int c) { return fabs(H->B[c]); })));
    __syncthreads();
    double f_cur = H->bcd[3];
    double sum_abs_b = np_sum(p, [&](int c) { return fabs(H->B[c]); });
    double f_sweep_start = f_cur;
    int sweeps = 1, steps = 0, conv = 0;
    const int j0 = (frozen == 0) ? 1 : 0;
    int j = j0;
    if (j >= p) {
        conv = 1;
    } else {
        for (;;) {
            block_step<PMAX>(M, n, p, j, lam, (sparse >> j) & 1u, r, f_cur, sum_abs_b);
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
            sum_abs_b = np_sum(p, [&](int c) { return fabs(H->B[c]); });
            j = j0;
        }
    }
    const double obj = block_objective<PMAX>(M, n, p, lam);
    const int D = C.D;
    const long long S = C.S;
    __syncwarp();
    if (lane < p) C.res_beta[lane] = H->B[lane];
    if (lane == 0) {
        C.res_obj = obj;
        C.res_conv = conv;
        C.res_sweeps = sweeps;
        C.res_steps = steps;
        C.D = D + 1;
        C.S = S + steps;
    }
    __syncwarp();
    __syncthreads();
}

template <int PMAX>
__global__ void __launch_bounds__(BLK_THREADS) locus_block_kernel(LocusArgs A)
{
    extern __shared__ __align__(16) unsigned char blk_smem[];
    const int n = A.n, p = A.p;
    const BlockLayout L = block_layout<PMAX>(n, p);
    BlockMem<PMAX> M;
    M.H = reinterpret_cast<BlockHead<PMAX> *>(blk_smem);
    M.X = reinterpret_cast<double *>(blk_smem + L.off_X);
    M.Y = reinterpret_cast<double *>(blk_smem + L.off_Y);
    M.loc = reinterpret_cast<double *>(blk_smem + L.off_loc);
    M.w = reinterpret_cast<double *>(blk_smem + L.off_w);
    M.sk = reinterpret_cast<double *>(blk_smem + L.off_sk);
    M.si = reinterpret_cast<int *>(blk_smem + L.off_si);
    M.aw = reinterpret_cast<double2 *>(blk_smem + L.off_aw);
    M.tmp = reinterpret_cast<double *>(blk_smem + L.off_tmp);
    M.pos = reinterpret_cast<int *>(blk_smem + L.off_pos);
    M.P2 = L.P2;
    M.xs = p | 1;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    Ctl<PMAX> &C = M.H->C[wp];
    if (threadIdx.x < PMAX) {
        M.H->cand[threadIdx.x] = 0;
    }
    if (lane == 0) C.pc = PC_FETCH;
    __syncthreads();
    BlockAccess<PMAX> acc{n, p, lane, M};
    for (;;) {
        const int act = controller<PMAX>(C, A, acc, blockIdx.x);
        __syncthreads();
        if (act == ACT_EXIT) break;
        block_descent<PMAX>(M, C, n, p);
    }
}

}  // namespace lad
