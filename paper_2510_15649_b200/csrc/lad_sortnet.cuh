// lad_sortnet.cuh -- register-resident sorting network for the weighted-median
// coordinate step (ccd.py:81-91 restated).
//
// The reference sorts the n+1 breakpoints with np.argsort(kind="stable"), i.e.
// by (location, original index).  A Batcher odd-even merge network over the
// next power of two, pruned to the live width NE (pads would be +inf and never
// move), sorts (key, idx) pairs lexicographically, which is exactly that stable
// order.  All indices are compile-time constants after unrolling, so the keys
// stay in registers.
#pragma once
#include <cuda_runtime.h>

namespace lad {

struct SortNet {
    int n;
    unsigned char a[512];
    unsigned char b[512];
};

__host__ __device__ constexpr int next_pow2(int v)
{
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// Batcher odd-even merge sort, comparators (i, j) with i < j, pruned to j < NE.
__host__ __device__ constexpr SortNet make_oddeven(int NE)
{
    SortNet net{};
    int ns = next_pow2(NE);
    int c = 0;
    for (int p = 1; p < ns; p += p)
        for (int k = p; k >= 1; k /= 2)
            for (int j = k % p; j + k < ns; j += k + k)
                for (int i = 0; i < k && i < ns - j - k; ++i)
                    if ((i + j) / (p + p) == (i + j + k) / (p + p)) {
                        int lo = i + j, hi = i + j + k;
                        if (hi < NE) {
                            net.a[c] = (unsigned char)lo;
                            net.b[c] = (unsigned char)hi;
                            ++c;
                        }
                    }
    net.n = c;
    return net;
}

template <int NE>
struct NetHolder {
    static constexpr SortNet net = make_oddeven(NE);
};

// Compare-exchange on (key, idx) lexicographic.  idx values are distinct.
__device__ __forceinline__ void cmpx(double &ka, int &ia, double &kb, int &ib)
{
    bool sw = (ka > kb) | ((ka == kb) & (ia > ib));
    double k0 = sw ? kb : ka, k1 = sw ? ka : kb;
    int i0 = sw ? ib : ia, i1 = sw ? ia : ib;
    ka = k0; kb = k1; ia = i0; ib = i1;
}

template <int NE>
__device__ __forceinline__ void sort_pairs(double (&key)[NE], int (&idx)[NE])
{
    constexpr SortNet net = make_oddeven(NE);
#pragma unroll
    for (int c = 0; c < net.n; ++c) cmpx(key[net.a[c]], idx[net.a[c]], key[net.b[c]], idx[net.b[c]]);
}

}  // namespace lad
