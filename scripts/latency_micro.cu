// Dependent-chain latencies (cycles per operation) of the operations on the locus kernel's
// critical path, measured with clock64 on one warp: DFMA / DADD / DMUL (the v_new FMA tail,
// the Markstein division), 32-bit SHFL, REDUX.SUM (+ the move out of the uniform register,
// as used by the median test), LDS.32 (pointer chase through shared memory).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency_micro scripts/latency_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void chains(long long *out, double *sink, const double *src)
{
    __shared__ int sh[64];
    const int lane = threadIdx.x;
    sh[lane] = (lane + 1) & 63;
    sh[lane + 32] = (lane + 33) & 63;
    __syncwarp();
    const int nxt = (lane + 1) & 31;
    double a = src[lane], b = src[lane + 32], c = 1.0;
    unsigned u = lane;
    int idx = lane;
    long long t0, t1;

    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) c = fma(a, c, b);
    t1 = clock64();
    out[0] = t1 - t0;

    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) c = __dadd_rn(c, b);
    t1 = clock64();
    out[1] = t1 - t0;

    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) c = __dmul_rn(c, a);
    t1 = clock64();
    out[2] = t1 - t0;

    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) u = __shfl_sync(0xffffffffu, u, nxt);
    t1 = clock64();
    out[3] = t1 - t0;

    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) u = __reduce_add_sync(0xffffffffu, u) & 31u;
    t1 = clock64();
    out[4] = t1 - t0;

    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) idx = sh[idx];
    t1 = clock64();
    out[5] = t1 - t0;

    sink[lane] = c + u + idx;
}

int main()
{
    long long *d_out, h_out[6];
    double *d_sink, *d_src, h_src[64];
    for (int i = 0; i < 64; ++i) h_src[i] = 1.0 + 1e-9 * i;
    cudaMalloc(&d_out, sizeof h_out);
    cudaMalloc(&d_sink, 64 * sizeof(double));
    cudaMalloc(&d_src, sizeof h_src);
    cudaMemcpy(d_src, h_src, sizeof h_src, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) chains<<<1, 32>>>(d_out, d_sink, d_src);
    cudaMemcpy(h_out, d_out, sizeof h_out, cudaMemcpyDeviceToHost);
    const char *names[6] = {"dfma", "dadd", "dmul", "shfl_idx_32", "redux_sum", "lds_32"};
    printf("{");
    for (int k = 0; k < 6; ++k) printf("%s\"%s\": %.2f", k ? ", " : "", names[k], (double)h_out[k] / N);
    printf("}\n");
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
