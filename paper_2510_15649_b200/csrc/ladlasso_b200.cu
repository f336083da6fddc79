// ladlasso_b200.cu -- C ABI over the sm_100a kernels (see include/ladlasso_b200.h).
//
// Dispatch picks a compile-time (n, p) instantiation of the locus kernel for
// the BASELINE.json shapes (register-resident sort network, fully unrolled
// reduction trees) and a runtime-shape instantiation for everything else.
#include <cuda_runtime.h>
#include <cstdlib>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <string>

#include "../../include/ladlasso_b200.h"
#include "lad_brute.cuh"
#include "lad_cert.cuh"
#include "lad_lp.cuh"
#include "lad_gen.cuh"
#include "lad_genspec.cuh"
#include "lad_locus.cuh"
#include "lad_locus_warp.cuh"
#include "lad_locus_block.cuh"

#define LAD_VERSION 103

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};  // kernels this library has launched (all threads)

static int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(expr)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess) return fail(LAD_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

extern "C" int lad_version(void) { return LAD_VERSION; }
extern "C" long long lad_kernel_launches(void) { return g_launches.load(); }
extern "C" const char *lad_last_error(void) { return g_err.c_str(); }

extern "C" void lad_default_params(lad_locus_params *prm)
{
    prm->outer_axis = -1;
    prm->outer_search = LAD_OUTER_TERNARY;
    prm->outer_tolerance = 1e-9;
    prm->outer_probes = 8;
    prm->outer_max_iterations = 200;
    prm->has_bracket = 0;
    prm->bracket_lo = -1.0;
    prm->bracket_hi = 1.0;
    prm->inner_sweep_tol = 1e-10;
    prm->inner_max_sweeps = 500;
    prm->lambda_floor = 1e-9;
    prm->seen_capacity = 0;
}

static_assert(sizeof(lad_locus_params) == sizeof(lad::LocusParamsDev), "params layout");

namespace {

using KernelFn = void (*)(lad::LocusArgs);

struct Variant {
    KernelFn fn;
    int nmax, pmax;
    size_t smem;      // dynamic shared memory per block
    int block;        // threads per block
    int slots_per_block;  // independent solvers (seen-list slots) per block
    bool warp_mapped;     // warp-per-problem kernel (the axis-parallel mode's work items)
    int carveout_blocks;  // > 0: ask for the smallest shared-memory carve-out that holds this many blocks per SM
};

template <int N, int P, bool EXACT>
Variant make_thread_variant()
{
    constexpr int w = lad::thread_warps<N, EXACT>;
    return Variant{lad::locus_kernel<N, P, EXACT>, N, P, lad::smem_doubles_per_warp<N, P, EXACT>() * sizeof(double) * w,
                   32 * w, 32 * w, false, EXACT ? lad::thread_min_blocks<N, EXACT> : 0};
}

template <int P, int NC, typename T = double>
Variant make_warp_variant()
{
    constexpr int wpb = lad::warps_per_block<P, T>;
    return Variant{lad::locus_warp_kernel<P, NC, T>, 31, P, sizeof(lad::WarpShared<P, T>) * wpb, 32 * wpb, wpb, true, 0};
}

int g_kernel_policy = LAD_KERNEL_AUTO;
int g_axis_parallel = 1;

bool pick_variant(int n, int p, Variant &v, bool f32)
{
    const bool warp_ok = n <= 31 && p <= 8;
    if (f32) {  // fp32 mode: warp-per-problem only
        if (!warp_ok) return false;
        if (n == 31 && p == 8) v = make_warp_variant<8, 31, float>();
        else if (n == 30 && p == 5) v = make_warp_variant<5, 30, float>();
        else if (p <= 3) v = make_warp_variant<3, 0, float>();
        else if (p <= 5) v = make_warp_variant<5, 0, float>();
        else v = make_warp_variant<8, 0, float>();
        return true;
    }
    const bool thread_exact = n == 10 && p == 2;  // config 1: thread-per-problem (north_star's tiny-n variant)
    int policy = g_kernel_policy;
    if (policy == LAD_KERNEL_AUTO) policy = (thread_exact || !warp_ok) ? LAD_KERNEL_THREAD : LAD_KERNEL_WARP;
    if (policy == LAD_KERNEL_WARP && warp_ok) {
        // compile-time shapes of BASELINE configs 0/2 (30,5), 3 (25,5), 4 (31,8)
        if (n == 30 && p == 5) v = make_warp_variant<5, 30>();
        else if (n == 25 && p == 5) v = make_warp_variant<5, 25>();
        else if (n == 31 && p == 8) v = make_warp_variant<8, 31>();
        else if (p <= 3) v = make_warp_variant<3, 0>();
        else if (p <= 5) v = make_warp_variant<5, 0>();
        else v = make_warp_variant<8, 0>();
        return true;
    }
    const bool block_ok = n >= 32 && n <= lad::BLK_NMAX && p <= 8;
    if (block_ok && !(g_kernel_policy == LAD_KERNEL_THREAD && n <= 32)) {  // block per problem (32 <= n <= 1023)
        const int threads = std::min(lad::BLK_THREADS, 32 * ((n + 1 + 31) / 32));
        v = Variant{lad::locus_block_kernel<8>, lad::BLK_NMAX, 8, lad::block_layout<8>(n, p).total, threads, 1, false, 0};
        return true;
    }
    if (thread_exact) v = make_thread_variant<10, 2, true>();
    else if (n <= 16 && p <= 4) v = make_thread_variant<16, 4, false>();
    else if (n <= 32 && p <= 8) v = make_thread_variant<32, 8, false>();
    else return false;
    return true;
}

int g_num_sms = 0;
int g_smem_per_sm = 228 * 1024;  // shared memory per SM (the carve-out preference is a percentage of it)
std::atomic<uint64_t> g_pool_devices{0};  // devices whose default pool keeps freed scratch mapped

// Per-process, per-device setup: the SM count (grid sizing) and the default
// stream-ordered pool's release threshold, so the per-call scratch (seen lists,
// counters) stays mapped between calls instead of being returned to the OS at
// every synchronize (default threshold 0).
cudaError_t device_init()
{
    int dev;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (g_num_sms == 0) {
        e = cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        int smem = 0;
        if (cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) == cudaSuccess && smem > 0)
            g_smem_per_sm = smem;
    }
    const uint64_t bit = 1ull << (dev & 63);
    if (!(g_pool_devices.load() & bit)) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = 2ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        g_pool_devices.fetch_or(bit);
    }
    return cudaSuccess;
}

// Curve points one _CurveEvaluator can record (locus.py:188-191, :210-212, :278-288): the bracket
// expansion (2 + 3 per iteration, at most 60: linesearch.py:247-268), the outer rounds (2 probes per
// ternary round, `probes` per quadrature round) and the final mid probe; a refine evaluator holds
// 1 + fan + 64.  The outer rounds are bounded by the tolerance (ternary shrinks the bracket to 2/3
// per round, quadrature to 2/(probes+1)) plus 32 rounds of slack, not by outer_max_iterations: a
// huge max_iterations costs nothing unless a search really stalls, and a search that outgrows the
// list ends with status 3 (the host API re-runs such problems with prm->seen_capacity = the worst
// case, worst_case_seen_capacity) instead of silently truncating the nearest-point scan.
long long worst_case_seen(const lad_locus_params *prm)
{
    long long outer = prm->outer_search == LAD_OUTER_TERNARY ? 2LL * prm->outer_max_iterations
                                                             : (long long)prm->outer_probes * prm->outer_max_iterations;
    return std::max(2 + 3 * 60 + outer + 1, 1LL + 12 + 64);
}

int seen_capacity(const lad_locus_params *prm, int p)
{
    if (p <= 2) return 0;  // no warm starts below d = 3 (locus.py:199-202)
    if (prm->seen_capacity > 0) return (int)std::min<long long>(prm->seen_capacity, worst_case_seen(prm));
    const double shrink = prm->outer_search == LAD_OUTER_TERNARY ? 2.0 / 3.0 : 2.0 / (prm->outer_probes + 1.0);
    long long rounds = (long long)std::ceil(std::log(prm->outer_tolerance) / std::log(shrink));
    rounds = std::max(0LL, rounds) + 32;
    rounds = std::min<long long>(rounds, prm->outer_max_iterations);
    const long long per_round = prm->outer_search == LAD_OUTER_TERNARY ? 2 : prm->outer_probes;
    return (int)std::min(std::max(2 + 3 * 60 + per_round * rounds + 1, 1LL + 12 + 64), worst_case_seen(prm));
}

// X, Y, lam are double* (f32 == false) or float* (f32 == true)
int run_locus(const void *X, const void *Y, const void *lam, const int64_t *data_index, int64_t Bd, int64_t B, int n, int p,
              const lad_locus_params *prm, const lad_locus_out *out, cudaStream_t st, int mode, const double *start,
              const int32_t *frozen, double desc_tol, int desc_sweeps, bool f32 = false,
              const double *brackets = nullptr)
{
    if (B < 0 || n < 1 || p < 1) return fail(LAD_E_INVALID, "need B >= 0, n >= 1, p >= 1 (got %lld, %d, %d)", (long long)B, n, p);
    if (B == 0) return LAD_OK;
    if (data_index && Bd < 1) return fail(LAD_E_INVALID, "Bd must be >= 1 with data_index");
    if (!data_index && Bd != B) return fail(LAD_E_INVALID, "Bd must equal B without data_index");
    if (!out || !out->beta || !out->objective || !out->iterations || !out->objective_evals || !out->converged ||
        !out->status)
        return fail(LAD_E_INVALID, "output pointers must be non-null");
    if (prm->outer_tolerance <= 0) return fail(LAD_E_INVALID, "outer_tolerance must be positive");
    if (prm->outer_probes < 3) return fail(LAD_E_INVALID, "probes must be at least 3");
    if (prm->outer_max_iterations < 1) return fail(LAD_E_INVALID, "max_iterations must be at least 1");
    if (prm->inner_sweep_tol <= 0) return fail(LAD_E_INVALID, "sweep_tolerance must be positive");
    if (prm->inner_max_sweeps < 1) return fail(LAD_E_INVALID, "max_sweeps must be at least 1");
    if (prm->outer_axis >= p) return fail(LAD_E_INVALID, "outer_axis %d out of range for d=%d", prm->outer_axis, p);
    if (prm->seen_capacity < 0) return fail(LAD_E_INVALID, "seen_capacity must be >= 0");
    if (!brackets && prm->has_bracket && !(prm->bracket_lo < prm->bracket_hi))
        return fail(LAD_E_INVALID, "bracket needs lo < hi");
    if (!(prm->lambda_floor > 0)) return fail(LAD_E_INVALID, "lambda_floor must be finite and > 0");
    Variant v;
    if (!pick_variant(n, p, v, f32))
        return fail(LAD_E_UNSUPPORTED, "n=%d p=%d beyond n<=%d, p<=8", n, p, f32 ? 31 : lad::BLK_NMAX);

    CK(device_init());
    if (v.smem > 48 * 1024) CK(cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem));
    if (v.carveout_blocks > 0) {
        // the thread kernel keeps its controller state in local memory: every KB of L1 counts, so
        // ask for the smallest carve-out that still holds its resident blocks (+1 KB reserved each)
        // (the preference is a percentage the driver rounds up to a supported size: name the size)
        const size_t need = (size_t)v.carveout_blocks * (v.smem + 1024);
        static const int kCarveKB[] = {0, 8, 16, 32, 64, 100, 132, 164, 196, 228};
        size_t pick = (size_t)g_smem_per_sm;
        for (int kb : kCarveKB)
            if ((size_t)kb * 1024 >= need) {
                pick = (size_t)kb * 1024;
                break;
            }
        const int pct = (int)std::min<size_t>(100, pick * 100 / (size_t)g_smem_per_sm);
        CK(cudaFuncSetAttribute(v.fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    }
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v.fn, v.block, v.smem));
    if (per_sm < 1) return fail(LAD_E_CUDA, "locus kernel does not fit on an SM (smem %zu)", v.smem);
    const int64_t max_grid = (int64_t)g_num_sms * per_sm;
    // Small batches leave most warps idle and are bound by one solve's latency:
    // run the independent per-axis searches as separate work items (warp kernel).
    // Up to two waves of problems it also wins: the finer items fill the grid's
    // tail (scripts/axis_threshold.py: B = 8,192 +11% for config 2 shapes, +5%
    // for config 4; equal at 16,384), despite searching every axis where the
    // serial scan stops after two confirmations.
    const bool axis_par = g_axis_parallel && mode == lad::MODE_LOCUS && v.warp_mapped && prm->outer_axis < 0 &&
                          p > 1 && (g_axis_parallel == 2 || B < 2 * max_grid * v.slots_per_block);
    const int64_t items = axis_par ? B * p : B;
    int64_t want = (items + v.slots_per_block - 1) / v.slots_per_block;
    int64_t grid = std::min<int64_t>(want, max_grid);
    int64_t slots = grid * v.slots_per_block;

    lad::LocusArgs A;
    memset(&A, 0, sizeof A);
    if (f32) {
        A.Xf = (const float *)X;
        A.Yf = (const float *)Y;
        A.lamf = (const float *)lam;
    } else {
        A.X = (const double *)X;
        A.Y = (const double *)Y;
        A.lam = (const double *)lam;
    }
    A.data_index = data_index;
    A.Bd = data_index ? Bd : B;
    A.B = B;
    A.n = n;
    A.p = p;
    memcpy(&A.prm, prm, sizeof A.prm);
    A.mode = mode;
    A.start = start;
    A.frozen = frozen;
    A.desc_tol = desc_tol;
    A.desc_sweeps = desc_sweeps;
    A.beta = out->beta;
    A.objective = out->objective;
    A.iterations = out->iterations;
    A.objective_evals = out->objective_evals;
    A.converged = out->converged;
    A.status = out->status;
    A.descents = out->descents;
    A.steps = out->steps;
    A.seen_cap = mode == lad::MODE_LOCUS ? seen_capacity(prm, p) : 0;
    A.brackets = mode == lad::MODE_LOCUS ? brackets : nullptr;
    size_t seen_bytes = (size_t)slots * A.seen_cap * (1 + v.pmax) * sizeof(double);
    A.axis_stride = v.pmax + 10;
    size_t axis_bytes = axis_par ? (size_t)B * p * A.axis_stride * sizeof(double) : 0;
    size_t done_bytes = axis_par ? (size_t)B * sizeof(unsigned) : 0;
    size_t scratch = 256 + seen_bytes + axis_bytes + done_bytes;
    char *buf = nullptr;
    CK(cudaMallocAsync((void **)&buf, scratch, st));
    A.counter = (unsigned long long *)buf;
    A.seen = A.seen_cap ? (double *)(buf + 256) : nullptr;
    A.axis_res = axis_par ? (double *)(buf + 256 + seen_bytes) : nullptr;
    A.axis_done = axis_par ? (unsigned *)(buf + 256 + seen_bytes + axis_bytes) : nullptr;
    CK(cudaMemsetAsync(buf, 0, 256, st));
    if (axis_par) CK(cudaMemsetAsync(A.axis_done, 0, done_bytes, st));
    cudaError_t le;
    if (!axis_par) {
        A.axis_mode = lad::AXIS_SERIAL;
        v.fn<<<(unsigned)grid, v.block, v.smem, st>>>(A); ++g_launches;
        le = cudaGetLastError();
    } else {
        // one launch: the per-axis searches as work items, each problem's finish
        // (agreement, refine, polish) run by the warp that completes its last search
        A.axis_mode = lad::AXIS_SEARCH;
        v.fn<<<(unsigned)grid, v.block, v.smem, st>>>(A); ++g_launches;
        le = cudaGetLastError();
    }
    cudaFreeAsync(buf, st);
    if (le != cudaSuccess) return fail(LAD_E_CUDA, "locus kernel launch: %s", cudaGetErrorString(le));
    return LAD_OK;
}

}  // namespace

extern "C" int lad_copy_h2d(void *dst, const void *src, size_t bytes, void *stream)
{
    if (bytes == 0) return LAD_OK;
    if (dst == nullptr || src == nullptr) return fail(LAD_E_INVALID, "lad_copy_h2d: null pointer");
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    return LAD_OK;
}

extern "C" int lad_set_axis_parallel(int32_t enable)
{
    g_axis_parallel = enable < 0 ? 0 : (enable > 2 ? 2 : enable);
    return LAD_OK;
}

extern "C" int lad_set_kernel_policy(int32_t policy)
{
    if (policy < LAD_KERNEL_AUTO || policy > LAD_KERNEL_WARP) return fail(LAD_E_INVALID, "unknown kernel policy %d", policy);
    g_kernel_policy = policy;
    return LAD_OK;
}

extern "C" int lad_locus_solve_f64(const double *X, const double *Y, const double *lam, const int64_t *data_index,
                                   int64_t Bd, int64_t B, int32_t n, int32_t p, const lad_locus_params *prm,
                                   const lad_locus_out *out, void *stream)
{
    lad_locus_params def;
    if (!prm) {
        lad_default_params(&def);
        prm = &def;
    }
    return run_locus(X, Y, lam, data_index, Bd, B, n, p, prm, out, (cudaStream_t)stream, lad::MODE_LOCUS, nullptr,
                     nullptr, 0.0, 0);
}

extern "C" int lad_locus_solve_bracketed_f64(const double *X, const double *Y, const double *lam,
                                             const int64_t *data_index, int64_t Bd, int64_t B, int32_t n, int32_t p,
                                             const double *brackets, const lad_locus_params *prm,
                                             const lad_locus_out *out, void *stream)
{
    lad_locus_params def;
    if (!prm) {
        lad_default_params(&def);
        prm = &def;
    }
    if (!brackets && B > 0) return fail(LAD_E_INVALID, "brackets must be non-null");
    return run_locus(X, Y, lam, data_index, Bd, B, n, p, prm, out, (cudaStream_t)stream, lad::MODE_LOCUS, nullptr,
                     nullptr, 0.0, 0, false, brackets);
}

extern "C" int lad_ccd_descend_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n,
                                   int32_t p, const double *start, const int32_t *frozen, double sweep_tolerance,
                                   int32_t max_sweeps, double lambda_floor, const lad_locus_out *out, void *stream)
{
    if (!(sweep_tolerance > 0)) return fail(LAD_E_INVALID, "sweep_tolerance must be positive");
    if (max_sweeps < 1) return fail(LAD_E_INVALID, "max_sweeps must be at least 1");
    if (!start && B > 0) return fail(LAD_E_INVALID, "start must be non-null");
    lad_locus_params prm;
    lad_default_params(&prm);
    prm.lambda_floor = lambda_floor;
    return run_locus(X, Y, lam, nullptr, B, B, n, p, &prm, out, (cudaStream_t)stream, lad::MODE_DESCENT, start, frozen,
                     sweep_tolerance, max_sweeps);
}

extern "C" int lad_locus_solve_f32(const float *X, const float *Y, const float *lam, const int64_t *data_index,
                                   int64_t Bd, int64_t B, int32_t n, int32_t p, const lad_locus_params *prm,
                                   const lad_locus_out *out, void *stream)
{
    lad_locus_params def;
    if (!prm) {
        lad_default_params(&def);
        prm = &def;
    }
    return run_locus(X, Y, lam, data_index, Bd, B, n, p, prm, out, (cudaStream_t)stream, lad::MODE_LOCUS, nullptr,
                     nullptr, 0.0, 0, true);
}

extern "C" int lad_ccd_descend_f32(const float *X, const float *Y, const float *lam, int64_t B, int32_t n, int32_t p,
                                   const double *start, const int32_t *frozen, double sweep_tolerance,
                                   int32_t max_sweeps, double lambda_floor, const lad_locus_out *out, void *stream)
{
    if (!(sweep_tolerance > 0)) return fail(LAD_E_INVALID, "sweep_tolerance must be positive");
    if (max_sweeps < 1) return fail(LAD_E_INVALID, "max_sweeps must be at least 1");
    if (!start && B > 0) return fail(LAD_E_INVALID, "start must be non-null");
    lad_locus_params prm;
    lad_default_params(&prm);
    prm.lambda_floor = lambda_floor;
    return run_locus(X, Y, lam, nullptr, B, B, n, p, &prm, out, (cudaStream_t)stream, lad::MODE_DESCENT, start, frozen,
                     sweep_tolerance, max_sweeps, true);
}

// problems per chunk of the pipelined host-buffer solve (below).  Config 1, 2^20 problems from pinned
// host arrays, same box: one launch 56.2 ms, chunks of 2^19 / 2^18 / 2^17 / 2^16: 53.1 / 52.8 / 56.5 / 57.7 ms
// (smaller chunks lose more to their launch tails than the overlap of the copies wins)
static const int64_t HOST_CHUNK = [] {
    const char *v = getenv("LAD_HOST_CHUNK");  // tuning knob (problems per chunk)
    const long long c = v ? atoll(v) : 0;
    return (int64_t)(c >= 1024 ? c : (1 << 18));
}();

template <typename T>
static int locus_solve_host(const T *X, const T *Y, const T *lam, const int64_t *data_index, int64_t Bd, int64_t B,
                            int32_t n, int32_t p, const lad_locus_params *prm, const lad_locus_out *out, void *stream,
                            const double *brackets = nullptr)
{
    cudaStream_t st = (cudaStream_t)stream;
    if (B < 0 || Bd < 0) return fail(LAD_E_INVALID, "B < 0");
    if (!data_index && Bd != B) return fail(LAD_E_INVALID, "Bd must equal B without data_index");
    if (B == 0) return LAD_OK;
    auto rup = [](size_t s) { return (s + 255) & ~(size_t)255; };
    const size_t es = sizeof(T);
    size_t bx = (size_t)Bd * n * p * es, by = (size_t)Bd * n * es, bl = (size_t)B * es, bb = (size_t)B * p * 8;
    size_t bi = data_index ? (size_t)B * 8 : 0;
    size_t bk = brackets ? (size_t)B * 16 : 0;
    size_t total = rup(bx) + rup(by) + rup(bl) + rup(bi) + rup(bk) + rup(bb) + rup(B * 8) + 2 * rup(B * 4) +
                   2 * rup(B) + rup(B * 4) + rup(B * 8);
    char *d = nullptr;
    CK(cudaMallocAsync((void **)&d, total, st));
    char *q = d;
    auto take = [&](size_t sz) {
        char *r = q;
        q += rup(sz);
        return r;
    };
    T *dX = (T *)take(bx), *dY = (T *)take(by), *dL = (T *)take(bl);
    int64_t *dI = data_index ? (int64_t *)take(bi) : nullptr;
    double *dK = brackets ? (double *)take(bk) : nullptr;
    lad_locus_out dout;
    dout.beta = (double *)take(bb);
    dout.objective = (double *)take(B * 8);
    dout.iterations = (int32_t *)take(B * 4);
    dout.objective_evals = (int32_t *)take(B * 4);
    dout.converged = (uint8_t *)take(B);
    dout.status = (uint8_t *)take(B);
    dout.descents = out->descents ? (int32_t *)take(B * 4) : nullptr;
    dout.steps = out->steps ? (int64_t *)take(B * 8) : nullptr;
    int rc = LAD_OK;
    cudaError_t e = cudaSuccess;
    // Large batches of independent problems (no data_index): the batch is cut into chunks that
    // alternate between two side streams, so one chunk's copies overlap the other's solve and the
    // solves fill each other's launch tails.  Results are those of the single launch (problems are
    // independent); the caller's stream is joined before the call returns.
    if (!data_index && !brackets && B >= 2 * HOST_CHUNK) {
        cudaStream_t ss[2] = {nullptr, nullptr};
        cudaEvent_t ev0 = nullptr, ev[2] = {nullptr, nullptr};
        e = cudaStreamCreateWithFlags(&ss[0], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ss[1], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
        for (int k = 0; k < 2 && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(ev0, st);  // after the allocation and the caller's earlier work
        for (int k = 0; k < 2 && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(ss[k], ev0, 0);
        int64_t c = 0;
        for (int64_t off = 0; off < B && e == cudaSuccess && rc == LAD_OK; off += HOST_CHUNK, ++c) {
            const int64_t nb = std::min<int64_t>(HOST_CHUNK, B - off);
            cudaStream_t sc = ss[c & 1];
            const size_t xo = (size_t)off * n * p, yo = (size_t)off * n;
            e = cudaMemcpyAsync(dX + xo, X + xo, (size_t)nb * n * p * es, cudaMemcpyHostToDevice, sc);
            if (e == cudaSuccess) e = cudaMemcpyAsync(dY + yo, Y + yo, (size_t)nb * n * es, cudaMemcpyHostToDevice, sc);
            if (e == cudaSuccess) e = cudaMemcpyAsync(dL + off, lam + off, (size_t)nb * es, cudaMemcpyHostToDevice, sc);
            if (e != cudaSuccess) break;
            lad_locus_out co = dout;
            co.beta += (size_t)off * p;
            co.objective += off;
            co.iterations += off;
            co.objective_evals += off;
            co.converged += off;
            co.status += off;
            if (co.descents) co.descents += off;
            if (co.steps) co.steps += off;
            if constexpr (sizeof(T) == 4) rc = lad_locus_solve_f32(dX + xo, dY + yo, dL + off, nullptr, nb, nb, n, p, prm, &co, sc);
            else rc = lad_locus_solve_f64(dX + xo, dY + yo, dL + off, nullptr, nb, nb, n, p, prm, &co, sc);
            if (rc != LAD_OK) break;
            struct { void *h; const void *d; size_t w; } cp[] = {
                {out->beta, dout.beta, (size_t)p * 8}, {out->objective, dout.objective, 8}, {out->iterations, dout.iterations, 4},
                {out->objective_evals, dout.objective_evals, 4}, {out->converged, dout.converged, 1},
                {out->status, dout.status, 1}, {out->descents, dout.descents, 4}, {out->steps, dout.steps, 8}};
            for (auto &q : cp)
                if (q.h && q.d && e == cudaSuccess)
                    e = cudaMemcpyAsync((char *)q.h + (size_t)off * q.w, (const char *)q.d + (size_t)off * q.w,
                                        (size_t)nb * q.w, cudaMemcpyDeviceToHost, sc);
        }
        for (int k = 0; k < 2; ++k)  // join the side streams into the caller's (also on an error: nothing may outlive d)
            if (ss[k] && ev[k] && cudaEventRecord(ev[k], ss[k]) == cudaSuccess) cudaStreamWaitEvent(st, ev[k], 0);
        cudaFreeAsync(d, st);
        cudaError_t se = cudaStreamSynchronize(st);
        for (int k = 0; k < 2; ++k) {
            if (ss[k]) cudaStreamSynchronize(ss[k]);
            if (ev[k]) cudaEventDestroy(ev[k]);
            if (ss[k]) cudaStreamDestroy(ss[k]);
        }
        if (ev0) cudaEventDestroy(ev0);
        if (e != cudaSuccess) return fail(LAD_E_CUDA, "host solve (chunked): %s", cudaGetErrorString(e));
        if (rc != LAD_OK) return rc;
        if (se != cudaSuccess) return fail(LAD_E_CUDA, "host solve (chunked): %s", cudaGetErrorString(se));
        return LAD_OK;
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(dX, X, bx, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dY, Y, by, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dL, lam, bl, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && dI) e = cudaMemcpyAsync(dI, data_index, bi, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && dK) e = cudaMemcpyAsync(dK, brackets, bk, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        if constexpr (sizeof(T) == 4) rc = lad_locus_solve_f32(dX, dY, dL, dI, Bd, B, n, p, prm, &dout, stream);
        else if (dK) rc = lad_locus_solve_bracketed_f64(dX, dY, dL, dI, Bd, B, n, p, dK, prm, &dout, stream);
        else rc = lad_locus_solve_f64(dX, dY, dL, dI, Bd, B, n, p, prm, &dout, stream);
    }
    if (e == cudaSuccess && rc == LAD_OK) {
        struct { void *h; const void *d; size_t s; } cp[] = {
            {out->beta, dout.beta, bb}, {out->objective, dout.objective, (size_t)B * 8},
            {out->iterations, dout.iterations, (size_t)B * 4}, {out->objective_evals, dout.objective_evals, (size_t)B * 4},
            {out->converged, dout.converged, (size_t)B}, {out->status, dout.status, (size_t)B},
            {out->descents, dout.descents, (size_t)B * 4}, {out->steps, dout.steps, (size_t)B * 8}};
        for (auto &c : cp)
            if (c.h && c.d && e == cudaSuccess) e = cudaMemcpyAsync(c.h, c.d, c.s, cudaMemcpyDeviceToHost, st);
    }
    cudaFreeAsync(d, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(LAD_E_CUDA, "host solve copies: %s", cudaGetErrorString(e));
    if (rc != LAD_OK) return rc;
    if (se != cudaSuccess) return fail(LAD_E_CUDA, "host solve: %s", cudaGetErrorString(se));
    return LAD_OK;
}

extern "C" int lad_locus_solve_host_f64(const double *X, const double *Y, const double *lam,
                                        const int64_t *data_index, int64_t Bd, int64_t B, int32_t n, int32_t p,
                                        const lad_locus_params *prm, const lad_locus_out *out, void *stream)
{
    return locus_solve_host<double>(X, Y, lam, data_index, Bd, B, n, p, prm, out, stream);
}

extern "C" int lad_locus_solve_bracketed_host_f64(const double *X, const double *Y, const double *lam,
                                                  const int64_t *data_index, int64_t Bd, int64_t B, int32_t n,
                                                  int32_t p, const double *brackets, const lad_locus_params *prm,
                                                  const lad_locus_out *out, void *stream)
{
    if (!brackets && B > 0) return fail(LAD_E_INVALID, "brackets must be non-null");
    return locus_solve_host<double>(X, Y, lam, data_index, Bd, B, n, p, prm, out, stream, brackets);
}

extern "C" int lad_locus_solve_host_f32(const float *X, const float *Y, const float *lam, const int64_t *data_index,
                                        int64_t Bd, int64_t B, int32_t n, int32_t p, const lad_locus_params *prm,
                                        const lad_locus_out *out, void *stream)
{
    return locus_solve_host<float>(X, Y, lam, data_index, Bd, B, n, p, prm, out, stream);
}

namespace {
// dense FMA throughput probe: 8 independent chains per thread
template <typename T>
__global__ void fma_peak_kernel(T *out, int iters)
{
    T a0 = T(threadIdx.x * 1e-9), a1 = a0 + T(1e-9), a2 = a0 + T(2e-9), a3 = a0 + T(3e-9), a4 = a0 + T(4e-9),
      a5 = a0 + T(5e-9), a6 = a0 + T(6e-9), a7 = a0 + T(7e-9);
    const T m = T(0.999999999), c = T(1e-12);
    for (int i = 0; i < iters; ++i) {
        a0 = lad::dfma(a0, m, c); a1 = lad::dfma(a1, m, c); a2 = lad::dfma(a2, m, c); a3 = lad::dfma(a3, m, c);
        a4 = lad::dfma(a4, m, c); a5 = lad::dfma(a5, m, c); a6 = lad::dfma(a6, m, c); a7 = lad::dfma(a7, m, c);
    }
    T s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == T(12345.0)) out[0] = s;  // keep the chain alive
}

template <typename T>
int fma_peak_tflops(double *tflops, cudaStream_t st)
{
    CK(device_init());
    const int block = 256, blocks = g_num_sms * 8, iters = 1 << 14;
    T *dout = nullptr;
    CK(cudaMallocAsync((void **)&dout, sizeof(T), st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    fma_peak_kernel<T><<<blocks, block, 0, st>>>(dout, iters); ++g_launches;  // warm-up
    CK(cudaEventRecord(e0, st));
    fma_peak_kernel<T><<<blocks, block, 0, st>>>(dout, iters); ++g_launches;
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(dout, st);
    double flops = 2.0 * 8.0 * iters * (double)block * blocks;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return LAD_OK;
}
}  // namespace

extern "C" int lad_fp64_peak_tflops(double *tflops, void *stream)
{
    return fma_peak_tflops<double>(tflops, (cudaStream_t)stream);
}

extern "C" int lad_fp32_peak_tflops(double *tflops, void *stream)
{
    return fma_peak_tflops<float>(tflops, (cudaStream_t)stream);
}

namespace {
template <int P>
int brute_dispatch(const double *X, const double *Y, const double *lam, int64_t B, int n, int64_t C,
                   double lambda_floor, double *beta, double *objective, int64_t *vertices, cudaStream_t st)
{
    lad::BruteArgs A;
    memset(&A, 0, sizeof A);
    A.X = X;
    A.Y = Y;
    A.lam = lam;
    A.B = B;
    A.n = n;
    A.lambda_floor = lambda_floor;
    A.C = C;
    A.beta = beta;
    A.objective = objective;
    A.vertices = vertices;
    if (C <= 4096) {
        int bs = 128;
        lad::brute_thread_kernel<P><<<(unsigned)((B + bs - 1) / bs), bs, 0, st>>>(A); ++g_launches;
        cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) return fail(LAD_E_CUDA, "brute kernel: %s", cudaGetErrorString(le));
        return LAD_OK;
    }
    A.chunk = 256 * 64;
    A.nchunks = (C + A.chunk - 1) / A.chunk;
    if (A.nchunks > 65535) {
        A.nchunks = 65535;
        A.chunk = (C + A.nchunks - 1) / A.nchunks;
    }
    // grid.y carries the problem: slices of at most 65535 problems (pointers offset per slice)
    const int64_t slice = std::min<int64_t>(B, 65535);
    size_t bytes = (size_t)slice * A.nchunks * (sizeof(lad::BruteKey) + 8);
    char *buf = nullptr;
    CK(cudaMallocAsync((void **)&buf, bytes, st));
    A.partial = (lad::BruteKey *)buf;
    A.pcount = (unsigned long long *)(buf + (size_t)slice * A.nchunks * sizeof(lad::BruteKey));
    cudaError_t le = cudaSuccess;
    for (int64_t s0 = 0; s0 < B && le == cudaSuccess; s0 += slice) {
        lad::BruteArgs S = A;
        S.B = std::min<int64_t>(slice, B - s0);
        S.X = X + (size_t)s0 * n * P;
        S.Y = Y + (size_t)s0 * n;
        S.lam = lam + s0;
        S.beta = beta + (size_t)s0 * P;
        S.objective = objective + s0;
        S.vertices = vertices ? vertices + s0 : nullptr;
        dim3 grid((unsigned)S.nchunks, (unsigned)S.B);
        lad::brute_chunk_kernel<P><<<grid, 256, 0, st>>>(S); ++g_launches;
        lad::brute_reduce_kernel<P><<<(unsigned)((S.B + 127) / 128), 128, 0, st>>>(S); ++g_launches;
        le = cudaGetLastError();
    }
    cudaFreeAsync(buf, st);
    if (le != cudaSuccess) return fail(LAD_E_CUDA, "brute kernel: %s", cudaGetErrorString(le));
    return LAD_OK;
}
}  // namespace

extern "C" int lad_brute_solve_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n,
                                   int32_t p, int32_t max_variables, int64_t max_candidates, double lambda_floor,
                                   double *beta, double *objective, int64_t *vertices, void *stream)
{
    if (n < 1 || p < 1 || B < 0) return fail(LAD_E_INVALID, "bad shape");
    if (n > 64) return fail(LAD_E_UNSUPPORTED, "brute supports n <= 64");
    int64_t C = lad::binom(n + p, p);
    if (p > max_variables)
        return fail(LAD_E_TOO_LARGE, "d=%d exceeds the enumeration limit of %d variables", p, max_variables);
    if (C > max_candidates)
        return fail(LAD_E_TOO_LARGE, "choose(%d, %d) = %lld candidate subsets exceeds the cap of %lld", n + p, p,
                    (long long)C, (long long)max_candidates);
    if (B == 0) return LAD_OK;
    cudaStream_t st = (cudaStream_t)stream;
    switch (p) {
    case 1: return brute_dispatch<1>(X, Y, lam, B, n, C, lambda_floor, beta, objective, vertices, st);
    case 2: return brute_dispatch<2>(X, Y, lam, B, n, C, lambda_floor, beta, objective, vertices, st);
    case 3: return brute_dispatch<3>(X, Y, lam, B, n, C, lambda_floor, beta, objective, vertices, st);
    case 4: return brute_dispatch<4>(X, Y, lam, B, n, C, lambda_floor, beta, objective, vertices, st);
    case 5: return brute_dispatch<5>(X, Y, lam, B, n, C, lambda_floor, beta, objective, vertices, st);
    case 6: return brute_dispatch<6>(X, Y, lam, B, n, C, lambda_floor, beta, objective, vertices, st);
    case 7: return brute_dispatch<7>(X, Y, lam, B, n, C, lambda_floor, beta, objective, vertices, st);
    case 8: return brute_dispatch<8>(X, Y, lam, B, n, C, lambda_floor, beta, objective, vertices, st);
    default: return fail(LAD_E_UNSUPPORTED, "brute supports p <= 8");
    }
}

extern "C" int lad_objective_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n, int32_t p,
                                 const double *beta, double lambda_floor, double *objective, void *stream)
{
    if (n < 1 || p < 1 || p > 8 || B < 0) return fail(LAD_E_INVALID, "bad shape");
    if (B == 0) return LAD_OK;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned g = (unsigned)((B + 127) / 128);
    switch (p) {
    case 1: lad::objective_kernel<1><<<g, 128, 0, st>>>(X, Y, lam, B, n, beta, lambda_floor, objective); ++g_launches; break;
    case 2: lad::objective_kernel<2><<<g, 128, 0, st>>>(X, Y, lam, B, n, beta, lambda_floor, objective); ++g_launches; break;
    case 3: lad::objective_kernel<3><<<g, 128, 0, st>>>(X, Y, lam, B, n, beta, lambda_floor, objective); ++g_launches; break;
    case 4: lad::objective_kernel<4><<<g, 128, 0, st>>>(X, Y, lam, B, n, beta, lambda_floor, objective); ++g_launches; break;
    case 5: lad::objective_kernel<5><<<g, 128, 0, st>>>(X, Y, lam, B, n, beta, lambda_floor, objective); ++g_launches; break;
    case 6: lad::objective_kernel<6><<<g, 128, 0, st>>>(X, Y, lam, B, n, beta, lambda_floor, objective); ++g_launches; break;
    case 7: lad::objective_kernel<7><<<g, 128, 0, st>>>(X, Y, lam, B, n, beta, lambda_floor, objective); ++g_launches; break;
    case 8: lad::objective_kernel<8><<<g, 128, 0, st>>>(X, Y, lam, B, n, beta, lambda_floor, objective); ++g_launches; break;
    }
    CK(cudaGetLastError());
    return LAD_OK;
}

extern "C" int lad_generate_f64(int32_t config, uint64_t seed, int64_t first, int64_t B, int32_t n, int32_t p,
                                double *X, double *Y, double *lam, double *beta_true, void *stream)
{
    if (config < 0 || config > 4 || config == 3) return fail(LAD_E_INVALID, "config must be 0, 1, 2 or 4");
    if (n < 1 || n > 64 || p < 1 || p > 8 || B < 0) return fail(LAD_E_INVALID, "bad shape");
    if (config == 1 && !lam) return fail(LAD_E_INVALID, "config 1 draws lambda per problem: lam must be non-null");
    if (B == 0) return LAD_OK;
    lad::GenArgs G{config, seed, first, B, n, p, X, Y, lam, beta_true};
    lad::gen_kernel<<<(unsigned)((B + 127) / 128), 128, 0, (cudaStream_t)stream>>>(G); ++g_launches;
    CK(cudaGetLastError());
    return LAD_OK;
}

extern "C" int lad_genspec_generate_f64(int64_t B, int32_t m, int32_t d, int32_t n_informative,
                                        const double *true_coefficients, double noise_sigma, double outlier_fraction,
                                        double outlier_scale, const uint64_t *seeds, double *X, double *Y,
                                        double *beta_true, void *stream)
{
    // GenSpec.__post_init__ (datagen.py:40-58)
    if (m < 1 || d < 1) return fail(LAD_E_INVALID, "need m >= 1 and d >= 1");
    if (n_informative < 1 || n_informative > d)
        return fail(LAD_E_INVALID, "n_informative must be in [1, %d], got %d", d, n_informative);
    if (!(noise_sigma >= 0)) return fail(LAD_E_INVALID, "noise_sigma must be >= 0");
    if (!(outlier_fraction >= 0 && outlier_fraction < 1)) return fail(LAD_E_INVALID, "outlier_fraction must be in [0, 1)");
    if (!(outlier_scale >= 1)) return fail(LAD_E_INVALID, "outlier_scale must be >= 1");
    if (d > 8 || m > 1024) return fail(LAD_E_UNSUPPORTED, "device GenSpec generation supports d <= 8, m <= 1024");
    if (B < 0 || (B > 0 && (!seeds || !X || !Y))) return fail(LAD_E_INVALID, "bad batch arguments");
    if (B == 0) return LAD_OK;
    lad::GenSpecArgs G;
    G.B = B;
    G.m = m;
    G.d = d;
    G.n_informative = n_informative;
    G.n_outliers = (int)std::floor(outlier_fraction * (double)m);  // math.floor(fraction * m)
    G.truth = true_coefficients;
    G.noise_sigma = noise_sigma;
    G.outlier_scale = outlier_scale;
    G.seeds = seeds;
    G.X = X;
    G.Y = Y;
    G.beta_true = beta_true;
    lad::genspec_kernel<<<(unsigned)((B + 63) / 64), 64, 0, (cudaStream_t)stream>>>(G); ++g_launches;
    CK(cudaGetLastError());
    return LAD_OK;
}

extern "C" int lad_subsets_f64(const double *X0, const double *Y0, int32_t n0, int32_t p, int32_t keep, int64_t first,
                               int64_t B, double *X, double *Y, void *stream)
{
    if (keep < 1 || keep > n0 || n0 > 64 || p < 1 || B < 0) return fail(LAD_E_INVALID, "bad subset shape");
    if (first < 0 || first + B > lad::binom(n0, keep)) return fail(LAD_E_INVALID, "subset index out of range");
    if (B == 0) return LAD_OK;
    lad::subsets_kernel<<<(unsigned)((B + 127) / 128), 128, 0, (cudaStream_t)stream>>>(X0, Y0, n0, p, keep, first, B,
                                                                                       X, Y); ++g_launches;
    CK(cudaGetLastError());
    return LAD_OK;
}

extern "C" int lad_axiswise_minimum_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n,
                                        int32_t p, const double *beta, const int32_t *skip, double tol,
                                        double lambda_floor, uint8_t *out, void *stream)
{
    if (B < 0 || n < 1 || p < 1) return fail(LAD_E_INVALID, "need B >= 0, n >= 1, p >= 1");
    if (n > 64 || p > 8) return fail(LAD_E_UNSUPPORTED, "n=%d p=%d beyond n<=64, p<=8", n, p);
    if (!(tol >= 0)) return fail(LAD_E_INVALID, "tol must be >= 0");
    if (!(lambda_floor > 0)) return fail(LAD_E_INVALID, "lambda_floor must be finite and > 0");
    if (B == 0) return LAD_OK;
    lad::CertArgs A{X, Y, lam, beta, skip, B, n, p, tol, lambda_floor, out};
    lad::axiswise_minimum_kernel<64, 8><<<(unsigned)((B + 127) / 128), 128, 0, (cudaStream_t)stream>>>(A); ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(LAD_E_CUDA, "certificate kernel: %s", cudaGetErrorString(e));
    return LAD_OK;
}

extern "C" int lad_lp_solve_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n, int32_t p,
                                int32_t max_pivots, int32_t pivot_rule, double feasibility_tolerance,
                                double lambda_floor, double *beta, double *objective, int32_t *pivots,
                                uint8_t *converged, uint8_t *status, double *x_full, int32_t *basis, double *trace,
                                int32_t trace_cap, void *stream)
{
    if (B < 0 || n < 1 || p < 1) return fail(LAD_E_INVALID, "need B >= 0, n >= 1, p >= 1");
    if (n > lad::LP_MMAX || p > lad::LP_DMAX) return fail(LAD_E_UNSUPPORTED, "n=%d p=%d beyond n<=46, p<=8", n, p);
    if (max_pivots < 0) return fail(LAD_E_INVALID, "max_pivots must be at least 1 (0 = default 50 * columns)");
    if (pivot_rule != LAD_PIVOT_DANTZIG_BLAND && pivot_rule != LAD_PIVOT_BLAND)
        return fail(LAD_E_INVALID, "unknown pivot rule %d", pivot_rule);
    if (!(lambda_floor > 0)) return fail(LAD_E_INVALID, "lambda_floor must be finite and > 0");
    if (B == 0) return LAD_OK;  // (empty outputs may be null)
    if (!beta || !objective || !pivots || !converged || !status) return fail(LAD_E_INVALID, "output pointers must be non-null");
    const int warp_doubles = lad::lp_warp_doubles(n, p);
    const size_t smem = (size_t)lad::LP_WARPS * warp_doubles * sizeof(double);
    CK(cudaFuncSetAttribute(lad::lp_simplex_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    lad::LpArgs A{X, Y, lam, B, n, p, max_pivots, pivot_rule == LAD_PIVOT_BLAND, feasibility_tolerance, lambda_floor,
                  beta, objective, x_full, pivots, basis, converged, status, trace, trace ? trace_cap : 0, warp_doubles};
    const unsigned grid = (unsigned)((B + lad::LP_WARPS - 1) / lad::LP_WARPS);
    lad::lp_simplex_kernel<<<grid, 32 * lad::LP_WARPS, smem, (cudaStream_t)stream>>>(A); ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(LAD_E_CUDA, "simplex kernel: %s", cudaGetErrorString(e));
    return LAD_OK;
}
