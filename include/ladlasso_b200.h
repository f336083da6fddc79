/*
 * ladlasso_b200.h -- C ABI of the B200-native batched LAD-LASSO solver.
 *
 * The reference (arxiv/paper_2510_15649, /root/reference/pkg/src/ladlasso) is
 * a pure-Python package with no FFI; its drop-in boundary is the Python
 * function API.  Each entry point below replaces one reference function,
 * batched over B independent problems (B, n, p) and cited file:line:
 *
 *   lad_locus_solve_f64     <- locus.solve_locus(spec, cfg)        locus.py:300-409
 *   lad_locus_solve_host_f64   same, host buffers (H2D + solve + D2H inside)
 *   lad_locus_solve_f32 / _host_f32 / lad_ccd_descend_f32: the fp32 mode
 *                              (BASELINE config 4 "fp64 and fp32"), see below
 *   lad_ccd_descend_f64     <- ccd.ccd_descend(spec, start, cfg)   ccd.py:126-206
 *   lad_brute_solve_f64     <- brute.solve_brute(spec, ...)        brute.py:106-145
 *   lad_objective_f64       <- model.evaluate_objective(spec, b)   model.py:151-154
 *   lad_axiswise_minimum_f64 <- ccd.is_axiswise_minimum(spec, b)   ccd.py:214-237
 *   lad_lp_solve_f64        <- lp.solve_lp(spec, SimplexConfig)    lp.py:106-215
 *   lad_generate_f64        <- (no reference counterpart) device-side generation
 *                              of the BASELINE.json config problems
 *
 * Conventions: device pointers unless the name says _host; calls are
 * asynchronous on `stream` (a cudaStream_t passed as void*, NULL = legacy
 * default stream); return 0 on success or a negative LAD_E_* code, with the
 * message available from lad_last_error() (thread-local).  Per-problem failures
 * never abort a batch; they are reported in `status`:
 *   0 ok, 1 unbounded direction (UnboundedDirectionError, linesearch.py:266),
 *   2 invalid input (InvalidInputError: non-finite data, lambda < 0, bad bracket),
 *   3 scratch capacity exceeded (the search recorded more curve points than
 *     prm->seen_capacity allows; re-run the problem with a larger capacity --
 *     the Python API does this automatically).
 * Non-convergence is not an error (converged = 0), as in the reference.
 */
#ifndef LADLASSO_B200_H
#define LADLASSO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAD_OK 0
#define LAD_E_INVALID (-1)     /* bad shape / argument (InvalidInputError) */
#define LAD_E_TOO_LARGE (-2)   /* brute caps exceeded (ProblemTooLargeError, brute.py:66-81) */
#define LAD_E_CUDA (-3)        /* CUDA runtime failure */
#define LAD_E_UNSUPPORTED (-4) /* p > 8, or n > 1023 (fp32 mode: n > 31; simplex: n > 46) */

#define LAD_OUTER_TERNARY 0
#define LAD_OUTER_QUADRATURE 1

/* LocusConfig + CcdConfig + ProblemSpec.lambda_floor (locus.py:52-58, ccd.py:55-59, model.py:27). */
typedef struct lad_locus_params {
    int32_t outer_axis;           /* -1 = None: scan every axis in influence order */
    int32_t outer_search;         /* LAD_OUTER_TERNARY | LAD_OUTER_QUADRATURE */
    double outer_tolerance;       /* 1e-9 */
    int32_t outer_probes;         /* 8 (quadrature) */
    int32_t outer_max_iterations; /* 200 */
    int32_t has_bracket;          /* initial_bracket given? */
    double bracket_lo, bracket_hi;
    double inner_sweep_tol;       /* 1e-10 */
    int32_t inner_max_sweeps;     /* 500 */
    double lambda_floor;          /* 1e-9 */
    int32_t seen_capacity;        /* curve points one evaluator keeps for the nearest-point warm start
                                     (locus.py:188-191): 0 = automatic (bounded by the outer tolerance,
                                     with slack); a problem that needs more ends with status 3 */
} lad_locus_params;

/* Per-problem outputs (SolveResult fields, model.py:113-133, plus work counters). */
typedef struct lad_locus_out {
    double *beta;             /* (B, p) */
    double *objective;        /* (B,) fresh evaluate_objective(beta) */
    int32_t *iterations;      /* locus: outer rounds; descent: sweeps */
    int32_t *objective_evals; /* locus: curve evaluations; descent: coordinate steps */
    uint8_t *converged;       /* (B,) */
    uint8_t *status;          /* (B,) see above */
    int32_t *descents;        /* (B,) ccd_descend calls (may be NULL) */
    int64_t *steps;           /* (B,) exact coordinate steps (may be NULL) */
} lad_locus_out;

#define LAD_KERNEL_AUTO 0   /* warp-per-problem for n <= 31, thread-per-problem for (n,p) = (10,2),
                               block-per-problem for 32 <= n <= 1023 */
#define LAD_KERNEL_THREAD 1 /* one thread per problem (n <= 32) */
#define LAD_KERNEL_WARP 2   /* one warp per problem, lane = row (n <= 31; larger n: block per problem) */

int lad_version(void);
const char *lad_last_error(void);
/* number of kernels this library has launched so far (process-wide) */
long long lad_kernel_launches(void);
/* process-wide choice of the locus kernel mapping (both are bit-identical) */
int lad_set_kernel_policy(int32_t policy);
/* small batches (fewer problems than resident warps): run the independent
 * per-axis searches of each problem as separate work items, then combine them
 * in influence order (bit-identical).  0 = off, 1 = small batches only
 * (default), 2 = every batch. */
int lad_set_axis_parallel(int32_t enable);
/* fills the defaults of LocusConfig()/CcdConfig() */
void lad_default_params(lad_locus_params *prm);

/* Batched solve_locus.  X (Bd, n, p), Y (Bd, n); lam (B,) raw lambdas;
 * data_index (B,) maps problem -> dataset row (NULL = identity, then Bd == B).
 * An index outside [0, Bd) marks that problem invalid (status 2); the call
 * never synchronizes the stream. */
int lad_locus_solve_f64(const double *X, const double *Y, const double *lam, const int64_t *data_index, int64_t Bd,
                        int64_t B, int32_t n, int32_t p, const lad_locus_params *prm, const lad_locus_out *out,
                        void *stream);

/* Same with HOST pointers for inputs and outputs (pinned or pageable); the
 * host<->device copies run inside the call on `stream`, which is synchronized
 * before returning.  out fields are host pointers.  X (Bd, n, p), Y (Bd, n);
 * data_index (B,) host array or NULL (then Bd == B). */
int lad_locus_solve_host_f64(const double *X, const double *Y, const double *lam, const int64_t *data_index,
                             int64_t Bd, int64_t B, int32_t n, int32_t p, const lad_locus_params *prm,
                             const lad_locus_out *out, void *stream);

/* solve_locus with a per-problem LocusConfig.initial_bracket (locus.py:56, consumed at :227 and
 * :364-365): brackets (B, 2) = (lo, hi) per problem (device pointer; the _host variant takes host
 * pointers like lad_locus_solve_host_f64).  A bracket that is not finite with lo < hi marks its
 * problem invalid (status 2), as Bracket() raises InvalidInputError (linesearch.py:85-89).
 * prm->has_bracket is ignored.  Used by the warm-started lambda path (bench.py --warm). */
int lad_locus_solve_bracketed_f64(const double *X, const double *Y, const double *lam, const int64_t *data_index,
                                  int64_t Bd, int64_t B, int32_t n, int32_t p, const double *brackets,
                                  const lad_locus_params *prm, const lad_locus_out *out, void *stream);
int lad_locus_solve_bracketed_host_f64(const double *X, const double *Y, const double *lam,
                                       const int64_t *data_index, int64_t Bd, int64_t B, int32_t n, int32_t p,
                                       const double *brackets, const lad_locus_params *prm,
                                       const lad_locus_out *out, void *stream);

/* Batched ccd_descend from `start` (B, p); frozen (B,) axis or -1 (NULL = none). */
int lad_ccd_descend_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n, int32_t p,
                        const double *start, const int32_t *frozen, double sweep_tolerance, int32_t max_sweeps,
                        double lambda_floor, const lad_locus_out *out, void *stream);

/* Batched solve_brute: exhaustive vertex evaluation (the check).  vertices (B,)
 * = nonsingular vertices evaluated.  Returns LAD_E_TOO_LARGE when p >
 * max_variables or C(n+p, p) > max_candidates (whole batch, like the reference). */
int lad_brute_solve_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n, int32_t p,
                        int32_t max_variables, int64_t max_candidates, double lambda_floor, double *beta,
                        double *objective, int64_t *vertices, void *stream);

/* fp32 mode.  The reference has no binary32 path (model.py:33 casts every
 * input to float64), so this mode is defined by this library: X, Y, lambda are
 * binary32 and every coordinate-descent operation (residuals, breakpoints, the
 * weighted median, v_new, objectives) runs in binary32 in the same order as
 * the fp64 path, while the outer search (brackets, probe positions, warm
 * starts, agreement and refine rules) stays binary64; a probe position or
 * warm start is rounded to binary32 when its descent starts.  Outputs are
 * binary64 (exact widenings).  Parity: bit-exact against the oracle compiled
 * for binary32 (oracle/orc_descent.inc); distance to the fp64 reference is a
 * reported statistic, not a guarantee.  n <= 31, p <= 8 (warp kernel). */
int lad_locus_solve_f32(const float *X, const float *Y, const float *lam, const int64_t *data_index, int64_t Bd,
                        int64_t B, int32_t n, int32_t p, const lad_locus_params *prm, const lad_locus_out *out,
                        void *stream);
int lad_locus_solve_host_f32(const float *X, const float *Y, const float *lam, const int64_t *data_index,
                             int64_t Bd, int64_t B, int32_t n, int32_t p, const lad_locus_params *prm,
                             const lad_locus_out *out, void *stream);
int lad_ccd_descend_f32(const float *X, const float *Y, const float *lam, int64_t B, int32_t n, int32_t p,
                        const double *start, const int32_t *frozen, double sweep_tolerance, int32_t max_sweeps,
                        double lambda_floor, const lad_locus_out *out, void *stream);

/* Roofline denominators: measured dense FP64 / FP32 FMA throughput of the
 * current device (TFLOP/s, 2 flops per FMA), timed with CUDA events on `stream`. */
int lad_fp64_peak_tflops(double *tflops, void *stream);
int lad_fp32_peak_tflops(double *tflops, void *stream);

/* Batched ccd.is_axiswise_minimum (ccd.py:214-237): out[i] = 1 iff no
 * axis-parallel move from beta (B, p) descends, except along skip[i] (-1 or
 * NULL = none); 0 otherwise; 2 for non-finite inputs.  tol as the reference
 * (1e-9, relative to max(1, |b_j|)). */
int lad_axiswise_minimum_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n, int32_t p,
                             const double *beta, const int32_t *skip, double tol, double lambda_floor, uint8_t *out,
                             void *stream);

/* Batched lp.solve_lp (lp.py:106-215): dense tableau simplex on the standard
 * form (bp, bn, rp, rn) from the sign-split residual basis.  pivot_rule:
 * LAD_PIVOT_DANTZIG_BLAND (Dantzig, permanent switch to Bland after n
 * degenerate pivots; default) or LAD_PIVOT_BLAND; max_pivots 0 = 50 * (2p+2n)
 * columns.  Outputs: beta (B, p), objective = evaluate_objective(beta), pivots,
 * converged; status 0 ok, 1 unbounded direction (SimplexError in
 * simplex_minimize), 2 invalid input, 3 the LP optimum does not reproduce the
 * objective within 1e-9 (SimplexError in simplex_solve).
 * x_full (B, 2p+2n), basis (B, n) and trace (B, trace_cap: the LP objective
 * after 0, 1, ... pivots, SimplexSolution.objective_trace) are optional (NULL). */
#define LAD_PIVOT_DANTZIG_BLAND 0
#define LAD_PIVOT_BLAND 1
int lad_lp_solve_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n, int32_t p,
                     int32_t max_pivots, int32_t pivot_rule, double feasibility_tolerance, double lambda_floor,
                     double *beta, double *objective, int32_t *pivots, uint8_t *converged, uint8_t *status,
                     double *x_full, int32_t *basis, double *trace, int32_t trace_cap, void *stream);

/* evaluate_objective for (B, p) coefficient vectors. */
int lad_objective_f64(const double *X, const double *Y, const double *lam, int64_t B, int32_t n, int32_t p,
                      const double *beta, double lambda_floor, double *objective, void *stream);

/* Batched datagen.generate(GenSpec) (datagen.py:63-80, rng.py:25-72) on the device: B
 * problems of one shape (m, d), problem i seeded with seeds[i] (the other GenSpec fields
 * shared).  true_coefficients (d,) or NULL (U[1,10] on the first n_informative axes).
 * Outputs X (B, m, d), Y (B, m), beta_true (B, d) or NULL; device pointers.  The
 * transcendentals are double-double and rounded once (see lad_genspec.cuh); equality with
 * the host generator is measured in tests/test_gpu_genspec.py (2 ulp per normal draw).
 * d <= 8, m <= 1024 (LAD_E_UNSUPPORTED beyond). */
int lad_genspec_generate_f64(int64_t B, int32_t m, int32_t d, int32_t n_informative,
                             const double *true_coefficients, double noise_sigma, double outlier_fraction,
                             double outlier_scale, const uint64_t *seeds, double *X, double *Y, double *beta_true,
                             void *stream);

/* Device-side problem generation for the BASELINE.json configs:
 *   config 0/2: X~N(0,1), 2 nonzeros +-U[1,3], Laplace(0,0.5), 10% rows +-10
 *   config 1:   X~U(-1,1), beta~N(0,1), Laplace(0,0.3), lambda~U(0.1,2)
 *   config 4:   X~t(3), 3 nonzeros +-U[1,3], Cauchy(0,0.2)
 * Problem i uses counter-based Philox keyed by (seed, first + i), so any shard
 * [first, first+B) is reproducible independently.  lam may be NULL except for config 1.
 * Every operation is a single IEEE operation with this library's own transcendental
 * polynomials (lad_gen.cuh), so oracle/gen_host.c reproduces the bytes on the CPU. */
int lad_generate_f64(int32_t config, uint64_t seed, int64_t first, int64_t B, int32_t n, int32_t p, double *X,
                     double *Y, double *lam, double *beta_true, void *stream);

/* Config 3: gather the k-th `keep`-row subset (lexicographic itertools.combinations
 * order) of one dataset (n0, p) for k in [first, first+B). */
int lad_subsets_f64(const double *X0, const double *Y0, int32_t n0, int32_t p, int32_t keep, int64_t first, int64_t B,
                    double *X, double *Y, void *stream);

/* Host -> device copy of `bytes` from a caller's host buffer, ordered on `stream`
 * (cudaMemcpyAsync on the raw pointer: DMA when the buffer is page-locked, driver
 * staging otherwise).  Used by the Python host-buffer paths of the batched calls
 * that have no _host entry point (brute force, simplex, descents, certificates). */
int lad_copy_h2d(void *dst, const void *src, size_t bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif
