/*
 * pcdm.h -- C ABI of libpcdm.so, the B200 (sm_100a) hot path of synchronous
 * PCDM1 (parallel coordinate descent, arXiv 1212.0873) on LASSO:
 *
 *     minimise  F(x) = 1/2 ||A x - b||^2 + lambda ||x||_1          (eq:P, PAPER.md:42-46;
 *                                                                     LASSO instance PAPER.md:1175)
 *
 * One PCDM1 iteration (alg:PCD1):
 *   draw a tau-nice sampling S_k (tau distinct coordinates, uniformly at random,
 *   PAPER.md:436-438); for each i in S_k, from the SAME snapshot r_k = A x_k - b:
 *     g_i = a_i^T r_k                                  (grad_i f)
 *     x_i+ = argmin_t g_i t + (beta L_i / 2) t^2 + lambda |x_i + t|  (+ x_i)
 *                                                      (eq:h(x) block form PAPER.md:214-216)
 *   with w = L, L_i = ||a_i||^2 and the tau-nice ESO constant
 *     beta = 1 + (omega - 1)(tau - 1) / max(1, n - 1)  (thm:ESO-nice PAPER.md:875-878),
 *     omega = max_j ||A_j||_0 (stored entries per row);
 *   then x_i <- x_i+ and r <- r + (x_i+ - x_i) a_i for all i in S_k.
 *
 * Conventions for every entry point
 *   - Array pointers may be HOST or DEVICE memory (CUDA device/managed pointers
 *     are used in place; host pointers, pinned or pageable, are copied).  The
 *     library detects which with cudaPointerGetAttributes.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All device work
 *     is enqueued on it.
 *   - Errors: every call returns a pcdm_status; nothing is thrown across the ABI.
 *     pcdm_last_error() returns a thread-local message for the last failing call.
 *   - Handles are not thread-safe; distinct handles are independent.
 *   - Sizes: 1 <= m < 2^31 (int32 row indices), 1 <= n < 2^31, 1 <= nnz < 2^62.
 */
#ifndef PCDM_H
#define PCDM_H

#include <stdint.h>

#if defined(__GNUC__)
#define PCDM_API __attribute__((visibility("default")))
#else
#define PCDM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pcdm_problem pcdm_problem; /* opaque, owned by the library */

typedef enum {
    PCDM_OK = 0,
    PCDM_EINVAL = 1,    /* bad argument or malformed CSC / non-finite input   */
    PCDM_ENOMEM = 2,    /* device allocation failed                           */
    PCDM_ECUDA = 3,     /* any other CUDA runtime failure                     */
    PCDM_EDIVERGED = 4, /* a non-finite step occurred during pcdm_run          */
    PCDM_ESAMPLER = 5   /* sampler round counter overflow (never in practice) */
} pcdm_status;

/* Execution variants of the iteration loop (pcdm_run_ex).  All compute the same
 * synchronous PCDM1 iteration; they differ only in where the barrier between the
 * read phase (all g_i of S_k from r_k) and the write phase (r += delta_i a_i)
 * runs and where the data lives. */
typedef enum {
    PCDM_VARIANT_AUTO = 0, /* pick by problem size: SMEM when A fits shared memory;
                             BATCHED for LASSO when 4m > 2 x L2 and E|S| >= 2^17 and
                             E|S| >= 0.8 tau (handing the rest of the run to PACKED if
                             its steps turn out dense); PACKED
                             otherwise; GRID when no packed copy of A fits in memory */
    PCDM_VARIANT_GRID = 1, /* persistent cooperative grid, r in HBM/L2, grid barriers    */
    PCDM_VARIANT_SMEM = 2, /* one CTA, A, r, x, L resident in shared memory (small A)    */
    PCDM_VARIANT_BLOCK = 3, /* one CTA, data in HBM/L2, __syncthreads barriers           */
    PCDM_VARIANT_PACKED = 4, /* persistent grid on packed column blocks (one coalesced line
                               per column); one barrier per iteration with double-buffered
                               r.  Uniform layout (every column G lanes, G from the longest
                               column <= 62 entries) or, chosen at create when a column is
                               longer than 62 entries or would double every column's lanes,
                               the ragged layout: per sampled column 2..32 lanes, a warp
                               (63..1024 entries) or a CTA (longer) by its length, the
                               slots binned by class after the sampler.  The previous
                               iteration's steps are replayed into the second residual
                               buffer from registers (grid covers tau in one round) or
                               from CTA-local shared-memory lists */
    PCDM_VARIANT_BATCHED = 5, /* packed blocks; per chunk of iterations the partial
                               derivatives a_i^T r_0 of all sampled columns are computed at
                               once from the chunk's starting residual (gathers sorted by
                               row bin, r streamed through L2 once per chunk), plus
                               a_i^T (r_k - r_0) on the rows the chunk's steps touched.
                               Same iteration (alg:PCD1), different summation order of g_i.
                               For r much larger than L2 and sparse steps (LASSO).  Needs
                               the uniform packed layout */
} pcdm_variant;

/* Doubly uniform samplings (tbl:ESO PAPER.md:324-355).  A run
 * draws one realisation S_k per iteration; its slot array has tau entries, -1 for
 * an idle processor (one that updates nothing this iteration).
 *   NICE         tau-nice: S_k uniform over tau-subsets -- the
 *                north_star sampling; rule: DESIGN.md R1.
 *   INDEPENDENT  tau-independent: tau processors pick a block each, uniformly and
 *                independently; a block picked twice is updated once (lowest
 *                processor), the others idle (R16).
 *   BINOMIAL     (tau, p_b)-binomial, Case 2 of PAPER.md:452-455: a tau-nice
 *                assignment, each processor available with probability p_b
 *                (R17; exponent reading R13).
 *   DU           general doubly uniform with size law q[0..tau] (eq:p(S),
 *                PAPER.md:418-422): |S_k| = K ~ q, S_k = the first K slots of the
 *                tau-nice slot array (needs 2 tau <= n; R18).
 * beta for every kind: thm:ESO-DU,
 *   beta = 1 + (omega-1)(E|S|^2/E|S| - 1)/max(1,n-1)  (= thm:ESO-nice for NICE). */
typedef enum {
    PCDM_SAMPLING_NICE = 0,
    PCDM_SAMPLING_INDEPENDENT = 1,
    PCDM_SAMPLING_BINOMIAL = 2,
    PCDM_SAMPLING_DU = 3
} pcdm_sampling_kind;

typedef struct {
    int32_t kind;      /* pcdm_sampling_kind                                      */
    int32_t reserved;  /* 0                                                       */
    int64_t tau;       /* processors / slots per iteration, 1 <= tau <= n          */
    double p_b;        /* BINOMIAL: availability probability, 0 < p_b <= 1        */
    const double *q;   /* DU: host array q[0..tau], q_k = P(|S| = k), sums to 1
                          (|sum - 1| <= 1e-9); borrowed for the call              */
} pcdm_sampling;

typedef struct {
    int64_t iters;              /* iterations executed by the last run              */
    int64_t nonzero_deltas;     /* number of (i in S_k, k) with delta_i != 0        */
    int64_t sampler_max_rounds; /* largest sampler round index used + 1            */
    int64_t refreshes;          /* residual refreshes performed (excl. the initial) */
    int64_t kernel_launches;    /* kernels of this library launched by the run      */
    int32_t variant;            /* pcdm_variant actually used                       */
    int32_t grid_ctas;          /* CTAs of the iteration kernel                     */
    int32_t threads_per_cta;
    int32_t lanes_per_column;   /* threads cooperating on one sampled column (0: chosen
                                   per column, the ragged packed layout)              */
    int64_t chunk_iters;        /* iterations per iteration-kernel launch (max)     */
    int64_t iter_launches;      /* launches of the iteration kernel                 */
    double iter_kernel_ms;      /* summed device time of the iteration kernel       */
    double sampler_ms;          /* summed device time of the sampler passes         */
    double setup_ms;            /* residual init/refresh + copies (device time)     */
    int64_t hot_rows;           /* PACKED: rows served from the per-CTA shared-memory
                                   copy of r (rows stored >= max(64, 32 x mean) times,
                                   the 2048 most frequent; 0 for uniform rows, and 0
                                   when tau x (count of the hottest row) < 1024 n)    */
    int64_t host_h2d_bytes;     /* host x: bytes copied host -> device by the run      */
    int64_t host_d2h_bytes;     /* host x: bytes copied device -> host (the changed
                                   entries only, as (index, value) pairs, when they are
                                   fewer than n/2; else the whole x)                  */
    int64_t screen_misses;      /* BATCHED, screened step pass: iterations in which a
                                   flagged (not speculative) slot took a nonzero step  */
    int64_t screen_scans;       /* ... and the later-slot scans those steps cost        */
    int64_t screen_spec;        /* ... speculative items (nonzero step from g0 alone)    */
    int64_t screen_flagged;     /* ... flagged items (share a row or the column with an
                                   earlier speculative step of the chunk)               */
} pcdm_run_stats;

/* pcdm_create -- build a problem handle for LASSO with A (m x n, CSC), b, lambda.
 *   colptr int64[n+1], rowidx int32[nnz], val float32[nnz]: CSC of A, column i has
 *     entries p in [colptr[i], colptr[i+1]); rows strictly increasing per column.
 *   b float32[m]; lambda >= 0 finite.
 * The library copies (and may repack) everything into its own device memory; the
 * caller may free its arrays when the call returns (the call synchronises `stream`).
 * Computes L_i = ||a_i||^2 (fp64 accumulation, stored fp32) and
 * omega = max row count.
 * Errors: EINVAL for m,n,nnz < 1, colptr[0] != 0, colptr[n] != nnz, decreasing
 * colptr, row index out of [0,m) or not strictly increasing within a column,
 * non-finite val or b, lambda < 0 or non-finite, NULL pointers. */
PCDM_API pcdm_status pcdm_create(int64_t m, int64_t n, int64_t nnz, const int64_t *colptr,
                        const int32_t *rowidx, const float *val, const float *b, double lambda,
                        void *stream, pcdm_problem **out);

/* pcdm_create_logistic -- the L2-regularised logistic regression problem of Sec. 8.4
 * (logistic loss of tbl:ML3 PAPER.md:68):
 *
 *     minimise  F(x) = sum_j log(1 + exp(-y_j A_j^T x)) + lambda ||x||_2^2,
 *
 * rows of A = examples, columns = features, labels y float32[m] in {+1, -1}.
 * Same CSC arguments, ownership and errors as pcdm_create (EINVAL also for a label
 * other than +-1).  The library stores A~ = diag(y) A; the maintained vector r is the
 * margin s = A~ x; L_i = ||a_i||^2 / 4; omega as for LASSO; the block step minimises
 * grad_i f t + (beta L_i / 2) t^2 + lambda (x_i + t)^2 exactly (R21).
 * pcdm_run / pcdm_run_ex / pcdm_run_sampling / pcdm_objective / pcdm_residual
 * (returns s) / pcdm_col_norms (returns L) work on the handle; pcdm_run_async does
 * not (EINVAL). */
PCDM_API pcdm_status pcdm_create_logistic(int64_t m, int64_t n, int64_t nnz, const int64_t *colptr,
                                 const int32_t *rowidx, const float *val, const float *y, double lambda,
                                 void *stream, pcdm_problem **out);

/* Frees every device buffer of the handle (NULL is a no-op). */
PCDM_API void pcdm_destroy(pcdm_problem *p);

/* Thread-local message describing the most recent failure (never NULL). */
PCDM_API const char *pcdm_last_error(void);

/* Degree of partial separability omega (host value cached at create). */
PCDM_API pcdm_status pcdm_omega(const pcdm_problem *p, int64_t *omega);

/* beta = 1 + (omega-1)(tau-1)/max(1,n-1) in fp64 (thm:ESO-nice). EINVAL if tau not in [1,n]. */
PCDM_API pcdm_status pcdm_beta(const pcdm_problem *p, int64_t tau, double *beta);

/* pcdm_run -- `iters` synchronous PCDM1 iterations k = 0..iters-1 with the
 * tau-nice sampling keyed by `seed`, starting from x (float32[n], in/out).
 * Equivalent to pcdm_run_ex(p, x, tau, iters, seed, 0, 0, 0.0, PCDM_VARIANT_AUTO, stream).
 * x is read at the start and written at the end (device x is updated in place).
 * Synchronises `stream` once after the initial residual and once at the end.
 * Errors: EINVAL for tau not in [1,n], iters < 0, non-finite x; EDIVERGED if a
 * step was non-finite (x then holds the diverged iterate). */
PCDM_API pcdm_status pcdm_run(pcdm_problem *p, float *x, int64_t tau, int64_t iters, uint64_t seed,
                     void *stream);

/* pcdm_run_ex -- pcdm_run with the knobs the tests and the bench need:
 *   first_iter    iteration index of the first step (resume: the sampler stream
 *                 continues bit-exactly); first_iter + iters <= 2^32.
 *   refresh_every residual r = Ax - b recomputed from scratch after every R-th
 *                 iteration (fp64 accumulation): 0 = default R = ceil(2n/tau),
 *                 -1 = never, > 0 = that R.  (reading R#8.)
 *   beta_override > 0 replaces the formula's beta (ESO inflation).
 *   variant       pcdm_variant. */
PCDM_API pcdm_status pcdm_run_ex(pcdm_problem *p, float *x, int64_t tau, int64_t iters, uint64_t seed,
                        int64_t first_iter, int64_t refresh_every, double beta_override,
                        int32_t variant, void *stream);

/* pcdm_run_ex with any doubly uniform sampling (pcdm_sampling above).  Same
 * arguments and errors as pcdm_run_ex, plus EINVAL for an invalid sampling (unknown
 * kind, tau not in [1,n], p_b not in (0,1], q NULL / negative / not summing to 1,
 * DU with 2 tau > n).  The default refresh period uses R = ceil(2n / tau). */
PCDM_API pcdm_status pcdm_run_sampling(pcdm_problem *p, float *x, const pcdm_sampling *sampling, int64_t iters,
                              uint64_t seed, int64_t first_iter, int64_t refresh_every, double beta_override,
                              int32_t variant, void *stream);

/* pcdm_run_async -- the asynchronous variant the paper's experiments ran
 * (SURVEY 8(f) NEXT-4), measured, not oracle-checked: every worker
 * (a group of lanes; pcdm_last_run_stats().grid_ctas x threads / lanes of them)
 * repeatedly picks a coordinate uniformly at random (update u = first_update ..
 * first_update+updates-1 picks i from Philox counter (u lo, u hi, rho, tag 6)) and
 * applies its soft-threshold step computed from whatever r holds at that moment;
 * x_i and r are updated with atomics, so r = Ax - b holds whatever the
 * interleaving (up to fp32 rounding) but the iterates are not deterministic.
 *   tau_beta      beta = 1 + (omega-1)(tau_beta-1)/max(1,n-1); 0 = the number of
 *                 concurrent workers (clamped to n)
 *   beta_override > 0 replaces that beta
 *   refresh_every r recomputed from scratch after every this many updates
 *                 (0 = 2n, -1 = never)
 * Needs the packed layout (max column length <= 62): EINVAL otherwise, or for
 * updates < 0, non-finite x.  EDIVERGED as pcdm_run. */
PCDM_API pcdm_status pcdm_run_async(pcdm_problem *p, float *x, int64_t updates, int64_t tau_beta,
                           double beta_override, int64_t refresh_every, uint64_t first_update, uint64_t seed,
                           void *stream);

/* beta of thm:ESO-DU for `sampling` on this problem (fp64, host). */
PCDM_API pcdm_status pcdm_beta_sampling(const pcdm_problem *p, const pcdm_sampling *sampling, double *beta);

/* F(x) = 1/2||Ax-b||^2 + lambda||x||_1, residual accumulated in fp64 from scratch,
 * sums in fp64 (eq:P). x float32[n] host or device. Synchronises `stream`. */
PCDM_API pcdm_status pcdm_objective(pcdm_problem *p, const float *x, double *F, void *stream);

/* Statistics of the most recent pcdm_run / pcdm_run_ex on this handle. */
PCDM_API pcdm_status pcdm_last_run_stats(const pcdm_problem *p, pcdm_run_stats *stats);

/* ---- test and measurement hooks (not the hot path) ---------------------- */

/* Slot arrays of S_k for k = first_iter .. first_iter+count-1 (int32[count*tau],
 * row-major by k), exactly as pcdm_run draws them.  1 <= tau <= n < 2^31. */
PCDM_API pcdm_status pcdm_sample(int64_t n, int64_t tau, uint64_t seed, int64_t first_iter, int64_t count,
                        int32_t *slots, void *stream);

/* pcdm_sample for any sampling: slot arrays int32[count*tau], -1 = idle slot. */
PCDM_API pcdm_status pcdm_sample_sampling(int64_t n, const pcdm_sampling *sampling, uint64_t seed, int64_t first_iter,
                                 int64_t count, int32_t *slots, void *stream);

/* L_i = ||a_i||^2 as stored by the library (float32[n]). */
PCDM_API pcdm_status pcdm_col_norms(const pcdm_problem *p, float *L, void *stream);

/* Row histogram counts[j] = #stored entries in row j (int32[m]); omega = max. */
PCDM_API pcdm_status pcdm_row_counts(const pcdm_problem *p, int32_t *counts, void *stream);

/* The maintained residual r (float32[m]) as left by the last run. */
PCDM_API pcdm_status pcdm_residual(const pcdm_problem *p, float *r, void *stream);

/* Philox4x32-10 of the library's device generator on `count` (ctr, key) pairs:
 * ctr uint32[4*count], key uint32[2*count] -> out uint32[4*count]. */
PCDM_API pcdm_status pcdm_philox(int64_t count, const uint32_t *ctr, const uint32_t *key, uint32_t *out,
                        void *stream);

/* Compares the library's device Philox with cuRAND's curand_Philox4x32_10 on
 * `count` pseudo-random (ctr, key) pairs derived from `seed`; *mismatches = number
 * of differing outputs. */
PCDM_API pcdm_status pcdm_philox_check_curand(int64_t count, uint64_t seed, int64_t *mismatches,
                                     void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PCDM_H */
