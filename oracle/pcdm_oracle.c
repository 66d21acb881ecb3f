/*
 * pcdm_oracle.c -- serial CPU ORACLE for synchronous PCDM1 on LASSO.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1212_0873_b200/) never links, imports or calls it,
 * and this file shares no code, header or constant generator with it.
 *
 * Plain, slow, obviously-correct: single thread, fp64 arithmetic on the fp32
 * inputs, no blocking/fusion/reordering beyond what the paper states.
 * Citations are PAPER.md:<line> (LaTeX source of arXiv 1212.0873) plus the
 * section / equation / algorithm label, and SURVEY.md section 8(c) readings
 * (O1..O8, R#n) where the paper is silent.
 *
 * Problem (eq:P, PAPER.md:42-46 with f = 1/2||Ax-b||^2, Omega = lambda||x||_1,
 * PAPER.md:1175):   F(x) = 1/2 ||Ax - b||^2 + lambda ||x||_1.
 * A is m x n, CSC: colptr int64[n+1], rowidx int32[nnz], val float[nnz].
 *
 * Parity status:
 *   or_omega, or_col_norms, or_beta, or_prox, or_run, or_objective,
 *   or_residual: pinned by tests/test_oracle_*.py (closed forms, brute force,
 *   paper-printed values, ESO identities, KKT).
 *   or_philox4x32_10: pinned by Random123 known-answer vectors.
 *   or_sample: law pinned (chi-square, moments, paper's q-values); the exact
 *   counter layout / ownership rule is a SURVEY 8(c) reading -> the specific
 *   slot ORDER is "parity unpinned" beyond cross-implementation agreement
 *   with the independent pure-Python twin (oracle/ref_sampler.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 counter-based generator (Salmon et al. 2011, Random123).     */
/* Used by the SAMPLE reading of SURVEY 8(c) (the paper gives only the law of */
/* S_k).  Multipliers and Weyl key increments are the       */
/* published Philox4x32 constants.                                            */
/* ------------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* One draw of the SAMPLE reading:
 *   key = (lo32(seed), hi32(seed)), counter = (slot j, k, round rho, tag),
 *   u = (out.y << 32) | out.x, Lemire map to [0,n): v = floor(u*n / 2^64),
 *   rejected iff (u*n mod 2^64) < (2^64 - n) mod n.
 * Returns 1 and sets *v if accepted, 0 if rejected. */
int or_draw(uint64_t seed, uint32_t k, uint32_t rho, uint32_t j, uint32_t tag,
            uint64_t n, uint64_t *v)
{
    uint32_t ctr[4] = { j, k, rho, tag };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t out[4];
    or_philox4x32_10(ctr, key, out);
    uint64_t u = ((uint64_t)out[1] << 32) | (uint64_t)out[0];
    unsigned __int128 prod = (unsigned __int128)u * (unsigned __int128)n;
    uint64_t lo = (uint64_t)prod;
    uint64_t threshold = (uint64_t)(0 - n) % n;
    if (lo < threshold) return 0;
    *v = (uint64_t)(prod >> 64);
    return 1;
}

/* O5: tau-nice sampling S_k (uniform over all tau-subsets
 * of [n]; alg:PCD1 step 3).  Rule (SURVEY 8(c) "SAMPLE"):
 * rounds rho = 0,1,...; pending slots, in ascending j, draw a value; a slot
 * owns its value iff the draw was accepted and the value is not already owned
 * (by an earlier round or by a lower slot of this round).  If 2*tau > n, run
 * the rule for n-tau slots with tag 2 and output [n] minus the owned set in
 * ascending order.
 * taken: caller scratch of n bytes, all zero on entry and on return (or NULL:
 * allocated here).  Returns 0 on success, -1 on bad arguments, -2 if the
 * round counter would overflow the (rho, j) code space (never in practice). */
int or_sample(uint64_t seed, int64_t k, int64_t tau, int64_t n, int32_t *slots,
              unsigned char *taken)
{
    if (n < 1 || tau < 1 || tau > n || k < 0 || k > 0xFFFFFFFFLL || n > 0x7FFFFFFFLL)
        return -1;
    int complement = (2 * tau > n);
    int64_t cnt = complement ? (n - tau) : tau;
    uint32_t tag = complement ? 2u : 1u;
    int own_taken = 0;
    if (!taken) {
        taken = (unsigned char *)calloc((size_t)n, 1);
        if (!taken) return -1;
        own_taken = 1;
    }
    int64_t *owned = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cnt > 0 ? cnt : 1));
    int64_t *pending = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cnt > 0 ? cnt : 1));
    int64_t npending = cnt;
    for (int64_t j = 0; j < cnt; ++j) { owned[j] = -1; pending[j] = j; }
    int rc = 0;
    for (uint64_t rho = 0; npending > 0; ++rho) {
        if ((rho + 1) * (uint64_t)cnt > 0x100000000ULL) { rc = -2; break; }
        int64_t still = 0;
        for (int64_t t = 0; t < npending; ++t) {
            int64_t j = pending[t];
            uint64_t v;
            int ok = or_draw(seed, (uint32_t)k, (uint32_t)rho, (uint32_t)j, tag, (uint64_t)n, &v);
            if (ok && !taken[v]) {
                taken[v] = 1;
                owned[j] = (int64_t)v;
            } else {
                pending[still++] = j;
            }
        }
        npending = still;
    }
    if (rc == 0) {
        if (!complement) {
            for (int64_t j = 0; j < cnt; ++j) slots[j] = (int32_t)owned[j];
        } else {
            int64_t t = 0;
            for (int64_t v = 0; v < n; ++v)
                if (!taken[v]) slots[t++] = (int32_t)v;
        }
    }
    for (int64_t j = 0; j < cnt; ++j)
        if (owned[j] >= 0) taken[owned[j]] = 0;
    free(owned);
    free(pending);
    if (own_taken) free(taken);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Other doubly uniform samplings.      */
/* Each returns tau slots; an idle slot (a processor that updates nothing) is  */
/* -1.  Readings (R16-R18) fix the concrete random stream.           */
/* ------------------------------------------------------------------------ */
enum { OR_NICE = 0, OR_INDEPENDENT = 1, OR_BINOMIAL = 2, OR_DU = 3 };

/* 64-bit word of counter (j, k, 0, tag) under key (lo32 seed, hi32 seed). */
static uint64_t or_word(uint64_t seed, uint32_t k, uint32_t j, uint32_t tag)
{
    uint32_t ctr[4] = { j, k, 0u, tag };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t out[4];
    or_philox4x32_10(ctr, key, out);
    return ((uint64_t)out[1] << 32) | (uint64_t)out[0];
}

/* floor(p * 2^64) for 0 <= p < 1; UINT64_MAX + "always" for p >= 1 (flag). */
static uint64_t or_threshold(double p, int *always)
{
    *always = 0;
    if (p >= 1.0) { *always = 1; return UINT64_MAX; }
    if (p <= 0.0) return 0;
    return (uint64_t)(p * 18446744073709551616.0); /* 2^64: exact scaling, then truncation */
}

/* tau-independent sampling: processor j = 0..tau-1 picks
 * the first accepted draw of counters (j, k, rho, tag 3), rho = 0,1,...,
 * independently of the others; "if two or more processors pick the same block,
 * all but one will be idle": the lowest j keeps it (reading R16). */
int or_sample_independent(uint64_t seed, int64_t k, int64_t tau, int64_t n, int32_t *slots)
{
    if (n < 1 || tau < 1 || tau > n || k < 0 || k > 0xFFFFFFFFLL || n > 0x7FFFFFFFLL) return -1;
    unsigned char *taken = (unsigned char *)calloc((size_t)n, 1);
    if (!taken) return -1;
    for (int64_t j = 0; j < tau; ++j) {
        uint64_t v = 0;
        uint32_t rho = 0;
        while (!or_draw(seed, (uint32_t)k, rho, (uint32_t)j, 3u, (uint64_t)n, &v)) ++rho;
        if (taken[v]) {
            slots[j] = -1;
        } else {
            taken[v] = 1;
            slots[j] = (int32_t)v;
        }
    }
    free(taken);
    return 0;
}

/* (tau, p_b)-binomial sampling, Case 2 of PAPER.md:452-455: a tau-nice set is
 * assigned to tau processors, processor j is available with probability p_b
 * independently (word of counter (j, k, 0, tag 4) < floor(p_b 2^64)); busy
 * processors are idle (reading R17). */
int or_sample_binomial(uint64_t seed, int64_t k, int64_t tau, int64_t n, double p_b, int32_t *slots)
{
    int rc = or_sample(seed, k, tau, n, slots, NULL);
    if (rc != 0) return rc;
    int always;
    uint64_t T = or_threshold(p_b, &always);
    for (int64_t j = 0; j < tau; ++j)
        if (!always && !(or_word(seed, (uint32_t)k, (uint32_t)j, 4u) < T)) slots[j] = -1;
    return 0;
}

/* Doubly uniform sampling with size law q[0..tau] (eq:p(S)):
 * |S| = K is the smallest K with u < floor(min(1, q_0 + ... + q_K) 2^64), u the
 * word of counter (0, k, 0, tag 5) (cumulative sums in fp64, left to right;
 * the last one counts as 1); S = the first K slots of the tau-nice slot array
 * (uniform over ordered tau-tuples, so its K-prefix is uniform over K-subsets;
 * needs 2 tau <= n: the complement path's sorted output has no such property)
 * (reading R18). */
int or_sample_du(uint64_t seed, int64_t k, int64_t tau, int64_t n, const double *q, int32_t *slots)
{
    if (2 * tau > n) return -1;
    int rc = or_sample(seed, k, tau, n, slots, NULL);
    if (rc != 0) return rc;
    uint64_t u = or_word(seed, (uint32_t)k, 0u, 5u);
    double cum = 0.0;
    int64_t K = tau;
    for (int64_t s = 0; s < tau; ++s) {
        cum += q[s];
        int always;
        uint64_t T = or_threshold(cum, &always);
        if (always || u < T) { K = s; break; }
    }
    for (int64_t j = K; j < tau; ++j) slots[j] = -1;
    return 0;
}

int or_sample_kind(int kind, uint64_t seed, int64_t k, int64_t tau, int64_t n, double p_b, const double *q,
                   int32_t *slots)
{
    switch (kind) {
    case OR_NICE: return or_sample(seed, k, tau, n, slots, NULL);
    case OR_INDEPENDENT: return or_sample_independent(seed, k, tau, n, slots);
    case OR_BINOMIAL: return or_sample_binomial(seed, k, tau, n, p_b, slots);
    case OR_DU: return or_sample_du(seed, k, tau, n, q, slots);
    default: return -1;
    }
}

/* First two moments of |S| (E|S|, E|S|^2) for each sampling:
 *   nice: tau, tau^2;
 *   independent: occupancy of n bins by tau balls, E|S| = n(1 - (1-1/n)^tau),
 *     E|S|^2 = E|S| + n(n-1)(1 - 2(1-1/n)^tau + (1-2/n)^tau)   (the law is the
 *     q_k of PAPER.md:440-444; tests pin these against that recursion);
 *   binomial: tau p_b and tau p_b (1 + tau p_b - p_b);
 *   DU: sum_k k q_k and sum_k k^2 q_k. */
int or_moments(int kind, int64_t tau, int64_t n, double p_b, const double *q, double *e1, double *e2)
{
    double t = (double)tau, nn = (double)n;
    switch (kind) {
    case OR_NICE: *e1 = t; *e2 = t * t; return 0;
    case OR_INDEPENDENT: {
        double a = pow(1.0 - 1.0 / nn, t);
        double b = (n >= 2) ? pow(1.0 - 2.0 / nn, t) : 0.0;
        *e1 = nn * (1.0 - a);
        *e2 = *e1 + nn * (nn - 1.0) * (1.0 - 2.0 * a + b);
        return 0;
    }
    case OR_BINOMIAL: *e1 = t * p_b; *e2 = t * p_b * (1.0 + t * p_b - p_b); return 0;
    case OR_DU: {
        double s1 = 0.0, s2 = 0.0;
        for (int64_t kk = 0; kk <= tau; ++kk) { s1 += (double)kk * q[kk]; s2 += (double)kk * (double)kk * q[kk]; }
        *e1 = s1; *e2 = s2;
        return 0;
    }
    default: return -1;
    }
}

/* ESO constant for a doubly uniform sampling (thm:ESO-DU, PAPER.md:955-960;
 * tbl:ESO PAPER.md:339,346):
 *   beta = 1 + (omega-1)(E|S|^2 / E|S| - 1) / max(1, n-1). */
double or_beta_du(int64_t omega, int64_t n, double e1, double e2)
{
    double denom = (double)(n - 1 > 1 ? n - 1 : 1);
    if (e1 <= 0.0) return 1.0;
    return 1.0 + (double)(omega - 1) * (e2 / e1 - 1.0) / denom;
}

/* O1: degree of partial separability for f = 1/2||Ax-b||^2 with unit blocks:
 * omega = max_j ||A_j||_0, the maximum number of (stored) entries in a row
 * (eq:omega PAPER.md:54; LASSO PAPER.md:303; reading R#3: count
 * stored entries). */
void or_row_counts(int64_t nnz, const int32_t *rowidx, int64_t *counts)
{
    for (int64_t p = 0; p < nnz; ++p) counts[rowidx[p]] += 1;
}

int64_t or_omega(int64_t m, int64_t nnz, const int32_t *rowidx)
{
    int64_t *counts = (int64_t *)calloc((size_t)m, sizeof(int64_t));
    or_row_counts(nnz, rowidx, counts);
    int64_t omega = 0;
    for (int64_t j = 0; j < m; ++j)
        if (counts[j] > omega) omega = counts[j];
    free(counts);
    return omega;
}

/* O2: block Lipschitz constants w = L, L_i = ||a_i||^2 (tbl:ESO
 * PAPER.md:344, w = L). */
void or_col_norms(int64_t n, const int64_t *colptr, const float *val, double *L)
{
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t p = colptr[i]; p < colptr[i + 1]; ++p)
            s += (double)val[p] * (double)val[p];
        L[i] = s;
    }
}

/* O3: ESO constant for the tau-nice sampling,
 * beta = 1 + (omega-1)(tau-1)/max(1,n-1)   (thm:ESO-nice, PAPER.md:875-878;
 * tbl:ESO PAPER.md:344; reading R#4 uses max(1,n-1)). */
double or_beta(int64_t omega, int64_t tau, int64_t n)
{
    double denom = (double)(n - 1 > 1 ? n - 1 : 1);
    return 1.0 + (double)(omega - 1) * (double)(tau - 1) / denom;
}

/* Block update for Omega_i = lambda|.|: the i-th block of h(x) (eq:h(x),
 * block form PAPER.md:214-216):
 *   h_i = argmin_t g t + (s/2) t^2 + lambda |x + t|,  s = beta * L_i.
 * Closed form: u = x - g/s, x+ = sign(u) max(|u| - lambda/s, 0), h = x+ - x.
 * Returns x+ (reading R#6: ties -> 0, x+ first then delta = x+ - x).
 * Empty column (s = 0; reading R#5): x+ = 0 if lambda > 0 else x. */
double or_prox(double x, double g, double s, double lambda)
{
    if (s == 0.0) return lambda > 0.0 ? 0.0 : x;
    double u = x - g / s;
    double mag = fabs(u) - lambda / s;
    if (mag <= 0.0) return 0.0;
    return u > 0.0 ? mag : -mag;
}

/* O4: residual r = Ax - b (implied by grad_i f = a_i^T (Ax - b)
 * with PAPER.md:303), in double, skipping x_i = 0 columns. */
void or_residual(int64_t m, int64_t n, const int64_t *colptr, const int32_t *rowidx,
                 const float *val, const float *b, const double *x, double *r)
{
    for (int64_t j = 0; j < m; ++j) r[j] = -(double)b[j];
    for (int64_t i = 0; i < n; ++i) {
        if (x[i] == 0.0) continue;
        for (int64_t p = colptr[i]; p < colptr[i + 1]; ++p)
            r[rowidx[p]] += (double)val[p] * x[i];
    }
}

/* F(x) = 1/2||Ax-b||^2 + lambda||x||_1 (eq:P PAPER.md:42 with PAPER.md:1175),
 * recomputed from scratch in double. */
double or_objective(int64_t m, int64_t n, const int64_t *colptr, const int32_t *rowidx,
                    const float *val, const float *b, double lambda, const double *x)
{
    double *r = (double *)malloc(sizeof(double) * (size_t)m);
    or_residual(m, n, colptr, rowidx, val, b, x, r);
    double f = 0.0;
    for (int64_t j = 0; j < m; ++j) f += r[j] * r[j];
    double l1 = 0.0;
    for (int64_t i = 0; i < n; ++i) l1 += fabs(x[i]);
    free(r);
    return 0.5 * f + lambda * l1;
}

/* Default residual-refresh period (reading R#8): R = ceil(2n / tau). */
int64_t or_refresh_period(int64_t n, int64_t tau, int64_t refresh_every)
{
    if (refresh_every < 0) return 0; /* off */
    if (refresh_every > 0) return refresh_every;
    return (2 * n + tau - 1) / tau;
}

static double now_seconds(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* Synchronous PCDM1 (alg:PCD1) for LASSO:
 *   for k = first_iter .. first_iter+iters-1:
 *     O5  S_k = SAMPLE(seed, k, tau, n)
 *     O6  read phase: for each i in S_k, g_i = a_i^T r_k (double, storage
 *         order), x_i+ = prox, delta_i = x_i+ - x_i   (all from snapshot r_k:
 *         "x_{k+1} <- x_k + (h(x_k))_[S_k]")
 *     O7  write phase, slots ascending: x_i <- x_i+, r += delta_i a_i
 *     O8  if (k-first_iter+1) % R == 0: r <- Ax - b from scratch
 * L: double[n] from or_col_norms; beta from or_beta (or any override).
 * x: double[n] in/out.  r_out (double[m]) / slots_out (int32[iters*tau]) /
 * loop_seconds may be NULL.  Returns 0, or <0 on bad args/sampler failure,
 * or 1 if a non-finite delta occurred (divergence). */
int or_run_kind(int64_t m, int64_t n, const int64_t *colptr, const int32_t *rowidx,
                const float *val, const float *b, double lambda, const double *L, double beta,
                double *x, int kind, int64_t tau, double p_b, const double *q, int64_t iters,
                uint64_t seed, int64_t first_iter, int64_t refresh_every, double *r_out,
                int32_t *slots_out, double *loop_seconds)
{
    if (m < 1 || n < 1 || tau < 1 || tau > n || iters < 0 || first_iter < 0) return -1;
    double *r = (double *)malloc(sizeof(double) * (size_t)m);
    int32_t *S = (int32_t *)malloc(sizeof(int32_t) * (size_t)tau);
    double *xplus = (double *)malloc(sizeof(double) * (size_t)tau);
    unsigned char *taken = (unsigned char *)calloc((size_t)n, 1);
    if (!r || !S || !xplus || !taken) return -1;
    int64_t R = or_refresh_period(n, tau, refresh_every);
    int rc = 0;

    or_residual(m, n, colptr, rowidx, val, b, x, r); /* O4 */

    double t0 = now_seconds();
    for (int64_t it = 0; it < iters && rc == 0; ++it) {
        int64_t k = first_iter + it;
        int src = (kind == OR_NICE) ? or_sample(seed, k, tau, n, S, taken) /* O5 */
                                    : or_sample_kind(kind, seed, k, tau, n, p_b, q, S);
        if (src != 0) { rc = -2; break; }
        if (slots_out) memcpy(slots_out + it * tau, S, sizeof(int32_t) * (size_t)tau);

        for (int64_t j = 0; j < tau; ++j) { /* O6: read phase */
            int64_t i = S[j];
            if (i < 0) continue; /* idle processor */
            double g = 0.0;
            for (int64_t p = colptr[i]; p < colptr[i + 1]; ++p)
                g += (double)val[p] * r[rowidx[p]];
            xplus[j] = or_prox(x[i], g, beta * L[i], lambda);
            if (!isfinite(xplus[j])) rc = 1;
        }
        for (int64_t j = 0; j < tau; ++j) { /* O7: write phase */
            int64_t i = S[j];
            if (i < 0) continue;
            double delta = xplus[j] - x[i];
            x[i] = xplus[j];
            for (int64_t p = colptr[i]; p < colptr[i + 1]; ++p)
                r[rowidx[p]] += (double)val[p] * delta;
        }
        if (R > 0 && (it + 1) % R == 0) /* O8 */
            or_residual(m, n, colptr, rowidx, val, b, x, r);
    }
    double t1 = now_seconds();
    if (loop_seconds) *loop_seconds = t1 - t0;
    if (r_out) memcpy(r_out, r, sizeof(double) * (size_t)m);
    free(r); free(S); free(xplus); free(taken);
    return rc;
}

/* Synchronous PCDM1 with the tau-nice sampling (the north_star path). */
int or_run(int64_t m, int64_t n, const int64_t *colptr, const int32_t *rowidx,
           const float *val, const float *b, double lambda, const double *L, double beta,
           double *x, int64_t tau, int64_t iters, uint64_t seed, int64_t first_iter,
           int64_t refresh_every, double *r_out, int32_t *slots_out, double *loop_seconds)
{
    return or_run_kind(m, n, colptr, rowidx, val, b, lambda, L, beta, x, OR_NICE, tau, 0.0, NULL, iters,
                       seed, first_iter, refresh_every, r_out, slots_out, loop_seconds);
}

/* ------------------------------------------------------------------------ */
/* L2-regularised logistic regression (Sec. 8.4,         */
/* PAPER.md:1381-1392; logistic loss of tbl:ML3 PAPER.md:68):                */
/*   F(x) = sum_j log(1 + exp(-y_j A_j^T x)) + lambda ||x||_2^2,             */
/* y_j in {+1,-1}.  Unit blocks, Omega_i(t) = lambda t^2 (eq:Psi_block_def   */
/* PAPER.md:155-159).  Reading R21: block Lipschitz constants    */
/* L_i = 1/4 ||a_i||^2 (the logistic loss has curvature <= 1/4), the update  */
/* minimises <grad_i f, t> + (beta L_i / 2) t^2 + lambda (x_i + t)^2 exactly: */
/*   t = -(grad_i f + 2 lambda x_i) / (beta L_i + 2 lambda),                 */
/* with grad_i f = -sum_j y_j a_ji sigma(-s_j), s_j = y_j A_j^T x (margins), */
/* sigma(z) = 1 / (1 + exp(-z)).                                            */
/* ------------------------------------------------------------------------ */
static double or_sigma(double z)
{
    return z >= 0.0 ? 1.0 / (1.0 + exp(-z)) : exp(z) / (1.0 + exp(z));
}

/* log(1 + exp(-s)) without overflow */
static double or_logloss(double s)
{
    return s >= 0.0 ? log1p(exp(-s)) : -s + log1p(exp(s));
}

/* margins s_j = y_j (A x)_j from scratch, in double */
void or_margins(int64_t m, int64_t n, const int64_t *colptr, const int32_t *rowidx, const float *val,
                const float *y, const double *x, double *s)
{
    for (int64_t j = 0; j < m; ++j) s[j] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (x[i] == 0.0) continue;
        for (int64_t p = colptr[i]; p < colptr[i + 1]; ++p)
            s[rowidx[p]] += (double)val[p] * x[i];
    }
    for (int64_t j = 0; j < m; ++j) s[j] *= (double)y[j];
}

double or_logistic_objective(int64_t m, int64_t n, const int64_t *colptr, const int32_t *rowidx, const float *val,
                             const float *y, double lambda, const double *x)
{
    double *s = (double *)malloc(sizeof(double) * (size_t)m);
    or_margins(m, n, colptr, rowidx, val, y, x, s);
    double f = 0.0;
    for (int64_t j = 0; j < m; ++j) f += or_logloss(s[j]);
    double q = 0.0;
    for (int64_t i = 0; i < n; ++i) q += x[i] * x[i];
    free(s);
    return f + lambda * q;
}

/* grad_i f at the margins s (for tests) */
double or_logistic_grad_i(const int64_t *colptr, const int32_t *rowidx, const float *val, const float *y,
                          const double *s, int64_t i)
{
    double g = 0.0;
    for (int64_t p = colptr[i]; p < colptr[i + 1]; ++p)
        g -= (double)y[rowidx[p]] * (double)val[p] * or_sigma(-s[rowidx[p]]);
    return g;
}

/* L_i = 1/4 ||a_i||^2 */
void or_logistic_L(int64_t n, const int64_t *colptr, const float *val, double *L)
{
    or_col_norms(n, colptr, val, L);
    for (int64_t i = 0; i < n; ++i) L[i] *= 0.25;
}

/* block update: x+ = x + t, t = -(g + 2 lambda x) / (s + 2 lambda), s = beta L_i.
 * s + 2 lambda = 0 (empty column, lambda = 0): x unchanged (reading R21). */
double or_logistic_step(double x, double g, double s, double lambda)
{
    double d = s + 2.0 * lambda;
    if (d == 0.0) return x;
    return x - (g + 2.0 * lambda * x) / d;
}

/* Synchronous PCDM1 for the logistic problem: the same O5-O8 structure as
 * or_run_kind with the margins s in place of r (O4: s = y .* (Ax); O6 reads
 * sigma(-s) of the snapshot; O7 adds y_j a_ji delta; O8 recomputes s). */
int or_logistic_run(int64_t m, int64_t n, const int64_t *colptr, const int32_t *rowidx, const float *val,
                    const float *y, double lambda, const double *L, double beta, double *x, int kind, int64_t tau,
                    double p_b, const double *q, int64_t iters, uint64_t seed, int64_t first_iter,
                    int64_t refresh_every, double *s_out, double *loop_seconds)
{
    if (m < 1 || n < 1 || tau < 1 || tau > n || iters < 0 || first_iter < 0) return -1;
    double *s = (double *)malloc(sizeof(double) * (size_t)m);
    int32_t *S = (int32_t *)malloc(sizeof(int32_t) * (size_t)tau);
    double *xplus = (double *)malloc(sizeof(double) * (size_t)tau);
    if (!s || !S || !xplus) return -1;
    int64_t R = or_refresh_period(n, tau, refresh_every);
    int rc = 0;
    or_margins(m, n, colptr, rowidx, val, y, x, s);
    double t0 = now_seconds();
    for (int64_t it = 0; it < iters && rc == 0; ++it) {
        int64_t k = first_iter + it;
        if (or_sample_kind(kind, seed, k, tau, n, p_b, q, S) != 0) { rc = -2; break; }
        for (int64_t j = 0; j < tau; ++j) {
            int64_t i = S[j];
            if (i < 0) continue;
            double g = or_logistic_grad_i(colptr, rowidx, val, y, s, i);
            xplus[j] = or_logistic_step(x[i], g, beta * L[i], lambda);
            if (!isfinite(xplus[j])) rc = 1;
        }
        for (int64_t j = 0; j < tau; ++j) {
            int64_t i = S[j];
            if (i < 0) continue;
            double delta = xplus[j] - x[i];
            x[i] = xplus[j];
            for (int64_t p = colptr[i]; p < colptr[i + 1]; ++p)
                s[rowidx[p]] += (double)y[rowidx[p]] * (double)val[p] * delta;
        }
        if (R > 0 && (it + 1) % R == 0)
            or_margins(m, n, colptr, rowidx, val, y, x, s);
    }
    double t1 = now_seconds();
    if (loop_seconds) *loop_seconds = t1 - t0;
    if (s_out) memcpy(s_out, s, sizeof(double) * (size_t)m);
    free(s); free(S); free(xplus);
    return rc;
}
