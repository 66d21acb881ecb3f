// kernels_iter.cu -- the PCDM1 iteration loop (the hot path).
//
// One synchronous PCDM1 iteration (alg:PCD1) for LASSO:
//   phase A (read):  for every i in S_k, from the snapshot r_k:
//                      g_i = a_i^T r_k
//                      x_i+ = soft-threshold step           (eq:h(x) block form)
//                      delta_i = x_i+ - x_i ; x_i <- x_i+   (distinct i: race-free)
//                      delta_i != 0 -> append (i, delta_i) to this iteration's list
//   barrier          (no iteration-k scatter may reach an iteration-k gather)
//   phase B (write): r += delta_i a_i for the listed columns (red.global.add.f32)
//   barrier          (iteration k+1 gathers see every iteration-k scatter)
// delta_i = 0 columns scatter nothing (r + 0 a_i = r exactly), so phase B only
// walks the compacted list of nonzero steps.
//
// Variants (same arithmetic, different barrier / data placement):
//   GRID  persistent cooperative grid over all SMs, r in HBM/L2, grid barriers.
//   BLOCK one CTA, data in HBM/L2, __syncthreads barriers.
//   SMEM  one CTA, colptr/rowidx/val/L/x/r copied into shared memory.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include <algorithm>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

using namespace pcdm;
using namespace pcdm_internal;

namespace {

constexpr int kGridThreads = 512;

template <int G>
__device__ __forceinline__ float group_sum(float v, unsigned gmask) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
    return v;
}

template <int G>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (G == 32) {
        return 0xffffffffu;
    } else {
        const unsigned lane = threadIdx.x & 31;
        return ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
    }
}

// G lanes per sampled column, U entries per lane in flight.
template <int G, int U, bool SINGLE, bool LOGISTIC>
__global__ void __launch_bounds__(kGridThreads) pcdm_iter_kernel(IterParams P) {
    const int lane_g = threadIdx.x & (G - 1);
    const unsigned gmask = group_mask<G>();
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
    unsigned bar_target = 0;
    const float beta = P.beta, lam = P.lambda;
    const int64_t tau = P.tau;

    for (int64_t it = 0; it < P.iters; ++it) {
        const int par = (int)(it & 1);
        const int* S = P.slots + it * tau;
        if (blockIdx.x == 0 && threadIdx.x == 0) P.nz_count[par ^ 1] = 0;

        // ---------------- phase A: gathers from the snapshot r_k
        for (int64_t j = gid; j < tau; j += ngroups) {
            const int i = ld_stream_s32(S + j);
            if (i < 0) continue;  // idle processor (non-nice samplings)
            const long long s = ld_stream_s64((const long long*)P.colptr + i);
            const long long e = ld_stream_s64((const long long*)P.colptr + i + 1);
            float acc = 0.0f;
            for (long long base = s; base < e; base += (long long)U * G) {
                int rr[U];
                float vv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const long long q = base + (long long)u * G + lane_g;
                    rr[u] = q < e ? ld_stream_s32(P.rowidx + q) : -1;
                    vv[u] = q < e ? ld_stream_f32(P.val + q) : 0.0f;
                }
                float gv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) gv[u] = rr[u] >= 0 ? grad_weight<LOGISTIC>(ld_l2_f32(P.r + rr[u])) : 0.0f;
#pragma unroll
                for (int u = 0; u < U; ++u) acc = fmaf(vv[u], gv[u], acc);
            }
            acc = group_sum<G>(acc, gmask);
            if (lane_g == 0) {
                const float Li = ld_stream_f32(P.L + i);
                const float xi = ld_l2_f32(P.x + i);
                const float xp = block_step<LOGISTIC>(xi, acc, beta * Li, lam);
                const float d = xp - xi;
                if (d != 0.0f) {
                    if (!isfinite(xp)) atomicOr(P.flags, FLAG_DIVERGED);
                    P.x[i] = xp;
                    const int pos = atomicAdd(P.nz_count + par, 1);
                    P.nz_idx[par * tau + pos] = i;
                    P.nz_delta[par * tau + pos] = d;
                }
            }
        }
        if (SINGLE) __syncthreads();
        else grid_barrier(P.barrier, bar_target);

        // ---------------- phase B: r += delta_i a_i for delta_i != 0
        const int cnt = ld_l2_s32(P.nz_count + par);
        for (int64_t t = gid; t < cnt; t += ngroups) {
            const int i = ld_l2_s32(P.nz_idx + par * tau + t);
            const float d = ld_l2_f32(P.nz_delta + par * tau + t);
            const long long s = ld_stream_s64((const long long*)P.colptr + i);
            const long long e = ld_stream_s64((const long long*)P.colptr + i + 1);
            for (long long q = s + lane_g; q < e; q += G)
                red_add_f32(P.r + ld_stream_s32(P.rowidx + q), ld_stream_f32(P.val + q) * d);
        }
        if (blockIdx.x == 0 && threadIdx.x == 0 && cnt) atomicAdd(P.nz_total, (unsigned long long)cnt);
        if (SINGLE) __syncthreads();
        else grid_barrier(P.barrier, bar_target);
    }
}

// ---------------------------------------------------------------- SMEM variant
// Everything of a small problem lives in shared memory of one CTA: colptr as
// int32 offsets, (row, val), L, x, r; lists of nonzero steps too.
constexpr int kSmemThreads = 1024;

template <int G, bool LOGISTIC>
__global__ void __launch_bounds__(kSmemThreads) pcdm_smem_kernel(IterParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = (int)P.m, n = (int)P.n;
    const int nnz = (int)P.colptr[n];
    const int tau = (int)P.tau;
    int* s_col = (int*)smem_raw;                 // n+1
    int* s_row = s_col + (n + 1);                // nnz
    float* s_val = (float*)(s_row + nnz);        // nnz
    float* s_L = s_val + nnz;                    // n
    float* s_x = s_L + n;                        // n
    float* s_r = s_x + n;                        // m
    int* s_nzi = (int*)(s_r + m);                // tau
    float* s_nzd = (float*)(s_nzi + tau);        // tau
    double* s_r64 = (double*)(((uintptr_t)(s_nzd + tau) + 7) & ~(uintptr_t)7);  // m (refresh scratch)
    __shared__ int s_cnt2[2];  // step counter, double-buffered (no reset barrier)

    for (int t = threadIdx.x; t <= n; t += blockDim.x) s_col[t] = (int)P.colptr[t];
    for (int t = threadIdx.x; t < nnz; t += blockDim.x) {
        s_row[t] = P.rowidx[t];
        s_val[t] = P.val[t];
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        s_L[t] = P.L[t];
        s_x[t] = P.x[t];
    }
    for (int t = threadIdx.x; t < m; t += blockDim.x) s_r[t] = P.r[t];
    if (threadIdx.x < 2) s_cnt2[threadIdx.x] = 0;
    __syncthreads();

    const int lane_g = threadIdx.x & (G - 1);
    const unsigned gmask = group_mask<G>();
    const int gid = threadIdx.x / G;
    const int ngroups = blockDim.x / G;
    const float beta = P.beta, lam = P.lambda;
    unsigned long long nz_total = 0;

    // one slot per group (tiny: tau = 32): the next iteration's slot id is loaded at the
    // top of this one, off the iteration's critical path
    const bool one = tau <= ngroups;
    int i_next = one && gid < tau && P.iters > 0 ? P.slots[gid] : -1;
    for (int64_t it = 0; it < P.iters; ++it) {
        const int* S = P.slots + it * tau;
        int* s_cnt = s_cnt2 + (it & 1);
        const int i_cur = i_next;
        if (one && gid < tau && it + 1 < P.iters) i_next = __ldg(P.slots + (it + 1) * tau + gid);
        for (int j = gid; j < tau; j += ngroups) {
            const int i = one ? i_cur : S[j];
            if (i < 0) continue;  // idle processor
            const int s = s_col[i], e = s_col[i + 1];
            float acc = 0.0f;
            for (int base = s; base < e; base += G) {
                const int q = base + lane_g;
                if (q < e) acc = fmaf(s_val[q], grad_weight<LOGISTIC>(s_r[s_row[q]]), acc);
            }
            acc = group_sum<G>(acc, gmask);
            if (lane_g == 0) {
                const float xi = s_x[i];
                const float xp = block_step<LOGISTIC>(xi, acc, beta * s_L[i], lam);
                const float d = xp - xi;
                if (d != 0.0f) {
                    if (!isfinite(xp)) atomicOr(P.flags, FLAG_DIVERGED);
                    s_x[i] = xp;
                    const int pos = atomicAdd(s_cnt, 1);
                    s_nzi[pos] = i;
                    s_nzd[pos] = d;
                }
            }
        }
        __syncthreads();
        const int cnt = *s_cnt;
        for (int t = gid; t < cnt; t += ngroups) {
            const int i = s_nzi[t];
            const float d = s_nzd[t];
            for (int q = s_col[i] + lane_g; q < s_col[i + 1]; q += G) atomicAdd(s_r + s_row[q], s_val[q] * d);
        }
        nz_total += (unsigned long long)cnt;
        if (threadIdx.x == 0) s_cnt2[(it + 1) & 1] = 0;  // the next iteration's counter (read last
                                                          // in iteration it-1, before the barrier above)
        __syncthreads();
        if (P.R > 0 && (P.k0 + it + 1) % P.R == 0) {
            // residual refresh (R8): r = fp32(A x - b) with fp64 accumulation, as the
            // host-side refresh of the other variants
            for (int t = threadIdx.x; t < m; t += blockDim.x) s_r64[t] = -(double)P.b[t];
            __syncthreads();
            for (int i = gid; i < n; i += ngroups) {
                const double xi = (double)s_x[i];
                if (xi == 0.0) continue;
                for (int q = s_col[i] + lane_g; q < s_col[i + 1]; q += G)
                    atomicAdd(s_r64 + s_row[q], (double)s_val[q] * xi);
            }
            __syncthreads();
            for (int t = threadIdx.x; t < m; t += blockDim.x) s_r[t] = (float)s_r64[t];
            __syncthreads();
        }
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x) P.x[t] = s_x[t];
    for (int t = threadIdx.x; t < m; t += blockDim.x) P.r[t] = s_r[t];
    if (threadIdx.x == 0 && nz_total) atomicAdd(P.nz_total, nz_total);
}


// ---------------------------------------------------------------- SMEM1 variant
// The same problem placement, one slot per G-lane group (tau * G <= 1024), each lane
// holding <= E entries of its column in registers, and ONE barrier per iteration: r is
// double-buffered in shared memory.  Iteration k gathers from buf[k & 1] (every step
// < k) and adds its own steps AND the previous iteration's steps (replayed from the
// group's registers) into buf[(k + 1) & 1] (every step < k - 1), which nobody reads in
// iteration k.  The barrier then publishes buf[(k + 1) & 1] = r_{k+1} (alg:PCD1 step 4,
// every g_i of iteration k from r_k).  No step list, no counter atomics;
// the group's lanes all hold the butterfly sum (bit-identical: fp addition commutes), so
// each takes the step and scatters its own entries.  The next slot's column is loaded
// into registers before the barrier (S and A do not depend on r).
// The slot ids stream through a shared-memory double buffer of W-iteration windows
// (cp.async, issued a window ahead): a global load per iteration on the critical path
// measured ~0.6 us per iteration on tiny.
__device__ __forceinline__ int smem1_window(int64_t tau) { return (int)max((int64_t)4, min((int64_t)64, 2048 / tau)); }

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}

// Per column, computed once per launch: inv_i = 1/(beta L_i) (logistic: 1/(beta L_i + 2
// lam)), 0 for an empty column, and lin_i = lam * inv_i (+inf for an empty column when
// lam > 0).  The step is then multiplications only: LASSO x+ = sign(u) max(|u| - lin, 0),
// u = x - g inv (prox_l1 with g/s -> g (1/s), lam/s -> lam (1/s): one rounding more
// each; an empty column gives u = x, |u| - inf < 0 -> 0 for lam > 0 and x for lam = 0,
// as prox_l1); logistic x+ = x - (g + 2 lam x) inv (x for a zero denominator).
// Column n is a dummy empty column with x = inv = lin = 0 (idle slots: d = 0).
template <bool LOGISTIC>
__device__ __forceinline__ float step_inv(float x, float g, float inv, float lin, float lam) {
    if (LOGISTIC) return x - (g + 2.0f * lam * x) * inv;
    const float u = fmaf(-g, inv, x);
    const float mag = fabsf(u) - lin;
    if (!(mag > 0.0f)) return (mag == mag) ? 0.0f : mag;  // keep NaN visible
    return copysignf(mag, u);
}

template <int G, int E, bool LOGISTIC>
__global__ void __launch_bounds__(kSmemThreads) pcdm_smem1_kernel(IterParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = (int)P.m, n = (int)P.n;
    const int nnz = (int)P.colptr[n];
    const int tau = (int)P.tau;
    const int iters = (int)P.iters;
    const int W = smem1_window(tau);
    const int WT = W * tau;
    double* s_r64 = (double*)smem_raw;           // m (refresh scratch)
    int* s_col = (int*)(s_r64 + m);              // n+2 (column n: the dummy)
    int* s_row = s_col + (n + 2);                // nnz
    float* s_val = (float*)(s_row + nnz);        // nnz
    float* s_inv = s_val + nnz;                  // n+1
    float* s_lin = s_inv + (n + 1);              // n+1
    float* s_x = s_lin + (n + 1);                // n+1
    float* s_rb = s_x + (n + 1);                 // 2 x m
    float* s_b = s_rb + 2 * m;                   // m
    int* s_sl = (int*)(s_b + m);                 // 2 x W x tau slot ids (a ring)
    const float beta = P.beta, lam = P.lambda;

    auto fetch_window = [&](int w, bool async) {
        const int it0 = w * W;
        const int cnt = min(W, iters - it0) * tau;
        int* dst = s_sl + (w & 1) * WT;
        const int* src = P.slots + (int64_t)it0 * tau;
        for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
            if (async) cp_async4(dst + t, src + t);
            else dst[t] = src[t];
        }
        if (async) asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int t = threadIdx.x; t <= n + 1; t += blockDim.x) s_col[t] = (int)P.colptr[min(t, n)];
    for (int t = threadIdx.x; t < nnz; t += blockDim.x) {
        s_row[t] = P.rowidx[t];
        s_val[t] = P.val[t];
    }
    for (int t = threadIdx.x; t <= n; t += blockDim.x) {
        float inv = 0.0f, lin = 0.0f, xv = 0.0f;
        if (t < n) {
            const float sL = beta * P.L[t];
            const float den = LOGISTIC ? sL + 2.0f * lam : sL;
            inv = den == 0.0f ? 0.0f : 1.0f / den;
            lin = LOGISTIC ? 0.0f : (sL == 0.0f ? (lam > 0.0f ? __int_as_float(0x7f800000) : 0.0f) : lam / sL);
            xv = P.x[t];
        }
        s_inv[t] = inv;
        s_lin[t] = lin;
        s_x[t] = xv;
    }
    for (int t = threadIdx.x; t < m; t += blockDim.x) {
        s_rb[t] = s_rb[m + t] = P.r[t];
        s_b[t] = P.b ? P.b[t] : 0.0f;
    }
    if (iters > 0) fetch_window(0, false);
    __syncthreads();

    const int lane_g = threadIdx.x & (G - 1);
    const int gid = threadIdx.x / G;
    const bool active = gid < tau;
    const int ring = 2 * WT;
    unsigned nzc = 0;

    // the current slot's column: entries (padding: row 0, value 0 -- the gathers are
    // unconditional, fmaf(0, r, acc) = acc), 1/(beta L), lam/(beta L)
    int crow[E];
    float cval[E];
    float cinv, clin;
    int ci;
    auto load_col = [&](int i) {
        ci = i < 0 ? n : i;
        const int s = s_col[ci], e = s_col[ci + 1];
        cinv = s_inv[ci];
        clin = s_lin[ci];
#pragma unroll
        for (int u = 0; u < E; ++u) {
            const int q = s + u * G + lane_g;
            const bool ok = q < e;
            crow[u] = ok ? s_row[q] : 0;
            cval[u] = ok ? s_val[q] : 0.0f;
        }
    };
    load_col(active && iters > 0 ? s_sl[gid] : -1);
    int pi = n;          // the previous iteration's column and step (replayed)
    float pd = 0.0f;
    int until_refresh = P.R > 0 ? (int)(P.R - (P.k0 % P.R)) : -1;
    int sp = tau + gid;  // ring position of the next iteration's slot id
    int pos = 0, win = 0;  // it = win * W + pos

    for (int it = 0; it < iters; ++it) {
        const float* rr = s_rb + (it & 1) * m;
        float* rw = s_rb + ((it + 1) & 1) * m;
        float acc = 0.0f, acc2 = 0.0f;  // two chains when a lane holds many entries
#pragma unroll
        for (int u = 0; u < E; ++u) {
            if (E >= 4 && (u & 1)) acc2 = fmaf(cval[u], grad_weight<LOGISTIC>(rr[crow[u]]), acc2);
            else acc = fmaf(cval[u], grad_weight<LOGISTIC>(rr[crow[u]]), acc);
        }
        acc += acc2;
        const float xi = s_x[ci];
        const int ni = (active && it + 1 < iters) ? s_sl[sp] : -1;
        sp += tau;
        if (sp >= ring) sp -= ring;
        // window win+1 into the ring half window win-1 used (its last id was read in
        // iteration win*W - 2, before the last barrier)
        if (pos == 0 && (win + 1) * W < iters) fetch_window(win + 1, true);
        // the previous iteration's step into the buffer that lacks it (rare)
        if (pd != 0.0f) {
            const int s = s_col[pi], e = s_col[pi + 1];
            for (int q = s + lane_g; q < e; q += G) atomicAdd(rw + s_row[q], s_val[q] * pd);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const float xp = step_inv<LOGISTIC>(xi, acc, cinv, clin, lam);
        const float d = xp - xi;
        if (d != 0.0f) {  // rare for LASSO
            if (lane_g == 0) {
                if (!isfinite(xp)) atomicOr(P.flags, FLAG_DIVERGED);
                s_x[ci] = xp;
                ++nzc;
            }
#pragma unroll
            for (int u = 0; u < E; ++u)
                if (cval[u] != 0.0f) atomicAdd(rw + crow[u], cval[u] * d);
        }
        pi = ci;
        pd = d;
        load_col(ni);  // S and A do not depend on r
        if (++pos == W) pos = 0, ++win;
        // the next window's copies land before the barrier that precedes its first read
        if (pos == W - 1) asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        if (--until_refresh == 0) {
            // residual refresh (R8): r = fp32(A x - b), fp64 accumulation; both buffers
            // then hold r_{k+1}, so nothing is replayed.  A warp takes 32 columns at a
            // time and walks the entries of the nonzero ones.
            until_refresh = (int)P.R;
            pd = 0.0f;
            for (int t = threadIdx.x; t < m; t += blockDim.x) s_r64[t] = -(double)s_b[t];
            __syncthreads();
            const int lane = threadIdx.x & 31;
            for (int base = (threadIdx.x >> 5) * 32; base < n; base += (blockDim.x >> 5) * 32) {
                const float xl = base + lane < n ? s_x[base + lane] : 0.0f;
                unsigned nzm = __ballot_sync(0xffffffffu, xl != 0.0f);
                while (nzm) {
                    const int j = __ffs(nzm) - 1;
                    nzm &= nzm - 1;
                    const double xj = (double)__shfl_sync(0xffffffffu, xl, j);
                    const int i = base + j;
                    for (int q = s_col[i] + lane; q < s_col[i + 1]; q += 32)
                        atomicAdd(s_r64 + s_row[q], (double)s_val[q] * xj);
                }
            }
            __syncthreads();
            for (int t = threadIdx.x; t < m; t += blockDim.x) s_rb[t] = s_rb[m + t] = (float)s_r64[t];
            __syncthreads();
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    const float* rf = s_rb + (iters & 1) * m;
    for (int t = threadIdx.x; t < n; t += blockDim.x) P.x[t] = s_x[t];
    for (int t = threadIdx.x; t < m; t += blockDim.x) P.r[t] = rf[t];
    if (nzc) atomicAdd(P.nz_total, (unsigned long long)nzc);
}

size_t smem1_bytes(int64_t m, int64_t n, int64_t nnz, int64_t tau) {
    const int64_t W = std::max<int64_t>(4, std::min<int64_t>(64, 2048 / std::max<int64_t>(tau, 1)));
    return (size_t)m * 8 + (size_t)(n + 2) * 4 + (size_t)nnz * 8 + (size_t)(n + 1) * 12 + (size_t)m * 12 +
           (size_t)(2 * W * tau) * 4;
}

size_t smem_bytes(int64_t m, int64_t n, int64_t nnz, int64_t tau) {
    return (size_t)(n + 1) * 4 + (size_t)nnz * 8 + (size_t)n * 8 + (size_t)m * 4 + (size_t)tau * 8 + 8 +
           (size_t)m * 8;  // + the refresh scratch
}

int pow2_clamp(int64_t v, int lo, int hi) {
    int g = 1;
    while (g < v && g < hi) g <<= 1;
    return g < lo ? lo : g;
}

template <int G, int U, bool SINGLE, bool LOG>
cudaError_t launch_one(const IterLaunch& L, const IterParams& P, cudaStream_t st) {
    if (SINGLE) {
        pcdm_iter_kernel<G, U, true, LOG><<<1, L.threads, 0, st>>>(P);
        return cudaGetLastError();
    }
    void* args[] = {(void*)&P};
    return cudaLaunchCooperativeKernel((const void*)pcdm_iter_kernel<G, U, false, LOG>, dim3(L.ctas),
                                       dim3(L.threads), args, 0, st);
}

template <int U, bool SINGLE, bool LOG>
cudaError_t launch_lanes(const IterLaunch& L, const IterParams& P, cudaStream_t st) {
    switch (L.lanes) {
        case 1: return launch_one<1, U, SINGLE, LOG>(L, P, st);
        case 2: return launch_one<2, U, SINGLE, LOG>(L, P, st);
        case 4: return launch_one<4, U, SINGLE, LOG>(L, P, st);
        case 8: return launch_one<8, U, SINGLE, LOG>(L, P, st);
        case 16: return launch_one<16, U, SINGLE, LOG>(L, P, st);
        default: return launch_one<32, U, SINGLE, LOG>(L, P, st);
    }
}

template <int G, int E, bool LOG>
cudaError_t launch_smem1(const IterLaunch& L, const IterParams& P, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(pcdm_smem1_kernel<G, E, LOG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L.smem);
    if (e != cudaSuccess) return e;
    pcdm_smem1_kernel<G, E, LOG><<<1, L.threads, L.smem, st>>>(P);
    return cudaGetLastError();
}

template <int E, bool LOG>
cudaError_t launch_smem1_lanes(const IterLaunch& L, const IterParams& P, cudaStream_t st) {
    switch (L.lanes) {
        case 1: return launch_smem1<1, E, LOG>(L, P, st);
        case 2: return launch_smem1<2, E, LOG>(L, P, st);
        case 4: return launch_smem1<4, E, LOG>(L, P, st);
        case 8: return launch_smem1<8, E, LOG>(L, P, st);
        case 16: return launch_smem1<16, E, LOG>(L, P, st);
        default: return launch_smem1<32, E, LOG>(L, P, st);
    }
}

// E > 4 entries per lane: one or two lanes per column
template <int E, bool LOG>
cudaError_t launch_smem1_few(const IterLaunch& L, const IterParams& P, cudaStream_t st) {
    return L.lanes == 1 ? launch_smem1<1, E, LOG>(L, P, st) : launch_smem1<2, E, LOG>(L, P, st);
}

template <int G, bool LOG>
cudaError_t launch_smem(const IterLaunch& L, const IterParams& P, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(pcdm_smem_kernel<G, LOG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L.smem);
    if (e != cudaSuccess) return e;
    pcdm_smem_kernel<G, LOG><<<1, L.threads, L.smem, st>>>(P);
    return cudaGetLastError();
}

}  // namespace

namespace {

template <bool LOG>
cudaError_t launch_iter_loss(const IterLaunch& L, const IterParams& P, cudaStream_t st) {
    constexpr int kU = 8;
    if (L.variant == 2 && L.entries > 0) {
        switch (L.entries) {
            case 1: return launch_smem1_lanes<1, LOG>(L, P, st);
            case 2: return launch_smem1_lanes<2, LOG>(L, P, st);
            case 3: return launch_smem1_lanes<3, LOG>(L, P, st);
            case 4: return launch_smem1_lanes<4, LOG>(L, P, st);
            case 6: return launch_smem1_few<6, LOG>(L, P, st);
            case 8: return launch_smem1_few<8, LOG>(L, P, st);
            case 12: return launch_smem1_few<12, LOG>(L, P, st);
            default: return launch_smem1_few<16, LOG>(L, P, st);
        }
    }
    if (L.variant == 2) {
        switch (L.lanes) {
            case 1: return launch_smem<1, LOG>(L, P, st);
            case 2: return launch_smem<2, LOG>(L, P, st);
            case 4: return launch_smem<4, LOG>(L, P, st);
            case 8: return launch_smem<8, LOG>(L, P, st);
            case 16: return launch_smem<16, LOG>(L, P, st);
            default: return launch_smem<32, LOG>(L, P, st);
        }
    }
    if (L.variant == 3) return launch_lanes<kU, true, LOG>(L, P, st);
    return launch_lanes<kU, false, LOG>(L, P, st);
}

}  // namespace

namespace pcdm_internal {

constexpr int kUnroll = 8;
constexpr size_t kSmemLimit = 200 * 1024;

IterLaunch plan_iter(int variant, int64_t m, int64_t n, int64_t nnz, int64_t tau, int sms, int device,
                     bool logistic, int64_t max_len) {
    IterLaunch L{};
    const int64_t avg = (nnz + n - 1) / n;
    const size_t sm = smem_bytes(m, n, nnz, tau);
    if (variant == 0) variant = (sm <= kSmemLimit && nnz < (1ll << 31)) ? 2 : 1;
    if (variant == 2 && !(sm <= kSmemLimit && nnz < (1ll << 31))) variant = 1;
    L.variant = variant;
    if (variant == 2) {
        L.ctas = 1;
        L.lanes = pow2_clamp(avg, 1, 32);
        if (const char* sl = knob("PCDM_SMEM_LANES")) L.lanes = pow2_clamp(atoi(sl), 1, 32);  // A/B
        // as many threads as the slots need (each __syncthreads waits for all of them)
        L.threads = std::max(64, std::min(kSmemThreads, pow2_clamp(tau * L.lanes, 64, kSmemThreads)));
        L.smem = sm;
        // the one-barrier kernel: one slot per group of G lanes (tau * G <= 1024 threads),
        // the longest column in E = ceil(max_len / G) entries per lane (E <= 4, or
        // E in {6, 8, 12, 16} for G <= 2); the most lanes that fit (E = 1 when tau allows):
        // fewer lanes shorten the butterfly but serialise the scatter of a nonzero step and
        // the refresh (tiny: G = 16 0.45, 4 0.52, 2 0.66, 1 1.13 us per iteration,
        // profiles/r02_smem1_ab.txt); PCDM_SMEM1=0 keeps the two-barrier list kernel
        // (A/B, tests), PCDM_SMEM_LANES forces G
        const char* s1 = knob("PCDM_SMEM1");
        const size_t sm1 = smem1_bytes(m, n, nnz, tau);
        if (max_len >= 0 && !(s1 && atoi(s1) == 0) && sm1 <= kSmemLimit) {
            int G = pow2_clamp(std::max<int64_t>(max_len, 1), 1, 32);
            while (G > 1 && tau * G > kSmemThreads) G >>= 1;
            if (const char* sl = knob("PCDM_SMEM_LANES")) G = pow2_clamp(atoi(sl), 1, 32);
            int64_t E = std::max<int64_t>(1, (max_len + G - 1) / G);
            if (E > 4) E = G > 2 ? 0 : E <= 6 ? 6 : E <= 8 ? 8 : E <= 12 ? 12 : E <= 16 ? 16 : 0;
            if (E > 0 && tau * G <= kSmemThreads) {
                L.entries = (int)E;
                L.lanes = G;
                L.threads = std::max(32, (int)((tau * G + 31) / 32 * 32));
                L.smem = sm1;
            }
        }
        return L;
    }
    L.lanes = pow2_clamp((avg + kUnroll - 1) / kUnroll, 1, 32);
    L.threads = kGridThreads;
    if (variant == 3) {
        L.ctas = 1;
        return L;
    }
    int per_sm = 1;
    const void* fn;
    switch (L.lanes) {
        case 1: fn = logistic ? (const void*)pcdm_iter_kernel<1, kUnroll, false, true> : (const void*)pcdm_iter_kernel<1, kUnroll, false, false>; break;
        case 2: fn = logistic ? (const void*)pcdm_iter_kernel<2, kUnroll, false, true> : (const void*)pcdm_iter_kernel<2, kUnroll, false, false>; break;
        case 4: fn = logistic ? (const void*)pcdm_iter_kernel<4, kUnroll, false, true> : (const void*)pcdm_iter_kernel<4, kUnroll, false, false>; break;
        case 8: fn = logistic ? (const void*)pcdm_iter_kernel<8, kUnroll, false, true> : (const void*)pcdm_iter_kernel<8, kUnroll, false, false>; break;
        case 16: fn = logistic ? (const void*)pcdm_iter_kernel<16, kUnroll, false, true> : (const void*)pcdm_iter_kernel<16, kUnroll, false, false>; break;
        default: fn = logistic ? (const void*)pcdm_iter_kernel<32, kUnroll, false, true> : (const void*)pcdm_iter_kernel<32, kUnroll, false, false>; break;
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGridThreads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    (void)device;
    L.ctas = per_sm * sms;
    return L;
}

cudaError_t launch_iter(const IterLaunch& L, const IterParams& P, cudaStream_t st, int64_t* launches) {
    ++*launches;
    return P.logistic ? launch_iter_loss<true>(L, P, st) : launch_iter_loss<false>(L, P, st);
}

}  // namespace pcdm_internal
