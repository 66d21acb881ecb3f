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
                     bool logistic) {
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
