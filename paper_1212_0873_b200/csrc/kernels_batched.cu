// kernels_batched.cu -- the synchronous PCDM1 loop with batched-snapshot partial
// gradients (BATCHED variant; for residuals much larger than L2, e.g. `huge`).
//
// Why: on `huge` (r = 400 MB) every sampled column costs ~10 random 4-byte gathers
// of r, each filling a 128-byte line from HBM; one iteration touches ~57 % of r's
// lines.  The partial derivative of alg:PCD1 at iteration k is
//
//     g_i = a_i^T r_k = a_i^T r_0 + a_i^T (r_k - r_0),
//
// r_0 the residual at the start of a chunk of c iterations.  The first term does
// not depend on the steps taken inside the chunk, so it is computed for all c tau
// sampled columns at once, with the gathers sorted by row bin so that r streams
// through L2 once per chunk (passes 1-2).  The second term is nonzero only on rows
// touched by the chunk's nonzero steps (a handful per iteration on LASSO), kept in
// a dense delta buffer D = r_k - r_0 and found through a per-CTA Bloom filter of
// those rows (pass 3).  The step itself is the packed loop's (kernels_packed.cu):
// same soft-threshold (eq:h(x)), same synchronous semantics; only
// the summation order of g_i changes (fp32 rounding, within the north_star
// tolerance).
//
//   pass 1  expand: per range q of Cq chunk slots, the sampled columns' blocks are
//           unpacked into (row, val) entries, counting-sorted by row bin (2^rb
//           rows) in shared memory and written coalesced: gent[q][x] =
//           (row_local | slot_local << rb, val), offs[q][b] = start of bin b.
//   pass 2  sweep: each CTA owns a group of slot ranges and walks the bins in order,
//           so the grid works on one or two 8 MB tiles of r at a time;
//           g0[t] += val * w(r[row]) accumulated in shared memory.
//   pass 3  steps: c iterations in one cooperative launch, one grid barrier each;
//           g = g0 + sum over Bloom-flagged rows of val * (w(r + D_P) - w(r));
//           nonzero steps scatter into D_Q (the one-barrier double buffer of
//           kernels_packed.cu applied to D instead of r) and are listed per
//           iteration.
//   fold    r += sum of the chunk's steps; D_P = D_Q = 0 on their rows.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

using namespace pcdm;
using namespace pcdm_internal;

namespace {

constexpr int kThreads = 512;
constexpr int kBloomLog = 19;  // dirty-row filter: 2^19 bits = 64 KB of shared memory per CTA
constexpr int kColLog = 16;    // stepped-column filter: 2^16 bits = 8 KB
#ifndef PCDM_EXPAND_THREADS
#define PCDM_EXPAND_THREADS 512
#endif
constexpr int kExpandThreads = PCDM_EXPAND_THREADS;  // pass 1 CTA size (its slot range scales with it)
constexpr int kSweepMaxSlots = 40 * 512;  // pass 2: slots per CTA (x 4 B of shared accumulators)
#ifndef PCDM_SWEEP_HW
#define PCDM_SWEEP_HW 16
#endif
#ifndef PCDM_EXPAND_U
#define PCDM_EXPAND_U 4  // pass 1: slots per group in flight
#endif
#ifndef PCDM_BATCHED_UP
#define PCDM_BATCHED_UP 1  // pass 3: slots per thread loaded before the filter update
#endif
#ifndef PCDM_EXPAND_MINB
#define PCDM_EXPAND_MINB 2
#endif

__device__ __forceinline__ int4 ld_l2_v4(const int4* p) {
    int4 v;
    asm volatile("ld.global.cg.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ int4 ld_stream_v4(const int4* p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ int2 ld_stream_v2(const int2* p) {
    int2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

template <int G>
__device__ __forceinline__ unsigned gmask_of() {
    if constexpr (G == 32) {
        return 0xffffffffu;
    } else {
        const unsigned lane = threadIdx.x & 31;
        return ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
    }
}

// lane t's 16-byte chunk of a column block inside the step kernels, which write x_i into
// the header (chunk 0 .z) when P.xlist: the header through L2, the immutable (row, val)
// chunks on the non-coherent path
__device__ __forceinline__ int4 ld_blk(const BatchedParams& P, const int4* p, int t) {
    return (t == 0 && P.xlist) ? ld_l2_v4(p) : ld_stream_v4(p);
}

// real row of a block entry (hot rows are stored as 0x80000000 | h, kernels_packed.cu)
__device__ __forceinline__ int real_row(int v, const int* hrow) { return v < 0 ? hrow[v & 0x7fffffff] : v; }

// two-hash Bloom filters (bit arrays of 2^LOG bits): a false positive costs one block
// read, a miss is impossible.  With k rows set, a row tests positive with probability
// ~(2k / 2^LOG)^2 (huge, k ~ 3000 per chunk: ~1.4e-4, against 6e-3 for one hash on
// 2^18 bits; one hit stalls the whole warp on the serial block read of pass 3)
template <int LOG>
__device__ __forceinline__ uint32_t bloom_h1(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - LOG); }
template <int LOG>
__device__ __forceinline__ uint32_t bloom_h2(uint32_t v) { return ((v ^ (v >> 15)) * 0x2C1B3C6Du) >> (32 - LOG); }
template <int LOG>
__device__ __forceinline__ void bloom_set(unsigned* bf, uint32_t v) {
    const uint32_t a = bloom_h1<LOG>(v), b = bloom_h2<LOG>(v);
    atomicOr(bf + (a >> 5), 1u << (a & 31));
    atomicOr(bf + (b >> 5), 1u << (b & 31));
}
template <int LOG>
__device__ __forceinline__ bool bloom_test(const unsigned* bf, uint32_t v) {
    const uint32_t a = bloom_h1<LOG>(v), b = bloom_h2<LOG>(v);
    return (bf[a >> 5] >> (a & 31)) & (bf[b >> 5] >> (b & 31)) & 1u;
}

// ---------------------------------------------------------------- pass 1: expand + sort
// Dynamic shared memory: stage int2[cq*maxe] | inv u16[cq*maxe] | cnt int[nb] | cur int[nb+1]
template <int G>
__global__ void __launch_bounds__(kExpandThreads, PCDM_EXPAND_MINB * 512 / kExpandThreads) batch_expand_kernel(BatchedParams P) {
    constexpr int MAXE = 2 * (G - 1);
    extern __shared__ int4 s_raw[];
    const int cq = 1 << P.cq_log;
    const int ne = cq * MAXE;
    int2* stage = (int2*)s_raw;
    unsigned short* inv = (unsigned short*)(stage + ne);
    int* cnt = (int*)(inv + ((ne + 7) & ~7));
    int* cur = cnt + P.nb;
    const int t = threadIdx.x & (G - 1);
    const int grp = threadIdx.x / G;
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int64_t total = P.iters * P.tau;
    const int rmask = (1 << P.rb) - 1;

    for (int q = blockIdx.x; q < P.nq; q += gridDim.x) {
        for (int b = threadIdx.x; b < P.nb; b += blockDim.x) cnt[b] = 0;
        __syncthreads();
        // U slots per group in flight: the slot ids, then their blocks, then the entries
        constexpr int U = PCDM_EXPAND_U;
        constexpr int GPC = kExpandThreads / G;  // groups per CTA
        for (int sl0 = grp; sl0 < cq; sl0 += GPC * U) {
            int iv[U];
            int4 cv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t tt = ((int64_t)q << P.cq_log) + sl0 + u * GPC;
                iv[u] = (sl0 + u * GPC < cq && tt < total) ? ld_stream_s32(P.slots + tt) : -1;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (iv[u] >= 0) cv[u] = ld_stream_v4(P.blocks + (int64_t)iv[u] * G + t);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int sl = sl0 + u * GPC;
                if (sl >= cq) break;
                const int64_t tt = ((int64_t)q << P.cq_log) + sl;
                int2 ea = make_int2(-1, 0), eb = make_int2(-1, 0);
                int len = 0;
                if (iv[u] >= 0) {
                    const int4 c = cv[u];
                    len = __shfl_sync(gm, c.y, src);
                    if (t > 0) {
                        if (2 * (t - 1) < len) {
                            ea = make_int2(real_row(c.x, P.hot_rows), c.y);
                            atomicAdd(cnt + (ea.x >> P.rb), 1);
                        }
                        if (2 * (t - 1) + 1 < len) {
                            eb = make_int2(real_row(c.z, P.hot_rows), c.w);
                            atomicAdd(cnt + (eb.x >> P.rb), 1);
                        }
                    }
                }
                if (t > 0) {
                    const int e0 = sl * MAXE + 2 * (t - 1);
                    stage[e0] = ea;
                    stage[e0 + 1] = eb;
                }
                // the slot record of pass 3, 8 bytes per lane: lane 0 {L_i, x_i}, lane t the
                // real rows of its two entries (-1 = none)
                if (tt < total && t < 2 * P.rnv)
                    P.rec[tt * 2 * P.rnv + t] = t == 0 ? make_int2(cv[u].x, cv[u].z) : make_int2(ea.x, eb.x);
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // exclusive scan of the bin counts (one warp, 32 bins per step)
            int carry = 0;
            for (int b0 = 0; b0 < P.nb; b0 += 32) {
                const int b = b0 + threadIdx.x;
                const int v = b < P.nb ? cnt[b] : 0;
                int incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (threadIdx.x >= o) incl += y;
                }
                if (b < P.nb) cur[b] = carry + incl - v;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (threadIdx.x == 0) cur[P.nb] = carry;
        }
        __syncthreads();
        int* offs = P.offs + (int64_t)q * (P.nb + 1);
        for (int b = threadIdx.x; b <= P.nb; b += blockDim.x) offs[b] = cur[b];
        __syncthreads();
        for (int e = threadIdx.x; e < ne; e += blockDim.x) {
            const int row = stage[e].x;
            if (row >= 0) inv[atomicAdd(cur + (row >> P.rb), 1)] = (unsigned short)e;
        }
        __syncthreads();
        const int n_ent = cur[P.nb - 1];  // end of the last bin = number of entries
        int2* out = P.gent + (int64_t)q * ne;
        for (int x = threadIdx.x; x < n_ent; x += blockDim.x) {
            const int e = inv[x];
            const int2 v = stage[e];
            out[x] = make_int2((v.x & rmask) | ((e / MAXE) << P.rb), v.y);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- pass 2: bin-major sweep
// One CTA owns a group of qpc consecutive slot ranges q and accumulates their g0 in
// shared memory (no global atomics); it walks the row bins in order, like every other
// CTA, so the grid works on one or two 8 MB tiles of r at a time and r streams
// through L2 once per chunk.  Half-warp h takes the (bin, q) segments h, h + 32, ...
// of the group in bin-major order (a segment holds ~100 entries on `huge`: ~7 per
// lane, all in flight); the next segment's bounds are loaded ahead.  (One CTA-wide
// list per bin was slower: 391 vs 288 us per 18 iterations, a barrier per bin.)
template <bool LOGISTIC>
__global__ void __launch_bounds__(kThreads, 2) batch_sweep_kernel(BatchedParams P, int qpc) {
    extern __shared__ float s_g[];
    constexpr int HW = PCDM_SWEEP_HW;  // lanes per segment
    const int hl = threadIdx.x & (HW - 1), hw = threadIdx.x / HW;
    constexpr int NH = kThreads / HW;
    const int ne = (1 << P.cq_log) * P.maxe;
    const int rmask = (1 << P.rb) - 1;
    const int64_t total = P.iters * P.tau;
    const int ngrp = (P.nq + qpc - 1) / qpc;
    for (int grp = blockIdx.x; grp < ngrp; grp += gridDim.x) {
        const int q0 = grp * qpc;
        const int nql = min(qpc, P.nq - q0);
        const int nacc = nql << P.cq_log;
        for (int k = threadIdx.x; k < nacc; k += blockDim.x) s_g[k] = 0.0f;
        __syncthreads();
        const int nseg = P.nb * nql;
        auto bounds = [&](int sg, int& lo, int& hi) {
            const int bb = sg / nql, ql = sg - bb * nql;
            const int* offs = P.offs + (int64_t)(q0 + ql) * (P.nb + 1) + bb;
            lo = __ldg(offs);
            hi = __ldg(offs + 1);
        };
        int lo = 0, hi = 0;
        if (hw < nseg) bounds(hw, lo, hi);
        for (int sg = hw; sg < nseg; sg += NH) {
            int nlo = 0, nhi = 0;
            if (sg + NH < nseg) bounds(sg + NH, nlo, nhi);
            const int bb = sg / nql, ql = sg - bb * nql;
            const int2* ent = P.gent + (int64_t)(q0 + ql) * ne;
            const float* rb = P.r + ((int64_t)bb << P.rb);
            float* acc = s_g + (ql << P.cq_log);
            constexpr int U = 8;
            for (int x0 = lo + hl; x0 < hi; x0 += HW * U) {
                int2 e[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (x0 + HW * u < hi) e[u] = ld_stream_v2(ent + x0 + HW * u);
                float rv[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (x0 + HW * u < hi) rv[u] = __ldcg(rb + (e[u].x & rmask));
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (x0 + HW * u < hi)
                        atomicAdd(acc + ((unsigned)e[u].x >> P.rb), __int_as_float(e[u].y) * grad_weight<LOGISTIC>(rv[u]));
            }
            lo = nlo;
            hi = nhi;
        }
        __syncthreads();
        float* g0 = P.g0 + ((int64_t)q0 << P.cq_log);
        const int64_t left = total - ((int64_t)q0 << P.cq_log);
        for (int k = threadIdx.x; k < nacc && k < left; k += blockDim.x) g0[k] = s_g[k];
        __syncthreads();
    }
}

// ---------------------------------------------------------------- pass 3: the steps
// correction of g_i on one entry: val * (w(r + D_P) - w(r)) if the row may be dirty
template <bool LOGISTIC>
__device__ __forceinline__ float dirty_term(const BatchedParams& P, const float* DP, const unsigned* bf, int row,
                                            float val) {
    if (!bloom_test<kBloomLog>(bf, (uint32_t)row)) return 0.0f;
    const float dv = ld_l2_f32(DP + row);
    if (dv == 0.0f) return 0.0f;
    if (!LOGISTIC) return val * dv;
    const float r0 = ld_l2_f32(P.r + row);
    return val * (grad_weight<true>(r0 + dv) - grad_weight<true>(r0));
}

template <int G, bool LOGISTIC>
__global__ void __launch_bounds__(kThreads, 2) pcdm_batched_kernel(BatchedParams P) {
    const int t = threadIdx.x & (G - 1);
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
    const int grp = threadIdx.x / G;
    const int pair0 = 2 * (t - 1);
    const int64_t tau = P.tau;
    // shared memory: Bloom filter of the chunk's dirty rows, of its stepped columns, hot-row ids
    extern __shared__ unsigned s_bf[];
    unsigned* s_cf = s_bf + (1 << (kBloomLog - 5));
    int* s_hrow = (int*)(s_cf + (1 << (kColLog - 5)));
    for (int w = threadIdx.x; w < (1 << (kBloomLog - 5)) + (1 << (kColLog - 5)); w += blockDim.x) s_bf[w] = 0u;
    for (int h = threadIdx.x; h < P.nhot; h += blockDim.x) s_hrow[h] = P.hot_rows[h];
    unsigned bar_target = 0;
    __syncthreads();

    for (int64_t it = 0; it < P.iters; ++it) {
        const float* DP = (it & 1) ? P.d1 : P.d0;
        float* DQ = (it & 1) ? P.d0 : P.d1;
        if (it > 0) {
            const int cntp = ld_l2_s32(P.nz_count + it - 1);
            const int* lidx = P.nz_idx + (it - 1) * tau;
            // every CTA: the rows of iteration it-1's steps into its filter
            for (int e = grp; e < cntp; e += kThreads / G) {
                const int i = ld_l2_s32(lidx + e);
                const int4 c = ld_blk(P, P.blocks + (int64_t)i * G + t, t);
                const int len = __shfl_sync(gm, c.y, src);
                if (t == 0) bloom_set<kColLog>(s_cf, (uint32_t)i);
                if (t > 0 && pair0 < len) bloom_set<kBloomLog>(s_bf, (uint32_t)real_row(c.x, s_hrow));
                if (t > 0 && pair0 + 1 < len) bloom_set<kBloomLog>(s_bf, (uint32_t)real_row(c.z, s_hrow));
            }
            // the grid: replay Delta_{it-1} into D_Q (one-barrier double buffer)
            for (int64_t e = gid; e < cntp; e += ngroups) {
                const int i = ld_l2_s32(lidx + e);
                const float d = ld_l2_f32(P.nz_delta + (it - 1) * tau + e);
                const int4 c = ld_blk(P, P.blocks + (int64_t)i * G + t, t);
                const int len = __shfl_sync(gm, c.y, src);
                if (t > 0 && pair0 < len) red_add_f32(DQ + real_row(c.x, s_hrow), __int_as_float(c.y) * d);
                if (t > 0 && pair0 + 1 < len) red_add_f32(DQ + real_row(c.z, s_hrow), __int_as_float(c.w) * d);
            }
            __syncthreads();
        }
        const int2* rec = P.rec + it * tau * G;
        const int* S = P.slots + it * tau;
        const float* g0 = P.g0 + it * tau;
        // U slot records per group in flight (coalesced, written by pass 1); the column's
        // block is read only when a row may be dirty (Bloom hit) or the step is nonzero
        constexpr int U = 2;
        for (int64_t j0 = gid; j0 < tau; j0 += U * ngroups) {
            int2 hv[U];
            int iv[U];
            float gv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t j = j0 + u * ngroups;
                iv[u] = -1;
                if (j < tau) {
                    iv[u] = ld_stream_s32(S + j);
                    hv[u] = ld_stream_v2(rec + j * G + t);
                    gv[u] = t == 0 ? __ldcg(g0 + j) : 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = iv[u];
                if (i < 0) continue;
                const int2 h = hv[u];
                const bool hit = t > 0 && ((h.x >= 0 && bloom_test<kBloomLog>(s_bf, (uint32_t)h.x)) ||
                                           (h.y >= 0 && bloom_test<kBloomLog>(s_bf, (uint32_t)h.y)));
                const bool need = __any_sync(gm, hit) != 0;
                int4 c = make_int4(0, 0, 0, 0);
                int len = 0;
                float acc = gv[u], xi = 0.0f;
                if (need) {
                    c = ld_l2_v4(P.blocks + (int64_t)i * G + t);
                    len = __shfl_sync(gm, c.y, src);
                    if (t > 0) {
                        if (pair0 < len) acc += dirty_term<LOGISTIC>(P, DP, s_bf, real_row(c.x, s_hrow), __int_as_float(c.y));
                        if (pair0 + 1 < len)
                            acc += dirty_term<LOGISTIC>(P, DP, s_bf, real_row(c.z, s_hrow), __int_as_float(c.w));
                    }
                }
                if (t == 0) {
                    // x_i as pass 1 read it, unless the column was stepped earlier in the chunk
                    if (!P.xlist) xi = ld_l2_f32(P.x + i);
                    else if (bloom_test<kColLog>(s_cf, (uint32_t)i)) xi = ld_l2_f32((const float*)(P.blocks + (int64_t)i * G) + 2);
                    else xi = __int_as_float(h.y);
                }
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gm, acc, o);
                float d = 0.0f;
                if (t == 0) {
                    const float xp = block_step<LOGISTIC>(xi, acc, P.beta * __int_as_float(h.x), P.lambda);
                    d = xp - xi;
                    if (d != 0.0f) {
                        if (!isfinite(xp)) atomicOr(P.flags, FLAG_DIVERGED);
                        if (P.xlist) {
                            ((float*)(P.blocks + (int64_t)i * G))[2] = xp;
                            if (P.xlist_cap > 0) {  // 0: dense iterate, no dirty list
                                const unsigned long long q = atomicAdd(P.xlist_count, 1ull);
                                if (q < (unsigned long long)P.xlist_cap) P.xlist[q] = i;
                            }
                        } else {
                            P.x[i] = xp;
                        }
                        const int pos = atomicAdd(P.nz_count + it, 1);
                        P.nz_idx[it * tau + pos] = i;
                        P.nz_delta[it * tau + pos] = d;
                    }
                }
                d = __shfl_sync(gm, d, src);
                if (d != 0.0f) {
                    if (!need) {
                        c = ld_blk(P, P.blocks + (int64_t)i * G + t, t);
                        len = __shfl_sync(gm, c.y, src);
                    }
                    if (t > 0 && pair0 < len) red_add_f32(DQ + real_row(c.x, s_hrow), __int_as_float(c.y) * d);
                    if (t > 0 && pair0 + 1 < len) red_add_f32(DQ + real_row(c.z, s_hrow), __int_as_float(c.w) * d);
                }
            }
        }
        if (it + 1 < P.iters) grid_barrier(P.barrier, bar_target);
    }
}

// Pass 3 with one thread per slot (G <= 8: the slot record is G/2 16-byte vectors,
// <= 14 rows).  Same arithmetic as pcdm_batched_kernel; a thread tests its slot's
// rows against the filter alone, so no group shuffles, and its first slot's record
// is loaded before the filter update so the two latencies overlap.  A Bloom hit or a
// nonzero step reads the column's block in the thread (rare on LASSO).
template <int G, bool LOGISTIC>
__global__ void __launch_bounds__(kThreads, 2) pcdm_batched_slot_kernel(BatchedParams P) {
    static_assert(G >= 2 && G <= 8, "one slot record per thread");
    constexpr int NV = G / 2;
    const int t = threadIdx.x & (G - 1);
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int grp = threadIdx.x / G;
    const int pair0 = 2 * (t - 1);
    const int64_t tau = P.tau;
    extern __shared__ unsigned s_bf[];
    unsigned* s_cf = s_bf + (1 << (kBloomLog - 5));
    int* s_hrow = (int*)(s_cf + (1 << (kColLog - 5)));
    for (int w = threadIdx.x; w < (1 << (kBloomLog - 5)) + (1 << (kColLog - 5)); w += blockDim.x) s_bf[w] = 0u;
    for (int h = threadIdx.x; h < P.nhot; h += blockDim.x) s_hrow[h] = P.hot_rows[h];
    unsigned bar_target = 0;
    __syncthreads();

    for (int64_t it = 0; it < P.iters; ++it) {
        const float* DP = (it & 1) ? P.d1 : P.d0;
        float* DQ = (it & 1) ? P.d0 : P.d1;
        const int4* rec = (const int4*)(P.rec + it * tau * 2 * P.rnv);
        const int* S = P.slots + it * tau;
        const float* g0 = P.g0 + it * tau;
        // this thread's first UP slots, in flight across the filter update
        constexpr int UP = PCDM_BATCHED_UP;
        int ipf[UP];
        int4 rpf[UP][NV];
        float gpf[UP];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
            const int64_t j = tid + u * nth;
            ipf[u] = -1;
            if (j < tau) {
                ipf[u] = ld_stream_s32(S + j);
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    rpf[u][v] = v < P.rnv ? ld_stream_v4(rec + j * P.rnv + v) : make_int4(-1, -1, -1, -1);
                gpf[u] = __ldcg(g0 + j);
            }
        }
        if (it > 0) {
            const int cntp = ld_l2_s32(P.nz_count + it - 1);
            const int* lidx = P.nz_idx + (it - 1) * tau;
            for (int e = grp; e < cntp; e += kThreads / G) {
                const int i = ld_l2_s32(lidx + e);
                const int4 c = ld_blk(P, P.blocks + (int64_t)i * G + t, t);
                const int len = __shfl_sync(gm, c.y, src);
                if (t == 0) bloom_set<kColLog>(s_cf, (uint32_t)i);
                if (t > 0 && pair0 < len) bloom_set<kBloomLog>(s_bf, (uint32_t)real_row(c.x, s_hrow));
                if (t > 0 && pair0 + 1 < len) bloom_set<kBloomLog>(s_bf, (uint32_t)real_row(c.z, s_hrow));
            }
            for (int64_t e = gid; e < cntp; e += ngroups) {
                const int i = ld_l2_s32(lidx + e);
                const float d = ld_l2_f32(P.nz_delta + (it - 1) * tau + e);
                const int4 c = ld_blk(P, P.blocks + (int64_t)i * G + t, t);
                const int len = __shfl_sync(gm, c.y, src);
                if (t > 0 && pair0 < len) red_add_f32(DQ + real_row(c.x, s_hrow), __int_as_float(c.y) * d);
                if (t > 0 && pair0 + 1 < len) red_add_f32(DQ + real_row(c.z, s_hrow), __int_as_float(c.w) * d);
            }
            __syncthreads();
        }
        auto process = [&](int64_t j, int i, const int4* rv, float acc) {
            const int4* blk = P.blocks + (int64_t)i * G;
            bool hit = false;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (v > 0) {
                    hit |= rv[v].x >= 0 && bloom_test<kBloomLog>(s_bf, (uint32_t)rv[v].x);
                    hit |= rv[v].y >= 0 && bloom_test<kBloomLog>(s_bf, (uint32_t)rv[v].y);
                }
                hit |= rv[v].z >= 0 && bloom_test<kBloomLog>(s_bf, (uint32_t)rv[v].z);
                hit |= rv[v].w >= 0 && bloom_test<kBloomLog>(s_bf, (uint32_t)rv[v].w);
            }
            int len = -1;
            if (hit) {
                len = ld_l2_v4(blk).y;
#pragma unroll
                for (int l = 1; l < G; ++l) {
                    const int4 c = ld_l2_v4(blk + l);
                    if (2 * (l - 1) < len) acc += dirty_term<LOGISTIC>(P, DP, s_bf, real_row(c.x, s_hrow), __int_as_float(c.y));
                    if (2 * (l - 1) + 1 < len)
                        acc += dirty_term<LOGISTIC>(P, DP, s_bf, real_row(c.z, s_hrow), __int_as_float(c.w));
                }
            }
            float xi;
            if (!P.xlist) xi = ld_l2_f32(P.x + i);
            else if (bloom_test<kColLog>(s_cf, (uint32_t)i)) xi = ld_l2_f32((const float*)blk + 2);
            else xi = __int_as_float(rv[0].y);
            const float xp = block_step<LOGISTIC>(xi, acc, P.beta * __int_as_float(rv[0].x), P.lambda);
            const float d = xp - xi;
            if (d == 0.0f) return;
            if (!isfinite(xp)) atomicOr(P.flags, FLAG_DIVERGED);
            if (P.xlist) {
                ((float*)blk)[2] = xp;
                if (P.xlist_cap > 0) {
                    const unsigned long long q = atomicAdd(P.xlist_count, 1ull);
                    if (q < (unsigned long long)P.xlist_cap) P.xlist[q] = i;
                }
            } else {
                P.x[i] = xp;
            }
            const int pos = atomicAdd(P.nz_count + it, 1);
            P.nz_idx[it * tau + pos] = i;
            P.nz_delta[it * tau + pos] = d;
            if (len < 0) len = (P.xlist ? ld_l2_v4(blk) : ld_stream_v4(blk)).y;
#pragma unroll
            for (int l = 1; l < G; ++l) {
                if (2 * (l - 1) >= len) break;
                const int4 c = ld_stream_v4(blk + l);
                red_add_f32(DQ + real_row(c.x, s_hrow), __int_as_float(c.y) * d);
                if (2 * (l - 1) + 1 < len) red_add_f32(DQ + real_row(c.z, s_hrow), __int_as_float(c.w) * d);
            }
        };
#pragma unroll
        for (int u = 0; u < UP; ++u)
            if (ipf[u] >= 0) process(tid + u * nth, ipf[u], rpf[u], gpf[u]);
        for (int64_t j = tid + UP * nth; j < tau; j += nth) {
            const int i = ld_stream_s32(S + j);
            if (i < 0) continue;
            int4 rv[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v)
                rv[v] = v < P.rnv ? ld_stream_v4(rec + j * P.rnv + v) : make_int4(-1, -1, -1, -1);
            process(j, i, rv, __ldcg(g0 + j));
        }
        if (it + 1 < P.iters) grid_barrier(P.barrier, bar_target);
    }
}

// ---------------------------------------------------------------- fold
// r += sum of the chunk's steps (a_i delta_i), D0 = D1 = 0 on their rows.
template <int G>
__global__ void batch_fold_kernel(BatchedParams P) {
    const int t = threadIdx.x & (G - 1);
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
    const int pair0 = 2 * (t - 1);
    unsigned long long nz = 0;
    for (int64_t it = 0; it < P.iters; ++it) {
        const int cnt = P.nz_count[it];
        if (gid == 0 && t == 0) nz += (unsigned long long)cnt;
        for (int64_t e = gid; e < cnt; e += ngroups) {
            const int i = P.nz_idx[it * P.tau + e];
            const float d = P.nz_delta[it * P.tau + e];
            const int4 c = ld_stream_v4(P.blocks + (int64_t)i * G + t);
            const int len = __shfl_sync(gm, c.y, src);
            if (t > 0 && pair0 < len) {
                const int row = real_row(c.x, P.hot_rows);
                red_add_f32(P.r_out + row, __int_as_float(c.y) * d);
                P.d0[row] = 0.0f;
                P.d1[row] = 0.0f;
            }
            if (t > 0 && pair0 + 1 < len) {
                const int row = real_row(c.z, P.hot_rows);
                red_add_f32(P.r_out + row, __int_as_float(c.w) * d);
                P.d0[row] = 0.0f;
                P.d1[row] = 0.0f;
            }
        }
    }
    if (nz) atomicAdd(P.nz_total, nz);
}

// pass 3: one thread per slot for G <= 8 (PCDM_BATCHED_GROUP=1: one group per slot)
template <int G>
const void* step_kernel(bool logistic) {
    if constexpr (G <= 8) {
        const bool group = [] {
            const char* v = knob("PCDM_BATCHED_GROUP");
            return v && atoi(v) != 0;
        }();
        if (!group)
            return logistic ? (const void*)pcdm_batched_slot_kernel<G, true>
                            : (const void*)pcdm_batched_slot_kernel<G, false>;
    }
    return logistic ? (const void*)pcdm_batched_kernel<G, true> : (const void*)pcdm_batched_kernel<G, false>;
}

template <int G>
size_t expand_smem(int cq_log, int nb) {
    const size_t ne = (size_t)1 << cq_log;
    const size_t n = ne * 2 * (G - 1);
    return n * sizeof(int2) + ((n + 7) & ~(size_t)7) * 2 + (size_t)(2 * nb + 1) * sizeof(int);
}

template <int G>
cudaError_t launch_all(const BatchedParams& P0, int ctas3, cudaStream_t st, int sms, int64_t* launches) {
    cudaError_t e;
    // slot records: P.rnv 16-byte vectors (rows 2 + 4 (rnv - 1) >= max column length);
    // the G-lane-group step kernel reads G / 2
    BatchedParams P = P0;
    if (step_kernel<G>(P.logistic) == (P.logistic ? (const void*)pcdm_batched_kernel<G, true>
                                                  : (const void*)pcdm_batched_kernel<G, false>))
        P.rnv = G / 2;
    P.rnv = std::max(1, std::min(P.rnv, G / 2));
    const size_t sm1 = expand_smem<G>(P.cq_log, P.nb);
    e = cudaFuncSetAttribute(batch_expand_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    if (e != cudaSuccess) return e;
    int per1 = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, batch_expand_kernel<G>, kExpandThreads, sm1);
    const int g1 = std::min(P.nq, std::max(1, per1) * sms);
    batch_expand_kernel<G><<<g1, kExpandThreads, sm1, st>>>(P);
    // pass 2: groups of qpc slot ranges per CTA, g0 accumulated in shared memory
    const int qpc = std::max(1, std::min(kSweepMaxSlots >> P.cq_log, (P.nq + 2 * sms - 1) / (2 * sms)));
    const size_t sm2 = ((size_t)qpc << P.cq_log) * sizeof(float);
    const void* sw = P.logistic ? (const void*)batch_sweep_kernel<true> : (const void*)batch_sweep_kernel<false>;
    e = cudaFuncSetAttribute(sw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    if (e != cudaSuccess) return e;
    const int ngrp = (P.nq + qpc - 1) / qpc;
    if (P.logistic)
        batch_sweep_kernel<true><<<std::min(ngrp, 2 * sms), kThreads, sm2, st>>>(P, qpc);
    else
        batch_sweep_kernel<false><<<std::min(ngrp, 2 * sms), kThreads, sm2, st>>>(P, qpc);
    void* args[] = {(void*)&P};
    const size_t sm3 = batched_step_smem(P.nhot);
    e = cudaLaunchCooperativeKernel(step_kernel<G>(P.logistic), dim3(ctas3), dim3(kThreads), args, sm3, st);
    if (e != cudaSuccess) return e;
    batch_fold_kernel<G><<<sms * 4, kThreads, 0, st>>>(P);
    *launches += 4;
    return cudaGetLastError();
}


}  // namespace

namespace pcdm_internal {

size_t batched_step_smem(int nhot) {
    return ((size_t)1 << (kBloomLog - 3)) + ((size_t)1 << (kColLog - 3)) + (size_t)nhot * sizeof(int);
}

int batched_cq_log(int G) {
    // Cq * maxlen_capacity <= 8192 entries staged in shared memory (64 KB + 16 KB) for a
    // 512-thread expand CTA, proportionally less for smaller ones
    const int maxe = 2 * (G - 1);
    int l = 0;
    while (((2 << l) * maxe) <= 8192 * kExpandThreads / 512) ++l;
    return l;
}

int batched_rb(int cq_log) { return std::min(21, 32 - cq_log); }

int batched_ctas(int G, int sms, bool logistic, int nhot) {
    const void* fn;
    switch (G) {
        case 2: fn = step_kernel<2>(logistic); break;
        case 4: fn = step_kernel<4>(logistic); break;
        case 8: fn = step_kernel<8>(logistic); break;
        case 16: fn = step_kernel<16>(logistic); break;
        default: fn = step_kernel<32>(logistic); break;
    }
    const size_t smem = batched_step_smem(nhot);
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    return per_sm * sms;
}

cudaError_t launch_batched(int G, const BatchedParams& P, int ctas3, cudaStream_t st, int sms, int64_t* launches) {
    switch (G) {
        case 2: return launch_all<2>(P, ctas3, st, sms, launches);
        case 4: return launch_all<4>(P, ctas3, st, sms, launches);
        case 8: return launch_all<8>(P, ctas3, st, sms, launches);
        case 16: return launch_all<16>(P, ctas3, st, sms, launches);
        default: return launch_all<32>(P, ctas3, st, sms, launches);
    }
}

}  // namespace pcdm_internal
