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
#ifndef PCDM_EXPAND_COALESCE
#define PCDM_EXPAND_COALESCE 1  // pass 1: slot records staged and written coalesced after the load phase
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

// multiplicative hash of a key onto 2^log buckets (the screened pass's tables and bitmaps)
__device__ __forceinline__ uint32_t key_hash(uint32_t v, int log) { return (v * 0x9E3779B1u) >> (32 - log); }
__device__ __forceinline__ uint32_t key_hash2(uint32_t v, int log) { return ((v ^ (v >> 15)) * 0x2C1B3C6Du) >> (32 - log); }

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

// debug timeline (PCDM_SCREEN_TIMELINE): per chunk and kernel, the first CTA start and
// the last CTA end (%globaltimer ns); start stored bitwise-negated so both use atomicMax
struct TLScope {
    unsigned long long* p;
    __device__ static unsigned long long now() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    }
    __device__ TLScope(unsigned long long* tl, int k) : p(tl ? tl + 2 * k : nullptr) {
        if (p && threadIdx.x == 0) atomicMax(p, ~now());
    }
    __device__ ~TLScope() {
        if (p && threadIdx.x == 0) atomicMax(p + 1, now());
    }
};

// ---------------------------------------------------------------- pass 1: expand + sort
// Dynamic shared memory: stage int2[cq*maxe] | inv u16[cq*maxe] | cnt int[nb] | cur int[nb+1]
template <int G>
__global__ void __launch_bounds__(kExpandThreads, PCDM_EXPAND_MINB * 512 / kExpandThreads) batch_expand_kernel(BatchedParams P) {
    TLScope tl_scope(P.tl, 0);
    // stage stride per slot: the problem's longest column rounded up to an even count
    // (P.maxe <= 2 (G - 1)); slot = e / MAXE by a 32-bit multiplicative inverse
    const int MAXE = P.maxe;
    const unsigned inv_me = 0xFFFFFFFFu / (unsigned)MAXE + 1u;
    extern __shared__ int4 s_raw[];
    const int cq = 1 << P.cq_log;
    const int ne = cq * MAXE;
    int2* stage = (int2*)s_raw;
    unsigned short* inv = (unsigned short*)(stage + ne);
    int* cnt = (int*)(inv + ((ne + 7) & ~7));
    int* cur = cnt + P.nb;
    int2* s_lx = (int2*)(cnt + ((2 * P.nb + 2) & ~1));  // [cq] {L, x} per slot (PCDM_EXPAND_COALESCE)
    const int t = threadIdx.x & (G - 1);
    const int grp = threadIdx.x / G;
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int64_t total = P.iters * P.tau;
    const int rmask = (1 << P.rb) - 1;

    // U slots per group in flight: the slot ids, then their blocks, then the entries
    constexpr int U = PCDM_EXPAND_U;
    constexpr int GPC = kExpandThreads / G;  // groups per CTA
    auto load_round = [&](int q, int sl0, int (&iv)[U], int4 (&cv)[U]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t tt = ((int64_t)q << P.cq_log) + sl0 + u * GPC;
            iv[u] = (sl0 + u * GPC < cq && tt < total) ? ld_stream_s32(P.slots + tt) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            // through L2 (ld.cg): the previous chunk's fix-up may be writing x_i into the
            // headers meanwhile (the non-coherent path requires data unchanged during the kernel)
            if (iv[u] >= 0) cv[u] = ld_l2_v4(P.blocks + (int64_t)iv[u] * G + t);
    };
    for (int q = blockIdx.x; q < P.nq; q += gridDim.x) {
        for (int b = threadIdx.x; b < P.nb; b += blockDim.x) cnt[b] = 0;
        __syncthreads();
        for (int sl0 = grp; sl0 < cq; sl0 += GPC * U) {
            int iv[U];
            int4 cv[U];
            load_round(q, sl0, iv, cv);
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
                if (t > 0 && 2 * (t - 1) < MAXE) {
                    const int e0 = sl * MAXE + 2 * (t - 1);
                    stage[e0] = ea;
                    stage[e0 + 1] = eb;
                }
                if (tt < total && P.screen && PCDM_EXPAND_COALESCE) {
                    // {L_i, x_i} staged; the rows are the staged entries: both written
                    // coalesced after the load phase
                    if (t == 0) {
                        int2 lx = make_int2(-1, 0);
                        if (iv[u] >= 0)
                            lx = make_int2(cv[u].x, P.xlist ? cv[u].z : __float_as_int(ld_l2_f32(P.x + iv[u])));
                        s_lx[sl] = lx;
                    }
                } else if (tt < total && P.screen) {
                    // screened step pass: {L_i, x_i} per slot (L = -1 bits: idle slot) and the
                    // slot's real rows, row-major by entry (coalesced for the test pass)
                    if (t == 0) {
                        int2 lx = make_int2(-1, 0);
                        if (iv[u] >= 0)
                            lx = make_int2(cv[u].x, P.xlist ? cv[u].z : __float_as_int(ld_l2_f32(P.x + iv[u])));
                        P.lx[tt] = lx;
                    } else {
                        const int p0 = 2 * (t - 1);
                        if (p0 < P.nrow) P.rows[p0 * P.rows_ld + tt] = ea.x;
                        if (p0 + 1 < P.nrow) P.rows[(p0 + 1) * P.rows_ld + tt] = eb.x;
                    }
                } else if (tt < total && t < 2 * P.rnv) {
                    // the slot record of pass 3, 8 bytes per lane: lane 0 {L_i, x_i}, lane t the
                    // real rows of its two entries (-1 = none)
                    P.rec[tt * 2 * P.rnv + t] = t == 0 ? make_int2(cv[u].x, cv[u].z) : make_int2(ea.x, eb.x);
                }
            }
        }
        __syncthreads();
        if (P.screen && PCDM_EXPAND_COALESCE) {
            // the range's slot records, coalesced: {L, x} per slot and its rows row-major by
            // entry (a warp writes 32 consecutive slots of one entry index per store)
            const int64_t tq = (int64_t)q << P.cq_log;
            for (int sl = threadIdx.x; sl < cq; sl += blockDim.x)
                if (tq + sl < total) P.lx[tq + sl] = s_lx[sl];
            for (int w = threadIdx.x; w < P.nrow * cq; w += blockDim.x) {
                const int pp = w >> P.cq_log, sl = w & (cq - 1);
                if (tq + sl < total) P.rows[pp * P.rows_ld + tq + sl] = stage[sl * MAXE + pp].x;
            }
        }
        int* offs = P.offs + (int64_t)q * (P.nb + 1);
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
                if (b < P.nb) {
                    cur[b] = carry + incl - v;
                    offs[b] = carry + incl - v;
                }
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (threadIdx.x == 0) {
                cur[P.nb] = carry;
                offs[P.nb] = carry;
            }
        }
        __syncthreads();
        int2* out = P.gent + (int64_t)q * ne;
        for (int e = threadIdx.x; e < ne; e += blockDim.x) {
            const int row = stage[e].x;
            if (row >= 0) inv[atomicAdd(cur + (row >> P.rb), 1)] = (unsigned short)e;
        }
        __syncthreads();
        const int n_ent = cur[P.nb - 1];  // end of the last bin = number of entries
        for (int x = threadIdx.x; x < n_ent; x += blockDim.x) {
            const int e = inv[x];
            const int2 v = stage[e];
            out[x] = make_int2((v.x & rmask) | ((int)__umulhi((unsigned)e, inv_me) << P.rb), v.y);
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
constexpr int kStaleLog = 16;  // sweep: bitmap of the columns the previous chunk stepped (8 KB)
template <bool LOGISTIC>
__global__ void __launch_bounds__(kThreads, 2) batch_sweep_kernel(BatchedParams P, int qpc) {
    TLScope tl_scope(P.tl, 1);
    extern __shared__ float s_g[];
    unsigned* s_stale = (unsigned*)(s_g + (qpc << P.cq_log));
    __shared__ int s_all_stale;
    if (!LOGISTIC && P.screen) {
        // the columns the previous chunk stepped: this chunk's expand may have read their
        // x_i before that chunk's fix-up wrote it (the two overlap), so the epilogue
        // re-reads x_i for them (all columns when there are too many steps)
        for (int w = threadIdx.x; w < (1 << (kStaleLog - 5)); w += blockDim.x) s_stale[w] = 0u;
        if (threadIdx.x == 0) s_all_stale = 0;
        __syncthreads();
        if (P.prev_nz_idx) {
            for (int k = 0; k < P.prev_iters; ++k) {
                const int cnt = ld_l2_s32(P.prev_nz_count + k);
                if (cnt > 4096) s_all_stale = 1;
                else
                    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
                        const uint32_t h = key_hash((uint32_t)ld_l2_s32(P.prev_nz_idx + k * P.tau + e), kStaleLog);
                        atomicOr(s_stale + (h >> 5), 1u << (h & 31));
                    }
            }
        }
        __syncthreads();
    }
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
        const int kend = (int)std::min<int64_t>(nacc, left);
        if (LOGISTIC || !P.screen) {
            for (int k = threadIdx.x; k < kend; k += blockDim.x) g0[k] = s_g[k];
        } else {
            // the speculative step of every slot: its step if no earlier step of the chunk
            // touched its rows or its column (the fix-up's arithmetic in that case, bit for
            // bit); nonzero ones become items of the fix-up.  Four slots per thread with
            // their loads in flight together.
            constexpr int EU = 4;
            for (int k0 = threadIdx.x; k0 < kend; k0 += EU * blockDim.x) {
                int2 lx[EU];
                int iv[EU];
#pragma unroll
                for (int u = 0; u < EU; ++u) {
                    const int k = k0 + u * blockDim.x;
                    const int64_t t = ((int64_t)q0 << P.cq_log) + k;
                    lx[u] = k < kend ? ld_stream_v2(P.lx + t) : make_int2(-1, 0);
                    iv[u] = k < kend && P.prev_nz_idx ? ld_stream_s32(P.slots + t) : -1;
                }
#pragma unroll
                for (int u = 0; u < EU; ++u) {
                    const int k = k0 + u * blockDim.x;
                    if (k >= kend) break;
                    const int64_t t = ((int64_t)q0 << P.cq_log) + k;
                    const float g = s_g[k];
                    g0[k] = g;
                    if (lx[u].x == -1) continue;
                    float xi = __int_as_float(lx[u].y);
                    if (iv[u] >= 0) {
                        // x_i may predate the previous chunk's fix-up: re-read it for the
                        // columns that chunk stepped
                        const uint32_t h = key_hash((uint32_t)iv[u], kStaleLog);
                        if (s_all_stale || ((s_stale[h >> 5] >> (h & 31)) & 1u))
                            xi = P.xlist ? ld_l2_f32((const float*)(P.blocks + (int64_t)iv[u] * P.G) + 2)
                                         : ld_l2_f32(P.x + iv[u]);
                    }
                    const float xp = prox_l1(xi, g, P.beta * __int_as_float(lx[u].x), P.lambda);
                    if (xp - xi != 0.0f) {
                        atomicOr(P.bits + (t >> 5), 1u << (t & 31));
                        P.items[atomicAdd(P.counts, 1)] = (int)t;
                    }
                }
            }
        }
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

// ---------------------------------------------------------------- screened step pass
// Pass 3 without a grid barrier per iteration (LASSO).  The sweep's epilogue took every
// slot's step from g0 alone, the step the slot takes exactly when no earlier step of the
// chunk changed a row of its column or its x_i; the nonzero ones are the speculative
// items.  Synchronous PCDM1 (alg:PCD1) differs from that only at
// slots sharing a row or the column with a step of an earlier iteration of the chunk:
//   3s test:  every slot of iteration k is tested against the rows and columns of the
//             speculative steps of iterations < k (a shared-memory key table with the
//             earliest iteration per key); hits become flagged items;
//   4s fix:   one CTA replays the chunk's iterations over the items only, in order: g =
//             g0 + sum of val * D[row] over the rows the chunk's earlier true steps
//             dirtied (D in a shared-memory map), x_i current if the column stepped earlier;
//             a nonzero step updates x_i, D and r (the fold) at once.  A flagged item that
//             steps is a "miss": its rows were not tested against, so the CTA scans the
//             later slots for them before going on.
// Same arithmetic as pass 3 per slot (g0 + corrections in fp32); items that never touch a
// dirty row take exactly the speculative step.
constexpr int kTestThreads = 1024;
constexpr int kTestLog = 13;    // test key table: 2^13 {key, iteration} pairs = 64 KB
constexpr int kTestBmLog = 20;  // ... and a 2^20-bit (128 KB) one-hash bitmap of its keys
constexpr int kColKey = (int)0x80000000;  // column keys i | 2^31 (rows are >= 0)


// keep the minimum stamp per key (open addressing, linear probing; never full: the
// callers keep the load <= 1/2)
__device__ __forceinline__ void stamp_insert(int* keys, int* stamps, int log, int key, int stamp) {
    const uint32_t mask = (1u << log) - 1u;
    uint32_t h = key_hash((uint32_t)key, log);
    for (;;) {
        const int prev = atomicCAS(keys + h, -1, key);
        if (prev == -1 || prev == key) {
            atomicMin(stamps + h, stamp);
            return;
        }
        h = (h + 1) & mask;
    }
}
__device__ __forceinline__ int stamp_find(const int* keys, const int* stamps, int log, int key) {
    const uint32_t mask = (1u << log) - 1u;
    uint32_t h = key_hash((uint32_t)key, log);
    for (;;) {
        const int k = keys[h];
        if (k == key) return stamps[h];
        if (k == -1) return 0x7fffffff;
        h = (h + 1) & mask;
    }
}

// slot t of the chunk becomes an item (once)
__device__ __forceinline__ bool claim_slot(unsigned* bits, int64_t t) {
    const unsigned bit = 1u << (t & 31);
    return !(atomicOr(bits + (t >> 5), bit) & bit);
}

// test pass over slots [t0, t1) against the keys in the table: a thread takes 4
// consecutive slots (16-byte row loads; rows_ld is a multiple of 4), all their rows in
// flight, then two bits per key in the Bloom bitmap `bm` (2^bmlog bits, set for every
// key of the table; nullptr: none) -- only a slot whose key tests positive probes the
// table (probing every key made the pass instruction-bound, 133 us per chunk on huge;
// with one bit per key 3 % of the slots took the divergent probe path)
__device__ __forceinline__ void test_slots(const BatchedParams& P, const int* keys, const int* stamps, int log,
                                           const unsigned* bm, int bmlog, int64_t t0, int64_t t1, int64_t tid,
                                           int64_t nth, int* out, int* out_count) {
    const int64_t tau = P.tau;
    constexpr int PB = 6;  // rows per batch of loads
    auto maybe = [&](int key) -> unsigned {
        if (!bm) return 1u;
        const uint32_t h1 = key_hash((uint32_t)key, bmlog), h2 = key_hash2((uint32_t)key, bmlog);
        return (bm[h1 >> 5] >> (h1 & 31)) & (bm[h2 >> 5] >> (h2 & 31)) & 1u;
    };
    for (int64_t tb = (t0 & ~(int64_t)3) + 4 * tid; tb < t1; tb += 4 * nth) {
        int iv[4];
        unsigned any[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) iv[u] = tb + u >= t0 && tb + u < t1 ? ld_stream_s32(P.slots + tb + u) : -1;
#pragma unroll
        for (int u = 0; u < 4; ++u) any[u] = iv[u] >= 0 ? maybe(iv[u] | kColKey) : 0u;
        for (int p0 = 0; p0 < P.nrow; p0 += PB) {
            int4 rv[PB];
#pragma unroll
            for (int u = 0; u < PB; ++u)
                rv[u] = p0 + u < P.nrow ? ld_stream_v4((const int4*)(P.rows + (int64_t)(p0 + u) * P.rows_ld + tb))
                                        : make_int4(-1, -1, -1, -1);
#pragma unroll
            for (int u = 0; u < PB; ++u) {
                any[0] |= rv[u].x >= 0 ? maybe(rv[u].x) : 0u;
                any[1] |= rv[u].y >= 0 ? maybe(rv[u].y) : 0u;
                any[2] |= rv[u].z >= 0 ? maybe(rv[u].z) : 0u;
                any[3] |= rv[u].w >= 0 ? maybe(rv[u].w) : 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (!any[u] || iv[u] < 0) continue;
            // a candidate: the exact test against the stamped keys
            const int64_t ts = tb + u;
            const int k = (int)(ts / tau);
            bool h = stamp_find(keys, stamps, log, iv[u] | kColKey) < k;
            for (int p = 0; p < P.nrow && !h; ++p) {
                const int row = ld_stream_s32(P.rows + (int64_t)p * P.rows_ld + ts);
                h = row >= 0 && stamp_find(keys, stamps, log, row) < k;
            }
            if (h && claim_slot(P.bits, ts)) out[atomicAdd(out_count, 1)] = (int)ts;
        }
    }
}

template <int G>
__global__ void __launch_bounds__(kTestThreads, 1) screen_test_kernel(BatchedParams P) {
    TLScope tl_scope(P.tl, 2);
    extern __shared__ int s_kt[];
    int* keys = s_kt;
    int* stamps = s_kt + (1 << kTestLog);
    unsigned* bm = (unsigned*)(stamps + (1 << kTestLog));  // 2^kTestBmLog bits
    __shared__ int s_kmin;
    const int t = threadIdx.x & (G - 1);
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int pair0 = 2 * (t - 1);
    const int64_t tau = P.tau;
    const int64_t total = P.iters * tau;
    const int nspec = ld_l2_s32(P.counts);
    auto insert = [&](int key, int k) {
        stamp_insert(keys, stamps, kTestLog, key, k);
        const uint32_t h1 = key_hash((uint32_t)key, kTestBmLog), h2 = key_hash2((uint32_t)key, kTestBmLog);
        atomicOr(bm + (h1 >> 5), 1u << (h1 & 31));
        atomicOr(bm + (h2 >> 5), 1u << (h2 & 31));
    };
    // speculative slots per table fill (keys <= half the table)
    const int per = std::max(1, ((1 << kTestLog) / 2) / (1 + P.nrow));
    for (int b0 = 0; b0 < nspec; b0 += per) {
        for (int w = threadIdx.x; w < (1 << kTestLog); w += blockDim.x) {
            keys[w] = -1;
            stamps[w] = 0x7fffffff;
        }
        for (int w = threadIdx.x; w < (1 << (kTestBmLog - 5)); w += blockDim.x) bm[w] = 0u;
        if (threadIdx.x == 0) s_kmin = 0x7fffffff;
        __syncthreads();
        const int b1 = std::min(nspec, b0 + per);
        // one group of G lanes per speculative slot: its column and its rows, stamped with
        // the slot's iteration
        for (int q = b0 + (int)(threadIdx.x / G); q < b1; q += blockDim.x / G) {
            const int ts = ld_l2_s32(P.items + q);
            const int k = (int)(ts / tau);
            const int i = ld_stream_s32(P.slots + ts);
            const int4 c = ld_stream_v4(P.blocks + (int64_t)i * G + t);
            const int len = __shfl_sync(gm, c.y, src);
            if (t == 0) {
                insert(i | kColKey, k);
                atomicMin(&s_kmin, k);
            } else {
                if (pair0 < len) insert(real_row(c.x, P.hot_rows), k);
                if (pair0 + 1 < len) insert(real_row(c.z, P.hot_rows), k);
            }
        }
        __syncthreads();
        // slots of iterations after the earliest stamp
        const int64_t t0 = ((int64_t)s_kmin + 1) * tau;
        test_slots(P, keys, stamps, kTestLog, bm, kTestBmLog, t0, total, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                   (int64_t)gridDim.x * blockDim.x, P.items + P.rows_ld, P.counts + 1);
        __syncthreads();
    }
}

// fix-up shared-memory shape (host-computed from the shared-memory budget)
struct FixShape {
    int icap;  // items staged in shared memory (meta + nl block lanes each)
    int nl;    // 16-byte lanes staged per item (1 + ceil(max length / 2))
    int dlog;  // D map: 2^dlog {row, value} entries
    int clog;  // stepped-column set: 2^clog keys
    int scap;  // steps of one iteration kept in shared memory (the rest in the global list)
    int mlog;  // miss-scan key table: 2^mlog {key, stamp}
    int c;     // iterations of the chunk (histogram size)
};

size_t fix_smem_bytes(const FixShape& F) {
    return (size_t)F.icap * 16 * (1 + F.nl) + ((size_t)8 << F.dlog) + ((size_t)4 << F.clog) + (size_t)F.icap * 4 +
           (size_t)F.scap * 8 + ((size_t)8 << F.mlog) + (size_t)(F.c + 1) * 8;
}

template <int G>
__global__ void __launch_bounds__(kTestThreads, 1) screen_fix_kernel(BatchedParams P, FixShape F) {
    TLScope tl_scope(P.tl, 3);
    extern __shared__ int4 s_fix[];
    int4* s_meta = s_fix;                        // [icap] {t, i, g0, x0}
    int4* s_blk = s_meta + F.icap;               // [icap][nl] the item's block
    int* s_dkey = (int*)(s_blk + (size_t)F.icap * F.nl);
    float* s_dval = (float*)(s_dkey + (1 << F.dlog));
    int2* s_step = (int2*)(s_dval + (1 << F.dlog));  // [scap] {item, delta}
    int* s_ckey = (int*)(s_step + F.scap);
    int* s_ord = s_ckey + (1 << F.clog);         // [icap] items by iteration
    int* s_mkey = s_ord + F.icap;                // [2^mlog] miss keys
    int* s_mstamp = s_mkey + (1 << F.mlog);
    int* s_start = s_mstamp + (1 << F.mlog);     // [c + 1]
    int* s_cur = s_start + (F.c + 1);            // [c]
    __shared__ int s_nstep, s_dcount, s_ccount, s_dspill, s_cfull, s_miss, s_nextra, s_mcount, s_total, s_nmiss,
        s_nscan;
    __shared__ unsigned long long s_xbase;

    const int tid = threadIdx.x, nth = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nth >> 5;
    const int64_t tau = P.tau;
    const int c = (int)P.iters;
    const int nspec = ld_l2_s32(P.counts), ncand = ld_l2_s32(P.counts + 1);
    const int nit = nspec + ncand;
    // items q < nstaged live in shared memory (at most two per thread; scan hits: q >= nit)
    const int nstaged = min(nit, min(F.icap, 2 * nth));
    int* const cand = P.items + P.rows_ld;       // flagged items, then the misses' scans
    int* const ord = nit <= F.icap ? s_ord : P.items + 2 * P.rows_ld;
    auto item_t = [&](int q) { return q < nspec ? ld_l2_s32(P.items + q) : ld_l2_s32(cand + (q - nspec)); };
    const int dmask = (1 << F.dlog) - 1, cmask = (1 << F.clog) - 1;
    const int dlimit = (7 << F.dlog) / 10, climit = (7 << F.clog) / 10;

    long long tclk0 = clock64();
    for (int w = tid; w < (1 << F.dlog); w += nth) {
        s_dkey[w] = -1;
        s_dval[w] = 0.0f;
    }
    for (int w = tid; w < (1 << F.clog); w += nth) s_ckey[w] = -1;
    for (int w = tid; w <= c; w += nth) s_start[w] = 0;
    if (tid == 0) {
        s_nstep = s_dcount = s_ccount = s_dspill = s_cfull = s_miss = s_nextra = s_total = s_nmiss = s_nscan = 0;
    }
    __syncthreads();
    // stage the items (slot id, g0, x0 and the column's block); count them per iteration
    // with warp-aggregated atomics (one per distinct iteration in a warp), each item
    // keeping its rank within its iteration
    int my_k[2], my_rank[2];  // this thread's items q = tid and tid + nth (nit <= 2 nth here)
    for (int r = 0, q = tid; r < 2; ++r, q += nth) {
        my_k[r] = -1;
        const bool has = q < nit;
        int t = 0, k = -1;
        if (has) {
            t = item_t(q);
            k = (int)(t / tau);
        }
        const unsigned act = __ballot_sync(0xffffffffu, has);
        if (has) {
            const unsigned peers = __match_any_sync(act, k);
            const int leader = __ffs(peers) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(s_start + k, __popc(peers));
            base = __shfl_sync(peers, base, leader);
            my_k[r] = k;
            my_rank[r] = base + __popc(peers & ((1u << lane) - 1u));
        }
        if (has && q < nstaged) {
            const int i = ld_stream_s32(P.slots + t);
            const int4* blk = P.blocks + (int64_t)i * G;
            int4 bl[8];
#pragma unroll
            for (int l = 0; l < 8; ++l)
                if (l < F.nl) bl[l] = ld_stream_v4(blk + l);
            const float g0 = ld_l2_f32(P.g0 + t);
#pragma unroll
            for (int l = 0; l < 8; ++l)
                if (l < F.nl) s_blk[(size_t)q * F.nl + l] = bl[l];
            for (int l = 8; l < F.nl; ++l) s_blk[(size_t)q * F.nl + l] = ld_stream_v4(blk + l);
            const float x0 = P.xlist ? __int_as_float(bl[0].z) : ld_l2_f32(P.x + i);
            s_meta[q] = make_int4(t, i, __float_as_int(g0), __float_as_int(x0));
        }
    }
    __syncthreads();  // the ranks above count ranked items only
    for (int q = 2 * nth + tid; q < nit; q += nth) {  // beyond 2 per thread: not staged, plain atomics
        const int t = item_t(q);
        atomicAdd(s_start + t / tau, 1);
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the per-iteration counts, 32 iterations per step
        int carry = 0;
        for (int k0 = 0; k0 < c; k0 += 32) {
            const int k = k0 + tid;
            const int v = k < c ? s_start[k] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += y;
            }
            if (k < c) {
                s_start[k] = carry + incl - v;
                s_cur[k] = carry + incl;  // items beyond 2 per thread are appended after the ranked ones
            }
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (tid == 0) s_start[c] = carry;
    }
    __syncthreads();
    // ranked items go to start + rank; the rest (nit > 2 nth) are placed from the end of
    // their iteration's range backwards
    for (int r = 0; r < 2; ++r)
        if (my_k[r] >= 0) ord[s_start[my_k[r]] + my_rank[r]] = tid + r * nth;
    for (int q = 2 * nth + tid; q < nit; q += nth) ord[atomicSub(s_cur + item_t(q) / tau, 1) - 1] = q;
    __syncthreads();

    // (every probe loop is bounded by the table size: concurrent inserts may overshoot the
    // load limit and fill a small table)
    auto dget = [&](int row) -> float {
        float v = 0.0f;
        int h = (int)key_hash((uint32_t)row, F.dlog);
        for (int pr = 0; pr <= dmask; ++pr) {
            const int k = s_dkey[h];
            if (k == row) {
                v = s_dval[h];
                break;
            }
            if (k == -1) break;
            h = (h + 1) & dmask;
        }
        if (s_dspill) v += ld_l2_f32(P.d0 + row);
        return v;
    };
    auto dadd = [&](int row, float v) {
        int h = (int)key_hash((uint32_t)row, F.dlog);
        for (int pr = 0; pr <= dmask; ++pr) {
            const int k = ((volatile int*)s_dkey)[h];
            if (k == row) {
                atomicAdd(s_dval + h, v);
                return;
            }
            if (k == -1) {
                if (*(volatile int*)&s_dcount >= dlimit) break;
                const int prev = atomicCAS(s_dkey + h, -1, row);
                if (prev == -1) atomicAdd(&s_dcount, 1);
                if (prev == -1 || prev == row) {
                    atomicAdd(s_dval + h, v);
                    return;
                }
            }
            h = (h + 1) & dmask;
        }
        s_dspill = 1;  // map full: this row's deltas go to the dense global buffer
        red_add_f32(P.d0 + row, v);
    };
    auto stepped = [&](int i) -> bool {  // column stepped earlier in the chunk (conservative)
        if (s_cfull) return true;
        int h = (int)key_hash((uint32_t)i, F.clog);
        for (int pr = 0; pr <= cmask; ++pr) {
            const int k = s_ckey[h];
            if (k == i) return true;
            if (k == -1) return false;
            h = (h + 1) & cmask;
        }
        return true;  // table full without the key: conservative
    };
    auto mark_stepped = [&](int i) {
        int h = (int)key_hash((uint32_t)i, F.clog);
        for (int pr = 0; pr <= cmask; ++pr) {
            const int k = ((volatile int*)s_ckey)[h];
            if (k == i) return;
            if (k == -1) {
                if (*(volatile int*)&s_ccount >= climit) break;
                const int prev = atomicCAS(s_ckey + h, -1, i);
                if (prev == -1) atomicAdd(&s_ccount, 1);
                if (prev == -1 || prev == i) return;
            }
            h = (h + 1) & cmask;
        }
        s_cfull = 1;
    };
    auto cur_x = [&](int i) -> float {
        return P.xlist ? ld_l2_f32((const float*)(P.blocks + (int64_t)i * G) + 2) : ld_l2_f32(P.x + i);
    };
    // entry e of a block given as lanes (staged copy or global)
    auto entry = [&](const int4* lanes, int e, bool staged) -> int2 {
        const int4 v = staged ? lanes[1 + (e >> 1)] : ld_stream_v4(lanes + 1 + (e >> 1));
        return (e & 1) ? make_int2(v.z, v.w) : make_int2(v.x, v.y);
    };
    // compute phase of one item of iteration k, one warp per item: lane e takes entry e
    // (and e + 32, ...), the corrections are summed over the warp (a thread walking the
    // entries serialised the lanes' divergent map probes: ~12 K cycles per iteration)
    auto process = [&](int q, int k) {
        const bool staged = q < nstaged;
        int i;
        float g0, x0;
        const int4* lanes;
        int4 h;
        if (staged) {
            const int4 m = s_meta[q];
            i = m.y;
            g0 = __int_as_float(m.z);
            x0 = __int_as_float(m.w);
            lanes = s_blk + (size_t)q * F.nl;
            h = lanes[0];
        } else {
            const int t = item_t(q);
            i = ld_stream_s32(P.slots + t);
            g0 = ld_l2_f32(P.g0 + t);
            lanes = P.blocks + (int64_t)i * G;
            h = ld_l2_v4(lanes);
            x0 = P.xlist ? __int_as_float(h.z) : ld_l2_f32(P.x + i);  // current x_i (this kernel writes it)
        }
        const int len = h.y;
        float corr = 0.0f;
        for (int e = lane; e < len; e += 32) {
            const int2 rv = entry(lanes, e, staged);
            const float dv = dget(real_row(rv.x, P.hot_rows));
            if (dv != 0.0f) corr += __int_as_float(rv.y) * dv;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) corr += __shfl_xor_sync(0xffffffffu, corr, o);
        if (lane != 0) return;
        const float xi = staged && stepped(i) ? cur_x(i) : x0;
        const float xp = prox_l1(xi, g0 + corr, P.beta * __int_as_float(h.x), P.lambda);
        const float d = xp - xi;
        if (d == 0.0f) return;
        if (!isfinite(xp)) atomicOr(P.flags, FLAG_DIVERGED);
        if (P.xlist) ((float*)(P.blocks + (int64_t)i * G))[2] = xp;
        else P.x[i] = xp;
        const int pos = atomicAdd(&s_nstep, 1);
        if (pos < F.scap) s_step[pos] = make_int2(q, __float_as_int(d));
        P.nz_idx[k * tau + pos] = i;
        P.nz_delta[k * tau + pos] = d;
        if (q >= nspec) s_miss = 1;
    };
    // apply phase, one warp per step e of iteration k: D, r (the fold) and the
    // stepped-column set
    auto apply = [&](int e, int k) {
        int q = -1, i;
        float d;
        if (e < F.scap) {
            const int2 st = s_step[e];
            q = st.x;
            d = __int_as_float(st.y);
            i = q < nstaged ? s_meta[q].y : ld_l2_s32(P.nz_idx + k * tau + e);
        } else {
            i = ld_l2_s32(P.nz_idx + k * tau + e);
            d = ld_l2_f32(P.nz_delta + k * tau + e);
        }
        const bool staged = q >= 0 && q < nstaged;
        const int4* lanes = staged ? s_blk + (size_t)q * F.nl : P.blocks + (int64_t)i * G;
        const int len = staged ? lanes[0].y : ld_l2_v4(lanes).y;
        for (int ee = lane; ee < len; ee += 32) {
            const int2 rv = entry(lanes, ee, staged);
            const int row = real_row(rv.x, P.hot_rows);
            const float v = __int_as_float(rv.y) * d;
            dadd(row, v);
            red_add_f32(P.r_out + row, v);
        }
        if (lane == 0) mark_stepped(i);  // (dirty-list appends: after the loop, one atomic)
    };

    const int64_t total = P.iters * tau;
    long long tclk1 = clock64(), tcomp = 0, tapply = 0;
    for (int k = 0; k < c; ++k) {
        long long ta = clock64();
        for (int p = s_start[k] + warp; p < s_start[k + 1]; p += nwarp) process(ord[p], k);
        // items added by the scans for earlier misses
        const int nextra = s_nextra;
        for (int e = warp; e < nextra; e += nwarp) {
            const int q = nit + e;
            if (item_t(q) / tau == k) process(q, k);
        }
        __syncthreads();
        long long tb = clock64();
        tcomp += tb - ta;
        const int nst = s_nstep;
        for (int e = warp; e < nst; e += nwarp) apply(e, k);
        if (tid == 0) {
            P.nz_count[k] = nst;
            s_total += nst;
        }
        __syncthreads();
        tapply += clock64() - tb;
        if (s_miss && k + 1 < c) {
            // a flagged item stepped: scan the later slots for its rows and column
            // (key batches of at most half the miss table)
            const int per = std::max(1, ((1 << F.mlog) / 2) / (1 + P.nrow));
            for (int b0 = 0; b0 < nst; b0 += per) {
                for (int w = tid; w < (1 << F.mlog); w += nth) {
                    s_mkey[w] = -1;
                    s_mstamp[w] = 0x7fffffff;
                }
                if (tid == 0) s_mcount = 0;
                __syncthreads();
                for (int e = b0 + tid; e < std::min(nst, b0 + per); e += nth) {
                    const int q = e < F.scap ? s_step[e].x : -1;
                    if (q >= 0 && q < nspec) continue;  // speculative: already tested against
                    const int i = ld_l2_s32(P.nz_idx + k * tau + e);
                    const int4* lanes = P.blocks + (int64_t)i * G;
                    const int len = ld_l2_v4(lanes).y;
                    stamp_insert(s_mkey, s_mstamp, F.mlog, i | kColKey, k);
                    for (int ee = 0; ee < len; ++ee)
                        stamp_insert(s_mkey, s_mstamp, F.mlog, real_row(entry(lanes, ee, false).x, P.hot_rows), k);
                    atomicAdd(&s_mcount, 1);
                }
                __syncthreads();
                if (s_mcount > 0) {
                    test_slots(P, s_mkey, s_mstamp, F.mlog, nullptr, 0, (int64_t)(k + 1) * tau, total, tid, nth, cand + ncand,
                               &s_nextra);
                    if (tid == 0) ++s_nscan;
                }
                __syncthreads();
            }
            if (tid == 0) ++s_nmiss;
        }
        if (tid == 0) {
            s_nstep = 0;
            s_miss = 0;
        }
        __syncthreads();
    }
    // the chunk's stepped columns onto the x dirty list: one atomic for all of them
    if (P.xlist && P.xlist_cap > 0 && s_total > 0) {
        if (tid == 0) {
            s_xbase = atomicAdd(P.xlist_count, (unsigned long long)s_total);
            int run = 0;
            for (int k = 0; k < c; ++k) {
                s_cur[k] = run;
                run += ld_l2_s32(P.nz_count + k);
            }
        }
        __syncthreads();
        const unsigned long long base = s_xbase;
        for (int k = 0; k < c; ++k) {
            const int cnt = ld_l2_s32(P.nz_count + k);
            for (int e = tid; e < cnt; e += nth) {
                const unsigned long long qq = base + s_cur[k] + e;
                if (qq < (unsigned long long)P.xlist_cap) P.xlist[qq] = ld_l2_s32(P.nz_idx + k * tau + e);
            }
        }
    }
    // clear what the chunk left: spilled D rows, the item bits, the item counters
    if (s_dspill) {
        for (int k = 0; k < c; ++k) {
            const int cnt = ld_l2_s32(P.nz_count + k);
            for (int e = tid; e < cnt; e += nth) {
                const int i = ld_l2_s32(P.nz_idx + k * tau + e);
                const int4* lanes = P.blocks + (int64_t)i * G;
                const int len = ld_l2_v4(lanes).y;
                for (int ee = 0; ee < len; ++ee) P.d0[real_row(entry(lanes, ee, false).x, P.hot_rows)] = 0.0f;
            }
        }
    }
    for (int q = tid; q < nit + s_nextra; q += nth) P.bits[item_t(q) >> 5] = 0u;
    __syncthreads();
    if (tid == 0) {
        P.counts[0] = 0;
        P.counts[1] = 0;
        P.counts[2] += s_nmiss;
        P.counts[3] += s_nscan;
        P.counts[4] += nspec;
        P.counts[5] += ncand + s_nextra;
        P.counts[6] += (int)((tclk1 - tclk0) >> 10);
        P.counts[7] += (int)(tcomp >> 10);
        P.counts[8] += (int)(tapply >> 10);
        P.counts[9] += (int)((clock64() - tclk1) >> 10);
        if (s_total) atomicAdd(P.nz_total, (unsigned long long)s_total);
    }
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

// the fix-up's shared-memory shape: D map 2^13 rows, 2^11 stepped columns, 1024 steps
// per iteration, a 2^10-key miss table; the rest stages items (PCDM_SCREEN_SMALL=1: tiny
// maps and staging, so that tests reach the spill and global paths)
FixShape fix_shape(const BatchedParams& P, int G) {
    FixShape F;
    F.nl = std::min(G, 1 + (P.nrow + 1) / 2);
    F.c = (int)P.iters;
    const char* sm = knob("PCDM_SCREEN_SMALL");
    if (sm && atoi(sm) != 0) {
        F.dlog = 4;
        F.clog = 3;
        F.scap = 2;
        F.mlog = 5;
        F.icap = 3;
        return F;
    }
    F.dlog = 13;
    F.clog = 11;
    F.scap = 1024;
    F.mlog = 10;
    F.icap = 0;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t fixed = fix_smem_bytes(F) + 1024;  // + static shared memory
    const size_t per = (size_t)16 * (1 + F.nl) + 4;
    if ((size_t)optin > fixed) F.icap = (int)std::min<size_t>(((size_t)optin - fixed) / per, 1 << 20);
    return F;
}

template <int G>
size_t expand_smem(int cq_log, int nb) {
    const size_t ne = (size_t)1 << cq_log;
    const size_t n = ne * 2 * (G - 1);
    return n * sizeof(int2) + ((n + 7) & ~(size_t)7) * 2 + (size_t)((2 * nb + 2) & ~1) * sizeof(int) + ne * sizeof(int2);
}

template <int G>
cudaError_t launch_all(const BatchedParams& P0, int ctas3, cudaStream_t st, int sms, int64_t* launches,
                       const ScreenSched* sch) {
    cudaError_t e;
    // slot records: P.rnv 16-byte vectors (rows 2 + 4 (rnv - 1) >= max column length);
    // the G-lane-group step kernel reads G / 2
    BatchedParams P = P0;
    P.G = G;
    if (step_kernel<G>(P.logistic) == (P.logistic ? (const void*)pcdm_batched_kernel<G, true>
                                                  : (const void*)pcdm_batched_kernel<G, false>))
        P.rnv = G / 2;
    P.rnv = std::max(1, std::min(P.rnv, G / 2));
    if (P.screen && P.logistic) P.screen = 0;  // dense steps: the grid-barrier pass
    const size_t sm1 = expand_smem<G>(P.cq_log, P.nb);
    e = cudaFuncSetAttribute(batch_expand_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    if (e != cudaSuccess) return e;
    int per1 = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, batch_expand_kernel<G>, kExpandThreads, sm1);
    // screened with the fix-up on its own stream: the expand leaves one SM to the previous
    // chunk's fix-up (one CTA that needs a whole SM), else two of its persistent CTAs would
    // start only after the fix-up and finish last
    const int esms = P.screen && sch && sms > 1 ? sms - 1 : sms;
    if (const char* v = knob("PCDM_EXPAND_PER_SM")) per1 = std::max(1, std::min(per1, atoi(v)));
    const int g1 = std::min(P.nq, std::max(1, per1) * esms);
    batch_expand_kernel<G><<<g1, kExpandThreads, sm1, st>>>(P);
    // the sweep reads r and (for the speculative steps) x: after the previous fix-up
    if (P.screen && sch) {
        e = cudaStreamWaitEvent(st, sch->ev_fix, 0);
        if (e != cudaSuccess) return e;
    }
    // pass 2: groups of qpc slot ranges per CTA, g0 accumulated in shared memory
    int sweep_per_sm = 2, sweep_max = kSweepMaxSlots;
    if (const char* v = knob("PCDM_SWEEP_PER_SM")) {
        sweep_per_sm = std::max(1, std::min(2, atoi(v)));
        if (sweep_per_sm == 1) sweep_max = 2 * kSweepMaxSlots;  // one CTA per SM: twice the accumulators
    }
    const int qpc = std::max(1, std::min(sweep_max >> P.cq_log, (P.nq + sweep_per_sm * sms - 1) / (sweep_per_sm * sms)));
    const size_t sm2 = ((size_t)qpc << P.cq_log) * sizeof(float) + ((size_t)1 << (kStaleLog - 3));
    const void* sw = P.logistic ? (const void*)batch_sweep_kernel<true> : (const void*)batch_sweep_kernel<false>;
    e = cudaFuncSetAttribute(sw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    if (e != cudaSuccess) return e;
    const int ngrp = (P.nq + qpc - 1) / qpc;
    if (P.logistic)
        batch_sweep_kernel<true><<<std::min(ngrp, sweep_per_sm * sms), kThreads, sm2, st>>>(P, qpc);
    else
        batch_sweep_kernel<false><<<std::min(ngrp, sweep_per_sm * sms), kThreads, sm2, st>>>(P, qpc);
    if (P.screen) {
        const size_t smt = ((size_t)8 << kTestLog) + ((size_t)1 << (kTestBmLog - 3));
        e = cudaFuncSetAttribute(screen_test_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smt);
        if (e != cudaSuccess) return e;
        screen_test_kernel<G><<<sms, kTestThreads, smt, st>>>(P);
        FixShape F = fix_shape(P, G);
        const size_t smf = fix_smem_bytes(F);
        e = cudaFuncSetAttribute(screen_fix_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf);
        if (e != cudaSuccess) return e;
        cudaStream_t sf = st;
        if (sch) {
            if ((e = cudaEventRecord(sch->ev_test, st)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(sch->st2, sch->ev_test, 0)) != cudaSuccess) return e;
            sf = sch->st2;
        }
        screen_fix_kernel<G><<<1, kTestThreads, smf, sf>>>(P, F);
        if (sch && (e = cudaEventRecord(sch->ev_fix, sf)) != cudaSuccess) return e;
        *launches += 4;
        return cudaGetLastError();
    }
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

cudaError_t launch_batched(int G, const BatchedParams& P, int ctas3, cudaStream_t st, int sms, int64_t* launches,
                           const ScreenSched* sch) {
    switch (G) {
        case 2: return launch_all<2>(P, ctas3, st, sms, launches, sch);
        case 4: return launch_all<4>(P, ctas3, st, sms, launches, sch);
        case 8: return launch_all<8>(P, ctas3, st, sms, launches, sch);
        case 16: return launch_all<16>(P, ctas3, st, sms, launches, sch);
        default: return launch_all<32>(P, ctas3, st, sms, launches, sch);
    }
}

}  // namespace pcdm_internal
