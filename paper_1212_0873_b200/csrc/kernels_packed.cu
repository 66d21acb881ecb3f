// kernels_packed.cu -- the PCDM1 hot loop on packed column blocks (PACKED variant).
//
// Why: on B200 a random global access costs one DRAM line activation whatever
// its width (measured: ~54 G random accesses/s from a 400 MB array, the same
// with 64 B or 128 B L2 fetches), so the hot loop is bounded by the number of
// distinct random lines touched per sampled column, not by bytes.  The CSC
// layout touches colptr, rowidx, val, L and x on separate lines (4-6 random
// lines) besides the c gathers of r.  Here column i is one slot of G x 16 B:
//
//   chunk 0       { L_i (f32), len (i32), 0, 0 }
//   chunk t >= 1  { row_{2t-2}, val_{2t-2}, row_{2t-1}, val_{2t-1} }   (pairs beyond len unused)
//
// with G = pow2 >= 1 + ceil(maxlen/2) lanes per column: one coalesced
// G x 16 B load per column (128 B for c = 10), each lane then gathers <= 2
// entries of r.  The arithmetic is the same synchronous PCDM1 step as
// kernels_iter.cu (alg:PCD1 PAPER.md:177-186; g_i = a_i^T r_k, soft-threshold
// block update eq:h(x) PAPER.md:214-216).
//
// Barrier schemes:
//   TWO_BARRIER  one residual buffer: phase A (gathers, steps, list of nonzero
//                steps) | barrier | phase B (r += delta a_i for the list) | barrier.
//   ONE_BARRIER  two residual buffers P = r_k (read-only in iteration k) and
//                Q = r_{k-1}: iteration k gathers from P and scatters both its
//                own steps Delta_k and the previous iteration's list Delta_{k-1}
//                into Q, so after ONE barrier Q = r_{k-1} + Delta_{k-1} + Delta_k
//                = r_{k+1} and the buffers swap (the default).  The replay of
//                Delta_{k-1} is issued at the start of iteration k, so its dependent
//                loads overlap the gathers; the first slot of iteration k+1 (S and its
//                block do not depend on r) is loaded between barrier arrival and wait.
// Step lists rotate over 3 buffers (append k%3, replay (k-1)%3, reset (k+1)%3).
//
// Hot rows (skewed row distributions, e.g. the Zipf config): a row stored in a
// large fraction of the columns is read by that fraction of all sampled columns
// every iteration, and same-address L2 requests serialise in one L2 slice.  The
// rows stored >= a threshold times (chosen at create from the row histogram) are
// encoded in the blocks as 0x80000000 | h; every CTA with work copies
// r_k[hot_rows[h]] into shared memory at the start of the iteration (r_k is
// read-only during iteration k in both barrier schemes) and gathers hot entries
// from there; scatters go to the real row hot_rows[h].
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

using namespace pcdm;
using namespace pcdm_internal;

namespace {

constexpr int kThreads = 512;

// L2 (coherent) 16-byte load: column blocks whose header holds the mutable x_i
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

template <int G>
__device__ __forceinline__ unsigned gmask_of() {
    if constexpr (G == 32) {
        return 0xffffffffu;
    } else {
        const unsigned lane = threadIdx.x & 31;
        return ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
    }
}

// real row of a block entry (hot rows stored as 0x80000000 | h)
__device__ __forceinline__ int real_row(int v, const int* hrow) { return v < 0 ? hrow[v & 0x7fffffff] : v; }

// r[row] += val * d for this lane's (<= 2) pairs of the chunk.
__device__ __forceinline__ void scatter_chunk(float* r, const int4 c, int pair0, int len, float d, const int* hrow) {
    if (pair0 < len) red_add_f32(r + real_row(c.x, hrow), __int_as_float(c.y) * d);
    if (pair0 + 1 < len) red_add_f32(r + real_row(c.z, hrow), __int_as_float(c.w) * d);
}

// Scatter with the hot rows staged (P.hot_stage): contributions to a hot row go to the
// CTA's shared-memory accumulator s_hacc[h] (shared atomics, no same-address L2
// serialisation across the grid), flushed with one red.global.add per touched hot row
// and CTA before the iteration's barrier; other rows as scatter_chunk.
__device__ __forceinline__ void scatter_chunk_staged(float* r, const int4 c, int pair0, int len, float d,
                                                     const int* hrow, float* s_hacc) {
    if (pair0 < len) {
        const float v = __int_as_float(c.y) * d;
        if (c.x < 0) atomicAdd(s_hacc + (c.x & 0x7fffffff), v);
        else red_add_f32(r + c.x, v);
    }
    if (pair0 + 1 < len) {
        const float v = __int_as_float(c.w) * d;
        if (c.z < 0) atomicAdd(s_hacc + (c.z & 0x7fffffff), v);
        else red_add_f32(r + c.z, v);
    }
}

// gathered r entry (hot rows from the shared-memory copy, or through the row table
// when the run does not cache them)
__device__ __forceinline__ float gather_r(const float* rP, int v, const float* s_hot, const int* s_hrow, bool cache) {
    if (v >= 0) return ld_l2_f32(rP + v);
    return cache ? s_hot[v & 0x7fffffff] : ld_l2_f32(rP + s_hrow[v & 0x7fffffff]);
}

#ifndef PCDM_PACKED_MINB
#define PCDM_PACKED_MINB 3  // CTAs of 512 threads per SM (register cap 40)
#endif
template <int G, bool ONE_BARRIER, bool LOGISTIC, int TPB = kThreads>
__global__ void __launch_bounds__(TPB, TPB == kThreads ? PCDM_PACKED_MINB : 1) pcdm_packed_kernel(PackedParams P) {
    const int t = threadIdx.x & (G - 1);  // lane within the column group
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
    const int pair0 = 2 * (t - 1);
    unsigned bar_target = 0;
    const int64_t tau = P.tau;
    extern __shared__ float s_dyn[];
    float* s_hot = s_dyn;                      // [nhot] r_k at the hot rows
    int* s_hrow = (int*)(s_dyn + P.nhot);      // [nhot] hot row ids
    const int nhot = P.nhot;
    // staged step list (P.list_cap > 0): [list_cap] ids, [list_cap] steps, count, base
    // CTA-local replay (P.local_cap > 0, one-barrier scheme): the slots of a CTA are the same
    // positions of every iteration, so the CTA that took a step replays it; its steps stay in
    // shared memory (3 rotating lists: append k%3, replay (k-1)%3, reset (k+1)%3), no global
    // step list, no list counter to read after the barrier
    const bool local = ONE_BARRIER && P.local_cap > 0;
    const bool stage = !local && P.list_cap > 0;
    int* s_li = s_hrow + nhot;
    float* s_ld = (float*)(s_li + P.list_cap);
    int* s_lc = (int*)(s_ld + P.list_cap);
    int* s_lbase = s_lc + 1;
    // staged hot-row scatters (P.hot_stage, one-barrier scheme): [nhot] accumulators
    float* s_hacc = stage ? (float*)(s_lbase + 1) : (float*)(s_hrow + nhot);
    const bool hstage = ONE_BARRIER && P.hot_stage && nhot > 0;
    const int lcap = P.local_cap;
    int* s_rcnt = (int*)(s_hacc + (P.hot_stage ? nhot : 0));  // [4]: 3 list counts
    int* s_ri = s_rcnt + 4;                                    // [3][lcap] column ids
    float* s_rd = (float*)(s_ri + 3 * lcap);                   // [3][lcap] steps
    unsigned nzl = 0;                                          // thread 0: the CTA's nonzero steps
    if (local && threadIdx.x < 3) s_rcnt[threadIdx.x] = 0;
    if (stage && threadIdx.x == 0) *s_lc = 0;
    if (hstage)
        for (int h = threadIdx.x; h < nhot; h += blockDim.x) s_hacc[h] = 0.0f;
    const bool cache = P.hot_cache != 0;
    // CTAs without slots in an iteration skip the hot-row copy
    const bool has_slots = (int64_t)blockIdx.x * (blockDim.x / G) < tau;
    if (nhot || stage || local) {
        for (int h = threadIdx.x; h < nhot; h += blockDim.x) s_hrow[h] = P.hot_rows[h];
        __syncthreads();
    }
    // a step list of the CTA replayed into `dst` (a group of G lanes per entry)
    auto replay_local = [&](int list, float* dst, bool staged) {
        const int cnt = s_rcnt[list];
        for (int e = threadIdx.x / G; e < cnt; e += blockDim.x / G) {
            const int i = s_ri[list * lcap + e];
            const float d = s_rd[list * lcap + e];
            const int4 c = ld_stream_v4(P.blocks + (int64_t)i * G + t);
            const int len = __shfl_sync(gm, c.y, src);
            if (t > 0) {
                if (staged) scatter_chunk_staged(dst, c, pair0, len, d, s_hrow, s_hacc);
                else scatter_chunk(dst, c, pair0, len, d, s_hrow);
            }
        }
    };

    // software pipeline: slot gid of iteration it and its block, loaded one iteration ahead
    // (pipelined slot loop: also the id of the group's second slot, so that no block load
    // waits for its slot id inside the loop)
    int i_pf = -1, i_pf2 = -1;
    int4 c_pf = make_int4(0, 0, 0, 0);
    auto prefetch = [&](int64_t it) {
        i_pf = -1;
        i_pf2 = -1;
        if (it < P.iters && gid < tau) {
            i_pf = ld_stream_s32(P.slots + it * tau + gid);
            if (P.pipeline && gid + ngroups < tau) i_pf2 = ld_stream_s32(P.slots + it * tau + gid + ngroups);
            if (i_pf >= 0)
                c_pf = P.xlist ? ld_l2_v4(P.blocks + (int64_t)i_pf * G + t) : ld_stream_v4(P.blocks + (int64_t)i_pf * G + t);
        }
    };
    prefetch(0);

    for (int64_t it = 0; it < P.iters; ++it) {
        const int64_t k = P.k0 + it;
        const int cur = (int)(k % 3), prev = (int)((k + 2) % 3), next = (int)((k + 1) % 3);
        const float* rP = (ONE_BARRIER && (k & 1)) ? P.r1 : P.r0;
        float* rQ = (ONE_BARRIER && (k & 1)) ? P.r0 : P.r1;
        const int* S = P.slots + it * tau;
        if (!local && blockIdx.x == 0 && threadIdx.x == 0) P.nz_count[next] = 0;
        if (local) {
            if (threadIdx.x == 0) s_rcnt[next] = 0;  // replayed in iteration k-1, before its barrier
            replay_local(prev, rQ, hstage);
        } else if (ONE_BARRIER) {
            // replay the previous iteration's nonzero steps into Q (first, so that its
            // dependent loads overlap phase A instead of following it)
            const int cntp = ld_l2_s32(P.nz_count + prev);
            for (int64_t e = gid; e < cntp; e += ngroups) {
                const int i = ld_l2_s32(P.nz_idx + prev * tau + e);
                const float d = ld_l2_f32(P.nz_delta + prev * tau + e);
                const int4 c = ld_stream_v4(P.blocks + (int64_t)i * G + t);
                const int len = __shfl_sync(gm, c.y, src);
                if (t > 0) {
                    if (hstage) scatter_chunk_staged(rQ, c, pair0, len, d, s_hrow, s_hacc);
                    else scatter_chunk(rQ, c, pair0, len, d, s_hrow);
                }
            }
        }
        if (cache && has_slots) {
            // the previous iteration's readers of s_hot passed the grid barrier's __syncthreads
            for (int h = threadIdx.x; h < nhot; h += blockDim.x) s_hot[h] = ld_l2_f32(rP + s_hrow[h]);
            __syncthreads();
        }

        // ---------------- phase A: one coalesced block load + <= 2 gathers per lane
        // Software pipeline over this group's slots: the next slot's id and block are
        // loaded before the current slot's gathers.  The first slot was loaded before
        // the previous barrier (S_k and A do not depend on r), so only its x_i, which a
        // step of iteration k-1 may have changed, is read again; later blocks are loaded
        // inside iteration k, after that barrier, and no other slot of iteration k changes
        // their column (the slots of one iteration are distinct).
        // (P.pipeline = 0, for DRAM-bound r: each block is loaded when its slot comes up)
        // x_i lives in the block header (chunk 0 .z) when P.xlist: the column's single line
        // brings it, no separate random x line; the header is then mutable, so the block is
        // read through L2 (ld.cg) instead of the non-coherent path
        auto load_block = [&](int col) {
            return P.xlist ? ld_l2_v4(P.blocks + (int64_t)col * G + t) : ld_stream_v4(P.blocks + (int64_t)col * G + t);
        };
        const bool pipeline = P.pipeline != 0;
        // pipelined: (i_cur, c_cur) = the slot being processed, i_n1 = the id of the next one
        // (loaded a slot ago), whose block is issued now; the id after that is issued too
        int i_cur = i_pf, i_n1 = i_pf2;
        int4 c_cur = c_pf;
        for (int64_t j = gid; j < tau; j += ngroups) {
            const bool first = j == gid;
            int i;
            int4 c;
            if (first || pipeline) {
                i = i_cur;
                c = c_cur;
            } else {
                i = ld_stream_s32(S + j);
                if (i >= 0) c = load_block(i);
            }
            const int64_t jn = j + ngroups;
            if (pipeline && jn < tau) {
                if (i_n1 >= 0) c_cur = load_block(i_n1);
                i_cur = i_n1;
                i_n1 = jn + ngroups < tau ? ld_stream_s32(S + jn + ngroups) : -1;
            }
            if (i < 0) continue;  // idle processor (non-nice samplings)
            float xi = 0.0f;
            if (t == 0) {
                if (!P.xlist) xi = ld_l2_f32(P.x + i);
                else xi = first ? ld_l2_f32((const float*)(P.blocks + (int64_t)i * G) + 2) : __int_as_float(c.z);
            }
            const int len = __shfl_sync(gm, c.y, src);
            float acc = 0.0f;
            if (t > 0) {
                const float ra = pair0 < len ? grad_weight<LOGISTIC>(gather_r(rP, c.x, s_hot, s_hrow, cache)) : 0.0f;
                const float rb = pair0 + 1 < len ? grad_weight<LOGISTIC>(gather_r(rP, c.z, s_hot, s_hrow, cache)) : 0.0f;
                acc = fmaf(__int_as_float(c.y), ra, __int_as_float(c.w) * rb);
            }
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gm, acc, o);
            float d = 0.0f;
            if (t == 0) {
                const float xp = block_step<LOGISTIC>(xi, acc, P.beta * __int_as_float(c.x), P.lambda);
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
                    if (local) {
                        const int pos = atomicAdd(s_rcnt + cur, 1);
                        s_ri[cur * lcap + pos] = i;
                        s_rd[cur * lcap + pos] = d;
                    } else if (stage) {  // CTA-local list, flushed with one global atomic per CTA
                        const int pos = atomicAdd(s_lc, 1);
                        s_li[pos] = i;
                        s_ld[pos] = d;
                    } else {
                        const int pos = atomicAdd(P.nz_count + cur, 1);
                        P.nz_idx[cur * tau + pos] = i;
                        P.nz_delta[cur * tau + pos] = d;
                    }
                }
            }
            if (ONE_BARRIER) {
                d = __shfl_sync(gm, d, src);
                if (d != 0.0f && t > 0) {
                    if (hstage) scatter_chunk_staged(rQ, c, pair0, len, d, s_hrow, s_hacc);
                    else scatter_chunk(rQ, c, pair0, len, d, s_hrow);
                }
            }
        }
        if (hstage) {
            // flush the CTA's hot-row sums into Q before the barrier publishes it
            __syncthreads();
            for (int h = threadIdx.x; h < nhot; h += blockDim.x) {
                const float v = s_hacc[h];
                if (v != 0.0f) {
                    red_add_f32(rQ + s_hrow[h], v);
                    s_hacc[h] = 0.0f;
                }
            }
        }
        if (stage) {
            __syncthreads();
            const int cnt = *s_lc;
            if (threadIdx.x == 0 && cnt) *s_lbase = atomicAdd(P.nz_count + cur, cnt);
            __syncthreads();
            for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
                P.nz_idx[cur * tau + *s_lbase + e] = s_li[e];
                P.nz_delta[cur * tau + *s_lbase + e] = s_ld[e];
            }
            __syncthreads();
            if (threadIdx.x == 0) *s_lc = 0;  // ordered before the next appends by the barrier
        }
        if (ONE_BARRIER && P.cluster_sync) {
            // a grid of one thread-block cluster: the hardware cluster barrier (release /
            // acquire at cluster scope, which covers the global-memory r, x and lists)
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            prefetch(it + 1);
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else if (ONE_BARRIER) {
            // the next iteration's first slot is loaded while the other CTAs arrive
            grid_arrive(P.barrier, bar_target);
            prefetch(it + 1);
            grid_wait(P.barrier, bar_target);
        } else {
            grid_barrier(P.barrier, bar_target);
            const int cnt = ld_l2_s32(P.nz_count + cur);
            for (int64_t e = gid; e < cnt; e += ngroups) {
                const int i = ld_l2_s32(P.nz_idx + cur * tau + e);
                const float d = ld_l2_f32(P.nz_delta + cur * tau + e);
                const int4 c = ld_stream_v4(P.blocks + (int64_t)i * G + t);
                const int len = __shfl_sync(gm, c.y, src);
                if (t > 0) scatter_chunk(P.r0, c, pair0, len, d, s_hrow);
            }
            grid_arrive(P.barrier, bar_target);
            prefetch(it + 1);
            grid_wait(P.barrier, bar_target);
        }
        if (local) {
            if (threadIdx.x == 0) nzl += (unsigned)s_rcnt[cur];  // complete since the barrier's __syncthreads
        } else if (blockIdx.x == 0 && threadIdx.x == 0) {
            const int cnt = ld_l2_s32(P.nz_count + cur);
            if (cnt) atomicAdd(P.nz_total, (unsigned long long)cnt);
        }
    }
    if (local && P.iters > 0) {
        // the last iteration's steps into the other buffer as well: both buffers leave the
        // launch equal to r_{k0+iters}, the next launch has nothing to replay
        replay_local((int)((P.k0 + P.iters - 1) % 3), ((P.k0 + P.iters) & 1) ? P.r0 : P.r1, false);
        if (threadIdx.x == 0 && nzl) atomicAdd(P.nz_total, (unsigned long long)nzl);
    }
}

// ---------------------------------------------------------------- one slot per group
// The one-barrier loop for grids that cover tau in one round (every group of G lanes owns
// at most one slot per iteration: the small-tau, latency-bound configs).  The group that
// took the step of iteration k-1 still holds that column's chunk and delta in registers,
// so the replay of Delta_{k-1} into Q needs no step list: no list counter to read after
// the barrier, no dependent list and block loads before the replay's scatters, no append
// atomics.  An iteration's dependent chain is then: barrier -> gathers of r_k (and x_i)
// -> shuffles, step -> scatters -> barrier.  The dirty-list append of a changed x_i (read
// only after the launch) is issued between barrier arrival and wait.  After the last
// iteration the last step is also added to the other buffer, so both buffers leave the
// launch equal to r_{k0+iters} and the next launch has nothing to replay; nonzero steps
// are counted in registers.  Same arithmetic as pcdm_packed_kernel (alg:PCD1
// PAPER.md:177-186; eq:h(x) PAPER.md:214-216).
template <int G, bool LOGISTIC, int TPB = kThreads>
__global__ void __launch_bounds__(TPB, TPB == kThreads ? PCDM_PACKED_MINB : 1) pcdm_packed1_kernel(PackedParams P) {
    const int t = threadIdx.x & (G - 1);
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int pair0 = 2 * (t - 1);
    unsigned bar_target = 0;
    const int64_t tau = P.tau;
    extern __shared__ float s_dyn[];
    float* s_hot = s_dyn;                  // [nhot] r_k at the hot rows
    int* s_hrow = (int*)(s_dyn + P.nhot);  // [nhot] hot row ids
    const int nhot = P.nhot;
    const bool cache = P.hot_cache != 0;
    const bool has_slots = (int64_t)blockIdx.x * (blockDim.x / G) < tau;
    if (nhot) {
        for (int h = threadIdx.x; h < nhot; h += blockDim.x) s_hrow[h] = P.hot_rows[h];
        __syncthreads();
    }
    // S and A do not depend on r: the slot id is loaded two iterations ahead and its block
    // one iteration ahead (at the start of the iteration before), so neither load sits on
    // the barrier-to-barrier chain (ncu on medium: the id -> block chain issued after the
    // barrier arrival was 25 % of the warp samples)
    const bool mine = gid < tau;
    auto slot_of = [&](int64_t it) { return it < P.iters && mine ? ld_stream_s32(P.slots + it * tau + gid) : -1; };
    auto block_of = [&](int col) {
        if (col < 0) return make_int4(0, 0, 0, 0);  // idle: length 0
        return P.xlist ? ld_l2_v4(P.blocks + (int64_t)col * G + t) : ld_stream_v4(P.blocks + (int64_t)col * G + t);
    };
    int i_cur = slot_of(0);
    int4 c_cur = block_of(i_cur);
    int i_nx = slot_of(1);
    int4 c_prev = make_int4(0, 0, 0, 0);
    float d_prev = 0.0f;
    int len_prev = 0;
    unsigned nzl = 0;
    int xl_i = -1;  // changed column whose dirty-list append is pending
    constexpr unsigned kFull = 0xffffffffu;  // every lane reaches the shuffles (idle groups carry zeros)

    for (int64_t it = 0; it < P.iters; ++it) {
        const int64_t k = P.k0 + it;
        const float* rP = (k & 1) ? P.r1 : P.r0;
        float* rQ = (k & 1) ? P.r0 : P.r1;
        const int4 c_nx = block_of(i_nx);
        const int i_nx2 = slot_of(it + 2);
        if (cache && has_slots) {
            // the previous iteration's readers of s_hot passed the barrier's __syncthreads
            for (int h = threadIdx.x; h < nhot; h += blockDim.x) s_hot[h] = ld_l2_f32(rP + s_hrow[h]);
            __syncthreads();
        }
        const int i = i_cur;
        const int4 c = c_cur;
        const bool act = i >= 0;
        // the gathers first: everything below overlaps their latency
        // (issuing the plain-row gathers before the hot-row copy and reading the hot entries
        // after it measured slower: medium 26.0 -> 38.6, skewed tau = 2^12 38.3 -> 50.6 ms per
        // 1e4 iterations, profiles/r02_reg_replay_ab.jsonl)
        float xi = 0.0f, ra = 0.0f, rb = 0.0f;
        // x_i may have been changed by iteration k-1 after the block was loaded
        if (act && t == 0) xi = P.xlist ? ld_l2_f32((const float*)(P.blocks + (int64_t)i * G) + 2) : ld_l2_f32(P.x + i);
        const int len = __shfl_sync(kFull, c.y, src);
        if (t > 0) {
            if (pair0 < len) ra = gather_r(rP, c.x, s_hot, s_hrow, cache);
            if (pair0 + 1 < len) rb = gather_r(rP, c.z, s_hot, s_hrow, cache);
        }
        // replay this group's step of iteration k-1 into Q, from registers
        if (d_prev != 0.0f && t > 0) scatter_chunk(rQ, c_prev, pair0, len_prev, d_prev, s_hrow);
        float acc = 0.0f;
        if (t > 0) {
            const float wa = pair0 < len ? grad_weight<LOGISTIC>(ra) : 0.0f;
            const float wb = pair0 + 1 < len ? grad_weight<LOGISTIC>(rb) : 0.0f;
            acc = fmaf(__int_as_float(c.y), wa, __int_as_float(c.w) * wb);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        float d = 0.0f;
        if (act && t == 0) {
            const float xp = block_step<LOGISTIC>(xi, acc, P.beta * __int_as_float(c.x), P.lambda);
            d = xp - xi;
            if (d != 0.0f) {
                if (!isfinite(xp)) atomicOr(P.flags, FLAG_DIVERGED);
                if (P.xlist) {
                    ((float*)(P.blocks + (int64_t)i * G))[2] = xp;
                    if (P.xlist_cap > 0) xl_i = i;  // 0: dense iterate, no dirty list
                } else {
                    P.x[i] = xp;
                }
                ++nzl;
            }
        }
        d = __shfl_sync(kFull, d, src);
        if (d != 0.0f && t > 0) scatter_chunk(rQ, c, pair0, len, d, s_hrow);
        c_prev = c;
        d_prev = d;
        len_prev = len;
        if (P.cluster_sync) {
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        } else {
            grid_arrive(P.barrier, bar_target);
        }
        if (xl_i >= 0) {
            const unsigned long long q = atomicAdd(P.xlist_count, 1ull);
            if (q < (unsigned long long)P.xlist_cap) P.xlist[q] = xl_i;
            xl_i = -1;
        }
        i_cur = i_nx;
        c_cur = c_nx;
        i_nx = i_nx2;
        if (P.cluster_sync) {
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            grid_wait(P.barrier, bar_target);
        }
    }
    // the last step into the other buffer as well (every gather of it passed the barrier)
    if (d_prev != 0.0f && t > 0) {
        float* rO = ((P.k0 + P.iters) & 1) ? P.r0 : P.r1;
        scatter_chunk(rO, c_prev, pair0, len_prev, d_prev, s_hrow);
    }
    if (nzl) atomicAdd(P.nz_total, (unsigned long long)nzl);
}

// ---------------------------------------------------------------- asynchronous variant
// What the paper's experiments ran: every worker repeatedly picks a
// coordinate uniformly at random and updates it from whatever r currently holds, with
// no barrier between workers.  Here a worker is a group of G lanes; update u (global
// index, u = u0 .. u0 + updates - 1) is done by group u mod ngroups and picks
// i = Lemire(Philox(counter (u lo, u hi, rho, tag 6), key seed)).  x_i and r are
// updated with atomics (x_i += delta, r += delta a_i) so that r = Ax - b is kept
// whatever the interleaving; the result is not deterministic (measured, not
// oracle-checked; R20).
template <int G>
__global__ void __launch_bounds__(kThreads, 3) pcdm_async_kernel(AsyncParams A) {
    const int t = threadIdx.x & (G - 1);
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
    const int pair0 = 2 * (t - 1);
    unsigned long long nz = 0;
    for (int64_t q = gid; q < A.updates; q += ngroups) {
        const uint64_t u = (uint64_t)(A.u0 + q);
        int i = 0;
        if (t == 0) {
            long long v;
            uint32_t rho = 0;
            do {
                u32x4 o = philox4x32_10(u32x4{(uint32_t)u, (uint32_t)(u >> 32), rho, 6u}, (uint32_t)A.seed,
                                        (uint32_t)(A.seed >> 32));
                const uint64_t w = ((uint64_t)o.y << 32) | (uint64_t)o.x;
                v = (w * (uint64_t)A.n < A.reject_below) ? -1 : (long long)__umul64hi(w, (uint64_t)A.n);
                ++rho;
            } while (v < 0);
            i = (int)v;
        }
        i = __shfl_sync(gm, i, src);
        float xi = 0.0f;
        if (t == 0) xi = ld_l2_f32(A.x + i);
        const int4 c = ld_stream_v4(A.blocks + (int64_t)i * G + t);
        const int len = __shfl_sync(gm, c.y, src);
        float acc = 0.0f;
        if (t > 0) {
            const float ra = pair0 < len ? ld_l2_f32(A.r + real_row(c.x, A.hot_rows)) : 0.0f;
            const float rb = pair0 + 1 < len ? ld_l2_f32(A.r + real_row(c.z, A.hot_rows)) : 0.0f;
            acc = fmaf(__int_as_float(c.y), ra, __int_as_float(c.w) * rb);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gm, acc, o);
        float d = 0.0f;
        if (t == 0) {
            const float xp = prox_l1(xi, acc, A.beta * __int_as_float(c.x), A.lambda);
            d = xp - xi;
            if (d != 0.0f) {
                if (!isfinite(xp)) atomicOr(A.flags, FLAG_DIVERGED);
                atomicAdd(A.x + i, d);
                ++nz;
            }
        }
        d = __shfl_sync(gm, d, src);
        if (d != 0.0f && t > 0) scatter_chunk(A.r, c, pair0, len, d, A.hot_rows);
    }
    if (nz) atomicAdd(A.nz_total, nz);
}

// ---------------------------------------------------------------- x in the block headers
// The run keeps x_i in chunk 0 .z of column i's block.  The dirty list D (indices
// whose header may be nonzero; duplicates allowed) ties the headers to the
// caller's x:  run start: headers of D zeroed, D cleared, every nonzero x_i copied
// into its header and appended to D (by the residual pass, kernels_setup.cu);
// during the run every changed i is appended;
// refresh / run end: x_i = header for i in D.  If D overflows its capacity the
// start / end passes walk all n columns instead.
__global__ void xhdr_clear_kernel(int4* __restrict__ blocks, int G, const long long* __restrict__ off,
                                  const int* __restrict__ list,
                                  const unsigned long long* __restrict__ count, int64_t cap, int64_t n) {
    const unsigned long long c = *count;
    const bool all = c > (unsigned long long)cap;
    const int64_t total = all ? n : (int64_t)c;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = all ? t : list[t];
        ((float*)(blocks + (off ? off[i] : i * G)))[2] = 0.0f;
    }
}

__global__ void xhdr_out_kernel(const int4* __restrict__ blocks, int G, const long long* __restrict__ off,
                                float* __restrict__ x, int64_t n,
                                const int* __restrict__ list, const unsigned long long* __restrict__ count,
                                int64_t cap) {
    const unsigned long long c = *count;
    const bool all = c > (unsigned long long)cap;
    const int64_t total = all ? n : (int64_t)c;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = all ? t : list[t];
        x[i] = __ldcg((const float*)(blocks + (off ? off[i] : i * G)) + 2);
    }
}

// out[t] = x[list[t]], t < count (the changed entries of a host iterate, copied back compactly)
__global__ void gather_list_kernel(const float* __restrict__ x, const int* __restrict__ list, int64_t count,
                                   float* __restrict__ out) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = x[list[t]];
}

// Pack the CSC into blocks: one thread per (column, chunk).
// row id as stored in a block: 0x80000000 | h if row == hot_rows[h] (ascending list)
__device__ __forceinline__ int encode_row(int row, const int* __restrict__ hot_rows, int nhot) {
    int lo = 0, hi = nhot;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (hot_rows[mid] < row) lo = mid + 1;
        else hi = mid;
    }
    return (lo < nhot && hot_rows[lo] == row) ? (int)(0x80000000u | (unsigned)lo) : row;
}

__global__ void pack_kernel(int64_t n, int G, const long long* __restrict__ colptr, const int* __restrict__ rowidx,
                            const float* __restrict__ val, const float* __restrict__ L, const int* __restrict__ hot_rows,
                            int nhot, int4* __restrict__ blocks) {
    const int64_t total = n * G;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / G;
        const int t = (int)(q - i * G);
        const long long s = colptr[i];
        const int len = (int)(colptr[i + 1] - s);
        int4 c;
        if (t == 0) {
            c = make_int4(__float_as_int(L[i]), len, 0, 0);
        } else {
            const int p0 = 2 * (t - 1);
            c.x = p0 < len ? encode_row(rowidx[s + p0], hot_rows, nhot) : 0;
            c.y = p0 < len ? __float_as_int(val[s + p0]) : 0;
            c.z = p0 + 1 < len ? encode_row(rowidx[s + p0 + 1], hot_rows, nhot) : 0;
            c.w = p0 + 1 < len ? __float_as_int(val[s + p0 + 1]) : 0;
        }
        blocks[q] = c;
    }
}

__global__ void max_len_kernel(int64_t n, const long long* __restrict__ colptr, int* __restrict__ out) {
    long long best = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        best = max(best, colptr[i + 1] - colptr[i]);
    int b = best > 0x7fffffff ? 0x7fffffff : (int)best;
    b = __reduce_max_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0) atomicMax(out, b);
}

template <int G, bool ONE, bool LOG>
cudaError_t launch_g(int ctas, const PackedParams& P, cudaStream_t st) {
    void* args[] = {(void*)&P};
    const int tpb = (ONE && P.cluster_sync == 2) ? 1024 : kThreads;
    const void* fn = tpb == 1024 ? (const void*)pcdm_packed_kernel<G, ONE, LOG, 1024>
                                 : (const void*)pcdm_packed_kernel<G, ONE, LOG>;
    if (ONE && P.reg_replay)  // every group owns <= 1 slot per iteration: replay from registers
        fn = tpb == 1024 ? (const void*)pcdm_packed1_kernel<G, LOG, 1024> : (const void*)pcdm_packed1_kernel<G, LOG>;
    const size_t smem = packed_smem_bytes(P.nhot, P.local_cap > 0 ? 0 : P.list_cap, P.hot_stage != 0, P.local_cap);
    if (P.cluster_sync) {  // the whole grid is one cluster (ctas <= 16)
        if (ctas > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(tpb);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = ctas;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelExC(&cfg, fn, args) == cudaSuccess) return cudaSuccess;
        cudaGetLastError();  // cluster of this size not available: grid barrier instead
        PackedParams Q = P;
        Q.cluster_sync = 0;
        void* qargs[] = {(void*)&Q};
        return cudaLaunchCooperativeKernel(fn, dim3(ctas), dim3(tpb), qargs, smem, st);
    }
    return cudaLaunchCooperativeKernel(fn, dim3(ctas), dim3(kThreads), args, smem, st);
}

template <bool ONE, bool LOG>
const void* kernel_ptr(int G) {
    switch (G) {
        case 2: return (const void*)pcdm_packed_kernel<2, ONE, LOG>;
        case 4: return (const void*)pcdm_packed_kernel<4, ONE, LOG>;
        case 8: return (const void*)pcdm_packed_kernel<8, ONE, LOG>;
        case 16: return (const void*)pcdm_packed_kernel<16, ONE, LOG>;
        default: return (const void*)pcdm_packed_kernel<32, ONE, LOG>;
    }
}

template <bool ONE, bool LOG>
cudaError_t launch_sel(int G, int ctas, const PackedParams& P, cudaStream_t st) {
    switch (G) {
        case 2: return launch_g<2, ONE, LOG>(ctas, P, st);
        case 4: return launch_g<4, ONE, LOG>(ctas, P, st);
        case 8: return launch_g<8, ONE, LOG>(ctas, P, st);
        case 16: return launch_g<16, ONE, LOG>(ctas, P, st);
        default: return launch_g<32, ONE, LOG>(ctas, P, st);
    }
}

}  // namespace

namespace pcdm_internal {

cudaError_t launch_xhdr_clear(int4* blocks, int G, const long long* off, const int* list,
                              const unsigned long long* count, int64_t cap, int64_t n, cudaStream_t st, int sms,
                              int64_t* launches) {
    xhdr_clear_kernel<<<sms * 8, 256, 0, st>>>(blocks, G, off, list, count, cap, n);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_xhdr_out(const int4* blocks, int G, const long long* off, float* x, int64_t n, const int* list,
                            const unsigned long long* count, int64_t cap, cudaStream_t st, int sms,
                            int64_t* launches) {
    xhdr_out_kernel<<<sms * 8, 256, 0, st>>>(blocks, G, off, x, n, list, count, cap);
    ++*launches;
    return cudaGetLastError();
}

int packed_lanes(int64_t max_len) {
    const int64_t chunks = 1 + (max_len + 1) / 2;
    int g = 2;
    while (g < chunks) g <<= 1;
    return g;
}

cudaError_t launch_max_len(int64_t n, const int64_t* colptr, int* out, cudaStream_t st, int sms, int64_t* launches) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    int64_t b = (n + 255) / 256;
    if (b > sms * 8) b = sms * 8;
    max_len_kernel<<<(int)b, 256, 0, st>>>(n, (const long long*)colptr, out);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_gather_list(const float* x, const int* list, int64_t count, float* out, cudaStream_t st, int sms,
                               int64_t* launches) {
    int64_t b = (count + 255) / 256;
    if (b < 1) b = 1;
    if (b > sms * 8) b = sms * 8;
    gather_list_kernel<<<(int)b, 256, 0, st>>>(x, list, count, out);
    ++*launches;
    return cudaGetLastError();
}

size_t packed_smem_bytes(int nhot, int list_cap, bool hot_stage, int local_cap) {
    return (size_t)nhot * (sizeof(float) + sizeof(int)) + (list_cap > 0 ? (size_t)list_cap * 8 + 8 : 0) +
           (hot_stage ? (size_t)nhot * sizeof(float) : 0) + (local_cap > 0 ? (size_t)local_cap * 24 + 16 : 0);
}

cudaError_t launch_pack(int64_t n, int G, const int64_t* colptr, const int* rowidx, const float* val, const float* L,
                        const int* hot_rows, int nhot, int4* blocks, cudaStream_t st, int sms, int64_t* launches) {
    int64_t b = (n * G + 255) / 256;
    if (b > sms * 16) b = sms * 16;
    pack_kernel<<<(int)b, 256, 0, st>>>(n, G, (const long long*)colptr, rowidx, val, L, hot_rows, nhot, blocks);
    ++*launches;
    return cudaGetLastError();
}

int async_groups(int G, int sms, int* ctas) {
    const void* fn;
    switch (G) {
        case 2: fn = (const void*)pcdm_async_kernel<2>; break;
        case 4: fn = (const void*)pcdm_async_kernel<4>; break;
        case 8: fn = (const void*)pcdm_async_kernel<8>; break;
        case 16: fn = (const void*)pcdm_async_kernel<16>; break;
        default: fn = (const void*)pcdm_async_kernel<32>; break;
    }
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    *ctas = per_sm * sms;
    return *ctas * (kThreads / G);
}

cudaError_t launch_async(int G, int ctas, const AsyncParams& A, cudaStream_t st, int64_t* launches) {
    ++*launches;
    switch (G) {
        case 2: pcdm_async_kernel<2><<<ctas, kThreads, 0, st>>>(A); break;
        case 4: pcdm_async_kernel<4><<<ctas, kThreads, 0, st>>>(A); break;
        case 8: pcdm_async_kernel<8><<<ctas, kThreads, 0, st>>>(A); break;
        case 16: pcdm_async_kernel<16><<<ctas, kThreads, 0, st>>>(A); break;
        default: pcdm_async_kernel<32><<<ctas, kThreads, 0, st>>>(A); break;
    }
    return cudaGetLastError();
}

int packed_ctas(int G, bool one_barrier, int sms, bool logistic, int nhot, int list_cap, bool hot_stage,
                int local_cap) {
    int per_sm = 1;
    const void* fn = logistic ? (one_barrier ? kernel_ptr<true, true>(G) : kernel_ptr<false, true>(G))
                              : (one_barrier ? kernel_ptr<true, false>(G) : kernel_ptr<false, false>(G));
    const size_t smem = packed_smem_bytes(nhot, list_cap, hot_stage, local_cap);
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    return per_sm * sms;
}

cudaError_t launch_packed(int G, bool one_barrier, int ctas, const PackedParams& P, cudaStream_t st,
                          int64_t* launches) {
    ++*launches;
    if (P.logistic) return one_barrier ? launch_sel<true, true>(G, ctas, P, st) : launch_sel<false, true>(G, ctas, P, st);
    return one_barrier ? launch_sel<true, false>(G, ctas, P, st) : launch_sel<false, false>(G, ctas, P, st);
}

}  // namespace pcdm_internal
