// kernels_ragged.cu -- the PCDM1 hot loop for matrices with ragged column lengths
// (RAGGED layout of the packed loop): a warp, sub-warp or whole CTA per sampled
// column, chosen by the column's number of nonzeros.
//
// The uniform packed layout (kernels_packed.cu) gives every column G x 16 B with G
// fixed by the LONGEST column, so one 62-entry column makes every 10-entry column
// a 32-lane group, and a column over 62 entries rules the layout out.  Here column
// i owns g_i consecutive 16-byte chunks at chunk offset off[i]:
//
//   chunk 0       { L_i (f32), len (i32), x_i (f32, when x lives in the headers), 0 }
//   chunk t >= 1  { row_{2t-2}, val_{2t-2}, row_{2t-1}, val_{2t-1} }
//
// with g_i = pow2 >= 1 + ceil(len_i / 2) (2 .. 32) for len_i <= 62: one coalesced
// g_i x 16 B load by a group of g_i lanes, as in the uniform layout; and
// g_i = 1 + ceil(len_i / 2) for a LONG column (len_i > 62): a whole warp loops over
// its chunks (62 < len_i <= 1024: at most 16 rounds of 32 lanes), a whole CTA beyond
// (each thread <= 2 entries per 1024-entry round, block reduction, one thread takes
// the step, every thread scatters its entries).
//
// Binning (PAPER.md's iteration does not fix an order within S_k: every g_i of
// iteration k is computed from the same r_k, alg:PCD1 PAPER.md:177-186): after the
// sampler draws S_k, bin_* kernels sort the slot array of each iteration by class
// (g = 2, 4, 8, 16, 32 lanes, warp-long, CTA-long) into entries {i, off[i]}, so the
// iteration kernel reads the offset with the slot (no extra random line) and runs
// one loop per class, each spread over the whole grid: the longest columns first
// (they are the stragglers), then warp-long columns, 32-, 16-, 8-, 4- and 2-lane groups.
//
// Synchronisation is the one-barrier double-buffered scheme of the packed loop
// (P = r_k read-only in iteration k, Q receives the previous iteration's replayed
// steps and this iteration's own steps; after the barrier Q = r_{k+1}).  Step list
// entries hold (chunk offset, delta); the replay walks a column's chunks with a warp.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "internal.h"

using namespace pcdm;
using namespace pcdm_internal;

namespace {

constexpr int kThreads = 512;
constexpr int kWarpClass = 5;    // 62 < len <= 1024: a warp loops over the chunks
constexpr int kCtaClass = 6;     // len > 1024: a CTA
constexpr int kNumClasses = 7;
constexpr long long kCtaChunks = 1 + 1024 / 2;  // chunk count of a 1024-entry column

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

// ---- bulk (TMA engine) copies global -> shared with mbarrier completion (CTA-long columns)
constexpr int kStageChunks = 2048;  // 32 KB of 16-byte chunks = 4096 entries per piece

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
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

__device__ __forceinline__ int real_row(int v, const int* hrow) { return v < 0 ? hrow[v & 0x7fffffff] : v; }

__device__ __forceinline__ float gather_r(const float* rP, int v, const float* s_hot, const int* s_hrow, bool cache) {
    if (v >= 0) return ld_l2_f32(rP + v);
    return cache ? s_hot[v & 0x7fffffff] : ld_l2_f32(rP + s_hrow[v & 0x7fffffff]);
}

// r[row] += val * d for the chunk's (<= 2) pairs; pair0 = index of the first pair
__device__ __forceinline__ void scatter_chunk(float* r, const int4 c, int pair0, int len, float d, const int* hrow) {
    if (pair0 < len) red_add_f32(r + real_row(c.x, hrow), __int_as_float(c.y) * d);
    if (pair0 + 1 < len) red_add_f32(r + real_row(c.z, hrow), __int_as_float(c.w) * d);
}

// chunks of a column of `len` entries in the ragged layout
__host__ __device__ __forceinline__ long long ragged_chunks(long long len) {
    const long long need = 1 + (len + 1) / 2;
    if (len > 62) return need;
    long long g = 2;
    while (g < need) g <<= 1;
    return g;
}

// class of a column from its chunk count: 0..4 = 2..32 lanes, 5 = warp-long, 6 = CTA-long
__device__ __forceinline__ int chunk_class(long long nch) {
    if (nch > kCtaChunks) return kCtaClass;
    if (nch > 32 || (nch & (nch - 1)) != 0) return kWarpClass;
    return 30 - __clz((int)nch);  // log2(nch) - 1
}

// Record a nonzero step: x_i (header or array), the dirty list, the step list (off, d).
template <bool LOGISTIC>
__device__ __forceinline__ void record_step(const PackedParams& P, int i, unsigned off, float xp, float d, int cur) {
    if (!isfinite(xp)) atomicOr(P.flags, FLAG_DIVERGED);
    if (P.xlist) {
        ((float*)(P.blocks + off))[2] = xp;
        if (P.xlist_cap > 0) {
            const unsigned long long q = atomicAdd(P.xlist_count, 1ull);
            if (q < (unsigned long long)P.xlist_cap) P.xlist[q] = i;
        }
    } else {
        P.x[i] = xp;
    }
    const int pos = atomicAdd(P.nz_count + cur, 1);
    P.nz_idx[cur * P.tau + pos] = (int)off;
    P.nz_delta[cur * P.tau + pos] = d;
}

// One class of G-lane groups over entries E[beg, end): gather, reduce, step, scatter into Q.
template <int G, bool LOGISTIC>
__device__ __forceinline__ void ragged_class(const PackedParams& P, const int2* E, int beg, int end, const float* rP,
                                             float* rQ, const float* s_hot, const int* s_hrow, bool cache, int cur) {
    const int t = threadIdx.x & (G - 1);
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
    const int pair0 = 2 * (t - 1);
    for (int64_t j = beg + gid; j < end; j += ng) {
        const int2 e = ld_stream_v2(E + j);
        const unsigned off = (unsigned)e.y;
        // header (mutable x_i) through L2, pair chunks on the non-coherent path
        const int4 c = (t == 0) ? ld_l2_v4(P.blocks + off) : ld_stream_v4(P.blocks + off + t);
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
            const float xi = P.xlist ? __int_as_float(c.z) : ld_l2_f32(P.x + e.x);
            const float xp = block_step<LOGISTIC>(xi, acc, P.beta * __int_as_float(c.x), P.lambda);
            d = xp - xi;
            if (d != 0.0f) record_step<LOGISTIC>(P, e.x, off, xp, d, cur);
        }
        d = __shfl_sync(gm, d, src);
        if (d != 0.0f && t > 0) scatter_chunk(rQ, c, pair0, len, d, s_hrow);
    }
}

// Warp-long columns (63..1024 entries): a warp per column, lanes over its chunks.
template <bool LOGISTIC>
__device__ __forceinline__ void ragged_warp(const PackedParams& P, const int2* E, int beg, int end, const float* rP,
                                            float* rQ, const float* s_hot, const int* s_hrow, bool cache, int cur) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = beg + gw; j < end; j += nw) {
        const int2 e = ld_stream_v2(E + j);
        const int4* blk = P.blocks + (unsigned)e.y;
        const int4 h = ld_l2_v4(blk);  // header: L_i, len, x_i (mutable: through L2)
        const int len = h.y;
        const int nch = 1 + (len + 1) / 2;
        float acc = 0.0f;
        for (int t = 1 + lane; t < nch; t += 32) {
            const int4 c = ld_stream_v4(blk + t);
            const int p0 = 2 * (t - 1);
            const float ra = grad_weight<LOGISTIC>(gather_r(rP, c.x, s_hot, s_hrow, cache));
            const float rb = p0 + 1 < len ? grad_weight<LOGISTIC>(gather_r(rP, c.z, s_hot, s_hrow, cache)) : 0.0f;
            acc += fmaf(__int_as_float(c.y), ra, __int_as_float(c.w) * rb);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        float d = 0.0f;
        if (lane == 0) {
            const float xi = P.xlist ? __int_as_float(h.z) : ld_l2_f32(P.x + e.x);
            const float xp = block_step<LOGISTIC>(xi, acc, P.beta * __int_as_float(h.x), P.lambda);
            d = xp - xi;
            if (d != 0.0f) record_step<LOGISTIC>(P, e.x, (unsigned)e.y, xp, d, cur);
        }
        d = __shfl_sync(0xffffffffu, d, 0);
        if (d != 0.0f)
            for (int t = 1 + lane; t < nch; t += 32) scatter_chunk(rQ, ld_stream_v4(blk + t), 2 * (t - 1), len, d, s_hrow);
    }
}

// CTA-long columns: one CTA per column (entries E[beg, end) dealt to CTAs round robin).
template <bool LOGISTIC>
__device__ __forceinline__ void ragged_long(const PackedParams& P, const int2* E, int beg, int end, const float* rP,
                                            float* rQ, const float* s_hot, const int* s_hrow, bool cache, int cur,
                                            float* s_red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int q = beg + blockIdx.x; q < end; q += gridDim.x) {
        const int2 e = ld_stream_v2(E + q);
        const int4* blk = P.blocks + (unsigned)e.y;
        const int len = ld_l2_v4(blk).y;  // the header line holds the mutable x_i: read it through L2
        const int nch = 1 + (len + 1) / 2;
        float acc = 0.0f;
        for (int t = 1 + threadIdx.x; t < nch; t += blockDim.x) {
            const int4 c = ld_stream_v4(blk + t);
            const int p0 = 2 * (t - 1);
            const float ra = grad_weight<LOGISTIC>(gather_r(rP, c.x, s_hot, s_hrow, cache));
            const float rb = p0 + 1 < len ? grad_weight<LOGISTIC>(gather_r(rP, c.z, s_hot, s_hrow, cache)) : 0.0f;
            acc += fmaf(__int_as_float(c.y), ra, __int_as_float(c.w) * rb);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) s_red[warp] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            float g = 0.0f;
            for (int w = 0; w < nwarps; ++w) g += s_red[w];
            const int4 h = ld_l2_v4(blk);
            const float xi = P.xlist ? __int_as_float(h.z) : ld_l2_f32(P.x + e.x);
            const float xp = block_step<LOGISTIC>(xi, g, P.beta * __int_as_float(h.x), P.lambda);
            const float d = xp - xi;
            if (d != 0.0f) record_step<LOGISTIC>(P, e.x, (unsigned)e.y, xp, d, cur);
            s_red[32] = d;
        }
        __syncthreads();
        const float d = s_red[32];
        if (d != 0.0f)
            for (int t = 1 + threadIdx.x; t < nch; t += blockDim.x)
                scatter_chunk(rQ, ld_stream_v4(blk + t), 2 * (t - 1), len, d, s_hrow);
        __syncthreads();  // s_red reused by the next long column
    }
}

#ifndef PCDM_RAGGED_MINB
#define PCDM_RAGGED_MINB 3  // CTAs of 512 threads per SM (register cap 40)
#endif
// CTA-long columns with the column slice staged in shared memory by bulk copies
// (P.bulk_stage): pieces of <= 4096 entries arrive through the TMA
// engine (one cp.async.bulk per piece, completion on an mbarrier), the threads gather
// from shared memory, and a column that fits one piece is scattered from the staged
// copy instead of being read from global memory a second time.
template <bool LOGISTIC>
__device__ __forceinline__ void ragged_long_bulk(const PackedParams& P, const int2* E, int beg, int end, const float* rP,
                                                 float* rQ, const float* s_hot, const int* s_hrow, bool cache, int cur,
                                                 float* s_red, int4* s_stage, unsigned long long* bar,
                                                 unsigned& phase) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int q = beg + blockIdx.x; q < end; q += gridDim.x) {
        const int2 e = ld_stream_v2(E + q);
        const int4* blk = P.blocks + (unsigned)e.y;
        const int len = ld_l2_v4(blk).y;
        const int npair = (len + 1) / 2;
        float acc = 0.0f;
        for (int base = 0; base < npair; base += kStageChunks) {
            const int cnt = min(kStageChunks, npair - base);
            if (threadIdx.x == 0) {
                // the generic-proxy reads of the previous piece (ordered by the __syncthreads
                // below) come before the async-proxy write of this one
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(bar, (unsigned)cnt * 16u);
                bulk_g2s(s_stage, blk + 1 + base, (unsigned)cnt * 16u, bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1u;
            for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
                const int4 c = s_stage[t];
                const int p0 = 2 * (base + t);
                const float ra = grad_weight<LOGISTIC>(gather_r(rP, c.x, s_hot, s_hrow, cache));
                const float rb = p0 + 1 < len ? grad_weight<LOGISTIC>(gather_r(rP, c.z, s_hot, s_hrow, cache)) : 0.0f;
                acc += fmaf(__int_as_float(c.y), ra, __int_as_float(c.w) * rb);
            }
            __syncthreads();
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) s_red[warp] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            float g = 0.0f;
            for (int w = 0; w < nwarps; ++w) g += s_red[w];
            const int4 h = ld_l2_v4(blk);
            const float xi = P.xlist ? __int_as_float(h.z) : ld_l2_f32(P.x + e.x);
            const float xp = block_step<LOGISTIC>(xi, g, P.beta * __int_as_float(h.x), P.lambda);
            const float d = xp - xi;
            if (d != 0.0f) record_step<LOGISTIC>(P, e.x, (unsigned)e.y, xp, d, cur);
            s_red[32] = d;
        }
        __syncthreads();
        const float d = s_red[32];
        if (d != 0.0f) {
            if (npair <= kStageChunks)  // the whole slice is still staged
                for (int t = threadIdx.x; t < npair; t += blockDim.x) scatter_chunk(rQ, s_stage[t], 2 * t, len, d, s_hrow);
            else
                for (int t = 1 + threadIdx.x; t <= npair; t += blockDim.x)
                    scatter_chunk(rQ, ld_stream_v4(blk + t), 2 * (t - 1), len, d, s_hrow);
        }
        __syncthreads();  // s_red and s_stage reused by the next long column
    }
}

template <bool LOGISTIC, bool BULK>
__global__ void __launch_bounds__(kThreads, PCDM_RAGGED_MINB) pcdm_ragged_kernel(PackedParams P) {
    unsigned bar_target = 0;
    extern __shared__ float s_dyn[];
    const int nhot = P.nhot;
    float* s_hot = s_dyn;                  // [nhot] r_k at the hot rows
    int* s_hrow = (int*)(s_dyn + nhot);    // [nhot] hot row ids
    float* s_red = (float*)(s_hrow + nhot);  // [33] block reduction + the long column's step
    int* s_cb = (int*)(s_red + 33);          // [2][8] class bounds of this / the next iteration
    // P.bulk_stage: [kStageChunks] staged column slice (16-byte aligned) + its mbarrier
    int4* s_stage = (int4*)(((uintptr_t)(s_cb + 16) + 15) & ~(uintptr_t)15);
    unsigned long long* s_bar = (unsigned long long*)(s_stage + kStageChunks);
    unsigned phase = 0;
    constexpr bool bulk = BULK;
    const bool cache = P.hot_cache != 0;
    for (int h = threadIdx.x; h < nhot; h += blockDim.x) s_hrow[h] = P.hot_rows[h];
    if (threadIdx.x < 8 && P.iters > 0) s_cb[threadIdx.x] = ld_stream_s32(P.bcnt + threadIdx.x);
    if (bulk && threadIdx.x == 0) {
        mbar_init(s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t it = 0; it < P.iters; ++it) {
        const int64_t k = P.k0 + it;
        const int cur = (int)(k % 3), prev = (int)((k + 2) % 3), next = (int)((k + 1) % 3);
        const float* rP = (k & 1) ? P.r1 : P.r0;
        float* rQ = (k & 1) ? P.r0 : P.r1;
        if (blockIdx.x == 0 && threadIdx.x == 0) P.nz_count[next] = 0;
        // replay the previous iteration's nonzero steps into Q: a warp per step
        const int cntp = ld_l2_s32(P.nz_count + prev);
        for (int64_t e = gwarp; e < cntp; e += nwarp) {
            const unsigned off = (unsigned)ld_l2_s32(P.nz_idx + prev * P.tau + e);
            const float d = ld_l2_f32(P.nz_delta + prev * P.tau + e);
            const int4* blk = P.blocks + off;
            const int len = ld_l2_v4(blk).y;
            const int nch = 1 + (len + 1) / 2;
            for (int t = 1 + lane; t < nch; t += 32) scatter_chunk(rQ, ld_stream_v4(blk + t), 2 * (t - 1), len, d, s_hrow);
        }
        if (cache) {
            for (int h = threadIdx.x; h < nhot; h += blockDim.x) s_hot[h] = ld_l2_f32(rP + s_hrow[h]);
            __syncthreads();
        }
        const int2* E = P.bins + it * P.tau;
        const int* cb = s_cb + (it & 1) * 8;  // class starts [0..6], end [7] (loaded before the barrier)
        if constexpr (bulk)
            ragged_long_bulk<LOGISTIC>(P, E, cb[6], cb[7], rP, rQ, s_hot, s_hrow, cache, cur, s_red, s_stage, s_bar,
                                       phase);
        else
            ragged_long<LOGISTIC>(P, E, cb[6], cb[7], rP, rQ, s_hot, s_hrow, cache, cur, s_red);
        ragged_warp<LOGISTIC>(P, E, cb[5], cb[6], rP, rQ, s_hot, s_hrow, cache, cur);
        ragged_class<32, LOGISTIC>(P, E, cb[4], cb[5], rP, rQ, s_hot, s_hrow, cache, cur);
        ragged_class<16, LOGISTIC>(P, E, cb[3], cb[4], rP, rQ, s_hot, s_hrow, cache, cur);
        ragged_class<8, LOGISTIC>(P, E, cb[2], cb[3], rP, rQ, s_hot, s_hrow, cache, cur);
        ragged_class<4, LOGISTIC>(P, E, cb[1], cb[2], rP, rQ, s_hot, s_hrow, cache, cur);
        ragged_class<2, LOGISTIC>(P, E, cb[0], cb[1], rP, rQ, s_hot, s_hrow, cache, cur);
        // the next iteration's class bounds (written before the launch) load while the
        // other CTAs arrive
        grid_arrive(P.barrier, bar_target);
        if (threadIdx.x < 8 && it + 1 < P.iters)
            s_cb[((it + 1) & 1) * 8 + threadIdx.x] = ld_stream_s32(P.bcnt + (it + 1) * 8 + threadIdx.x);
        grid_wait(P.barrier, bar_target);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const int cnt = ld_l2_s32(P.nz_count + cur);
            if (cnt) atomicAdd(P.nz_total, (unsigned long long)cnt);
        }
    }
}

// ---------------------------------------------------------------- layout
__global__ void ragged_sizes_kernel(int64_t n, const long long* __restrict__ colptr, long long* __restrict__ sizes,
                                    unsigned char* __restrict__ cls) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const long long nch = ragged_chunks(colptr[i + 1] - colptr[i]);
        sizes[i] = nch;
        cls[i] = (unsigned char)chunk_class(nch);
    }
}

// one thread per chunk q: its column by binary search in off[0..n]
__global__ void ragged_pack_kernel(int64_t n, int64_t total, const long long* __restrict__ off,
                                   const long long* __restrict__ colptr, const int* __restrict__ rowidx,
                                   const float* __restrict__ val, const float* __restrict__ L,
                                   const int* __restrict__ hot_rows, int nhot, int4* __restrict__ blocks) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;  // largest i with off[i] <= q
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (off[mid] <= q) lo = mid;
            else hi = mid;
        }
        const int64_t i = lo;
        const int t = (int)(q - off[i]);
        const long long s = colptr[i];
        const int len = (int)(colptr[i + 1] - s);
        int4 c;
        if (t == 0) {
            c = make_int4(__float_as_int(L[i]), len, 0, 0);
        } else {
            const int p0 = 2 * (t - 1);
            auto enc = [&](int row) {
                int a = 0, b = nhot;
                while (a < b) {
                    const int mid = (a + b) >> 1;
                    if (hot_rows[mid] < row) a = mid + 1;
                    else b = mid;
                }
                return (a < nhot && hot_rows[a] == row) ? (int)(0x80000000u | (unsigned)a) : row;
            };
            c.x = p0 < len ? enc(rowidx[s + p0]) : 0;
            c.y = p0 < len ? __float_as_int(val[s + p0]) : 0;
            c.z = p0 + 1 < len ? enc(rowidx[s + p0 + 1]) : 0;
            c.w = p0 + 1 < len ? __float_as_int(val[s + p0 + 1]) : 0;
        }
        blocks[q] = c;
    }
}

// ---------------------------------------------------------------- binning
// Per iteration `it` (blockIdx.y) of a sampler pass: class counts of its slots.
__global__ void bin_count_kernel(const int* __restrict__ slots, int64_t tau, const unsigned char* __restrict__ cls,
                                 int* __restrict__ gcnt) {
    __shared__ int s_c[8];
    if (threadIdx.x < 8) s_c[threadIdx.x] = 0;
    __syncthreads();
    const int* S = slots + (int64_t)blockIdx.y * tau;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < tau; j += (int64_t)gridDim.x * blockDim.x) {
        const int i = __ldg(S + j);
        if (i < 0) continue;  // idle processor
        atomicAdd(&s_c[cls[i]], 1);
    }
    __syncthreads();
    if (threadIdx.x < kNumClasses && s_c[threadIdx.x])
        atomicAdd(gcnt + blockIdx.y * 16 + threadIdx.x, s_c[threadIdx.x]);
}

// class starts (bcnt[it][0..6]) and end (bcnt[it][7]); cursors gcnt[it][8..14] = starts
__global__ void bin_scan_kernel(int64_t count, int* __restrict__ gcnt, int* __restrict__ bcnt) {
    const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= count) return;
    int* g = gcnt + it * 16;
    int s = 0;
    for (int c = 0; c < kNumClasses; ++c) {
        bcnt[it * 8 + c] = s;
        g[8 + c] = s;
        s += g[c];
    }
    bcnt[it * 8 + 7] = s;
}

__global__ void bin_scatter_kernel(const int* __restrict__ slots, int64_t tau, const long long* __restrict__ off,
                                   const unsigned char* __restrict__ cls, int* __restrict__ gcnt,
                                   int2* __restrict__ bins) {
    __shared__ int s_c[8], s_base[8];
    const int* S = slots + (int64_t)blockIdx.y * tau;
    int2* E = bins + (int64_t)blockIdx.y * tau;
    const int64_t per = (tau + gridDim.x - 1) / gridDim.x;
    const int64_t j0 = (int64_t)blockIdx.x * per, j1 = min(tau, j0 + per);
    if (threadIdx.x < 8) s_c[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
        const int i = __ldg(S + j);
        if (i >= 0) atomicAdd(&s_c[cls[i]], 1);
    }
    __syncthreads();
    if (threadIdx.x < kNumClasses) {
        s_base[threadIdx.x] = s_c[threadIdx.x] ? atomicAdd(gcnt + blockIdx.y * 16 + 8 + threadIdx.x, s_c[threadIdx.x]) : 0;
        s_c[threadIdx.x] = 0;
    }
    __syncthreads();
    for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
        const int i = __ldg(S + j);
        if (i < 0) continue;
        const int c = cls[i];
        const int pos = s_base[c] + atomicAdd(&s_c[c], 1);
        E[pos] = make_int2(i, (int)(unsigned)off[i]);
    }
}

}  // namespace

namespace pcdm_internal {

cudaError_t build_ragged(const DevCSC& A, const float* L, const int* hot_rows, int nhot, long long** off_out,
                         unsigned char** cls_out, int4** blocks_out, long long* total_out, cudaStream_t st, int sms,
                         int64_t* launches) {
    *off_out = nullptr;
    *cls_out = nullptr;
    *blocks_out = nullptr;
    long long* off = nullptr;
    unsigned char* cls = nullptr;
    cudaError_t e = cudaMalloc((void**)&off, sizeof(long long) * (A.n + 1));
    if (e != cudaSuccess) return e;
    e = cudaMalloc((void**)&cls, A.n);
    if (e != cudaSuccess) {
        cudaFree(off);
        return e;
    }
    e = cudaMemsetAsync(off, 0, sizeof(long long), st);
    int64_t b = (A.n + 255) / 256;
    if (b > sms * 16) b = sms * 16;
    if (e == cudaSuccess) {
        ragged_sizes_kernel<<<(int)b, 256, 0, st>>>(A.n, (const long long*)A.colptr, off + 1, cls);
        ++*launches;
        e = cudaGetLastError();
    }
    size_t tmp_bytes = 0;
    void* tmp = nullptr;
    if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, off + 1, off + 1, A.n, st);
    if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes);
    if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, off + 1, off + 1, A.n, st);
    long long total = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&total, off + A.n, sizeof(long long), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(tmp);
    if (e == cudaSuccess && total >= (1ll << 32)) e = cudaErrorInvalidValue;  // offsets are 32-bit in the bins
    int4* blocks = nullptr;
    if (e == cudaSuccess) e = cudaMalloc((void**)&blocks, sizeof(int4) * total);
    if (e == cudaSuccess) {
        int64_t bb = (total + 255) / 256;
        if (bb > sms * 32) bb = sms * 32;
        ragged_pack_kernel<<<(int)bb, 256, 0, st>>>(A.n, total, off, (const long long*)A.colptr, A.rowidx, A.val, L,
                                                    hot_rows, nhot, blocks);
        ++*launches;
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) {
        cudaFree(off);
        cudaFree(cls);
        cudaFree(blocks);
        return e;
    }
    *off_out = off;
    *cls_out = cls;
    *blocks_out = blocks;
    *total_out = total;
    return cudaSuccess;
}

size_t bin_scratch_bytes(int64_t count) { return (size_t)count * 16 * sizeof(int); }

cudaError_t bin_chunk(const int* slots, int64_t tau, int64_t count, const long long* off, const unsigned char* cls,
                      int* scratch, int2* bins, int* bcnt, cudaStream_t st, int sms, int64_t* launches) {
    if (count <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(scratch, 0, bin_scratch_bytes(count), st);
    if (e != cudaSuccess) return e;
    // blocks per iteration: ~2 waves of the device over the whole pass
    int64_t per_it = (2 * sms * 4 + count - 1) / count;
    per_it = std::max<int64_t>(1, std::min<int64_t>(per_it, (tau + 255) / 256));
    const dim3 grid((unsigned)per_it, (unsigned)count);
    bin_count_kernel<<<grid, 256, 0, st>>>(slots, tau, cls, scratch);
    bin_scan_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(count, scratch, bcnt);
    bin_scatter_kernel<<<grid, 256, 0, st>>>(slots, tau, off, cls, scratch, bins);
    *launches += 3;
    return cudaGetLastError();
}

size_t ragged_smem_bytes(int nhot, bool bulk_stage) {
    return (size_t)nhot * (sizeof(float) + sizeof(int)) + (33 + 16) * sizeof(float) +
           (bulk_stage ? 16 + (size_t)kStageChunks * 16 + 8 : 0);
}

static const void* ragged_fn(bool logistic, bool bulk) {
    if (bulk) return logistic ? (const void*)pcdm_ragged_kernel<true, true> : (const void*)pcdm_ragged_kernel<false, true>;
    return logistic ? (const void*)pcdm_ragged_kernel<true, false> : (const void*)pcdm_ragged_kernel<false, false>;
}

int ragged_ctas(int sms, bool logistic, int nhot, bool bulk_stage) {
    const void* fn = ragged_fn(logistic, bulk_stage);
    const size_t smem = ragged_smem_bytes(nhot, bulk_stage);
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    return per_sm * sms;
}

cudaError_t launch_ragged(int ctas, const PackedParams& P, cudaStream_t st, int64_t* launches) {
    ++*launches;
    void* args[] = {(void*)&P};
    const void* fn = ragged_fn(P.logistic != 0, P.bulk_stage != 0);
    return cudaLaunchCooperativeKernel(fn, dim3(ctas), dim3(kThreads), args,
                                       ragged_smem_bytes(P.nhot, P.bulk_stage != 0), st);
}

}  // namespace pcdm_internal
