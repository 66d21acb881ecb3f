// common.cuh -- device helpers shared by the libpcdm kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PCDM_EMPTY_SLOT 0xFFFFFFFFFFFFFFFFull

// error-flag bits (device int written with atomicOr)
enum : int {
    FLAG_BAD_COLPTR = 1,
    FLAG_BAD_ROW = 2,
    FLAG_ROW_ORDER = 4,
    FLAG_NONFINITE_VAL = 8,
    FLAG_NONFINITE_B = 16,
    FLAG_NONFINITE_X = 32,
    FLAG_DIVERGED = 64,
    FLAG_SAMPLER = 128,
};

namespace pcdm {

// ---------------------------------------------------------------- loads
// Read-only data (A, L, colptr, slots): non-coherent path, no L1 allocation for
// streamed column data.
__device__ __forceinline__ float ld_stream_f32(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_stream_s32(const int* p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ long long ld_stream_s64(const long long* p) {
    long long v;
    asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
// Mutable data written by other CTAs inside the same launch (r, x, delta lists):
// bypass L1 (which is not coherent) and read the L2 copy.
__device__ __forceinline__ float ld_l2_f32(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_l2_s32(const int* p) {
    int v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void red_add_f32(float* p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ---------------------------------------------------------------- grid barrier
// Monotone-counter barrier for a co-resident (cooperative) grid.  `target`
// advances by gridDim.x per call; the counter is zeroed before each launch.
// Arrive: __syncthreads, then thread 0's red.release.gpu (cumulative over the
// CTA's writes that __syncthreads ordered before it); wait: thread 0 spins with
// ld.acquire.gpu, then __syncthreads releases the CTA.  No sequentially consistent
// fences (-DPCDM_SC_BARRIER restores the __threadfence + atomicAdd form).  Work
// issued between arrive and wait overlaps the other CTAs' arrival (it must not
// write anything the barrier is meant to publish).
// PCDM_BARRIER_SPLIT = K > 1: CTA b arrives on counter b % K (K counters 128 bytes
// apart, so the arrivals do not serialise on one L2 address) and warp 0 polls all K.
// The barrier memory is kBarrierWords words (zeroed before each launch).
#ifndef PCDM_BARRIER_SPLIT
#define PCDM_BARRIER_SPLIT 1
#endif
constexpr int kBarrierWords = 8 * 32;
static_assert(PCDM_BARRIER_SPLIT >= 1 && PCDM_BARRIER_SPLIT <= 8, "at most 8 barrier counters");
#ifndef PCDM_SC_BARRIER
__device__ __forceinline__ void grid_arrive(unsigned* counter, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        unsigned* c = counter + (PCDM_BARRIER_SPLIT > 1 ? (blockIdx.x % PCDM_BARRIER_SPLIT) * 32 : 0);
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
    }
}
__device__ __forceinline__ void grid_wait(const unsigned* counter, unsigned target) {
    if (PCDM_BARRIER_SPLIT == 1) {
        if (threadIdx.x == 0) {
            while ((int)(ld_acquire_u32(counter) - target) < 0) {
#ifdef PCDM_BARRIER_SLEEP
                __nanosleep(PCDM_BARRIER_SLEEP);
#endif
            }
        }
    } else if (threadIdx.x < 32) {
        const unsigned lane = threadIdx.x;
        for (;;) {
            const unsigned v = lane < PCDM_BARRIER_SPLIT ? ld_acquire_u32(counter + lane * 32) : 0u;
            if ((int)(__reduce_add_sync(0xffffffffu, v) - target) >= 0) break;
        }
    }
    __syncthreads();
}
#else
__device__ __forceinline__ void grid_arrive(unsigned* counter, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
    }
}
__device__ __forceinline__ void grid_wait(const unsigned* counter, unsigned target) {
    if (threadIdx.x == 0) {
        while ((int)(ld_acquire_u32(counter) - target) < 0) {
        }
        __threadfence();
    }
    __syncthreads();
}
#endif
__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned& target) {
    grid_arrive(counter, target);
    grid_wait(counter, target);
}

// ---------------------------------------------------------------- Philox4x32-10
struct u32x4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        u32x4 o;
        o.x = hi1 ^ c.y ^ k0;
        o.y = lo1;
        o.z = hi0 ^ c.w ^ k1;
        o.w = lo0;
        c = o;
    }
    return c;
}

// One sampler draw: counter (j, k, rho, tag), key = seed halves, Lemire map of
// the 64-bit word (y<<32)|x onto [0, n).  `reject_below` = (2^64 - n) mod n.
// Returns the value or -1 if the word is rejected.
__device__ __forceinline__ long long draw_value(uint64_t seed, uint32_t k, uint32_t rho, uint32_t j,
                                                uint32_t tag, uint64_t n, uint64_t reject_below) {
    u32x4 c{j, k, rho, tag};
    u32x4 o = philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t u = ((uint64_t)o.y << 32) | (uint64_t)o.x;
    const uint64_t lo = u * n;
    if (lo < reject_below) return -1;
    return (long long)__umul64hi(u, n);
}

// Fibonacci hash of a value onto a table of 2^log2h entries.
__device__ __forceinline__ uint32_t hash_slot(uint32_t v, int log2h) {
    return log2h == 0 ? 0u : (uint32_t)((v * 0x9E3779B1u) >> (32 - log2h));
}

// Insert (value v, owner code) so that the table keeps, per value, the minimum
// code: entry = (v << 32) | code; equal-key entries merge with a 64-bit atomicMin.
__device__ __forceinline__ void table_insert(unsigned long long* table, int log2h, uint32_t v,
                                             uint32_t code) {
    const unsigned long long key = ((unsigned long long)v << 32) | code;
    const uint32_t mask = (1u << log2h) - 1u;
    uint32_t h = hash_slot(v, log2h);
    while (true) {
        unsigned long long cur = *((volatile unsigned long long*)&table[h]);
        if (cur == PCDM_EMPTY_SLOT) {
            unsigned long long prev = atomicCAS(&table[h], PCDM_EMPTY_SLOT, key);
            if (prev == PCDM_EMPTY_SLOT) return;
            cur = prev;
        }
        if ((uint32_t)(cur >> 32) == v) {
            atomicMin(&table[h], key);
            return;
        }
        h = (h + 1) & mask;
    }
}

// Same result as table_insert, starting with the CAS on the home entry (no load
// first): one L2 operation per insert when the home entry is empty.
// Returns the entry index the value occupies (values never move: linear probing
// without deletion).
__device__ __forceinline__ uint32_t table_insert_cas_first(unsigned long long* table, int log2h, uint32_t v,
                                                           uint32_t code) {
    const unsigned long long key = ((unsigned long long)v << 32) | code;
    const uint32_t mask = (1u << log2h) - 1u;
    uint32_t h = hash_slot(v, log2h);
    while (true) {
        const unsigned long long prev = atomicCAS(&table[h], PCDM_EMPTY_SLOT, key);
        if (prev == PCDM_EMPTY_SLOT) return h;
        if ((uint32_t)(prev >> 32) == v) {
            atomicMin(&table[h], key);
            return h;
        }
        h = (h + 1) & mask;
    }
}

__device__ __forceinline__ uint32_t table_owner(const unsigned long long* table, int log2h,
                                                uint32_t v) {
    const uint32_t mask = (1u << log2h) - 1u;
    uint32_t h = hash_slot(v, log2h);
    while (true) {
        unsigned long long cur = __ldcg(&table[h]);
        if ((uint32_t)(cur >> 32) == v && cur != PCDM_EMPTY_SLOT) return (uint32_t)cur;
        h = (h + 1) & mask;
    }
}

// ---------------------------------------------------------------- soft threshold
// x+ = argmin_t g t + (s/2) t^2 + lam |x + t|  (+ x): u = x - g/s,
// x+ = sign(u) max(|u| - lam/s, 0); s == 0 (empty column): x+ = lam > 0 ? 0 : x.
__device__ __forceinline__ float prox_l1(float x, float g, float s, float lam) {
    if (s == 0.0f) return lam > 0.0f ? 0.0f : x;
    const float u = x - g / s;
    const float mag = fabsf(u) - lam / s;
    if (!(mag > 0.0f)) return (mag == mag) ? 0.0f : mag;  // keep NaN visible
    return u > 0.0f ? mag : -mag;
}

// ---------------------------------------------------------------- losses
// LASSO (square loss): the gathered vector is r = Ax - b, grad_i f = sum_j a_ji r_j,
// block step = soft-threshold (eq:h(x) block form).
// L2-regularised logistic (Sec. 8.4; R21): the library
// stores A~ = diag(y) A, the gathered vector is the margin s = A~ x,
// grad_i f = -sum_j a~_ji sigma(-s_j) = sum_j a~_ji w(s_j), w(s) = -1/(1+e^s), and the
// step minimises g t + (beta L_i/2) t^2 + lambda (x+t)^2 exactly.
template <bool LOGISTIC>
__device__ __forceinline__ float grad_weight(float v) {
    if (LOGISTIC) return -1.0f / (1.0f + __expf(v));
    return v;
}

template <bool LOGISTIC>
__device__ __forceinline__ float block_step(float x, float g, float s, float lam) {
    if (LOGISTIC) {
        const float d = s + 2.0f * lam;
        return d == 0.0f ? x : x - (g + 2.0f * lam * x) / d;
    }
    return prox_l1(x, g, s, lam);
}

}  // namespace pcdm
