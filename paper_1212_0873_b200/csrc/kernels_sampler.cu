// kernels_sampler.cu -- seeded tau-nice sampler on the device.
//
// Law: S_k uniform over all tau-subsets of [n] (tau-nice).
// Concrete rule (reading R#1, SURVEY 8(c) "SAMPLE"): slot j of
// iteration k draws, in rounds rho = 0, 1, ..., the Lemire-mapped Philox4x32-10
// word of counter (j, k, rho, tag) under key (lo32 seed, hi32 seed); each value
// is owned by the lexicographically smallest (rho, j) that drew it; unowned
// slots redraw in the next round.  If 2 tau > n the n - tau EXCLUDED values are
// drawn (tag 2) and S_k is the complement in ascending order.
//
// Device realisation: round 0 for every (iteration, slot) of a chunk is one
// grid-wide pass inserting (value, code = rho*cnt + j) into a per-iteration
// open-addressing table that keeps the minimum code per value (64-bit
// atomicMin on (value << 32 | code); the insert CASes the home entry first and
// records the entry the value landed in); a second pass keeps the owners by
// reading that entry; the few leftover slots finish their rounds inside one CTA
// per iteration.  The result depends only on the codes, never on thread timing.
#include <cub/block/block_scan.cuh>
#include <cuda_runtime.h>
#include <curand_kernel.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"

using namespace pcdm;

namespace {

struct DrawArgs {
    uint64_t seed;
    uint64_t n;
    uint64_t reject_below;
    uint32_t tag;
    int64_t cnt;
    int log2h;
};

// Contest mode (round 0 without a check pass): a draw that finds its value already in
// the table is a duplicate; it records (entry, its code, the code it found) in the
// iteration's contest list (second half of the pending area, cnt/3 records) and lowers
// the entry to the minimum code; a rejected draw goes straight to the pending list.  The
// rounds kernel then knows every slot that drew a contested value: the one that wrote
// the entry first appears as a found code (the first duplicate's CAS reads it before
// any atomicMin), all others as recording codes.  Too many records for the list: the
// iteration's counter passes cnt/3 and the rounds kernel checks all its slots.
__device__ __forceinline__ void contest_record(int* pending, int* ncontest, int64_t it, int64_t cnt, uint32_t h,
                                               uint32_t code, uint32_t found) {
    const int cap = (int)(cnt / 3);
    const int q = atomicAdd(ncontest + it, 1);
    if (q < cap) {
        int* rec = pending + it * 2 * cnt + cnt + 3 * q;
        rec[0] = (int)h;
        rec[1] = (int)code;
        rec[2] = (int)found;
    }
}

template <bool CAS_FIRST>
__global__ void sample_round0_kernel(DrawArgs a, int64_t k0, int64_t count, unsigned long long* tables,
                                     int* cand, int* pending, int* npending, int contest) {
    const int64_t total = count * a.cnt;
    const uint32_t mask = (1u << a.log2h) - 1u;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t it = t / a.cnt;
        const uint32_t j = (uint32_t)(t - it * a.cnt);
        const long long v = draw_value(a.seed, (uint32_t)(k0 + it), 0u, j, a.tag, a.n, a.reject_below);
        cand[t] = (int)v;
        if (CAS_FIRST && contest) {
            if (v < 0) {
                pending[it * 2 * a.cnt + atomicAdd(npending + it, 1)] = (int)j;
                continue;
            }
            unsigned long long* table = tables + (it << a.log2h);
            const unsigned long long key = ((unsigned long long)v << 32) | j;
            uint32_t h = hash_slot((uint32_t)v, a.log2h);
            while (true) {
                const unsigned long long prev = atomicCAS(&table[h], PCDM_EMPTY_SLOT, key);
                if (prev == PCDM_EMPTY_SLOT) break;
                if ((uint32_t)(prev >> 32) == (uint32_t)v) {
                    atomicMin(&table[h], key);
                    contest_record(pending, npending + count, it, a.cnt, h, j, (uint32_t)prev);
                    break;
                }
                h = (h + 1) & mask;
            }
            continue;
        }
        if (v >= 0) {
            if (CAS_FIRST) {
                // the entry index goes to the (still unused) second half of the iteration's
                // pending area, so the check pass reads one entry instead of probing
                const uint32_t at = table_insert_cas_first(tables + (it << a.log2h), a.log2h, (uint32_t)v, j);
                if (pending) pending[it * 2 * a.cnt + a.cnt + j] = (int)at;
            } else {
                table_insert(tables + (it << a.log2h), a.log2h, (uint32_t)v, j);
            }
        }
    }
}

template <bool AT>
__global__ void sample_check_kernel(DrawArgs a, int64_t count, const unsigned long long* tables,
                                    const int* cand, int* pending, int* npending) {
    const int64_t total = count * a.cnt;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t it = t / a.cnt;
        const uint32_t j = (uint32_t)(t - it * a.cnt);
        const int v = cand[t];
        const unsigned long long* table = tables + (it << a.log2h);
        const bool owned =
            v >= 0 && (AT ? (uint32_t)__ldcg(table + pending[it * 2 * a.cnt + a.cnt + j]) == j
                          : table_owner(table, a.log2h, (uint32_t)v) == j);
        if (!owned) {
            const int pos = atomicAdd(npending + it, 1);
            pending[it * 2 * a.cnt + pos] = (int)j;
        }
    }
}

// One CTA per iteration finishes rounds rho >= 1 for its pending slots.
__global__ void sample_rounds_kernel(DrawArgs a, int64_t k0, int64_t count, unsigned long long* tables, int* cand,
                                     int* pending, const int* npending, int* rounds_max, int* flags, int contest) {
    const int64_t it = blockIdx.x;
    unsigned long long* table = tables + (it << a.log2h);
    int* c = cand + it * a.cnt;
    int* pin = pending + it * 2 * a.cnt;
    int* pout = pin + a.cnt;
    __shared__ int s_next;
    int np = npending[it];
    if (contest) {
        // the losers of round 0: from the contest records, or (list overflow) every slot
        const int nrec = npending[count + it];
        if (nrec == 0 && np == 0) return;
        if (threadIdx.x == 0) s_next = np;
        __syncthreads();
        auto lose = [&](uint32_t code) {  // append once (mark the slot's value -2)
            if (atomicExch(c + code, -2) != -2) pin[atomicAdd(&s_next, 1)] = (int)code;
        };
        if (nrec > (int)(a.cnt / 3)) {
            for (int t = threadIdx.x; t < a.cnt; t += blockDim.x) {
                const int v = c[t];
                if (v >= 0 && table_owner(table, a.log2h, (uint32_t)v) != (uint32_t)t) lose((uint32_t)t);
            }
        } else {
            const int* rec = pin + a.cnt;
            for (int q = threadIdx.x; q < nrec; q += blockDim.x) {
                const uint32_t owner = (uint32_t)__ldcg(table + rec[3 * q]);
                const uint32_t code = (uint32_t)rec[3 * q + 1], found = (uint32_t)rec[3 * q + 2];
                if (code != owner) lose(code);
                if (found != owner) lose(found);
            }
        }
        __syncthreads();
        np = s_next;
        __syncthreads();
    }
    if (np == 0) return;
    uint32_t rho = 1;
    for (; np > 0; ++rho) {
        if ((uint64_t)(rho + 1) * (uint64_t)a.cnt > 0x100000000ull) {
            if (threadIdx.x == 0) atomicOr(flags, FLAG_SAMPLER);
            return;
        }
        // the entry each of this thread's first kPos slots landed in (CAS-first insert)
        constexpr int kPos = 4;
        uint32_t at[kPos];
        for (int t = threadIdx.x, q = 0; t < np; t += blockDim.x, ++q) {
            const uint32_t j = (uint32_t)pin[t];
            const long long v = draw_value(a.seed, (uint32_t)(k0 + it), rho, j, a.tag, a.n, a.reject_below);
            c[j] = (int)v;
            if (v >= 0) {
                const uint32_t h = table_insert_cas_first(table, a.log2h, (uint32_t)v, rho * (uint32_t)a.cnt + j);
                if (q < kPos) at[q] = h;
            }
        }
        if (threadIdx.x == 0) s_next = 0;
        __syncthreads();
        for (int t = threadIdx.x, q = 0; t < np; t += blockDim.x, ++q) {
            const uint32_t j = (uint32_t)pin[t];
            const int v = c[j];
            const uint32_t code = rho * (uint32_t)a.cnt + j;
            const bool owned = v >= 0 && (q < kPos ? (uint32_t)__ldcg(table + at[q]) == code
                                                   : table_owner(table, a.log2h, (uint32_t)v) == code);
            if (!owned) pout[atomicAdd(&s_next, 1)] = (int)j;
        }
        __syncthreads();
        np = s_next;
        int* tmp = pin;
        pin = pout;
        pout = tmp;
        __syncthreads();
    }
    if (threadIdx.x == 0) atomicMax(rounds_max, (int)rho);
}

// ---------------------------------------------------------------- other DU samplings
// 64-bit word of counter (j, k, 0, tag) (the same Philox stream as the draws).
__device__ __forceinline__ uint64_t sampler_word(uint64_t seed, uint32_t k, uint32_t j, uint32_t tag) {
    u32x4 o = philox4x32_10(u32x4{j, k, 0u, tag}, (uint32_t)seed, (uint32_t)(seed >> 32));
    return ((uint64_t)o.y << 32) | (uint64_t)o.x;
}

// tau-independent (R16): processor j picks the first
// accepted draw of counters (j, k, rho, tag 3); the lowest j keeps a shared pick.
// (CAS-first insert; the entry index is recorded in `at` for the check pass, as in round 0)
__global__ void sample_indep_insert_kernel(DrawArgs a, int64_t k0, int64_t count, unsigned long long* tables,
                                           int* slots, int* at) {
    const int64_t total = count * a.cnt;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t it = t / a.cnt;
        const uint32_t j = (uint32_t)(t - it * a.cnt);
        long long v;
        uint32_t rho = 0;
        while ((v = draw_value(a.seed, (uint32_t)(k0 + it), rho, j, 3u, a.n, a.reject_below)) < 0) ++rho;
        slots[t] = (int)v;
        at[t] = (int)table_insert_cas_first(tables + (it << a.log2h), a.log2h, (uint32_t)v, j);
    }
}

__global__ void sample_indep_check_kernel(DrawArgs a, int64_t count, const unsigned long long* tables, int* slots,
                                          const int* at) {
    const int64_t total = count * a.cnt;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t it = t / a.cnt;
        const uint32_t j = (uint32_t)(t - it * a.cnt);
        if ((uint32_t)__ldcg(tables + (it << a.log2h) + at[t]) != j) slots[t] = -1;
    }
}

// (tau, p_b)-binomial, Case 2 of PAPER.md:452-455 (R17): processor j of
// the tau-nice assignment is available iff word(j, k, 0, tag 4) < T.
__global__ void sample_thin_kernel(uint64_t seed, int64_t k0, int64_t count, int64_t tau, uint64_t T, int* slots) {
    const int64_t total = count * tau;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t it = t / tau;
        const uint32_t j = (uint32_t)(t - it * tau);
        if (!(sampler_word(seed, (uint32_t)(k0 + it), j, 4u) < T)) slots[t] = -1;
    }
}

// DU(q) (eq:p(S); R18): K = first s with u < T[s]
// (or s >= always_from), u = word(0, k, 0, tag 5); slots j >= K are idle.
__global__ void sample_du_size_kernel(uint64_t seed, int64_t k0, int64_t count, int64_t tau, const uint64_t* T,
                                      int64_t always_from, int* K) {
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < count;
         it += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t u = sampler_word(seed, (uint32_t)(k0 + it), 0u, 5u);
        int64_t lo = 0, hi = tau;  // first s in [0, tau) with the predicate, else tau
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (mid >= always_from || u < T[mid]) hi = mid;
            else lo = mid + 1;
        }
        K[it] = (int)lo;
    }
}

__global__ void sample_du_mask_kernel(int64_t count, int64_t tau, const int* K, int* slots) {
    const int64_t total = count * tau;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t it = t / tau;
        if (t - it * tau >= K[it]) slots[t] = -1;
    }
}

// Complement: S_k = [n] minus the owned (excluded) values, ascending.
constexpr int kScanThreads = 512;
__global__ void __launch_bounds__(kScanThreads) sample_complement_kernel(int64_t n, int64_t tau, int64_t cnt,
                                                                         const int* cand, unsigned char* marks,
                                                                         int* slots) {
    using Scan = cub::BlockScan<int, kScanThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int s_base;
    const int64_t it = blockIdx.x;
    unsigned char* mk = marks + it * n;
    const int* c = cand + it * cnt;
    for (int64_t j = threadIdx.x; j < cnt; j += blockDim.x) mk[c[j]] = 1;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    int* out = slots + it * tau;
    for (int64_t v0 = 0; v0 < n; v0 += kScanThreads) {
        const int64_t v = v0 + threadIdx.x;
        const int keep = (v < n && !mk[v]) ? 1 : 0;
        int pos, total;
        Scan(tmp).ExclusiveSum(keep, pos, total);
        if (keep) out[s_base + pos] = (int)v;
        __syncthreads();
        if (threadIdx.x == 0) s_base += total;
        __syncthreads();
    }
}

__global__ void philox_kernel(int64_t count, const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        u32x4 c{ctr[4 * t], ctr[4 * t + 1], ctr[4 * t + 2], ctr[4 * t + 3]};
        u32x4 o = philox4x32_10(c, key[2 * t], key[2 * t + 1]);
        out[4 * t] = o.x;
        out[4 * t + 1] = o.y;
        out[4 * t + 2] = o.z;
        out[4 * t + 3] = o.w;
    }
}

__global__ void philox_curand_kernel(int64_t count, uint64_t seed, unsigned long long* mismatches) {
    unsigned long long bad = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        // pseudo-random (ctr, key) derived from t and seed through our own generator
        u32x4 h = philox4x32_10(u32x4{(uint32_t)t, (uint32_t)(t >> 32), 0x1234567u, 0x89abcdefu},
                                (uint32_t)seed, (uint32_t)(seed >> 32));
        u32x4 h2 = philox4x32_10(u32x4{h.w, h.z, h.y, h.x}, h.x, h.y);
        const uint4 c4 = make_uint4(h.x, h.y, h.z, h.w);
        const uint2 k2 = make_uint2(h2.x, h2.y);
        const uint4 ref = curand_Philox4x32_10(c4, k2);
        const u32x4 ours = philox4x32_10(u32x4{h.x, h.y, h.z, h.w}, h2.x, h2.y);
        bad += (ref.x != ours.x) + (ref.y != ours.y) + (ref.z != ours.z) + (ref.w != ours.w);
    }
    if (bad) atomicAdd(mismatches, bad);
}

inline int blocks_for(int64_t work, int threads, int max_blocks) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (int)b;
}

}  // namespace

namespace pcdm_internal {

size_t sampler_bytes_per_iter(int64_t n, int64_t tau, int* log2h_out, bool no_complement) {
    const bool comp = 2 * tau > n && !no_complement;
    const int64_t cnt = comp ? n - tau : tau;
    int log2h = 0;
    while ((int64_t(1) << log2h) < 2 * cnt) ++log2h;
    if (log2h_out) *log2h_out = log2h;
    size_t bytes = ((size_t)1 << log2h) * 8 + (size_t)cnt * 4 * 2 + sizeof(int);
    if (comp) bytes += (size_t)cnt * 4 + (size_t)n;
    return bytes;
}

cudaError_t sample_chunk(const SamplerWork& w, const SamplingDev& sd, uint64_t seed, int64_t k0, int64_t count,
                         int* slots, int* flags, cudaStream_t st, int sms, int64_t* launches) {
    cudaError_t e;
    DrawArgs a;
    a.seed = seed;
    a.n = (uint64_t)w.n;
    a.reject_below = (uint64_t)(0 - (uint64_t)w.n) % (uint64_t)w.n;
    a.tag = w.complement ? 2u : 1u;
    a.cnt = w.cnt;
    a.log2h = w.log2h;
    const int blocks = blocks_for(count * w.cnt, 256, sms * 8);
    if (sd.kind == 1) {  // tau-independent: one ownership pass, no redraws of collisions
        e = cudaMemsetAsync(w.tables, 0xFF, (size_t)count * ((size_t)1 << w.log2h) * 8, st);
        if (e != cudaSuccess) return e;
        // entry indices in the (otherwise unused) pending area: count * cnt ints; the insert
        // pass in 128-thread blocks, up to 8 waves (as round 0 of the tau-nice sampler)
        const int ib = blocks_for(count * w.cnt, 128, sms * 16 * 8);
        sample_indep_insert_kernel<<<ib, 128, 0, st>>>(a, k0, count, w.tables, slots, w.pending);
        sample_indep_check_kernel<<<blocks, 256, 0, st>>>(a, count, w.tables, slots, w.pending);
        *launches += 2;
        return cudaGetLastError();
    }
    int* cand = w.complement ? w.cand : slots;
    if (w.cnt > 0) {
        e = cudaMemsetAsync(w.tables, 0xFF, (size_t)count * ((size_t)1 << w.log2h) * 8, st);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(w.npending, 0, (size_t)count * 2 * sizeof(int), st);  // + contest counters
        if (e != cudaSuccess) return e;
        // CAS straight on the home entry (the tables were just cleared): huge sampler
        // 8.23 -> 7.05 ms/step, large 8.80 -> 7.68 (profiles/r01_sampler_cas_first_ab.jsonl);
        // PCDM_CAS_FIRST=0 restores load-then-CAS
        const bool cas_first = [] {
            const char* v = knob("PCDM_CAS_FIRST");
            return !(v && atoi(v) == 0);
        }();
        // round 0 records where each value landed, so the check pass reads that entry
        // instead of probing (huge sampler 7.57 -> 6.03 ms/step,
        // profiles/r01_sampler_check_at_ab.jsonl); PCDM_CHECK_AT=0 probes
        const bool rec_at = [] {
            const char* v = knob("PCDM_CHECK_AT");
            return !(v && atoi(v) == 0);
        }();
        // contest mode (default with CAS-first): duplicates recorded at insert time, no
        // check pass over all slots (PCDM_CONTEST=0: check pass)
        const bool contest = [] {
            const char* v = knob("PCDM_CONTEST");
            return !(v && atoi(v) == 0);
        }();
        const int cm = cas_first && contest ? 1 : 0;
        if (cas_first) {
            // round 0 in 128-thread blocks, up to 8 waves of them: fewer draws per thread and
            // block-level load balance for the CAS round trips (huge sampler 4.0 -> 3.5 ms/step,
            // profiles/r01_sampler_r0_shape_ab.jsonl; PCDM_R0_TPB / PCDM_R0_WAVES for A/B)
            const int r0_tpb = [] {
                const char* v = knob("PCDM_R0_TPB");
                const int x = v ? atoi(v) : 128;
                return (x == 64 || x == 128 || x == 256 || x == 512 || x == 1024) ? x : 128;
            }();
            const int r0_waves = [] {
                const char* v = knob("PCDM_R0_WAVES");
                const int x = v ? atoi(v) : 8;
                return x >= 1 && x <= 64 ? x : 8;
            }();
            const int r0_blocks = blocks_for(count * w.cnt, r0_tpb, sms * (2048 / r0_tpb) * r0_waves);
            sample_round0_kernel<true><<<r0_blocks, r0_tpb, 0, st>>>(a, k0, count, w.tables, cand,
                                                               (rec_at || cm) ? w.pending : nullptr, w.npending, cm);
        } else {
            sample_round0_kernel<false><<<blocks, 256, 0, st>>>(a, k0, count, w.tables, cand, nullptr, w.npending, 0);
        }
        if (!cm) {
            if (cas_first && rec_at)
                sample_check_kernel<true><<<blocks, 256, 0, st>>>(a, count, w.tables, cand, w.pending, w.npending);
            else
                sample_check_kernel<false><<<blocks, 256, 0, st>>>(a, count, w.tables, cand, w.pending, w.npending);
            ++*launches;
        }
        sample_rounds_kernel<<<(unsigned)count, 1024, 0, st>>>(a, k0, count, w.tables, cand, w.pending, w.npending,
                                                               w.rounds_max, flags, cm);
        *launches += 2;
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (w.complement) {
        e = cudaMemsetAsync(w.marks, 0, (size_t)count * (size_t)w.n, st);
        if (e != cudaSuccess) return e;
        sample_complement_kernel<<<(unsigned)count, kScanThreads, 0, st>>>(w.n, w.tau, w.cnt, w.cand, w.marks,
                                                                          slots);
        ++*launches;
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const int tblocks = blocks_for(count * w.tau, 256, sms * 8);
    if (sd.kind == 2 && !sd.thin_always) {
        sample_thin_kernel<<<tblocks, 256, 0, st>>>(seed, k0, count, w.tau, sd.thin_T, slots);
        ++*launches;
        e = cudaGetLastError();
    } else if (sd.kind == 3) {
        sample_du_size_kernel<<<blocks_for(count, 128, sms), 128, 0, st>>>(seed, k0, count, w.tau, sd.du_T,
                                                                           sd.du_always_from, w.npending);
        sample_du_mask_kernel<<<tblocks, 256, 0, st>>>(count, w.tau, w.npending, slots);
        *launches += 2;
        e = cudaGetLastError();
    }
    return e;
}

cudaError_t launch_philox(int64_t count, const uint32_t* ctr, const uint32_t* key, uint32_t* out,
                          cudaStream_t st) {
    philox_kernel<<<blocks_for(count, 256, 4096), 256, 0, st>>>(count, ctr, key, out);
    return cudaGetLastError();
}

cudaError_t launch_philox_check_curand(int64_t count, uint64_t seed, unsigned long long* mismatches,
                                       cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(mismatches, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    philox_curand_kernel<<<blocks_for(count, 256, 4096), 256, 0, st>>>(count, seed, mismatches);
    return cudaGetLastError();
}

}  // namespace pcdm_internal
