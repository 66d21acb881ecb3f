// internal.h -- launch functions shared between the libpcdm translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pcdm_internal {

// Tuning and test knobs (A/B measurements, forced layouts / loops in tests) are
// environment variables read ONLY when PCDM_DEBUG_KNOBS=1, on every call (no
// process-wide caching); any other process runs the measured defaults whatever its
// environment holds.  Returns the variable's value or nullptr.
const char* knob(const char* name);

struct DevCSC {
    int64_t m, n, nnz;
    const int64_t* colptr;  // device int64[n+1]
    const int* rowidx;      // device int32[nnz]
    const float* val;       // device float[nnz]
};

// ---- setup / occasional kernels (kernels_setup.cu)
// L != nullptr: the same pass also writes L_i = ||a_i||^2 (fp64 sums) for valid column tiles
cudaError_t launch_validate(const DevCSC& A, int* flags, cudaStream_t st, int sms, int64_t* launches,
                            float* L = nullptr);
cudaError_t launch_check_finite(int64_t count, const float* v, int flag_bit, int* flags, cudaStream_t st,
                                int sms, int64_t* launches);
cudaError_t launch_row_counts(const DevCSC& A, int* counts, cudaStream_t st, int sms, int64_t* launches);
cudaError_t launch_max(int64_t count, const int* v, int* out, cudaStream_t st, int sms, int64_t* launches);
// rows with counts[j] >= threshold -> (rows, cnts)[0 .. min(*n_out, cap)), *n_out = all of them
cudaError_t launch_hot_candidates(int64_t m, const int* counts, int threshold, int* rows, int* cnts, int* n_out,
                                  int cap, cudaStream_t st, int sms, int64_t* launches);
cudaError_t launch_col_norms(const DevCSC& A, float* L, cudaStream_t st, int sms, int64_t* launches);
// x in the packed block headers (kernels_packed.cu): the residual pass also copies every
// nonzero x_i into its header and appends i to the dirty list
struct XHeaders {
    int4* blocks;
    int G;
    const long long* off;  // ragged layout: chunk offset of column i (nullptr: uniform, i * G)
    int* list;
    unsigned long long* count;
    int64_t cap;
};
// Row-major copy of A (built for dense iterates: the logistic problem)
struct DevCSR {
    const int64_t* rowptr;  // [m+1]
    const int* col;         // [nnz]
    const float* val;       // [nnz]
};
// r64 = A x - b in fp64: column scatter with fp64 atomics, or (csr given) a warp per row
// without atomics; both also copy nonzero x_i into the block headers when xh is given
cudaError_t launch_residual64(const DevCSC& A, const float* b, const float* x, double* r64, int* flags,
                              cudaStream_t st, int sms, int64_t* launches, const XHeaders* xh = nullptr,
                              const DevCSR* csr = nullptr);
cudaError_t build_csr(const DevCSC& A, const int* counts, DevCSR* out, cudaStream_t st, int sms, int64_t* launches);
cudaError_t launch_round_r(int64_t m, const double* r64, float* r, cudaStream_t st, int sms,
                           int64_t* launches, float* r2 = nullptr, int* zero = nullptr, int nzero = 0);
cudaError_t launch_objective_sums(int64_t m, int64_t n, const double* r64, const float* x, double* out,
                                  cudaStream_t st, int sms, int64_t* launches);

// L2-regularised logistic problem (NEXT-3): label check (+-1, flags FLAG_NONFINITE_B
// otherwise) and A~ = diag(y) A in place; L scaling; objective sums
cudaError_t launch_logistic_setup(int64_t m, int64_t nnz, const int* rowidx, const float* y, float* val, int* flags,
                                  cudaStream_t st, int sms, int64_t* launches);
cudaError_t launch_scale(int64_t n, float a, float* v, cudaStream_t st, int sms, int64_t* launches);
cudaError_t launch_objective_logistic(int64_t m, int64_t n, const double* s64, const float* x, double* out,
                                      cudaStream_t st, int sms, int64_t* launches);

// ---- samplers (kernels_sampler.cu)
// Doubly uniform samplings of PAPER.md:418-456 (pcdm_sampling_kind); the slot
// arrays hold tau entries per iteration, -1 for an idle processor.
struct SamplingDev {
    int kind;                  // 0 nice, 1 independent, 2 binomial, 3 du
    uint64_t thin_T;           // binomial: processor available iff word < thin_T ...
    int thin_always;           // ... or always (p_b >= 1)
    const uint64_t* du_T;      // du: device thresholds floor(cum_s 2^64), s < tau
    int64_t du_always_from;    // du: first s with cum_s >= 1 (tau if none)
};
struct SamplerWork {
    int64_t n, tau, cnt;        // cnt = slots drawn per iteration (tau or n - tau)
    bool complement;            // 2 tau > n: draw the n - tau excluded values
    int log2h;                  // hash table of 2^log2h uint64 entries per iteration
    int64_t chunk;              // iterations per sampler pass
    unsigned long long* tables; // [chunk][2^log2h]
    int* cand;                  // [chunk][cnt] owned values (== slots when !complement)
    int* pending;               // [chunk][cnt] pending slot lists
    int* npending;              // [chunk]
    unsigned char* marks;       // [chunk][n] (complement only)
    int* rounds_max;            // device scalar
};
// Fill slots[it * tau + j] for it in [0, count), iterations k = k0 + it.
cudaError_t sample_chunk(const SamplerWork& w, const SamplingDev& sd, uint64_t seed, int64_t k0, int64_t count,
                         int* slots, int* flags, cudaStream_t st, int sms, int64_t* launches);
size_t sampler_bytes_per_iter(int64_t n, int64_t tau, int* log2h_out, bool no_complement = false);

cudaError_t launch_philox(int64_t count, const uint32_t* ctr, const uint32_t* key, uint32_t* out,
                          cudaStream_t st);
cudaError_t launch_philox_check_curand(int64_t count, uint64_t seed, unsigned long long* mismatches,
                                       cudaStream_t st);

// ---- iteration kernels (kernels_iter.cu)
struct IterParams {
    const int64_t* colptr;
    const int* rowidx;
    const float* val;
    const float* L;
    float* x;
    float* r;
    const int* slots;     // [iters][tau]
    int64_t tau;
    int64_t iters;
    float beta;
    float lambda;
    int* nz_idx;          // [2][tau]
    float* nz_delta;      // [2][tau]
    int* nz_count;        // [2]
    unsigned* barrier;    // zeroed before launch
    int* flags;
    unsigned long long* nz_total;  // accumulates #delta != 0
    int64_t m, n;
    int logistic;         // 1: L2-regularised logistic loss (margins in r)
    // shared-memory variant: residual refreshes inside the kernel (r = fp32(Ax - b),
    // fp64 accumulation) after every run-local iteration k with (k + 1) % R == 0
    const float* b;
    int64_t k0;           // run-local index of this launch's first iteration
    int64_t R;            // refresh period (0: none)
};

struct IterLaunch {
    int variant;          // pcdm_variant actually used
    int ctas, threads, lanes;
    size_t smem;
    int entries;          // SMEM: 0 = the two-barrier list kernel; E > 0 = the one-barrier
                          // kernel (one slot per lane group, <= E entries per lane)
};

// ---- packed-block hot loop (kernels_packed.cu)
struct PackedParams {
    int4* blocks;         // [n][G] 16-byte chunks: {L, len, x (xlist), 0}, then (row, val) pairs
    float* x;
    float* r0;            // residual buffer (TWO_BARRIER: the residual)
    float* r1;            // second buffer (ONE_BARRIER only)
    const int* slots;     // [iters][tau]
    int64_t tau;
    int64_t iters;
    int64_t k0;           // run-local index of the first iteration of this launch
    float beta;
    float lambda;
    int* nz_idx;          // [3][tau]
    float* nz_delta;      // [3][tau]
    int* nz_count;        // [3]
    unsigned* barrier;
    int* flags;
    unsigned long long* nz_total;
    int logistic;         // 1: L2-regularised logistic loss (margins in r0/r1)
    int* xlist;           // non-null: x lives in the block headers; dirty list D of changed i
    unsigned long long* xlist_count;
    int64_t xlist_cap;
    const int* hot_rows;  // [nhot] ascending row ids of the hot rows (block row field 0x80000000 | h)
    int nhot;             // 0: no hot rows (blocks hold plain row ids)
    int pipeline;         // 1: the next slot's block is loaded before the current slot's gathers
    int cluster_sync;     // 1 / 2: the grid is one thread-block cluster of 512- / 1024-thread CTAs,
                          //        the barriers are barrier.cluster
    int list_cap;         // > 0: nonzero steps staged per CTA in shared memory (capacity), one
                          //      global atomic per CTA and iteration (dense-step workloads)
    int hot_cache;        // 1: copy r_k[hot_rows] into shared memory every iteration (else
                          //    hot entries are gathered through the row table)
    int bulk_stage;       // ragged layout: CTA-long column slices staged in shared memory by
                          //    cp.async.bulk (TMA engine) pieces, scattered from the staged copy
    int hot_stage;        // 1 (one-barrier scheme): scatters into hot rows accumulate in shared
                          //    memory per CTA, one red.global.add per hot row and CTA per iteration
    int local_cap;        // > 0 (one-barrier scheme): each CTA keeps its own steps in shared memory (capacity
                          //    per list) and replays them itself; no global step lists
    int reg_replay;       // 1 (one-barrier scheme, grid covers tau in one round): pcdm_packed1_kernel,
                          //    the previous step replayed from the registers of the group that took it
    // ragged layout (kernels_ragged.cu): per iteration the slots binned by class
    const int2* bins;     // [iters][tau] {i, chunk offset of column i}, grouped by class
    const int* bcnt;      // [iters][8] class starts (2, 4, 8, 16, 32 lanes, warp-long, CTA-long) and end
};
cudaError_t launch_xhdr_clear(int4* blocks, int G, const long long* off, const int* list,
                              const unsigned long long* count, int64_t cap, int64_t n, cudaStream_t st, int sms,
                              int64_t* launches);
cudaError_t launch_xhdr_out(const int4* blocks, int G, const long long* off, float* x, int64_t n, const int* list,
                            const unsigned long long* count, int64_t cap, cudaStream_t st, int sms,
                            int64_t* launches);
// ---- ragged layout (kernels_ragged.cu): a warp, sub-warp or CTA per sampled column by its length
// off[n+1] chunk offsets (g_i = pow2 >= 1 + ceil(len/2) for len <= 62, 1 + ceil(len/2) beyond);
// fails with cudaErrorInvalidValue when the blocks would exceed 2^32 chunks
// cls[n]: class of each column (0..4: 2..32 lanes, 5: warp-long, 6: CTA-long)
cudaError_t build_ragged(const DevCSC& A, const float* L, const int* hot_rows, int nhot, long long** off_out,
                         unsigned char** cls_out, int4** blocks_out, long long* total_out, cudaStream_t st, int sms,
                         int64_t* launches);
size_t bin_scratch_bytes(int64_t count);
// slots [count][tau] -> bins [count][tau] {i, off[i]} grouped by class, bcnt [count][8]
cudaError_t bin_chunk(const int* slots, int64_t tau, int64_t count, const long long* off, const unsigned char* cls,
                      int* scratch, int2* bins, int* bcnt, cudaStream_t st, int sms, int64_t* launches);
size_t ragged_smem_bytes(int nhot, bool bulk_stage);
int ragged_ctas(int sms, bool logistic, int nhot, bool bulk_stage);
cudaError_t launch_ragged(int ctas, const PackedParams& P, cudaStream_t st, int64_t* launches);
// asynchronous variant (NEXT-4): no barriers, no sampler pass
struct AsyncParams {
    const int4* blocks;
    float* x;
    float* r;
    int64_t n;
    int64_t updates;      // coordinate updates of this launch (all groups together)
    int64_t u0;           // global index of this launch's first update (resume)
    uint64_t seed;
    uint64_t reject_below;
    float beta;
    float lambda;
    int* flags;
    unsigned long long* nz_total;
    const int* hot_rows;  // decodes hot-row entries of the blocks (see PackedParams)
};
int async_groups(int G, int sms, int* ctas);
cudaError_t launch_async(int G, int ctas, const AsyncParams& A, cudaStream_t st, int64_t* launches);
int packed_lanes(int64_t max_len);
cudaError_t launch_gather_list(const float* x, const int* list, int64_t count, float* out, cudaStream_t st, int sms,
                               int64_t* launches);
cudaError_t launch_max_len(int64_t n, const int64_t* colptr, int* out, cudaStream_t st, int sms, int64_t* launches);
// rows listed in hot_rows[0..nhot) (ascending) are stored as 0x80000000 | h
cudaError_t launch_pack(int64_t n, int G, const int64_t* colptr, const int* rowidx, const float* val, const float* L,
                        const int* hot_rows, int nhot, int4* blocks, cudaStream_t st, int sms, int64_t* launches);
int packed_ctas(int G, bool one_barrier, int sms, bool logistic = false, int nhot = 0, int list_cap = 0,
                bool hot_stage = false, int local_cap = 0);
cudaError_t launch_packed(int G, bool one_barrier, int ctas, const PackedParams& P, cudaStream_t st,
                          int64_t* launches);
size_t packed_smem_bytes(int nhot, int list_cap = 0, bool hot_stage = false, int local_cap = 0);

// ---- batched-snapshot loop (kernels_batched.cu): passes expand / sweep / steps / fold
struct BatchedParams {
    int4* blocks;         // packed column blocks (as PackedParams)
    const int* slots;     // [iters][tau] of the chunk
    int64_t tau;
    int64_t iters;        // iterations of the chunk (c)
    float beta;
    float lambda;
    const float* r;       // residual (margins) r_0 at the start of the chunk, read-only in passes 1-3
    float* r_out;         // the same buffer, updated by the fold
    float* d0;            // D = r_k - r_0 double buffer, zero outside the chunk's dirty rows
    float* d1;
    float* g0;            // [iters * tau] a_i^T w(r_0) per chunk slot
    int2* gent;           // [nq][cq * maxe] sorted entries (row_local | slot_local << rb, val)
    int* offs;            // [nq][nb + 1] bin starts
    int nq, cq_log, nb, rb, maxe;
    int2* rec;            // [iters * tau][2 rnv] slot records: lane 0 {L_i, x_i}, lane t real rows 2t-2, 2t-1 (-1: none)
    int rnv;              // 16-byte vectors per slot record: 1 + ceil((max column length - 2) / 4), <= G / 2
    int* nz_idx;          // [iters][tau] nonzero steps per iteration
    float* nz_delta;      // [iters][tau]
    int* nz_count;        // [iters], zeroed before the chunk
    unsigned* barrier;
    int* flags;
    unsigned long long* nz_total;
    float* x;
    int* xlist;
    unsigned long long* xlist_count;
    int64_t xlist_cap;
    const int* hot_rows;
    int nhot;
    int logistic;
    // SCREENED step pass (LASSO; kernels_batched.cu passes 3s-4s): no grid barrier per
    // iteration.  The sweep takes every slot's step from g0 alone (the "speculative" step),
    // the test pass flags the slots a speculative step of an earlier iteration of the
    // chunk could change (shared row or column), and one CTA replays the chunk's
    // iterations over the speculative and flagged slots only, with the exact corrections.
    int screen;           // 1: passes 3s-4s replace pass 3 + fold
    int2* lx;             // [iters * tau] {L_i, x_i at the chunk start} (pass 1; L = -1 bits: idle slot)
    int* rows;            // [nrow][rows_ld] real rows of every slot (pass 1; -1: none)
    int64_t rows_ld;      // leading dimension of rows (>= iters * tau)
    int nrow;             // rows stored per slot (max column length)
    unsigned* bits;       // [ceil(rows_ld / 32)] slot is already an item (zero between chunks)
    int* items;           // [2][rows_ld]: speculative slots, then flagged slots
    int* counts;          // [4]: #speculative, #flagged, misses (run total), scans (run total)
    int fix_cap;          // (unused)
    int G;                // 16-byte chunks per column block (set by launch_batched)
    unsigned long long* tl;  // debug timeline of the chunk's kernels (nullptr: off)
    // the previous chunk's step lists (its fix-up may still run while this chunk's expand
    // reads x_i): the sweep re-reads x_i of the columns listed there; nullptr: none
    const int* prev_nz_idx;
    const int* prev_nz_count;
    int prev_iters;
};
// screened pass scheduling: the fix-up runs on its own stream after the test pass
// (ev_test) and the next chunk's sweep waits for it (ev_fix)
struct ScreenSched {
    cudaStream_t st2;
    cudaEvent_t ev_test, ev_fix;
};
size_t batched_step_smem(int nhot);
int batched_cq_log(int G);
int batched_rb(int cq_log);
int batched_ctas(int G, int sms, bool logistic, int nhot);
cudaError_t launch_batched(int G, const BatchedParams& P, int ctas3, cudaStream_t st, int sms, int64_t* launches,
                           const ScreenSched* sch = nullptr);



// Choose the launch shape for `variant` (AUTO resolved) given problem sizes.
IterLaunch plan_iter(int variant, int64_t m, int64_t n, int64_t nnz, int64_t tau, int sms, int device,
                     bool logistic = false, int64_t max_len = -1);
cudaError_t launch_iter(const IterLaunch& L, const IterParams& P, cudaStream_t st, int64_t* launches);

}  // namespace pcdm_internal
