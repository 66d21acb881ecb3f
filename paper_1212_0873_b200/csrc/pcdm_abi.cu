// pcdm_abi.cu -- host side of libpcdm.so: the C ABI declared in include/pcdm.h.
//
// Owns the problem handle (device copies of A, b, L, r, scratch), drives the
// create-time kernels, and runs the PCDM1 loop as alternating sampler passes
// and persistent iteration-kernel launches on the caller's stream.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/pcdm.h"
#include "common.cuh"
#include "internal.h"

using namespace pcdm_internal;

namespace pcdm_internal {
const char* knob(const char* name) {
    const char* dbg = getenv("PCDM_DEBUG_KNOBS");
    if (!dbg || atoi(dbg) == 0) return nullptr;
    return getenv(name);
}
}  // namespace pcdm_internal

namespace {

thread_local std::string g_error = "no error";

pcdm_status fail(pcdm_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_error = buf;
    return s;
}

pcdm_status cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? PCDM_ENOMEM : PCDM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(call, what)                                  \
    do {                                                \
        cudaError_t _e = (call);                        \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Scalars living in one small device block.
struct Scalars {
    int flags;
    int nz_count[3];
    int max_out;
    int rounds_max;
    unsigned long long nz_total;
    unsigned long long mismatches;
    double sums[2];
    alignas(128) unsigned barrier[pcdm::kBarrierWords];  // grid-barrier counter(s), common.cuh
};

}  // namespace

struct pcdm_problem {
    int device = 0;
    int sms = 148;
    int64_t m = 0, n = 0, nnz = 0;
    double lambda = 0.0;
    int64_t omega = 0;
    int loss = 0;              // 0: LASSO (square loss), 1: L2-regularised logistic
    int64_t* colptr = nullptr;
    int* rowidx = nullptr;
    float* val = nullptr;
    float* b = nullptr;
    float* L = nullptr;
    float* r = nullptr;        // residual (buffer 0)
    float* r2 = nullptr;       // second residual buffer (one-barrier packed loop)
    float* r_cur = nullptr;    // buffer holding the residual after the last run
    int4* blocks = nullptr;    // packed column blocks (PACKED variant), [n][packed_G]
    int* xlist = nullptr;      // dirty list D of columns whose block header may hold x_i != 0
    unsigned long long* xlist_count = nullptr;  // |D| (> cap: overflowed, walk all n)
    int64_t xlist_cap = 0;
    int packed_G = 0;          // uniform packed layout: lanes per column (0: none)
    // RAGGED packed layout (kernels_ragged.cu): column i at chunk offset blk_off[i], a warp,
    // sub-warp or CTA per sampled column by its length; chosen at create when a column is
    // longer than 62 entries or the longest column would at least double every column's lanes
    bool ragged = false;
    long long* blk_off = nullptr;
    unsigned char* blk_cls = nullptr;
    long long ragged_chunks = 0;
    int* bin_scr = nullptr;    // binning scratch of one sampler pass
    size_t bin_scr_cap = 0;
    int2* bins = nullptr;      // binned slot entries of the run's sampled windows / presampled run
    int* bcnt = nullptr;
    size_t bins_cap = 0;       // entries
    int* hot_rows = nullptr;   // ascending ids of the hot rows cached in shared memory (packed loop)
    int nhot = 0;
    int64_t hot_max_count = 0; // stored entries of the most frequent row
    DevCSR csr{};              // row-major copy of A (logistic problems: dense iterates)
    bool has_csr = false;
    float* d0 = nullptr;       // BATCHED: D = r_k - r_0 double buffer (zero between chunks)
    float* d1 = nullptr;
    void* bat_mem = nullptr;   // BATCHED per-chunk workspace (g0, sorted entries, offsets, lists)
    cudaStream_t fix_st = nullptr;  // screened step pass: the fix-up's stream (high priority)
    cudaEvent_t ev_test = nullptr, ev_fix = nullptr;
    size_t bat_cap = 0;
    int64_t max_len = 0;
    double* r64 = nullptr;
    float* xbuf = nullptr;     // device iterate when the caller passes host x
    float* xcomp = nullptr;    // changed entries of xbuf, gathered for the compact copy back
    int* hidx = nullptr;       // pinned host staging of the compact copy (indices, values)
    float* hval = nullptr;
    int64_t comp_cap = 0;
    int* slot_buf = nullptr;   // slot arrays of one iteration-kernel launch (when it spans several sampler chunks)
    size_t slot_cap = 0;
    int* pre_slots = nullptr;  // host-x runs: the whole run's slot arrays, drawn during the x copy
    size_t pre_cap = 0;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_s0 = nullptr, ev_s1 = nullptr;
    std::vector<cudaEvent_t> pass_ev;  // PCDM_PRESAMPLE_DEV: one event per presampler pass
    // AUTO BATCHED guard: the nonzero-step count, read back without stalling the stream
    unsigned long long* nz_host = nullptr;
    cudaEvent_t ev_nz = nullptr;
    Scalars* sc = nullptr;     // device scalars
    // per-run workspaces (grown on demand)
    int* nz_idx = nullptr;
    float* nz_delta = nullptr;
    int64_t nz_cap = 0;
    void* samp_mem = nullptr;
    size_t samp_cap = 0;
    uint64_t* du_T = nullptr;  // DU-sampling thresholds
    size_t du_cap = 0;
    pcdm_run_stats stats{};
    std::vector<cudaEvent_t> events;  // timing events, reused across runs
    DevCSC csc() const { return DevCSC{m, n, nnz, colptr, rowidx, val}; }
};

namespace {

template <typename T>
pcdm_status dev_copy_in(T** dst, const T* src, size_t count, cudaStream_t st, const char* what) {
    CK(cudaMalloc((void**)dst, sizeof(T) * (count ? count : 1)), what);
    if (count) CK(cudaMemcpyAsync(*dst, src, sizeof(T) * count, cudaMemcpyDefault, st), what);
    return PCDM_OK;
}

void free_problem(pcdm_problem* p) {
    if (!p) return;
    cudaFree(p->colptr);
    cudaFree(p->rowidx);
    cudaFree(p->val);
    cudaFree(p->b);
    cudaFree(p->L);
    cudaFree(p->r);
    cudaFree(p->r64);
    cudaFree(p->r2);
    cudaFree(p->blocks);
    cudaFree(p->blk_off);
    cudaFree(p->blk_cls);
    cudaFree(p->bin_scr);
    cudaFree(p->bins);
    cudaFree(p->bcnt);
    cudaFree(p->hot_rows);
    if (p->has_csr) {
        cudaFree((void*)p->csr.rowptr);
        cudaFree((void*)p->csr.col);
        cudaFree((void*)p->csr.val);
    }
    cudaFree(p->d0);
    cudaFree(p->d1);
    cudaFree(p->bat_mem);
    if (p->fix_st) {
        cudaStreamDestroy(p->fix_st);
        cudaEventDestroy(p->ev_test);
        cudaEventDestroy(p->ev_fix);
    }
    cudaFree(p->xlist);
    cudaFree(p->xlist_count);
    cudaFree(p->xbuf);
    cudaFree(p->xcomp);
    cudaFreeHost(p->hidx);
    cudaFreeHost(p->hval);
    cudaFree(p->pre_slots);
    cudaFree(p->slot_buf);
    if (p->side) {
        cudaStreamDestroy(p->side);
        cudaEventDestroy(p->ev_fork);
        cudaEventDestroy(p->ev_s0);
        cudaEventDestroy(p->ev_s1);
    }
    for (cudaEvent_t e : p->pass_ev) cudaEventDestroy(e);
    if (p->ev_nz) cudaEventDestroy(p->ev_nz);
    cudaFreeHost(p->nz_host);
    cudaFree(p->sc);
    cudaFree(p->nz_idx);
    cudaFree(p->nz_delta);
    cudaFree(p->samp_mem);
    cudaFree(p->du_T);
    for (cudaEvent_t e : p->events) cudaEventDestroy(e);
    delete p;
}

const char* flag_text(int f) {
    if (f & FLAG_BAD_COLPTR) return "colptr must start at 0, end at nnz and be non-decreasing";
    if (f & FLAG_BAD_ROW) return "row index out of [0, m)";
    if (f & FLAG_ROW_ORDER) return "row indices must be strictly increasing within each column";
    if (f & FLAG_NONFINITE_VAL) return "non-finite value in val";
    if (f & FLAG_NONFINITE_B) return "non-finite value in b";
    if (f & FLAG_NONFINITE_X) return "non-finite value in x";
    return "invalid input";
}

pcdm_status read_scalars(pcdm_problem* p, Scalars* host, cudaStream_t st) {
    CK(cudaMemcpyAsync(host, p->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st), "read scalars");
    CK(cudaStreamSynchronize(st), "stream synchronize");
    return PCDM_OK;
}

// r <- A x - b with fp64 accumulation (x device pointer).
// r2 / zero: the rounding pass also fills the one-barrier loop's second buffer and
// clears its step-list counters
pcdm_status residual_from(pcdm_problem* p, const float* x, cudaStream_t st, int64_t* launches,
                          const XHeaders* xh = nullptr, float* r2 = nullptr, int* zero = nullptr, int nzero = 0) {
    CK(launch_residual64(p->csc(), p->b, x, p->r64, &p->sc->flags, st, p->sms, launches, xh,
                         p->has_csr ? &p->csr : nullptr),
       "residual kernels");
    CK(launch_round_r(p->m, p->r64, p->r, st, p->sms, launches, r2, zero, nzero), "residual rounding");
    return PCDM_OK;
}

// Device-time accounting of a run: event pairs recorded on the run's stream
// around each phase; summed after the final synchronisation.
struct RunTimer {
    pcdm_problem* p;
    cudaStream_t st;
    std::vector<std::pair<int, int>> marks;  // (kind, index of the start event)
    int used = 0;
    cudaError_t record(int* idx) {
        if ((int)p->events.size() <= used) {
            cudaEvent_t e;
            cudaError_t err = cudaEventCreate(&e);
            if (err != cudaSuccess) return err;
            p->events.push_back(e);
        }
        *idx = used++;
        return cudaEventRecord(p->events[*idx], st);
    }
    cudaError_t begin(int* idx) { return record(idx); }
    cudaError_t end(int kind, int start_idx) {
        int e;
        cudaError_t err = record(&e);
        marks.push_back({kind, start_idx});
        return err;
    }
    void sum(double out[3]) {
        out[0] = out[1] = out[2] = 0.0;
        for (auto& mk : marks) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, p->events[mk.second], p->events[mk.second + 1]) == cudaSuccess)
                out[mk.first] += ms;
        }
        cudaGetLastError();
    }
};
enum { T_ITER = 0, T_SAMPLER = 1, T_SETUP = 2 };

int64_t refresh_period(int64_t n, int64_t tau, int64_t refresh_every) {
    if (refresh_every < 0) return 0;
    if (refresh_every > 0) return refresh_every;
    return (2 * n + tau - 1) / tau;
}

struct SamplerPlan {
    SamplerWork w;
    int* slots;
};

// Carve the sampler + slot workspace for `chunk` iterations out of p->samp_mem.
pcdm_status sampler_workspace(void** mem, size_t* cap, int64_t n, int64_t tau, int64_t chunk, SamplerPlan* sp,
                              bool no_complement = false) {
    int log2h = 0;
    sampler_bytes_per_iter(n, tau, &log2h, no_complement);
    const bool comp = 2 * tau > n && !no_complement;
    const int64_t cnt = comp ? n - tau : tau;
    auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
    size_t off = 0;
    const size_t o_tables = off; off += al((size_t)chunk * ((size_t)1 << log2h) * 8);
    const size_t o_slots = off; off += al((size_t)chunk * tau * 4);
    const size_t o_cand = off; off += comp ? al((size_t)chunk * cnt * 4) : 0;
    const size_t o_pend = off; off += al((size_t)chunk * 2 * (cnt ? cnt : 1) * 4);
    const size_t o_np = off; off += al((size_t)chunk * 8);  // npending[chunk] + ncontest[chunk]
    const size_t o_marks = off; off += comp ? al((size_t)chunk * n) : 0;
    const size_t o_rmax = off; off += 256;
    if (off > *cap) {
        cudaFree(*mem);
        *mem = nullptr;
        *cap = 0;
        CK(cudaMalloc(mem, off), "sampler workspace");
        *cap = off;
    }
    char* base = (char*)*mem;
    sp->w.n = n;
    sp->w.tau = tau;
    sp->w.cnt = cnt;
    sp->w.complement = comp;
    sp->w.log2h = log2h;
    sp->w.chunk = chunk;
    sp->w.tables = (unsigned long long*)(base + o_tables);
    sp->w.cand = comp ? (int*)(base + o_cand) : nullptr;
    sp->w.pending = (int*)(base + o_pend);
    sp->w.npending = (int*)(base + o_np);
    sp->w.marks = comp ? (unsigned char*)(base + o_marks) : nullptr;
    sp->w.rounds_max = (int*)(base + o_rmax);
    sp->slots = (int*)(base + o_slots);
    return PCDM_OK;
}

int64_t choose_chunk(int64_t n, int64_t tau, int64_t iters) {
    // one sampler pass's tables + slots within a budget: large enough that the per-pass
    // launches amortise, small enough that the random atomics mostly stay in L2
    const size_t per = sampler_bytes_per_iter(n, tau, nullptr) + (size_t)tau * 4;
    // 128 MB per sampler pass: huge 5.90 -> 5.17 ms/step of sampler, large 6.87 -> 5.54
    // (profiles/r01_sampler_mb_ab.jsonl; 256 MB is no better)
    size_t budget = (size_t)128 << 20;
    if (const char* mb = knob("PCDM_SAMPLER_MB")) budget = (size_t)std::max(1, atoi(mb)) << 20;
    int64_t c = (int64_t)std::max<size_t>(1, budget / per);
    c = std::min<int64_t>(c, 8192);
    if (const char* fc = knob("PCDM_CHUNK")) c = std::max<int64_t>(1, atoll(fc));  // tests / tuning
    return std::min<int64_t>(c, std::max<int64_t>(iters, 1));
}

// A sampling of the run (pcdm_sampling, validated) plus what the device needs.
struct SamplingSpec {
    int kind = PCDM_SAMPLING_NICE;
    int64_t tau = 1;
    double p_b = 1.0;
    std::vector<double> q;
};

pcdm_status check_sampling(const pcdm_sampling* sp, int64_t n, SamplingSpec* out) {
    if (!sp) return fail(PCDM_EINVAL, "NULL sampling");
    out->kind = sp->kind;
    out->tau = sp->tau;
    out->p_b = sp->p_b;
    if (sp->kind < PCDM_SAMPLING_NICE || sp->kind > PCDM_SAMPLING_DU) return fail(PCDM_EINVAL, "unknown sampling kind %d", sp->kind);
    if (sp->tau < 1 || sp->tau > n) return fail(PCDM_EINVAL, "tau must be in [1, n]");
    if (sp->kind == PCDM_SAMPLING_BINOMIAL && !(sp->p_b > 0.0 && sp->p_b <= 1.0))
        return fail(PCDM_EINVAL, "binomial sampling needs 0 < p_b <= 1");
    if (sp->kind == PCDM_SAMPLING_DU) {
        if (!sp->q) return fail(PCDM_EINVAL, "DU sampling needs q[0..tau]");
        if (2 * sp->tau > n) return fail(PCDM_EINVAL, "DU sampling needs 2 tau <= n");
        double sum = 0.0;
        out->q.assign(sp->q, sp->q + sp->tau + 1);
        for (double v : out->q) {
            if (!(v >= 0.0 && v <= 1.0)) return fail(PCDM_EINVAL, "q entries must be in [0, 1]");
            sum += v;
        }
        if (!(fabs(sum - 1.0) <= 1e-9)) return fail(PCDM_EINVAL, "q must sum to 1 (sum %.17g)", sum);
    }
    return PCDM_OK;
}

// (E|S|, E|S|^2) of the sampling (thm:ESO-DU inputs):
//   nice tau, tau^2; binomial tau p_b, tau p_b (1 + tau p_b - p_b);
//   DU sum k q_k, sum k^2 q_k; tau-independent = occupied bins of tau balls in n
//   bins: E|S| = n(1 - a), E|S|^2 = E|S| + n(n-1)(1 - 2a + b), a = (1-1/n)^tau,
//   b = (1-2/n)^tau, evaluated through expm1/log1p (1-2a+b = 2(1-a) - (1-b)).
void sampling_moments(const SamplingSpec& sp, int64_t n, double* e1, double* e2) {
    const double t = (double)sp.tau, nn = (double)n;
    switch (sp.kind) {
        case PCDM_SAMPLING_INDEPENDENT: {
            const double one_minus_a = -expm1(t * log1p(-1.0 / nn));
            const double one_minus_b = n >= 2 ? -expm1(t * log1p(-2.0 / nn)) : 1.0;
            *e1 = nn * one_minus_a;
            *e2 = *e1 + nn * (nn - 1.0) * (2.0 * one_minus_a - one_minus_b);
            return;
        }
        case PCDM_SAMPLING_BINOMIAL:
            *e1 = t * sp.p_b;
            *e2 = t * sp.p_b * (1.0 + t * sp.p_b - sp.p_b);
            return;
        case PCDM_SAMPLING_DU: {
            double a1 = 0.0, a2 = 0.0;
            for (size_t k = 0; k < sp.q.size(); ++k) {
                a1 += (double)k * sp.q[k];
                a2 += (double)k * (double)k * sp.q[k];
            }
            *e1 = a1;
            *e2 = a2;
            return;
        }
        default:
            *e1 = t;
            *e2 = t * t;
    }
}

// beta = 1 + (omega-1)(E|S|^2/E|S| - 1)/max(1,n-1)  (thm:ESO-DU)
double sampling_beta(const SamplingSpec& sp, int64_t omega, int64_t n) {
    if (sp.kind == PCDM_SAMPLING_NICE) {  // the north_star form, thm:ESO-nice
        const double denom = (double)std::max<int64_t>(1, n - 1);
        return 1.0 + (double)(omega - 1) * (double)(sp.tau - 1) / denom;
    }
    double e1, e2;
    sampling_moments(sp, n, &e1, &e2);
    if (!(e1 > 0.0)) return 1.0;
    return 1.0 + (double)(omega - 1) * (e2 / e1 - 1.0) / (double)std::max<int64_t>(1, n - 1);
}

// floor(p 2^64) (p < 1) or "always" (p >= 1), exactly as the oracle's reading R17/R18
uint64_t prob_threshold(double p, int* always) {
    *always = 0;
    if (p >= 1.0) {
        *always = 1;
        return ~0ull;
    }
    if (p <= 0.0) return 0;
    return (uint64_t)(p * 18446744073709551616.0);
}

// Device-side description; DU thresholds go to `dev_T` (tau entries).
pcdm_status sampling_dev(const SamplingSpec& sp, uint64_t** dev_T, size_t* cap, cudaStream_t st, SamplingDev* out) {
    out->kind = sp.kind;
    out->thin_T = 0;
    out->thin_always = 1;
    out->du_T = nullptr;
    out->du_always_from = sp.tau;
    if (sp.kind == PCDM_SAMPLING_BINOMIAL) out->thin_T = prob_threshold(sp.p_b, &out->thin_always);
    if (sp.kind == PCDM_SAMPLING_DU) {
        std::vector<uint64_t> T((size_t)sp.tau);
        double cum = 0.0;
        for (int64_t s = 0; s < sp.tau; ++s) {
            cum += sp.q[(size_t)s];
            int always = 0;
            T[(size_t)s] = prob_threshold(cum, &always);
            if (always && out->du_always_from == sp.tau) out->du_always_from = s;
        }
        if (*cap < T.size()) {
            cudaFree(*dev_T);
            *dev_T = nullptr;
            *cap = 0;
            CK(cudaMalloc((void**)dev_T, sizeof(uint64_t) * T.size()), "DU thresholds");
            *cap = T.size();
        }
        CK(cudaMemcpyAsync(*dev_T, T.data(), sizeof(uint64_t) * T.size(), cudaMemcpyHostToDevice, st), "DU thresholds");
        CK(cudaStreamSynchronize(st), "DU thresholds");  // T is a stack vector
        out->du_T = *dev_T;
    }
    return PCDM_OK;
}

pcdm_status run_impl(pcdm_problem* p, float* x, const SamplingSpec& spec, int64_t iters, uint64_t seed,
                     int64_t first_iter, int64_t refresh_every, double beta_override, int32_t variant, void* stream);
pcdm_status create_impl(int64_t m, int64_t n, int64_t nnz, const int64_t* colptr, const int32_t* rowidx,
                        const float* val, const float* b, double lambda, int loss, void* stream, pcdm_problem** out);

}  // namespace

extern "C" {

const char* pcdm_last_error(void) { return g_error.c_str(); }

pcdm_status pcdm_create(int64_t m, int64_t n, int64_t nnz, const int64_t* colptr, const int32_t* rowidx,
                        const float* val, const float* b, double lambda, void* stream, pcdm_problem** out) {
    return create_impl(m, n, nnz, colptr, rowidx, val, b, lambda, 0, stream, out);
}

pcdm_status pcdm_create_logistic(int64_t m, int64_t n, int64_t nnz, const int64_t* colptr, const int32_t* rowidx,
                                 const float* val, const float* y, double lambda, void* stream, pcdm_problem** out) {
    return create_impl(m, n, nnz, colptr, rowidx, val, y, lambda, 1, stream, out);
}

}  // extern "C"

namespace {

// Hot rows of the packed loop (kernels_packed.cu): rows stored at least
// max(64, 32 x the mean row count) times, the PCDM_HOT_MAX (default 2048) most
// frequent of them.  Every iteration reads such a row about count_j tau / n times;
// those same-address reads serialise in one L2 slice unless they are served from
// the per-CTA shared-memory copy.  Uniform-row configs have none (omega is far
// below the threshold).  PCDM_HOT_ROWS=0 disables.
pcdm_status select_hot_rows(pcdm_problem* p, const int* counts, cudaStream_t st, int64_t* launches) {
    p->nhot = 0;
    const char* en = knob("PCDM_HOT_ROWS");
    if (en && atoi(en) == 0) return PCDM_OK;
    int hmax = 2048;
    if (const char* hm = knob("PCDM_HOT_MAX")) hmax = std::max(0, std::min(8192, atoi(hm)));
    if (hmax == 0) return PCDM_OK;
    const int64_t mean = (p->nnz + p->m - 1) / p->m;
    const int64_t thr64 = std::max<int64_t>(64, 32 * mean);
    if (thr64 > 0x7fffffff) return PCDM_OK;
    const int cap = 1 << 16;
    int *rows = nullptr, *cnts = nullptr, *nout = nullptr;
    cudaError_t e = cudaMalloc((void**)&rows, sizeof(int) * (2 * cap + 1));
    if (e != cudaSuccess) return cuda_fail(e, "alloc hot candidates");
    cnts = rows + cap;
    nout = rows + 2 * cap;
    int total = 0;
    std::vector<int> hr, hc;
    e = launch_hot_candidates(p->m, counts, (int)thr64, rows, cnts, nout, cap, st, p->sms, launches);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&total, nout, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    const int got = std::min(total, cap);
    if (e == cudaSuccess && got > 0) {
        hr.resize(got);
        hc.resize(got);
        e = cudaMemcpyAsync(hr.data(), rows, sizeof(int) * got, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), cnts, sizeof(int) * got, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    cudaFree(rows);
    if (e != cudaSuccess) return cuda_fail(e, "hot rows");
    if (got == 0) return PCDM_OK;
    // most frequent first (ties: lower row), keep hmax, then ascending row ids
    std::vector<int> order(got);
    for (int q = 0; q < got; ++q) order[q] = q;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return hc[a] != hc[b] ? hc[a] > hc[b] : hr[a] < hr[b]; });
    const int keep = std::min(got, hmax);
    std::vector<int> sel(keep);
    for (int q = 0; q < keep; ++q) sel[q] = hr[order[q]];
    std::sort(sel.begin(), sel.end());
    e = cudaMalloc((void**)&p->hot_rows, sizeof(int) * keep);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->hot_rows, sel.data(), sizeof(int) * keep, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "hot rows");
    p->nhot = keep;
    p->hot_max_count = hc[order[0]];
    return PCDM_OK;
}

// loss 0: LASSO with b; loss 1: L2-regularised logistic with labels y (the library
// stores A~ = diag(y) A, b = 0, L = ||a_i||^2 / 4; R21)
pcdm_status create_impl(int64_t m, int64_t n, int64_t nnz, const int64_t* colptr, const int32_t* rowidx,
                        const float* val, const float* b, double lambda, int loss, void* stream, pcdm_problem** out) {
    if (!out) return fail(PCDM_EINVAL, "out must not be NULL");
    *out = nullptr;
    if (m < 1 || n < 1 || nnz < 1) return fail(PCDM_EINVAL, "need m, n, nnz >= 1 (no loss terms otherwise)");
    if (m >= (1ll << 31) || n >= (1ll << 31)) return fail(PCDM_EINVAL, "m and n must be < 2^31");
    if (!colptr || !rowidx || !val || !b) return fail(PCDM_EINVAL, "NULL array argument");
    if (!(lambda >= 0.0) || lambda > 1e308) return fail(PCDM_EINVAL, "lambda must be finite and >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    pcdm_problem* p = new pcdm_problem();
    p->m = m;
    p->n = n;
    p->nnz = nnz;
    p->lambda = lambda;
    p->loss = loss;
    pcdm_status s = PCDM_OK;
    int64_t launches = 0;
    Scalars hs{};
    do {
        if (cudaGetDevice(&p->device) != cudaSuccess) { s = cuda_fail(cudaGetLastError(), "cudaGetDevice"); break; }
        cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, p->device);
        if ((s = dev_copy_in(&p->colptr, colptr, (size_t)n + 1, st, "copy colptr")) != PCDM_OK) break;
        if ((s = dev_copy_in(&p->rowidx, rowidx, (size_t)nnz, st, "copy rowidx")) != PCDM_OK) break;
        if ((s = dev_copy_in(&p->val, val, (size_t)nnz, st, "copy val")) != PCDM_OK) break;
        if ((s = dev_copy_in(&p->b, b, (size_t)m, st, loss ? "copy y" : "copy b")) != PCDM_OK) break;
        cudaError_t e;
        if ((e = cudaMalloc((void**)&p->sc, sizeof(Scalars))) != cudaSuccess) { s = cuda_fail(e, "scalars"); break; }
        if ((e = cudaMemsetAsync(p->sc, 0, sizeof(Scalars), st)) != cudaSuccess) { s = cuda_fail(e, "memset"); break; }
        // validation and the column norms L_i (a1) in one pass over the tiles of A
        if ((e = cudaMalloc((void**)&p->L, sizeof(float) * n)) != cudaSuccess) { s = cuda_fail(e, "alloc L"); break; }
        if ((e = launch_validate(p->csc(), &p->sc->flags, st, p->sms, &launches, p->L)) != cudaSuccess) { s = cuda_fail(e, "validate"); break; }
        if (loss == 0) {
            if ((e = launch_check_finite(m, p->b, FLAG_NONFINITE_B, &p->sc->flags, st, p->sms, &launches)) != cudaSuccess) { s = cuda_fail(e, "check b"); break; }
        } else {
            // labels +-1 (flagged as FLAG_NONFINITE_B otherwise), A~ = diag(y) A, then b = 0: r holds s = A~ x
            if ((e = launch_logistic_setup(m, nnz, p->rowidx, p->b, p->val, &p->sc->flags, st, p->sms, &launches)) != cudaSuccess) { s = cuda_fail(e, "labels"); break; }
            if ((e = cudaMemsetAsync(p->b, 0, sizeof(float) * m, st)) != cudaSuccess) { s = cuda_fail(e, "memset b"); break; }
        }
        if ((s = read_scalars(p, &hs, st)) != PCDM_OK) break;
        if (hs.flags) {
            s = fail(PCDM_EINVAL, "invalid input: %s",
                     (loss && (hs.flags & FLAG_NONFINITE_B)) ? "labels y must be +1 or -1" : flag_text(hs.flags));
            break;
        }
        if (loss == 1 && (e = launch_scale(n, 0.25f, p->L, st, p->sms, &launches)) != cudaSuccess) { s = cuda_fail(e, "L"); break; }
        int* counts = nullptr;
        if ((e = cudaMalloc((void**)&counts, sizeof(int) * m)) != cudaSuccess) { s = cuda_fail(e, "alloc counts"); break; }
        e = launch_row_counts(p->csc(), counts, st, p->sms, &launches);
        if (e == cudaSuccess) e = launch_max(m, counts, &p->sc->max_out, st, p->sms, &launches);
        if (e != cudaSuccess) { cudaFree(counts); s = cuda_fail(e, "row histogram"); break; }
        s = read_scalars(p, &hs, st);
        if (s == PCDM_OK) s = select_hot_rows(p, counts, st, &launches);
        // logistic problems: every visited coordinate becomes nonzero, so the margins
        // s = A~ x are recomputed at each run start / refresh from a row-major copy (a warp
        // per row, fp64 in registers) instead of nnz fp64 atomics (PCDM_ROW_RESIDUAL=0: off)
        const char* rr = knob("PCDM_ROW_RESIDUAL");
        if (s == PCDM_OK && loss == 1 && !(rr && atoi(rr) == 0)) {
            if (build_csr(p->csc(), counts, &p->csr, st, p->sms, &launches) == cudaSuccess) p->has_csr = true;
            else cudaGetLastError();  // out of memory: the column scatter stays
        }
        cudaFree(counts);
        if (s != PCDM_OK) break;
        p->omega = hs.max_out;
        // packed column blocks for the PACKED hot loop (skipped if a column is too long
        // or the device cannot hold the copy)
        if ((e = launch_max_len(n, p->colptr, &p->sc->max_out, st, p->sms, &launches)) != cudaSuccess) { s = cuda_fail(e, "max len"); break; }
        if ((s = read_scalars(p, &hs, st)) != PCDM_OK) break;
        p->max_len = hs.max_out;
        // layout: uniform G x 16 B blocks when every column fits 62 entries and the longest
        // column does not at least double the lanes of an average one; ragged otherwise
        // (PCDM_LAYOUT=uniform|ragged forces one, for tests and A/B runs)
        const int64_t avg_len = (nnz + n - 1) / n;
        const char* lay = knob("PCDM_LAYOUT");
        bool want_ragged = lay ? strcmp(lay, "ragged") == 0
                               : (p->max_len > 62 || packed_lanes(p->max_len) > 2 * packed_lanes(avg_len));
        if (want_ragged && !knob("PCDM_NO_PACK")) {
            e = build_ragged(p->csc(), p->L, p->hot_rows, p->nhot, &p->blk_off, &p->blk_cls, &p->blocks,
                             &p->ragged_chunks, st, p->sms, &launches);
            if (e == cudaSuccess) {
                p->ragged = true;
            } else {
                cudaGetLastError();  // too large / out of memory: the uniform layout or none
                want_ragged = false;
            }
        }
        if (!p->ragged && p->max_len <= 62 && !knob("PCDM_NO_PACK")) {
            const int G = packed_lanes(p->max_len);
            if (cudaMalloc((void**)&p->blocks, (size_t)n * G * 16) == cudaSuccess) {
                p->packed_G = G;
                if ((e = launch_pack(n, G, p->colptr, p->rowidx, p->val, p->L, p->hot_rows, p->nhot, p->blocks, st, p->sms, &launches)) != cudaSuccess) { s = cuda_fail(e, "pack"); break; }
            } else {
                cudaGetLastError();
                p->blocks = nullptr;
            }
        }
        if ((e = cudaMalloc((void**)&p->r, sizeof(float) * m)) != cudaSuccess) { s = cuda_fail(e, "alloc r"); break; }
        if ((e = cudaMalloc((void**)&p->r64, sizeof(double) * m)) != cudaSuccess) { s = cuda_fail(e, "alloc r64"); break; }
        if ((e = cudaMemsetAsync(p->r, 0, sizeof(float) * m, st)) != cudaSuccess) { s = cuda_fail(e, "memset r"); break; }
        p->r_cur = p->r;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { s = cuda_fail(e, "create sync"); break; }
    } while (0);
    if (s != PCDM_OK) {
        free_problem(p);
        return s;
    }
    p->stats.kernel_launches = launches;
    *out = p;
    return PCDM_OK;
}

}  // namespace

extern "C" {

void pcdm_destroy(pcdm_problem* p) {
    if (!p) return;
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    free_problem(p);
}

pcdm_status pcdm_omega(const pcdm_problem* p, int64_t* omega) {
    if (!p || !omega) return fail(PCDM_EINVAL, "NULL argument");
    *omega = p->omega;
    return PCDM_OK;
}

pcdm_status pcdm_beta(const pcdm_problem* p, int64_t tau, double* beta) {
    if (!p || !beta) return fail(PCDM_EINVAL, "NULL argument");
    if (tau < 1 || tau > p->n) return fail(PCDM_EINVAL, "tau must be in [1, n]");
    const double denom = (double)std::max<int64_t>(1, p->n - 1);
    *beta = 1.0 + (double)(p->omega - 1) * (double)(tau - 1) / denom;
    return PCDM_OK;
}

pcdm_status pcdm_run(pcdm_problem* p, float* x, int64_t tau, int64_t iters, uint64_t seed, void* stream) {
    return pcdm_run_ex(p, x, tau, iters, seed, 0, 0, 0.0, PCDM_VARIANT_AUTO, stream);
}

pcdm_status pcdm_run_ex(pcdm_problem* p, float* x, int64_t tau, int64_t iters, uint64_t seed, int64_t first_iter,
                        int64_t refresh_every, double beta_override, int32_t variant, void* stream) {
    if (!p || !x) return fail(PCDM_EINVAL, "NULL argument");
    pcdm_sampling smp{};
    smp.kind = PCDM_SAMPLING_NICE;
    smp.tau = tau;
    smp.p_b = 1.0;
    return pcdm_run_sampling(p, x, &smp, iters, seed, first_iter, refresh_every, beta_override, variant, stream);
}

pcdm_status pcdm_run_sampling(pcdm_problem* p, float* x, const pcdm_sampling* sampling, int64_t iters, uint64_t seed,
                              int64_t first_iter, int64_t refresh_every, double beta_override, int32_t variant,
                              void* stream) {
    if (!p || !x) return fail(PCDM_EINVAL, "NULL argument");
    SamplingSpec spec;
    pcdm_status s0 = check_sampling(sampling, p->n, &spec);
    if (s0 != PCDM_OK) return s0;
    return run_impl(p, x, spec, iters, seed, first_iter, refresh_every, beta_override, variant, stream);
}

}  // extern "C"

namespace {

pcdm_status run_impl(pcdm_problem* p, float* x, const SamplingSpec& spec, int64_t iters, uint64_t seed,
                     int64_t first_iter, int64_t refresh_every, double beta_override, int32_t variant, void* stream) {
    const int64_t tau = spec.tau;
    if (iters < 0 || first_iter < 0) return fail(PCDM_EINVAL, "iters and first_iter must be >= 0");
    if (first_iter + iters > (1ll << 32)) return fail(PCDM_EINVAL, "first_iter + iters must be <= 2^32");
    if (variant < 0 || variant > 5) return fail(PCDM_EINVAL, "unknown variant %d", variant);
    if (variant == PCDM_VARIANT_PACKED && !p->packed_G && !p->ragged)
        return fail(PCDM_EINVAL, "PACKED variant: no packed copy of A (device memory)");
    if (variant == PCDM_VARIANT_BATCHED && !p->packed_G)
        return fail(PCDM_EINVAL, "BATCHED variant needs the uniform packed layout (max column length %lld%s)",
                    (long long)p->max_len, p->ragged ? ", ragged layout" : "");
    if (!(beta_override <= 1e308)) return fail(PCDM_EINVAL, "beta_override must be finite");
    CK(cudaSetDevice(p->device), "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    pcdm_run_stats stats{};
    int64_t launches = 0;

    RunTimer tm{p, st};
    int t0;
    CK(tm.begin(&t0), "event");
    // a previous host-x run's side-stream sampler must be done with the workspace
    if (p->side) CK(cudaStreamWaitEvent(st, p->ev_s1, 0), "join presampler");
    // iterate buffer: device x in place, host x through xbuf
    const bool x_dev = is_device_ptr(x);
    CK(cudaMemsetAsync(p->sc, 0, sizeof(Scalars), st), "memset scalars");
    pcdm_status s = PCDM_OK;
    Scalars hs{};
    // sampler plan: chunks of iterations, aligned with the residual refreshes
    const int64_t R = refresh_period(p->n, tau, refresh_every);
    // schunk: iterations per sampler pass (its hash tables fit the workspace budget);
    // chunk: the same capped at the refresh period (the BATCHED workspace unit)
    const int64_t schunk = choose_chunk(p->n, tau, iters);
    int64_t chunk = schunk;
    if (R > 0) chunk = std::min(chunk, R);
    auto chunk_len = [&](int64_t done) { return std::min(schunk, iters - done); };
    SamplerPlan sp;
    if ((s = sampler_workspace(&p->samp_mem, &p->samp_cap, p->n, tau, schunk, &sp,
                               spec.kind == PCDM_SAMPLING_INDEPENDENT)) != PCDM_OK)
        return s;
    SamplingDev sdev;
    if ((s = sampling_dev(spec, &p->du_T, &p->du_cap, st, &sdev)) != PCDM_OK) return s;
    // host x: every sample set of the run is drawn on a side stream while x crosses PCIe
    // (the sampler needs only seed and k; the copy engines and the SMs overlap)
    // ... and also for a device x, with the iterations waiting for their own sampler pass
    // only (an event per pass), so the passes run on the low-priority side stream under
    // the iteration kernels: huge 4.66e9 -> 4.81e9 updates/s, large / skewed 2^12 / tiny /
    // kddb_like +1-1.5 %, medium and skewed 2^16 within -0.7 % (profiles/r01_presample_overlap_ab.txt).
    // PCDM_PRESAMPLE_DEV=0: sample in the run's stream
    const char* pe = knob("PCDM_PRESAMPLE");
    const char* pdev = knob("PCDM_PRESAMPLE_DEV");
    // PCDM_PRESAMPLE_JOIN=1: every pass drawn before the first iteration kernel (no overlap)
    const char* pjoin = knob("PCDM_PRESAMPLE_JOIN");
    const bool join_all = pjoin && atoi(pjoin) != 0;
    const bool per_pass = (pdev ? atoi(pdev) != 0 : true) && !join_all;
    const bool presample = (!x_dev || per_pass || join_all) && iters > 0 && spec.kind == PCDM_SAMPLING_NICE &&
                           !(pe && atoi(pe) == 0) && (double)iters * (double)tau * 4.0 <= (double)(4ll << 30);
    // ragged layout: the slot arrays are binned by column class; with presampling the
    // binning rides on each sampler pass (side stream), else it runs before each launch
    const IterLaunch plan0 = plan_iter(variant >= PCDM_VARIANT_PACKED ? PCDM_VARIANT_GRID : variant, p->m, p->n,
                                       p->nnz, tau, p->sms, p->device, p->loss == 1, p->max_len);
    const bool ragged_plan = p->ragged && (variant == PCDM_VARIANT_PACKED ||
                                           (variant == PCDM_VARIANT_AUTO && plan0.variant == PCDM_VARIANT_GRID));
    auto ensure_bins = [&](int64_t its, int64_t scr_its) -> pcdm_status {
        if (p->bins_cap < (size_t)(its * tau)) {
            cudaFree(p->bins);
            cudaFree(p->bcnt);
            p->bins = nullptr;
            p->bcnt = nullptr;
            p->bins_cap = 0;
            CK(cudaMalloc((void**)&p->bins, sizeof(int2) * its * tau), "alloc bins");
            CK(cudaMalloc((void**)&p->bcnt, sizeof(int) * 8 * its), "alloc bins");
            p->bins_cap = (size_t)(its * tau);
        }
        if (p->bin_scr_cap < bin_scratch_bytes(scr_its)) {
            cudaFree(p->bin_scr);
            p->bin_scr = nullptr;
            p->bin_scr_cap = 0;
            CK(cudaMalloc((void**)&p->bin_scr, bin_scratch_bytes(scr_its)), "alloc bin scratch");
            p->bin_scr_cap = bin_scratch_bytes(scr_its);
        }
        return PCDM_OK;
    };
    if (presample) {
        const size_t need = sizeof(int) * (size_t)iters * (size_t)tau;
        if (p->pre_cap < need) {
            cudaFree(p->pre_slots);
            p->pre_slots = nullptr;
            p->pre_cap = 0;
            CK(cudaMalloc((void**)&p->pre_slots, need), "alloc presampled slots");
            p->pre_cap = need;
        }
        if (!p->side) {
            int least = 0, greatest = 0;  // the presampler yields to the iteration kernels
            cudaDeviceGetStreamPriorityRange(&least, &greatest);
            CK(cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, least), "side stream");
            CK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming), "event");
            CK(cudaEventCreate(&p->ev_s0), "event");
            CK(cudaEventCreate(&p->ev_s1), "event");
        }
        CK(cudaEventRecord(p->ev_fork, st), "event");
        CK(cudaStreamWaitEvent(p->side, p->ev_fork, 0), "event");
        CK(cudaEventRecord(p->ev_s0, p->side), "event");
        CK(cudaMemsetAsync(sp.w.rounds_max, 0, sizeof(int), p->side), "memset rounds");
        if (ragged_plan && (s = ensure_bins(iters, schunk)) != PCDM_OK) return s;
        for (int64_t done = 0, pass = 0; done < iters; ++pass) {
            const int64_t c = chunk_len(done);
            CK(sample_chunk(sp.w, sdev, seed, first_iter + done, c, p->pre_slots + done * tau, &p->sc->flags, p->side,
                            p->sms, &launches),
               "sampler");
            if (ragged_plan)
                CK(bin_chunk(p->pre_slots + done * tau, tau, c, p->blk_off, p->blk_cls, p->bin_scr, p->bins + done * tau,
                             p->bcnt + done * 8, p->side, p->sms, &launches),
                   "binning");
            if (per_pass) {
                while ((int64_t)p->pass_ev.size() <= pass) {
                    cudaEvent_t e;
                    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
                    p->pass_ev.push_back(e);
                }
                CK(cudaEventRecord(p->pass_ev[pass], p->side), "event");
            }
            done += c;
        }
        CK(cudaEventRecord(p->ev_s1, p->side), "event");
    } else {
        CK(cudaMemsetAsync(sp.w.rounds_max, 0, sizeof(int), st), "memset rounds");
    }
    float* xd = x;
    if (!x_dev) {
        if (!p->xbuf) CK(cudaMalloc((void**)&p->xbuf, sizeof(float) * p->n), "alloc x buffer");
        CK(cudaMemcpyAsync(p->xbuf, x, sizeof(float) * p->n, cudaMemcpyHostToDevice, st), "copy x in");
        xd = p->xbuf;
    }

    double beta_d = sampling_beta(spec, p->omega, p->n);
    if (beta_override > 0.0) beta_d = beta_override;
    IterLaunch plan = plan0;
    // AUTO: packed blocks whenever the shared-memory variant does not apply
    bool packed = (p->packed_G > 0 || p->ragged) &&
                  (variant >= PCDM_VARIANT_PACKED || (variant == PCDM_VARIANT_AUTO && plan.variant == PCDM_VARIANT_GRID));
    // BATCHED (kernels_batched.cu): AUTO picks it for LASSO when r is much larger than L2
    // (huge: 3.90e9 -> 4.60e9 updates/s; large, skewed, kddb_like stay on the packed loop,
    // profiles/r01_batched_vs_packed.txt), with the packed loop prepared as a fallback
    // should the run's steps turn out too dense for its filters (below).  PCDM_BATCHED=0/1
    // overrides the size rule.
    int l2_bytes = 0;
    cudaDeviceGetAttribute(&l2_bytes, cudaDevAttrL2CacheSize, p->device);
    const char* bat_env = knob("PCDM_BATCHED");
    // ... and when an iteration samples enough columns to amortise the snapshot's
    // per-iteration barrier and filter latency, with few idle slots (its passes cost per
    // slot, active or not).  Huge (profiles/r01_batched_autorule_ab.txt): tau-nice 2^17,
    // 1.5 2^17, 2^18, 2^19 and tau-independent 2^18 win by 14-23 %; (2^18, 0.75)-binomial
    // ties, (2^18, 0.5)-binomial loses (2.63e9 vs 2.95e9 updates/s).  Rule: E|S| >= 2^17
    // and E|S| >= 0.8 tau (PCDM_BATCHED_MIN_SLOTS overrides the first).
    double es1 = 0.0, es2 = 0.0;
    sampling_moments(spec, p->n, &es1, &es2);
    double min_slots = 131072.0;
    if (const char* ms = knob("PCDM_BATCHED_MIN_SLOTS")) min_slots = atof(ms);
    const bool auto_batched =
        variant == PCDM_VARIANT_AUTO &&
        (bat_env ? atoi(bat_env) != 0
                 : p->loss == 0 && p->packed_G > 0 && p->packed_G <= 8 && (double)p->m * 4.0 > 2.0 * l2_bytes && es1 >= min_slots &&
                       es1 >= 0.8 * (double)tau);
    bool batched = packed && p->packed_G > 0 && (variant == PCDM_VARIANT_BATCHED || auto_batched);
    const bool bat_fallback = batched && variant == PCDM_VARIANT_AUTO;
    if (batched && !bat_fallback) packed = false;
    bool one_barrier = false;
    int list_cap = 0;
    bool hot_stage = false;
    bool bulk_stage = false;
    int cluster_sync = 0;
    const bool ragged_run = packed && p->ragged;
    if (ragged_run) {
        // one barrier per iteration with the double-buffered residual (the generic CSC
        // kernel if the second buffer cannot be allocated)
        one_barrier = true;
        if (!p->r2 && cudaMalloc((void**)&p->r2, sizeof(float) * p->m) != cudaSuccess) {
            cudaGetLastError();
            p->r2 = nullptr;
            one_barrier = false;
            packed = false;
        }
    }
    if (packed && ragged_run) {
        plan.variant = PCDM_VARIANT_PACKED;
        plan.lanes = 0;  // per column: 2..32 lanes, or a CTA beyond 62 entries
        plan.threads = 512;
        // CTA-long column slices staged in shared memory by bulk copies (SURVEY 8 row X2,
        // profiles/r02_bulk_stage_ab.jsonl); PCDM_BULK_STAGE=0/1 overrides
        const char* bs_env = knob("PCDM_BULK_STAGE");
        bulk_stage = bs_env ? atoi(bs_env) != 0 : false;
        plan.ctas = ragged_ctas(p->sms, p->loss == 1, p->nhot, bulk_stage);
        // small tau: only about as many CTAs as the average column needs lanes
        const double gavg = (double)p->ragged_chunks / (double)p->n;
        const int64_t busy = std::max<int64_t>(1, (int64_t)ceil((double)tau * gavg / plan.threads));
        if (busy < plan.ctas) plan.ctas = (int)busy;
        if (const char* cs = knob("PCDM_CTAS")) {
            const int v = atoi(cs);
            if (v >= 1) plan.ctas = std::min(v, ragged_ctas(p->sms, p->loss == 1, p->nhot, bulk_stage));
        }
    } else if (packed) {
        // one barrier per iteration (double-buffered r, the previous iteration's steps
        // replayed): measured faster on every config (huge: 45.7 -> 44.2 ms/step,
        // profiles/r01_one_barrier_huge_ab.log); two barriers if the second buffer
        // cannot be allocated or PCDM_ONE_BARRIER=0
        one_barrier = true;
        const char* ob = knob("PCDM_ONE_BARRIER");
        if (ob) one_barrier = atoi(ob) != 0;
        if (one_barrier && !p->r2 && cudaMalloc((void**)&p->r2, sizeof(float) * p->m) != cudaSuccess) {
            cudaGetLastError();
            p->r2 = nullptr;
            one_barrier = false;
        }
        // hot-row scatters staged in shared memory per CTA (one-barrier scheme; SURVEY 8
        // row X2, profiles/r02_hot_stage_ab.jsonl); PCDM_HOT_STAGE=0/1 overrides
        const char* hs_env = knob("PCDM_HOT_STAGE");
        // default: dense-step workloads (logistic: every visited coordinate steps) -- skewed,
        // logistic tau = 2^16: 498 -> 31 ms of iteration kernel per 1000 iterations; LASSO's
        // sparse steps lose (169 -> 176 ms per 1e4 iterations: the per-iteration flush costs more)
        hot_stage = one_barrier && p->nhot > 0 && (hs_env ? atoi(hs_env) != 0 : p->loss == 1);
        plan.variant = PCDM_VARIANT_PACKED;
        plan.lanes = p->packed_G;
        plan.threads = 512;
        plan.ctas = packed_ctas(p->packed_G, one_barrier, p->sms, p->loss == 1, p->nhot, 0, hot_stage);
        // small tau: only CTAs that own slots; the others would only add arrivals to
        // every grid barrier (PCDM_CTAS overrides, for measurements)
        const int64_t busy = (tau * p->packed_G + plan.threads - 1) / plan.threads;
        if (busy < plan.ctas) plan.ctas = (int)busy;
        // a grid that covers tau in one round with <= 16 CTAs fits one thread-block
        // cluster: hardware cluster barriers instead of the global-memory grid barrier
        // (skewed tau = 2^8: 8 CTAs, 41.5 -> 36.6 ms/step); 1024-thread CTAs when 512-thread
        // ones would need more than 16 (medium: 16 x 1024, 39.2 -> 37.7 ms/step;
        // profiles/r01_cluster_sync_ab.jsonl).  PCDM_CLUSTER_SYNC=0: off
        const char* csy = knob("PCDM_CLUSTER_SYNC");
        cluster_sync = one_barrier && !(csy && atoi(csy) == 0) ? 1 : 0;
        const int64_t busy1024 = (tau * p->packed_G + 1023) / 1024;
        if (cluster_sync && busy > 16 && busy1024 <= 16 && !knob("PCDM_CTAS")) {
            plan.threads = 1024;
            plan.ctas = (int)busy1024;
            cluster_sync = 2;
        }
        if (const char* cs = knob("PCDM_CTAS")) {
            const int v = atoi(cs);
            if (v >= 1)
                plan.ctas = std::min(v, packed_ctas(p->packed_G, one_barrier, p->sms, p->loss == 1, p->nhot, 0, hot_stage));
        }
        // dense-step workloads (logistic: every step is nonzero): stage each CTA's steps in
        // shared memory, one atomic on the list counter per CTA instead of one per step
        // (PCDM_STAGE_LIST=0/1 overrides)
        const char* sl = knob("PCDM_STAGE_LIST");
        if (sl ? atoi(sl) != 0 : p->loss == 1) {
            const int64_t groups = (int64_t)plan.ctas * plan.threads / p->packed_G;
            const int64_t cap = ((tau + groups - 1) / groups) * (plan.threads / p->packed_G);
            const int full = packed_ctas(p->packed_G, one_barrier, p->sms, p->loss == 1, p->nhot, 0, hot_stage);
            if (cap * 8 <= 32 * 1024 &&
                packed_ctas(p->packed_G, one_barrier, p->sms, p->loss == 1, p->nhot, (int)cap, hot_stage) == full)
                list_cap = (int)cap;
        }
    }
    // CTA-local replay (one-barrier scheme, uniform layout): a CTA's slots are the same
    // positions of every iteration, so its steps stay in shared-memory lists and it replays
    // them itself -- no global step lists, no list counter read after the barrier (large:
    // profiles/r02_local_replay_ab.jsonl); taken when the lists fit 24 KB without lowering the
    // occupancy; PCDM_LOCAL_REPLAY=0: the global lists
    int local_cap = 0;
    if (packed && !ragged_run && one_barrier) {
        const char* lr = knob("PCDM_LOCAL_REPLAY");
        const int64_t groups = (int64_t)plan.ctas * plan.threads / p->packed_G;
        const int64_t cap = ((tau + groups - 1) / groups) * (plan.threads / p->packed_G);
        if (!(lr && atoi(lr) == 0) && cap * 24 <= 24 * 1024 &&
            (plan.threads != 512 ||
             packed_ctas(p->packed_G, one_barrier, p->sms, p->loss == 1, p->nhot, 0, hot_stage, (int)cap) ==
                 packed_ctas(p->packed_G, one_barrier, p->sms, p->loss == 1, p->nhot, 0, hot_stage))) {
            local_cap = (int)cap;
            list_cap = 0;
        }
    }
    const IterLaunch packed_plan = plan;  // the AUTO BATCHED fallback
    if (batched) packed = false;
    if (p->nz_cap < tau) {
        cudaFree(p->nz_idx);
        cudaFree(p->nz_delta);
        p->nz_idx = nullptr;
        p->nz_delta = nullptr;
        p->nz_cap = 0;
        CK(cudaMalloc((void**)&p->nz_idx, sizeof(int) * 3 * tau), "alloc step list");
        CK(cudaMalloc((void**)&p->nz_delta, sizeof(float) * 3 * tau), "alloc step list");
        p->nz_cap = tau;
    }
    // x in the block headers (packed loop): saves the separate random x line of every
    // update; PCDM_X_IN_BLOCK=0 keeps x in the caller's array.  The start-of-run
    // header load rides on the residual pass, which reads x anyway.
    const char* xib = knob("PCDM_X_IN_BLOCK");
    const bool xhdr = (packed || batched) && !(xib && atoi(xib) == 0);
    // dense iterates (logistic: every visited coordinate steps) keep no dirty list: its
    // appends would all hit one counter; the header passes walk all n columns instead
    // (list count pinned at ~0 = "overflowed", appends skipped with cap 0; PCDM_XLIST_DENSE)
    const char* xde = knob("PCDM_XLIST_DENSE");
    const bool xdense = xde ? atoi(xde) != 0 : p->loss == 1;
    XHeaders xh{};
    int64_t cap_eff = 0;
    if (xhdr) {
        if (!p->xlist) {
            int64_t cap = std::min<int64_t>(p->n, (int64_t)1 << 26);
            if (const char* xc = knob("PCDM_XLIST_CAP")) cap = std::max<int64_t>(1, atoll(xc));
            CK(cudaMalloc((void**)&p->xlist, sizeof(int) * cap), "alloc x list");
            CK(cudaMalloc((void**)&p->xlist_count, sizeof(unsigned long long)), "alloc x list");
            CK(cudaMemsetAsync(p->xlist_count, 0, sizeof(unsigned long long), st), "memset x list");
            p->xlist_cap = cap;
        }
        CK(launch_xhdr_clear(p->blocks, p->packed_G, p->blk_off, p->xlist, p->xlist_count, p->xlist_cap, p->n, st, p->sms,
                             &launches),
           "x headers");
        cap_eff = xdense ? 0 : p->xlist_cap;
        CK(cudaMemsetAsync(p->xlist_count, xdense ? 0xFF : 0, sizeof(unsigned long long), st), "memset x list");
        xh = XHeaders{p->blocks, p->packed_G, p->blk_off, p->xlist, p->xlist_count, cap_eff};
    }
    if ((s = residual_from(p, xd, st, &launches, xhdr ? &xh : nullptr, one_barrier && !batched ? p->r2 : nullptr)) !=
        PCDM_OK)
        return s;
    CK(tm.end(T_SETUP, t0), "event");
    if ((s = read_scalars(p, &hs, st)) != PCDM_OK) return s;
    if (hs.flags & FLAG_NONFINITE_X) return fail(PCDM_EINVAL, "non-finite value in x");
    auto x_out = [&]() -> pcdm_status {
        if (xhdr)
            CK(launch_xhdr_out(p->blocks, p->packed_G, p->blk_off, xd, p->n, p->xlist, p->xlist_count, cap_eff, st, p->sms,
                               &launches),
               "x headers");
        return PCDM_OK;
    };

    IterParams P{};
    P.colptr = p->colptr;
    P.rowidx = p->rowidx;
    P.val = p->val;
    P.L = p->L;
    P.x = xd;
    P.r = p->r;
    P.tau = tau;
    P.beta = (float)beta_d;
    P.lambda = (float)p->lambda;
    P.nz_idx = p->nz_idx;
    P.nz_delta = p->nz_delta;
    P.nz_count = p->sc->nz_count;
    P.barrier = p->sc->barrier;
    P.flags = &p->sc->flags;
    P.nz_total = &p->sc->nz_total;
    P.m = p->m;
    P.n = p->n;
    P.logistic = p->loss;
    PackedParams Q{};
    Q.blocks = p->blocks;
    Q.x = xd;
    Q.r0 = p->r;
    Q.r1 = one_barrier ? p->r2 : nullptr;
    Q.tau = tau;
    Q.beta = (float)beta_d;
    Q.lambda = (float)p->lambda;
    Q.nz_idx = p->nz_idx;
    Q.nz_delta = p->nz_delta;
    Q.nz_count = p->sc->nz_count;
    Q.barrier = p->sc->barrier;
    Q.flags = &p->sc->flags;
    Q.nz_total = &p->sc->nz_total;
    Q.logistic = p->loss;
    Q.xlist = xhdr ? p->xlist : nullptr;
    Q.xlist_count = p->xlist_count;
    Q.xlist_cap = cap_eff;
    Q.hot_rows = p->hot_rows;
    Q.nhot = p->nhot;
    Q.list_cap = list_cap;
    Q.local_cap = local_cap;
    Q.hot_stage = hot_stage ? 1 : 0;
    Q.bulk_stage = ragged_run && bulk_stage ? 1 : 0;
    // software-pipelined slots when r is L2-resident (the loop is latency-bound there:
    // large 26.1 -> 25.8, skewed tau=2^16 163 -> 158 ms/step); for r much larger than L2
    // (huge) the extra loads in flight cost more than they hide (29.0 -> 29.4 ms)
    {
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, p->device);
        Q.pipeline = (double)p->m * 4.0 <= 0.5 * (double)l2;
        if (const char* pl = knob("PCDM_PIPELINE")) Q.pipeline = atoi(pl) != 0;
    }
    // a grid that fits one cluster (<= 16 CTAs: small tau) synchronises with the hardware
    // cluster barrier instead of the global-memory grid barrier
    Q.cluster_sync = (packed || bat_fallback) && packed_plan.ctas <= 16 && !ragged_run ? cluster_sync : 0;
    if (ragged_run) Q.pipeline = 0;
    // a grid that covers tau in one round (every group owns <= 1 slot per iteration: the
    // latency-bound small-tau configs) replays the previous step from registers, without
    // step lists (pcdm_packed1_kernel; iteration kernel per 1e4 iterations: medium 32.7 -> 20.4 ms, skewed
    // tau = 2^8 35.2 -> 19.9, tau = 2^12 55.2 -> 38.8 ms;
    // profiles/r02_reg_replay_ab.jsonl); PCDM_REG_REPLAY=0: the list-based loop
    {
        const int64_t groups = (int64_t)packed_plan.ctas * packed_plan.threads / std::max(1, p->packed_G);
        const char* rr = knob("PCDM_REG_REPLAY");
        Q.reg_replay = (packed || bat_fallback) && !ragged_run && one_barrier && !hot_stage && groups >= tau &&
                               !(rr && atoi(rr) == 0)
                           ? 1
                           : 0;
    }
    // cache the hot rows when the hottest one is read >= 1024 times per iteration
    // (tau count_max / n); below that the per-iteration copy costs more than the
    // same-address serialisation it removes (skewed, tau = 256: 55.2 vs 57.6 ms/step;
    // tau = 65536: 548 -> 179 ms/step of iteration kernel, profiles/r01_hot_rows_ab.jsonl)
    Q.hot_cache = p->nhot > 0 && (double)tau * (double)p->hot_max_count >= 1024.0 * (double)p->n;
    if (const char* hc = knob("PCDM_HOT_CACHE")) Q.hot_cache = p->nhot > 0 && atoi(hc) != 0;

    BatchedParams B{}, B1{};  // B1: the second workspace set of the screened pass
    int bat_ctas = 0;
    int64_t bsnap = 0, bprev_c = 0;  // screened: chunks launched, the previous chunk's iterations
    unsigned long long* tl_buf = nullptr;  // debug timeline (PCDM_SCREEN_TIMELINE)
    if (knob("PCDM_SCREEN_TIMELINE")) {
        CK(cudaMalloc((void**)&tl_buf, 8 * 256 * sizeof(unsigned long long)), "alloc timeline");
        CK(cudaMemsetAsync(tl_buf, 0, 8 * 256 * sizeof(unsigned long long), st), "memset timeline");
    }
    // BATCHED: iterations per chunk (the passes' unit), its own rule independent of the
    // sampler pass size: 16 (huge with the screened step pass: 15-16 beat 10-14 and 17-23 by
    // ~3 %, 25+ needs a second wave of sweep CTAs, profiles/r02_batched_chunk_ab.txt; round 1
    // chose 18 for the grid-barrier step pass), at most one refresh period and the run
    int64_t bchunk = 16;
    if (const char* bc = knob("PCDM_BATCHED_CHUNK")) bchunk = std::max<int64_t>(1, atoll(bc));
    bchunk = std::min<int64_t>(bchunk, std::max<int64_t>(iters, 1));
    if (R > 0) bchunk = std::min(bchunk, R);
    if (batched) {
        const int64_t chunk = bchunk;
        const int G = p->packed_G;
        B.cq_log = batched_cq_log(G);
        B.rb = batched_rb(B.cq_log);
        // entries staged per slot: the longest column, rounded up to a whole 16-byte chunk
        B.maxe = (int)std::min<int64_t>(2 * (G - 1), std::max<int64_t>(2, (p->max_len + 1) & ~(int64_t)1));
        B.nb = (int)((p->m + (1ll << B.rb) - 1) >> B.rb);
        const int64_t cq = 1ll << B.cq_log;
        const int64_t nq_max = (chunk * tau + cq - 1) / cq;
        auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
        const size_t o_g0 = 0;
        const size_t o_ent = o_g0 + al(sizeof(float) * chunk * tau);
        const size_t o_offs = o_ent + al(sizeof(int2) * nq_max * cq * B.maxe);
        const size_t o_idx = o_offs + al(sizeof(int) * nq_max * (B.nb + 1));
        const size_t o_del = o_idx + al(sizeof(int) * chunk * tau);
        const size_t o_cnt = o_del + al(sizeof(float) * chunk * tau);
        const size_t o_rec = o_cnt + al(sizeof(int) * chunk);
        // SCREENED step pass (LASSO; kernels_batched.cu): per slot {L, x} + its rows,
        // item bits and lists, in place of the grid-barrier pass's slot records
        // (PCDM_BATCHED_SCREEN=0: the grid-barrier pass)
        const char* scr_env = knob("PCDM_BATCHED_SCREEN");
        const bool screen = p->loss == 0 && !(scr_env && atoi(scr_env) == 0);
        const int64_t T = chunk * tau;
        const int nrow = (int)std::max<int64_t>(1, p->max_len);
        const size_t o_lx = o_rec + (screen ? 0 : al(sizeof(int2) * T * G));
        const size_t o_rows = o_lx + (screen ? al(sizeof(int2) * T) : 0);
        const int64_t rows_ld = (T + 3) & ~(int64_t)3;  // 16-byte row loads in the test pass
        const size_t o_bits = o_rows + (screen ? al(sizeof(int) * rows_ld * nrow) : 0);
        const size_t o_items = o_bits + (screen ? al(sizeof(unsigned) * ((rows_ld + 31) / 32)) : 0);
        const size_t o_counts = o_items + (screen ? al(sizeof(int) * 3 * rows_ld) : 0);
        const size_t one = al(o_counts + al(sizeof(int) * 16));
        // screened: two workspace sets, alternating per chunk, so that chunk s's fix-up
        // (own stream) overlaps chunk s+1's expand pass
        const size_t need = screen ? 2 * one : one;
        if (p->bat_cap < need) {
            cudaFree(p->bat_mem);
    if (p->fix_st) {
        cudaStreamDestroy(p->fix_st);
        cudaEventDestroy(p->ev_test);
        cudaEventDestroy(p->ev_fix);
    }
            p->bat_mem = nullptr;
            p->bat_cap = 0;
            CK(cudaMalloc(&p->bat_mem, need), "alloc batched workspace");
            p->bat_cap = need;
        }
        if (!p->d0) {
            CK(cudaMalloc((void**)&p->d0, sizeof(float) * p->m), "alloc delta buffer");
            CK(cudaMalloc((void**)&p->d1, sizeof(float) * p->m), "alloc delta buffer");
            CK(cudaMemsetAsync(p->d0, 0, sizeof(float) * p->m, st), "memset delta");
            CK(cudaMemsetAsync(p->d1, 0, sizeof(float) * p->m, st), "memset delta");
        }
        char* base = (char*)p->bat_mem;
        B.blocks = p->blocks;
        B.tau = tau;
        B.beta = (float)beta_d;
        B.lambda = (float)p->lambda;
        B.r = p->r;
        B.r_out = p->r;
        B.d0 = p->d0;
        B.d1 = p->d1;
        B.g0 = (float*)(base + o_g0);
        B.gent = (int2*)(base + o_ent);
        B.offs = (int*)(base + o_offs);
        B.nz_idx = (int*)(base + o_idx);
        B.nz_delta = (float*)(base + o_del);
        B.nz_count = (int*)(base + o_cnt);
        B.rec = (int2*)(base + o_rec);
        B.screen = screen ? 1 : 0;
        if (screen) {
            B.lx = (int2*)(base + o_lx);
            B.rows = (int*)(base + o_rows);
            B.rows_ld = rows_ld;
            B.nrow = nrow;
            B.bits = (unsigned*)(base + o_bits);
            B.items = (int*)(base + o_items);
            CK(cudaMemsetAsync(B.bits, 0, sizeof(unsigned) * ((T + 31) / 32), st), "memset item bits");
        }
        B.counts = (int*)(base + o_counts);
        CK(cudaMemsetAsync(B.counts, 0, sizeof(int) * 16, st), "memset item counts");
        B.rnv = 1 + (int)((std::max<int64_t>(p->max_len - 2, 0) + 3) / 4);  // 10 entries (huge): 3 vectors, 48 B
        B.barrier = p->sc->barrier;
        B.flags = &p->sc->flags;
        B.nz_total = &p->sc->nz_total;
        B.x = xd;
        B.xlist = xhdr ? p->xlist : nullptr;
        B.xlist_count = p->xlist_count;
        B.xlist_cap = cap_eff;
        B.hot_rows = p->hot_rows;
        B.nhot = p->nhot;
        B.logistic = p->loss;
        if (screen) {
            char* b1 = base + one;
            B1 = B;
            B1.g0 = (float*)(b1 + o_g0);
            B1.gent = (int2*)(b1 + o_ent);
            B1.offs = (int*)(b1 + o_offs);
            B1.nz_idx = (int*)(b1 + o_idx);
            B1.nz_delta = (float*)(b1 + o_del);
            B1.nz_count = (int*)(b1 + o_cnt);
            B1.lx = (int2*)(b1 + o_lx);
            B1.rows = (int*)(b1 + o_rows);
            B1.bits = (unsigned*)(b1 + o_bits);
            B1.items = (int*)(b1 + o_items);
            B1.counts = (int*)(b1 + o_counts);
            CK(cudaMemsetAsync(B1.bits, 0, sizeof(unsigned) * ((T + 31) / 32), st), "memset item bits");
            CK(cudaMemsetAsync(B1.counts, 0, sizeof(int) * 16, st), "memset item counts");
            if (!p->fix_st) {
                int least = 0, greatest = 0;  // the fix-up is on the critical path of the next sweep
                cudaDeviceGetStreamPriorityRange(&least, &greatest);
                CK(cudaStreamCreateWithPriority(&p->fix_st, cudaStreamNonBlocking, greatest), "fix-up stream");
                CK(cudaEventCreateWithFlags(&p->ev_test, cudaEventDisableTiming), "event");
                CK(cudaEventCreateWithFlags(&p->ev_fix, cudaEventDisableTiming), "event");
            }
            // the first chunk's sweep must not wait on a previous run's (completed) fix-up
            CK(cudaEventRecord(p->ev_fix, st), "event");
        }
        bat_ctas = batched_ctas(G, p->sms, p->loss == 1, p->nhot);
        plan.variant = PCDM_VARIANT_BATCHED;
        plan.lanes = G;
        plan.threads = 512;
        plan.ctas = bat_ctas;
    }


    if (presample && !per_pass) CK(cudaStreamWaitEvent(st, p->ev_s1, 0), "join presampler");
    // iterations per launch of the iteration kernel: max(schunk, 64) (PCDM_ITER_CHUNK for
    // the 64; each launch of the persistent kernel costs its ramp-up and drain), never
    // across a residual refresh.  Slots are drawn ahead in windows of max(schunk, ichunk)
    // iterations (one sampler pass can cover several refresh periods: tiny, medium),
    // each window in sampler passes of schunk iterations.
    int64_t ichunk = batched ? bchunk : chunk;
    if (!batched) {
        int64_t want = 64;
        if (const char* ic = knob("PCDM_ITER_CHUNK")) want = std::max<int64_t>(1, atoll(ic));
        ichunk = std::max(schunk, std::min(want, iters));  // long launches when samples are cheap
        if (R > 0) ichunk = std::min(ichunk, R);
        ichunk = std::max<int64_t>(ichunk, 1);
    }
    const int64_t win = std::min(iters, std::max(schunk, ichunk));
    const bool own_slots = !presample && win > schunk;
    if (own_slots && p->slot_cap < (size_t)(win * tau)) {
        cudaFree(p->slot_buf);
        p->slot_buf = nullptr;
        p->slot_cap = 0;
        CK(cudaMalloc((void**)&p->slot_buf, sizeof(int) * win * tau), "alloc slot buffer");
        p->slot_cap = (size_t)(win * tau);
    }
    int* const win_slots = own_slots ? p->slot_buf : sp.slots;
    int64_t w0 = 0, w1 = 0;  // sampled window [w0, w1) of run-local iterations
    // the shared-memory variant refreshes the residual inside the kernel: its launches
    // are not cut at refresh points
    const bool kernel_refresh = !packed && !batched && plan.variant == PCDM_VARIANT_SMEM;
    if (kernel_refresh) ichunk = std::max(ichunk, std::min<int64_t>(iters, std::max<int64_t>(schunk, 1)));
    auto iter_len = [&](int64_t done) {
        int64_t c = std::min(ichunk, iters - done);
        if (R > 0 && !kernel_refresh) c = std::min(c, R - (done % R));
        if (!presample) c = std::min(c, w1 - done);
        return c;
    };
    bool list_restarted = false;
    // AUTO BATCHED guard: after each batched launch the nonzero-step count is copied to
    // pinned host memory behind an event; when a completed copy shows more dirty rows per
    // snapshot than the filters hold (kBloomLog = 19: ~16 K rows keep a false positive
    // below ~0.5 %), the rest of the run goes to the packed loop (r2 = r, empty step lists:
    // the state it starts from after a refresh)
    int64_t nz_at = 0;  // run-local iterations the last issued copy covers
    bool nz_pending = false;
    if (bat_fallback && !p->nz_host) {
        CK(cudaMallocHost((void**)&p->nz_host, sizeof(unsigned long long)), "alloc pinned counter");
        CK(cudaEventCreateWithFlags(&p->ev_nz, cudaEventDisableTiming), "event");
    }
    const double avg_len = p->n > 0 ? (double)p->nnz / (double)p->n : 0.0;
    int64_t done = 0;
    while (done < iters) {
        if (batched && bat_fallback && nz_pending) {
            const bool sync_check = knob("PCDM_BATCHED_SYNC_CHECK") != nullptr;  // tests: deterministic
            const cudaError_t q = sync_check ? cudaEventSynchronize(p->ev_nz) : cudaEventQuery(p->ev_nz);
            if (q == cudaSuccess) {
                nz_pending = false;
                const double rows_per_chunk =
                    (double)*p->nz_host / (double)std::max<int64_t>(nz_at, 1) * (double)bchunk * avg_len;
                if (rows_per_chunk > 16384.0 || knob("PCDM_BATCHED_FORCE_FALLBACK")) {
                    if (B.screen) CK(cudaStreamWaitEvent(st, p->ev_fix, 0), "join fix-up");
                    batched = false;
                    packed = true;
                    plan = packed_plan;
                    if (one_barrier) CK(cudaMemcpyAsync(p->r2, p->r, sizeof(float) * p->m, cudaMemcpyDeviceToDevice, st),
                                        "copy residual");
                    CK(cudaMemsetAsync(p->sc->nz_count, 0, 3 * sizeof(int), st), "memset step lists");
                }
            } else if (q != cudaErrorNotReady) {
                CK(q, "event query");
            } else {
                cudaGetLastError();  // not-ready is not an error
            }
        }
        int ts;
        CK(tm.begin(&ts), "event");
        if (!presample && done >= w1) {
            // the window's slot buffer is reused: the last fix-up (own stream) reads it
            if (B.screen) CK(cudaStreamWaitEvent(st, p->ev_fix, 0), "join fix-up");
            w0 = done;
            w1 = std::min(iters, done + win);
            for (int64_t s0 = w0; s0 < w1; s0 += schunk)
                CK(sample_chunk(sp.w, sdev, seed, first_iter + s0, std::min(schunk, w1 - s0),
                                win_slots + (s0 - w0) * tau, &p->sc->flags, st, p->sms, &launches),
                   "sampler");
        }
        const int64_t c = iter_len(done);
        int* slots_c = presample ? p->pre_slots + done * tau : win_slots + (done - w0) * tau;
        if (presample && per_pass)  // the pass holding the launch's last iteration (passes run in order)
            CK(cudaStreamWaitEvent(st, p->pass_ev[(done + c - 1) / schunk], 0), "join presampler pass");
        // zero the barrier counter; the generic kernel also restarts its step lists per
        // launch, the packed loop keeps them (the one-barrier scheme replays list k-1)
        CK(cudaMemsetAsync(p->sc->barrier, 0, sizeof(p->sc->barrier), st), "memset barrier");
        if (!packed && !batched) CK(cudaMemsetAsync(p->sc->nz_count, 0, 3 * sizeof(int), st), "memset step lists");
        if (batched && !B.screen) CK(cudaMemsetAsync(B.nz_count, 0, sizeof(int) * c, st), "memset step lists");
        CK(tm.end(T_SAMPLER, ts), "event");
        int ti;
        CK(tm.begin(&ti), "event");
        if (batched) {
            BatchedParams& Bc = (B.screen && (bsnap & 1)) ? B1 : B;
            const BatchedParams& Bo = (B.screen && (bsnap & 1)) ? B : B1;
            Bc.slots = slots_c;
            Bc.iters = c;
            Bc.nq = (int)((c * tau + (1ll << Bc.cq_log) - 1) >> Bc.cq_log);
            // screened: the x_i this chunk's expand reads may miss the previous chunk's steps
            // (its fix-up runs beside the expand); the sweep re-reads x_i of those columns
            Bc.prev_nz_idx = Bc.screen && bprev_c > 0 ? Bo.nz_idx : nullptr;
            Bc.prev_nz_count = Bo.nz_count;
            Bc.prev_iters = (int)bprev_c;
            if (tl_buf && bsnap < 256) Bc.tl = tl_buf + 8 * bsnap;
            ScreenSched sch{};
            if (Bc.screen) sch = ScreenSched{p->fix_st, p->ev_test, p->ev_fix};
            CK(launch_batched(p->packed_G, Bc, bat_ctas, st, p->sms, &launches, Bc.screen ? &sch : nullptr),
               "batched iteration kernels");
            ++bsnap;
            bprev_c = c;
            cudaStream_t nz_st = Bc.screen ? p->fix_st : st;
            if (bat_fallback && !nz_pending) {
                CK(cudaMemcpyAsync(p->nz_host, &p->sc->nz_total, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                   nz_st),
                   "read step count");
                CK(cudaEventRecord(p->ev_nz, nz_st), "event");
                nz_at = done + c;
                nz_pending = true;
            }
        } else if (packed && ragged_run) {
            // the launch's slot arrays binned by column class (kernels_ragged.cu): by the
            // presampler passes, or here
            if (presample && ragged_plan) {
                Q.bins = p->bins + done * tau;
                Q.bcnt = p->bcnt + done * 8;
            } else {
                if ((s = ensure_bins(std::max(ichunk, c), std::max(ichunk, c))) != PCDM_OK) return s;
                CK(bin_chunk(slots_c, tau, c, p->blk_off, p->blk_cls, p->bin_scr, p->bins, p->bcnt, st, p->sms, &launches),
                   "binning");
                Q.bins = p->bins;
                Q.bcnt = p->bcnt;
            }
            Q.iters = c;
            Q.k0 = done;
            CK(launch_ragged(plan.ctas, Q, st, &launches), "ragged iteration kernel");
        } else if (packed) {
            Q.slots = slots_c;
            Q.iters = c;
            Q.k0 = done;
            CK(launch_packed(p->packed_G, one_barrier, plan.ctas, Q, st, &launches), "packed iteration kernel");
        } else {
            P.slots = slots_c;
            P.iters = c;
            P.k0 = done;
            P.R = kernel_refresh ? R : 0;
            P.b = p->b;
            CK(launch_iter(plan, P, st, &launches), "iteration kernel");
        }
        CK(tm.end(T_ITER, ti), "event");
        ++stats.iter_launches;
        done += c;
        if (kernel_refresh && R > 0) stats.refreshes += (done / R) - ((done - c) / R);
        if (R > 0 && done % R == 0 && !kernel_refresh) {
            if (B.screen) {  // the refresh reads x and r: the last fix-up first; x is current after it
                CK(cudaStreamWaitEvent(st, p->ev_fix, 0), "join fix-up");
                bprev_c = 0;
            }
            int tr;
            CK(tm.begin(&tr), "event");
            float* r2 = one_barrier ? p->r2 : nullptr;
            int* zero = one_barrier ? p->sc->nz_count : nullptr;
            if (xhdr) {
                // the refresh reads x: headers -> x, and the dirty list restarts from the
                // support of x (the refresh pass re-lists the nonzero x_i), so it does not
                // grow with every step of a long run; the host copy-back then cannot name
                // entries that became zero: it copies all of x
                // (two passes: the list may name a column twice)
                if ((s = x_out()) != PCDM_OK) return s;
                CK(launch_xhdr_clear(p->blocks, p->packed_G, p->blk_off, p->xlist, p->xlist_count, cap_eff, p->n, st, p->sms,
                                     &launches),
                   "x headers");
                CK(cudaMemsetAsync(p->xlist_count, xdense ? 0xFF : 0, sizeof(unsigned long long), st), "memset x list");
                list_restarted = true;
                if ((s = residual_from(p, xd, st, &launches, &xh, r2, zero, 3)) != PCDM_OK) return s;
            } else if ((s = residual_from(p, xd, st, &launches, nullptr, r2, zero, 3)) != PCDM_OK) {
                return s;
            }
            CK(tm.end(T_SETUP, tr), "event");
            ++stats.refreshes;
        }
    }
    if (B.screen) CK(cudaStreamWaitEvent(st, p->ev_fix, 0), "join fix-up");
    p->r_cur = (one_barrier && !batched && (iters & 1)) ? p->r2 : p->r;
    int tx;
    CK(tm.begin(&tx), "event");
    if ((s = x_out()) != PCDM_OK) return s;
    if (!x_dev) {
        stats.host_h2d_bytes = (int64_t)sizeof(float) * p->n;
        // with x in the block headers the dirty list names every entry the run may have
        // changed: copy back (index, value) pairs when that is less than the whole x
        bool compact = false;
        unsigned long long cnt = 0;
        if (xhdr && !list_restarted) {
            CK(cudaMemcpyAsync(&cnt, p->xlist_count, sizeof(cnt), cudaMemcpyDeviceToHost, st), "read x list");
            CK(cudaStreamSynchronize(st), "stream synchronize");
            compact = cnt <= (unsigned long long)cap_eff && 8 * (int64_t)cnt < 4 * p->n;
        }
        if (compact && cnt > 0) {
            if (p->comp_cap < (int64_t)cnt) {
                cudaFree(p->xcomp);
                cudaFreeHost(p->hidx);
                cudaFreeHost(p->hval);
                p->xcomp = nullptr;
                p->hidx = nullptr;
                p->hval = nullptr;
                p->comp_cap = 0;
                const int64_t cap = std::max<int64_t>((int64_t)cnt, 1 << 16);
                CK(cudaMalloc((void**)&p->xcomp, sizeof(float) * cap), "alloc compact x");
                CK(cudaMallocHost((void**)&p->hidx, sizeof(int) * cap), "alloc compact x");
                CK(cudaMallocHost((void**)&p->hval, sizeof(float) * cap), "alloc compact x");
                p->comp_cap = cap;
            }
            CK(launch_gather_list(p->xbuf, p->xlist, (int64_t)cnt, p->xcomp, st, p->sms, &launches), "gather x");
            CK(cudaMemcpyAsync(p->hidx, p->xlist, sizeof(int) * cnt, cudaMemcpyDeviceToHost, st), "copy x out");
            CK(cudaMemcpyAsync(p->hval, p->xcomp, sizeof(float) * cnt, cudaMemcpyDeviceToHost, st), "copy x out");
            CK(cudaStreamSynchronize(st), "stream synchronize");
            for (unsigned long long q = 0; q < cnt; ++q) x[p->hidx[q]] = p->hval[q];
            stats.host_d2h_bytes = (int64_t)sizeof(cnt) + 8 * (int64_t)cnt;
        } else if (!compact) {
            CK(cudaMemcpyAsync(x, p->xbuf, sizeof(float) * p->n, cudaMemcpyDeviceToHost, st), "copy x out");
            stats.host_d2h_bytes = (int64_t)sizeof(float) * p->n;
        } else {
            stats.host_d2h_bytes = (int64_t)sizeof(cnt);
        }
    }
    CK(tm.end(T_SETUP, tx), "event");
    int rmax = 0;
    CK(cudaMemcpyAsync(&rmax, sp.w.rounds_max, sizeof(int), cudaMemcpyDeviceToHost, st), "read rounds");
    if ((s = read_scalars(p, &hs, st)) != PCDM_OK) return s;

    stats.iters = iters;
    stats.nonzero_deltas = (int64_t)hs.nz_total;
    stats.sampler_max_rounds = iters > 0 ? std::max(1, rmax) : 0;
    stats.kernel_launches = launches;
    stats.variant = plan.variant;
    stats.grid_ctas = plan.ctas;
    stats.threads_per_cta = plan.threads;
    stats.lanes_per_column = plan.lanes;
    stats.chunk_iters = ichunk;
    stats.hot_rows = packed && Q.hot_cache ? p->nhot : 0;
    double tms[3];
    tm.sum(tms);
    stats.iter_kernel_ms = tms[T_ITER];
    stats.sampler_ms = tms[T_SAMPLER];
    if (presample) {
        // the run's stream waited only for the pass events: ev_s1 may still be pending
        cudaEventSynchronize(p->ev_s1);
        float pms = 0.f;
        if (cudaEventElapsedTime(&pms, p->ev_s0, p->ev_s1) == cudaSuccess) stats.sampler_ms += pms;
        cudaGetLastError();
    }
    stats.setup_ms = tms[T_SETUP];
    if (B.screen && B.counts) {
        int cnt[16] = {0}, cnt1[16] = {0};
        CK(cudaMemcpy(cnt, B.counts, sizeof(cnt), cudaMemcpyDeviceToHost), "read screen counts");
        CK(cudaMemcpy(cnt1, B1.counts, sizeof(cnt1), cudaMemcpyDeviceToHost), "read screen counts");
        for (int w = 0; w < 16; ++w) cnt[w] += cnt1[w];
        stats.screen_misses = cnt[2];
        stats.screen_scans = cnt[3];
        stats.screen_spec = cnt[4];
        stats.screen_flagged = cnt[5];
        if (knob("PCDM_SCREEN_CLOCKS"))
            fprintf(stderr, "screen clocks (kcyc): stage %d compute %d apply %d loop %d probes %d dgets %d\n", cnt[6], cnt[7],
                    cnt[8], cnt[9], cnt[10], cnt[11]);
    }
    if (tl_buf) {
        unsigned long long h[8 * 256];
        cudaMemcpy(h, tl_buf, sizeof(h), cudaMemcpyDeviceToHost);
        const int ns = (int)std::min<int64_t>(bsnap, 256);
        for (int q = 0; q < ns; ++q) {
            const unsigned long long t0 = ~h[8 * q];
            fprintf(stderr, "timeline chunk %d (us from expand start):", q);
            for (int k = 0; k < 4; ++k)
                fprintf(stderr, " [%.1f %.1f]", h[8 * q + 2 * k] ? ((double)(~h[8 * q + 2 * k]) - (double)t0) / 1e3 : -1.0,
                        h[8 * q + 2 * k + 1] ? ((double)h[8 * q + 2 * k + 1] - (double)t0) / 1e3 : -1.0);
            fprintf(stderr, "\n");
        }
        cudaFree(tl_buf);
    }
    p->stats = stats;
    if (hs.flags & FLAG_SAMPLER) return fail(PCDM_ESAMPLER, "sampler round counter overflow");
    if (hs.flags & FLAG_DIVERGED) return fail(PCDM_EDIVERGED, "non-finite step (diverged)");
    return PCDM_OK;
}

}  // namespace

extern "C" {

pcdm_status pcdm_run_async(pcdm_problem* p, float* x, int64_t updates, int64_t tau_beta, double beta_override,
                           int64_t refresh_every, uint64_t first_update, uint64_t seed, void* stream) {
    if (!p || !x) return fail(PCDM_EINVAL, "NULL argument");
    if (updates < 0 || tau_beta < 0) return fail(PCDM_EINVAL, "updates and tau_beta must be >= 0");
    if (!p->packed_G)
        return fail(PCDM_EINVAL, "asynchronous variant needs the uniform packed layout (max column length %lld)",
                    (long long)p->max_len);
    if (p->loss != 0) return fail(PCDM_EINVAL, "asynchronous variant: LASSO problems only");
    if (!(beta_override <= 1e308)) return fail(PCDM_EINVAL, "beta_override must be finite");
    CK(cudaSetDevice(p->device), "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    pcdm_run_stats stats{};
    int64_t launches = 0;
    RunTimer tm{p, st};
    int t0;
    CK(tm.begin(&t0), "event");
    const bool x_dev = is_device_ptr(x);
    float* xd = x;
    if (!x_dev) {
        if (!p->xbuf) CK(cudaMalloc((void**)&p->xbuf, sizeof(float) * p->n), "alloc x buffer");
        CK(cudaMemcpyAsync(p->xbuf, x, sizeof(float) * p->n, cudaMemcpyHostToDevice, st), "copy x in");
        xd = p->xbuf;
    }
    CK(cudaMemsetAsync(p->sc, 0, sizeof(Scalars), st), "memset scalars");
    pcdm_status s = residual_from(p, xd, st, &launches);
    if (s != PCDM_OK) return s;
    CK(tm.end(T_SETUP, t0), "event");
    Scalars hs{};
    if ((s = read_scalars(p, &hs, st)) != PCDM_OK) return s;
    if (hs.flags & FLAG_NONFINITE_X) return fail(PCDM_EINVAL, "non-finite value in x");

    int ctas = 0;
    const int64_t workers = async_groups(p->packed_G, p->sms, &ctas);
    const int64_t tb = std::min<int64_t>(tau_beta > 0 ? tau_beta : workers, p->n);
    double beta_d = 1.0 + (double)(p->omega - 1) * (double)(tb - 1) / (double)std::max<int64_t>(1, p->n - 1);
    if (beta_override > 0.0) beta_d = beta_override;
    const int64_t R = refresh_every < 0 ? 0 : (refresh_every > 0 ? refresh_every : 2 * p->n);
    AsyncParams A{};
    A.blocks = p->blocks;
    A.x = xd;
    A.r = p->r;
    A.n = p->n;
    A.seed = seed;
    A.reject_below = (uint64_t)(0 - (uint64_t)p->n) % (uint64_t)p->n;
    A.beta = (float)beta_d;
    A.lambda = (float)p->lambda;
    A.flags = &p->sc->flags;
    A.nz_total = &p->sc->nz_total;
    A.hot_rows = p->hot_rows;
    for (int64_t done = 0; done < updates;) {
        const int64_t c = R > 0 ? std::min(R, updates - done) : updates - done;
        A.updates = c;
        A.u0 = (int64_t)(first_update + (uint64_t)done);
        int ti;
        CK(tm.begin(&ti), "event");
        CK(launch_async(p->packed_G, ctas, A, st, &launches), "async kernel");
        CK(tm.end(T_ITER, ti), "event");
        ++stats.iter_launches;
        done += c;
        if (R > 0 && done < updates) {
            int tr;
            CK(tm.begin(&tr), "event");
            if ((s = residual_from(p, xd, st, &launches)) != PCDM_OK) return s;
            CK(tm.end(T_SETUP, tr), "event");
            ++stats.refreshes;
        }
    }
    p->r_cur = p->r;
    int tx;
    CK(tm.begin(&tx), "event");
    if (!x_dev) CK(cudaMemcpyAsync(x, p->xbuf, sizeof(float) * p->n, cudaMemcpyDeviceToHost, st), "copy x out");
    CK(tm.end(T_SETUP, tx), "event");
    if ((s = read_scalars(p, &hs, st)) != PCDM_OK) return s;
    stats.iters = updates;
    stats.nonzero_deltas = (int64_t)hs.nz_total;
    stats.kernel_launches = launches;
    stats.variant = -1;
    stats.grid_ctas = ctas;
    stats.threads_per_cta = 512;
    stats.lanes_per_column = p->packed_G;
    stats.chunk_iters = R > 0 ? R : updates;
    double tms[3];
    tm.sum(tms);
    stats.iter_kernel_ms = tms[T_ITER];
    stats.sampler_ms = 0.0;
    stats.setup_ms = tms[T_SETUP];
    p->stats = stats;
    if (hs.flags & FLAG_DIVERGED) return fail(PCDM_EDIVERGED, "non-finite step (diverged)");
    return PCDM_OK;
}

pcdm_status pcdm_objective(pcdm_problem* p, const float* x, double* F, void* stream) {
    if (!p || !x || !F) return fail(PCDM_EINVAL, "NULL argument");
    CK(cudaSetDevice(p->device), "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t launches = 0;
    const float* xd = x;
    float* tmp = nullptr;
    if (!is_device_ptr(x)) {
        CK(cudaMalloc((void**)&tmp, sizeof(float) * p->n), "alloc x");
        CK(cudaMemcpyAsync(tmp, x, sizeof(float) * p->n, cudaMemcpyHostToDevice, st), "copy x");
        xd = tmp;
    }
    pcdm_status s = PCDM_OK;
    Scalars hs{};
    do {
        cudaError_t e = cudaMemsetAsync(&p->sc->flags, 0, sizeof(int), st);
        if (e != cudaSuccess) { s = cuda_fail(e, "memset"); break; }
        if ((e = launch_residual64(p->csc(), p->b, xd, p->r64, &p->sc->flags, st, p->sms, &launches, nullptr, p->has_csr ? &p->csr : nullptr)) != cudaSuccess) { s = cuda_fail(e, "residual"); break; }
        if (p->loss == 0) {
            if ((e = launch_objective_sums(p->m, p->n, p->r64, xd, p->sc->sums, st, p->sms, &launches)) != cudaSuccess) { s = cuda_fail(e, "objective"); break; }
        } else if ((e = launch_objective_logistic(p->m, p->n, p->r64, xd, p->sc->sums, st, p->sms, &launches)) != cudaSuccess) {
            s = cuda_fail(e, "objective");
            break;
        }
        s = read_scalars(p, &hs, st);
    } while (0);
    cudaFree(tmp);
    if (s != PCDM_OK) return s;
    if (hs.flags & FLAG_NONFINITE_X) return fail(PCDM_EINVAL, "non-finite value in x");
    *F = (p->loss == 0 ? 0.5 * hs.sums[0] : hs.sums[0]) + p->lambda * hs.sums[1];
    return PCDM_OK;
}

pcdm_status pcdm_last_run_stats(const pcdm_problem* p, pcdm_run_stats* stats) {
    if (!p || !stats) return fail(PCDM_EINVAL, "NULL argument");
    *stats = p->stats;
    return PCDM_OK;
}

pcdm_status pcdm_sample(int64_t n, int64_t tau, uint64_t seed, int64_t first_iter, int64_t count, int32_t* slots,
                        void* stream) {
    pcdm_sampling smp{};
    smp.kind = PCDM_SAMPLING_NICE;
    smp.tau = tau;
    smp.p_b = 1.0;
    return pcdm_sample_sampling(n, &smp, seed, first_iter, count, slots, stream);
}

pcdm_status pcdm_sample_sampling(int64_t n, const pcdm_sampling* sampling, uint64_t seed, int64_t first_iter,
                                 int64_t count, int32_t* slots, void* stream) {
    if (!slots) return fail(PCDM_EINVAL, "NULL argument");
    if (n < 1 || n >= (1ll << 31)) return fail(PCDM_EINVAL, "n must be in [1, 2^31)");
    SamplingSpec spec;
    pcdm_status s = check_sampling(sampling, n, &spec);
    if (s != PCDM_OK) return s;
    const int64_t tau = spec.tau;
    if (count < 0 || first_iter < 0 || first_iter + count > (1ll << 32))
        return fail(PCDM_EINVAL, "bad iteration range");
    if (count == 0) return PCDM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t chunk = choose_chunk(n, tau, count);
    void* mem = nullptr;
    size_t cap = 0;
    int* flags = nullptr;
    uint64_t* dT = nullptr;
    size_t dcap = 0;
    SamplerPlan sp;
    SamplingDev sdev;
    s = sampler_workspace(&mem, &cap, n, tau, chunk, &sp, spec.kind == PCDM_SAMPLING_INDEPENDENT);
    if (s == PCDM_OK) s = sampling_dev(spec, &dT, &dcap, st, &sdev);
    if (s != PCDM_OK) {
        cudaFree(mem);
        cudaFree(dT);
        return s;
    }
    int64_t launches = 0;
    cudaError_t e = cudaMalloc((void**)&flags, sizeof(int));
    if (e == cudaSuccess) e = cudaMemsetAsync(flags, 0, sizeof(int), st);
    const bool dev_out = is_device_ptr(slots);
    for (int64_t done = 0; e == cudaSuccess && done < count;) {
        const int64_t c = std::min(chunk, count - done);
        e = sample_chunk(sp.w, sdev, seed, first_iter + done, c, sp.slots, flags, st, sms, &launches);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(slots + done * tau, sp.slots, sizeof(int) * c * tau,
                                dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st);
        done += c;
    }
    int hflags = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hflags, flags, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(mem);
    cudaFree(flags);
    cudaFree(dT);
    if (e != cudaSuccess) return cuda_fail(e, "pcdm_sample");
    if (hflags & FLAG_SAMPLER) return fail(PCDM_ESAMPLER, "sampler round counter overflow");
    return PCDM_OK;
}

pcdm_status pcdm_beta_sampling(const pcdm_problem* p, const pcdm_sampling* sampling, double* beta) {
    if (!p || !beta) return fail(PCDM_EINVAL, "NULL argument");
    SamplingSpec spec;
    pcdm_status s = check_sampling(sampling, p->n, &spec);
    if (s != PCDM_OK) return s;
    *beta = sampling_beta(spec, p->omega, p->n);
    return PCDM_OK;
}

pcdm_status pcdm_col_norms(const pcdm_problem* p, float* L, void* stream) {
    if (!p || !L) return fail(PCDM_EINVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemcpyAsync(L, p->L, sizeof(float) * p->n, cudaMemcpyDefault, st), "copy L");
    CK(cudaStreamSynchronize(st), "sync");
    return PCDM_OK;
}

pcdm_status pcdm_row_counts(const pcdm_problem* p, int32_t* counts, void* stream) {
    if (!p || !counts) return fail(PCDM_EINVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t launches = 0;
    int* d = nullptr;
    CK(cudaMalloc((void**)&d, sizeof(int) * p->m), "alloc counts");
    cudaError_t e = launch_row_counts(p->csc(), d, st, p->sms, &launches);
    if (e == cudaSuccess) e = cudaMemcpyAsync(counts, d, sizeof(int) * p->m, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "row counts");
    return PCDM_OK;
}

pcdm_status pcdm_residual(const pcdm_problem* p, float* r, void* stream) {
    if (!p || !r) return fail(PCDM_EINVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemcpyAsync(r, p->r_cur, sizeof(float) * p->m, cudaMemcpyDefault, st), "copy r");
    CK(cudaStreamSynchronize(st), "sync");
    return PCDM_OK;
}

pcdm_status pcdm_philox(int64_t count, const uint32_t* ctr, const uint32_t* key, uint32_t* out, void* stream) {
    if (count < 0 || (count > 0 && (!ctr || !key || !out))) return fail(PCDM_EINVAL, "bad arguments");
    if (count == 0) return PCDM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *dc = nullptr, *dk = nullptr, *dout = nullptr;
    cudaError_t e = cudaMalloc((void**)&dc, 16 * count);
    if (e == cudaSuccess) e = cudaMalloc((void**)&dk, 8 * count);
    if (e == cudaSuccess) e = cudaMalloc((void**)&dout, 16 * count);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dc, ctr, 16 * count, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dk, key, 8 * count, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = launch_philox(count, dc, dk, dout, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, 16 * count, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(dc);
    cudaFree(dk);
    cudaFree(dout);
    if (e != cudaSuccess) return cuda_fail(e, "pcdm_philox");
    return PCDM_OK;
}

pcdm_status pcdm_philox_check_curand(int64_t count, uint64_t seed, int64_t* mismatches, void* stream) {
    if (!mismatches || count < 0) return fail(PCDM_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* d = nullptr;
    unsigned long long h = 0;
    cudaError_t e = cudaMalloc((void**)&d, sizeof(unsigned long long));
    if (e == cudaSuccess) e = launch_philox_check_curand(count, seed, d, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "pcdm_philox_check_curand");
    *mismatches = (int64_t)h;
    return PCDM_OK;
}

}  // extern "C"
