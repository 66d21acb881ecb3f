// l2_policy.cu -- what does one random 4-byte load out of a 400 MB array cost in DRAM
// traffic on B200, and can the L2 be told to fetch less or keep more of the array?
//
// ncu on the PCDM hot loop (huge config) showed ~4 DRAM sectors (128 B) read per
// random r gather.  Cases (each a separate kernel launch, rate printed; run under
// ncu --metrics dram__sectors_read.sum,lts__t_sector_hit_rate.pct for the bytes):
//   fetch_default        no limit set
//   fetch_limit_{32,64}  cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g)
//   persist_window       cudaAccessPolicyWindow over the array, hitRatio = set-aside / size
//   evict_last_frac      ld with createpolicy.fractional.L2::evict_last (fraction f)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2_policy tools/l2_policy.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

template <int MODE>
__device__ __forceinline__ float ld(const float* p, uint64_t pol) {
    float v;
    if (MODE == 0) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    if (MODE == 1) asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// random gathers: hash-generated addresses (no index traffic), U loads in flight per thread
template <int MODE, int U>
__global__ void gather_kernel(const float* __restrict__ a, uint64_t len, int rounds, float frac, uint32_t salt,
                              float* out) {
    uint64_t pol = 0;
    if (MODE == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(pol) : "f"(frac));
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    uint32_t h = (uint32_t)tid * 0x9E3779B1u + salt;
    for (int r = 0; r < rounds; ++r) {
        uint64_t idx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            h ^= h << 13;
            h ^= h >> 17;
            h ^= h << 5;
            idx[u] = ((uint64_t)h * len) >> 32;
        }
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld<MODE>(a + idx[u], pol);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 12345.678f) *out = acc;
}

__global__ void flush_kernel(float* f, int64_t n, float v) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) f[t] = v;
}

int main() {
    int sms = 0, l2 = 0, persist_max = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
    CK(cudaDeviceGetAttribute(&persist_max, cudaDevAttrMaxPersistingL2CacheSize, 0));
    const uint64_t len = 100000000ull;  // 400 MB, like r of the huge config
    float *a, *out, *fl;
    CK(cudaMalloc(&a, len * 4));
    CK(cudaMemset(a, 0, len * 4));
    CK(cudaMalloc(&out, 4));
    const int64_t fln = 64ll << 20;
    CK(cudaMalloc(&fl, fln * 4));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{\"bench\": \"device\", \"l2\": %d, \"persist_max\": %d}\n", l2, persist_max);
    const int ctas = sms * 4, threads = 512, rounds = 8, U = 8;
    const double loads = (double)ctas * threads * rounds * U;
    auto run = [&](const char* name, auto kern, float frac) {
        // warm pass (L2 reaches its steady state for this policy), then 5 timed passes
        flush_kernel<<<sms * 4, 512, 0, st>>>(fl, fln, 1.f);
        kern<<<ctas, threads, 0, st>>>(a, len, rounds, frac, 1u, out);
        float best = 1e30f;
        for (int t = 0; t < 5; ++t) {
            cudaEventRecord(e0, st);
            kern<<<ctas, threads, 0, st>>>(a, len, rounds, frac, 100u + t, out);
            cudaEventRecord(e1, st);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("{\"bench\": \"%s\", \"frac\": %.2f, \"loads\": %.0f, \"us\": %.1f, \"Gloads_per_s\": %.2f}\n", name, frac,
               loads, best * 1e3, loads / best / 1e6);
    };
    run("fetch_default", gather_kernel<0, 8>, 0.f);
    for (int g : {32, 64, 128}) {
        CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g));
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        char nm[64];
        snprintf(nm, sizeof nm, "fetch_limit_%d_got_%zu", g, got);
        run(nm, gather_kernel<0, 8>, 0.f);
    }
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 0));
    for (float f : {0.25f, 0.5f, 1.0f}) run("evict_last_frac", gather_kernel<1, 8>, f);
    // persisting window over the array
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist_max));
    size_t setaside = 0;
    cudaDeviceGetLimit(&setaside, cudaLimitPersistingL2CacheSize);
    int maxwin = 0;
    cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, 0);
    const size_t win = len * 4 < (size_t)maxwin ? len * 4 : (size_t)maxwin;
    printf("{\"bench\": \"window\", \"max_window\": %d, \"window\": %zu}\n", maxwin, win);
    for (float hr : {(float)setaside / (float)win, 0.5f, 1.0f}) {
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.base_ptr = a;
        v.accessPolicyWindow.num_bytes = win;
        v.accessPolicyWindow.hitRatio = hr > 1.f ? 1.f : hr;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v));
        run("persist_window_hitratio", gather_kernel<0, 8>, v.accessPolicyWindow.hitRatio);
    }
    printf("{\"bench\": \"persist_setaside\", \"bytes\": %zu}\n", setaside);
    return 0;
}
