// loadflavors.cu -- which global-load flavour fetches the fewest DRAM bytes per
// random 4-byte access on B200 (run under ncu for dram__bytes_read.sum).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

template <int V>
__device__ __forceinline__ float ldv(const float* p) {
    float v;
    if (V == 0) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    if (V == 1) asm volatile("ld.global.cv.f32 %0, [%1];" : "=f"(v) : "l"(p));
    if (V == 2) asm volatile("ld.global.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
    if (V == 3) asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    if (V == 4) {
        unsigned u;
        asm volatile("atom.global.or.b32 %0, [%1], 0;" : "=r"(u) : "l"(p) : "memory");
        v = __uint_as_float(u);
    }
    if (V == 5) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    if (V == 6) asm volatile("ld.volatile.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    if (V == 7) asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(v) : "l"(p));
    if (V == 8) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    }
    if (V == 9) asm volatile("ld.global.lu.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

template <int V>
__global__ void gather(const float* __restrict__ a, uint64_t len, int rounds, float* out) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    uint32_t h = (uint32_t)tid * 0x9E3779B1u + 0x7F4A7C15u;
    for (int r = 0; r < rounds; ++r) {
        uint64_t idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            h ^= h << 13; h ^= h >> 17; h ^= h << 5;
            idx[u] = ((uint64_t)h * len) >> 32;
        }
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ldv<V>(a + idx[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    if (acc == 12345.678f) *out = acc;
}

template <int V>
void run(const float* a, float* out, uint64_t len, int sms, const char* name) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    const int rounds = 32;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        gather<V><<<sms * 4, 512>>>(a, len, rounds, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double loads = (double)sms * 4 * 512 * rounds * 8;
    printf("{\"bench\": \"flavor\", \"v\": %d, \"name\": \"%s\", \"array_MB\": %.0f, \"Gloads_per_s\": %.3f, \"err\": \"%s\"}\n",
           V, name, len * 4 / 1e6, loads / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    if (argc > 1) {  // set the fetch granularity limit before anything else touches the context
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1]));
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        printf("{\"bench\": \"limit\", \"set\": %s, \"got\": %zu, \"err\": \"%s\"}\n", argv[1], got, cudaGetErrorString(e));
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t len = 100000000ull;
    float *a, *out;
    cudaMalloc(&a, len * 4); cudaMalloc(&out, 4); cudaMemset(a, 0, len * 4);
    run<0>(a, out, len, sms, "ld.global.cg");
    if (argc > 1) return 0;
    run<1>(a, out, len, sms, "ld.global.cv");
    run<2>(a, out, len, sms, "ld.global.L2::64B");
    run<3>(a, out, len, sms, "ld.relaxed.gpu");
    run<4>(a, out, len, sms, "atom.or 0");
    run<5>(a, out, len, sms, "ld.nc.L1::no_allocate");
    run<6>(a, out, len, sms, "ld.volatile");
    run<7>(a, out, len, sms, "ld.global.cs");
    run<8>(a, out, len, sms, "ld.L2::cache_hint evict_first");
    run<9>(a, out, len, sms, "ld.global.lu");
    return 0;
}
