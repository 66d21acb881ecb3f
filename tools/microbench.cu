// microbench.cu -- B200 microbenchmarks that decide the PCDM kernel design:
//   1. grid-barrier latency of several barrier implementations vs grid size;
//   2. random 4-byte gather throughput from HBM-sized and L2-sized arrays;
//   3. streaming read bandwidth (L2-resident and HBM) for roofline denominators.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
// Output: one JSON object per line.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e = (x);                                                             \
        if (e != cudaSuccess) {                                                          \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));    \
            exit(1);                                                                     \
        }                                                                                \
    } while (0)

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// variant 0: everyone polls the arrival counter
// variant 1: last arriver publishes a generation flag, others poll the flag
// variant 2: as 1, with release/acquire atomics (no separate fences)
// variant 3: as 2, with __nanosleep backoff while polling
template <int V>
__global__ void barrier_kernel(unsigned* count, unsigned* flag, int reps, unsigned long long* cycles) {
    unsigned target = 0, gen = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        if (threadIdx.x == 0) {
            if (V == 0) {
                target += gridDim.x;
                __threadfence();
                atomicAdd(count, 1u);
                while ((int)(ld_acquire(count) - target) < 0) {
                }
                __threadfence();
            } else if (V == 1) {
                ++gen;
                __threadfence();
                const unsigned arrived = atomicAdd(count, 1u) + 1;
                if (arrived == gen * gridDim.x) {
                    st_release(flag, gen);
                } else {
                    while ((int)(ld_acquire(flag) - gen) < 0) {
                    }
                }
                __threadfence();
            } else {
                ++gen;
                const unsigned arrived = atom_add_release(count, 1u) + 1;
                if (arrived == gen * gridDim.x) {
                    st_release(flag, gen);
                } else {
                    while ((int)(ld_acquire(flag) - gen) < 0) {
                        if (V == 3) __nanosleep(20);
                    }
                }
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = (unsigned long long)(clock64() - t0);
}

template <int V>
void run_barrier(int ctas, int threads, int reps) {
    unsigned *count, *flag;
    unsigned long long* cyc;
    CK(cudaMalloc(&count, 4));
    CK(cudaMalloc(&flag, 4));
    CK(cudaMalloc(&cyc, 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int trial = 0; trial < 3; ++trial) {
        CK(cudaMemset(count, 0, 4));
        CK(cudaMemset(flag, 0, 4));
        void* args[] = {&count, &flag, &reps, &cyc};
        cudaEventRecord(a);
        CK(cudaLaunchCooperativeKernel((void*)barrier_kernel<V>, ctas, threads, args, 0, 0));
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    printf("{\"bench\": \"barrier\", \"variant\": %d, \"ctas\": %d, \"threads\": %d, \"reps\": %d, \"us_per_barrier\": %.4f}\n",
           V, ctas, threads, reps, best * 1e3 / reps);
    cudaFree(count);
    cudaFree(flag);
    cudaFree(cyc);
}

// Random gather: each thread issues U independent 4-byte loads per round at
// pseudo-random positions (hash of thread, round) in an array of `len` floats.
template <int U, bool CG>
__global__ void gather_kernel(const float* __restrict__ a, uint64_t len, int rounds, float* out) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    uint32_t h = (uint32_t)tid * 0x9E3779B1u + 0x7F4A7C15u;
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
        for (int u = 0; u < U; ++u) {
            if (CG) v[u] = __ldcg(a + idx[u]);
            else v[u] = __ldg(a + idx[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 12345.678f) *out = acc;
}

template <int U, bool CG>
void run_gather(uint64_t len, int ctas, int threads, int rounds) {
    float* a;
    float* out;
    CK(cudaMalloc(&a, len * 4));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(a, 0, len * 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 4; ++t) {
        cudaEventRecord(e0);
        gather_kernel<U, CG><<<ctas, threads>>>(a, len, rounds, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double loads = (double)ctas * threads * rounds * U;
    printf("{\"bench\": \"gather\", \"array_MB\": %.1f, \"U\": %d, \"cg\": %d, \"ctas\": %d, \"threads\": %d, "
           "\"Gloads_per_s\": %.3f, \"GBps_4B\": %.1f, \"GBps_32Bsector\": %.1f, \"GBps_64B\": %.1f}\n",
           len * 4 / 1e6, U, (int)CG, ctas, threads, loads / best / 1e6, loads * 4 / best / 1e6,
           loads * 32 / best / 1e6, loads * 64 / best / 1e6);
    cudaFree(a);
    cudaFree(out);
}

__global__ void stream_read_kernel(const float4* __restrict__ a, uint64_t n4, int reps, float* out) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(a + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 12345.678f) *out = acc;
}

void run_stream(uint64_t bytes, int reps, int sms) {
    float4* a;
    float* out;
    CK(cudaMalloc(&a, bytes));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(a, 0, bytes));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
        cudaEventRecord(e0);
        stream_read_kernel<<<sms * 8, 512>>>(a, bytes / 16, reps, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf("{\"bench\": \"stream_read\", \"buffer_MB\": %.1f, \"reps\": %d, \"GBps\": %.1f}\n", bytes / 1e6, reps,
           (double)bytes * reps / best / 1e6);
    cudaFree(a);
    cudaFree(out);
}

int main(int argc, char** argv) {
    int dev = 0, sms = 0;
    if (argc > 1 && argv[1][0] == 'g') {  // fetch-granularity sweep only
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        for (int g : {0, 32, 64, 128}) {
            CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g));
            size_t got = 0;
            cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
            printf("{\"bench\": \"l2_fetch_granularity\", \"set\": %d, \"got\": %zu}\n", g, got);
            run_gather<8, true>(100000000ull, sms * 4, 512, 64);
            run_gather<8, true>(500000000ull, sms * 4, 512, 64);
        }
        return 0;
    }
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    printf("{\"bench\": \"device\", \"sms\": %d, \"l2_bytes\": %d}\n", sms, l2);
    const int reps = 2000;
    for (int per : {1, 2, 3, 4}) {
        run_barrier<0>(sms * per, 512, reps);
        run_barrier<1>(sms * per, 512, reps);
        run_barrier<2>(sms * per, 512, reps);
        run_barrier<3>(sms * per, 512, reps);
    }
    run_barrier<2>(sms, 1024, reps);
    run_barrier<2>(sms * 2, 1024, reps);
    // random gathers: 400 MB (huge r), 8 MB (large r), 2 GB
    for (uint64_t len : {100000000ull, 2000000ull, 500000000ull}) {
        run_gather<8, true>(len, sms * 4, 512, 64);
        run_gather<16, true>(len, sms * 4, 512, 32);
        run_gather<8, false>(len, sms * 4, 512, 64);
    }
    run_gather<4, true>(100000000ull, sms * 4, 512, 128);
    run_gather<32, true>(100000000ull, sms * 2, 512, 16);
    // streaming reads: L2-resident (l2/4) and HBM (4 GB)
    run_stream((uint64_t)l2 / 4, 200, sms);
    run_stream((uint64_t)l2 / 2, 100, sms);
    run_stream(4ull << 30, 3, sms);
    return 0;
}
