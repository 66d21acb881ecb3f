// atomic_rate.cu -- L2 atomic throughput on random addresses in a 4 MB table
// (the sampler's per-iteration hash table): 64-bit CAS (the round-0 insert) vs
// 32-bit CAS, 64-bit load, and 32-bit red.add, 262144 x 9 operations per launch.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/atomic_rate tools/atomic_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <algorithm>
#include <vector>

__device__ __forceinline__ uint32_t hsh(uint64_t t) {
    t ^= t >> 31; t *= 0xBF58476D1CE4E5B9ull; t ^= t >> 29; t *= 0x94D049BB133111EBull; t ^= t >> 32;
    return (uint32_t)t;
}

template <int OP>
__global__ void k(unsigned long long* t64, unsigned* t32, int64_t total, int log2h, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t it = q >> 18;
        const uint32_t h = hsh(q) >> (32 - log2h);
        if (OP == 0) acc += atomicCAS(t64 + (it << log2h) + h, ~0ull, (unsigned long long)q);
        if (OP == 1) acc += atomicCAS(t32 + (it << log2h) + h, ~0u, (unsigned)q);
        if (OP == 2) acc += __ldcg(t64 + (it << log2h) + h);
        if (OP == 3) atomicAdd(t32 + (it << log2h) + h, 1u);
        if (OP == 4) acc += atomicAdd(t32 + (it << log2h) + h, 1u);
        if (OP == 5) acc += atomicMin(t64 + (it << log2h) + h, (unsigned long long)q);
    }
    if (acc == 42) *sink = acc;
}

int main() {
    const int log2h = 19, iters = 9;
    const int64_t total = (int64_t)iters << 18;
    unsigned long long *t64, *sink;
    unsigned* t32;
    cudaMalloc(&t64, ((size_t)iters << log2h) * 8);
    cudaMalloc(&t32, ((size_t)iters << log2h) * 4);
    cudaMalloc(&sink, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"cas64", "cas32", "ld64", "red32", "atomadd32_ret", "min64"};
    for (int op = 0; op < 6; ++op) {
        std::vector<float> ts;
        for (int rep = 0; rep < 7; ++rep) {
            cudaMemset(t64, 0xFF, ((size_t)iters << log2h) * 8);
            cudaMemset(t32, 0xFF, ((size_t)iters << log2h) * 4);
            cudaEventRecord(a);
            switch (op) {
                case 0: k<0><<<sms * 8, 256>>>(t64, t32, total, log2h, sink); break;
                case 1: k<1><<<sms * 8, 256>>>(t64, t32, total, log2h, sink); break;
                case 2: k<2><<<sms * 8, 256>>>(t64, t32, total, log2h, sink); break;
                case 3: k<3><<<sms * 8, 256>>>(t64, t32, total, log2h, sink); break;
                case 4: k<4><<<sms * 8, 256>>>(t64, t32, total, log2h, sink); break;
                case 5: k<5><<<sms * 8, 256>>>(t64, t32, total, log2h, sink); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        printf("{\"op\": \"%s\", \"ops\": %lld, \"us_median\": %.2f, \"Gops\": %.1f}\n", names[op], (long long)total,
               ts[3] * 1e3, total / (ts[3] * 1e6));
    }
    return 0;
}
