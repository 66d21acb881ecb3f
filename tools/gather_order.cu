// gather_order.cu -- does address order change the random-access rate of HBM on B200?
//
// The huge config's iteration is ~2.6M random 4-byte gathers of r (400 MB, far
// larger than L2) plus ~0.5M random column/x accesses.  This measures, for
// N = 2.6M accesses into a 400 MB array:
//   * gather / red.add rate with the indices in random order,
//   * the same indices sorted on bits [s, 27) only (bucketed: random order inside
//     buckets of 2^s floats), for several s, and fully sorted (s = 0),
//   * the cost of the radix sort itself (cub, keys only / pairs).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/gather_order tools/gather_order.cu
#include <cub/cub.cuh>
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

__global__ void make_indices(uint32_t* idx, int64_t total, uint32_t len, uint32_t salt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = (uint64_t)t * 0x9E3779B97F4A7C15ull + salt;
        h ^= h >> 31;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
        idx[t] = (uint32_t)(((h & 0xffffffffull) * len) >> 32);
    }
}

template <int U>
__global__ void gather(const float* __restrict__ a, const uint32_t* __restrict__ idx, int64_t N, float* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < N; base += stride * U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = base + u * stride;
            v[u] = q < N ? __ldcg(a + __ldg(idx + q)) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = base + u * stride;
            if (q < N) out[q] = v[u];
        }
    }
}

// CTA-blocked variant: CTA b owns the contiguous index range [b*chunk, (b+1)*chunk), so with
// sorted indices each CTA sweeps one address region and all CTAs sweep in parallel.
template <int U>
__global__ void gather_blocked(const float* __restrict__ a, const uint32_t* __restrict__ idx, int64_t N, float* __restrict__ out) {
    const int64_t chunk = (N + gridDim.x - 1) / gridDim.x;
    const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(N, lo + chunk);
    for (int64_t base = lo + threadIdx.x; base < hi; base += (int64_t)blockDim.x * U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = base + u * blockDim.x;
            v[u] = q < hi ? __ldcg(a + __ldg(idx + q)) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = base + u * blockDim.x;
            if (q < hi) out[q] = v[u];
        }
    }
}

__global__ void scatter_red(float* __restrict__ a, const uint32_t* __restrict__ idx, int64_t N) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (int64_t)gridDim.x * blockDim.x)
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(a + __ldg(idx + q)), "f"(1.0f) : "memory");
}

__global__ void flush_kernel(float* f, int64_t n, float v) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) f[t] = v;
}

int main(int argc, char** argv) {
    const uint32_t len = argc > 1 ? (uint32_t)atoll(argv[1]) : 100000000u;
    const int64_t N = argc > 2 ? atoll(argv[2]) : 2621440;
    const int SETS = 8;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float *a, *out, *fl;
    uint32_t *idx, *sorted, *tmpk;
    CK(cudaMalloc(&a, (size_t)len * 4));
    CK(cudaMemset(a, 0, (size_t)len * 4));
    CK(cudaMalloc(&out, N * 4));
    const int64_t fln = 64ll << 20;  // 256 MB flush buffer
    CK(cudaMalloc(&fl, fln * 4));
    CK(cudaMalloc(&idx, N * SETS * 4));
    CK(cudaMalloc(&sorted, N * SETS * 4));
    CK(cudaMalloc(&tmpk, N * 4));
    make_indices<<<sms * 8, 256>>>(idx, N * SETS, len, 12345u);
    CK(cudaDeviceSynchronize());
    int endbit = 0;
    while ((1ull << endbit) < len) ++endbit;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, idx, sorted, (int)N, 0, endbit);
    void* tmp;
    CK(cudaMalloc(&tmp, tmp_bytes * 2 + (1 << 20)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{\"bench\": \"setup\", \"array_MB\": %.1f, \"N\": %lld, \"sets\": %d, \"endbit\": %d}\n", len * 4 / 1e6,
           (long long)N, SETS, endbit);

    auto timed = [&](const char* what, int s_bits, auto&& launch) {
        float tot = 0.f;
        for (int s = 0; s < SETS; ++s) {
            flush_kernel<<<sms * 4, 512>>>(fl, fln, (float)s);
            cudaEventRecord(e0);
            launch(s);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (s > 0) tot += ms;  // set 0 = warm-up
        }
        const double us = tot * 1e3 / (SETS - 1);
        printf("{\"bench\": \"%s\", \"bucket_bits\": %d, \"us\": %.2f, \"Gaccess_per_s\": %.2f, \"GBps_32B\": %.0f}\n", what,
               s_bits, us, N / us / 1e3, N * 32.0 / us / 1e3);
    };

    for (int sb : {-1, 22, 18, 14, 12, 10, 8, 0}) {
        // order: -1 = random; else sorted on bits [sb, endbit)
        for (int s = 0; s < SETS; ++s) {
            if (sb < 0) {
                CK(cudaMemcpy(sorted + s * N, idx + s * N, N * 4, cudaMemcpyDeviceToDevice));
            } else {
                size_t tb = tmp_bytes * 2;
                CK(cub::DeviceRadixSort::SortKeys(tmp, tb, idx + s * N, sorted + s * N, (int)N, sb, endbit));
            }
        }
        CK(cudaDeviceSynchronize());
        timed("gather_U8", sb, [&](int s) { gather<8><<<sms * 4, 512>>>(a, sorted + s * N, N, out); });
        timed("gather_U4", sb, [&](int s) { gather<4><<<sms * 4, 512>>>(a, sorted + s * N, N, out); });
        timed("gather_blocked_U8", sb, [&](int s) { gather_blocked<8><<<sms * 4, 512>>>(a, sorted + s * N, N, out); });
        timed("gather_blocked_U4_8cta", sb, [&](int s) { gather_blocked<4><<<sms * 8, 256>>>(a, sorted + s * N, N, out); });
        timed("red_add", sb, [&](int s) { scatter_red<<<sms * 8, 512>>>(a, sorted + s * N, N); });
        if (sb >= 0) {
            timed("sort_keys", sb, [&](int s) {
                size_t tb = tmp_bytes * 2;
                cub::DeviceRadixSort::SortKeys(tmp, tb, idx + s * N, tmpk, (int)N, sb, endbit);
            });
        }
    }
    return 0;
}
