// Latency calibration for the one-CTA shared-memory loop (tiny): cycles and ns per
// iteration of (a) a bare __syncthreads loop, (b) a dependent shared-memory load chain
// + barrier, (c) (b) + a 4-lane butterfly + an fp32 division, for 128 and 512 threads.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int MODE>
__global__ void probe(int iters, unsigned long long* out, float* sink) {
    __shared__ int s_idx[4096];
    __shared__ float s_f[4096];
    for (int t = threadIdx.x; t < 4096; t += blockDim.x) {
        s_idx[t] = (t * 7 + 13) & 4095;
        s_f[t] = 1.0f + t;
    }
    __syncthreads();
    int p = threadIdx.x;
    float acc = 0.f;
    const unsigned long long c0 = clock64(), t0 = gtime();
    for (int it = 0; it < iters; ++it) {
        if (MODE >= 1) {
            p = s_idx[p];
            p = s_idx[p];
            p = s_idx[p];
            acc += s_f[p];
        }
        if (MODE >= 2) {
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            acc = 1.0f - acc / (3.0f + s_f[p & 7]);
        }
        __syncthreads();
    }
    const unsigned long long c1 = clock64(), t1 = gtime();
    if (threadIdx.x == 0) {
        out[0] = c1 - c0;
        out[1] = t1 - t0;
    }
    sink[threadIdx.x] = acc + p;
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 16);
    cudaMalloc(&sink, 4096);
    const int iters = 100000;
    for (int threads : {32, 128, 512}) {
        for (int mode = 0; mode < 3; ++mode) {
            unsigned long long h[2];
            for (int rep = 0; rep < 3; ++rep) {
                if (mode == 0) probe<0><<<1, threads>>>(iters, d, sink);
                if (mode == 1) probe<1><<<1, threads>>>(iters, d, sink);
                if (mode == 2) probe<2><<<1, threads>>>(iters, d, sink);
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            }
            printf("threads=%d mode=%d cycles/iter=%.1f ns/iter=%.1f clock=%.0f MHz\n", threads, mode,
                   (double)h[0] / iters, (double)h[1] / iters, 1e3 * (double)h[0] / (double)h[1]);
        }
    }
    return 0;
}
