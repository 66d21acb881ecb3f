// tile_pass.cu -- costs of the pieces of a row-tiled ("propagation-blocked") gather on B200.
//
// Batched-snapshot design for the huge config: the B*tau*c gathers of B iterations
// are binned by row tile (r tile <= ~50 MB, L2-resident), then each tile's entries
// gather r from L2 and accumulate into per-slot sums.  Measured here for one tile
// (12.5M rows = 50 MB of a 400 MB r) with E = 2.6M entries:
//   gather_only      sum of val*r[row] (rows inside the tile), cold and warm L2
//   red_slot         red.add.f32 of val*r[row] into G[dest], G = 2^21 floats (8 MB)
//   st_pos           st.global of val*r[row] into P[pos], P = 21M floats (84 MB), pos random
//   bin_pass         read 262K random 128-byte blocks, bin their 10 entries into 8 tiles
//                    through shared memory, write 12-byte entries
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tile_pass tools/tile_pass.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t err_ = (x);                                                          \
        if (err_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(err_)); \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t h) {
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    h *= 0x94D049BB133111EBull;
    h ^= h >> 32;
    return h;
}

struct Entry {
    int row;
    int dest;
    float val;
};

__global__ void make_entries(Entry* e, int64_t E, uint32_t tile_rows, uint32_t ndest, uint64_t salt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < E; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix((uint64_t)t + salt);
        e[t].row = (int)(((h & 0xffffffffull) * tile_rows) >> 32);
        e[t].dest = (int)(((h >> 32) * ndest) >> 32);
        e[t].val = 1.0f;
    }
}

__global__ void gather_only(const float* __restrict__ r, const Entry* __restrict__ e, int64_t E, float* out) {
    float acc = 0.f;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < E; t += (int64_t)gridDim.x * blockDim.x) {
        const Entry q = e[t];
        acc += q.val * __ldcg(r + q.row);
    }
    if (acc == 1234.5f) *out = acc;
}

__global__ void red_slot(const float* __restrict__ r, const Entry* __restrict__ e, int64_t E, float* G) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < E; t += (int64_t)gridDim.x * blockDim.x) {
        const Entry q = e[t];
        const float v = q.val * __ldcg(r + q.row);
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(G + q.dest), "f"(v) : "memory");
    }
}

__global__ void st_pos(const float* __restrict__ r, const Entry* __restrict__ e, int64_t E, float* P, uint32_t npos) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < E; t += (int64_t)gridDim.x * blockDim.x) {
        const Entry q = e[t];
        const float v = q.val * __ldcg(r + q.row);
        const uint32_t pos = (uint32_t)(((uint64_t)(uint32_t)(q.dest * 2654435761u) * npos) >> 32);
        __stcg(P + pos, v);
    }
}

// bin pass: warp per 4 columns (8 lanes x 16 B per column block), 8 tiles, smem staging per CTA
constexpr int kTiles = 8;
constexpr int kStage = 448;  // entries per tile staged per CTA (one round of 256 threads adds <= 320)
__global__ void __launch_bounds__(256) bin_pass(const int4* __restrict__ blocks, const int* __restrict__ cols, int64_t ncols,
                                                uint32_t tile_shift, Entry* __restrict__ bins, int64_t bin_cap,
                                                unsigned long long* __restrict__ bin_fill) {
    __shared__ Entry stage[kTiles][kStage];
    __shared__ int cnt[kTiles];
    __shared__ unsigned long long base[kTiles];
    if (threadIdx.x < kTiles) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int lane8 = threadIdx.x & 7;
    const int64_t groups = ((int64_t)gridDim.x * blockDim.x) >> 3;
    const int64_t per_round = (int64_t)blockDim.x >> 3;
    for (int64_t g0 = (int64_t)blockIdx.x * per_round; g0 < ncols; g0 += groups) {
        const int64_t g = g0 + (threadIdx.x >> 3);
        if (g < ncols) {
            const int i = cols[g];
            const int4 c = __ldcs(blocks + (int64_t)i * 8 + lane8);
            if (lane8 >= 1 && lane8 <= 5) {
                const int rr[2] = {c.x, c.z};
                const float vv[2] = {__int_as_float(c.y), __int_as_float(c.w)};
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int t = rr[u] >> tile_shift;
                    const int p = atomicAdd(&cnt[t], 1);
                    if (p < kStage) stage[t][p] = Entry{rr[u] & ((1 << tile_shift) - 1), (int)g, vv[u]};
                }
            }
        }
        __syncthreads();
        // flush when any tile's stage is more than half full (always at the end)
        bool flush = (g0 + groups >= ncols);
        if (threadIdx.x == 0) {
            for (int t = 0; t < kTiles; ++t) flush |= cnt[t] > kStage - 320;
        }
        flush = __syncthreads_or(flush);
        if (flush) {
            if (threadIdx.x < kTiles) {
                const int k = min(cnt[threadIdx.x], kStage);
                base[threadIdx.x] = atomicAdd(bin_fill + threadIdx.x, (unsigned long long)k);
            }
            __syncthreads();
            for (int t = 0; t < kTiles; ++t) {
                const int k = min(cnt[t], kStage);
                for (int q = threadIdx.x; q < k; q += blockDim.x)
                    if (base[t] + q < (unsigned long long)bin_cap) bins[t * bin_cap + base[t] + q] = stage[t][q];
            }
            __syncthreads();
            if (threadIdx.x < kTiles) cnt[threadIdx.x] = 0;
            __syncthreads();
        }
    }
}

__global__ void make_blocks(int4* b, int64_t n, uint32_t m) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n * 8; q += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix((uint64_t)q);
        const int t = (int)(q & 7);
        int4 c = make_int4(0, 0, 0, 0);
        if (t >= 1 && t <= 5)
            c = make_int4((int)(((h & 0xffffffffull) * m) >> 32), __float_as_int(1.f), (int)(((h >> 32) * m) >> 32),
                          __float_as_int(1.f));
        b[q] = c;
    }
}

__global__ void make_cols(int* cols, int64_t k, uint32_t n, uint64_t salt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < k; t += (int64_t)gridDim.x * blockDim.x)
        cols[t] = (int)(((mix(t + salt) & 0xffffffffull) * n) >> 32);
}

__global__ void flush_kernel(float* f, int64_t n, float v) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) f[t] = v;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t m = 100000000u, tile_rows = m / 8, ndest = 1u << 21;
    const int64_t E = 2621440;
    float *r, *G, *P, *fl, *out;
    Entry* e;
    CK(cudaMalloc(&r, (size_t)m * 4));
    CK(cudaMemset(r, 0, (size_t)m * 4));
    CK(cudaMalloc(&G, ndest * 4));
    CK(cudaMalloc(&P, (size_t)21000000 * 4));
    CK(cudaMalloc(&e, E * sizeof(Entry)));
    CK(cudaMalloc(&out, 4));
    const int64_t fln = 64ll << 20;
    CK(cudaMalloc(&fl, fln * 4));
    make_entries<<<sms * 4, 256>>>(e, E, tile_rows, ndest, 7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, bool cold, auto&& launch) {
        float best = 1e30f;
        for (int t = 0; t < 5; ++t) {
            if (cold) flush_kernel<<<sms * 4, 512>>>(fl, fln, (float)t);
            else launch();  // warm the tile
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("{\"bench\": \"%s\", \"cold\": %d, \"entries\": %lld, \"us\": %.2f, \"Gentries_per_s\": %.1f}\n", name,
               (int)cold, (long long)E, best * 1e3, E / (best * 1e6));
    };
    for (int cold : {1, 0}) {
        timeit("gather_only", cold, [&] { gather_only<<<sms * 4, 512>>>(r, e, E, out); });
        timeit("red_slot", cold, [&] { red_slot<<<sms * 4, 512>>>(r, e, E, G); });
        timeit("st_pos", cold, [&] { st_pos<<<sms * 4, 512>>>(r, e, E, P, 21000000u); });
    }
    // bin pass over 262144 random columns of a 5e8-column packed matrix (64 GB of blocks is too
    // much for a microbenchmark: use 1e8 columns = 12.8 GB)
    const int64_t n = 100000000, k = 262144;
    int4* blocks;
    int* cols;
    Entry* bins;
    unsigned long long* fill;
    CK(cudaMalloc(&blocks, (size_t)n * 8 * 16));
    make_blocks<<<sms * 8, 256>>>(blocks, n, m);
    CK(cudaMalloc(&cols, k * 4));
    make_cols<<<sms, 256>>>(cols, k, (uint32_t)n, 3);
    const int64_t cap = 1 << 20;
    CK(cudaMalloc(&bins, kTiles * cap * sizeof(Entry)));
    CK(cudaMalloc(&fill, kTiles * 8));
    int shift = 0;
    while ((m >> shift) > (uint32_t)kTiles - 1 && (1u << shift) * kTiles < m) ++shift;
    timeit("bin_pass_262k_cols", true, [&] {
        cudaMemsetAsync(fill, 0, kTiles * 8);
        bin_pass<<<sms * 4, 256>>>(blocks, cols, k, shift, bins, cap, fill);
    });
    unsigned long long hf[kTiles];
    CK(cudaMemcpy(hf, fill, sizeof hf, cudaMemcpyDeviceToHost));
    printf("{\"bench\": \"bin_fill\", \"shift\": %d, \"fill\": [%llu, %llu, %llu, %llu, %llu, %llu, %llu, %llu]}\n", shift,
           hf[0], hf[1], hf[2], hf[3], hf[4], hf[5], hf[6], hf[7]);
    return 0;
}
