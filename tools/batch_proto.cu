// batch_proto.cu -- prototype of the batched-snapshot partial-gradient pass for `huge`.
//
// Question: the huge iteration is bound by random 128-byte line fills of r
// (2.6 M random 4-byte gathers per iteration over a 400 MB r, ~3 sectors each).
// If the gathers of B iterations are computed from one snapshot r_0 (the
// synchronous PCDM1 g_i = a_i^T r_k = a_i^T r_0 + a_i^T (r_k - r_0), the second
// term only on rows dirtied inside the batch), they can be partitioned by row
// bins and swept in row order, so every r line is fetched once per batch.
// This measures, on huge-shaped data:
//   direct : the current layout, one G=8 group per slot: block line + 10 random r gathers
//   hdr    : block line + g0[s] only (the per-iteration pass left once g0 is known)
//   expand : pass 1, block line -> (bin, q) regions of 8-byte entries (row_local|slot_local, val)
//   sweepR : pass 2, bin-major sweep of the regions, g0 accumulated with red.global.add.f32
//   sweepS : pass 2, CTA owns NQ slot ranges, g0 accumulated in shared memory
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/batch_proto tools/batch_proto.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

constexpr int G = 8;
constexpr int NNZ = 10;
constexpr int RB = 21;  // rows per bin = 2^21
constexpr int CQ_LOG = 11;
constexpr int CQ = 1 << CQ_LOG;  // slots per range

__device__ __forceinline__ uint64_t mix(uint64_t h) {
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    h *= 0x94D049BB133111EBull;
    h ^= h >> 32;
    return h;
}

__global__ void make_blocks(int4* blocks, int64_t ncols, uint32_t m) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < ncols * G; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / G;
        const int t = (int)(q % G);
        int4 c = make_int4(0, 0, 0, 0);
        if (t == 0) {
            c = make_int4(__float_as_int(10.0f), NNZ, 0, 0);
        } else if (2 * (t - 1) < NNZ) {
            const uint64_t h = mix((uint64_t)q * 0x9E3779B97F4A7C15ull + 7);
            c.x = (int)(((h & 0xffffffffull) * m) >> 32);
            c.y = __float_as_int(((float)((h >> 40) & 0xffff) - 32768.f) / 32768.f);
            const uint64_t h2 = mix(h + 1);
            c.z = (int)(((h2 & 0xffffffffull) * m) >> 32);
            c.w = __float_as_int(((float)((h2 >> 40) & 0xffff) - 32768.f) / 32768.f);
        }
        blocks[q] = c;
    }
}

__global__ void make_r(float* r, int64_t m) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
        r[q] = (float)((mix(q) & 0xffff)) / 65536.f - 0.5f;
}

__global__ void make_slots(int* s, int64_t total, uint32_t ncols) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x)
        s[q] = (int)(((mix(q + 12345) & 0xffffffffull) * ncols) >> 32);
}

__device__ __forceinline__ int4 ldv4(const int4* p) {
    int4 v;
    asm volatile("ld.global.cg.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__global__ void __launch_bounds__(512) direct_kernel(const int4* blocks, const float* r, const int* S, int64_t total, float* g) {
    const int t = threadIdx.x & (G - 1);
    const unsigned gm = 0xffu << ((threadIdx.x & 31) & ~(G - 1));
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
    const int p0 = 2 * (t - 1);
    for (int64_t j = gid; j < total; j += ng) {
        const int i = __ldg(S + j);
        const int4 c = ldv4(blocks + (int64_t)i * G + t);
        float acc = 0.f;
        if (t > 0) {
            const float ra = p0 < NNZ ? __ldcg(r + c.x) : 0.f;
            const float rb = p0 + 1 < NNZ ? __ldcg(r + c.z) : 0.f;
            acc = fmaf(__int_as_float(c.y), ra, __int_as_float(c.w) * rb);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gm, acc, o);
        if (t == 0) g[j] = acc;
    }
}

__global__ void __launch_bounds__(512) hdr_kernel(const int4* blocks, const float* g0, const int* S, int64_t total, float* out) {
    const int t = threadIdx.x & (G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
    for (int64_t j = gid; j < total; j += ng) {
        const int i = __ldg(S + j);
        const int4 c = ldv4(blocks + (int64_t)i * G + t);
        if (t == 0) out[j] = __ldcg(g0 + j) * __int_as_float(c.x) + __int_as_float(c.z);
    }
}

// pass 1: CTA per slot range q (CQ slots); entries of bin b go to region (b*nq + q)*cap.
__global__ void __launch_bounds__(512) expand_kernel(const int4* blocks, const int* S, int nq, int nb, int cap,
                                                      int2* ent, int* cnt, int* spill_n, int4* spill) {
    __shared__ int c_s[64];
    const int t = threadIdx.x & (G - 1);
    const int grp = threadIdx.x / G;
    const int p0 = 2 * (t - 1);
    for (int q = blockIdx.x; q < nq; q += gridDim.x) {
        if (threadIdx.x < 64) c_s[threadIdx.x] = 0;
        __syncthreads();
        for (int sl = grp; sl < CQ; sl += 512 / G) {
            const int i = __ldg(S + (int64_t)q * CQ + sl);
            const int4 c = ldv4(blocks + (int64_t)i * G + t);
            if (t > 0) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (p0 + h < NNZ) {
                        const int row = h ? c.z : c.x;
                        const int v = h ? c.w : c.y;
                        const int b = row >> RB;
                        const int pos = atomicAdd(&c_s[b], 1);
                        const int key = (row & ((1 << RB) - 1)) | (sl << RB);
                        if (pos < cap) {
                            ent[((int64_t)b * nq + q) * cap + pos] = make_int2(key, v);
                        } else {
                            const int z = atomicAdd(spill_n, 1);
                            spill[z] = make_int4(row, v, q * CQ + sl, 0);
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < nb) cnt[threadIdx.x * nq + q] = min(c_s[threadIdx.x], cap);
        __syncthreads();
    }
}

__device__ __forceinline__ void red_add(float* p, float v) { asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory"); }

// pass 2 (global reds): bin-major sweep of all regions.
template <int U>
__global__ void __launch_bounds__(512) sweep_red_kernel(const int2* ent, const int* cnt, int nq, int nb, int cap, const float* r, float* g0) {
    const int64_t total = (int64_t)nb * nq * cap;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < total; base += stride * U) {
        float v[U];
        int dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = base + u * stride;
            dst[u] = -1;
            v[u] = 0.f;
            if (e < total) {
                const int64_t reg = e / cap;
                const int pos = (int)(e - reg * cap);
                if (pos < __ldg(cnt + reg)) {
                    const int2 x = __ldcs(ent + e);
                    const int b = (int)(reg / nq), q = (int)(reg - (int64_t)b * nq);
                    const int row = (b << RB) | (x.x & ((1 << RB) - 1));
                    v[u] = __int_as_float(x.y) * __ldcg(r + row);
                    dst[u] = q * CQ + ((unsigned)x.x >> RB);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (dst[u] >= 0) red_add(g0 + dst[u], v[u]);
    }
}

// pass 2 (shared accumulators): CTA owns NQ consecutive ranges.
template <int NQ>
__global__ void __launch_bounds__(1024) sweep_smem_kernel(const int2* ent, const int* cnt, int nq, int nb, int cap, const float* r, float* g0) {
    extern __shared__ float gs[];
    for (int q0 = blockIdx.x * NQ; q0 < nq; q0 += gridDim.x * NQ) {
        for (int u = threadIdx.x; u < NQ * CQ; u += blockDim.x) gs[u] = 0.f;
        __syncthreads();
        for (int b = 0; b < nb; ++b) {
#pragma unroll 1
            for (int u = 0; u < NQ; ++u) {
                const int q = q0 + u;
                if (q >= nq) break;
                const int64_t reg = (int64_t)b * nq + q;
                const int c = __ldg(cnt + reg);
                for (int pos = threadIdx.x; pos < c; pos += blockDim.x) {
                    const int2 x = __ldcs(ent + reg * cap + pos);
                    const int row = (b << RB) | (x.x & ((1 << RB) - 1));
                    atomicAdd(gs + u * CQ + ((unsigned)x.x >> RB), __int_as_float(x.y) * __ldcg(r + row));
                }
            }
        }
        __syncthreads();
        for (int u = threadIdx.x; u < NQ * CQ; u += blockDim.x)
            if (q0 * CQ + u < nq * CQ) g0[(int64_t)q0 * CQ + u] = gs[u];
        __syncthreads();
    }
}

__global__ void spill_kernel(const int4* spill, const int* spill_n, const float* r, float* g0) {
    const int n = *spill_n;
    for (int z = blockIdx.x * blockDim.x + threadIdx.x; z < n; z += gridDim.x * blockDim.x) {
        const int4 s = spill[z];
        red_add(g0 + s.z, __int_as_float(s.y) * __ldcg(r + s.x));
    }
}

__global__ void flush_kernel(float* f, int64_t n) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) f[q] += 1.f;
}

int main(int argc, char** argv) {
    const uint32_t m = 100000000u;
    const int64_t ncols = argc > 1 ? atoll(argv[1]) : 50000000ll;
    const int64_t tau = 1 << 18;
    const int B = argc > 2 ? atoi(argv[2]) : 8;
    const int64_t total = B * tau;
    const int nq = (int)(total / CQ);
    const int nb = (int)((m + (1u << RB) - 1) >> RB);
    const double expct = (double)CQ * NNZ / nb * ((double)(1u << RB) * nb / m);
    const int cap = (int)(expct + 8.0 * sqrt(expct) + 32) & ~31;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    printf("{\"m\": %u, \"ncols\": %lld, \"tau\": %lld, \"B\": %d, \"nq\": %d, \"nb\": %d, \"cap\": %d, \"expect\": %.1f}\n", m,
           (long long)ncols, (long long)tau, B, nq, nb, cap, expct);

    int4 *blocks, *spill;
    float *r, *g_dir, *g0, *out, *flush;
    int *S, *cnt, *spill_n;
    int2* ent;
    CK(cudaMalloc(&blocks, ncols * G * sizeof(int4)));
    CK(cudaMalloc(&r, (size_t)m * 4));
    CK(cudaMalloc(&S, total * 4));
    CK(cudaMalloc(&g_dir, total * 4));
    CK(cudaMalloc(&g0, total * 4));
    CK(cudaMalloc(&out, total * 4));
    CK(cudaMalloc(&ent, (size_t)nb * nq * cap * sizeof(int2)));
    CK(cudaMalloc(&cnt, (size_t)nb * nq * 4));
    CK(cudaMalloc(&spill_n, 4));
    CK(cudaMalloc(&spill, (size_t)1 << 24));
    const int64_t nflush = 64ll << 20;
    CK(cudaMalloc(&flush, nflush * 4));
    make_blocks<<<sms * 16, 256>>>(blocks, ncols, m);
    make_r<<<sms * 16, 256>>>(r, m);
    make_slots<<<sms * 16, 256>>>(S, total, (uint32_t)ncols);
    CK(cudaDeviceSynchronize());

    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](const char* name, auto&& fn, int reps) {
        std::vector<float> ts;
        for (int k = 0; k < reps; ++k) {
            flush_kernel<<<sms * 8, 256>>>(flush, nflush);
            CK(cudaEventRecord(e0));
            fn();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        printf("{\"kernel\": \"%s\", \"ms_median\": %.4f, \"ms_best\": %.4f, \"us_per_iter\": %.2f}\n", name, ts[reps / 2],
               ts[0], 1000.0 * ts[reps / 2] / B);
        return ts[reps / 2];
    };
    const int reps = 7;
    timeit("direct", [&] { direct_kernel<<<sms * 3, 512>>>(blocks, r, S, total, g_dir); }, reps);
    timeit("hdr", [&] { hdr_kernel<<<sms * 3, 512>>>(blocks, g_dir, S, total, out); }, reps);
    timeit("expand", [&] {
        cudaMemsetAsync(spill_n, 0, 4);
        expand_kernel<<<sms * 3, 512>>>(blocks, S, nq, nb, cap, ent, cnt, spill_n, spill);
    }, reps);
    int hsp = 0;
    CK(cudaMemcpy(&hsp, spill_n, 4, cudaMemcpyDeviceToHost));
    printf("{\"spill\": %d}\n", hsp);
    std::vector<float> a(total), b(total);
    CK(cudaMemcpy(a.data(), g_dir, total * 4, cudaMemcpyDeviceToHost));
    auto check = [&](const char* name) {
        CK(cudaMemcpy(b.data(), g0, total * 4, cudaMemcpyDeviceToHost));
        double worst = 0;
        for (int64_t j = 0; j < total; ++j) worst = std::max(worst, (double)fabsf(a[j] - b[j]) / (1e-3 + fabsf(a[j])));
        printf("{\"check\": \"%s\", \"max_rel\": %.3g}\n", name, worst);
    };
    timeit("sweepR_u4", [&] {
        cudaMemsetAsync(g0, 0, total * 4);
        sweep_red_kernel<4><<<sms * 4, 512>>>(ent, cnt, nq, nb, cap, r, g0);
        spill_kernel<<<sms, 256>>>(spill, spill_n, r, g0);
    }, reps);
    check("sweepR_u4");
    timeit("sweepR_u8", [&] {
        cudaMemsetAsync(g0, 0, total * 4);
        sweep_red_kernel<8><<<sms * 4, 512>>>(ent, cnt, nq, nb, cap, r, g0);
        spill_kernel<<<sms, 256>>>(spill, spill_n, r, g0);
    }, reps);
    check("sweepR_u8");
    {
        constexpr int NQ = 6;
        CK(cudaFuncSetAttribute(sweep_smem_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, NQ * CQ * 4));
        const int ctas = (nq + NQ - 1) / NQ;
        timeit("sweepS_nq6", [&] {
            sweep_smem_kernel<NQ><<<ctas, 1024, NQ * CQ * 4>>>(ent, cnt, nq, nb, cap, r, g0);
            spill_kernel<<<sms, 256>>>(spill, spill_n, r, g0);
        }, reps);
        check("sweepS_nq6");
    }
    {
        constexpr int NQ = 3;
        CK(cudaFuncSetAttribute(sweep_smem_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, NQ * CQ * 4));
        const int ctas = (nq + NQ - 1) / NQ;
        timeit("sweepS_nq3", [&] {
            sweep_smem_kernel<NQ><<<ctas, 1024, NQ * CQ * 4>>>(ent, cnt, nq, nb, cap, r, g0);
            spill_kernel<<<sms, 256>>>(spill, spill_n, r, g0);
        }, reps);
        check("sweepS_nq3");
    }
    return 0;
}
