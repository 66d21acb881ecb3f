// kernels_cluster.cu -- the PCDM1 loop for residuals that fit in one thread-block
// cluster's distributed shared memory (CLUSTER variant; e.g. `medium`, m = 1e5).
//
// Why: for small tau the synchronous iteration (alg:PCD1) is
// bound by the latency of its barriers and of the dependent L2 round trips, not
// by bytes (medium: 1024 columns x 20 entries per iteration, r = 400 KB).  A grid
// barrier over global memory costs ~1.5-2 us; the hardware cluster barrier
// (barrier.cluster) a few hundred cycles.  So one cluster of up to 16 CTAs runs
// the whole iteration: r is split row-wise over the CTAs' shared memories,
// gathers g_i = a_i^T r_k are distributed-shared-memory loads (~200 cycles),
// and the synchronous semantics come from two cluster barriers per iteration:
//
//   phase A  every sampled column: g_i from r_k (DSMEM), soft-threshold step
//            (eq:h(x) block form) in registers, x_i updated,
//            nonzero steps listed in the CTA's shared memory      | cluster barrier
//   phase B  r += delta_i a_i for the listed steps (DSMEM red.add) | cluster barrier
//
// The packed column blocks (kernels_packed.cu) come from L2/HBM; the next
// iteration's first slot id and block are loaded during phase B.  r is loaded
// from global memory at launch start and written back at launch end.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;
using namespace pcdm;
using namespace pcdm_internal;

namespace {

constexpr int kThreads = 1024;

__device__ __forceinline__ int4 ld_stream_v4(const int4* p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

template <int G>
__device__ __forceinline__ unsigned gmask_of() {
    if constexpr (G == 32) {
        return 0xffffffffu;
    } else {
        const unsigned lane = threadIdx.x & 31;
        return ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
    }
}

__device__ __forceinline__ int real_row(int v, const int* hrow) { return v < 0 ? hrow[v & 0x7fffffff] : v; }

// Dynamic shared memory: r slice f32[rpc] | hot-row ids int[nhot] | step list {i, d}[list_cap]
template <int G, bool LOGISTIC>
__global__ void __launch_bounds__(kThreads, 1) pcdm_cluster_kernel(ClusterParams P) {
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    const unsigned csize = cluster.num_blocks();
    extern __shared__ float s_r[];
    int* s_hrow = (int*)(s_r + P.rpc);
    int2* s_list = (int2*)(s_hrow + P.nhot + (P.nhot & 1));
    __shared__ int s_cnt;
    __shared__ unsigned long long s_nz;

    const int t = threadIdx.x & (G - 1);
    const unsigned gm = gmask_of<G>();
    const int src = (threadIdx.x & 31) & ~(G - 1);
    const int grp = threadIdx.x / G;
    const int64_t gid = ((int64_t)rank * kThreads + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)csize * kThreads) / G;
    const int pair0 = 2 * (t - 1);
    const int64_t tau = P.tau;
    const int rpc = P.rpc;

    // this CTA's rows [rank * rpc, (rank+1) * rpc) of r
    const int64_t row0 = (int64_t)rank * rpc;
    for (int q = threadIdx.x; q < rpc; q += kThreads) s_r[q] = row0 + q < P.m ? P.r[row0 + q] : 0.0f;
    for (int h = threadIdx.x; h < P.nhot; h += kThreads) s_hrow[h] = P.hot_rows[h];
    if (threadIdx.x == 0) {
        s_cnt = 0;
        s_nz = 0;
    }
    cluster.sync();

    // r[row] in the owning CTA's shared memory
    auto rptr = [&](int row) -> float* {
        const unsigned owner = (unsigned)row / (unsigned)rpc;
        return cluster.map_shared_rank(s_r + (row - (int)owner * rpc), owner);
    };

    // first slot of each group, loaded one iteration ahead
    int i_pf = -1;
    int4 c_pf = make_int4(0, 0, 0, 0);
    auto prefetch = [&](int64_t it) {
        i_pf = -1;
        if (it < P.iters && gid < tau) {
            i_pf = ld_stream_s32(P.slots + it * tau + gid);
            if (i_pf >= 0) c_pf = ld_stream_v4(P.blocks + (int64_t)i_pf * G + t);
        }
    };
    prefetch(0);

    for (int64_t it = 0; it < P.iters; ++it) {
        const int* S = P.slots + it * tau;
        // ---------------- phase A: gathers from r_k (distributed shared memory), steps
        for (int64_t j = gid; j < tau; j += ngroups) {
            int i;
            int4 c;
            if (j == gid) {
                i = i_pf;
                c = c_pf;
            } else {
                i = ld_stream_s32(S + j);
                if (i >= 0) c = ld_stream_v4(P.blocks + (int64_t)i * G + t);
            }
            if (i < 0) continue;
            float xi = 0.0f;
            if (t == 0) xi = P.xlist ? ld_l2_f32((const float*)(P.blocks + (int64_t)i * G) + 2) : ld_l2_f32(P.x + i);
            const int len = __shfl_sync(gm, c.y, src);
            float acc = 0.0f;
            if (t > 0) {
                const float ra = pair0 < len ? grad_weight<LOGISTIC>(*rptr(real_row(c.x, s_hrow))) : 0.0f;
                const float rb = pair0 + 1 < len ? grad_weight<LOGISTIC>(*rptr(real_row(c.z, s_hrow))) : 0.0f;
                acc = fmaf(__int_as_float(c.y), ra, __int_as_float(c.w) * rb);
            }
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gm, acc, o);
            if (t == 0) {
                const float xp = block_step<LOGISTIC>(xi, acc, P.beta * __int_as_float(c.x), P.lambda);
                const float d = xp - xi;
                if (d != 0.0f) {
                    if (!isfinite(xp)) atomicOr(P.flags, FLAG_DIVERGED);
                    if (P.xlist) {
                        ((float*)(P.blocks + (int64_t)i * G))[2] = xp;
                        if (P.xlist_cap > 0) {  // 0: dense iterate, no dirty list
                            const unsigned long long q = atomicAdd(P.xlist_count, 1ull);
                            if (q < (unsigned long long)P.xlist_cap) P.xlist[q] = i;
                        }
                    } else {
                        P.x[i] = xp;
                    }
                    // list_cap >= the slots a CTA handles per iteration: never full
                    s_list[atomicAdd(&s_cnt, 1)] = make_int2(i, __float_as_int(d));
                }
            }
        }
        cluster.sync();
        // ---------------- phase B: r += delta a_i for this CTA's steps; next slot prefetched
        prefetch(it + 1);
        const int cnt = s_cnt;
        for (int e = grp; e < cnt; e += kThreads / G) {
            const int2 st = s_list[e];
            const float d = __int_as_float(st.y);
            const int4 c = ld_stream_v4(P.blocks + (int64_t)st.x * G + t);
            const int len = __shfl_sync(gm, c.y, src);
            if (t > 0 && pair0 < len) atomicAdd(rptr(real_row(c.x, s_hrow)), __int_as_float(c.y) * d);
            if (t > 0 && pair0 + 1 < len) atomicAdd(rptr(real_row(c.z, s_hrow)), __int_as_float(c.w) * d);
        }
        cluster.sync();
        if (threadIdx.x == 0) {
            s_nz += (unsigned long long)cnt;
            s_cnt = 0;
        }
        __syncthreads();  // the reset before the next iteration's appends
    }
    for (int q = threadIdx.x; q < rpc; q += kThreads)
        if (row0 + q < P.m) P.r[row0 + q] = s_r[q];
    if (threadIdx.x == 0 && s_nz) atomicAdd(P.nz_total, s_nz);
}

template <int G, bool LOG>
const void* kfn() {
    return (const void*)pcdm_cluster_kernel<G, LOG>;
}

template <bool LOG>
const void* kfn_g(int G) {
    switch (G) {
        case 2: return kfn<2, LOG>();
        case 4: return kfn<4, LOG>();
        case 8: return kfn<8, LOG>();
        case 16: return kfn<16, LOG>();
        default: return kfn<32, LOG>();
    }
}

}  // namespace

namespace pcdm_internal {

size_t cluster_smem_bytes(int rpc, int nhot, int list_cap) {
    return (size_t)rpc * sizeof(float) + (size_t)(nhot + (nhot & 1)) * sizeof(int) + (size_t)list_cap * sizeof(int2);
}

// Largest usable cluster size (16 if the device allows non-portable clusters, else 8)
// for this kernel with `smem` bytes of dynamic shared memory; 0 if none fits.
int cluster_plan(int G, bool logistic, size_t smem, int want) {
    const void* fn = logistic ? kfn_g<true>(G) : kfn_g<false>(G);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaGetLastError();
    for (int cs = want; cs >= 1; cs >>= 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) == cudaSuccess && nclusters >= 1) return cs;
        cudaGetLastError();
    }
    return 0;
}

cudaError_t launch_cluster(int G, int cs, const ClusterParams& P, size_t smem, cudaStream_t st, int64_t* launches) {
    const void* fn = P.logistic ? kfn_g<true>(G) : kfn_g<false>(G);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {(void*)&P};
    ++*launches;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace pcdm_internal
