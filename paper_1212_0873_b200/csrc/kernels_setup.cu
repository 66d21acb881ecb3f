// kernels_setup.cu -- create-time and occasional kernels of libpcdm:
//   CSC validation, row histogram + omega, column norms
//   L_i = ||a_i||^2, residual r = Ax - b (fp64 scratch), and
//   the objective F = 1/2||r||^2 + lambda||x||_1 (eq:P).
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

using namespace pcdm;
using pcdm_internal::DevCSR;
using pcdm_internal::XHeaders;

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t work, int per_block, int max_blocks) {
    int64_t b = (work + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (int)b;
}

// Hot rows (packed loop, kernels_packed.cu): rows stored >= threshold times are
// appended (row, count) to a candidate list of capacity cap (n_out counts all).
__global__ void hot_candidates_kernel(int64_t m, const int* __restrict__ counts, int threshold, int* __restrict__ rows,
                                      int* __restrict__ cnts, int* __restrict__ n_out, int cap) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        const int c = counts[j];
        if (c >= threshold) {
            const int q = atomicAdd(n_out, 1);
            if (q < cap) {
                rows[q] = (int)j;
                cnts[q] = c;
            }
        }
    }
}

// Column tiles: a warp takes 32 consecutive columns and walks their entries
// [colptr[i0], colptr[i0 + 32]) with all lanes, coalesced (a warp per column leaves 22
// of 32 lanes idle on 10-entry columns and is latency-bound).  tile_bounds loads the 33
// boundaries (lane l holds b_l = colptr[i0 + l], lane 0 also b_32 in *b32);
// tile_col finds the tile-local column of entry p: the largest k with b_k <= p.
__device__ __forceinline__ long long tile_bounds(const long long* __restrict__ colptr, int64_t n, int64_t i0,
                                                 long long* b32) {
    const int lane = threadIdx.x & 31;
    const int64_t i = i0 + lane;
    const long long b = colptr[i < n ? i : n];
    *b32 = colptr[i0 + 32 < n ? i0 + 32 : n];
    return b;
}
__device__ __forceinline__ int tile_col(long long p, long long b) {
    int k = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
        const long long bk = __shfl_sync(0xffffffffu, b, k + step);
        if (bk <= p) k += step;
    }
    return k;
}

// L_i = sum_p val_p^2 on column tiles: fp64 segmented warp sums (entries of a column are
// consecutive lanes), one fp64 accumulator per tile column in shared memory (acc[32]).
__device__ __forceinline__ void tile_norms_scan(const float* __restrict__ val, int64_t n, int64_t i0, long long b,
                                                long long e32, double* acc, float* __restrict__ L) {
    const int lane = threadIdx.x & 31;
    acc[lane] = 0.0;
    __syncwarp();
    const long long s = __shfl_sync(0xffffffffu, b, 0);
    for (long long p0 = s; p0 < e32; p0 += 32) {
        const long long p = p0 + lane;
        const bool valid = p < e32;
        const double v = valid ? (double)ld_stream_f32(val + p) : 0.0;
        const int kt = tile_col(p, b);  // all lanes (shuffles)
        const int k = valid ? kt : 32;
        double sum = v * v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // segmented inclusive scan (keys non-decreasing)
            const double y = __shfl_up_sync(0xffffffffu, sum, o);
            const int ky = __shfl_up_sync(0xffffffffu, k, o);
            if (lane >= o && ky == k) sum += y;
        }
        const int kn = __shfl_down_sync(0xffffffffu, k, 1);
        if (valid && (lane == 31 || kn != k)) acc[k] += sum;  // the segment's last lane
        __syncwarp();
    }
    if (i0 + lane < n) L[i0 + lane] = (float)acc[lane];
    __syncwarp();
}

__global__ void col_norms_tile_kernel(int64_t n, const long long* __restrict__ colptr, const float* __restrict__ val,
                                      float* __restrict__ L) {
    __shared__ double s_acc[kThreads];
    double* acc = s_acc + (threadIdx.x & ~31);
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i0 = warp * 32; i0 < n; i0 += nwarps * 32) {
        long long e32;
        const long long b = tile_bounds(colptr, n, i0, &e32);
        tile_norms_scan(val, n, i0, b, e32, acc, L);
    }
}

// CSC validation on column tiles: colptr monotone and within [0, nnz], rows in [0, m)
// and strictly increasing within a column, values finite.
__global__ void validate_tile_kernel(int64_t m, int64_t n, int64_t nnz, const long long* __restrict__ colptr,
                                     const int* __restrict__ rowidx, const float* __restrict__ val,
                                     int* __restrict__ flags, float* __restrict__ L) {
    __shared__ double s_acc[kThreads];
    double* acc = s_acc + (threadIdx.x & ~31);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int bad = 0;
    if (warp == 0 && lane == 0 && (colptr[0] != 0 || colptr[n] != nnz)) bad |= FLAG_BAD_COLPTR;
    for (int64_t i0 = warp * 32; i0 < n; i0 += nwarps * 32) {
        long long e32;
        const long long b = tile_bounds(colptr, n, i0, &e32);
        const long long bn = __shfl_down_sync(0xffffffffu, b, 1);
        const long long next = lane == 31 ? e32 : bn;
        const bool col_ok = next >= b && b >= 0 && next <= nnz;
        if (!__all_sync(0xffffffffu, col_ok)) {
            bad |= FLAG_BAD_COLPTR;
            continue;
        }
        const long long s = __shfl_sync(0xffffffffu, b, 0);
        for (long long p0 = s; p0 < e32; p0 += 32) {  // all lanes (tile_col shuffles)
            const long long p = p0 + lane;
            const int k = tile_col(p, b);
            const bool start = __shfl_sync(0xffffffffu, b, k) == p;  // first entry of its column
            if (p < e32) {
                const int r = rowidx[p];
                if (r < 0 || (int64_t)r >= m) bad |= FLAG_BAD_ROW;
                if (!start && rowidx[p - 1] >= r) bad |= FLAG_ROW_ORDER;
                if (!isfinite(val[p])) bad |= FLAG_NONFINITE_VAL;
            }
        }
        if (L) {
            // L_i = sum val^2 (fp64) of the tile's columns, read again while the tile is in
            // L2: a lane per column when the tile's columns are short (no shuffles), the
            // segmented warp scan otherwise
            const int len = (int)min(next - b, (long long)INT_MAX);
            if (__reduce_max_sync(0xffffffffu, len) <= 64) {
                double sum = 0.0;
                for (long long p = b; p < next; ++p) {
                    const double v = (double)val[p];
                    sum = fma(v, v, sum);
                }
                if (i0 + lane < n) L[i0 + lane] = (float)sum;
            } else {
                tile_norms_scan(val, n, i0, b, e32, acc, L);
            }
        }
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicOr(flags, bad);
}

// counts[row]++ restricted to rows in [lo, hi): the row range's counters stay in L2
// while every pass streams the whole row-index array (16-byte loads).
__global__ void row_counts_range_kernel(int64_t nnz, const int* __restrict__ rowidx, int lo, int hi,
                                        int* __restrict__ counts) {
    const int64_t nv = nnz / 4;
    const int4* r4 = (const int4*)rowidx;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nv; q += (int64_t)gridDim.x * blockDim.x) {
        int4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(r4 + q));
        if (v.x >= lo && v.x < hi) atomicAdd(counts + v.x, 1);
        if (v.y >= lo && v.y < hi) atomicAdd(counts + v.y, 1);
        if (v.z >= lo && v.z < hi) atomicAdd(counts + v.z, 1);
        if (v.w >= lo && v.w < hi) atomicAdd(counts + v.w, 1);
    }
    for (int64_t p = nv * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int r = rowidx[p];
        if (r >= lo && r < hi) atomicAdd(counts + r, 1);
    }
}

// Byte counters: counts of rows [lo, hi) as 8-bit fields of 32-bit words (4 rows per word,
// a 2^26-row range in 64 MB of L2), atomicAdd of 1 << 8 (r & 3); a field that was 255
// before the add has carried into its neighbour: *overflow is set and the caller recounts
// with 32-bit counters (a row with more than 255 stored entries).
__global__ void row_counts_u8_kernel(int64_t nnz, const int* __restrict__ rowidx, int lo, int hi,
                                     unsigned* __restrict__ words, int* __restrict__ overflow) {
    const int64_t nv = nnz / 4;
    const int4* r4 = (const int4*)rowidx;
    bool ovf = false;
    auto count = [&](int r) {
        if (r >= lo && r < hi) {
            const int q = r - lo;
            const unsigned sh = 8u * (unsigned)(q & 3);
            const unsigned old = atomicAdd(words + (q >> 2), 1u << sh);
            ovf |= ((old >> sh) & 0xFFu) == 0xFFu;
        }
    };
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nv; q += (int64_t)gridDim.x * blockDim.x) {
        int4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(r4 + q));
        count(v.x);
        count(v.y);
        count(v.z);
        count(v.w);
    }
    for (int64_t p = nv * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
         p += (int64_t)gridDim.x * blockDim.x)
        count(rowidx[p]);
    if (__any_sync(0xffffffffu, ovf) && (threadIdx.x & 31) == 0) atomicExch(overflow, 1);
}

// counts[lo + t] = byte t of the range's words
__global__ void row_counts_expand_kernel(int lo, int cnt, const unsigned* __restrict__ words, int* __restrict__ counts) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x)
        counts[lo + t] = (int)((words[t >> 2] >> (8u * (unsigned)(t & 3))) & 0xFFu);
}

__global__ void check_finite_kernel(int64_t count, const float* __restrict__ v, int flag_bit,
                                    int* __restrict__ flags) {
    int bad = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(v[t])) bad = flag_bit;
    bad = __reduce_or_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(flags, bad);
}

// counts[row]++ for every stored entry; warp-aggregated for hot rows.
__global__ void row_counts_kernel(int64_t nnz, const int* __restrict__ rowidx, int* __restrict__ counts) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int r = ld_stream_s32(rowidx + p);
        const unsigned active = __activemask();
        const unsigned peers = __match_any_sync(active, r);
        const int leader = __ffs(peers) - 1;
        if ((threadIdx.x & 31) == leader) atomicAdd(counts + r, __popc(peers));
    }
}

__global__ void max_kernel(int64_t count, const int* __restrict__ v, int* __restrict__ out) {
    int best = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x)
        best = max(best, v[t]);
    best = __reduce_max_sync(0xffffffffu, best);
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

__global__ void neg_b_kernel(int64_t m, const float* __restrict__ b, double* __restrict__ r64) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x)
        r64[t] = -(double)b[t];
}

// r64 += x_i a_i for x_i != 0; also flags non-finite x.  One pass over x with
// 16-byte loads (x is read in full every run; its support is usually small), a
// thread per 4 columns for the (rare) nonzero ones.
__device__ __forceinline__ void scatter_col(int64_t i, float xi, const long long* __restrict__ colptr,
                                            const int* __restrict__ rowidx, const float* __restrict__ val,
                                            double* __restrict__ r64, int& bad, const XHeaders& xh) {
    if (xi == 0.0f) return;
    if (!isfinite(xi)) {
        bad = FLAG_NONFINITE_X;
        return;
    }
    if (xh.blocks) {
        ((float*)(xh.blocks + (xh.off ? xh.off[i] : i * xh.G)))[2] = xi;
        if (xh.cap > 0) {  // 0: dense iterate, no dirty list
            const unsigned long long q = atomicAdd(xh.count, 1ull);
            if (q < (unsigned long long)xh.cap) xh.list[q] = (int)i;
        }
    }
    if (!colptr) return;
    const double xd = (double)xi;
    for (long long p = colptr[i]; p < colptr[i + 1]; ++p) atomicAdd(r64 + rowidx[p], (double)val[p] * xd);
}

// Row-major residual (dense iterates, e.g. the logistic margins): one warp per row,
// r64_j = -b_j + sum_{(j,i) stored} a_ji x_i in fp64 registers, no atomics.
__global__ void residual_rows_kernel(int64_t m, const long long* __restrict__ rowptr, const int* __restrict__ ccol,
                                     const float* __restrict__ cval, const float* __restrict__ b,
                                     const float* __restrict__ x, double* __restrict__ r64) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < m; j += nw) {
        const long long s = rowptr[j], e = rowptr[j + 1];
        double acc = 0.0;
        for (long long q = s + lane; q < e; q += 32) acc += (double)cval[q] * (double)__ldg(x + ccol[q]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) r64[j] = acc - (double)b[j];
    }
}

// CSR fill: entry (i, row, val) goes to the next free position of its row
__global__ void csr_fill_kernel(int64_t n, const long long* __restrict__ colptr, const int* __restrict__ rowidx,
                                const float* __restrict__ val, unsigned long long* __restrict__ cursor,
                                int* __restrict__ ccol, float* __restrict__ cval) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
        for (long long p = colptr[i] + lane; p < colptr[i + 1]; p += 32) {
            const unsigned long long pos = atomicAdd(cursor + rowidx[p], 1ull);
            ccol[pos] = (int)i;
            cval[pos] = val[p];
        }
    }
}

__global__ void counts64_kernel(int64_t m, const int* __restrict__ counts, unsigned long long* __restrict__ out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= m; j += (int64_t)gridDim.x * blockDim.x)
        out[j] = j < m ? (unsigned long long)counts[j] : 0ull;
}

// scatter = false: only the header copy / dirty list / non-finite check (the row-major
// residual below computes r64 without atomics)
__global__ void scatter_x_kernel(int64_t n, const long long* __restrict__ colptr,
                                 const int* __restrict__ rowidx, const float* __restrict__ val,
                                 const float* __restrict__ x, double* __restrict__ r64,
                                 int* __restrict__ flags, XHeaders xh, bool scatter) {
    if (!scatter) colptr = nullptr;
    int bad = 0;
    const int64_t n4 = ((uintptr_t)x % 16 == 0) ? n / 4 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
        const float4 v = __ldcs((const float4*)x + q);
        if (v.x != 0.0f || v.y != 0.0f || v.z != 0.0f || v.w != 0.0f) {
            scatter_col(4 * q, v.x, colptr, rowidx, val, r64, bad, xh);
            scatter_col(4 * q + 1, v.y, colptr, rowidx, val, r64, bad, xh);
            scatter_col(4 * q + 2, v.z, colptr, rowidx, val, r64, bad, xh);
            scatter_col(4 * q + 3, v.w, colptr, rowidx, val, r64, bad, xh);
        }
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        scatter_col(i, x[i], colptr, rowidx, val, r64, bad, xh);
    bad = __reduce_or_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(flags, bad);
}

// r = (float) r64; also into r2 (the one-barrier loop's second buffer) and zeroes
// zero[0 .. nzero) when given
__global__ void round_r_kernel(int64_t m, const double* __restrict__ r64, float* __restrict__ r,
                               float* __restrict__ r2, int* __restrict__ zero, int nzero) {
    if (zero && blockIdx.x == 0 && threadIdx.x < nzero) zero[threadIdx.x] = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x) {
        const float v = (float)r64[t];
        r[t] = v;
        if (r2) r2[t] = v;
    }
}

// out[0] += sum r64^2 ; out[1] += sum |x|
__global__ void objective_sums_kernel(int64_t m, int64_t n, const double* __restrict__ r64,
                                      const float* __restrict__ x, double* __restrict__ out) {
    double s2 = 0.0, s1 = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += stride)
        s2 += r64[t] * r64[t];
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride)
        s1 += fabs((double)x[t]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    __shared__ double sh[2][32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sh[0][w] = s2;
        sh[1][w] = s1;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        s2 = lane < nw ? sh[0][lane] : 0.0;
        s1 = lane < nw ? sh[1][lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        if (lane == 0) {
            atomicAdd(out, s2);
            atomicAdd(out + 1, s1);
        }
    }
}

// L2-regularised logistic problem: labels must be +-1; A~ = diag(y) A in place.
__global__ void check_labels_kernel(int64_t m, const float* __restrict__ y, int* __restrict__ flags) {
    int bad = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
        if (!(y[t] == 1.0f || y[t] == -1.0f)) bad = FLAG_NONFINITE_B;
    bad = __reduce_or_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(flags, bad);
}

__global__ void fold_labels_kernel(int64_t nnz, const int* __restrict__ rowidx, const float* __restrict__ y,
                                   float* __restrict__ val) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
        val[p] *= y[rowidx[p]];
}

__global__ void scale_kernel(int64_t n, float a, float* __restrict__ v) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        v[t] *= a;
}

// out[0] += sum log(1 + exp(-s_j)) (fp64, stable), out[1] += sum x_i^2
__global__ void objective_logistic_kernel(int64_t m, int64_t n, const double* __restrict__ s64,
                                          const float* __restrict__ x, double* __restrict__ out) {
    double a = 0.0, q = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += stride) {
        const double v = s64[t];
        a += v >= 0.0 ? log1p(exp(-v)) : -v + log1p(exp(v));
    }
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const double xv = (double)x[t];
        q += xv * xv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, a);
        atomicAdd(out + 1, q);
    }
}

}  // namespace

namespace pcdm_internal {

cudaError_t launch_logistic_setup(int64_t m, int64_t nnz, const int* rowidx, const float* y, float* val, int* flags,
                                  cudaStream_t st, int sms, int64_t* launches) {
    check_labels_kernel<<<grid_for(m, kThreads, sms * 8), kThreads, 0, st>>>(m, y, flags);
    fold_labels_kernel<<<grid_for(nnz, kThreads, sms * 16), kThreads, 0, st>>>(nnz, rowidx, y, val);
    *launches += 2;
    return cudaGetLastError();
}

cudaError_t launch_scale(int64_t n, float a, float* v, cudaStream_t st, int sms, int64_t* launches) {
    scale_kernel<<<grid_for(n, kThreads, sms * 8), kThreads, 0, st>>>(n, a, v);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_objective_logistic(int64_t m, int64_t n, const double* s64, const float* x, double* out,
                                      cudaStream_t st, int sms, int64_t* launches) {
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(double), st);
    if (e != cudaSuccess) return e;
    objective_logistic_kernel<<<grid_for(m > n ? m : n, kThreads, sms * 4), kThreads, 0, st>>>(m, n, s64, x, out);
    ++*launches;
    return cudaGetLastError();
}


cudaError_t launch_validate(const DevCSC& A, int* flags, cudaStream_t st, int sms, int64_t* launches, float* L) {
    const int blocks = grid_for(A.n, kThreads, sms * 16);  // a warp per 32-column tile
    validate_tile_kernel<<<blocks, kThreads, 0, st>>>(A.m, A.n, A.nnz, (const long long*)A.colptr, A.rowidx,
                                                      A.val, flags, L);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_check_finite(int64_t count, const float* v, int flag_bit, int* flags, cudaStream_t st,
                                int sms, int64_t* launches) {
    const int blocks = grid_for(count, kThreads, sms * 8);
    check_finite_kernel<<<blocks, kThreads, 0, st>>>(count, v, flag_bit, flags);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_row_counts(const DevCSC& A, int* counts, cudaStream_t st, int sms, int64_t* launches) {
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int) * (size_t)A.m, st);
    if (e != cudaSuccess) return e;
    // counters of at most 2^24 rows (64 MB) per pass stay in L2 (huge: 189 -> see
    // profiles/r02_create_ab.jsonl); small m: one pass with warp-aggregated atomics
    const int64_t tile = (int64_t)1 << 24;
    if (A.m <= tile) {
        const int blocks = grid_for(A.nnz, kThreads, sms * 16);
        row_counts_kernel<<<blocks, kThreads, 0, st>>>(A.nnz, A.rowidx, counts);
        ++*launches;
        return cudaGetLastError();
    }
    const int blocks = grid_for(A.nnz / 4 + 1, kThreads, sms * 8);
    // byte counters first: 2^26 rows per pass (huge: 2 passes instead of 6; 53 -> see
    // profiles/r02_create_ab.txt), 32-bit counters again if a row overflowed a byte
    const int64_t tile8 = (int64_t)1 << 26;
    unsigned* words = nullptr;
    int* ovf = nullptr;
    if (cudaMalloc((void**)&words, sizeof(unsigned) * (size_t)(std::min(A.m, tile8) / 4 + 1) + 16) == cudaSuccess) {
        ovf = (int*)(words + std::min(A.m, tile8) / 4 + 1);
        int h_ovf = 0;
        e = cudaMemsetAsync(ovf, 0, sizeof(int), st);
        for (int64_t lo = 0; e == cudaSuccess && lo < A.m; lo += tile8) {
            const int cnt = (int)std::min(tile8, A.m - lo);
            e = cudaMemsetAsync(words, 0, sizeof(unsigned) * (size_t)(cnt / 4 + 1), st);
            if (e != cudaSuccess) break;
            row_counts_u8_kernel<<<blocks, kThreads, 0, st>>>(A.nnz, A.rowidx, (int)lo, (int)(lo + cnt), words, ovf);
            row_counts_expand_kernel<<<grid_for(cnt, kThreads, sms * 8), kThreads, 0, st>>>((int)lo, cnt, words, counts);
            *launches += 2;
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h_ovf, ovf, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        cudaFree(words);
        if (e != cudaSuccess) return e;
        if (!h_ovf) return cudaSuccess;
        if ((e = cudaMemsetAsync(counts, 0, sizeof(int) * (size_t)A.m, st)) != cudaSuccess) return e;
    } else {
        cudaGetLastError();  // no room for the byte counters: 32-bit passes
    }
    for (int64_t lo = 0; lo < A.m; lo += tile) {
        row_counts_range_kernel<<<blocks, kThreads, 0, st>>>(A.nnz, A.rowidx, (int)lo, (int)std::min(A.m, lo + tile),
                                                             counts);
        ++*launches;
    }
    return cudaGetLastError();
}

cudaError_t launch_hot_candidates(int64_t m, const int* counts, int threshold, int* rows, int* cnts, int* n_out,
                                  int cap, cudaStream_t st, int sms, int64_t* launches) {
    cudaError_t e = cudaMemsetAsync(n_out, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    hot_candidates_kernel<<<grid_for(m, kThreads, sms * 8), kThreads, 0, st>>>(m, counts, threshold, rows, cnts, n_out,
                                                                               cap);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_max(int64_t count, const int* v, int* out, cudaStream_t st, int sms, int64_t* launches) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    const int blocks = grid_for(count, kThreads, sms * 8);
    max_kernel<<<blocks, kThreads, 0, st>>>(count, v, out);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_col_norms(const DevCSC& A, float* L, cudaStream_t st, int sms, int64_t* launches) {
    const int blocks = grid_for(A.n, kThreads, sms * 16);  // a warp per 32-column tile
    col_norms_tile_kernel<<<blocks, kThreads, 0, st>>>(A.n, (const long long*)A.colptr, A.val, L);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_residual64(const DevCSC& A, const float* b, const float* x, double* r64, int* flags,
                              cudaStream_t st, int sms, int64_t* launches, const XHeaders* xh, const DevCSR* csr) {
    const XHeaders none{nullptr, 0, nullptr, nullptr, nullptr, 0};
    if (csr) {
        scatter_x_kernel<<<grid_for((A.n + 3) / 4, kThreads, sms * 8), kThreads, 0, st>>>(
            A.n, (const long long*)A.colptr, A.rowidx, A.val, x, r64, flags, xh ? *xh : none, false);
        residual_rows_kernel<<<grid_for(A.m * 32, kThreads, sms * 16), kThreads, 0, st>>>(
            A.m, (const long long*)csr->rowptr, csr->col, csr->val, b, x, r64);
        *launches += 2;
        return cudaGetLastError();
    }
    neg_b_kernel<<<grid_for(A.m, kThreads, sms * 8), kThreads, 0, st>>>(A.m, b, r64);
    scatter_x_kernel<<<grid_for((A.n + 3) / 4, kThreads, sms * 8), kThreads, 0, st>>>(
        A.n, (const long long*)A.colptr, A.rowidx, A.val, x, r64, flags, xh ? *xh : none, true);
    *launches += 2;
    return cudaGetLastError();
}

cudaError_t build_csr(const DevCSC& A, const int* counts, DevCSR* out, cudaStream_t st, int sms, int64_t* launches) {
    unsigned long long* rowptr = nullptr;
    unsigned long long* cursor = nullptr;
    int* ccol = nullptr;
    float* cval = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t e = cudaMalloc((void**)&rowptr, sizeof(unsigned long long) * (A.m + 1));
    if (e == cudaSuccess) e = cudaMalloc((void**)&cursor, sizeof(unsigned long long) * (A.m + 1));
    if (e == cudaSuccess) e = cudaMalloc((void**)&ccol, sizeof(int) * A.nnz);
    if (e == cudaSuccess) e = cudaMalloc((void**)&cval, sizeof(float) * A.nnz);
    if (e == cudaSuccess) {
        counts64_kernel<<<grid_for(A.m + 1, kThreads, sms * 8), kThreads, 0, st>>>(A.m, counts, cursor);
        ++*launches;
        e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cursor, rowptr, A.m + 1, st);
    }
    if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cursor, rowptr, A.m + 1, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(cursor, rowptr, sizeof(unsigned long long) * (A.m + 1), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) {
        csr_fill_kernel<<<grid_for(A.n * 32, kThreads, sms * 16), kThreads, 0, st>>>(
            A.n, (const long long*)A.colptr, A.rowidx, A.val, cursor, ccol, cval);
        ++*launches;
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(tmp);
    cudaFree(cursor);
    if (e != cudaSuccess) {
        cudaFree(rowptr);
        cudaFree(ccol);
        cudaFree(cval);
        cudaGetLastError();
        return e;
    }
    out->rowptr = (const int64_t*)rowptr;
    out->col = ccol;
    out->val = cval;
    return cudaSuccess;
}

cudaError_t launch_round_r(int64_t m, const double* r64, float* r, cudaStream_t st, int sms,
                           int64_t* launches, float* r2, int* zero, int nzero) {
    round_r_kernel<<<grid_for(m, kThreads, sms * 8), kThreads, 0, st>>>(m, r64, r, r2, zero, nzero);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_objective_sums(int64_t m, int64_t n, const double* r64, const float* x, double* out,
                                  cudaStream_t st, int sms, int64_t* launches) {
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(double), st);
    if (e != cudaSuccess) return e;
    objective_sums_kernel<<<grid_for(m > n ? m : n, kThreads, sms * 4), kThreads, 0, st>>>(m, n, r64, x, out);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace pcdm_internal
