// pd_csr.cu -- a13 CSR compaction (row gather after the device prefix scan of pd_sort.cu), plus the
// Morton-order slice export / reassembly used by the sharded (multi-GPU) build.
#include <cuda_runtime.h>
#include <stdint.h>

#include "pd_bvh.cuh"

namespace pd {
namespace {

inline unsigned blocks(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// One warp per 32 rows: lanes cooperate on each row so the copies are coalesced.
__global__ void k_csr_gather(const int32_t* __restrict__ cnt, const int64_t* __restrict__ aoff,
                             const int64_t* __restrict__ offsets, const int32_t* __restrict__ anbr,
                             const float* __restrict__ aarea, int64_t n, int32_t* __restrict__ nbr,
                             float* __restrict__ area) {
    int64_t row0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll;
    int lane = threadIdx.x & 31;
    int64_t my = row0 + lane;
    int c = my < n ? cnt[my] : 0;
    int64_t src = my < n ? aoff[my] : 0, dst = my < n ? offsets[my] : 0;
    for (int r = 0; r < 32; ++r) {
        int cr = __shfl_sync(0xffffffffu, c, r);
        long long s = __shfl_sync(0xffffffffu, (long long)src, r);
        long long d = __shfl_sync(0xffffffffu, (long long)dst, r);
        for (int e = lane; e < cr; e += 32) {
            nbr[d + e] = anbr[s + e];
            area[d + e] = aarea[s + e];
        }
    }
}

__global__ void k_export_meta(const int32_t* __restrict__ perm, int64_t begin, int64_t len, const int32_t* __restrict__ cnt,
                              const float* __restrict__ vol, const float* __restrict__ surf, const uint8_t* __restrict__ flags,
                              int32_t* cnt_m, float* vol_m, float* surf_m, uint8_t* flags_m) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= len) return;
    int i = perm[begin + k];
    cnt_m[k] = cnt[i];
    vol_m[k] = vol[i];
    surf_m[k] = surf[i];
    flags_m[k] = flags[i];
}

__global__ void k_export_rows(const int32_t* __restrict__ perm, int64_t begin, int64_t len, const int32_t* __restrict__ cnt_m,
                              const int64_t* __restrict__ moff, const int64_t* __restrict__ offsets,
                              const int32_t* __restrict__ nbr, const float* __restrict__ area, int32_t* rows_nbr,
                              float* rows_area) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= len) return;
    int i = perm[begin + k];
    int64_t s = offsets[i], d = moff[k];
    for (int e = 0; e < cnt_m[k]; ++e) {
        rows_nbr[d + e] = nbr[s + e];
        rows_area[d + e] = area[s + e];
    }
}

__global__ void k_assemble_meta(const int32_t* __restrict__ perm, int64_t n, const int32_t* __restrict__ cnt_m,
                                const float* __restrict__ vol_m, const float* __restrict__ surf_m,
                                const uint8_t* __restrict__ flags_m, int32_t* cnt_o, float* vol_o, float* surf_o,
                                uint8_t* flags_o) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    int i = perm[k];
    cnt_o[i] = cnt_m[k];
    vol_o[i] = vol_m[k];
    surf_o[i] = surf_m[k];
    flags_o[i] = flags_m[k];
}

__global__ void k_assemble_rows(const int32_t* __restrict__ perm, int64_t n, const int32_t* __restrict__ cnt_m,
                                const int64_t* __restrict__ moff, const int64_t* __restrict__ offsets,
                                const int32_t* __restrict__ rows_nbr, const float* __restrict__ rows_area,
                                int32_t* nbr, float* area) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    int i = perm[k];
    int64_t s = moff[k], d = offsets[i];
    for (int e = 0; e < cnt_m[k]; ++e) {
        nbr[d + e] = rows_nbr[s + e];
        area[d + e] = rows_area[s + e];
    }
}

// dual tetrahedra: one thread per cell copies its rows (int4 each)
__global__ void k_tet_gather(const int32_t* __restrict__ tcnt, const int64_t* __restrict__ taoff,
                             const int64_t* __restrict__ toff, const int4* __restrict__ tarena, int64_t n,
                             int4* __restrict__ tets) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = tcnt[i];
    const int64_t s = taoff[i], d = toff[i];
    for (int e = 0; e < c; ++e) tets[d + e] = tarena[s + e];
}

__global__ void k_fill_u8(uint8_t* p, int64_t n, uint8_t v) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) p[k] = v;
}

__global__ void k_gather_cost(const int32_t* __restrict__ perm, const int32_t* __restrict__ pos, int64_t ns,
                              const int32_t* __restrict__ cost, int32_t* __restrict__ out) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < ns) out[k] = cost[perm[pos[k]]];
}


// Longest-first order of a capacity tier's overflow list: one CTA bitonic-sorts up to
// kListSortMax (cell, cost) pairs in shared memory by (cost descending, Morton index ascending); a
// longer list keeps its (arbitrary) order.  Runs on the device so no host round trip separates the
// tiers.
constexpr int kListSortMax = 8192;
__global__ void __launch_bounds__(1024) k_sort_list(int32_t* __restrict__ list, const int32_t* __restrict__ cost,
                                                    const int32_t* __restrict__ count) {
    extern __shared__ unsigned long long key[];  // kListSortMax entries (64 KB, dynamic)
    const int n = *count;
    if (n <= 1 || n > kListSortMax) return;
    int m = 2;
    while (m < n) m <<= 1;
    for (int k = threadIdx.x; k < m; k += blockDim.x)
        key[k] = k < n ? ((unsigned long long)(uint32_t)(0x7fffffff - max(cost[k], 0)) << 32) | (uint32_t)list[k]
                       : ~0ull;
    __syncthreads();
    for (int size = 2; size <= m; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int k = threadIdx.x; k < m; k += blockDim.x) {
                const int o = k ^ stride;
                if (o > k) {
                    const bool up = (k & size) == 0;
                    const unsigned long long a = key[k], b = key[o];
                    if ((a > b) == up) { key[k] = b; key[o] = a; }
                }
            }
            __syncthreads();
        }
    }
    for (int k = threadIdx.x; k < n; k += blockDim.x) list[k] = (int32_t)(uint32_t)key[k];
}

}  // namespace

cudaError_t gather_sample_cost(const int32_t* perm, const int32_t* pos, int64_t ns, const int32_t* cost, int32_t* out,
                               cudaStream_t st, int* launches) {
    k_gather_cost<<<blocks(ns, 256), 256, 0, st>>>(perm, pos, ns, cost, out);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t sort_list_by_cost(int32_t* list, const int32_t* cost, const int32_t* count, cudaStream_t st, int* launches) {
    static bool attr[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
        cudaFuncSetAttribute(k_sort_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kListSortMax * sizeof(unsigned long long)));
        attr[dev & 63] = true;
    }
    k_sort_list<<<1, 1024, kListSortMax * sizeof(unsigned long long), st>>>(list, cost, count);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t csr_gather(const int32_t* cnt, const int64_t* aoff, const int64_t* offsets, const int32_t* arena_nbr,
                       const float* arena_area, int64_t n, int32_t* nbr, float* area, cudaStream_t st, int* launches) {
    k_csr_gather<<<blocks(n, 256), 256, 0, st>>>(cnt, aoff, offsets, arena_nbr, arena_area, n, nbr, area);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t slice_export_meta(const int32_t* perm, int64_t begin, int64_t len, const int32_t* cnt, const float* vol,
                              const float* surf, const uint8_t* flags, int32_t* cnt_m, float* vol_m, float* surf_m,
                              uint8_t* flags_m, cudaStream_t st, int* launches) {
    if (len <= 0) return cudaSuccess;
    k_export_meta<<<blocks(len, 256), 256, 0, st>>>(perm, begin, len, cnt, vol, surf, flags, cnt_m, vol_m, surf_m, flags_m);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t slice_export_rows(const int32_t* perm, int64_t begin, int64_t len, const int32_t* cnt_m,
                              const int64_t* moff, const int64_t* offsets, const int32_t* nbr, const float* area,
                              int32_t* rows_nbr, float* rows_area, cudaStream_t st, int* launches) {
    if (len <= 0) return cudaSuccess;
    k_export_rows<<<blocks(len, 256), 256, 0, st>>>(perm, begin, len, cnt_m, moff, offsets, nbr, area, rows_nbr, rows_area);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t assemble_meta(const int32_t* perm, int64_t n, const int32_t* cnt_m, const float* vol_m, const float* surf_m,
                          const uint8_t* flags_m, int32_t* cnt_o, float* vol_o, float* surf_o, uint8_t* flags_o,
                          cudaStream_t st, int* launches) {
    k_assemble_meta<<<blocks(n, 256), 256, 0, st>>>(perm, n, cnt_m, vol_m, surf_m, flags_m, cnt_o, vol_o, surf_o, flags_o);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t assemble_rows(const int32_t* perm, int64_t n, const int32_t* cnt_m, const int64_t* moff,
                          const int64_t* offsets, const int32_t* rows_nbr, const float* rows_area, int32_t* nbr,
                          float* area, cudaStream_t st, int* launches) {
    k_assemble_rows<<<blocks(n, 256), 256, 0, st>>>(perm, n, cnt_m, moff, offsets, rows_nbr, rows_area, nbr, area);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t tet_gather(const int32_t* tcnt, const int64_t* taoff, const int64_t* toff, const int4* tarena, int64_t n,
                       int4* tets, cudaStream_t st, int* launches) {
    k_tet_gather<<<blocks(n, 256), 256, 0, st>>>(tcnt, taoff, toff, tarena, n, tets);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t fill_flags(uint8_t* flags, int64_t n, uint8_t v, cudaStream_t st, int* launches) {
    k_fill_u8<<<blocks(n, 256), 256, 0, st>>>(flags, n, v);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace pd
