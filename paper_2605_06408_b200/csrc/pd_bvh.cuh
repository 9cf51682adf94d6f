// pd_bvh.cuh -- host entry points of the BVH builder (pd_bvh.cu) and CSR stage (pd_csr.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pd_internal.cuh"

namespace pd {

constexpr int kCollapseCounters = 128;

struct BvhScratch {
    int2* child = nullptr;      // n-1
    int2* range = nullptr;      // n-1
    int* parent_int = nullptr;  // n-1
    int* parent_leaf = nullptr; // n
    int* visit = nullptr;       // n-1
    float4* blo = nullptr;      // n-1
    float4* bhi = nullptr;      // n-1
    int2* tasks[2] = {nullptr, nullptr};  // collapse work lists (binary node, wide node)
    int* counters = nullptr;    // kCollapseCounters ints: [0] wide-node count, [1] overflow, [2+L] level-L tasks, barrier
    int max_wide = 0;
};

cudaError_t bvh_pack(const float* pts, const float* w, int64_t n, const pd_box* box, float4* sites, float* box_dev,
                     unsigned long long* errs, int* aabb, cudaStream_t st, int* launches);
cudaError_t bvh_morton(const float4* sites, int64_t n, const float* box_dev, uint64_t* keys, uint32_t* vals,
                       cudaStream_t st, int* launches);
cudaError_t bvh_gather(const float4* sites, const uint32_t* perm, int64_t n, float4* sorted, int32_t* perm_i32,
                       cudaStream_t st, int* launches);
cudaError_t bvh_topology(const uint64_t* keys_sorted, const float4* sorted, int n, int leaf, BvhScratch& sc, Bvh& out,
                         cudaStream_t st, int* launches);

// radix sort of (u64 key, u32 value) pairs on bits [0, 63)
cudaError_t sort_pairs(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                       int64_t n, void* temp, size_t* temp_bytes, cudaStream_t st, int* launches);

// exclusive scan of int32 counts into int64 offsets[n+1]
cudaError_t scan_counts(const int32_t* cnt, int64_t* offsets, int64_t n, void* temp, size_t* temp_bytes,
                        cudaStream_t st, int* launches);

// CSR rows: copy arena rows (per original id) into the CSR arrays
cudaError_t csr_gather(const int32_t* cnt, const int64_t* aoff, const int64_t* offsets, const int32_t* arena_nbr,
                       const float* arena_area, int64_t n, int32_t* nbr, float* area, cudaStream_t st, int* launches);

// dual tetrahedra rows: copy each cell's arena tets into the final order
cudaError_t tet_gather(const int32_t* tcnt, const int64_t* taoff, const int64_t* toff, const int4* tarena, int64_t n,
                       int4* tets, cudaStream_t st, int* launches);

// longest-first order of a capacity tier's overflow list (device count; <= 8192 entries, else unchanged)
cudaError_t sort_list_by_cost(int32_t* list, const int32_t* cost, const int32_t* count, cudaStream_t st, int* launches);

// sharding helpers
cudaError_t slice_export_meta(const int32_t* perm, int64_t begin, int64_t len, const int32_t* cnt, const float* vol,
                              const float* surf, const uint8_t* flags, int32_t* cnt_m, float* vol_m, float* surf_m,
                              uint8_t* flags_m, cudaStream_t st, int* launches);
cudaError_t slice_export_rows(const int32_t* perm, int64_t begin, int64_t len, const int32_t* cnt_m,
                              const int64_t* moff, const int64_t* offsets, const int32_t* nbr, const float* area,
                              int32_t* rows_nbr, float* rows_area, cudaStream_t st, int* launches);
cudaError_t assemble_meta(const int32_t* perm, int64_t n, const int32_t* cnt_m, const float* vol_m, const float* surf_m,
                          const uint8_t* flags_m, int32_t* cnt_o, float* vol_o, float* surf_o, uint8_t* flags_o,
                          cudaStream_t st, int* launches);
cudaError_t assemble_rows(const int32_t* perm, int64_t n, const int32_t* cnt_m, const int64_t* moff,
                          const int64_t* offsets, const int32_t* rows_nbr, const float* rows_area, int32_t* nbr,
                          float* area, cudaStream_t st, int* launches);
cudaError_t fill_flags(uint8_t* flags, int64_t n, uint8_t v, cudaStream_t st, int* launches);
// out[k] = cost[perm[pos[k]]] for the sampled Morton positions (cost-balanced slicing)
cudaError_t gather_sample_cost(const int32_t* perm, const int32_t* pos, int64_t ns, const int32_t* cost, int32_t* out,
                               cudaStream_t st, int* launches);

}  // namespace pd
