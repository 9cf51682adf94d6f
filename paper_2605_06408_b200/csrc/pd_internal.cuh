// pd_internal.cuh -- shared device types of the CUDA path (never included by oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pd.h"

namespace pd {

// Child record stored in its parent so that the two children of a node are one 64-byte read.
//   lo_w = (lo.x, lo.y, lo.z, max weight in subtree)   -- PAPER.md:527 "maxweight"
//   hi_l = (hi.x, hi.y, hi.z, link as int bits)
// link >= 0 : internal node index; link < 0 : leaf range, ~link = (first << 5) | (count - 1).
struct __align__(16) NodeChild {
    float4 lo_w;
    float4 hi_l;
};
// 8-wide BVH node (the binary LBVH collapsed top-down): lane k of a warp reads child k, so one node
// visit is a single coalesced 256-byte read and 8 parallel child tests.
constexpr int WIDE = 8;
constexpr int EMPTY_LINK = 0x7fffffff;  // unused child slot
struct __align__(256) WideNode {
    NodeChild c[WIDE];
};

__host__ __device__ inline int leaf_link(int first, int count) { return ~((first << 5) | (count - 1)); }
__host__ __device__ inline int leaf_first(int link) { return (~link) >> 5; }
__host__ __device__ inline int leaf_count(int link) { return ((~link) & 31) + 1; }

struct Bvh {
    WideNode* nodes = nullptr;  // wide nodes (<= 2n/l + 2); unused when n <= leaf
    NodeChild* root = nullptr;  // device: 1 record describing the root (bounds + link)
    int n_wide = 0;
    int levels = 0;
};

// Per-cell outputs of the cell kernel, indexed by ORIGINAL id (cells outside a shard untouched).
struct CellOut {
    int32_t* cnt;        // neighbour count
    int64_t* aoff;       // offset of the row in the arena
    float* vol;
    float* surf;
    uint8_t* flags;
    int32_t* arena_nbr;
    float* arena_area;
    unsigned long long* arena_top;  // atomic bump pointer (entries)
    int64_t arena_cap;
    int* arena_overflow;            // set to 1 when a row did not fit
    int32_t* cost;                  // optional per-cell work (PD_COST)
    // optional dual tetrahedra (PD_TETS): per original id count + arena offset, arena of int4 tets
    int32_t* tcnt;
    int64_t* taoff;
    int4* tarena;
    unsigned long long* ttop;
    int64_t tcap;
    int* tovf;
};

struct Stats {  // device counters (PD_STATS), robustness counters (always)
    unsigned long long nodes, leaves, sites, clip_tests, clips, cells, tier[3], overflow, spills, cyc[10];
    unsigned long long dropped, small, degraded;
};

struct CellParams {
    const float4* sites;  // Morton-sorted (x, y, z, w)
    const int32_t* perm;  // Morton position -> original id
    const WideNode* nodes;
    const NodeChild* root;
    float box_lo[3], box_hi[3];
    unsigned flags;
    // work: either the Morton range [begin, begin+count) or list[0..*list_count)
    int64_t begin;
    int64_t count;
    const int32_t* list;
    const int32_t* list_count;
    unsigned long long* work_counter;
    // overflow hand-off to the next tier
    int32_t* next_list;
    int32_t* next_count;
    int32_t* next_cost;   // parallel to next_list: the work a cell had done when it outgrew this tier
    int last_tier;
    CellOut out;
    Stats* stats;
    NodeChild* spill;   // per-warp queue spill stacks (global memory)
    int spill_cap;      // entries per warp
    int exact_after;    // exact node tests once a cell has visited this many nodes
    void* gstate;       // top tier: per-warp cell state in global memory
    int prof_tier;      // PD_PROFILE builds: tier whose phase cycles are recorded (-1 = all)
    const int32_t* knn; // PD_WARM_START: K = 8 nearest sites per Morton index (-1 = none), else NULL
    int64_t n_sites;    // number of sites (Morton positions 0..n_sites-1)
    int start_tier;     // test knob ($PD_START_TIER): cells skip the tiers below it (default 0)
    int coop_min_v;     // top tier: vertex count from which O(V) passes use the whole CTA ($PD_COOP_MIN_V)
    int trace_cell;     // debug ($PD_TRACE_CELL): print the work counters of this original id (-1 = none)
    // Deferred finalize (tier 1): the cell program stores each finished cell's topology -- its planes as
    // neighbour ids and its vertices as plane-index triplets -- and a separate kernel rebuilds the FP64 planes
    // and vertices from it and computes faces, areas and volume (keeps the finalize code out of the cell
    // program's instruction-cache working set).  rec_index == NULL: finalize in the cell kernel.
    uint32_t* rec_index;           // per Morton position: word offset of its record, ~0u = not deferred
    uint32_t* rec_arena;           // records: [nv | np << 16, degraded, pid[np], vt[nv]]
    unsigned long long* rec_top;   // bump pointer (words)
    int64_t rec_cap;               // words (< 2^32); a cell that does not fit is built again by tier 2
};

cudaError_t launch_cells(int tier, const CellParams& p, cudaStream_t st, int num_sms, int* launches,
                         bool with_finalize = true);
// the tier-1 finalize (deferred records) alone; cpw > 0: non-persistent grid, cpw cells per warp
cudaError_t launch_finalize(const CellParams& p, cudaStream_t st, int num_sms, int cpw, int* launches);
int cells_grid_warps(int tier, int num_sms);
size_t cells_global_state_bytes(int num_sms);
constexpr int KNN_K = 8;  // warm-start neighbours per site
// K nearest sites (Euclidean, coincident sites excluded) of the Morton positions [begin, end) -> knn[s*K + k]
// adaptive != 0: only sites dominated at their own position by their power-nearest neighbour keep a list
// list != NULL: the positions list[begin..end) instead of the Morton range [begin, end)
cudaError_t knn_query(const float4* sites, const WideNode* nodes, const NodeChild* root, int begin, int end, int adaptive,
                      int32_t* knn, int num_sms, cudaStream_t st, int* launches, const int32_t* list = nullptr);

}  // namespace pd
