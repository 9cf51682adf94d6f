// pd_knn.cu -- the optional KNN warm start (App. "KNN warm start"; SURVEY.md §8(f)
// NEXT-1): before the BVH traversal of the cell kernel, a K = 8 nearest-neighbour query on the same
// BVH gives each site candidates that pre-clip its cell, so the directional culling
// already prunes from the root.
//
// "Nearest" is in power distance from the site, pi_j(p_i) = |p_i - p_j|^2 - w_j (PAPER.md:545 bounds the
// initial search radius "to approximately the power distance to the K-th nearest neighbor"; for
// Voronoi input it is the Euclidean KNN): the sites whose power cells reach furthest over p_i, which
// for a light site among heavy ones are the planes that empty its cell.
// One warp per site over the 8-wide BVH: lanes 0..7 test the 8 child boxes of a node (squared
// distance from the site to the box minus the subtree's max weight, a lower bound of the power
// distance), the nearest surviving child is descended, the others go on a
// per-warp stack in shared memory (popped nearest-last-pushed, re-checked against the current K-th
// distance); at a leaf lane k takes site first+k and the candidates closer than the current K-th are
// inserted one at a time into the sorted best list held by lanes 0..7.
//
// The result only orders work: the warm start is correctness-neutral ("warm-start
// transparency"), so a stack overflow simply drops the deepest entries (the KNN becomes approximate,
// never wrong for the diagram).  Coincident sites (D = 0) are excluded: their ownership is decided by
// the leaf processing of the cell kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include "pd_bvh.cuh"
#include "pd_internal.cuh"

namespace pd {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int KNN_WARPS = 4;
constexpr int KNN_STACK = 128;

__device__ __forceinline__ int fordk(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}

__global__ void __launch_bounds__(KNN_WARPS * 32) k_knn(const float4* __restrict__ sites, const WideNode* __restrict__ nodes,
                                                        const NodeChild* __restrict__ root, int begin, int end, int adaptive,
                                                        int32_t* __restrict__ knn, const int32_t* __restrict__ list) {
    __shared__ int st_node[KNN_WARPS][KNN_STACK];
    __shared__ float st_d[KNN_WARPS][KNN_STACK];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gw = blockIdx.x * KNN_WARPS + wid, nw = gridDim.x * KNN_WARPS;
    const int root_link = __float_as_int(__ldg(&root->hi_l.w));
    for (int it = begin + gw; it < end; it += nw) {
        const int s = list ? __ldg(&list[it]) : it;  // a Morton range, or the listed positions list[begin..end)
        const float4 p = __ldg(&sites[s]);
        float bd = INFINITY;  // lanes 0..K-1: sorted K best squared distances
        int bi = -1;
        float kth = INFINITY;
        int sp = 0;
        int node = root_link;
        bool have = true;
        for (;;) {
            if (have) {
                while (node >= 0) {  // descend, nearest surviving child first
                    float d = INFINITY;
                    int link = EMPTY_LINK;
                    if (lane < WIDE) {
                        const NodeChild* rec = nodes[node].c;
                        float4 lo = __ldg(&rec[lane].lo_w), hi = __ldg(&rec[lane].hi_l);
                        link = __float_as_int(hi.w);
                        if (link != EMPTY_LINK) {  // lower bound of the power distance over the box
                            float gx = fmaxf(fmaxf(lo.x - p.x, p.x - hi.x), 0.f);
                            float gy = fmaxf(fmaxf(lo.y - p.y, p.y - hi.y), 0.f);
                            float gz = fmaxf(fmaxf(lo.z - p.z, p.z - hi.z), 0.f);
                            d = gx * gx + gy * gy + gz * gz - lo.w;
                        }
                    }
                    const bool ok = d < kth;
                    if (!__any_sync(FULL, ok)) { have = false; break; }
                    const int dmin = __reduce_min_sync(FULL, ok ? fordk(d) : 0x7fffffff);
                    const int near = __ffs(__ballot_sync(FULL, ok && fordk(d) == dmin)) - 1;
                    const bool push = ok && lane != near;
                    const unsigned pm = __ballot_sync(FULL, push);
                    if (push) {
                        const int pos = sp + __popc(pm & ((1u << lane) - 1u));
                        if (pos < KNN_STACK) { st_node[wid][pos] = link; st_d[wid][pos] = d; }
                    }
                    sp = min(sp + __popc(pm), KNN_STACK);
                    node = __shfl_sync(FULL, link, near);
                }
            }
            if (have) {  // leaf: node is a leaf link
                const int first = leaf_first(node), count = leaf_count(node);
                const int j = first + lane;
                float d = INFINITY;
                if (lane < count && j != s) {
                    const float4 q = __ldg(&sites[j]);
                    const float dx = q.x - p.x, dy = q.y - p.y, dz = q.z - p.z;
                    if (dx != 0.f || dy != 0.f || dz != 0.f) d = dx * dx + dy * dy + dz * dz - q.w;
                }
                unsigned cm = __ballot_sync(FULL, d < kth);
                while (cm) {  // insert the candidates below the K-th distance, one at a time
                    const int src = __ffs(cm) - 1;
                    cm &= cm - 1;
                    const float cd = __shfl_sync(FULL, d, src);
                    if (!(cd < kth)) continue;
                    const int pos = __popc(__ballot_sync(FULL, lane < KNN_K && bd <= cd));
                    const float ud = __shfl_up_sync(FULL, bd, 1);
                    const int ui = __shfl_up_sync(FULL, bi, 1);
                    if (lane < KNN_K && lane > pos) { bd = ud; bi = ui; }
                    if (lane == pos) { bd = cd; bi = first + src; }
                    kth = __shfl_sync(FULL, bd, KNN_K - 1);
                }
            }
            // pop the most recently stacked node that is still closer than the K-th distance
            __syncwarp();
            have = false;
            while (sp > 0) {
                --sp;
                if (st_d[wid][sp] < kth) { node = st_node[wid][sp]; have = true; break; }
            }
            __syncwarp();
            if (!have) break;
        }
        // adaptive mode: keep the list only for a site that its power-nearest neighbour dominates at
        // its own position (pi_j(p_i) < pi_i(p_i) = -w_i: p_i lies outside its cell, as for every EMPTY
        // cell), where pre-clipping pays; other sites start the traversal from the box as usual
        const bool keep = !adaptive || __shfl_sync(FULL, bd, 0) < -p.w;
        if (lane < KNN_K) knn[(int64_t)s * KNN_K + lane] = keep ? bi : -1;
    }
}

}  // namespace

cudaError_t knn_query(const float4* sites, const WideNode* nodes, const NodeChild* root, int begin, int end, int adaptive,
                      int32_t* knn, int num_sms, cudaStream_t st, int* launches, const int32_t* list) {
    if (end <= begin) return cudaSuccess;
    int grid = num_sms * 16;
    int need = (end - begin + KNN_WARPS - 1) / KNN_WARPS;
    if (grid > need) grid = need;
    k_knn<<<grid, KNN_WARPS * 32, 0, st>>>(sites, nodes, root, begin, end, adaptive, knn, list);
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace pd
