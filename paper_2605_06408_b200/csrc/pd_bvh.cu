// pd_bvh.cu -- input packing, Morton codes, radix sort, Karras LBVH topology and
// the bottom-up refit of per-node AABB + max weight ("power-augmented BVH").
// The paper uses the cuBQL builder; this is an own LBVH (Karras 2012 topology over 63-bit Morton
// codes), collapsed to leaves of <= l sites at traversal time via the leaf-range links.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pd_bvh.cuh"
#include "pd_internal.cuh"

namespace pd {
namespace {

__device__ __forceinline__ int ford(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float iford(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

// a1: pack (x,y,z,w) into one float4 per site; validate finite and (if a box is given) inside it.
__global__ void k_pack(const float* __restrict__ pts, const float* __restrict__ w, int64_t n, float4* __restrict__ out,
                       int has_box, float lx, float ly, float lz, float hx, float hy, float hz,
                       unsigned long long* err_nonfinite, unsigned long long* err_outside, int* aabb) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    if (i < n) {
        float x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
        float ww = w ? w[i] : 0.f;
        out[i] = make_float4(x, y, z, ww);
        bool fin = isfinite(x) && isfinite(y) && isfinite(z) && isfinite(ww);
        if (!fin) atomicMin(err_nonfinite, (unsigned long long)i);
        else if (has_box && !(x >= lx && x <= hx && y >= ly && y <= hy && z >= lz && z <= hz))
            atomicMin(err_outside, (unsigned long long)i);
        if (fin) { mn[0] = mx[0] = x; mn[1] = mx[1] = y; mn[2] = mx[2] = z; }
    }
    if (!has_box) {  // a2: AABB of the points
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            int a = __reduce_min_sync(0xffffffffu, ford(mn[k]));
            int b = __reduce_max_sync(0xffffffffu, ford(mx[k]));
            if ((threadIdx.x & 31) == 0) {
                atomicMin(&aabb[k], a);
                atomicMax(&aabb[3 + k], b);
            }
        }
    }
}

__device__ __forceinline__ uint64_t spread21(uint32_t v) {
    uint64_t x = v & 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

// a3: 63-bit Morton code, 21 bits per axis over the box.
__global__ void k_morton(const float4* __restrict__ s, int64_t n, const float* __restrict__ box, uint64_t* __restrict__ keys,
                         uint32_t* __restrict__ vals) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 p = s[i];
    float c[3] = {p.x, p.y, p.z};
    uint32_t q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float ext = box[3 + k] - box[k];
        float t = ext > 0.f ? (c[k] - box[k]) / ext : 0.f;
        t = fminf(fmaxf(t, 0.f), 1.f);
        uint32_t v = (uint32_t)(t * 2097152.0f);
        q[k] = v > 2097151u ? 2097151u : v;
    }
    keys[i] = spread21(q[0]) | (spread21(q[1]) << 1) | (spread21(q[2]) << 2);
    vals[i] = (uint32_t)i;
}

// a5: sites in Morton order
__global__ void k_gather(const float4* __restrict__ s, const uint32_t* __restrict__ perm, int64_t n, float4* __restrict__ out,
                         int32_t* __restrict__ perm_i32) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t p = perm[i];
    out[i] = s[p];
    perm_i32[i] = (int32_t)p;
}

__device__ __forceinline__ int delta(const uint64_t* __restrict__ k, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    uint64_t a = k[i], b = k[j];
    if (a == b) return 64 + __clz((unsigned)(i ^ j));
    return __clzll((long long)(a ^ b));
}

// a6: Karras (2012) radix-tree topology.  child >= 0 internal index, child < 0 leaf ~prim.
__global__ void k_karras(const uint64_t* __restrict__ k, int n, int2* __restrict__ child, int2* __restrict__ range,
                         int* __restrict__ parent_int, int* __restrict__ parent_leaf) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = delta(k, n, i, i - d);
    int lmax = 2;
    while (delta(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
    int j = i + l * d;
    int dnode = delta(k, n, i, j);
    int s = 0;
    int t = l;
    do {
        t = (t + 1) >> 1;
        if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    int gamma = i + s * d + (d < 0 ? d : 0);
    int lo = min(i, j), hi = max(i, j);
    int left = (lo == gamma) ? ~gamma : gamma;
    int right = (hi == gamma + 1) ? ~(gamma + 1) : gamma + 1;
    child[i] = make_int2(left, right);
    range[i] = make_int2(lo, hi);
    if (left < 0) parent_leaf[~left] = i; else parent_int[left] = i;
    if (right < 0) parent_leaf[~right] = i; else parent_int[right] = i;
    if (i == 0) parent_int[0] = -1;
}

// a7: bottom-up refit of AABB + max weight (atomic visit counters; second arrival computes).
__global__ void k_refit(const float4* __restrict__ s, int n, const int2* __restrict__ child, const int* __restrict__ parent_int,
                        const int* __restrict__ parent_leaf, int* __restrict__ visit, float4* __restrict__ blo,
                        float4* __restrict__ bhi) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int node = parent_leaf[p];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&visit[node], 1) == 0) return;
        __threadfence();
        int2 c = child[node];
        float4 lo = make_float4(INFINITY, INFINITY, INFINITY, -INFINITY);
        float4 hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            int ch = q ? c.y : c.x;
            float4 a, b;
            if (ch < 0) {
                a = s[~ch];
                b = a;
            } else {
                a = __ldcg(&blo[ch]);
                b = __ldcg(&bhi[ch]);
            }
            lo.x = fminf(lo.x, a.x); lo.y = fminf(lo.y, a.y); lo.z = fminf(lo.z, a.z); lo.w = fmaxf(lo.w, a.w);
            hi.x = fmaxf(hi.x, b.x); hi.y = fmaxf(hi.y, b.y); hi.z = fmaxf(hi.z, b.z);
        }
        __stcg(&blo[node], lo);
        __stcg(&bhi[node], hi);
        node = parent_int[node];
    }
}

__device__ __forceinline__ float box_area(float4 lo, float4 hi) {
    float dx = hi.x - lo.x, dy = hi.y - lo.y, dz = hi.z - lo.z;
    return dx * dy + dy * dz + dz * dx;
}

// Collapse the binary LBVH into 8-wide nodes.  Task (b, w): wide node w covers binary subtree b.
// Its children start as b's two children; the internal child (more than l sites) with the largest
// surface area is replaced by its two children until there are 8.  Children with <= l sites become
// leaf-range links (the collapse of PAPER.md:527's leaf size l); larger ones become new wide nodes
// (next level's tasks).
// Capacity: every wide node is a distinct binary node with > l sites.  Those nodes form an upward-
// closed subtree whose lowest members are disjoint sets of > l sites, so there are at most n/(l+1)
// of them and the subtree has at most 2n/(l+1) - 1 nodes <= max_wide = min(2n/l + 2, n).  The guard
// below therefore never fires on a well-formed tree; it turns a violated invariant into an error
// (ovf) instead of an out-of-bounds write.
__device__ __forceinline__ void collapse_task(int2 task, const int2* __restrict__ child, const int2* __restrict__ range,
                                              const float4* __restrict__ blo, const float4* __restrict__ bhi,
                                              const float4* __restrict__ s, int leaf, WideNode* __restrict__ wide,
                                              int* wide_count, int* next_count, int2* __restrict__ tasks_out, int max_wide,
                                              int* ovf) {
    int ref[WIDE];
    int2 c0 = child[task.x];
    ref[0] = c0.x;
    ref[1] = c0.y;
    int m = 2;
    while (m < WIDE) {
        int best = -1;
        float bestA = -1.f;
        for (int k = 0; k < m; ++k) {
            int r = ref[k];
            if (r < 0) continue;
            int2 rg = range[r];
            if (rg.y - rg.x + 1 <= leaf) continue;
            float A = box_area(__ldcg(&blo[r]), __ldcg(&bhi[r]));
            if (A > bestA) { bestA = A; best = k; }
        }
        if (best < 0) break;
        int2 cc = child[ref[best]];
        ref[best] = cc.x;
        ref[m++] = cc.y;
    }
    WideNode out;
    for (int k = 0; k < WIDE; ++k) {
        float4 a, b;
        int link;
        if (k >= m) {
            a = make_float4(INFINITY, INFINITY, INFINITY, -INFINITY);
            b = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
            link = EMPTY_LINK;
        } else if (ref[k] < 0) {
            a = s[~ref[k]];
            b = a;
            link = leaf_link(~ref[k], 1);
        } else {
            int r = ref[k];
            int2 rg = range[r];
            int cnt = rg.y - rg.x + 1;
            a = __ldcg(&blo[r]);
            b = __ldcg(&bhi[r]);
            if (cnt <= leaf) {
                link = leaf_link(rg.x, cnt);
            } else {
                link = atomicAdd(wide_count, 1);
                int q = atomicAdd(next_count, 1);
                if (link < max_wide && q < max_wide) tasks_out[q] = make_int2(r, link);
                else { atomicExch(ovf, 1); link = EMPTY_LINK; }
            }
        }
        out.c[k].lo_w = a;
        out.c[k].hi_l = make_float4(b.x, b.y, b.z, __int_as_float(link));
    }
    if (task.y < max_wide) wide[task.y] = out;
}

// Grid-wide barrier for a cooperative launch (every block co-resident): arrive on a counter, the last
// block bumps the generation word the others spin on.
__device__ __forceinline__ void grid_barrier(unsigned* arrive, volatile unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(arrive, 1u) == nblocks - 1) {
            *arrive = 0u;
            __threadfence();
            atomicAdd((unsigned*)gen, 1u);
        } else {
            while (*gen == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// All collapse levels in ONE cooperative launch (no host round trip per level): level L reads its
// tasks from tasks[L & 1] (count counters[2 + L]) and appends the next level's to tasks[(L+1) & 1].
// counters: [0] wide-node count, [1] overflow flag, [2 + L] task count of level L, [kMaxLevels + 2]
// barrier arrive, [kMaxLevels + 3] barrier generation.
constexpr int kMaxLevels = 120;  // binary depth <= 63 key bits + 32 index bits (duplicate codes)
__global__ void __launch_bounds__(256) k_collapse_all(int2* __restrict__ tasks0, int2* __restrict__ tasks1,
                                                      const int2* __restrict__ child, const int2* __restrict__ range,
                                                      const float4* __restrict__ blo, const float4* __restrict__ bhi,
                                                      const float4* __restrict__ s, int leaf, WideNode* __restrict__ wide,
                                                      int* counters, int max_wide) {
    volatile int* vc = counters;
    const unsigned nb = gridDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
    for (int L = 0; L < kMaxLevels; ++L) {
        const int ntask = vc[2 + L];
        if (ntask == 0 || vc[1]) break;  // uniform over the grid (written before the last barrier)
        const int2* tin = (L & 1) ? tasks1 : tasks0;
        int2* tout = (L & 1) ? tasks0 : tasks1;
        for (int t = tid; t < ntask; t += nthreads)
            collapse_task(__ldcg(&tin[t]), child, range, blo, bhi, s, leaf, wide, &counters[0], &counters[2 + L + 1],
                          tout, max_wide, &counters[1]);
        grid_barrier((unsigned*)&counters[kMaxLevels + 2], (volatile unsigned*)&counters[kMaxLevels + 3], nb);
    }
}

__global__ void k_root(const float4* __restrict__ blo, const float4* __restrict__ bhi, int n, int leaf,
                       NodeChild* root, int2* tasks, int* counters) {
    float4 lo = blo[0], hi = bhi[0];
    int link = n <= leaf ? leaf_link(0, n) : 0;
    root->lo_w = lo;
    root->hi_l = make_float4(hi.x, hi.y, hi.z, __int_as_float(link));
    tasks[0] = make_int2(0, 0);
    counters[0] = 1;  // wide node 0 = the root's node
    counters[2] = 1;  // level 0: one task (the root)
}

__global__ void k_root_single(NodeChild* root) {
    root->lo_w = make_float4(0, 0, 0, 0);
    root->hi_l = make_float4(0, 0, 0, __int_as_float(leaf_link(0, 1)));
}

__global__ void k_box_from_aabb(const int* aabb, float* box) {
    int k = threadIdx.x;
    if (k < 6) box[k] = iford(aabb[k]);
}

inline unsigned blocks(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

cudaError_t bvh_pack(const float* pts, const float* w, int64_t n, const pd_box* box, float4* sites, float* box_dev,
                     unsigned long long* errs, int* aabb, cudaStream_t st, int* launches) {
    if (box) {
        k_pack<<<blocks(n, 256), 256, 0, st>>>(pts, w, n, sites, 1, box->lo[0], box->lo[1], box->lo[2], box->hi[0],
                                               box->hi[1], box->hi[2], errs, errs + 1, aabb);
        ++*launches;
    } else {
        k_pack<<<blocks(n, 256), 256, 0, st>>>(pts, w, n, sites, 0, 0, 0, 0, 0, 0, 0, errs, errs + 1, aabb);
        k_box_from_aabb<<<1, 32, 0, st>>>(aabb, box_dev);
        *launches += 2;
    }
    return cudaGetLastError();
}

cudaError_t bvh_morton(const float4* sites, int64_t n, const float* box_dev, uint64_t* keys, uint32_t* vals,
                       cudaStream_t st, int* launches) {
    k_morton<<<blocks(n, 256), 256, 0, st>>>(sites, n, box_dev, keys, vals);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t bvh_gather(const float4* sites, const uint32_t* perm, int64_t n, float4* sorted, int32_t* perm_i32,
                       cudaStream_t st, int* launches) {
    k_gather<<<blocks(n, 256), 256, 0, st>>>(sites, perm, n, sorted, perm_i32);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t bvh_topology(const uint64_t* keys_sorted, const float4* sorted, int n, int leaf, BvhScratch& sc, Bvh& out,
                         cudaStream_t st, int* launches) {
    cudaMemsetAsync(sc.counters, 0, sizeof(int) * kCollapseCounters, st);  // [1] is read back after the cells
    if (n <= 1) {
        k_root_single<<<1, 1, 0, st>>>(out.root);
        ++*launches;
        return cudaGetLastError();
    }
    k_karras<<<blocks(n - 1, 256), 256, 0, st>>>(keys_sorted, n, sc.child, sc.range, sc.parent_int, sc.parent_leaf);
    cudaMemsetAsync(sc.visit, 0, sizeof(int) * (size_t)(n - 1), st);
    k_refit<<<blocks(n, 256), 256, 0, st>>>(sorted, n, sc.child, sc.parent_int, sc.parent_leaf, sc.visit, sc.blo, sc.bhi);
    k_root<<<1, 1, 0, st>>>(sc.blo, sc.bhi, n, leaf, out.root, sc.tasks[0], sc.counters);
    *launches += 3;
    out.n_wide = 0;
    out.levels = 0;
    if (n <= leaf) return cudaGetLastError();
    // every collapse level in one cooperative launch (grid = co-resident blocks); no host round trip
    static int grid[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!grid[dev & 63]) {
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_collapse_all, 256, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        grid[dev & 63] = std::max(1, std::min(per_sm, 4)) * std::max(sms, 1);
    }
    int max_wide = sc.max_wide;
    void* args[] = {(void*)&sc.tasks[0], (void*)&sc.tasks[1], (void*)&sc.child, (void*)&sc.range, (void*)&sc.blo,
                    (void*)&sc.bhi, (void*)&sorted, (void*)&leaf, (void*)&out.nodes, (void*)&sc.counters,
                    (void*)&max_wide};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_collapse_all, dim3(grid[dev & 63]), dim3(256), args, 0, st);
    if (e != cudaSuccess) return e;
    ++*launches;
    out.levels = -1;  // not read back (the cell kernel never needs it)
    return cudaGetLastError();
}

}  // namespace pd
