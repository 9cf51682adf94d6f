// pd_cells.cu -- the cell kernel: one WARP per power cell, polyhedron kept on-chip (shared memory),
// best-first BVH traversal with a per-warp priority queue, directional culling, warp-parallel
// half-space clipping, and an FP64 finalize (face areas, volume).
//
// Paper mapping:
//   * cell = box, then clip by bisecting planes (§4.1; App. PAPER.md:548-558)
//   * bisector distance d_ij = (|p_i-p_j|^2 + w_i - w_j) / (2|p_i-p_j|)
//   * site culling d_ij > r_i with the directional radius of p_j's octant
//   * node culling with the max-weight lower bound
//   * best-first traversal, near child first, far child pushed if valid, pop + re-validate
//     (Alg. 1); unsorted queue with min-scan pop
//   * plane garbage collection at 85% occupancy
// B200 design (differs from the paper's thread-per-cell, global-memory state):
//   * a warp owns a cell; vertices (FP64 positions in site-local coordinates + plane-index triplets,
//     plus an FP32 copy) and planes live in shared memory;
//   * every classification runs in FP32 against a proven error margin and is certified in FP64 only
//     when |s| is within that margin, so each decision equals the FP64 predicate's (PAPER.md:872
//     runs FP32 only; SURVEY.md §7 "Precision");
//   * the hole of a clip is found without the serial circular list of PAPER.md:556: a removed
//     vertex's directed dual edge (x->y) is on the hole boundary iff no other removed vertex holds
//     (y->x); every boundary edge independently spawns the vertex (h, x, y);
//   * a leaf's candidates are culled and cut-tested in parallel (lane = candidate); planes that do
//     not cut the current cell are dropped for good (the cell only shrinks);
//   * the queue is re-validated in parallel at every pop, and spills to global memory when full;
//   * heavy cells switch on an exact polytope-vs-box node test;
//   * capacity tiers: cells that outgrow the tier's on-chip arrays are handed to a larger tier.
#include <cuda_runtime.h>
#include <stdint.h>
#include <assert.h>
#include <stdio.h>

#include <type_traits>

#include "pd_internal.cuh"

namespace pd {
namespace {

constexpr unsigned FULL = 0xffffffffu;
// Bounds checks of the on-chip arrays (a -DPD_CHECKS build: device asserts; tools/checks.sh runs the GPU parity
// tests under it).  Compiled out of the product build.
#ifdef PD_CHECKS
#define PD_ASSERT(c) assert(c)
#else
#define PD_ASSERT(c) (void)0
#endif

#ifndef PD_LAZY_POP_TOP
#define PD_LAZY_POP_TOP 1  // cooperative top tier: lazy pop (its queue is long; the plane-distance keys never go stale)
#endif
#ifndef PD_LAZY_POP
#define PD_LAZY_POP 0
#endif
#ifndef PD_BATCH_CUT
#define PD_BATCH_CUT 0
#endif
#ifndef PD_MATCH
#define PD_MATCH 1
#endif
#ifndef PD_CLEAN_POP
#define PD_CLEAN_POP 0  // tier 1: no re-validation at a pop when the cell has not changed since the last one (measured 10% slower on C4)
#endif
#ifndef PD_LAZY_COMPACT
#define PD_LAZY_COMPACT 0  // swap-remove the popped queue entry while >= 3/4 are alive (all tiers)
#endif
#ifndef PD_LEAF_AABB
#define PD_LEAF_AABB 1  // tier 1: the cell AABB refreshed once per leaf (after its clips), not after every clip (C4 -3%)
#endif
#ifndef PD_FUSED_AABB
#define PD_FUSED_AABB 1  // tier 1: the new AABB from the classification pass (measured 3.5% faster on C4)
#endif
#ifndef PD_INL_AABB
#define PD_INL_AABB __forceinline__
#endif
#ifndef PD_INL_CLIP
#define PD_INL_CLIP __forceinline__
#endif
#ifndef PD_INL_LEAF
#define PD_INL_LEAF __forceinline__
#endif
#ifndef PD_EXACT_LEAVES
#define PD_EXACT_LEAVES 0
#endif
#ifndef PD_EDGE_BITMAP
#define PD_EDGE_BITMAP 0
#endif
#ifndef PD_FAST_REJECT
#define PD_FAST_REJECT 0  // per candidate, FP32-only "can this plane cut at all" pass (superseded by the pre-test)
#endif
#ifndef PD_PRETEST
#define PD_PRETEST 1  // per leaf: every candidate against every vertex at once (lane = vertex), FP32 only
#endif
#ifndef PD_INL_EXACT
#define PD_INL_EXACT __noinline__  // the exact polytope-vs-box node test (rare unless PD_EXACT_LEAVES)
#endif
#ifndef PD_PK_CULL
#define PD_PK_CULL 1  // node bound (1) on the plane-distance lower bound (keeps w_i - w_max > 0) vs the radius
#endif
#ifndef PD_FIN_BATCH
#define PD_FIN_BATCH 0  // finalize_kernel (chunked): per-chunk batched loads of the record headers / sites / ids (no gain measured)
#endif
#ifndef PD_KEY_SMEM
#define PD_KEY_SMEM 1  // the leaf candidates' order keys in shared memory instead of a register held through clip()
#endif
#ifndef PD_FAST_RCP
#define PD_FAST_RCP 1  // solve3: 1/det by a MUFU seed + 2 Newton steps instead of the IEEE FP64 division
#endif
#ifndef PD_PARK
#define PD_PARK 1  // park the queue counts in shared memory across a leaf (lower register pressure)
#endif
#ifndef PD_FLAT_NODES
#define PD_FLAT_NODES 1  // descent: node tests on all 32 lanes (child lane & 7) instead of a lane < 8 branch
#endif
#ifndef PD_FLAT_CLASSIFY
#define PD_FLAT_CLASSIFY 1  // clip classification without divergent branches (certification behind a warp vote)
#endif
#ifndef PD_REFILTER
#define PD_REFILTER 0  // re-run the pre-test on a leaf's remaining candidates after each clip
#endif
#ifndef PD_REFILTER_MIN
#define PD_REFILTER_MIN 2  // ... when at least this many remain
#endif
#ifndef PD_VISITS_BY_WORK
#define PD_VISITS_BY_WORK 1  // exact node tests switch on by the work counter (work/16) instead of a visit counter
#endif
#define PD_VISITS(cnt) (PD_VISITS_BY_WORK ? (unsigned long long)((cnt).work >> 4) : (unsigned long long)(cnt).visited)
#ifndef PD_PRETEST_MIN
#define PD_PRETEST_MIN 1  // pre-test a leaf's candidates only when at least this many survive the site cull (2: 8% slower)
#endif
#ifndef PD_PRETEST_COMPACT
#define PD_PRETEST_COMPACT 1  // the pre-test's candidate planes packed by rank (no empty groups of 4)
#endif

template <int V, int P, int Q, int W, int MINB, bool GLOB = false, bool CO = false, bool SPH = false, bool F64 = true,
          bool FINAL = false>
struct TierCfg {
    // the state of finalize_kernel only: no clipping scratch (candidate planes, plane-GC map)
    static constexpr bool FIN = FINAL;
    // FP64 vertex copies in the state.  Tier 1 keeps none (its finalize is deferred to finalize_kernel, which
    // rebuilds every vertex from its plane triplet): the rare FP64 certification of an ambiguous FP32
    // classification re-solves the vertex from its three FP64 planes instead (same solve3, same operands).
    static constexpr bool F64V = F64;
    static constexpr bool GLOBAL = GLOB;     // warp state in global memory (top tier) instead of smem
    // CTA-cooperative cell (top tier): warp 0 runs the cell program, warps 1..W-1 join its O(V) passes
    static constexpr bool COOP = CO;
    // bounding-sphere companion of the site cull (tiers whose cells grow large; see site_culled)
    static constexpr bool SPHERE = SPH;
    using trip_t = typename std::conditional<(P <= 1024), uint32_t, uint64_t>::type;
    static constexpr int VMAX = V;   // vertices
    static constexpr int PMAX = P;   // planes (<= 1024: 10-bit triplet fields)
    static constexpr int QMAX = Q;   // on-chip priority-queue entries
    static constexpr int WARPS = W;  // warps per block
    static constexpr int MIN_BLOCKS = MINB;  // __launch_bounds__ residency target (register cap)
    static constexpr int VC = V / 32;
    static constexpr int QC = Q / 32;
    // hole edges via an XOR bitmap over unordered plane pairs when it is small enough
    static constexpr bool EDGE_BITMAP = PD_EDGE_BITMAP && P <= 256;
    static constexpr int EBW = EDGE_BITMAP ? (P * P + 31) / 32 : 1;
};

#ifndef PD_T1_MINB
#define PD_T1_MINB 7  // resident CTAs per SM (register cap 72, with the candidate keys in shared memory and no visit counter; 6: 80 registers, 0.5% slower on C4, 1.2% on C3; 5: 96 registers, 3% slower)
#endif
#ifndef PD_T1_WARPS
#define PD_T1_WARPS 4  // 1: one-warp CTAs (constant smem address) measured 9% lower issue efficiency on C4
#endif
#ifndef PD_T1_Q
#define PD_T1_Q 64
#endif
#ifndef PD_T1_V
#define PD_T1_V 96
#endif
#ifndef PD_T1_P
#define PD_T1_P 64
#endif
#ifndef PD_T1_SPHERE
#define PD_T1_SPHERE 0
#endif
#ifndef PD_T1_F64V
#define PD_T1_F64V 0
#endif
using Tier1 = TierCfg<PD_T1_V, PD_T1_P, PD_T1_Q, PD_T1_WARPS, PD_T1_MINB, false, false, PD_T1_SPHERE != 0, PD_T1_F64V != 0>;
// the state finalize_kernel rebuilds a deferred tier-1 cell into (with the FP64 vertices finalize() reads)
using Tier1F = TierCfg<PD_T1_V, PD_T1_P, PD_T1_Q, PD_T1_WARPS, PD_T1_MINB, false, false, PD_T1_SPHERE != 0, true, true>;
// Tier 2: one cell per CTA of 4 warps (state in shared memory, O(V) passes CTA-wide from 128 vertices):
// the few heavy cells of a light-weight workload (C4: 78) no longer run on one warp each, which
// mattered most for the per-rank critical path of sharded builds.
#ifndef PD_T2_COOP
#define PD_T2_COOP 0  // measured slower on C3/C4 (the heavy tier-2 cells are traversal-bound), kept as an option
#endif
#ifndef PD_T2_WARPS
#define PD_T2_WARPS 6  // warps (cells) per tier-2 CTA, one CTA per SM (35.6 KB of shared memory per warp; 4: C3 +7%)
#endif
using Tier2 = TierCfg<384, 192, 256, PD_T2_WARPS, PD_T2_COOP ? 4 : 1, false, PD_T2_COOP != 0, true>;
// Top tier: state in global memory (L1/L2-cached), 64-bit plane-index triplets; for the rare cells
// with thousands of faces (heavy-tailed weights, SURVEY.md §7 hard part 3).
// One cell per CTA: its 16 warps share every O(V) pass (classification, exact node tests, AABB,
// finalize) of the heavy cells (heavy-tailed weights: thousands of vertices).
#ifndef PD_T3_COOP
#define PD_T3_COOP 1
#endif
#ifndef PD_T3_WARPS
#define PD_T3_WARPS 16
#endif
using Tier3 = TierCfg<16384, 8192, 4096, PD_T3_COOP ? PD_T3_WARPS : 2, 1, true, PD_T3_COOP != 0, true>;
constexpr int kTier3BlocksPerSM = 1;

// Per-warp cell state (warp-uniform).  Lives in the warp's shared-memory block (read by broadcast):
// passing a register-resident struct by reference to non-inlined functions would put it on the
// thread stack (local memory), which thrashes L1 once shared memory takes the carveout.
struct Cell {
    double px, py, pz, pw;  // site (world), weight
    float fpx, fpy, fpz, fpw;
    float flo[3], fhi[3];   // cell AABB, site-local, rounded outward
    float glo[3], ghi[3];   // the same box grown to contain the site: min(flo, 0), max(fhi, 0) (node bound (2))
    float flo2[3], fhi2[3]; // flo^2, fhi^2 (the directional radius of node bound (1))
    float vmax;             // max_k max(|lo_k|, |hi_k|)
    float sc[3], srad;      // bounding sphere of the cell (SPHERE tiers): center (site-local), radius
    int nv, np, nq;
    int degraded;           // a topology-consistency check failed (PD_CELL_DEGRADED)
    int t_nq, t_ns;         // traversal state parked across a leaf (PD_PARK)
    int self;               // Morton index
    int self_orig;
};

template <class T>
struct __align__(16) WarpState {
    Cell c;                       // warp-uniform cell state
    double4 pl[T::PMAX];          // plane n.y <= d (n = p_j - p_i, local coordinates), exact
    float4 fv[T::VMAX];           // FP32 copy of the vertex positions (x, y, z, 0)
    double vx[T::F64V ? T::VMAX : 1], vy[T::F64V ? T::VMAX : 1], vz[T::F64V ? T::VMAX : 1];
    typename T::trip_t vt[T::VMAX];  // plane-index triplet (a, b, c), CCW seen from outside
    int32_t pid[T::PMAX];         // >= 0 Morton index of the neighbour site; -1-k box wall k
    union {
        struct {                  // traversal: priority queue of pushed child records
            float4 qlo[T::QMAX];  // (lo, maxw)
            float4 qhi[T::QMAX];  // (hi, link)
            float qkey[(PD_LAZY_POP || PD_CLEAN_POP || (PD_LAZY_POP_TOP && T::COOP)) ? T::QMAX : 1];  // priority
        };
        struct {                  // finalize (the queue is dead by then)
            union {
                uint16_t tw[3][T::VMAX];     // twin vertex across edges a->b, b->c, c->a
                uint16_t flist[3 * T::VMAX]; // face walk (tier 1): vertices bucketed by face, u | y << 7
            };
            union {
                uint32_t etab[256];   // edge hash (tier 1): unordered plane pair -> its two vertices
                struct {
                    union {
                        struct {
                            int32_t nb_id[T::PMAX];   // neighbour staging
                            float nb_area[T::PMAX];
                        };
                        struct {                      // face walk: per-face CSR offsets and fill cursors
                            uint32_t fcnt[T::PMAX];
                            uint32_t ffill[T::PMAX];
                        };
                    };
                    double farea[T::PMAX];    // face areas
                };
            };
        };
    };
    uint16_t rem[T::VMAX];        // removed-vertex slots of the current clip
    uint32_t omask[T::VC];        // outside-vertex ballots of the current clip
    uint32_t qmask[T::QC];        // alive-entry ballots of the current pop
    uint32_t bnd[T::VMAX];        // boundary edges (x | y << 16) of the current clip (B <= VMAX unless overflow)
    uint16_t pmap[T::FIN ? 1 : T::PMAX];  // plane GC remap
    float4 cpl[T::FIN ? 1 : 32];  // a leaf's candidates, by rank: FP32 plane (D = p_j - p_i, dd = q/2)
    __align__(16) float cmg[T::FIN ? 4 : 32];  //   and its certification margin (kept in smem, not registers, through clip())
    int ckey[(T::FIN || !PD_KEY_SMEM) ? 1 : 32];  // the candidates' order keys (PD_KEY_SMEM), by slot
    uint32_t ebits[T::EBW];       // hole-edge parity bitmap (zero between clips)
};

__device__ __forceinline__ int ford(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float iford(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

// Plane-index triplets: 10-bit fields in a u32 (<= 1024 planes) or 21-bit fields in a u64.
template <class TR>
__device__ __forceinline__ TR tpack(int a, int b, int c);
template <>
__device__ __forceinline__ uint32_t tpack<uint32_t>(int a, int b, int c) {
    return (uint32_t)a | ((uint32_t)b << 10) | ((uint32_t)c << 20);
}
template <>
__device__ __forceinline__ uint64_t tpack<uint64_t>(int a, int b, int c) {
    return (uint64_t)a | ((uint64_t)b << 21) | ((uint64_t)c << 42);
}
__device__ __forceinline__ int ta(uint32_t t) { return t & 1023; }
__device__ __forceinline__ int tb(uint32_t t) { return (t >> 10) & 1023; }
__device__ __forceinline__ int tc(uint32_t t) { return (t >> 20) & 1023; }
__device__ __forceinline__ int ta(uint64_t t) { return (int)(t & 0x1fffff); }
__device__ __forceinline__ int tb(uint64_t t) { return (int)((t >> 21) & 0x1fffff); }
__device__ __forceinline__ int tc(uint64_t t) { return (int)((t >> 42) & 0x1fffff); }
// does triplet t contain the directed dual edge x->y ?
template <class TR>
__device__ __forceinline__ bool has_edge(TR t, int x, int y) {
    int a = ta(t), b = tb(t), c = tc(t);
    return (a == x && b == y) || (b == x && c == y) || (c == x && a == y);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Global-space atomics (the generic atomicAdd emits a shared/global runtime dispatch).
__device__ __forceinline__ void red_add_g(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_g(unsigned long long* p, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ int atom_add_g32(int* p, int v) {
    int old;
    asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// Compile-time culling/traversal mode.  Tier 1 is instantiated per common mode so that the default
// kernel carries none of the ablation branches (instruction-fetch stalls dominate otherwise);
// kDynMode reads the mode bits from the runtime flags (mode combinations, tiers 2-3).
constexpr unsigned kModeBits = PD_ISOTROPIC | PD_DFS | PD_PAPER_BOUND | PD_EXACT_NODES | PD_NO_EXACT | PD_WARM_START;
constexpr unsigned kDynMode = 0xffffffffu;
template <unsigned MODE>
__device__ __forceinline__ unsigned mode_flags(unsigned runtime_flags) {
    return MODE == kDynMode ? runtime_flags : ((MODE & kModeBits) | (runtime_flags & ~kModeBits));
}
template <unsigned MODE>
constexpr bool kStats = MODE == kDynMode || (MODE & PD_STATS) != 0;  // u64 pd_stats counters compiled in

// Exact node tests switch on once a cell has visited `after` nodes (heavy cells), or always with
// PD_EXACT_NODES; PD_NO_EXACT disables them.
__device__ __forceinline__ bool exact_on(unsigned flags, unsigned long long visited, int after) {
    if (flags & PD_NO_EXACT) return false;
    return (flags & PD_EXACT_NODES) || visited > (unsigned long long)after;
}

enum { ST_OK = 0, ST_EMPTY = 1, ST_OVERFLOW = 2, ST_DUP = 3 };
enum { CLIP_NONE = 0, CLIP_DONE = 1, CLIP_EMPTY = 2, CLIP_OVF = 3 };

#ifndef PD_PROFILE
#define PD_PROFILE 0
#endif
// Work counters.  The u64 totals (pd_stats) are compiled in only for kernels instantiated with PD_STATS (or the
// generic-mode kernels of the higher tiers): in the default tier-1 kernel they would hold ~12 registers across
// the whole cell program.  `work` (nodes + sites + 8 clips of the current cell: PD_COST, the longest-first
// order of the next tier) and `visited` (nodes of the current cell: the exact-test switch) are always kept.
struct Counters {
    unsigned long long nodes, leaves, sites, tests, clips, spills;
    unsigned work, visited;             // per cell
    unsigned ncl;                       // clips so far (running; the traversal compares it across a leaf)
#if PD_PROFILE
    unsigned long long cyc[10];  // init, descend, leaf, clip, pop, finalize | clip: classify, boundary, create, aabb
#endif
};
#if PD_PROFILE
#define PT_BEGIN(v) long long v = clock64()
#define PT_END(v, k) cnt.cyc[k] += (unsigned long long)(clock64() - v)
#else
#define PT_BEGIN(v) (void)0
#define PT_END(v, k) (void)0
#endif


// An FP32 plane with its certification margin: |s32 - s| <= err < m for s = n.v - d evaluated in
// FP32 from the FP32 copies (all inputs carry <= 2^-24 relative rounding; the FMA chain adds a few
// more).  m = 1e-6 (|n|_1 vmax + |D|^2 + |w_i - w_j|) is > 8x the worst-case error.
struct FPlane {
    float nx, ny, nz, d, m;
};
// FP64 certification tolerance 1e-12 |n| R (reading R9), in FP32; only evaluated on the rare certification path.
#ifndef PD_FAST_SQRT
#define PD_FAST_SQRT 0  // bounds' square roots by MUFU.RSQ, rounded up (measured no different on C2-C5; IEEE sqrtf kept)
#endif
// sqrt for the culling bounds (1e-5 relative margins): x * rsqrt(x) is within a few ulp; x (1 + 1e-6) covers it
__device__ __forceinline__ float sqrt_up(float x) {
    if (!PD_FAST_SQRT) return sqrtf(x);
    return x > 0.f ? x * rsqrtf(x) * (1.f + 1e-6f) : 0.f;
}
// Max corner distance of the cell AABB (the isotropic radius R of P:211 and the scale of the FP64 certification
// tolerance, R9): computed where it is used (rarely: certification, isotropic ablation) from the stored AABB.
__device__ __forceinline__ float cell_r2(const Cell& c) {
    float rm2 = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) rm2 += fmaxf(c.flo[k] * c.flo[k], c.fhi[k] * c.fhi[k]);
    return rm2;
}
__device__ __forceinline__ float cell_rmax(const Cell& c) { return sqrt_up(cell_r2(c)); }
__device__ __forceinline__ float cert_tol(const FPlane& f, float rmax) {
    const float f2 = f.nx * f.nx + f.ny * f.ny + f.nz * f.nz;
    return 1e-12f * (f2 * rsqrtf(f2)) * rmax;
}

// r^2 of the directional radius for an octant set (one corner per octant is
// sound).  allow bit 2k: + side on axis k; bit 2k+1: - side.
__device__ __forceinline__ float dir_r2(const Cell& c, unsigned allow, bool iso) {
    float r2 = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float h2 = c.fhi2[k], l2 = c.flo2[k];
        float a = (iso || (allow & (1u << (2 * k)))) ? h2 : 0.f;
        float b = (iso || (allow & (2u << (2 * k)))) ? l2 : 0.f;
        r2 += fmaxf(a, b);
    }
    return r2;
}

// Node test.  Two sound culls, a node is discarded if EITHER holds (FP32, 1e-5 relative margins so
// rounding can only keep a node):
//  (1) the paper's: the lower bound d/2 + min(0, w_i - w_max)/(2d) on d_ij over
//      the box exceeds the directional radius r of the octants the box occupies, i.e.
//      d^2 + min(0, w_i - w_max) - 2 r d > 0;
//  (2) a companion bound from the same cell AABB: for p_j in B and y in the cell,
//      y.D <= H = sum_k max(lo_k a_k, lo_k b_k, hi_k a_k, hi_k b_k) with D_k in [a_k, b_k] (the box
//      minus p_i), while the plane offset is (|D|^2 + w_i - w_j)/2 >= (d^2 + w_i - w_max)/2;
//      so no plane of B cuts the cell if d^2 + w_i - w_max > 2H.  (2) is never looser than (1) for
//      small far boxes (Cauchy-Schwarz) and is disabled by PD_PAPER_BOUND / PD_ISOTROPIC.
// Returns the Alg. 1 priority delta = NodeSqrDist - r^2 (+ the weight term): order only.
#ifndef PD_NODE_KEY
#define PD_NODE_KEY 0  // default mode's queue priority: 0 Alg. 1's d^2 + min(0,dw) - r^2 (with bound (1)); 1 d^2 + min(0,dw)
#endif
// Priority (order only, the diagram is unchanged) with PK: a lower bound on the plane distance
// d_ij = (|D|^2 + w_i - w_j) / (2|D|) of the node's sites (|D| >= d, w_j <= w_max).  As a function of
// t = |D| it is minimal at t = sqrt(w_i - w_j) when w_i > w_j: the nearest planes of a heavy site come from
// sites at distance ~sqrt(dw), not from the nearest boxes, so Alg. 1's distance order clips a heavy cell with
// thousands of planes that later ones supersede.  Equal weights: d/2, the same order as d^2.
#ifndef PD_PLANE_KEY
#define PD_PLANE_KEY 2  // 0: Alg. 1's priority everywhere; 1: plane-distance bound in tiers 2-3; 2: in every tier
#endif
__device__ __forceinline__ float plane_key(float d2, float dw) {
    // branch-free, one MUFU.RSQ: m = max(d2, dw) is d2 unless d2 < dw (then the bound is sqrt(dw) = dw / sqrt(dw));
    // d2 = 0 with dw <= 0 gives a huge negative value (the bound is -inf there; 0 when dw = 0 too)
    const float m = fmaxf(fmaxf(d2, dw), 1e-30f);
    const float rs = rsqrtf(m);
    return d2 < dw ? dw * rs : 0.5f * (d2 + dw) * rs;
}
template <bool PK = false>
__device__ __forceinline__ float node_test(const Cell& c, float4 lo_w, float4 hi_l, unsigned flags, bool& culled) {
    const bool iso = (flags & PD_ISOTROPIC) != 0;
    const bool paper = (flags & (PD_PAPER_BOUND | PD_ISOTROPIC)) != 0;
    float a0 = lo_w.x - c.fpx, a1 = lo_w.y - c.fpy, a2 = lo_w.z - c.fpz;
    float b0 = hi_l.x - c.fpx, b1 = hi_l.y - c.fpy, b2 = hi_l.z - c.fpz;
    float g0 = fmaxf(fmaxf(a0, -b0), 0.f), g1 = fmaxf(fmaxf(a1, -b1), 0.f), g2 = fmaxf(fmaxf(a2, -b2), 0.f);
    float d2 = g0 * g0 + g1 * g1 + g2 * g2;
    if (PD_NODE_KEY == 1 && !paper) {
        // the AABB-support bound (2) alone: it is the tighter one wherever a node is near the cell, and the
        // paper's (1) costs a directional radius and a square root per node (culling only; output identical)
        const float dw = c.fpw - lo_w.w;
        const float h0 = fmaxf(fmaxf(c.flo[0] * a0, c.flo[0] * b0), fmaxf(c.fhi[0] * a0, c.fhi[0] * b0));
        const float h1 = fmaxf(fmaxf(c.flo[1] * a1, c.flo[1] * b1), fmaxf(c.fhi[1] * a1, c.fhi[1] * b1));
        const float h2 = fmaxf(fmaxf(c.flo[2] * a2, c.flo[2] * b2), fmaxf(c.fhi[2] * a2, c.fhi[2] * b2));
        const float H = h0 + h1 + h2;
        const float mag = c.vmax * (fmaxf(fabsf(a0), fabsf(b0)) + fmaxf(fabsf(a1), fabsf(b1)) + fmaxf(fabsf(a2), fabsf(b2)));
        culled = d2 + dw - 2.f * H > 1e-5f * (d2 + fabsf(dw) + 2.f * mag);
        return PK ? plane_key(d2, dw) : d2 + fminf(0.f, dw);
    }
    unsigned allow = (b0 >= 0.f ? 1u : 0u) | (a0 <= 0.f ? 2u : 0u) | (b1 >= 0.f ? 4u : 0u) | (a1 <= 0.f ? 8u : 0u) |
                     (b2 >= 0.f ? 16u : 0u) | (a2 <= 0.f ? 32u : 0u);
    float dw = c.fpw - lo_w.w;
    float dwn = fminf(0.f, dw);
    float r2 = dir_r2(c, allow, iso);
    float pk = 0.f;
    if (PD_PK_CULL && PK && !paper) {
        // (1) with the plane-distance bound of the priority, which keeps a positive w_i - w_max (the paper's
        // d/2 + min(0, dw)/(2d) drops it): no site of the node has a plane nearer than pk, and no point of the
        // cell is farther than r in the node's octants -- cull iff pk > r
        pk = plane_key(d2, dw);
        const float r = r2 > 0.f ? r2 * rsqrtf(r2) * (1.f + 1e-6f) : 0.f;  // within the 1e-5 margin
        culled = pk - r > 1e-5f * (fabsf(pk) + r);
    } else {
        float rd = sqrt_up(r2 * d2);
        culled = d2 + dwn - 2.f * rd > 1e-5f * (d2 - dwn + 2.f * rd);
    }
    if (!paper) {
        // max over y in the box grown to contain the site (glo <= 0 <= ghi) and D_k in [a_k, b_k] of y_k D_k:
        // with glo <= 0, glo a >= glo b; with ghi >= 0, ghi b >= ghi a -- two products per axis, not four
        float h0 = fmaxf(c.glo[0] * a0, c.ghi[0] * b0);
        float h1 = fmaxf(c.glo[1] * a1, c.ghi[1] * b1);
        float h2 = fmaxf(c.glo[2] * a2, c.ghi[2] * b2);
        float H = h0 + h1 + h2;
        float mag = c.vmax * (fmaxf(fabsf(a0), fabsf(b0)) + fmaxf(fabsf(a1), fabsf(b1)) + fmaxf(fabsf(a2), fabsf(b2)));
        culled |= d2 + dw - 2.f * H > 1e-5f * (d2 + fabsf(dw) + 2.f * mag);
    }
    if (PK && PD_PLANE_KEY == 3) return plane_key(d2, dw) - sqrtf(r2);  // the nearest plane's depth in the cell
    if (PD_PK_CULL && PK && !paper) return pk;
    if (PK) return plane_key(d2, dw);
    return d2 + dwn - r2;
}
template <class T>
constexpr bool kCleanPop = PD_CLEAN_POP && !PD_LAZY_POP && !T::COOP;
// Lazy pop (the paper's): pop the least key, test only that entry.  With the plane-distance keys (which
// do not depend on the cell) the order is exact; dead entries are found one at a time when they reach the top.
// Measured slower in tier 1 (short queues, many dead entries), used in the cooperative top tier (long queues).
template <class T>
constexpr bool kLazyPop = PD_LAZY_POP || (PD_LAZY_POP_TOP && T::COOP && (PD_PLANE_KEY >= 1));
template <class T>
constexpr bool kPlaneKey = PD_PLANE_KEY >= 2 || (PD_PLANE_KEY == 1 && T::SPHERE);

// ---------------------------------------------------------------- CTA-cooperative passes (top tier)
// Warp 0 of a COOP CTA runs the cell program; at an O(V) pass it publishes a job in shared memory and
// meets warps 1..W-1 at named barrier 1, every warp takes a strided share of the vertex (or face)
// slots, and all meet again at barrier 2, after which warp 0 combines the per-warp partials in a fixed
// order (so the result is deterministic).
enum { JOB_EXIT = 0, JOB_CLASSIFY = 1, JOB_EXACT = 2, JOB_AABB = 3, JOB_TWINS = 4, JOB_AREAS = 5, JOB_BATCH = 6,
       JOB_REVAL = 7 };
constexpr int kCoopMaxW = 32;
struct CoopJob {
    int kind, nv, np;
    int min_v;  // passes over fewer vertices stay on warp 0 (CellParams::coop_min_v)
    unsigned mask;
    FPlane f;
    float4 sj;
    float4 lo[WIDE], hi[WIDE];
    int ipart[kCoopMaxW][WIDE];
    double dpart[kCoopMaxW][2];
    unsigned flags;     // JOB_REVAL: culling mode
    int nq;             // JOB_REVAL: queue length
    float4 cD[32];      // JOB_BATCH: candidate planes (D, d) of a leaf, lane = candidate,
    float cm[32];       //            their FP32 certification margins
    float4 csj[32];     //            and sites (for the FP64 certification of ambiguous vertices)
};
extern __shared__ __align__(16) unsigned char pd_smem[];
__device__ __forceinline__ CoopJob& coop_job() { return *reinterpret_cast<CoopJob*>(pd_smem); }
template <class T>
__device__ __forceinline__ int P_coop_min_v(const WarpState<T>&) { return coop_job().min_v; }
// Cooperative tier: the priority queue lives in shared memory after the job record.
template <class T>
__device__ __forceinline__ float4* coop_queue_lo() { return reinterpret_cast<float4*>(pd_smem + ((sizeof(CoopJob) + 15) & ~15)); }
template <class T>
__device__ __forceinline__ float4* coop_queue_hi() { return coop_queue_lo<T>() + T::QMAX; }
template <class T>
__device__ __forceinline__ uint32_t* coop_queue_mask() { return reinterpret_cast<uint32_t*>(coop_queue_hi<T>() + T::QMAX); }
template <class T>
constexpr size_t coop_smem_bytes() { return ((sizeof(CoopJob) + 15) & ~(size_t)15) + 2 * sizeof(float4) * T::QMAX + 4 * T::QC; }
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    // barrier.sync (not the .aligned bar.sync): legal where the compiler has not reconverged the warp
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Exact polytope-vs-box node test (not in the paper; strictly tighter than any AABB bound).  The
// plane of p_j (D = p_j - p_i) cuts the cell iff some vertex v has v.D - |D|^2/2 > (w_i - w_j)/2.
// Over all p_j in the box, D_k in [a_k, b_k] and w_j <= w_max, and
//   max_{D in box} (v.D - |D|^2/2) = sum_k (v_k c_k - c_k^2/2),  c_k = clamp(v_k, a_k, b_k),
// (a separable concave maximisation), so the node is culled iff for every vertex that sum is
// <= (w_i - w_max)/2.  Lanes = vertices, FP32 with a 1e-5 relative margin (only keeps nodes).
__device__ __forceinline__ float exact_partial(const float4* fv, const Cell& c, float4 lo_w, float4 hi_l, int s0, int nv,
                                               int stride) {
    const float a0 = lo_w.x - c.fpx, a1 = lo_w.y - c.fpy, a2 = lo_w.z - c.fpz;
    const float b0 = hi_l.x - c.fpx, b1 = hi_l.y - c.fpy, b2 = hi_l.z - c.fpz;
    float best = -INFINITY;
    for (int s = s0; s < nv; s += stride) {
        float4 v = fv[s];
        float cx = fminf(fmaxf(v.x, a0), b0), cy = fminf(fmaxf(v.y, a1), b1), cz = fminf(fmaxf(v.z, a2), b2);
        best = fmaxf(best, cx * (v.x - 0.5f * cx) + cy * (v.y - 0.5f * cy) + cz * (v.z - 0.5f * cz));
    }
    return best;
}
__device__ __forceinline__ bool exact_decide(const Cell& c, float4 lo_w, float4 hi_l, float best) {
    const float a0 = lo_w.x - c.fpx, a1 = lo_w.y - c.fpy, a2 = lo_w.z - c.fpz;
    const float b0 = hi_l.x - c.fpx, b1 = hi_l.y - c.fpy, b2 = hi_l.z - c.fpz;
    const float B0 = fmaxf(fabsf(a0), fabsf(b0)), B1 = fmaxf(fabsf(a1), fabsf(b1)), B2 = fmaxf(fabsf(a2), fabsf(b2));
    const float mag = B0 * (c.vmax + B0) + B1 * (c.vmax + B1) + B2 * (c.vmax + B2) + fabsf(c.fpw) + fabsf(lo_w.w);
    return best < 0.5f * (c.fpw - lo_w.w) - 1e-5f * mag;
}

template <class T>
__device__ __forceinline__ void coop_run(WarpState<T>& S, CoopJob& J, int w, int lane);

// warp 0: run the published job with all warps of the CTA
template <class T>
__device__ __forceinline__ void coop_go(WarpState<T>& S, CoopJob& J, int lane) {
    __syncwarp();
    named_bar(1, T::WARPS * 32);
    coop_run<T>(S, J, 0, lane);
    named_bar(2, T::WARPS * 32);
}

template <class T>
__device__ PD_INL_EXACT bool node_exact_culled(const WarpState<T>& S, const Cell& c, int lane, float4 lo_w, float4 hi_l) {
    float best;
    if (T::COOP && c.nv >= P_coop_min_v(S)) {
        CoopJob& J = coop_job();
        if (lane == 0) { J.kind = JOB_EXACT; J.nv = c.nv; J.mask = 1u; J.lo[0] = lo_w; J.hi[0] = hi_l; }
        coop_go<T>(const_cast<WarpState<T>&>(S), J, lane);
        int b = lane < T::WARPS ? J.ipart[lane][0] : ford(-INFINITY);
        best = iford(__reduce_max_sync(FULL, b));
    } else {
        best = exact_partial(S.fv, c, lo_w, hi_l, lane, c.nv, 32);
        best = iford(__reduce_max_sync(FULL, ford(best)));
    }
    return exact_decide(c, lo_w, hi_l, best);
}

// Per-lane partial AABB of vertex positions (FP32 copies).
struct Box6 {
    float lo0, lo1, lo2, hi0, hi1, hi2;
    __device__ __forceinline__ void reset() {
        lo0 = lo1 = lo2 = INFINITY;
        hi0 = hi1 = hi2 = -INFINITY;
    }
    __device__ __forceinline__ void add(float4 v) {
        lo0 = fminf(lo0, v.x); hi0 = fmaxf(hi0, v.x);
        lo1 = fminf(lo1, v.y); hi1 = fmaxf(hi1, v.y);
        lo2 = fminf(lo2, v.z); hi2 = fmaxf(hi2, v.z);
    }
};

// Warp-reduce the partial boxes into the cell AABB (widened by 2 ulp) and its radius bounds.
__device__ __forceinline__ void finish_aabb(Cell& c, const Box6& b) {
    float lo[3], hi[3];
    lo[0] = iford(__reduce_min_sync(FULL, ford(b.lo0)));
    lo[1] = iford(__reduce_min_sync(FULL, ford(b.lo1)));
    lo[2] = iford(__reduce_min_sync(FULL, ford(b.lo2)));
    hi[0] = iford(__reduce_max_sync(FULL, ford(b.hi0)));
    hi[1] = iford(__reduce_max_sync(FULL, ford(b.hi1)));
    hi[2] = iford(__reduce_max_sync(FULL, ford(b.hi2)));
    float vm = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        // the FP32 copies are rounded to nearest: widen by 2 ulp so the box contains the FP64 cell
        lo[k] -= fabsf(lo[k]) * 2.4e-7f + 1e-30f;
        hi[k] += fabsf(hi[k]) * 2.4e-7f + 1e-30f;
        vm = fmaxf(vm, fmaxf(-lo[k], hi[k]));
    }
    // every lane writes the same warp-uniform fields: no lane may still be reading the old ones, and all
    // writes land before any lane reads the new ones
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        c.flo[k] = lo[k]; c.fhi[k] = hi[k];
        c.glo[k] = fminf(lo[k], 0.f); c.ghi[k] = fmaxf(hi[k], 0.f);
        c.flo2[k] = lo[k] * lo[k]; c.fhi2[k] = hi[k] * hi[k];
    }
    c.vmax = vm;
    __syncwarp();
}

// Cell AABB (and, in SPHERE tiers, a bounding sphere centred at the previous AABB's centre: any
// fixed centre gives a valid sphere, and the previous box is known before the pass).
template <class T>
__device__ PD_INL_AABB void update_aabb(const WarpState<T>& S, Cell& c, int lane) {
    Box6 b;
    b.reset();
    float m0 = 0.f, m1 = 0.f, m2 = 0.f, r2 = 0.f;
    if (T::SPHERE) {
        m0 = 0.5f * (c.flo[0] + c.fhi[0]); m1 = 0.5f * (c.flo[1] + c.fhi[1]); m2 = 0.5f * (c.flo[2] + c.fhi[2]);
    }
    if (T::COOP && c.nv >= P_coop_min_v(S)) {
        CoopJob& J = coop_job();
        if (lane == 0) { J.kind = JOB_AABB; J.nv = c.nv; J.lo[0] = make_float4(m0, m1, m2, 0.f); }
        coop_go<T>(const_cast<WarpState<T>&>(S), J, lane);
        if (lane < T::WARPS) {
            b.lo0 = iford(J.ipart[lane][0]); b.lo1 = iford(J.ipart[lane][1]); b.lo2 = iford(J.ipart[lane][2]);
            b.hi0 = iford(J.ipart[lane][3]); b.hi1 = iford(J.ipart[lane][4]); b.hi2 = iford(J.ipart[lane][5]);
            r2 = iford(J.ipart[lane][6]);
        }
    } else {
        for (int s = lane; s < c.nv; s += 32) {
            const float4 v = S.fv[s];
            b.add(v);
            if (T::SPHERE) {
                const float dx = v.x - m0, dy = v.y - m1, dz = v.z - m2;
                r2 = fmaxf(r2, dx * dx + dy * dy + dz * dz);
            }
        }
    }
    if (T::SPHERE) r2 = iford(__reduce_max_sync(FULL, ford(r2)));
    finish_aabb(c, b);
    if (T::SPHERE) {
        // FP32 vertex copies are within 2^-24 |v| of the FP64 cell: 1e-6 vmax covers it
        c.sc[0] = m0; c.sc[1] = m1; c.sc[2] = m2;
        c.srad = sqrtf(r2) * (1.f + 1e-6f) + 1e-6f * c.vmax;
        __syncwarp();
    }
}

template <class T>
__device__ __forceinline__ void put_vertex(WarpState<T>& S, int s, double x, double y, double z) {
    float4* fv = S.fv;
    if (T::F64V) { S.vx[s] = x; S.vy[s] = y; S.vz[s] = z; }
    fv[s] = make_float4((float)x, (float)y, (float)z, 0.f);
}

// Plane garbage collection: drop planes no vertex references.
template <class T>
__device__ __noinline__ void plane_gc(WarpState<T>& S, Cell& c, int lane) {
    const int np0 = c.np, nv0 = c.nv;
    for (int f = lane; f < np0; f += 32) S.pmap[f] = 0;
    __syncwarp();
    for (int s = lane; s < nv0; s += 32) {
        auto t = S.vt[s];
        S.pmap[ta(t)] = 1; S.pmap[tb(t)] = 1; S.pmap[tc(t)] = 1;
    }
    __syncwarp();
    int base = 0;
    for (int f0 = 0; f0 < np0; f0 += 32) {
        int f = f0 + lane;
        bool live = f < np0 && S.pmap[f];
        unsigned m = __ballot_sync(FULL, live);
        int dst = base + __popc(m & lanemask_lt());
        double4 pl;
        int id = 0;
        if (live) { pl = S.pl[f]; id = S.pid[f]; }
        __syncwarp();
        if (live) { S.pl[dst] = pl; S.pid[dst] = id; S.pmap[f] = (uint16_t)dst; }
        __syncwarp();
        base += __popc(m);
    }
    __syncwarp();
    for (int s = lane; s < nv0; s += 32) {
        auto t = S.vt[s];
        S.vt[s] = tpack<typename T::trip_t>(S.pmap[ta(t)], S.pmap[tb(t)], S.pmap[tc(t)]);
    }
    c.np = base;
    __syncwarp();
}

// Vertex of three planes n.y = d (Cramer's rule), staged so that only one cross product is live at a time
// (register pressure of the inlined hot loop): x = (a.w (b x c) + b.w (c x a) + c.w (a x b)) / (a . (b x c)).
__device__ __forceinline__ void solve3(const double4* pl, int ia, int ib, int ic, double& x, double& y, double& z) {
    const double4 b = pl[ib], c = pl[ic];
    double det;
    {
        const double bcx = b.y * c.z - b.z * c.y, bcy = b.z * c.x - b.x * c.z, bcz = b.x * c.y - b.y * c.x;
        const double4 a = pl[ia];
        det = a.x * bcx + a.y * bcy + a.z * bcz;
        x = a.w * bcx; y = a.w * bcy; z = a.w * bcz;
    }
    {
        const double4 a = pl[ia];
        const double cax = c.y * a.z - c.z * a.y, cay = c.z * a.x - c.x * a.z, caz = c.x * a.y - c.y * a.x;
        x += b.w * cax; y += b.w * cay; z += b.w * caz;
        const double abx = a.y * b.z - a.z * b.y, aby = a.z * b.x - a.x * b.z, abz = a.x * b.y - a.y * b.x;
        x += c.w * abx; y += c.w * aby; z += c.w * abz;
    }
    double inv;
    if (PD_FAST_RCP) {
        // MUFU reciprocal seed + two Newton steps (quadratic convergence: full FP64 precision, within 1 ulp of
        // 1/det) instead of the IEEE division sequence; the same function builds every vertex everywhere
        // (clip, certification, finalize_kernel), so all FP64 positions stay consistent
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(det));
        inv = fma(inv, fma(-det, inv, 1.0), inv);
        inv = fma(inv, fma(-det, inv, 1.0), inv);
    } else {
        inv = 1.0 / det;
    }
    x *= inv; y *= inv; z *= inv;
}

#ifndef PD_SOLVE_OOL
#define PD_SOLVE_OOL 0  // the new vertices' FP64 solve out of line (measured: not the register peak; kept off)
#endif
__device__ __noinline__ void solve3_ool(const double4* pl, int ia, int ib, int ic, double& x, double& y, double& z) {
    solve3(pl, ia, ib, ic, x, y, z);
}

// FP64 position of vertex slot s: the stored copy, or (tiers without FP64 copies) re-solved from its plane
// triplet exactly as it was created (solve3 on the same FP64 planes: the same value; box corners are exact).
template <class T>
__device__ __forceinline__ void vertex64(const WarpState<T>& S, int s, double& x, double& y, double& z) {
    if (T::F64V) {
        x = S.vx[s]; y = S.vy[s]; z = S.vz[s];
    } else {
        const auto t = S.vt[s];
        solve3(S.pl, ta(t), tb(t), tc(t), x, y, z);
    }
}

// Clip the cell by {y : n.y <= d} (re-designed warp-parallel).
__device__ __forceinline__ double4 exact_plane(const Cell& c, float4 sj) {
    // the exact FP64 plane of candidate site sj: n = p_j - p_i, d = (|n|^2 + w_i - w_j)/2
    double ex = (double)sj.x - c.px, ey = (double)sj.y - c.py, ez = (double)sj.z - c.pz;
    return make_double4(ex, ey, ez, 0.5 * (ex * ex + ey * ey + ez * ez + (c.pw - (double)sj.w)));
}

// Removed-vertex slots (ascending) from the per-chunk outside ballots; returns their number.
template <class T>
__device__ __noinline__ int rem_from_omask(WarpState<T>& S, int nch, int lane) {
    int R = 0;
    for (int c0 = 0; c0 < nch; c0 += 32) {
        const int ch = c0 + lane;
        unsigned m = ch < nch ? S.omask[ch] : 0u;
        const int k = __popc(m);
        int inc = k;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += v;
        }
        int off = R + inc - k;
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            S.rem[off++] = (uint16_t)(ch * 32 + b);
        }
        R += __shfl_sync(FULL, inc, 31);
    }
    __syncwarp();
    return R;
}

// FP64 certification of one vertex whose FP32 classification fell within the margin (rare):
// outside <=> n.v - d > tol in FP64 (R9/R10); the tolerance comes precomputed with the plane so the
// hot loop carries no FP64 set-up.
__device__ __forceinline__ bool outside_fp64(const Cell& c, float4 sj, const FPlane& f, double vx, double vy, double vz) {
    const double4 pe = exact_plane(c, sj);
    return fma(pe.x, vx, fma(pe.y, vy, pe.z * vz)) - pe.w > (double)cert_tol(f, cell_rmax(c));
}

// The FP64 certification of an ambiguous FP32 classification (rare).  Out of line in the tiers without FP64
// vertex copies: re-solving the vertex must not add its FP64 registers to the inlined hot loop's pressure.
template <class T>
__device__ __noinline__ bool outside_cert_solve(const WarpState<T>& S, const Cell& c, float4 sj, FPlane f, int s) {
    double x, y, z;
    vertex64(S, s, x, y, z);
    return outside_fp64(c, sj, f, x, y, z);
}
template <class T>
__device__ __forceinline__ bool outside_cert(const WarpState<T>& S, const Cell& c, float4 sj, const FPlane& f, int s) {
    if (T::F64V) return outside_fp64(c, sj, f, S.vx[s], S.vy[s], S.vz[s]);
    return outside_cert_solve(S, c, sj, f, s);
}

template <class T>
constexpr bool kLeafAabb = PD_LEAF_AABB && !T::COOP && !T::SPHERE;

template <class T>
__device__ PD_INL_CLIP int clip(WarpState<T>& S, Cell& c, int lane, float4 sj, FPlane f, int pidn, Counters& cnt) {
    PT_BEGIN(t_cls);
    // warp-uniform counts snapshotted in registers; published to the shared Cell only at the end,
    // after a __syncwarp, so no lane can observe a half-updated cell
    const int nv0 = c.nv;
    // 1. classify (outside <=> s > tol; on-plane vertices are kept)
    int R = 0;
    const int nch = (nv0 + 31) >> 5;
    Box6 box;  // AABB of the kept vertices, fused into the classification pass
    box.reset();
    if (T::COOP && nv0 >= P_coop_min_v(S)) {  // all warps of the CTA classify; removed slots from the ballots
        CoopJob& J = coop_job();
        if (lane == 0) { J.kind = JOB_CLASSIFY; J.nv = nv0; J.f = f; J.sj = sj; }
        coop_go<T>(S, J, lane);
        R = rem_from_omask(S, nch, lane);
    } else
    for (int ch = 0; ch < nch; ++ch) {
        int s = ch * 32 + lane;
        bool out = false;
        if (PD_FLAT_CLASSIFY) {
            // branch-free: every lane loads a valid slot and the rare FP64 certification is a warp-uniform branch
            const bool in = s < nv0;
            const float4 v = S.fv[in ? s : 0];
            const float s32 = fmaf(f.nx, v.x, fmaf(f.ny, v.y, f.nz * v.z)) - f.d;
            out = in && s32 > f.m;
            const bool amb = in && fabsf(s32) <= f.m;
            if (__any_sync(FULL, amb)) {
                if (amb) out = outside_cert(S, c, sj, f, s);
            }
            if (!kLeafAabb<T> && in && !out) box.add(v);
        } else
        if (s < nv0) {
            float4 v = S.fv[s];
            float s32 = fmaf(f.nx, v.x, fmaf(f.ny, v.y, f.nz * v.z)) - f.d;
            if (fabsf(s32) > f.m) out = s32 > 0.f;
            else out = outside_cert(S, c, sj, f, s);
            if (!kLeafAabb<T> && !out) box.add(v);
        }
        unsigned m = __ballot_sync(FULL, out);
        if (out) {
            PD_ASSERT(R + __popc(m & lanemask_lt()) < T::VMAX);
            S.rem[R + __popc(m & lanemask_lt())] = (uint16_t)s;  // removed slots, ascending
        }
        if (lane == 0) S.omask[ch] = m;
        R += __popc(m);
    }
    PT_END(t_cls, 6);
    if (R == 0) return CLIP_NONE;
    if (R == nv0) return CLIP_EMPTY;
    __syncwarp();
    PT_BEGIN(t_bnd);
    int np0 = c.np;
    if (np0 >= (T::PMAX * 85) / 100) {  // plane garbage collection (vertex slots are unaffected)
        plane_gc(S, c, lane);
        np0 = c.np;
        if (np0 >= T::PMAX) return CLIP_OVF;
    }
    // 2. hole boundary: edge x->y of a removed vertex is a boundary edge iff its reverse y->x is not
    //    held by another removed vertex, i.e. iff the unordered edge {x,y} occurs once among the
    //    removed vertices (an interior edge occurs exactly twice).  Up to 10 removed vertices: one
    //    edge per lane and a single __match_any_sync; otherwise the pairwise scan below.
    int B = 0;
    if (PD_MATCH && 3 * R <= 32) {
        const int r = lane / 3, e = lane - 3 * r;
        const bool act = lane < 3 * R;
        uint32_t key = 0xffff0000u | (uint32_t)lane;  // unique for idle lanes
        uint32_t dir = 0;
        if (act) {
            auto t = S.vt[S.rem[r]];
            int a = ta(t), b = tb(t), cc = tc(t);
            int x = e == 0 ? a : (e == 1 ? b : cc);
            int y = e == 0 ? b : (e == 1 ? cc : a);
            key = (uint32_t)min(x, y) | ((uint32_t)max(x, y) << 16);
            dir = (uint32_t)x | ((uint32_t)y << 16);
        }
        const unsigned same = __match_any_sync(FULL, key);  // every lane must execute it
        const bool bnd = act && __popc(same) == 1;
        const unsigned bm = __ballot_sync(FULL, bnd);
        if (bnd) S.bnd[__popc(bm & lanemask_lt())] = dir;
        B = __popc(bm);
    } else {
        if (T::EDGE_BITMAP) {
            for (int r = lane; r < R; r += 32) {
                auto t = S.vt[S.rem[r]];
                int a = ta(t), b = tb(t), cc = tc(t);
                int k0 = min(a, b) * T::PMAX + max(a, b), k1 = min(b, cc) * T::PMAX + max(b, cc),
                    k2 = min(cc, a) * T::PMAX + max(cc, a);
                atomicXor(&S.ebits[k0 >> 5], 1u << (k0 & 31));
                atomicXor(&S.ebits[k1 >> 5], 1u << (k1 & 31));
                atomicXor(&S.ebits[k2 >> 5], 1u << (k2 & 31));
            }
            __syncwarp();
        }
        for (int r0 = 0; r0 < R; r0 += 32) {
            int r = r0 + lane;
            int nb = 0;
            uint32_t e0 = 0, e1 = 0, e2 = 0;
            if (r < R) {
                auto t = S.vt[S.rem[r]];
                int a = ta(t), b = tb(t), cc = tc(t);
                bool f0 = false, f1 = false, f2 = false;
                if (T::EDGE_BITMAP) {
                    int k0 = min(a, b) * T::PMAX + max(a, b), k1 = min(b, cc) * T::PMAX + max(b, cc),
                        k2 = min(cc, a) * T::PMAX + max(cc, a);
                    f0 = !((S.ebits[k0 >> 5] >> (k0 & 31)) & 1u);
                    f1 = !((S.ebits[k1 >> 5] >> (k1 & 31)) & 1u);
                    f2 = !((S.ebits[k2 >> 5] >> (k2 & 31)) & 1u);
                } else {
#pragma unroll 1
                    for (int k = 0; k < R; ++k) {
                        auto u = S.vt[S.rem[k]];
                        f0 |= has_edge(u, b, a);
                        f1 |= has_edge(u, cc, b);
                        f2 |= has_edge(u, a, cc);
                    }
                }
                // compact the (up to 3) boundary edges without local-memory arrays
                uint32_t ab = (uint32_t)a | ((uint32_t)b << 16), bc = (uint32_t)b | ((uint32_t)cc << 16),
                         ca = (uint32_t)cc | ((uint32_t)a << 16);
                if (!f0) { e0 = ab; nb = 1; }
                if (!f1) { if (nb == 0) e0 = bc; else e1 = bc; nb++; }
                if (!f2) { if (nb == 0) e0 = ca; else if (nb == 1) e1 = ca; else e2 = ca; nb++; }
            }
            int inc = nb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int v = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += v;
            }
            int tot = __shfl_sync(FULL, inc, 31);
            int pos = B + inc - nb;
            if (B + tot <= T::VMAX) {
                if (nb > 0) S.bnd[pos] = e0;
                if (nb > 1) S.bnd[pos + 1] = e1;
                if (nb > 2) S.bnd[pos + 2] = e2;
            }
            B += tot;
        }
        if (T::EDGE_BITMAP) {  // restore the all-zero bitmap
            __syncwarp();
            for (int r = lane; r < R; r += 32) {
                auto t = S.vt[S.rem[r]];
                int a = ta(t), b = tb(t), cc = tc(t);
                S.ebits[(min(a, b) * T::PMAX + max(a, b)) >> 5] = 0u;
                S.ebits[(min(b, cc) * T::PMAX + max(b, cc)) >> 5] = 0u;
                S.ebits[(min(cc, a) * T::PMAX + max(cc, a)) >> 5] = 0u;
            }
            __syncwarp();
        }
    }
    PT_END(t_bnd, 7);
    PT_BEGIN(t_cre);
    // topology check: the hole of a proper cut is bounded by one cycle of >= 3 edges, i.e.
    // B >= 3 and every plane starts as many boundary edges as it ends (checked cheaply: B >= 3)
    if (B < 3 && lane == 0) c.degraded = 1;
    int nvn = nv0 - R + B;
    if (nvn > T::VMAX || B > T::VMAX || np0 + 1 > T::PMAX) return CLIP_OVF;
    // 3. append the plane, create (h, x, y) for every boundary edge
    int hs = np0;
    if (lane == 0) {  // the exact FP64 plane goes straight to shared memory (read back by every new vertex)
        PD_ASSERT(hs < T::PMAX);
        S.pl[hs] = exact_plane(c, sj);
        S.pid[hs] = pidn;
    }
    __syncwarp();
    for (int e0 = 0; e0 < B; e0 += 32) {
        int e = e0 + lane;
        if (e < B) {
            uint32_t be = S.bnd[e];
            int x = be & 0xffff, y = be >> 16;
            double vx, vy, vz;
            if (PD_SOLVE_OOL) solve3_ool(S.pl, hs, x, y, vx, vy, vz);
            else solve3(S.pl, hs, x, y, vx, vy, vz);
            int slot = e < R ? S.rem[e] : nv0 + (e - R);
            put_vertex(S, slot, vx, vy, vz);
            PD_ASSERT(slot >= 0 && slot < T::VMAX && x < hs && y < hs && x != y);
            S.vt[slot] = tpack<typename T::trip_t>(hs, x, y);
            if (!kLeafAabb<T>) box.add(make_float4((float)vx, (float)vy, (float)vz, 0.f));
        }
    }
    // 4. if fewer vertices were created than removed, move kept vertices from the tail into holes
    if (B < R) {
        int moved = 0;
        for (int ch = nvn >> 5; ch < nch; ++ch) {
            int s = ch * 32 + lane;
            bool mover = s >= nvn && s < nv0 && !((S.omask[ch] >> lane) & 1u);
            unsigned mm = __ballot_sync(FULL, mover);
            if (mover) {
                int dst = S.rem[B + moved + __popc(mm & lanemask_lt())];
                if (T::F64V) { S.vx[dst] = S.vx[s]; S.vy[dst] = S.vy[s]; S.vz[dst] = S.vz[s]; }
                S.fv[dst] = S.fv[s];
                S.vt[dst] = S.vt[s];
            }
            moved += __popc(mm);
        }
    }
    c.nv = nvn;  // safe without a prior sync: no lane reads c.nv/c.np in clip after the snapshot
    c.np = hs + 1;
    __syncwarp();
    PT_END(t_cre, 8);
    PT_BEGIN(t_ab);
    // fused: the AABB of the kept + created vertices gathered by this clip's passes (not in the
    // cooperative tier, whose classification runs on all warps, nor with the sphere bound)
    // (a stale AABB contains the smaller cell: every bound that reads it stays sound, only looser)
    if (kLeafAabb<T>) {
    } else if (PD_FUSED_AABB && !T::COOP && !T::SPHERE) finish_aabb(c, box);
    else update_aabb(S, c, lane);
    PT_END(t_ab, 9);
    return CLIP_DONE;
}

// Site test in FP32: cull iff the plane y.D <= q/2 (q = |D|^2 + w_i - w_j)
// cannot cut the cell.  Paper: d_ij = q/(2|D|) > r with r the directional radius of p_j's octant.
// Default: the exact support of the cell AABB in direction D, h = sum_k max(lo_k D_k, hi_k D_k)
// <= r |D| (Cauchy-Schwarz), cull iff q/2 > h: never looser.  Margins only ever keep a site.
// SPHERE tiers also bound the support by the cell's bounding sphere, h <= m.D + rho |D|: much tighter
// than the box for the huge, round cells of heavy sites, whose AABB holds thousands of candidates.
template <bool SPH>
__device__ __forceinline__ bool site_culled_hq(const Cell& c, float Dx, float Dy, float Dz, float D2, float hq, float dqa,
                                               unsigned flags) {
    if (!(flags & (PD_PAPER_BOUND | PD_ISOTROPIC))) {
        float h = Dx * (Dx >= 0.f ? c.fhi[0] : c.flo[0]) + Dy * (Dy >= 0.f ? c.fhi[1] : c.flo[1]) +
                  Dz * (Dz >= 0.f ? c.fhi[2] : c.flo[2]);
        float mag = c.vmax * (fabsf(Dx) + fabsf(Dy) + fabsf(Dz));
        if (SPH) {
            const float rd = c.srad * sqrtf(D2);
            h = fminf(h, fmaf(c.sc[0], Dx, fmaf(c.sc[1], Dy, c.sc[2] * Dz)) + rd);
            mag += rd;
        }
        return hq - h > 1e-5f * (D2 + dqa + mag);
    }
    float r2;
    if (flags & PD_ISOTROPIC) {
        r2 = cell_r2(c);
    } else {
        float hx = Dx >= 0.f ? c.fhi[0] : c.flo[0], hy = Dy >= 0.f ? c.fhi[1] : c.flo[1], hz = Dz >= 0.f ? c.fhi[2] : c.flo[2];
        r2 = hx * hx + hy * hy + hz * hz;
    }
    float rd = sqrtf(r2 * D2);
    return 2.f * hq - 2.f * rd > 1e-5f * (D2 + dqa + 2.f * rd);
}
template <bool SPH>
__device__ __forceinline__ bool site_culled(const Cell& c, float Dx, float Dy, float Dz, float D2, float dq,
                                            unsigned flags) {
    return site_culled_hq<SPH>(c, Dx, Dy, Dz, D2, 0.5f * (D2 + dq), fabsf(dq), flags);
}
// Re-cull from a candidate's stored plane (D, dd = q/2): |dq| = |2 dd - D2| only sizes the relative margin.
template <bool SPH>
__device__ __forceinline__ bool site_culled_pl(const Cell& c, float4 pl, unsigned flags) {
    const float D2 = pl.x * pl.x + pl.y * pl.y + pl.z * pl.z;
    return site_culled_hq<SPH>(c, pl.x, pl.y, pl.z, D2, pl.w, fabsf(2.f * pl.w - D2), flags);
}

// FP64 certification of a candidate whose FP32 cut test was ambiguous (rare; kept out of line).
template <class T>
__device__ __noinline__ bool cuts_fp64(const WarpState<T>& S, const Cell& c, float4 sj, float D2) {
    double ex = (double)sj.x - c.px, ey = (double)sj.y - c.py, ez = (double)sj.z - c.pz;
    double ed = 0.5 * (ex * ex + ey * ey + ez * ez + (c.pw - (double)sj.w));
    double tol = 1e-12 * (double)sqrtf(D2) * (double)cell_rmax(c);
    for (int k = 0; k < c.nv; ++k) {
        double x, y, z;
        vertex64(S, k, x, y, z);
        if (fma(ex, x, fma(ey, y, ez * z)) - ed > tol) return true;
    }
    return false;
}

// Candidate processing (lane = candidate site j, Morton index): a BVH leaf's sites, or the warm
// start's K nearest sites.
template <class T, unsigned MODE>
__device__ PD_INL_LEAF int process_cands(WarpState<T>& S, Cell& c, int lane, int j, bool valid, int count,
                                         const CellParams& P, Counters& cnt) {
    const unsigned flags = mode_flags<MODE>(P.flags);
    float4 sj = make_float4(0.f, 0.f, 0.f, 0.f);
    float Dx = 0.f, Dy = 0.f, Dz = 0.f, D2 = 0.f, dq = 0.f;
    bool dup_kill = false;
    if (valid) {
        sj = __ldg(&P.sites[j]);
        Dx = sj.x - c.fpx; Dy = sj.y - c.fpy; Dz = sj.z - c.fpz;  // exact iff zero: duplicates are detected exactly
        D2 = Dx * Dx + Dy * Dy + Dz * Dz;
        dq = c.fpw - sj.w;
        if (Dx == 0.f && Dy == 0.f && Dz == 0.f) {
            // coincident sites: the heavier owns, ties to the lower id
            if (sj.w > c.fpw || (sj.w == c.fpw && __ldg(&P.perm[j]) < c.self_orig)) dup_kill = true;
            valid = false;
        }
    }
    if (__any_sync(FULL, dup_kill)) return ST_DUP;
    if (kStats<MODE>) cnt.sites += count;
    cnt.work += count;
    bool cand = valid && !site_culled<T::SPHERE>(c, Dx, Dy, Dz, D2, dq, flags);
    unsigned mask = __ballot_sync(FULL, cand);
    if (!mask) return ST_OK;
    // Batch cut test, lane = candidate: does the plane cut the CURRENT cell?  A plane that does not
    // cut it cannot cut any later (smaller) cell, so it is dropped for good.  Same certified
    // predicate as clip().
    const float dd = 0.5f * (D2 + dq);
    const float m = 1e-6f * ((fabsf(Dx) + fabsf(Dy) + fabsf(Dz)) * c.vmax + D2 + fabsf(dq));
    if (PD_BATCH_CUT) {
        bool cuts = false, amb = false;
        if (cand) {
#pragma unroll 4
            for (int k = 0; k < c.nv; ++k) {
                float4 v = S.fv[k];
                float s = fmaf(Dx, v.x, fmaf(Dy, v.y, Dz * v.z)) - dd;
                cuts |= s > m;
                amb |= fabsf(s) <= m;
            }
            if (!cuts && amb) cuts = cuts_fp64(S, c, sj, D2);  // certify in FP64 (rare)
        }
        if (kStats<MODE>) cnt.tests += __popc(mask);
        cand = cand && cuts;
        mask = __ballot_sync(FULL, cand);
    }
    bool batched = PD_BATCH_CUT;
    if (T::COOP && !PD_BATCH_CUT && c.nv >= P_coop_min_v(S) && (mask & (mask - 1))) {
        // cooperative tier: one CTA-wide pass tests every candidate of the leaf against the current
        // cell (same certified predicate); only the planes that cut go on to clip()
        CoopJob& J = coop_job();
        if (cand) { J.cD[lane] = make_float4(Dx, Dy, Dz, dd); J.cm[lane] = m; J.csj[lane] = sj; }
        if (lane == 0) { J.kind = JOB_BATCH; J.nv = c.nv; J.mask = mask; }
        coop_go<T>(S, J, lane);
        unsigned cut = 0u;
        for (int w = 0; w < T::WARPS; ++w) cut |= (unsigned)J.ipart[w][0];
        const bool cuts = (cut >> lane) & 1u;
        if (kStats<MODE>) cnt.tests += __popc(mask);
        cand = cand && cuts;
        mask = __ballot_sync(FULL, cand);
        batched = true;
    }
    if (!batched && kStats<MODE>) cnt.tests += __popc(mask);
    float key = cand ? dd * rsqrtf(D2) : INFINITY;  // d_ij: nearest plane first
    // the candidates' planes wait in shared memory (lane = candidate), so that no per-candidate value but
    // the key stays in registers through clip()
    // candidate planes stored by rank among the candidates (the pre-test runs over ceil(k/4) groups, no gaps)
    const unsigned mask0 = mask;
    const int ncand = __popc(mask0);
    const int myslot = PD_PRETEST_COMPACT ? __popc(mask0 & lanemask_lt()) : lane;
    if (cand) {
        S.cpl[myslot] = make_float4(Dx, Dy, Dz, dd);
        S.cmg[myslot] = m;
        if (PD_KEY_SMEM) S.ckey[myslot] = ford(key);
    }
    if (PD_PRETEST_COMPACT && lane >= ncand && lane < ((ncand + 3) & ~3)) {  // the last group's padding
        S.cpl[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
        S.cmg[lane] = 0.f;
    }
    __syncwarp();
    // Pre-test, lane = vertex, all candidates at once (independent FMA chains, groups of 4 planes in
    // flight): bit k <=> candidate slot k has some FP32 value above -m_k on the CURRENT cell.  A candidate
    // with none has every vertex strictly inside (|s32 - s| < m), i.e. the certified classification
    // of clip() would remove nothing now or on any later (smaller) cell: dropped for good.  Run on the
    // leaf's candidates, and again on the remaining ones after each clip (PD_REFILTER): most planes that cut
    // the cell the leaf started with no longer cut it once the nearest have clipped.
    auto pretest = [&](unsigned smask) -> unsigned {
        unsigned hit = 0u;
        const int nv0 = c.nv;
        for (int sv = lane; sv - lane < nv0; sv += 32) {
            const bool vin = sv < nv0;
            const float4 v = vin ? S.fv[sv] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
            for (int k0 = 0; k0 < ncand; k0 += 4) {
                if (!((smask >> k0) & 0xfu)) continue;
                const float4 mg = *reinterpret_cast<const float4*>(&S.cmg[k0]);
                const float4 p0 = S.cpl[k0], p1 = S.cpl[k0 + 1], p2 = S.cpl[k0 + 2], p3 = S.cpl[k0 + 3];
                const bool h0 = fmaf(p0.x, v.x, fmaf(p0.y, v.y, p0.z * v.z)) - p0.w > -mg.x;
                const bool h1 = fmaf(p1.x, v.x, fmaf(p1.y, v.y, p1.z * v.z)) - p1.w > -mg.y;
                const bool h2 = fmaf(p2.x, v.x, fmaf(p2.y, v.y, p2.z * v.z)) - p2.w > -mg.z;
                const bool h3 = fmaf(p3.x, v.x, fmaf(p3.y, v.y, p3.z * v.z)) - p3.w > -mg.w;
                if (vin) hit |= ((h0 ? 1u : 0u) | (h1 ? 2u : 0u) | (h2 ? 4u : 0u) | (h3 ? 8u : 0u)) << k0;
            }
        }
        return __reduce_or_sync(FULL, hit);
    };
    if (PD_PRETEST && PD_PRETEST_COMPACT && !batched && ncand >= PD_PRETEST_MIN) {
        const unsigned hr = pretest(ncand == 32 ? FULL : (1u << ncand) - 1u);
        cand = cand && ((hr >> myslot) & 1u);
        mask = __ballot_sync(FULL, cand);
    } else if (PD_PRETEST && !batched) {  // candidates stored by lane (PD_PRETEST_COMPACT=0)
        unsigned hit = 0u;
        const int nv0 = c.nv;
        for (int sv = lane; sv - lane < nv0; sv += 32) {
            const bool vin = sv < nv0;
            const float4 v = vin ? S.fv[sv] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
            for (int k0 = 0; k0 < 32; k0 += 4) {
                if (!((mask >> k0) & 0xfu)) continue;
                const float4 mg = *reinterpret_cast<const float4*>(&S.cmg[k0]);
                const float4 p0 = S.cpl[k0], p1 = S.cpl[k0 + 1], p2 = S.cpl[k0 + 2], p3 = S.cpl[k0 + 3];
                const bool h0 = fmaf(p0.x, v.x, fmaf(p0.y, v.y, p0.z * v.z)) - p0.w > -mg.x;
                const bool h1 = fmaf(p1.x, v.x, fmaf(p1.y, v.y, p1.z * v.z)) - p1.w > -mg.y;
                const bool h2 = fmaf(p2.x, v.x, fmaf(p2.y, v.y, p2.z * v.z)) - p2.w > -mg.z;
                const bool h3 = fmaf(p3.x, v.x, fmaf(p3.y, v.y, p3.z * v.z)) - p3.w > -mg.w;
                if (vin) hit |= ((h0 ? 1u : 0u) | (h1 ? 2u : 0u) | (h2 ? 4u : 0u) | (h3 ? 8u : 0u)) << k0;
            }
        }
        mask &= __reduce_or_sync(FULL, hit);
        cand = (mask >> lane) & 1u;
    }
    int nclip = 0;
    while (mask) {
        const int kk = !cand ? 0x7fffffff : (PD_KEY_SMEM ? S.ckey[myslot] : ford(key));  // smem: not live across clip
        int kmin = __reduce_min_sync(FULL, kk);
        unsigned lead = __ballot_sync(FULL, cand && kk == kmin);
        int src = __ffs(lead) - 1;
        if (lane == src) cand = false;
        // Fast reject, lane = vertex: the plane (D, dd) of the leaf's candidate pass, its margin m (from the
        // leaf-time vmax >= the current one: only larger).  No FP32 value above -m means every vertex is
        // strictly inside (|s32 - s| < m), which is exactly when the certified classification of clip()
        // would remove nothing: such a plane never cuts this or any later (smaller) cell.
        FPlane f;
        {
            const int sl = PD_PRETEST_COMPACT ? __popc(mask0 & ((1u << src) - 1u)) : src;
            const float4 pl = S.cpl[sl];
            f.nx = pl.x; f.ny = pl.y; f.nz = pl.z; f.d = pl.w;
            f.m = S.cmg[sl];
        }
        if (PD_FAST_REJECT) {
            const int nv0 = c.nv;
            bool maybe = false;
            for (int sv = lane; sv < nv0; sv += 32) {
                const float4 v = S.fv[sv];
                maybe |= fmaf(f.nx, v.x, fmaf(f.ny, v.y, f.nz * v.z)) - f.d > -f.m;
            }
            if (!__any_sync(FULL, maybe)) {
                mask = __ballot_sync(FULL, cand);
                continue;
            }
        }
        const int jsrc = __shfl_sync(FULL, j, src);
        const float4 sjs = __ldg(&P.sites[jsrc]);  // the site itself (FP64 plane of the certification)
        PT_BEGIN(t_clip);
#ifdef PD_COUNT_CALLS  // measurement build: clip() calls counted in the queue-spill counter
        if (kStats<MODE>) cnt.spills++;
#endif
        int st = clip(S, c, lane, sjs, f, jsrc, cnt);
        PT_END(t_clip, 3);
        if (st == CLIP_EMPTY) return ST_EMPTY;
        if (st == CLIP_OVF) return ST_OVERFLOW;
        if (st == CLIP_DONE) {
            ++nclip;
            if (kStats<MODE>) cnt.clips++;
            cnt.ncl++;
            cnt.work += 8;
            // (with the per-leaf AABB the box has not changed since the leaf's site cull: nothing new to cull)
            if (!kLeafAabb<T> && cand && site_culled_pl<T::SPHERE>(c, S.cpl[myslot], flags)) cand = false;
            if (PD_REFILTER && PD_PRETEST_COMPACT && !batched) {
                if (__popc(__ballot_sync(FULL, cand)) >= PD_REFILTER_MIN) {
                    const unsigned hr = pretest(__reduce_or_sync(FULL, cand ? 1u << myslot : 0u));
                    cand = cand && ((hr >> myslot) & 1u);
                }
            }
        }
        mask = __ballot_sync(FULL, cand);
    }
    if (kLeafAabb<T> && nclip) update_aabb(S, c, lane);
    return ST_OK;
}

// A BVH leaf's sites -- or, once per cell with the KNN warm start, the site's K
// power-nearest sites, clipped before the traversal through this same (single, inlined) candidate
// path.  The warm-start sites are met again in their leaves, where their planes no longer cut
// (on-plane vertices are kept), so the diagram is unchanged.  Coincident sites
// are never in the list; they share a Morton code, so they sit next to each other in Morton order, and
// the duplicate rule (R5) is settled from the 16 positions on either side before any warm-start clip
// (so a cell that the power-nearest planes empty is still flagged DUPLICATE when it is one; the leaf
// processing keeps deciding the rare runs of > 16 sites in one Morton cell).
template <class T, unsigned MODE>
__device__ __forceinline__ int process_leaf(WarpState<T>& S, Cell& c, int lane, int link, bool warm, const CellParams& P,
                                            Counters& cnt) {
    int j, count;
    bool valid;
    if ((mode_flags<MODE>(P.flags) & PD_WARM_START) && warm) {
        j = lane < KNN_K ? __ldg(&P.knn[(int64_t)c.self * KNN_K + lane]) : -1;
        if (!__any_sync(FULL, j >= 0)) return ST_OK;  // no list (adaptive mode: not dominated)
        const int64_t t = lane < 16 ? (int64_t)c.self - 1 - lane : (int64_t)c.self + 1 + (lane - 16);
        bool kill = false;
        if (t >= 0 && t < P.n_sites) {
            const float4 q = __ldg(&P.sites[t]);
            if (q.x == c.fpx && q.y == c.fpy && q.z == c.fpz)
                kill = q.w > c.fpw || (q.w == c.fpw && __ldg(&P.perm[t]) < c.self_orig);
        }
        if (__any_sync(FULL, kill)) return ST_DUP;
        valid = j >= 0;
        count = KNN_K;
    } else {
        const int first = leaf_first(link);
        count = leaf_count(link);
        j = first + lane;
        valid = lane < count && j != c.self;
    }
    return process_cands<T, MODE>(S, c, lane, j, valid, count, P, cnt);
}

// Best-first traversal (Alg. 1).  Queue entries are the pushed child records;
// when the on-chip queue is full, entries spill to a per-warp stack in global memory (order is
// relaxed, correctness is not affected) and are refilled when the on-chip queue drains.
template <class T, unsigned MODE>
__device__ int traverse(WarpState<T>& S, Cell& c, int lane, const CellParams& P, Counters& cnt, NodeChild* spill,
                        int spill_cap) {
    const unsigned flags = mode_flags<MODE>(P.flags);
    const bool dfs = (flags & PD_DFS) != 0;
    // the queue: in the warp's state, or (cooperative top tier, state in global memory) in shared memory
    float4* const qlo = T::COOP ? coop_queue_lo<T>() : S.qlo;
    float4* const qhi = T::COOP ? coop_queue_hi<T>() : S.qhi;
    uint32_t* const qmask = T::COOP ? coop_queue_mask<T>() : S.qmask;
    int node = __float_as_int(__ldg(&P.root->hi_l.w));
    bool have = true;
    // warm start: the first "leaf" is the KNN list (then the traversal starts at the root)
    bool warm = (mode_flags<MODE>(P.flags) & PD_WARM_START) && P.knn;
    const int root_link = node;
    int ns = 0;  // spilled entries
    int nq = 0;  // queue length (warp-uniform register)
    bool dirty = true;  // the cell changed since the queue was last re-validated (clean pop)
    for (;;) {
        if (have) {
            PT_BEGIN(t_desc);
            while (node >= 0 && !warm) {  // descend (Alg. 1 lines 4-18), 8 children per visit
                if (kStats<MODE>) cnt.nodes++;
                cnt.work++;
                if (!PD_VISITS_BY_WORK) cnt.visited++;
                float key = INFINITY;
                bool culled = true;
                float4 lo_w = make_float4(0, 0, 0, 0), hi_l = make_float4(0, 0, 0, 0);
                const NodeChild* rec = P.nodes[node].c;
                if (PD_FLAT_NODES) {  // every lane tests child lane & 7 (no divergent branch); lanes >= 8 are culled
                    lo_w = __ldg(&rec[lane & (WIDE - 1)].lo_w);
                    hi_l = __ldg(&rec[lane & (WIDE - 1)].hi_l);
                    key = node_test<kPlaneKey<T>>(c, lo_w, hi_l, flags, culled);
                    culled = culled || lane >= WIDE || __float_as_int(hi_l.w) == EMPTY_LINK;
                } else if (lane < WIDE) {
                    lo_w = __ldg(&rec[lane].lo_w);
                    hi_l = __ldg(&rec[lane].hi_l);
                    if (__float_as_int(hi_l.w) != EMPTY_LINK) key = node_test<kPlaneKey<T>>(c, lo_w, hi_l, flags, culled);
                }
                unsigned surv = __ballot_sync(FULL, !culled);
                const bool ex_all = exact_on(flags, PD_VISITS(cnt), P.exact_after);
                // exact test on every surviving LEAF child (a leaf costs far more than the test), and on
                // internal children too once the cell is heavy
                const unsigned leafm = __ballot_sync(FULL, lane < WIDE && __float_as_int(hi_l.w) < 0);
                const unsigned exm = ex_all ? surv : (PD_EXACT_LEAVES == 1 && !(flags & PD_NO_EXACT) ? (surv & leafm) : 0u);
                if (exm && T::COOP && c.nv >= P_coop_min_v(S)) {  // all children in one CTA-wide pass
                    CoopJob& J = coop_job();
                    const bool mine = lane < WIDE && ((exm >> lane) & 1u);
                    if (mine) { J.lo[lane] = lo_w; J.hi[lane] = hi_l; }
                    if (lane == 0) { J.kind = JOB_EXACT; J.nv = c.nv; J.mask = exm; }
                    coop_go<T>(S, J, lane);
                    bool cull = false;
                    if (mine) {
                        int b = J.ipart[0][lane];
                        for (int w = 1; w < T::WARPS; ++w) b = max(b, J.ipart[w][lane]);
                        cull = exact_decide(c, lo_w, hi_l, iford(b));
                    }
                    surv &= ~__ballot_sync(FULL, cull);
                    culled = !((surv >> lane) & 1u);
                } else if (exm) {
                    unsigned s2 = exm;
                    while (s2) {
                        int k = __ffs(s2) - 1;
                        s2 &= s2 - 1;
                        if (node_exact_culled(S, c, lane, __ldg(&rec[k].lo_w), __ldg(&rec[k].hi_l))) surv &= ~(1u << k);
                    }
                    culled = !((surv >> lane) & 1u);
                }
                if (!surv) {
                    have = false;
                    PT_END(t_desc, 1);
                    break;
                }
                // go to the child with the smallest priority delta, queue the other survivors
                int kmin = __reduce_min_sync(FULL, culled ? 0x7fffffff : ford(key));
                int near = __ffs(__ballot_sync(FULL, !culled && ford(key) == kmin)) - 1;
                int lnear = __shfl_sync(FULL, __float_as_int(hi_l.w), near);
                bool push = !culled && lane != near;
                unsigned pm = __ballot_sync(FULL, push);
                int npush = __popc(pm);
                if (npush) {
                    int rank = __popc(pm & lanemask_lt());
                    int room = T::QMAX - nq;
                    int tos = max(npush - room, 0);
                    if (ns + tos > spill_cap) return ST_OVERFLOW;
                    if (push) {
                        if (rank < room) {
                            if (kLazyPop<T> || kCleanPop<T>) S.qkey[nq + rank] = key;
                            PD_ASSERT(nq + rank < T::QMAX);
                            qlo[nq + rank] = lo_w;
                            qhi[nq + rank] = hi_l;
                        } else {
                            spill[ns + rank - room].lo_w = lo_w;
                            spill[ns + rank - room].hi_l = hi_l;
                        }
                    }
                    nq += npush - tos;
                    ns += tos;
                    if (kStats<MODE>) cnt.spills += tos;
                }
                // PD_EXACT_LEAVES 2: the leaf about to be processed gets the exact polytope-vs-box test (a leaf
                // costs far more than one warp pass over the vertices; 60% of the leaves the AABB tests keep fail it)
                if (PD_EXACT_LEAVES == 2 && lnear < 0 && !ex_all && !(flags & PD_NO_EXACT) &&
                    node_exact_culled(S, c, lane, __ldg(&rec[near].lo_w), __ldg(&rec[near].hi_l))) {
                    have = false;
                    PT_END(t_desc, 1);
                    break;
                }
                node = lnear;
            }
            if (have) {
                PT_END(t_desc, 1);
                if (kStats<MODE>) cnt.leaves++;
                __syncwarp();
                PT_BEGIN(t_leaf);
                const unsigned ncl0 = cnt.ncl;
                // PD_PARK: warp-uniform traversal state parked in shared memory across the leaf (register
                // pressure of the inlined clip), reloaded below
                if (PD_PARK) { c.t_nq = nq; c.t_ns = ns; }
                int st = process_leaf<T, MODE>(S, c, lane, node, warm, P, cnt);
                if (PD_PARK) { nq = *(volatile int*)&c.t_nq; ns = *(volatile int*)&c.t_ns; }
                PT_END(t_leaf, 2);
                if (st != ST_OK) return st;
                if (cnt.ncl != ncl0) dirty = true;
                if (warm) {
                    warm = false;
                    node = root_link;
                    continue;
                }
            }
        }
        // pop (Alg. 1 lines 21-31): re-validate every queued entry against the shrunk cell
        PT_BEGIN(t_pop);
        __syncwarp();
        if (nq == 0 && ns > 0) {  // refill from the spill stack
            __threadfence_block();
            dirty = true;  // refilled entries carry no key
            int mm = min(ns, T::QMAX);
            for (int t = lane; t < mm; t += 32) {
                NodeChild e = spill[ns - mm + t];
                if (kLazyPop<T>) {
                    bool cu;
                    S.qkey[t] = node_test<kPlaneKey<T>>(c, e.lo_w, e.hi_l, flags, cu);
                }
                qlo[t] = e.lo_w;
                qhi[t] = e.hi_l;
            }
            ns -= mm;
            nq = mm;
            __syncwarp();
        }
        if (nq == 0) return ST_OK;
        if (dfs) {
            bool ok = false;
            while (nq > 0 && !ok) {
                int t = nq - 1;
                bool culled;
                node_test<kPlaneKey<T>>(c, qlo[t], qhi[t], flags, culled);
                node = __float_as_int(qhi[t].w);
                nq--;
                ok = !culled;
            }
            __syncwarp();
            if (!ok) {
                if (ns > 0) continue;
                return ST_OK;
            }
            have = true;
            continue;
        }
        if (kLazyPop<T>) {
            // the paper's unsorted-queue pop: min over the push-time priorities,
            // re-validate only the popped entry (Alg. 1 lines 25-29), fill its hole with the last one
            int bk = 0x7fffffff, bs = -1;
            for (int s = lane; s < nq; s += 32) {
                int k = ford(S.qkey[s]);
                if (k < bk) { bk = k; bs = s; }
            }
            int gk = __reduce_min_sync(FULL, bk);
            int bslot = __shfl_sync(FULL, bs, __ffs(__ballot_sync(FULL, bk == gk)) - 1);
            float4 lo = qlo[bslot], hi = qhi[bslot];
            __syncwarp();
            if (lane == 0 && bslot != nq - 1) {
                qlo[bslot] = qlo[nq - 1];
                qhi[bslot] = qhi[nq - 1];
                S.qkey[bslot] = S.qkey[nq - 1];
            }
            --nq;
            __syncwarp();
            bool culled;
            node_test<kPlaneKey<T>>(c, lo, hi, flags, culled);
            if (!culled && (exact_on(flags, PD_VISITS(cnt), P.exact_after) ||
                            (PD_EXACT_LEAVES && !(flags & PD_NO_EXACT) && __float_as_int(hi.w) < 0)))
                culled = node_exact_culled(S, c, lane, lo, hi);
            node = __float_as_int(hi.w);
            have = !culled;
            PT_END(t_pop, 4);
            continue;
        }
        if (kCleanPop<T> && !dirty && !dfs) {
            // the cell is unchanged since the last re-validation: every queued entry is alive and its key
            // current (entries pushed since were tested against this same cell); pop the least key
            int bk = 0x7fffffff, bs = 0x7fffffff;
            for (int sq = lane; sq < nq; sq += 32) {
                const int k = ford(S.qkey[sq]);
                if (k < bk) { bk = k; bs = sq; }
            }
            const int gk = __reduce_min_sync(FULL, bk);
            const int bslot = __reduce_min_sync(FULL, bk == gk ? bs : 0x7fffffff);
            node = __float_as_int(qhi[bslot].w);
            const bool popped_dead = (exact_on(flags, PD_VISITS(cnt), P.exact_after) ||
                                      (PD_EXACT_LEAVES && !(flags & PD_NO_EXACT) && node < 0)) &&
                                     node_exact_culled(S, c, lane, qlo[bslot], qhi[bslot]);
            __syncwarp();
            if (lane == 0 && bslot != nq - 1) {
                qlo[bslot] = qlo[nq - 1];
                qhi[bslot] = qhi[nq - 1];
                S.qkey[bslot] = S.qkey[nq - 1];
            }
            __syncwarp();
            --nq;
            have = !popped_dead;
            PT_END(t_pop, 4);
            continue;
        }
        int bestk = 0x7fffffff, bests = -1;
        const int qch = (nq + 31) >> 5;
        int alive_total = -1;
        if (T::COOP && nq >= 8 * 32) {  // the whole CTA re-validates a long queue
            CoopJob& J = coop_job();
            if (lane == 0) { J.kind = JOB_REVAL; J.nq = nq; J.flags = flags; }
            coop_go<T>(S, J, lane);
            const int k = lane < T::WARPS ? J.ipart[lane][0] : 0x7fffffff;
            const int sl = lane < T::WARPS ? J.ipart[lane][1] : 0x7fffffff;
            const int g = __reduce_min_sync(FULL, k);
            bestk = g;
            bests = __reduce_min_sync(FULL, k == g ? sl : 0x7fffffff);
            alive_total = __reduce_add_sync(FULL, lane < T::WARPS ? J.ipart[lane][2] : 0);
        } else
        for (int ch = 0; ch < qch; ++ch) {
            int s = ch * 32 + lane;
            bool al = false;
            if (PD_FLAT_NODES) {  // no divergent branch: lanes past the queue test slot 0 and are dropped
                const bool in = s < nq;
                bool culled;
                const float k = node_test<kPlaneKey<T>>(c, qlo[in ? s : 0], qhi[in ? s : 0], flags, culled);
                al = in && !culled;
                if (al && ford(k) < bestk) { bestk = ford(k); bests = s; }
                if (kCleanPop<T> && in) S.qkey[s] = k;
            } else
            if (s < nq) {
                bool culled;
                float k = node_test<kPlaneKey<T>>(c, qlo[s], qhi[s], flags, culled);
                al = !culled;
                if (al && ford(k) < bestk) { bestk = ford(k); bests = s; }
                if (kCleanPop<T>) S.qkey[s] = k;
            }
            unsigned am = __ballot_sync(FULL, al);
            if (lane == 0) qmask[ch] = am;
        }
        __syncwarp();
        int gk = __reduce_min_sync(FULL, bestk);
        if (gk == 0x7fffffff) {
            nq = 0;
            have = false;
            if (ns > 0) continue;
            return ST_OK;
        }
        unsigned lead = __ballot_sync(FULL, bestk == gk);
        int bslot = __shfl_sync(FULL, bests, __ffs(lead) - 1);
        node = __float_as_int(qhi[bslot].w);
        bool popped_dead = (exact_on(flags, PD_VISITS(cnt), P.exact_after) ||
                            (PD_EXACT_LEAVES && !(flags & PD_NO_EXACT) && node < 0)) &&
                           node_exact_culled(S, c, lane, qlo[bslot], qhi[bslot]);
        if (PD_LAZY_COMPACT && alive_total < 0) {  // warp path: alive count from the chunk ballots
            int a = 0;
            for (int ch = lane; ch < qch; ch += 32) a += __popc(qmask[ch]);
            alive_total = __reduce_add_sync(FULL, a);
        }
        if ((T::COOP || PD_LAZY_COMPACT) && alive_total * 4 > nq * 3) {
            // mostly alive: remove only the popped entry (the last one fills its slot);
            // the few dead entries stay and are found dead again (culling is monotone), until a
            // re-validation finds a quarter of the queue dead and compacts it below
            __syncwarp();
            if (lane == 0 && bslot != nq - 1) { qlo[bslot] = qlo[nq - 1]; qhi[bslot] = qhi[nq - 1]; }
            __syncwarp();
            nq -= 1;
            have = !popped_dead;
            PT_END(t_pop, 4);
            continue;
        }
        // compact: keep alive entries except the popped one
        int base = 0;
        for (int ch = 0; ch < qch; ++ch) {
            int s = ch * 32 + lane;
            bool keep = ((qmask[ch] >> lane) & 1u) && s != bslot;
            unsigned km = __ballot_sync(FULL, keep);
            float4 lo = make_float4(0, 0, 0, 0), hi = make_float4(0, 0, 0, 0);
            float ky = 0.f;
            if (keep) {
                lo = qlo[s]; hi = qhi[s];
                if (kCleanPop<T>) ky = S.qkey[s];
            }
            __syncwarp();
            if (keep) {
                int dst = base + __popc(km & lanemask_lt());
                qlo[dst] = lo;
                qhi[dst] = hi;
                if (kCleanPop<T>) S.qkey[dst] = ky;
            }
            __syncwarp();
            base += __popc(km);
        }
        nq = base;
        have = !popped_dead;
        dirty = false;
        PT_END(t_pop, 4);
    }
}

template <class T>
__device__ __noinline__ void init_cell(WarpState<T>& S, Cell& c, int lane, const CellParams& P) {
    // the box as 6 wall planes + 8 vertices, site-local coordinates
    double lo[3] = {(double)P.box_lo[0] - c.px, (double)P.box_lo[1] - c.py, (double)P.box_lo[2] - c.pz};
    double hi[3] = {(double)P.box_hi[0] - c.px, (double)P.box_hi[1] - c.py, (double)P.box_hi[2] - c.pz};
    if (lane < 6) {
        int ax = lane >> 1, pos = lane & 1;
        double n[3] = {0, 0, 0};
        n[ax] = pos ? 1.0 : -1.0;
        S.pl[lane] = make_double4(n[0], n[1], n[2], pos ? hi[ax] : -lo[ax]);
        S.pid[lane] = -1 - lane;
    }
    if (lane < 8) {
        int sx = lane & 1, sy = (lane >> 1) & 1, sz = (lane >> 2) & 1;
        put_vertex(S, lane, sx ? hi[0] : lo[0], sy ? hi[1] : lo[1], sz ? hi[2] : lo[2]);
        int X = sx, Y = 2 + sy, Z = 4 + sz;
        int sgn = (sx ? 1 : -1) * (sy ? 1 : -1) * (sz ? 1 : -1);  // det of the outward normals
        S.vt[lane] = sgn > 0 ? tpack<typename T::trip_t>(X, Y, Z) : tpack<typename T::trip_t>(X, Z, Y);
    }
    c.nv = 8;
    c.np = 6;
    c.nq = 0;
    c.degraded = 0;
    if (T::SPHERE) {
        c.flo[0] = c.flo[1] = c.flo[2] = 0.f;
        c.fhi[0] = c.fhi[1] = c.fhi[2] = 0.f;
        __syncwarp();
        update_aabb(S, c, lane);
        return;
    }
    // the AABB of the box's corners: what update_aabb computes from their FP32 copies, without the warp reductions
    // (keeps the once-per-cell code small: it shares the instruction cache with the hot loop)
    float vm = 0.f, flo[3], fhi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        flo[k] = (float)lo[k];
        fhi[k] = (float)hi[k];
        flo[k] -= fabsf(flo[k]) * 2.4e-7f + 1e-30f;
        fhi[k] += fabsf(fhi[k]) * 2.4e-7f + 1e-30f;
        vm = fmaxf(vm, fmaxf(-flo[k], fhi[k]));
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        c.flo[k] = flo[k]; c.fhi[k] = fhi[k];
        c.glo[k] = fminf(flo[k], 0.f); c.ghi[k] = fmaxf(fhi[k], 0.f);
        c.flo2[k] = flo[k] * flo[k]; c.fhi2[k] = fhi[k] * fhi[k];
    }
    c.vmax = vm;
    __syncwarp();
}

// Twins: the vertex across each directed edge of vertex u (slots u0, u0+stride, ...).
template <class T>
__device__ __forceinline__ void twins_range(WarpState<T>& S, int nv, int u0, int stride) {
    for (int u = u0; u < nv; u += stride) {
        auto t = S.vt[u];
        int a = ta(t), b = tb(t), cc = tc(t);
        uint16_t t0 = 0xffff, t1 = 0xffff, t2 = 0xffff;
#pragma unroll 1
        for (int k = 0; k < nv; ++k) {
            auto w = S.vt[k];
            if (has_edge(w, b, a)) t0 = (uint16_t)k;
            if (has_edge(w, cc, b)) t1 = (uint16_t)k;
            if (has_edge(w, a, cc)) t2 = (uint16_t)k;
        }
        S.tw[0][u] = t0; S.tw[1][u] = t1; S.tw[2][u] = t2;
    }
}

// Face vector areas (1/2 sum v x next(v)), face areas, and this thread's volume / surface partials
// (faces f0, f0+stride, ...).
template <class T>
__device__ __forceinline__ void areas_range(WarpState<T>& S, int nv, int np, int f0, int stride, double& vol, double& surf,
                                            bool& missing) {
    for (int f = f0; f < np; f += stride) {
        double Ax = 0, Ay = 0, Az = 0;
#pragma unroll 1
        for (int u = 0; u < nv; ++u) {
            auto t = S.vt[u];
            int which = ta(t) == f ? 2 : (tb(t) == f ? 0 : (tc(t) == f ? 1 : -1));
            if (which >= 0) {
                int w = S.tw[which][u];
                if (w == 0xffff) {  // an edge without its reverse: the final cell is not closed
                    missing = true;
                    continue;
                }
                double ux = S.vx[u], uy = S.vy[u], uz = S.vz[u];
                double wx = S.vx[w], wy = S.vy[w], wz = S.vz[w];
                Ax += uy * wz - uz * wy;
                Ay += uz * wx - ux * wz;
                Az += ux * wy - uy * wx;
            }
        }
        Ax *= 0.5; Ay *= 0.5; Az *= 0.5;
        double area = sqrt(Ax * Ax + Ay * Ay + Az * Az);
        S.farea[f] = area;
        double4 pl = S.pl[f];
        double nn = pl.x * pl.x + pl.y * pl.y + pl.z * pl.z;
        vol += (Ax * pl.x + Ay * pl.y + Az * pl.z) * pl.w / nn;
        surf += area;
    }
}

// Tier 1 (<= 64 planes, <= 127 vertices): twins from a 256-entry edge hash and face areas by walking each
// face's loop (lane = face), O(V) per cell instead of the O(V^2) scans above.  Every edge {x, y} of the closed
// polytope is held by exactly two vertices (as x->y and y->x): entry = key(12) | A(7) | B(7), 127 = none.
// A third holder or a missing partner is a topology failure (PD_CELL_DEGRADED).
template <class T>
#ifndef PD_HASH_TWINS
#define PD_HASH_TWINS 0  // 1: O(V) edge-hash finalize; measured 40% slower on C4 (645 vs 456 ms), kept as an option
#endif
constexpr bool kHashTwins = PD_HASH_TWINS && T::PMAX <= 64 && T::VMAX <= 127 && !T::COOP;
constexpr uint32_t kEtEmpty = 0xffffffffu;
__device__ __forceinline__ int et_hash(uint32_t key) { return (int)((key * 2654435761u) >> 24); }

template <class T>
__device__ __forceinline__ bool twins_hash(WarpState<T>& S, int nv, int lane) {
    bool bad = false;
    for (int k = lane; k < 256; k += 32) S.etab[k] = kEtEmpty;
    __syncwarp();
    for (int u = lane; u < nv; u += 32) {
        const auto t = S.vt[u];
        const int p[3] = {ta(t), tb(t), tc(t)};
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const int x = p[e], y = p[e == 2 ? 0 : e + 1];
            const uint32_t key = (uint32_t)(min(x, y) << 6 | max(x, y));
            int h = et_hash(key);
            for (int probe = 0; probe < 256; ++probe) {
                const uint32_t w = S.etab[h];
                if (w == kEtEmpty) {
                    if (atomicCAS(&S.etab[h], kEtEmpty, key << 14 | (uint32_t)u << 7 | 127u) == kEtEmpty) break;
                    --probe;  // lost the race for this slot: look at it again
                    continue;
                }
                if ((w >> 14) == key) {
                    if ((w & 127u) != 127u) { bad = true; break; }  // a third vertex on one edge
                    if (atomicCAS(&S.etab[h], w, (w & ~127u) | (uint32_t)u) == w) break;
                    --probe;
                    continue;
                }
                h = (h + 1) & 255;
            }
        }
    }
    __syncwarp();
    for (int u = lane; u < nv; u += 32) {
        const auto t = S.vt[u];
        const int p[3] = {ta(t), tb(t), tc(t)};
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const int x = p[e], y = p[e == 2 ? 0 : e + 1];
            const uint32_t key = (uint32_t)(min(x, y) << 6 | max(x, y));
            int h = et_hash(key);
            uint32_t w = S.etab[h];
            while (w != kEtEmpty && (w >> 14) != key) { h = (h + 1) & 255; w = S.etab[h]; }
            int tw = 0xffff;
            if (w != kEtEmpty) {
                const int a = (int)(w >> 7) & 127, b = (int)(w & 127u);
                tw = a == u ? b : a;
                if (tw == 127) tw = 0xffff;
            }
            bad |= tw == 0xffff;
            S.tw[e][u] = (uint16_t)tw;  // e = 0: across a->b, 1: b->c, 2: c->a (as twins_range)
        }
    }
    __syncwarp();
    return bad;
}

// Face areas by walking each face's vertex loop from its lowest vertex slot (deterministic order), lane = face.
template <class T>
__device__ __forceinline__ bool areas_walk(WarpState<T>& S, int nv, int np, int lane, double& vol, double& surf) {
    uint32_t* start = S.bnd;  // dead outside clip(): the lowest vertex slot of every face
    for (int f = lane; f < np; f += 32) start[f] = 0xffffffffu;
    __syncwarp();
    for (int u = lane; u < nv; u += 32) {
        const auto t = S.vt[u];
        atomicMin(&start[ta(t)], (uint32_t)u);
        atomicMin(&start[tb(t)], (uint32_t)u);
        atomicMin(&start[tc(t)], (uint32_t)u);
    }
    __syncwarp();
    bool bad = false;
    for (int f = lane; f < np; f += 32) {
        double Ax = 0, Ay = 0, Az = 0;
        const uint32_t s0 = start[f];
        if (s0 != 0xffffffffu) {
            int u = (int)s0;
            double ux = S.vx[u], uy = S.vy[u], uz = S.vz[u];
            for (int step = 0; step < T::VMAX; ++step) {
                const auto t = S.vt[u];
                const int slot = ta(t) == f ? 2 : (tb(t) == f ? 0 : (tc(t) == f ? 1 : -1));
                const int w = slot < 0 ? 0xffff : S.tw[slot][u];
                if (w == 0xffff) { bad = true; break; }
                const double wx = S.vx[w], wy = S.vy[w], wz = S.vz[w];
                Ax += uy * wz - uz * wy;
                Ay += uz * wx - ux * wz;
                Az += ux * wy - uy * wx;
                u = w; ux = wx; uy = wy; uz = wz;
                if (u == (int)s0) break;
                if (step == T::VMAX - 1) bad = true;  // the loop never closed
            }
        }
        Ax *= 0.5; Ay *= 0.5; Az *= 0.5;
        const double area = sqrt(Ax * Ax + Ay * Ay + Az * Az);
        S.farea[f] = area;
        const double4 pl = S.pl[f];
        const double nn = pl.x * pl.x + pl.y * pl.y + pl.z * pl.z;
        vol += (Ax * pl.x + Ay * pl.y + Az * pl.z) * pl.w / nn;
        surf += area;
    }
    return bad;
}

// Tier 1 (<= 64 planes, <= 128 vertices, one warp): face areas by walking each face's vertex loop, lane = face,
// with the vertices bucketed by face first (CSR built with shared-memory atomics), O(sum_f k_f^2) per cell instead
// of the O(V^2) twin scan + O(F V) area scan above.  Vertex u = (a, b, c) (CCW from outside) rotated to put face f
// first, (f, y, z): its successor on face f's loop is the vertex whose rotated triplet is (f, z, .) -- the holder
// of the reverse of u's dual edge z -> f, i.e. its twin (areas_range's tw[which][u]).  Each walk starts at the
// lowest vertex slot of the face (deterministic summation order).  A face whose vertices do not form exactly one
// cycle is a topology failure (PD_CELL_DEGRADED).
#ifndef PD_FACE_WALK
#define PD_FACE_WALK 1
#endif
template <class T>
constexpr bool kFaceWalk = PD_FACE_WALK && T::PMAX <= 64 && T::VMAX <= 128 && !T::COOP && !T::GLOBAL;

template <class T>
__device__ __forceinline__ bool areas_facewalk(WarpState<T>& S, int nv, int np, int lane, double& vol, double& surf) {
    uint32_t* const off = S.fcnt;   // per face: CSR offset of its entries
    uint32_t* const cur = S.ffill;  // per face: entry count
    // scratch in arrays the finalize does not read: the FP32 vertex copies hold the entries (u | y << 7 | f << 14:
    // vertex u on face f, y = the plane after f in u's CCW triplet), tw the successor vertex of every entry and,
    // per vertex, the entry index of each of its three faces
    uint32_t* const ent = reinterpret_cast<uint32_t*>(S.fv);
    uint16_t* const succ = &S.tw[0][0];
    for (int f = lane; f < np; f += 32) { off[f] = 0u; cur[f] = 0u; }
    __syncwarp();
    for (int u = lane; u < nv; u += 32) {
        const auto t = S.vt[u];
        atomicAdd(&off[ta(t)], 1u);
        atomicAdd(&off[tb(t)], 1u);
        atomicAdd(&off[tc(t)], 1u);
    }
    __syncwarp();
    {   // exclusive scan of the per-face counts (np <= 64: two faces per lane)
        const int f0 = 2 * lane;
        const uint32_t c0 = f0 < np ? off[f0] : 0u, c1 = f0 + 1 < np ? off[f0 + 1] : 0u;
        uint32_t inc = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += v;
        }
        __syncwarp();
        if (f0 < np) off[f0] = inc - c0 - c1;
        if (f0 + 1 < np) off[f0 + 1] = inc - c1;
    }
    __syncwarp();
    // fill; every vertex remembers the entry index of its faces a (in rem) and b, c (the halves of bnd)
    for (int u = lane; u < nv; u += 32) {
        const auto t = S.vt[u];
        const int a = ta(t), b = tb(t), cc = tc(t);
        const uint32_t ea = off[a] + atomicAdd(&cur[a], 1u), eb = off[b] + atomicAdd(&cur[b], 1u),
                       ec = off[cc] + atomicAdd(&cur[cc], 1u);
        ent[ea] = (uint32_t)u | (uint32_t)b << 7 | (uint32_t)a << 14;   // on face a: (a, b, c), y = b
        ent[eb] = (uint32_t)u | (uint32_t)cc << 7 | (uint32_t)b << 14;  // on face b: (b, c, a), y = c
        ent[ec] = (uint32_t)u | (uint32_t)a << 7 | (uint32_t)cc << 14;  // on face c: (c, a, b), y = a
        S.rem[u] = (uint16_t)ea;
        S.bnd[u] = eb | ec << 16;
    }
    __syncwarp();
    const int ne = 3 * nv;
    bool bad = false;
    // successor of every entry (lane = entry): vertex u on face f, (f, y, z) rotated; its successor on f's loop is
    // the entry of f whose y equals z (the holder of the reverse of u's dual edge z -> f)
    for (int e = lane; e < ne; e += 32) {
        const uint32_t x = ent[e];
        const int u = (int)(x & 127u), f = (int)(x >> 14);
        const auto t = S.vt[u];
        const int a = ta(t), b = tb(t), cc = tc(t);
        const int z = a == f ? cc : (b == f ? a : b);
        const int o = (int)off[f], k = (int)cur[f];
        int w = 0xffff;
        for (int q = 0; q < k; ++q) {
            const uint32_t y = ent[o + q];
            if ((int)((y >> 7) & 127u) == z) w = (int)(y & 127u);
        }
        bad |= w == 0xffff;
        succ[e] = (uint16_t)w;
    }
    __syncwarp();
    // walk each face's loop (lane = face) from its lowest vertex slot: deterministic summation order
    for (int f = lane; f < np; f += 32) {
        const int o = (int)off[f], k = (int)cur[f];
        double Ax = 0, Ay = 0, Az = 0;
        if (k > 0) {
            int e0 = o;
            for (int q = 1; q < k; ++q)
                if ((ent[o + q] & 127u) < (ent[e0] & 127u)) e0 = o + q;
            int e = e0, steps = 0;
            int u = (int)(ent[e] & 127u);
            double ux = S.vx[u], uy = S.vy[u], uz = S.vz[u];
            for (;;) {
                const int w = succ[e];
                if (w == 0xffff) { bad = true; break; }
                const double wx = S.vx[w], wy = S.vy[w], wz = S.vz[w];
                Ax += uy * wz - uz * wy;
                Ay += uz * wx - ux * wz;
                Az += ux * wy - uy * wx;
                ++steps;
                // w's entry on face f: its triplet slot holding f
                const auto t = S.vt[w];
                const uint32_t bc = S.bnd[w];
                e = ta(t) == f ? (int)S.rem[w] : (tb(t) == f ? (int)(bc & 0xffffu) : (int)(bc >> 16));
                u = w; ux = wx; uy = wy; uz = wz;
                if (e == e0 || steps >= k) break;
            }
            bad |= e != e0 || steps != k;  // not exactly one cycle through the face's k vertices
        }
        Ax *= 0.5; Ay *= 0.5; Az *= 0.5;
        const double area = sqrt(Ax * Ax + Ay * Ay + Az * Az);
        S.farea[f] = area;
        const double4 pl = S.pl[f];
        const double nn = pl.x * pl.x + pl.y * pl.y + pl.z * pl.z;
        vol += (Ax * pl.x + Ay * pl.y + Az * pl.z) * pl.w / nn;
        surf += area;
    }
    return bad;
}

// One warp's share of a cooperative job (warp w of T::WARPS; warp 0 is the cell's own warp).
template <class T>
__device__ __forceinline__ void coop_run(WarpState<T>& S, CoopJob& J, int w, int lane) {
    const Cell& c = S.c;
    const int kind = J.kind, nv = J.nv;
    constexpr int stride = T::WARPS * 32;
    if (kind == JOB_CLASSIFY) {  // same certified predicate as clip()
        const FPlane f = J.f;
        const float4 sj = J.sj;
        const int nch = (nv + 31) >> 5;
        constexpr int U = 4;  // chunks in flight per warp (the vertex loads are independent)
        for (int ch0 = w; ch0 < nch; ch0 += U * T::WARPS) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int s = (ch0 + u * T::WARPS) * 32 + lane;
                v[u] = s < nv ? S.fv[s] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int ch = ch0 + u * T::WARPS;
                if (ch >= nch) break;
                const int s = ch * 32 + lane;
                bool out = false;
                if (s < nv) {
                    float s32 = fmaf(f.nx, v[u].x, fmaf(f.ny, v[u].y, f.nz * v[u].z)) - f.d;
                    if (fabsf(s32) > f.m) out = s32 > 0.f;
                    else out = outside_fp64(c, sj, f, S.vx[s], S.vy[s], S.vz[s]);
                }
                const unsigned m = __ballot_sync(FULL, out);
                if (lane == 0) S.omask[ch] = m;
            }
        }
    } else if (kind == JOB_EXACT) {
        const unsigned mask = J.mask;
        for (int k = 0; k < WIDE; ++k) {
            if (!((mask >> k) & 1u)) continue;
            float b = exact_partial(S.fv, c, J.lo[k], J.hi[k], w * 32 + lane, nv, stride);
            int bi = __reduce_max_sync(FULL, ford(b));
            if (lane == 0) J.ipart[w][k] = bi;
        }
    } else if (kind == JOB_AABB) {
        Box6 b;
        b.reset();
        const float4 m = J.lo[0];
        float sr2 = 0.f;
#pragma unroll 4
        for (int s = w * 32 + lane; s < nv; s += stride) {
            const float4 v = S.fv[s];
            b.add(v);
            if (T::SPHERE) {
                const float dx = v.x - m.x, dy = v.y - m.y, dz = v.z - m.z;
                sr2 = fmaxf(sr2, dx * dx + dy * dy + dz * dz);
            }
        }
        const int r6 = __reduce_max_sync(FULL, ford(sr2));
        if (lane == 0) J.ipart[w][6] = r6;
        int r0 = __reduce_min_sync(FULL, ford(b.lo0)), r1 = __reduce_min_sync(FULL, ford(b.lo1)),
            r2 = __reduce_min_sync(FULL, ford(b.lo2)), r3 = __reduce_max_sync(FULL, ford(b.hi0)),
            r4 = __reduce_max_sync(FULL, ford(b.hi1)), r5 = __reduce_max_sync(FULL, ford(b.hi2));
        if (lane == 0) {
            J.ipart[w][0] = r0; J.ipart[w][1] = r1; J.ipart[w][2] = r2;
            J.ipart[w][3] = r3; J.ipart[w][4] = r4; J.ipart[w][5] = r5;
        }
    } else if (kind == JOB_BATCH) {
        // does candidate k's plane cut the cell?  Some vertex outside, by the same certified predicate as
        // clip(): FP32 beyond the margin, else FP64 against the tolerance 1e-12 |D| R (R9/R10) -- done
        // right here by the thread holding the vertex (heavy cells' weights make many tests ambiguous)
        const unsigned cmask = J.mask;
        unsigned cut = 0u;
        constexpr int U = 4;
        for (int s0 = w * 32 + lane; s0 < nv; s0 += U * stride) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int sv = s0 + u * stride;
                v[u] = sv < nv ? S.fv[sv] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            unsigned mm = cmask;
            while (mm) {
                const int k = __ffs(mm) - 1;
                mm &= mm - 1;
                const float4 D = J.cD[k];
                const float mk = J.cm[k];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int sv_i = s0 + u * stride;
                    if (sv_i < nv) {
                        const float sv = fmaf(D.x, v[u].x, fmaf(D.y, v[u].y, D.z * v[u].z)) - D.w;
                        if (sv > mk) cut |= 1u << k;
                        else if (fabsf(sv) <= mk && !((cut >> k) & 1u)) {
                            FPlane f;
                            f.nx = D.x; f.ny = D.y; f.nz = D.z; f.d = D.w; f.m = mk;
                            if (outside_fp64(c, J.csj[k], f, S.vx[sv_i], S.vy[sv_i], S.vz[sv_i])) cut |= 1u << k;
                        }
                    }
                }
            }
        }
        cut = __reduce_or_sync(FULL, cut);
        if (lane == 0) { J.ipart[w][0] = (int)cut; J.ipart[w][1] = 0; }
    } else if (kind == JOB_REVAL) {
        // re-validate the queue against the shrunk cell: alive ballots per chunk + this warp's best
        const int nq = J.nq;
        const unsigned flags = J.flags;
        float4* const qlo = coop_queue_lo<T>();
        float4* const qhi = coop_queue_hi<T>();
        uint32_t* const qmask = coop_queue_mask<T>();
        const int qch = (nq + 31) >> 5;
        int bestk = 0x7fffffff, bests = 0x7fffffff;
        for (int ch = w; ch < qch; ch += T::WARPS) {
            const int sq = ch * 32 + lane;
            bool al = false;
            if (sq < nq) {
                bool culled;
                const float k = node_test<kPlaneKey<T>>(c, qlo[sq], qhi[sq], flags, culled);
                al = !culled;
                if (al && ford(k) < bestk) { bestk = ford(k); bests = sq; }
            }
            const unsigned am = __ballot_sync(FULL, al);
            if (lane == 0) qmask[ch] = am;
        }
        const int gk = __reduce_min_sync(FULL, bestk);
        const int gs = __reduce_min_sync(FULL, bestk == gk ? bests : 0x7fffffff);
        int alive = 0;
        for (int ch = w + lane * T::WARPS; ch < qch; ch += 32 * T::WARPS) alive += __popc(qmask[ch]);
        alive = __reduce_add_sync(FULL, alive);
        if (lane == 0) { J.ipart[w][0] = gk; J.ipart[w][1] = gs; J.ipart[w][2] = alive; }
    } else if (kind == JOB_TWINS) {
        twins_range(S, nv, w * 32 + lane, stride);
    } else if (kind == JOB_AREAS) {
        double vol = 0, surf = 0;
        bool missing = false;
        areas_range(S, nv, J.np, w * 32 + lane, stride, vol, surf, missing);
        vol = warp_sum_d(vol);
        surf = warp_sum_d(surf);
        missing = __any_sync(FULL, missing);
        if (lane == 0) { J.dpart[w][0] = vol; J.dpart[w][1] = surf; J.ipart[w][0] = missing ? 1 : 0; }
    }
}

// Warps 1..W-1 of a COOP CTA: serve jobs until warp 0 publishes JOB_EXIT.
template <class T>
__device__ __noinline__ void coop_worker(WarpState<T>& S, int w, int lane) {
    CoopJob& J = coop_job();
    for (;;) {
        named_bar(1, T::WARPS * 32);
        if (*(volatile int*)&J.kind == JOB_EXIT) return;
        coop_run<T>(S, J, w, lane);
        named_bar(2, T::WARPS * 32);
    }
}

// Dual tetrahedra (PD_TETS): vertex (a, b, c) of cell i whose three planes are bisector faces of
// positive area is the power-equidistant centre of {i, j_a, j_b, j_c}; the tet is written by the cell
// of its lowest original id, as (i, sorted others).  Needs S.farea (finalize).
template <class T>
__device__ __noinline__ void emit_tets(WarpState<T>& S, const Cell& c, int lane, const CellParams& P, double amin) {
    const CellOut& O = P.out;
    const int i = c.self_orig;
    int total = 0;
    for (int pass = 0; pass < 2; ++pass) {
        long long base = 0;
        if (pass == 1) {
            if (lane == 0) base = (long long)atom_add_g(O.ttop, (unsigned long long)total);
            base = __shfl_sync(FULL, base, 0);
            if (base + total > O.tcap) {  // arena full: the build is re-run with a larger one
                if (lane == 0) { *O.tovf = 1; O.tcnt[i] = 0; O.taoff[i] = 0; }
                break;
            }
            if (lane == 0) { O.tcnt[i] = total; O.taoff[i] = base; }
        }
        int k = 0;
        for (int u0 = 0; u0 < c.nv; u0 += 32) {
            const int u = u0 + lane;
            bool em = false;
            int x = 0, y = 0, z = 0;
            if (u < c.nv) {
                const auto t = S.vt[u];
                const int a = ta(t), b = tb(t), cc = tc(t);
                const int pa = S.pid[a], pb = S.pid[b], pc = S.pid[cc];
                if (pa >= 0 && pb >= 0 && pc >= 0 && S.farea[a] > amin && S.farea[b] > amin && S.farea[cc] > amin) {
                    x = __ldg(&P.perm[pa]); y = __ldg(&P.perm[pb]); z = __ldg(&P.perm[pc]);
                    if (x > y) { int q = x; x = y; y = q; }
                    if (y > z) { int q = y; y = z; z = q; }
                    if (x > y) { int q = x; x = y; y = q; }
                    em = i < x;
                }
            }
            const unsigned m = __ballot_sync(FULL, em);
            if (pass == 1 && em) O.tarena[base + k + __popc(m & lanemask_lt())] = make_int4(i, x, y, z);
            k += __popc(m);
        }
        total = k;
    }
}

// Face areas (vector area 1/2 sum v x next(v) around each face), volume, neighbours; FP64.
// Returns the cell's robustness counts packed: faces dropped (bits 0-14), near-degenerate neighbour faces
// (bits 15-29), degraded (bit 30) -- returned rather than added to the caller's Counters, which would
// otherwise have its address taken by this out-of-line call and live on the thread stack.
// The per-cell output of a cell without a polytope (EMPTY, DUPLICATE, or OVERFLOW in the last tier).
__device__ __forceinline__ void finalize_status(const Cell& c, int lane, const CellParams& P, int status) {
    const int i = c.self_orig;
    const CellOut& O = P.out;
    if (lane == 0) {
        if (O.tarena) { O.tcnt[i] = 0; O.taoff[i] = 0; }
        O.cnt[i] = 0;
        O.aoff[i] = 0;
        O.vol[i] = 0.f;
        O.surf[i] = 0.f;
        O.flags[i] = (uint8_t)(status == ST_OVERFLOW ? PD_CELL_OVERFLOW
                                                     : (PD_CELL_EMPTY | (status == ST_DUP ? PD_CELL_DUPLICATE : 0)));
    }
}

template <class T>
__device__ __noinline__ unsigned finalize(WarpState<T>& S, Cell& c, int lane, const CellParams& P, int status) {
    const int i = c.self_orig;
    const CellOut& O = P.out;
    if (status == ST_EMPTY || status == ST_DUP || status == ST_OVERFLOW) {
        finalize_status(c, lane, P, status);
        return 0u;
    }
#ifdef PD_SKIP_FIN
    if (!T::COOP && !T::GLOBAL) {  // EXPERIMENT ONLY: wrong output, measures the cell program without finalize
        if (lane == 0) { O.cnt[i] = 0; O.aoff[i] = 0; O.vol[i] = 0.f; O.surf[i] = 0.f; O.flags[i] = 0; }
        return 0u;
    }
#endif
    double vol = 0, surf = 0;
    if (T::COOP && c.nv >= P_coop_min_v(S)) {  // twins and faces over all warps of the CTA
        CoopJob& J = coop_job();
        if (lane == 0) { J.kind = JOB_TWINS; J.nv = c.nv; J.np = c.np; }
        coop_go<T>(S, J, lane);
        if (lane == 0) J.kind = JOB_AREAS;
        coop_go<T>(S, J, lane);
        bool missing = false;
        for (int w = 0; w < T::WARPS; ++w) { vol += J.dpart[w][0]; surf += J.dpart[w][1]; missing |= J.ipart[w][0] != 0; }
        vol /= 3.0;
        if (missing && lane == 0) c.degraded = 1;
    } else if (kFaceWalk<T>) {
        const bool bad = areas_facewalk(S, c.nv, c.np, lane, vol, surf);
        vol = warp_sum_d(vol) / 3.0;
        surf = warp_sum_d(surf);
        if (__any_sync(FULL, bad) && lane == 0) c.degraded = 1;
    } else if (kHashTwins<T>) {
        bool bad = twins_hash(S, c.nv, lane);
        bad |= areas_walk(S, c.nv, c.np, lane, vol, surf);
        vol = warp_sum_d(vol) / 3.0;
        surf = warp_sum_d(surf);
        if (__any_sync(FULL, bad) && lane == 0) c.degraded = 1;
    } else {
        twins_range(S, c.nv, lane, 32);
        __syncwarp();
        bool missing = false;
        areas_range(S, c.nv, c.np, lane, 32, vol, surf, missing);
        vol = warp_sum_d(vol) / 3.0;
        surf = warp_sum_d(surf);
        if (__any_sync(FULL, missing) && lane == 0) c.degraded = 1;
    }
    __syncwarp();
    // A face counts when its area exceeds 1e-13 S: below that it is a rounding artefact of a
    // zero-area (edge / vertex) contact of a degenerate configuration (reading R2).
    const double amin = 1e-13 * surf, asmall = 1e-9 * surf;
    bool boundary = false;
    int K = 0;
    unsigned ndrop = 0, nsmall = 0;
    for (int f0 = 0; f0 < c.np; f0 += 32) {
        int f = f0 + lane;
        bool nb = false, drop = false;
        double area = 0;
        if (f < c.np) {
            area = S.farea[f];
            if (area > amin) {
                if (S.pid[f] < 0) boundary = true;
                else nb = true;
            } else if (S.pid[f] >= 0 && area > 0) {
                drop = true;  // a zero-area contact (reading R2): counted, not a neighbour
            }
        }
        ndrop += __popc(__ballot_sync(FULL, drop));
        nsmall += __popc(__ballot_sync(FULL, nb && area < asmall));
        unsigned mb = __ballot_sync(FULL, nb);
        if (nb) {
            int pos = K + __popc(mb & lanemask_lt());
            S.nb_id[pos] = __ldg(&P.perm[S.pid[f]]);
            S.nb_area[pos] = (float)area;
        }
        K += __popc(mb);
    }
    boundary = __any_sync(FULL, boundary);
    __syncwarp();
    // arena row (ascending original ids)
    long long base = 0;
    if (lane == 0) base = (long long)atom_add_g(O.arena_top, (unsigned long long)K);
    base = __shfl_sync(FULL, base, 0);
    bool fits = base + K <= O.arena_cap;
    if (fits) {
        for (int e = lane; e < K; e += 32) {
            int id = S.nb_id[e];
            int rank = 0;
#pragma unroll 1
            for (int k = 0; k < K; ++k) rank += S.nb_id[k] < id;
            O.arena_nbr[base + rank] = id;
            O.arena_area[base + rank] = S.nb_area[e];
        }
    } else if (lane == 0) {
        *O.arena_overflow = 1;
    }
    if (O.tarena) emit_tets(S, c, lane, P, amin);
    const bool degraded = c.degraded != 0;
    if (lane == 0) {
        O.cnt[i] = K;
        O.aoff[i] = base;
        O.vol[i] = (float)vol;
        O.surf[i] = (float)surf;
        O.flags[i] = (uint8_t)((boundary ? PD_CELL_BOUNDARY : 0) | (vol > 0 ? 0 : PD_CELL_EMPTY) |
                               (degraded ? PD_CELL_DEGRADED : 0));
    }
    return min(ndrop, 0x7fffu) | (min(nsmall, 0x7fffu) << 15) | (degraded ? 1u << 30 : 0u);
}

// Deferred finalize (tier 1, CellParams::rec_*): store the finished cell's topology for finalize_kernel.
template <class T>
constexpr bool kDefer = std::is_same<T, Tier1>::value;  // finalize_kernel runs right after the tier-1 launch
template <class T>
__device__ __forceinline__ bool defer_cell(const WarpState<T>& S, const Cell& c, int lane, const CellParams& P, int s) {
    const int nv = c.nv, np = c.np;
    const unsigned words = 2u + (unsigned)np + (unsigned)nv;
    unsigned long long off = 0;
    if (lane == 0) off = atom_add_g(P.rec_top, words);
    off = __shfl_sync(FULL, off, 0);
    if (off + words > (unsigned long long)P.rec_cap) return false;  // arena full: finalize here
    uint32_t* rec = P.rec_arena + off;
    if (lane == 0) { rec[0] = (uint32_t)nv | ((uint32_t)np << 16); rec[1] = (uint32_t)c.degraded; }
    for (int f = lane; f < np; f += 32) rec[2 + f] = (uint32_t)S.pid[f];
    for (int u = lane; u < nv; u += 32) rec[2 + np + u] = (uint32_t)S.vt[u];
    if (lane == 0) P.rec_index[s] = (uint32_t)off;
    return true;
}

// Deferred finalize of tier 1: warp per recorded cell, Morton order.  The FP64 planes are rebuilt from the
// neighbour ids exactly as the cell program built them (exact_plane / the walls of init_cell) and every vertex
// by solve3 of its three planes -- the same function on the same operands, so the same values -- then the
// same finalize() as in the cell kernel.
// cpw = 0: persistent grid, grid-stride over the cells; cpw > 0: one chunk of cpw consecutive cells per warp
// (CTAs retire as they finish, so kernels of other streams -- the higher tiers -- get SMs as they free up).
template <class T>
__global__ void __launch_bounds__(T::WARPS * 32) finalize_kernel(const __grid_constant__ CellParams P, int cpw) {
    const int lane = threadIdx.x & 31, wid = (int)(threadIdx.x >> 5);
    WarpState<T>& S = reinterpret_cast<WarpState<T>*>(pd_smem)[wid];
    Cell& c = S.c;
    const int64_t gw = (int64_t)blockIdx.x * T::WARPS + wid;
    const int64_t nw = cpw > 0 ? 1 : (int64_t)gridDim.x * T::WARPS;
    const int64_t i0 = cpw > 0 ? gw * cpw : gw, i1 = cpw > 0 ? min(P.count, i0 + cpw) : P.count;
    // chunked mode (cpw <= 32): the chunk's record offsets, headers, degraded words, sites and original ids are
    // loaded once, lane = cell, and handed out by shuffles (one round of global latency per chunk, not per cell)
    const bool batch = PD_FIN_BATCH && cpw > 0 && cpw <= 32;
    uint32_t b_off = 0xffffffffu, b_h0 = 0u, b_deg = 0u;
    int b_orig = 0;
    float4 b_site = make_float4(0.f, 0.f, 0.f, 0.f);
    if (batch && i0 + lane < i1) {
        const int sl = (int)(P.begin + i0 + lane);
        b_off = P.rec_index[sl];
        b_site = __ldg(&P.sites[sl]);
        b_orig = __ldg(&P.perm[sl]);
        if (b_off != 0xffffffffu) { b_h0 = P.rec_arena[b_off]; b_deg = P.rec_arena[b_off + 1]; }
    }
    for (int64_t idx = i0; idx < i1; idx += nw) {
        const int s = (int)(P.begin + idx);
        const int k = (int)(idx - i0);
        const uint32_t off = batch ? __shfl_sync(FULL, b_off, k) : P.rec_index[s];
        if (off == 0xffffffffu) continue;
        const uint32_t* rec = P.rec_arena + off;
        const uint32_t h0 = batch ? __shfl_sync(FULL, b_h0, k) : rec[0];
        const int nv = (int)(h0 & 0xffffu), np = (int)(h0 >> 16);
        PD_ASSERT(nv >= 4 && nv <= T::VMAX && np >= 4 && np <= T::PMAX && off + 2u + (uint32_t)(nv + np) <= P.rec_cap);
        float4 site;
        int orig;
        uint32_t deg;
        if (batch) {
            site.x = __shfl_sync(FULL, b_site.x, k); site.y = __shfl_sync(FULL, b_site.y, k);
            site.z = __shfl_sync(FULL, b_site.z, k); site.w = __shfl_sync(FULL, b_site.w, k);
            orig = __shfl_sync(FULL, b_orig, k);
            deg = __shfl_sync(FULL, b_deg, k);
        } else {
            site = __ldg(&P.sites[s]);
            orig = __ldg(&P.perm[s]);
            deg = rec[1];
        }
        __syncwarp();
        if (lane == 0) {
            c.fpx = site.x; c.fpy = site.y; c.fpz = site.z; c.fpw = site.w;
            c.px = site.x; c.py = site.y; c.pz = site.z; c.pw = site.w;
            c.self = s;
            c.self_orig = orig;
            c.nv = nv;
            c.np = np;
            c.degraded = (int)deg;
        }
        __syncwarp();
        for (int f = lane; f < np; f += 32) {
            const int pid = (int)rec[2 + f];
            double4 pl;
            if (pid < 0) {  // box wall k (init_cell)
                const int k = -1 - pid, ax = k >> 1, pos = k & 1;
                const double lo = (double)P.box_lo[ax] - (ax == 0 ? c.px : ax == 1 ? c.py : c.pz);
                const double hi = (double)P.box_hi[ax] - (ax == 0 ? c.px : ax == 1 ? c.py : c.pz);
                double n[3] = {0, 0, 0};
                n[ax] = pos ? 1.0 : -1.0;
                pl = make_double4(n[0], n[1], n[2], pos ? hi : -lo);
            } else {
                pl = exact_plane(c, __ldg(&P.sites[pid]));
            }
            S.pl[f] = pl;
            S.pid[f] = pid;
        }
        __syncwarp();
        for (int u = lane; u < nv; u += 32) {
            const auto t = (typename T::trip_t)rec[2 + np + u];
            double x, y, z;
            solve3(S.pl, ta(t), tb(t), tc(t), x, y, z);
            put_vertex(S, u, x, y, z);
            S.vt[u] = t;
        }
        __syncwarp();
        const unsigned rob = finalize(S, c, lane, P, ST_OK);
        if (rob && lane == 0) {
            red_add_g(&P.stats->dropped, rob & 0x7fffu);
            red_add_g(&P.stats->small, (rob >> 15) & 0x7fffu);
            red_add_g(&P.stats->degraded, rob >> 30);
        }
    }
}

__device__ __noinline__ void trace_print(int tier, const Cell& c, const Counters& a, const Counters& b, int st, long long cyc) {
    printf("PD_TRACE cell=%d tier=%d status=%d nv=%d np=%d cycles=%lld nodes=%llu leaves=%llu sites=%llu tests=%llu "
           "clips=%llu spills=%llu\n",
           c.self_orig, tier, st, c.nv, c.np, cyc, a.nodes - b.nodes, a.leaves - b.leaves, a.sites - b.sites,
           a.tests - b.tests, a.clips - b.clips, a.spills - b.spills);
#if PD_PROFILE
        printf("PD_TRACE cell=%d phase_cycles init=%llu descend=%llu leaf=%llu clip=%llu pop=%llu finalize=%llu "
               "classify=%llu boundary=%llu create=%llu aabb=%llu\n",
               c.self_orig, a.cyc[0] - b.cyc[0], a.cyc[1] - b.cyc[1], a.cyc[2] - b.cyc[2], a.cyc[3] - b.cyc[3],
               a.cyc[4] - b.cyc[4], a.cyc[5] - b.cyc[5], a.cyc[6] - b.cyc[6], a.cyc[7] - b.cyc[7], a.cyc[8] - b.cyc[8],
               a.cyc[9] - b.cyc[9]);
#endif
}

template <class T, unsigned MODE>
__global__ void __launch_bounds__(T::WARPS * 32, T::MIN_BLOCKS) cells_kernel(const __grid_constant__ CellParams P, int tier) {
    const int lane = threadIdx.x & 31, wid = T::WARPS == 1 ? 0 : (int)(threadIdx.x >> 5);
    WarpState<T>& S = T::COOP     ? (T::GLOBAL ? reinterpret_cast<WarpState<T>*>(P.gstate)[blockIdx.x]
                                               : *reinterpret_cast<WarpState<T>*>(pd_smem + coop_smem_bytes<T>()))
                      : T::GLOBAL ? reinterpret_cast<WarpState<T>*>(P.gstate)[blockIdx.x * T::WARPS + wid]
                                  : reinterpret_cast<WarpState<T>*>(pd_smem)[wid];
    if (T::COOP) {
        if (threadIdx.x == 0) coop_job().min_v = P.coop_min_v;
        __syncthreads();
        if (wid != 0) {  // helper warps of a cooperative CTA
            coop_worker<T>(S, wid, lane);
            return;
        }
    }
    const int64_t total = P.list ? (int64_t)(*P.list_count) : P.count;
    Counters cnt = {};
    // spill stack per cell program: per warp, or per CTA in a cooperative tier (only warp 0 traverses)
    const int gw = T::COOP ? blockIdx.x : blockIdx.x * T::WARPS + wid;
    NodeChild* spill = P.spill + (size_t)gw * P.spill_cap;
    for (int k = lane; k < T::EBW; k += 32) S.ebits[k] = 0u;
    __syncwarp();
    unsigned long long ncells = 0, novf = 0;
    // Morton-consecutive batches of 4 in the first tier (locality); one cell at a time from the
    // (cost-ordered) lists of the higher tiers, so that their heaviest cells spread over the CTAs
#ifndef PD_T1_BATCH
#define PD_T1_BATCH 4
#endif
    const int BATCH = P.list ? 1 : PD_T1_BATCH;
    for (;;) {
        long long b0 = 0;
        if (lane == 0) b0 = (long long)atom_add_g(P.work_counter, (unsigned long long)BATCH);
        b0 = __shfl_sync(FULL, b0, 0);
        if (b0 >= total) break;
        for (int b = 0; b < BATCH && b0 + b < total; ++b) {
            int64_t idx = b0 + b;
            int s = P.list ? P.list[idx] : (int)(P.begin + idx);
            if (tier < P.start_tier) {  // test knob: hand every cell to the next tier untouched
                if (lane == 0) P.next_list[atom_add_g32(P.next_count, 1)] = s;
                continue;
            }
            Cell& c = S.c;
#if PD_PROFILE
            const Counters before = cnt;
#endif
            cnt.work = 0;
            cnt.visited = 0;
            float4 site = __ldg(&P.sites[s]);
            c.fpx = site.x; c.fpy = site.y; c.fpz = site.z; c.fpw = site.w;
            c.px = site.x; c.py = site.y; c.pz = site.z; c.pw = site.w;
            c.self = s;
            c.self_orig = __ldg(&P.perm[s]);
            __syncwarp();  // warp-uniform cell fields written by every lane
#if PD_PROFILE
            const long long t_cell = clock64();
#endif
            PT_BEGIN(t_init);
            init_cell(S, c, lane, P);
            PT_END(t_init, 0);
            int st = traverse<T, MODE>(S, c, lane, P, cnt, spill, P.spill_cap);
            __syncwarp();
            if (st == ST_OVERFLOW && !P.last_tier) {
                if (lane == 0) {
                    int k = atom_add_g32(P.next_count, 1);
                    P.next_list[k] = s;
                    if (P.next_cost) {  // the host starts the next tier's costliest cells first
                        P.next_cost[k] = (int32_t)min(cnt.work, 0x7fffffffu);
                    }
                }
                continue;
            }
            if (kStats<MODE> && st == ST_OVERFLOW) novf++;
            PT_BEGIN(t_fin);
            const bool deferred = kDefer<T> && st == ST_OK && P.rec_index && defer_cell(S, c, lane, P, s);
            unsigned rob = 0u;
            if constexpr (T::F64V) {
                if (!deferred) rob = finalize(S, c, lane, P, st);
            } else {
                // a finished cell whose record did not fit (never seen) is built again by the next tier; the
                // cost-sampling runs (no records: only the work counts are read) skip the output
                if (st == ST_OK && !deferred && P.rec_index) {
                    if (lane == 0) P.next_list[atom_add_g32(P.next_count, 1)] = s;
                    continue;
                }
                if (st != ST_OK) finalize_status(c, lane, P, st);
            }
            if (rob && lane == 0) {  // robustness counters (rare, always published): straight to the device totals
                red_add_g(&P.stats->dropped, rob & 0x7fffu);
                red_add_g(&P.stats->small, (rob >> 15) & 0x7fffu);
                red_add_g(&P.stats->degraded, rob >> 30);
            }
            PT_END(t_fin, 5);
            if (kStats<MODE>) ncells++;
#if PD_PROFILE
            if (c.self_orig == P.trace_cell && lane == 0) trace_print(tier, c, cnt, before, st, clock64() - t_cell);
#endif
            if ((P.flags & PD_COST) && lane == 0) {  // deterministic work count (balanced cuts must agree)
                P.out.cost[c.self_orig] = (int32_t)min(cnt.work, 0x7fffffffu);
            }
            __syncwarp();
        }
    }
    if (T::COOP) {  // release the helper warps
        if (lane == 0) coop_job().kind = JOB_EXIT;
        __syncwarp();
        named_bar(1, T::WARPS * 32);
    }
    // counters of every tier, or only of tier $PD_PROF_TIER when it is set (per-tier profiles)
    if (kStats<MODE> && (P.flags & PD_STATS) && lane == 0 && (P.prof_tier < 0 || P.prof_tier == tier)) {
        red_add_g(&P.stats->nodes, cnt.nodes);
        red_add_g(&P.stats->leaves, cnt.leaves);
        red_add_g(&P.stats->sites, cnt.sites);
        red_add_g(&P.stats->clip_tests, cnt.tests);
        red_add_g(&P.stats->clips, cnt.clips);
        red_add_g(&P.stats->cells, ncells);
        red_add_g(&P.stats->tier[tier], ncells);
        red_add_g(&P.stats->overflow, novf);
        red_add_g(&P.stats->spills, cnt.spills);
#if PD_PROFILE
        for (int k = 0; k < 10; ++k) red_add_g(&P.stats->cyc[k], cnt.cyc[k]);
#endif
    }

}

template <class T, unsigned MODE>
int tier_grid(int num_sms) {
    if (T::GLOBAL) {
        if (T::COOP) cudaFuncSetAttribute(cells_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coop_smem_bytes<T>());
        return num_sms * kTier3BlocksPerSM;
    }
    size_t smem = T::COOP ? coop_smem_bytes<T>() + sizeof(WarpState<T>) : sizeof(WarpState<T>) * T::WARPS;
    cudaFuncSetAttribute(cells_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cells_kernel<T, MODE>, T::WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    return num_sms * per_sm;
}

template <class T, unsigned MODE>
cudaError_t launch_tier(const CellParams& p, int tier, cudaStream_t st, int num_sms) {
    size_t smem = T::COOP ? coop_smem_bytes<T>() + (T::GLOBAL ? 0 : sizeof(WarpState<T>))
                          : T::GLOBAL ? 0 : sizeof(WarpState<T>) * T::WARPS;
    int grid = tier_grid<T, MODE>(num_sms);
    cells_kernel<T, MODE><<<grid, T::WARPS * 32, smem, st>>>(p, tier);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tier1(const CellParams& p, cudaStream_t st, int num_sms);

cudaError_t launch_finalize(const CellParams& p, cudaStream_t st, int num_sms, int cpw, int* launches) {
    if (!p.rec_index || p.count <= 0) return cudaSuccess;
    if (launches) ++*launches;
    const size_t smem = sizeof(WarpState<Tier1F>) * Tier1F::WARPS;
    cudaFuncSetAttribute(finalize_kernel<Tier1F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int grid;
    if (cpw > 0) {
        const int64_t warps = (p.count + cpw - 1) / cpw;
        grid = (int)((warps + Tier1F::WARPS - 1) / Tier1F::WARPS);
    } else {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, finalize_kernel<Tier1F>, Tier1F::WARPS * 32, smem);
        grid = num_sms * (per_sm < 1 ? 1 : per_sm);
    }
    finalize_kernel<Tier1F><<<grid, Tier1F::WARPS * 32, smem, st>>>(p, cpw);
    return cudaGetLastError();
}

cudaError_t launch_cells(int tier, const CellParams& p, cudaStream_t st, int num_sms, int* launches, bool with_finalize) {
    if (launches) ++*launches;
    if (tier == 0) {
        cudaError_t e = launch_tier1(p, st, num_sms);
        if (e != cudaSuccess || !with_finalize) return e;
        return launch_finalize(p, st, num_sms, 0, launches);
    }
    if (tier == 1) return launch_tier<Tier2, kDynMode>(p, 1, st, num_sms);
    return launch_tier<Tier3, kDynMode>(p, 2, st, num_sms);
}

cudaError_t launch_tier1(const CellParams& p, cudaStream_t st, int num_sms) {
    {
        // tier 1: specialized kernels for the common modes, each with and without the pd_stats counters
        constexpr unsigned S = PD_STATS;
        switch (p.flags & (kModeBits | PD_STATS)) {
            case 0: return launch_tier<Tier1, 0u>(p, 0, st, num_sms);
            case S: return launch_tier<Tier1, S>(p, 0, st, num_sms);
            case PD_PAPER_BOUND: return launch_tier<Tier1, PD_PAPER_BOUND>(p, 0, st, num_sms);
            case PD_PAPER_BOUND | S: return launch_tier<Tier1, PD_PAPER_BOUND | S>(p, 0, st, num_sms);
            case PD_ISOTROPIC: return launch_tier<Tier1, PD_ISOTROPIC>(p, 0, st, num_sms);
            case PD_ISOTROPIC | S: return launch_tier<Tier1, PD_ISOTROPIC | S>(p, 0, st, num_sms);
            case PD_DFS: return launch_tier<Tier1, PD_DFS>(p, 0, st, num_sms);
            case PD_DFS | S: return launch_tier<Tier1, PD_DFS | S>(p, 0, st, num_sms);
            case PD_WARM_START: return launch_tier<Tier1, PD_WARM_START>(p, 0, st, num_sms);
            case PD_WARM_START | S: return launch_tier<Tier1, PD_WARM_START | S>(p, 0, st, num_sms);
            default: return launch_tier<Tier1, kDynMode>(p, 0, st, num_sms);
        }
    }
}

size_t cells_global_state_bytes(int num_sms) {
    return (size_t)tier_grid<Tier3, kDynMode>(num_sms) * (Tier3::COOP ? 1 : Tier3::WARPS) * sizeof(WarpState<Tier3>);
}

int cells_grid_warps(int tier, int num_sms) {
    // all tier-1 instantiations share one register/smem footprint bound; take the largest grid
    if (tier == 0) {
        int g = tier_grid<Tier1, 0u>(num_sms);
        g = max(g, tier_grid<Tier1, PD_STATS>(num_sms));
        g = max(g, tier_grid<Tier1, PD_PAPER_BOUND>(num_sms));
        g = max(g, tier_grid<Tier1, PD_ISOTROPIC>(num_sms));
        g = max(g, tier_grid<Tier1, PD_DFS>(num_sms));
        g = max(g, tier_grid<Tier1, PD_WARM_START>(num_sms));
        g = max(g, tier_grid<Tier1, kDynMode>(num_sms));
        return g * Tier1::WARPS;
    }
    // cell programs (spill stacks): one per warp, or one per CTA in a cooperative tier
    if (tier == 1) return tier_grid<Tier2, kDynMode>(num_sms) * (Tier2::COOP ? 1 : Tier2::WARPS);
    return tier_grid<Tier3, kDynMode>(num_sms) * (Tier3::COOP ? 1 : Tier3::WARPS);
}

}  // namespace pd
