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
//   * a warp owns a cell; vertices (FP64 positions in site-local coordinates + plane-index triplets)
//     and planes live in shared memory; classification is one FMA chain per lane + __ballot_sync;
//   * the hole of a clip is found without the serial circular list of PAPER.md:556: a removed
//     vertex's directed dual edge (x->y) is on the hole boundary iff no other removed vertex holds
//     (y->x); every boundary edge independently spawns the vertex (h, x, y);
//   * the queue is re-validated in parallel at every pop (all lanes, all entries), dropping entries
//     the shrunk cell has made cullable;
//   * capacity tiers: cells that outgrow the tier's on-chip arrays are handed to a larger tier.
#include <cuda_runtime.h>
#include <stdint.h>

#include "pd_internal.cuh"

namespace pd {
namespace {

constexpr unsigned FULL = 0xffffffffu;

template <int V, int P, int Q, int W>
struct TierCfg {
    static constexpr int VMAX = V;   // vertices
    static constexpr int PMAX = P;   // planes (<= 1024: 10-bit triplet fields)
    static constexpr int QMAX = Q;   // priority-queue entries
    static constexpr int WARPS = W;  // warps per block
    static constexpr int VC = V / 32;
    static constexpr int PC = P / 32;
    static constexpr int QC = Q / 32;
};

using Tier1 = TierCfg<96, 64, 96, 4>;
using Tier2 = TierCfg<384, 192, 384, 4>;
using Tier3 = TierCfg<2048, 1024, 2048, 1>;

template <class T>
struct __align__(16) WarpState {
    double4 pl[T::PMAX];          // plane n.y <= d (n = p_j - p_i, local coordinates)
    double vx[T::VMAX], vy[T::VMAX], vz[T::VMAX];
    uint32_t vt[T::VMAX];         // triplet a | b << 10 | c << 20, CCW seen from outside
    int32_t pid[T::PMAX];         // >= 0 Morton index of the neighbour site; -1-k box wall k
    float4 qlo[T::QMAX];          // priority queue: the pushed child records (lo, maxw), (hi, link)
    float4 qhi[T::QMAX];
    uint16_t rem[T::VMAX];        // removed-vertex slots of the current clip
    uint32_t omask[T::VC];        // outside-vertex ballots of the current clip
    uint32_t qmask[T::QC];        // alive-entry ballots of the current pop
    uint32_t bnd[T::VMAX + 64];   // boundary edges (x | y << 16) of the current clip
    uint16_t tw[3][T::VMAX];      // finalize: twin vertex across edges a->b, b->c, c->a
    uint16_t pmap[T::PMAX];       // plane GC remap
    int32_t nb_id[T::PMAX];       // finalize: neighbour staging
    float nb_area[T::PMAX];
};

__device__ __forceinline__ int ford(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float iford(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__device__ __forceinline__ uint32_t tpack(int a, int b, int c) { return (uint32_t)a | ((uint32_t)b << 10) | ((uint32_t)c << 20); }
__device__ __forceinline__ int ta(uint32_t t) { return t & 1023; }
__device__ __forceinline__ int tb(uint32_t t) { return (t >> 10) & 1023; }
__device__ __forceinline__ int tc(uint32_t t) { return (t >> 20) & 1023; }
// does triplet t contain the directed dual edge x->y ?
__device__ __forceinline__ bool has_edge(uint32_t t, int x, int y) {
    int a = ta(t), b = tb(t), c = tc(t);
    return (a == x && b == y) || (b == x && c == y) || (c == x && a == y);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(FULL, v, src); }
__device__ __forceinline__ float4 shfl_f4(float4 v, int src) {
    return make_float4(__shfl_sync(FULL, v.x, src), __shfl_sync(FULL, v.y, src), __shfl_sync(FULL, v.z, src),
                       __shfl_sync(FULL, v.w, src));
}
// Exact node tests switch on once a cell has visited this many nodes (heavy cells), or always with
// PD_EXACT_NODES; PD_NO_EXACT disables them.
constexpr unsigned long long kExactAfterNodes = 64;
__device__ __forceinline__ bool exact_on(unsigned flags, unsigned long long visited) {
    if (flags & PD_NO_EXACT) return false;
    return (flags & PD_EXACT_NODES) || visited > kExactAfterNodes;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

enum { ST_OK = 0, ST_EMPTY = 1, ST_OVERFLOW = 2, ST_DUP = 3 };
enum { CLIP_NONE = 0, CLIP_DONE = 1, CLIP_EMPTY = 2, CLIP_OVF = 3 };

struct Counters {
    unsigned long long nodes, leaves, sites, tests, clips, spills;
};

// Per-warp register state (identical in all lanes).
struct Cell {
    double px, py, pz, pw;  // site (world), weight
    float fpx, fpy, fpz, fpw;
    float flo[3], fhi[3];   // cell AABB, site-local, rounded outward
    float rmax;             // max corner distance of the AABB (isotropic radius bound)
    int nv, np, nq;
    int self;               // Morton index
    int self_orig;
};

// r^2 of the directional radius for an octant set (one corner per octant is
// sound).  allow bit 2k: + side on axis k; bit 2k+1: - side.
__device__ __forceinline__ float dir_r2(const Cell& c, unsigned allow, bool iso) {
    float r2 = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float h2 = c.fhi[k] * c.fhi[k], l2 = c.flo[k] * c.flo[k];
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
__device__ __forceinline__ float node_test(const Cell& c, float4 lo_w, float4 hi_l, unsigned flags, bool& culled) {
    const bool iso = (flags & PD_ISOTROPIC) != 0;
    const bool paper = (flags & (PD_PAPER_BOUND | PD_ISOTROPIC)) != 0;
    float a0 = lo_w.x - c.fpx, a1 = lo_w.y - c.fpy, a2 = lo_w.z - c.fpz;
    float b0 = hi_l.x - c.fpx, b1 = hi_l.y - c.fpy, b2 = hi_l.z - c.fpz;
    float g0 = fmaxf(fmaxf(a0, -b0), 0.f), g1 = fmaxf(fmaxf(a1, -b1), 0.f), g2 = fmaxf(fmaxf(a2, -b2), 0.f);
    float d2 = g0 * g0 + g1 * g1 + g2 * g2;
    unsigned allow = (b0 >= 0.f ? 1u : 0u) | (a0 <= 0.f ? 2u : 0u) | (b1 >= 0.f ? 4u : 0u) | (a1 <= 0.f ? 8u : 0u) |
                     (b2 >= 0.f ? 16u : 0u) | (a2 <= 0.f ? 32u : 0u);
    float dw = c.fpw - lo_w.w;
    float dwn = fminf(0.f, dw);
    float r2 = dir_r2(c, allow, iso);
    float rd = sqrtf(r2 * d2);
    culled = d2 + dwn - 2.f * rd > 1e-5f * (d2 - dwn + 2.f * rd);
    if (!paper) {
        float h0 = fmaxf(fmaxf(c.flo[0] * a0, c.flo[0] * b0), fmaxf(c.fhi[0] * a0, c.fhi[0] * b0));
        float h1 = fmaxf(fmaxf(c.flo[1] * a1, c.flo[1] * b1), fmaxf(c.fhi[1] * a1, c.fhi[1] * b1));
        float h2 = fmaxf(fmaxf(c.flo[2] * a2, c.flo[2] * b2), fmaxf(c.fhi[2] * a2, c.fhi[2] * b2));
        float H = h0 + h1 + h2;
        float mag = fmaxf(fabsf(c.flo[0]), c.fhi[0]) * fmaxf(fabsf(a0), fabsf(b0)) +
                    fmaxf(fabsf(c.flo[1]), c.fhi[1]) * fmaxf(fabsf(a1), fabsf(b1)) +
                    fmaxf(fabsf(c.flo[2]), c.fhi[2]) * fmaxf(fabsf(a2), fabsf(b2));
        culled |= d2 + dw - 2.f * H > 1e-5f * (d2 + fabsf(dw) + 2.f * mag);
    }
    return d2 + dwn - r2;
}

template <class T>
__device__ __noinline__ void update_aabb(WarpState<T>& S, Cell& c, int lane) {
    float lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY, hi2 = -INFINITY;
    for (int s = lane; s < c.nv; s += 32) {
        double x = S.vx[s], y = S.vy[s], z = S.vz[s];
        lo0 = fminf(lo0, __double2float_rd(x)); hi0 = fmaxf(hi0, __double2float_ru(x));
        lo1 = fminf(lo1, __double2float_rd(y)); hi1 = fmaxf(hi1, __double2float_ru(y));
        lo2 = fminf(lo2, __double2float_rd(z)); hi2 = fmaxf(hi2, __double2float_ru(z));
    }
    c.flo[0] = iford(__reduce_min_sync(FULL, ford(lo0)));
    c.flo[1] = iford(__reduce_min_sync(FULL, ford(lo1)));
    c.flo[2] = iford(__reduce_min_sync(FULL, ford(lo2)));
    c.fhi[0] = iford(__reduce_max_sync(FULL, ford(hi0)));
    c.fhi[1] = iford(__reduce_max_sync(FULL, ford(hi1)));
    c.fhi[2] = iford(__reduce_max_sync(FULL, ford(hi2)));
    float rm2 = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) rm2 += fmaxf(c.flo[k] * c.flo[k], c.fhi[k] * c.fhi[k]);
    c.rmax = sqrtf(rm2);
}

// Plane garbage collection: drop planes no vertex references.
template <class T>
__device__ __noinline__ void plane_gc(WarpState<T>& S, Cell& c, int lane) {
    for (int f = lane; f < c.np; f += 32) S.pmap[f] = 0;
    __syncwarp();
    for (int s = lane; s < c.nv; s += 32) {
        uint32_t t = S.vt[s];
        S.pmap[ta(t)] = 1; S.pmap[tb(t)] = 1; S.pmap[tc(t)] = 1;
    }
    __syncwarp();
    int base = 0;
    for (int f0 = 0; f0 < c.np; f0 += 32) {
        int f = f0 + lane;
        bool live = f < c.np && S.pmap[f];
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
    for (int s = lane; s < c.nv; s += 32) {
        uint32_t t = S.vt[s];
        S.vt[s] = tpack(S.pmap[ta(t)], S.pmap[tb(t)], S.pmap[tc(t)]);
    }
    c.np = base;
    __syncwarp();
}

__device__ __forceinline__ void solve3(double4 a, double4 b, double4 c, double& x, double& y, double& z) {
    double bcx = b.y * c.z - b.z * c.y, bcy = b.z * c.x - b.x * c.z, bcz = b.x * c.y - b.y * c.x;
    double cax = c.y * a.z - c.z * a.y, cay = c.z * a.x - c.x * a.z, caz = c.x * a.y - c.y * a.x;
    double abx = a.y * b.z - a.z * b.y, aby = a.z * b.x - a.x * b.z, abz = a.x * b.y - a.y * b.x;
    double det = a.x * bcx + a.y * bcy + a.z * bcz;
    double inv = 1.0 / det;
    x = (a.w * bcx + b.w * cax + c.w * abx) * inv;
    y = (a.w * bcy + b.w * cay + c.w * aby) * inv;
    z = (a.w * bcz + b.w * caz + c.w * abz) * inv;
}

// Clip the cell by {y : n.y <= d} (re-designed warp-parallel).
template <class T>
__device__ __noinline__ int clip(WarpState<T>& S, Cell& c, int lane, double nx, double ny, double nz, double d,
                                 double tol, int pidn) {
    if (c.np >= (T::PMAX * 85) / 100) {
        plane_gc(S, c, lane);
        if (c.np >= T::PMAX) return CLIP_OVF;
    }
    // 1. classify (outside <=> s > tol; on-plane vertices are kept)
    int R = 0;
    const int nch = (c.nv + 31) >> 5;
    for (int ch = 0; ch < nch; ++ch) {
        int s = ch * 32 + lane;
        bool out = false;
        if (s < c.nv) out = fma(nx, S.vx[s], fma(ny, S.vy[s], nz * S.vz[s])) - d > tol;
        unsigned m = __ballot_sync(FULL, out);
        if (out) S.rem[R + __popc(m & lanemask_lt())] = (uint16_t)s;  // removed slots, ascending
        if (lane == 0) S.omask[ch] = m;
        R += __popc(m);
    }
    if (R == 0) return CLIP_NONE;
    if (R == c.nv) return CLIP_EMPTY;
    __syncwarp();
    // 2. hole boundary: edge x->y of a removed vertex is a boundary edge iff its reverse y->x is not
    //    held by another removed vertex.
    int B = 0;
    for (int r0 = 0; r0 < R; r0 += 32) {
        int r = r0 + lane;
        int nb = 0;
        uint32_t e[3];
        if (r < R) {
            uint32_t t = S.vt[S.rem[r]];
            int a = ta(t), b = tb(t), cc = tc(t);
            bool f0 = false, f1 = false, f2 = false;
            #pragma unroll 1
            for (int k = 0; k < R; ++k) {
                uint32_t u = S.vt[S.rem[k]];
                f0 |= has_edge(u, b, a);
                f1 |= has_edge(u, cc, b);
                f2 |= has_edge(u, a, cc);
            }
            if (!f0) e[nb++] = (uint32_t)a | ((uint32_t)b << 16);
            if (!f1) e[nb++] = (uint32_t)b | ((uint32_t)cc << 16);
            if (!f2) e[nb++] = (uint32_t)cc | ((uint32_t)a << 16);
        }
        // inclusive scan of nb
        int inc = nb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += v;
        }
        int tot = __shfl_sync(FULL, inc, 31);
        int pos = B + inc - nb;
        if (B + tot <= T::VMAX + 64) {
            for (int k = 0; k < nb; ++k) S.bnd[pos + k] = e[k];
        }
        B += tot;
    }
    int nvn = c.nv - R + B;
    if (nvn > T::VMAX || B > T::VMAX + 64 || c.np + 1 > T::PMAX) return CLIP_OVF;
    // 3. append the plane, create (h, x, y) for every boundary edge
    int hs = c.np;
    if (lane == 0) {
        S.pl[hs] = make_double4(nx, ny, nz, d);
        S.pid[hs] = pidn;
    }
    __syncwarp();
    double4 ph = make_double4(nx, ny, nz, d);
    for (int e0 = 0; e0 < B; e0 += 32) {
        int e = e0 + lane;
        if (e < B) {
            uint32_t be = S.bnd[e];
            int x = be & 0xffff, y = be >> 16;
            double vx, vy, vz;
            solve3(ph, S.pl[x], S.pl[y], vx, vy, vz);
            int slot = e < R ? S.rem[e] : c.nv + (e - R);
            S.vx[slot] = vx; S.vy[slot] = vy; S.vz[slot] = vz;
            S.vt[slot] = tpack(hs, x, y);
        }
    }
    // 4. if fewer vertices were created than removed, move kept vertices from the tail into holes
    if (B < R) {
        int moved = 0;
        for (int ch = nvn >> 5; ch < nch; ++ch) {
            int s = ch * 32 + lane;
            bool mover = s >= nvn && s < c.nv && !((S.omask[ch] >> lane) & 1u);
            unsigned mm = __ballot_sync(FULL, mover);
            if (mover) {
                int dst = S.rem[B + moved + __popc(mm & lanemask_lt())];
                S.vx[dst] = S.vx[s]; S.vy[dst] = S.vy[s]; S.vz[dst] = S.vz[s];
                S.vt[dst] = S.vt[s];
            }
            moved += __popc(mm);
        }
    }
    c.nv = nvn;
    c.np = hs + 1;
    __syncwarp();
    update_aabb(S, c, lane);
    return CLIP_DONE;
}

// Site test in FP64: cull iff the plane y.D <= q/2 (q = |D|^2 + w_i - w_j)
// cannot cut the cell.  Paper: d_ij = q/(2|D|) > r with r the directional radius of p_j's octant,
// i.e. q > 0 and q^2 > 4 r^2 |D|^2.  Default: the exact support of the cell AABB in direction D,
// h = sum_k max(lo_k D_k, hi_k D_k) <= r |D| (Cauchy-Schwarz), cull iff q/2 > h: never looser.
__device__ __forceinline__ bool site_culled(const Cell& c, double Dx, double Dy, double Dz, double q, double D2,
                                            unsigned flags) {
    if (!(flags & (PD_PAPER_BOUND | PD_ISOTROPIC))) {
        double h = Dx * (Dx >= 0 ? (double)c.fhi[0] : (double)c.flo[0]) + Dy * (Dy >= 0 ? (double)c.fhi[1] : (double)c.flo[1]) +
                   Dz * (Dz >= 0 ? (double)c.fhi[2] : (double)c.flo[2]);
        return 0.5 * q > h + 1e-9 * (fabs(h) + D2);
    }
    double r2;
    if (flags & PD_ISOTROPIC) {
        r2 = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) r2 += (double)fmaxf(c.flo[k] * c.flo[k], c.fhi[k] * c.fhi[k]);
    } else {
        double hx = Dx >= 0 ? c.fhi[0] : c.flo[0], hy = Dy >= 0 ? c.fhi[1] : c.flo[1], hz = Dz >= 0 ? c.fhi[2] : c.flo[2];
        r2 = hx * hx + hy * hy + hz * hz;
    }
    return q > 0 && q * q > 4.0 * r2 * D2 * (1.0 + 1e-9);
}

// Exact polytope-vs-box node test (not in the paper; strictly tighter than any AABB bound).  The
// plane of p_j (D = p_j - p_i) cuts the cell iff some vertex v has v.D - |D|^2/2 > (w_i - w_j)/2.
// Over all p_j in the box, D_k in [a_k, b_k] and w_j <= w_max, and
//   max_{D in box} (v.D - |D|^2/2) = sum_k (v_k c_k - c_k^2/2),  c_k = clamp(v_k, a_k, b_k),
// (a separable concave maximisation), so the node is culled iff for every vertex that sum is
// <= (w_i - w_max)/2.  Lanes = vertices, FP64, relative margin so rounding only keeps nodes.
template <class T>
__device__ __noinline__ bool node_exact_culled(const WarpState<T>& S, const Cell& c, int lane, float4 lo_w, float4 hi_l) {
    const double a0 = (double)lo_w.x - c.px, a1 = (double)lo_w.y - c.py, a2 = (double)lo_w.z - c.pz;
    const double b0 = (double)hi_l.x - c.px, b1 = (double)hi_l.y - c.py, b2 = (double)hi_l.z - c.pz;
    const double rhs = 0.5 * (c.pw - (double)lo_w.w);
    double best = -1e300, mag = 0.0;
    for (int s = lane; s < c.nv; s += 32) {
        double vx = S.vx[s], vy = S.vy[s], vz = S.vz[s];
        double cx = fmin(fmax(vx, a0), b0), cy = fmin(fmax(vy, a1), b1), cz = fmin(fmax(vz, a2), b2);
        double f = cx * (vx - 0.5 * cx) + cy * (vy - 0.5 * cy) + cz * (vz - 0.5 * cz);
        best = fmax(best, f);
        mag = fmax(mag, fabs(cx * vx) + fabs(cy * vy) + fabs(cz * vz));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        best = fmax(best, __shfl_xor_sync(FULL, best, o));
        mag = fmax(mag, __shfl_xor_sync(FULL, mag, o));
    }
    return best < rhs - 1e-12 * (mag + fabs(rhs));
}

template <class T>
__device__ __noinline__ int process_leaf(WarpState<T>& S, Cell& c, int lane, int link, const CellParams& P, Counters& cnt) {
    int first = leaf_first(link), count = leaf_count(link);
    int j = first + lane;
    bool valid = lane < count && j != c.self;
    double Dx = 0, Dy = 0, Dz = 0, q = 0, D2 = 0;
    float wj = 0.f;
    bool dup_kill = false;
    if (valid) {
        float4 s = __ldg(&P.sites[j]);
        wj = s.w;
        Dx = (double)s.x - c.px; Dy = (double)s.y - c.py; Dz = (double)s.z - c.pz;
        D2 = Dx * Dx + Dy * Dy + Dz * Dz;
        q = D2 + (c.pw - (double)s.w);
        if (D2 == 0.0) {
            // coincident sites: the heavier owns, ties to the lower id
            if (s.w > c.fpw || (s.w == c.fpw && __ldg(&P.perm[j]) < c.self_orig)) dup_kill = true;
            valid = false;
        }
    }
    if (__any_sync(FULL, dup_kill)) return ST_DUP;
    cnt.sites += __popc(__ballot_sync(FULL, lane < count));
    bool cand = valid && !site_culled(c, Dx, Dy, Dz, q, D2, P.flags);
    unsigned mask = __ballot_sync(FULL, cand);
    if (!mask) return ST_OK;
    // Batch cut test, lane = candidate: does the plane cut the CURRENT cell?  A plane that does not
    // cut it cannot cut any later (smaller) cell, so it is dropped for good.  Same FP64 predicate
    // as clip().
    const float nD = sqrtf((float)D2);
    const double tol = 1e-12 * (double)nD * (double)c.rmax;
    const double dd = 0.5 * q;
    {
        bool cuts = false;
#pragma unroll 2
        for (int k = 0; k < c.nv; ++k) {
            double s = fma(Dx, S.vx[k], fma(Dy, S.vy[k], Dz * S.vz[k])) - dd;
            cuts |= s > tol;
        }
        cnt.tests += __popc(mask);
        cand = cand && cuts;
        mask = __ballot_sync(FULL, cand);
    }
    float key = cand ? (float)(q / (double)nD) : INFINITY;  // 2 d_ij: nearest plane first
    while (mask) {
        int kmin = __reduce_min_sync(FULL, cand ? ford(key) : 0x7fffffff);
        unsigned lead = __ballot_sync(FULL, cand && ford(key) == kmin);
        int src = __ffs(lead) - 1;
        double nx = shfl_d(Dx, src), ny = shfl_d(Dy, src), nz = shfl_d(Dz, src), qq = shfl_d(dd, src);
        double tt = shfl_d(tol, src);
        int jj = __shfl_sync(FULL, j, src);
        if (lane == src) cand = false;
        int st = clip(S, c, lane, nx, ny, nz, qq, tt, jj);
        if (st == CLIP_EMPTY) return ST_EMPTY;
        if (st == CLIP_OVF) return ST_OVERFLOW;
        if (st == CLIP_DONE) {
            cnt.clips++;
            if (cand && site_culled(c, Dx, Dy, Dz, q, D2, P.flags)) cand = false;
        }
        mask = __ballot_sync(FULL, cand);
    }
    return ST_OK;
}

// Best-first traversal (Alg. 1).  Queue entries are the pushed child records;
// when the on-chip queue is full, entries spill to a per-warp stack in global memory (order is
// relaxed, correctness is not affected) and are refilled when the on-chip queue drains.
template <class T>
__device__ int traverse(WarpState<T>& S, Cell& c, int lane, const CellParams& P, Counters& cnt, NodeChild* spill,
                        int spill_cap) {
    const bool dfs = (P.flags & PD_DFS) != 0;
    int node = __float_as_int(__ldg(&P.root->hi_l.w));
    bool have = true;
    int ns = 0;  // spilled entries
    const unsigned long long nodes0 = cnt.nodes;
    c.nq = 0;
    for (;;) {
        if (have) {
            while (node >= 0) {  // descend (Alg. 1 lines 4-18)
                cnt.nodes++;
                float key = INFINITY;
                bool culled = true;
                float4 lo_w = make_float4(0, 0, 0, 0), hi_l = make_float4(0, 0, 0, 0);
                if (lane < 2) {
                    const NodeChild* ch = &P.nodes[node].c[lane];
                    lo_w = __ldg(&ch->lo_w);
                    hi_l = __ldg(&ch->hi_l);
                    key = node_test(c, lo_w, hi_l, P.flags, culled);
                }
                bool c0 = __shfl_sync(FULL, culled, 0), c1 = __shfl_sync(FULL, culled, 1);
                if (exact_on(P.flags, cnt.nodes - nodes0)) {
                    float4 l0 = shfl_f4(lo_w, 0), h0 = shfl_f4(hi_l, 0), l1 = shfl_f4(lo_w, 1), h1 = shfl_f4(hi_l, 1);
                    if (!c0) c0 = node_exact_culled(S, c, lane, l0, h0);
                    if (!c1) c1 = node_exact_culled(S, c, lane, l1, h1);
                    if (lane == 0) culled = c0;
                    if (lane == 1) culled = c1;
                }
                if (c0 && c1) { have = false; break; }
                float k0 = __shfl_sync(FULL, key, 0), k1 = __shfl_sync(FULL, key, 1);
                int near = (!c0 && (c1 || k0 <= k1)) ? 0 : 1;
                int far = 1 - near;
                bool cfar = far ? c1 : c0;
                int lnear = __shfl_sync(FULL, __float_as_int(hi_l.w), near);
                if (!cfar) {
                    if (c.nq < T::QMAX) {
                        if (lane == far) { S.qlo[c.nq] = lo_w; S.qhi[c.nq] = hi_l; }
                        c.nq++;
                    } else {
                        if (ns >= spill_cap) return ST_OVERFLOW;
                        if (lane == far) { spill[ns].lo_w = lo_w; spill[ns].hi_l = hi_l; }
                        ns++;
                        cnt.spills++;
                    }
                }
                node = lnear;
            }
            if (have) {
                cnt.leaves++;
                __syncwarp();
                int st = process_leaf(S, c, lane, node, P, cnt);
                if (st != ST_OK) return st;
            }
        }
        // pop (Alg. 1 lines 21-31): re-validate every queued entry against the shrunk cell
        __syncwarp();
        if (c.nq == 0 && ns > 0) {  // refill from the spill stack
            __threadfence_block();
            int m = min(ns, T::QMAX);
            for (int t = lane; t < m; t += 32) {
                NodeChild e = spill[ns - m + t];
                S.qlo[t] = e.lo_w;
                S.qhi[t] = e.hi_l;
            }
            ns -= m;
            c.nq = m;
            __syncwarp();
        }
        if (c.nq == 0) return ST_OK;
        if (dfs) {
            bool ok = false;
            while (c.nq > 0 && !ok) {
                int t = c.nq - 1;
                bool culled;
                node_test(c, S.qlo[t], S.qhi[t], P.flags, culled);
                node = __float_as_int(S.qhi[t].w);
                c.nq--;
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
        int bestk = 0x7fffffff, bests = -1;
        const int qch = (c.nq + 31) >> 5;
        for (int ch = 0; ch < qch; ++ch) {
            int s = ch * 32 + lane;
            bool al = false;
            if (s < c.nq) {
                bool culled;
                float k = node_test(c, S.qlo[s], S.qhi[s], P.flags, culled);
                al = !culled;
                if (al && ford(k) < bestk) { bestk = ford(k); bests = s; }
            }
            unsigned am = __ballot_sync(FULL, al);
            if (lane == 0) S.qmask[ch] = am;
        }
        __syncwarp();
        int gk = __reduce_min_sync(FULL, bestk);
        if (gk == 0x7fffffff) {
            c.nq = 0;
            have = false;
            if (ns > 0) continue;
            return ST_OK;
        }
        unsigned lead = __ballot_sync(FULL, bestk == gk);
        int bslot = __shfl_sync(FULL, bests, __ffs(lead) - 1);
        node = __float_as_int(S.qhi[bslot].w);
        bool popped_dead = exact_on(P.flags, cnt.nodes - nodes0) && node_exact_culled(S, c, lane, S.qlo[bslot], S.qhi[bslot]);
        // compact: keep alive entries except the popped one
        int base = 0;
        for (int ch = 0; ch < qch; ++ch) {
            int s = ch * 32 + lane;
            bool keep = ((S.qmask[ch] >> lane) & 1u) && s != bslot;
            unsigned km = __ballot_sync(FULL, keep);
            float4 lo = make_float4(0, 0, 0, 0), hi = make_float4(0, 0, 0, 0);
            if (keep) { lo = S.qlo[s]; hi = S.qhi[s]; }
            __syncwarp();
            if (keep) {
                int dst = base + __popc(km & lanemask_lt());
                S.qlo[dst] = lo;
                S.qhi[dst] = hi;
            }
            __syncwarp();
            base += __popc(km);
        }
        c.nq = base;
        have = !popped_dead;
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
        S.vx[lane] = sx ? hi[0] : lo[0];
        S.vy[lane] = sy ? hi[1] : lo[1];
        S.vz[lane] = sz ? hi[2] : lo[2];
        int X = sx, Y = 2 + sy, Z = 4 + sz;
        int sgn = (sx ? 1 : -1) * (sy ? 1 : -1) * (sz ? 1 : -1);  // det of the outward normals
        S.vt[lane] = sgn > 0 ? tpack(X, Y, Z) : tpack(X, Z, Y);
    }
    float rm2 = 0.f;
    for (int k = 0; k < 3; ++k) {
        c.flo[k] = __double2float_rd(lo[k]);
        c.fhi[k] = __double2float_ru(hi[k]);
        rm2 += fmaxf(c.flo[k] * c.flo[k], c.fhi[k] * c.fhi[k]);
    }
    c.rmax = sqrtf(rm2);
    c.nv = 8;
    c.np = 6;
    c.nq = 0;
    __syncwarp();
}

// Face areas (vector area 1/2 sum v x next(v) around each face), volume, neighbours.
template <class T>
__device__ __noinline__ void finalize(WarpState<T>& S, Cell& c, int lane, const CellParams& P, int status) {
    const int i = c.self_orig;
    const CellOut& O = P.out;
    if (status == ST_EMPTY || status == ST_DUP || status == ST_OVERFLOW) {
        if (lane == 0) {
            O.cnt[i] = 0;
            O.aoff[i] = 0;
            O.vol[i] = 0.f;
            O.surf[i] = 0.f;
            O.flags[i] = (uint8_t)(status == ST_OVERFLOW ? PD_CELL_OVERFLOW
                                                         : (PD_CELL_EMPTY | (status == ST_DUP ? PD_CELL_DUPLICATE : 0)));
        }
        return;
    }
    // twins: vertex across each directed edge
    for (int u = lane; u < c.nv; u += 32) {
        uint32_t t = S.vt[u];
        int a = ta(t), b = tb(t), cc = tc(t);
        uint16_t t0 = 0xffff, t1 = 0xffff, t2 = 0xffff;
        #pragma unroll 1
        for (int k = 0; k < c.nv; ++k) {
            uint32_t w = S.vt[k];
            if (has_edge(w, b, a)) t0 = (uint16_t)k;
            if (has_edge(w, cc, b)) t1 = (uint16_t)k;
            if (has_edge(w, a, cc)) t2 = (uint16_t)k;
        }
        S.tw[0][u] = t0; S.tw[1][u] = t1; S.tw[2][u] = t2;
    }
    __syncwarp();
    double vol = 0, surf = 0;
    bool boundary = false;
    int K = 0;
    for (int f0 = 0; f0 < c.np; f0 += 32) {
        int f = f0 + lane;
        double Ax = 0, Ay = 0, Az = 0;
        if (f < c.np) {
            #pragma unroll 1
            for (int u = 0; u < c.nv; ++u) {
                uint32_t t = S.vt[u];
                int which = ta(t) == f ? 2 : (tb(t) == f ? 0 : (tc(t) == f ? 1 : -1));
                if (which >= 0) {
                    int w = S.tw[which][u];
                    if (w == 0xffff) continue;
                    double ux = S.vx[u], uy = S.vy[u], uz = S.vz[u];
                    double wx = S.vx[w], wy = S.vy[w], wz = S.vz[w];
                    Ax += uy * wz - uz * wy;
                    Ay += uz * wx - ux * wz;
                    Az += ux * wy - uy * wx;
                }
            }
        }
        Ax *= 0.5; Ay *= 0.5; Az *= 0.5;
        double area = sqrt(Ax * Ax + Ay * Ay + Az * Az);
        bool nb = false;
        if (f < c.np && area > 0) {
            double4 pl = S.pl[f];
            double nn = pl.x * pl.x + pl.y * pl.y + pl.z * pl.z;
            vol += (Ax * pl.x + Ay * pl.y + Az * pl.z) * pl.w / nn;
            surf += area;
            int id = S.pid[f];
            if (id < 0) boundary = true;
            else nb = true;
        }
        unsigned mb = __ballot_sync(FULL, nb);
        if (nb) {
            int pos = K + __popc(mb & lanemask_lt());
            S.nb_id[pos] = __ldg(&P.perm[S.pid[f]]);
            S.nb_area[pos] = (float)area;
        }
        K += __popc(mb);
    }
    vol = warp_sum_d(vol) / 3.0;
    surf = warp_sum_d(surf);
    boundary = __any_sync(FULL, boundary);
    __syncwarp();
    // arena row (ascending original ids)
    long long base = 0;
    if (lane == 0) base = (long long)atomicAdd(O.arena_top, (unsigned long long)K);
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
    if (lane == 0) {
        O.cnt[i] = K;
        O.aoff[i] = base;
        O.vol[i] = (float)vol;
        O.surf[i] = (float)surf;
        O.flags[i] = (uint8_t)((boundary ? PD_CELL_BOUNDARY : 0) | (vol > 0 ? 0 : PD_CELL_EMPTY));
    }
}

template <class T>
__global__ void __launch_bounds__(T::WARPS * 32) cells_kernel(CellParams P, int tier) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpState<T>& S = reinterpret_cast<WarpState<T>*>(smem_raw)[wid];
    const int64_t total = P.list ? (int64_t)(*P.list_count) : P.count;
    Counters cnt = {0, 0, 0, 0, 0, 0};
    const int gw = blockIdx.x * T::WARPS + wid;
    NodeChild* spill = P.spill + (size_t)gw * P.spill_cap;
    unsigned long long ncells = 0, novf = 0;
    constexpr int BATCH = 4;
    for (;;) {
        long long b0 = 0;
        if (lane == 0) b0 = (long long)atomicAdd(P.work_counter, (unsigned long long)BATCH);
        b0 = __shfl_sync(FULL, b0, 0);
        if (b0 >= total) break;
        for (int b = 0; b < BATCH && b0 + b < total; ++b) {
            int64_t idx = b0 + b;
            int s = P.list ? P.list[idx] : (int)(P.begin + idx);
            Cell c;
            const Counters before = cnt;
            float4 site = __ldg(&P.sites[s]);
            c.fpx = site.x; c.fpy = site.y; c.fpz = site.z; c.fpw = site.w;
            c.px = site.x; c.py = site.y; c.pz = site.z; c.pw = site.w;
            c.self = s;
            c.self_orig = __ldg(&P.perm[s]);
            init_cell(S, c, lane, P);
            int st = traverse(S, c, lane, P, cnt, spill, P.spill_cap);
            __syncwarp();
            if (st == ST_OVERFLOW && !P.last_tier) {
                if (lane == 0) {
                    int k = atomicAdd(P.next_count, 1);
                    P.next_list[k] = s;
                }
                continue;
            }
            if (st == ST_OVERFLOW) novf++;
            finalize(S, c, lane, P, st);
            ncells++;
            if ((P.flags & PD_COST) && lane == 0) {
                unsigned long long w = (cnt.nodes - before.nodes) + (cnt.sites - before.sites) + 8 * (cnt.clips - before.clips);
                P.out.cost[c.self_orig] = (int32_t)min(w, 0x7fffffffull);
            }
            __syncwarp();
        }
    }
    if ((P.flags & PD_STATS) && lane == 0) {
        atomicAdd(&P.stats->nodes, cnt.nodes);
        atomicAdd(&P.stats->leaves, cnt.leaves);
        atomicAdd(&P.stats->sites, cnt.sites);
        atomicAdd(&P.stats->clip_tests, cnt.tests);
        atomicAdd(&P.stats->clips, cnt.clips);
        atomicAdd(&P.stats->cells, ncells);
        atomicAdd(&P.stats->tier[tier], ncells);
        atomicAdd(&P.stats->overflow, novf);
        atomicAdd(&P.stats->spills, cnt.spills);
    }
}

template <class T>
int tier_grid(int num_sms) {
    size_t smem = sizeof(WarpState<T>) * T::WARPS;
    cudaFuncSetAttribute(cells_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cells_kernel<T>, T::WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    return num_sms * per_sm;
}

template <class T>
cudaError_t launch_tier(const CellParams& p, int tier, cudaStream_t st, int num_sms) {
    size_t smem = sizeof(WarpState<T>) * T::WARPS;
    int grid = tier_grid<T>(num_sms);
    cells_kernel<T><<<grid, T::WARPS * 32, smem, st>>>(p, tier);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_cells(int tier, const CellParams& p, cudaStream_t st, int num_sms, int* launches) {
    if (launches) ++*launches;
    if (tier == 0) return launch_tier<Tier1>(p, 0, st, num_sms);
    if (tier == 1) return launch_tier<Tier2>(p, 1, st, num_sms);
    return launch_tier<Tier3>(p, 2, st, num_sms);
}

int cells_grid_warps(int tier, int num_sms) {
    if (tier == 0) return tier_grid<Tier1>(num_sms) * Tier1::WARPS;
    if (tier == 1) return tier_grid<Tier2>(num_sms) * Tier2::WARPS;
    return tier_grid<Tier3>(num_sms) * Tier3::WARPS;
}

}  // namespace pd
