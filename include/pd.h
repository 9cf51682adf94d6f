/*
 * pd.h -- C ABI of the B200 (sm_100a) power / Voronoi diagram cell-construction library (libpd.so).
 *
 * Problem (§3 Eq. 1): given sites p_i with weights w_i, the power cell
 *     C_i = { x : |x - p_i|^2 - w_i <= |x - p_j|^2 - w_j  for all j != i }
 * restricted to the box B (App. "Initialization").  Equal weights give Voronoi.
 * Two sites are neighbours iff their cells share a polygonal face of positive area.
 *
 * Method (the hot path): per cell, progressive half-space clipping of B (§4.1,
 * App. "Convex cell clipping" PAPER.md:548-558) by the bisecting planes of candidates found by a
 * best-first traversal (Alg. 1) of a weight-augmented BVH (PAPER.md:295-297,
 * 526-527) pruned by the directional bound (§4.2).  Output: CSR adjacency,
 * per-face areas, per-cell volumes and flags (EMPTY etc.) -- SURVEY.md §8(b).
 *
 * Conventions (all entry points):
 *  - No C++ exceptions cross this boundary; every call returns a pd_status.
 *  - Inputs are BORROWED for the duration of the call and never retained.  They are host pointers
 *    unless PD_IN_DEVICE is set, in which case they must be device pointers on opt->device.
 *  - Outputs are OWNED by the pd_result and released by pd_free.  They live on the device unless
 *    PD_OUT_HOST is set (then they are host memory).  Accessors never transfer ownership.
 *  - Calls are synchronous with respect to the host: on return the result is complete.  Work is
 *    enqueued on opt->stream (a cudaStream_t; NULL = the legacy default stream).
 *  - On error *out is set to NULL and no partial output exists.
 *  - Thread safety: distinct pd_result objects may be built concurrently from different threads.
 *  - Ids are int32 (n <= PD_MAX_SITES).  Output is deterministic: byte-identical across runs.
 */
#ifndef PD_H
#define PD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PD_ABI_VERSION 1
#define PD_MAX_SITES ((int64_t)1 << 26) /* leaf-range encoding of the BVH: 26-bit first index */

typedef struct { float lo[3], hi[3]; } pd_box;

typedef enum {
    PD_OK = 0,
    PD_EINVAL = 1,      /* bad argument: n > PD_MAX_SITES, lo >= hi on an axis, NULL where required */
    PD_EEMPTY = 2,      /* n == 0 */
    PD_ENONFINITE = 3,  /* a coordinate or weight is NaN/Inf; pd_error_index() names it */
    PD_EOUTSIDE = 4,    /* a point lies outside the closed box; pd_error_index() names it */
    PD_ENOMEM = 5,      /* device or host allocation failed */
    PD_ECUDA = 6,       /* a CUDA runtime error (message via pd_last_cuda_error()) */
    PD_ENCCL = 7,       /* an NCCL call failed, or libnccl.so.2 is missing (message via pd_last_nccl_error()) */
    PD_EINTERNAL = 8    /* an internal invariant failed (e.g. output arena overflow twice) */
} pd_status;

/* pd_options.flags */
enum {
    PD_IN_DEVICE = 1u << 0,   /* points/weights are device pointers (else host) */
    PD_OUT_HOST = 1u << 1,    /* copy the outputs to host memory before returning */
    PD_STATS = 1u << 2,       /* collect traversal/clipping counters (pd_get_stats) */
    PD_ISOTROPIC = 1u << 3,   /* ablation: isotropic radius instead of the directional one */
    PD_DFS = 1u << 4,         /* ablation: depth-first LIFO traversal instead of best-first */
    PD_WARM_START = 1u << 5,  /* KNN warm start (K = 8): a K-nearest-neighbour query (in power
                                 distance pi_j(p_i) = |p_i-p_j|^2 - w_j) on the same BVH pre-clips every cell
                                 before its traversal; same diagram, different work (the neighbour sets are
                                 identical, areas/volumes agree to rounding) */
    PD_PAPER_BOUND = 1u << 6, /* ablation: the paper's culling bounds only (no AABB-support companion) */
    PD_COST = 1u << 7,        /* record per-cell work (pd_cell_cost): BVH nodes + leaf sites + 8 x clips (deterministic) */
    PD_EXACT_NODES = 1u << 8, /* exact polytope-vs-box node test on every node the AABB tests keep */
    PD_NO_EXACT = 1u << 9,    /* never use the exact polytope-vs-box node test (pure AABB culling) */
    PD_BALANCE = 1u << 10,    /* sharded build: equal-cost Morton slices from a sampled cost estimate
                                 (default: equal-count slices, measured better balanced on C4) */
    PD_WARM_ADAPTIVE = 1u << 12, /* warm start only the sites whose power-nearest neighbour dominates them at
                                    their own position (every EMPTY cell is such a site): the KNN query runs for
                                    all, the pre-clip only where it pays (heavy-tailed weights) */
    PD_TETS = 1u << 11,       /* also output the dual tetrahedra (the "explicit mesh"
                                 of PAPER.md:343/398): see pd_tets.  Not with shard_world > 1 (PD_EINVAL). */
    PD_NO_AUTO_WARM = 1u << 13, /* accepted for compatibility: the automatic warm-start decision is now opt-in
                                   (PD_AUTO_WARM), so this is the default */
    PD_AUTO_WARM = 1u << 14   /* decide the KNN warm start by measurement: with weights and neither PD_WARM_START
                                  nor PD_WARM_ADAPTIVE given, the tier-1 cell program runs on a strided 8k-site
                                  sample with and without the KNN pre-clip (deterministic per-cell work counters,
                                  PD_COST) and PD_WARM_START is used when sampled work with it (x 1.10, plus ~60
                                  units per site for the KNN query) is below 0.9 x the work without
                                  (pd_stats.warm_gain).  Costs two sample launches + one sync (~2-5 ms); every rank
                                  of a sharded build measures the same sample and takes the same decision.  Off by
                                  default since the queue priority became the plane-distance bound:
                                  the warm start then measured slower on every configuration (C3 170 -> 280 ms,
                                  C4 381 -> 636 ms, C5 632 -> 1079 ms) and the sample alone cost ~0.5% of C4.  The
                                  diagram is the same either way (areas/volumes to rounding). */
};

/* pd_cell_flags values */
enum {
    PD_CELL_EMPTY = 1,     /* vol == 0 (power cell empty inside the box) */
    PD_CELL_BOUNDARY = 2,  /* a box wall contributes a face of positive area */
    PD_CELL_OVERFLOW = 4,  /* exceeded the largest on-chip capacity tier: output incomplete */
    PD_CELL_DUPLICATE = 8, /* bit-identical position with a heavier (or equal, lower-id) site */
    PD_CELL_DEGRADED = 16, /* topology-consistency check failed: a clip's hole boundary
                              was not one cycle of >= 3 edges, or a face edge of the final cell has no
                              unique reverse edge; the cell's output is still written, and counted in
                              pd_stats.degraded_cells */
    PD_CELL_NOT_OWNED = 32 /* sharded build: this cell belongs to another rank's slice */
};

typedef struct {
    int device;        /* CUDA device ordinal */
    void* stream;      /* cudaStream_t (NULL = default stream) */
    int leaf_size;     /* BVH leaf size l, 1..32 (0 = default 32); PAPER.md:527 uses 17 / 10 */
    unsigned flags;    /* PD_* flags above */
    int shard_rank;    /* sharded build: this rank's slice of the Morton order (0 when world=1) */
    int shard_world;   /* number of slices (0 or 1 = whole diagram) */
} pd_options;

typedef struct {
    int64_t cells;             /* cells built by this call */
    int64_t nodes_visited;     /* internal BVH nodes whose children were tested (Alg. 1 line 5) */
    int64_t leaves_visited;    /* leaves processed (Alg. 1 ProcessLeaf) */
    int64_t sites_tested;      /* leaf sites tested against the directional bound (§4.2) */
    int64_t clip_tests;        /* candidate planes classified against the cell's vertices */
    int64_t clips;             /* clips that changed the cell */
    int64_t tier_cells[3];     /* cells finished in each capacity tier */
    int64_t overflow_cells;    /* cells flagged PD_CELL_OVERFLOW */
    int64_t queue_spills;      /* queue entries spilled to global memory */
    int64_t nnz;               /* total neighbour entries */
    double ms_bvh, ms_cells, ms_csr, ms_total; /* phase times (CUDA events) */
    double ms_tier[3];         /* cell-kernel time per capacity tier (CUDA events) */
    int64_t warp_cycles[10];   /* PD_PROFILE builds only: warp clock64 in init/descend/leaf/clip/pop/finalize,
                                  then clip's classify/boundary/create/aabb */
    double ms_knn;             /* PD_WARM_START: the K-nearest-neighbour query (part of ms_cells) */
    /* Robustness counters, always collected (BASELINE.json north_star: near-degenerate faces "counted and
     * reported"; "never silently dropped"): */
    int64_t faces_dropped;         /* bisector faces with area <= 1e-13 S_i: zero-area contacts, not neighbours
                                      (reading R2) */
    int64_t faces_near_degenerate; /* reported neighbour faces with area < 1e-9 S_i (the parity excusal band) */
    int64_t degraded_cells;        /* cells flagged PD_CELL_DEGRADED */
    double warm_gain;              /* auto warm start: sampled work ratio with / without it (0 when not sampled) */
    int64_t warm_start;            /* 1 if the KNN warm start ran (given or switched on automatically) */
} pd_stats;

typedef struct pd_result pd_result;

/* Build the diagram of n sites.
 *  points  : xyz interleaved, 3*n floats (host, or device with PD_IN_DEVICE).
 *  weights : n floats, or NULL for the Voronoi diagram (all weights 0).
 *  box     : the domain B (host struct); NULL = the tight AABB of the points.
 *            Every point must lie in the closed box.
 *  opt     : options (host struct); NULL = defaults on device 0, default stream.
 *  out     : receives the result handle (release with pd_free).
 * Errors: PD_EEMPTY (n == 0), PD_EINVAL, PD_ENONFINITE / PD_EOUTSIDE (index via pd_error_index),
 *         PD_ENOMEM, PD_ECUDA, PD_EINTERNAL. */
pd_status pd_build(const float* points, const float* weights, int64_t n, const pd_box* box,
                   const pd_options* opt, pd_result** out);

/* Accessors (valid until pd_free).  Arrays are in ORIGINAL site order. */
int64_t pd_num_cells(const pd_result* r);
int64_t pd_nnz(const pd_result* r);
int pd_on_host(const pd_result* r);              /* 1 if the arrays below are host memory */
const int64_t* pd_offsets(const pd_result* r);   /* n+1; offsets[0] = 0, offsets[n] = nnz */
const int32_t* pd_neighbors(const pd_result* r); /* nnz; per row ascending original ids; never self */
const float* pd_face_areas(const pd_result* r);  /* nnz; aligned with pd_neighbors */
const float* pd_volumes(const pd_result* r);     /* n; 0 for EMPTY */
const float* pd_surface(const pd_result* r);     /* n; total surface area incl. box walls */
const uint8_t* pd_cell_flags(const pd_result* r);/* n; PD_CELL_* bits */
const int32_t* pd_cell_cost(const pd_result* r); /* n (device); per-cell work count, only with PD_COST, else NULL */
/* Dual tetrahedra (PD_TETS): the regular (weighted Delaunay) triangulation dual to the diagram, restricted
 * to the box.  Every cell vertex where three bisector faces of positive area meet (no box wall) is the
 * centre of the tet {i, a, b, c} (the vertex is equidistant in power from the four
 * sites); each tet is listed once, by its lowest id i.  pd_tets: 4*pd_num_tets int32 original ids,
 * (i < a < b < c) per tet, grouped by i ascending, within a group in the emitting cell's vertex order.
 * NULL / 0 without PD_TETS.  Near-degenerate (cospherical) configurations may list sliver tets
 * of zero volume: the triplet dual splits a vertex of degree > 3. */
int64_t pd_num_tets(const pd_result* r);
const int32_t* pd_tets(const pd_result* r);
pd_status pd_get_stats(const pd_result* r, pd_stats* s);
void pd_free(pd_result* r);

/* Sharded builds (pd_options.shard_world > 1) compute only this rank's contiguous slice of the
 * Morton order; the slice's rows are exported in Morton order so that ranks can exchange them and
 * reassemble the full diagram with pd_assemble (the exchange itself is torch.distributed/NCCL in
 * the Python layer). */
int64_t pd_slice_begin(const pd_result* r);      /* first Morton position of this rank's slice */
int64_t pd_slice_end(const pd_result* r);
const int32_t* pd_morton_perm(const pd_result* r); /* n; Morton position -> original id (device) */

/* Reassemble a full CSR (original order) from Morton-ordered per-cell blocks gathered from all
 * ranks.  All pointers are DEVICE pointers on opt->device (rows_nbr/rows_area may be NULL only when
 * total == 0):
 *   perm[n] (Morton pos -> original id), cnt[n] (row length per Morton pos), vol/surf/flags[n]
 *   per Morton pos, rows_nbr/rows_area[total] concatenated rows in Morton order.
 * Returns a result whose arrays are in original order (on device unless PD_OUT_HOST).
 * Errors: PD_EINVAL if a pointer is NULL, n <= 0, or the row lengths cnt[] do not add up to `total`
 * (checked on the device before any row is written). */
pd_status pd_assemble(const int32_t* perm, const int32_t* cnt, const float* vol, const float* surf,
                      const uint8_t* flags, const int32_t* rows_nbr, const float* rows_area,
                      int64_t n, int64_t total, const pd_options* opt, pd_result** out);

/* Morton-ordered export of a (sharded) result, for the exchange: copies, for Morton positions
 * [pd_slice_begin, pd_slice_end), the row lengths, volumes, surfaces, flags and concatenated rows
 * into caller-provided DEVICE buffers.  Returns the number of row entries written via *total. */
pd_status pd_export_slice(const pd_result* r, int32_t* cnt, float* vol, float* surf,
                          uint8_t* flags, int32_t* rows_nbr, float* rows_area, int64_t* total,
                          void* stream);
int64_t pd_slice_nnz(const pd_result* r);

/* ---- Multi-GPU (the paper itself is single-GPU; the sharding rests on the n
 * independent clipping tasks of PAPER.md:151).  One process per GPU; NCCL (libnccl.so.2, opened at the first
 * call) over NVLink/NVSwitch inside the library, torch.distributed (or any channel) only to hand the 128-byte
 * unique id from rank 0 to the others. */
typedef struct pd_comm pd_comm;

/* Rank 0 creates the communicator's unique id (an ncclUniqueId, 128 bytes) and sends the bytes to the other
 * ranks by any means.  Errors: PD_EINVAL (uid NULL), PD_ENCCL. */
pd_status pd_comm_unique_id(unsigned char uid[128]);

/* Collective over `world` ranks: join the communicator of `uid` as `rank` on CUDA device `device`.
 * *comm receives the handle (release with pd_comm_free after the last pd_build_sharded).
 * Errors: PD_EINVAL (rank/world/device out of range, NULL), PD_ECUDA, PD_ENCCL. */
pd_status pd_comm_init(const unsigned char uid[128], int rank, int world, int device, pd_comm** comm);

/* Collective: the diagram of n sites built by all ranks of `comm` together.
 *  points/weights/box : as pd_build, read on RANK 0 ONLY (other ranks may pass NULL); every rank passes the
 *                       same n.  opt->device is ignored (the communicator's device is used); PD_TETS is
 *                       not available (PD_EINVAL).
 * Rank 0 packs and validates the input and builds the LBVH; NCCL broadcasts a header (status, n, box) and the
 * LBVH -- Morton-sorted sites (16 B/site), the permutation (4 B/site) and the wide nodes -- to every rank.
 * Each rank builds the cells of its contiguous slice of the Morton order (equal count, or equal estimated cost
 * with PD_BALANCE); the per-cell fields and rows of every slice are then broadcast by their owner (grouped
 * NCCL broadcasts) and EVERY rank assembles the full original-order CSR into *out (same accessors as
 * pd_build; pd_slice_begin/end give this rank's slice).  The result is byte-identical to pd_build's.
 * Errors: as pd_build (an input error found on rank 0 is returned by every rank, with pd_error_index),
 *         PD_EINVAL (n differs from rank 0's, comm NULL), PD_ENCCL. */
pd_status pd_build_sharded(pd_comm* comm, const float* points, const float* weights, int64_t n, const pd_box* box,
                           const pd_options* opt, pd_result** out);

int pd_comm_rank(const pd_comm* comm);
int pd_comm_world(const pd_comm* comm);
void pd_comm_free(pd_comm* comm);
const char* pd_last_nccl_error(void); /* thread-local message of the last PD_ENCCL */

/* ---- Roofline denominators measured on the box (bench.py, not the hot path). */
/* FP32 FFMA throughput in lane-ops/s (one FFMA = one lane-op): best of `reps` launches of independent FFMA
 * chains at full occupancy.  Errors: PD_EINVAL, PD_ECUDA. */
pd_status pd_measure_fp32_peak(int device, int reps, double* lane_ops_per_s);
/* L2 read bandwidth in bytes/s: `bytes` (>= 1 MiB; <= 64 MiB to stay L2-resident) swept 32 times per launch
 * with L1-bypassing 16-byte loads after a warming launch; best of `reps`.  Errors: PD_EINVAL, PD_ECUDA. */
pd_status pd_measure_l2_peak(int device, int64_t bytes, int reps, double* bytes_per_s);

/* Test hook for the path's own LSD radix sort: stable sort of n (key < 2^64,
 * value) pairs, all DEVICE pointers on the current device, enqueued on `stream` and synchronized.
 * keys_in/vals_in are not modified; temp storage is allocated internally. */
pd_status pd_sort_pairs_u64(const uint64_t* keys_in, const uint32_t* vals_in, int64_t n, uint64_t* keys_out,
                            uint32_t* vals_out, void* stream);

/* Release the per-device build workspace (temporaries are cached across builds in persistent device
 * chunks, DESIGN.md §6 "Memory"), the internal high-priority stream the capacity tiers 2-3 run on, and
 * the cached pinned host buffers of freed PD_OUT_HOST results.
 * Waits for a build in flight on `device`; results stay valid.  Errors: PD_EINVAL (device out of
 * range), PD_ECUDA. */
pd_status pd_trim(int device);

const char* pd_strerror(pd_status s);
int64_t pd_error_index(void);      /* thread-local: offending point of the last NONFINITE/OUTSIDE */
const char* pd_last_cuda_error(void); /* thread-local message of the last PD_ECUDA */
int pd_abi_version(void);
/* Number of kernels launched by the last pd_build/pd_assemble on this thread (for bench.py). */
int64_t pd_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PD_H */
