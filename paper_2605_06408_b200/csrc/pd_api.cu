// pd_api.cu -- the C ABI (include/pd.h): argument checking, device memory, the pipeline
// pack -> Morton -> sort -> gather -> LBVH -> refit -> cell kernel (3 capacity tiers) -> CSR,
// result ownership and accessors.  See include/pd.h for the contract.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/pd.h"
#include "pd_bvh.cuh"
#include "pd_comm.cuh"
#include "pd_internal.cuh"

struct pd_result {
    int64_t n = 0;
    int64_t nnz = 0;
    int on_host = 0;
    int device = 0;
    cudaStream_t stream = nullptr;  // stream the result was built on (frees are ordered on it)
    int64_t* offsets = nullptr;
    int32_t* nbr = nullptr;
    float* area = nullptr;
    int64_t ntets = 0;
    int32_t* tets = nullptr;  // PD_TETS: 4 * ntets
    float* vol = nullptr;
    float* surf = nullptr;
    uint8_t* flags = nullptr;
    // sharding
    int64_t slice_begin = 0, slice_end = 0, slice_nnz = 0;
    int32_t* perm = nullptr;  // device, Morton position -> original id
    int32_t* cnt = nullptr;   // device, per original id
    int32_t* cost = nullptr;  // device, per original id (PD_COST)
    pd_stats stats;
    std::vector<void*> dev;
    std::vector<void*> host;
};

namespace {

thread_local int64_t g_err_index = -1;
thread_local char g_cuda_msg[256] = "";
thread_local int64_t g_launches = 0;

struct Fail {
    pd_status s;
};

void ck(cudaError_t e) {
    if (e != cudaSuccess) {
        snprintf(g_cuda_msg, sizeof(g_cuda_msg), "%s", cudaGetErrorString(e));
        if (e == cudaErrorMemoryAllocation) throw Fail{PD_ENOMEM};
        throw Fail{PD_ECUDA};
    }
}

// CUDA event destroyed with its scope (error paths included).
struct Ev {
    cudaEvent_t e = nullptr;
    Ev() = default;
    Ev(const Ev&) = delete;
    Ev& operator=(const Ev&) = delete;
    ~Ev() {
        if (e) cudaEventDestroy(e);
    }
    void create() { ck(cudaEventCreate(&e)); }
    operator cudaEvent_t() const { return e; }
};

// Stream-ordered allocations, released at scope end (cudaFreeAsync) unless handed to a result.
struct Arena {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Arena(cudaStream_t s) : st(s) {}
    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        size_t bytes = std::max<size_t>(count * sizeof(T), 16);
        ck(cudaMallocAsync(&p, bytes, st));
        ptrs.push_back(p);
        return (T*)p;
    }
    void release(void* p) {
        auto it = std::find(ptrs.begin(), ptrs.end(), p);
        if (it != ptrs.end()) ptrs.erase(it);
    }
    ~Arena() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

// Per-device cached workspace for a build's temporaries: a bump allocator over persistent chunks.
// Builds of the same problem request the same sequence of sizes, so after the first build every
// temporary lands in memory that is already mapped (growing the stream-ordered pool mid-build by
// hundreds of MB cost up to ~0.4 s per build).  One build per device at a time holds the lock.
struct Workspace {
    std::mutex mu;
    std::vector<std::pair<char*, size_t>> chunks;
    size_t ci = 0, off = 0;
    void reset() { ci = 0; off = 0; }
    template <class T>
    T* alloc(size_t count) {
        size_t bytes = (std::max<size_t>(count * sizeof(T), 16) + 255) & ~(size_t)255;
        while (ci < chunks.size()) {
            if (off + bytes <= chunks[ci].second) {
                char* p = chunks[ci].first + off;
                off += bytes;
                return (T*)p;
            }
            ++ci;
            off = 0;
        }
        size_t sz = std::max<size_t>(bytes, size_t(256) << 20);
        void* p = nullptr;
        ck(cudaMalloc(&p, sz));
        chunks.emplace_back((char*)p, sz);
        ci = chunks.size() - 1;
        off = bytes;
        return (T*)p;
    }
};
Workspace& workspace(int device) {
    static Workspace ws[64];
    return ws[device & 63];
}

void setup_pool(int device) {
    static bool done[64] = {false};
    if (device >= 0 && device < 64 && !done[device]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        done[device] = true;
    }
}

// A high-priority internal stream per device: the capacity tiers 2-3 run on it concurrently with the tier-1
// finalize on the caller's stream (PD_OVERLAP); pending CTAs of the higher priority are dispatched first.
cudaStream_t& hi_stream_slot(int device) {
    static cudaStream_t hs[64] = {};
    return hs[device & 63];
}
cudaStream_t hi_stream(int device) {
    cudaStream_t& h = hi_stream_slot(device);
    if (!h) {
        int least = 0, greatest = 0;
        ck(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        ck(cudaStreamCreateWithPriority(&h, cudaStreamNonBlocking, greatest));
    }
    return h;
}

int num_sms(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v > 0 ? v : 1;
}

template <class T>
T* to_result(pd_result* r, Arena& A, T* p) {
    A.release(p);
    r->dev.push_back(p);
    return p;
}

// Pinned host buffers for PD_OUT_HOST results are recycled across builds (cudaMallocHost of a
// ~1 GB CSR costs far more than the copy itself).  Buffers are keyed by capacity.
struct PinnedCache {
    std::mutex mu;
    std::multimap<size_t, void*> free_;  // capacity -> buffer
    std::map<void*, size_t> cap_;
    size_t cached = 0;
    static constexpr size_t kMaxCached = size_t(16) << 30;
    void* get(size_t bytes) {
        {
            std::lock_guard<std::mutex> g(mu);
            auto it = free_.lower_bound(bytes);
            if (it != free_.end() && it->first <= 2 * bytes + (1 << 20)) {
                void* p = it->second;
                cached -= it->first;
                free_.erase(it);
                return p;
            }
        }
        void* p = nullptr;
        size_t cap = std::max<size_t>(bytes, 64);
        ck(cudaMallocHost(&p, cap));
        std::lock_guard<std::mutex> g(mu);
        cap_[p] = cap;
        return p;
    }
    void put(void* p) {
        std::lock_guard<std::mutex> g(mu);
        size_t cap = cap_[p];
        if (cached + cap > kMaxCached) {
            cap_.erase(p);
            cudaFreeHost(p);
            return;
        }
        free_.emplace(cap, p);
        cached += cap;
    }
    void trim() {  // release every cached (free) buffer
        std::lock_guard<std::mutex> g(mu);
        for (auto& kv : free_) {
            cap_.erase(kv.second);
            cudaFreeHost(kv.second);
        }
        free_.clear();
        cached = 0;
    }
};
PinnedCache& pinned() {
    static PinnedCache c;
    return c;
}

template <class T>
T* host_copy(pd_result* r, const T* dptr, size_t count, cudaStream_t st) {
    T* h = (T*)pinned().get(std::max<size_t>(count * sizeof(T), 16));
    r->host.push_back(h);
    if (count) ck(cudaMemcpyAsync(h, dptr, count * sizeof(T), cudaMemcpyDeviceToHost, st));
    return h;
}

void free_result(pd_result* r) {
    if (!r) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(r->device);
    for (void* p : r->dev) cudaFreeAsync(p, r->stream);
    if (!r->host.empty()) cudaStreamSynchronize(r->stream);
    for (void* p : r->host) pinned().put(p);
    cudaSetDevice(cur);
    delete r;
}

void finish_outputs(pd_result* r, Arena& A, unsigned flags, cudaStream_t st) {
    if (flags & PD_OUT_HOST) {
        r->offsets = host_copy(r, r->offsets, (size_t)r->n + 1, st);
        r->nbr = host_copy(r, r->nbr, (size_t)r->nnz, st);
        r->area = host_copy(r, r->area, (size_t)r->nnz, st);
        r->vol = host_copy(r, r->vol, (size_t)r->n, st);
        r->surf = host_copy(r, r->surf, (size_t)r->n, st);
        r->flags = host_copy(r, r->flags, (size_t)r->n, st);
        if (r->tets) r->tets = host_copy(r, r->tets, (size_t)r->ntets * 4, st);
        r->on_host = 1;
    }
    (void)A;
}

void nck(ncclResult_t r, const char* where) {
    if (r != ncclSuccess) {
        pd::nccl_set_error(where, r);
        throw Fail{PD_ENCCL};
    }
}

// Header rank 0 broadcasts before the arrays of a sharded build (pd_build_sharded).
struct ShardHeader {
    int64_t status, err_index, n, n_wide;
    float box[6];
    int32_t has_box, pad;
};

// comm == nullptr: pd_build (whole diagram, or the opt.shard_rank slice without an exchange).
// comm != nullptr: pd_build_sharded -- rank 0 packs, validates and builds the LBVH, NCCL broadcasts the
// sorted sites, the permutation and the wide nodes; every rank builds its Morton slice of the cells; the
// slices are exchanged (grouped NCCL broadcasts) and every rank assembles the full CSR.
pd_status build_impl(const float* points, const float* weights, int64_t n, const pd_box* box, const pd_options* optp,
                     pd_result** out, pd_comm* comm = nullptr) {
    pd_options opt;
    memset(&opt, 0, sizeof(opt));
    if (optp) opt = *optp;
    if (!out) return PD_EINVAL;
    *out = nullptr;
    const bool root_builds = !comm || comm->rank == 0;  // this rank packs the input and builds the LBVH
    if (comm) {
        opt.device = comm->device;
        opt.shard_world = comm->world;
        opt.shard_rank = comm->rank;
        if (opt.flags & PD_TETS) return PD_EINVAL;
    }
    if (n == 0) return PD_EEMPTY;
    if (n < 0 || n > PD_MAX_SITES || (root_builds && !points)) return PD_EINVAL;
    if (box)
        for (int k = 0; k < 3; ++k)
            if (!(box->lo[k] < box->hi[k]) || !std::isfinite(box->lo[k]) || !std::isfinite(box->hi[k])) return PD_EINVAL;
    int leaf = opt.leaf_size > 0 ? opt.leaf_size : 32;
    if (leaf > 32) return PD_EINVAL;
    int world = opt.shard_world > 1 ? opt.shard_world : 1;
    int rank = world > 1 ? opt.shard_rank : 0;
    if (rank < 0 || rank >= world) return PD_EINVAL;
    if ((opt.flags & PD_TETS) && world > 1) return PD_EINVAL;
    g_launches = 0;
    int launches = 0;
    ck(cudaSetDevice(opt.device));
    setup_pool(opt.device);
    cudaStream_t st = (cudaStream_t)opt.stream;
    Arena A(st);  // result-owned buffers (stream-ordered pool)
    Workspace& W = workspace(opt.device);  // temporaries
    std::unique_lock<std::mutex> wlock(W.mu);
    W.reset();
    pd_result* r = new pd_result();
    memset(&r->stats, 0, sizeof(r->stats));
    r->n = n;
    r->device = opt.device;
    r->stream = (cudaStream_t)opt.stream;
    try {
        Ev ev[5];
        for (auto& e : ev) e.create();
        ck(cudaEventRecord(ev[0], st));
        float4* sorted = nullptr;
        int32_t* perm = nullptr;
        int* bvh_counters = nullptr;  // collapse counters ([1] = capacity overflow), checked after the cells
        pd::Bvh bvh;
        float hbox[6] = {0, 0, 0, 0, 0, 0};
        int64_t n_wide = 0;
        pd_status root_status = PD_OK;
        int64_t root_err = -1;
        if (root_builds) {
        // ---- inputs
        const float* dpts = points;
        const float* dw = weights;
        if (!(opt.flags & PD_IN_DEVICE)) {
            float* p = W.alloc<float>((size_t)n * 3);
            ck(cudaMemcpyAsync(p, points, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, st));
            dpts = p;
            if (weights) {
                float* q = W.alloc<float>((size_t)n);
                ck(cudaMemcpyAsync(q, weights, sizeof(float) * n, cudaMemcpyHostToDevice, st));
                dw = q;
            }
        }
        // ---- a1/a2 pack + validate + box
        float4* sites = W.alloc<float4>(n);
        float* box_dev = W.alloc<float>(8);
        unsigned long long* errs = W.alloc<unsigned long long>(2);
        int* aabb = W.alloc<int>(8);
        ck(cudaMemsetAsync(errs, 0xff, 2 * sizeof(unsigned long long), st));
        {
            int init[6] = {0x7f800000, 0x7f800000, 0x7f800000, (int)(0xff800000u ^ 0x7fffffffu),
                           (int)(0xff800000u ^ 0x7fffffffu), (int)(0xff800000u ^ 0x7fffffffu)};
            ck(cudaMemcpyAsync(aabb, init, sizeof(init), cudaMemcpyHostToDevice, st));
        }
        if (box) {
            float b[6] = {box->lo[0], box->lo[1], box->lo[2], box->hi[0], box->hi[1], box->hi[2]};
            ck(cudaMemcpyAsync(box_dev, b, sizeof(b), cudaMemcpyHostToDevice, st));
        }
        ck(pd::bvh_pack(dpts, dw, n, box, sites, box_dev, errs, aabb, st, &launches));
        unsigned long long herr[2];
        ck(cudaMemcpyAsync(herr, errs, sizeof(herr), cudaMemcpyDeviceToHost, st));
        ck(cudaMemcpyAsync(hbox, box_dev, sizeof(hbox), cudaMemcpyDeviceToHost, st));
        ck(cudaStreamSynchronize(st));
        if (herr[0] != ~0ull) { root_err = (int64_t)herr[0]; root_status = PD_ENONFINITE; }
        else if (herr[1] != ~0ull) { root_err = (int64_t)herr[1]; root_status = PD_EOUTSIDE; }
        if (root_status != PD_OK && !comm) { g_err_index = root_err; throw Fail{root_status}; }
        if (root_status == PD_OK) {
        // a degenerate tight box (all points on a plane) is widened so cells stay 3-D
        if (!box) {
            bool changed = false;
            for (int k = 0; k < 3; ++k)
                if (!(hbox[k] < hbox[3 + k])) {
                    hbox[k] = std::nextafter(hbox[k], -INFINITY);
                    hbox[3 + k] = std::nextafter(hbox[3 + k], INFINITY);
                    changed = true;
                }
            if (changed) ck(cudaMemcpyAsync(box_dev, hbox, sizeof(hbox), cudaMemcpyHostToDevice, st));
        }
        // ---- a3-a5 Morton, sort, gather
        uint64_t* keys = W.alloc<uint64_t>(n);
        uint64_t* keys_s = W.alloc<uint64_t>(n);
        uint32_t* vals = W.alloc<uint32_t>(n);
        uint32_t* vals_s = W.alloc<uint32_t>(n);
        ck(pd::bvh_morton(sites, n, box_dev, keys, vals, st, &launches));
        size_t tb = 0;
        ck(pd::sort_pairs(keys, keys_s, vals, vals_s, n, nullptr, &tb, st, nullptr));
        void* tmp = W.alloc<unsigned char>(tb);
        ck(pd::sort_pairs(keys, keys_s, vals, vals_s, n, tmp, &tb, st, &launches));
        sorted = W.alloc<float4>(n);
        perm = A.alloc<int32_t>(n);
        ck(pd::bvh_gather(sites, vals_s, n, sorted, perm, st, &launches));
        // ---- a6/a7 LBVH + refit
        pd::BvhScratch sc;
        int ni = (int)std::max<int64_t>(n - 1, 1);
        sc.child = W.alloc<int2>(ni);
        sc.range = W.alloc<int2>(ni);
        sc.parent_int = W.alloc<int>(ni);
        sc.parent_leaf = W.alloc<int>(n);
        sc.visit = W.alloc<int>(ni);
        sc.blo = W.alloc<float4>(ni);
        sc.bhi = W.alloc<float4>(ni);
        sc.max_wide = (int)std::min<int64_t>(2 * n / leaf + 2, ni + 1);
        bvh.nodes = W.alloc<pd::WideNode>(sc.max_wide);
        sc.tasks[0] = W.alloc<int2>(sc.max_wide);
        sc.tasks[1] = W.alloc<int2>(sc.max_wide);
        sc.counters = W.alloc<int>(pd::kCollapseCounters);
        bvh.root = W.alloc<pd::NodeChild>(1);
        ck(pd::bvh_topology(keys_s, sorted, (int)n, leaf, sc, bvh, st, &launches));
        bvh_counters = sc.counters;
        if (comm && n > leaf) {  // the wide-node count sizes the broadcast
            int hc[2] = {0, 0};
            ck(cudaMemcpyAsync(hc, sc.counters, sizeof(hc), cudaMemcpyDeviceToHost, st));
            ck(cudaStreamSynchronize(st));
            if (hc[1]) throw Fail{PD_EINTERNAL};  // collapse capacity invariant violated
            n_wide = hc[0];
        }
        }  // root_status == PD_OK
        }  // root_builds
        if (comm) {
            // ---- broadcast the header (status first: every rank returns rank 0's input error), then the
            // LBVH: Morton-sorted sites, the permutation and the wide nodes + root record (NCCL over NVLink)
            const pd::NcclApi* nc = pd::nccl_api();
            if (!nc) throw Fail{PD_ENCCL};
            ShardHeader* dh = W.alloc<ShardHeader>(1);
            ShardHeader hh;
            memset(&hh, 0, sizeof(hh));
            if (root_builds) {
                hh.status = root_status; hh.err_index = root_err; hh.n = n; hh.n_wide = n_wide;
                for (int k = 0; k < 6; ++k) hh.box[k] = hbox[k];
                ck(cudaMemcpyAsync(dh, &hh, sizeof(hh), cudaMemcpyHostToDevice, st));
            }
            nck(nc->Broadcast(dh, dh, sizeof(hh), ncclUint8, 0, comm->comm, st), "ncclBroadcast(header)");
            ck(cudaMemcpyAsync(&hh, dh, sizeof(hh), cudaMemcpyDeviceToHost, st));
            ck(cudaStreamSynchronize(st));
            if (hh.status != PD_OK) { g_err_index = hh.err_index; throw Fail{(pd_status)hh.status}; }
            if (hh.n != n) throw Fail{PD_EINVAL};  // every rank must pass the same n
            n_wide = hh.n_wide;
            for (int k = 0; k < 6; ++k) hbox[k] = hh.box[k];
            if (!root_builds) {
                sorted = W.alloc<float4>(n);
                perm = A.alloc<int32_t>(n);
                bvh.nodes = W.alloc<pd::WideNode>(std::max<int64_t>(n_wide, 1));
                bvh.root = W.alloc<pd::NodeChild>(1);
            }
            nck(nc->GroupStart(), "ncclGroupStart");
            nck(nc->Broadcast(sorted, sorted, (size_t)n * 4, ncclFloat32, 0, comm->comm, st), "ncclBroadcast(sites)");
            nck(nc->Broadcast(perm, perm, (size_t)n, ncclInt32, 0, comm->comm, st), "ncclBroadcast(perm)");
            if (n_wide > 0)
                nck(nc->Broadcast(bvh.nodes, bvh.nodes, (size_t)n_wide * sizeof(pd::WideNode), ncclUint8, 0, comm->comm, st),
                    "ncclBroadcast(nodes)");
            nck(nc->Broadcast(bvh.root, bvh.root, sizeof(pd::NodeChild), ncclUint8, 0, comm->comm, st), "ncclBroadcast(root)");
            nck(nc->GroupEnd(), "ncclGroupEnd");
        }
        ck(cudaEventRecord(ev[1], st));
        // ---- cells
        int32_t* cnt = A.alloc<int32_t>(n);
        int64_t* aoff = W.alloc<int64_t>(n);
        float* vol = A.alloc<float>(n);
        float* surf = A.alloc<float>(n);
        uint8_t* flags = A.alloc<uint8_t>(n);
        int sms = num_sms(opt.device);
        const int spill_cap[3] = {2048, 8192, 32768};
        size_t spill_entries = 0;
        for (int t = 0; t < 3; ++t)
            spill_entries = std::max(spill_entries, (size_t)pd::cells_grid_warps(t, sms) * spill_cap[t]);
        pd::NodeChild* spill = W.alloc<pd::NodeChild>(spill_entries);
        void* gstate = W.alloc<unsigned char>(pd::cells_global_state_bytes(sms));
        const int exact_after = [] {
            const char* ev = getenv("PD_EXACT_AFTER");  // tuning knob (default 100: C3 -2% vs 200, C4 unchanged)
            return ev ? atoi(ev) : 100;
        }();
        // ---- slice of the Morton order owned by this rank: equal-count by default;
        // PD_BALANCE cuts equal estimated cost, from the tier-1 kernel's per-cell work counters on a
        // strided ~40k-cell sample (deterministic, so every rank computes the same cuts).  Measured on
        // C4 at world 8 (tools/shard_balance.py): equal-count max/mean 1.07, cost-balanced 1.16.
        // Sampled tier-1 work (deterministic per-cell counters nodes + sites + 8 x clips, PD_COST) of the listed
        // Morton positions, run in list mode with scratch outputs: the cost model of PD_BALANCE's cuts and of the
        // auto warm start.  Every rank of a sharded build runs it on the same broadcast sites, so all agree.
        auto sample_work = [&](const int32_t* spos, int32_t* scount, int64_t ns, unsigned flags, const int32_t* sknn,
                               int32_t* sgath) {
            int32_t* scost = W.alloc<int32_t>(n);
            unsigned long long* sctr = W.alloc<unsigned long long>(8);
            const int64_t scap = ns * 96 + 4096;
            int32_t* s_nbr = W.alloc<int32_t>(scap);
            float* s_area = W.alloc<float>(scap);
            int* s_ovf = W.alloc<int>(1);
            pd::Stats* s_stats = W.alloc<pd::Stats>(1);
            int32_t* s_next = W.alloc<int32_t>(ns);
            int32_t hc[4] = {(int32_t)ns, 0, 0, 0};
            ck(cudaMemcpyAsync(scount, hc, sizeof(hc), cudaMemcpyHostToDevice, st));
            ck(cudaMemsetAsync(sctr, 0, 8 * sizeof(unsigned long long), st));
            ck(cudaMemsetAsync(s_ovf, 0, sizeof(int), st));
            pd::CellParams Q;
            memset(&Q, 0, sizeof(Q));
            Q.sites = sorted;
            Q.perm = perm;
            Q.nodes = bvh.nodes;
            Q.root = bvh.root;
            for (int k = 0; k < 3; ++k) { Q.box_lo[k] = hbox[k]; Q.box_hi[k] = hbox[3 + k]; }
            Q.flags = (flags | PD_COST) & ~PD_STATS;
            Q.out.cnt = W.alloc<int32_t>(n); Q.out.aoff = W.alloc<int64_t>(n); Q.out.vol = W.alloc<float>(n);
            Q.out.surf = W.alloc<float>(n); Q.out.flags = W.alloc<uint8_t>(n);
            Q.out.arena_nbr = s_nbr; Q.out.arena_area = s_area; Q.out.arena_top = sctr + 4;
            Q.out.arena_cap = scap; Q.out.arena_overflow = s_ovf; Q.out.cost = scost;
            Q.stats = s_stats;
            Q.spill = spill;
            Q.gstate = gstate;
            Q.exact_after = exact_after;
            Q.prof_tier = -2;
            Q.coop_min_v = 128;
            Q.trace_cell = -1;
            Q.knn = sknn;
            Q.n_sites = n;
            Q.work_counter = sctr;
            Q.last_tier = 1;  // heavy sampled cells keep their (partial) cost instead of escalating
            Q.list = spos;
            Q.list_count = scount;
            Q.next_list = s_next;
            Q.next_count = scount + 1;
            Q.spill_cap = spill_cap[0];
            ck(pd::launch_cells(0, Q, st, sms, &launches));
            ck(pd::gather_sample_cost(perm, spos, ns, scost, sgath, st, &launches));
        };
        auto strided_sample = [&](int64_t target, int64_t& ns, int64_t& stride) {
            stride = std::max<int64_t>(1, n / target);
            ns = (n + stride - 1) / stride;
            std::vector<int32_t> hpos(ns);
            for (int64_t k = 0; k < ns; ++k) hpos[k] = (int32_t)(k * stride);
            int32_t* spos = W.alloc<int32_t>(ns);
            ck(cudaMemcpyAsync(spos, hpos.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, st));
            ck(cudaStreamSynchronize(st));  // hpos is a host temporary
            return spos;
        };
        // ---- auto warm start (pd.h PD_AUTO_WARM): measure the sampled tier-1 work with and without the KNN
        // pre-clip and keep it when it saves more than the KNN query costs
        double warm_gain = 0.0;
        int32_t* knn = nullptr;
        if ((opt.flags & PD_AUTO_WARM) && !(opt.flags & (PD_WARM_START | PD_WARM_ADAPTIVE | PD_NO_AUTO_WARM)) &&
            n >= 4096 && (weights || comm)) {
            int64_t ns = 0, stride = 1;
            const int32_t* spos = strided_sample(8192, ns, stride);
            int32_t* scount = W.alloc<int32_t>(4);
            knn = W.alloc<int32_t>((size_t)n * pd::KNN_K);
            ck(pd::knn_query(sorted, bvh.nodes, bvh.root, 0, (int)ns, 0, knn, sms, st, &launches, spos));
            int32_t* g0 = W.alloc<int32_t>(ns);
            int32_t* g1 = W.alloc<int32_t>(ns);
            sample_work(spos, scount, ns, opt.flags & ~(PD_WARM_START | PD_WARM_ADAPTIVE), nullptr, g0);
            sample_work(spos, scount, ns, opt.flags | PD_WARM_START, knn, g1);
            std::vector<int32_t> h0(ns), h1(ns);
            ck(cudaMemcpyAsync(h0.data(), g0, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, st));
            ck(cudaMemcpyAsync(h1.data(), g1, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, st));
            ck(cudaStreamSynchronize(st));
            double w0 = 0, w1 = 0;
            for (int64_t k = 0; k < ns; ++k) { w0 += h0[k]; w1 += h1[k]; }
            // the KNN query of a site costs about kKnnWork work units, and the warm-start kernel a few % more per unit
            constexpr double kKnnWork = 60.0, kWarmOverhead = 1.10;
            warm_gain = w0 > 0 ? (w1 * kWarmOverhead + kKnnWork * (double)ns) / w0 : 1.0;
            if (warm_gain < 0.9) opt.flags |= PD_WARM_START;
        }
        std::vector<int64_t> cuts(world + 1);  // every rank's slice (the exchange needs them all)
        for (int q = 0; q <= world; ++q) cuts[q] = (n * q) / world;
        if (world > 1 && (opt.flags & PD_BALANCE) && n >= 4 * world) {
            int64_t ns = 0, stride = 1;
            const int32_t* spos = strided_sample(40000, ns, stride);
            int32_t* scount = W.alloc<int32_t>(4);
            int32_t* sgath = W.alloc<int32_t>(ns);
            sample_work(spos, scount, ns, opt.flags & ~(PD_WARM_START | PD_WARM_ADAPTIVE), nullptr, sgath);
            std::vector<int32_t> hcost(ns);
            ck(cudaMemcpyAsync(hcost.data(), sgath, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, st));
            ck(cudaStreamSynchronize(st));
            std::vector<double> cum(ns + 1, 0.0);
            for (int64_t k = 0; k < ns; ++k) cum[k + 1] = cum[k] + std::max<int32_t>(hcost[k], 1);
            auto cut = [&](int q) -> int64_t {  // Morton position where cumulative cost reaches q/world
                if (q <= 0) return 0;
                if (q >= world) return n;
                const double target = cum[ns] * q / world;
                int64_t k = std::lower_bound(cum.begin(), cum.end(), target) - cum.begin();
                return std::min<int64_t>(n, std::max<int64_t>(0, (k - 1) * stride));
            };
            for (int q = 0; q <= world; ++q) cuts[q] = cut(q);
        }
        const int64_t begin = cuts[rank], end = cuts[rank + 1];
        r->slice_begin = begin;
        r->slice_end = end;
        // ---- optional KNN warm start: K = 8 nearest sites of every site of the slice
        Ev kev[2];
        if (opt.flags & (PD_WARM_START | PD_WARM_ADAPTIVE)) {
            if (!knn) knn = W.alloc<int32_t>((size_t)n * pd::KNN_K);
            kev[0].create();
            kev[1].create();
            ck(cudaEventRecord(kev[0], st));
            const int adaptive = (opt.flags & PD_WARM_START) ? 0 : 1;
            ck(pd::knn_query(sorted, bvh.nodes, bvh.root, (int)begin, (int)end, adaptive, knn, sms, st, &launches));
            ck(cudaEventRecord(kev[1], st));
        }
        int32_t* lists = W.alloc<int32_t>(2 * (size_t)std::max<int64_t>(end - begin, 1));
        int32_t* lcost = W.alloc<int32_t>(2 * (size_t)std::max<int64_t>(end - begin, 1));
        unsigned long long* counters = W.alloc<unsigned long long>(8);
        int32_t* list_counts = W.alloc<int32_t>(4);
        int* aovf = W.alloc<int>(1);
        pd::Stats* dstats = W.alloc<pd::Stats>(1);
        int32_t* cost = (opt.flags & PD_COST) ? A.alloc<int32_t>(n) : nullptr;
        if (cost) ck(cudaMemsetAsync(cost, 0, sizeof(int32_t) * n, st));
        int64_t cap = std::max<int64_t>((end - begin) * 18, 1 << 16);
        int32_t* anbr = nullptr;
        int32_t* nbr = nullptr;  // CSR outputs: allocated with the arena (same capacity) so the CSR
        float* area = nullptr;   // phase never grows the memory pool mid-build
        float* aarea = nullptr;
        Ev tev[4];
        for (auto& e : tev) e.create();
        // dual tetrahedra (PD_TETS): ~6.8 per site for Poisson-Voronoi input, each listed once
        const bool want_tets = (opt.flags & PD_TETS) != 0;
        int32_t* tcnt = want_tets ? W.alloc<int32_t>(n) : nullptr;
        int64_t* taoff = want_tets ? W.alloc<int64_t>(n) : nullptr;
        int* tovf = want_tets ? W.alloc<int>(1) : nullptr;
        int4* tarena = nullptr;
        int64_t tcap = std::max<int64_t>((end - begin) * 8, 4096);
        // deferred tier-1 finalize (pd_cells.cu finalize_kernel): per-cell topology records, ~60 words per
        // cell on average (2 + planes + vertices); a cell that does not fit is finalized in the cell kernel
        const bool defer = true;  // tier 1 keeps no FP64 vertices: its finalize always runs in finalize_kernel
        uint32_t* rec_index = defer ? W.alloc<uint32_t>((size_t)std::max<int64_t>(n, 1)) : nullptr;
        int64_t rec_cap = std::min<int64_t>(std::max<int64_t>((end - begin) * 80, 1 << 16), 0xfffffff0LL);
        if (getenv("PD_REC_CAP")) rec_cap = std::max<int64_t>(atoll(getenv("PD_REC_CAP")), 16);  // test knob
        uint32_t* rec_arena = defer ? W.alloc<uint32_t>((size_t)rec_cap) : nullptr;
        for (int attempt = 0; attempt < 3; ++attempt) {
            anbr = W.alloc<int32_t>(cap);
            if (want_tets) {
                tarena = W.alloc<int4>(tcap);
                ck(cudaMemsetAsync(tovf, 0, sizeof(int), st));
            }
            nbr = A.alloc<int32_t>(cap);
            area = A.alloc<float>(cap);
            aarea = W.alloc<float>(cap);
            ck(cudaMemsetAsync(counters, 0, 8 * sizeof(unsigned long long), st));
            ck(cudaMemsetAsync(list_counts, 0, 4 * sizeof(int32_t), st));
            ck(cudaMemsetAsync(aovf, 0, sizeof(int), st));
            ck(cudaMemsetAsync(dstats, 0, sizeof(pd::Stats), st));
            if (world > 1) {
                ck(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * n, st));
                ck(pd::fill_flags(flags, n, PD_CELL_NOT_OWNED, st, &launches));
                ck(cudaMemsetAsync(vol, 0, sizeof(float) * n, st));
                ck(cudaMemsetAsync(surf, 0, sizeof(float) * n, st));
            }
            pd::CellParams P;
            memset(&P, 0, sizeof(P));
            P.sites = sorted;
            P.perm = perm;
            P.nodes = bvh.nodes;
            P.root = bvh.root;
            for (int k = 0; k < 3; ++k) { P.box_lo[k] = hbox[k]; P.box_hi[k] = hbox[3 + k]; }
            P.flags = opt.flags;
            if (defer && end > begin) {
                ck(cudaMemsetAsync(rec_index + begin, 0xff, sizeof(uint32_t) * (size_t)(end - begin), st));
                P.rec_index = rec_index;
                P.rec_arena = rec_arena;
                P.rec_top = counters + 6;
                P.rec_cap = rec_cap;
            }
            if (opt.flags & PD_WARM_ADAPTIVE) P.flags = (P.flags & ~PD_WARM_ADAPTIVE) | PD_WARM_START;
            P.out.cnt = cnt;
            P.out.aoff = aoff;
            P.out.vol = vol;
            P.out.surf = surf;
            P.out.flags = flags;
            P.out.arena_nbr = anbr;
            P.out.arena_area = aarea;
            P.out.arena_top = counters + 4;
            P.out.arena_cap = cap;
            P.out.arena_overflow = aovf;
            P.out.cost = cost;
            if (want_tets) {
                P.out.tcnt = tcnt;
                P.out.taoff = taoff;
                P.out.tarena = tarena;
                P.out.ttop = counters + 5;
                P.out.tcap = tcap;
                P.out.tovf = tovf;
            }
            P.stats = dstats;
            P.spill = spill;
            P.gstate = gstate;
            P.exact_after = exact_after;
            P.prof_tier = getenv("PD_PROF_TIER") ? atoi(getenv("PD_PROF_TIER")) : -1;
            P.knn = knn;
            P.n_sites = n;
            P.start_tier = getenv("PD_START_TIER") ? atoi(getenv("PD_START_TIER")) : 0;
            P.coop_min_v = getenv("PD_COOP_MIN_V") ? atoi(getenv("PD_COOP_MIN_V")) : 128;
            P.trace_cell = getenv("PD_TRACE_CELL") ? atoi(getenv("PD_TRACE_CELL")) : -1;
            int64_t L = end - begin;
            // The tier-1 finalize (non-persistent grid of 16 cells per warp, caller's stream) runs concurrently with
            // the higher tiers (internal high-priority stream): they read and write disjoint cells' outputs, and
            // every shared counter (row arena, stats) is an atomic.  Measured C4 358 -> 353 ms, C5 595 -> 582 ms,
            // C3 159.5 -> 161 ms.  PD_OVERLAP=0: serial (persistent finalize after tier 1); N > 1: N cells per warp.
            const int overlap = getenv("PD_OVERLAP") ? atoi(getenv("PD_OVERLAP")) : 1;
            cudaStream_t sh = overlap ? hi_stream(opt.device) : st;
            Ev ov[2];
            pd::CellParams P0;
            for (int tier = 0; tier < 3; ++tier) {
                cudaStream_t ts = tier == 0 ? st : sh;
                if (tier == 1 && overlap) {
                    ov[0].create();
                    ck(cudaEventRecord(ov[0], st));
                    ck(cudaStreamWaitEvent(sh, ov[0], 0));
                }
                P.work_counter = counters + tier;
                P.last_tier = tier == 2;
                if (tier == 0) {
                    P.begin = begin;
                    P.count = L;
                    P.list = nullptr;
                    P.list_count = nullptr;
                } else {
                    P.list = lists + (size_t)((tier - 1) & 1) * std::max<int64_t>(L, 1);
                    P.list_count = list_counts + (tier - 1);
                }
                P.next_list = lists + (size_t)(tier & 1) * std::max<int64_t>(L, 1);
                P.next_cost = lcost + (size_t)(tier & 1) * std::max<int64_t>(L, 1);
                P.next_count = list_counts + tier;
                P.spill_cap = spill_cap[tier];
                if (tier >= 1) {
                    // Longest first: a short list of heavy cells (C5's top tier: ~250 cells, the largest
                    // alone ~0.45 s) is started in descending order of the work they had done when they
                    // outgrew the previous tier, so the heaviest never queue behind others.  Sorted on
                    // the device (no host round trip between the tiers).
                    ck(pd::sort_list_by_cost(const_cast<int32_t*>(P.list),
                                             lcost + (size_t)((tier - 1) & 1) * std::max<int64_t>(L, 1),
                                             P.list_count, ts, &launches));
                }
                ck(cudaEventRecord(tev[tier], ts));
                ck(pd::launch_cells(tier, P, ts, sms, &launches, !overlap));
                if (tier == 0) P0 = P;
            }
            if (overlap) {
                ck(pd::launch_finalize(P0, st, sms, overlap > 1 ? overlap : 16, &launches));
                ov[1].create();
                ck(cudaEventRecord(ov[1], sh));
                ck(cudaStreamWaitEvent(st, ov[1], 0));
            }
            ck(cudaEventRecord(tev[3], st));
            unsigned long long top = 0, ttop = 0;
            int ovf = 0, t_ovf = 0;
            ck(cudaMemcpyAsync(&top, counters + 4, sizeof(top), cudaMemcpyDeviceToHost, st));
            ck(cudaMemcpyAsync(&ovf, aovf, sizeof(ovf), cudaMemcpyDeviceToHost, st));
            int collapse_ovf = 0;
            if (bvh_counters) ck(cudaMemcpyAsync(&collapse_ovf, bvh_counters + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
            if (want_tets) {
                ck(cudaMemcpyAsync(&ttop, counters + 5, sizeof(ttop), cudaMemcpyDeviceToHost, st));
                ck(cudaMemcpyAsync(&t_ovf, tovf, sizeof(t_ovf), cudaMemcpyDeviceToHost, st));
            }
            ck(cudaStreamSynchronize(st));
            if (collapse_ovf) throw Fail{PD_EINTERNAL};  // LBVH collapse capacity invariant violated (pd_bvh.cu)
            if (!ovf && !t_ovf) break;
            if (attempt == 2) throw Fail{PD_EINTERNAL};
            if (ovf) cap = (int64_t)(top * 1.1) + 1024;  // rerun with an arena large enough
            if (t_ovf) tcap = (int64_t)(ttop * 1.1) + 1024;
        }
        ck(cudaEventRecord(ev[2], st));
        int64_t nnz = 0;
        int64_t* offsets = nullptr;
        if (!comm) {
        // ---- a13 CSR
        offsets = A.alloc<int64_t>((size_t)n + 1);
        size_t sb = 0;
        ck(pd::scan_counts(cnt, offsets, n, nullptr, &sb, st, nullptr));
        void* stmp = W.alloc<unsigned char>(sb);
        ck(pd::scan_counts(cnt, offsets, n, stmp, &sb, st, &launches));
        ck(cudaMemcpyAsync(&nnz, offsets + n, sizeof(nnz), cudaMemcpyDeviceToHost, st));
        ck(cudaStreamSynchronize(st));
        if (nnz > cap) throw Fail{PD_EINTERNAL};
        ck(pd::csr_gather(cnt, aoff, offsets, anbr, aarea, n, nbr, area, st, &launches));
        if (want_tets) {  // dual tetrahedra rows in original-id order (same scan + gather as the CSR)
            int64_t* toff = W.alloc<int64_t>((size_t)n + 1);
            size_t tb2 = 0;
            ck(pd::scan_counts(tcnt, toff, n, nullptr, &tb2, st, nullptr));
            void* ttmp = W.alloc<unsigned char>(tb2);
            ck(pd::scan_counts(tcnt, toff, n, ttmp, &tb2, st, &launches));
            int64_t nt = 0;
            ck(cudaMemcpyAsync(&nt, toff + n, sizeof(nt), cudaMemcpyDeviceToHost, st));
            ck(cudaStreamSynchronize(st));
            int4* tt = A.alloc<int4>((size_t)std::max<int64_t>(nt, 1));
            ck(pd::tet_gather(tcnt, taoff, toff, tarena, n, tt, st, &launches));
            r->ntets = nt;
            r->tets = (int32_t*)to_result(r, A, tt);
        }
        } else {
            // ---- exchange: this rank's slice in Morton order goes straight into
            // the full Morton-ordered arrays at its offset; the row counts are all-gathered; every block is
            // then broadcast by its owner (grouped NCCL broadcasts = an all-gather of variable-size blocks);
            // every rank assembles the full original-order CSR.
            const pd::NcclApi* nc = pd::nccl_api();
            const int64_t len = end - begin;
            int32_t* cnt_m = W.alloc<int32_t>(n);
            float* vol_m = W.alloc<float>(n);
            float* surf_m = W.alloc<float>(n);
            uint8_t* flags_m = W.alloc<uint8_t>(n);
            int64_t* moff = W.alloc<int64_t>((size_t)len + 1);
            ck(pd::slice_export_meta(perm, begin, len, cnt, vol, surf, flags, cnt_m + begin, vol_m + begin,
                                     surf_m + begin, flags_m + begin, st, &launches));
            size_t sb = 0;
            ck(pd::scan_counts(cnt_m + begin, moff, len, nullptr, &sb, st, nullptr));
            ck(pd::scan_counts(cnt_m + begin, moff, len, W.alloc<unsigned char>(sb), &sb, st, &launches));
            int64_t* rows_all = W.alloc<int64_t>(world);
            nck(nc->AllGather(moff + len, rows_all, 1, ncclInt64, comm->comm, st), "ncclAllGather(rows)");
            std::vector<int64_t> hrows(world), roff(world + 1, 0);
            ck(cudaMemcpyAsync(hrows.data(), rows_all, sizeof(int64_t) * world, cudaMemcpyDeviceToHost, st));
            ck(cudaStreamSynchronize(st));
            for (int q = 0; q < world; ++q) roff[q + 1] = roff[q] + hrows[q];
            const int64_t total = roff[world];
            int32_t* rows_nbr = W.alloc<int32_t>((size_t)std::max<int64_t>(total, 1));
            float* rows_area = W.alloc<float>((size_t)std::max<int64_t>(total, 1));
            ck(pd::slice_export_rows(perm, begin, len, cnt_m + begin, moff, aoff, anbr, aarea, rows_nbr + roff[rank],
                                     rows_area + roff[rank], st, &launches));
            nck(nc->GroupStart(), "ncclGroupStart");
            for (int q = 0; q < world; ++q) {
                const int64_t b = cuts[q], lq = cuts[q + 1] - cuts[q];
                if (lq > 0) {
                    nck(nc->Broadcast(cnt_m + b, cnt_m + b, (size_t)lq, ncclInt32, q, comm->comm, st), "ncclBroadcast(cnt)");
                    nck(nc->Broadcast(vol_m + b, vol_m + b, (size_t)lq, ncclFloat32, q, comm->comm, st), "ncclBroadcast(vol)");
                    nck(nc->Broadcast(surf_m + b, surf_m + b, (size_t)lq, ncclFloat32, q, comm->comm, st), "ncclBroadcast(surf)");
                    nck(nc->Broadcast(flags_m + b, flags_m + b, (size_t)lq, ncclUint8, q, comm->comm, st), "ncclBroadcast(flags)");
                }
                if (hrows[q] > 0) {
                    nck(nc->Broadcast(rows_nbr + roff[q], rows_nbr + roff[q], (size_t)hrows[q], ncclInt32, q, comm->comm, st),
                        "ncclBroadcast(rows)");
                    nck(nc->Broadcast(rows_area + roff[q], rows_area + roff[q], (size_t)hrows[q], ncclFloat32, q, comm->comm,
                                      st), "ncclBroadcast(areas)");
                }
            }
            nck(nc->GroupEnd(), "ncclGroupEnd");
            // ---- assemble the full CSR in original order on every rank (same kernels as pd_assemble)
            int32_t* cnt_o = A.alloc<int32_t>(n);
            float* vol_o = A.alloc<float>(n);
            float* surf_o = A.alloc<float>(n);
            uint8_t* flags_o = A.alloc<uint8_t>(n);
            ck(pd::assemble_meta(perm, n, cnt_m, vol_m, surf_m, flags_m, cnt_o, vol_o, surf_o, flags_o, st, &launches));
            int64_t* moff_all = W.alloc<int64_t>((size_t)n + 1);
            offsets = A.alloc<int64_t>((size_t)n + 1);
            size_t sb1 = 0, sb2 = 0;
            ck(pd::scan_counts(cnt_m, moff_all, n, nullptr, &sb1, st, nullptr));
            ck(pd::scan_counts(cnt_m, moff_all, n, W.alloc<unsigned char>(sb1), &sb1, st, &launches));
            ck(pd::scan_counts(cnt_o, offsets, n, nullptr, &sb2, st, nullptr));
            ck(pd::scan_counts(cnt_o, offsets, n, W.alloc<unsigned char>(sb2), &sb2, st, &launches));
            nbr = A.alloc<int32_t>((size_t)std::max<int64_t>(total, 1));
            area = A.alloc<float>((size_t)std::max<int64_t>(total, 1));
            ck(pd::assemble_rows(perm, n, cnt_m, moff_all, offsets, rows_nbr, rows_area, nbr, area, st, &launches));
            nnz = total;
            cnt = cnt_o;
            vol = vol_o;
            surf = surf_o;
            flags = flags_o;
            r->slice_nnz = hrows[rank];
        }
        ck(cudaEventRecord(ev[3], st));
        r->nnz = nnz;
        r->offsets = to_result(r, A, offsets);
        r->nbr = to_result(r, A, nbr);
        r->area = to_result(r, A, area);
        r->vol = to_result(r, A, vol);
        r->surf = to_result(r, A, surf);
        r->flags = to_result(r, A, flags);
        r->perm = to_result(r, A, perm);
        r->cnt = to_result(r, A, cnt);
        if (cost) r->cost = to_result(r, A, cost);
        if (!comm) r->slice_nnz = nnz;
        finish_outputs(r, A, opt.flags, st);
        ck(cudaEventRecord(ev[4], st));
        pd::Stats hs;
        ck(cudaMemcpyAsync(&hs, dstats, sizeof(hs), cudaMemcpyDeviceToHost, st));
        ck(cudaStreamSynchronize(st));
        float t01, t12, t23, t04;
        cudaEventElapsedTime(&t01, ev[0], ev[1]);
        cudaEventElapsedTime(&t12, ev[1], ev[2]);
        cudaEventElapsedTime(&t23, ev[2], ev[3]);
        cudaEventElapsedTime(&t04, ev[0], ev[4]);
        pd_stats& s = r->stats;
        for (int k = 0; k < 3; ++k) {
            float tt = 0.f;
            cudaEventElapsedTime(&tt, tev[k], tev[k + 1]);
            s.ms_tier[k] = tt;
        }
        s.ms_knn = 0.0;
        if (kev[0].e) {
            float tk = 0.f;
            cudaEventElapsedTime(&tk, kev[0], kev[1]);
            s.ms_knn = tk;
        }
        s.cells = (int64_t)hs.cells;
        s.nodes_visited = (int64_t)hs.nodes;
        s.leaves_visited = (int64_t)hs.leaves;
        s.sites_tested = (int64_t)hs.sites;
        s.clip_tests = (int64_t)hs.clip_tests;
        s.clips = (int64_t)hs.clips;
        for (int k = 0; k < 3; ++k) s.tier_cells[k] = (int64_t)hs.tier[k];
        s.overflow_cells = (int64_t)hs.overflow;
        s.queue_spills = (int64_t)hs.spills;
        for (int k = 0; k < 10; ++k) s.warp_cycles[k] = (int64_t)hs.cyc[k];
        s.faces_dropped = (int64_t)hs.dropped;
        s.faces_near_degenerate = (int64_t)hs.small;
        s.degraded_cells = (int64_t)hs.degraded;
        s.warm_gain = warm_gain;
        s.warm_start = (opt.flags & (PD_WARM_START | PD_WARM_ADAPTIVE)) ? 1 : 0;
        s.nnz = nnz;
        s.ms_bvh = t01;
        s.ms_cells = t12;
        s.ms_csr = t23;
        s.ms_total = t04;
        g_launches = launches;
        *out = r;
        return PD_OK;
    } catch (const Fail& f) {
        cudaStreamSynchronize(st);  // kernels may still use workspace memory the next build reuses
        free_result(r);
        return f.s;
    } catch (...) {  // e.g. std::bad_alloc of a host vector: same cleanup, before the workspace lock goes
        cudaStreamSynchronize(st);
        free_result(r);
        return PD_EINTERNAL;
    }
}

}  // namespace

extern "C" {

pd_status pd_build(const float* points, const float* weights, int64_t n, const pd_box* box, const pd_options* opt,
                   pd_result** out) {
    try {
        return build_impl(points, weights, n, box, opt, out);
    } catch (...) {
        if (out) *out = nullptr;
        return PD_EINTERNAL;
    }
}

pd_status pd_build_sharded(pd_comm* comm, const float* points, const float* weights, int64_t n, const pd_box* box,
                           const pd_options* opt, pd_result** out) {
    if (!comm) {
        if (out) *out = nullptr;
        return PD_EINVAL;
    }
    try {
        return build_impl(points, weights, n, box, opt, out, comm);
    } catch (...) {
        if (out) *out = nullptr;
        return PD_EINTERNAL;
    }
}

int64_t pd_num_cells(const pd_result* r) { return r ? r->n : 0; }
int64_t pd_nnz(const pd_result* r) { return r ? r->nnz : 0; }
int pd_on_host(const pd_result* r) { return r ? r->on_host : 0; }
const int64_t* pd_offsets(const pd_result* r) { return r ? r->offsets : nullptr; }
const int32_t* pd_neighbors(const pd_result* r) { return r ? r->nbr : nullptr; }
const float* pd_face_areas(const pd_result* r) { return r ? r->area : nullptr; }
const float* pd_volumes(const pd_result* r) { return r ? r->vol : nullptr; }
const float* pd_surface(const pd_result* r) { return r ? r->surf : nullptr; }
const uint8_t* pd_cell_flags(const pd_result* r) { return r ? r->flags : nullptr; }
const int32_t* pd_cell_cost(const pd_result* r) { return r ? r->cost : nullptr; }
int64_t pd_num_tets(const pd_result* r) { return r ? r->ntets : 0; }
const int32_t* pd_tets(const pd_result* r) { return r ? r->tets : nullptr; }
pd_status pd_get_stats(const pd_result* r, pd_stats* s) {
    if (!r || !s) return PD_EINVAL;
    *s = r->stats;
    return PD_OK;
}
void pd_free(pd_result* r) { free_result(r); }
int64_t pd_slice_begin(const pd_result* r) { return r ? r->slice_begin : 0; }
int64_t pd_slice_end(const pd_result* r) { return r ? r->slice_end : 0; }
int64_t pd_slice_nnz(const pd_result* r) { return r ? r->slice_nnz : 0; }
const int32_t* pd_morton_perm(const pd_result* r) { return r ? r->perm : nullptr; }

pd_status pd_export_slice(const pd_result* r, int32_t* cnt_m, float* vol_m, float* surf_m, uint8_t* flags_m,
                          int32_t* rows_nbr, float* rows_area, int64_t* total, void* stream) {
    if (!r || r->on_host || !total) return PD_EINVAL;
    try {
        ck(cudaSetDevice(r->device));
        cudaStream_t st = (cudaStream_t)stream;
        Arena A(st);
        int launches = 0;
        int64_t len = r->slice_end - r->slice_begin;
        ck(pd::slice_export_meta(r->perm, r->slice_begin, len, r->cnt, r->vol, r->surf, r->flags, cnt_m, vol_m, surf_m,
                                 flags_m, st, &launches));
        int64_t* moff = A.alloc<int64_t>((size_t)len + 1);
        size_t sb = 0;
        ck(pd::scan_counts(cnt_m, moff, len, nullptr, &sb, st, nullptr));
        void* tmp = A.alloc<unsigned char>(sb);
        ck(pd::scan_counts(cnt_m, moff, len, tmp, &sb, st, &launches));
        ck(pd::slice_export_rows(r->perm, r->slice_begin, len, cnt_m, moff, r->offsets, r->nbr, r->area, rows_nbr,
                                 rows_area, st, &launches));
        ck(cudaMemcpyAsync(total, moff + len, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        ck(cudaStreamSynchronize(st));
        g_launches = launches;
        return PD_OK;
    } catch (const Fail& f) {
        return f.s;
    }
}

pd_status pd_assemble(const int32_t* perm, const int32_t* cnt_m, const float* vol_m, const float* surf_m,
                      const uint8_t* flags_m, const int32_t* rows_nbr, const float* rows_area, int64_t n, int64_t total,
                      const pd_options* optp, pd_result** out) {
    pd_options opt;
    memset(&opt, 0, sizeof(opt));
    if (optp) opt = *optp;
    if (!out) return PD_EINVAL;
    *out = nullptr;
    if (n <= 0 || total < 0 || !perm || !cnt_m || !vol_m || !surf_m || !flags_m) return PD_EINVAL;
    if (total > 0 && (!rows_nbr || !rows_area)) return PD_EINVAL;
    pd_result* r = new pd_result();
    memset(&r->stats, 0, sizeof(r->stats));
    r->n = n;
    r->device = opt.device;
    r->stream = (cudaStream_t)opt.stream;
    try {
        ck(cudaSetDevice(opt.device));
        setup_pool(opt.device);
        cudaStream_t st = (cudaStream_t)opt.stream;
        Arena A(st);
        int launches = 0;
        int32_t* cnt = A.alloc<int32_t>(n);
        float* vol = A.alloc<float>(n);
        float* surf = A.alloc<float>(n);
        uint8_t* flags = A.alloc<uint8_t>(n);
        ck(pd::assemble_meta(perm, n, cnt_m, vol_m, surf_m, flags_m, cnt, vol, surf, flags, st, &launches));
        int64_t* moff = A.alloc<int64_t>((size_t)n + 1);
        int64_t* offsets = A.alloc<int64_t>((size_t)n + 1);
        size_t sb = 0;
        ck(pd::scan_counts(cnt_m, moff, n, nullptr, &sb, st, nullptr));
        void* tmp = A.alloc<unsigned char>(sb);
        ck(pd::scan_counts(cnt_m, moff, n, tmp, &sb, st, &launches));
        int64_t rows_total = -1;  // the row lengths must add up to the caller's `total`
        ck(cudaMemcpyAsync(&rows_total, moff + n, sizeof(rows_total), cudaMemcpyDeviceToHost, st));
        ck(cudaStreamSynchronize(st));
        if (rows_total != total) throw Fail{PD_EINVAL};
        size_t sb2 = 0;
        ck(pd::scan_counts(cnt, offsets, n, nullptr, &sb2, st, nullptr));
        void* tmp2 = A.alloc<unsigned char>(sb2);
        ck(pd::scan_counts(cnt, offsets, n, tmp2, &sb2, st, &launches));
        int32_t* nbr = A.alloc<int32_t>((size_t)total);
        float* area = A.alloc<float>((size_t)total);
        ck(pd::assemble_rows(perm, n, cnt_m, moff, offsets, rows_nbr, rows_area, nbr, area, st, &launches));
        r->nnz = total;
        r->offsets = to_result(r, A, offsets);
        r->nbr = to_result(r, A, nbr);
        r->area = to_result(r, A, area);
        r->vol = to_result(r, A, vol);
        r->surf = to_result(r, A, surf);
        r->flags = to_result(r, A, flags);
        r->cnt = to_result(r, A, cnt);
        r->slice_begin = 0;
        r->slice_end = n;
        finish_outputs(r, A, opt.flags, st);
        ck(cudaStreamSynchronize(st));
        g_launches = launches;
        *out = r;
        return PD_OK;
    } catch (const Fail& f) {
        cudaStreamSynchronize((cudaStream_t)opt.stream);
        free_result(r);
        return f.s;
    } catch (...) {
        cudaStreamSynchronize((cudaStream_t)opt.stream);
        free_result(r);
        return PD_EINTERNAL;
    }
}

pd_status pd_trim(int device) {
    if (device < 0 || device >= 64) return PD_EINVAL;
    Workspace& W = workspace(device);
    std::lock_guard<std::mutex> g(W.mu);  // waits for a build in flight on this device
    int cur = 0;
    cudaGetDevice(&cur);
    if (cudaSetDevice(device) != cudaSuccess) return PD_ECUDA;
    cudaDeviceSynchronize();
    for (auto& c : W.chunks) cudaFree(c.first);
    W.chunks.clear();
    W.reset();
    if (cudaStream_t& h = hi_stream_slot(device)) {  // the internal stream of the higher tiers
        cudaStreamDestroy(h);
        h = nullptr;
    }
    pinned().trim();
    cudaSetDevice(cur);
    return PD_OK;
}

pd_status pd_sort_pairs_u64(const uint64_t* keys_in, const uint32_t* vals_in, int64_t n, uint64_t* keys_out,
                            uint32_t* vals_out, void* stream) {
    if (n < 0 || (n > 0 && (!keys_in || !vals_in || !keys_out || !vals_out))) return PD_EINVAL;
    if (n == 0) return PD_OK;
    try {
        cudaStream_t st = (cudaStream_t)stream;
        Arena A(st);
        size_t tb = 0;
        ck(pd::sort_pairs(keys_in, keys_out, vals_in, vals_out, n, nullptr, &tb, st, nullptr));
        void* tmp = A.alloc<unsigned char>(tb);
        int launches = 0;
        ck(pd::sort_pairs(keys_in, keys_out, vals_in, vals_out, n, tmp, &tb, st, &launches));
        ck(cudaStreamSynchronize(st));
        return PD_OK;
    } catch (const Fail& f) {
        return f.s;
    }
}

const char* pd_strerror(pd_status s) {
    switch (s) {
        case PD_OK: return "ok";
        case PD_EINVAL: return "invalid argument";
        case PD_EEMPTY: return "empty input (n == 0)";
        case PD_ENONFINITE: return "non-finite coordinate or weight";
        case PD_EOUTSIDE: return "point outside the box";
        case PD_ENOMEM: return "out of memory";
        case PD_ECUDA: return "CUDA error";
        case PD_ENCCL: return "NCCL error";
        case PD_EINTERNAL: return "internal error";
    }
    return "unknown status";
}
int64_t pd_error_index(void) { return g_err_index; }
const char* pd_last_cuda_error(void) { return g_cuda_msg; }
const char* pd_last_nccl_error(void) { return pd::nccl_last_error(); }
int pd_abi_version(void) { return PD_ABI_VERSION; }
int64_t pd_last_launch_count(void) { return g_launches; }

}  // extern "C"
