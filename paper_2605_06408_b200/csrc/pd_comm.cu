// pd_comm.cu -- NCCL communicator of the sharded build (include/pd.h: pd_comm_unique_id, pd_comm_init,
// pd_comm_free; the collectives themselves are issued by pd_build_sharded in pd_api.cu).
// PAPER.md:452 ("targets single-GPU execution") leaves multi-GPU open; the sharding rests on the n
// independent per-site clipping tasks of PAPER.md:151.
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "pd_comm.cuh"

namespace pd {

namespace {
NcclApi g_api;
bool g_ok = false;
std::once_flag g_once;
thread_local char g_msg[256] = "";

template <class F>
bool sym(void* h, const char* name, F& out) {
    out = reinterpret_cast<F>(dlsym(h, name));
    return out != nullptr;
}

void load() {
    // RTLD_NOLOAD first: reuse an NCCL already in the process (PyTorch's), else open the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_ok = sym(h, "ncclGetUniqueId", g_api.GetUniqueId) && sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
           sym(h, "ncclCommDestroy", g_api.CommDestroy) && sym(h, "ncclBroadcast", g_api.Broadcast) &&
           sym(h, "ncclAllGather", g_api.AllGather) && sym(h, "ncclGroupStart", g_api.GroupStart) &&
           sym(h, "ncclGroupEnd", g_api.GroupEnd) && sym(h, "ncclGetErrorString", g_api.GetErrorString) &&
           sym(h, "ncclGetVersion", g_api.GetVersion);
}
}  // namespace

const NcclApi* nccl_api() {
    std::call_once(g_once, load);
    return g_ok ? &g_api : nullptr;
}

void nccl_set_error(const char* where, ncclResult_t r) {
    const NcclApi* a = nccl_api();
    snprintf(g_msg, sizeof(g_msg), "%s: %s", where, a ? a->GetErrorString(r) : "libnccl.so.2 not found");
}

const char* nccl_last_error() { return g_msg; }

}  // namespace pd

extern "C" {

pd_status pd_comm_unique_id(unsigned char uid[128]) {
    if (!uid) return PD_EINVAL;
    const pd::NcclApi* a = pd::nccl_api();
    if (!a) {
        pd::nccl_set_error("dlopen", ncclSystemError);
        return PD_ENCCL;
    }
    ncclUniqueId id;
    ncclResult_t r = a->GetUniqueId(&id);
    if (r != ncclSuccess) {
        pd::nccl_set_error("ncclGetUniqueId", r);
        return PD_ENCCL;
    }
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(uid, &id, 128);
    return PD_OK;
}

pd_status pd_comm_init(const unsigned char uid[128], int rank, int world, int device, pd_comm** out) {
    if (!out) return PD_EINVAL;
    *out = nullptr;
    if (!uid || world < 1 || rank < 0 || rank >= world || device < 0) return PD_EINVAL;
    const pd::NcclApi* a = pd::nccl_api();
    if (!a) {
        pd::nccl_set_error("dlopen", ncclSystemError);
        return PD_ENCCL;
    }
    int cur = 0;
    cudaGetDevice(&cur);
    if (cudaSetDevice(device) != cudaSuccess) return PD_ECUDA;
    ncclUniqueId id;
    memcpy(&id, uid, 128);
    pd_comm* c = new pd_comm();
    c->rank = rank;
    c->world = world;
    c->device = device;
    ncclResult_t r = a->CommInitRank(&c->comm, world, id, rank);
    cudaSetDevice(cur);
    if (r != ncclSuccess) {
        pd::nccl_set_error("ncclCommInitRank", r);
        delete c;
        return PD_ENCCL;
    }
    *out = c;
    return PD_OK;
}

void pd_comm_free(pd_comm* c) {
    if (!c) return;
    const pd::NcclApi* a = pd::nccl_api();
    if (a && c->comm) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(c->device);
        a->CommDestroy(c->comm);
        cudaSetDevice(cur);
    }
    delete c;
}

int pd_comm_rank(const pd_comm* c) { return c ? c->rank : -1; }
int pd_comm_world(const pd_comm* c) { return c ? c->world : 0; }

}  // extern "C"
