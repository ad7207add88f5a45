// nccl_merge.cu -- the only collective of the sequence-sharded path (config 5):
// every rank's per-lane softmax partial (m, l, o[d]) is all-gathered over NCCL (NVLink /
// NVSwitch between the GPUs of one box) and merged by log-sum-exp (kvt_lse_merge), stream-
// ordered in one C-ABI call.  NCCL is bound at run time with dlopen("libnccl.so.2") -- the
// process's NCCL when one is already loaded (torch's) -- so the library keeps no link-time
// dependency besides the CUDA driver.  Communicators come from kvt_nccl_comm_init (the unique
// id travels through any out-of-band channel, e.g. torch.distributed over gloo).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather;
    });
    return api;
}

int nccl_status(ncclResult_t r) {
    if (r == ncclSuccess) return KVT_OK;
    NcclApi& api = nccl();
    return kvt_set_error_text(api.error_string ? api.error_string(r) : "NCCL error");
}

}  // namespace

extern "C" int kvt_nccl_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int kvt_nccl_unique_id(void* id_out) {
    if (!id_out) return KVT_ERR_ARG;
    NcclApi& api = nccl();
    if (!api.ok) return KVT_ERR_ARG;
    ncclUniqueId id;
    const ncclResult_t r = api.get_unique_id(&id);
    if (r != ncclSuccess) return nccl_status(r);
    std::memcpy(id_out, &id, sizeof(id));
    return KVT_OK;
}

extern "C" int kvt_nccl_comm_init(void** comm_out, int nranks, int rank, const void* id) {
    if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks) return KVT_ERR_ARG;
    NcclApi& api = nccl();
    if (!api.ok) return KVT_ERR_ARG;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    const ncclResult_t r = api.comm_init_rank(&c, nranks, uid, rank);
    if (r != ncclSuccess) return nccl_status(r);
    *comm_out = c;
    return KVT_OK;
}

extern "C" int kvt_nccl_comm_destroy(void* comm) {
    if (!comm) return KVT_ERR_ARG;
    NcclApi& api = nccl();
    if (!api.ok) return KVT_ERR_ARG;
    return nccl_status(api.comm_destroy((ncclComm_t)comm));
}

// part_local [n_lanes][d + 2] f64 (m, l, o normalised) of this rank; gather_buf [nranks]
// [n_lanes][d + 2] f64 (device); out / out64 [n_lanes][d].
extern "C" int kvt_lse_allgather_merge(void* comm, int nranks, const double* part_local, int64_t n_lanes, int d,
                                       double logit_scale, double* gather_buf, float* out, double* out64,
                                       void* stream) {
    if (!comm || !part_local || !gather_buf || (!out && !out64) || nranks < 1 || nranks > 64 || n_lanes < 0 || d < 1)
        return KVT_ERR_ARG;
    NcclApi& api = nccl();
    if (!api.ok) return KVT_ERR_ARG;
    if (n_lanes == 0) return KVT_OK;
    const size_t count = (size_t)n_lanes * (size_t)(d + 2);
    const ncclResult_t r = api.all_gather(part_local, gather_buf, count, ncclFloat64, (ncclComm_t)comm,
                                          (cudaStream_t)stream);
    if (r != ncclSuccess) return nccl_status(r);
    return kvt_lse_merge(gather_buf, nranks, n_lanes, d, logit_scale, out, out64, stream);
}
