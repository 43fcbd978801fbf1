// im_comm.cu -- the library's own NCCL communicator for simulation sharding (
// include/im.h im_comm_nccl_*).  NCCL (over NVLink 5 / NVSwitch) is loaded with dlopen at the first
// call, so the library has no build- or load-time dependency on it; the three collectives of the
// exchange protocol are enqueued on the library's stream (stream-ordered, no host round trip).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "im_internal.h"

namespace im {

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi api;

template <class F>
bool sym(F& f, const char* name) {
    f = reinterpret_cast<F>(dlsym(api.h, name));
    return f != nullptr;
}

// libnccl.so.2: torch's copy if the process already loaded it (same soname), else the system one
int load_nccl(char* err, size_t errn) {
    if (api.h) return 0;
    const char* env = getenv("IM_NCCL_LIB");
    void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        snprintf(err, errn, "dlopen(%s) failed: %s", env ? env : "libnccl.so.2", dlerror());
        return -1;
    }
    api.h = h;
    if (!(sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
          sym(api.CommDestroy, "ncclCommDestroy") && sym(api.AllReduce, "ncclAllReduce") &&
          sym(api.ReduceScatter, "ncclReduceScatter") && sym(api.AllGather, "ncclAllGather") &&
          sym(api.GetErrorString, "ncclGetErrorString"))) {
        snprintf(err, errn, "libnccl.so.2 lacks a required symbol");
        api = NcclApi{};
        return -1;
    }
    return 0;
}

struct NcclState {
    ncclComm_t comm = nullptr;
};

ncclDataType_t dt(int32_t dtype) { return dtype == IM_DTYPE_I64 ? ncclInt64 : ncclInt32; }

int nccl_allreduce(void* buf, int64_t count, int32_t dtype, int32_t op, void* stream, void* user) {
    auto* s = static_cast<NcclState*>(user);
    return (int)api.AllReduce(buf, buf, (size_t)count, dt(dtype), op == IM_OP_MAX ? ncclMax : ncclSum, s->comm,
                              (cudaStream_t)stream);
}
int nccl_reduce_scatter(const void* send, void* recv, int64_t recvcount, int32_t dtype, void* stream, void* user) {
    auto* s = static_cast<NcclState*>(user);
    return (int)api.ReduceScatter(send, recv, (size_t)recvcount, dt(dtype), ncclSum, s->comm, (cudaStream_t)stream);
}
int nccl_allgather(const void* send, void* recv, int64_t sendcount, int32_t dtype, void* stream, void* user) {
    auto* s = static_cast<NcclState*>(user);
    return (int)api.AllGather(send, recv, (size_t)sendcount, dt(dtype), s->comm, (cudaStream_t)stream);
}

}  // namespace

int nccl_unique_id(void* out, char* err, size_t errn) {
    if (load_nccl(err, errn)) return -1;
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) {
        snprintf(err, errn, "ncclGetUniqueId: %s", api.GetErrorString(r));
        return -1;
    }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out, &id, sizeof id);
    return 0;
}

// creates the communicator on the current device and fills `comm` (stream-ordered collectives)
int nccl_init(const void* id128, int rank, int nranks, im_comm* comm, void** state, char* err, size_t errn) {
    if (load_nccl(err, errn)) return -1;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    auto* s = new NcclState;
    ncclResult_t r = api.CommInitRank(&s->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        snprintf(err, errn, "ncclCommInitRank(rank %d of %d): %s", rank, nranks, api.GetErrorString(r));
        delete s;
        return -1;
    }
    *comm = im_comm{};
    comm->rank = rank;
    comm->nranks = nranks;
    comm->stream_ordered = 1;
    comm->allreduce = nccl_allreduce;
    comm->reduce_scatter = nccl_reduce_scatter;
    comm->allgather = nccl_allgather;
    comm->user = s;
    *state = s;
    return 0;
}

void nccl_release(void* state) {
    auto* s = static_cast<NcclState*>(state);
    if (!s) return;
    if (s->comm && api.CommDestroy) api.CommDestroy(s->comm);
    delete s;
}

}  // namespace im
