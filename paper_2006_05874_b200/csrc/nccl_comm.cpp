// nccl_comm.cpp — the collectives of the row-sharded path, through NCCL.
//
// libnccl is resolved at run time (dlopen of libnccl.so.2) the first time a
// multi-rank problem needs it, so a process that already loaded PyTorch's
// NCCL shares that copy and single-GPU users never load NCCL at all. Only
// the types come from the system nccl.h.
#include "common.cuh"

#include <cstring>
#include <dlfcn.h>
#include <mutex>
#include <nccl.h>

namespace ihs_b200 {

namespace {
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.AllGather && a.GetErrorString;
    });
    if (!a.ok) fail(IHS_NCCL_ERROR, "libnccl.so.2 could not be loaded");
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(IHS_NCCL_ERROR, std::string(what) + ": " + api().GetErrorString(r));
}
}  // namespace

void nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    check(api().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId layout");
    std::memcpy(out, &id, 128);
}

void* nccl_comm_create(const uint8_t id_bytes[128], int world, int rank) {
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, 128);
    ncclComm_t comm = nullptr;
    check(api().CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
    return comm;
}

void nccl_comm_destroy(void* comm) {
    if (comm) api().CommDestroy(static_cast<ncclComm_t>(comm));
}

void nccl_allreduce_sum(double* buf, size_t count, void* comm, cudaStream_t st) {
    check(api().AllReduce(buf, buf, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), st), "ncclAllReduce");
}

void nccl_allgather(const double* send, double* recv, size_t count_per_rank, void* comm, cudaStream_t st) {
    check(api().AllGather(send, recv, count_per_rank, ncclFloat64, static_cast<ncclComm_t>(comm), st),
          "ncclAllGather");
}

}  // namespace ihs_b200
