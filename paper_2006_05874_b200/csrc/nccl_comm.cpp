// nccl_comm.cpp — the collectives of the row-sharded path.
//
// A communicator is either
//   * NCCL: libnccl is resolved at run time (dlopen of libnccl.so.2) the first time a multi-rank problem needs
//     it, so a process that already loaded PyTorch's NCCL shares that copy and single-GPU users never load
//     NCCL at all (only the types come from the system nccl.h); or
//   * emulated: world_size ranks of ONE process, each driven by its own host thread and stream, usually on one
//     device (ihs_gpu_emu_comm_create). Every collective is a host barrier among the rank threads plus
//     device-side copies ordered by CUDA events — no kernel ever waits on another launch — so the library's
//     real world_size > 1 code (sharded sketches, gradient and Gram all-reduces, the adaptive loop) runs and is
//     tested without a multi-GPU box. Sums are taken in rank order, so every rank gets identical bytes.
#include "common.cuh"

#include <condition_variable>
#include <cstring>
#include <dlfcn.h>
#include <memory>
#include <mutex>
#include <nccl.h>
#include <vector>

namespace ihs_b200 {

namespace {
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
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
        a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(h, "ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(h, "ncclRecv"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.AllGather && a.GetErrorString &&
               a.Send && a.Recv && a.GroupStart && a.GroupEnd;
    });
    if (!a.ok) fail(IHS_NCCL_ERROR, "libnccl.so.2 could not be loaded");
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(IHS_NCCL_ERROR, std::string(what) + ": " + api().GetErrorString(r));
}
}  // namespace

// ---------------------------------------------------------------- emulated group
struct EmuGroup {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t gen = 0;
    std::vector<const double*> src;  // per rank: posted buffer of the collective in flight
    std::vector<cudaEvent_t> ready, done;
    explicit EmuGroup(int w) : world(w), src(w, nullptr), ready(w, nullptr), done(w, nullptr) {
        for (int r = 0; r < w; ++r) {
            CUDA_CHECK(cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming));
            CUDA_CHECK(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
        }
    }
    ~EmuGroup() {
        for (auto e : ready) cudaEventDestroy(e);
        for (auto e : done) cudaEventDestroy(e);
    }
    void barrier() {  // host barrier of the rank threads (generation counted, reusable)
        std::unique_lock<std::mutex> lk(mu);
        const int64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct Comm {
    bool emulated = false;
    ncclComm_t nccl = nullptr;
    std::shared_ptr<EmuGroup> grp;
    int rank = 0, world = 1;
    double* tmp = nullptr;  // emulated all-reduce scratch (this rank's sum)
    size_t tmp_count = 0;
    ~Comm() {
        if (tmp) cudaFree(tmp);
    }
};

__global__ void emu_sum_kernel(const double* const* __restrict__ srcs, int world, size_t count,
                               double* __restrict__ out) {
    pdl_wait();
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        double s = srcs[0][i];
        for (int p = 1; p < world; ++p) s += srcs[p][i];  // rank order: identical on every rank
        out[i] = s;
    }
}

// every rank posts its buffer (and the event after which it is ready), then waits for all others' events
void emu_post(Comm* c, const double* buf, cudaStream_t st) {
    EmuGroup& g = *c->grp;
    g.src[c->rank] = buf;
    CUDA_CHECK(cudaEventRecord(g.ready[c->rank], st));
    g.barrier();
    for (int p = 0; p < g.world; ++p)
        if (p != c->rank) CUDA_CHECK(cudaStreamWaitEvent(st, g.ready[p], 0));
}
// no rank may reuse its posted buffer before every rank has read it
void emu_finish(Comm* c, cudaStream_t st) {
    EmuGroup& g = *c->grp;
    CUDA_CHECK(cudaEventRecord(g.done[c->rank], st));
    g.barrier();
    for (int p = 0; p < g.world; ++p)
        if (p != c->rank) CUDA_CHECK(cudaStreamWaitEvent(st, g.done[p], 0));
}

void emu_allreduce_sum(Comm* c, double* buf, size_t count, cudaStream_t st) {
    EmuGroup& g = *c->grp;
    if (c->tmp_count < count + (size_t)g.world) {
        if (c->tmp) CUDA_CHECK(cudaFree(c->tmp));
        CUDA_CHECK(cudaMalloc(&c->tmp, (count + (size_t)g.world) * sizeof(double)));
        c->tmp_count = count + (size_t)g.world;
    }
    emu_post(c, buf, st);
    // the source pointer table rides in front of the sum buffer
    std::vector<const double*> srcs(g.src.begin(), g.src.end());
    const double** d_srcs = reinterpret_cast<const double**>(c->tmp + count);
    CUDA_CHECK(cudaMemcpyAsync(d_srcs, srcs.data(), srcs.size() * sizeof(double*), cudaMemcpyHostToDevice, st));
    const int blocks = (int)std::min<size_t>(ceil_div((int64_t)count, 256), 148 * 8);
    if (count > 0) LAUNCH_PDL(emu_sum_kernel, std::max(blocks, 1), 256, 0, st, d_srcs, g.world, count, c->tmp);
    emu_finish(c, st);
    CUDA_CHECK(cudaMemcpyAsync(buf, c->tmp, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CUDA_CHECK(cudaStreamSynchronize(st));  // the host copy of the pointer table must outlive the transfer
}

void emu_allgather(Comm* c, const double* send, double* recv, size_t count, cudaStream_t st) {
    EmuGroup& g = *c->grp;
    emu_post(c, send, st);
    for (int p = 0; p < g.world; ++p)
        if (recv + (size_t)p * count != g.src[p])
            CUDA_CHECK(cudaMemcpyAsync(recv + (size_t)p * count, g.src[p], count * sizeof(double),
                                       cudaMemcpyDeviceToDevice, st));
    emu_finish(c, st);
}

void emu_alltoall(Comm* c, const double* send, double* recv, size_t count, cudaStream_t st) {
    EmuGroup& g = *c->grp;
    emu_post(c, send, st);
    for (int p = 0; p < g.world; ++p)  // block `rank` of rank p's send buffer
        CUDA_CHECK(cudaMemcpyAsync(recv + (size_t)p * count, g.src[p] + (size_t)c->rank * count, count * sizeof(double),
                                   cudaMemcpyDeviceToDevice, st));
    emu_finish(c, st);
}

void nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    check(api().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId layout");
    std::memcpy(out, &id, 128);
}

void* nccl_comm_create(const uint8_t id_bytes[128], int world, int rank) {
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, 128);
    ncclComm_t nc = nullptr;
    check(api().CommInitRank(&nc, world, id, rank), "ncclCommInitRank");
    auto* c = new Comm;
    c->nccl = nc;
    c->rank = rank;
    c->world = world;
    return c;
}

void emu_comm_create(int world, void** out) {
    auto grp = std::make_shared<EmuGroup>(world);
    for (int r = 0; r < world; ++r) {
        auto* c = new Comm;
        c->emulated = true;
        c->grp = grp;
        c->rank = r;
        c->world = world;
        out[r] = c;
    }
}

int comm_world(const void* comm) { return comm ? static_cast<const Comm*>(comm)->world : 1; }
int comm_rank(const void* comm) { return comm ? static_cast<const Comm*>(comm)->rank : 0; }

void nccl_comm_destroy(void* comm) {
    auto* c = static_cast<Comm*>(comm);
    if (!c) return;
    if (!c->emulated && c->nccl) api().CommDestroy(c->nccl);
    delete c;
}

void nccl_allreduce_sum(double* buf, size_t count, void* comm, cudaStream_t st) {
    auto* c = static_cast<Comm*>(comm);
    if (c->emulated) return emu_allreduce_sum(c, buf, count, st);
    check(api().AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->nccl, st), "ncclAllReduce");
}

void nccl_allgather(const double* send, double* recv, size_t count_per_rank, void* comm, cudaStream_t st) {
    auto* c = static_cast<Comm*>(comm);
    if (c->emulated) return emu_allgather(c, send, recv, count_per_rank, st);
    check(api().AllGather(send, recv, count_per_rank, ncclFloat64, c->nccl, st), "ncclAllGather");
}

void nccl_alltoall(const double* send, double* recv, size_t count_per_rank, void* comm, cudaStream_t st) {
    auto* c = static_cast<Comm*>(comm);
    if (c->emulated) return emu_alltoall(c, send, recv, count_per_rank, st);
    NcclApi& a = api();
    check(a.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < c->world; ++p) {
        check(a.Send(send + (size_t)p * count_per_rank, count_per_rank, ncclFloat64, p, c->nccl, st), "ncclSend");
        check(a.Recv(recv + (size_t)p * count_per_rank, count_per_rank, ncclFloat64, p, c->nccl, st), "ncclRecv");
    }
    check(a.GroupEnd(), "ncclGroupEnd");
}

}  // namespace ihs_b200
