// Communication for the 1D-partitioned BFS (Alg. 2/3):
//   allgather_inplace  -- bottom-up pull of every partition's next-frontier slice
//                         (Alg. 3 PullFrontiers)
//   alltoallv          -- top-down push of (vertex, parent) claims to their owners
//                         (Alg. 2 PushFrontiers), variable sizes
//   allreduce_sum_i64  -- the per-level switch counters (every rank then applies
//                         the same integer rule: no coordinator, contrast P:153)
// Two backends behind one interface:
//   NcclComm   one process per GPU; NCCL is dlopen'ed ("libnccl.so.2") so the
//              single-GPU library has no NCCL dependency.
//   LocalComm  p ranks as p host threads of ONE process on ONE device, exchanging
//              through device memcpy -- a test vehicle that runs the exact same
//              partitioned host/kernels code on a single GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <algorithm>
#include <memory>
#include <mutex>

#include "internal.cuh"

namespace bfsb {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // prefer an already-loaded NCCL (torch's), then the default search path
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.h = h;
#define LOAD(field, sym) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym))
        LOAD(GetUniqueId, "ncclGetUniqueId");
        LOAD(CommInitRank, "ncclCommInitRank");
        LOAD(CommDestroy, "ncclCommDestroy");
        LOAD(AllGather, "ncclAllGather");
        LOAD(AllReduce, "ncclAllReduce");
        LOAD(Send, "ncclSend");
        LOAD(Recv, "ncclRecv");
        LOAD(GroupStart, "ncclGroupStart");
        LOAD(GroupEnd, "ncclGroupEnd");
        LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
    });
    if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.AllReduce || !api.Send ||
        !api.Recv || !api.GroupStart || !api.GroupEnd)
        fail(BFS_ERR_NCCL, std::string("cannot load NCCL (libnccl.so.2): ") + (dlerror() ? dlerror() : "missing symbols"));
    return api;
}

#define NCCL_TRY(expr)                                                                                   \
    do {                                                                                                 \
        ncclResult_t _r = (expr);                                                                        \
        if (_r != ncclSuccess)                                                                           \
            fail(BFS_ERR_NCCL, std::string(#expr) + ": " +                                               \
                                   (nccl().GetErrorString ? nccl().GetErrorString(_r) : "nccl error")); \
    } while (0)

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
    }
    void allgather_inplace(void* buf, size_t bytes_per_rank, cudaStream_t s) override {
        char* b = static_cast<char*>(buf);
        NCCL_TRY(nccl().AllGather(b + (size_t)rank * bytes_per_rank, b, bytes_per_rank, ncclUint8, comm, s));
    }
    void allreduce_sum_i64(int64_t* buf, int count, cudaStream_t s) override {
        NCCL_TRY(nccl().AllReduce(buf, buf, (size_t)count, ncclInt64, ncclSum, comm, s));
    }
    void allreduce_max_i64(int64_t* buf, int count, cudaStream_t s) override {
        NCCL_TRY(nccl().AllReduce(buf, buf, (size_t)count, ncclInt64, ncclMax, comm, s));
    }
    void alltoallv(const void* const* sendp, const size_t* sendb, void* const* recvp, const size_t* recvb,
                   cudaStream_t s) override {
        NCCL_TRY(nccl().GroupStart());
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            if (sendb[q]) NCCL_TRY(nccl().Send(sendp[q], sendb[q], ncclUint8, q, comm, s));
            if (recvb[q]) NCCL_TRY(nccl().Recv(recvp[q], recvb[q], ncclUint8, q, comm, s));
        }
        NCCL_TRY(nccl().GroupEnd());
    }
};

// ------------------------------------------------------------------ local (threads, one device)
struct LocalGroup {
    int n;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<void*> ptr;          // published per-rank pointer
    std::vector<const void* const*> sendp;
    std::vector<const size_t*> sendb;
    std::vector<std::vector<int64_t>> host;
    explicit LocalGroup(int n_) : n(n_), ptr(n_), sendp(n_), sendb(n_), host(n_) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        uint64_t gen = generation;
        if (++arrived == n) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

struct LocalComm final : Comm {
    std::shared_ptr<LocalGroup> grp;
    void allgather_inplace(void* buf, size_t bytes_per_rank, cudaStream_t s) override {
        BFS_CUDA(cudaStreamSynchronize(s));
        grp->ptr[rank] = buf;
        grp->barrier();
        char* me = static_cast<char*>(buf);
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            const char* src = static_cast<const char*>(grp->ptr[q]) + (size_t)q * bytes_per_rank;
            BFS_CUDA(cudaMemcpyAsync(me + (size_t)q * bytes_per_rank, src, bytes_per_rank, cudaMemcpyDeviceToDevice, s));
        }
        BFS_CUDA(cudaStreamSynchronize(s));
        grp->barrier();
    }
    void reduce(int64_t* buf, int count, cudaStream_t s, bool is_max) {
        auto& mine = grp->host[rank];
        mine.resize((size_t)count);
        BFS_CUDA(cudaMemcpyAsync(mine.data(), buf, (size_t)count * 8, cudaMemcpyDeviceToHost, s));
        BFS_CUDA(cudaStreamSynchronize(s));
        grp->barrier();
        std::vector<int64_t> acc(grp->host[0]);
        for (int q = 1; q < nranks; ++q)
            for (int i = 0; i < count; ++i)
                acc[i] = is_max ? std::max(acc[i], grp->host[q][i]) : acc[i] + grp->host[q][i];
        grp->barrier();
        BFS_CUDA(cudaMemcpyAsync(buf, acc.data(), (size_t)count * 8, cudaMemcpyHostToDevice, s));
        BFS_CUDA(cudaStreamSynchronize(s));
    }
    void allreduce_sum_i64(int64_t* buf, int count, cudaStream_t s) override { reduce(buf, count, s, false); }
    void allreduce_max_i64(int64_t* buf, int count, cudaStream_t s) override { reduce(buf, count, s, true); }
    void alltoallv(const void* const* sendp, const size_t* sendb, void* const* recvp, const size_t* recvb,
                   cudaStream_t s) override {
        BFS_CUDA(cudaStreamSynchronize(s));
        grp->sendp[rank] = sendp;
        grp->sendb[rank] = sendb;
        grp->barrier();
        for (int q = 0; q < nranks; ++q) {
            if (q == rank || !recvb[q]) continue;
            if (grp->sendb[q][rank] != recvb[q]) fail(BFS_ERR_INTERNAL, "alltoallv size mismatch");
            BFS_CUDA(cudaMemcpyAsync(recvp[q], grp->sendp[q][rank], recvb[q], cudaMemcpyDeviceToDevice, s));
        }
        BFS_CUDA(cudaStreamSynchronize(s));
        grp->barrier();
    }
};

void comm_unique_id(uint8_t id[128]) {
    ncclUniqueId u;
    NCCL_TRY(nccl().GetUniqueId(&u));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    std::memcpy(id, &u, 128);
}

Comm* comm_create_nccl(int nranks, int rank, const uint8_t id[128], int device) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(BFS_ERR_INVALID_ARG, "bad nranks/rank");
    BFS_CUDA(cudaSetDevice(device));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    auto* c = new NcclComm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        fail(BFS_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
    }
    return c;
}

void comm_create_local(int nparts, int device, Comm** out) {
    if (nparts < 1 || nparts > 64) fail(BFS_ERR_INVALID_ARG, "nparts must be in [1, 64]");
    auto grp = std::make_shared<LocalGroup>(nparts);
    for (int r = 0; r < nparts; ++r) {
        auto* c = new LocalComm();
        c->grp = grp;
        c->nranks = nparts;
        c->rank = r;
        c->device = device;
        out[r] = c;
    }
}

}  // namespace bfsb
