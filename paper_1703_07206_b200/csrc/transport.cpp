// transport.cpp — see transport.hpp.
#include "transport.hpp"

#include <dlfcn.h>
#include <nccl.h>  // types only: the library is opened at run time

#include <algorithm>
#include <chrono>
#include <cstring>

#include "engine.hpp"

namespace sgmlb {

// ---------------------------------------------------------------------------
// in-process ranks
// ---------------------------------------------------------------------------

LocalGroup::LocalGroup(int n)
    : size(n), a(n, nullptr), nz(n, 0), flags(n, nullptr), red(n, nullptr), host(n) {}

void LocalGroup::barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == size) {
        arrived = 0;
        ++generation;
        cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != gen; })) {
        // a rank failed before this exchange: do not hang the others
        --arrived;
        fail(SGML_ELOGIC, "local clique: a rank did not reach the exchange within 120 s");
    }
}

LocalTransport::LocalTransport(std::shared_ptr<LocalGroup> g, int r) : g_(std::move(g)) {
    size = g_->size;
    rank = r;
}

void LocalTransport::halo(double* a, long long plane, int nz, int* flags, cudaStream_t s) {
    SGML_CUDA(cudaStreamSynchronize(s));
    g_->a[rank] = a;
    g_->nz[rank] = nz;
    g_->flags[rank] = flags;
    g_->barrier();
    const size_t bytes = (size_t)plane * sizeof(double);
    if (rank > 0) {  // my plane 0 <- lower rank's last own plane
        const int p = rank - 1;
        SGML_CUDA(cudaMemcpyAsync(a, g_->a[p] + plane * g_->nz[p], bytes, cudaMemcpyDeviceToDevice, s));
        SGML_CUDA(cudaMemcpyAsync(flags + 2, g_->flags[p] + 1, sizeof(int), cudaMemcpyDeviceToDevice, s));
    }
    if (rank + 1 < size) {  // my plane nz + 1 <- upper rank's first own plane
        const int p = rank + 1;
        SGML_CUDA(cudaMemcpyAsync(a + plane * (nz + 1), g_->a[p] + plane, bytes, cudaMemcpyDeviceToDevice, s));
        SGML_CUDA(cudaMemcpyAsync(flags + 3, g_->flags[p] + 1, sizeof(int), cudaMemcpyDeviceToDevice, s));
    }
    SGML_CUDA(cudaStreamSynchronize(s));
    g_->barrier();
}

void LocalTransport::allgather(double* a, const std::vector<long long>& off, const std::vector<long long>& cnt,
                               cudaStream_t s) {
    SGML_CUDA(cudaStreamSynchronize(s));
    g_->a[rank] = a;
    g_->barrier();
    for (int p = 0; p < size; ++p)
        if (p != rank && cnt[p] > 0)
            SGML_CUDA(cudaMemcpyAsync(a + off[p], g_->a[p] + off[p], (size_t)cnt[p] * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
    SGML_CUDA(cudaStreamSynchronize(s));
    g_->barrier();
}

template <typename T>
void LocalTransport::reduce_max(T* d, int n, cudaStream_t s) {
    std::vector<unsigned long long>& mine = g_->host[rank];
    mine.assign(n, 0);
    std::vector<T> tmp(n);
    SGML_CUDA(cudaMemcpyAsync(tmp.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    SGML_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < n; ++i) mine[i] = (unsigned long long)tmp[i];
    g_->barrier();
    for (int p = 0; p < size; ++p)
        for (int i = 0; i < n; ++i) tmp[i] = std::max(tmp[i], (T)g_->host[p][i]);
    g_->barrier();
    SGML_CUDA(cudaMemcpyAsync(d, tmp.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    SGML_CUDA(cudaStreamSynchronize(s));
}

void LocalTransport::allreduce_max_u64(unsigned long long* d, int n, cudaStream_t s) { reduce_max(d, n, s); }
void LocalTransport::allreduce_max_i32(int* d, int n, cudaStream_t s) { reduce_max(d, n, s); }

// ---------------------------------------------------------------------------
// NCCL
// ---------------------------------------------------------------------------

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // an already loaded libnccl.so.2 (e.g. torch's) is reused by soname
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
        auto sym = [](const char* s) { return dlsym(api.h, s); };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.Send = (decltype(api.Send))sym("ncclSend");
        api.Recv = (decltype(api.Recv))sym("ncclRecv");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    });
    if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.AllReduce ||
        !api.Broadcast || !api.GroupStart || !api.GroupEnd)
        fail(SGML_ENCCL, "libnccl.so.2 could not be opened (multi-GPU solves need NCCL)");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        fail(SGML_ENCCL, std::string("NCCL error ") + msg + " at " + what);
    }
}
#define SGML_NCCL(call) nccl_check((call), #call)

class NcclTransport : public Transport {
public:
    NcclTransport(int n, int r, const unsigned char id[128]) {
        size = n;
        rank = r;
        ncclUniqueId uid;
        static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(&uid, id, 128);
        SGML_NCCL(nccl().CommInitRank(&comm_, n, uid, r));
    }
    ~NcclTransport() override {
        if (comm_ && nccl().CommDestroy) nccl().CommDestroy(comm_);
    }
    void halo(double* a, long long plane, int nz, int* flags, cudaStream_t s) override {
        const auto& N = nccl();
        SGML_NCCL(N.GroupStart());
        if (rank > 0) {
            SGML_NCCL(N.Send(a + plane, (size_t)plane, ncclFloat64, rank - 1, comm_, s));
            SGML_NCCL(N.Recv(a, (size_t)plane, ncclFloat64, rank - 1, comm_, s));
            SGML_NCCL(N.Send(flags + 1, 1, ncclInt32, rank - 1, comm_, s));
            SGML_NCCL(N.Recv(flags + 2, 1, ncclInt32, rank - 1, comm_, s));
        }
        if (rank + 1 < size) {
            SGML_NCCL(N.Send(a + plane * nz, (size_t)plane, ncclFloat64, rank + 1, comm_, s));
            SGML_NCCL(N.Recv(a + plane * (nz + 1), (size_t)plane, ncclFloat64, rank + 1, comm_, s));
            SGML_NCCL(N.Send(flags + 1, 1, ncclInt32, rank + 1, comm_, s));
            SGML_NCCL(N.Recv(flags + 3, 1, ncclInt32, rank + 1, comm_, s));
        }
        SGML_NCCL(N.GroupEnd());
    }
    void allgather(double* a, const std::vector<long long>& off, const std::vector<long long>& cnt,
                   cudaStream_t s) override {
        const auto& N = nccl();
        SGML_NCCL(N.GroupStart());
        for (int p = 0; p < size; ++p)
            if (cnt[p] > 0)
                SGML_NCCL(N.Broadcast(a + off[p], a + off[p], (size_t)cnt[p], ncclFloat64, p, comm_, s));
        SGML_NCCL(N.GroupEnd());
    }
    void allreduce_max_u64(unsigned long long* d, int n, cudaStream_t s) override {
        SGML_NCCL(nccl().AllReduce(d, d, (size_t)n, ncclUint64, ncclMax, comm_, s));
    }
    void allreduce_max_i32(int* d, int n, cudaStream_t s) override {
        SGML_NCCL(nccl().AllReduce(d, d, (size_t)n, ncclInt32, ncclMax, comm_, s));
    }
    // NCCL send/recv/broadcast are graph-capturable (SGML_NO_SLAB_GRAPHS=1: eager)
    bool graph_capturable() const override { return std::getenv("SGML_NO_SLAB_GRAPHS") == nullptr; }

private:
    ncclComm_t comm_ = nullptr;
};

}  // namespace

void nccl_unique_id(unsigned char out[128]) {
    ncclUniqueId uid;
    SGML_NCCL(nccl().GetUniqueId(&uid));
    std::memcpy(out, &uid, 128);
}

std::unique_ptr<Transport> make_nccl_transport(int nranks, int rank, const unsigned char id[128]) {
    return std::unique_ptr<Transport>(new NcclTransport(nranks, rank, id));
}

}  // namespace sgmlb
