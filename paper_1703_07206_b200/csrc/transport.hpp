// transport.hpp — the exchange steps of the z-slab decomposition
// (SURVEY.md §8e): halo planes between neighbouring ranks, plane all-gathers
// of replicated coarse levels and of the dense result, and the per-cycle max
// reductions.  Two implementations with one contract:
//
//  * NcclTransport: one process per GPU, NCCL send/recv/all-reduce on the
//    engine stream over NVLink (libnccl is opened at run time, so single-GPU
//    users never need it).
//  * LocalTransport: P ranks as P host threads of one process sharing one
//    device (the parity tests run the decomposition on a single GPU).  Every
//    exchange synchronises the rank's stream, meets the others at a host
//    barrier, pulls the peers' planes with device copies and meets again;
//    no kernel ever waits on another rank's kernel.
//
// Every rank calls the same sequence of operations (the schedule is the
// same on all ranks), which is what pairs them up, as with NCCL.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace sgmlb {

class Transport {
public:
    virtual ~Transport() = default;
    int size = 1;
    int rank = 0;
    // Halo planes of a z-slab array: `a` holds ext planes 0 .. nz + 1 of
    // `plane` doubles each (0 and nz + 1 are the halos).  Own plane 1 goes to
    // rank - 1 (its plane nz' + 1), own plane nz to rank + 1 (its plane 0).
    // flags[1] (this rank's tiny-value flag) travels along: it lands in the
    // receiver's flags[2] (from rank - 1) and flags[3] (from rank + 1).
    virtual void halo(double* a, long long plane, int nz, int* flags, cudaStream_t s) = 0;
    // Replicated buffer `a`: rank r owns doubles [off[r], off[r] + cnt[r]);
    // afterwards every rank holds every rank's part.
    virtual void allgather(double* a, const std::vector<long long>& off, const std::vector<long long>& cnt,
                           cudaStream_t s) = 0;
    // element-wise max over ranks (non-negative doubles as u64, or flags)
    virtual void allreduce_max_u64(unsigned long long* d, int n, cudaStream_t s) = 0;
    virtual void allreduce_max_i32(int* d, int n, cudaStream_t s) = 0;
    // every exchange is stream-ordered device work (no host synchronisation),
    // so a cycle with its exchanges can be captured into a CUDA graph
    virtual bool graph_capturable() const { return false; }
};

// ---- in-process ranks ------------------------------------------------------
struct LocalGroup {
    explicit LocalGroup(int n);
    int size;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    // per-rank posted operands of the current exchange
    std::vector<double*> a;
    std::vector<int> nz;
    std::vector<int*> flags;
    std::vector<void*> red;
    std::vector<std::vector<unsigned long long>> host;
    void barrier();
};

class LocalTransport : public Transport {
public:
    LocalTransport(std::shared_ptr<LocalGroup> g, int rank);
    void halo(double* a, long long plane, int nz, int* flags, cudaStream_t s) override;
    void allgather(double* a, const std::vector<long long>& off, const std::vector<long long>& cnt,
                   cudaStream_t s) override;
    void allreduce_max_u64(unsigned long long* d, int n, cudaStream_t s) override;
    void allreduce_max_i32(int* d, int n, cudaStream_t s) override;

private:
    std::shared_ptr<LocalGroup> g_;
    template <typename T>
    void reduce_max(T* d, int n, cudaStream_t s);
};

// ---- NCCL (one process per GPU) ------------------------------------------
// unique id of a new clique (128 bytes, rank 0 creates it and shares it)
void nccl_unique_id(unsigned char out[128]);
std::unique_ptr<Transport> make_nccl_transport(int nranks, int rank, const unsigned char id[128]);

}  // namespace sgmlb
