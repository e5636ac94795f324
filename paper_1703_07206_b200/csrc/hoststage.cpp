// hoststage.cpp — host <-> device copies of PAGEABLE host buffers at pinned
// speed (the reference's Fields are std::vector<double>: every drop-in call
// moves pageable memory).
//
// A plain cudaMemcpy from pageable memory goes through the driver's small
// bounce buffers at well below the PCIe rate (measured: a 513^3 solve through
// sgml_solve spent ~145 ms moving 2 x 1.08 GB).  Here the copy is pipelined
// through a ring of pinned chunks owned by the context: host worker threads
// copy chunk i + 1 between the user's buffer and a pinned slot while the DMA
// engine moves chunk i, so the transfer runs at min(PCIe, host memcpy
// bandwidth of the workers).  Already-pinned buffers (sgml_host_alloc,
// cudaHostRegister) take the direct path.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.hpp"

namespace sgmlb {

namespace {

constexpr size_t kChunk = size_t(32) << 20;  // bytes per pinned slot
constexpr int kSlots = 4;
constexpr size_t kDirect = size_t(4) << 20;  // smaller copies: plain cudaMemcpyAsync

// fixed pool of memcpy workers; run() splits one copy over all of them (the
// calling thread takes a share) and returns when every part is done
class CopyPool {
public:
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (std::thread& t : workers_) t.join();
    }
    void run(char* dst, const char* src, size_t bytes) {
        const int parts = (int)workers_.size() + 1;
        // (rounded up: a chunk of fewer bytes than parts still gets copied)
        const size_t per = ((bytes + parts - 1) / parts + 63) & ~size_t(63);
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = dst;
            src_ = src;
            bytes_ = bytes;
            per_ = per;
            pending_ = (int)workers_.size();
            ++gen_;
        }
        cv_.notify_all();
        part(parts - 1);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }

private:
    void part(int i) {
        const size_t b = std::min(bytes_, per_ * (size_t)i), e = std::min(bytes_, b + per_);
        if (e > b) std::memcpy(dst_ + b, src_ + b, e - b);
    }
    void loop(int i) {
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            part(i);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    bool stop_ = false;
    unsigned long long gen_ = 0;
    int pending_ = 0;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0, per_ = 0;
};

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace

struct HostStager {
    char* slot[kSlots] = {};
    cudaEvent_t done[kSlots] = {};
    bool used[kSlots] = {};
    CopyPool pool;
    HostStager() : pool(std::clamp((int)std::thread::hardware_concurrency() / 2, 1, 8) - 1) {
        for (int s = 0; s < kSlots; ++s) {
            SGML_CUDA(cudaMallocHost((void**)&slot[s], kChunk));
            SGML_CUDA(cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming));
        }
    }
    ~HostStager() {
        for (int s = 0; s < kSlots; ++s) {
            if (done[s]) {
                cudaEventSynchronize(done[s]);
                cudaEventDestroy(done[s]);
            }
            if (slot[s]) cudaFreeHost(slot[s]);
        }
    }
    void reuse(int s) {
        if (used[s]) SGML_CUDA(cudaEventSynchronize(done[s]));
        used[s] = true;
    }
};

void destroy_stager(HostStager* st) { delete st; }

static HostStager& stager(sgml_ctx* ctx) {
    if (!ctx->stager) ctx->stager = new HostStager();
    return *ctx->stager;
}

// host (any) -> device, in the context's stream order.  Returns once `src` has
// been consumed (the caller may overwrite it); the device copy completes in
// stream order.  Call with the context lock held.
void copy_h2d(sgml_ctx* ctx, void* dst, const void* src, size_t bytes) {
    const cudaStream_t s = ctx->stream;
    if (bytes <= kDirect || is_pinned(src)) {
        // (from pageable memory the source is consumed when the call returns)
        SGML_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    HostStager& st = stager(ctx);
    const char* in = static_cast<const char*>(src);
    char* out = static_cast<char*>(dst);
    for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
        const int sl = (int)(i % kSlots);
        const size_t n = std::min(kChunk, bytes - off);
        st.reuse(sl);  // the slot's previous DMA has finished
        st.pool.run(st.slot[sl], in + off, n);
        SGML_CUDA(cudaMemcpyAsync(out + off, st.slot[sl], n, cudaMemcpyHostToDevice, s));
        SGML_CUDA(cudaEventRecord(st.done[sl], s));
    }
}

// device -> host (any); returns when `dst` holds the data.  Call with the
// context lock held.
void copy_d2h(sgml_ctx* ctx, void* dst, const void* src, size_t bytes) {
    const cudaStream_t s = ctx->stream;
    if (bytes <= kDirect || is_pinned(dst)) {
        SGML_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
        return;
    }
    HostStager& st = stager(ctx);
    const char* in = static_cast<const char*>(src);
    char* out = static_cast<char*>(dst);
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t i) {
        const int sl = (int)(i % kSlots);
        const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
        st.reuse(sl);
        SGML_CUDA(cudaMemcpyAsync(st.slot[sl], in + off, n, cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaEventRecord(st.done[sl], s));
    };
    for (size_t i = 0; i < std::min<size_t>(nch, kSlots); ++i) issue(i);
    for (size_t i = 0; i < nch; ++i) {
        const int sl = (int)(i % kSlots);
        const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
        SGML_CUDA(cudaEventSynchronize(st.done[sl]));
        st.pool.run(out + off, st.slot[sl], n);
        st.used[sl] = false;  // drained by the host
        if (i + kSlots < nch) issue(i + kSlots);
    }
}

}  // namespace sgmlb
