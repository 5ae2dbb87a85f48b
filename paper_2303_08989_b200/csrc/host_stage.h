// Pinned staging ring for host-buffer entry points called with PAGEABLE
// memory (a reference user's std::vector storage).  A cudaMemcpyAsync from
// pageable memory is synchronous for the calling thread, so the overlapped
// host pipeline would serialise behind it.  Instead every pageable transfer is
// cut into slot-sized pieces: a CUDA host function (stream `host`) copies the
// piece between the user buffer and a pinned slot with a small thread pool,
// and the DMA (the caller's copy stream) moves the slot to / from the device.
// Events order slot reuse, so the CPU copy of piece i+1 overlaps the DMA of
// piece i and the whole exchange stays asynchronous to the calling thread.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

namespace tcec {

// Fixed worker pool running one parallel loop at a time (the host functions
// of a stream run one after another, so there is a single caller).
class CopyPool {
  public:
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    int size() const { return int(workers_.size()) + 1; }
    // fn(part) for part in [0, parts), the calling thread takes part 0
    void run(int parts, const std::function<void(int)>& fn) {
        {
            std::lock_guard<std::mutex> g(mu_);
            fn_ = &fn;
            parts_ = parts;
            pending_ = int(workers_.size());
            ++gen_;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }

  private:
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* f;
            int parts;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                f = fn_;
                parts = parts_;
            }
            if (i + 1 < parts) (*f)(i + 1);
            std::lock_guard<std::mutex> g(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* fn_ = nullptr;
    int parts_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// 2-D host copy (rows of `width` bytes) split by rows over the pool
inline void pool_copy2d(CopyPool& pool, uint8_t* dst, size_t dpitch, const uint8_t* src, size_t spitch,
                        size_t width, size_t height) {
    const int parts = pool.size();
    pool.run(parts, [&](int p) {
        const size_t r0 = height * size_t(p) / size_t(parts), r1 = height * size_t(p + 1) / size_t(parts);
        if (dpitch == width && spitch == width) {
            std::memcpy(dst + r0 * width, src + r0 * width, (r1 - r0) * width);
            return;
        }
        for (size_t r = r0; r < r1; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, width);
    });
}

struct StageRing {
    static constexpr int kSlots = 8;
    static constexpr size_t kSlotBytes = size_t(32) << 20;
    uint8_t* buf = nullptr;  // pinned, kSlots * kSlotBytes
    cudaStream_t host = nullptr;
    cudaEvent_t filled[kSlots] = {}, freed[kSlots] = {};
    int next = 0;
    std::unique_ptr<CopyPool> pool;
    struct Job {
        StageRing* ring;
        uint8_t* dst;
        const uint8_t* src;
        size_t dpitch, spitch, width, height;
    };
    std::vector<std::unique_ptr<Job>> jobs;  // alive until the call synchronises

    ~StageRing() {
        if (host) cudaStreamSynchronize(host);
        for (auto& e : filled)
            if (e) cudaEventDestroy(e);
        for (auto& e : freed)
            if (e) cudaEventDestroy(e);
        if (host) cudaStreamDestroy(host);
        if (buf) cudaFreeHost(buf);
    }

    cudaError_t init() {
        if (buf) return cudaSuccess;
        cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&buf), kSlots * kSlotBytes);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&host, cudaStreamNonBlocking);
        for (int i = 0; i < kSlots && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&filled[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming);
        }
        if (e == cudaSuccess) {
            // copy threads (TCEC_STAGE_THREADS overrides): all but two host cores, <= 16
            const int hc = int(std::thread::hardware_concurrency());
            int t = std::max(1, std::min(16, hc - 2));
            if (const char* env = std::getenv("TCEC_STAGE_THREADS")) t = std::max(1, std::min(64, std::atoi(env)));
            pool = std::make_unique<CopyPool>(t - 1);
        }
        return e;
    }

    static void CUDART_CB run_job(void* p) {
        const Job* j = static_cast<const Job*>(p);
        pool_copy2d(*j->ring->pool, j->dst, j->dpitch, j->src, j->spitch, j->width, j->height);
    }

    // host (pageable, rows of `width` at spitch) -> device (dst, rows at dpitch) on dma
    cudaError_t h2d(uint8_t* dst, size_t dpitch, const uint8_t* src, size_t spitch, size_t width,
                    size_t height, cudaStream_t dma) {
        if (width > kSlotBytes)  // rows wider than a slot: the driver's own staging
            return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, dma);
        const size_t rows = kSlotBytes / width;
        for (size_t r0 = 0; r0 < height; r0 += rows) {
            const size_t nr = std::min(rows, height - r0);
            const int s = next++ % kSlots;
            uint8_t* slot = buf + size_t(s) * kSlotBytes;
            jobs.push_back(std::make_unique<Job>(Job{this, slot, src + r0 * spitch, width, spitch, width, nr}));
            cudaError_t e = cudaStreamWaitEvent(host, freed[s], 0);
            if (e == cudaSuccess) e = cudaLaunchHostFunc(host, run_job, jobs.back().get());
            if (e == cudaSuccess) e = cudaEventRecord(filled[s], host);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(dma, filled[s], 0);
            if (e == cudaSuccess)
                e = cudaMemcpy2DAsync(dst + r0 * dpitch, dpitch, slot, width, width, nr, cudaMemcpyHostToDevice,
                                      dma);
            if (e == cudaSuccess) e = cudaEventRecord(freed[s], dma);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }

    // device (src, rows at spitch) -> host (pageable dst, rows at dpitch), DMA on dma
    cudaError_t d2h(uint8_t* dst, size_t dpitch, const uint8_t* src, size_t spitch, size_t width,
                    size_t height, cudaStream_t dma) {
        if (width > kSlotBytes)
            return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost, dma);
        const size_t rows = kSlotBytes / width;
        for (size_t r0 = 0; r0 < height; r0 += rows) {
            const size_t nr = std::min(rows, height - r0);
            const int s = next++ % kSlots;
            uint8_t* slot = buf + size_t(s) * kSlotBytes;
            jobs.push_back(std::make_unique<Job>(Job{this, dst + r0 * dpitch, slot, dpitch, width, width, nr}));
            cudaError_t e = cudaStreamWaitEvent(dma, freed[s], 0);
            if (e == cudaSuccess)
                e = cudaMemcpy2DAsync(slot, width, src + r0 * spitch, spitch, width, nr, cudaMemcpyDeviceToHost,
                                      dma);
            if (e == cudaSuccess) e = cudaEventRecord(filled[s], dma);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(host, filled[s], 0);
            if (e == cudaSuccess) e = cudaLaunchHostFunc(host, run_job, jobs.back().get());
            if (e == cudaSuccess) e = cudaEventRecord(freed[s], host);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }

    // after the caller synchronised `host` (and its DMA streams)
    void finish() { jobs.clear(); }
};

// true for memory the driver can DMA directly (pinned / registered / managed)
inline bool dma_capable(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type != cudaMemoryTypeUnregistered;
}

}  // namespace tcec
