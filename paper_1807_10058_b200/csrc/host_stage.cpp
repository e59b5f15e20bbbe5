// Host-side staging: pageable detection, pinned bounce buffers, and a
// persistent copy pool (host_stage.hpp).
#include "host_stage.hpp"

#include <algorithm>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>

namespace fcct {

bool is_pageable_host(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // older drivers report unregistered memory as an error
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

PinnedBuf::~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
}

void PinnedBuf::reserve(size_t b) {
    if (b <= bytes) return;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    const cudaError_t e = cudaHostAlloc(&ptr, b, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        ptr = nullptr;
        throw std::runtime_error(std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    }
    bytes = b;
}

namespace {

// Fixed set of workers; one job at a time (callers serialise on job_mu).
class CopyPool {
public:
    CopyPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        nworkers_ = static_cast<int>(std::min(7u, hw > 1 ? hw / 2 : 0u));
        for (int w = 0; w < nworkers_; ++w) threads_.emplace_back([this, w] { loop(w); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    void copy(void* dst, const void* src, size_t bytes) {
        constexpr size_t kMinPiece = 1 << 20;
        const int parts = static_cast<int>(std::min<size_t>(nworkers_ + 1, std::max<size_t>(1, bytes / kMinPiece)));
        if (parts <= 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> job(job_mu_);
        auto piece = [=](int i) {
            const size_t a = bytes * i / parts, b = bytes * (i + 1) / parts;
            std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
        };
        {
            std::lock_guard<std::mutex> lk(mu_);
            work_ = piece;
            active_ = parts - 1;  // workers 0 .. parts-2 take pieces 1 .. parts-1
            pending_ = parts - 1;
            ++gen_;
        }
        cv_.notify_all();
        piece(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
    }

private:
    void loop(int w) {
        uint64_t seen = 0;
        for (;;) {
            std::function<void(int)> fn;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                if (w >= active_) continue;
                fn = work_;
            }
            fn(w + 1);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    int nworkers_ = 0;
    std::vector<std::thread> threads_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_, done_cv_;
    std::function<void(int)> work_;
    int active_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

CopyPool& pool() {
    static CopyPool p;
    return p;
}

}  // namespace

void par_memcpy(void* dst, const void* src, size_t bytes) { pool().copy(dst, src, bytes); }

}  // namespace fcct
