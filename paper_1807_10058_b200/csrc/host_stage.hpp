// Host-side staging for the *_host entry points (fcct_gpu.h): pageable caller
// buffers go through pinned bounce buffers, with the host-side copies split
// over a small persistent thread pool so that they keep up with PCIe / C2C.
// (The reference's Eigen::VectorXcd storage, transform.hpp:21,32, is ordinary
// pageable heap memory, which is what a drop-in caller hands over.)
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <mutex>
#include <thread>
#include <vector>

namespace fcct {

// True when `p` is ordinary (pageable, unregistered) host memory.
bool is_pageable_host(const void* p);

// memcpy split over the pool's workers (and the calling thread).
void par_memcpy(void* dst, const void* src, size_t bytes);

// Page-locked host buffer (cudaHostAlloc), grown on demand, never shrunk.
struct PinnedBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf();
    void reserve(size_t b);
};

}  // namespace fcct
