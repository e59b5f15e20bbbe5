// Small device helpers shared by the FCC-DCT kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fcct {
namespace dev {

template <typename R>
struct C2;
template <>
struct __align__(16) C2<double> {
    double x, y;
};
template <>
struct __align__(8) C2<float> {
    float x, y;
};

template <typename R>
__device__ __forceinline__ void cmac(C2<R>& acc, const C2<R>& a, const C2<R>& b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// --- mbarrier + TMA bulk copies (cp.async.bulk, 1D) ----------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
// wait until at most n (0..15) of this thread's most recent bulk groups still read shared memory
__device__ __forceinline__ void tma_store_wait_read_n(int n) {
    switch (n) {
        case 0: tma_store_wait_read<0>(); break;
        case 1: tma_store_wait_read<1>(); break;
        case 2: tma_store_wait_read<2>(); break;
        case 3: tma_store_wait_read<3>(); break;
        case 4: tma_store_wait_read<4>(); break;
        case 5: tma_store_wait_read<5>(); break;
        case 6: tma_store_wait_read<6>(); break;
        case 7: tma_store_wait_read<7>(); break;
        case 8: tma_store_wait_read<8>(); break;
        case 9: tma_store_wait_read<9>(); break;
        case 10: tma_store_wait_read<10>(); break;
        case 11: tma_store_wait_read<11>(); break;
        case 12: tma_store_wait_read<12>(); break;
        case 13: tma_store_wait_read<13>(); break;
        case 14: tma_store_wait_read<14>(); break;
        default: tma_store_wait_read<15>(); break;
    }
}
__device__ __forceinline__ void tma_store_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// --- programmatic dependent launch ---------------------------------------
// pdl_wait: block until the preceding kernel in the stream has completed and
// its memory is visible (a no-op without the launch attribute); pdl_trigger:
// let the next kernel's CTAs be scheduled (their prologue overlaps this tail)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// --- cp.async 16B with zero fill ----------------------------------------
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(sz)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// --- FP64 tensor core: mma.sync.m8n8k4 ----------------------------------
// Fragments (verified by tests/test_gpu_kernels.py::test_dmma_fragment_layout):
//   A 8x4 row:  a = A[lane>>2][lane&3]
//   B 4x8 col:  b = B[lane&3][lane>>2]
//   C 8x8:      c0,c1 = C[lane>>2][2*(lane&3) + {0,1}]
// m16n8k4: rows lane/4 and lane/4 + 8 of A (a0, a1) and of C (c0, c1 | c2, c3)
__device__ __forceinline__ void dmma1684(double& c0, double& c1, double& c2, double& c3, double a0, double a1,
                                         double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
                 : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

}  // namespace dev
}  // namespace fcct
