// fp32 direct transform on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// naive_apply / inverse_apply(dense) (transform.cpp:146-169) for an fp32 plan is
// the real-form GEMM  C[M][Nn] = A[M][K] . W[Nn][K]^T  (A = the batch of blocks,
// complex64 interleaved, K = Nn = 2 n^3; W = D or D^{-1} in real form, both
// K-major). TF32 alone carries 11 significant bits, short of the 1e-5 fp32 bar,
// so the product runs split (3xTF32):
//     A.W ~= A_hi.W_hi + A_hi.W_lo + A_lo.W_hi,   W_hi = rna_tf32(W), A_hi = trunc_tf32(A),
//     x_lo = rna_tf32(x - x_hi)
// with W_hi / W_lo split from the fp64 table at plan time and A split in shared
// memory as each stage lands. All three products accumulate into one fp32
// accumulator in tensor memory.
//
// Persistent kernel, one CTA per SM, warp-specialised (320 threads):
//   warp 0      TMA producer: A, W_hi, W_lo tiles (BK = 32 fp32 = one 128-byte
//               swizzle row) into a 3-stage ring, mbarrier complete_tx
//   warp 1      MMA issuer (one thread): 3 x 4 tcgen05.mma.kind::tf32 per stage,
//               M = 128, N = 128, K = 8; TMEM (512 columns): two hi.hi chunk
//               accumulators (ping-pong every K = 128) and two tile accumulators
//               for the hi.lo + lo.hi corrections; tcgen05.commit frees the stage
//               and hands finished accumulators to the epilogue
//   warps 2-9   epilogue: every K = 128 the hi.hi chunk accumulator is read with
//               tcgen05.ld 32x32b.x32 and added into fp32 registers (one row,
//               64 columns per thread); the tile's hi.lo + lo.hi accumulator is
//               added last, then fp32 stores
//   warps 10-13 converter: A stage -> A_lo (A_hi is the landed tile: kind::tf32
//               drops the low 13 bits), fence.proxy.async
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "device.cuh"
#include "kernels.hpp"

namespace fcct {

using namespace dev;

namespace {

constexpr int kBM = 128, kBN = 128, kBK = 32, kStages = 3;
constexpr int kTileA = kBM * kBK * 4;                   // 16 KB
constexpr int kTileB = kBN * kBK * 4;                   // 16 KB
constexpr int kStageBytes = 2 * kTileA + 2 * kTileB;    // A_hi (landed raw), A_lo, W_hi, W_lo
constexpr int kTxBytes = kTileA + 2 * kTileB;           // what TMA brings per stage
constexpr int kTmemCols = 4 * kBN;                      // 2 main chunk + 2 correction fp32 accumulators
// the hi.hi chain is promoted to fp32 registers every kChunkKb k-blocks (K = 128):
// the tensor core's accumulator alignment rounding grows with the chain length
// (forward error 2.8e-6 at K = 1024 with one chain, ~K-linear)
constexpr int kChunkKb = 4;
constexpr int kEpiThreads = 256, kConvThreads = 128;
constexpr int kThreads = 64 + kEpiThreads + kConvThreads;  // producer, MMA, 8 epilogue, 4 converter warps
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /* barriers */ + 1024 /* alignment */;

// smem matrix descriptor, K-major, 128-byte swizzle (8-row atoms of 1024 bytes)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16)  // LBO (unused for swizzled K-major)
           | (static_cast<uint64_t>(1024 >> 4) << 32)                     // SBO: 8-row group stride
           | (1ull << 46)                                                 // descriptor version (sm_100)
           | (2ull << 61);                                                // SWIZZLE_128B
}

// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(kBN >> 3) << 17) |
                            (static_cast<uint32_t>(kBM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return r;
}

#define TMEM_LD_32(taddr, v)                                                                                      \
    asm volatile(                                                                                                 \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"  \
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                                     \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),        \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),  \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),             \
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),             \
          "=r"(v[30]), "=r"(v[31])                                                                                \
        : "r"(taddr))

__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmWhi,
                       const __grid_constant__ CUtensorMap tmWlo, float* __restrict__ C, int64_t M, int Nn, int K) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128-byte swizzle atoms
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* conv = full + kStages;      // converter -> MMA: A_hi / A_lo written
    uint64_t* empty = conv + kStages;     // MMA -> producer: stage read
    uint64_t* cfull = empty + kStages;    // MMA -> epilogue: a main chunk accumulator is complete
    uint64_t* cempty = cfull + 2;         // epilogue -> MMA: chunk accumulator drained
    uint64_t* rfull = cempty + 2;         // MMA -> epilogue: the tile's correction accumulator
    uint64_t* rempty = rfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tiles = Nn / kBN;
    const int64_t m_tiles = (M + kBM - 1) / kBM;
    const int64_t tiles = m_tiles * n_tiles;
    const int kblocks = K / kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], kConvThreads);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&cfull[a], 1);
            mbar_init(&cempty[a], kEpiThreads);
            mbar_init(&rfull[a], 1);
            mbar_init(&rempty[a], kEpiThreads);
        }
        fence_mbar_init();
    }
    if (warp == 1) {  // TMEM, owned (and freed) by this warp
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmWhi)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmWlo)) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // TMEM columns: [0, 2 BN) two main chunk accumulators, [2 BN, 4 BN) two tile correction accumulators

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            int s = 0;
            uint32_t ph = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int m0 = static_cast<int>((t / n_tiles) * kBM), n0 = static_cast<int>((t % n_tiles) * kBN);
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1u);
                    uint8_t* st = smem + s * kStageBytes;
                    mbar_arrive_expect_tx(&full[s], kTxBytes);
                    tma_load_2d(st, &tmA, kb * kBK, m0, &full[s]);
                    tma_load_2d(st + 2 * kTileA, &tmWhi, kb * kBK, n0, &full[s]);
                    tma_load_2d(st + 2 * kTileA + kTileB, &tmWlo, kb * kBK, n0, &full[s]);
                    if (++s == kStages) s = 0, ph ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            int s = 0, cb = 0, rb = 0;
            uint32_t ph = 0, cph = 0, rph = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                mbar_wait(&rempty[rb], rph ^ 1u);  // the epilogue read this correction accumulator
                const uint32_t dr = tmem_base + static_cast<uint32_t>((2 + rb) * kBN);
                for (int kb = 0; kb < kblocks; ++kb) {
                    const bool chunk_start = kb % kChunkKb == 0;
                    if (chunk_start) mbar_wait(&cempty[cb], cph ^ 1u);  // the epilogue drained this chunk buffer
                    mbar_wait(&conv[s], ph);
                    tc_fence_after();
                    const uint32_t dm = tmem_base + static_cast<uint32_t>(cb * kBN);
                    const uint32_t st = smem_u32(smem + s * kStageBytes);
                    const uint64_t ahi = sw128_desc(st), alo = sw128_desc(st + kTileA);
                    const uint64_t bhi = sw128_desc(st + 2 * kTileA), blo = sw128_desc(st + 2 * kTileA + kTileB);
#pragma unroll
                    for (int k = 0; k < kBK / 8; ++k) {  // K = 8 tf32 = 32 bytes along the swizzled row
                        const uint64_t dk = static_cast<uint64_t>(k * 2);  // 32 bytes in 16-byte units
                        mma_tf32(dm, ahi + dk, bhi + dk, !(chunk_start && k == 0));
                        mma_tf32(dr, ahi + dk, blo + dk, (kb | k) != 0);
                        mma_tf32(dr, alo + dk, bhi + dk, 1u);
                    }
                    mma_commit(&empty[s]);  // the stage is free once these MMAs have read it
                    if (++s == kStages) s = 0, ph ^= 1u;
                    if (kb % kChunkKb == kChunkKb - 1 || kb == kblocks - 1) {
                        mma_commit(&cfull[cb]);  // chunk complete: promote to the epilogue's fp32 registers
                        if (++cb == 2) cb = 0, cph ^= 1u;
                    }
                }
                mma_commit(&rfull[rb]);
                if (++rb == 2) rb = 0, rph ^= 1u;
            }
        }
    } else if (warp < 2 + kEpiThreads / 32) {  // ---- epilogue: chunk promotion + store
        const int e = warp - 2;
        const int quarter = warp & 3;        // TMEM lanes 32*quarter .. +31 belong to this warp
        const int half = e >> 2;             // columns half*64 .. +63 of the tile
        int cb = 0, rb = 0;
        uint32_t cph = 0, rph = 0;
        const int nchunks = (kblocks + kChunkKb - 1) / kChunkKb;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            const int64_t row = (t / n_tiles) * kBM + quarter * 32 + lane;
            const int n0 = static_cast<int>((t % n_tiles) * kBN) + half * 64;
            const uint32_t lanes = static_cast<uint32_t>(quarter * 32) << 16;
            float sum[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) sum[j] = 0.f;
            for (int c = 0; c < nchunks; ++c) {
                mbar_wait(&cfull[cb], cph);
                tc_fence_after();
                const uint32_t ta = tmem_base + lanes + cb * kBN + half * 64;
                uint32_t v[32];
                TMEM_LD_32(ta, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; ++j) sum[j] += __uint_as_float(v[j]);
                TMEM_LD_32(ta + 32, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; ++j) sum[32 + j] += __uint_as_float(v[j]);
                tc_fence_before();
                mbar_arrive(&cempty[cb]);
                if (++cb == 2) cb = 0, cph ^= 1u;
            }
            mbar_wait(&rfull[rb], rph);
            tc_fence_after();
            {
                const uint32_t ta = tmem_base + lanes + (2 + rb) * kBN + half * 64;
                uint32_t v[32];
                TMEM_LD_32(ta, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; ++j) sum[j] += __uint_as_float(v[j]);
                TMEM_LD_32(ta + 32, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; ++j) sum[32 + j] += __uint_as_float(v[j]);
            }
            tc_fence_before();
            mbar_arrive(&rempty[rb]);
            if (++rb == 2) rb = 0, rph ^= 1u;
            if (row < M) {
                float4* dst = reinterpret_cast<float4*>(C + row * Nn + n0);
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    dst[q] = make_float4(sum[4 * q], sum[4 * q + 1], sum[4 * q + 2], sum[4 * q + 3]);
            }
        }
    } else {  // ---- converter: A stage -> A_hi (in place) + A_lo, then hand to the MMA issuer
        const int ct = threadIdx.x - (2 * 32 + kEpiThreads);  // 0..127
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&full[s], ph);
                float4* a = reinterpret_cast<float4*>(smem + s * kStageBytes);
                float4* lo = reinterpret_cast<float4*>(smem + s * kStageBytes + kTileA);
#pragma unroll
                for (int q = 0; q < kTileA / 16 / kConvThreads; ++q) {  // elementwise: the swizzle is irrelevant
                    const int i = q * kConvThreads + ct;
                    // A_hi is the landed tile itself: kind::tf32 reads the upper 19 bits of
                    // each fp32 (the low 13 are dropped), so only A_lo = x - trunc(x) is written
                    const float4 x = a[i];
                    float4 l;
                    l.x = __uint_as_float(to_tf32(x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u)));
                    l.y = __uint_as_float(to_tf32(x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u)));
                    l.z = __uint_as_float(to_tf32(x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u)));
                    l.w = __uint_as_float(to_tf32(x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u)));
                    lo[i] = l;
                }
                fence_proxy_async_smem();  // generic-proxy writes -> tensor-core (async proxy) reads
                mbar_arrive(&conv[s]);
                if (++s == kStages) s = 0, ph ^= 1u;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kTmemCols)
                     : "memory");
    }
}

// ===========================================================================
// fp64 direct transform on tcgen05: Ozaki-scheme split into int8 slices.
//
// Each row of A (a block) and of W (an output of D or D^{-1}) is scaled by a
// power of two sigma >= its max |entry| and cut into kOzS int8 slices,
//     a / sigma = sum_p 2^{-7p} a_p,   |a_p| <= 127   (round to nearest, p = 1..kOzS).
// Every slice product a_p . w_q is an exact int8 GEMM with int32 accumulation
// (K 127^2 * pairs < 2^31 up to K = 8192), and
//     C = sigma_A sigma_W sum_{p+q <= kOzS+1} 2^{-7(p+q)} (a_p . w_q^T).
// Products of equal order d = p + q share a scale and one int32 TMEM accumulator.
// N = 128 per MMA (the A operand's shared-memory reads amortised over 128
// columns); 512 TMEM columns hold four 128-column accumulators, so a tile runs
// in two passes over K: orders d = 0..3 (10 products, slices 0..3), drained into
// fp64 registers by the epilogue, then d = 4..6 (18 products, slices 0..6).
// S = 7 slices (28 products): forward 4.5e-15, inverse 1.6e-14 relative L2 at
// n = 8 against fp64; S = 8 (36 products): 6.5e-16 / 8.7e-16 (tools/ozaki_sim.py).
// The inverse, whose error the conditioning of D^{-1} amplifies, runs S = 8.
constexpr int kOzSMax = 8;                                  // 7 slices forward, 8 inverse (capi.cpp)
constexpr int kOzPass1 = 4;                                 // orders d = 0..3 in the first pass
constexpr int kOzBM = 128, kOzBN = 128, kOzBK = 32;         // BK = 32 int8 = one 32-byte swizzle row
constexpr int kOzStages = 3;
constexpr int kOzTileA = kOzSMax * kOzBM * kOzBK;          // 32 KB: all slices of the A tile
constexpr int kOzTileB = kOzSMax * kOzBN * kOzBK;          // 32 KB
constexpr int kOzStage = kOzTileA + kOzTileB;
constexpr int kOzEpi = 256;                                 // 8 epilogue warps: lane quarter x column half
constexpr int kOzThreads = 64 + kOzEpi;                     // producer, MMA issuer, epilogue
constexpr int kOzSmem = kOzStages * kOzStage + 1024 + 1024;
constexpr int kOzTmemCols = 512;                           // 4 x 128

// smem descriptor, K-major, 32-byte swizzle (8-row atoms of 256 bytes)
__device__ __forceinline__ uint64_t sw32_desc(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (static_cast<uint64_t>(256 >> 4) << 32) |
           (1ull << 46) | (6ull << 61);
}
// D s32, A/B signed int8, K-major, M = 128, N = 128
constexpr uint32_t kOzIdesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kOzBN >> 3) << 17) |
                              (static_cast<uint32_t>(kOzBM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kOzIdesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// rows of A [rows][K] fp64 -> slices [kOzS][rows][K] int8 and scale[rows] = 2^e >= max |row|.
// One warp per row; each lane takes 8 consecutive elements per step (two 32-byte
// loads, one 8-byte store per slice: 256-byte warp stores). K % 8 == 0.
template <int S>
__global__ void ozaki_slice_kernel(const double* __restrict__ a, int64_t rows, int K, int8_t* __restrict__ sl,
                                   double* __restrict__ scale) {
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const double* r = a + row * K;
    double m = 0.0;
    bool nan = false;  // fmax drops NaN operands: track them apart
    for (int k = 8 * lane; k < K; k += 256) {
        const double4* v = reinterpret_cast<const double4*>(r + k);
        const double4 x0 = v[0], x1 = v[1];
        m = fmax(m, fmax(fmax(fabs(x0.x), fabs(x0.y)), fmax(fabs(x0.z), fabs(x0.w))));
        m = fmax(m, fmax(fmax(fabs(x1.x), fabs(x1.y)), fmax(fabs(x1.z), fabs(x1.w))));
        nan |= isnan(x0.x + x0.y + x0.z + x0.w + x1.x + x1.y + x1.z + x1.w);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    nan = __any_sync(0xffffffffu, nan);
    int e = 0;
    const bool finite = isfinite(m) && !nan;
    if (m > 0.0 && finite) frexp(m, &e);  // m = f 2^e, f in [0.5, 1): 2^e > m
    const double inv = (m > 0.0 && finite) ? ldexp(1.0, -e) : 0.0;
    // a row holding inf / NaN gets a NaN scale: its outputs are NaN (the fp64
    // GEMM would propagate them too) instead of silently finite
    if (lane == 0) scale[row] = !finite ? __longlong_as_double(0x7FF8000000000000LL) : (m > 0.0 ? ldexp(1.0, e) : 1.0);
    const int64_t plane = rows * static_cast<int64_t>(K);
    for (int k = 8 * lane; k < K; k += 256) {
        const double4* v4 = reinterpret_cast<const double4*>(r + k);
        const double4 x0 = v4[0], x1 = v4[1];
        double v[8] = {x0.x * inv, x0.y * inv, x0.z * inv, x0.w * inv, x1.x * inv, x1.y * inv, x1.z * inv, x1.w * inv};
#pragma unroll
        for (int q = 1; q <= S; ++q) {
            const double sc = ldexp(1.0, 7 * q), isc = ldexp(1.0, -7 * q);
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const double t = fmin(127.0, fmax(-127.0, rint(v[j] * sc)));
                v[j] = fma(-t, isc, v[j]);  // exact: removes the leading part
                const uint32_t byte = static_cast<uint32_t>(static_cast<int>(t)) & 0xFFu;
                if (j < 4)
                    lo |= byte << (8 * j);
                else
                    hi |= byte << (8 * (j - 4));
            }
            *reinterpret_cast<uint2*>(sl + (q - 1) * plane + row * K + k) = make_uint2(lo, hi);
        }
    }
}

template <int S>
__global__ void __launch_bounds__(kOzThreads, 1)
    gemm_ozaki_kernel(const __grid_constant__ CUtensorMap tmA4, const __grid_constant__ CUtensorMap tmA7,
                      const __grid_constant__ CUtensorMap tmW4, const __grid_constant__ CUtensorMap tmW7,
                      const double* __restrict__ sa, const double* __restrict__ sw, double* __restrict__ C,
                      int64_t M, int Nn, int K) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOzStages * kOzStage);
    uint64_t* empty = full + kOzStages;
    uint64_t* tfull = empty + kOzStages;  // MMA -> epilogue: a pass's accumulators are complete
    uint64_t* tempty = tfull + 1;         // epilogue -> MMA: drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tiles = Nn / kOzBN;
    const int64_t tiles = ((M + kOzBM - 1) / kOzBM) * n_tiles;
    const int kblocks = K / kOzBK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kOzStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, kOzEpi);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "r"(kOzTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        for (const CUtensorMap* m : {&tmA4, &tmA7, &tmW4, &tmW7})
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer: pass 1 slices 0..3, pass 2 slices 0..6 (3-D boxes)
            int s = 0;
            uint32_t ph = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int m0 = static_cast<int>((t / n_tiles) * kOzBM), n0 = static_cast<int>((t % n_tiles) * kOzBN);
                for (int pass = 0; pass < 2; ++pass) {
                    const uint32_t tx = (pass ? S : kOzPass1) * (kOzBM + kOzBN) * kOzBK;
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait(&empty[s], ph ^ 1u);
                        uint8_t* st = smem + s * kOzStage;
                        mbar_arrive_expect_tx(&full[s], tx);
                        tma_load_3d(st, pass ? &tmA7 : &tmA4, kb * kOzBK, m0, 0, &full[s]);
                        tma_load_3d(st + kOzTileA, pass ? &tmW7 : &tmW4, kb * kOzBK, n0, 0, &full[s]);
                        if (++s == kOzStages) s = 0, ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            int s = 0;
            uint32_t ph = 0, tph = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                for (int pass = 0; pass < 2; ++pass) {
                    mbar_wait(tempty, tph ^ 1u);  // the epilogue drained the accumulators
                    tph ^= 1u;
                    tc_fence_after();
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait(&full[s], ph);
                        tc_fence_after();
                        const uint32_t st = smem_u32(smem + s * kOzStage);
                        if (pass == 0) {
#pragma unroll
                            for (int d = 0; d < kOzPass1; ++d)
#pragma unroll
                                for (int pq = 0; pq <= d; ++pq)
                                    mma_i8(tmem_base + static_cast<uint32_t>(d * kOzBN),
                                           sw32_desc(st + pq * kOzBM * kOzBK),
                                           sw32_desc(st + kOzTileA + (d - pq) * kOzBN * kOzBK),
                                           (kb > 0 || pq > 0) ? 1u : 0u);
                        } else {
#pragma unroll
                            for (int d = kOzPass1; d < S; ++d)
#pragma unroll
                                for (int pq = 0; pq <= d; ++pq)
                                    mma_i8(tmem_base + static_cast<uint32_t>((d - kOzPass1) * kOzBN),
                                           sw32_desc(st + pq * kOzBM * kOzBK),
                                           sw32_desc(st + kOzTileA + (d - pq) * kOzBN * kOzBK),
                                           (kb > 0 || pq > 0) ? 1u : 0u);
                        }
                        mma_commit(&empty[s]);
                        if (++s == kOzStages) s = 0, ph ^= 1u;
                    }
                    mma_commit(tfull);
                }
            }
        }
    } else {  // ---- epilogue: C = sigma_A sigma_W sum_d 2^{-7(d+2)} acc_d, 64 columns per thread
        const int e = warp - 2, quarter = warp & 3, half = e >> 2;
        uint32_t tph = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            const int64_t row = (t / n_tiles) * kOzBM + quarter * 32 + lane;
            const int n0 = static_cast<int>((t % n_tiles) * kOzBN) + half * 64;
            const uint32_t tl = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + half * 64;
            double acc[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) acc[j] = 0.0;
            for (int pass = 0; pass < 2; ++pass) {
                mbar_wait(tfull, tph);
                tph ^= 1u;
                tc_fence_after();
                const int d0 = pass ? kOzPass1 : 0, nd = pass ? S - kOzPass1 : kOzPass1;
#pragma unroll 1
                for (int dd = nd - 1; dd >= 0; --dd) {
                    const double sc = ldexp(1.0, -7 * (d0 + dd + 2));
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t v[32];
                        TMEM_LD_32(tl + dd * kOzBN + c * 32, v);
                        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            acc[c * 32 + j] = fma(static_cast<double>(static_cast<int>(v[j])), sc, acc[c * 32 + j]);
                    }
                }
                tc_fence_before();
                mbar_arrive(tempty);
            }
            if (row < M) {
                const double ra = sa[row];
                double2* dst = reinterpret_cast<double2*>(C + row * Nn + n0);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int c = n0 + 2 * j;
                    dst[j] = make_double2(acc[2 * j] * ra * __ldg(sw + c), acc[2 * j + 1] * ra * __ldg(sw + c + 1));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kOzTmemCols)
                     : "memory");
    }
}

// W (fp64 real form) -> W_hi = rna_tf32(W), W_lo = W - W_hi (rounded to fp32)
__global__ void split_tf32_kernel(const double* __restrict__ w, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t count) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    const double v = w[i];
    const float h = __uint_as_float(to_tf32(static_cast<float>(v)));
    hi[i] = h;
    lo[i] = __uint_as_float(to_tf32(static_cast<float>(v - static_cast<double>(h))));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// [rows][cols] fp32 row-major, box = 32 columns (128 bytes) x 128 rows, 128-byte swizzle
bool make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
    const cuuint32_t box[2] = {kBK, 128};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// slices [S][rows][K] int8, box = 32 bytes x brows rows x S slices, 32-byte swizzle
bool make_slice_map(CUtensorMap* m, const int8_t* base, int64_t rows, int64_t K, int brows, int bslices,
                    int nslices) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows),
                                static_cast<cuuint64_t>(nslices)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(K) * static_cast<cuuint64_t>(rows)};
    const cuuint32_t box[3] = {kOzBK, static_cast<cuuint32_t>(brows), static_cast<cuuint32_t>(bslices)};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int ozaki_slices() { return kOzSMax; }

bool gemm_ozaki_supported(int Nn, int K) { return Nn % kOzBN == 0 && K % kOzBK == 0 && Nn >= kOzBN && K <= 8192; }
// (the slicing kernel also needs K % 8 == 0 and 32-byte aligned rows: K % 32 == 0 holds)

cudaError_t ozaki_slice(const double* a, int64_t rows, int K, int S, int8_t* slices, double* scale, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    const int64_t threads = rows * 32;
    const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
    if (S == 7)
        ozaki_slice_kernel<7><<<grid, 256, 0, st>>>(a, rows, K, slices, scale);
    else if (S == 8)
        ozaki_slice_kernel<8><<<grid, 256, 0, st>>>(a, rows, K, slices, scale);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

template <int S>
cudaError_t launch_ozaki_t(const int8_t* a_slices, const double* a_scale, const int8_t* w_slices, const double* w_scale,
                           double* C, int64_t M, int Nn, int K, int num_sms, cudaStream_t st) {
    CUtensorMap ma4, ma7, mw4, mw7;
    if (!make_slice_map(&ma4, a_slices, M, K, kOzBM, kOzPass1, S) || !make_slice_map(&ma7, a_slices, M, K, kOzBM, S, S) ||
        !make_slice_map(&mw4, w_slices, Nn, K, kOzBN, kOzPass1, S) || !make_slice_map(&mw7, w_slices, Nn, K, kOzBN, S, S))
        return cudaErrorInvalidValue;
    int per_sm = 0;
    cudaError_t e = prepare_launch(reinterpret_cast<const void*>(gemm_ozaki_kernel<S>), kOzThreads, kOzSmem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t tiles = ((M + kOzBM - 1) / kOzBM) * (Nn / kOzBN);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(tiles, num_sms));
    gemm_ozaki_kernel<S><<<grid, kOzThreads, kOzSmem, st>>>(ma4, ma7, mw4, mw7, a_scale, w_scale, C, M, Nn, K);
    return cudaGetLastError();
}

cudaError_t launch_gemm_ozaki(const int8_t* a_slices, const double* a_scale, const int8_t* w_slices,
                              const double* w_scale, double* C, int64_t M, int Nn, int K, int S, int num_sms,
                              cudaStream_t st) {
    if (M <= 0) return cudaSuccess;
    if (!gemm_ozaki_supported(Nn, K)) return cudaErrorInvalidValue;
    if (S == 7) return launch_ozaki_t<7>(a_slices, a_scale, w_slices, w_scale, C, M, Nn, K, num_sms, st);
    if (S == 8) return launch_ozaki_t<8>(a_slices, a_scale, w_slices, w_scale, C, M, Nn, K, num_sms, st);
    return cudaErrorInvalidValue;
}

bool gemm_tf32x3_supported(int Nn, int K) { return Nn % kBN == 0 && K % kBK == 0 && Nn >= kBN && K >= kBK; }

cudaError_t split_tf32(const double* w, float* hi, float* lo, int64_t count, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    split_tf32_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, st>>>(w, hi, lo, count);
    return cudaGetLastError();
}

cudaError_t launch_gemm_tf32x3(const float* A, const float* Whi, const float* Wlo, float* C, int64_t M, int Nn, int K,
                               int num_sms, cudaStream_t st) {
    if (M <= 0) return cudaSuccess;
    if (!gemm_tf32x3_supported(Nn, K)) return cudaErrorInvalidValue;
    CUtensorMap ma, mh, ml;
    if (!make_map(&ma, A, M, K) || !make_map(&mh, Whi, Nn, K) || !make_map(&ml, Wlo, Nn, K))
        return cudaErrorInvalidValue;
    int per_sm = 0;
    cudaError_t e = prepare_launch(reinterpret_cast<const void*>(gemm_tf32x3_kernel), kThreads, kSmemBytes, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t tiles = ((M + kBM - 1) / kBM) * (Nn / kBN);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(tiles, num_sms));
    gemm_tf32x3_kernel<<<grid, kThreads, kSmemBytes, st>>>(ma, mh, ml, C, M, Nn, K);
    return cudaGetLastError();
}

}  // namespace fcct
