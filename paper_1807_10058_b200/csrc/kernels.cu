// sm_100a kernels of the B200 FCC-DCT (arXiv 1807.10058).
//
//  * fast pipeline  — the paper's radix-2x2x2 factorization applied stage by
//                     stage to a tile of TB transform blocks resident in shared
//                     memory (TMA bulk load/store, in-place two-phase stages);
//  * direct GEMMs   — D x as a real-form GEMM on the FP64 tensor pipe (DMMA)
//                     or FFMA for fp32;
//  * table generation — D, D^{-1}, nodes and permutations built on the device.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "device.cuh"
#include "kernels.hpp"

namespace fcct {

// Per (device, kernel, dynamic smem) cache of the smem attribute and the
// occupancy query: both are host round trips that would otherwise cost
// microseconds on every launch (the latency of single-transform calls).
cudaError_t prepare_launch(const void* kern, int threads, int smem, int* per_sm) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int, int>, int> cache;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const auto key = std::make_tuple(dev, kern, threads, smem);
    {
        std::lock_guard<std::mutex> lock(mu);
        const auto it = cache.find(key);
        if (it != cache.end()) {
            if (per_sm) *per_sm = it->second;
            return cudaSuccess;
        }
    }
    // the attribute is raised to the device maximum once per kernel, so any
    // cached smem size stays launchable whatever was prepared last
    int max_optin = 0;
    e = cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    const int dyn_max = max_optin - static_cast<int>(fa.sharedSizeBytes);
    if (smem > dyn_max) return cudaErrorInvalidConfiguration;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = occ;
    if (per_sm) *per_sm = occ;
    return cudaSuccess;
}

namespace {
}  // namespace

using namespace dev;

__constant__ int c_group[24 * 9];  // S4 in the reference's BFS order (weyl_s4.cpp:54-92)

static cudaError_t upload_group() {
    static bool done = false;
    if (done) return cudaSuccess;
    // BFS closure of the generators; identical to plan.cpp's s4_group (kept
    // here as the device constant the generation kernels read).
    extern const int* host_group_table();
    cudaError_t e = cudaMemcpyToSymbol(c_group, host_group_table(), sizeof(int) * 24 * 9);
    if (e == cudaSuccess) done = true;
    return e;
}

// ===========================================================================
// Fast pipeline
// ===========================================================================
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kJ = 16;  // complex outputs a lane may hold per stage

template <typename R, int TB>
__device__ __forceinline__ void sparse_stage(const StageDesc& sd, C2<R>* data, int N1, int warp, int lane) {
    constexpr int RG = 32 / TB;
    const int rr = lane / TB, t = lane % TB;
    C2<R>* row_t = data + t * N1;
    const C2<R>* coef = static_cast<const C2<R>*>(sd.ecoef);
    C2<R> acc[kJ];
    int outpos[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
        const int g = warp + j * kWarps;
        outpos[j] = -1;
        acc[j].x = 0;
        acc[j].y = 0;
        if (g < sd.ngroups) {
            const int2 gi = __ldg(sd.ginfo + g);
            outpos[j] = __ldg(sd.grow + g * RG + rr);
            C2<R> a;
            a.x = 0;
            a.y = 0;
            for (int k = 0; k < gi.y; ++k) {
                const int e = gi.x + k * RG + rr;
                const int col = __ldg(sd.ecol + e);
                const C2<R> c = coef[e];
                cmac(a, c, row_t[col]);
            }
            acc[j] = a;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kJ; ++j)
        if (outpos[j] >= 0) row_t[outpos[j]] = acc[j];
    __syncthreads();
}

template <typename R, int TB>
__device__ __forceinline__ void mix8_stage(const StageDesc& sd, C2<R>* data, int N1, int warp, int lane) {
    constexpr int RG = 32 / TB;
    constexpr int kItems = kJ / 8;
    const int rr = lane / TB, t = lane % TB;
    C2<R>* row_t = data + t * N1;
    const C2<R>* Kall = static_cast<const C2<R>*>(sd.K);
    const int items = sd.nodes * sd.m3;
    C2<R> acc[kItems][8];
    int base[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const int item = (warp * RG + rr) + j * (kWarps * RG);
        base[j] = -1;
        if (item < items) {
            const int q = item / sd.m3, h = item - q * sd.m3;
            base[j] = q * 8 * sd.m3 + h;
            C2<R> x[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                int p = base[j] + g * sd.m3;
                if (sd.gather) p = __ldg(sd.gather + p);
                x[g] = row_t[p];
            }
            const C2<R>* Kq = Kall + q * 64;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                C2<R> a;
                a.x = 0;
                a.y = 0;
#pragma unroll
                for (int g = 0; g < 8; ++g) cmac(a, Kq[b * 8 + g], x[g]);
                acc[j][b] = a;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kItems; ++j)
        if (base[j] >= 0) {
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                int p = base[j] + b * sd.m3;
                if (sd.scatter) p = __ldg(sd.scatter + p);
                row_t[p] = acc[j][b];
            }
        }
    __syncthreads();
}

template <typename R, int TB>
__global__ void __launch_bounds__(kThreads, 1)
    pipeline_kernel(const __grid_constant__ PipelineDesc d, const C2<R>* __restrict__ in, C2<R>* __restrict__ out,
                    int64_t batch) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    C2<R>* data = reinterpret_cast<C2<R>*>(smem_raw + 128);
    // row stride: one padding element (fp64) or two (fp32) keep every row
    // 16-B aligned for the bulk copies and rotate the bank of consecutive rows
    const int N = d.N, N1 = d.N + (sizeof(C2<R>) == 8 ? 2 : 1);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t ntiles = (batch + TB - 1) / TB;
    const uint32_t row_bytes = static_cast<uint32_t>(N * sizeof(C2<R>));
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t t0 = tile * TB;
        const int nvalid = static_cast<int>(batch - t0 < TB ? batch - t0 : TB);
        if (threadIdx.x == 0) {
            tma_store_wait_read0();  // previous tile's stores have read the buffer
            mbar_arrive_expect_tx(bar, row_bytes * nvalid);
            for (int t = 0; t < nvalid; ++t) tma_load_1d(data + t * N1, in + (t0 + t) * N, row_bytes, bar);
            const int64_t nt = tile + gridDim.x;
            if (nt < ntiles) {
                const int64_t n0 = nt * TB;
                const int nv = static_cast<int>(batch - n0 < TB ? batch - n0 : TB);
                prefetch_l2_bulk(in + n0 * N, row_bytes * nv);
            }
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        for (int s = 0; s < d.nstages; ++s) {
            const StageDesc& sd = d.stage[s];
            if (sd.kind == 0)
                sparse_stage<R, TB>(sd, data, N1, warp, lane);
            else
                mix8_stage<R, TB>(sd, data, N1, warp, lane);
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int t = 0; t < nvalid; ++t) tma_store_1d(out + (t0 + t) * N, data + t * N1, row_bytes);
            tma_store_commit();
        }
    }
    if (threadIdx.x == 0) tma_store_wait0();
}

template <typename R, int TB>
cudaError_t launch_pipeline_t(const PipelineDesc& d, const void* in, void* out, int64_t batch, cudaStream_t st,
                              int num_sms) {
    const int smem = 128 + TB * (d.N + (sizeof(C2<R>) == 8 ? 2 : 1)) * static_cast<int>(sizeof(C2<R>));
    auto kern = pipeline_kernel<R, TB>;
    int per_sm = 0;
    cudaError_t e = prepare_launch(reinterpret_cast<const void*>(kern), kThreads, smem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t ntiles = (batch + TB - 1) / TB;
    const int64_t grid = std::min<int64_t>(ntiles, static_cast<int64_t>(per_sm) * num_sms);
    kern<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(d, static_cast<const C2<R>*>(in),
                                                               static_cast<C2<R>*>(out), batch);
    return cudaGetLastError();
}

}  // namespace

int pipeline_smem_bytes(const PipelineDesc& d, bool f32) {
    return 128 + d.tb * (d.N + (f32 ? 2 : 1)) * (f32 ? 8 : 16);
}

cudaError_t launch_pipeline(const PipelineDesc& d, bool f32, const void* in, void* out, int64_t batch,
                            cudaStream_t st, int num_sms) {
    if (batch <= 0) return cudaSuccess;
#define FCCT_PIPE(TBV)                                                                   \
    case TBV:                                                                            \
        return f32 ? launch_pipeline_t<float, TBV>(d, in, out, batch, st, num_sms)       \
                   : launch_pipeline_t<double, TBV>(d, in, out, batch, st, num_sms);
    switch (d.tb) {
        FCCT_PIPE(1)
        FCCT_PIPE(2)
        FCCT_PIPE(4)
        FCCT_PIPE(8)
        FCCT_PIPE(16)
        FCCT_PIPE(32)
        default:
            return cudaErrorInvalidValue;
    }
#undef FCCT_PIPE
}

// ===========================================================================
// Fast pipeline v2: every stage on the FP64 tensor pipe (DMMA m8n8k4), see
// tiling.hpp. smem X[t][slot][part], 16 blocks, row stride 2N + 8 doubles.
// Lane l: data row r = l/4 -> (t_sub = r/2, part = r%2), k = l%4.
//   A fragment (data, 8 x 4): X[t = 4 mt + t_sub][slot_k][part]
//   B fragment (table, 4 x 8): T[k][n = l/4], (Re, Im)
//   C fragment (8 x 8):        rows r, outputs n = 2k, 2k+1
// ===========================================================================
namespace {

// CTA shapes: <TB blocks, WARPS warps>; units per warp U = 64 / WARPS

// v with its sign bit xor-ed by `s` (0 or 0x80000000) on the integer pipe: a
// plain negation compiles to DADD, which competes with DMMA for the FP64 pipe.
__device__ __forceinline__ double xor_hi(double v, uint32_t s) {
    uint32_t lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
    asm("xor.b32 %0, %0, %1;" : "+r"(hi) : "r"(s));
    double o;
    asm("mov.b64 %0, {%1, %2};" : "=d"(o) : "r"(lo), "r"(hi));
    return o;
}

template <int MT>
__device__ __forceinline__ void store_unit(double* X, int stride, int t_sub, int part, int o0, int o1,
                                           const double (&acc)[MT][2]) {
    double* Xw = X + t_sub * stride + part;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        Xw[(4 * mt) * stride + 2 * o0] = acc[mt][0];
        Xw[(4 * mt) * stride + 2 * o1] = acc[mt][1];
    }
}

// Output sink of the last stage: global rows of the tile (natural layout).
struct TileOut {
    double* out;  // nullptr: write back into shared memory
    int64_t t0;
    int nvalid;
    int dimr;
};

template <int MT>
__device__ __forceinline__ void store_unit_global(const TileOut& to, int t_sub, int part, int o0, int o1,
                                                  const double (&acc)[MT][2]) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        const int t = 4 * mt + t_sub;
        if (t < to.nvalid) {
            double* row = to.out + (to.t0 + t) * to.dimr + part;
            row[2 * o0] = acc[mt][0];
            row[2 * o1] = acc[mt][1];
        }
    }
}

// Issued by thread 0 between the compute and the store phase of the last
// stage: the shared tile is free, so the next tile's bulk load overlaps the
// global stores of this one.
struct NextLoad {
    const double* in;
    uint64_t* bar;
    double* X;
    int stride;
    int shift;     // doubles added to odd rows (natural input layout)
    int dimr;
    int64_t tile;  // next tile index (< 0: none)
    int64_t batch;
    int64_t after; // tile after next (L2 prefetch), < 0: none
};

template <int TB>
__device__ __forceinline__ void issue_tile_load(const NextLoad& nl) {
    const uint32_t row_bytes = static_cast<uint32_t>(nl.dimr * sizeof(double));
    if (nl.tile >= 0) {
        const int64_t t0 = nl.tile * TB;
        const int nv = static_cast<int>(nl.batch - t0 < TB ? nl.batch - t0 : TB);
        mbar_arrive_expect_tx(nl.bar, row_bytes * nv);
        for (int t = 0; t < nv; ++t)
            tma_load_1d(nl.X + t * nl.stride + ((t & 1) ? nl.shift : 0), nl.in + (t0 + t) * nl.dimr, row_bytes, nl.bar);
    }
    if (nl.after >= 0) {
        const int64_t a0 = nl.after * TB;
        const int nv = static_cast<int>(nl.batch - a0 < TB ? nl.batch - a0 : TB);
        prefetch_l2_bulk(nl.in + a0 * nl.dimr, row_bytes * nv);
    }
}


constexpr int kRing = 4;  // table entries in flight per warp (cp.async ring depth)

// Stage barrier: the whole CTA, or only the warp group of one root child
// (named barrier 1 + group, WARPS/8 warps) when the stage keeps every group's
// data inside its own slot range.
template <int WARPS>
__device__ __forceinline__ void stage_sync(int group_scope, int warp) {
    if (group_scope) {
        constexpr int wpg = WARPS / 8;
        asm volatile("bar.sync %0, %1;\n" ::"r"(1 + warp / wpg), "r"(32 * wpg) : "memory");
    } else {
        __syncthreads();
    }
}

__device__ __forceinline__ double2 lds128(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ void sts128(uint32_t addr, double a, double b) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(a), "d"(b) : "memory");
}

// One stage of the fast pipeline on the FP64 tensor pipe.
//
// The complex stage operator is applied in real form: for an 8-block m-tile
// the DMMA A operand is an 8 x 4 fragment of real parts (a_re) or imaginary
// parts (a_im) of 4 input slots; the B operand is a 4 x 8 table tile T = Tr +
// i Ti; the C accumulators are the real and imaginary outputs:
//     C_re += a_re Tr - a_im Ti,   C_im += a_re Ti + a_im Tr
// (real tiles skip the Ti terms). One 16-byte shared load per lane returns a
// slot's (re, im) pair, i.e. both A fragments, and one 16-byte store writes an
// output's (re, im): every shared access moves unique data, conflict-free for
// the edge-coloured slot layouts (tiling.cpp), and no operand needs a sign flip
// or a part select except -Ti, one integer xor per table entry.
// Per-warp table-entry ring (kRing x 32 lanes x 16 B in shared memory).
struct RingCtx {
    double2* ring;
};

template <int TB, int WARPS>
__device__ __forceinline__ void stage2(const Stage2Dev& sd, double* X, int stride, int warp, int lane,
                                       const unsigned char* arena, const TileOut& to, const NextLoad& nl,
                                       unsigned long long* tcomp, RingCtx& rc, unsigned long long* wt = nullptr) {
    const long long wt0 = wt != nullptr ? clock64() : 0;
    const int r = lane >> 2, k = lane & 3;
    constexpr int kU2 = 64 / WARPS;  // units per warp
    constexpr int MT = TB / 8;       // m-tiles (8 blocks each)
    double2* ring = rc.ring;
    double acc[kU2][MT][2][2];       // [unit][m-tile][re, im][c0, c1]
    int o0[kU2], o1[kU2];
    const uint32_t xb = smem_u32(X) + static_cast<uint32_t>(r * stride) * 8u;  // block r of m-tile 0
    const uint32_t xl = xb + ((r & 1) ? sd.ld_shift : 0);                         // A-load base
    const uint32_t xsb = xb + ((r & 1) ? sd.st_shift : 0);                        // store base
    const uint32_t mstep = static_cast<uint32_t>(8 * stride) * 8u;             // next m-tile (8 blocks)
    const int* __restrict__ s_units = reinterpret_cast<const int*>(arena + sd.o_warp_units);
    const int* __restrict__ s_uout = reinterpret_cast<const int*>(arena + sd.o_u_out);
    int units[kU2];
#pragma unroll
    for (int j = 0; j < kU2; ++j) {
        units[j] = s_units[warp * kU2 + j];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) acc[j][mt][0][0] = acc[j][mt][0][1] = acc[j][mt][1][0] = acc[j][mt][1][1] = 0.0;
        o0[j] = o1[j] = -1;
    }
    if (sd.kind == 0) {
        // This warp's entry stream (tiling.hpp): (Re, Im) of the table tiles
        // stream through a kRing-deep per-warp cp.async ring (each lane copies
        // and reads back only its own 16 bytes: no warp synchronisation). Per
        // unit the real tiles come first, then the complex ones, so both
        // loops are branch-free (a predicated-off DMMA would still take its
        // tensor-pipe slot).
        const int* __restrict__ s_wbase = reinterpret_cast<const int*>(arena + sd.o_w_base);
        const int* __restrict__ s_wcount = reinterpret_cast<const int*>(arena + sd.o_w_count);
        const int* __restrict__ s_wccount = reinterpret_cast<const int*>(arena + sd.o_w_ccount);
        const int base = s_wbase[warp];
        const int total = s_wbase[warp + 1] - base;
        const int* __restrict__ psl = reinterpret_cast<const int*>(arena + sd.o_e_slots) + base * 4 + k;
        const uint32_t rs = smem_u32(ring + warp * kRing * 32 + lane);
        const double2* __restrict__ pri = sd.e_ri + static_cast<size_t>(base) * 32 + lane;
#pragma unroll
        for (int q = 0; q < kRing - 1; ++q) {
            if (q < total)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(rs + q * 512), "l"(pri + q * 32)
                             : "memory");
            cp_async_commit();
        }
        // issues entry f + kRing - 1, loads entry f's A fragments and table tile
        auto next = [&](int f, double2 (&a)[MT]) -> double2 {
            const int q = f + kRing - 1;
            if (q < total)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(rs + (q & (kRing - 1)) * 512),
                             "l"(pri + q * 32)
                             : "memory");
            cp_async_commit();
            const uint32_t xa = xl + static_cast<uint32_t>(psl[f * 4] & ~(1 << 30)) * 16u;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) a[mt] = lds128(xa + mt * mstep);
            cp_async_wait<kRing - 1>();
            return lds128(rs + (f & (kRing - 1)) * 512);
        };
        int f = 0;
#pragma unroll
        for (int j = 0; j < kU2; ++j) {
            const int nc = s_wccount[warp * kU2 + j];
            const int nr = s_wcount[warp * kU2 + j] - nc;
            for (int e = 0; e < nr; ++e, ++f) {
                double2 a[MT];
                const double2 t = next(f, a);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    dmma884(acc[j][mt][0][0], acc[j][mt][0][1], a[mt].x, t.x);
                    dmma884(acc[j][mt][1][0], acc[j][mt][1][1], a[mt].y, t.x);
                }
            }
            for (int e = 0; e < nc; ++e, ++f) {
                double2 a[MT];
                const double2 t = next(f, a);
                const double nti = xor_hi(t.y, 0x80000000u);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    dmma884(acc[j][mt][0][0], acc[j][mt][0][1], a[mt].x, t.x);
                    dmma884(acc[j][mt][1][0], acc[j][mt][1][1], a[mt].y, t.x);
                    dmma884(acc[j][mt][0][0], acc[j][mt][0][1], a[mt].y, nti);
                    dmma884(acc[j][mt][1][0], acc[j][mt][1][1], a[mt].x, t.y);
                }
            }
            if (units[j] >= 0) {
                o0[j] = s_uout[units[j] * 8 + 2 * k];
                o1[j] = s_uout[units[j] * 8 + 2 * k + 1];
            }
        }
        cp_async_wait<0>();
    } else {
        // 8x8 complex K per unit (B fragment: K[b = n][g = 4 kt + k]); the next
        // unit's K fragments and input slots are prefetched into registers
        const int* __restrict__ s_unode = reinterpret_cast<const int*>(arena + sd.o_u_node);
        const int* __restrict__ s_uin = reinterpret_cast<const int*>(arena + sd.o_u_in);
        const bool k_smem = sd.o_K >= 0;
        const double2* __restrict__ Ks = reinterpret_cast<const double2*>(arena + (k_smem ? sd.o_K : 0));
        const int kidx = r * 8 + k;  // K[b = r][g = k] (+ 4 kt)
#pragma unroll
        for (int j = 0; j < kU2; ++j) {
            if (units[j] < 0) continue;
            const int u = units[j];
            const int node = s_unode[u] * 64 + kidx;
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) {
                const int slot = s_uin[u * 8 + kt * 4 + k];
                const double2 kf = k_smem ? Ks[node + kt * 4] : __ldg(sd.K + node + kt * 4);
                const uint32_t xa = xl + static_cast<uint32_t>(slot) * 16u;
                double2 a[MT];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) a[mt] = lds128(xa + mt * mstep);
                const double nki = xor_hi(kf.y, 0x80000000u);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    dmma884(acc[j][mt][0][0], acc[j][mt][0][1], a[mt].x, kf.x);
                    dmma884(acc[j][mt][1][0], acc[j][mt][1][1], a[mt].y, kf.x);
                    dmma884(acc[j][mt][0][0], acc[j][mt][0][1], a[mt].y, nki);
                    dmma884(acc[j][mt][1][0], acc[j][mt][1][1], a[mt].x, kf.y);
                }
            }
            o0[j] = s_uout[u * 8 + 2 * k];
            o1[j] = s_uout[u * 8 + 2 * k + 1];
        }
    }
    if (wt != nullptr && lane == 0)
        atomicAdd(wt + warp, static_cast<unsigned long long>(clock64() - wt0));
    stage_sync<WARPS>(sd.sync_mid, warp);
    if (tcomp != nullptr) *tcomp = clock64();
    if (to.out != nullptr) {
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            issue_tile_load<TB>(nl);
        }
#pragma unroll
        for (int j = 0; j < kU2; ++j)
            if (o0[j] >= 0) {
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const int t = 8 * mt + r;
                    if (t < to.nvalid) {
                        double2* row = reinterpret_cast<double2*>(to.out + (to.t0 + t) * to.dimr);
                        row[o0[j]] = make_double2(acc[j][mt][0][0], acc[j][mt][1][0]);
                        row[o1[j]] = make_double2(acc[j][mt][0][1], acc[j][mt][1][1]);
                    }
                }
            }
        return;
    }
#pragma unroll
    for (int j = 0; j < kU2; ++j)
        if (o0[j] >= 0) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                sts128(xsb + mt * mstep + static_cast<uint32_t>(o0[j]) * 16u, acc[j][mt][0][0], acc[j][mt][1][0]);
                sts128(xsb + mt * mstep + static_cast<uint32_t>(o1[j]) * 16u, acc[j][mt][0][1], acc[j][mt][1][1]);
            }
        }
    stage_sync<WARPS>(sd.sync_end, warp);
}

template <int TB, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 512 / (WARPS * 32))
    pipeline2_kernel(const __grid_constant__ Pipeline2Desc d, const void* __restrict__ in_raw, void* __restrict__ out_raw,
                     int64_t batch) {
    const double* __restrict__ in = static_cast<const double*>(in_raw);
    double* __restrict__ out = static_cast<double*>(out_raw);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    double* X = reinterpret_cast<double*>(smem_raw + 128);
    const int stride = d.stride;
    unsigned char* arena = smem_raw + 128 + static_cast<size_t>(TB) * stride * sizeof(double);
    double2* ring = d.ring ? reinterpret_cast<double2*>(arena + d.arena_bytes) : nullptr;
    RingCtx rc{ring};
    const int dimr = 2 * d.N;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t ntiles = (batch + TB - 1) / TB;
    const uint32_t row_bytes = static_cast<uint32_t>(dimr * sizeof(double));
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    {  // per-CTA copy of the small stage tables (identical for every tile)
        uint4* dst = reinterpret_cast<uint4*>(arena);
        for (int i = threadIdx.x; i < d.arena_bytes / 16; i += blockDim.x) dst[i] = __ldg(d.arena + i);
    }
    __syncthreads();
    uint32_t phase = 0;
    if (d.direct_store && !d.real_in && !d.real_out) {
        if (threadIdx.x == 0 && static_cast<int64_t>(blockIdx.x) < ntiles) {
            const int64_t nt = blockIdx.x + gridDim.x;
            issue_tile_load<TB>(NextLoad{in, bar, X, stride, d.shift_in, dimr, static_cast<int64_t>(blockIdx.x), batch,
                                     nt < ntiles ? nt : -1});
        }
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int64_t t0 = tile * TB;
            const int nvalid = static_cast<int>(batch - t0 < TB ? batch - t0 : TB);
            mbar_wait(bar, phase);
            phase ^= 1;
            const TileOut none{nullptr, 0, 0, 0};
            const int64_t nt = tile + gridDim.x, nn = tile + 2 * static_cast<int64_t>(gridDim.x);
            const NextLoad nl{in, bar, X, stride, d.shift_in, dimr, nt < ntiles ? nt : -1, batch, nn < ntiles ? nn : -1};
            for (int s = 0; s + 1 < d.nstages; ++s) stage2<TB, WARPS>(d.st[s], X, stride, warp, lane, arena, none, nl, nullptr, rc);
            stage2<TB, WARPS>(d.st[d.nstages - 1], X, stride, warp, lane, arena, TileOut{out, t0, nvalid, dimr}, nl,
                              nullptr, rc);
        }
        return;
    }
    const TileOut none{nullptr, 0, 0, 0};
    const NextLoad nonl{in, bar, X, stride, d.shift_in, dimr, -1, batch, -1};
    const bool timing = d.timing != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    __shared__ unsigned long long tacc[kMaxStages + 2];
    if (threadIdx.x < kMaxStages + 2) tacc[threadIdx.x] = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t t0 = tile * TB;
        const int nvalid = static_cast<int>(batch - t0 < TB ? batch - t0 : TB);
        long long c0 = timing ? clock64() : 0;
        if (d.real_in) {
            // z_transform fused into the load: real rows -> (re, 0) pairs of the fp64 tile
            if (threadIdx.x == 0) tma_store_wait_read0();  // the previous tile's bulk store has read X
            __syncthreads();
            if (d.io_f32) {
                const int per_row = d.N / 4;
                const float4* src = reinterpret_cast<const float4*>(in_raw) + t0 * per_row;
                for (int i = threadIdx.x; i < nvalid * per_row; i += blockDim.x) {
                    const int t = i / per_row, q = i - t * per_row;
                    const float4 v = __ldg(src + static_cast<int64_t>(t) * per_row + q);
                    double2* xr = reinterpret_cast<double2*>(X + t * stride + ((t & 1) ? d.shift_in : 0)) + 4 * q;
                    xr[0] = make_double2(v.x, 0.0);
                    xr[1] = make_double2(v.y, 0.0);
                    xr[2] = make_double2(v.z, 0.0);
                    xr[3] = make_double2(v.w, 0.0);
                }
            } else {
                const int per_row = d.N / 2;
                const double2* src = reinterpret_cast<const double2*>(in_raw) + t0 * per_row;
                for (int i = threadIdx.x; i < nvalid * per_row; i += blockDim.x) {
                    const int t = i / per_row, q = i - t * per_row;
                    const double2 v = __ldg(src + static_cast<int64_t>(t) * per_row + q);
                    double2* xr = reinterpret_cast<double2*>(X + t * stride + ((t & 1) ? d.shift_in : 0)) + 2 * q;
                    xr[0] = make_double2(v.x, 0.0);
                    xr[1] = make_double2(v.y, 0.0);
                }
            }
            if (threadIdx.x == 0) {
                const int64_t nt = tile + gridDim.x;
                if (nt < ntiles) {
                    const int64_t n0 = nt * TB;
                    const int nv = static_cast<int>(batch - n0 < TB ? batch - n0 : TB);
                    const size_t eb = d.io_f32 ? sizeof(float) : sizeof(double);
                    prefetch_l2_bulk(static_cast<const char*>(in_raw) + n0 * d.N * eb,
                                     static_cast<uint32_t>(nv * d.N * eb));
                }
            }
            __syncthreads();
        } else if (d.io_f32) {
            // complex64 rows -> fp64 tile (coalesced float4 loads, 2 points each)
            const float4* src = reinterpret_cast<const float4*>(in_raw) + t0 * (d.N / 2);
            const int per_row = d.N / 2;
            for (int i = threadIdx.x; i < nvalid * per_row; i += blockDim.x) {
                const int t = i / per_row, q = i - t * per_row;
                const float4 v = __ldg(src + static_cast<int64_t>(t) * per_row + q);
                double2* xr = reinterpret_cast<double2*>(X + t * stride + ((t & 1) ? d.shift_in : 0)) + 2 * q;
                xr[0] = make_double2(v.x, v.y);
                xr[1] = make_double2(v.z, v.w);
            }
            if (threadIdx.x == 0) {
                const int64_t nt = tile + gridDim.x;
                if (nt < ntiles) {
                    const int64_t n0 = nt * TB;
                    const int nv = static_cast<int>(batch - n0 < TB ? batch - n0 : TB);
                    prefetch_l2_bulk(reinterpret_cast<const float*>(in_raw) + n0 * dimr,
                                     static_cast<uint32_t>(nv * dimr * sizeof(float)));
                }
            }
            __syncthreads();
        } else {
            if (threadIdx.x == 0) {
                // the previous tile left row by row (one bulk group per row):
                // each row of this tile is loaded as soon as the copy engine
                // has read that row out, so the stores and loads overlap
                const int nv = nvalid;
                mbar_arrive_expect_tx(bar, row_bytes * nv);
#pragma unroll
                for (int t = 0; t < TB; ++t) {
                    if (t >= nv) break;
                    tma_store_wait_read_n(TB - 1 - t);
                    tma_load_1d(X + t * stride + ((t & 1) ? d.shift_in : 0), in + (t0 + t) * d.row_in, row_bytes, bar);
                }
                const int64_t na = tile + gridDim.x;
                if (na < ntiles) {
                    const int64_t a0 = na * TB;
                    const int nva = static_cast<int>(batch - a0 < TB ? batch - a0 : TB);
                    if (d.row_in == dimr)
                        prefetch_l2_bulk(in + a0 * dimr, row_bytes * nva);
                    else
                        for (int t = 0; t < nva; ++t) prefetch_l2_bulk(in + (a0 + t) * d.row_in, row_bytes);
                }
            }
            mbar_wait(bar, phase);
            phase ^= 1;
        }
        if (timing) {
            const long long c1 = clock64();
            tacc[0] += c1 - c0;
            c0 = c1;
        }
        for (int s = 0; s < d.nstages; ++s) {
            __shared__ unsigned long long tmid;
            if ((d.stage_mask >> s) & 1)
                stage2<TB, WARPS>(d.st[s], X, stride, warp, lane, arena, none, nonl, timing ? &tmid : nullptr, rc,
                                  (d.timing != nullptr && blockIdx.x == 0) ? d.timing + kMaxStages + 2 + s * 16 : nullptr);
            if (timing) {
                const long long c1 = clock64();
                tacc[1 + s] += tmid - c0;              // compute phase (to the mid barrier)
                tacc[1 + kMaxStages / 2 + s] += c1 - tmid;  // store phase + final barrier
                c0 = c1;
            }
        }
        if (d.real_out) {
            // grid_from_signal fused into the store: real parts only
            if (d.io_f32) {
                const int per_row = d.N / 4;
                float4* dst = reinterpret_cast<float4*>(out_raw) + t0 * per_row;
                for (int i = threadIdx.x; i < nvalid * per_row; i += blockDim.x) {
                    const int t = i / per_row, q = i - t * per_row;
                    const double* xr = X + t * stride + ((t & 1) ? d.shift_out : 0) + 8 * q;
                    dst[static_cast<int64_t>(t) * per_row + q] =
                        make_float4(static_cast<float>(xr[0]), static_cast<float>(xr[2]), static_cast<float>(xr[4]),
                                    static_cast<float>(xr[6]));
                }
            } else {
                const int per_row = d.N / 2;
                double2* dst = reinterpret_cast<double2*>(out_raw) + t0 * per_row;
                for (int i = threadIdx.x; i < nvalid * per_row; i += blockDim.x) {
                    const int t = i / per_row, q = i - t * per_row;
                    const double* xr = X + t * stride + ((t & 1) ? d.shift_out : 0) + 4 * q;
                    dst[static_cast<int64_t>(t) * per_row + q] = make_double2(xr[0], xr[2]);
                }
            }
            __syncthreads();
            continue;
        }
        if (d.io_f32) {
            float4* dst = reinterpret_cast<float4*>(out_raw) + t0 * (d.N / 2);
            const int per_row = d.N / 2;
            for (int i = threadIdx.x; i < nvalid * per_row; i += blockDim.x) {
                const int t = i / per_row, q = i - t * per_row;
                const double2* xr = reinterpret_cast<const double2*>(X + t * stride + ((t & 1) ? d.shift_out : 0)) + 2 * q;
                const double2 a = xr[0], b = xr[1];
                dst[static_cast<int64_t>(t) * per_row + q] = make_float4(static_cast<float>(a.x), static_cast<float>(a.y),
                                                                       static_cast<float>(b.x), static_cast<float>(b.y));
            }
            __syncthreads();
            continue;
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            // one bulk group per row, and always TB groups (empty ones for a
            // ragged last tile) so the next tile's per-row waits line up
            for (int t = 0; t < TB; ++t) {
                if (t < nvalid)
                    tma_store_1d(out + (t0 + t) * d.row_out, X + t * stride + ((t & 1) ? d.shift_out : 0), row_bytes);
                tma_store_commit();
            }
        }
    }
    if (threadIdx.x == 0) tma_store_wait0();
    if (timing)
        for (int i = 0; i < kMaxStages + 2; ++i) d.timing[i] = tacc[i];
}

}  // namespace

template <int TB, int WARPS>
cudaError_t launch_pipeline2_t(const Pipeline2Desc& d, const void* in, void* out, int64_t batch, cudaStream_t st,
                               int num_sms) {
    const int smem = 128 + TB * d.stride * static_cast<int>(sizeof(double)) + d.arena_bytes +
                     (d.ring ? WARPS * kRing * 32 * static_cast<int>(sizeof(double2)) : 0);
    auto kern = pipeline2_kernel<TB, WARPS>;
    int per_sm = 0;
    cudaError_t e = prepare_launch(reinterpret_cast<const void*>(kern), WARPS * 32, smem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t ntiles = (batch + TB - 1) / TB;
    const int64_t grid = std::min<int64_t>(ntiles, static_cast<int64_t>(per_sm) * num_sms);
    kern<<<static_cast<unsigned>(grid), WARPS * 32, smem, st>>>(d, in, out, batch);
    return cudaGetLastError();
}

cudaError_t launch_pipeline2(const Pipeline2Desc& d, const void* in, void* out, int64_t batch, cudaStream_t st,
                             int num_sms) {
    if (batch <= 0) return cudaSuccess;
    if (d.tb == 16 && d.warps == 16) return launch_pipeline2_t<16, 16>(d, in, out, batch, st, num_sms);
    if (d.tb == 8 && d.warps == 8) return launch_pipeline2_t<8, 8>(d, in, out, batch, st, num_sms);
    return cudaErrorInvalidValue;
}

namespace {

template <typename R>
__global__ void complexify_kernel(const R* __restrict__ in, C2<R>* __restrict__ out, int64_t count) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        C2<R> v;
        v.x = __ldg(in + i);
        v.y = 0;
        out[i] = v;
    }
}

template <typename R>
__global__ void real_part_kernel(const C2<R>* __restrict__ in, R* __restrict__ out, int64_t count) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = in[i].x;
}

unsigned elementwise_grid(int64_t count) {
    const int64_t blocks = (count + 255) / 256;
    return static_cast<unsigned>(blocks < 148 * 32 ? (blocks > 0 ? blocks : 1) : 148 * 32);
}

}  // namespace

cudaError_t launch_complexify(const void* in_real, void* out_cplx, int64_t count, bool f32, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    if (f32)
        complexify_kernel<float><<<elementwise_grid(count), 256, 0, st>>>(static_cast<const float*>(in_real),
                                                                          static_cast<C2<float>*>(out_cplx), count);
    else
        complexify_kernel<double><<<elementwise_grid(count), 256, 0, st>>>(static_cast<const double*>(in_real),
                                                                           static_cast<C2<double>*>(out_cplx), count);
    return cudaGetLastError();
}

cudaError_t launch_real_part(const void* in_cplx, void* out_real, int64_t count, bool f32, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    if (f32)
        real_part_kernel<float><<<elementwise_grid(count), 256, 0, st>>>(static_cast<const C2<float>*>(in_cplx),
                                                                         static_cast<float*>(out_real), count);
    else
        real_part_kernel<double><<<elementwise_grid(count), 256, 0, st>>>(static_cast<const C2<double>*>(in_cplx),
                                                                          static_cast<double*>(out_real), count);
    return cudaGetLastError();
}

// ===========================================================================
// Two-level executor: root pass (SIMT FP64), children on pipeline2
// ===========================================================================
namespace {

__device__ __forceinline__ double2 load_point(int mode, const void* __restrict__ src, int64_t i) {
    if (mode == 0) return __ldg(static_cast<const double2*>(src) + i);
    if (mode == 1) {
        const float2 f = __ldg(static_cast<const float2*>(src) + i);
        return make_double2(f.x, f.y);
    }
    if (mode == 2) return make_double2(__ldg(static_cast<const double*>(src) + i), 0.0);
    return make_double2(__ldg(static_cast<const float*>(src) + i), 0.0);
}

__device__ __forceinline__ void store_point(int mode, void* __restrict__ dst, int64_t i, double2 v) {
    if (mode == 0)
        static_cast<double2*>(dst)[i] = v;
    else if (mode == 1)
        static_cast<float2*>(dst)[i] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
    else if (mode == 2)
        static_cast<double*>(dst)[i] = v.x;
    else
        static_cast<float*>(dst)[i] = static_cast<float>(v.x);
}

__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}

constexpr int kRootBlk = 3;  // blocks per CTA pass: each table entry serves kRootBlk blocks

// Sparse rows of one ELL group for the kRootBlk blocks held in shared memory.
__device__ __forceinline__ void root_rows(const RootDesc& d, int g, int h, const double2* xs, double2 (&acc)[kRootBlk]) {
    // entries are fetched 8 at a time into registers before any is used, so
    // eight table loads (L2) are in flight per thread
    const int e_end = d.ell_off[g + 1];
    for (int base = d.ell_off[g] + h; base < e_end; base += 8 * d.m3) {
        int c[8];
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = base + u * d.m3;
            c[u] = idx < e_end ? __ldg(d.col + idx) : 0;
            v[u] = idx < e_end ? __ldg(d.val + idx) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int b = 0; b < kRootBlk; ++b) cfma(acc[b], v[u], xs[(b << d.lgN) + c[u]]);
    }
}

__global__ void __launch_bounds__(512, 1)
    root_forward_kernel(const RootDesc d, const void* __restrict__ x, int in_mode, double2* __restrict__ z,
                        int64_t batch) {
    extern __shared__ double2 xs[];  // [kRootBlk][N]
    __shared__ double2 Ks[64];
    __shared__ uint64_t bar;
    if (threadIdx.x < 64) Ks[threadIdx.x] = d.K[threadIdx.x];
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    uint32_t phase = 0;
    const int64_t step = static_cast<int64_t>(gridDim.x) * kRootBlk;
    for (int64_t b0 = static_cast<int64_t>(blockIdx.x) * kRootBlk; b0 < batch; b0 += step) {
        const int nb = static_cast<int>(batch - b0 < kRootBlk ? batch - b0 : kRootBlk);
        __syncthreads();
        if (in_mode == 0) {  // complex128 blocks are contiguous: one bulk copy, next pass prefetched into L2
            if (threadIdx.x == 0) {
                const uint32_t bytes = static_cast<uint32_t>(nb) << (d.lgN + 4);
                mbar_arrive_expect_tx(&bar, bytes);
                tma_load_1d(xs, static_cast<const double2*>(x) + (b0 << d.lgN), bytes, &bar);
                const int64_t nx = b0 + step;
                if (nx < batch) {
                    const int nn = static_cast<int>(batch - nx < kRootBlk ? batch - nx : kRootBlk);
                    prefetch_l2_bulk(static_cast<const double2*>(x) + (nx << d.lgN), static_cast<uint32_t>(nn) << (d.lgN + 4));
                }
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
        } else {
            if (threadIdx.x == 0) {  // the next pass's samples into L2
                const int64_t nx = b0 + step;
                const int esz = in_mode == 1 ? 8 : (in_mode == 2 ? 8 : 4);
                if (nx < batch) {
                    const int nn = static_cast<int>(batch - nx < kRootBlk ? batch - nx : kRootBlk);
                    prefetch_l2_bulk(static_cast<const char*>(x) + (nx << d.lgN) * esz,
                                     static_cast<uint32_t>(nn) * (static_cast<uint32_t>(esz) << d.lgN));
                }
            }
#pragma unroll 8
            for (int i = threadIdx.x; i < (nb << d.lgN); i += blockDim.x) xs[i] = load_point(in_mode, x, (b0 << d.lgN) + i);
        }
        __syncthreads();
        for (int h = threadIdx.x; h < d.m3; h += blockDim.x) {
            double2 t[kRootBlk][8];
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                double2 acc[kRootBlk];
#pragma unroll
                for (int b = 0; b < kRootBlk; ++b) acc[b] = make_double2(0.0, 0.0);
                root_rows(d, g, h, xs, acc);
#pragma unroll
                for (int b = 0; b < kRootBlk; ++b) t[b][g] = acc[b];
            }
            // K-mix: z[c m3 + h] = sum_g K[c][g] t[g]
#pragma unroll
            for (int b = 0; b < kRootBlk; ++b)
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (b >= nb) break;
                    double2 s = make_double2(0.0, 0.0);
#pragma unroll
                    for (int g = 0; g < 8; ++g) cfma(s, Ks[c * 8 + g], t[b][g]);
                    z[((b0 + b) << d.lgN) + c * d.m3 + h] = s;
                }
        }
    }
}

__global__ void __launch_bounds__(512, 1)
    root_inverse_kernel(const RootDesc d, const double2* __restrict__ z, void* __restrict__ y, int out_mode,
                        int64_t batch) {
    extern __shared__ double2 xs[];  // [kRootBlk][N]
    __shared__ double2 Ks[64];
    __shared__ uint64_t bar;
    if (threadIdx.x < 64) Ks[threadIdx.x] = d.K[threadIdx.x];
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    uint32_t phase = 0;
    const int64_t step = static_cast<int64_t>(gridDim.x) * kRootBlk;
    for (int64_t b0 = static_cast<int64_t>(blockIdx.x) * kRootBlk; b0 < batch; b0 += step) {
        const int nb = static_cast<int>(batch - b0 < kRootBlk ? batch - b0 : kRootBlk);
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t bytes = static_cast<uint32_t>(nb) << (d.lgN + 4);
            mbar_arrive_expect_tx(&bar, bytes);
            tma_load_1d(xs, z + (b0 << d.lgN), bytes, &bar);
            const int64_t nx = b0 + step;
            if (nx < batch) {
                const int nn = static_cast<int>(batch - nx < kRootBlk ? batch - nx : kRootBlk);
                prefetch_l2_bulk(z + (nx << d.lgN), static_cast<uint32_t>(nn) << (d.lgN + 4));
            }
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        __syncthreads();
        // K^{-1} unmix in place: every thread owns positions g m3 + h of its h
        for (int h = threadIdx.x; h < d.m3; h += blockDim.x)
#pragma unroll 1
            for (int b = 0; b < nb; ++b) {
                double2 u[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) u[c] = xs[(b << d.lgN) + c * d.m3 + h];
#pragma unroll 1
                for (int g = 0; g < 8; ++g) {  // not unrolled: the 64 K values would be hoisted into registers
                    double2 s = make_double2(0.0, 0.0);
#pragma unroll
                    for (int c = 0; c < 8; ++c) cfma(s, Ks[g * 8 + c], u[c]);
                    xs[(b << d.lgN) + g * d.m3 + h] = s;
                }
            }
        __syncthreads();
        // B^{-1}: natural rows j m3 + h
        for (int h = threadIdx.x; h < d.m3; h += blockDim.x)
#pragma unroll 1
            for (int j = 0; j < 8; ++j) {
                double2 acc[kRootBlk];
#pragma unroll
                for (int b = 0; b < kRootBlk; ++b) acc[b] = make_double2(0.0, 0.0);
                root_rows(d, j, h, xs, acc);
#pragma unroll
                for (int b = 0; b < kRootBlk; ++b)
                    if (b < nb) store_point(out_mode, y, ((b0 + b) << d.lgN) + j * d.m3 + h, acc[b]);
            }
    }
}

__global__ void child_to_natural_kernel(const RootDesc d, const double2* __restrict__ src, void* __restrict__ dst,
                                        int out_mode, int64_t total) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t b = i >> d.lgN;
        const int P = static_cast<int>(i & (d.N - 1));
        store_point(out_mode, dst, i, __ldg(src + (b << d.lgN) + __ldg(d.pinv + P)));
    }
}

__global__ void natural_to_child_kernel(const RootDesc d, const void* __restrict__ src, int in_mode,
                                        double2* __restrict__ dst, int64_t total) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t b = i >> d.lgN;
        const int q = static_cast<int>(i & (d.N - 1));
        dst[i] = load_point(in_mode, src, (b << d.lgN) + __ldg(d.perm + q));
    }
}

unsigned root_grid(int64_t batch, int num_sms) {
    const int64_t passes = (batch + kRootBlk - 1) / kRootBlk;
    return static_cast<unsigned>(std::min<int64_t>(passes, num_sms));
}

}  // namespace

cudaError_t launch_root_forward(const RootDesc& d, const void* x, int in_mode, double* z, int64_t batch,
                                cudaStream_t st, int num_sms) {
    if (batch <= 0) return cudaSuccess;
    const int smem = kRootBlk * d.N * static_cast<int>(sizeof(double2));
    cudaError_t e = prepare_launch(reinterpret_cast<const void*>(root_forward_kernel), 512, smem, nullptr);
    if (e != cudaSuccess) return e;
    root_forward_kernel<<<root_grid(batch, num_sms), 512, smem, st>>>(d, x, in_mode, reinterpret_cast<double2*>(z),
                                                                      batch);
    return cudaGetLastError();
}

cudaError_t launch_root_inverse(const RootDesc& d, const double* z, void* y, int out_mode, int64_t batch,
                                cudaStream_t st, int num_sms) {
    if (batch <= 0) return cudaSuccess;
    const int smem = kRootBlk * d.N * static_cast<int>(sizeof(double2));
    cudaError_t e = prepare_launch(reinterpret_cast<const void*>(root_inverse_kernel), 512, smem, nullptr);
    if (e != cudaSuccess) return e;
    root_inverse_kernel<<<root_grid(batch, num_sms), 512, smem, st>>>(d, reinterpret_cast<const double2*>(z), y,
                                                                      out_mode, batch);
    return cudaGetLastError();
}

cudaError_t launch_child_to_natural(const RootDesc& d, const double* src, void* dst, int out_mode, int64_t batch,
                                    cudaStream_t st) {
    const int64_t total = batch << d.lgN;
    if (total <= 0) return cudaSuccess;
    child_to_natural_kernel<<<elementwise_grid(total), 256, 0, st>>>(d, reinterpret_cast<const double2*>(src), dst,
                                                                     out_mode, total);
    return cudaGetLastError();
}

cudaError_t launch_natural_to_child(const RootDesc& d, const void* src, int in_mode, double* dst, int64_t batch,
                                    cudaStream_t st) {
    const int64_t total = batch << d.lgN;
    if (total <= 0) return cudaSuccess;
    natural_to_child_kernel<<<elementwise_grid(total), 256, 0, st>>>(d, src, in_mode, reinterpret_cast<double2*>(dst),
                                                                     total);
    return cudaGetLastError();
}

// ===========================================================================
// Global-memory multi-pass pipeline (one launch per stage)
// ===========================================================================
namespace {

template <typename R>
__global__ void gstage_sparse_kernel(const GStage st, int N, const C2<R>* __restrict__ x, C2<R>* __restrict__ y) {
    const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (r >= N) return;
    const int64_t b = blockIdx.y;
    const C2<R>* xb = x + b * N;
    const C2<R>* coef = static_cast<const C2<R>*>(st.coef);
    C2<R> acc;
    acc.x = 0;
    acc.y = 0;
    const int64_t sl = r >> 5;
    const int64_t e0 = __ldg(st.rowptr + sl) + (r & 31), e1 = __ldg(st.rowptr + sl + 1);
#pragma unroll 4
    for (int64_t e = e0; e < e1; e += 32) cmac(acc, coef[e], xb[__ldg(st.col + e)]);
    const int64_t o = __ldg(st.out_row + r);
    y[b * N + o] = acc;
}

template <typename R>
__global__ void gstage_mix_kernel(const GStage st, int N, const C2<R>* __restrict__ x, C2<R>* __restrict__ y) {
    const int64_t item = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (item >= static_cast<int64_t>(st.nodes) * st.m3) return;
    const int64_t b = blockIdx.y;
    const int q = static_cast<int>(item / st.m3), h = static_cast<int>(item % st.m3);
    const int64_t base = static_cast<int64_t>(q) * 8 * st.m3 + h;
    const C2<R>* Kq = static_cast<const C2<R>*>(st.K) + static_cast<int64_t>(q) * 64;
    C2<R> in[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        int64_t p = base + static_cast<int64_t>(g) * st.m3;
        if (st.gather) p = __ldg(st.gather + p);
        in[g] = x[b * N + p];
    }
#pragma unroll
    for (int bo = 0; bo < 8; ++bo) {
        C2<R> acc;
        acc.x = 0;
        acc.y = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g) cmac(acc, Kq[bo * 8 + g], in[g]);
        int64_t p = base + static_cast<int64_t>(bo) * st.m3;
        if (st.scatter) p = __ldg(st.scatter + p);
        y[b * N + p] = acc;
    }
}

template <typename R>
cudaError_t launch_global_t(const GlobalPipelineDesc& d, const void* in, void* out, void* s0, void* s1, int64_t batch,
                            cudaStream_t stream) {
    const C2<R>* src = static_cast<const C2<R>*>(in);
    for (int s = 0; s < d.nstages; ++s) {
        C2<R>* dst = (s + 1 == d.nstages) ? static_cast<C2<R>*>(out) : static_cast<C2<R>*>(s % 2 ? s1 : s0);
        const GStage& st = d.st[s];
        for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
            const unsigned nb = static_cast<unsigned>(std::min<int64_t>(65535, batch - b0));
            const int64_t off = b0 * d.N;
            if (st.kind == 0) {
                dim3 grid(static_cast<unsigned>((d.N + 255) / 256), nb);
                gstage_sparse_kernel<R><<<grid, 256, 0, stream>>>(st, d.N, src + off, dst + off);
            } else {
                const int64_t items = static_cast<int64_t>(st.nodes) * st.m3;
                dim3 grid(static_cast<unsigned>((items + 255) / 256), nb);
                gstage_mix_kernel<R><<<grid, 256, 0, stream>>>(st, d.N, src + off, dst + off);
            }
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
        src = dst;
    }
    return cudaSuccess;
}

}  // namespace

cudaError_t launch_global_pipeline(const GlobalPipelineDesc& d, bool f32, const void* in, void* out, void* scratch0,
                                   void* scratch1, int64_t batch, cudaStream_t stream) {
    if (batch <= 0) return cudaSuccess;
    return f32 ? launch_global_t<float>(d, in, out, scratch0, scratch1, batch, stream)
               : launch_global_t<double>(d, in, out, scratch0, scratch1, batch, stream);
}

// ===========================================================================
// Direct transform GEMMs (real form: C[M][Nn] = A[M][K] * Wt[Nn][K]^T)
// ===========================================================================
namespace {

constexpr int GBM = 64, GBN = 128, GBK = 16, GLD = 20;  // GLD: padded row (doubles)

__global__ void __launch_bounds__(256) gemm_f64_kernel(const double* __restrict__ A, const double* __restrict__ W,
                                                       double* __restrict__ C, int64_t M, int Nn, int K) {
    extern __shared__ __align__(16) double gsm[];
    double* As = gsm;                    // [2][GBM][GLD]
    double* Bs = gsm + 2 * GBM * GLD;    // [2][GBN][GLD]
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int wm = warp / 4, wn = warp % 4;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * GBM;
    const int n0 = blockIdx.x * GBN;
    double c[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j][0] = c[i][j][1] = 0.0;

    auto load_tile = [&](int buf, int k0) {
        // A: 64 rows x 16 doubles = 512 chunks of 16B; 2 per thread
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int chunk = tid + q * 256;
            const int r = chunk / 8, cc = chunk % 8;
            const int64_t gr = m0 + r;
            const int gk = k0 + cc * 2;
            const bool ok = gr < M && gk < K;
            cp_async16(As + (buf * GBM + r) * GLD + cc * 2, ok ? A + gr * K + gk : A, ok);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int chunk = tid + q * 256;
            const int r = chunk / 8, cc = chunk % 8;
            const int gn = n0 + r;
            const int gk = k0 + cc * 2;
            const bool ok = gn < Nn && gk < K;
            cp_async16(Bs + (buf * GBN + r) * GLD + cc * 2, ok ? W + static_cast<int64_t>(gn) * K + gk : W, ok);
        }
        cp_async_commit();
    };

    const int ktiles = (K + GBK - 1) / GBK;
    load_tile(0, 0);
    for (int kt = 0; kt < ktiles; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < ktiles) {
            load_tile(buf ^ 1, (kt + 1) * GBK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* as = As + buf * GBM * GLD;
        const double* bs = Bs + buf * GBN * GLD;
#pragma unroll
        for (int kk = 0; kk < GBK; kk += 4) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = as[(wm * 32 + i * 8 + (lane >> 2)) * GLD + kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = bs[(wn * 32 + j * 8 + (lane >> 2)) * GLD + kk + (lane & 3)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(c[i][j][0], c[i][j][1], a[i], b[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t row = m0 + wm * 32 + i * 8 + (lane >> 2);
            const int col = n0 + wn * 32 + j * 8 + 2 * (lane & 3);
            if (row < M && col + 1 < Nn + 1) {
                if (col + 1 < Nn) {
                    *reinterpret_cast<double2*>(C + row * Nn + col) = make_double2(c[i][j][0], c[i][j][1]);
                } else if (col < Nn) {
                    C[row * Nn + col] = c[i][j][0];
                }
            }
        }
}

// fp32: classic 128x128x8 SIMT tile, 8x8 outputs per thread.
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, const float* __restrict__ W,
                                                       float* __restrict__ C, int64_t M, int Nn, int K) {
    __shared__ __align__(16) float As[2][8][128 + 4];
    __shared__ __align__(16) float Bs[2][8][128 + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * 128;
    const int n0 = blockIdx.x * 128;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    // each thread loads 4 A values and 4 B values per k-tile: row = tid/2, k = (tid%2)*4 .. +3
    const int lr = tid / 2, lk = (tid % 2) * 4;
    float ra[4], rb[4];
    auto gload = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t gr = m0 + lr;
            const int gk = k0 + lk + q;
            ra[q] = (gr < M && gk < K) ? __ldg(A + gr * K + gk) : 0.f;
            const int gn = n0 + lr;
            rb[q] = (gn < Nn && gk < K) ? __ldg(W + static_cast<int64_t>(gn) * K + gk) : 0.f;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            As[buf][lk + q][lr] = ra[q];
            Bs[buf][lk + q][lr] = rb[q];
        }
    };
    const int ktiles = (K + 7) / 8;
    gload(0);
    sstore(0);
    __syncthreads();
    for (int kt = 0; kt < ktiles; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < ktiles) gload((kt + 1) * 8);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float a[8], b[8];
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
            a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
            b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (kt + 1 < ktiles) sstore(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int col = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
            if (col < Nn) C[row * Nn + col] = acc[i][j];
        }
    }
}

}  // namespace

cudaError_t launch_gemm_f64(const double* A, const double* Wt, double* C, int64_t M, int Nn, int K,
                            cudaStream_t st) {
    if (M <= 0) return cudaSuccess;
    const int smem = 2 * (GBM + GBN) * GLD * static_cast<int>(sizeof(double));
    cudaError_t e = prepare_launch(reinterpret_cast<const void*>(gemm_f64_kernel), 256, smem, nullptr);
    if (e != cudaSuccess) return e;
    dim3 grid((Nn + GBN - 1) / GBN, static_cast<unsigned>((M + GBM - 1) / GBM));
    gemm_f64_kernel<<<grid, 256, smem, st>>>(A, Wt, C, M, Nn, K);
    return cudaGetLastError();
}

cudaError_t launch_gemm_f32(const float* A, const float* Wt, float* C, int64_t M, int Nn, int K,
                            cudaStream_t st) {
    if (M <= 0) return cudaSuccess;
    dim3 grid((Nn + 127) / 128, static_cast<unsigned>((M + 127) / 128));
    gemm_f32_kernel<<<grid, 256, 0, st>>>(A, Wt, C, M, Nn, K);
    return cudaGetLastError();
}

// ===========================================================================
// Device-side table generation
// ===========================================================================
namespace {

// e^{2 pi i (frac + ip/n)}: frac = (w kappa).p / n in double (exact for
// dyadic offsets), ip reduced mod n exactly in integers.
__device__ __forceinline__ double2 phase_turns(double turns) {
    turns -= floor(turns);
    double s, c;
    sincospi(2.0 * turns, &s, &c);
    return make_double2(c, s);
}

__device__ double2 dense_entry_dev(int n, double r, double s, double t, int i0, int i1, int i2, int k0, int k1,
                                   int k2) {
    double re = 0.0, im = 0.0;
    for (int e = 0; e < 24; ++e) {
        const int* w = c_group + e * 9;
        const int a0 = w[0] * k0 + w[1] * k1 + w[2] * k2;
        const int a1 = w[3] * k0 + w[4] * k1 + w[5] * k2;
        const int a2 = w[6] * k0 + w[7] * k1 + w[8] * k2;
        const double frac = (r * a0 + s * a1 + t * a2) / n;
        long long ip = static_cast<long long>(a0) * i0 + static_cast<long long>(a1) * i1 +
                       static_cast<long long>(a2) * i2;
        ip %= n;
        if (ip < 0) ip += n;
        const double2 ph = phase_turns(frac + static_cast<double>(ip) / n);
        re += ph.x;
        im += ph.y;
    }
    return make_double2(re / 24.0, im / 24.0);
}

template <typename R>
__global__ void gen_dense_realform_kernel(int n, double r, double s, double t, R* Wt) {
    const int64_t N = static_cast<int64_t>(n) * n * n;
    const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (idx >= N * N) return;
    const int64_t node = idx / N, kap = idx % N;
    const int i0 = static_cast<int>(node / (n * n)), i1 = static_cast<int>((node / n) % n), i2 = static_cast<int>(node % n);
    const int k0 = static_cast<int>(kap / (n * n)), k1 = static_cast<int>((kap / n) % n), k2 = static_cast<int>(kap % n);
    const double2 v = dense_entry_dev(n, r, s, t, i0, i1, i2, k0, k1, k2);
    const int64_t K = 2 * N;
    Wt[(2 * node) * K + 2 * kap] = static_cast<R>(v.x);
    Wt[(2 * node) * K + 2 * kap + 1] = static_cast<R>(-v.y);
    Wt[(2 * node + 1) * K + 2 * kap] = static_cast<R>(v.y);
    Wt[(2 * node + 1) * K + 2 * kap + 1] = static_cast<R>(v.x);
}

__global__ void gen_dense_colmajor_kernel(int n, double r, double s, double t, double2* D) {
    const int64_t N = static_cast<int64_t>(n) * n * n;
    const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (idx >= N * N) return;
    const int64_t kap = idx / N, node = idx % N;
    const int i0 = static_cast<int>(node / (n * n)), i1 = static_cast<int>((node / n) % n), i2 = static_cast<int>(node % n);
    const int k0 = static_cast<int>(kap / (n * n)), k1 = static_cast<int>((kap / n) % n), k2 = static_cast<int>(kap % n);
    D[idx] = dense_entry_dev(n, r, s, t, i0, i1, i2, k0, k1, k2);
}

// ||D_n(p)||_1 column sums (the norm factor of the reference's condition
// estimate, condition_with_lu, transform.cpp:93): one CTA per column kappa
// (grid-stride), the 24 group terms a_w = w kappa (reduced mod n) with
// c_w = e^{2 pi i (w kappa).p/n}/24 (unreduced exponent, transform.cpp:51-53) in
// shared memory, then every node x sums c_w e^{2 pi i (a_w.x mod n)/n} from a
// twiddle table. Plan-time only.
__global__ void dense_colnorm_kernel(int n, double r, double s, double t, double* colsum) {
    extern __shared__ double2 tw[];  // n twiddles
    __shared__ int aw[24][3];
    __shared__ double2 cw[24];
    __shared__ double red[32];
    const int64_t N = static_cast<int64_t>(n) * n * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) tw[i] = phase_turns(static_cast<double>(i) / n);
    for (int64_t kap = blockIdx.x; kap < N; kap += gridDim.x) {
        if (threadIdx.x < 24) {
            const int* w = c_group + threadIdx.x * 9;
            const int k0 = static_cast<int>(kap / (n * n)), k1 = static_cast<int>((kap / n) % n),
                      k2 = static_cast<int>(kap % n);
            const int a0 = w[0] * k0 + w[1] * k1 + w[2] * k2;
            const int a1 = w[3] * k0 + w[4] * k1 + w[5] * k2;
            const int a2 = w[6] * k0 + w[7] * k1 + w[8] * k2;
            const double2 c = phase_turns((r * a0 + s * a1 + t * a2) / n);
            cw[threadIdx.x] = make_double2(c.x / 24.0, c.y / 24.0);
            aw[threadIdx.x][0] = ((a0 % n) + n) % n;
            aw[threadIdx.x][1] = ((a1 % n) + n) % n;
            aw[threadIdx.x][2] = ((a2 % n) + n) % n;
        }
        __syncthreads();
        double acc = 0.0;
        for (int64_t x = threadIdx.x; x < N; x += blockDim.x) {
            const int x0 = static_cast<int>(x / (n * n)), x1 = static_cast<int>((x / n) % n), x2 = static_cast<int>(x % n);
            double re = 0.0, im = 0.0;
#pragma unroll 4
            for (int e = 0; e < 24; ++e) {
                const int ip = (aw[e][0] * x0 + aw[e][1] * x1 + aw[e][2] * x2) % n;
                const double2 f = tw[ip], c = cw[e];
                re = fma(c.x, f.x, fma(-c.y, f.y, re));
                im = fma(c.x, f.y, fma(c.y, f.x, im));
            }
            acc += hypot(re, im);
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) tot += red[i];
            colsum[kap] = tot;
        }
        __syncthreads();
    }
}

// D^{-1}[kappa][node] = (1/N) sum_{a in O(kappa)} Sinv[kappa][a] e^{-2 pi i a.node/n}
template <typename R>
__global__ void gen_dense_inv_realform_kernel(int n, OrbitDev od, R* Wt) {
    const int64_t N = static_cast<int64_t>(n) * n * n;
    const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (idx >= N * N) return;
    const int64_t kap = idx / N, node = idx % N;
    const int i0 = static_cast<int>(node / (n * n)), i1 = static_cast<int>((node / n) % n), i2 = static_cast<int>(node % n);
    const int O = od.orbit_of[kap], pk = od.pos[kap];
    const int off = od.mem_off[O], d = od.mem_off[O + 1] - off;
    const double* S = od.sinv + 2 * (od.sinv_off[O] + static_cast<int64_t>(pk) * d);
    double re = 0.0, im = 0.0;
    for (int i = 0; i < d; ++i) {
        const int a = od.mem[off + i];
        const int a0 = a / (n * n), a1 = (a / n) % n, a2 = a % n;
        const long long ip = (static_cast<long long>(a0) * i0 + static_cast<long long>(a1) * i1 +
                              static_cast<long long>(a2) * i2) % n;
        const double2 ph = phase_turns(-static_cast<double>(ip) / n);
        const double sr = S[2 * i], si = S[2 * i + 1];
        re += sr * ph.x - si * ph.y;
        im += sr * ph.y + si * ph.x;
    }
    re /= static_cast<double>(N);
    im /= static_cast<double>(N);
    const int64_t K = 2 * N;
    Wt[(2 * kap) * K + 2 * node] = static_cast<R>(re);
    Wt[(2 * kap) * K + 2 * node + 1] = static_cast<R>(-im);
    Wt[(2 * kap + 1) * K + 2 * node] = static_cast<R>(im);
    Wt[(2 * kap + 1) * K + 2 * node + 1] = static_cast<R>(re);
}

__device__ double wrap_turn(double a) {  // TorusPoint::wrapped (chebyshev.cpp:30-39)
    double f = a - floor(a);
    if (f >= 1.0 - 1e-15) f = 0.0;
    return f;
}

__device__ double2 cmul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ double2 crecip(double2 a) {
    const double d = a.x * a.x + a.y * a.y;
    return make_double2(a.x / d, -a.y / d);
}
__device__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

__global__ void gen_nodes_kernel(int n, double r, double s, double t, double2* out) {
    const int64_t N = static_cast<int64_t>(n) * n * n;
    const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (idx >= N) return;
    const int i = static_cast<int>(idx / (n * n)), j = static_cast<int>((idx / n) % n), k = static_cast<int>(idx % n);
    const double th0 = wrap_turn((r + i) / n), th1 = wrap_turn((s + j) / n), th2 = wrap_turn((t + k) / n);
    double s0, c0, s1, c1, s2, c2;
    sincospi(2.0 * th0, &s0, &c0);
    sincospi(2.0 * th1, &s1, &c1);
    sincospi(2.0 * th2, &s2, &c2);
    const double2 u = make_double2(c0, s0), v = make_double2(c1, s1), w = make_double2(c2, s2);
    const double2 ui = crecip(u), vi = crecip(v), wi = crecip(w);
    // coords_from_uvw (chebyshev.cpp:76-85)
    const double2 x = cscale(cadd(cadd(u, cmul(ui, v)), cadd(cmul(vi, w), wi)), 0.25);
    const double2 y = cscale(cadd(cadd(cadd(vi, v), cadd(cmul(u, wi), cmul(cmul(ui, v), wi))),
                                  cadd(cmul(ui, w), cmul(cmul(u, vi), w))),
                             1.0 / 6.0);
    const double2 z = cscale(cadd(cadd(ui, cmul(u, vi)), cadd(cmul(v, wi), w)), 0.25);
    double2* o = out + idx * 6;
    o[0] = u;
    o[1] = v;
    o[2] = w;
    o[3] = x;
    o[4] = y;
    o[5] = z;
}

// check_not_degenerate (spectral.cpp:26-43): any pair closer than 1e-9.
__global__ void degenerate_kernel(int64_t N, const double2* nodes, int* flag) {
    const int64_t a = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (a >= N) return;
    const double2* pa = nodes + a * 6;
    for (int64_t b = a + 1; b < N; ++b) {
        const double2* pb = nodes + b * 6;
        double d = 0.0;
        for (int c = 3; c < 6; ++c) {
            const double dx = pa[c].x - pb[c].x, dy = pa[c].y - pb[c].y;
            d += dx * dx + dy * dy;
        }
        if (d < 1e-18) {
            atomicExch(flag, 1);
            return;
        }
    }
}

__global__ void radix_perm_kernel(int n, unsigned long long* out) {
    const int64_t N = static_cast<int64_t>(n) * n * n;
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= N) return;
    const int m = n / 2;
    const int64_t m3 = static_cast<int64_t>(m) * m * m;
    const int blk = static_cast<int>(i / m3);
    const int64_t k = i % m3;
    const int kr = static_cast<int>(k / (m * m)), ks = static_cast<int>((k / m) % m), kt = static_cast<int>(k % m);
    const int ir = blk >> 2, is = (blk >> 1) & 1, it = blk & 1;
    out[i] = static_cast<unsigned long long>((static_cast<int64_t>(ir + 2 * kr) * n + (is + 2 * ks)) * n + (it + 2 * kt));
}

__global__ void residual_kernel(const double2* Y, const double2* D, int N, double* partial) {
    __shared__ double red[256];
    double best = 0.0;
    const int64_t total = static_cast<int64_t>(N) * N;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        // Y[k][i] vs D column-major D[k*N + i]
        const double2 y = Y[idx], dd = D[idx];
        const double dx = y.x - dd.x, dy = y.y - dd.y;
        best = fmax(best, sqrt(dx * dx + dy * dy));
    }
    red[threadIdx.x] = best;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

template <typename R>
__global__ void identity_kernel(int N, R* E) {
    const int64_t total = static_cast<int64_t>(N) * N;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = idx / N, i = idx % N;
        E[2 * idx] = (k == i) ? R(1) : R(0);
        E[2 * idx + 1] = R(0);
    }
}

__global__ void dmma_probe_kernel(const double* A, const double* B, double* C) {
    const int lane = threadIdx.x;
    const double a = A[(lane >> 2) * 4 + (lane & 3)];
    const double b = B[(lane & 3) * 8 + (lane >> 2)];
    double c0 = 0.0, c1 = 0.0;
    dmma884(c0, c1, a, b);
    C[(lane >> 2) * 8 + 2 * (lane & 3)] = c0;
    C[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = c1;
}

inline unsigned blocks_for(int64_t total, int threads) {
    return static_cast<unsigned>((total + threads - 1) / threads);
}

}  // namespace

cudaError_t gen_dense_realform(int n, double r, double s, double t, void* Wt, bool f32, cudaStream_t st) {
    cudaError_t e = upload_group();
    if (e != cudaSuccess) return e;
    const int64_t N = static_cast<int64_t>(n) * n * n;
    if (f32)
        gen_dense_realform_kernel<float><<<blocks_for(N * N, 256), 256, 0, st>>>(n, r, s, t, static_cast<float*>(Wt));
    else
        gen_dense_realform_kernel<double><<<blocks_for(N * N, 256), 256, 0, st>>>(n, r, s, t, static_cast<double*>(Wt));
    return cudaGetLastError();
}

cudaError_t gen_dense_inv_realform(int n, const OrbitDev& od, void* Wt, bool f32, cudaStream_t st) {
    const int64_t N = static_cast<int64_t>(n) * n * n;
    if (f32)
        gen_dense_inv_realform_kernel<float><<<blocks_for(N * N, 256), 256, 0, st>>>(n, od, static_cast<float*>(Wt));
    else
        gen_dense_inv_realform_kernel<double><<<blocks_for(N * N, 256), 256, 0, st>>>(n, od, static_cast<double*>(Wt));
    return cudaGetLastError();
}

cudaError_t dense_colnorm(int n, double r, double s, double t, double* colsum, cudaStream_t st) {
    cudaError_t e = upload_group();
    if (e != cudaSuccess) return e;
    const int64_t N = static_cast<int64_t>(n) * n * n;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(N, 148 * 16));
    dense_colnorm_kernel<<<grid, 256, sizeof(double2) * n, st>>>(n, r, s, t, colsum);
    return cudaGetLastError();
}

cudaError_t gen_dense_colmajor(int n, double r, double s, double t, double* D, cudaStream_t st) {
    cudaError_t e = upload_group();
    if (e != cudaSuccess) return e;
    const int64_t N = static_cast<int64_t>(n) * n * n;
    gen_dense_colmajor_kernel<<<blocks_for(N * N, 256), 256, 0, st>>>(n, r, s, t, reinterpret_cast<double2*>(D));
    return cudaGetLastError();
}

cudaError_t gen_nodes(int n, double r, double s, double t, double* out, int* flag, cudaStream_t st) {
    const int64_t N = static_cast<int64_t>(n) * n * n;
    gen_nodes_kernel<<<blocks_for(N, 256), 256, 0, st>>>(n, r, s, t, reinterpret_cast<double2*>(out));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || flag == nullptr || n > 16) return e;
    degenerate_kernel<<<blocks_for(N, 128), 128, 0, st>>>(N, reinterpret_cast<const double2*>(out), flag);
    return cudaGetLastError();
}

cudaError_t gen_radix_permutation(int n, unsigned long long* out, cudaStream_t st) {
    const int64_t N = static_cast<int64_t>(n) * n * n;
    radix_perm_kernel<<<blocks_for(N, 256), 256, 0, st>>>(n, out);
    return cudaGetLastError();
}

cudaError_t residual_max(const double* Y, const double* D, int N, double* partial, int nblocks, cudaStream_t st) {
    residual_kernel<<<nblocks, 256, 0, st>>>(reinterpret_cast<const double2*>(Y), reinterpret_cast<const double2*>(D), N,
                                             partial);
    return cudaGetLastError();
}

cudaError_t gen_identity(int N, void* E, bool f32, cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(N) * N;
    const unsigned nb = static_cast<unsigned>(std::min<int64_t>(blocks_for(total, 256), 4096));
    if (f32)
        identity_kernel<float><<<nb, 256, 0, st>>>(N, static_cast<float*>(E));
    else
        identity_kernel<double><<<nb, 256, 0, st>>>(N, static_cast<double*>(E));
    return cudaGetLastError();
}

cudaError_t dmma_probe(const double* A, const double* B, double* C, cudaStream_t st) {
    dmma_probe_kernel<<<1, 32, 0, st>>>(A, B, C);
    return cudaGetLastError();
}

}  // namespace fcct
