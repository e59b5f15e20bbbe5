// Two-pass orbit-FFT executor (orbit16.hpp): pass A, the orbit-block base
// change on the FP64 tensor pipe over gathered chunks of 8 blocks; pass B, the
// radix-2 3D FFT per block.
#include <algorithm>

#include "orbit16.hpp"
#include "orbit_dev.cuh"

namespace fcct {

using namespace dev;
using namespace odev;

namespace {

// ---------------------------------------------------------------------------
// Pass A: base change. One persistent CTA per SM (16 warps), 8 blocks per
// group, chunks of <= kO16Chunk member slots. Stage slot (s, b) at element
// index s * 8 + (b ^ 2 (s & 3)): the quarter-warp of a fragment load (2 blocks
// x 4 slots of one k-tile) touches 8 distinct bank groups for every element
// size (16, 8 and 4 bytes), and the gather's 8 lanes of one slot too.
// ---------------------------------------------------------------------------
constexpr int kRingA = kO16Wrap;  // operator tiles in flight per warp (L2 latency)

template <int DIR, int MI, int MO>
__global__ void __launch_bounds__(kO16Warps * 32, 1)
    orbit16_base_kernel(const __grid_constant__ Orbit16Desc d, const void* __restrict__ in, void* __restrict__ out,
                        int64_t batch) {
    constexpr int SM = DIR == 0 ? MI : OF_C128;  // stage element (the z side is complex128)
    constexpr int DM = DIR == 0 ? OF_C128 : MO;
    constexpr int SEB = eb_of(SM);
    constexpr bool REAL = SM == OF_R64 || SM == OF_R32;
    constexpr int SBUF = kO16Chunk * 8 * SEB;
    extern __shared__ __align__(128) unsigned char smem[];
    const int N = d.N, tmax = d.tmax, nch = d.nchunks;
    // shared: stage[2] | gather lists | tile metadata | output positions (all chunks, copied once)
    char* stage = reinterpret_cast<char*>(smem);
    int* g_s = reinterpret_cast<int*>(smem + 3 * SBUF);
    int* tm_s = g_s + nch * kO16Chunk;
    int* op_s = tm_s + nch * kO16Warps * tmax;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, k = lane & 3;
    for (int i = tid; i < nch * kO16Chunk; i += blockDim.x) g_s[i] = __ldg(d.gather + i);
    for (int i = tid; i < nch * kO16Warps * tmax; i += blockDim.x) tm_s[i] = __ldg(d.tile_meta + i);
    for (int i = tid; i < nch * kO16Warps * tmax * 4; i += blockDim.x) op_s[i] = __ldg(d.out_pos + i);
    const int64_t in_row = static_cast<int64_t>(N) * eb_of(DIR == 0 ? MI : OF_C128);
    const int64_t out_row = static_cast<int64_t>(N) * eb_of(DM);
    const int64_t ngroups = (batch + 7) / 8;
    __syncthreads();
    // stream of (group, chunk) work items of this CTA
    const int64_t items = (ngroups > blockIdx.x ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0) * nch;
    int gc = 0;            // chunk of the next gather
    int64_t ggrp = blockIdx.x;  // group of the next gather
    int gbuf = 0;  // stage buffer of the next gather (rotates 0, 1, 2)
    auto gather = [&]() {
        char* st = stage + gbuf * SBUF;
        gbuf = gbuf == 2 ? 0 : gbuf + 1;
        const int c = gc;
        const int64_t grp = ggrp;
        if (++gc == nch) {
            gc = 0;
            ggrp += gridDim.x;
        }
        // thread tid copies block b = tid & 7 of slots s = tid / 8 + 64 e: its
        // block, source row and bank xor are fixed, only the slot advances
        const int b = tid & 7, s0 = tid >> 3;
        const int* gl = g_s + c * kO16Chunk + s0;
        const bool bvalid = b < batch - grp * 8;
        const char* srow = static_cast<const char*>(in) + (grp * 8 + (bvalid ? b : 0)) * in_row;
        char* dst = st + (s0 * 8 + (b ^ (2 * (s0 & 3)))) * SEB;
        // all list entries first: each cp.async is a compiler memory barrier,
        // a load between two of them would wait out its full latency
        constexpr int E = kO16Chunk * 8 / (kO16Warps * 32);
        int pe[E];
#pragma unroll
        for (int e = 0; e < E; ++e) pe[e] = gl[e * 64];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int p = pe[e];
            if (p >= 0 || (s0 & 3) != 0)  // slots of an unused k-tile are never read
                cp_async_n<SEB>(dst + e * 64 * 8 * SEB, srow + static_cast<int64_t>(p > 0 ? p : 0) * SEB,
                                p >= 0 && bvalid);
        }
        cp_async_commit();
    };
    // operator tile stream of this warp (chunk-major, tmax tiles per chunk),
    // kRingA fragments in flight, loaded L2-only (they are read once per group)
    // this warp's operator tiles are contiguous over the chunks, followed by
    // copies of its first kRingA tiles: the look-ahead reads tp[32 q] and the
    // pointer resets once per group
    const double2* tbase = d.table + static_cast<size_t>(warp) * (static_cast<size_t>(nch) * tmax + kRingA) * 32 + lane;
    const double2* tp = tbase;
    const int lane_off = (8 * k + (r ^ (2 * k))) * SEB;  // this lane's element of a k-tile's 32 slots
    double2 ring[kRingA];
#pragma unroll
    for (int q = 0; q < kRingA; ++q) ring[q] = __ldcg(tp + q * 32);
    tp += kRingA * 32;
    // three stage buffers: chunk item + 2 is gathered while item is computed,
    // one barrier per chunk
    if (items > 0) gather();
    if (items > 1) gather(); else cp_async_commit();
    int c = 0, cbuf = 0;
    int64_t grp = blockIdx.x;
    for (int64_t item = 0; item < items; ++item) {
        cp_async_wait<1>();  // this thread's copies of chunk `item` have landed
        __syncthreads();     // ... everyone's; and every warp is done with chunk item - 1
        if (item + 2 < items)
            gather();  // chunk item + 2, into the buffer chunk item - 1 used
        else
            cp_async_commit();  // keep one group per iteration
        const char* st = stage + cbuf * SBUF;
        cbuf = cbuf == 2 ? 0 : cbuf + 1;
        const int64_t nv = batch - grp * 8;
        const bool live = r < nv;
        char* d_row = static_cast<char*>(out) + (grp * 8 + r) * out_row;
        const int* tm = tm_s + (c * kO16Warps + warp) * tmax;
        const int* op = op_s + (c * kO16Warps + warp) * tmax * 4;
        double cr0 = 0.0, cr1 = 0.0, ci0 = 0.0, ci1 = 0.0;
        // software pipeline: metadata two tiles ahead, the fragment one tile ahead
        auto frag = [&](int m, double& ar, double& ai) {
            if (m & (1 << 17))
                ld_el<SM>(st + (m & 0xFFFF) * (32 * SEB) + lane_off, 0, ar, ai);
            else
                ar = ai = 0.0;
        };
        int m_cur = tm[0], m_nxt = tmax > 1 ? tm[1] : 0;
        double ar, ai;
        frag(m_cur, ar, ai);
        for (int t0 = 0; t0 < tmax; t0 += kRingA) {
#pragma unroll
            for (int q = 0; q < kRingA; ++q) {
                const int t = t0 + q;
                const double2 tb = ring[q];
                ring[q] = __ldcg(tp + q * 32);  // kRingA tiles ahead
                const int m_nn = t + 2 < tmax ? tm[t + 2] : 0;
                double arn, ain;
                frag(m_nxt, arn, ain);
                if (m_cur & (1 << 17)) {  // real tile (padding tiles close each warp's list)
                    dmma884(cr0, cr1, ar, tb.x);
                    dmma884(ci0, ci1, ar, tb.y);
                    if constexpr (!REAL) {
                        dmma884(cr0, cr1, neg_hi16(ai), tb.y);
                        dmma884(ci0, ci1, ai, tb.x);
                    }
                    if (m_cur & (1 << 16)) {  // chain end
                        const int o = op[t * 4 + k];
                        const int o0 = o & 0xFFFF, o1 = (o >> 16) & 0xFFFF;
                        if (live && o0 != 0xFFFF) st_el<DM>(d_row, o0, cr0, ci0);
                        if (live && o1 != 0xFFFF) st_el<DM>(d_row, o1, cr1, ci1);
                        cr0 = cr1 = ci0 = ci1 = 0.0;
                    }
                }
                m_cur = m_nxt;
                m_nxt = m_nn;
                ar = arn;
                ai = ain;
            }
            tp += kRingA * 32;
        }
        if (++c == nch) {
            c = 0;
            grp += gridDim.x;
            tp = tbase + kRingA * 32;  // the ring holds the group's first tiles (the wrap copies)
        }
    }
}

// ---------------------------------------------------------------------------
// Pass B: 3D radix-2 FFT of NN^3 points per block. 256 threads, one line of
// NN points per thread per pass; the tile is loaded by cp.async (complex128
// input) into the (k ^ j)-swizzled layout, the block after next is prefetched.
// ---------------------------------------------------------------------------

constexpr int kFftThreads = 256;

template <int NN, int SIGN, int MI, int MO>
__global__ void __launch_bounds__(kFftThreads, 2)
    fft_cube_kernel(const void* __restrict__ in, void* __restrict__ out, int64_t batch, const int* __restrict__ zperm) {
    constexpr int N = NN * NN * NN, LINES = NN * NN;
    static_assert(LINES == kFftThreads, "one line per thread per pass");
    // one 64 KB tile and the orbit-order permutation per CTA, two CTAs per SM:
    // the block after this one is prefetched into L2 while the tile is transformed
    extern __shared__ __align__(128) unsigned char smem[];
    double2* X = reinterpret_cast<double2*>(smem);
    int* zp = reinterpret_cast<int*>(smem + N * 16);
    const int tid = threadIdx.x, hi = tid / NN, lo = tid % NN;
    for (int a = tid; a < N; a += kFftThreads) zp[a] = __ldg(zperm + a);
    __syncthreads();
    auto swz = [](int i, int j, int k) { return (i * NN + j) * NN + (k ^ (j & (NN - 1))); };
    constexpr int64_t in_row = int64_t{N} * eb_of(MI), out_row = int64_t{N} * eb_of(MO);
    for (int64_t blk = blockIdx.x; blk < batch; blk += gridDim.x) {
        const int64_t nx = blk + gridDim.x;
        if (tid == 0 && nx < batch) prefetch_l2_bulk(static_cast<const char*>(in) + nx * in_row, static_cast<uint32_t>(in_row));
        const char* src = static_cast<const char*>(in) + blk * in_row;
        for (int a = tid; a < N; a += kFftThreads) {  // natural (or orbit-ordered z) -> tile
            const int k = a % NN, j = (a / NN) % NN, i = a / (NN * NN);
            if constexpr (SIGN > 0) {  // forward: z (orbit order) copied contiguously; un-permuted by the k pass
                cp_async_n<16>(X + a, src + static_cast<int64_t>(a) * 16, true);
            } else if constexpr (MI == OF_C128) {
                cp_async_n<16>(X + swz(i, j, k), src + static_cast<int64_t>(a) * 16, true);
            } else {
                double re, im;
                ld_el<MI>(src, a, re, im);
                X[swz(i, j, k)] = make_double2(re, im);
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        double2 v[NN];
        // k axis: line (i, j) = (hi, lo)
        if constexpr (SIGN > 0) {  // the tile holds z in orbit order: gather, then write the swizzled layout
#pragma unroll
            for (int x = 0; x < NN; ++x) v[x] = X[zp[(hi * NN + lo) * NN + x]];
            __syncthreads();  // every line has been read before the tile is rewritten
        } else {
#pragma unroll
            for (int x = 0; x < NN; ++x) v[x] = X[swz(hi, lo, x)];
        }
        fft_line16<NN, SIGN>(v);
#pragma unroll
        for (int x = 0; x < NN; ++x) X[swz(hi, lo, x)] = v[x];
        __syncthreads();
        // j axis: line (i, k) = (hi, lo)
#pragma unroll
        for (int x = 0; x < NN; ++x) v[x] = X[swz(hi, x, lo)];
        fft_line16<NN, SIGN>(v);
#pragma unroll
        for (int x = 0; x < NN; ++x) X[swz(hi, x, lo)] = v[x];
        __syncthreads();
        // i axis: line (j, k) = (hi, lo), stored to HBM (lanes vary k: coalesced)
#pragma unroll
        for (int x = 0; x < NN; ++x) v[x] = X[swz(x, hi, lo)];
        fft_line16<NN, SIGN>(v);
        char* dst = static_cast<char*>(out) + blk * out_row;
        if constexpr (SIGN > 0) {
#pragma unroll
            for (int x = 0; x < NN; ++x) st_el<MO>(dst, (x * NN + hi) * NN + lo, v[x].x, v[x].y);
        } else {
            // inverse: z is stored in orbit order; the lines go back into the
            // tile at their orbit-order slots first, then the row leaves in
            // contiguous 16-byte stores
            __syncthreads();  // every line of the i pass has been read
#pragma unroll
            for (int x = 0; x < NN; ++x) X[zp[(x * NN + hi) * NN + lo]] = v[x];
            __syncthreads();
            double2* d2 = reinterpret_cast<double2*>(dst);
            for (int a = tid; a < N; a += kFftThreads) d2[a] = X[a];
        }
        __syncthreads();  // the tile is refilled by the next block
    }
}

template <int DIR, int MI, int MO>
cudaError_t launch_a(const Orbit16Desc& d, const void* in, void* out, int64_t batch, cudaStream_t st, int num_sms) {
    constexpr int SM = DIR == 0 ? MI : OF_C128;
    const int smem = 3 * kO16Chunk * 8 * eb_of(SM) + d.nchunks * kO16Chunk * 4 + d.nchunks * kO16Warps * d.tmax * 5 * 4;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    auto kern = orbit16_base_kernel<DIR, MI, MO>;
    static thread_local int prepared = -1;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (prepared != dev) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        prepared = dev;
    }
    const int64_t groups = (batch + 7) / 8;
    kern<<<static_cast<unsigned>(std::min<int64_t>(groups, num_sms)), kO16Warps * 32, smem, st>>>(d, in, out, batch);
    return cudaGetLastError();
}

template <int NN, int SIGN, int MI, int MO>
cudaError_t launch_b(const void* in, void* out, int64_t batch, const int* zperm, cudaStream_t st, int num_sms) {
    const int smem = NN * NN * NN * (16 + 4);
    auto kern = fft_cube_kernel<NN, SIGN, MI, MO>;
    static thread_local int prepared = -1;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (prepared != dev) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        prepared = dev;
    }
    kern<<<static_cast<unsigned>(std::min<int64_t>(batch, 2 * static_cast<int64_t>(num_sms))), kFftThreads, smem, st>>>(
        in, out, batch, zperm);
    return cudaGetLastError();
}

// out[b][a] = in[b][zperm[a]]: the inverse base change's orbit-ordered rows
// back to natural positions: one CTA per row. The orbit-ordered row is copied
// into shared memory with coalesced 16-byte cp.async, then every thread
// gathers 16 bytes' worth of natural positions from it and stores them with
// one 16-byte store (the earlier element-per-thread gather kept one 8-byte
// load in flight per thread: 3.7 TB/s).
constexpr int kUnpThreads = 256;
// unaligned buffers / rows (user output pointers): element per thread
template <int M>
__global__ void __launch_bounds__(256) unpermute_elem_kernel(const char* __restrict__ in, char* __restrict__ out,
                                                             int N, int64_t batch, const int* __restrict__ zperm) {
    constexpr int EB = eb_of(M);
    const int64_t total = batch * N;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t b = i / N;
        const int a = static_cast<int>(i - b * N);
        const char* src = in + (b * N + __ldg(zperm + a)) * EB;
        char* dst = out + i * EB;
        if constexpr (EB == 16)
            *reinterpret_cast<double2*>(dst) = *reinterpret_cast<const double2*>(src);
        else if constexpr (EB == 8)
            *reinterpret_cast<double*>(dst) = *reinterpret_cast<const double*>(src);
        else
            *reinterpret_cast<float*>(dst) = *reinterpret_cast<const float*>(src);
    }
}
template <int M>
__global__ void __launch_bounds__(kUnpThreads) unpermute_kernel(const char* __restrict__ in, char* __restrict__ out,
                                                               int N, const int* __restrict__ zperm) {
    constexpr int EB = eb_of(M), V = 16 / EB;  // elements per 16-byte store
    extern __shared__ __align__(16) unsigned char srow[];
    const int64_t b = blockIdx.x;
    const char* row = in + b * N * EB;
    const int pieces = N * EB / 16;
    for (int q = threadIdx.x; q < pieces; q += kUnpThreads) cp_async_n<16>(srow + q * 16, row + q * 16, true);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    char* orow = out + b * N * EB;
    for (int q = threadIdx.x; q < pieces; q += kUnpThreads) {
        if constexpr (V == 1) {
            reinterpret_cast<uint4*>(orow)[q] = reinterpret_cast<const uint4*>(srow)[__ldg(zperm + q)];
        } else if constexpr (V == 2) {
            const int2 a = __ldg(reinterpret_cast<const int2*>(zperm) + q);
            const uint2 lo = reinterpret_cast<const uint2*>(srow)[a.x], hi = reinterpret_cast<const uint2*>(srow)[a.y];
            reinterpret_cast<uint4*>(orow)[q] = make_uint4(lo.x, lo.y, hi.x, hi.y);
        } else {
            const int4 a = __ldg(reinterpret_cast<const int4*>(zperm) + q);
            const unsigned* s = reinterpret_cast<const unsigned*>(srow);
            reinterpret_cast<uint4*>(orow)[q] = make_uint4(s[a.x], s[a.y], s[a.z], s[a.w]);
        }
    }
}

}  // namespace

cudaError_t launch_unpermute(int mode, const void* in, void* out, int N, int64_t batch, const int* zperm,
                             cudaStream_t st, int num_sms) {
    if (batch <= 0) return cudaSuccess;
    const int eb = eb_of(mode);
    auto* i = static_cast<const char*>(in);
    auto* o = static_cast<char*>(out);
    // the row-staged kernel needs whole 16-byte pieces per row and 16-byte
    // aligned buffers; anything else takes the element-per-thread kernel
    if ((N * eb) % 16 != 0 || ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) != 0 ||
        batch > 0x7FFFFFFF || N * eb > 227 * 1024) {
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>((batch * N + 255) / 256, 8 * int64_t{num_sms}));
        switch (mode) {
            case OF_C128: unpermute_elem_kernel<OF_C128><<<grid, 256, 0, st>>>(i, o, N, batch, zperm); break;
            case OF_C64: unpermute_elem_kernel<OF_C64><<<grid, 256, 0, st>>>(i, o, N, batch, zperm); break;
            case OF_R64: unpermute_elem_kernel<OF_R64><<<grid, 256, 0, st>>>(i, o, N, batch, zperm); break;
            default: unpermute_elem_kernel<OF_R32><<<grid, 256, 0, st>>>(i, o, N, batch, zperm); break;
        }
        return cudaGetLastError();
    }
    const int smem = N * eb;
    auto go = [&](auto kern) {
        if (smem > 48 * 1024) {
            const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
        }
        kern<<<static_cast<unsigned>(batch), kUnpThreads, smem, st>>>(i, o, N, zperm);
        return cudaGetLastError();
    };
    switch (mode) {
        case OF_C128: return go(unpermute_kernel<OF_C128>);
        case OF_C64: return go(unpermute_kernel<OF_C64>);
        case OF_R64: return go(unpermute_kernel<OF_R64>);
        default: return go(unpermute_kernel<OF_R32>);
    }
}

cudaError_t launch_orbit16_base(const Orbit16Desc& d, int in_mode, int out_mode, const void* in, void* out,
                                int64_t batch, cudaStream_t st, int num_sms) {
    if (batch <= 0) return cudaSuccess;
    if (d.tmax % kRingA != 0) return cudaErrorInvalidValue;  // the ring stays chunk-aligned
    if (d.dir == 0 && out_mode == OF_C128) {
        switch (in_mode) {
            case OF_C128: return launch_a<0, OF_C128, OF_C128>(d, in, out, batch, st, num_sms);
            case OF_C64: return launch_a<0, OF_C64, OF_C128>(d, in, out, batch, st, num_sms);
            case OF_R64: return launch_a<0, OF_R64, OF_C128>(d, in, out, batch, st, num_sms);
            case OF_R32: return launch_a<0, OF_R32, OF_C128>(d, in, out, batch, st, num_sms);
        }
    }
    if (d.dir == 1 && in_mode == OF_C128) {
        switch (out_mode) {
            case OF_C128: return launch_a<1, OF_C128, OF_C128>(d, in, out, batch, st, num_sms);
            case OF_C64: return launch_a<1, OF_C128, OF_C64>(d, in, out, batch, st, num_sms);
            case OF_R64: return launch_a<1, OF_C128, OF_R64>(d, in, out, batch, st, num_sms);
            case OF_R32: return launch_a<1, OF_C128, OF_R32>(d, in, out, batch, st, num_sms);
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_fft_cube(int n, int sign, int in_mode, int out_mode, const void* in, void* out, int64_t batch,
                            const int* zperm, cudaStream_t st, int num_sms) {
    if (batch <= 0) return cudaSuccess;
    if (n != 16) return cudaErrorInvalidValue;
    // forward: z (complex128) -> y (c128 / c64); inverse: y (c128 / c64) -> z (complex128)
    if (sign > 0 && in_mode == OF_C128) {
        if (out_mode == OF_C128) return launch_b<16, +1, OF_C128, OF_C128>(in, out, batch, zperm, st, num_sms);
        if (out_mode == OF_C64) return launch_b<16, +1, OF_C128, OF_C64>(in, out, batch, zperm, st, num_sms);
    }
    if (sign < 0 && out_mode == OF_C128) {
        if (in_mode == OF_C128) return launch_b<16, -1, OF_C128, OF_C128>(in, out, batch, zperm, st, num_sms);
        if (in_mode == OF_C64) return launch_b<16, -1, OF_C64, OF_C128>(in, out, batch, zperm, st, num_sms);
    }
    return cudaErrorInvalidValue;
}

}  // namespace fcct
