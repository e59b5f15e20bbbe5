// Orbit-FFT executor (orbit_fft.hpp): one persistent CTA per SM, 16 warps.
//
// Tile = 8 * G transform blocks (G = 1 at n = 8, 8 at n = 4). Shared memory:
//   X[2]  input tiles as they arrive from HBM (TMA bulk row copies, raw I/O
//         element type), double-buffered; in the inverse the same buffer
//         stages the output rows for the TMA bulk store;
//   Y     the complex128 FFT tile, swizzled (of_swizzle) so that the k-, j-
//         and i-axis line passes are free of bank conflicts;
//   meta  per-warp tile metadata of the base change.
// Forward:  S_n x on DMMA (X -> Y), FFT(+) along k, j, i; the i pass stores
//           its lines straight to HBM (coalesced 16-byte stores).
// Inverse:  FFT(-) along i (X -> Y), j, k; S_n^{-1}/n^3 on DMMA (Y -> X);
//           TMA bulk store of the rows.
// The base-change operator is register resident: each warp owns a fixed set
// of DMMA tiles (<= TMAX) for the whole kernel, so no table traffic remains.
#include <algorithm>

#include "device.cuh"
#include "orbit_fft.hpp"

namespace fcct {

using namespace dev;

namespace {

__host__ __device__ constexpr double cos16(int e) {
    switch (e & 15) {
        case 0: return 1.0;
        case 1: return 0.92387953251128675613;
        case 2: return 0.70710678118654752440;
        case 3: return 0.38268343236508977173;
        case 4: return 0.0;
        case 5: return -0.38268343236508977173;
        case 6: return -0.70710678118654752440;
        case 7: return -0.92387953251128675613;
        case 8: return -1.0;
        case 9: return -0.92387953251128675613;
        case 10: return -0.70710678118654752440;
        case 11: return -0.38268343236508977173;
        case 12: return 0.0;
        case 13: return 0.38268343236508977173;
        case 14: return 0.70710678118654752440;
        default: return 0.92387953251128675613;
    }
}

__host__ __device__ constexpr int bitrev(int q, int nn) {
    int r = 0;
    for (int b = 1; b < nn; b <<= 1) {
        r = (r << 1) | (q & 1);
        q >>= 1;
    }
    return r;
}

// d * e^{SIGN 2 pi i e / NN}; e is a compile-time constant after unrolling
template <int NN, int SIGN>
__device__ __forceinline__ double2 twiddle(double2 d, int e) {
    if (e == 0) return d;
    if (4 * e == NN) return SIGN > 0 ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
    const double c = cos16(e * (16 / NN)), s = SIGN * cos16(e * (16 / NN) - 4);
    return make_double2(fma(d.x, c, -d.y * s), fma(d.x, s, d.y * c));
}

// v[q] <- sum_p v[p] e^{SIGN 2 pi i p q / NN} (radix-2 decimation in frequency;
// the bit reversal is a register renaming)
template <int NN, int SIGN>
__device__ __forceinline__ void fft_line(double2 (&v)[NN]) {
#pragma unroll
    for (int half = NN / 2; half >= 1; half >>= 1) {
#pragma unroll
        for (int st = 0; st < NN; st += 2 * half) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double2 a = v[st + j], b = v[st + j + half];
                v[st + j] = make_double2(a.x + b.x, a.y + b.y);
                v[st + j + half] = twiddle<NN, SIGN>(make_double2(a.x - b.x, a.y - b.y), j * (NN / (2 * half)));
            }
        }
    }
    double2 t[NN];
#pragma unroll
    for (int q = 0; q < NN; ++q) t[q] = v[bitrev(q, NN)];
#pragma unroll
    for (int q = 0; q < NN; ++q) v[q] = t[q];
}

__host__ __device__ constexpr int mode_bytes(int m) { return m == OF_C128 ? 16 : (m == OF_R32 ? 4 : 8); }

template <int M>
__device__ __forceinline__ void load_elem(const char* row, int pos, double& re, double& im) {
    if constexpr (M == OF_C128) {
        const double2 v = *reinterpret_cast<const double2*>(row + pos * 16);
        re = v.x;
        im = v.y;
    } else if constexpr (M == OF_C64) {
        const float2 v = *reinterpret_cast<const float2*>(row + pos * 8);
        re = v.x;
        im = v.y;
    } else if constexpr (M == OF_R64) {
        re = *reinterpret_cast<const double*>(row + pos * 8);
        im = 0.0;
    } else {
        re = *reinterpret_cast<const float*>(row + pos * 4);
        im = 0.0;
    }
}

template <int M>
__device__ __forceinline__ void store_elem(char* row, int pos, double re, double im) {
    if constexpr (M == OF_C128) {
        *reinterpret_cast<double2*>(row + pos * 16) = make_double2(re, im);
    } else if constexpr (M == OF_C64) {
        *reinterpret_cast<float2*>(row + pos * 8) = make_float2(static_cast<float>(re), static_cast<float>(im));
    } else if constexpr (M == OF_R64) {
        *reinterpret_cast<double*>(row + pos * 8) = re;
    } else {
        *reinterpret_cast<float*>(row + pos * 4) = static_cast<float>(re);
    }
}

__device__ __forceinline__ double neg_hi(double v) {  // -v on the integer pipe (a DADD would take an FP64 slot)
    return __hiloint2double(__double2hiint(v) ^ static_cast<int>(0x80000000u), __double2loint(v));
}

// Base change on the FP64 tensor pipe: C[block][out] += A[block][in] T[in][out]
// over this warp's register-resident tiles (every warp runs exactly TMAX,
// padded with zero tiles), for each 8-block group. The four real products go
// to four independent accumulator pairs (two DMMA chains per accumulator
// instead of four), and the next tile's metadata and A fragment are loaded
// before this tile's DMMAs.
template <int TMAX, int G, int SM, int DM>
__device__ __forceinline__ void base_change(const double2 (&tab)[TMAX], const int2* __restrict__ meta_w,
                                            const char* src, int srow, char* dst, int drow, int r, int k) {
    constexpr bool real_src = SM == OF_R64 || SM == OF_R32;
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
        const char* s_row = src + (8 * g + r) * srow;
        char* d_row = dst + (8 * g + r) * drow;
        double rr0 = 0.0, rr1 = 0.0, ri0 = 0.0, ri1 = 0.0;  // a_re Tr, -a_im Ti  -> Re
        double ir0 = 0.0, ir1 = 0.0, ii0 = 0.0, ii1 = 0.0;  // a_re Ti,  a_im Tr  -> Im
        int2 m = meta_w[k];
        double ar, ai;
        load_elem<SM>(s_row, m.x & 0xFFFF, ar, ai);
#pragma unroll
        for (int t = 0; t < TMAX; ++t) {
            int2 mn = m;
            double arn = 0.0, ain = 0.0;
            if (t + 1 < TMAX) {
                mn = meta_w[(t + 1) * 4 + k];
                load_elem<SM>(s_row, mn.x & 0xFFFF, arn, ain);
            }
            dmma884(rr0, rr1, ar, tab[t].x);
            dmma884(ir0, ir1, ar, tab[t].y);
            if constexpr (!real_src) {
                // -a_im Ti: the sign goes on the data (a table-side negation is
                // loop invariant and the compiler would keep TMAX of them live)
                dmma884(ri0, ri1, neg_hi(ai), tab[t].y);
                dmma884(ii0, ii1, ai, tab[t].x);
            }
            if (m.x & (2 << 16)) {  // chain end (warp-uniform)
                const int o0 = m.y & 0xFFFF, o1 = (m.y >> 16) & 0xFFFF;
                if constexpr (real_src) {
                    if (o0 != 0xFFFF) store_elem<DM>(d_row, o0, rr0, ir0);
                    if (o1 != 0xFFFF) store_elem<DM>(d_row, o1, rr1, ir1);
                } else {
                    if (o0 != 0xFFFF) store_elem<DM>(d_row, o0, rr0 + ri0, ir0 + ii0);
                    if (o1 != 0xFFFF) store_elem<DM>(d_row, o1, rr1 + ri1, ir1 + ii1);
                }
                rr0 = rr1 = ri0 = ri1 = ir0 = ir1 = ii0 = ii1 = 0.0;
            }
            m = mn;
            ar = arn;
            ai = ain;
        }
    }
}

// One FFT pass along axis AX (0 = i, 1 = j, 2 = k) over every block of the tile.
// Source / sink: the swizzled Y tile, or (SRC_G / DST_G) natural raw rows.
template <int NN, int SIGN, int TB, int AX, int SRCM, int DSTM>
__device__ __forceinline__ void fft_pass(const char* src, int srow, bool src_nat, char* dst, int drow, bool dst_nat,
                                         int nvalid) {
    constexpr int L = TB * NN * NN;
#pragma unroll 1
    for (int line = threadIdx.x; line < L; line += blockDim.x) {
        const int b = line / (NN * NN), l = line % (NN * NN), hi = l / NN, lo = l % NN;
        double2 v[NN];
        // natural / swizzled position of element x of this line (recomputed at the
        // store: the 2 NN indices would otherwise stay live across the butterflies)
        auto pos = [&](int x, bool natural) {
            const int i = AX == 0 ? x : hi, j = AX == 0 ? hi : (AX == 1 ? x : lo), kk = AX == 2 ? x : lo;
            return (i * NN + j) * NN + (natural ? kk : (kk ^ (j & (NN - 1))));
        };
        const char* srow_p = src + b * srow;
#pragma unroll
        for (int x = 0; x < NN; ++x) load_elem<SRCM>(srow_p, pos(x, src_nat), v[x].x, v[x].y);
        fft_line<NN, SIGN>(v);
        if (dst_nat && b >= nvalid) continue;
        char* drow_p = dst + b * drow;
#pragma unroll
        for (int x = 0; x < NN; ++x) store_elem<DSTM>(drow_p, pos(x, dst_nat), v[x].x, v[x].y);
    }
}

template <int NN, int DIR, int MI, int MO, int TMAX>
struct OfCfg {
    static constexpr int N = NN * NN * NN;
    static constexpr int G = 512 / N >= 1 ? 512 / N : 1;
    static constexpr int TB = 8 * G;
    static constexpr int EB = mode_bytes(MI) > mode_bytes(MO) ? mode_bytes(MI) : mode_bytes(MO);
    // Block rows rotate by 4 elements of the base change's access width: the 8
    // lanes of a quarter-warp (2 blocks x 4 members with positions distinct
    // mod 4, orbit_fft_host.cpp) then hit distinct banks. X is read by the
    // forward base change (MI) and written by the inverse one (MO).
    static constexpr int XROW = N * EB + 4 * mode_bytes(DIR == 0 ? MI : MO);
    static constexpr int YROW = (N + 4) * 16;
    static constexpr int META = kOfWarps * TMAX * 4 * 8;
    static constexpr int SMEM = 128 + META + 2 * TB * XROW + TB * YROW;
};

template <int NN, int DIR, int MI, int MO, int TMAX>
__global__ void __launch_bounds__(kOfWarps * 32, 1)
    orbit_fft_kernel(const __grid_constant__ OrbitFftDesc d, const void* __restrict__ in, void* __restrict__ out,
                     int64_t batch) {
    using C = OfCfg<NN, DIR, MI, MO, TMAX>;
    constexpr int N = C::N, TB = C::TB, G = C::G;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    int2* meta_s = reinterpret_cast<int2*>(smem + 128);
    char* Xb = reinterpret_cast<char*>(smem + 128 + C::META);
    char* Y = Xb + 2 * TB * C::XROW;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, k = lane & 3;

    double2 tab[TMAX];
#pragma unroll
    for (int t = 0; t < TMAX; ++t)
        tab[t] = t < d.tmax ? __ldg(d.table + (static_cast<size_t>(warp) * d.tmax + t) * 32 + lane) : make_double2(0, 0);
    for (int i = tid; i < kOfWarps * TMAX * 4; i += blockDim.x) {  // tiles beyond d.tmax: zero padding
        const int w = i / (TMAX * 4), rest = i - w * TMAX * 4;
        meta_s[i] = rest < d.tmax * 4 ? __ldg(d.meta + w * d.tmax * 4 + rest) : make_int2(0, -1);
    }
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int2* meta_w = meta_s + warp * TMAX * 4;

    const int64_t ntiles = (batch + TB - 1) / TB;
    constexpr uint32_t in_row = N * mode_bytes(MI), out_row = N * mode_bytes(MO);
    auto issue_load = [&](int buf, int64_t tile) {
        const int64_t t0 = tile * TB;
        const int nv = static_cast<int>(batch - t0 < TB ? batch - t0 : TB);
        char* X = Xb + buf * TB * C::XROW;
        mbar_arrive_expect_tx(bar + buf, in_row * nv);
        const char* src = static_cast<const char*>(in) + t0 * in_row;
        for (int b = 0; b < nv; ++b) tma_load_1d(X + b * C::XROW, src + static_cast<int64_t>(b) * in_row, in_row, bar + buf);
    };
    if (tid == 0) {
        if (static_cast<int64_t>(blockIdx.x) < ntiles) issue_load(0, blockIdx.x);
        if (static_cast<int64_t>(blockIdx.x) + gridDim.x < ntiles) issue_load(1, blockIdx.x + gridDim.x);
    }
    uint32_t phases = 0;  // bit b: parity of X[b]'s barrier
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        char* X = Xb + buf * TB * C::XROW;
        const int64_t t0 = tile * TB;
        const int nvalid = static_cast<int>(batch - t0 < TB ? batch - t0 : TB);
        if (DIR == 1 && it >= 1 && tid == 0) {
            // X[buf ^ 1] staged the previous tile's output: reload it once the bulk store has read it
            tma_store_wait_read0();
            const int64_t nx = tile + gridDim.x;
            if (nx < ntiles) issue_load(buf ^ 1, nx);
        }
        mbar_wait(bar + buf, (phases >> buf) & 1);
        phases ^= 1u << buf;
        if constexpr (DIR == 0) {
            base_change<TMAX, G, MI, OF_C128>(tab, meta_w, X, C::XROW, Y, C::YROW, r, k);
            __syncthreads();
            if (tid == 0) {
                const int64_t nx = tile + 2 * static_cast<int64_t>(gridDim.x);
                if (nx < ntiles) issue_load(buf, nx);  // X[buf] has been consumed
            }
            fft_pass<NN, +1, TB, 2, OF_C128, OF_C128>(Y, C::YROW, false, Y, C::YROW, false, TB);
            __syncthreads();
            fft_pass<NN, +1, TB, 1, OF_C128, OF_C128>(Y, C::YROW, false, Y, C::YROW, false, TB);
            __syncthreads();
            fft_pass<NN, +1, TB, 0, OF_C128, MO>(Y, C::YROW, false, static_cast<char*>(out) + t0 * out_row, out_row, true,
                                                 nvalid);
            __syncthreads();
        } else {
            fft_pass<NN, -1, TB, 0, MI, OF_C128>(X, C::XROW, true, Y, C::YROW, false, TB);
            __syncthreads();
            fft_pass<NN, -1, TB, 1, OF_C128, OF_C128>(Y, C::YROW, false, Y, C::YROW, false, TB);
            __syncthreads();
            fft_pass<NN, -1, TB, 2, OF_C128, OF_C128>(Y, C::YROW, false, Y, C::YROW, false, TB);
            __syncthreads();
            base_change<TMAX, G, OF_C128, MO>(tab, meta_w, Y, C::YROW, X, C::XROW, r, k);
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
                char* dst = static_cast<char*>(out) + t0 * out_row;
                for (int b = 0; b < nvalid; ++b) tma_store_1d(dst + static_cast<int64_t>(b) * out_row, X + b * C::XROW, out_row);
                tma_store_commit();
            }
        }
    }
    if (DIR == 1 && tid == 0) tma_store_wait0();
}

template <int NN, int DIR, int MI, int MO, int TMAX>
cudaError_t launch_t(const OrbitFftDesc& d, const void* in, void* out, int64_t batch, cudaStream_t st, int num_sms) {
    using C = OfCfg<NN, DIR, MI, MO, TMAX>;
    auto kern = orbit_fft_kernel<NN, DIR, MI, MO, TMAX>;
    static thread_local int prepared_dev = -1;  // attribute set once per device and thread
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (prepared_dev != dev) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        prepared_dev = dev;
    }
    const int64_t ntiles = (batch + C::TB - 1) / C::TB;
    const int64_t grid = std::min<int64_t>(ntiles, num_sms);
    kern<<<static_cast<unsigned>(grid), kOfWarps * 32, C::SMEM, st>>>(d, in, out, batch);
    return cudaGetLastError();
}

template <int NN, int TMAX>
cudaError_t launch_n(const OrbitFftDesc& d, int mi, int mo, const void* in, void* out, int64_t batch, cudaStream_t st,
                     int num_sms) {
    if (d.dir == 0) {
        if (mi == OF_C128 && mo == OF_C128) return launch_t<NN, 0, OF_C128, OF_C128, TMAX>(d, in, out, batch, st, num_sms);
        if (mi == OF_R64 && mo == OF_C128) return launch_t<NN, 0, OF_R64, OF_C128, TMAX>(d, in, out, batch, st, num_sms);
        if (mi == OF_C64 && mo == OF_C64) return launch_t<NN, 0, OF_C64, OF_C64, TMAX>(d, in, out, batch, st, num_sms);
        if (mi == OF_R32 && mo == OF_C64) return launch_t<NN, 0, OF_R32, OF_C64, TMAX>(d, in, out, batch, st, num_sms);
    } else {
        if (mi == OF_C128 && mo == OF_C128) return launch_t<NN, 1, OF_C128, OF_C128, TMAX>(d, in, out, batch, st, num_sms);
        if (mi == OF_C128 && mo == OF_R64) return launch_t<NN, 1, OF_C128, OF_R64, TMAX>(d, in, out, batch, st, num_sms);
        if (mi == OF_C64 && mo == OF_C64) return launch_t<NN, 1, OF_C64, OF_C64, TMAX>(d, in, out, batch, st, num_sms);
        if (mi == OF_C64 && mo == OF_R32) return launch_t<NN, 1, OF_C64, OF_R32, TMAX>(d, in, out, batch, st, num_sms);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_orbit_fft(const OrbitFftDesc& d, int in_mode, int out_mode, const void* in, void* out,
                             int64_t batch, cudaStream_t st, int num_sms) {
    if (batch <= 0) return cudaSuccess;
    if (d.n == 8 && d.tmax <= kOfTmax8) return launch_n<8, kOfTmax8>(d, in_mode, out_mode, in, out, batch, st, num_sms);
    if (d.n == 4 && d.tmax <= kOfTmax4) return launch_n<4, kOfTmax4>(d, in_mode, out_mode, in, out, batch, st, num_sms);
    return cudaErrorInvalidValue;
}

}  // namespace fcct
