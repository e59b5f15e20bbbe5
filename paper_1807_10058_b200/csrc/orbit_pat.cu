// Single-pass orbit-pattern executor (orbit_pat.hpp): one transform block per
// CTA iteration, resident in a 64 KB shared tile from load to store — the base
// change as a register-resident constant-operator DMMA over the block's own
// orbits, in place, and the 16^3 radix-2 FFT in the same tile.
#include <algorithm>

#include "orbit_dev.cuh"
#include "orbit_pat.hpp"

namespace fcct {

using namespace dev;
using namespace odev;

namespace {

constexpr int kPatThreads = kPatWarps * 32;
constexpr int kPatCtas = kPatWarps == 4 ? 3 : 2;        // CTAs per SM
constexpr int kPatLines = 256 / kPatThreads;             // FFT lines per thread per pass

// One DMMA class: orbits of D members sharing the operator M (D x D complex).
// MMA roles: A = data, 8 orbits x 4 members per k-step (lane: orbit lane / 4,
// member 4 q + lane % 4); B = M^T fragments in registers (k = member, n = output
// row); C[orbit][row]: this lane's rows 8 nt + 2 (lane % 4) + {0, 1}.
// An orbit is read and written by this warp only, and every fragment of a tile
// is loaded before its last DMMA issues, so the tile is updated in place.
template <int D>
struct PatOp {
    static constexpr int KT = D / 4, NT = (D + 7) / 8;
    double br[KT][NT], bi[KT][NT];
    __device__ __forceinline__ void load(const double2* __restrict__ op, int lane) {
#pragma unroll
        for (int q = 0; q < KT; ++q)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const double2 v = __ldg(op + (q * NT + nt) * 32 + lane);
                br[q][nt] = v.x;
                bi[q][nt] = v.y;
            }
    }
};

template <int D, bool RIN, bool ROUT>
__device__ __forceinline__ void pat_class(double* Re, double* Im, const uint16_t* ix0, const PatOp<D>& op, int first,
                                          int count, int cnt, int lane) {
    constexpr int KT = D / 4, NT = (D + 7) / 8;
    const int o = lane >> 2, k = lane & 3;
    for (int t = first; t < first + count; ++t) {
        const uint16_t* ix = ix0 + t * (D * 8);
        double cr[NT][2], ci[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) cr[nt][0] = cr[nt][1] = ci[nt][0] = ci[nt][1] = 0.0;
        double ar[KT], ai[KT];
#pragma unroll
        for (int q = 0; q < KT; ++q) {
            const int slot = ix[(4 * q + k) * 8 + o];
            ar[q] = Re[slot];
            ai[q] = RIN ? 0.0 : Im[slot];
        }
#pragma unroll
        for (int q = 0; q < KT; ++q) {
            const double xr = ar[q], xi = ai[q], nxi = neg_hi16(xi);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                dmma884(cr[nt][0], cr[nt][1], xr, op.br[q][nt]);
                if constexpr (!ROUT) dmma884(ci[nt][0], ci[nt][1], xr, op.bi[q][nt]);
                if constexpr (!RIN) {
                    dmma884(cr[nt][0], cr[nt][1], nxi, op.bi[q][nt]);
                    if constexpr (!ROUT) dmma884(ci[nt][0], ci[nt][1], xi, op.br[q][nt]);
                }
            }
        }
        const bool valid = t * 8 + o < cnt;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = 8 * nt + 2 * k + e;
                if ((D % 8 == 0 || row < D) && valid) {
                    const int slot = ix[row * 8 + o];
                    Re[slot] = cr[nt][e];
                    if constexpr (!ROUT) Im[slot] = ci[nt][e];
                }
            }
    }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// The tile: two planes of n^3 doubles (Re, Im). Natural order (slot = lexicographic
// index) while the base change runs and on the load / store side, so a real block
// is ONE bulk copy (TMA) into / out of the Re plane; (i, j, k ^ j) for the k-axis
// pass. The j-axis pass converts between the two for free: a row (i, j, .) is
// read and written by the 16 lanes of one instruction.
template <int DIR, int MI, int MO>
__global__ void __launch_bounds__(kPatThreads, kPatCtas)
    orbit_pat_kernel(const __grid_constant__ OrbitPatDesc d, const void* __restrict__ in, void* __restrict__ out,
                     int64_t batch) {
    constexpr int NN = 16, N = NN * NN * NN, SIGN = DIR == 0 ? +1 : -1;
    constexpr bool RIN = DIR == 0 && (MI == OF_R64 || MI == OF_R32);
    constexpr bool ROUT = DIR == 1 && (MO == OF_R64 || MO == OF_R32);
    constexpr bool TMA_IN = DIR == 0 && MI == OF_R64, TMA_OUT = DIR == 1 && MO == OF_R64;
    extern __shared__ __align__(128) unsigned char smem[];
    double* Re = reinterpret_cast<double*>(smem);
    double* Im = Re + N;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + N * 16);
    uint16_t* ix_s = reinterpret_cast<uint16_t*>(smem + N * 16 + 16);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (TMA_IN && tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    for (int i = tid; i < d.idx_count / 2; i += kPatThreads)
        reinterpret_cast<uint32_t*>(ix_s)[i] = __ldg(reinterpret_cast<const uint32_t*>(d.idx) + i);
    const int2 wa = __ldg(d.warp_tiles + warp), wb = __ldg(d.warp_tiles + kPatWarps + warp);
    const uint16_t* ix_b = ix_s + d.ntiles[0] * (24 * 8);
    int rout[kPatMaxRare];  // this thread's rare rows (SIMT): output slots
#pragma unroll
    for (int u = 0; u < kPatMaxRare; ++u)
        rout[u] = tid + u * kPatThreads < d.nrare ? __ldg(d.rare_out + tid + u * kPatThreads) : -1;
    __syncthreads();
    constexpr int64_t in_row = int64_t{N} * eb_of(MI), out_row = int64_t{N} * eb_of(MO);
    auto nat = [](int i, int j, int k) { return (i * NN + j) * NN + k; };
    auto swz = [](int i, int j, int k) { return (i * NN + j) * NN + (k ^ j); };
    // one line of the cube FFT in registers; the axis' share of Lambda multiplies
    // it before (forward) or after (inverse) the butterflies
    auto line_fft = [&](double2 (&v)[NN], const double2 (&lax)[16]) {
        if constexpr (DIR == 0) {
#pragma unroll
            for (int x = 0; x < NN; ++x) v[x] = cmul(v[x], lax[x]);
        }
        fft_line16<NN, SIGN>(v);
        if constexpr (DIR == 1) {
#pragma unroll
            for (int x = 0; x < NN; ++x) v[x] = cmul(v[x], lax[x]);
        }
    };
    // in-place pass over the tile, two lines per thread: rd / wr give the slot of
    // element x of line (hi, lo)
    auto pass = [&](auto rd, auto wr, const double2 (&lax)[16]) {
#pragma unroll 1
        for (int h = 0; h < kPatLines; ++h) {
            const int line = tid + h * kPatThreads, hi = line >> 4, lo = line & 15;
            double2 v[NN];
#pragma unroll
            for (int x = 0; x < NN; ++x) v[x] = make_double2(Re[rd(hi, lo, x)], Im[rd(hi, lo, x)]);
            line_fft(v, lax);
#pragma unroll
            for (int x = 0; x < NN; ++x) {
                Re[wr(hi, lo, x)] = v[x].x;
                Im[wr(hi, lo, x)] = v[x].y;
            }
        }
    };
    uint32_t phase = 0;
    for (int64_t blk = blockIdx.x; blk < batch; blk += gridDim.x) {
        const char* src = static_cast<const char*>(in) + blk * in_row;
        char* dst = static_cast<char*>(out) + blk * out_row;
        PatOp<24> opa;
        if (tid == 0 && blk + gridDim.x < batch)  // the block after this one, into L2
            prefetch_l2_bulk(src + static_cast<int64_t>(gridDim.x) * in_row, static_cast<uint32_t>(in_row));
        if constexpr (DIR == 0) {
            if constexpr (TMA_IN) {  // a real block: one bulk copy into the Re plane
                if (tid == 0) {
                    mbar_arrive_expect_tx(bar, N * 8);
                    tma_load_1d(Re, src, N * 8, bar);
                }
            } else {
#pragma unroll 8
                for (int a = tid; a < N; a += kPatThreads) {
                    {
                        double re, im;
                        ld_el<MI>(src, a, re, im);
                        Re[a] = re;
                        if constexpr (!RIN) Im[a] = im;
                    }
                }
                cp_async_commit();
            }
            opa.load(d.op[0], lane);  // the operator fragments arrive while the tile loads
            if constexpr (TMA_IN) {
                mbar_wait(bar, phase);
                phase ^= 1;
            } else {
                cp_async_wait<0>();
                __syncthreads();
            }
        } else {
            // i axis straight from HBM (lanes vary k: coalesced), written in the k-pass layout
            if constexpr (kPatLines == 1) {
                const int hi = tid >> 4, lo = tid & 15;
                double2 v[NN];
#pragma unroll
                for (int x = 0; x < NN; ++x) ld_el<MI>(src, nat(x, hi, lo), v[x].x, v[x].y);
                line_fft(v, d.lax[0]);
#pragma unroll
                for (int x = 0; x < NN; ++x) {
                    Re[swz(x, hi, lo)] = v[x].x;
                    Im[swz(x, hi, lo)] = v[x].y;
                }
            } else {
                const int hi = tid >> 4, lo = tid & 15;  // lines tid and tid + 128: (hi, lo) and (hi + 8, lo)
                double2 v[NN], w[NN];
#pragma unroll
                for (int x = 0; x < NN; ++x) ld_el<MI>(src, nat(x, hi, lo), v[x].x, v[x].y);
#pragma unroll
                for (int x = 0; x < NN; ++x) ld_el<MI>(src, nat(x, hi + 8, lo), w[x].x, w[x].y);
                line_fft(v, d.lax[0]);
#pragma unroll
                for (int x = 0; x < NN; ++x) {
                    Re[swz(x, hi, lo)] = v[x].x;
                    Im[swz(x, hi, lo)] = v[x].y;
                }
                line_fft(w, d.lax[0]);
#pragma unroll
                for (int x = 0; x < NN; ++x) {
                    Re[swz(x, hi + 8, lo)] = w[x].x;
                    Im[swz(x, hi + 8, lo)] = w[x].y;
                }
            }
            __syncthreads();
            pass([&](int hi, int lo, int x) { return swz(hi, lo, x); }, [&](int hi, int lo, int x) { return swz(hi, lo, x); },
                 d.lax[2]);
            __syncthreads();
            pass([&](int hi, int lo, int x) { return swz(hi, x, lo); }, [&](int hi, int lo, int x) { return nat(hi, x, lo); },
                 d.lax[1]);
            opa.load(d.op[0], lane);
            __syncthreads();
        }
        // base change, in place: the rare rows first (into registers, all their
        // loads in flight at once), then the two DMMA classes
        double2 racc[kPatMaxRare];
#pragma unroll
        for (int u = 0; u < kPatMaxRare; ++u) {
            racc[u] = make_double2(0.0, 0.0);
            if (rout[u] >= 0) {
                const int r = tid + u * kPatThreads;
                double2 c[kPatRareTerms];
                int sl[kPatRareTerms];
#pragma unroll
                for (int t = 0; t < kPatRareTerms; ++t) {
                    c[t] = __ldg(d.rare_coef + t * d.rare_pitch + r);
                    sl[t] = __ldg(d.rare_in + t * d.rare_pitch + r);
                }
#pragma unroll
                for (int t = 0; t < kPatRareTerms; ++t) {
                    const double xr = Re[sl[t]];
                    racc[u].x = fma(c[t].x, xr, racc[u].x);
                    racc[u].y = fma(c[t].y, xr, racc[u].y);
                    if constexpr (!RIN) {
                        const double xi = Im[sl[t]];
                        racc[u].x = fma(-c[t].y, xi, racc[u].x);
                        racc[u].y = fma(c[t].x, xi, racc[u].y);
                    }
                }
            }
        }
        pat_class<24, RIN, ROUT>(Re, Im, ix_s, opa, wa.x, wa.y, d.cnt[0], lane);
        PatOp<12> opb;
        opb.load(d.op[1], lane);
        pat_class<12, RIN, ROUT>(Re, Im, ix_b, opb, wb.x, wb.y, d.cnt[1], lane);
        __syncthreads();  // the rare rows have been read by everyone
#pragma unroll
        for (int u = 0; u < kPatMaxRare; ++u)
            if (rout[u] >= 0) {
                Re[rout[u]] = racc[u].x;
                if constexpr (!ROUT) Im[rout[u]] = racc[u].y;
            }
        if constexpr (TMA_OUT) fence_proxy_async_smem();
        __syncthreads();
        if constexpr (DIR == 0) {
            pass([&](int hi, int lo, int x) { return nat(hi, x, lo); }, [&](int hi, int lo, int x) { return swz(hi, x, lo); },
                 d.lax[1]);
            __syncthreads();
            pass([&](int hi, int lo, int x) { return swz(hi, lo, x); }, [&](int hi, int lo, int x) { return swz(hi, lo, x); },
                 d.lax[2]);
            __syncthreads();
            // i axis, stored to HBM from registers (lanes vary k: coalesced)
#pragma unroll 1
            for (int h = 0; h < kPatLines; ++h) {
                const int line = tid + h * kPatThreads, hi = line >> 4, lo = line & 15;
                double2 v[NN];
#pragma unroll
                for (int x = 0; x < NN; ++x) v[x] = make_double2(Re[swz(x, hi, lo)], Im[swz(x, hi, lo)]);
                line_fft(v, d.lax[0]);
#pragma unroll
                for (int x = 0; x < NN; ++x) st_el<MO>(dst, nat(x, hi, lo), v[x].x, v[x].y);
            }
            __syncthreads();  // the tile is refilled by the next block
        } else if constexpr (TMA_OUT) {  // a real block: one bulk copy out of the Re plane
            if (tid == 0) {
                tma_store_1d(dst, Re, N * 8);
                tma_store_commit();
                tma_store_wait_read0();
            }
            __syncthreads();
        } else {
#pragma unroll 8
            for (int a = tid; a < N; a += kPatThreads) st_el<MO>(dst, a, Re[a], ROUT ? 0.0 : Im[a]);
            __syncthreads();
        }
    }
}

template <int DIR, int MI, int MO>
cudaError_t launch_pat(const OrbitPatDesc& d, const void* in, void* out, int64_t batch, cudaStream_t st, int num_sms) {
    const int smem = 16 * 16 * 16 * 16 + 16 + ((d.idx_count * 2 + 15) / 16) * 16;
    auto kern = orbit_pat_kernel<DIR, MI, MO>;
    static thread_local int prepared = -1;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (prepared != dev) {  // the bound compile_orbit_pat enforces on the slot lists (10 KB), not this plan's size
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 16 * 16 * 16 + 16 + 10 * 1024);
        if (e != cudaSuccess) return e;
        prepared = dev;
    }
    kern<<<static_cast<unsigned>(std::min<int64_t>(batch, kPatCtas * static_cast<int64_t>(num_sms))), kPatThreads, smem, st>>>(
        d, in, out, batch);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Large n (32, 64): the S pass of a transform that lives in L2. One warp per
// tile of 8 orbits: fragments gathered from global memory, the constant
// operator in registers, results scattered to the output row; Lambda from
// three n-entry tables in shared memory. The CTAs after the tile CTAs run the
// rare shapes' rows, one thread per row.
// ---------------------------------------------------------------------------
struct LamTab {
    const double2* t;  // shared: [3][n]
    int n, lg;
    __device__ __forceinline__ double2 operator()(int a) const {
        const int k = a & (n - 1), j = (a >> lg) & (n - 1), i = a >> (2 * lg);
        return cmul(cmul(t[i], t[n + j]), t[2 * n + k]);
    }
};

template <int D, int DIR>
__device__ __forceinline__ void pat_big_tile(const OrbitPatBigDesc& d, const LamTab& lam, const int32_t* __restrict__ ix,
                                             const double2* __restrict__ opt, int valid_orbits,
                                             const double2* __restrict__ x, double2* __restrict__ y, int64_t batch,
                                             int lane) {
    constexpr int KT = D / 4, NT = (D + 7) / 8;
    PatOp<D> op;
    op.load(opt, lane);
    const int o = lane >> 2, k = lane & 3;
    int gs[KT], ss[NT][2];
#pragma unroll
    for (int q = 0; q < KT; ++q) gs[q] = __ldg(ix + (4 * q + k) * 8 + o);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int row = 8 * nt + 2 * k + e;
            ss[nt][e] = (D % 8 == 0 || row < D) && o < valid_orbits ? __ldg(ix + row * 8 + o) : -1;
        }
    pdl_wait();  // x is the previous kernel's output; the tables above are the plan's
    for (int64_t b = 0; b < batch; ++b) {
        const double2* xb = x + b * d.N;
        double2* yb = y + b * d.N;
        double2 a[KT];
#pragma unroll
        for (int q = 0; q < KT; ++q) a[q] = __ldg(xb + gs[q]);
        double cr[NT][2], ci[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) cr[nt][0] = cr[nt][1] = ci[nt][0] = ci[nt][1] = 0.0;
#pragma unroll
        for (int q = 0; q < KT; ++q) {
            if constexpr (DIR == 1) a[q] = cmul(a[q], lam(gs[q]));
            const double xr = a[q].x, xi = a[q].y, nxi = neg_hi16(xi);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                dmma884(cr[nt][0], cr[nt][1], xr, op.br[q][nt]);
                dmma884(ci[nt][0], ci[nt][1], xr, op.bi[q][nt]);
                dmma884(cr[nt][0], cr[nt][1], nxi, op.bi[q][nt]);
                dmma884(ci[nt][0], ci[nt][1], xi, op.br[q][nt]);
            }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (ss[nt][e] >= 0) {
                    double2 v = make_double2(cr[nt][e], ci[nt][e]);
                    if constexpr (DIR == 0) v = cmul(v, lam(ss[nt][e]));
                    yb[ss[nt][e]] = v;
                }
    }
}

template <int DIR>
__global__ void __launch_bounds__(128, 3)
    orbit_pat_big_kernel(const __grid_constant__ OrbitPatBigDesc d, const double2* __restrict__ x,
                         double2* __restrict__ y, int64_t batch, int tile_ctas) {
    __shared__ double2 lax_s[3 * 64];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 3 * d.n; i += 128) lax_s[i] = __ldg(d.lax + i);
    __syncthreads();
    const LamTab lam{lax_s, d.n, d.log2n};
    if (static_cast<int>(blockIdx.x) < tile_ctas) {
        const int t = blockIdx.x * 4 + warp, ta = d.ntiles[0];
        if (t < ta)
            pat_big_tile<24, DIR>(d, lam, d.idx + static_cast<int64_t>(t) * (24 * 8), d.op[0], d.cnt[0] - t * 8, x, y,
                                  batch, lane);
        else if (t < ta + d.ntiles[1])
            pat_big_tile<12, DIR>(d, lam, d.idx + static_cast<int64_t>(ta) * (24 * 8) + static_cast<int64_t>(t - ta) * (12 * 8),
                                  d.op[1], d.cnt[1] - (t - ta) * 8, x, y, batch, lane);
        return;
    }
    const int r = (blockIdx.x - tile_ctas) * 128 + tid;
    if (r >= d.nrare) return;
    double2 c[kPatRareTerms];
    int sl[kPatRareTerms];
#pragma unroll
    for (int t = 0; t < kPatRareTerms; ++t) {
        c[t] = __ldg(d.rare_coef + static_cast<int64_t>(t) * d.rare_pitch + r);
        sl[t] = __ldg(d.rare_in + static_cast<int64_t>(t) * d.rare_pitch + r);
    }
    const int out = __ldg(d.rare_out + r);
    pdl_wait();
    for (int64_t b = 0; b < batch; ++b) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < kPatRareTerms; ++t) {
            double2 v = __ldg(x + b * d.N + sl[t]);
            if constexpr (DIR == 1) v = cmul(v, lam(sl[t]));
            acc.x = fma(c[t].x, v.x, acc.x);
            acc.x = fma(-c[t].y, v.y, acc.x);
            acc.y = fma(c[t].x, v.y, acc.y);
            acc.y = fma(c[t].y, v.x, acc.y);
        }
        if constexpr (DIR == 0) acc = cmul(acc, lam(out));
        y[b * d.N + out] = acc;
    }
}

}  // namespace

cudaError_t launch_orbit_pat_big(const OrbitPatBigDesc& d, const void* in, void* out, int64_t batch, cudaStream_t st) {
    if (batch <= 0) return cudaSuccess;
    if (d.n > 64 || in == out) return cudaErrorInvalidValue;
    const int tile_ctas = (d.ntiles[0] + d.ntiles[1] + 3) / 4, rare_ctas = (d.nrare + 127) / 128;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(tile_ctas + rare_ctas));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto* x = static_cast<const double2*>(in);
    auto* y = static_cast<double2*>(out);
    return d.dir == 0 ? cudaLaunchKernelEx(&cfg, orbit_pat_big_kernel<0>, d, x, y, batch, tile_ctas)
                      : cudaLaunchKernelEx(&cfg, orbit_pat_big_kernel<1>, d, x, y, batch, tile_ctas);
}

cudaError_t launch_orbit_pat(const OrbitPatDesc& d, int in_mode, int out_mode, const void* in, void* out,
                             int64_t batch, cudaStream_t st, int num_sms) {
    if (batch <= 0) return cudaSuccess;
    if (d.n != 16 || d.nrare > kPatMaxRare * kPatThreads) return cudaErrorInvalidValue;
    if (d.dir == 0) {
        if (out_mode == OF_C128) switch (in_mode) {
                case OF_C128: return launch_pat<0, OF_C128, OF_C128>(d, in, out, batch, st, num_sms);
                case OF_C64: return launch_pat<0, OF_C64, OF_C128>(d, in, out, batch, st, num_sms);
                case OF_R64: return launch_pat<0, OF_R64, OF_C128>(d, in, out, batch, st, num_sms);
                case OF_R32: return launch_pat<0, OF_R32, OF_C128>(d, in, out, batch, st, num_sms);
            }
        if (out_mode == OF_C64) switch (in_mode) {
                case OF_C128: return launch_pat<0, OF_C128, OF_C64>(d, in, out, batch, st, num_sms);
                case OF_C64: return launch_pat<0, OF_C64, OF_C64>(d, in, out, batch, st, num_sms);
                case OF_R64: return launch_pat<0, OF_R64, OF_C64>(d, in, out, batch, st, num_sms);
                case OF_R32: return launch_pat<0, OF_R32, OF_C64>(d, in, out, batch, st, num_sms);
            }
    } else {
        if (in_mode == OF_C128) switch (out_mode) {
                case OF_C128: return launch_pat<1, OF_C128, OF_C128>(d, in, out, batch, st, num_sms);
                case OF_C64: return launch_pat<1, OF_C128, OF_C64>(d, in, out, batch, st, num_sms);
                case OF_R64: return launch_pat<1, OF_C128, OF_R64>(d, in, out, batch, st, num_sms);
                case OF_R32: return launch_pat<1, OF_C128, OF_R32>(d, in, out, batch, st, num_sms);
            }
        if (in_mode == OF_C64) switch (out_mode) {
                case OF_C128: return launch_pat<1, OF_C64, OF_C128>(d, in, out, batch, st, num_sms);
                case OF_C64: return launch_pat<1, OF_C64, OF_C64>(d, in, out, batch, st, num_sms);
                case OF_R64: return launch_pat<1, OF_C64, OF_R64>(d, in, out, batch, st, num_sms);
                case OF_R32: return launch_pat<1, OF_C64, OF_R32>(d, in, out, batch, st, num_sms);
            }
    }
    return cudaErrorInvalidValue;
}

}  // namespace fcct
