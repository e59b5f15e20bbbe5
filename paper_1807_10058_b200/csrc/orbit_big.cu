// Large-n orbit-FFT executor (orbit_big.hpp): the orbit-block base change as a
// coalesced SIMT pass, and radix-2 line FFTs in shared memory per axis.
#include <algorithm>

#include "device.cuh"
#include "orbit_big.hpp"

namespace fcct {

using namespace dev;

namespace {

// y[b][members[off + r]] = sum_c coef[cbase + c s + r] x[b][members[off + c]]
// __launch_bounds__(256, 4): a 64-register cap. Unbounded, ptxas compiled 34
// registers and kept ~2 of a row's 24 coefficient loads in flight (latency
// bound: 29 us at n = 64). 62 registers hoist most of them with 4 CTAs per SM:
// 44 -> 35 us per direction. (256, 1) / 3 / 5 measured 46 / 36 / 38 us.
__global__ void __launch_bounds__(256, 4) orbit_big_s_kernel(const __grid_constant__ OrbitBigDesc d,
                                                          const double2* __restrict__ x, double2* __restrict__ y,
                                                          int64_t batch) {
    // no early trigger: this grid runs in several waves, and dependents
    // scheduled during them slowed the forward (60 vs 50 us at n = 64)
    const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= d.rows) return;
    // plan tables (constant) before the wait; x is the previous kernel's output
    const int o = __ldg(d.row_orbit + row), r = __ldg(d.row_index + row);
    const int off = __ldg(d.orbit_off + o), s = __ldg(d.orbit_off + o + 1) - off;
    const double2* __restrict__ cf = d.coef + __ldg(d.coef_off + o) + r;
    const int* __restrict__ mem = d.members + off;
    const int out = __ldg(mem + r);
    pdl_wait();
    for (int64_t b = 0; b < batch; ++b) {
        const double2* xb = x + b * d.N;
        double re = 0.0, im = 0.0;
        if (s == 24) {  // free orbits (almost every row at n = 64): all 24 coefficient loads in flight at once
            double2 m[24];
#pragma unroll
            for (int c = 0; c < 24; ++c) m[c] = __ldcs(cf + c * 24);
#pragma unroll
            for (int c = 0; c < 24; ++c) {
                const double2 v = __ldg(xb + __ldg(mem + c));
                re = fma(m[c].x, v.x, re);
                re = fma(-m[c].y, v.y, re);
                im = fma(m[c].x, v.y, im);
                im = fma(m[c].y, v.x, im);
            }
        } else {
#pragma unroll 4
            for (int c = 0; c < s; ++c) {
                const double2 m = __ldcs(cf + static_cast<int64_t>(c) * s);  // read once: streaming
                const double2 v = __ldg(xb + __ldg(mem + c));
                re = fma(m.x, v.x, re);
                re = fma(-m.y, v.y, re);
                im = fma(m.x, v.y, im);
                im = fma(m.y, v.x, im);
            }
        }
        y[b * d.N + out] = make_double2(re, im);
    }
}

// Forward S pass with generated coefficients (OrbitBigDesc::gen): rows of free
// orbits form S[r][c] = base_r T[t_c][g_r g_c^{-1}] from two small shared-memory
// tables instead of streaming the 104 MB coefficient stream (n = 64); rows of the
// few non-free orbits keep their coefficient blocks. Persistent grid-stride rows.
constexpr int kGenMaxCarry = 64;
constexpr int kGenOrbits = 10;  // free orbits per CTA: 240 of 256 threads, one row each
// CTAs after the tail: the members of 10 free orbits are staged in shared
// memory (x values and their decoded (T row, g) words), then each thread forms
// its row from shared memory only: y_r = base_r sum_c T[t_c][g_r g_c^-1] x_c.
// The first CTAs run the non-free orbits' rows on their coefficient blocks.
__global__ void __launch_bounds__(256, 4) orbit_big_sgen_kernel(const __grid_constant__ OrbitBigDesc d,
                                                                const double2* __restrict__ x,
                                                                double2* __restrict__ y, int64_t batch) {
    __shared__ __align__(16) double2 T[kGenMaxCarry * 24];
    __shared__ __align__(16) uint8_t Mt[24 * 24];
    __shared__ double2 xs[kGenOrbits * 24];
    __shared__ int ws[kGenOrbits * 24];   // T row offset (carry id x 24) of each member
    // the non-free orbits' rows (long serial coefficient chains) are scheduled first;
    // the remaining CTAs are persistent over groups of 10 free orbits, so the two
    // tables are loaded once per CTA (bulk copies, overlapped with the first group's
    // member words)
    const int tail_ctas = (d.ntail + 255) / 256;
    const int tid = threadIdx.x;
    if (static_cast<int>(blockIdx.x) >= tail_ctas) {
        __shared__ __align__(8) uint64_t tbar;
        const int nfc = static_cast<int>(gridDim.x) - tail_ctas;  // free-orbit CTAs
        const int groups = (d.nfree + kGenOrbits - 1) / kGenOrbits;
        const uint32_t tbytes = static_cast<uint32_t>(d.ncarry) * 24 * 16;
        if (tid == 0) {
            mbar_init(&tbar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(&tbar, tbytes + 24 * 24);
            tma_load_1d(T, d.ttab, tbytes, &tbar);
            tma_load_1d(Mt, d.mtab, 24 * 24, &tbar);
        }
        __syncthreads();  // the barrier is initialised before anyone waits on it
        const int ob = tid - tid % 24;  // first slot of this thread's orbit in the stage
        // slots are ordered by group element, so this row's g_r = tid % 24 and its
        // 24 values w = g_r g_c^-1 are one fixed row of the product table: packed
        // into registers once (bytes), no table lookup per term
        uint32_t wp[6] = {0, 0, 0, 0, 0, 0};
        bool waited = false;
        for (int grp = static_cast<int>(blockIdx.x) - tail_ctas; grp < groups; grp += nfc) {
            const int orbit = grp * kGenOrbits + tid / 24;
            const bool live = tid < kGenOrbits * 24 && orbit < d.nfree;
            const int64_t slot = static_cast<int64_t>(orbit) * 24 + tid % 24;
            const uint32_t me = live ? __ldg(d.fpack + slot) : 0u;
            const double2 base = live ? __ldg(d.fbase + slot) : make_double2(0.0, 0.0);
            const int nat = static_cast<int>(me & 0x3FFFFu), gr = static_cast<int>((me >> 24) & 31u);
            if (!waited) {
                pdl_wait();  // x is the previous kernel's output
                mbar_wait(&tbar, 0);
                waited = true;
                const int g0 = tid % 24;
#pragma unroll
                for (int q = 0; q < 6; ++q)
                    wp[q] = static_cast<uint32_t>(Mt[g0 * 24 + 4 * q]) | (static_cast<uint32_t>(Mt[g0 * 24 + 4 * q + 1]) << 8) |
                            (static_cast<uint32_t>(Mt[g0 * 24 + 4 * q + 2]) << 16) |
                            (static_cast<uint32_t>(Mt[g0 * 24 + 4 * q + 3]) << 24);
            } else {
                __syncthreads();  // the previous group's stage is consumed
            }
            if (live) ws[tid] = static_cast<int>((me >> 18) & 63u) * 24;
            (void)gr;
            for (int64_t b = 0; b < batch; ++b) {
                if (b > 0) __syncthreads();
                if (live) xs[tid] = __ldg(x + b * d.N + nat);
                __syncthreads();
                if (!live) continue;
                double re = 0.0, im = 0.0;
#pragma unroll
                for (int c = 0; c < 24; ++c) {
                    const double2 v = xs[ob + c];
                    const int w = static_cast<int>((wp[c >> 2] >> (8 * (c & 3))) & 0xFFu);
                    const double2 m = T[ws[ob + c] + w];
                    re = fma(m.x, v.x, re);
                    re = fma(-m.y, v.y, re);
                    im = fma(m.x, v.y, im);
                    im = fma(m.y, v.x, im);
                }
                y[b * d.N + nat] = make_double2(base.x * re - base.y * im, base.x * im + base.y * re);
            }
        }
        if (!waited) {
            pdl_wait();
            mbar_wait(&tbar, 0);  // the bulk copies must land before the CTA exits
        }
        return;
    }
    // non-free orbits (<= 12 members): their coefficient blocks, all loads in flight
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + tid;
    if (q >= d.ntail) return;
    const int64_t row = __ldg(d.tail + q);
    const int o = __ldg(d.row_orbit + row), r = __ldg(d.row_index + row);
    const int off = __ldg(d.orbit_off + o), s = __ldg(d.orbit_off + o + 1) - off;
    const double2* __restrict__ cf = d.coef + __ldg(d.coef_off + o) + r;
    const int* __restrict__ mem = d.members + off;
    const int out = __ldg(mem + r);
    int mi[12];
    double2 mc[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) {
        mi[c] = c < s ? __ldg(mem + c) : 0;
        mc[c] = c < s ? __ldg(cf + static_cast<int64_t>(c) * s) : make_double2(0.0, 0.0);
    }
    pdl_wait();
    for (int64_t b = 0; b < batch; ++b) {
        const double2* xb = x + b * d.N;
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
            const double2 v = c < s ? __ldg(xb + mi[c]) : make_double2(0.0, 0.0);
            re = fma(mc[c].x, v.x, re);
            re = fma(-mc[c].y, v.y, re);
            im = fma(mc[c].x, v.y, im);
            im = fma(mc[c].y, v.x, im);
        }
        y[b * d.N + out] = make_double2(re, im);
    }
}

constexpr int kLines = 8;  // lines per CTA (neighbours in the contiguous dimension)

// One radix-2 DIF FFT along `axis` for kLines neighbouring lines of n points.
template <int NN, int SIGN>
__global__ void __launch_bounds__(256) line_fft_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                       int axis, int64_t batch) {
    constexpr int N = NN * NN * NN, LOG = NN == 32 ? 5 : 6;
    __shared__ double2 buf[kLines][NN];
    __shared__ double2 tw[NN / 2];
    const int tid = threadIdx.x;
    pdl_trigger();
    for (int e = tid; e < NN / 2; e += blockDim.x) {
        double sv, cv;
        sincospi(2.0 * e / NN, &sv, &cv);
        tw[e] = make_double2(cv, SIGN * sv);
    }
    pdl_wait();  // the twiddles overlap the previous kernel's tail
    // line group g: lines (u, ., v0 + l) along the axis, l = 0..7 contiguous in memory
    const int64_t groups_per_block = static_cast<int64_t>(NN) * NN / kLines;
    const int64_t g = blockIdx.x;
    const int64_t b = g / groups_per_block;
    const int gi = static_cast<int>(g % groups_per_block);
    if (b >= batch) return;
    // strides: the line's own stride and the neighbour stride (1: contiguous)
    int64_t base, step;
    if (axis == 2) {  // k lines: rows (i, j) = consecutive lines, neighbours l -> j + l
        const int i = gi / (NN / kLines), j0 = (gi % (NN / kLines)) * kLines;
        base = (static_cast<int64_t>(i) * NN + j0) * NN;
        step = 1;  // along the line
    } else {
        const int u = gi / (NN / kLines), v0 = (gi % (NN / kLines)) * kLines;  // u: the other axis, v0: k
        base = axis == 1 ? static_cast<int64_t>(u) * NN * NN + v0 : static_cast<int64_t>(u) * NN + v0;
        step = axis == 1 ? NN : static_cast<int64_t>(NN) * NN;
    }
    const double2* src = in + b * N;
    double2* dst = out + b * N;
    for (int e = tid; e < kLines * NN; e += blockDim.x) {
        int l, x;
        if (axis == 2) {
            l = e / NN;
            x = e % NN;
        } else {  // neighbours innermost: coalesced 128-byte rows
            l = e % kLines;
            x = e / kLines;
        }
        const int64_t off = axis == 2 ? base + static_cast<int64_t>(l) * NN + x : base + l + x * step;
        buf[l][x] = src[off];
    }
    __syncthreads();
#pragma unroll 1
    for (int st = 0; st < LOG; ++st) {
        const int half = NN >> (st + 1);
        for (int e = tid; e < kLines * NN / 2; e += blockDim.x) {
            const int l = e / (NN / 2), q = e % (NN / 2);
            const int grp = q / half, j = q % half;
            const int i0 = grp * 2 * half + j, i1 = i0 + half;
            const double2 a = buf[l][i0], c = buf[l][i1];
            const double2 d = make_double2(a.x - c.x, a.y - c.y);
            const double2 w = tw[j << st];
            buf[l][i0] = make_double2(a.x + c.x, a.y + c.y);
            buf[l][i1] = make_double2(d.x * w.x - d.y * w.y, d.x * w.y + d.y * w.x);
        }
        __syncthreads();
    }
    for (int e = tid; e < kLines * NN; e += blockDim.x) {
        int l, x;
        if (axis == 2) {
            l = e / NN;
            x = e % NN;
        } else {
            l = e % kLines;
            x = e / kLines;
        }
        const int rx = __brev(static_cast<unsigned>(x)) >> (32 - LOG);  // DIF output is bit-reversed
        const int64_t off = axis == 2 ? base + static_cast<int64_t>(l) * NN + x : base + l + x * step;
        dst[off] = buf[l][rx];
    }
}

// 64-point lines as 8 x 8: thread t (0..7) of a line takes x[t + 8 m], runs
// an 8-point DFT over m, multiplies by w64^{t q}, exchanges through shared
// memory, and runs the 8-point DFT over t: X[q + 8 u] = sum_t w8^{t u} w64^{t q}
// sum_m w8^{m q} x[t + 8 m]. 32 lines per CTA (8 threads each), two barriers.
template <int SIGN>
__device__ __forceinline__ void dft8(double2 (&v)[8]) {
    // radix-2 DIF on 8 points, output in natural order
    const double h = 0.70710678118654752440;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double2 a = v[j], b = v[j + 4];
        v[j] = make_double2(a.x + b.x, a.y + b.y);
        double2 d = make_double2(a.x - b.x, a.y - b.y);
        if (j == 1) d = make_double2(h * (d.x - SIGN * d.y), h * (d.y + SIGN * d.x));
        if (j == 2) d = SIGN > 0 ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
        if (j == 3) d = make_double2(h * (-d.x - SIGN * d.y), h * (-d.y + SIGN * d.x));
        v[j + 4] = d;
    }
#pragma unroll
    for (int g = 0; g < 8; g += 4)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const double2 a = v[g + j], b = v[g + j + 2];
            v[g + j] = make_double2(a.x + b.x, a.y + b.y);
            double2 d = make_double2(a.x - b.x, a.y - b.y);
            if (j == 1) d = SIGN > 0 ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
            v[g + j + 2] = d;
        }
#pragma unroll
    for (int g = 0; g < 8; g += 2) {
        const double2 a = v[g], b = v[g + 1];
        v[g] = make_double2(a.x + b.x, a.y + b.y);
        v[g + 1] = make_double2(a.x - b.x, a.y - b.y);
    }
    double2 t[8];
    constexpr int br[8] = {0, 4, 2, 6, 1, 5, 3, 7};
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = v[br[q]];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = t[q];
}

template <int SIGN>
__global__ void __launch_bounds__(256) line_fft64_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                         int axis, int64_t batch) {
    constexpr int NN = 64, N = NN * NN * NN, LPC = 32;  // lines per CTA
    __shared__ double2 ex[LPC][8][9];                   // [line][t][q], padded
    __shared__ double2 tw[NN];                          // w64^e
    const int tid = threadIdx.x, t = tid & 7, li = tid >> 3;  // 8 threads per line
    pdl_trigger();
    if (tid < NN) {
        double sv, cv;
        sincospi(2.0 * tid / NN, &sv, &cv);
        tw[tid] = make_double2(cv, SIGN * sv);
    }
    __syncthreads();
    pdl_wait();  // the twiddles overlap the previous kernel's tail
    const int64_t line = static_cast<int64_t>(blockIdx.x) * LPC + li;  // global line id
    const int64_t b = line / (NN * NN);
    if (b >= batch) return;
    const int gi = static_cast<int>(line % (NN * NN));
    // line start and stride along the axis; neighbouring lines are adjacent in
    // the contiguous dimension for the i and j axes (coalesced across li)
    int64_t base, step;
    if (axis == 2) {
        base = static_cast<int64_t>(gi) * NN;
        step = 1;
    } else if (axis == 1) {
        base = static_cast<int64_t>(gi / NN) * NN * NN + gi % NN;
        step = NN;
    } else {
        base = gi;
        step = static_cast<int64_t>(NN) * NN;
    }
    const double2* src = in + b * N + base;
    double2* dst = out + b * N + base;
    double2 v[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) v[m] = src[(t + 8 * m) * step];
    dft8<SIGN>(v);  // over m -> q
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const double2 w = tw[t * q];  // t q < 64
        ex[li][t][q] = make_double2(v[q].x * w.x - v[q].y * w.y, v[q].x * w.y + v[q].y * w.x);
    }
    __syncwarp();
    // thread t now takes q = t: the 8 values over t' (the second DFT's input)
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ex[li][u][t];
    dft8<SIGN>(v);  // over t' -> u: X[t + 8 u]
#pragma unroll
    for (int u = 0; u < 8; ++u) dst[(t + 8 * u) * step] = v[u];
}

bool pdl_enabled() {
    static const bool on = [] {
#ifdef FCCT_AB_SWITCHES  // A/B timing builds only (capi.cpp ab_env)
        const char* e = std::getenv("FCCT_PDL");
        return !(e && e[0] == '0');
#else
        return true;
#endif
    }();
    return on;
}

// launch with programmatic stream serialisation: the kernel may start while
// the previous one in the stream drains; it waits (pdl_wait) before touching
// that kernel's output
template <typename... P, typename... A>
cudaError_t launch_pdl(void (*kern)(P...), unsigned grid, unsigned block, cudaStream_t st, A... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<P>(args)...);
}

}  // namespace

cudaError_t launch_orbit_big_s(const OrbitBigDesc& d, const void* in, void* out, int64_t batch, cudaStream_t st) {
    if (batch <= 0) return cudaSuccess;
    const int64_t blocks = (d.rows + 255) / 256;
    if (d.gen) {
        if (d.ncarry > kGenMaxCarry) return cudaErrorInvalidValue;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t grid = std::min<int64_t>((d.nfree + kGenOrbits - 1) / kGenOrbits, 4LL * sms) + (d.ntail + 255) / 256;
        return launch_pdl(orbit_big_sgen_kernel, static_cast<unsigned>(grid), 256, st, d,
                          static_cast<const double2*>(in), static_cast<double2*>(out), batch);
    }
    return launch_pdl(orbit_big_s_kernel, static_cast<unsigned>(blocks), 256, st, d, static_cast<const double2*>(in),
                      static_cast<double2*>(out), batch);
}

cudaError_t launch_line_fft(int n, int axis, int sign, const void* in, void* out, int64_t batch, cudaStream_t st) {
    if (batch <= 0) return cudaSuccess;
    const int64_t grid = batch * static_cast<int64_t>(n) * n / kLines;
    auto* i = static_cast<const double2*>(in);
    auto* o = static_cast<double2*>(out);
    if (n == 64) {  // 8 x 8 decomposition, 32 lines per CTA
        const unsigned g64 = static_cast<unsigned>(batch * 64 * 64 / 32);
        return sign > 0 ? launch_pdl(line_fft64_kernel<1>, g64, 256, st, i, o, axis, batch)
                        : launch_pdl(line_fft64_kernel<-1>, g64, 256, st, i, o, axis, batch);
    }
    if (n == 32)
        return sign > 0 ? launch_pdl(line_fft_kernel<32, 1>, static_cast<unsigned>(grid), 256, st, i, o, axis, batch)
                        : launch_pdl(line_fft_kernel<32, -1>, static_cast<unsigned>(grid), 256, st, i, o, axis, batch);
    return cudaErrorInvalidValue;
}

}  // namespace fcct
