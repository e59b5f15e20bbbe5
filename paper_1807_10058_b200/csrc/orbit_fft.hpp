// Orbit-FFT executor of a fast plan: the paper's radix-2x2x2 recursion with
// its inner base changes telescoped.
//
// A radix node factors D_n(p) = P (+)_c D_m(p_c) (K (x) I) B (transform.cpp:
// 429-460), and the exact derivation of B (plan.hpp) reads
//     (K (x) I) B = (+)_c S_m(p_c)^{-1} Phi S_n(p),     D_m(p_c) = F_m S_m(p_c),
// so every child's base change S_m(p_c) cancels against its parent's
// S_m(p_c)^{-1}:
//     D_n(p) = P (+)_c F_m  Phi  S_n(p) = F_n S_n(p),
// P (+)F_m Phi being one radix-2 decimation step of the DFT on Z_n^3.
// Recursing to the leaves leaves ONE base change (the orbit-block diagonal
// S_n(p), blocks <= 24 x 24) followed by the radix-2 FFT in each axis:
//     forward  y = F_n S_n x           (F_n[ijk, a] = e^{+2 pi i a.ijk / n})
//     inverse  x = S_n^{-1} F_n^{-1} y (F_n^{-1} = conj(F_n)^T / n^3)
// The base change runs on the FP64 tensor pipe (DMMA m8n8k4, 8 transform
// blocks per m-tile, complex operator in real form), the FFT on the FP64
// SIMT pipe from shared memory. Per point at n = 8 this is sum|O|^2 / N =
// 15.7 complex MACs plus 3 x 7 FFT flops: ~60% of the stage-by-stage tree.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <vector>

namespace fcct {

constexpr int kOfWarps = 16;   // warps per CTA (one CTA per SM)
// Phased kernel: all 16 warps run the base change, then the FFT passes.
constexpr int kOfTmax8 = 19;   // register-resident table tiles per warp, n = 8
constexpr int kOfTmax4 = 4;    // n = 4
// Warp-specialised kernel: 12 base-change warps (the register-resident table
// split 12 ways) and 4 FFT warps that run the previous tile's line passes
// concurrently, through three rotating tile buffers. Warp w runs on SMSP
// w % 4: each SMSP carries 3 base-change warps and 1 FFT warp. (Measured:
// 14 + 2 warps leaves the FFT group the bottleneck, 0.397 vs 0.311 ms.)
constexpr int kOfBcWarps = 12;
constexpr int kOfWsTmax8 = 25;
constexpr int kOfWsTmax4 = 4;

// I/O element modes of the global rows (same codes as the two-level executor).
enum OfMode { OF_C128 = 0, OF_C64 = 1, OF_R64 = 2, OF_R32 = 3 };

struct OrbitFftDesc {
    int n = 0;
    int N = 0;        // n^3
    int dir = 0;      // 0 forward (S then FFT+), 1 inverse (FFT- then S^{-1}/N)
    int groups = 1;   // 8-block m-tile groups per CTA tile (tile = 8 * groups blocks)
    int tmax = 0;     // table tiles per warp (<= the kernel's compile-time bound)
    int warps = kOfWarps;  // base-change warps the table is split over (16 phased, 12 specialised)
    int64_t in_stride = 0;   // bytes between input block rows (0: dense rows); specialised kernel only
    int64_t out_stride = 0;  // bytes between output block rows (0: dense rows)
    // B fragments of the orbit-block operator, [warp][tmax][32 lanes] (Re, Im):
    // lane l holds M[row 8 nt + l/4][col 4 kt + l%4] of its tile (0 outside the block)
    const double2* table = nullptr;
    // per tile and lane quad k = lane % 4: x = in_pos | flags << 16 (bit 0 chain start,
    // bit 1 chain end), y = out_pos(2k) | out_pos(2k+1) << 16 (0xFFFF: padding row)
    const int2* meta = nullptr;  // [warp][tmax][4]
    const int* ntiles = nullptr; // [warp]
};

// Host image of the tables (also what the CPU emulation runs).
struct OrbitFftHost {
    int n = 0, N = 0, dir = 0, groups = 1, tmax = 0, warps = kOfWarps;
    std::vector<double> table;    // [warp][tmax][32][2]
    std::vector<int32_t> meta;    // [warp][tmax][4][2]
    std::vector<int32_t> ntiles;  // [warp]
    int64_t tiles = 0;            // DMMA tiles (4 x 8) over all warps
    // FP64-pipe flops per block: DMMA tiles (4 real products each, 8 blocks per
    // m-tile, zero padding included) plus the radix-2 butterflies
    double exec_flops() const;
};

struct PlanNode;
struct Params;

// Swizzled position of Fourier index a = (i, j, k) in the FFT buffer:
// (i n + j) n + (k ^ j): the k-, j- and i-axis line passes are all free of
// shared-memory bank conflicts (8 lanes of a quarter-warp vary j or k).
inline int of_swizzle(int a, int n) {
    const int k = a % n, j = (a / n) % n, i = a / (n * n);
    return (i * n + j) * n + (k ^ (j & (n - 1)));
}

// Compiles the orbit-block operator of S_n(p) (forward) or S_n(p)^{-1} / n^3
// (inverse) into per-warp DMMA tiles. Returns false when n is not supported.
bool compile_orbit_fft(int n, const Params& p, bool inverse, OrbitFftHost& h, int warps = kOfWarps);

// Host emulation of the kernel's arithmetic on the compiled tables (tests):
// in/out complex128 rows [batch][N].
void emulate_orbit_fft(const OrbitFftHost& h, const double* in, double* out, int64_t batch);

cudaError_t launch_orbit_fft(const OrbitFftDesc& d, int in_mode, int out_mode, const void* in, void* out,
                             int64_t batch, cudaStream_t st, int num_sms);

}  // namespace fcct
