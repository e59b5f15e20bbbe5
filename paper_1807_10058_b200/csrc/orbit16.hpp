// Orbit-FFT executor for n = 16 (and any n whose 8-block tile does not fit a
// CTA): D_n(p) = F_n S_n(p) as two passes over HBM (orbit_fft.hpp derives the
// telescoped factorisation).
//
//  pass A  base change S_n(p) (forward) or S_n(p)^{-1} / n^3 (inverse) on the
//          FP64 tensor pipe. A CTA owns 8 transform blocks (one DMMA m-tile)
//          at a time and walks the orbits in chunks: the chunk's members of
//          the 8 blocks are gathered (cp.async, 16 or 8 bytes each) into a
//          [slot][8 blocks] stage whose block index is xor-ed by 2 (slot mod 4)
//          (conflict-free fragment loads), its operator tiles are copied from
//          L2 into shared memory, both one chunk ahead; outputs are stored at
//          their natural positions (the 8 blocks' rows stay L2-resident while
//          the CTA covers them, so DRAM sees each sector once).
//  pass B  the 3D FFT on Z_n^3 per block: a cp.async tile load into a
//          (k ^ j)-swizzled shared tile (conflict-free line passes), k, j and
//          i passes, the last one storing to HBM.
// Forward: A (x -> z) then B (z -> y); inverse: B (y -> z) then A (z -> x).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace fcct {

struct Params;

constexpr int kO16Warps = 16;
constexpr int kO16Chunk = 256;  // member slots per chunk (4 per k-tile)
constexpr int kO16Tmax = 16;    // tiles per warp per chunk
constexpr int kO16Wrap = 12;    // operator tiles in flight per warp (the stream's look-ahead)

struct Orbit16Desc {
    int n = 0, N = 0, dir = 0;
    int nchunks = 0;
    int tmax = 0;                      // tiles per warp per chunk (<= kO16Tmax)
    const double2* table = nullptr;    // [warp][chunk * tmax + kO16Wrap][32] B fragments (Re, Im)
    const int* tile_meta = nullptr;    // [chunk][warp][tmax]: k-tile index | chain end << 16 | valid << 17
    const int* out_pos = nullptr;      // [chunk][warp][tmax][4]: orbit-order positions o(2k) | o(2k+1) << 16 (0xFFFF none)
    const int* gather = nullptr;       // [chunk][kO16Chunk]: natural position of each slot (-1: zero padding)
    const int* chunk_slots = nullptr;  // [chunk]: slots used
    const int* zperm = nullptr;        // [N]: orbit-order index of natural position a in z
};

struct Orbit16Host {
    int n = 0, N = 0, dir = 0, nchunks = 0, tmax = 0;
    std::vector<double> table;
    std::vector<int32_t> tile_meta, out_pos, gather, chunk_slots;
    std::vector<int32_t> zperm;  // natural position -> index in the orbit-ordered scratch z
    int64_t tiles = 0;  // real DMMA tiles
    double exec_flops() const;  // FP64-pipe flops per block (tiles + FFT butterflies)
};

// Compiles the orbit blocks of S_n(p) (or S_n(p)^{-1} / n^3) for pass A.
// Throws IllConditioned like compile_orbit_fft; false when n is unsupported.
bool compile_orbit16(int n, const Params& p, bool inverse, Orbit16Host& h);

// Host emulation of both passes on the compiled tables (CPU tests), complex128 rows.
void emulate_orbit16(const Orbit16Host& h, const double* in, double* out, int64_t batch);

// Pass A: in/out modes as OfMode (orbit_fft.hpp); the z side is complex128.
cudaError_t launch_orbit16_base(const Orbit16Desc& d, int in_mode, int out_mode, const void* in, void* out,
                                int64_t batch, cudaStream_t st, int num_sms);
// Inverse epilogue: rows stored in orbit order by pass A -> natural positions.
cudaError_t launch_unpermute(int mode, const void* in, void* out, int N, int64_t batch, const int* zperm,
                             cudaStream_t st, int num_sms);
// Pass B: sign +1 (forward F_n) or -1 (F_n^{-1} without the 1/n^3, folded into pass A).
// zperm: the z side (forward input / inverse output, complex128) is in orbit
// order, z[zperm[a]] holding natural position a.
cudaError_t launch_fft_cube(int n, int sign, int in_mode, int out_mode, const void* in, void* out, int64_t batch,
                            const int* zperm, cudaStream_t st, int num_sms);

}  // namespace fcct
