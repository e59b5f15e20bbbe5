// Single-pass orbit-pattern executor for n = 16 (executor 10): D_n(p) = F_n S_n(p)
// with one transform block resident in shared memory from load to store.
//
// The orbit blocks of S_n(p) (ColumnEvaluator's symmetrised plane waves,
// transform.cpp:46-68, restated in orbit_fft.hpp) come in very few shapes.
// List an orbit's members in group order from its lexicographically smallest
// member k0 (member r = g_r k0 mod n, first appearance), and split off the
// separable phase of the reduced index,
//     S_O = diag(Lambda[a_r]) M,  Lambda[a] = e^{2 pi i a.p/n} / 24,
// then M holds only the carry phases e^{2 pi i t.p} (g k = a + n t) and is the
// SAME matrix for every free orbit (24 members), and one of two matrices for the
// 12-member orbits, ... : 8 distinct M for any n and p (measured n = 8 .. 64;
// tools/orbit_shapes.py counts them from the group alone).
// So the base change of a block is a GEMM with a constant 24 x 24 (and a
// 12 x 12) complex operator over the block's OWN orbits:
//   - the operator lives in registers as DMMA m8n8k4 B fragments (36 doubles);
//   - the M dimension of the MMA is 8 orbits of the same block, so a CTA needs
//     one block (64 KB complex128), not 8 — the block stays in shared memory,
//     the base change runs in place (an orbit is read and written by one warp),
//     and the 16^3 FFT follows (forward) or precedes (inverse) it in the same
//     tile. HBM sees every sample once: no z round trip (orbit16.hpp moves z
//     through HBM twice), no operator stream from L2, no tile metadata;
//   - Lambda is separable, Lambda[(i, j, k)] = L0[i] L1[j] L2[k]: each axis pass of
//     the FFT multiplies its line by 16 constants read from the kernel
//     parameters (constant bank operands: no load instructions, no table) —
//     before the butterflies in the forward, after them (conjugated, 24 n^-3
//     folded into axis 0) in the inverse;
//   - the few orbits of the rare shapes (28 of 245 at n = 16) are SIMT rows,
//     their coefficients stored term-major so a warp's loads are coalesced.
// Real samples in (forward) and out (inverse) halve the DMMA count.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace fcct {

struct Params;

constexpr int kPatWarps = 4;     // warps per CTA (4: three CTAs per SM; 8: two)
constexpr int kPatMaxRare = 2;   // rare rows per thread
constexpr int kPatRareTerms = 12;  // terms of a rare row (padded with zero coefficients)

// slot of Fourier / sample index a = (i, j, k) in the shared tile's Re / Im planes
// while the base change runs: natural order (the FFT's j-axis pass converts to and
// from the conflict-free (i, j, k ^ j) layout of the k-axis pass)
__host__ __device__ constexpr int pat_slot(int a) { return a; }

struct OrbitPatDesc {
    int n = 0, N = 0, dir = 0;
    int cnt[2] = {0, 0};      // orbits of the two DMMA classes (24 and 12 members)
    int ntiles[2] = {0, 0};   // tiles of 8 orbits
    int idx_count = 0;        // uint16 entries of idx (copied to shared memory)
    int nrare = 0;            // SIMT rows
    const double2* op[2] = {nullptr, nullptr};   // [q][nt][32] B fragments (Re, Im) of M (or M^-1)
    const uint16_t* idx = nullptr;               // class 0: [tile][24][8], then class 1: [tile][12][8] slots
    const int2* warp_tiles = nullptr;            // [2][kPatWarps]: (first tile, tiles) of a warp per class
    int rare_pitch = 0;                          // nrare rounded up to a warp
    const uint16_t* rare_out = nullptr;          // [nrare] output slots
    const uint16_t* rare_in = nullptr;           // [kPatRareTerms][rare_pitch] input slots
    const double2* rare_coef = nullptr;          // [kPatRareTerms][rare_pitch]
    double2 lax[3][16];                          // per-axis phases of Lambda (forward) / its scaled inverse
};

// Large n (32, 64; orbit_big.hpp's executor): the same tables drive the S pass of
// a single transform that lives in L2 — one warp per tile of 8 orbits, fragments
// gathered from / scattered to global memory, Lambda from three n-entry tables
// in shared memory. Nothing is streamed: the 104 MB coefficient stream of
// S_64^-1 (and S_64's generated coefficients) become a 9 KB register operand.
struct OrbitPatBigDesc {
    int n = 0, N = 0, dir = 0, log2n = 0;
    int cnt[2] = {0, 0}, ntiles[2] = {0, 0};
    const double2* op[2] = {nullptr, nullptr};
    const int32_t* idx = nullptr;        // class 0: [tile][24][8], then class 1: [tile][12][8] natural positions
    int nrare = 0, rare_pitch = 0;
    const int32_t* rare_out = nullptr;   // [nrare]
    const int32_t* rare_in = nullptr;    // [kPatRareTerms][rare_pitch]
    const double2* rare_coef = nullptr;  // [kPatRareTerms][rare_pitch]
    const double2* lax = nullptr;        // [3][n] per-axis phases
};

struct OrbitPatHost {
    int n = 0, N = 0, dir = 0;
    int cnt[2] = {0, 0}, ntiles[2] = {0, 0};
    std::vector<double> op[2];
    double lax[3][64][2] = {};        // per-axis phases (Re, Im), n entries per axis
    std::vector<int32_t> idx;
    std::vector<int32_t> warp_tiles;  // [2][kPatWarps][2]
    int nrare = 0, rare_pitch = 0;
    std::vector<int32_t> rare_out;    // [nrare]
    std::vector<int32_t> rare_in;     // [kPatRareTerms][rare_pitch]
    std::vector<double> rare_coef;    // [kPatRareTerms][rare_pitch][2]
    int64_t rare_terms = 0;           // non-zero terms
    int patterns = 0;                 // distinct shapes found
    int64_t dmma = 0;                 // complex-input DMMA count per block
    // FP64-pipe flops per block; real_io: real samples in (forward) / out
    // (inverse), where half of the DMMA products are not issued
    double exec_flops(bool real_io = false) const;
    // modelled shared-memory wavefronts per block and plane of the fragment gathers
    // and result scatters (8-byte accesses, half-warps), and their conflict-free floor
    int64_t wavefronts = 0, wavefronts_floor = 0;
};

// Compiles S_n(p) (forward) or S_n(p)^{-1} / n^3 (inverse); false when n is not
// 16, 32 or 64, an orbit block is singular or the shapes do not fit the kernel.
bool compile_orbit_pat(int n, const Params& p, bool inverse, OrbitPatHost& h);
// Both directions from one derivation of the orbit blocks.
bool compile_orbit_pat_pair(int n, const Params& p, OrbitPatHost& fwd, OrbitPatHost& inv);

// Host emulation on the compiled tables, complex128 rows (CPU tests).
void emulate_orbit_pat(const OrbitPatHost& h, const double* in, double* out, int64_t batch);

// in / out modes as OfMode (orbit_fft.hpp).
cudaError_t launch_orbit_pat(const OrbitPatDesc& d, int in_mode, int out_mode, const void* in, void* out,
                             int64_t batch, cudaStream_t st, int num_sms);

// Large-n S pass (complex128 in and out, [batch][N] rows; in != out).
cudaError_t launch_orbit_pat_big(const OrbitPatBigDesc& d, const void* in, void* out, int64_t batch, cudaStream_t st);

}  // namespace fcct
