// Plan-time compilation of the fast transform into DMMA stages (pipeline v2).
//
// One CTA tile holds TB = 16 transform blocks in shared memory as
// X[t][slot][part] (complex positions at "slots", row stride 2N + 8 doubles).
// Every stage of the factorization (basis change B, K-mix, leaf D_2) is a
// complex linear map y = A x on the n^3 positions, executed on the FP64 tensor
// pipe as C(32 x 8) += D(32 x 4) * T(4 x 8) with mma.sync.m8n8k4.f64:
//   * the 32 rows are the 16 blocks x {re, im} (4 m-tiles of 8 data rows),
//   * T is a 4 x 8 tile of A (4 input positions x 8 output positions), kept as
//     (Re, Im) pairs; a complex tile costs a second DMMA on the part-swapped,
//     sign-flipped data,
//   * a "unit" is 8 output positions (an n-tile of a sparse stage, or one
//     8 x 8 K-mix item) and accumulates over its non-zero k-tiles.
// Layout rules (all conflict-free on the 32 shared-memory banks):
//   * every k-tile reads 4 consecutive slots (the previous stage writes its
//     outputs in the next stage's k-tile order);
//   * the 4 even and the 4 odd outputs of every unit land on slots with
//     distinct residues mod 4 (a proper 4-edge-colouring of the regular
//     bipartite graph "k-tile -- unit half", König).
// The first stage reads the natural layout produced by the TMA bulk load and
// the last stage writes the natural (composite-permuted) output layout.
#pragma once

#include <cstdint>
#include <vector>

#include "plan.hpp"

namespace fcct {

// CTA shape: `tb` blocks per tile (4 data rows per block pair -> tb/4 m-tiles
// per unit), `warps` warps per CTA, at most `units` units per warp per stage.
struct Shape2 {
    int tb = 16;
    int warps = 16;
    int units = 4;
};

struct Stage2Host {
    int kind = 0;  // 0 sparse (tiles), 1 mix (8x8 complex per unit)
    int n_units = 0;
    std::vector<int32_t> warp_units;  // [warps][units] unit index or -1
    std::vector<int32_t> u_out;       // [n_units][8] output slot of output n
    // sparse: entries stored warp-major (the per-warp stream the kernel's
    // cp.async ring walks): warp w owns entries [w_base[w], w_base[w+1]),
    // unit j of warp w has w_count[w][j] of them.
    std::vector<int32_t> w_base;      // [warps + 1]
    std::vector<int32_t> w_count;     // [warps][units]
    std::vector<int32_t> w_ccount;    // [warps][units] complex entries (stored after the real ones)
    std::vector<uint32_t> w_cplx;     // [warps][4]: bit f = flat entry f of the warp is complex (<= 128 entries)
    std::vector<int32_t> e_slots;     // [n_entries][4] input slot of k-column; bit 30 = complex tile
    std::vector<double> e_re;         // [n_entries][32] Re T[k][n], lane order
    std::vector<double> e_im;         // [n_entries][32] Im T[k][n] (zeros for real tiles, never fetched)
    // mix
    std::vector<int32_t> u_node;      // [n_units]
    std::vector<int32_t> u_in;        // [n_units][8] input slot of input g
    std::vector<double> K;            // [nodes][8 b][8 g][2]
    int64_t dmma_per_tile = 0;        // DMMA.884 per 16-block tile
    int sync_mid = 0;                 // barrier between compute and store: 0 CTA, 1 warp group
    int sync_end = 0;                 // barrier after the store: 0 CTA, 1 warp group
};

struct Pipeline2Host {
    Shape2 shape;
    int n = 0;
    int N = 0;
    int stride = 0;  // doubles per block row in smem (2N + 8)
    std::vector<Stage2Host> stages;
    int64_t dmma_per_tile = 0;
    // natural-layout row shift (in 16-byte slots) of odd block rows: a leaf
    // mix touches 8 natural positions that share their residue mod 4, so odd
    // rows are moved by one slot to spread them over twice the banks
    int shift_in = 0, shift_out = 0;
};

// Builds the stage list for a full radix tree (every leaf n == 1, n <= 8).
// Returns false when the tree is not supported (odd leaves, n > 8).
bool compile_pipeline2(const PlanNode& root, bool inverse, const Shape2& shape, Pipeline2Host& out);

}  // namespace fcct
