// Orbit-FFT executor for large n (32, 64): D_n(p) = F_n S_n(p) (orbit_fft.hpp)
// for a single transform or a small batch, where one block's state (4 MB at
// n = 64) is L2-resident and the work is bound by streaming the operator.
//
//  S pass   one thread per output row of an orbit block (rows of an orbit are
//           consecutive threads); the orbit's coefficients are stored column
//           major, so a warp reads them coalesced while the input member is a
//           broadcast; every coefficient is read once per launch and reused
//           across the batch.
//  F pass   one kernel per axis: a CTA loads 8 neighbouring lines of n points
//           (coalesced 128-byte rows), runs the radix-2 stages in shared
//           memory, and writes them back (in place, or to the output on the
//           last axis).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace fcct {

struct Params;

struct OrbitBigDesc {
    int n = 0, N = 0, dir = 0;
    int64_t rows = 0;                 // = N (every natural position is one row of one orbit)
    const int* row_orbit = nullptr;   // [rows]: orbit of the row (rows are grouped by orbit)
    const int* row_index = nullptr;   // [rows]: row index r inside its orbit
    const int* orbit_off = nullptr;   // [orbits + 1]: first member slot of each orbit
    const int64_t* coef_off = nullptr;// [orbits]: first coefficient of each orbit
    const int* members = nullptr;     // [N]: natural position of each member slot
    const double2* coef = nullptr;    // column-major blocks: coef[coef_off + c s + r] = M[r][c]
    // forward only: free orbits (24 members) generate S_n(p)'s coefficients instead
    // of streaming them (coef_off[o] < 0 marks such an orbit). With member j = g_j k0
    // - n t_j (k0 = member 0, g_j in S4, carry t_j),
    //   S[r][c] = e^{2 pi i (g_r k0).p/n} / 24 * e^{-2 pi i t_c.(w^T p)},  w = g_r g_c^{-1}
    int gen = 0;
    double pr = 0, ps = 0, pt = 0;    // grid offsets (turns)
    const uint32_t* mpack = nullptr;  // [N] member slot: natural | carry id << 18 | g << 24 | generated << 31
    const double2* ttab = nullptr;    // [ncarry][24]: e^{-2 pi i t.(w^T p)}
    const uint8_t* mtab = nullptr;    // [24][24]: index of g_a g_b^{-1}
    const int* grp = nullptr;         // [24][9]: the group matrices (s4_group order)
    int ncarry = 0;
    // the kernel's work lists: free orbits (24 packed members each, 10 orbits per
    // CTA) and the rows of the remaining (non-free) orbits as slot indices
    const uint32_t* fpack = nullptr;
    const double2* fbase = nullptr;   // [nfree * 24]: base phase of each free row
    int nfree = 0;
    const int* tail = nullptr;
    int ntail = 0;
};

struct OrbitBigHost {
    int n = 0, N = 0, dir = 0;
    std::vector<int32_t> row_orbit, row_index, orbit_off, members;
    std::vector<int64_t> coef_off;
    std::vector<double> coef;  // (Re, Im) pairs
    // generated forward coefficients (OrbitBigDesc::gen)
    int gen = 0;
    double pr = 0, ps = 0, pt = 0;
    std::vector<uint32_t> mpack;
    std::vector<double> ttab;
    std::vector<uint8_t> mtab;
    std::vector<int32_t> grp;
    int ncarry = 0;
    int64_t gen_rows = 0;  // rows whose coefficients are generated
    std::vector<uint32_t> fpack;  // free orbits, 24 packed members each
    std::vector<double> fbase;    // e^{2 pi i (g_j k0).p/n} / 24 per fpack slot, (Re, Im)
    std::vector<int32_t> tail;    // slots of the rows in non-free orbits
    double exec_flops() const;
};

// Builds the S_n(p) (forward) or S_n(p)^{-1} / n^3 (inverse) blocks for n = 32, 64.
// generate (forward only): free orbits carry no coefficient block; the kernel
// generates their coefficients from the group structure (OrbitBigDesc::gen).
bool compile_orbit_big(int n, const Params& p, bool inverse, OrbitBigHost& h, bool generate = true);

// Host emulation of both passes on the compiled tables (CPU tests), complex128 rows.
void emulate_orbit_big(const OrbitBigHost& h, const double* in, double* out, int64_t batch);

// S pass: complex128 in and out, [batch][N] rows.
cudaError_t launch_orbit_big_s(const OrbitBigDesc& d, const void* in, void* out, int64_t batch, cudaStream_t st);
// F pass along axis (0 = i, 1 = j, 2 = k) with sign +-1; in == out allowed.
cudaError_t launch_line_fft(int n, int axis, int sign, const void* in, void* out, int64_t batch, cudaStream_t st);

}  // namespace fcct
