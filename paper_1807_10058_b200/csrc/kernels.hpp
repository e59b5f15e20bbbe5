// Launch interface of the sm_100a kernels (implemented in kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fcct {

constexpr int kMaxStages = 16;

// One stage of the fast pipeline: a sparse operator on the n^3 state vector.
//  kind 0 (sparse): ELL row groups of RG = 32/TB rows. Entry e of group g,
//        row slot rr, step k is e = ginfo[g].x + k*RG + rr.
//  kind 1 (mix8):  for every node q of the level and slice h < m3,
//        out[pos_out(blk)] = sum_g K[q][blk][g] * in[pos_in(g)],
//        pos(g) = q*8*m3 + g*m3 + h, optionally remapped through gather /
//        scatter (the composite radix permutation at the first/last stage).
struct StageDesc {
    int kind;
    int ngroups;
    const int2* ginfo;
    const int* grow;
    const int* ecol;
    const void* ecoef;
    int m3;
    int nodes;
    const void* K;
    const int* gather;
    const int* scatter;
};

struct PipelineDesc {
    int n;
    int N;
    int tb;       // transforms per CTA tile
    int nstages;
    StageDesc stage[kMaxStages];
};

// Pipeline v2 (fp64, n <= 8): every stage on the FP64 tensor pipe, see tiling.hpp.
// Small per-stage tables live in a per-CTA shared-memory arena (copied once
// per kernel, they are identical for every tile): fields named o_* are byte
// offsets into it (-1: absent). Fragment values and large K tables stay global.
struct Stage2Dev {
    int kind;  // 0 sparse tiles, 1 mix
    int n_units;
    int o_warp_units;  // int [warps][units]
    int o_u_out;       // int [units][8]
    int o_w_base;      // sparse: int [warps + 1] warp-major entry ranges
    int o_w_count;     // sparse: int [warps][units]
    int o_w_ccount;    // sparse: int [warps][units] complex entries (after the real ones)
    int o_e_slots;     // sparse: int [entries][4] input slots (bit 30: complex tile)
    int o_u_node;      // mix: int [units]
    int o_u_in;        // mix: int [units][8]
    int o_K;           // mix: double2 [nodes][8][8] when small enough, else -1
    const double* e_re;  // sparse: [entries][32] Re T[k][n], lane order (global)
    const double* e_im;  // sparse: [entries][32] Im T[k][n] (global)
    const double2* e_ri; // sparse: [entries][32] (Re, Im) interleaved: the cp.async ring's source
    const double2* K;    // mix: global copy of the K tables
    int sync_mid;        // barrier between compute and store: 0 CTA, 1 warp group (root child)
    int sync_end;        // barrier after the store: 0 CTA, 1 warp group
    int ld_shift;        // bytes added to the A-load address of odd block rows (natural input layout)
    int st_shift;        // bytes added to the store address of odd block rows (natural output layout)
};

struct Pipeline2Desc {
    const uint4* arena;  // global image of the shared-memory table arena
    int arena_bytes;     // multiple of 16
    int tb;     // blocks per tile (16 or 8)
    int warps;  // warps per CTA (16 or 8)
    int N;
    int stride;  // doubles per block row in shared memory
    int nstages;
    int direct_store;  // 1: last stage stores to global from registers; 0: smem + TMA bulk store
    int io_f32;        // 1: global data is complex64 (converted to/from fp64 at tile load/store)
    int real_in;       // 1: input rows are real samples (z_transform fused into the tile load)
    int real_out;      // 1: only real parts are stored (grid_from_signal fused into the tile store)
    int64_t row_in;    // doubles between consecutive block rows of the input (2N when dense)
    int64_t row_out;   // same for the output (the two-level executor runs children in place of a parent)
    int ring;          // 1: sparse-stage table entries stream through a per-warp cp.async ring in smem
    int shift_in;      // doubles: odd block rows of the natural input tile start this far into their row
    int shift_out;     // doubles: same for the natural output tile (spreads the leaf mix's banks)
    int stage_mask;    // debug/timing only: stages with a cleared bit are skipped
    unsigned long long* timing;  // debug: CTA 0 accumulates clock64 per phase (nullptr: off)
    Stage2Dev st[kMaxStages];
};

cudaError_t launch_pipeline2(const Pipeline2Desc& d, const void* in, void* out, int64_t batch, cudaStream_t stream,
                             int num_sms);

// Two-level executor (n = 16): the root level runs as its own pass, the eight
// n = 8 children on pipeline2 (row-strided into a child-major scratch).
// Root tables: ELL per unit h (m3 = N / 8 units); entries of output row
// g m3 + h (forward B) or j m3 + h (inverse B^-1) at [off[g] + e * m3 + h].
struct RootDesc {
    int N, m3, lgN;
    int ell_off[9];           // prefix offsets (in entries) of the 8 row groups; ell_off[8] = total
    const int* col;           // [entries] input column (padding: 0 with value 0)
    const double2* val;       // [entries]
    const double2* K;         // [8][8] K (forward) or K^{-1} (inverse), row-major
    const int* perm;          // [N] radix permutation: child-major index c m3 + j -> natural position
    const int* pinv;          // [N] its inverse
};
// forward: x (natural, mode 0 c128 / 1 c64 / 2 r64 / 3 r32) -> z child-major c128
cudaError_t launch_root_forward(const RootDesc& d, const void* x, int in_mode, double* z, int64_t batch,
                                cudaStream_t st, int num_sms);
// inverse: z child-major c128 -> y natural (out_mode as above)
cudaError_t launch_root_inverse(const RootDesc& d, const double* z, void* y, int out_mode, int64_t batch,
                                cudaStream_t st, int num_sms);
// child-major c128 <-> natural (mode conversions on the natural side)
cudaError_t launch_child_to_natural(const RootDesc& d, const double* src, void* dst, int out_mode, int64_t batch,
                                    cudaStream_t st);
cudaError_t launch_natural_to_child(const RootDesc& d, const void* src, int in_mode, double* dst, int64_t batch,
                                    cudaStream_t st);

// z_transform / grid_from_signal for executors without fused real I/O:
// real[count] -> complex[count] (zero imaginary parts) and back (real parts).
cudaError_t launch_complexify(const void* in_real, void* out_cplx, int64_t count, bool f32, cudaStream_t st);
cudaError_t launch_real_part(const void* in_cplx, void* out_real, int64_t count, bool f32, cudaStream_t st);

// Global-memory multi-pass pipeline (any full radix tree; used when a block's
// state does not fit one CTA tile, e.g. n = 32, 64): one launch per stage.
struct GStage {
    int kind;              // 0 sparse (sliced ELL), 1 mix8
    const int64_t* rowptr; // sparse: slice offsets [N / 32 + 1] (entries of slice s at rowptr[s] + e 32 + lane)
    const int* col;        // sparse (gather folded in for the first inverse stage)
    const void* coef;      // sparse: complex values
    const int* out_row;    // sparse: output position of row r (scatter folded in), nullptr = identity
    int nodes, m3;         // mix
    const void* K;         // mix: [nodes][8][8] complex, row-major [b][g]
    const int* gather;     // mix: input position map or nullptr
    const int* scatter;    // mix: output position map or nullptr
};

struct GlobalPipelineDesc {
    int N;
    int nstages;
    GStage st[kMaxStages];
};

cudaError_t launch_global_pipeline(const GlobalPipelineDesc& d, bool f32, const void* in, void* out, void* scratch0,
                                   void* scratch1, int64_t batch, cudaStream_t stream);

// Fast transform pipeline (forward or inverse, decided by the stage list).
cudaError_t launch_pipeline(const PipelineDesc& d, bool f32, const void* in, void* out, int64_t batch,
                            cudaStream_t stream, int num_sms);
int pipeline_smem_bytes(const PipelineDesc& d, bool f32);

// Direct transform: out[b][:] = real-form GEMM of in[b][:] with Wt (2N x 2N, [col][k]).
// Raises the kernel's dynamic shared-memory limit once per (device, kernel) and
// caches the occupancy (CTAs per SM) for (threads, smem); host round trips that
// would otherwise cost microseconds per launch.
cudaError_t prepare_launch(const void* kern, int threads, int smem, int* per_sm);

// fp32 direct GEMM on tcgen05 (gemm_tc.cu): C = A . W^T with W = W_hi + W_lo,
// 3xTF32 (A split on chip). Needs Nn % 128 == 0 and K % 32 == 0.
bool gemm_tf32x3_supported(int Nn, int K);
cudaError_t launch_gemm_tf32x3(const float* A, const float* Whi, const float* Wlo, float* C, int64_t M, int Nn, int K,
                               int num_sms, cudaStream_t st);
// fp64 direct GEMM on tcgen05 by the Ozaki scheme (gemm_tc.cu): int8 slices of
// A and W with per-row power-of-two scales, exact int8 products, fp64 epilogue.
int ozaki_slices();
bool gemm_ozaki_supported(int Nn, int K);
// S = 7 or 8 slices ([S][rows][K] int8); ozaki_slices() = the largest S
cudaError_t ozaki_slice(const double* a, int64_t rows, int K, int S, int8_t* slices, double* scale, cudaStream_t st);
cudaError_t launch_gemm_ozaki(const int8_t* a_slices, const double* a_scale, const int8_t* w_slices,
                              const double* w_scale, double* C, int64_t M, int Nn, int K, int S, int num_sms,
                              cudaStream_t st);
// fp64 table -> (rna_tf32 part, fp32 remainder)
cudaError_t split_tf32(const double* w, float* hi, float* lo, int64_t count, cudaStream_t st);

cudaError_t launch_gemm_f64(const double* A, const double* Wt, double* C, int64_t M, int Nn, int K,
                            cudaStream_t stream);
cudaError_t launch_gemm_f32(const float* A, const float* Wt, float* C, int64_t M, int Nn, int K,
                            cudaStream_t stream);

// Device-side table generation.
struct OrbitDev {
    const int* orbit_of;
    const int* pos;
    const int* mem_off;   // per orbit: offset into members
    const int* mem;       // lex members
    const int* sinv_off;  // per orbit: offset (complex elements) into sinv
    const double* sinv;   // complex128 blocks, row-major [kappa-pos][a-pos]
};
// Real-form forward operator Wt[2N][2N] of D_n(p) (fp64 or fp32 output).
cudaError_t gen_dense_realform(int n, double r, double s, double t, void* Wt, bool f32, cudaStream_t st);
// Real-form inverse operator of D_n(p) from the orbit blocks of S_n(p)^{-1}.
cudaError_t gen_dense_inv_realform(int n, const OrbitDev& od, void* Wt, bool f32, cudaStream_t st);
// Complex column-major D (dense_transform(n,p).matrix layout).
cudaError_t gen_dense_colmajor(int n, double r, double s, double t, double* D, cudaStream_t st);
// Column 1-norms of D_n(p) (plan-time condition estimate): colsum[kappa], N doubles.
cudaError_t dense_colnorm(int n, double r, double s, double t, double* colsum, cudaStream_t st);
// Skew nodes: 6 complex per node (u,v,w,x,y,z); degenerate flag via *flag (device int).
cudaError_t gen_nodes(int n, double r, double s, double t, double* out, int* flag, cudaStream_t st);
// Composite radix permutation.
cudaError_t gen_radix_permutation(int n, unsigned long long* out, cudaStream_t st);
// max |Y[k][i] - D[i][k]| per CTA (Y: batch N of complex128 rows, D column-major).
cudaError_t residual_max(const double* Y, const double* D, int N, double* partial, int nblocks,
                         cudaStream_t st);
// Unit-vector batch: E[k][i] = (i == k).
cudaError_t gen_identity(int N, void* E, bool f32, cudaStream_t st);

// DMMA fragment-layout probe: C (8x8) = A (8x4 row-major) * B (4x8 row-major).
cudaError_t dmma_probe(const double* A, const double* B, double* C, cudaStream_t st);

}  // namespace fcct
