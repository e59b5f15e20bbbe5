/*
 * fcct_gpu.h — C ABI of the B200-native FCC-lattice cosine transform
 * (arXiv 1807.10058). Drop-in replacement for the hot path of the reference
 * C++ library `fcct` (/root/reference/proj/include/fcct/transform.hpp).
 *
 * Each entry point cites the reference interface it replaces. Plain C types
 * only: no torch, no Eigen, no C++ exceptions cross this boundary. Errors are
 * returned as fcct_status codes; fcct_last_error() gives the message of the
 * last failing call on the calling thread.
 *
 * Data layout (byte-compatible with one Eigen::VectorXcd per block,
 * transform.hpp:17-33): block-major [batch][n^3], each point an interleaved
 * (re, im) pair — complex128 for FCCT_F64 plans, complex64 for FCCT_F32 —
 * lexicographic point order (i*n + j)*n + k, last index fastest.
 *
 * Buffers passed to fcct_forward / fcct_inverse are DEVICE pointers owned by
 * the caller; the *_host variants take HOST pointers and do the copies
 * themselves: the batch moves in chunks alternating over two streams, so the
 * H2D copy, the transform and the D2H copy of neighbouring chunks overlap.
 * Page-locked caller buffers are DMA'd directly; pageable ones (a std::vector,
 * an Eigen::VectorXcd) are staged through plan-owned pinned bounce buffers,
 * the host-side copies split over a small thread pool. The plan
 * owns its device tables. Calls on distinct streams are safe to run
 * concurrently; results are deterministic (no atomics in any reduction).
 */
#ifndef FCCT_GPU_H
#define FCCT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error taxonomy: fcct/errors.hpp:9-63 (ErrorCategory math -> CLI exit 2,
 * io -> exit 3; fcct.cpp:702-707). */
typedef enum {
    FCCT_OK = 0,
    FCCT_INVALID_ARGUMENT = 1, /* std::invalid_argument (n < 1, bad params) */
    FCCT_SIZE_MISMATCH = 2,    /* SizeMismatch (transform.cpp:147-154,498-521) */
    FCCT_ODD_SIZE = 3,         /* OddSize (transform.cpp:173-175,315-317) */
    FCCT_DEGENERATE_NODES = 4, /* DegenerateNodes (spectral.cpp:26-43) */
    FCCT_ILL_CONDITIONED = 5,  /* IllConditioned (transform.cpp:113-117,377-378) */
    FCCT_PARAMS_MISMATCH = 6,  /* invalid_argument "different skew grid" (:163-165,515-517) */
    FCCT_IO = 7,               /* MalformedFile / IoFailure */
    FCCT_CUDA = 8,             /* CUDA runtime failure */
    FCCT_DERIVATION = 9,       /* basis-change derivation residual (transform.cpp:301-304) */
    FCCT_MALFORMED = 10,       /* MalformedFile (errors.hpp:52-56), io category */
    FCCT_SIZE_MISMATCH_IO = 11 /* SizeMismatch(..., ErrorCategory::io): a file promises another length */
} fcct_status;

typedef enum { FCCT_DIRECT = 0, FCCT_FAST = 1 } fcct_method;
typedef enum { FCCT_F64 = 0, FCCT_F32 = 1 } fcct_precision;
/* TransformPlan::Kind (transform.hpp:69) */
typedef enum { FCCT_KIND_DIRECT = 0, FCCT_KIND_RADIX2 = 1 } fcct_kind;

typedef struct fcct_plan_s* fcct_plan;

typedef struct {
    int n;
    double r, s, t;          /* SkewParams of the root */
    int kind;                /* fcct_kind of the root */
    int method;              /* fcct_method the plan executes */
    int precision;           /* fcct_precision */
    int levels;              /* radix levels (log2 n for powers of two) */
    int64_t points;          /* n^3 */
    int64_t tree_nnz;        /* sum of nnz(B) over radix nodes, B_2 = I excluded */
    int64_t tree_nnz_inv;    /* same for the explicit B^{-1} factors */
    int64_t root_nnz;        /* nnz(B) of the root */
    int64_t table_bytes;     /* device bytes owned by the plan */
    double condition;        /* the reference's condition estimate of D (direct plans,
                                condition_with_lu, transform.cpp:91-111), or the largest
                                estimate gated while building a fast plan's tree (radix
                                kernels and every child transform) */
    double flops_forward;    /* algorithmic flops per block */
    double flops_inverse;
    int executor;            /* 0 direct GEMM, 1 tile interpreter, 2 FP64-tensor-pipe
                                pipeline, 3 global-memory multi-pass pipeline,
                                4 two-level (n = 16: root pass + eight n = 8 pipelines),
                                5 orbit-FFT (the radix tree telescoped to S_n + radix-2 FFT),
                                6 two-pass orbit-FFT (n = 16: S_n pass + cube FFT pass),
                                7 large-n orbit-FFT (n = 32, 64: S_n pass + three line-FFT passes),
                                8 direct GEMM on tcgen05 (fp32 plans, 3xTF32, gemm_tc.cu),
                                9 direct GEMM on tcgen05 (fp64 plans, Ozaki int8 slices, gemm_tc.cu),
                                10 single-pass orbit-pattern executor (n = 16: the block resident in
                                   shared memory, constant-operator DMMA base change + cube FFT, orbit_pat.hpp) */
    double exec_flops_forward; /* flops the executor issues on the FP64 pipes per block (tensor-core
                                  tiles including their zero padding, plus FFT butterflies); 0 when
                                  equal to the algorithmic count */
    double exec_flops_inverse;
    int64_t table_bytes_forward; /* device bytes of the forward executor's own tables (fast plans) */
    double exec_flops_forward_real; /* same as exec_flops_*, for real samples in (fcct_forward_real) / out
                                       (fcct_inverse_real) where the executor skips the imaginary half of its
                                       tensor-core products (executor 10); 0 when equal to exec_flops_* */
    double exec_flops_inverse_real;
} fcct_plan_info_t;

/* Last error message on this thread ("" if none). */
const char* fcct_last_error(void);

/* Plan creation: replaces build_plan(n, params) (transform.hpp:118-119,
 * transform.cpp:382-408) for method FAST and dense_transform(n, params)
 * (transform.hpp:46, transform.cpp:130-144) for method DIRECT. Tables are
 * derived exactly (orbit-block structure, extended precision) and generated
 * on `device`. n odd or n == 1 always yields a direct plan (transform.cpp:385-386). */
fcct_status fcct_plan_create(int n, double r, double s, double t, int method, int precision,
                             int device, fcct_plan* out);

/* Executors of a FAST plan (fcct_plan_info_t.executor). FCCT_EXEC_AUTO is the
 * default choice of fcct_plan_create; the others force one executor (parity tests
 * of every executor, A/B timing). All compute the same transform; a forced
 * executor that cannot run this plan falls through to the next in the order
 * orbit -> pipeline2 -> two-level -> tile / global. No environment variable
 * selects executors in the product build. */
typedef enum {
    FCCT_EXEC_AUTO = 0,
    FCCT_EXEC_ORBIT = 1,          /* orbit-FFT executors (n = 4, 8 warp-specialised; 16 single pass; 32, 64) */
    FCCT_EXEC_ORBIT_PHASED = 2,   /* n = 4, 8: the phased orbit-FFT kernel (16 warps alternate roles) */
    FCCT_EXEC_PIPELINE2 = 3,      /* stage-by-stage FP64 DMMA pipeline (n <= 8) */
    FCCT_EXEC_TWO_LEVEL = 4,      /* n = 16: root pass + eight n = 8 orbit-FFT children */
    FCCT_EXEC_TWO_LEVEL_V2 = 5,   /* n = 16: root pass + eight n = 8 stage-pipeline children */
    FCCT_EXEC_TILE = 6,           /* shared-memory tile interpreter */
    FCCT_EXEC_GLOBAL = 7,         /* global-memory multi-pass pipeline */
    FCCT_EXEC_ORBIT_TWO_PASS = 8, /* n = 16: the two-pass orbit-FFT executor (S_n pass + cube FFT pass through HBM) */
    FCCT_EXEC_ORBIT_STREAMED = 9  /* n = 32, 64: the S pass on streamed / generated orbit blocks (one thread per row)
                                     instead of the constant-operator DMMA tiles (orbit_pat.hpp) */
} fcct_executor;

/* build_plan with a forced executor (method FAST; see fcct_executor). */
fcct_status fcct_plan_create_executor(int n, double r, double s, double t, int precision, int device, int executor,
                                      fcct_plan* out);
fcct_status fcct_plan_destroy(fcct_plan plan);
fcct_status fcct_plan_info(fcct_plan plan, fcct_plan_info_t* info);

/* Forward: replaces fast_apply(plan, signal) (transform.hpp:123-124,
 * transform.cpp:496-507) and naive_apply(dense, signal) (transform.hpp:48,
 * transform.cpp:146-156), batched. in/out are device buffers of
 * batch * n^3 complex values; stream is a cudaStream_t (NULL = default). */
fcct_status fcct_forward(fcct_plan plan, const void* in, void* out, int64_t batch, void* stream);

/* Inverse: replaces inverse_apply(plan, spectrum) (transform.hpp:127-128,
 * transform.cpp:509-524) and inverse_apply(dense, spectrum) (transform.hpp:49,
 * transform.cpp:158-169). `r, s, t` of the spectrum must equal the plan's
 * (FCCT_PARAMS_MISMATCH otherwise, transform.cpp:515-517). */
fcct_status fcct_inverse(fcct_plan plan, const void* in, void* out, int64_t batch, void* stream);
fcct_status fcct_inverse_checked(fcct_plan plan, double r, double s, double t, const void* in,
                                 void* out, int64_t batch, void* stream);

/* Host-buffer variants (the call a CPU caller of fcct makes): host -> device
 * copy, transform, device -> host copy, synchronous on `stream`. */
fcct_status fcct_forward_host(fcct_plan plan, const void* in_host, void* out_host, int64_t batch,
                              void* stream);
fcct_status fcct_inverse_host(fcct_plan plan, const void* in_host, void* out_host, int64_t batch,
                              void* stream);

/* Real-sample I/O (the steps either side of the path, voxel_io.hpp:40-46).
 * fcct_forward_real replaces z_transform (voxel_io.cpp:178-186) followed by
 * fast_apply / naive_apply: `in_real` holds [batch][n^3] real samples (f64,
 * or f32 for an FCCT_F32 plan) and `out` the complex spectrum. fcct_inverse_real
 * replaces inverse_apply followed by grid_from_signal (voxel_io.cpp:188-198):
 * `out_real` receives the real parts only. The fast fp64/fp32 pipeline fuses
 * the (de)complexification into its tile load/store, halving the bytes moved
 * on the real side. */
fcct_status fcct_forward_real(fcct_plan plan, const void* in_real, void* out, int64_t batch, void* stream);
fcct_status fcct_inverse_real(fcct_plan plan, const void* in, void* out_real, int64_t batch, void* stream);
fcct_status fcct_forward_real_host(fcct_plan plan, const void* in_real_host, void* out_host, int64_t batch,
                                   void* stream);
fcct_status fcct_inverse_real_host(fcct_plan plan, const void* in_host, void* out_real_host, int64_t batch,
                                   void* stream);

/* radix_permutation(n) (transform.hpp:55, transform.cpp:171-194): n^3 entries,
 * bit-exact. Computed on the device from the closed-form digit interleave. */
fcct_status fcct_radix_permutation(int n, uint64_t* out_host);

/* dense_transform(n, params).matrix (transform.hpp:39-46): column-major n^3 x n^3
 * complex128, generated on the device into the caller's device buffer. */
fcct_status fcct_dense_matrix(int n, double r, double s, double t, void* out_device, void* stream);
/* Same matrix into HOST memory (column-major n^3 x n^3 complex128), generated
 * on `device`: the DenseTransform::matrix of the C++ shim (include/fcct_b200.hpp). */
fcct_status fcct_dense_matrix_host(int n, double r, double s, double t, int device, void* out_host);

/* Skew node set (skew_nodes, spectral.cpp:155-171) generated on the device:
 * per node 6 complex128 values (u, v, w, x, y, z); runs the degeneracy check
 * for n <= 16 (spectral.cpp:26-43). */
fcct_status fcct_skew_nodes(int n, double r, double s, double t, void* out_device, void* stream);

/* TransformPlan accessors (transform.hpp:71-84). kernel(): 8x8 column-major
 * complex128. basis(): CSC export (colptr[n^3+1], rowidx[nnz], values[2*nnz]);
 * pass NULL arrays to query *nnz only. child: index 0..7 of a radix plan. */
fcct_status fcct_plan_kernel(fcct_plan plan, double* out128);
fcct_status fcct_plan_basis(fcct_plan plan, int64_t* nnz, int64_t* colptr, int32_t* rowidx,
                            double* values);
fcct_status fcct_plan_child(fcct_plan plan, int index, int* n, double* r, double* s, double* t,
                            int* kind);

/* factorization_residual(plan, dense) (transform.hpp:132-133,
 * transform.cpp:526-540): max |fast(e_k) - D e_k| over all k, evaluated on the
 * device. */
fcct_status fcct_factorization_residual(fcct_plan plan, double* out);

/* with_perturbed_basis(plan, delta) (transform.hpp:138-139,
 * transform.cpp:542-554): copy of a FAST plan with delta added to the first
 * stored basis entry of the root; children shared. */
fcct_status fcct_plan_perturbed_basis(fcct_plan plan, double delta, fcct_plan* out);

/* basis_change(n, params) (transform.hpp:57-62, transform.cpp:314-320): the
 * sparse factor B (inverse = 0) or its explicit inverse (inverse = 1) in CSC,
 * derived on the host (no GPU needed). Pass NULL arrays to query *nnz. */
fcct_status fcct_basis_change(int n, double r, double s, double t, int inverse, int64_t* nnz, int64_t* colptr,
                              int32_t* rowidx, double* values);

/* condition_estimate_1norm(dense_transform(n, params).matrix) (transform.hpp:141-143,
 * transform.cpp:91-122): the reference's probe-based 1-norm condition estimate of
 * D_n(p) — exact ||D||_1 times the largest ||D^{-1} v||_1 / ||v||_1 over its eight
 * probes — without forming D (D = F_n S_n(p), D^{-1} v = S^{-1} F^{-1} v). This is
 * the value IllConditioned is raised on and DenseTransform.condition_estimate holds.
 * Host computation; column norms on the current GPU for n^3 >= 4096 when one is
 * present. inf when D is singular. */
fcct_status fcct_condition_estimate(int n, double r, double s, double t, double* out);

/* Host-side tree statistics of the fast plan (no GPU needed): tree nnz of B and
 * B^{-1} (B_2 = I excluded) and the algorithmic flops per block. */
fcct_status fcct_plan_tree_stats(int n, double r, double s, double t, int64_t* tree_nnz_fwd, int64_t* tree_nnz_inv,
                                 double* flops_fwd, double* flops_inv);

/* Plan cache (PlanStore, plan_cache.hpp:30-51): one `.fccplan` file per
 * (n, params), byte-compatible with the reference's format (plan_cache.hpp:11-27),
 * children as separate entries, corrupt files rebuilt in place with a warning.
 * Files written by the reference load here (the inverse factor is recomputed
 * from the stored B). */
typedef struct fcct_store_s* fcct_store;
fcct_status fcct_store_open(const char* dir, fcct_store* out);
fcct_status fcct_store_close(fcct_store store);
/* load_or_build on the host only (no GPU): warms the cache for (n, params). */
fcct_status fcct_store_warm(fcct_store store, int n, double r, double s, double t);
fcct_status fcct_store_stats(fcct_store store, int* hits, int* misses, int* rebuilt);
/* Path of the cache entry for (n, params) (PlanStore::path_for); len = buffer size. */
fcct_status fcct_store_path(fcct_store store, int n, double r, double s, double t, char* buf, int len);
/* build_plan(n, params, store) (transform.cpp:404-408): fast plan through the store. */
fcct_status fcct_plan_create_from_store(fcct_store store, int n, double r, double s, double t, int precision,
                                        int device, fcct_plan* out);

/* Batch scheduler for one process of a multi-GPU job: contiguous block range
 * [begin, end) of `total` blocks owned by `rank` of `world` (ceil split,
 * uneven tail allowed). No collective is involved. */
fcct_status fcct_shard_range(int64_t total, int rank, int world, int64_t* begin, int64_t* end);

/* ---------------------------------------------------------------------------
 * I/O either side of the path. Host buffers; text
 * outputs go to `path`, where NULL or "-" means stdout (fcct.cpp:44-54).
 * ------------------------------------------------------------------------- */

/* parse_params / SkewParams::encode (spectral.cpp:77-117): "r,s,t" with
 * fields "a/b" or decimals. encode writes at most `len` bytes incl. the NUL. */
fcct_status fcct_parse_params(const char* text, double* r, double* s, double* t);
fcct_status fcct_encode_params(double r, double s, double t, char* buf, int64_t len);

/* export_nodes_csv of skew_nodes(n, params) (spectral.cpp:155-171,180-188; CLI `zeros`):
 * "i,j,k,x,y,z" + one %.17g row per node. DEGENERATE_NODES as skew_nodes. */
fcct_status fcct_export_nodes_csv(int n, double r, double s, double t, const char* path);

/* export_geometry (voxel_io.cpp:330-334): "dx,dy,dz" + the 14 FCC shifts. */
fcct_status fcct_export_geometry(const char* path);

/* export_spectrum (voxel_io.cpp:238-261): `values_host` is one spectrum of n^3
 * complex128 values; writes "# n=.. params=..", the column header
 * "i,j,k,x,y,z,re,im,magnitude" and one %.17g row per node. */
fcct_status fcct_export_spectrum(int n, double r, double s, double t, const void* values_host, const char* path);

/* load_spectrum_csv (voxel_io.cpp:263-328). With values_host == NULL only the
 * header is read (n and params returned); otherwise the whole file is checked
 * and n^3 complex128 values written (capacity counts points). Errors: IO
 * (cannot open), MALFORMED (header / row problems), SIZE_MISMATCH_IO (row count). */
fcct_status fcct_load_spectrum_csv(const char* path, int* n, double* r, double* s, double* t, void* values_host,
                                   int64_t capacity);

/* load_grid / save_grid (voxel_io.cpp:158-176): ".json" paths hold one JSON
 * object {"metadata":{..},"n":..,"values":[..]}; other paths a little-endian
 * f64 payload plus a ".json" sidecar. metadata travels as a JSON object of
 * strings. values_host == NULL reads n (and metadata) only. */
fcct_status fcct_grid_load(const char* path, int* n, double* values_host, int64_t capacity, char* metadata_json,
                           int64_t metadata_len);
fcct_status fcct_grid_save(const char* path, int n, const double* values_host, const char* metadata_json);

/* synthetic_sword (voxel_io.cpp:200-236), n >= 8: writes n^3 samples in {0,1}
 * (metadata {"solid":"sword"}); occupancy_checksum (:336-344): FNV-1a 64. */
fcct_status fcct_synthetic_sword(int n, double* values_host);
fcct_status fcct_occupancy_checksum(const double* values_host, int64_t count, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* FCCT_GPU_H */
