// Host-side plan construction for the B200 FCC-DCT (arXiv 1807.10058).
//
// The reference derives the basis-change factor B numerically: it factors the
// eight dense child transforms with PartialPivLU and solves one column of the
// dense parent matrix at a time (transform.cpp:202-310), which is O(n^9),
// needs ~137 GB at n = 64 and leaves 1e-13..1e-9 noise in B.
//
// Here B is derived EXACTLY from the orbit structure of the transform:
//   D_n(p) = F_n S_n(p)
// with F_n[ijk, a] = e^{2 pi i a.ijk/n} (unnormalised DFT on Z_n^3) and
// S_n[a, k] = (1/24) sum_{w : wk = a mod n} e^{2 pi i (wk).p/n}. S_n is block
// diagonal over the orbits of S4 acting on Z_n^3 (blocks <= 24 x 24). The
// radix split then reads
//   (K (x) I) B = blockdiag_blk( S_m(child_blk)^{-1} ) Phi S_n,
//   Phi[(blk, a'), a] = [a mod m == a'] e^{2 pi i a.(ir,is,it)/n},
// so every column of B (and of B^{-1}) costs O(24^2) operations, in long
// double. The result reproduces the reference factor (same sparsity, same
// values up to the reference's own derivation noise) and scales to n = 64.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace fcct {

using cld = std::complex<long double>;
using Index3 = std::array<int, 3>;

// Status codes shared with include/fcct_gpu.h.
enum Status {
    ST_OK = 0,
    ST_INVALID_ARGUMENT = 1,
    ST_SIZE_MISMATCH = 2,
    ST_ODD_SIZE = 3,
    ST_DEGENERATE_NODES = 4,
    ST_ILL_CONDITIONED = 5,
    ST_PARAMS_MISMATCH = 6,
    ST_IO = 7,
    ST_CUDA = 8,
    ST_DERIVATION = 9,
    ST_MALFORMED = 10,        // MalformedFile (io category)
    ST_SIZE_MISMATCH_IO = 11, // SizeMismatch(..., ErrorCategory::io)
};

struct FcctError : std::runtime_error {
    int code;
    FcctError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// SkewParams (spectral.hpp:13-27): grid offsets in turns.
struct Params {
    double r = 0.0, s = 0.0, t = 0.0;
    bool operator==(const Params& o) const { return r == o.r && s == o.s && t == o.t; }
    static Params canonical() { return Params{0.125, 0.0, 0.375}; }  // spectral.cpp:47
    // SkewParams::child (spectral.cpp:49-51)
    Params child(int ir, int is, int it) const {
        return Params{(r + ir) / 2.0, (s + is) / 2.0, (t + it) / 2.0};
    }
};

inline int64_t cube(int n) { return static_cast<int64_t>(n) * n * n; }

// The 24 matrices of S4 in the reference's BFS order (weyl_s4.cpp:54-92).
const std::array<std::array<int, 9>, 24>& s4_group();

// e^{2 pi i turns}, argument reduced mod 1 in long double first.
cld unit_phase_ld(long double turns);

// Orbits of S4 acting on Z_n^3 (lex index a = (a0*n + a1)*n + a2).
struct Orbits {
    int n = 0;
    std::vector<int32_t> orbit_of;  // lex index -> orbit id
    std::vector<int32_t> pos;       // lex index -> position inside its orbit
    std::vector<std::vector<int32_t>> members;
};
const Orbits& orbits(int n);  // cached per n

// S_n(p) restricted to each orbit (|O| x |O| row-major, rows = Fourier index,
// cols = polynomial index), and its inverse.
struct OrbitBlocks {
    int n = 0;
    Params p;
    const Orbits* orb = nullptr;
    std::vector<std::vector<cld>> S, Sinv;
    double worst_condition = 0.0;  // max 1-norm condition over the blocks
};
OrbitBlocks orbit_blocks(int n, const Params& p);

// The reference's condition estimate (condition_with_lu, transform.cpp:91-111):
// the exact 1-norm of A times the largest ||A^{-1} v||_1 / ||v||_1 over the unit
// vectors e_0, e_{dim/2}, e_{dim-1} and five mt19937(12345) (+-1 +- i) probes.
// It is what IllConditioned is raised on (require_condition, transform.cpp:113-117):
// dense_transform (n^3 <= 512), assemble_direct, every child of derive_basis and
// the radix kernel. inf when A is singular.
double reference_condition_dense(const std::vector<cld>& A, const std::vector<cld>& Ainv, int64_t dim);
// Same estimate for D_n(p) = F_n S_n(p) without forming D: ||D||_1 column by
// column (each column is <= 24 plane waves), A^{-1} v = S^{-1} F^{-1} v.
double reference_condition(int n, const Params& p);
// ||D_n(p)||_1 on a GPU (registered by the C-ABI layer; < 0 = unavailable).
// Used for n^3 >= 4096, where the host column sums cost seconds.
using ColNormHook = double (*)(int n, const Params& p);
void set_colnorm_hook(ColNormHook hook);

// Sparse matrix in CSR (rows), long double values.
struct SparseLD {
    int64_t dim = 0;
    std::vector<int64_t> rowptr;
    std::vector<int32_t> col;
    std::vector<cld> val;
    int64_t nnz() const { return static_cast<int64_t>(val.size()); }
};

// One node of the plan tree (TransformPlan, transform.hpp:67-114).
struct PlanNode {
    int n = 0;
    Params p;
    bool radix = false;
    // radix2: K = D_2(p) row-major [blk][g], K^{-1}, B and B^{-1}, children
    std::array<cld, 64> K{}, Kinv{};
    SparseLD B, Binv;
    std::array<std::shared_ptr<const PlanNode>, 8> children;
    // direct (n odd or n == 1): D and D^{-1}, row-major N x N
    std::vector<cld> D, Dinv;
    double condition = 0.0;
};

// One radix node over given children (build_plan_node with a child source,
// plan_internal.hpp:10-13): K, K^{-1}, B, B^{-1} derived exactly.
std::shared_ptr<const PlanNode> build_radix_node(int n, const Params& p,
                                                 const std::array<std::shared_ptr<const PlanNode>, 8>& children);

// B^{-1} by connected components of B, each inverted densely in long double
// (plan_cache.cpp): used for a loaded or a perturbed basis factor.
SparseLD invert_sparse(const SparseLD& B);

// True when B is the identity (entries within 1e-15 of 1, derivation rounding). B_2 = I holds for every offset, so the
// executors skip that stage; a perturbed B_2 (with_perturbed_basis) is applied.
bool basis_is_identity(const SparseLD& B);

inline bool level_identity(const std::vector<const PlanNode*>& level, bool inverse) {
    for (const PlanNode* nd : level)
        if (!basis_is_identity(inverse ? nd->Binv : nd->B)) return false;
    return true;
}

// Dense inverse (Gauss-Jordan, partial pivoting, long double), row-major;
// *cond receives the exact 1-norm condition.
std::vector<cld> dense_inverse(const std::vector<cld>& a, int64_t dim, double* cond);

// Text encoding of an offset (encode_param, spectral.cpp:53-75).
std::string encode_param(double value);

// Builds the tree (PlanBuilder::make, transform.cpp:382-401): direct for odd n
// or n == 1, radix2 with 8 children otherwise. Throws FcctError.
std::shared_ptr<const PlanNode> build_tree(int n, const Params& p);

// radix_permutation (transform.cpp:171-194). Throws OddSize / invalid_argument.
std::vector<uint64_t> radix_permutation(int n);

// Composite output position of stacked (deepest-level) element i for a
// full radix tree of size n (power of two): Z_s(i) = perm_s[blk*m^3 + Z_m(j)].
std::vector<int32_t> output_order(int n);

// Dense D_n(p) entry (ColumnEvaluator semantics, transform.cpp:35-82).
cld dense_entry(int n, const Params& p, const Index3& node, const Index3& kappa);

// Spectral coordinates (x, y, z) of the skew nodes in lexicographic order
// (skew_nodes + coords_from_uvw, spectral.cpp:155-171, chebyshev.cpp:30-85).
std::vector<std::array<std::complex<double>, 3>> node_coords(int n, const Params& p);

// Node degeneracy check (check_not_degenerate, spectral.cpp:26-43), n <= 16.
void check_nodes(int n, const Params& p);

// Tree statistics.
int64_t tree_nnz(const PlanNode& node, bool inverse, bool with_b2);
int tree_levels(int n);

// Per-block algorithmic flops: 8 * (nnz_tree + 8 N log2 n).
double algorithmic_flops(const PlanNode& root, bool inverse);

}  // namespace fcct
