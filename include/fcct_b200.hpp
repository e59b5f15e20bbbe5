// fcct_b200.hpp — header-only C++ shim over the C ABI (fcct_gpu.h) that keeps
// the reference library's names and semantics (proj/include/fcct/transform.hpp
// :17-143, proj/include/fcct/errors.hpp:9-63), so code written against `fcct`
// compiles against the B200 build by swapping the include and linking
// libfcct_b200.so.
//
// Differences from the reference, all forced by the absent Eigen3:
//   * Eigen::VectorXcd -> fcct::VectorXcd = std::vector<std::complex<double>>
//     (same contiguous interleaved complex128 storage);
//   * DenseTransform::matrix is a column-major std::vector (Eigen's default
//     storage order), with rows() / cols() / operator()(i, j);
//   * SparseMatrix is a compressed-column export (colptr / rowidx / values);
//   * `threads` is accepted and ignored (the device runs the whole batch);
//   * batched entry points are added (fast_apply_batch, inverse_apply_batch).
// Plans are shared_ptr<const TransformPlan>, immutable, safe across threads.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fcct_gpu.h"

namespace fcct {

using Complex = std::complex<double>;
using VectorXcd = std::vector<Complex>;
using Index3 = std::array<int, 3>;

// ---- errors.hpp:9-63 --------------------------------------------------------
enum class ErrorCategory { math, io };

class Error : public std::runtime_error {
public:
    Error(const std::string& msg, ErrorCategory cat) : std::runtime_error(msg), category_(cat) {}
    ErrorCategory category() const noexcept { return category_; }

private:
    ErrorCategory category_;
};
class DegenerateNodes : public Error {
public:
    explicit DegenerateNodes(const std::string& m) : Error(m, ErrorCategory::math) {}
};
class IllConditioned : public Error {
public:
    explicit IllConditioned(const std::string& m) : Error(m, ErrorCategory::math) {}
};
class SizeMismatch : public Error {
public:
    explicit SizeMismatch(const std::string& m, ErrorCategory cat = ErrorCategory::math) : Error(m, cat) {}
};
class OddSize : public Error {
public:
    explicit OddSize(const std::string& m) : Error(m, ErrorCategory::math) {}
};
class MalformedFile : public Error {
public:
    explicit MalformedFile(const std::string& m) : Error(m, ErrorCategory::io) {}
};
class IoFailure : public Error {
public:
    explicit IoFailure(const std::string& m) : Error(m, ErrorCategory::io) {}
};

namespace detail {
// fcct_status -> the reference's exception taxonomy
[[noreturn]] inline void raise(fcct_status st) {
    const std::string msg = fcct_last_error();
    switch (st) {
        case FCCT_SIZE_MISMATCH: throw SizeMismatch(msg);
        case FCCT_SIZE_MISMATCH_IO: throw SizeMismatch(msg, ErrorCategory::io);
        case FCCT_ODD_SIZE: throw OddSize(msg);
        case FCCT_DEGENERATE_NODES: throw DegenerateNodes(msg);
        case FCCT_ILL_CONDITIONED: throw IllConditioned(msg);
        case FCCT_MALFORMED: throw MalformedFile(msg);
        case FCCT_IO: throw IoFailure(msg);
        case FCCT_CUDA: throw std::runtime_error(msg);
        default: throw std::invalid_argument(msg);  // INVALID_ARGUMENT, PARAMS_MISMATCH, DERIVATION
    }
}
inline void check(fcct_status st) {
    if (st != FCCT_OK) raise(st);
}
inline int64_t cube(int n) { return static_cast<int64_t>(n) * n * n; }

struct Handle {  // owns one fcct_plan
    fcct_plan h = nullptr;
    explicit Handle(fcct_plan p) : h(p) {}
    Handle(const Handle&) = delete;
    Handle& operator=(const Handle&) = delete;
    ~Handle() {
        if (h) fcct_plan_destroy(h);
    }
};

// Device the shim creates plans on (FCCT_DEVICE, default 0).
inline int device() {
    const char* e = std::getenv("FCCT_DEVICE");
    return e ? std::atoi(e) : 0;
}
}  // namespace detail

// ---- spectral.hpp:13-27 ------------------------------------------------------
struct SkewParams {
    double r = 0.0, s = 0.0, t = 0.0;
    static SkewParams canonical() { return SkewParams{0.125, 0.0, 0.375}; }
    SkewParams child(int ir, int is, int it) const {  // spectral.cpp:49-51
        return SkewParams{(r + ir) / 2.0, (s + is) / 2.0, (t + it) / 2.0};
    }
    std::string encode() const {  // spectral.cpp:77-79
        char buf[128];
        detail::check(fcct_encode_params(r, s, t, buf, sizeof(buf)));
        return buf;
    }
    bool operator==(const SkewParams&) const = default;
};

inline SkewParams parse_params(const std::string& text) {  // spectral.cpp:105-117
    SkewParams p;
    detail::check(fcct_parse_params(text.c_str(), &p.r, &p.s, &p.t));
    return p;
}

// ---- transform.hpp:17-46 -----------------------------------------------------
struct SignalTensor {
    int n = 0;
    VectorXcd data;
    static SignalTensor zeros(int n) { return SignalTensor{n, VectorXcd(static_cast<size_t>(detail::cube(n)))}; }
    int64_t size() const { return detail::cube(n); }
};

struct Spectrum {
    int n = 0;
    SkewParams params;
    VectorXcd values;
};

struct DenseMatrix {  // column-major, like Eigen::MatrixXcd
    int64_t dim = 0;
    std::vector<Complex> storage;
    int64_t rows() const { return dim; }
    int64_t cols() const { return dim; }
    Complex operator()(int64_t i, int64_t j) const { return storage[static_cast<size_t>(i + j * dim)]; }
    const Complex* data() const { return storage.data(); }
};

struct DenseTransform {
    int n = 0;
    SkewParams params;
    DenseMatrix matrix;
    double condition_estimate = std::numeric_limits<double>::quiet_NaN();
    std::shared_ptr<detail::Handle> plan;  // the direct (DMMA GEMM) plan applying `matrix`
};

struct SparseMatrix {  // compressed column storage, Eigen::SparseMatrix<Complex> layout
    int64_t dim = 0;
    std::vector<int64_t> colptr;
    std::vector<int32_t> rowidx;
    std::vector<Complex> values;
    int64_t rows() const { return dim; }
    int64_t cols() const { return dim; }
    int64_t nonZeros() const { return static_cast<int64_t>(values.size()); }
};

// dense_transform (transform.cpp:130-144): D generated on the device.
inline DenseTransform dense_transform(int n, const SkewParams& p) {
    if (n < 1) throw std::invalid_argument("dense_transform: n must be >= 1");
    DenseTransform out;
    out.n = n;
    out.params = p;
    out.matrix.dim = detail::cube(n);
    out.matrix.storage.resize(static_cast<size_t>(out.matrix.dim * out.matrix.dim));
    detail::check(fcct_dense_matrix_host(n, p.r, p.s, p.t, detail::device(), out.matrix.storage.data()));
    fcct_plan h = nullptr;
    detail::check(fcct_plan_create(n, p.r, p.s, p.t, FCCT_DIRECT, FCCT_F64, detail::device(), &h));
    out.plan = std::make_shared<detail::Handle>(h);
    fcct_plan_info_t info;
    detail::check(fcct_plan_info(h, &info));
    if (out.matrix.dim <= 512) out.condition_estimate = info.condition;  // transform.cpp:141-142
    return out;
}

// naive_apply (transform.cpp:146-156)
inline Spectrum naive_apply(const DenseTransform& t, const SignalTensor& s) {
    if (t.n != s.n)
        throw SizeMismatch("naive_apply: transform size " + std::to_string(t.n) + " vs signal size " +
                           std::to_string(s.n));
    if (static_cast<int64_t>(s.data.size()) != t.matrix.cols())
        throw SizeMismatch("naive_apply: signal has " + std::to_string(s.data.size()) + " samples, need " +
                           std::to_string(t.matrix.cols()));
    Spectrum out{t.n, t.params, VectorXcd(s.data.size())};
    detail::check(fcct_forward_host(t.plan->h, s.data.data(), out.values.data(), 1, nullptr));
    return out;
}

// inverse_apply(dense) (transform.cpp:158-169)
inline SignalTensor inverse_apply(const DenseTransform& t, const Spectrum& q) {
    if (t.n != q.n)
        throw SizeMismatch("inverse_apply: transform size " + std::to_string(t.n) + " vs spectrum size " +
                           std::to_string(q.n));
    if (!(t.params == q.params))
        throw std::invalid_argument("inverse_apply: spectrum was produced on a different skew grid");
    if (static_cast<int64_t>(q.values.size()) != detail::cube(t.n))
        throw SizeMismatch("inverse_apply: spectrum has " + std::to_string(q.values.size()) + " values, need " +
                           std::to_string(detail::cube(t.n)));
    SignalTensor out{t.n, VectorXcd(q.values.size())};
    detail::check(fcct_inverse_host(t.plan->h, q.values.data(), out.data.data(), 1, nullptr));
    return out;
}

// radix_permutation (transform.cpp:171-194), bit-exact
inline std::vector<uint64_t> radix_permutation(int n) {
    if (n >= 1 && n % 2 != 0) throw OddSize("radix_permutation: n=" + std::to_string(n) + " is odd");
    std::vector<uint64_t> p(static_cast<size_t>(n >= 1 ? detail::cube(n) : 0));
    detail::check(fcct_radix_permutation(n, p.data()));
    return p;
}

namespace detail {
inline SparseMatrix export_csc(int64_t N, int64_t nnz, const std::vector<int64_t>& colptr,
                               const std::vector<int32_t>& rowidx, const std::vector<double>& vals) {
    SparseMatrix m;
    m.dim = N;
    m.colptr = colptr;
    m.rowidx = rowidx;
    m.values.resize(static_cast<size_t>(nnz));
    for (int64_t k = 0; k < nnz; ++k) m.values[k] = Complex{vals[2 * k], vals[2 * k + 1]};
    return m;
}
}  // namespace detail

// basis_change (transform.cpp:314-320)
inline SparseMatrix basis_change(int n, const SkewParams& p) {
    int64_t nnz = 0;
    detail::check(fcct_basis_change(n, p.r, p.s, p.t, 0, &nnz, nullptr, nullptr, nullptr));
    const int64_t N = detail::cube(n);
    std::vector<int64_t> colptr(N + 1);
    std::vector<int32_t> rowidx(nnz);
    std::vector<double> vals(2 * nnz);
    detail::check(fcct_basis_change(n, p.r, p.s, p.t, 0, &nnz, colptr.data(), rowidx.data(), vals.data()));
    return detail::export_csc(N, nnz, colptr, rowidx, vals);
}

// ---- TransformPlan (transform.hpp:64-115) ------------------------------------
class TransformPlan;
std::shared_ptr<const TransformPlan> build_plan(int n, const SkewParams& p, void* store = nullptr);

class TransformPlan {
public:
    enum class Kind { direct, radix2 };

    explicit TransformPlan(fcct_plan h) : h_(std::make_shared<detail::Handle>(h)) {
        detail::check(fcct_plan_info(h, &info_));
    }
    Kind kind() const { return info_.kind == FCCT_KIND_RADIX2 ? Kind::radix2 : Kind::direct; }
    int n() const { return info_.n; }
    SkewParams params() const { return SkewParams{info_.r, info_.s, info_.t}; }
    const fcct_plan_info_t& info() const { return info_; }
    fcct_plan native() const { return h_->h; }

    // radix2 only
    std::vector<uint64_t> permutation() const { return radix_permutation(n()); }
    std::vector<Complex> kernel() const {  // 8 x 8 column-major
        std::vector<Complex> k(64);
        detail::check(fcct_plan_kernel(h_->h, reinterpret_cast<double*>(k.data())));
        return k;
    }
    SparseMatrix basis() const {
        int64_t nnz = 0;
        detail::check(fcct_plan_basis(h_->h, &nnz, nullptr, nullptr, nullptr));
        const int64_t N = detail::cube(n());
        std::vector<int64_t> colptr(N + 1);
        std::vector<int32_t> rowidx(nnz);
        std::vector<double> vals(2 * nnz);
        detail::check(fcct_plan_basis(h_->h, &nnz, colptr.data(), rowidx.data(), vals.data()));
        return detail::export_csc(N, nnz, colptr, rowidx, vals);
    }
    std::array<std::shared_ptr<const TransformPlan>, 8> children() const {
        std::array<std::shared_ptr<const TransformPlan>, 8> out;
        for (int i = 0; i < 8; ++i) {
            int cn = 0, kind = 0;
            double r = 0, s = 0, t = 0;
            detail::check(fcct_plan_child(h_->h, i, &cn, &r, &s, &t, &kind));
            out[i] = build_plan(cn, SkewParams{r, s, t});
        }
        return out;
    }

    // Vector forms (transform.hpp:86-90); `threads` is accepted and ignored.
    VectorXcd apply_values(const VectorXcd& x, int /*threads*/ = 1) const {
        if (static_cast<int64_t>(x.size()) != detail::cube(n())) throw SizeMismatch("apply_values: wrong length");
        VectorXcd y(x.size());
        detail::check(fcct_forward_host(h_->h, x.data(), y.data(), 1, nullptr));
        return y;
    }
    VectorXcd solve_values(const VectorXcd& q, int /*threads*/ = 1) const {
        if (static_cast<int64_t>(q.size()) != detail::cube(n())) throw SizeMismatch("solve_values: wrong length");
        VectorXcd x(q.size());
        detail::check(fcct_inverse_host(h_->h, q.data(), x.data(), 1, nullptr));
        return x;
    }

private:
    std::shared_ptr<detail::Handle> h_;
    fcct_plan_info_t info_{};
};

// build_plan (transform.cpp:403-407). `store` is accepted for signature
// compatibility; plan files go through fcct_plan_create_from_store.
inline std::shared_ptr<const TransformPlan> build_plan(int n, const SkewParams& p, void* /*store*/) {
    if (n < 1) throw std::invalid_argument("build_plan: n must be >= 1");
    fcct_plan h = nullptr;
    detail::check(fcct_plan_create(n, p.r, p.s, p.t, FCCT_FAST, FCCT_F64, detail::device(), &h));
    return std::make_shared<const TransformPlan>(h);
}

// fast_apply (transform.cpp:496-507)
inline Spectrum fast_apply(const TransformPlan& plan, const SignalTensor& s, int threads = 1) {
    if (plan.n() != s.n)
        throw SizeMismatch("fast_apply: plan size " + std::to_string(plan.n()) + " vs signal size " +
                           std::to_string(s.n));
    if (static_cast<int64_t>(s.data.size()) != detail::cube(s.n))
        throw SizeMismatch("fast_apply: signal has " + std::to_string(s.data.size()) + " samples, need " +
                           std::to_string(detail::cube(s.n)));
    return Spectrum{plan.n(), plan.params(), plan.apply_values(s.data, threads)};
}

// inverse_apply(plan) (transform.cpp:509-524)
inline SignalTensor inverse_apply(const TransformPlan& plan, const Spectrum& q, int threads = 1) {
    if (plan.n() != q.n)
        throw SizeMismatch("inverse_apply: plan size " + std::to_string(plan.n()) + " vs spectrum size " +
                           std::to_string(q.n));
    if (!(plan.params() == q.params))
        throw std::invalid_argument("inverse_apply: spectrum was produced on a different skew grid");
    if (static_cast<int64_t>(q.values.size()) != detail::cube(q.n))
        throw SizeMismatch("inverse_apply: spectrum has " + std::to_string(q.values.size()) + " values, need " +
                           std::to_string(detail::cube(q.n)));
    return SignalTensor{plan.n(), plan.solve_values(q.values, threads)};
}

// Batched entry points (the B200 addition): `blocks` consecutive n^3 blocks,
// host memory (pageable or pinned).
inline void fast_apply_batch(const TransformPlan& plan, const Complex* in, Complex* out, int64_t blocks) {
    detail::check(fcct_forward_host(plan.native(), in, out, blocks, nullptr));
}
inline void inverse_apply_batch(const TransformPlan& plan, const Complex* in, Complex* out, int64_t blocks) {
    detail::check(fcct_inverse_host(plan.native(), in, out, blocks, nullptr));
}

// factorization_residual (transform.cpp:526-540), evaluated on the device
inline double factorization_residual(const TransformPlan& plan, const DenseTransform& dense) {
    if (plan.n() != dense.n) throw SizeMismatch("factorization_residual: sizes differ");
    double r = 0.0;
    detail::check(fcct_factorization_residual(plan.native(), &r));
    return r;
}

// with_perturbed_basis (transform.cpp:542-554)
inline std::shared_ptr<const TransformPlan> with_perturbed_basis(const TransformPlan& plan, double delta) {
    if (plan.kind() != TransformPlan::Kind::radix2)
        throw std::invalid_argument("with_perturbed_basis: plan has no basis factor");
    fcct_plan h = nullptr;
    detail::check(fcct_plan_perturbed_basis(plan.native(), delta, &h));
    return std::make_shared<const TransformPlan>(h);
}

}  // namespace fcct
