// Calls the B200 build through the C++ shim (include/fcct_b200.hpp) the way
// reference code calls fcct (transform.hpp names), following the checks of
// proj/tests/unit/test_transform.cpp. Built and run by tests/test_cpp_shim.py.
// Usage: shim_test <out.bin>   (writes x and fast_apply(x) for n = 8, 4 blocks)
#include <cmath>
#include <cstdio>
#include <fstream>

#include "fcct_b200.hpp"

static int failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static double splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    return (static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

static double rel(const fcct::VectorXcd& a, const fcct::VectorXcd& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) num += std::norm(a[i] - b[i]), den += std::norm(b[i]);
    return std::sqrt(num / den);
}

int main(int argc, char** argv) {
    using namespace fcct;
    const SkewParams p = SkewParams::canonical();
    // radix_permutation (test_transform.cpp:105-107) and OddSize
    const auto p4 = radix_permutation(4);
    CHECK(p4.size() == 64 && p4[46] == 57);
    CHECK(throws<OddSize>([] { radix_permutation(3); }));
    // plan structure
    const auto plan = build_plan(8, p);
    CHECK(plan->kind() == TransformPlan::Kind::radix2 && plan->n() == 8);
    const auto kids = plan->children();
    CHECK(kids[5]->n() == 4 && kids[5]->params() == p.child(1, 0, 1));
    CHECK(basis_change(4, p).nonZeros() == 245);
    CHECK(build_plan(2, p)->basis().nonZeros() == 8);  // B_2 = I
    // fast vs naive, round trip (test_transform.cpp:138-183)
    const int n = 8, blocks = 4;
    const int64_t N = n * n * n;
    std::vector<Complex> x(blocks * N), y(blocks * N);
    for (int64_t i = 0; i < blocks * N; ++i) x[i] = Complex{splitmix(2 * i), splitmix(2 * i + 1)};
    const DenseTransform dense = dense_transform(n, p);
    CHECK(dense.matrix.rows() == N && std::isfinite(dense.condition_estimate));
    for (int b = 0; b < blocks; ++b) {
        SignalTensor s{n, VectorXcd(x.begin() + b * N, x.begin() + (b + 1) * N)};
        const Spectrum q = fast_apply(*plan, s, 8);
        const Spectrum qn = naive_apply(dense, s);
        CHECK(rel(q.values, qn.values) < 1e-12);
        CHECK(rel(inverse_apply(*plan, q).data, s.data) < 1e-12);
        CHECK(rel(inverse_apply(dense, qn).data, s.data) < 1e-12);
        // D(:, kappa) column of the host matrix equals the direct plan on e_kappa
        if (b == 0) {
            SignalTensor e = SignalTensor::zeros(n);
            e.data[77] = 1.0;
            const auto col = naive_apply(dense, e).values;
            double worst = 0;
            for (int64_t i = 0; i < N; ++i) worst = std::max(worst, std::abs(col[i] - dense.matrix(i, 77)));
            CHECK(worst < 1e-14);
        }
        std::copy(q.values.begin(), q.values.end(), y.begin() + b * N);
    }
    // batched entry on pageable std::vector storage: bitwise the per-block calls
    std::vector<Complex> yb(blocks * N);
    fast_apply_batch(*plan, x.data(), yb.data(), blocks);
    CHECK(yb == y);
    // errors (transform.cpp:147-154,498-521)
    CHECK(throws<SizeMismatch>([&] { fast_apply(*plan, SignalTensor::zeros(4)); }));
    CHECK(throws<std::invalid_argument>([&] {
        inverse_apply(*plan, Spectrum{n, SkewParams{0.2, 0.1, 0.3}, VectorXcd(N)});
    }));
    CHECK(throws<SizeMismatch>([&] { naive_apply(dense, SignalTensor::zeros(4)); }));
    CHECK(throws<std::invalid_argument>([] { build_plan(0, SkewParams::canonical()); }));
    CHECK(throws<DegenerateNodes>([] { build_plan(2, SkewParams{0.0, 0.0, 0.0}); }));
    // factorization residual and its negative control (test_transform.cpp:120-136,212-220)
    CHECK(factorization_residual(*plan, dense) < 1e-12);
    CHECK(factorization_residual(*with_perturbed_basis(*plan, 1e-3), dense) > 1e-5);
    CHECK(parse_params(p.encode()) == p);
    if (argc > 1) {
        std::ofstream f(argv[1], std::ios::binary);
        f.write(reinterpret_cast<const char*>(x.data()), x.size() * sizeof(Complex));
        f.write(reinterpret_cast<const char*>(y.data()), y.size() * sizeof(Complex));
    }
    std::printf("%s: %d failures\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
