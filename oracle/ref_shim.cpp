// ===========================================================================
// REFERENCE SHIM — TEST INFRASTRUCTURE ONLY.
//
// A C entry layer over the reference's own Eigen-free sources, compiled in
// place from /root/reference/proj/src/{weyl_s4,chebyshev,spectral}.cpp by
// oracle/ref.mk into oracle/_ref/libfcct_ref.so (git-ignored). The reference's
// transform.cpp needs Eigen3 and cannot be built here, but
// these three files carry the group, the node set and the Chebyshev
// evaluation that every entry of D_n is made of:
//   D_n[node i, kappa] = T_kappa(node_i) = cheb_eval_uvw(kappa, uvw_i)
// (chebyshev.cpp:67-74; the ColumnEvaluator of transform.cpp:35-82 evaluates
// the same Laurent sum through axis tables). tests/test_ref_pins.py checks
// the oracle (fcct_oracle.cpp) against these functions, and
// tests/golden/make_ref_golden.py freezes their outputs into
// tests/golden/ref_*.npz for the GPU parity tests (the GPU box has no
// /root/reference).
// ===========================================================================
#include <complex>
#include <cstdint>
#include <cstring>
#include <string>

#include "fcct/chebyshev.hpp"
#include "fcct/errors.hpp"
#include "fcct/spectral.hpp"
#include "fcct/weyl_s4.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const fcct::DegenerateNodes& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void put(double* out, const std::complex<double>& v) {
    out[0] = v.real();
    out[1] = v.imag();
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// WeylGroup::s4() (weyl_s4.cpp:89-92): 24 x 9 ints in the group's own order.
int ref_group(int* out) {
    return guarded([&] {
        const auto& g = fcct::WeylGroup::s4();
        for (std::size_t e = 0; e < g.elements.size(); ++e)
            for (int k = 0; k < 9; ++k) out[e * 9 + k] = g.elements[e].m[k];
    });
}

// skew_nodes(n, p) (spectral.cpp:155-171): per node 12 doubles
// (u, v, w, x, y, z as re, im), lexicographic; status 4 = DegenerateNodes.
int ref_skew_nodes(int n, double r, double s, double t, double* out) {
    return guarded([&] {
        const auto grid = fcct::skew_nodes(n, fcct::SkewParams{r, s, t});
        for (std::size_t i = 0; i < grid.nodes.size(); ++i) {
            const auto& nd = grid.nodes[i];
            const std::complex<double> v[6] = {nd.uvw.u, nd.uvw.v, nd.uvw.w, nd.xyz.x, nd.xyz.y, nd.xyz.z};
            for (int c = 0; c < 6; ++c) put(out + i * 12 + 2 * c, v[c]);
        }
    });
}

// common_zeros(n) (spectral.cpp:136-153), same layout.
int ref_common_zeros(int n, double* out) {
    return guarded([&] {
        const auto grid = fcct::common_zeros(n);
        for (std::size_t i = 0; i < grid.nodes.size(); ++i) {
            const auto& nd = grid.nodes[i];
            const std::complex<double> v[6] = {nd.uvw.u, nd.uvw.v, nd.uvw.w, nd.xyz.x, nd.xyz.y, nd.xyz.z};
            for (int c = 0; c < 6; ++c) put(out + i * 12 + 2 * c, v[c]);
        }
    });
}

// cheb_eval_uvw(k, uvw) (chebyshev.cpp:67-74) at one point (6 doubles).
int ref_cheb_eval_uvw(int k0, int k1, int k2, const double* uvw, double* out) {
    return guarded([&] {
        const fcct::UVWPoint p{{uvw[0], uvw[1]}, {uvw[2], uvw[3]}, {uvw[4], uvw[5]}};
        put(out, fcct::cheb_eval_uvw(fcct::Index3{k0, k1, k2}, p, fcct::WeylGroup::s4()));
    });
}

// Columns [c0, c1) of D_n(p) by the reference's own evaluation: entry
// (i, kappa) = cheb_eval_uvw(kappa, skew_nodes(n, p)[i].uvw), kappa = (j, k, q)
// lexicographic (transform.cpp:84-89). Output column-major [c1 - c0][n^3]
// complex128.
int ref_dense_columns(int n, double r, double s, double t, int64_t c0, int64_t c1, double* out) {
    return guarded([&] {
        const auto grid = fcct::skew_nodes(n, fcct::SkewParams{r, s, t});
        const auto& g = fcct::WeylGroup::s4();
        const int64_t n3 = static_cast<int64_t>(n) * n * n;
        for (int64_t col = c0; col < c1; ++col) {
            const fcct::Index3 kap{static_cast<int>(col / (n * n)), static_cast<int>((col / n) % n),
                                   static_cast<int>(col % n)};
            for (int64_t i = 0; i < n3; ++i)
                put(out + 2 * ((col - c0) * n3 + i), fcct::cheb_eval_uvw(kap, grid.nodes[i].uvw, g));
        }
    });
}

// real_coords (chebyshev.cpp:87-97) of every node of skew_nodes(n, p): [n^3][3].
int ref_real_coords(int n, double r, double s, double t, double* out) {
    return guarded([&] {
        const auto grid = fcct::skew_nodes(n, fcct::SkewParams{r, s, t});
        for (std::size_t i = 0; i < grid.nodes.size(); ++i) {
            const auto c = fcct::real_coords(grid.nodes[i].xyz);
            for (int a = 0; a < 3; ++a) out[i * 3 + a] = c[a];
        }
    });
}

// SkewParams::child (spectral.cpp:49-51) -> out[3]; encode_param
// (spectral.cpp:53-75) of one value into buf (NUL-terminated, cap bytes).
int ref_child(double r, double s, double t, int ir, int is, int it, double* out) {
    return guarded([&] {
        const auto c = fcct::SkewParams{r, s, t}.child(ir, is, it);
        out[0] = c.r;
        out[1] = c.s;
        out[2] = c.t;
    });
}

int ref_encode_param(double v, char* buf, int cap) {
    return guarded([&] {
        const std::string e = fcct::encode_param(v);
        std::strncpy(buf, e.c_str(), static_cast<std::size_t>(cap));
        buf[cap - 1] = 0;
    });
}

}  // extern "C"
