// Host side of the large-n orbit-FFT executor (orbit_big.hpp): the orbit blocks
// of S_n(p) / S_n(p)^{-1} as column-major coefficient blocks, one row per
// natural position.
#include <cmath>
#include <complex>
#include <numbers>

#include "orbit_big.hpp"
#include "plan.hpp"

namespace fcct {

bool compile_orbit_big(int n, const Params& p, bool inverse, OrbitBigHost& h) {
    if (n != 32 && n != 64) return false;
    const int N = static_cast<int>(cube(n));
    OrbitBlocks ob = orbit_blocks(n, p);
    // the plan tree carries the reference's condition gates (plan.cpp); a singular
    // orbit block (no S^{-1}) leaves this executor unbuilt
    if (!std::isfinite(ob.worst_condition)) return false;
    const Orbits& orb = *ob.orb;
    h = OrbitBigHost{};
    h.n = n;
    h.N = N;
    h.dir = inverse ? 1 : 0;
    const int norb = static_cast<int>(orb.members.size());
    h.orbit_off.resize(norb + 1);
    h.coef_off.resize(norb);
    h.row_orbit.resize(N);
    h.row_index.resize(N);
    h.members.resize(N);
    int64_t slots = 0, coefs = 0;
    for (int o = 0; o < norb; ++o) {
        const int s = static_cast<int>(orb.members[o].size());
        h.orbit_off[o] = static_cast<int32_t>(slots);
        h.coef_off[o] = coefs;
        for (int m = 0; m < s; ++m) {
            h.members[slots + m] = orb.members[o][m];
            h.row_orbit[slots + m] = o;
            h.row_index[slots + m] = m;
        }
        slots += s;
        coefs += static_cast<int64_t>(s) * s;
    }
    h.orbit_off[norb] = static_cast<int32_t>(slots);
    h.coef.resize(2 * static_cast<size_t>(coefs));
    const long double scale = inverse ? 1.0L / N : 1.0L;
    for (int o = 0; o < norb; ++o) {
        const int s = static_cast<int>(orb.members[o].size());
        const std::vector<cld>& M = inverse ? ob.Sinv[o] : ob.S[o];  // [row][col]
        for (int r = 0; r < s; ++r)
            for (int c = 0; c < s; ++c) {
                const cld v = M[static_cast<size_t>(r) * s + c] * scale;
                const size_t e = static_cast<size_t>(h.coef_off[o] + static_cast<int64_t>(c) * s + r);
                h.coef[2 * e] = static_cast<double>(v.real());
                h.coef[2 * e + 1] = static_cast<double>(v.imag());
            }
    }
    return true;
}

double OrbitBigHost::exec_flops() const {
    // 8 flops per complex MAC of the orbit blocks, plus the radix-2 lines
    const double cmacs = static_cast<double>(coef.size() / 2);
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    double twiddles = 0;
    for (int half = n / 2; half >= 1; half /= 2)
        for (int j = 0; j < half; ++j) {
            const int e = j * (n / (2 * half));
            if (e != 0 && 4 * e != n) twiddles += n / (2 * half);
        }
    return 8.0 * cmacs + 3.0 * n * n * ((n / 2.0) * lg * 4.0 + 6.0 * twiddles);
}

// Host emulation (CPU tests): the S pass exactly as the kernel indexes the
// coefficient blocks, then the three axis DFTs. in / out: complex128 rows.
void emulate_orbit_big(const OrbitBigHost& h, const double* in, double* out, int64_t batch) {
    using cd = std::complex<double>;
    const int n = h.n, N = h.N;
    auto dft3 = [&](std::vector<cd>& v, int sign) {
        std::vector<cd> line(n), res(n);
        for (int axis = 0; axis < 3; ++axis)
            for (int u = 0; u < n; ++u)
                for (int w = 0; w < n; ++w) {
                    auto at = [&](int x) {
                        int ijk[3];
                        ijk[axis] = x;
                        ijk[axis == 0 ? 1 : 0] = u;
                        ijk[axis == 2 ? 1 : 2] = w;
                        return (ijk[0] * n + ijk[1]) * n + ijk[2];
                    };
                    for (int x = 0; x < n; ++x) line[x] = v[at(x)];
                    for (int q = 0; q < n; ++q) {
                        cd acc{0, 0};
                        for (int x = 0; x < n; ++x) {
                            const double ang = sign * 2.0 * std::numbers::pi * ((x * q) % n) / n;
                            acc += line[x] * cd{std::cos(ang), std::sin(ang)};
                        }
                        res[q] = acc;
                    }
                    for (int x = 0; x < n; ++x) v[at(x)] = res[x];
                }
    };
    std::vector<cd> x(N), y(N);
    for (int64_t b = 0; b < batch; ++b) {
        for (int a = 0; a < N; ++a) x[a] = cd{in[2 * (b * N + a)], in[2 * (b * N + a) + 1]};
        if (h.dir == 1) dft3(x, -1);
        for (int row = 0; row < N; ++row) {
            const int o = h.row_orbit[row], r = h.row_index[row];
            const int off = h.orbit_off[o], s = h.orbit_off[o + 1] - off;
            cd acc{0, 0};
            for (int c = 0; c < s; ++c) {
                const size_t e = static_cast<size_t>(h.coef_off[o] + static_cast<int64_t>(c) * s + r);
                acc += cd{h.coef[2 * e], h.coef[2 * e + 1]} * x[h.members[off + c]];
            }
            y[h.members[off + r]] = acc;
        }
        if (h.dir == 0) dft3(y, +1);
        for (int a = 0; a < N; ++a) {
            out[2 * (b * N + a)] = y[a].real();
            out[2 * (b * N + a) + 1] = y[a].imag();
        }
    }
}

}  // namespace fcct
