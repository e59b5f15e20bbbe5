// Host side of the large-n orbit-FFT executor (orbit_big.hpp): the orbit blocks
// of S_n(p) / S_n(p)^{-1} as column-major coefficient blocks, one row per
// natural position.
#include <array>
#include <cmath>
#include <complex>
#include <numbers>

#include "orbit_big.hpp"
#include "plan.hpp"

namespace fcct {

namespace {

int group_index(const std::array<int, 9>& m) {
    const auto& g = s4_group();
    for (int i = 0; i < 24; ++i)
        if (g[i] == m) return i;
    return -1;
}

std::array<int, 9> mat_mul(const std::array<int, 9>& a, const std::array<int, 9>& b) {
    std::array<int, 9> c{};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k) c[3 * i + j] += a[3 * i + k] * b[3 * k + j];
    return c;
}

std::array<int, 3> mat_vec(const std::array<int, 9>& a, const std::array<int, 3>& v) {
    return {a[0] * v[0] + a[1] * v[1] + a[2] * v[2], a[3] * v[0] + a[4] * v[1] + a[5] * v[2],
            a[6] * v[0] + a[7] * v[1] + a[8] * v[2]};
}

int floor_div(int a, int n) { return (a >= 0) ? a / n : -((-a + n - 1) / n); }

}  // namespace

bool compile_orbit_big(int n, const Params& p, bool inverse, OrbitBigHost& h, bool generate) {
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
    const auto& G = s4_group();
    h.gen = (!inverse && generate) ? 1 : 0;
    h.pr = p.r;
    h.ps = p.s;
    h.pt = p.t;
    if (h.gen) {
        h.mpack.assign(N, 0u);
        h.mtab.resize(24 * 24);
        for (int a = 0; a < 24; ++a)
            for (int b = 0; b < 24; ++b) {
                // g_b^{-1}: the group element whose product with g_b is the identity
                int binv = -1;
                for (int c = 0; c < 24 && binv < 0; ++c)
                    if (group_index(mat_mul(G[c], G[b])) == 0) binv = c;
                h.mtab[a * 24 + b] = static_cast<uint8_t>(group_index(mat_mul(G[a], G[binv])));
            }
        for (const auto& g : G) h.grp.insert(h.grp.end(), g.begin(), g.end());
    }
    std::vector<std::array<int, 3>> carries;  // distinct t vectors
    int64_t slots = 0, coefs = 0;
    for (int o = 0; o < norb; ++o) {
        const auto& mem = orb.members[o];
        const int s = static_cast<int>(mem.size());
        h.orbit_off[o] = static_cast<int32_t>(slots);
        bool gen_orbit = h.gen && s == 24;
        if (h.gen && s != 24 && s > 12) return false;  // (S4 orbits are 24 or at most 12)
        std::array<uint32_t, 24> pack{};
        if (gen_orbit) {  // member j = g_j k0 - n t_j: g_j is unique on a free orbit
            const Index3 k0 = {static_cast<int>(mem[0] / (n * n)), static_cast<int>((mem[0] / n) % n),
                               static_cast<int>(mem[0] % n)};
            for (int j = 0; j < 24 && gen_orbit; ++j) {
                int gj = -1;
                std::array<int, 3> t{};
                for (int g = 0; g < 24; ++g) {
                    const auto u = mat_vec(G[g], {k0[0], k0[1], k0[2]});
                    const int64_t red = (static_cast<int64_t>(((u[0] % n) + n) % n) * n + ((u[1] % n) + n) % n) * n +
                                        ((u[2] % n) + n) % n;
                    if (red == mem[j]) {
                        gj = g;
                        t = {floor_div(u[0], n), floor_div(u[1], n), floor_div(u[2], n)};
                        break;
                    }
                }
                int tid = -1;
                for (size_t q = 0; q < carries.size(); ++q)
                    if (carries[q] == t) tid = static_cast<int>(q);
                if (tid < 0 && gj >= 0 && carries.size() < 64) {
                    tid = static_cast<int>(carries.size());
                    carries.push_back(t);
                }
                if (gj < 0 || tid < 0) {
                    gen_orbit = false;  // (not expected on a free orbit) keep its coefficient block
                    break;
                }
                pack[j] = static_cast<uint32_t>(mem[j]) | (static_cast<uint32_t>(tid) << 18) |
                          (static_cast<uint32_t>(gj) << 24) | 0x80000000u;  // bit 31: generated row
            }
        }
        h.coef_off[o] = gen_orbit ? -1 : coefs;
        for (int m = 0; m < s; ++m) {
            h.members[slots + m] = mem[m];
            h.row_orbit[slots + m] = o;
            h.row_index[slots + m] = m;
            if (h.gen) h.mpack[slots + m] = gen_orbit ? pack[m] : static_cast<uint32_t>(mem[m]);
        }
        if (h.gen) {
            if (gen_orbit) {
                // device order: slot g holds the member generated by group element g
                // (slot index = g_r, so a row's w = g_r g_c^-1 comes from a fixed table row)
                std::array<uint32_t, 24> by_g{};
                for (int j = 0; j < 24; ++j) by_g[(pack[j] >> 24) & 31u] = pack[j];
                std::copy(by_g.begin(), by_g.end(), pack.begin());
                h.fpack.insert(h.fpack.end(), pack.begin(), pack.end());
                // base_j = e^{2 pi i (g_j k0).p / n} / 24 in long double
                const Index3 k0 = {static_cast<int>(mem[0] / (n * n)), static_cast<int>((mem[0] / n) % n),
                                   static_cast<int>(mem[0] % n)};
                for (int j = 0; j < 24; ++j) {
                    const auto u = mat_vec(G[(pack[j] >> 24) & 31u], {k0[0], k0[1], k0[2]});
                    const cld b = unit_phase_ld((static_cast<long double>(p.r) * u[0] + static_cast<long double>(p.s) * u[1] +
                                                 static_cast<long double>(p.t) * u[2]) / n) / 24.0L;
                    h.fbase.push_back(static_cast<double>(b.real()));
                    h.fbase.push_back(static_cast<double>(b.imag()));
                }
            }
            else
                for (int m = 0; m < s; ++m) h.tail.push_back(static_cast<int32_t>(slots + m));
        }
        slots += s;
        if (gen_orbit)
            h.gen_rows += s;
        else
            coefs += static_cast<int64_t>(s) * s;
    }
    h.orbit_off[norb] = static_cast<int32_t>(slots);
    if (h.gen) {  // T[t][w] = e^{-2 pi i t.(w^T p)} in long double
        h.ncarry = static_cast<int>(carries.size());
        h.ttab.resize(2 * static_cast<size_t>(h.ncarry) * 24);
        for (int q = 0; q < h.ncarry; ++q)
            for (int w = 0; w < 24; ++w) {
                const auto tw = mat_vec(G[w], carries[q]);  // (w t).p = t.(w^T p)
                const long double turns = -(static_cast<long double>(p.r) * tw[0] +
                                            static_cast<long double>(p.s) * tw[1] +
                                            static_cast<long double>(p.t) * tw[2]);
                const cld v = unit_phase_ld(turns);
                h.ttab[2 * (q * 24 + w)] = static_cast<double>(v.real());
                h.ttab[2 * (q * 24 + w) + 1] = static_cast<double>(v.imag());
            }
    }
    h.coef.resize(2 * static_cast<size_t>(coefs));
    const long double scale = inverse ? 1.0L / N : 1.0L;
    for (int o = 0; o < norb; ++o) {
        if (h.coef_off[o] < 0) continue;
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
    const double cmacs = static_cast<double>(coef.size() / 2) + 24.0 * static_cast<double>(gen_rows);
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
            if (h.coef_off[o] < 0) {  // generated coefficients, exactly as the kernel forms them
                const uint32_t me = h.mpack[off + r], m0 = h.mpack[off];
                const int gr = static_cast<int>((me >> 24) & 31u), k = static_cast<int>(m0 & 0x3FFFFu);
                const int* g = &h.grp[gr * 9];
                const int k0 = k / (n * n), k1 = (k / n) % n, k2 = k % n;
                const double u0 = g[0] * k0 + g[1] * k1 + g[2] * k2, u1 = g[3] * k0 + g[4] * k1 + g[5] * k2,
                             u2 = g[6] * k0 + g[7] * k1 + g[8] * k2;
                double turns = (h.pr * u0 + h.ps * u1 + h.pt * u2) / n;
                turns -= std::floor(turns);
                const cd base = cd{std::cos(2 * std::numbers::pi * turns), std::sin(2 * std::numbers::pi * turns)} / 24.0;
                for (int c = 0; c < s; ++c) {
                    const uint32_t mc = h.mpack[off + c];
                    const int w = h.mtab[gr * 24 + ((mc >> 24) & 31u)], q = static_cast<int>((mc >> 18) & 63u);
                    acc += cd{h.ttab[2 * (q * 24 + w)], h.ttab[2 * (q * 24 + w) + 1]} * x[mc & 0x3FFFFu];
                }
                acc *= base;
            } else {
                for (int c = 0; c < s; ++c) {
                    const size_t e = static_cast<size_t>(h.coef_off[o] + static_cast<int64_t>(c) * s + r);
                    acc += cd{h.coef[2 * e], h.coef[2 * e + 1]} * x[h.members[off + c]];
                }
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
