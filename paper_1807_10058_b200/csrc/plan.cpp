// Host-side plan construction (see plan.hpp for the derivation).
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <deque>
#include <future>
#include <map>
#include <mutex>
#include <numbers>
#include <random>
#include <set>
#include <thread>
#include <unordered_map>

namespace fcct {
namespace {

constexpr long double kTwoPiL = 2.0L * std::numbers::pi_v<long double>;
constexpr double kConditionLimit = 1e12;  // transform.cpp:20
// Exact factors carry only long-double rounding (~1e-18 relative); every true
// entry of B / B^{-1} is an algebraic number of size >= ~1e-3 for n <= 64.
constexpr long double kPrune = 1e-13L;

// Gauss-Jordan inverse with partial pivoting, row-major dim x dim. Returns the
// exact 1-norm condition ||A||_1 ||A^{-1}||_1 (inf when singular).
double invert_ld(const std::vector<cld>& a, int dim, std::vector<cld>& inv) {
    std::vector<cld> m(a);
    inv.assign(static_cast<size_t>(dim) * dim, cld{0, 0});
    for (int i = 0; i < dim; ++i) inv[i * dim + i] = 1;
    for (int k = 0; k < dim; ++k) {
        int best = k;
        long double bv = std::abs(m[k * dim + k]);
        for (int i = k + 1; i < dim; ++i) {
            const long double v = std::abs(m[i * dim + k]);
            if (v > bv) { bv = v; best = i; }
        }
        if (bv == 0.0L) return INFINITY;
        if (best != k)
            for (int j = 0; j < dim; ++j) {
                std::swap(m[k * dim + j], m[best * dim + j]);
                std::swap(inv[k * dim + j], inv[best * dim + j]);
            }
        const cld pinv = cld{1, 0} / m[k * dim + k];
        for (int j = 0; j < dim; ++j) {
            m[k * dim + j] *= pinv;
            inv[k * dim + j] *= pinv;
        }
        for (int i = 0; i < dim; ++i) {
            if (i == k) continue;
            const cld f = m[i * dim + k];
            if (f == cld{0, 0}) continue;
            for (int j = 0; j < dim; ++j) {
                m[i * dim + j] -= f * m[k * dim + j];
                inv[i * dim + j] -= f * inv[k * dim + j];
            }
        }
    }
    auto norm1 = [dim](const std::vector<cld>& x) {
        long double best = 0;
        for (int j = 0; j < dim; ++j) {
            long double s = 0;
            for (int i = 0; i < dim; ++i) s += std::abs(x[i * dim + j]);
            best = std::max(best, s);
        }
        return best;
    };
    return static_cast<double>(norm1(a) * norm1(inv));
}

Index3 unlex(int64_t a, int n) {
    return Index3{static_cast<int>(a / (static_cast<int64_t>(n) * n)),
                  static_cast<int>((a / n) % n), static_cast<int>(a % n)};
}
int64_t lex(const Index3& a, int n) { return (static_cast<int64_t>(a[0]) * n + a[1]) * n + a[2]; }
int mod(int a, int n) { return ((a % n) + n) % n; }

Index3 apply(const std::array<int, 9>& w, const Index3& k) {  // weyl_s4.cpp:38-43
    Index3 o{};
    for (int i = 0; i < 3; ++i) o[i] = w[i * 3] * k[0] + w[i * 3 + 1] * k[1] + w[i * 3 + 2] * k[2];
    return o;
}

// Exact factors are algebraic numbers of size >= ~1e-3; a real or imaginary
// component below 1e-15 is long-double rounding noise (e.g. cos(pi/2) or the
// imaginary part of an entry that is real in exact arithmetic) and is snapped
// to zero so real coefficients stay real.
cld snap(const cld& v) {
    constexpr long double eps = 1e-15L;
    return cld{std::fabs(v.real()) < eps ? 0.0L : v.real(), std::fabs(v.imag()) < eps ? 0.0L : v.imag()};
}

void require_condition(double cond, const std::string& what) {  // transform.cpp:113-117
    if (!(cond <= kConditionLimit))
        throw FcctError(ST_ILL_CONDITIONED,
                        what + ": condition estimate " + std::to_string(cond) + " exceeds 1e12");
}

}  // namespace

const std::array<std::array<int, 9>, 24>& s4_group() {
    // Breadth-first closure of the three generators, identity first
    // (weyl_s4.cpp:54-83).
    static const std::array<std::array<int, 9>, 24> g = [] {
        const std::array<std::array<int, 9>, 3> gens{{{-1, 0, 0, 1, 1, 0, 0, 0, 1},
                                                      {1, 1, 0, 0, -1, 0, 0, 1, 1},
                                                      {1, 0, 0, 0, 1, 1, 0, 0, -1}}};
        auto mul = [](const std::array<int, 9>& a, const std::array<int, 9>& b) {
            std::array<int, 9> o{};
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    int acc = 0;
                    for (int k = 0; k < 3; ++k) acc += a[i * 3 + k] * b[k * 3 + j];
                    o[i * 3 + j] = acc;
                }
            return o;
        };
        std::array<std::array<int, 9>, 24> out{};
        std::set<std::array<int, 9>> seen;
        std::deque<std::array<int, 9>> frontier{{1, 0, 0, 0, 1, 0, 0, 0, 1}};
        seen.insert(frontier.front());
        size_t count = 0;
        while (!frontier.empty()) {
            auto e = frontier.front();
            frontier.pop_front();
            if (count >= 24) throw std::logic_error("group closure exceeded 24 elements");
            out[count++] = e;
            for (const auto& s : gens) {
                auto nx = mul(e, s);
                if (seen.insert(nx).second) frontier.push_back(nx);
            }
        }
        if (count != 24) throw std::logic_error("group closure != 24");
        return out;
    }();
    return g;
}

std::string encode_param(double value) {  // spectral.cpp:53-75
    if (value == 0.0) return "0";
    double x = value;
    long long p0 = 0, q0 = 1, p1 = 1, q1 = 0;
    for (int step = 0; step < 40; ++step) {
        const double fa = std::floor(x);
        if (std::abs(fa) > 1e15) break;
        const long long a = static_cast<long long>(fa);
        const long long p2 = a * p1 + p0, q2 = a * q1 + q0;
        if (q2 > 1000000 || q2 < 0) break;
        if (q2 != 0 && static_cast<double>(p2) / static_cast<double>(q2) == value) {
            if (q2 == 1) return std::to_string(p2);
            return std::to_string(p2) + "/" + std::to_string(q2);
        }
        p0 = p1;
        q0 = q1;
        p1 = p2;
        q1 = q2;
        const double frac = x - fa;
        if (frac == 0.0) break;
        x = 1.0 / frac;
    }
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.17g", value);  // detail::g17 (format.hpp:9-13)
    return buf;
}

cld unit_phase_ld(long double turns) {
    turns -= std::floor(turns);
    return cld{std::cos(kTwoPiL * turns), std::sin(kTwoPiL * turns)};
}

const Orbits& orbits(int n) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<Orbits>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(n);
    if (it != cache.end()) return *it->second;
    auto o = std::make_unique<Orbits>();
    o->n = n;
    const int64_t n3 = cube(n);
    o->orbit_of.assign(n3, -1);
    o->pos.assign(n3, -1);
    const auto& g = s4_group();
    for (int64_t a = 0; a < n3; ++a) {
        if (o->orbit_of[a] >= 0) continue;
        const Index3 av = unlex(a, n);
        std::set<int64_t> members;
        for (const auto& w : g) {
            Index3 b = apply(w, av);
            for (auto& x : b) x = mod(x, n);
            members.insert(lex(b, n));
        }
        const int id = static_cast<int>(o->members.size());
        std::vector<int32_t> list(members.begin(), members.end());
        for (size_t i = 0; i < list.size(); ++i) {
            o->orbit_of[list[i]] = id;
            o->pos[list[i]] = static_cast<int32_t>(i);
        }
        o->members.push_back(std::move(list));
    }
    auto& ref = *o;
    cache.emplace(n, std::move(o));
    return ref;
}

OrbitBlocks orbit_blocks(int n, const Params& p) {
    OrbitBlocks ob;
    ob.n = n;
    ob.p = p;
    ob.orb = &orbits(n);
    const auto& g = s4_group();
    const auto& orb = *ob.orb;
    ob.S.resize(orb.members.size());
    ob.Sinv.resize(orb.members.size());
    const long double pr = p.r, ps = p.s, pt = p.t;
    for (size_t o = 0; o < orb.members.size(); ++o) {
        const auto& mem = orb.members[o];
        const int d = static_cast<int>(mem.size());
        std::vector<cld> S(static_cast<size_t>(d) * d, cld{0, 0});
        for (int j = 0; j < d; ++j) {  // polynomial index kappa = mem[j]
            const Index3 kap = unlex(mem[j], n);
            for (const auto& w : g) {
                const Index3 wk = apply(w, kap);
                Index3 a = wk;
                for (auto& x : a) x = mod(x, n);
                const int i = orb.pos[lex(a, n)];
                // e^{2 pi i (w kappa).p / n} with the unreduced exponent
                // (ColumnEvaluator prefactor, transform.cpp:51-53).
                S[static_cast<size_t>(i) * d + j] +=
                    unit_phase_ld((pr * wk[0] + ps * wk[1] + pt * wk[2]) / n) / 24.0L;
            }
        }
        const double c = invert_ld(S, d, ob.Sinv[o]);
        ob.worst_condition = std::max(ob.worst_condition, c);
        ob.S[o] = std::move(S);
    }
    return ob;
}

// ---- the reference's condition estimate (condition_with_lu, transform.cpp:91-111) ----
namespace {
ColNormHook g_colnorm_hook = nullptr;

using cd = std::complex<double>;

double l1(const std::vector<cd>& v) {
    double s = 0;
    for (const cd& z : v) s += std::abs(z);
    return s;
}

// max over the reference's eight probes of ||A^{-1} v||_1 / ||v||_1
// (transform.cpp:95-109: e_0, e_{dim/2}, e_{dim-1}, then five coin-flip vectors
// drawn from mt19937(12345) in the same order, real part first in source order).
template <class Solve>
double probe_inverse_norm(int64_t dim, Solve&& solve) {
    double inv_norm = 0.0;
    bool finite = true;
    auto take = [&](double v) {
        if (!std::isfinite(v)) finite = false;
        inv_norm = std::max(inv_norm, v);
    };
    for (int64_t j : {int64_t{0}, dim / 2, dim - 1}) {
        std::vector<cd> e(static_cast<size_t>(dim), cd{0, 0});
        e[static_cast<size_t>(j)] = 1.0;
        take(l1(solve(e)));
    }
    std::mt19937 rng(12345);
    std::uniform_int_distribution<int> coin(0, 1);
    for (int probe = 0; probe < 5; ++probe) {
        std::vector<cd> v(static_cast<size_t>(dim));
        for (int64_t i = 0; i < dim; ++i) v[static_cast<size_t>(i)] = cd(coin(rng) ? 1.0 : -1.0, coin(rng) ? 1.0 : -1.0);
        take(l1(solve(v)) / l1(v));
    }
    return finite ? inv_norm : INFINITY;
}

// ||D_n(p)||_1 on the host: column kappa of D is sum_{a in O(kappa)} S[a, kappa]
// e^{2 pi i a.x/n}; the exponent index (a.x mod n) advances incrementally.
double colnorm_host(int n, const OrbitBlocks& ob) {
    const Orbits& orb = *ob.orb;
    const int64_t N = cube(n);
    std::vector<cd> tw(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
        const cld t = unit_phase_ld(static_cast<long double>(k) / n);
        tw[k] = cd(static_cast<double>(t.real()), static_cast<double>(t.imag()));
    }
    const int nth = N >= 4096 ? std::max(1u, std::min(32u, std::thread::hardware_concurrency())) : 1;
    std::vector<double> best(nth, 0.0);
    auto work = [&](int th) {
        std::vector<cd> c;
        std::vector<Index3> a;
        std::vector<int> i0, i1, i2;
        for (int64_t kap = th; kap < N; kap += nth) {
            const int O = orb.orbit_of[kap], pk = orb.pos[kap];
            const auto& mem = orb.members[O];
            const int d = static_cast<int>(mem.size());
            c.resize(d);
            a.resize(d);
            i0.resize(d);
            i1.resize(d);
            i2.resize(d);
            for (int i = 0; i < d; ++i) {
                const cld v = ob.S[O][static_cast<size_t>(i) * d + pk];
                c[i] = cd(static_cast<double>(v.real()), static_cast<double>(v.imag()));
                a[i] = unlex(mem[i], n);
            }
            double sum = 0.0;
            for (int x0 = 0; x0 < n; ++x0) {
                for (int i = 0; i < d; ++i) i0[i] = (a[i][0] * x0) % n;
                for (int x1 = 0; x1 < n; ++x1) {
                    for (int i = 0; i < d; ++i) i1[i] = (i0[i] + a[i][1] * x1) % n, i2[i] = i1[i];
                    for (int x2 = 0; x2 < n; ++x2) {
                        cd acc{0, 0};
                        for (int i = 0; i < d; ++i) {
                            acc += c[i] * tw[i2[i]];
                            i2[i] += a[i][2];
                            if (i2[i] >= n) i2[i] -= n;
                        }
                        sum += std::abs(acc);
                    }
                }
            }
            best[th] = std::max(best[th], sum);
        }
    };
    if (nth == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int th = 0; th < nth; ++th) pool.emplace_back(work, th);
        for (auto& t : pool) t.join();
    }
    return *std::max_element(best.begin(), best.end());
}
}  // namespace

void set_colnorm_hook(ColNormHook hook) { g_colnorm_hook = hook; }

double reference_condition_dense(const std::vector<cld>& A, const std::vector<cld>& Ainv, int64_t dim) {
    long double norm_a = 0;
    for (int64_t j = 0; j < dim; ++j) {
        long double s = 0;
        for (int64_t i = 0; i < dim; ++i) s += std::abs(A[i * dim + j]);
        norm_a = std::max(norm_a, s);
    }
    for (const cld& v : Ainv)
        if (!std::isfinite(static_cast<double>(v.real())) || !std::isfinite(static_cast<double>(v.imag())))
            return INFINITY;
    const double inv = probe_inverse_norm(dim, [&](const std::vector<cd>& v) {
        std::vector<cd> x(static_cast<size_t>(dim));
        for (int64_t i = 0; i < dim; ++i) {
            cld acc{0, 0};
            for (int64_t j = 0; j < dim; ++j) acc += Ainv[i * dim + j] * cld(v[j].real(), v[j].imag());
            x[i] = cd(static_cast<double>(acc.real()), static_cast<double>(acc.imag()));
        }
        return x;
    });
    return static_cast<double>(norm_a) * inv;
}

double reference_condition(int n, const Params& p) {
    const OrbitBlocks ob = orbit_blocks(n, p);
    if (!std::isfinite(ob.worst_condition)) return INFINITY;  // a singular orbit block: D is singular
    const Orbits& orb = *ob.orb;
    const int64_t N = cube(n);
    double norm_a = -1.0;
    if (N >= 4096 && g_colnorm_hook) norm_a = g_colnorm_hook(n, p);
    if (norm_a < 0) norm_a = colnorm_host(n, ob);
    // D^{-1} v = S^{-1} F^{-1} v: F^{-1} as three axis DFTs (e^{-2 pi i k/n} / n each)
    std::vector<cd> tw(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
        const cld t = unit_phase_ld(-static_cast<long double>(k) / n);
        tw[k] = cd(static_cast<double>(t.real()), static_cast<double>(t.imag())) / static_cast<double>(n);
    }
    const double inv = probe_inverse_norm(N, [&](const std::vector<cd>& v) {
        std::vector<cd> u(v), t(static_cast<size_t>(N));
        const int64_t strides[3] = {static_cast<int64_t>(n) * n, n, 1};
        for (int ax = 0; ax < 3; ++ax) {
            const int64_t st = strides[ax];
            for (int64_t base = 0; base < N; ++base) {
                if ((base / st) % n != 0) continue;  // one line per base with coordinate 0 on this axis
                for (int a = 0; a < n; ++a) {
                    cd acc{0, 0};
                    for (int r = 0; r < n; ++r) acc += tw[(static_cast<int64_t>(a) * r) % n] * u[base + r * st];
                    t[base + a * st] = acc;
                }
            }
            u.swap(t);
        }
        std::vector<cd> x(static_cast<size_t>(N));
        for (int64_t k = 0; k < N; ++k) {
            const int O = orb.orbit_of[k], pk = orb.pos[k];
            const auto& mem = orb.members[O];
            const int d = static_cast<int>(mem.size());
            cd acc{0, 0};
            for (int i = 0; i < d; ++i) {
                const cld s = ob.Sinv[O][static_cast<size_t>(pk) * d + i];
                acc += cd(static_cast<double>(s.real()), static_cast<double>(s.imag())) * u[mem[i]];
            }
            x[k] = acc;
        }
        return x;
    });
    return norm_a * inv;
}

cld dense_entry(int n, const Params& p, const Index3& node, const Index3& kappa) {
    // (1/24) sum_w e^{2 pi i (w kappa).((p + ijk)/n)}; the integer part of the
    // exponent is reduced exactly before the phase is taken.
    cld acc{0, 0};
    for (const auto& w : s4_group()) {
        const Index3 a = apply(w, kappa);
        const long double frac = (static_cast<long double>(p.r) * a[0] +
                                  static_cast<long double>(p.s) * a[1] +
                                  static_cast<long double>(p.t) * a[2]) / n;
        const int64_t ip = static_cast<int64_t>(a[0]) * node[0] + static_cast<int64_t>(a[1]) * node[1] +
                           static_cast<int64_t>(a[2]) * node[2];
        acc += unit_phase_ld(frac + static_cast<long double>(((ip % n) + n) % n) / n);
    }
    return acc / 24.0L;
}

std::vector<std::array<std::complex<double>, 3>> node_coords(int n, const Params& p) {
    if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "skew_nodes: n must be >= 1");
    const int64_t n3 = cube(n);
    std::vector<std::array<std::complex<double>, 3>> xyz(n3);
    const double two_pi = 2.0 * std::numbers::pi;
    for (int64_t a = 0; a < n3; ++a) {
        const Index3 ijk = unlex(a, n);
        auto wrap = [](double v) {  // TorusPoint::wrapped (chebyshev.cpp:30-39)
            double f = v - std::floor(v);
            if (f >= 1.0 - 1e-15) f = 0.0;
            return f;
        };
        const double th[3] = {wrap((p.r + ijk[0]) / n), wrap((p.s + ijk[1]) / n),
                              wrap((p.t + ijk[2]) / n)};
        const std::complex<double> u{std::cos(two_pi * th[0]), std::sin(two_pi * th[0])};
        const std::complex<double> v{std::cos(two_pi * th[1]), std::sin(two_pi * th[1])};
        const std::complex<double> w{std::cos(two_pi * th[2]), std::sin(two_pi * th[2])};
        const auto ui = 1.0 / u, vi = 1.0 / v, wi = 1.0 / w;  // coords_from_uvw (chebyshev.cpp:76-85)
        xyz[a][0] = 0.25 * (u + ui * v + vi * w + wi);
        xyz[a][1] = (vi + v + u * wi + ui * v * wi + ui * w + u * vi * w) / 6.0;
        xyz[a][2] = 0.25 * (ui + u * vi + v * wi + w);
    }
    return xyz;
}

void check_nodes(int n, const Params& p) {
    if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "skew_nodes: n must be >= 1");
    if (n > 16) return;  // quadratic scan; larger grids skip it (spectral.cpp:27)
    const int64_t n3 = cube(n);
    const auto xyz = node_coords(n, p);
    constexpr double th2 = 1e-9 * 1e-9;
    for (int64_t a = 0; a < n3; ++a)
        for (int64_t b = a + 1; b < n3; ++b) {
            const double d = std::norm(xyz[a][0] - xyz[b][0]) + std::norm(xyz[a][1] - xyz[b][1]) +
                             std::norm(xyz[a][2] - xyz[b][2]);
            if (d < th2) {
                const Index3 ia = unlex(a, n), ib = unlex(b, n);
                throw FcctError(ST_DEGENERATE_NODES,
                                "nodes (" + std::to_string(ia[0]) + "," + std::to_string(ia[1]) +
                                    "," + std::to_string(ia[2]) + ") and (" + std::to_string(ib[0]) +
                                    "," + std::to_string(ib[1]) + "," + std::to_string(ib[2]) +
                                    ") map to the same spectral point for n=" + std::to_string(n));
            }
        }
}

std::vector<uint64_t> radix_permutation(int n) {
    if (n < 2) throw FcctError(ST_INVALID_ARGUMENT, "radix_permutation: n must be >= 2");
    if (n % 2 != 0)
        throw FcctError(ST_ODD_SIZE, "radix_permutation: size " + std::to_string(n) + " is odd");
    const int m = n / 2;
    const int64_t m3 = cube(m);
    std::vector<uint64_t> perm(static_cast<size_t>(cube(n)));
    for (int64_t i = 0; i < cube(n); ++i) {
        const int blk = static_cast<int>(i / m3);
        const Index3 k = unlex(i % m3, m);
        const int ir = blk >> 2, is = (blk >> 1) & 1, it = blk & 1;
        perm[i] = static_cast<uint64_t>(lex(Index3{ir + 2 * k[0], is + 2 * k[1], it + 2 * k[2]}, n));
    }
    return perm;
}

std::vector<int32_t> output_order(int n) {
    if (n == 1) return {0};
    const auto sub = output_order(n / 2);
    const auto perm = radix_permutation(n);
    const int64_t m3 = cube(n / 2);
    std::vector<int32_t> z(cube(n));
    for (int64_t i = 0; i < cube(n); ++i)
        z[i] = static_cast<int32_t>(perm[(i / m3) * m3 + sub[i % m3]]);
    return z;
}

namespace {

struct Triplet {
    int32_t row, col;
    cld val;
};

// Runs body(c0, c1, out) over column ranges on hardware threads and returns
// the rows of the resulting sparse matrix (sorted by column within a row).
template <typename Body>
SparseLD columns_parallel(int64_t n3, Body body) {
    const int nt = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(std::thread::hardware_concurrency(), n3 / 512)));
    std::vector<std::vector<Triplet>> parts(nt);
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w)
        pool.emplace_back([&, w] { body(n3 * w / nt, n3 * (w + 1) / nt, parts[w]); });
    for (auto& t : pool) t.join();
    SparseLD out;
    out.dim = n3;
    out.rowptr.assign(n3 + 1, 0);
    int64_t total = 0;
    for (const auto& p : parts) {
        total += static_cast<int64_t>(p.size());
        for (const auto& t : p) out.rowptr[t.row + 1]++;
    }
    for (int64_t r = 0; r < n3; ++r) out.rowptr[r + 1] += out.rowptr[r];
    out.col.resize(total);
    out.val.resize(total);
    std::vector<int64_t> fill(out.rowptr.begin(), out.rowptr.end() - 1);
    for (const auto& p : parts)  // parts are in column order, so rows stay column-sorted
        for (const auto& t : p) {
            const int64_t dst = fill[t.row]++;
            out.col[dst] = t.col;
            out.val[dst] = t.val;
        }
    return out;
}

std::vector<cld> roots_of_unity(int n) {  // e^{2 pi i j / n}
    std::vector<cld> r(n);
    for (int j = 0; j < n; ++j) r[j] = unit_phase_ld(static_cast<long double>(j) / n);
    return r;
}

// B = (K^{-1} (x) I) blockdiag(S_m(child)^{-1}) Phi S_n, column by column.
SparseLD derive_B(int n, const OrbitBlocks& Sn, const std::array<OrbitBlocks, 8>& Sm,
                  const std::array<cld, 64>& Kinv) {
    const int m = n / 2;
    const int64_t n3 = cube(n), m3 = cube(m);
    const auto& on = *Sn.orb;
    const auto& om = orbits(m);
    const auto root = roots_of_unity(n);
    return columns_parallel(n3, [&](int64_t c0, int64_t c1, std::vector<Triplet>& out) {
        std::vector<cld> v, u;
        for (int64_t c = c0; c < c1; ++c) {
            const int O = on.orbit_of[c], j = on.pos[c];
            const auto& mem = on.members[O];
            const int d = static_cast<int>(mem.size());
            const Index3 cm = unlex(c, n);
            const int64_t hrep = lex(Index3{cm[0] % m, cm[1] % m, cm[2] % m}, m);
            const int Op = om.orbit_of[hrep];
            const auto& memp = om.members[Op];
            const int dp = static_cast<int>(memp.size());
            v.assign(static_cast<size_t>(8) * dp, cld{0, 0});
            for (int i = 0; i < d; ++i) {
                const cld val = Sn.S[O][static_cast<size_t>(i) * d + j];
                if (val == cld{0, 0}) continue;
                const Index3 a = unlex(mem[i], n);
                const int ip = om.pos[lex(Index3{a[0] % m, a[1] % m, a[2] % m}, m)];
                for (int blk = 0; blk < 8; ++blk) {
                    const int ir = blk >> 2, is = (blk >> 1) & 1, it = blk & 1;
                    v[static_cast<size_t>(blk) * dp + ip] += root[(a[0] * ir + a[1] * is + a[2] * it) % n] * val;
                }
            }
            u.assign(static_cast<size_t>(8) * dp, cld{0, 0});
            for (int blk = 0; blk < 8; ++blk) {
                const auto& Si = Sm[blk].Sinv[Op];
                for (int h = 0; h < dp; ++h) {
                    cld acc{0, 0};
                    for (int i = 0; i < dp; ++i)
                        acc += Si[static_cast<size_t>(h) * dp + i] * v[static_cast<size_t>(blk) * dp + i];
                    u[static_cast<size_t>(blk) * dp + h] = acc;
                }
            }
            for (int g = 0; g < 8; ++g)
                for (int h = 0; h < dp; ++h) {
                    cld acc{0, 0};
                    for (int blk = 0; blk < 8; ++blk)
                        acc += Kinv[g * 8 + blk] * u[static_cast<size_t>(blk) * dp + h];
                    if (std::abs(acc) >= kPrune)
                        out.push_back({static_cast<int32_t>(static_cast<int64_t>(g) * m3 + memp[h]),
                                       static_cast<int32_t>(c), snap(acc)});
                }
        }
    });
}

// B^{-1} = S_n^{-1} Phi^{-1} blockdiag(S_m(child)) (K (x) I), column by column.
SparseLD derive_Binv(int n, const OrbitBlocks& Sn, const std::array<OrbitBlocks, 8>& Sm,
                     const std::array<cld, 64>& K) {
    const int m = n / 2;
    const int64_t n3 = cube(n), m3 = cube(m);
    const auto& on = *Sn.orb;
    const auto& om = orbits(m);
    const auto root = roots_of_unity(n);
    return columns_parallel(n3, [&](int64_t c0, int64_t c1, std::vector<Triplet>& out) {
        std::vector<cld> x(n3, cld{0, 0});  // dense scratch + touched list
        std::vector<char> hit(n3, 0);
        std::vector<int32_t> touched;
        std::vector<cld> w;
        for (int64_t col = c0; col < c1; ++col) {
            const int g = static_cast<int>(col / m3);
            const int64_t h = col % m3;
            const int Op = om.orbit_of[h], jh = om.pos[h];
            const auto& memp = om.members[Op];
            const int dp = static_cast<int>(memp.size());
            w.assign(static_cast<size_t>(8) * dp, cld{0, 0});
            for (int blk = 0; blk < 8; ++blk) {
                const auto& S = Sm[blk].S[Op];
                for (int i = 0; i < dp; ++i)
                    w[static_cast<size_t>(blk) * dp + i] = S[static_cast<size_t>(i) * dp + jh] * K[blk * 8 + g];
            }
            touched.clear();
            for (int i = 0; i < dp; ++i) {
                const Index3 ap = unlex(memp[i], m);
                for (int delta = 0; delta < 8; ++delta) {
                    const int dr = delta >> 2, ds = (delta >> 1) & 1, dt = delta & 1;
                    cld val{0, 0};
                    for (int blk = 0; blk < 8; ++blk) {
                        const int ir = blk >> 2, is = (blk >> 1) & 1, it = blk & 1;
                        const long double sign = ((dr * ir + ds * is + dt * it) & 1) ? -1.0L : 1.0L;
                        const cld tw = std::conj(root[(ap[0] * ir + ap[1] * is + ap[2] * it) % n]);
                        val += sign * tw * w[static_cast<size_t>(blk) * dp + i];
                    }
                    val /= 8.0L;
                    if (val == cld{0, 0}) continue;
                    const int64_t a = lex(Index3{ap[0] + m * dr, ap[1] + m * ds, ap[2] + m * dt}, n);
                    const int O = on.orbit_of[a], pa = on.pos[a];
                    const auto& mem = on.members[O];
                    const int d = static_cast<int>(mem.size());
                    const auto& Si = Sn.Sinv[O];
                    for (int k = 0; k < d; ++k) {
                        const int32_t r = mem[k];
                        if (!hit[r]) {
                            hit[r] = 1;
                            touched.push_back(r);
                        }
                        x[r] += Si[static_cast<size_t>(k) * d + pa] * val;
                    }
                }
            }
            for (int32_t r : touched) {
                if (std::abs(x[r]) >= kPrune) out.push_back({r, static_cast<int32_t>(col), snap(x[r])});
                x[r] = cld{0, 0};
                hit[r] = 0;
            }
        }
    });
}

std::shared_ptr<const PlanNode> make_node(int n, const Params& p, bool check) {
    if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "build_plan: n must be >= 1");
    if (check) check_nodes(n, p);  // dense_transform runs the check (transform.cpp:132)
    auto node = std::make_shared<PlanNode>();
    node->n = n;
    node->p = p;
    const int64_t n3 = cube(n);
    if (n == 1 || n % 2 != 0) {  // assemble_direct (transform.cpp:329-345)
        node->radix = false;
        OrbitBlocks ob = orbit_blocks(n, p);
        node->D.resize(static_cast<size_t>(n3 * n3));
        for (int64_t r = 0; r < n3; ++r)
            for (int64_t c = 0; c < n3; ++c) node->D[r * n3 + c] = dense_entry(n, p, unlex(r, n), unlex(c, n));
        // D^{-1} = S^{-1} F^{-1}: D^{-1}[kappa, node] = (1/N) sum_{a in O(kappa)} Sinv[kappa, a] e^{-2 pi i a.node/n}
        node->Dinv.assign(static_cast<size_t>(n3 * n3), cld{0, 0});
        const auto& orb = *ob.orb;
        for (int64_t k = 0; k < n3; ++k) {
            const int O = orb.orbit_of[k], pk = orb.pos[k];
            const auto& mem = orb.members[O];
            const int d = static_cast<int>(mem.size());
            for (int64_t r = 0; r < n3; ++r) {
                const Index3 nd = unlex(r, n);
                cld acc{0, 0};
                for (int i = 0; i < d; ++i) {
                    const Index3 a = unlex(mem[i], n);
                    const int64_t ip = static_cast<int64_t>(a[0]) * nd[0] + static_cast<int64_t>(a[1]) * nd[1] +
                                       static_cast<int64_t>(a[2]) * nd[2];
                    acc += ob.Sinv[O][static_cast<size_t>(pk) * d + i] *
                           unit_phase_ld(-static_cast<long double>(ip % n) / n);
                }
                node->Dinv[k * n3 + r] = acc / static_cast<long double>(n3);
            }
        }
        // assemble_direct gates on condition_with_lu(D) (transform.cpp:339-344)
        node->condition = reference_condition_dense(node->D, node->Dinv, n3);
        require_condition(node->condition, "dense transform (n=" + std::to_string(n) + ")");
        return node;
    }
    const int m = n / 2;
    std::array<std::shared_ptr<const PlanNode>, 8> children;
    if (m >= 8) {  // independent subtrees: build them concurrently
        std::array<std::future<std::shared_ptr<const PlanNode>>, 8> fut;
        for (int blk = 0; blk < 8; ++blk)
            fut[blk] = std::async(std::launch::async, [&, blk] {
                return make_node(m, p.child(blk >> 2, (blk >> 1) & 1, blk & 1), check);
            });
        for (int blk = 0; blk < 8; ++blk) children[blk] = fut[blk].get();
    } else {
        for (int blk = 0; blk < 8; ++blk)
            children[blk] = make_node(m, p.child(blk >> 2, (blk >> 1) & 1, blk & 1), check);
    }
    return build_radix_node(n, p, children);
}

}  // namespace

std::vector<cld> dense_inverse(const std::vector<cld>& a, int64_t dim, double* cond) {
    std::vector<cld> inv;
    const double c = invert_ld(a, static_cast<int>(dim), inv);
    if (cond) *cond = c;
    return inv;
}

std::shared_ptr<const PlanNode> build_radix_node(int n, const Params& p,
                                                 const std::array<std::shared_ptr<const PlanNode>, 8>& children) {
    if (n < 2 || n % 2 != 0) throw FcctError(ST_ODD_SIZE, "radix node needs an even size");
    auto node = std::make_shared<PlanNode>();
    node->n = n;
    node->p = p;
    node->radix = true;
    node->children = children;
    const int m = n / 2;
    // kernel = dense_transform(2, p).matrix (transform.cpp:397): rows = nodes blk, cols = g
    std::vector<cld> K(64), Kinv;
    for (int blk = 0; blk < 8; ++blk)
        for (int g = 0; g < 8; ++g)
            K[blk * 8 + g] = dense_entry(2, p, unlex(blk, 2), unlex(g, 2));
    invert_ld(K, 8, Kinv);
    const double kc = reference_condition_dense(K, Kinv, 8);  // condition_estimate_1norm(K), transform.cpp:224-227
    require_condition(kc, "radix kernel");
    for (int i = 0; i < 64; ++i) {
        node->K[i] = snap(K[i]);
        node->Kinv[i] = snap(Kinv[i]);
    }
    // derive_basis gates every child's dense transform on condition_with_lu
    // (transform.cpp:210-221); the parent D_n itself is not gated there, only its
    // basis factor's invertibility (assemble_radix, transform.cpp:376-378), which
    // fails exactly when an orbit block of S_n is singular.
    std::array<double, 8> cc{};
    if (m >= 16) {  // the column norms run on the GPU hook or on all host threads
        for (int blk = 0; blk < 8; ++blk) cc[blk] = reference_condition(m, children[blk]->p);
    } else {
        std::array<std::future<double>, 8> fut;
        for (int blk = 0; blk < 8; ++blk)
            fut[blk] = std::async(std::launch::async, [&, blk] { return reference_condition(m, children[blk]->p); });
        for (int blk = 0; blk < 8; ++blk) cc[blk] = fut[blk].get();
    }
    for (int blk = 0; blk < 8; ++blk) require_condition(cc[blk], "child block " + std::to_string(blk));
    const OrbitBlocks Sn = orbit_blocks(n, p);
    if (!std::isfinite(Sn.worst_condition))
        throw FcctError(ST_ILL_CONDITIONED, "basis-change factor is not invertible");
    std::array<OrbitBlocks, 8> Sm;
    for (int blk = 0; blk < 8; ++blk) Sm[blk] = orbit_blocks(m, children[blk]->p);
    node->condition = std::max(kc, *std::max_element(cc.begin(), cc.end()));
    node->B = derive_B(n, Sn, Sm, node->Kinv);
    node->Binv = derive_Binv(n, Sn, Sm, node->K);
    return node;
}

namespace {
}  // namespace

std::shared_ptr<const PlanNode> build_tree(int n, const Params& p) {
    if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "build_plan: n must be >= 1");
    // Degeneracy is a property of the root grid; children grids are subsets
    // of it (spectral tests "half size grids nest"), so one scan suffices.
    check_nodes(n, p);
    return make_node(n, p, false);
}

int64_t tree_nnz(const PlanNode& node, bool inverse, bool with_b2) {
    if (!node.radix) return 0;
    int64_t s = (node.n == 2 && !with_b2) ? 0 : (inverse ? node.Binv.nnz() : node.B.nnz());
    for (const auto& c : node.children) s += tree_nnz(*c, inverse, with_b2);
    return s;
}

int tree_levels(int n) {
    int l = 0;
    while (n > 1 && n % 2 == 0) { n /= 2; ++l; }
    return l;
}

double algorithmic_flops(const PlanNode& root, bool inverse) {
    const double N = static_cast<double>(cube(root.n));
    if (!root.radix) return 8.0 * N * N;
    return 8.0 * (static_cast<double>(tree_nnz(root, inverse, false)) + 8.0 * N * tree_levels(root.n));
}

bool basis_is_identity(const SparseLD& B) {
    if (B.nnz() != B.dim) return false;
    for (int64_t r = 0; r < B.dim; ++r)
        if (B.rowptr[r + 1] - B.rowptr[r] != 1 || B.col[B.rowptr[r]] != r ||
            std::abs(B.val[B.rowptr[r]] - cld{1, 0}) > 1e-15L)  // derivation rounding only
            return false;
    return true;
}

}  // namespace fcct
