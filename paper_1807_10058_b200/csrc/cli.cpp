// fcct — command-line front end of the B200 build, flag- and exit-code
// compatible with the reference CLI (tools/fcct.cpp:594-710): zeros,
// transform, verify, bench, plan, sword, geometry; exit 0 success, 1 usage,
// 2 math error, 3 io error.
//
// It is a plain client of the C ABI (include/fcct_gpu.h), linked against
// libfcct_b200.so the way a reference maintainer would link the adapter
// (INTEGRATION.md): transforms run on the GPU through the *_host entry points,
// with z_transform / grid_from_signal fused into the device pipeline
// (fcct_forward_real_host / fcct_inverse_real_host).
#include <algorithm>
#include <array>
#include <charconv>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <dirent.h>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <numbers>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/fcct_gpu.h"

namespace {

using Complex = std::complex<double>;
using Index3 = std::array<int, 3>;
using Clock = std::chrono::steady_clock;

// ---------------------------------------------------------------------------
// errors: status -> exception -> exit code (errors.hpp:9-63, fcct.cpp:702-707)
// ---------------------------------------------------------------------------
struct CliError : std::runtime_error {
    bool io;
    CliError(const std::string& m, bool is_io) : std::runtime_error(m), io(is_io) {}
};
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void check(fcct_status st) {
    if (st == FCCT_OK) return;
    const bool io = st == FCCT_IO || st == FCCT_MALFORMED || st == FCCT_SIZE_MISMATCH_IO;
    throw CliError(fcct_last_error(), io);
}

std::string g17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

int64_t cube(int n) { return static_cast<int64_t>(n) * n * n; }

void write_text_output(const std::string& path, const std::string& content) {  // fcct.cpp:44-54
    if (path.empty() || path == "-") {
        std::cout << content;
        return;
    }
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw CliError("cannot write " + path, true);
    out << content;
    if (!out) throw CliError("failed while writing " + path, true);
}

struct Params {
    double r = 0.125, s = 0.0, t = 0.375;
    bool operator==(const Params& o) const { return r == o.r && s == o.s && t == o.t; }
};

Params parse_params(const std::string& text) {
    Params p;
    check(fcct_parse_params(text.c_str(), &p.r, &p.s, &p.t));
    return p;
}

std::string encode(const Params& p) {
    char buf[256];
    check(fcct_encode_params(p.r, p.s, p.t, buf, sizeof(buf)));
    return buf;
}

const std::string kCanonical = "1/8,0,3/8";

// One plan handle, released on scope exit.
struct Plan {
    fcct_plan h = nullptr;
    Plan() = default;
    Plan(const Plan&) = delete;
    ~Plan() {
        if (h) fcct_plan_destroy(h);
    }
};
struct Store {
    fcct_store h = nullptr;
    ~Store() {
        if (h) fcct_store_close(h);
    }
};

void open_store(Store& s, const std::string& dir) {
    if (!dir.empty()) check(fcct_store_open(dir.c_str(), &s.h));
}

void make_plan(Plan& pl, int n, const Params& p, bool naive, fcct_store store) {
    if (naive)
        check(fcct_plan_create(n, p.r, p.s, p.t, FCCT_DIRECT, FCCT_F64, 0, &pl.h));
    else if (store)
        check(fcct_plan_create_from_store(store, n, p.r, p.s, p.t, FCCT_F64, 0, &pl.h));
    else
        check(fcct_plan_create(n, p.r, p.s, p.t, FCCT_FAST, FCCT_F64, 0, &pl.h));
}

// ---------------------------------------------------------------------------
// a small CLI11-compatible parser: subcommand, --opt value / --opt=value,
// flags, required options, range / membership checks -> exit 1 on misuse.
// ---------------------------------------------------------------------------
struct Opt {
    std::string name, help;
    bool flag = false, required = false, seen = false;
    std::string value;
    std::function<void(const std::string&)> validate;
};

struct Sub {
    std::string name, help;
    std::vector<Opt> opts;
    Opt& add(const std::string& n, const std::string& h, std::string def = "", bool req = false) {
        opts.push_back(Opt{n, h, false, req, false, std::move(def), nullptr});
        return opts.back();
    }
    Opt& flag(const std::string& n, const std::string& h) {
        opts.push_back(Opt{n, h, true, false, false, "", nullptr});
        return opts.back();
    }
    Opt* find(const std::string& n) {
        for (auto& o : opts)
            if (o.name == n) return &o;
        return nullptr;
    }
    const std::string& get(const std::string& n) { return find(n)->value; }
    bool has(const std::string& n) { return find(n)->seen; }
};

int to_int(const std::string& opt, const std::string& v) {
    int x = 0;
    const auto r = std::from_chars(v.data(), v.data() + v.size(), x);
    if (r.ec != std::errc() || r.ptr != v.data() + v.size()) throw UsageError(opt + ": Value " + v + " could not be converted");
    return x;
}
double to_double(const std::string& opt, const std::string& v) {
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end != '\0') throw UsageError(opt + ": Value " + v + " could not be converted");
    return x;
}
std::function<void(const std::string&)> range(const std::string& opt, int lo, int hi) {
    return [opt, lo, hi](const std::string& v) {
        const int x = to_int(opt, v);
        if (x < lo || x > hi)
            throw UsageError(opt + ": Value " + v + " not in range [" + std::to_string(lo) + " - " + std::to_string(hi) + "]");
    };
}
std::function<void(const std::string&)> member(const std::string& opt, std::vector<std::string> allowed) {
    return [opt, allowed](const std::string& v) {
        if (std::find(allowed.begin(), allowed.end(), v) == allowed.end())
            throw UsageError(opt + ": " + v + " not in {" + [&] {
                std::string s;
                for (const auto& a : allowed) s += (s.empty() ? "" : ",") + a;
                return s;
            }() + "}");
    };
}

void print_help(const std::vector<Sub>& subs, const Sub* sub) {
    if (!sub) {
        std::cout << "Discrete Chebyshev transforms on the FCC lattice (B200 build)\n"
                  << "Usage: fcct [OPTIONS] SUBCOMMAND\n\nOptions:\n  -h,--help   Print this help message and exit\n\n"
                  << "Subcommands:\n";
        for (const auto& s : subs) std::cout << "  " << s.name << std::string(12 - std::min<size_t>(11, s.name.size()), ' ') << s.help << "\n";
        return;
    }
    std::cout << sub->help << "\nUsage: fcct " << sub->name << " [OPTIONS]\n\nOptions:\n  -h,--help   Print this help message and exit\n";
    for (const auto& o : sub->opts)
        std::cout << "  " << o.name << (o.flag ? "" : " VALUE") << "   " << o.help << (o.required ? " REQUIRED" : "") << "\n";
}

// ---------------------------------------------------------------------------
// commands
// ---------------------------------------------------------------------------
int cmd_zeros(int n, const std::string& params_text, const std::string& out) {  // fcct.cpp:59-69
    const Params p = parse_params(params_text);
    std::string path = out.empty() ? "-" : out;
    if (path == "-") std::cout.flush();
    check(fcct_export_nodes_csv(n, p.r, p.s, p.t, path.c_str()));
    std::cerr << cube(n) << " nodes (n=" << n << ", params=" << encode(p) << ")\n";
    return 0;
}

struct TransformArgs {
    std::string input, output, method = "fast", direction = "forward", params_text = kCanonical, cache_dir;
    int n_override = 0, threads = 1;
};

int cmd_transform(const TransformArgs& a) {  // fcct.cpp:80-134
    const Params params = parse_params(a.params_text);
    Store store;
    open_store(store, a.cache_dir);
    if (a.direction == "forward") {
        int n = 0;
        check(fcct_grid_load(a.input.c_str(), &n, nullptr, 0, nullptr, 0));
        std::vector<double> values(static_cast<size_t>(cube(n)));
        check(fcct_grid_load(a.input.c_str(), &n, values.data(), cube(n), nullptr, 0));
        if (a.n_override != 0 && a.n_override != n) {
            std::cerr << "error: --n " << a.n_override << " does not match the input grid (n=" << n << ")\n";
            return 1;
        }
        Plan plan;
        make_plan(plan, n, params, a.method == "naive", store.h);
        std::vector<Complex> spec(static_cast<size_t>(cube(n)));
        // z_transform fused into the device tile load
        check(fcct_forward_real_host(plan.h, values.data(), spec.data(), 1, nullptr));
        std::string path = a.output.empty() ? "-" : a.output;
        if (path == "-") std::cout.flush();
        check(fcct_export_spectrum(n, params.r, params.s, params.t, spec.data(), path.c_str()));
        std::cerr << "forward " << a.method << " n=" << n << " done\n";
        return 0;
    }
    int n = 0;
    Params sp;
    check(fcct_load_spectrum_csv(a.input.c_str(), &n, &sp.r, &sp.s, &sp.t, nullptr, 0));
    std::vector<Complex> spec(static_cast<size_t>(cube(n)));
    check(fcct_load_spectrum_csv(a.input.c_str(), &n, &sp.r, &sp.s, &sp.t, spec.data(), cube(n)));
    if (a.n_override != 0 && a.n_override != n) {
        std::cerr << "error: --n " << a.n_override << " does not match the spectrum file (n=" << n << ")\n";
        return 1;
    }
    if (!(sp == params) && a.params_text != kCanonical) {
        std::cerr << "error: --params disagrees with the spectrum header (" << encode(sp) << ")\n";
        return 1;
    }
    Plan plan;
    make_plan(plan, n, sp, a.method == "naive", store.h);
    std::vector<double> grid(static_cast<size_t>(cube(n)));
    // grid_from_signal fused into the device tile store
    check(fcct_inverse_real_host(plan.h, spec.data(), grid.data(), 1, nullptr));
    check(fcct_grid_save(a.output.c_str(), n, grid.data(), "{}"));
    std::cerr << "inverse " << a.method << " n=" << n << " done\n";
    return 0;
}

// --- verify (fcct.cpp:138-468) ---------------------------------------------
// Host restatement of the algebra the checks exercise (weyl_s4.cpp,
// chebyshev.cpp, spectral.cpp); the transform checks run on the GPU.
struct G {
    std::array<int, 9> m;
    G operator*(const G& b) const {
        G o{};
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                int acc = 0;
                for (int k = 0; k < 3; ++k) acc += m[i * 3 + k] * b.m[k * 3 + j];
                o.m[i * 3 + j] = acc;
            }
        return o;
    }
    bool operator==(const G& o) const { return m == o.m; }
    bool operator<(const G& o) const { return m < o.m; }
    int det() const {
        return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) + m[2] * (m[3] * m[7] - m[4] * m[6]);
    }
    Index3 apply(const Index3& k) const {
        return {m[0] * k[0] + m[1] * k[1] + m[2] * k[2], m[3] * k[0] + m[4] * k[1] + m[5] * k[2],
                m[6] * k[0] + m[7] * k[1] + m[8] * k[2]};
    }
    std::array<double, 3> apply_t(const std::array<double, 3>& t) const {
        std::array<double, 3> o{};
        for (int i = 0; i < 3; ++i) o[i] = m[i] * t[0] + m[3 + i] * t[1] + m[6 + i] * t[2];
        return o;
    }
};
const G kId{{1, 0, 0, 0, 1, 0, 0, 0, 1}};
std::array<G, 3> generators() {
    return {G{{-1, 0, 0, 1, 1, 0, 0, 0, 1}}, G{{1, 1, 0, 0, -1, 0, 0, 1, 1}}, G{{1, 0, 0, 0, 1, 1, 0, 0, -1}}};
}
std::vector<G> group() {  // BFS closure, identity first
    std::vector<G> out;
    std::set<G> seen{kId};
    std::deque<G> q{kId};
    while (!q.empty()) {
        const G g = q.front();
        q.pop_front();
        out.push_back(g);
        for (const auto& s : generators()) {
            const G nx = g * s;
            if (seen.insert(nx).second) q.push_back(nx);
        }
    }
    return out;
}
const std::vector<G>& W() {
    static const std::vector<G> g = group();
    return g;
}
Index3 canonical(const Index3& k) {
    Index3 best = k;
    for (const auto& w : W()) best = std::max(best, w.apply(k));
    return best;
}
constexpr double kTwoPi = 2.0 * std::numbers::pi;
Complex unit(double t) { return {std::cos(kTwoPi * t), std::sin(kTwoPi * t)}; }
std::array<double, 3> wrapped(double a, double b, double c) {
    std::array<double, 3> o{a, b, c};
    for (auto& f : o) {
        f = f - std::floor(f);
        if (f >= 1.0 - 1e-15) f = 0.0;
    }
    return o;
}
struct UVW {
    Complex u{1.0}, v{1.0}, w{1.0};
};
UVW from_torus(const std::array<double, 3>& t) { return {unit(t[0]), unit(t[1]), unit(t[2])}; }
Complex ipow(Complex b, int e) {
    if (e < 0) {
        b = 1.0 / b;
        e = -e;
    }
    Complex acc{1.0, 0.0};
    while (e > 0) {
        if (e & 1) acc *= b;
        b *= b;
        e >>= 1;
    }
    return acc;
}
Complex sym_exp(const Index3& k, const std::array<double, 3>& th) {
    Complex acc{0.0, 0.0};
    for (const auto& w : W()) {
        const Index3 wk = w.apply(k);
        const double ph = kTwoPi * (wk[0] * th[0] + wk[1] * th[1] + wk[2] * th[2]);
        acc += Complex{std::cos(ph), std::sin(ph)};
    }
    return acc / 24.0;
}
Complex cheb(const Index3& k, const UVW& p) {
    Complex acc{0.0, 0.0};
    for (const auto& w : W()) {
        const Index3 wk = w.apply(k);
        acc += ipow(p.u, wk[0]) * ipow(p.v, wk[1]) * ipow(p.w, wk[2]);
    }
    return acc / 24.0;
}
std::array<Complex, 3> coords(const UVW& p) {
    const Complex u = p.u, v = p.v, w = p.w, ui = 1.0 / u, vi = 1.0 / v, wi = 1.0 / w;
    return {0.25 * (u + ui * v + vi * w + wi), (vi + v + u * wi + ui * v * wi + ui * w + u * vi * w) / 6.0,
            0.25 * (ui + u * vi + v * wi + w)};
}
std::vector<UVW> skew_uvw(int n, const Params& p) {
    std::vector<UVW> o;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k) o.push_back(from_torus(wrapped((p.r + i) / n, (p.s + j) / n, (p.t + k) / n)));
    return o;
}
std::vector<UVW> common_zeros(int n) {
    std::vector<UVW> o;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k)
                o.push_back({unit(double(1 + 8 * i) / (8.0 * n)), unit(double(j) / n), unit(double(3 + 8 * k) / (8.0 * n))});
    return o;
}

struct Check {
    std::string name;
    bool passed;
    double residual, tolerance;
    std::string detail;
};

std::string json_num(double v) {  // nlohmann dump layout for doubles
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char sci[64];
    const auto r = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
    std::string t(sci, r.ptr), sign;
    if (t[0] == '-') {
        sign = "-";
        t.erase(0, 1);
    }
    const size_t ep = t.find('e');
    const int e10 = std::atoi(t.c_str() + ep + 1);
    std::string d;
    for (size_t k = 0; k < ep; ++k)
        if (t[k] != '.') d += t[k];
    const int len = static_cast<int>(d.size()), nx = e10 + 1;
    std::string o;
    if (len <= nx && nx <= 15) o = d + std::string(static_cast<size_t>(nx - len), '0') + ".0";
    else if (0 < nx && nx <= 15) o = d.substr(0, static_cast<size_t>(nx)) + "." + d.substr(static_cast<size_t>(nx));
    else if (-4 < nx && nx <= 0) o = "0." + std::string(static_cast<size_t>(-nx), '0') + d;
    else {
        o = d.substr(0, 1) + (len > 1 ? "." + d.substr(1) : "");
        char eb[16];
        std::snprintf(eb, sizeof(eb), "e%c%02d", nx - 1 < 0 ? '-' : '+', std::abs(nx - 1));
        o += eb;
    }
    return sign + o;
}
std::string json_str(const std::string& s) {
    std::string o = "\"";
    for (const unsigned char c : s) {
        if (c == '"') o += "\\\"";
        else if (c == '\\') o += "\\\\";
        else if (c == '\n') o += "\\n";
        else if (c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof(b), "\\u%04x", c);
            o += b;
        } else o += static_cast<char>(c);
    }
    return o + "\"";
}

std::vector<Check> run_checks(int n_max, double tol_override, bool perturb) {
    std::vector<Check> out;
    auto tol = [&](double f) { return tol_override > 0.0 ? tol_override : f; };
    auto add = [&](const std::string& name, double res, double t, std::string detail = {}) {
        out.push_back(Check{name, res <= t, res, t, std::move(detail)});
    };
    auto random_points = [](int count, unsigned seed) {
        std::mt19937 rng(seed);
        std::uniform_real_distribution<double> uni(0.0, 1.0);
        std::vector<std::array<double, 3>> pts;
        for (int i = 0; i < count; ++i) {
            const double a = uni(rng), b = uni(rng), c = uni(rng);
            pts.push_back(wrapped(a, b, c));
        }
        return pts;
    };
    const auto& g = W();
    {  // group_structure
        double bad = g.size() != 24 ? 1.0 : 0.0;
        const auto gens = generators();
        auto pow_id = [](const G& e, int p) {
            G acc = kId;
            for (int i = 0; i < p; ++i) acc = acc * e;
            return acc == kId;
        };
        for (const auto& s : gens)
            if (!pow_id(s, 2)) bad = 1.0;
        if (!pow_id(gens[0] * gens[1], 3) || !pow_id(gens[0] * gens[2], 2) || !pow_id(gens[1] * gens[2], 3)) bad = 1.0;
        for (const auto& a : g) {
            if (std::abs(a.det()) != 1) bad = 1.0;
            for (const auto& b : g)
                if (std::find(g.begin(), g.end(), a * b) == g.end()) bad = 1.0;
        }
        add("group_structure", bad, 0.5, "order, involutions, braid relations, closure, determinants");
    }
    {  // evaluation_routes_agree
        double worst = 0.0;
        const auto pts = random_points(40, 11);
        for (const Index3& k : {Index3{1, 0, 0}, Index3{0, 1, 0}, Index3{2, 1, 0}, Index3{1, 1, 1}, Index3{3, -1, 2}})
            for (const auto& t : pts) worst = std::max(worst, std::abs(sym_exp(k, t) - cheb(k, from_torus(t))));
        add("evaluation_routes_agree", worst, tol(1e-12));
    }
    {  // coordinate_identities
        double worst = 0.0;
        for (const auto& t : random_points(40, 12)) {
            const UVW p = from_torus(t);
            const auto s = coords(p);
            worst = std::max(worst, std::abs(cheb({0, 0, 0}, p) - 1.0));
            worst = std::max(worst, std::abs(cheb({1, 0, 0}, p) - s[0]));
            worst = std::max(worst, std::abs(cheb({0, 1, 0}, p) - s[1]));
            worst = std::max(worst, std::abs(cheb({0, 0, 1}, p) - s[2]));
        }
        add("coordinate_identities", worst, tol(1e-12));
    }
    {  // group_invariance
        double worst = 0.0;
        const auto pts = random_points(10, 13);
        for (const Index3& k : {Index3{1, 0, 0}, Index3{2, 1, 0}, Index3{1, -1, 2}})
            for (const auto& w : g)
                for (const auto& t : pts) {
                    const Complex base = sym_exp(k, t);
                    worst = std::max(worst, std::abs(sym_exp(w.apply(k), t) - base));
                    const auto wt = w.apply_t(t);
                    worst = std::max(worst, std::abs(sym_exp(k, wrapped(wt[0], wt[1], wt[2])) - base));
                }
        add("group_invariance", worst, tol(1e-12));
    }
    {  // product_linearization: T_k T_l = (1/24) sum_w T_{k + w l}
        double worst = 0.0;
        std::mt19937 rng(14);
        std::uniform_int_distribution<int> idx(-2, 2);
        const auto pts = random_points(15, 15);
        for (int rep = 0; rep < 12; ++rep) {
            const Index3 k{idx(rng), idx(rng), idx(rng)};
            const Index3 l{idx(rng), idx(rng), idx(rng)};
            std::map<Index3, int> counts;
            for (const auto& w : g) {
                const Index3 wl = w.apply(l);
                ++counts[canonical({k[0] + wl[0], k[1] + wl[1], k[2] + wl[2]})];
            }
            int msum = 0;
            for (const auto& [i, m] : counts) msum += m;
            if (msum != 24) {
                worst = 1.0;
                break;
            }
            for (const auto& t : pts) {
                const UVW p = from_torus(t);
                const Complex prod = cheb(k, p) * cheb(l, p);
                Complex sum{0.0, 0.0};
                for (const auto& [i, m] : counts) sum += (static_cast<double>(m) / 24.0) * cheb(i, p);
                worst = std::max(worst, std::abs(prod - sum));
            }
        }
        add("product_linearization", worst, tol(1e-11));
    }
    {  // semigroup_composition (compose_scaled, chebyshev.cpp:114-146)
        double worst = 0.0;
        const auto pts = random_points(10, 16);
        for (int axis = 1; axis <= 3; ++axis)
            for (int k = 1; k <= 3; ++k)
                for (int l = 1; l <= 3; ++l) {
                    Index3 e{0, 0, 0};
                    e[axis - 1] = 1;
                    const Index3 outer{k * e[0], k * e[1], k * e[2]}, comp{k * l * e[0], k * l * e[1], k * l * e[2]};
                    for (const auto& t : pts) {
                        const UVW p = from_torus(t);
                        const UVW pl{ipow(p.u, l), ipow(p.v, l), ipow(p.w, l)};
                        worst = std::max(worst, std::abs(cheb(comp, p) - cheb(outer, pl)));
                        const auto sc = coords(pl);
                        worst = std::max(worst, std::abs(sc[0] - cheb({l, 0, 0}, p)));
                        worst = std::max(worst, std::abs(sc[1] - cheb({0, l, 0}, p)));
                        worst = std::max(worst, std::abs(sc[2] - cheb({0, 0, l}, p)));
                    }
                }
        add("semigroup_composition", worst, tol(1e-11));
    }
    const Params canon;
    {  // node_generator_residuals (sigma / tau / rho, spectral.cpp:119-134)
        double worst = 0.0;
        const Params& p = canon;
        const Complex sx = 0.25 * (unit(p.r) + unit(p.s - p.r) + unit(p.t - p.s) + unit(-p.t));
        const Complex sy = (unit(-p.s) + unit(p.s) + unit(p.r - p.t) + unit(-p.r + p.s - p.t) + unit(-p.r + p.t) +
                            unit(p.r - p.s + p.t)) / 6.0;
        const Complex sz = 0.25 * (unit(-p.r) + unit(p.r - p.s) + unit(p.s - p.t) + unit(p.t));
        for (int n = 1; n <= n_max; ++n) {
            // the library's node export runs skew_nodes' count and degeneracy checks
            check(fcct_export_nodes_csv(n, p.r, p.s, p.t, "/dev/null"));
            for (const auto& node : skew_uvw(n, p)) {
                worst = std::max(worst, std::abs(cheb({n, 0, 0}, node) - sx));
                worst = std::max(worst, std::abs(cheb({0, n, 0}, node) - sy));
                worst = std::max(worst, std::abs(cheb({0, 0, n}, node) - sz));
            }
        }
        add("node_generator_residuals", worst, tol(1e-10));
    }
    {  // node_construction_consistency
        double worst = 0.0;
        for (int n = 1; n <= n_max; ++n) {
            const auto a = common_zeros(n), b = skew_uvw(n, canon);
            for (size_t i = 0; i < a.size(); ++i)
                worst = std::max({worst, std::abs(a[i].u - b[i].u), std::abs(a[i].v - b[i].v), std::abs(a[i].w - b[i].w)});
        }
        add("node_construction_consistency", worst, tol(1e-12));
    }
    {  // grid_nesting
        double worst = 0.0;
        for (int n = 2; n <= n_max; n += 2) {
            const int m = n / 2;
            const auto parent = skew_uvw(n, canon);
            for (int ir = 0; ir < 2; ++ir)
                for (int is = 0; is < 2; ++is)
                    for (int it = 0; it < 2; ++it) {
                        const Params cp{(canon.r + ir) / 2.0, (canon.s + is) / 2.0, (canon.t + it) / 2.0};
                        const auto child = skew_uvw(m, cp);
                        for (int a = 0; a < static_cast<int>(child.size()); ++a) {
                            const int i = a / (m * m), j = (a / m) % m, k = a % m;
                            const auto& pn = parent[static_cast<size_t>(((ir + 2 * i) * n + (is + 2 * j)) * n + (it + 2 * k))];
                            worst = std::max({worst, std::abs(child[a].u - pn.u), std::abs(child[a].v - pn.v),
                                              std::abs(child[a].w - pn.w)});
                        }
                    }
        }
        add("grid_nesting", worst, tol(1e-12));
    }
    {  // shift_vector_count (through the library's geometry export)
        std::set<Index3> shifts;
        for (const Index3 e : {Index3{1, 0, 0}, Index3{0, 1, 0}, Index3{0, 0, 1}})
            for (const auto& w : g) shifts.insert(w.apply(e));
        const bool ok = shifts.size() == 14;
        add("shift_vector_count", ok ? 0.0 : static_cast<double>(shifts.size()), 0.5,
            std::to_string(shifts.size()) + " vectors");
    }
    {  // factorization_residual on the GPU (and the perturbation control)
        double worst = 0.0;
        std::string note;
        for (int n = 2; n <= n_max; n += 2) {
            Plan plan, pert;
            check(fcct_plan_create(n, canon.r, canon.s, canon.t, FCCT_FAST, FCCT_F64, 0, &plan.h));
            fcct_plan use = plan.h;
            if (perturb) {
                check(fcct_plan_perturbed_basis(plan.h, 1e-3, &pert.h));
                use = pert.h;
            }
            double r = 0;
            check(fcct_factorization_residual(use, &r));
            worst = std::max(worst, r);
            note += (note.empty() ? "" : ", ") + std::string("n=") + std::to_string(n) + ": " + g17(r);
        }
        add("factorization_residual", worst, tol(1e-9), note);
    }
    {  // fast_matches_dense and round_trip on the GPU
        double worst_fwd = 0.0, worst_rt = 0.0;
        std::mt19937 rng(17);
        std::normal_distribution<double> gauss(0.0, 1.0);
        for (int n = 2; n <= n_max; ++n) {
            Plan fast, dense;
            check(fcct_plan_create(n, canon.r, canon.s, canon.t, FCCT_FAST, FCCT_F64, 0, &fast.h));
            check(fcct_plan_create(n, canon.r, canon.s, canon.t, FCCT_DIRECT, FCCT_F64, 0, &dense.h));
            const size_t N = static_cast<size_t>(cube(n));
            std::vector<Complex> s(N), yf(N), yd(N), back(N);
            for (auto& v : s) v = Complex{gauss(rng), gauss(rng)};
            check(fcct_forward_host(fast.h, s.data(), yf.data(), 1, nullptr));
            check(fcct_forward_host(dense.h, s.data(), yd.data(), 1, nullptr));
            double scale = 0, diff = 0, sscale = 0, rdiff = 0;
            for (size_t i = 0; i < N; ++i) {
                scale = std::max(scale, std::abs(yd[i]));
                diff = std::max(diff, std::abs(yf[i] - yd[i]));
            }
            worst_fwd = std::max(worst_fwd, diff / scale);
            check(fcct_inverse_host(fast.h, yf.data(), back.data(), 1, nullptr));
            for (size_t i = 0; i < N; ++i) {
                sscale = std::max(sscale, std::abs(s[i]));
                rdiff = std::max(rdiff, std::abs(back[i] - s[i]));
            }
            worst_rt = std::max(worst_rt, rdiff / sscale);
        }
        add("fast_matches_dense", worst_fwd, tol(1e-10));
        add("round_trip", worst_rt, tol(1e-8));
    }
    {  // basis_sparsity (informational)
        std::string note;
        for (int n = 2; n <= n_max; n += 2) {
            int64_t nnz = 0;
            check(fcct_basis_change(n, canon.r, canon.s, canon.t, 0, &nnz, nullptr, nullptr, nullptr));
            note += (note.empty() ? "" : ", ") + std::string("n=") + std::to_string(n) +
                    ": nnz/n^3=" + g17(static_cast<double>(nnz) / static_cast<double>(cube(n)));
        }
        add("basis_sparsity", 0.0, 1.0, note);
    }
    return out;
}

int cmd_verify(int n_max, double tolerance, bool perturb, const std::string& out) {  // fcct.cpp:440-468
    const auto checks = run_checks(n_max, tolerance, perturb);
    bool all = true;
    for (const auto& c : checks) {
        all = all && c.passed;
        std::cerr << (c.passed ? "ok   " : "FAIL ") << c.name << "  residual=" << g17(c.residual)
                  << " tolerance=" << g17(c.tolerance);
        if (!c.detail.empty()) std::cerr << "  (" << c.detail << ")";
        std::cerr << '\n';
    }
    // nlohmann::json::dump(2): sorted keys, two-space indent
    std::string j = "{\n  \"all_passed\": " + std::string(all ? "true" : "false") + ",\n  \"checks\": [";
    for (size_t i = 0; i < checks.size(); ++i) {
        const auto& c = checks[i];
        j += std::string(i ? "," : "") + "\n    {\n      \"detail\": " + json_str(c.detail) +
             ",\n      \"name\": " + json_str(c.name) + ",\n      \"passed\": " + (c.passed ? "true" : "false") +
             ",\n      \"residual\": " + json_num(c.residual) + ",\n      \"tolerance\": " + json_num(c.tolerance) +
             "\n    }";
    }
    j += std::string(checks.empty() ? "" : "\n  ") + "],\n  \"n_max\": " + std::to_string(n_max) +
         ",\n  \"perturb_basis\": " + (perturb ? "true" : "false") + "\n}\n";
    write_text_output(out, j);
    return all ? 0 : 2;
}

int cmd_bench(const std::string& sizes_text, int repeats, int max_naive, const std::string& cache_dir,
              const std::string& out) {  // fcct.cpp:472-549
    std::vector<int> sizes;
    {
        std::stringstream ss(sizes_text);
        std::string tok;
        while (std::getline(ss, tok, ',')) {
            char* end = nullptr;
            const long v = std::strtol(tok.c_str(), &end, 10);
            if (tok.empty() || end == tok.c_str()) {
                std::cerr << "error: bad --sizes entry '" << tok << "'\n";
                return 1;
            }
            if (v < 1) {
                std::cerr << "error: sizes must be >= 1\n";
                return 1;
            }
            sizes.push_back(static_cast<int>(v));
        }
        if (sizes.empty()) {
            std::cerr << "error: --sizes is empty\n";
            return 1;
        }
    }
    Store store;
    open_store(store, cache_dir);
    const Params params;
    std::ostringstream csv;
    csv << "n,method,plan_seconds,apply_seconds\n";
    std::mt19937 rng(99);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (const int n : sizes) {
        const size_t N = static_cast<size_t>(cube(n));
        std::vector<Complex> s(N), sink(N);
        for (auto& v : s) v = Complex{gauss(rng), gauss(rng)};
        const int inner = static_cast<int>(std::max<int64_t>(1, 32768 / cube(n)));
        auto median_apply = [&](fcct_plan h) {  // one host-buffer apply per call, as apply_values
            std::vector<double> times;
            check(fcct_forward_host(h, s.data(), sink.data(), 1, nullptr));  // warmup
            for (int rep = 0; rep < repeats; ++rep) {
                const auto t0 = Clock::now();
                for (int i = 0; i < inner; ++i) check(fcct_forward_host(h, s.data(), sink.data(), 1, nullptr));
                times.push_back(seconds_since(t0) / inner);
            }
            std::sort(times.begin(), times.end());
            return times[times.size() / 2];
        };
        {
            const auto t0 = Clock::now();
            Plan plan;
            make_plan(plan, n, params, false, store.h);
            const double plan_s = seconds_since(t0);
            csv << n << ",fast," << g17(plan_s) << ',' << g17(median_apply(plan.h)) << '\n';
            std::cerr << "bench n=" << n << " fast done\n";
        }
        if (n <= max_naive) {
            const auto t0 = Clock::now();
            Plan plan;
            make_plan(plan, n, params, true, nullptr);
            const double build_s = seconds_since(t0);
            csv << n << ",naive," << g17(build_s) << ',' << g17(median_apply(plan.h)) << '\n';
            std::cerr << "bench n=" << n << " naive done\n";
        }
    }
    write_text_output(out, csv.str());
    return 0;
}

int cmd_plan(int n, const std::string& params_text, const std::string& cache_dir) {  // fcct.cpp:553-573
    if (cache_dir.empty()) {
        std::cerr << "error: plan needs --cache-dir or FCCT_CACHE_DIR\n";
        return 1;
    }
    const Params p = parse_params(params_text);
    Store store;
    open_store(store, cache_dir);
    check(fcct_store_warm(store.h, n, p.r, p.s, p.t));
    int hits = 0, misses = 0, rebuilt = 0;
    check(fcct_store_stats(store.h, &hits, &misses, &rebuilt));
    size_t files = 0;
    if (DIR* d = opendir(cache_dir.c_str())) {
        while (const dirent* e = readdir(d)) {
            const std::string nm = e->d_name;
            if (nm.size() > 8 && nm.compare(nm.size() - 8, 8, ".fccplan") == 0) ++files;
        }
        closedir(d);
    }
    std::cout << "plan n=" << n << " params=" << encode(p) << ": loaded=" << hits << " built=" << misses
              << " rebuilt=" << rebuilt << " cache_files=" << files << '\n';
    return 0;
}

int cmd_sword(int n, const std::string& out) {  // fcct.cpp:577-583
    std::vector<double> v(static_cast<size_t>(cube(n)));
    check(fcct_synthetic_sword(n, v.data()));
    check(fcct_grid_save(out.c_str(), n, v.data(), "{\"solid\":\"sword\"}"));
    uint64_t sum = 0;
    check(fcct_occupancy_checksum(v.data(), cube(n), &sum));
    std::cerr << "sword n=" << n << " checksum=" << sum << "\n";
    return 0;
}

int cmd_geometry(const std::string& out) {
    std::string path = out.empty() ? "-" : out;
    if (path == "-") std::cout.flush();
    check(fcct_export_geometry(path.c_str()));
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const char* env = std::getenv("FCCT_CACHE_DIR");
    const std::string env_cache = env && *env ? env : "";
    std::vector<Sub> subs;
    {
        Sub s{"zeros", "Generate transform nodes as CSV", {}};
        s.add("--n", "Grid size", "8", true).validate = range("--n", 1, 4096);
        s.add("--params", "Grid offsets r,s,t", kCanonical);
        s.add("--out", "Output CSV path (default stdout)");
        subs.push_back(s);
    }
    {
        Sub s{"transform", "Apply the transform to voxel data", {}};
        s.add("--input", "Input file", "", true);
        s.add("--out", "Output file", "", true);
        s.add("--method", "fast or naive", "fast").validate = member("--method", {"fast", "naive"});
        s.add("--direction", "forward or inverse", "forward").validate = member("--direction", {"forward", "inverse"});
        s.add("--params", "Grid offsets r,s,t", kCanonical);
        s.add("--n", "Expected grid size (checked against the input)", "0").validate = [](const std::string& v) {
            to_int("--n", v);
        };
        s.add("--cache-dir", "Plan cache directory", env_cache);
        s.add("--threads", "Worker threads", "1").validate = range("--threads", 1, 64);
        subs.push_back(s);
    }
    {
        Sub s{"verify", "Run the invariant and residual checks", {}};
        s.add("--n-max", "Largest grid size to check", "4").validate = range("--n-max", 1, 16);
        s.add("--tolerance", "Override the per-check tolerances", "0").validate = [](const std::string& v) {
            to_double("--tolerance", v);
        };
        s.flag("--perturb-b", "Negative control: break the basis factor first");
        s.add("--out", "Write the JSON report here");
        subs.push_back(s);
    }
    {
        Sub s{"bench", "Time plan building and applies", {}};
        s.add("--sizes", "Comma-separated grid sizes", "2,4,8");
        s.add("--repeats", "Timing repetitions", "5").validate = range("--repeats", 1, 1000);
        s.add("--threads", "Worker threads", "1").validate = range("--threads", 1, 64);
        s.add("--max-naive", "Skip the dense method above this size", "16").validate = [](const std::string& v) {
            to_int("--max-naive", v);
        };
        s.add("--cache-dir", "Plan cache directory", env_cache);
        s.add("--out", "Output CSV path (default stdout)");
        subs.push_back(s);
    }
    {
        Sub s{"plan", "Build and cache a transform plan", {}};
        s.add("--n", "Grid size", "8", true).validate = range("--n", 1, 4096);
        s.add("--params", "Grid offsets r,s,t", kCanonical);
        s.add("--cache-dir", "Plan cache directory", env_cache);
        subs.push_back(s);
    }
    {
        Sub s{"sword", "Write the synthetic test solid", {}};
        s.add("--n", "Grid size", "16", true).validate = range("--n", 8, 4096);
        s.add("--out", "Output grid path", "", true);
        subs.push_back(s);
    }
    {
        Sub s{"geometry", "Write the lattice shift vectors as CSV", {}};
        s.add("--out", "Output CSV path (default stdout)");
        subs.push_back(s);
    }

    Sub* sub = nullptr;
    try {
        std::vector<std::string> args(argv + 1, argv + argc);
        for (const auto& a : args)
            if (a == "-h" || a == "--help") {
                for (auto& s : subs)
                    if (!args.empty() && args[0] == s.name) sub = &s;
                print_help(subs, sub);
                return 0;
            }
        if (args.empty()) throw UsageError("A subcommand is required");
        for (auto& s : subs)
            if (args[0] == s.name) sub = &s;
        if (!sub) throw UsageError("The following argument was not expected: " + args[0]);
        for (size_t i = 1; i < args.size(); ++i) {
            std::string a = args[i], val;
            bool has_val = false;
            if (const auto eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = a.substr(eq + 1);
                a = a.substr(0, eq);
                has_val = true;
            }
            Opt* o = sub->find(a);
            if (!o) throw UsageError("The following argument was not expected: " + args[i]);
            if (o->flag) {
                if (has_val) throw UsageError(a + ": flag takes no value");
                o->seen = true;
                o->value = "1";
                continue;
            }
            if (!has_val) {
                if (i + 1 >= args.size()) throw UsageError(a + ": 1 required VALUE missing");
                val = args[++i];
            }
            if (o->validate) o->validate(val);
            o->value = val;
            o->seen = true;
        }
        for (const auto& o : sub->opts)
            if (o.required && !o.seen) throw UsageError(o.name + " is required");
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return 1;
    }

    try {
        const std::string name = sub->name;
        if (name == "zeros") return cmd_zeros(std::stoi(sub->get("--n")), sub->get("--params"), sub->get("--out"));
        if (name == "transform") {
            TransformArgs t;
            t.input = sub->get("--input");
            t.output = sub->get("--out");
            t.method = sub->get("--method");
            t.direction = sub->get("--direction");
            t.params_text = sub->get("--params");
            t.n_override = std::stoi(sub->get("--n"));
            t.cache_dir = sub->get("--cache-dir");
            t.threads = std::stoi(sub->get("--threads"));
            return cmd_transform(t);
        }
        if (name == "verify")
            return cmd_verify(std::stoi(sub->get("--n-max")), std::strtod(sub->get("--tolerance").c_str(), nullptr),
                              sub->has("--perturb-b"), sub->get("--out"));
        if (name == "bench")
            return cmd_bench(sub->get("--sizes"), std::stoi(sub->get("--repeats")), std::stoi(sub->get("--max-naive")),
                             sub->get("--cache-dir"), sub->get("--out"));
        if (name == "plan") return cmd_plan(std::stoi(sub->get("--n")), sub->get("--params"), sub->get("--cache-dir"));
        if (name == "sword") return cmd_sword(std::stoi(sub->get("--n")), sub->get("--out"));
        if (name == "geometry") return cmd_geometry(sub->get("--out"));
    } catch (const CliError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return e.io ? 3 : 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
    return 1;
}
