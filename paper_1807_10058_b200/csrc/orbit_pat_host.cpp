// Host side of the single-pass orbit-pattern executor (orbit_pat.hpp): the
// orbit blocks of S_n(p) classified by shape, the two big shapes compiled into
// DMMA fragment tables, the rare ones into SIMT rows.
#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <map>
#include <mutex>
#include <numbers>

#include "orbit_pat.hpp"
#include "plan.hpp"

namespace fcct {

namespace {

using cd = std::complex<double>;

struct Shape {
    int d = 0;
    std::vector<cld> M, Minv;  // d x d row-major, members in group order
    std::vector<int> orbits;
};

long double max_diff(const std::vector<cld>& a, const std::vector<cld>& b) {
    long double m = 0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

// wavefronts of one 8-byte access per lane into a plane of doubles: half-warps
// of 16 lanes, 16 banks of 8 bytes; equal addresses are one broadcast
int wavefronts8(const std::array<int, 32>& slot, const std::array<bool, 32>& on) {
    int total = 0;
    for (int h = 0; h < 2; ++h) {
        int worst = 0;
        for (int bank = 0; bank < 16; ++bank) {
            std::array<int, 16> seen{};
            int ns = 0;
            for (int l = 16 * h; l < 16 * h + 16; ++l) {
                if (!on[l] || (slot[l] & 15) != bank) continue;
                if (std::find(seen.begin(), seen.begin() + ns, slot[l]) == seen.begin() + ns) seen[ns++] = slot[l];
            }
            worst = std::max(worst, ns);
        }
        total += worst;
    }
    return total;
}

// Bank-conflict search for one DMMA class. The kernel's fragment gather of
// k-step q touches, per half-warp, members pi[4 q .. 4 q + 3] of 4 orbits (16
// doubles of one plane), its scatter of n-tile nt members pi[8 nt + e + 2 kk];
// banks are slot mod 16. Free choices: the order of the orbits (which 4 share a
// half-warp) and the member order pi (shared by the class: it permutes the
// operator's rows and columns). Deterministic hill climbing: orbit swaps
// between half-warps, now and then a swap inside pi.
struct ConflictSearch {
    int d = 0;
    const std::vector<std::vector<int>>* L = nullptr;
    std::vector<int> ord;  // orbit ids; slots beyond ord.size() in the last tile are padding
    std::vector<int> pi;   // member order
    int wl = 1, ws = 1;    // planes read by a gather / written by a scatter
    std::vector<std::array<int, 4>> quads_ld, quads_st;
    std::vector<int> st_live;  // live members of a store quad (d = 12: rows 8..11 only)

    void quads() {
        quads_ld.clear();
        quads_st.clear();
        st_live.clear();
        for (int q = 0; q < d / 4; ++q) quads_ld.push_back({pi[4 * q], pi[4 * q + 1], pi[4 * q + 2], pi[4 * q + 3]});
        for (int nt = 0; nt < (d + 7) / 8; ++nt)
            for (int e = 0; e < 2; ++e) {
                std::array<int, 4> qd{};
                int live = 0;
                for (int kk = 0; kk < 4; ++kk)
                    if (8 * nt + e + 2 * kk < d) qd[live++] = pi[8 * nt + e + 2 * kk];
                quads_st.push_back(qd);
                st_live.push_back(live);
            }
    }
    int quad_cost(int g, const std::array<int, 4>& qd, int live) const {  // half-warp g: orbits ord[4 g ..]
        int cnt[16] = {};
        int worst = 0;
        for (int o = 4 * g; o < 4 * g + 4 && o < static_cast<int>(ord.size()); ++o)
            for (int m = 0; m < live; ++m) worst = std::max(worst, ++cnt[(*L)[ord[o]][qd[m]] & 15]);
        return worst;
    }
    int group_cost(int g) const {
        int c = 0;
        for (const auto& qd : quads_ld) c += wl * quad_cost(g, qd, 4);
        for (size_t i = 0; i < quads_st.size(); ++i) c += ws * quad_cost(g, quads_st[i], st_live[i]);
        return c;
    }
    int groups() const { return (static_cast<int>(ord.size()) + 3) / 4; }
    int total() const {
        int c = 0;
        for (int g = 0; g < groups(); ++g) c += group_cost(g);
        return c;
    }
    void run(int rounds, int swaps_per_round) {
        uint64_t rng = 0x9E3779B97F4A7C15ull;
        auto next = [&](int mod) {
            rng = rng * 6364136223846793005ull + 1442695040888963407ull;
            return static_cast<int>((rng >> 33) % static_cast<uint64_t>(mod));
        };
        quads();
        const int G = groups(), n_orb = static_cast<int>(ord.size());
        std::vector<int> gc(G);
        for (int g = 0; g < G; ++g) gc[g] = group_cost(g);
        auto sweep = [&]() {
            for (int it = 0; it < swaps_per_round; ++it) {
                const int a = next(n_orb), b = next(n_orb), ga = a / 4, gb = b / 4;
                if (ga == gb) continue;
                std::swap(ord[a], ord[b]);
                const int ca = group_cost(ga), cb = group_cost(gb);
                if (ca + cb <= gc[ga] + gc[gb]) {
                    gc[ga] = ca;
                    gc[gb] = cb;
                } else {
                    std::swap(ord[a], ord[b]);
                }
            }
        };
        sweep();
        for (int r = 0; r < rounds; ++r) {
            const std::vector<int> ord0 = ord, gc0 = gc;
            int before = 0;
            for (int g = 0; g < G; ++g) before += gc[g];
            const int a = next(d), b = next(d);
            if (a == b) continue;
            std::swap(pi[a], pi[b]);
            quads();
            for (int g = 0; g < G; ++g) gc[g] = group_cost(g);
            sweep();
            int after = 0;
            for (int g = 0; g < G; ++g) after += gc[g];
            if (after > before) {
                std::swap(pi[a], pi[b]);
                quads();
                ord = ord0;
                gc = gc0;
            }
        }
    }
};

}  // namespace

namespace {
bool compile_from_blocks(int n, const Params& p, const OrbitBlocks& ob, bool inverse, OrbitPatHost& h);
}

bool compile_orbit_pat(int n, const Params& p, bool inverse, OrbitPatHost& h) {
    if (n != 16 && n != 32 && n != 64) return false;
    const OrbitBlocks ob = orbit_blocks(n, p);
    return compile_from_blocks(n, p, ob, inverse, h);
}

bool compile_orbit_pat_pair(int n, const Params& p, OrbitPatHost& fwd, OrbitPatHost& inv) {
    if (n != 16 && n != 32 && n != 64) return false;
    const OrbitBlocks ob = orbit_blocks(n, p);  // the long-double blocks once for both directions
    return compile_from_blocks(n, p, ob, false, fwd) && compile_from_blocks(n, p, ob, true, inv);
}

namespace {

bool compile_from_blocks(int n, const Params& p, const OrbitBlocks& ob, bool inverse, OrbitPatHost& h) {
    const int N = static_cast<int>(cube(n));
    if (!std::isfinite(ob.worst_condition)) return false;
    const Orbits& orb = *ob.orb;
    const auto& grp = s4_group();
    const long double pr = p.r, ps = p.s, pt = p.t;
    auto lam = [&](int a) {  // Lambda[a] = e^{2 pi i a.p/n} / 24
        const int i = a / (n * n), j = (a / n) % n, k = a % n;
        return unit_phase_ld((pr * i + ps * j + pt * k) / n) / 24.0L;
    };
    const int norb = static_cast<int>(orb.members.size());
    // members in group order from the smallest member
    std::vector<std::vector<int>> L(norb);
    std::vector<Shape> shapes;
    for (int o = 0; o < norb; ++o) {
        const auto& mem = orb.members[o];
        const int d = static_cast<int>(mem.size());
        const int a0 = mem[0];
        const int k0[3] = {a0 / (n * n), (a0 / n) % n, a0 % n};
        for (const auto& w : grp) {
            int b[3];
            for (int i = 0; i < 3; ++i) {
                const int v = w[3 * i] * k0[0] + w[3 * i + 1] * k0[1] + w[3 * i + 2] * k0[2];
                b[i] = ((v % n) + n) % n;
            }
            const int a = (b[0] * n + b[1]) * n + b[2];
            if (std::find(L[o].begin(), L[o].end(), a) == L[o].end()) L[o].push_back(a);
        }
        if (static_cast<int>(L[o].size()) != d) return false;
        std::vector<cld> M(static_cast<size_t>(d) * d), Mi(static_cast<size_t>(d) * d), lv(d);
        for (int r = 0; r < d; ++r) lv[r] = lam(L[o][r]);
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c) {
                const size_t src = static_cast<size_t>(orb.pos[L[o][r]]) * d + orb.pos[L[o][c]];
                M[static_cast<size_t>(r) * d + c] = ob.S[o][src] / lv[r];
                Mi[static_cast<size_t>(r) * d + c] = ob.Sinv[o][src] * lv[c];
            }
        bool found = false;
        for (Shape& s : shapes)
            if (s.d == d && max_diff(s.M, M) < 1e-12L && max_diff(s.Minv, Mi) < 1e-10L) {
                s.orbits.push_back(o);
                found = true;
                break;
            }
        if (!found) shapes.push_back(Shape{d, std::move(M), std::move(Mi), {o}});
    }
    h = OrbitPatHost{};
    h.n = n;
    h.N = N;
    h.dir = inverse ? 1 : 0;
    h.patterns = static_cast<int>(shapes.size());
    // DMMA classes: the most populated shape of 24 and of 12 members
    const int cls_d[2] = {24, 12};
    int cls[2] = {-1, -1};
    for (int c = 0; c < 2; ++c)
        for (size_t s = 0; s < shapes.size(); ++s)
            if (shapes[s].d == cls_d[c] && (cls[c] < 0 || shapes[s].orbits.size() > shapes[cls[c]].orbits.size()))
                cls[c] = static_cast<int>(s);
    if (cls[0] < 0) return false;
    std::vector<char> in_class(norb, 0);
    for (int c = 0; c < 2; ++c) {
        if (cls[c] < 0) continue;
        h.cnt[c] = static_cast<int>(shapes[cls[c]].orbits.size());
        h.ntiles[c] = (h.cnt[c] + 7) / 8;
        for (int o : shapes[cls[c]].orbits) in_class[o] = 1;
    }
    const long double inv_scale = 1.0L / N;
    {  // Lambda[(i, j, k)] = L0[i] L1[j] L2[k]; 1/24 (forward) or 24 / N (inverse, conjugated) on axis 0
        const long double off[3] = {pr, ps, pt};
        for (int ax = 0; ax < 3; ++ax)
            for (int x = 0; x < n; ++x) {
                cld v = unit_phase_ld((inverse ? -off[ax] : off[ax]) * x / n);
                if (ax == 0) v *= inverse ? 24.0L * inv_scale : 1.0L / 24.0L;
                h.lax[ax][x][0] = static_cast<double>(v.real());
                h.lax[ax][x][1] = static_cast<double>(v.imag());
            }
    }
    for (int c = 0; c < 2; ++c) {
        if (cls[c] < 0) continue;
        const Shape& sh = shapes[cls[c]];
        const int d = sh.d, KT = d / 4, NT = (d + 7) / 8;
        // orbit order and member order with the fewest modelled bank conflicts
        ConflictSearch cs;
        cs.d = d;
        cs.L = &L;
        cs.ord = sh.orbits;
        cs.pi.resize(d);
        for (int m = 0; m < d; ++m) cs.pi[m] = m;
        cs.wl = 2;  // planes (Re, Im) a gather reads / a scatter writes; real I/O halves one side
        cs.ws = 2;
        {  // the search does not depend on the direction or the offsets: once per (n, class)
            static std::mutex mu;
            static std::map<std::pair<int, int>, std::pair<std::vector<int>, std::vector<int>>> cache;
            std::lock_guard<std::mutex> lock(mu);
            auto it = cache.find({n, d});
            if (n > 16) {
                // large n gathers from global memory (L2): no banks to avoid
            } else if (it == cache.end() || it->second.first.size() != cs.ord.size()) {
                cs.run(300, 2000);
                cache[{n, d}] = {cs.ord, cs.pi};
            } else {
                cs.ord = it->second.first;
                cs.pi = it->second.second;
            }
        }
        const std::vector<int>& pi = cs.pi;
        std::vector<cld> M(static_cast<size_t>(d) * d);
        for (int r = 0; r < d; ++r)
            for (int cc = 0; cc < d; ++cc)
                M[static_cast<size_t>(r) * d + cc] = (inverse ? sh.Minv : sh.M)[static_cast<size_t>(pi[r]) * d + pi[cc]];
        auto member = [&](int o, int m) { return L[o][pi[m]]; };
        h.op[c].assign(static_cast<size_t>(KT) * NT * 32 * 2, 0.0);
        for (int q = 0; q < KT; ++q)
            for (int nt = 0; nt < NT; ++nt)
                for (int l = 0; l < 32; ++l) {
                    const int row = 8 * nt + l / 4, col = 4 * q + l % 4;
                    const cld v = row < d ? M[static_cast<size_t>(row) * d + col] : cld{0, 0};
                    h.op[c][((static_cast<size_t>(q) * NT + nt) * 32 + l) * 2] = static_cast<double>(v.real());
                    h.op[c][((static_cast<size_t>(q) * NT + nt) * 32 + l) * 2 + 1] = static_cast<double>(v.imag());
                }
        const int T = h.ntiles[c];
        auto orbit_at = [&](int t, int o) {  // padding slots of the last tile repeat its first orbit
            const int i = t * 8 + o;
            return cs.ord[i < h.cnt[c] ? i : t * 8];
        };
        for (int t = 0; t < T; ++t)
            for (int m = 0; m < d; ++m)
                for (int o = 0; o < 8; ++o) h.idx.push_back(pat_slot(member(orbit_at(t, o), m)));
        h.dmma += static_cast<int64_t>(T) * KT * NT * 4;
        // shared-memory conflict model of the gathers and scatters
        for (int t = 0; t < T; ++t) {
            std::array<int, 32> slot{};
            std::array<bool, 32> on{};
            for (int q = 0; q < KT; ++q) {
                for (int l = 0; l < 32; ++l) {
                    slot[l] = pat_slot(member(orbit_at(t, l / 4), 4 * q + l % 4));
                    on[l] = true;
                }
                h.wavefronts += wavefronts8(slot, on);
                h.wavefronts_floor += 2;
            }
            for (int nt = 0; nt < NT; ++nt)
                for (int e = 0; e < 2; ++e) {
                    int live = 0;
                    for (int l = 0; l < 32; ++l) {
                        const int row = 8 * nt + 2 * (l % 4) + e;
                        on[l] = row < d && t * 8 + l / 4 < h.cnt[c];
                        slot[l] = on[l] ? pat_slot(member(orbit_at(t, l / 4), row)) : 0;
                        live += on[l];
                    }
                    h.wavefronts += wavefronts8(slot, on);
                    h.wavefronts_floor += (live + 15) / 16;
                }
        }
    }
    // tiles to warps: class 0 round robin, class 1 to the least loaded warp
    {
        int na[kPatWarps] = {}, nb[kPatWarps] = {}, load[kPatWarps] = {};
        for (int t = 0; t < h.ntiles[0]; ++t) {
            ++na[t % kPatWarps];
            load[t % kPatWarps] += 72;
        }
        for (int t = 0; t < h.ntiles[1]; ++t) {
            const int w = static_cast<int>(std::min_element(load, load + kPatWarps) - load);
            ++nb[w];
            load[w] += 24;
        }
        h.warp_tiles.assign(2 * kPatWarps * 2, 0);
        int fa = 0, fb = 0;
        for (int w = 0; w < kPatWarps; ++w) {
            h.warp_tiles[(0 * kPatWarps + w) * 2] = fa;
            h.warp_tiles[(0 * kPatWarps + w) * 2 + 1] = na[w];
            h.warp_tiles[(1 * kPatWarps + w) * 2] = fb;
            h.warp_tiles[(1 * kPatWarps + w) * 2 + 1] = nb[w];
            fa += na[w];
            fb += nb[w];
        }
    }
    // rare shapes: one SIMT row per output member, the entries of S / S^-1 with Lambda divided out,
    // term-major and padded to kPatRareTerms (zero coefficient on the row's own
    // first input)
    {
        struct Row { int out; std::vector<std::pair<int, cld>> terms; };
        std::vector<Row> rows;
        for (int o = 0; o < norb; ++o) {
            if (in_class[o]) continue;
            const auto& mem = orb.members[o];
            const int d = static_cast<int>(mem.size());
            const std::vector<cld>& M = inverse ? ob.Sinv[o] : ob.S[o];
            for (int r = 0; r < d; ++r) {
                Row row{pat_slot(mem[r]), {}};
                for (int c = 0; c < d; ++c) {
                    // Lambda is applied by the FFT passes to every element: divide it out
                    const cld v = inverse ? M[static_cast<size_t>(r) * d + c] * lam(mem[c])
                                          : M[static_cast<size_t>(r) * d + c] / lam(mem[r]);
                    if (v != cld{0, 0}) row.terms.emplace_back(pat_slot(mem[c]), v);
                }
                if (row.terms.empty()) row.terms.emplace_back(pat_slot(mem[0]), cld{0, 0});
                if (static_cast<int>(row.terms.size()) > kPatRareTerms) return false;
                h.rare_terms += static_cast<int64_t>(row.terms.size());
                rows.push_back(std::move(row));
            }
        }
        h.nrare = static_cast<int>(rows.size());
        if (n == 16 && h.nrare > kPatMaxRare * kPatWarps * 32) return false;
        h.rare_pitch = (h.nrare + 31) / 32 * 32;
        h.rare_out.assign(h.nrare, 0);
        h.rare_in.assign(static_cast<size_t>(kPatRareTerms) * h.rare_pitch, 0);
        h.rare_coef.assign(static_cast<size_t>(kPatRareTerms) * h.rare_pitch * 2, 0.0);
        for (int r = 0; r < h.nrare; ++r) {
            h.rare_out[r] = rows[r].out;
            for (int t = 0; t < kPatRareTerms; ++t) {
                const bool on = t < static_cast<int>(rows[r].terms.size());
                const size_t at = static_cast<size_t>(t) * h.rare_pitch + r;
                h.rare_in[at] = on ? rows[r].terms[t].first : rows[r].terms[0].first;
                h.rare_coef[2 * at] = on ? static_cast<double>(rows[r].terms[t].second.real()) : 0.0;
                h.rare_coef[2 * at + 1] = on ? static_cast<double>(rows[r].terms[t].second.imag()) : 0.0;
            }
        }
    }
    if (n == 16 && h.idx.size() * 2 > 10 * 1024) return false;  // the slot lists share the CTA's shared memory with the tile
    // structural check of the tables (the kernels index shared / global memory through
    // them unchecked): every slot in range, and every position of the block written
    // exactly once — by one live orbit slot of a tile or by one rare row
    {
        std::vector<int> written(N, 0);
        size_t base = 0;
        for (int c = 0; c < 2; ++c) {
            const int d = cls_d[c];
            for (int t = 0; t < h.ntiles[c]; ++t)
                for (int m = 0; m < d; ++m)
                    for (int o = 0; o < 8; ++o) {
                        const int slot = h.idx[base + (static_cast<size_t>(t) * d + m) * 8 + o];
                        if (slot < 0 || slot >= N) return false;
                        if (t * 8 + o < h.cnt[c]) ++written[slot];
                    }
            base += static_cast<size_t>(h.ntiles[c]) * d * 8;
        }
        if (base != h.idx.size()) return false;
        for (int r = 0; r < h.nrare; ++r) {
            if (h.rare_out[r] < 0 || h.rare_out[r] >= N) return false;
            ++written[h.rare_out[r]];
        }
        for (int v : h.rare_in)
            if (v < 0 || v >= N) return false;
        for (int a = 0; a < N; ++a)
            if (written[a] != 1) return false;
        int tiles[2] = {0, 0};
        for (int c = 0; c < 2; ++c)
            for (int w = 0; w < kPatWarps; ++w) {
                if (h.warp_tiles[(c * kPatWarps + w) * 2] != tiles[c]) return false;  // contiguous, complete
                tiles[c] += h.warp_tiles[(c * kPatWarps + w) * 2 + 1];
            }
        if (tiles[0] != h.ntiles[0] || tiles[1] != h.ntiles[1]) return false;
    }
    return true;
}

}  // namespace

double OrbitPatHost::exec_flops(bool real_io) const {
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    double twiddles = 0;
    for (int half = n / 2; half >= 1; half /= 2)
        for (int j = 0; j < half; ++j) {
            const int e = j * (n / (2 * half));
            if (e != 0 && 4 * e != n) twiddles += n / (2 * half);
        }
    const double fft = 3.0 * n * n * ((n / 2.0) * lg * 4.0 + 6.0 * twiddles);
    return static_cast<double>(real_io ? dmma / 2 : dmma) * 512.0 + fft + 8.0 * static_cast<double>(rare_terms) + 3.0 * 6.0 * N;
}

namespace {

void dft3(std::vector<cd>& buf, int n, int sign) {
    std::vector<cd> line(n), res(n);
    for (int axis = 0; axis < 3; ++axis)
        for (int u = 0; u < n; ++u)
            for (int v = 0; v < n; ++v) {
                auto at = [&](int x) {
                    int ijk[3];
                    ijk[axis] = x;
                    ijk[axis == 0 ? 1 : 0] = u;
                    ijk[axis == 2 ? 1 : 2] = v;
                    return (ijk[0] * n + ijk[1]) * n + ijk[2];
                };
                for (int x = 0; x < n; ++x) line[x] = buf[at(x)];
                for (int q = 0; q < n; ++q) {
                    cd acc{0, 0};
                    for (int x = 0; x < n; ++x) {
                        const double ang = sign * 2.0 * std::numbers::pi * ((x * q) % n) / n;
                        acc += line[x] * cd{std::cos(ang), std::sin(ang)};
                    }
                    res[q] = acc;
                }
                for (int x = 0; x < n; ++x) buf[at(x)] = res[x];
            }
}

// the base change on the tile X (physical slots), as the kernel indexes its tables
void base_change(const OrbitPatHost& h, std::vector<cd>& X) {
    const int nrare = h.nrare;
    std::vector<cd> rare(nrare);
    for (int r = 0; r < nrare; ++r) {
        cd acc{0, 0};
        for (int t = 0; t < kPatRareTerms; ++t) {
            const size_t at = static_cast<size_t>(t) * h.rare_pitch + r;
            acc += cd{h.rare_coef[2 * at], h.rare_coef[2 * at + 1]} * X[h.rare_in[at]];
        }
        rare[r] = acc;
    }
    size_t idx_base = 0;
    const int cls_d[2] = {24, 12};
    for (int c = 0; c < 2; ++c) {
        const int d = cls_d[c], KT = d / 4, NT = (d + 7) / 8;
        for (int w = 0; w < kPatWarps; ++w) {
            const int first = h.warp_tiles[(c * kPatWarps + w) * 2], count = h.warp_tiles[(c * kPatWarps + w) * 2 + 1];
            for (int t = first; t < first + count; ++t) {
                const int32_t* ix = h.idx.data() + idx_base + static_cast<size_t>(t) * d * 8;
                cd acc[8][24];
                for (int o = 0; o < 8; ++o)
                    for (int nt = 0; nt < NT; ++nt)
                        for (int nl = 0; nl < 8; ++nl) {
                            cd s{0, 0};
                            for (int q = 0; q < KT; ++q)
                                for (int k = 0; k < 4; ++k) {
                                    const cd a = X[ix[(4 * q + k) * 8 + o]];
                                    const size_t ot = ((static_cast<size_t>(q) * NT + nt) * 32 + nl * 4 + k) * 2;
                                    s += a * cd{h.op[c][ot], h.op[c][ot + 1]};
                                }
                            acc[o][8 * nt + nl] = s;
                        }
                for (int o = 0; o < 8; ++o) {
                    if (t * 8 + o >= h.cnt[c]) continue;
                    for (int row = 0; row < d; ++row) {
                        X[ix[row * 8 + o]] = acc[o][row];
                    }
                }
            }
        }
        idx_base += static_cast<size_t>(h.ntiles[c]) * d * 8;
    }
    for (int r = 0; r < nrare; ++r) X[h.rare_out[r]] = rare[r];
}

}  // namespace

void emulate_orbit_pat(const OrbitPatHost& h, const double* in, double* out, int64_t batch) {
    const int N = h.N;
    std::vector<cd> x(N), X(N);
    for (int64_t b = 0; b < batch; ++b) {
        for (int a = 0; a < N; ++a) x[a] = cd{in[2 * (b * N + a)], in[2 * (b * N + a) + 1]};
        auto phases = [&]() {  // the axis passes' constant multiplies
            for (int a = 0; a < N; ++a) {
                const int ijk[3] = {a / (h.n * h.n), (a / h.n) % h.n, a % h.n};
                for (int ax = 0; ax < 3; ++ax) x[a] *= cd{h.lax[ax][ijk[ax]][0], h.lax[ax][ijk[ax]][1]};
            }
        };
        if (h.dir == 1) {
            dft3(x, h.n, -1);
            phases();
        }
        for (int a = 0; a < N; ++a) X[pat_slot(a)] = x[a];
        base_change(h, X);
        for (int a = 0; a < N; ++a) x[a] = X[pat_slot(a)];
        if (h.dir == 0) {
            phases();
            dft3(x, h.n, +1);
        }
        for (int a = 0; a < N; ++a) {
            out[2 * (b * N + a)] = x[a].real();
            out[2 * (b * N + a) + 1] = x[a].imag();
        }
    }
}

}  // namespace fcct
