// Host side of the orbit-FFT executor (orbit_fft.hpp): compiles the orbit
// blocks of S_n(p) (or S_n(p)^{-1} / n^3) into register-resident DMMA tiles.
#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <numbers>
#include <cstdio>
#include <cstdlib>

#include "orbit_fft.hpp"
#include "plan.hpp"

namespace fcct {

namespace {

// One n-tile (8 output rows) of one orbit block and its k-tiles (4 input
// columns each); -1 marks a padding row / column (zero table entries).
struct Chain {
    int orbit;
    std::array<int, 8> rows;
    std::vector<std::array<int, 4>> ktiles;
};

// Partitions members (indices 0..s-1) into groups of <= 4 whose positions are
// distinct mod 4 wherever the residues allow: with a block-row rotation of 4
// bank groups (orbit_fft.cu) the 8 lanes of a quarter-warp (2 blocks x 4
// members) then touch 8 distinct bank groups.
std::vector<std::array<int, 4>> residue_groups(const std::vector<int>& pos) {
    std::array<std::vector<int>, 4> bucket;
    for (int m = 0; m < static_cast<int>(pos.size()); ++m) bucket[pos[m] & 3].push_back(m);
    auto by_size = [&] {
        std::array<int, 4> order{0, 1, 2, 3};
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return bucket[x].size() > bucket[y].size(); });
        return order;
    };
    std::vector<std::array<int, 4>> groups;
    for (int left = static_cast<int>(pos.size()); left > 0;) {
        const int want = std::min(4, left);
        std::array<int, 4> g{-1, -1, -1, -1};
        int filled = 0;
        for (int q : by_size())  // one member from each residue class first
            if (filled < want && !bucket[q].empty()) {
                g[filled++] = bucket[q].back();
                bucket[q].pop_back();
            }
        while (filled < want) {  // then the largest classes (a conflict, but no extra tile)
            const int q = by_size()[0];
            g[filled++] = bucket[q].back();
            bucket[q].pop_back();
        }
        left -= want;
        groups.push_back(g);
    }
    return groups;
}

}  // namespace

bool compile_orbit_fft(int n, const Params& p, bool inverse, OrbitFftHost& h, int warps) {
    if (n != 4 && n != 8) return false;
    if (warps != kOfWarps && warps != kOfBcWarps) return false;
    const int N = static_cast<int>(cube(n));
    const bool ws = warps == kOfBcWarps;
    const int tmax_bound = n == 8 ? (ws ? kOfWsTmax8 : kOfTmax8) : (ws ? kOfWsTmax4 : kOfTmax4);
    OrbitBlocks ob = orbit_blocks(n, p);
    // the plan tree carries the reference's condition gates (plan.cpp); a singular
    // orbit block (no S^{-1}) leaves this executor unbuilt
    if (!std::isfinite(ob.worst_condition)) return false;
    const Orbits& orb = *ob.orb;
    // positions: forward reads natural kappa and writes swizzled a; inverse the reverse
    auto in_pos = [&](int lex) { return inverse ? of_swizzle(lex, n) : lex; };
    auto out_pos = [&](int lex) { return inverse ? lex : of_swizzle(lex, n); };
    std::vector<Chain> chains;
    for (int o = 0; o < static_cast<int>(orb.members.size()); ++o) {
        const auto& mem = orb.members[o];
        std::vector<int> ip, op;
        for (int m : mem) {
            ip.push_back(in_pos(m));
            op.push_back(out_pos(m));
        }
        const auto kt = residue_groups(ip);
        const auto rg = residue_groups(op);
        // n-tile = two row groups: the first on the even output columns (the
        // lanes' first store), the second on the odd ones (the second store)
        for (size_t g = 0; g < rg.size(); g += 2) {
            Chain c{o, {}, kt};
            for (int k = 0; k < 4; ++k) {
                c.rows[2 * k] = rg[g][k];
                c.rows[2 * k + 1] = g + 1 < rg.size() ? rg[g + 1][k] : -1;
            }
            chains.push_back(std::move(c));
        }
    }
    // longest chains first onto the least loaded warp (LPT); ties keep orbit order.
    // Specialised kernel: balance the FP64 pipe of each SMSP first (SMSPs 2 and
    // 3 also run an FFT warp: its butterflies are worth ~14 DMMA tile steps per
    // tile), then the warps inside each SMSP.
    std::stable_sort(chains.begin(), chains.end(),
                     [](const Chain& a, const Chain& b) { return a.ktiles.size() > b.ktiles.size(); });
    std::vector<std::vector<const Chain*>> per_warp(warps);
    std::vector<int> load(warps, 0);
    if (ws) {
        const int fft_steps = n == 8 ? 14 : 0;
        std::array<double, 4> sm_load{};
        std::array<int, 4> sm_warps{};
        for (int w = 0; w < warps; ++w) ++sm_warps[w % 4];
        for (int q = 0; q < 4; ++q)
            if (sm_warps[q] < (warps + 3) / 4) sm_load[q] = fft_steps * sm_warps[q];  // hosts an FFT warp
        for (const Chain& c : chains) {
            // least loaded SMSP (its FP64 pipe is shared by its warps), then its least loaded warp
            int q = 0;
            for (int x = 1; x < 4; ++x)
                if (sm_load[x] < sm_load[q]) q = x;
            int w = q;
            for (int x = q; x < warps; x += 4)
                if (load[x] < load[w]) w = x;
            per_warp[w].push_back(&c);
            load[w] += static_cast<int>(c.ktiles.size());
            sm_load[q] += static_cast<double>(c.ktiles.size());
        }
    } else {
        for (const Chain& c : chains) {
            const int w = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
            per_warp[w].push_back(&c);
            load[w] += static_cast<int>(c.ktiles.size());
        }
    }
    const int tmax = *std::max_element(load.begin(), load.end());
#ifdef FCCT_AB_SWITCHES
    if (std::getenv("FCCT_DEBUG_OFFT_LOAD")) {
        for (int w = 0; w < warps; ++w) fprintf(stderr, "%d ", load[w]);
        fprintf(stderr, "\n");
    }
#endif
    if (tmax > tmax_bound) return false;
    h = OrbitFftHost{};
    h.n = n;
    h.N = N;
    h.dir = inverse ? 1 : 0;
    h.groups = 512 / N >= 1 ? 512 / N : 1;
    h.tmax = tmax;
    h.warps = warps;
    // every warp runs exactly tmax tiles: the padding tiles are zero, flagged
    // neither chain start nor end, and read slot 0 (no per-tile branch remains)
    h.table.assign(static_cast<size_t>(warps) * tmax * 32 * 2, 0.0);
    h.meta.assign(static_cast<size_t>(warps) * tmax * 4 * 2, 0);
    for (size_t e = 1; e < h.meta.size(); e += 2) h.meta[e] = 0xFFFF | (0xFFFF << 16);
    h.ntiles.assign(warps, tmax);  // set to each warp's real count below
    const long double scale = inverse ? 1.0L / N : 1.0L;
    for (int w = 0; w < warps; ++w) {
        int t = 0;
        for (const Chain* c : per_warp[w]) {
            const auto& mem = orb.members[c->orbit];
            const int s = static_cast<int>(mem.size());
            const std::vector<cld>& M = inverse ? ob.Sinv[c->orbit] : ob.S[c->orbit];  // [row][col], s x s
            const int kts = static_cast<int>(c->ktiles.size());
            for (int kt = 0; kt < kts; ++kt, ++t) {
                const auto& cols = c->ktiles[kt];
                for (int l = 0; l < 32; ++l) {
                    const int row = c->rows[l / 4], col = cols[l % 4];
                    cld v{0, 0};
                    if (row >= 0 && col >= 0) v = M[static_cast<size_t>(row) * s + col] * scale;
                    const size_t e = ((static_cast<size_t>(w) * tmax + t) * 32 + l) * 2;
                    h.table[e] = static_cast<double>(v.real());
                    h.table[e + 1] = static_cast<double>(v.imag());
                }
                const int flags = (kt == 0 ? 1 : 0) | (kt == kts - 1 ? 2 : 0);
                for (int k = 0; k < 4; ++k) {
                    const int ip = in_pos(mem[cols[k] >= 0 ? cols[k] : cols[0]]);
                    const int r0 = c->rows[2 * k], r1 = c->rows[2 * k + 1];
                    const int o0 = r0 >= 0 ? out_pos(mem[r0]) : 0xFFFF, o1 = r1 >= 0 ? out_pos(mem[r1]) : 0xFFFF;
                    const size_t e = ((static_cast<size_t>(w) * tmax + t) * 4 + k) * 2;
                    h.meta[e] = ip | (flags << 16);
                    h.meta[e + 1] = o0 | (o1 << 16);
                }
                ++h.tiles;
            }
        }
        h.ntiles[w] = t;
    }
    return true;
}

double OrbitFftHost::exec_flops() const {
    const double dmma = static_cast<double>(tiles) * 4.0 * 512.0 / 8.0;
    // radix-2 line of n points: (n/2) log2 n butterflies of 2 complex add/sub
    // (4 flops each) plus 6 flops per twiddle other than 1 and +-i
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    double twiddles = 0;
    for (int half = n / 2; half >= 1; half /= 2)
        for (int j = 0; j < half; ++j) {
            const int e = j * (n / (2 * half));
            if (e != 0 && 4 * e != n) twiddles += n / (2 * half);
        }
    const double line = (n / 2.0) * lg * 4.0 + 6.0 * twiddles;
    return dmma + 3.0 * n * n * line;
}

namespace {

using cd = std::complex<double>;

// v[q] <- sum_p v[p] e^{sign 2 pi i p q / n} along one axis of an n^3 cube
// stored at positions pos(i, j, k).
template <typename Pos>
void dft_axis(std::vector<cd>& buf, int n, int axis, int sign, Pos pos) {
    std::vector<cd> line(n), res(n);
    for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v) {
            auto at = [&](int x) {
                int ijk[3];
                ijk[axis] = x;
                ijk[axis == 0 ? 1 : 0] = u;
                ijk[axis == 2 ? 1 : 2] = v;
                return pos(ijk[0], ijk[1], ijk[2]);
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

}  // namespace

void emulate_orbit_fft(const OrbitFftHost& h, const double* in, double* out, int64_t batch) {
    const int n = h.n, N = h.N;
    auto swz = [&](int i, int j, int k) { return of_swizzle((i * n + j) * n + k, n); };
    std::vector<cd> y(N), x(N);
    for (int64_t b = 0; b < batch; ++b) {
        const double* src = in + b * 2 * N;
        double* dst = out + b * 2 * N;
        auto base_change = [&](const std::vector<cd>& from, std::vector<cd>& to) {
            for (int w = 0; w < h.warps; ++w) {
                cd acc[8];
                for (int t = 0; t < h.ntiles[w]; ++t) {
                    const int32_t* m = &h.meta[(static_cast<size_t>(w) * h.tmax + t) * 8];
                    const int flags = m[0] >> 16;
                    if (flags & 1)
                        for (auto& a : acc) a = cd{0, 0};
                    for (int l = 0; l < 32; ++l) {
                        const int k = l % 4, col_n = l / 4;
                        const size_t e = ((static_cast<size_t>(w) * h.tmax + t) * 32 + l) * 2;
                        acc[col_n] += cd{h.table[e], h.table[e + 1]} * from[m[2 * k] & 0xFFFF];
                    }
                    if (flags & 2)
                        for (int k = 0; k < 4; ++k) {
                            const int o0 = m[2 * k + 1] & 0xFFFF, o1 = (m[2 * k + 1] >> 16) & 0xFFFF;
                            if (o0 != 0xFFFF) to[o0] = acc[2 * k];
                            if (o1 != 0xFFFF) to[o1] = acc[2 * k + 1];
                        }
                }
            }
        };
        for (int a = 0; a < N; ++a) x[a] = cd{src[2 * a], src[2 * a + 1]};
        if (h.dir == 0) {
            base_change(x, y);  // y at swizzled positions
            for (int axis = 2; axis >= 0; --axis) dft_axis(y, n, axis, +1, swz);
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    for (int k = 0; k < n; ++k) {
                        const cd v = y[swz(i, j, k)];
                        const int a = (i * n + j) * n + k;
                        dst[2 * a] = v.real();
                        dst[2 * a + 1] = v.imag();
                    }
        } else {
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    for (int k = 0; k < n; ++k) y[swz(i, j, k)] = x[(i * n + j) * n + k];
            for (int axis = 0; axis < 3; ++axis) dft_axis(y, n, axis, -1, swz);
            std::vector<cd> o(N);
            base_change(y, o);
            for (int a = 0; a < N; ++a) {
                dst[2 * a] = o[a].real();
                dst[2 * a + 1] = o[a].imag();
            }
        }
    }
}

}  // namespace fcct
