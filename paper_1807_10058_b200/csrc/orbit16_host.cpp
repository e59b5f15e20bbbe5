// Host side of the two-pass orbit-FFT executor (orbit16.hpp): the orbit blocks
// of S_n(p) packed into chunks of <= kO16Chunk member slots, their DMMA tiles
// balanced over the warps of a CTA per chunk.
#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <numbers>

#include "orbit16.hpp"
#include "plan.hpp"

namespace fcct {

namespace {

struct Chain16 {
    int orbit;
    int nt;                 // n-tile: rows 8 nt .. 8 nt + 7 of the orbit block
    int kt0;                // chunk-local index of the orbit's first k-tile
    int kts;                // k-tiles of the orbit
};

}  // namespace

bool compile_orbit16(int n, const Params& p, bool inverse, Orbit16Host& h) {
    if (n != 16) return false;
    const int N = static_cast<int>(cube(n));
    OrbitBlocks ob = orbit_blocks(n, p);
    // the plan tree carries the reference's condition gates (plan.cpp); a singular
    // orbit block (no S^{-1}) leaves this executor unbuilt
    if (!std::isfinite(ob.worst_condition)) return false;
    const Orbits& orb = *ob.orb;
    // chunks of whole orbits, <= kO16Chunk slots (4 per k-tile), formed
    // greedily so that orbits whose members share 32-byte sectors (four
    // consecutive positions: real f64 input) land in the same chunk: a chunk's
    // gather then reads each sector once instead of once per chunk touching it
    const int norb = static_cast<int>(orb.members.size());
    auto need = [&](int o) { return 4 * ((static_cast<int>(orb.members[o].size()) + 3) / 4); };
    std::vector<std::vector<int>> orb_keys(norb);
    for (int o = 0; o < norb; ++o) {
        for (int m : orb.members[o]) orb_keys[o].push_back(m >> 2);
        std::sort(orb_keys[o].begin(), orb_keys[o].end());
        orb_keys[o].erase(std::unique(orb_keys[o].begin(), orb_keys[o].end()), orb_keys[o].end());
    }
    std::vector<std::vector<int>> chunk_orbits;
    std::vector<char> taken(norb, 0);
    std::vector<int> key_hits(N / 4 + 1, 0);
    for (int left = norb; left > 0;) {
        chunk_orbits.emplace_back();
        std::fill(key_hits.begin(), key_hits.end(), 0);
        int used = 0;
        while (true) {
            int best = -1, best_score = -1;
            for (int o = 0; o < norb; ++o) {
                if (taken[o] || used + need(o) > kO16Chunk) continue;
                int score = 0;
                for (int key : orb_keys[o]) score += key_hits[key] ? 1 : 0;
                // shared sectors first, then larger orbits, then orbit order
                score = score * 64 + static_cast<int>(orb.members[o].size());
                if (score > best_score) {
                    best_score = score;
                    best = o;
                }
            }
            if (best < 0) break;
            taken[best] = 1;
            --left;
            used += need(best);
            chunk_orbits.back().push_back(best);
            for (int key : orb_keys[best]) key_hits[key] = 1;
        }
    }
    const int nchunks = static_cast<int>(chunk_orbits.size());
    std::vector<std::vector<std::vector<Chain16>>> per_warp(nchunks, std::vector<std::vector<Chain16>>(kO16Warps));
    std::vector<int> chunk_slots(nchunks, 0);
    int tmax = 0;
    for (int c = 0; c < nchunks; ++c) {
        std::vector<Chain16> chains;
        int kt = 0;
        for (int o : chunk_orbits[c]) {
            const int s = static_cast<int>(orb.members[o].size()), kts = (s + 3) / 4;
            for (int nt = 0; nt < (s + 7) / 8; ++nt) chains.push_back(Chain16{o, nt, kt, kts});
            kt += kts;
        }
        chunk_slots[c] = 4 * kt;
        std::stable_sort(chains.begin(), chains.end(), [](const Chain16& a, const Chain16& b) { return a.kts > b.kts; });
        std::vector<int> load(kO16Warps, 0);
        for (const Chain16& ch : chains) {
            const int w = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
            per_warp[c][w].push_back(ch);
            load[w] += ch.kts;
        }
        tmax = std::max(tmax, *std::max_element(load.begin(), load.end()));
    }
    tmax = (tmax + kO16Wrap - 1) / kO16Wrap * kO16Wrap;  // the kernel's operator ring stays chunk-aligned
    if (tmax > kO16Tmax) return false;
    h = Orbit16Host{};
    h.n = n;
    h.N = N;
    h.dir = inverse ? 1 : 0;
    h.nchunks = nchunks;
    h.tmax = tmax;
    // operator tiles per warp, contiguous over the chunks ([warp][chunk][tmax]),
    // plus kO16Wrap copies of the warp's first tiles: the kernel streams them
    // with a fixed look-ahead and no per-tile wrap logic
    const size_t per_warp_tiles = static_cast<size_t>(nchunks) * tmax + kO16Wrap;
    h.table.assign(kO16Warps * per_warp_tiles * 32 * 2, 0.0);
    h.tile_meta.assign(static_cast<size_t>(nchunks) * kO16Warps * tmax, 0);
    h.out_pos.assign(static_cast<size_t>(nchunks) * kO16Warps * tmax * 4, -1);
    h.gather.assign(static_cast<size_t>(nchunks) * kO16Chunk, -1);
    h.chunk_slots = chunk_slots;
    const long double scale = inverse ? 1.0L / N : 1.0L;
    // z (the spectrum-side scratch between the passes) is kept in orbit order:
    // orbits in chunk order, members in orbit order. Pass A then reads (inverse)
    // or writes (forward) z in contiguous runs; the cube FFT pass permutes.
    std::vector<int32_t> ord(N, -1);
    {
        int q = 0;
        for (int c = 0; c < nchunks; ++c)
            for (int o : chunk_orbits[c])
                for (int m : orb.members[o]) ord[m] = q++;
    }
    h.zperm = ord;
    auto zside = [&](int lex) { return ord[lex]; };
    for (int c = 0; c < nchunks; ++c) {
        int kt = 0;
        for (int o : chunk_orbits[c]) {  // slot 4 kt + k holds member 4 k-tile + k of the orbit
            const auto& mem = orb.members[o];
            for (size_t m = 0; m < mem.size(); ++m)  // forward: x natural; inverse: z in orbit order
                h.gather[static_cast<size_t>(c) * kO16Chunk + 4 * kt + m] = inverse ? zside(mem[m]) : mem[m];
            kt += (static_cast<int>(mem.size()) + 3) / 4;
        }
        for (int w = 0; w < kO16Warps; ++w) {
            int t = 0;
            for (const Chain16& ch : per_warp[c][w]) {
                const auto& mem = orb.members[ch.orbit];
                const int s = static_cast<int>(mem.size());
                const std::vector<cld>& M = inverse ? ob.Sinv[ch.orbit] : ob.S[ch.orbit];  // [row][col], s x s
                for (int q = 0; q < ch.kts; ++q, ++t) {
                    const size_t ti = (static_cast<size_t>(c) * kO16Warps + w) * tmax + t;
                    const size_t tt = w * per_warp_tiles + static_cast<size_t>(c) * tmax + t;  // table position
                    for (int l = 0; l < 32; ++l) {
                        const int row = 8 * ch.nt + l / 4, col = 4 * q + l % 4;
                        cld v{0, 0};
                        if (row < s && col < s) v = M[static_cast<size_t>(row) * s + col] * scale;
                        h.table[(tt * 32 + l) * 2] = static_cast<double>(v.real());
                        h.table[(tt * 32 + l) * 2 + 1] = static_cast<double>(v.imag());
                    }
                    const bool end = q == ch.kts - 1;
                    h.tile_meta[ti] = (ch.kt0 + q) | (end ? 1 << 16 : 0) | (1 << 17);
                    for (int k = 0; k < 4; ++k) {
                        const int r0 = 8 * ch.nt + 2 * k, r1 = r0 + 1;
                        // both directions store in orbit order (contiguous runs): forward
                        // z, inverse x (un-permuted by a coalesced pass afterwards)
                        auto op = [&](int row) { return row < s ? zside(mem[row]) : 0xFFFF; };
                        const int o0 = op(r0), o1 = op(r1);
                        h.out_pos[ti * 4 + k] = o0 | (o1 << 16);
                    }
                    ++h.tiles;
                }
            }
        }
    }
    for (int w = 0; w < kO16Warps; ++w)  // wrap copies
        for (int t = 0; t < kO16Wrap; ++t)
            for (int e = 0; e < 64; ++e)
                h.table[((w * per_warp_tiles + nchunks * tmax + t) * 32) * 2 + e] =
                    h.table[((w * per_warp_tiles + t) * 32) * 2 + e];
    return true;
}

double Orbit16Host::exec_flops() const {
    const double dmma = static_cast<double>(tiles) * 4.0 * 512.0 / 8.0;
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    double twiddles = 0;
    for (int half = n / 2; half >= 1; half /= 2)
        for (int j = 0; j < half; ++j) {
            const int e = j * (n / (2 * half));
            if (e != 0 && 4 * e != n) twiddles += n / (2 * half);
        }
    return dmma + 3.0 * n * n * ((n / 2.0) * lg * 4.0 + 6.0 * twiddles);
}

namespace {

using cd = std::complex<double>;

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

}  // namespace

void emulate_orbit16(const Orbit16Host& h, const double* in, double* out, int64_t batch) {
    const int N = h.N;
    std::vector<cd> x(N), z(N), stage(kO16Chunk);
    for (int64_t b = 0; b < batch; ++b) {
        for (int a = 0; a < N; ++a) x[a] = cd{in[2 * (b * N + a)], in[2 * (b * N + a) + 1]};
        if (h.dir == 1) {  // z in orbit order
            dft3(x, h.n, -1);
            std::vector<cd> t(N);
            for (int a = 0; a < N; ++a) t[h.zperm[a]] = x[a];
            x = t;
        }
        std::fill(z.begin(), z.end(), cd{0, 0});
        for (int c = 0; c < h.nchunks; ++c) {
            for (int s = 0; s < kO16Chunk; ++s) {
                const int p = h.gather[static_cast<size_t>(c) * kO16Chunk + s];
                stage[s] = p >= 0 ? x[p] : cd{0, 0};
            }
            for (int w = 0; w < kO16Warps; ++w) {
                cd acc[8];
                for (int t = 0; t < h.tmax; ++t) {
                    const size_t ti = (static_cast<size_t>(c) * kO16Warps + w) * h.tmax + t;
                    const int m = h.tile_meta[ti];
                    if (!(m & (1 << 17))) continue;
                    const int kt = m & 0xFFFF;
                    const size_t tt = w * (static_cast<size_t>(h.nchunks) * h.tmax + kO16Wrap) + c * h.tmax + t;
                    for (int l = 0; l < 32; ++l)
                        acc[l / 4] += cd{h.table[(tt * 32 + l) * 2], h.table[(tt * 32 + l) * 2 + 1]} * stage[4 * kt + l % 4];
                    if (m & (1 << 16)) {
                        for (int k = 0; k < 4; ++k) {
                            const int o0 = h.out_pos[ti * 4 + k] & 0xFFFF, o1 = (h.out_pos[ti * 4 + k] >> 16) & 0xFFFF;
                            if (o0 != 0xFFFF) z[o0] = acc[2 * k];
                            if (o1 != 0xFFFF) z[o1] = acc[2 * k + 1];
                        }
                        for (auto& a : acc) a = cd{0, 0};
                    }
                }
            }
        }
        {  // z (forward) / x (inverse) in orbit order -> natural
            std::vector<cd> t(N);
            for (int a = 0; a < N; ++a) t[a] = z[h.zperm[a]];
            z = t;
        }
        if (h.dir == 0) dft3(z, h.n, +1);
        for (int a = 0; a < N; ++a) {
            out[2 * (b * N + a)] = z[a].real();
            out[2 * (b * N + a) + 1] = z[a].imag();
        }
    }
}

}  // namespace fcct
