// Plan-time compilation of the fast transform into DMMA stages (tiling.hpp).
#include "tiling.hpp"

#include <algorithm>
#include <cstdlib>
#include <array>
#include <functional>
#include <map>
#include <numeric>

namespace fcct {
namespace {

// Z_s(i): stacked position -> output position of a full radix tree.
std::vector<int32_t> stacked_order(const PlanNode& nd) {
    const int64_t s3 = cube(nd.n);
    std::vector<int32_t> z(s3);
    if (!nd.radix) {
        std::iota(z.begin(), z.end(), 0);
        return z;
    }
    const auto sub = stacked_order(*nd.children[0]);
    const auto perm = radix_permutation(nd.n);
    const int64_t m3 = s3 / 8;
    for (int64_t i = 0; i < s3; ++i) z[i] = static_cast<int32_t>(perm[(i / m3) * m3 + sub[i % m3]]);
    return z;
}

std::vector<int32_t> positions_of(const std::vector<int32_t>& ord) {
    std::vector<int32_t> p(ord.size());
    for (size_t i = 0; i < ord.size(); ++i) p[ord[i]] = static_cast<int32_t>(i);
    return p;
}

int64_t count_tiles(const std::vector<std::vector<int32_t>>& rc, const std::vector<int32_t>& rpos,
                    const std::vector<int32_t>& cpos) {
    std::vector<std::pair<int32_t, int32_t>> t;
    for (size_t r = 0; r < rc.size(); ++r)
        for (int32_t c : rc[r]) t.emplace_back(rpos[r] / 8, cpos[c] / 4);
    std::sort(t.begin(), t.end());
    return std::unique(t.begin(), t.end()) - t.begin();
}

// Greedy co-ordering of one component: alternately sort rows (outputs, groups
// of 8) by the k-tile signature of their columns and columns (inputs, groups
// of 4) by the n-tile signature of their rows; keep the fewest 8x4 tiles.
void order_component(const std::vector<std::vector<int32_t>>& rc, int ncols, std::vector<int32_t>& rord,
                     std::vector<int32_t>& cord) {
    const int nr = static_cast<int>(rc.size());
    rord.resize(nr);
    cord.resize(ncols);
    std::iota(rord.begin(), rord.end(), 0);
    std::iota(cord.begin(), cord.end(), 0);
    std::vector<int> cdeg(ncols, 0);
    for (const auto& r : rc)
        for (int32_t c : r) cdeg[c]++;
    std::stable_sort(cord.begin(), cord.end(), [&](int a, int b) { return cdeg[a] > cdeg[b]; });
    std::vector<int32_t> br = rord, bc = cord;
    int64_t best = count_tiles(rc, positions_of(rord), positions_of(cord));
    for (int it = 0; it < 24; ++it) {
        {
            const auto cp = positions_of(cord);
            std::vector<std::vector<int32_t>> sig(nr);
            for (int r = 0; r < nr; ++r) {
                for (int32_t c : rc[r]) sig[r].push_back(cp[c] / 4);
                std::sort(sig[r].begin(), sig[r].end());
                sig[r].erase(std::unique(sig[r].begin(), sig[r].end()), sig[r].end());
            }
            std::stable_sort(rord.begin(), rord.end(), [&](int a, int b) { return sig[a] < sig[b]; });
        }
        {
            const auto rp = positions_of(rord);
            std::vector<std::vector<int32_t>> sig(ncols);
            for (int r = 0; r < nr; ++r)
                for (int32_t c : rc[r]) sig[c].push_back(rp[r] / 8);
            for (auto& s : sig) {
                std::sort(s.begin(), s.end());
                s.erase(std::unique(s.begin(), s.end()), s.end());
            }
            std::stable_sort(cord.begin(), cord.end(), [&](int a, int b) { return sig[a] < sig[b]; });
        }
        const int64_t t = count_tiles(rc, positions_of(rord), positions_of(cord));
        if (t < best) {
            best = t;
            br = rord;
            bc = cord;
        }
    }
    rord = br;
    cord = bc;
}

using Rows = std::vector<std::vector<std::pair<int32_t, cld>>>;

struct Tiling {
    std::vector<int32_t> row_order, col_order;  // length N
    // per n-tile: (k-tile, 32 lanes x (Re, Im)) of T[k][n] = A[row n][col k]
    std::vector<std::vector<std::pair<int32_t, std::array<double, 64>>>> tiles;
};

Tiling tile_rows(int N, const Rows& rows) {
    std::vector<int32_t> par(2 * N);
    std::iota(par.begin(), par.end(), 0);
    std::function<int32_t(int32_t)> find = [&](int32_t a) {
        while (par[a] != a) a = par[a] = par[par[a]];
        return a;
    };
    for (int32_t r = 0; r < N; ++r)
        for (const auto& e : rows[r]) par[find(r)] = find(N + e.first);
    std::map<int32_t, std::pair<std::vector<int32_t>, std::vector<int32_t>>> comps;
    for (int32_t i = 0; i < 2 * N; ++i) {
        auto& cp = comps[find(i)];
        (i < N ? cp.first : cp.second).push_back(i < N ? i : i - N);
    }
    std::vector<std::pair<std::vector<int32_t>, std::vector<int32_t>>> list;
    for (auto& kv : comps) list.push_back(kv.second);
    std::stable_sort(list.begin(), list.end(), [](const auto& a, const auto& b) {
        return a.first.size() + a.second.size() > b.first.size() + b.second.size();
    });
    Tiling T;
    for (const auto& [rws, cls] : list) {
        std::map<int32_t, int32_t> cl;
        for (size_t j = 0; j < cls.size(); ++j) cl[cls[j]] = static_cast<int32_t>(j);
        std::vector<std::vector<int32_t>> rc(rws.size());
        for (size_t r = 0; r < rws.size(); ++r)
            for (const auto& e : rows[rws[r]]) rc[r].push_back(cl[e.first]);
        std::vector<int32_t> ro, co;
        order_component(rc, static_cast<int>(cls.size()), ro, co);
        for (int32_t r : ro) T.row_order.push_back(rws[r]);
        for (int32_t c : co) T.col_order.push_back(cls[c]);
    }
    const auto rpos = positions_of(T.row_order), cpos = positions_of(T.col_order);
    const int nt = N / 8;
    std::vector<std::map<int32_t, std::array<double, 64>>> acc(nt);
    for (int32_t r = 0; r < N; ++r)
        for (const auto& [c, v] : rows[r]) {
            const double re = static_cast<double>(v.real()), im = static_cast<double>(v.imag());
            if (re == 0.0 && im == 0.0) continue;
            const int rp = rpos[r], cp = cpos[c];
            auto it = acc[rp / 8].find(cp / 4);
            if (it == acc[rp / 8].end()) it = acc[rp / 8].emplace(cp / 4, std::array<double, 64>{}).first;
            const int lane = (rp % 8) * 4 + (cp % 4);  // lane l: n = l/4, k = l%4
            it->second[2 * lane] += re;
            it->second[2 * lane + 1] += im;
        }
    T.tiles.resize(nt);
    for (int m = 0; m < nt; ++m)
        for (auto& kv : acc[m]) T.tiles[m].emplace_back(kv.first, kv.second);
    return T;
}

// Block-diagonal operator (one diagonal block of size s3 per node): every
// node is tiled on its own, so units and k-tiles never straddle two nodes and
// the k-tiles of node q are exactly [q s3/4, (q+1) s3/4).
Tiling tile_rows_nodes(int N, const Rows& rows, int s3) {
    if (s3 >= N) return tile_rows(N, rows);
    Tiling T;
    T.tiles.resize(N / 8);
    for (int q = 0; q < N / s3; ++q) {
        const int off = q * s3;
        Rows sub(s3);
        for (int r = 0; r < s3; ++r)
            for (const auto& [c, v] : rows[off + r]) {
                if (c < off || c >= off + s3) throw FcctError(ST_INVALID_ARGUMENT, "tiling: operator is not block diagonal");
                sub[r].emplace_back(c - off, v);
            }
        const Tiling t = tile_rows(s3, sub);
        for (int32_t r : t.row_order) T.row_order.push_back(off + r);
        for (int32_t c : t.col_order) T.col_order.push_back(off + c);
        for (int m = 0; m < s3 / 8; ++m)
            for (const auto& [kt, vals] : t.tiles[m]) T.tiles[off / 8 + m].emplace_back(off / 4 + kt, vals);
    }
    return T;
}

// Proper 4-edge-colouring of a 4-regular bipartite multigraph given as edges
// (left, right); returns the colour of every edge. Peels 4 perfect matchings
// (each exists by König's theorem) found with Kuhn's augmenting paths.
std::vector<int> edge_colour4(int nleft, int nright, const std::vector<std::pair<int, int>>& edges) {
    const int E = static_cast<int>(edges.size());
    std::vector<int> colour(E, -1);
    for (int c = 0; c < 4; ++c) {
        std::vector<std::vector<int>> adj(nleft);
        for (int e = 0; e < E; ++e)
            if (colour[e] < 0) adj[edges[e].first].push_back(e);
        std::vector<int> match_r(nright, -1);  // right -> edge
        for (int l = 0; l < nleft; ++l) {
            std::vector<char> seen(nright, 0);
            std::function<bool(int)> aug = [&](int u) -> bool {
                for (int e : adj[u]) {
                    const int r = edges[e].second;
                    if (seen[r]) continue;
                    seen[r] = 1;
                    if (match_r[r] < 0 || aug(edges[match_r[r]].first)) {
                        match_r[r] = e;
                        return true;
                    }
                }
                return false;
            };
            if (!aug(l)) throw FcctError(ST_INVALID_ARGUMENT, "edge colouring: no perfect matching");
        }
        for (int r = 0; r < nright; ++r) colour[match_r[r]] = c;
    }
    return colour;
}

struct Logical {
    int kind = 0;
    Rows rows;                           // sparse
    std::vector<const PlanNode*> nodes;  // mix
    bool inverse = false;
    int s3 = 0;                          // points per node of this level
};

}  // namespace

bool compile_pipeline2(const PlanNode& root, bool inverse, const Shape2& shape, Pipeline2Host& out) {
    const int kWarps2 = shape.warps, kUnits2 = shape.units;
    if (!root.radix || root.n > 8) return false;
    std::vector<std::vector<const PlanNode*>> levels;
    std::vector<const PlanNode*> cur{&root};
    while (!cur.empty() && cur[0]->radix) {
        levels.push_back(cur);
        std::vector<const PlanNode*> next;
        for (const PlanNode* nd : cur)
            for (const auto& c : nd->children) next.push_back(c.get());
        cur = next;
    }
    if (cur.empty() || cur[0]->n != 1) return false;
    const int n = root.n;
    const int N = static_cast<int>(cube(n));
    if (N / 8 > kWarps2 * kUnits2) return false;
    const auto Z = stacked_order(root);

    auto sparse_level = [&](const std::vector<const PlanNode*>& lv, bool inv) {
        Logical L;
        L.kind = 0;
        L.rows.resize(N);
        const int64_t s3 = cube(lv[0]->n);
        L.s3 = static_cast<int>(s3);
        for (size_t q = 0; q < lv.size(); ++q) {
            const SparseLD& S = inv ? lv[q]->Binv : lv[q]->B;
            const int64_t off = static_cast<int64_t>(q) * s3;
            for (int64_t r = 0; r < s3; ++r)
                for (int64_t k = S.rowptr[r]; k < S.rowptr[r + 1]; ++k)
                    L.rows[off + r].emplace_back(static_cast<int32_t>(off + S.col[k]), S.val[k]);
        }
        return L;
    };
    auto mix_level = [&](const std::vector<const PlanNode*>& lv, bool inv) {
        Logical L;
        L.kind = 1;
        L.nodes = lv;
        L.inverse = inv;
        L.s3 = static_cast<int>(cube(lv[0]->n));
        return L;
    };
    std::vector<Logical> logical;
    if (!inverse) {
        for (auto& lv : levels) {
            if (!level_identity(lv, false)) logical.push_back(sparse_level(lv, false));
            logical.push_back(mix_level(lv, false));
        }
    } else {
        for (auto it = levels.rbegin(); it != levels.rend(); ++it) {
            logical.push_back(mix_level(*it, true));
            if (!level_identity(*it, true)) logical.push_back(sparse_level(*it, true));
        }
    }
    const int S = static_cast<int>(logical.size());
    // a stage is group-local when its level has more than one node (n > 2:
    // every node lies inside one root child)
    std::vector<char> local(S, 0);
    if (n >= 4)
        for (int s = 0; s < S; ++s) local[s] = logical[s].s3 * 8 <= N;

    // Units: for each stage, its units' 8 output positions and k-tiles' 4 input positions.
    std::vector<Tiling> tilings(S);
    std::vector<std::vector<std::array<int32_t, 8>>> unit_outs(S);  // positions
    std::vector<std::vector<std::array<int32_t, 4>>> ktiles(S);     // positions
    for (int s = 0; s < S; ++s) {
        auto& L = logical[s];
        if (L.kind == 0) {
            tilings[s] = tile_rows_nodes(N, L.rows, L.s3);
            const auto& T = tilings[s];
            for (int m = 0; m < N / 8; ++m) {
                std::array<int32_t, 8> o{};
                for (int i = 0; i < 8; ++i) o[i] = T.row_order[m * 8 + i];
                unit_outs[s].push_back(o);
            }
            for (int j = 0; j < N / 4; ++j) {
                std::array<int32_t, 4> k{};
                for (int i = 0; i < 4; ++i) k[i] = T.col_order[j * 4 + i];
                ktiles[s].push_back(k);
            }
        } else {
            const int s3 = static_cast<int>(cube(L.nodes[0]->n)), m3 = s3 / 8;
            for (size_t q = 0; q < L.nodes.size(); ++q)
                for (int h = 0; h < m3; ++h) {
                    std::array<int32_t, 8> o{};
                    std::array<int32_t, 4> k0{}, k1{};
                    for (int b = 0; b < 8; ++b) o[b] = static_cast<int32_t>(q) * s3 + b * m3 + h;
                    for (int g = 0; g < 4; ++g) {
                        k0[g] = static_cast<int32_t>(q) * s3 + g * m3 + h;
                        k1[g] = static_cast<int32_t>(q) * s3 + (g + 4) * m3 + h;
                    }
                    unit_outs[s].push_back(o);
                    ktiles[s].push_back(k0);
                    ktiles[s].push_back(k1);
                }
        }
    }
    // Layouts: lam[s][position] = slot at the input of stage s.
    std::vector<std::vector<int32_t>> lam(S + 1, std::vector<int32_t>(N));
    for (int i = 0; i < N; ++i) {
        lam[0][i] = inverse ? Z[i] : i;  // stacked i of the inverse input sits at Z(i)
        lam[S][i] = inverse ? i : Z[i];
    }
    for (int s = 1; s < S; ++s) {
        // edge (k-tile of stage s, half of a unit of stage s-1) per position
        std::vector<int> kt_of(N), half_of(N);
        for (size_t j = 0; j < ktiles[s].size(); ++j)
            for (int32_t p : ktiles[s][j]) kt_of[p] = static_cast<int>(j);
        for (size_t u = 0; u < unit_outs[s - 1].size(); ++u)
            for (int i = 0; i < 8; ++i) half_of[unit_outs[s - 1][u][i]] = static_cast<int>(2 * u + (i & 1));
        std::vector<std::pair<int, int>> edges(N);
        for (int p = 0; p < N; ++p) edges[p] = {kt_of[p], half_of[p]};
        const auto col = edge_colour4(static_cast<int>(ktiles[s].size()),
                                      static_cast<int>(2 * unit_outs[s - 1].size()), edges);
        for (int p = 0; p < N; ++p) lam[s][p] = 4 * kt_of[p] + col[p];
    }

    out = Pipeline2Host{};
    out.shape = shape;
    out.n = n;
    out.N = N;
    out.stride = 2 * N + 8;
    struct Entry {
        std::array<int32_t, 4> slots;
        std::array<double, 32> re, im;
        bool cplx;
    };
    for (int s = 0; s < S; ++s) {
        const auto& L = logical[s];
        Stage2Host st;
        st.n_units = static_cast<int>(unit_outs[s].size());
        std::vector<int64_t> cost(st.n_units, 0);
        for (int u = 0; u < st.n_units; ++u)
            for (int i = 0; i < 8; ++i) st.u_out.push_back(lam[s + 1][unit_outs[s][u][i]]);
        // Leaf-level mixes (one slice per node, a distinct K per unit) go
        // through the entry ring like sparse stages: their K tables would
        // otherwise stream from L2 with only one unit of prefetch.
        const bool leaf_mix = false && L.kind == 1 && L.nodes[0]->n == 2;  // measured slower than the mix path
        std::vector<std::vector<Entry>> uent(st.n_units);
        if (L.kind == 0) {
            const Tiling& T = tilings[s];
            for (int u = 0; u < st.n_units; ++u)
                for (const auto& [kt, vals] : T.tiles[u]) {
                    Entry e{};
                    e.cplx = false;
                    for (int l = 0; l < 32; ++l) {
                        e.re[l] = vals[2 * l];
                        e.im[l] = vals[2 * l + 1];
                        e.cplx |= e.im[l] != 0.0;
                    }
                    for (int k = 0; k < 4; ++k) e.slots[k] = lam[s][T.col_order[kt * 4 + k]];
                    uent[u].push_back(e);
                }
        } else if (leaf_mix) {
            for (size_t q = 0; q < L.nodes.size(); ++q) {
                const auto& Kq = L.inverse ? L.nodes[q]->Kinv : L.nodes[q]->K;
                for (int kt = 0; kt < 2; ++kt) {
                    Entry e{};
                    e.cplx = false;
                    for (int l = 0; l < 32; ++l) {
                        const int nn = l / 4, k = l % 4;  // T[k][n] = K[b = n][g = 4 kt + k]
                        e.re[l] = static_cast<double>(Kq[nn * 8 + kt * 4 + k].real());
                        e.im[l] = static_cast<double>(Kq[nn * 8 + kt * 4 + k].imag());
                        e.cplx |= e.im[l] != 0.0;
                    }
                    for (int k = 0; k < 4; ++k) e.slots[k] = lam[s][static_cast<int32_t>(q) * 8 + kt * 4 + k];
                    uent[q].push_back(e);
                }
            }
        }
        if (L.kind == 0 || leaf_mix) {
            st.kind = 0;
            for (int u = 0; u < st.n_units; ++u)
                for (const auto& e : uent[u]) {
                    cost[u] += e.cplx ? 2 : 1;
                    st.dmma_per_tile += (shape.tb / 4) * (e.cplx ? 2 : 1);
                }
        } else {
            st.kind = 1;
            const int s3 = static_cast<int>(cube(L.nodes[0]->n)), m3 = s3 / 8;
            for (size_t q = 0; q < L.nodes.size(); ++q) {
                const auto& Kq = L.inverse ? L.nodes[q]->Kinv : L.nodes[q]->K;
                for (int i = 0; i < 64; ++i) {
                    st.K.push_back(static_cast<double>(Kq[i].real()));
                    st.K.push_back(static_cast<double>(Kq[i].imag()));
                }
                for (int h = 0; h < m3; ++h) {
                    st.u_node.push_back(static_cast<int32_t>(q));
                    for (int g = 0; g < 8; ++g)
                        st.u_in.push_back(lam[s][static_cast<int32_t>(q) * s3 + g * m3 + h]);
                }
            }
            for (int u = 0; u < st.n_units; ++u) cost[u] = 4;
            st.dmma_per_tile += static_cast<int64_t>(st.n_units) * 4 * (shape.tb / 4);
        }
        // LPT assignment of units to warps, at most kUnits2 per warp. In a
        // group-local stage (a level below the root: every unit lives inside
        // one root child's N/8 positions) the units of child c go to warp
        // group c only, so the group can run the stage on its own barrier.
        std::vector<int32_t> order(st.n_units);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
        st.warp_units.assign(kWarps2 * kUnits2, -1);
        std::vector<int64_t> load(kWarps2, 0);
        std::vector<int> cnt(kWarps2, 0);
        const bool grouped = local[s] && kWarps2 % 8 == 0;
        const int wpg = kWarps2 / 8;
        for (int32_t u : order) {
            int best = -1;
            const int g = unit_outs[s][u][0] / (N / 8);
            for (int w = 0; w < kWarps2; ++w) {
                if (grouped && w / wpg != g) continue;
                if (cnt[w] < kUnits2 && (best < 0 || load[w] < load[best])) best = w;
            }
            if (best < 0) return false;
            st.warp_units[best * kUnits2 + cnt[best]++] = u;
            load[best] += cost[u];
        }
        // barrier scope between compute and store (sync_mid) and after the
        // store (sync_end): a warp group suffices when the group's inputs and
        // outputs stay inside its own slot range [c N/8, (c+1) N/8)
        const bool in_closed = grouped && s >= 1;
        const bool out_closed = grouped && s + 1 <= S - 1 && local[s + 1];
        st.sync_mid = (in_closed && out_closed) ? 1 : 0;
        st.sync_end = out_closed ? 1 : 0;
        if (st.kind == 0) {
            st.w_base.assign(kWarps2 + 1, 0);
            st.w_count.assign(kWarps2 * kUnits2, 0);
            st.w_ccount.assign(kWarps2 * kUnits2, 0);
            st.w_cplx.assign(kWarps2 * 4, 0u);
            int32_t flat = 0;
            for (int w = 0; w < kWarps2; ++w) {
                st.w_base[w] = flat;
                for (int j = 0; j < kUnits2; ++j) {
                    const int u = st.warp_units[w * kUnits2 + j];
                    if (u < 0) continue;
                    st.w_count[w * kUnits2 + j] = static_cast<int32_t>(uent[u].size());
                    // real tiles first, complex after: the kernel runs one
                    // branch-free loop for each kind
                    std::stable_sort(uent[u].begin(), uent[u].end(),
                                     [](const Entry& a, const Entry& b) { return a.cplx < b.cplx; });
                    int32_t nc = 0;
                    for (const auto& e : uent[u]) nc += e.cplx ? 1 : 0;
                    st.w_ccount[w * kUnits2 + j] = nc;
                    for (const auto& e : uent[u]) {
                        for (int k = 0; k < 4; ++k) st.e_slots.push_back(e.slots[k] | (e.cplx ? (1 << 30) : 0));
                        st.e_re.insert(st.e_re.end(), e.re.begin(), e.re.end());
                        st.e_im.insert(st.e_im.end(), e.im.begin(), e.im.end());
                        const int fw = flat - st.w_base[w];
                        if (fw >= 128) return false;
                        if (e.cplx) st.w_cplx[w * 4 + fw / 32] |= 1u << (fw % 32);
                        ++flat;
                    }
                }
            }
            st.w_base[kWarps2] = flat;
        }
        out.dmma_per_tile += st.dmma_per_tile;
        out.stages.push_back(std::move(st));
    }
    out.shift_in = logical.front().kind == 1 ? 1 : 0;
    out.shift_out = logical.back().kind == 1 ? 1 : 0;
    return true;
}

}  // namespace fcct
