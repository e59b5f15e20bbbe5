"""Pins the CPU oracle (oracle/fcct_oracle.cpp + oracle/oracle.py) against the
reference's own known-answer tests. The reference cannot be built here (no
Eigen3 / doctest), so these checks are what make the oracle
trustworthy as the parity checker. Each test cites the reference test it
restates.
"""
import itertools
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle

GOLD = Path(__file__).resolve().parent / "golden"
CANON = (0.125, 0.0, 0.375)


def test_group_matches_reference_table():
    # test_weyl_s4.cpp:38-45,74-84: closes to 24, identity first, equals the expected set
    G = oracle.group()
    assert G.shape == (24, 3, 3)
    assert np.array_equal(G[0], np.eye(3, dtype=np.int32))
    exp = json.loads((GOLD / "weyl_s4_expected.json").read_text())["elements"]
    assert {tuple(m.flatten()) for m in G} == {tuple(e) for e in exp}
    assert len({tuple(m.flatten()) for m in G}) == 24


def test_generator_relations():
    # test_weyl_s4.cpp:47-58 (the code's relations, not the paper's)
    gens = [np.array(g).reshape(3, 3) for g in ([-1, 0, 0, 1, 1, 0, 0, 0, 1], [1, 1, 0, 0, -1, 0, 0, 1, 1],
                                                [1, 0, 0, 0, 1, 1, 0, 0, -1])]
    eye = np.eye(3, dtype=int)
    for s in gens:
        assert np.array_equal(s @ s, eye)
    mp = np.linalg.matrix_power
    assert np.array_equal(mp(gens[0] @ gens[1], 3), eye)
    assert np.array_equal(mp(gens[0] @ gens[2], 2), eye)
    assert np.array_equal(mp(gens[1] @ gens[2], 3), eye)
    assert not np.array_equal(mp(gens[0] @ gens[1], 2), eye)
    assert not np.array_equal(mp(gens[1] @ gens[2], 2), eye)
    G = oracle.group()
    for a in G:
        assert round(abs(np.linalg.det(a))) == 1 and np.abs(a).max() <= 1
        assert any(np.array_equal(a @ b, eye) for b in G)


def _orbit(k, G):
    return sorted({tuple(int(v) for v in w @ np.array(k)) for w in G})


def test_orbit_sizes_and_canonical_index():
    # test_weyl_s4.cpp:86-124
    G = oracle.group()
    sizes = {(0, 0, 0): 1, (1, 0, 0): 4, (0, 1, 0): 6, (0, 0, 1): 4, (2, 1, 0): 12, (1, 1, 0): 12, (1, 1, 1): 24}
    for k, sz in sizes.items():
        assert len(_orbit(k, G)) == sz
    assert _orbit((1, 0, 0), G) == [(-1, 1, 0), (0, -1, 1), (0, 0, -1), (1, 0, 0)]
    canon = lambda k: max(_orbit(k, G))  # noqa: E731
    assert canon((1, 0, 0)) == (1, 0, 0)
    assert canon((0, 1, 0)) == (1, 0, -1)
    assert canon((0, 0, 1)) == (1, -1, 0)
    # 14 shift vectors (test_spectral.cpp:138-151)
    shifts = set()
    for e in ((1, 0, 0), (0, 1, 0), (0, 0, 1)):
        shifts |= set(_orbit(e, G))
    assert len(shifts) == 14
    assert all(tuple(-v for v in s) in shifts for s in shifts)


def test_radix_permutation_known_answers():
    # test_transform.cpp:88-108
    with pytest.raises(oracle.OracleError):
        oracle.radix_permutation(3)
    with pytest.raises(oracle.OracleError):
        oracle.radix_permutation(0)
    assert np.array_equal(oracle.radix_permutation(2), np.arange(8))
    p4 = oracle.radix_permutation(4)
    assert sorted(p4.tolist()) == list(range(64))
    assert p4[5 * 8 + 6] == (3 * 4 + 2) * 4 + 1
    assert np.array_equal(p4, np.load(GOLD / "vectors.npz")["perm4"])


def test_dense_known_columns():
    # test_transform.cpp:42-72
    D1 = oracle.dense_transform(1, CANON)
    assert abs(D1[0, 0] - 1.0) < 1e-15
    n = 4
    D = oracle.dense_transform(n, CANON)
    nodes = oracle.skew_nodes(n, CANON)
    assert np.abs(D[:, 0] - 1.0).max() < 1e-12
    col_y = (0 * n + 1) * n + 0
    assert np.abs(D[:, col_y] - nodes[:, 4]).max() < 1e-12
    delta = np.zeros(n**3, complex)
    delta[0] = 1
    assert np.abs(D @ delta - 1.0).max() < 1e-12


def test_dense_vs_brute_force_entries():
    # test_transform.cpp:74-86: n = 3, seed 5, nodes {0,1,7,13,26}, 1e-11
    n = 3
    x = oracle.random_signal(n, 5)
    q = oracle.dense_transform(n, CANON) @ x
    nodes = oracle.skew_nodes(n, CANON)
    for node in (0, 1, 7, 13, 26):
        acc = 0j
        for j, k, p in itertools.product(range(n), repeat=3):
            c = x[(j * n + k) * n + p]
            acc += c * oracle.cheb_eval_uvw((j, k, p), nodes[node, :3])
        assert abs(q[node] - acc) < 1e-11


def test_nodes_common_zeros_nesting_and_degeneracy():
    # test_spectral.cpp:56-67 (residual), 84-95 (skew == common zeros), 108-136
    for n in (1, 2, 3, 4, 8):
        cz = oracle.common_zeros(n)
        assert cz.shape == (n**3, 6)
        worst = 0.0
        for node in cz:
            for k in ((n, 0, 0), (0, n, 0), (0, 0, n)):
                worst = max(worst, abs(oracle.cheb_eval_uvw(k, node[:3])))
        assert worst < 1e-10
    for n in (1, 2, 4):
        a = oracle.common_zeros(n)
        b = oracle.skew_nodes(n, CANON)
        assert np.abs(a[:, :3] - b[:, :3]).max() < 1e-12
    for n in (2, 4):
        big = oracle.skew_nodes(n, CANON)
        m = n // 2
        for ir, is_, it in itertools.product(range(2), repeat=3):
            cp = ((CANON[0] + ir) / 2, (CANON[1] + is_) / 2, (CANON[2] + it) / 2)
            child = oracle.skew_nodes(m, cp)
            for i, j, k in itertools.product(range(m), repeat=3):
                c = child[(i * m + j) * m + k, :3]
                p = big[((ir + 2 * i) * n + (is_ + 2 * j)) * n + (it + 2 * k), :3]
                assert np.abs(c - p).max() < 1e-12
    with pytest.raises(oracle.OracleError) as e:
        oracle.skew_nodes(2, (0.0, 0.0, 0.0))
    assert e.value.code == 4  # DEGENERATE_NODES
    # real coordinates are pairwise distinct at n = 8 (test_spectral.cpp:97-106)
    nodes = oracle.common_zeros(8)
    x, y, z = nodes[:, 3], nodes[:, 4], nodes[:, 5]
    rc = np.stack([(0.5 * (x + z)).real, y.real, ((x - z) / 2j).real], axis=1)
    assert len({tuple(np.round(r * 1e6).astype(np.int64)) for r in rc}) == 512


def test_basis_change_known_answers():
    # B_2 == I with nnz 8 (test_transform.cpp:110-118); nnz(B_4) = 245,
    # nnz(B_8) = 3438 and tree nnz 5550 (noise-free counts)
    p2 = oracle.RefPlan(2, CANON)
    assert p2.basis_nnz() == 8
    assert np.abs(p2.basis_dense() - np.eye(8)).max() < 1e-12
    p4 = oracle.RefPlan(4, CANON)
    assert p4.basis_nnz() == 245
    assert np.abs(p4.basis_dense() - np.load(GOLD / "vectors.npz")["B4_ref"]).max() == 0.0
    p8 = oracle.RefPlan(8, CANON)
    assert p8.basis_nnz() == 3438
    assert p8.tree_nnz() == 5550
    # nnz/n^3 growth 4 -> 8 stays below 4x (acceptance/main.cpp:454-467)
    assert (3438 / 512) / (245 / 64) <= 4.0


@pytest.mark.parametrize("n", [2, 4, 8])
def test_fast_vs_naive_and_round_trip(n):
    # test_transform.cpp:138-151 (seeds 40+n, 1e-10), 166-183 (seeds 90+n, 1e-8)
    plan = oracle.RefPlan(n, CANON)
    D = oracle.dense_transform(n, CANON)
    x = oracle.random_signal(n, 40 + n)
    slow = D @ x
    fast = plan.apply(x)
    assert np.abs(fast - slow).max() / np.abs(slow).max() < 1e-10
    s = oracle.random_signal(n, 90 + n)
    q = plan.apply(s)
    back = plan.solve(q)
    assert np.abs(back - s).max() / np.abs(s).max() < 1e-8
    again = plan.apply(plan.solve(q))
    assert np.abs(again - q).max() / np.abs(q).max() < 1e-8


def test_factorization_residual():
    # test_transform.cpp:120-136 and acceptance #6 (main.cpp:325-348)
    for n in (2, 4):
        assert oracle.RefPlan(n, CANON).factorization_residual() < 1e-9
    for p in (CANON, (0.21, 0.055, 0.4), (0.37, 0.61, 0.085)):
        assert oracle.RefPlan(4, p).factorization_residual() < 1e-9
        assert oracle.RefPlan(8, p).factorization_residual() < 1e-9


def test_odd_size_direct_plan():
    # test_transform.cpp:185-195
    plan = oracle.RefPlan(3, CANON)
    assert oracle.lib().oracle_plan_kind(plan.h) == 0
    s = oracle.random_signal(3, 13)
    q = plan.apply(s)
    assert np.abs(q - oracle.dense_transform(3, CANON) @ s).max() < 1e-10
    assert np.abs(plan.solve(q) - s).max() < 1e-8


def test_condition_estimator():
    # test_transform.cpp:222-232
    well = 2.0 * np.eye(6)
    assert abs(oracle.condition_estimate_matrix(well) - 1.0) <= 0.5
    sick = np.eye(6)
    sick[5, 5] = 1e-14
    assert oracle.condition_estimate_matrix(sick) > 1e12


def test_long_double_dense_oracle_matches_fp64_dense():
    for n in (2, 4, 8):
        x = oracle.random_signal(n, 7)
        y = oracle.forward_dense(n, CANON, x)
        y64 = oracle.dense_transform(n, CANON) @ x
        assert np.linalg.norm(y - y64) / np.linalg.norm(y) < 2e-15
        xb = oracle.inverse_dense(n, CANON, y)
        assert np.linalg.norm(xb - x) / np.linalg.norm(x) < 1e-14


def test_golden_vectors_frozen():
    g = np.load(GOLD / "vectors.npz")
    for n, seed in ((4, 44), (8, 48)):
        x = oracle.random_signal(n, seed)
        assert np.array_equal(x, g[f"x_n{n}"])  # libstdc++ mt19937 stream reproduced
        y = oracle.forward_dense(n, CANON, x)
        assert np.abs(y - g[f"y_n{n}"]).max() <= 1e-14 * np.abs(y).max()


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_orbit_route_oracle(n):
    # FFT / orbit route (oracle for n >= 16) agrees with the dense oracle
    p = CANON if n != 4 else (0.21, 0.055, 0.4)
    route = oracle.OrbitRoute(n, p)
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, (2, n**3)) + 1j * rng.uniform(-1, 1, (2, n**3))
    y = route.forward(x)
    if n <= 8:
        yd = oracle.forward_dense(n, p, x)
        assert np.linalg.norm(y - yd) / np.linalg.norm(yd) < 1e-14
    else:
        nodes = rng.integers(0, n**3, 16)
        direct = oracle.symmetrized_rows(n, p, nodes, x[0])
        assert np.linalg.norm(y[0, nodes] - direct) / np.linalg.norm(direct) < 1e-13
    xb = route.inverse(y)
    assert np.linalg.norm(xb - x) / np.linalg.norm(x) < 1e-13
