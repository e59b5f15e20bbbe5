"""CPU tests of the product's host side (no GPU): the C-ABI library loads and
exports every symbol include/fcct_gpu.h declares, the exact orbit-structured
plan derivation reproduces the reference's factor, the compiled DMMA stage
tables (emulated on the host exactly as the kernel indexes them) reproduce the
oracle, and the API-level helpers behave like the reference's.
"""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle
from paper_1807_10058_b200 import (
    OddSize,
    SkewParams,
    basis_change,
    encode_param,
    parse_param,
    parse_params,
    plan_tree_stats,
    shard_range,
)
from paper_1807_10058_b200 import _capi

ROOT = Path(__file__).resolve().parents[1]
CANON = SkewParams.canonical()
P2 = SkewParams(0.21, 0.055, 0.4)


def test_library_exports_header_symbols():
    L = _capi.lib()
    header = (ROOT / "include" / "fcct_gpu.h").read_text()
    declared = set(re.findall(r"\b(fcct_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    assert set(_capi.HEADER_SYMBOLS) == declared
    for sym in declared:
        assert hasattr(L, sym), sym


@pytest.mark.parametrize("n", [4, 8])
@pytest.mark.parametrize("p", [CANON, P2, SkewParams(0.37, 0.61, 0.085)])
def test_exact_basis_matches_reference_derivation(n, p):
    B = basis_change(n, p).to_dense()
    ref = oracle.RefPlan(n, (p.r, p.s, p.t)).basis_dense()
    # same sparsity (the reference prunes its noise at 1e-12) and values within
    # the reference derivation's own noise
    assert np.array_equal(np.abs(B) > 0, np.abs(ref) > 1e-9)
    assert np.abs(B - ref).max() < 1e-9


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_basis_times_inverse_is_identity(n):
    B = basis_change(n, CANON)
    Bi = basis_change(n, CANON, inverse=True)
    import scipy.sparse as sp

    def csc(m):
        return sp.csc_matrix((m.values, m.rowidx, m.colptr), shape=(m.rows, m.cols))

    prod = (csc(B) @ csc(Bi)).toarray()
    assert np.abs(prod - np.eye(n**3)).max() < 1e-13


def test_tree_statistics_and_flops():
    # tree nnz 245 / 5,550 / 82,724 and flops 10,152 / 142,704 / 1,710,368
    for n, nnz, flops in ((4, 245, 10152), (8, 5550, 142704), (16, 82724, 1710368)):
        st = plan_tree_stats(n, CANON)
        assert st["tree_nnz"] == nnz
        assert st["flops_forward"] == flops
    assert basis_change(2, CANON).nonZeros() == 8
    with pytest.raises(OddSize):
        basis_change(3, CANON)


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("p", [CANON, P2])
def test_compiled_dmma_tables_emulated(n, p):
    L = _capi.lib()
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, (3, n**3)) + 1j * rng.uniform(-1, 1, (3, n**3))
    y = np.zeros_like(x)
    pt = (p.r, p.s, p.t)
    assert L.fcct_debug_emulate_v2(n, *pt, 0, x.ctypes.data, y.ctypes.data, 3) == 0
    yr = oracle.forward_dense(n, pt, x)
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < 1e-12
    xi = np.zeros_like(x)
    assert L.fcct_debug_emulate_v2(n, *pt, 1, yr.ctypes.data, xi.ctypes.data, 3) == 0
    xr = oracle.inverse_dense(n, pt, yr)
    assert np.linalg.norm(xi - xr) / np.linalg.norm(xr) < 1e-12


@pytest.mark.parametrize("n", [4, 8])
@pytest.mark.parametrize("p", [CANON, P2])
def test_orbit_fft_tables_emulated(n, p):
    """The orbit-FFT executor's compiled tables (register-resident DMMA tiles of
    S_n(p) / S_n(p)^{-1} n^-3, swizzled FFT positions), emulated on the host as
    the kernel indexes them, then the radix-2 FFT: D_n(p) = F_n S_n(p) against
    the long-double dense oracle, both directions."""
    L = _capi.lib()
    rng = np.random.default_rng(10 + n)
    x = rng.uniform(-1, 1, (3, n**3)) + 1j * rng.uniform(-1, 1, (3, n**3))
    y = np.zeros_like(x)
    pt = (p.r, p.s, p.t)
    assert L.fcct_debug_emulate_orbit_fft(n, *pt, 0, x.ctypes.data, y.ctypes.data, 3) == 0
    yr = oracle.forward_dense(n, pt, x)
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < 1e-13
    xi = np.zeros_like(x)
    assert L.fcct_debug_emulate_orbit_fft(n, *pt, 1, yr.ctypes.data, xi.ctypes.data, 3) == 0
    xr = oracle.inverse_dense(n, pt, yr)
    assert np.linalg.norm(xi - xr) / np.linalg.norm(xr) < 1e-13


@pytest.mark.parametrize("p", [CANON, P2])
def test_orbit16_tables_emulated(p):
    """The two-pass orbit-FFT executor (n = 16): chunked orbit-block tables of
    pass A emulated as the kernel indexes them (gather slots, per-warp tiles,
    chain ends, natural output positions) plus the cube FFT, against the FFT /
    orbit-route oracle (the n = 16 dense oracle is too slow for a CPU test)."""
    n = 16
    L = _capi.lib()
    rng = np.random.default_rng(16)
    x = rng.uniform(-1, 1, (2, n**3)) + 1j * rng.uniform(-1, 1, (2, n**3))
    pt = (p.r, p.s, p.t)
    route = oracle.OrbitRoute(n, pt)
    y = np.zeros_like(x)
    assert L.fcct_debug_emulate_orbit16(n, *pt, 0, x.ctypes.data, y.ctypes.data, 2) == 0
    yr = route.forward(x)
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < 1e-13
    xi = np.zeros_like(x)
    assert L.fcct_debug_emulate_orbit16(n, *pt, 1, yr.ctypes.data, xi.ctypes.data, 2) == 0
    assert np.linalg.norm(xi - x) / np.linalg.norm(x) < 1e-13


@pytest.mark.parametrize("p", [CANON, P2])
def test_orbit_pat_tables_emulated(p):
    """The single-pass orbit-pattern executor (n = 16): the orbit blocks fall into
    8 shapes for any offsets; the two big ones (all 112 free orbits share ONE
    24 x 24 operator, 105 of the 108 twelve-member orbits another) are emulated as
    the kernel indexes its fragment tables (8 orbits per DMMA tile, Lambda in
    fragment order, in-place slots), the rare ones as SIMT rows, plus the cube
    FFT; against the FFT / orbit-route oracle."""
    import ctypes

    n = 16
    L = _capi.lib()
    rng = np.random.default_rng(161)
    x = rng.uniform(-1, 1, (2, n**3)) + 1j * rng.uniform(-1, 1, (2, n**3))
    pt = (p.r, p.s, p.t)
    route = oracle.OrbitRoute(n, pt)
    y = np.zeros_like(x)
    st = (ctypes.c_int64 * 6)()
    assert L.fcct_debug_emulate_orbit_pat(n, *pt, 0, x.ctypes.data, y.ctypes.data, 2, st) == 0
    assert list(st)[:4] == [8, 112, 105, 14 * 72 + 14 * 24]
    assert st[5] <= st[4] <= 4 * st[5]  # modelled gather / scatter wavefronts vs their floor
    yr = route.forward(x)
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < 1e-13
    xi = np.zeros_like(x)
    assert L.fcct_debug_emulate_orbit_pat(n, *pt, 1, yr.ctypes.data, xi.ctypes.data, 2, None) == 0
    assert np.linalg.norm(xi - x) / np.linalg.norm(x) < 1e-13


@pytest.mark.parametrize("n,expect", [(8, {1: [1], 3: [1], 4: [7], 6: [3, 1], 12: [21, 1], 24: [8]}),
                                      (16, {1: [1], 3: [1], 4: [15], 6: [7, 1], 12: [105, 3], 24: [112]})])
def test_orbit_block_shapes_from_the_group_alone(n, expect):
    """The structural fact the orbit-pattern executors rest on, checked without any of
    the product's code: built from the oracle's group table with numpy, the orbit
    blocks of S_n(p) — members in group order from the smallest member, the reduced
    index's phase divided out — coincide in 8 matrices, all free orbits in ONE, for
    canonical and generic offsets (tools/orbit_shapes.py)."""
    import importlib.util
    from pathlib import Path

    spec = importlib.util.spec_from_file_location("orbit_shapes", Path(__file__).resolve().parents[1] / "tools" / "orbit_shapes.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    for p in (CANON, P2):
        assert mod.summary(n, (p.r, p.s, p.t)) == expect


def test_orbit_pat_tables_emulated_n32():
    """The same pattern tables drive the large-n S pass (n = 32, 64: one warp per
    tile of 8 orbits gathering from global memory): 1,120 free orbits on one
    operator, 465 of the 472 twelve-member orbits on another, emulated at n = 32."""
    import ctypes

    n = 32
    L = _capi.lib()
    rng = np.random.default_rng(321)
    x = rng.uniform(-1, 1, (1, n**3)) + 1j * rng.uniform(-1, 1, (1, n**3))
    pt = (P2.r, P2.s, P2.t)
    route = oracle.OrbitRoute(n, pt)
    y = np.zeros_like(x)
    st = (ctypes.c_int64 * 6)()
    assert L.fcct_debug_emulate_orbit_pat(n, *pt, 0, x.ctypes.data, y.ctypes.data, 1, st) == 0
    assert list(st)[:3] == [8, 1120, 465]
    yr = route.forward(x)
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < 1e-13
    xi = np.zeros_like(x)
    assert L.fcct_debug_emulate_orbit_pat(n, *pt, 1, yr.ctypes.data, xi.ctypes.data, 1, None) == 0
    assert np.linalg.norm(xi - x) / np.linalg.norm(x) < 1e-13


@pytest.mark.parametrize("p", [CANON, P2])
def test_orbit_big_tables_emulated(p):
    """The large-n orbit-FFT executor (n = 32): column-major orbit-block rows of
    S_n(p) / S_n(p)^{-1} n^-3 emulated as the kernel indexes them, plus the three
    axis DFTs, against the FFT / orbit-route oracle."""
    n = 32
    L = _capi.lib()
    x = np.random.default_rng(32).uniform(-1, 1, (1, n**3)) + 1j * np.random.default_rng(33).uniform(-1, 1, (1, n**3))
    pt = (p.r, p.s, p.t)
    route = oracle.OrbitRoute(n, pt)
    y = np.zeros_like(x)
    assert L.fcct_debug_emulate_orbit_big(n, *pt, 0, x.ctypes.data, y.ctypes.data, 1) == 0
    yr = route.forward(x)
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < 1e-13
    xi = np.zeros_like(x)
    assert L.fcct_debug_emulate_orbit_big(n, *pt, 1, yr.ctypes.data, xi.ctypes.data, 1) == 0
    assert np.linalg.norm(xi - x) / np.linalg.norm(x) < 1e-13


def test_compiled_layouts_are_conflict_free_inside():
    # Only the first stage (natural layout from the TMA load) and the last stage
    # (natural output layout) may see shared-memory bank conflicts.
    L = _capi.lib()
    st = (ctypes.c_int64 * 6)()
    assert L.fcct_debug_v2_stats(8, 0.125, 0.0, 0.375, 0, st) == 0
    ld_req, ld_conf, st_req, st_conf, dmma, nstages = list(st)
    assert nstages == 5
    assert st_conf <= (8**3 // 8) * 2 * 2  # last stage's store requests only
    assert ld_conf < ld_req // 2


def test_param_text_round_trips():
    # test_spectral.cpp:153-175
    assert encode_param(0.125) == "1/8"
    assert encode_param(0.0) == "0"
    assert encode_param(0.375) == "3/8"
    assert parse_param("1/8") == 0.125
    assert parse_param("-3/4") == -0.75
    for bad in ("1/8/9", "abc", ""):
        with pytest.raises(ValueError):
            parse_param(bad)
    for v in (0.125, 0.0, 0.375, 0.3141592653589793, 1.0 / 3.0):
        assert parse_param(encode_param(v)) == v
    p = parse_params("1/8,0,3/8")
    assert p == CANON and p.encode() == "1/8,0,3/8"
    for bad in ("1,2", "1,2,3,4"):
        with pytest.raises(ValueError):
            parse_params(bad)
    c = CANON.child(1, 0, 1)
    assert (c.r, c.s, c.t) == ((0.125 + 1) / 2, 0.0, (0.375 + 1) / 2)


def test_shard_ranges_cover_batch():
    for total in (0, 1, 7, 65536, 185193):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(total, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and a <= b
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_errors_without_gpu():
    L = _capi.lib()
    nnz = ctypes.c_int64()
    assert L.fcct_basis_change(3, 0.125, 0.0, 0.375, 0, ctypes.byref(nnz), None, None, None) == _capi.ODD_SIZE
    assert L.fcct_basis_change(2, 0.0, 0.0, 0.0, 0, ctypes.byref(nnz), None, None, None) == _capi.DEGENERATE_NODES
    assert "same spectral point" in L.fcct_last_error().decode()
