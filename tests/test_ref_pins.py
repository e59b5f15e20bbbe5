"""Pins the oracle to the REFERENCE'S OWN code, not only to its known answers.

oracle/_ref/libfcct_ref.so is built in place from the reference's Eigen-free
sources (/root/reference/proj/src/{weyl_s4,chebyshev,spectral}.cpp, recipe
oracle/ref.mk). They hold the group (weyl_s4.cpp:54-92), the node set
(spectral.cpp:155-171 with TorusPoint::wrapped, chebyshev.cpp:30-46,76-85) and
the Chebyshev evaluation (cheb_eval_uvw, chebyshev.cpp:67-74) that every entry
of D_n is made of. transform.cpp itself needs Eigen3 (absent), so the matrix is
compared entry by entry: D[i, kappa] = cheb_eval_uvw(kappa, uvw_i).

Skipped where /root/reference is absent (the GPU box); tests/golden/
ref_golden.npz carries the same reference outputs there.
"""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="reference sources absent")

PSETS = [(0.125, 0.0, 0.375), (0.21, 0.055, 0.4), (0.37, 0.61, 0.085)]


@pytest.fixture(scope="module")
def R(oracle_mod):
    oracle.build_ref()
    return oracle.Ref


def test_group_bit_exact(R):
    assert np.array_equal(R.group(), oracle.group())


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("p", PSETS)
def test_skew_nodes_bit_exact(R, n, p):
    assert np.array_equal(R.skew_nodes(n, p), oracle.skew_nodes(n, p))


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_common_zeros_bit_exact(R, n):
    assert np.array_equal(R.common_zeros(n), oracle.common_zeros(n))


def test_degenerate_nodes_agree(R):
    # DegenerateNodes (spectral.cpp:26-43) fires for the same grids
    for n, p in [(2, (0.0, 0.0, 0.0)), (4, (0.3, 0.1, 0.7)), (8, (0.0, 0.0, 0.0))]:
        with pytest.raises(oracle.OracleError) as a:
            R.skew_nodes(n, p)
        with pytest.raises(oracle.OracleError) as b:
            oracle.skew_nodes(n, p)
        assert a.value.code == b.value.code == 4


def test_cheb_eval_uvw_off_torus(R):
    rng = np.random.default_rng(7)
    for _ in range(50):
        k = rng.integers(-3, 6, 3)
        uvw = rng.uniform(0.6, 1.4, 3) * np.exp(2j * np.pi * rng.uniform(0, 1, 3))
        a, b = R.cheb_eval_uvw(k, uvw), oracle.cheb_eval_uvw(k, uvw)
        assert a == b  # same Laurent sum, same ipow, same order


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("p", PSETS)
def test_dense_matrix_matches_reference_evaluation(R, n, p):
    """The oracle's ColumnEvaluator restatement (axis tables) against the
    reference's own per-entry Laurent evaluation: max |diff| <= 1e-14 (the
    reference's ipow route carries ~5e-15 of rounding at n = 8; the long-double
    oracle D sits within the same distance)."""
    N = n**3
    D_ref = R.dense_columns(n, p, 0, N)
    assert np.abs(D_ref - oracle.dense_transform(n, p)).max() <= 1e-14
    assert np.abs(D_ref - oracle.dense_transform(n, p, ext=True)).max() <= 1e-14


def test_dense_rows_match_reference_columns_n16(R):
    """The long-double row oracle (used for n = 16 GPU parity) against the
    reference's evaluation of D_16 on 8 columns: e_kappa inputs pick columns."""
    n, p = 16, PSETS[0]
    cols = np.array([0, 1, 16, 256, 1234, 3000, 4095])
    D_ref = np.stack([R.dense_columns(n, p, int(c), int(c) + 1)[:, 0] for c in cols], axis=1)
    rows = np.arange(0, n**3, 13)
    E = np.zeros((len(cols), n**3), dtype=np.complex128)
    E[np.arange(len(cols)), cols] = 1.0
    got = oracle.dense_rows(n, p, rows, E)  # [len(cols), len(rows)]
    assert np.abs(got.T - D_ref[rows]).max() <= 1e-13


def test_real_coords_and_child_and_encode(R):
    from paper_1807_10058_b200 import SkewParams, encode_param

    p = PSETS[0]
    nodes = oracle.skew_nodes(8, p)
    x, y, z = nodes[:, 3], nodes[:, 4], nodes[:, 5]
    mine = np.stack([(0.5 * (x + z)).real, y.real, ((x - z) / 2j).real], axis=1)
    assert np.abs(R.real_coords(8, p) - mine).max() <= 1e-15
    for q in PSETS:
        for c in range(8):
            ir, is_, it = c >> 2, (c >> 1) & 1, c & 1
            ch = SkewParams(*q).child(ir, is_, it)
            assert R.child(q, ir, is_, it) == (ch.r, ch.s, ch.t)
    for v in [0.0, 0.125, 0.375, 1 / 3, 0.21, 0.055, -0.5, 1e-7, 0.1 + 0.2, 5.0, 0.0625, 7 / 1024, 2.0 / 3.0]:
        assert R.encode_param(v) == encode_param(v), v


def test_golden_fixture_is_the_live_reference_output(R):
    """tests/golden/ref_golden.npz (read by the GPU tests) still equals what
    the reference computes here."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    import make_ref_golden

    frozen = np.load(Path(__file__).resolve().parent / "golden" / "ref_golden.npz")
    live = make_ref_golden.build()
    assert sorted(frozen.files) == sorted(live)
    for k in live:
        assert np.array_equal(frozen[k], live[k]), k
