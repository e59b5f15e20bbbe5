"""The reference's condition estimate (condition_with_lu, transform.cpp:91-111)
and where IllConditioned is raised on it (require_condition, :113-117).

The product computes the estimate of D_n(p) without forming D (plan.cpp
reference_condition: exact ||D||_1 column by column, the eight probes solved as
S^{-1} F^{-1} v). The oracle runs the reference's own recipe on the dense matrix
(partial-pivot LU solves against the same mt19937(12345) probes), so the two
must agree to rounding. No GPU needed: the column norms run on the host here.
"""
import numpy as np
import pytest

from paper_1807_10058_b200 import DegenerateNodes, SkewParams, condition_estimate_1norm

PSETS = [(0.125, 0.0, 0.375), (0.1, 0.27, 0.61), (0.3, 0.05, 0.9)]
N16_CANON_HOST = 25622.451093811218


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8])
@pytest.mark.parametrize("p", PSETS)
def test_estimate_matches_reference_recipe(oracle_mod, n, p):
    got = condition_estimate_1norm(n, SkewParams(*p))
    want = oracle_mod.condition_estimate_matrix(oracle_mod.dense_transform(n, p))
    assert abs(got - want) <= 1e-12 * want


def test_estimate_grows_towards_degenerate_grids():
    """cond(D_4) ~ 4.2 / delta as the offsets approach the degenerate (1/4, 1/4, 1/4)
    grid; the degeneracy scan (spectral.cpp:26-43) stops it before 1e12 at n = 4."""
    c = [condition_estimate_1norm(4, SkewParams(0.25 + d, 0.25, 0.25 + d)) for d in (1e-4, 1e-6, 1e-8)]
    assert 4e5 < c[0] < 4.3e5 and 4e7 < c[1] < 4.3e7 and 4e9 < c[2] < 4.3e9
    with pytest.raises(DegenerateNodes):
        condition_estimate_1norm(4, SkewParams(0.25 + 1e-11, 0.25, 0.25 + 1e-11))


def test_estimate_n16_host_path():
    """n = 16 (N = 4096): the threaded host column sums (the GPU hook is used when
    a device is present); the estimate is the same order as the canonical n = 8 one
    scaled by the growth of ||D||_1 ~ N."""
    c8 = condition_estimate_1norm(8, SkewParams(*PSETS[0]))
    c16 = condition_estimate_1norm(16, SkewParams(*PSETS[0]))
    assert np.isfinite(c16) and 4 * c8 < c16 < 64 * c8
    # the host column sums as computed in the CPU container (tests/test_gpu_ref_pins.py
    # checks the GPU hook's ||D||_1 reproduces it)
    assert abs(c16 - N16_CANON_HOST) <= 1e-12 * c16

