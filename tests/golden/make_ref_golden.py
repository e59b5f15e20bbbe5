"""Freezes outputs of the REFERENCE'S OWN code into tests/golden/ref_golden.npz.

oracle/_ref/libfcct_ref.so is compiled (oracle/ref.mk) from the reference's
Eigen-free sources where they lie under /root/reference/proj/src
(weyl_s4.cpp, chebyshev.cpp, spectral.cpp). Every entry of D_n is the
reference's cheb_eval_uvw(kappa, uvw_i) (chebyshev.cpp:67-74) at the
reference's skew_nodes (spectral.cpp:155-171), so these columns are
reference-computed values of the transform matrix, not the oracle's.

The GPU box has no /root/reference: tests/test_gpu_parity.py reads this file
to pin the device-generated node set and matrix D against the reference, and
tests/test_ref_pins.py checks that the file still equals the live reference
output here.

Contents (canonical offsets C = (1/8, 0, 3/8) and two non-dyadic sets):
  group            [24, 3, 3] int32, WeylGroup::s4() order
  nodes_{n}_{k}    [n^3, 6] complex128 (u, v, w, x, y, z) for n in 4, 8, 16
  dense4_{k}       D_4 in full, [64, 64] complex128 ([node, kappa])
  dense8_{k}_cols / dense8_{k}  columns COLS8 of D_8, [512, 48]
  dense16_0_cols / dense16_0    columns COLS16 of D_16 (canonical), [4096, 8]
  real_coords8_0   [512, 3] real_coords of the canonical n = 8 nodes

Run from the repo root:  python tests/golden/make_ref_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle  # noqa: E402

HERE = Path(__file__).resolve().parent
OUT = HERE / "ref_golden.npz"
PSETS = [(0.125, 0.0, 0.375), (0.21, 0.055, 0.4), (0.37, 0.61, 0.085)]


def columns(n, count, seed):
    rng = np.random.default_rng(seed)
    N = n**3
    fixed = [0, 1, n, n * n, N - 1]  # constant column, unit indices, the last
    rest = rng.choice(np.setdiff1d(np.arange(N), fixed), size=count - len(fixed), replace=False)
    return np.sort(np.concatenate([fixed, rest])).astype(np.int64)


def dense_cols(n, p, cols):
    return np.stack([oracle.Ref.dense_columns(n, p, int(c), int(c) + 1)[:, 0] for c in cols], axis=1)


def build() -> dict:
    R = oracle.Ref
    out = {"group": R.group()}
    for k, p in enumerate(PSETS):
        for n in (4, 8) + ((16,) if k == 0 else ()):
            out[f"nodes_{n}_{k}"] = R.skew_nodes(n, p)
        out[f"dense4_{k}"] = R.dense_columns(4, p, 0, 64)
        if k < 2:
            c8 = columns(8, 48, 80 + k)
            out[f"dense8_{k}_cols"] = c8
            out[f"dense8_{k}"] = dense_cols(8, p, c8)
    c16 = columns(16, 8, 160)
    out["dense16_0_cols"] = c16
    out["dense16_0"] = dense_cols(16, PSETS[0], c16)
    out["real_coords8_0"] = R.real_coords(8, PSETS[0])
    return out


def main():
    data = build()
    np.savez_compressed(OUT, **data)
    print(OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
