"""Counts the distinct shapes of the orbit blocks of S_n(p).

S_n[a, k] = (1/24) sum_{w : w k = a mod n} e^{2 pi i (w k).p / n} (ColumnEvaluator's
unreduced exponent, transform.cpp:51-53) is block diagonal over the S4-orbits of Z_n^3.
With an orbit's members listed in group order from its smallest member and the phase of
the reduced index e^{2 pi i a.p/n} / 24 divided out of the rows, only the carry phases
e^{2 pi i t.p} (w k = a + n t) remain — and the blocks coincide in 8 matrices for every n
and offset triple tried. Uses nothing but the group (oracle.group(), numpy).

    python tools/orbit_shapes.py [n ...]
"""
import itertools
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402


def shapes(n, p):
    """{(size, block bytes): orbit count} of the normalised orbit blocks."""
    G = oracle.group().astype(np.int64)
    p = np.asarray(p, dtype=np.float64)
    idx = np.array(list(itertools.product(range(n), repeat=3)), dtype=np.int64)
    wk = np.einsum("gij,kj->gki", G, idx)  # [24, N, 3], unreduced
    a = np.mod(wk, n)
    carry = (wk - a) // n
    row = (a[..., 0] * n + a[..., 1]) * n + a[..., 2]
    seen = np.zeros(n**3, dtype=bool)
    out = {}
    for k in range(n**3):
        if seen[k]:
            continue
        mem = []
        for g in range(24):
            if int(row[g, k]) not in mem:
                mem.append(int(row[g, k]))
        seen[mem] = True
        pos = {m: i for i, m in enumerate(mem)}
        S = np.zeros((len(mem), len(mem)), dtype=np.complex128)
        for j, c in enumerate(mem):
            for g in range(24):
                S[pos[int(row[g, c])], j] += np.exp(2j * np.pi * float(carry[g, c] @ p))
        key = (len(mem), np.round(S, 9).tobytes())
        out[key] = out.get(key, 0) + 1
    return out


def summary(n, p):
    by_size = {}
    for (d, _), c in shapes(n, p).items():
        by_size.setdefault(d, []).append(c)
    return {d: sorted(v, reverse=True) for d, v in sorted(by_size.items())}


if __name__ == "__main__":
    ns = [int(x) for x in sys.argv[1:]] or [8, 16]
    for n in ns:
        for p in ((0.125, 0.0, 0.375), (0.21, 0.055, 0.4)):
            s = summary(n, p)
            print(f"n = {n:2d} p = {p}: {sum(len(v) for v in s.values())} shapes; orbits per shape by size: {s}")
