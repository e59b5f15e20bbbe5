"""Ozaki-scheme accuracy model (numpy): real-form D_n / D_n^{-1} applied through
kOzS int8 slices with per-row power-of-two scales, keeping the products with
p + q <= S + 1, against fp64. Picks the slice count of gemm_ozaki_kernel.
  python tools/ozaki_sim.py [n]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402


def realform(A):
    N = A.shape[0]
    W = np.zeros((2 * N, 2 * N))
    W[0::2, 0::2] = A.real
    W[0::2, 1::2] = -A.imag
    W[1::2, 0::2] = A.imag
    W[1::2, 1::2] = A.real
    return W


def slices(A, S):
    amax = np.abs(A).max(axis=1, keepdims=True)
    _, e = np.frexp(np.where(amax > 0, amax, 1.0))
    sig = np.ldexp(1.0, e)
    R = A / sig
    out = []
    for q in range(1, S + 1):
        sl = np.clip(np.rint(R * 2.0 ** (7 * q)), -127, 127)
        out.append(sl)
        R = R - sl * 2.0 ** (-7 * q)
    return out, sig


def ozaki(X, W, S):
    xs, sx = slices(X, S)
    ws, sw = slices(W, S)
    C = np.zeros((X.shape[0], W.shape[0]))
    for a in range(S):
        for b in range(S - a):
            C += (xs[a] @ ws[b].T) * 2.0 ** (-7 * (a + b + 2))
    return C * sx * sw.T


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    N = n**3
    D = oracle.dense_transform(n, (0.125, 0.0, 0.375))
    Wf, Wi = realform(D), realform(np.linalg.inv(D))
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (8, N)) + 1j * rng.uniform(-1, 1, (8, N))
    X = np.zeros((8, 2 * N))
    X[:, 0::2], X[:, 1::2] = x.real, x.imag
    Y = X @ Wf.T
    for S in (5, 6, 7, 8):
        e1 = np.linalg.norm(ozaki(X, Wf, S) - Y) / np.linalg.norm(Y)
        Xb = Y @ Wi.T
        e2 = np.linalg.norm(ozaki(Y, Wi, S) - Xb) / np.linalg.norm(Xb)
        print(f"n={n} S={S}: forward {e1:.2e}  inverse {e2:.2e}")
