"""ctypes wrapper of the C++ oracle (oracle/fcct_oracle.cpp) plus the numpy
FFT/orbit-route oracle for large n. TEST INFRASTRUCTURE ONLY.

Parity pinning: see fcct_oracle.cpp's header and tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import itertools
import subprocess
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint, c_uint64, c_void_p
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
LIB = BUILD / "liboracle.so"


def build(force: bool = False) -> None:
    srcs = [HERE / "fcct_oracle.cpp", HERE / "Makefile"]
    if not force and LIB.exists() and all(s.stat().st_mtime <= LIB.stat().st_mtime for s in srcs if s.exists()):
        return
    subprocess.run(["make", "-C", str(HERE), "-s", "all"], check=True)


def _host_key() -> str:
    """Key of this machine's CPU (model name + ISA flags): the -march=native
    CPU baseline is built per host, never carried across machines."""
    import hashlib
    import platform

    info = platform.machine()
    try:
        text = Path("/proc/cpuinfo").read_text()
        model = next((ln for ln in text.splitlines() if ln.startswith("model name")), "")
        flags = next((ln for ln in text.splitlines() if ln.startswith("flags")), "")
        info += model + flags
    except OSError:
        pass
    return hashlib.sha1(info.encode()).hexdigest()[:12]


def cpu_baseline_path(force: bool = False) -> Path:
    """oracle/_build/host-<key>/cpu_baseline, compiled here with -march=native
    on first use (a few seconds)."""
    hostdir = BUILD / f"host-{_host_key()}"
    exe = hostdir / "cpu_baseline"
    srcs = [HERE / "cpu_baseline.cpp", HERE / "fcct_oracle.cpp", HERE / "Makefile"]
    if force or not exe.exists() or any(s.stat().st_mtime > exe.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-C", str(HERE), "-s", "baseline", f"HOSTDIR={hostdir}"], check=True)
    return exe


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        d3 = [c_double, c_double, c_double]
        sig = {
            "oracle_group": (c_int, [POINTER(c_int)]),
            "oracle_skew_nodes": (c_int, [c_int, *d3, c_int, POINTER(c_double)]),
            "oracle_common_zeros": (c_int, [c_int, POINTER(c_double)]),
            "oracle_cheb_eval_uvw": (c_int, [c_int, c_int, c_int, POINTER(c_double), POINTER(c_double)]),
            "oracle_dense_transform": (c_int, [c_int, *d3, c_int, POINTER(c_double)]),
            "oracle_forward_dense": (c_int, [c_int, *d3, c_int64, POINTER(c_double), POINTER(c_double)]),
            "oracle_inverse_dense": (c_int, [c_int, *d3, c_int64, POINTER(c_double), POINTER(c_double)]),
            "oracle_dense_rows": (c_int, [c_int, *d3, c_int64, POINTER(c_int64), c_int64, POINTER(c_double), POINTER(c_double)]),
            "oracle_condition_estimate": (c_int, [c_int, *d3, POINTER(c_double)]),
            "oracle_condition_estimate_matrix": (c_int, [c_int64, POINTER(c_double), POINTER(c_double)]),
            "oracle_radix_permutation": (c_int, [c_int, POINTER(c_uint64)]),
            "oracle_random_signal": (c_int, [c_int, c_uint, POINTER(c_double)]),
            "oracle_plan_build": (c_void_p, [c_int, *d3, POINTER(c_int)]),
            "oracle_plan_free": (None, [c_void_p]),
            "oracle_plan_kind": (c_int, [c_void_p]),
            "oracle_plan_basis_nnz": (c_int64, [c_void_p]),
            "oracle_plan_basis": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int32), POINTER(c_double)]),
            "oracle_plan_tree_nnz": (c_int64, [c_void_p, c_int]),
            "oracle_plan_apply": (c_int, [c_void_p, c_int64, POINTER(c_double), POINTER(c_double)]),
            "oracle_plan_solve": (c_int, [c_void_p, c_int64, POINTER(c_double), POINTER(c_double)]),
            "oracle_plan_factorization_residual": (c_int, [c_void_p, POINTER(c_double)]),
            "oracle_last_error": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _ck(st):
    if st != 0:
        raise OracleError(st, lib().oracle_last_error().decode())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(POINTER(c_double))


def group() -> np.ndarray:
    out = np.zeros(24 * 9, dtype=np.int32)
    _ck(lib().oracle_group(out.ctypes.data_as(POINTER(c_int))))
    return out.reshape(24, 3, 3)


def skew_nodes(n, p, check=True) -> np.ndarray:
    out = np.zeros(n**3 * 12)
    _ck(lib().oracle_skew_nodes(n, p[0], p[1], p[2], int(check), _dp(out)))
    return out.view(np.complex128).reshape(n**3, 6)


def common_zeros(n) -> np.ndarray:
    out = np.zeros(n**3 * 12)
    _ck(lib().oracle_common_zeros(n, _dp(out)))
    return out.view(np.complex128).reshape(n**3, 6)


def cheb_eval_uvw(k, uvw) -> complex:
    a = np.array([uvw[0].real, uvw[0].imag, uvw[1].real, uvw[1].imag, uvw[2].real, uvw[2].imag])
    out = np.zeros(2)
    _ck(lib().oracle_cheb_eval_uvw(int(k[0]), int(k[1]), int(k[2]), _dp(a), _dp(out)))
    return complex(out[0], out[1])


def dense_transform(n, p, ext=False) -> np.ndarray:
    """D_n(p) as a [node, kappa] complex128 array (ColumnEvaluator restatement)."""
    N = n**3
    out = np.zeros(2 * N * N)
    _ck(lib().oracle_dense_transform(n, p[0], p[1], p[2], int(ext), _dp(out)))
    return out.view(np.complex128).reshape(N, N).T.copy()


def forward_dense(n, p, x: np.ndarray) -> np.ndarray:
    """Primary forward oracle: long-double D and long-double accumulation."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    batch = x.size // n**3
    y = np.zeros_like(x)
    _ck(lib().oracle_forward_dense(n, p[0], p[1], p[2], batch, _dp(x.view(np.float64)), _dp(y.view(np.float64))))
    return y


def dense_rows(n, p, rows, x: np.ndarray) -> np.ndarray:
    """Rows `rows` of D_n(p) x, each row generated and accumulated in long
    double (independent of the orbit / FFT route): [batch, len(rows)]."""
    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.complex128)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    y = np.zeros((x.shape[0], len(rows)), dtype=np.complex128)
    _ck(lib().oracle_dense_rows(n, p[0], p[1], p[2], len(rows), rows.ctypes.data_as(POINTER(c_int64)), x.shape[0],
                                _dp(x.view(np.float64)), _dp(y.view(np.float64))))
    return y


def inverse_dense(n, p, y: np.ndarray) -> np.ndarray:
    """Primary inverse oracle: long-double partial-pivot LU (n <= 8)."""
    y = np.ascontiguousarray(y, dtype=np.complex128)
    batch = y.size // n**3
    x = np.zeros_like(y)
    _ck(lib().oracle_inverse_dense(n, p[0], p[1], p[2], batch, _dp(y.view(np.float64)), _dp(x.view(np.float64))))
    return x


def condition_estimate(n, p) -> float:
    out = c_double()
    _ck(lib().oracle_condition_estimate(n, p[0], p[1], p[2], ctypes.byref(out)))
    return out.value


def condition_estimate_matrix(a: np.ndarray) -> float:
    a = np.asfortranarray(a.astype(np.complex128))
    out = c_double()
    _ck(lib().oracle_condition_estimate_matrix(a.shape[0], _dp(a.reshape(-1, order="F").view(np.float64)), ctypes.byref(out)))
    return out.value


def radix_permutation(n) -> np.ndarray:
    out = np.zeros(n**3, dtype=np.uint64)
    _ck(lib().oracle_radix_permutation(n, out.ctypes.data_as(POINTER(c_uint64))))
    return out


def random_signal(n, seed) -> np.ndarray:
    """test_transform.cpp:14-21: std::mt19937(seed) + uniform_real(-1,1), re then im."""
    out = np.zeros(2 * n**3)
    _ck(lib().oracle_random_signal(n, seed, _dp(out)))
    return out.view(np.complex128)


class RefPlan:
    """Reference-faithful fast plan (numeric derive_basis, transform.cpp:202-494)."""

    def __init__(self, n, p):
        st = c_int()
        h = lib().oracle_plan_build(n, p[0], p[1], p[2], ctypes.byref(st))
        _ck(st.value)
        self.h = c_void_p(h)
        self.n = n

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_plan_free(self.h)
            self.h = None

    def basis_nnz(self):
        return lib().oracle_plan_basis_nnz(self.h)

    def tree_nnz(self, with_b2=False):
        return lib().oracle_plan_tree_nnz(self.h, int(with_b2))

    def basis_dense(self) -> np.ndarray:
        N = self.n**3
        nnz = self.basis_nnz()
        cp = np.zeros(N + 1, dtype=np.int64)
        ri = np.zeros(nnz, dtype=np.int32)
        v = np.zeros(2 * nnz)
        _ck(lib().oracle_plan_basis(self.h, cp.ctypes.data_as(POINTER(c_int64)), ri.ctypes.data_as(POINTER(c_int32)), _dp(v)))
        v = v.view(np.complex128)
        B = np.zeros((N, N), dtype=np.complex128)
        for c in range(N):
            B[ri[cp[c]:cp[c + 1]], c] = v[cp[c]:cp[c + 1]]
        return B

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.zeros_like(x)
        _ck(lib().oracle_plan_apply(self.h, x.size // self.n**3, _dp(x.view(np.float64)), _dp(y.view(np.float64))))
        return y

    def solve(self, q):
        q = np.ascontiguousarray(q, dtype=np.complex128)
        x = np.zeros_like(q)
        _ck(lib().oracle_plan_solve(self.h, q.size // self.n**3, _dp(q.view(np.float64)), _dp(x.view(np.float64))))
        return x

    def factorization_residual(self):
        out = c_double()
        _ck(lib().oracle_plan_factorization_residual(self.h, ctypes.byref(out)))
        return out.value


# ---------------------------------------------------------------------------
# FFT / orbit route (independent oracle for n >= 16, incl. n = 64).
#   D_n(p) x = n^3 * IFFT3(S x),  S[a, k] = (1/24) sum_{w: wk = a mod n} e^{2 pi i (wk).p/n}
#   D_n(p)^{-1} y = S^{-1} FFT3(y) / n^3, S^{-1} block diagonal over S4-orbits of Z_n^3.
# Restates ColumnEvaluator's "rank-one tensor of n-th roots of unity" structure
# (transform.cpp:32-34); SURVEY.md Appendix A.
# ---------------------------------------------------------------------------


class OrbitRoute:
    def __init__(self, n, p):
        self.n = n
        self.p = np.array(p, dtype=np.float64)
        G = group()
        N = n**3
        idx = np.array(list(itertools.product(range(n), repeat=3)), dtype=np.int64)  # lex kappa
        wk = np.einsum("gij,kj->gki", G, idx)  # [24, N, 3] unreduced
        abar = np.mod(wk, n)
        arow = (abar[..., 0] * n + abar[..., 1]) * n + abar[..., 2]  # [24, N]
        phase = np.exp(2j * np.pi * (wk @ self.p) / n) / 24.0  # [24, N]
        self.rows = arow
        self.phase = phase
        # orbit decomposition for the inverse
        orbit_of = -np.ones(N, dtype=np.int64)
        blocks = []
        for k in range(N):
            if orbit_of[k] >= 0:
                continue
            mem = np.unique(arow[:, k])
            orbit_of[mem] = len(blocks)
            blocks.append(mem)
        self.blocks = []
        for mem in blocks:
            d = len(mem)
            pos = {int(a): i for i, a in enumerate(mem)}
            S = np.zeros((d, d), dtype=np.complex128)
            for j, k in enumerate(mem):
                for g in range(24):
                    S[pos[int(arow[g, k])], j] += phase[g, k]
            self.blocks.append((mem, np.linalg.inv(S)))

    def S_apply(self, x):
        x = np.atleast_2d(x)
        N = self.n**3
        z = np.zeros((x.shape[0], N), dtype=np.complex128)
        for g in range(24):
            np.add.at(z, (slice(None), self.rows[g]), x * self.phase[g][None, :])
        return z

    def forward(self, x):
        n = self.n
        z = self.S_apply(x).reshape(-1, n, n, n)
        y = np.fft.ifftn(z, axes=(1, 2, 3)) * n**3
        return y.reshape(-1, n**3)

    def inverse(self, y):
        n = self.n
        y = np.atleast_2d(y)
        z = (np.fft.fftn(y.reshape(-1, n, n, n), axes=(1, 2, 3)) / n**3).reshape(-1, n**3)
        x = np.zeros_like(z)
        for mem, Sinv in self.blocks:
            x[:, mem] = z[:, mem] @ Sinv.T
        return x


def symmetrized_rows(n, p, node_idx, x):
    """Per-node direct evaluation sum_k x_k T_k(theta_node) with
    T_k(theta) = (1/24) sum_w e^{2 pi i (w k).theta} (chebyshev.cpp:54-65);
    the acceptance #7 spot check (acceptance/main.cpp:368-388), vectorised."""
    G = group()
    kap = np.array(list(itertools.product(range(n), repeat=3)), dtype=np.int64)
    wk = np.einsum("gij,kj->gki", G, kap).astype(np.float64)  # [24, N, 3]
    out = []
    for a in np.atleast_1d(node_idx):
        ijk = np.array([a // (n * n), (a // n) % n, a % n], dtype=np.float64)
        theta = (np.array(p) + ijk) / n
        theta = theta - np.floor(theta)
        T = np.exp(2j * np.pi * (wk @ theta)).sum(axis=0) / 24.0
        out.append(T @ x)
    return np.array(out)


# ---------------------------------------------------------------------------
# The reference's own Eigen-free sources (weyl_s4.cpp, chebyshev.cpp,
# spectral.cpp), compiled in place by oracle/ref.mk into oracle/_ref/ — the
# checker of this oracle. Only available where /root/reference exists (this
# build container); the GPU box uses the frozen fixtures in tests/golden/.
# ---------------------------------------------------------------------------
REF_DIR = HERE / "_ref"
REF_LIB = REF_DIR / "libfcct_ref.so"
REF_SRC = Path("/root/reference/proj")
_ref = None


def ref_available() -> bool:
    return REF_LIB.exists() or (REF_SRC / "src" / "spectral.cpp").exists()


def build_ref(force: bool = False) -> bool:
    """Compile oracle/_ref/libfcct_ref.so from the reference sources; False
    when the reference tree is absent and no prebuilt library exists."""
    if not (REF_SRC / "src" / "spectral.cpp").exists():
        return REF_LIB.exists()
    srcs = [REF_SRC / "src" / f for f in ("weyl_s4.cpp", "chebyshev.cpp", "spectral.cpp")]
    srcs += [HERE / "ref_shim.cpp", HERE / "ref.mk"]
    if force or not REF_LIB.exists() or any(s.stat().st_mtime > REF_LIB.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-s", "-f", str(HERE / "ref.mk"), f"REF={REF_SRC}"], check=True, cwd=str(HERE.parent))
    return True


def ref_lib() -> ctypes.CDLL:
    global _ref
    if _ref is None:
        if not build_ref():
            raise FileNotFoundError("reference sources absent and oracle/_ref not built")
        L = ctypes.CDLL(str(REF_LIB))
        d3 = [c_double, c_double, c_double]
        sig = {
            "ref_group": (c_int, [POINTER(c_int)]),
            "ref_skew_nodes": (c_int, [c_int, *d3, POINTER(c_double)]),
            "ref_common_zeros": (c_int, [c_int, POINTER(c_double)]),
            "ref_cheb_eval_uvw": (c_int, [c_int, c_int, c_int, POINTER(c_double), POINTER(c_double)]),
            "ref_dense_columns": (c_int, [c_int, *d3, c_int64, c_int64, POINTER(c_double)]),
            "ref_real_coords": (c_int, [c_int, *d3, POINTER(c_double)]),
            "ref_child": (c_int, [*d3, c_int, c_int, c_int, POINTER(c_double)]),
            "ref_encode_param": (c_int, [c_double, ctypes.c_char_p, c_int]),
            "ref_last_error": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _ref = L
    return _ref


def _rck(st):
    if st != 0:
        raise OracleError(st, ref_lib().ref_last_error().decode())


class Ref:
    """The reference's own functions (oracle/_ref), numpy in / out."""

    @staticmethod
    def group() -> np.ndarray:
        out = np.zeros(24 * 9, dtype=np.int32)
        _rck(ref_lib().ref_group(out.ctypes.data_as(POINTER(c_int))))
        return out.reshape(24, 3, 3)

    @staticmethod
    def skew_nodes(n, p) -> np.ndarray:
        out = np.zeros(n**3 * 12)
        _rck(ref_lib().ref_skew_nodes(n, p[0], p[1], p[2], _dp(out)))
        return out.view(np.complex128).reshape(n**3, 6)

    @staticmethod
    def common_zeros(n) -> np.ndarray:
        out = np.zeros(n**3 * 12)
        _rck(ref_lib().ref_common_zeros(n, _dp(out)))
        return out.view(np.complex128).reshape(n**3, 6)

    @staticmethod
    def cheb_eval_uvw(k, uvw) -> complex:
        a = np.array([uvw[0].real, uvw[0].imag, uvw[1].real, uvw[1].imag, uvw[2].real, uvw[2].imag])
        out = np.zeros(2)
        _rck(ref_lib().ref_cheb_eval_uvw(int(k[0]), int(k[1]), int(k[2]), _dp(a), _dp(out)))
        return complex(out[0], out[1])

    @staticmethod
    def dense_columns(n, p, c0, c1) -> np.ndarray:
        """Columns [c0, c1) of D_n(p), [node, column] complex128."""
        N = n**3
        out = np.zeros(2 * N * (c1 - c0))
        _rck(ref_lib().ref_dense_columns(n, p[0], p[1], p[2], c0, c1, _dp(out)))
        return out.view(np.complex128).reshape(c1 - c0, N).T.copy()

    @staticmethod
    def real_coords(n, p) -> np.ndarray:
        out = np.zeros(n**3 * 3)
        _rck(ref_lib().ref_real_coords(n, p[0], p[1], p[2], _dp(out)))
        return out.reshape(n**3, 3)

    @staticmethod
    def child(p, ir, is_, it):
        out = np.zeros(3)
        _rck(ref_lib().ref_child(p[0], p[1], p[2], ir, is_, it, _dp(out)))
        return tuple(out)

    @staticmethod
    def encode_param(v) -> str:
        buf = ctypes.create_string_buffer(64)
        _rck(ref_lib().ref_encode_param(v, buf, 64))
        return buf.value.decode()
