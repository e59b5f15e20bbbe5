"""Python mirror of the reference `fcct` transform API (proj/include/fcct/transform.hpp).

Same names, argument meaning and error behaviour as the reference C++ library,
executed by the sm_100a CUDA library through the C ABI (include/fcct_gpu.h).
Tensors are torch complex tensors: complex128 for fp64 plans (the reference's
Eigen::VectorXcd), complex64 for the fp32 variant. A tensor of shape
[batch, n^3] is a batch of independent blocks (the reference applies one vector
per call; batching is the B200 addition). CPU tensors go through the host-buffer
entry points (H2D + transform + D2H); CUDA tensors stay on the device.
"""
from __future__ import annotations

import ctypes
import json
import os
import enum
import math
from dataclasses import dataclass, field
from fractions import Fraction
from typing import List, Optional

import numpy as np
import torch

from . import _capi

# ---------------------------------------------------------------------------
# errors: fcct/errors.hpp:9-63
# ---------------------------------------------------------------------------


class ErrorCategory(enum.Enum):
    math = "math"  # CLI exit code 2
    io = "io"  # CLI exit code 3


class FcctError(RuntimeError):
    category = ErrorCategory.math


class DegenerateNodes(FcctError):
    pass


class IllConditioned(FcctError):
    pass


class SizeMismatch(FcctError):
    pass


class OddSize(FcctError):
    pass


class DerivationError(FcctError):
    pass


class MalformedFile(FcctError):
    category = ErrorCategory.io


class IoFailure(FcctError):
    category = ErrorCategory.io


class CudaError(FcctError):
    pass


def _raise(status: int) -> None:
    if status == _capi.OK:
        return
    msg = _capi.lib().fcct_last_error().decode(errors="replace")
    exc = {
        _capi.INVALID_ARGUMENT: ValueError,  # std::invalid_argument
        _capi.PARAMS_MISMATCH: ValueError,
        _capi.SIZE_MISMATCH: SizeMismatch,
        _capi.ODD_SIZE: OddSize,
        _capi.DEGENERATE_NODES: DegenerateNodes,
        _capi.ILL_CONDITIONED: IllConditioned,
        _capi.IO: IoFailure,
        _capi.CUDA: CudaError,
        _capi.DERIVATION: DerivationError,
        _capi.MALFORMED: MalformedFile,
        _capi.SIZE_MISMATCH_IO: SizeMismatch,
    }.get(status, FcctError)
    err = exc(msg)
    if status == _capi.SIZE_MISMATCH_IO:
        err.category = ErrorCategory.io  # SizeMismatch(..., ErrorCategory::io)
    raise err


# ---------------------------------------------------------------------------
# SkewParams: fcct/spectral.hpp:13-27, src/spectral.cpp:47-117
# ---------------------------------------------------------------------------


def encode_param(value: float) -> str:
    """Exact small rational as 'a/b', else %.17g (spectral.cpp:53-75)."""
    if value == 0.0:
        return "0"
    x = value
    p0, q0, p1, q1 = 0, 1, 1, 0
    for _ in range(40):
        fa = math.floor(x)
        if abs(fa) > 1e15:
            break
        a = int(fa)
        p2, q2 = a * p1 + p0, a * q1 + q0
        if q2 > 1000000 or q2 < 0:
            break
        if q2 != 0 and p2 / q2 == value:
            return str(p2) if q2 == 1 else f"{p2}/{q2}"
        p0, q0, p1, q1 = p1, q1, p2, q2
        frac = x - fa
        if frac == 0.0:
            break
        x = 1.0 / frac
    return f"{value:.17g}"


def parse_param(text: str) -> float:
    """Inverse of encode_param (spectral.cpp:81-103)."""
    if not text:
        raise ValueError("empty grid offset")
    try:
        if "/" in text:
            num, den = text.split("/", 1)
            if "/" in den or float(den) == 0.0:
                raise ValueError
            return float(num) / float(den)
        return float(text)
    except ValueError:
        raise ValueError(f"cannot parse grid offset '{text}'") from None


@dataclass(frozen=True)
class SkewParams:
    r: float = 0.0
    s: float = 0.0
    t: float = 0.0

    @staticmethod
    def canonical() -> "SkewParams":
        return SkewParams(0.125, 0.0, 0.375)

    def child(self, ir: int, is_: int, it: int) -> "SkewParams":
        return SkewParams((self.r + ir) / 2.0, (self.s + is_) / 2.0, (self.t + it) / 2.0)

    def encode(self) -> str:
        return f"{encode_param(self.r)},{encode_param(self.s)},{encode_param(self.t)}"


def parse_params(text: str) -> SkewParams:
    parts = text.split(",")
    if len(parts) != 3:
        raise ValueError(f"grid offsets must be 'r,s,t', got '{text}'")
    return SkewParams(*(parse_param(p) for p in parts))


# ---------------------------------------------------------------------------
# value types: transform.hpp:17-44
# ---------------------------------------------------------------------------


@dataclass
class SignalTensor:
    """Samples at the nodes, [..., n^3]. `data` is complex, or real (float64 /
    float32) when produced by z_transform: the identity complexification
    (voxel_io.cpp:178-186) is then fused into the device tile load."""

    n: int
    data: torch.Tensor

    @staticmethod
    def zeros(n: int, batch: Optional[int] = None, dtype=torch.complex128, device="cpu") -> "SignalTensor":
        shape = (n**3,) if batch is None else (batch, n**3)
        return SignalTensor(n, torch.zeros(shape, dtype=dtype, device=device))

    def size(self) -> int:
        return self.n**3


@dataclass
class Spectrum:
    n: int
    params: SkewParams
    values: torch.Tensor


@dataclass
class DenseTransform:
    """Dense matrix D_n(r,s,t) (rows = nodes, cols = polynomial index), generated
    on the device, plus the direct plan that applies it (DMMA GEMM)."""

    n: int
    params: SkewParams
    matrix: torch.Tensor
    condition_estimate: float = float("nan")
    _plan: Optional["TransformPlan"] = field(default=None, repr=False)


class Kind(enum.Enum):
    direct = 0
    radix2 = 1


@dataclass
class SparseMatrix:
    """CSC export of a basis factor (Eigen::SparseMatrix<Complex> layout)."""

    rows: int
    cols: int
    colptr: np.ndarray
    rowidx: np.ndarray
    values: np.ndarray

    def nonZeros(self) -> int:  # noqa: N802 (reference name)
        return int(self.values.size)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols), dtype=np.complex128)
        for c in range(self.cols):
            sl = slice(self.colptr[c], self.colptr[c + 1])
            out[self.rowidx[sl], c] = self.values[sl]
        return out


def _dtype_of(precision: str) -> torch.dtype:
    return torch.complex64 if precision == "f32" else torch.complex128


def _real_dtype_of(precision: str) -> torch.dtype:
    return torch.float32 if precision == "f32" else torch.float64


class TransformPlan:
    """Executable plan (transform.hpp:67-114). Immutable once built."""

    def __init__(self, handle: int, precision: str, device: int):
        self._h = ctypes.c_void_p(handle)
        self.precision = precision
        self.device = device
        info = _capi.PlanInfo()
        _raise(_capi.lib().fcct_plan_info(self._h, ctypes.byref(info)))
        self.info = info

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _capi.lib().fcct_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    # accessors ------------------------------------------------------------
    def kind(self) -> Kind:
        return Kind(self.info.kind)

    def n(self) -> int:
        return self.info.n

    def params(self) -> SkewParams:
        return SkewParams(self.info.r, self.info.s, self.info.t)

    def permutation(self) -> np.ndarray:
        if self.kind() != Kind.radix2:
            raise ValueError("permutation(): plan is direct")
        return radix_permutation(self.n())

    def kernel(self) -> np.ndarray:
        out = (ctypes.c_double * 128)()
        _raise(_capi.lib().fcct_plan_kernel(self._h, out))
        return np.frombuffer(out, dtype=np.complex128).reshape(8, 8, order="F").copy()

    def basis(self) -> SparseMatrix:
        L = _capi.lib()
        nnz = ctypes.c_int64()
        _raise(L.fcct_plan_basis(self._h, ctypes.byref(nnz), None, None, None))
        N = self.n() ** 3
        colptr = np.zeros(N + 1, dtype=np.int64)
        rowidx = np.zeros(nnz.value, dtype=np.int32)
        vals = np.zeros(2 * nnz.value, dtype=np.float64)
        _raise(
            L.fcct_plan_basis(
                self._h,
                ctypes.byref(nnz),
                colptr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                rowidx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                vals.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            )
        )
        return SparseMatrix(N, N, colptr, rowidx, vals.view(np.complex128))

    def children(self) -> List[tuple]:
        out = []
        for i in range(8):
            n, r, s, t, k = ctypes.c_int(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
            _raise(
                _capi.lib().fcct_plan_child(
                    self._h, i, ctypes.byref(n), ctypes.byref(r), ctypes.byref(s), ctypes.byref(t), ctypes.byref(k)
                )
            )
            out.append((n.value, SkewParams(r.value, s.value, t.value), Kind(k.value)))
        return out

    # raw vector forms (apply_values / solve_values, transform.cpp:429-494) ------
    def _run(
        self, x: torch.Tensor, inverse: bool, params: Optional[SkewParams] = None, real_out: bool = False
    ) -> torch.Tensor:
        N = self.n() ** 3
        dt = _dtype_of(self.precision)
        rdt = _real_dtype_of(self.precision)
        real_in = not inverse and x.dtype == rdt
        if x.dtype != dt and not real_in:
            raise TypeError(f"expected {dt} (or {rdt} real samples) for a {self.precision} plan, got {x.dtype}")
        if x.shape[-1] != N:
            raise SizeMismatch(f"signal has {x.shape[-1]} samples, need {N}")
        if inverse and params is not None and params != self.params():
            raise ValueError("inverse_apply: spectrum was produced on a different skew grid")
        batch = x.numel() // N
        L = _capi.lib()
        x = x.contiguous()
        out = torch.empty(x.shape, dtype=rdt if real_out else dt, device=x.device)
        if x.is_cuda:
            if x.device.index != self.device:
                raise ValueError(f"tensor on {x.device}, plan on cuda:{self.device}")
            stream = torch.cuda.current_stream(x.device).cuda_stream
            if real_in:
                st = L.fcct_forward_real(self._h, x.data_ptr(), out.data_ptr(), batch, stream)
            elif real_out:
                st = L.fcct_inverse_real(self._h, x.data_ptr(), out.data_ptr(), batch, stream)
            elif inverse and params is not None:
                st = L.fcct_inverse_checked(
                    self._h, params.r, params.s, params.t, x.data_ptr(), out.data_ptr(), batch, stream
                )
            else:
                fn = L.fcct_inverse if inverse else L.fcct_forward
                st = fn(self._h, x.data_ptr(), out.data_ptr(), batch, stream)
            _raise(st)
            return out
        if real_in:
            fn = L.fcct_forward_real_host
        elif real_out:
            fn = L.fcct_inverse_real_host
        else:
            fn = L.fcct_inverse_host if inverse else L.fcct_forward_host
        _raise(fn(self._h, x.data_ptr(), out.data_ptr(), batch, None))
        return out

    def apply_values(self, x: torch.Tensor, threads: int = 1) -> torch.Tensor:
        return self._run(x, False)

    def solve_values(self, q: torch.Tensor, threads: int = 1) -> torch.Tensor:
        return self._run(q, True)


# ---------------------------------------------------------------------------
# free functions: transform.hpp:46-143
# ---------------------------------------------------------------------------


# fcct_executor (include/fcct_gpu.h): executors a FAST plan can be forced onto
EXECUTORS = {"auto": 0, "orbit": 1, "orbit-phased": 2, "pipeline2": 3, "two-level": 4, "two-level-v2": 5,
             "tile": 6, "global": 7, "orbit-two-pass": 8, "orbit-streamed": 9}


def _create(n: int, p: SkewParams, method: int, precision: str, device: int, executor: str = "auto") -> TransformPlan:
    if not isinstance(n, int):
        raise TypeError("n must be an int")
    if executor not in EXECUTORS:
        raise ValueError(f"unknown executor {executor!r} (one of {sorted(EXECUTORS)})")
    h = ctypes.c_void_p()
    prec = _capi.F32 if precision == "f32" else _capi.F64
    if executor == "auto":
        _raise(_capi.lib().fcct_plan_create(n, p.r, p.s, p.t, method, prec, device, ctypes.byref(h)))
    else:
        _raise(_capi.lib().fcct_plan_create_executor(n, p.r, p.s, p.t, prec, device, EXECUTORS[executor],
                                                     ctypes.byref(h)))
    return TransformPlan(h.value, precision, device)


def _device_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    return torch.device(device).index or 0


def dense_transform(n: int, p: SkewParams, precision: str = "f64", device=None) -> DenseTransform:
    """dense_transform (transform.cpp:130-144): matrix generated on the GPU."""
    if n < 1:
        raise ValueError("dense_transform: n must be >= 1")
    dev = _device_index(device)
    plan = _create(n, p, _capi.DIRECT, precision, dev)
    N = n**3
    mat = torch.empty((N, N), dtype=torch.complex128, device=f"cuda:{dev}")
    # the C ABI writes column-major; a row-major [N][N] view of it is D^T
    stream = torch.cuda.current_stream(dev).cuda_stream
    _raise(_capi.lib().fcct_dense_matrix(n, p.r, p.s, p.t, mat.data_ptr(), stream))
    # the reference stores its estimate only for n^3 <= 512 (transform.cpp:141-142)
    cond = plan.info.condition if N <= 512 else float("nan")
    return DenseTransform(n, p, mat.t(), cond, plan)


def naive_apply(t: DenseTransform, s: SignalTensor) -> Spectrum:
    """naive_apply (transform.cpp:146-156): y = D x on the DMMA GEMM."""
    if t.n != s.n:
        raise SizeMismatch(f"naive_apply: transform size {t.n} vs signal size {s.n}")
    if s.data.shape[-1] != t.n**3:
        raise SizeMismatch(f"naive_apply: signal has {s.data.shape[-1]} samples, need {t.n ** 3}")
    return Spectrum(t.n, t.params, t._plan.apply_values(s.data))


def inverse_apply(t, q: Spectrum, threads: int = 1, real_output: bool = False) -> SignalTensor:
    """inverse_apply for a DenseTransform (transform.cpp:158-169) or a
    TransformPlan (transform.cpp:509-524).

    real_output=True fuses grid_from_signal (voxel_io.cpp:188-198) into the
    device store: the returned SignalTensor carries only the real parts."""
    if isinstance(t, DenseTransform):
        if t.n != q.n:
            raise SizeMismatch(f"inverse_apply: transform size {t.n} vs spectrum size {q.n}")
        if t.params != q.params:
            raise ValueError("inverse_apply: spectrum was produced on a different skew grid")
        if q.values.shape[-1] != t.n**3:
            raise SizeMismatch(f"inverse_apply: spectrum has {q.values.shape[-1]} values, need {t.n ** 3}")
        return SignalTensor(t.n, t._plan._run(q.values, True, q.params, real_out=real_output))
    plan: TransformPlan = t
    if plan.n() != q.n:
        raise SizeMismatch(f"inverse_apply: plan size {plan.n()} vs spectrum size {q.n}")
    if plan.params() != q.params:
        raise ValueError("inverse_apply: spectrum was produced on a different skew grid")
    if q.values.shape[-1] != q.n**3:
        raise SizeMismatch(f"inverse_apply: spectrum has {q.values.shape[-1]} values, need {q.n ** 3}")
    return SignalTensor(plan.n(), plan._run(q.values, True, q.params, real_out=real_output))


def radix_permutation(n: int) -> np.ndarray:
    """radix_permutation (transform.cpp:171-194), generated on the device."""
    if n < 2:
        raise ValueError("radix_permutation: n must be >= 2")
    if n % 2:
        raise OddSize(f"radix_permutation: size {n} is odd")
    out = np.zeros(n**3, dtype=np.uint64)
    _raise(_capi.lib().fcct_radix_permutation(n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return out


def build_plan(n: int, p: SkewParams, store=None, precision: str = "f64", device=None,
               executor: str = "auto") -> TransformPlan:
    """build_plan (transform.cpp:404-408): radix2 tree for even n, direct otherwise.
    `executor` (EXECUTORS) forces one of the fast executors; "auto" is the default choice."""
    if n < 1:
        raise ValueError("build_plan: n must be >= 1")
    if store is not None:
        return store.load_or_build(n, p, precision=precision, device=device)
    if executor != "auto" and (n == 1 or n % 2):
        executor = "auto"  # odd n / n == 1: a direct plan (transform.cpp:385-386)
    return _create(n, p, _capi.FAST, precision, _device_index(device), executor)


@dataclass
class PlanStoreStats:
    hits: int = 0
    misses: int = 0
    rebuilt: int = 0


class PlanStore:
    """On-disk plan cache (plan_cache.hpp:30-51), one reference-compatible
    `.fccplan` file per (n, params); corrupt entries are rebuilt with a
    warning on stderr, writes are temp + rename."""

    def __init__(self, directory):
        self._h = ctypes.c_void_p()
        _raise(_capi.lib().fcct_store_open(str(directory).encode(), ctypes.byref(self._h)))
        self.directory = str(directory)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _capi.lib().fcct_store_close(h)
            except Exception:
                pass
            self._h = None

    @staticmethod
    def cache_key(n: int, p: SkewParams) -> str:
        return f"n{n}_r{encode_param(p.r)}_s{encode_param(p.s)}_t{encode_param(p.t)}"

    def path_for(self, n: int, p: SkewParams) -> str:
        buf = ctypes.create_string_buffer(4096)
        _raise(_capi.lib().fcct_store_path(self._h, n, p.r, p.s, p.t, buf, 4096))
        return buf.value.decode()

    def warm(self, n: int, p: SkewParams) -> None:
        """load_or_build on the host only (no GPU needed)."""
        _raise(_capi.lib().fcct_store_warm(self._h, n, p.r, p.s, p.t))

    def load_or_build(self, n: int, p: SkewParams, precision: str = "f64", device=None) -> TransformPlan:
        h = ctypes.c_void_p()
        prec = _capi.F32 if precision == "f32" else _capi.F64
        dev = _device_index(device)
        _raise(_capi.lib().fcct_plan_create_from_store(self._h, n, p.r, p.s, p.t, prec, dev, ctypes.byref(h)))
        return TransformPlan(h.value, precision, dev)

    def stats(self) -> PlanStoreStats:
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _raise(_capi.lib().fcct_store_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return PlanStoreStats(a.value, b.value, c.value)


def basis_change(n: int, p: SkewParams, inverse: bool = False) -> SparseMatrix:
    """basis_change (transform.cpp:314-320): the exact sparse factor B (or its
    explicit inverse), derived on the host from the orbit structure."""
    if n < 2 or n % 2:
        raise OddSize(f"basis_change: needs an even size, got {n}")
    L = _capi.lib()
    nnz = ctypes.c_int64()
    _raise(L.fcct_basis_change(n, p.r, p.s, p.t, int(inverse), ctypes.byref(nnz), None, None, None))
    N = n**3
    colptr = np.zeros(N + 1, dtype=np.int64)
    rowidx = np.zeros(nnz.value, dtype=np.int32)
    vals = np.zeros(2 * nnz.value, dtype=np.float64)
    _raise(
        L.fcct_basis_change(
            n, p.r, p.s, p.t, int(inverse), ctypes.byref(nnz),
            colptr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            rowidx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            vals.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
        )
    )
    return SparseMatrix(N, N, colptr, rowidx, vals.view(np.complex128))


def condition_estimate_1norm(n: int, p: SkewParams) -> float:
    """condition_estimate_1norm(dense_transform(n, p).matrix) (transform.cpp:91-122):
    the reference's probe-based estimate, the value IllConditioned is raised on."""
    out = ctypes.c_double()
    _raise(_capi.lib().fcct_condition_estimate(n, p.r, p.s, p.t, ctypes.byref(out)))
    return out.value


def plan_tree_stats(n: int, p: SkewParams) -> dict:
    """Host-side statistics of the fast plan tree (no GPU)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    f, g = ctypes.c_double(), ctypes.c_double()
    _raise(_capi.lib().fcct_plan_tree_stats(n, p.r, p.s, p.t, ctypes.byref(a), ctypes.byref(b), ctypes.byref(f), ctypes.byref(g)))
    return {"tree_nnz": a.value, "tree_nnz_inv": b.value, "flops_forward": f.value, "flops_inverse": g.value}


def fast_apply(plan: TransformPlan, s: SignalTensor, threads: int = 1) -> Spectrum:
    """fast_apply (transform.cpp:496-507). `threads` is accepted for API
    compatibility; the GPU result does not depend on it (bitwise, as in the
    reference, transform.hpp:121-122)."""
    if plan.n() != s.n:
        raise SizeMismatch(f"fast_apply: plan size {plan.n()} vs signal size {s.n}")
    if s.data.shape[-1] != s.n**3:
        raise SizeMismatch(f"fast_apply: signal has {s.data.shape[-1]} samples, need {s.n ** 3}")
    return Spectrum(plan.n(), plan.params(), plan.apply_values(s.data, max(1, threads)))


def factorization_residual(plan: TransformPlan, dense: DenseTransform) -> float:
    """factorization_residual (transform.cpp:526-540), evaluated on the GPU
    against the device-generated dense matrix."""
    if plan.n() != dense.n:
        raise SizeMismatch("factorization_residual: sizes differ")
    out = ctypes.c_double()
    _raise(_capi.lib().fcct_factorization_residual(plan._h, ctypes.byref(out)))
    return out.value


def with_perturbed_basis(plan: TransformPlan, delta: float) -> TransformPlan:
    """with_perturbed_basis (transform.cpp:542-554): negative-control hook."""
    h = ctypes.c_void_p()
    _raise(_capi.lib().fcct_plan_perturbed_basis(plan._h, delta, ctypes.byref(h)))
    return TransformPlan(h.value, plan.precision, plan.device)


def skew_nodes(n: int, p: SkewParams, device=None) -> torch.Tensor:
    """Node set (spectral.cpp:155-171) generated on the device: [n^3, 6]
    complex128 columns (u, v, w, x, y, z). Raises DegenerateNodes for n <= 16."""
    dev = _device_index(device)
    out = torch.empty((n**3, 6), dtype=torch.complex128, device=f"cuda:{dev}")
    stream = torch.cuda.current_stream(dev).cuda_stream
    _raise(_capi.lib().fcct_skew_nodes(n, p.r, p.s, p.t, out.data_ptr(), stream))
    return out


def shard_range(total: int, rank: int, world: int) -> tuple:
    """Contiguous block range of one rank (ceil split): the batch scheduler."""
    b, e = ctypes.c_int64(), ctypes.c_int64()
    _raise(_capi.lib().fcct_shard_range(total, rank, world, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def exact_fraction(x: float) -> Fraction:
    return Fraction(x)


# ---------------------------------------------------------------------------
# I/O either side of the path: voxel_io.hpp, spectral.cpp:173-188 (native, C ABI)
# ---------------------------------------------------------------------------


@dataclass
class VoxelGrid:
    """VoxelGrid (voxel_io.hpp:16-22): real samples on an n^3 grid."""

    n: int
    values: np.ndarray
    metadata: dict = field(default_factory=dict)

    def size(self) -> int:
        return self.n**3


def _path(p) -> Optional[bytes]:
    return None if p is None else os.fsencode(p)


def load_grid(path) -> VoxelGrid:
    """load_grid (voxel_io.cpp:158-164): JSON for '.json' paths, raw + sidecar otherwise."""
    L = _capi.lib()
    n = ctypes.c_int()
    _raise(L.fcct_grid_load(_path(path), ctypes.byref(n), None, 0, None, 0))
    vals = np.empty(n.value**3, dtype=np.float64)
    meta = ctypes.create_string_buffer(1 << 16)
    _raise(L.fcct_grid_load(_path(path), ctypes.byref(n), vals.ctypes.data, vals.size, meta, len(meta)))
    return VoxelGrid(n.value, vals, json.loads(meta.value.decode()))


def save_grid(grid: VoxelGrid, path) -> None:
    """save_grid (voxel_io.cpp:166-176)."""
    vals = np.ascontiguousarray(grid.values, dtype=np.float64)
    if vals.size != grid.n**3 or grid.n < 1:
        raise SizeMismatch(f"grid carries {vals.size} values for n={grid.n}")
    meta = json.dumps(grid.metadata or {}, sort_keys=True).encode()
    _raise(_capi.lib().fcct_grid_save(_path(path), grid.n, vals.ctypes.data, meta))


def z_transform(grid: VoxelGrid, device=None) -> SignalTensor:
    """z_transform (voxel_io.cpp:178-186). The identity complexification is
    not materialised: the SignalTensor carries the real samples and the fast /
    direct apply fuses (re, 0) into its device tile load (fcct_forward_real)."""
    if grid.n < 1 or np.asarray(grid.values).size != grid.n**3:
        raise SizeMismatch(f"grid carries {np.asarray(grid.values).size} values for n={grid.n}")
    data = torch.from_numpy(np.ascontiguousarray(grid.values, dtype=np.float64))
    if device is not None:
        data = data.to(device)
    return SignalTensor(grid.n, data)


def grid_from_signal(s: SignalTensor) -> VoxelGrid:
    """grid_from_signal (voxel_io.cpp:188-198): real parts of one signal."""
    if s.data.shape[-1] != s.n**3 or s.data.numel() != s.n**3:
        raise SizeMismatch(f"signal carries {s.data.numel()} samples for n={s.n}")
    d = s.data.detach().cpu()
    vals = (d.real if d.is_complex() else d).to(torch.float64).numpy().copy()
    return VoxelGrid(s.n, vals.reshape(-1))


def synthetic_sword(n: int) -> VoxelGrid:
    """synthetic_sword (voxel_io.cpp:200-236)."""
    vals = np.empty(max(n, 0) ** 3, dtype=np.float64)
    _raise(_capi.lib().fcct_synthetic_sword(n, vals.ctypes.data if vals.size else None))
    return VoxelGrid(n, vals, {"solid": "sword"})


def occupancy_checksum(grid: VoxelGrid) -> int:
    """occupancy_checksum (voxel_io.cpp:336-344): FNV-1a 64 over '0'/'1' bytes."""
    vals = np.ascontiguousarray(grid.values, dtype=np.float64)
    out = ctypes.c_uint64()
    _raise(_capi.lib().fcct_occupancy_checksum(vals.ctypes.data if vals.size else None, vals.size, ctypes.byref(out)))
    return out.value


def _spectrum_host(spec: Spectrum) -> np.ndarray:
    v = spec.values.detach()
    if v.numel() != spec.n**3:
        raise SizeMismatch("spectrum value count does not match node count")
    return np.ascontiguousarray(v.cpu().to(torch.complex128).numpy().reshape(-1))


def export_spectrum(spec: Spectrum, path=None, params: Optional[SkewParams] = None) -> None:
    """export_spectrum (voxel_io.cpp:238-261) to `path` (None / '-' = stdout).
    `params` stands for the node grid's offsets: they must match the spectrum's."""
    if params is not None and params != spec.params:
        raise ValueError("export_spectrum: spectrum and node grid use different offsets")
    vals = _spectrum_host(spec)
    p = spec.params
    _raise(_capi.lib().fcct_export_spectrum(spec.n, p.r, p.s, p.t, vals.ctypes.data, _path(path)))


def load_spectrum_csv(path) -> Spectrum:
    """load_spectrum_csv (voxel_io.cpp:263-328): MalformedFile / IoFailure /
    SizeMismatch(io) exactly where the reference raises them."""
    L = _capi.lib()
    n, r, s_, t = ctypes.c_int(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _raise(L.fcct_load_spectrum_csv(_path(path), ctypes.byref(n), ctypes.byref(r), ctypes.byref(s_), ctypes.byref(t), None, 0))
    vals = np.empty(n.value**3, dtype=np.complex128)
    _raise(
        L.fcct_load_spectrum_csv(
            _path(path), ctypes.byref(n), ctypes.byref(r), ctypes.byref(s_), ctypes.byref(t), vals.ctypes.data, vals.size
        )
    )
    return Spectrum(n.value, SkewParams(r.value, s_.value, t.value), torch.from_numpy(vals))


def export_nodes_csv(n: int, p: SkewParams, path=None) -> None:
    """export_nodes_csv(skew_nodes(n, p)) (spectral.cpp:155-171,180-188; CLI `zeros`)."""
    _raise(_capi.lib().fcct_export_nodes_csv(n, p.r, p.s, p.t, _path(path)))


def export_geometry(path=None) -> None:
    """export_geometry (voxel_io.cpp:330-334): the 14 FCC shift vectors."""
    _raise(_capi.lib().fcct_export_geometry(_path(path)))
