"""ctypes binding of include/fcct_gpu.h (the C ABI of libfcct_b200.so).

There is no fallback: if the CUDA library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint64, c_void_p

from . import _build

OK = 0
INVALID_ARGUMENT = 1
SIZE_MISMATCH = 2
ODD_SIZE = 3
DEGENERATE_NODES = 4
ILL_CONDITIONED = 5
PARAMS_MISMATCH = 6
IO = 7
CUDA = 8
DERIVATION = 9
MALFORMED = 10
SIZE_MISMATCH_IO = 11

DIRECT = 0
FAST = 1
F64 = 0
F32 = 1
KIND_DIRECT = 0
KIND_RADIX2 = 1


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("n", c_int),
        ("r", c_double),
        ("s", c_double),
        ("t", c_double),
        ("kind", c_int),
        ("method", c_int),
        ("precision", c_int),
        ("levels", c_int),
        ("points", c_int64),
        ("tree_nnz", c_int64),
        ("tree_nnz_inv", c_int64),
        ("root_nnz", c_int64),
        ("table_bytes", c_int64),
        ("condition", c_double),
        ("flops_forward", c_double),
        ("flops_inverse", c_double),
        ("executor", c_int),
        ("exec_flops_forward", c_double),
        ("exec_flops_inverse", c_double),
        ("table_bytes_forward", c_int64),
        ("exec_flops_forward_real", c_double),
        ("exec_flops_inverse_real", c_double),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if not path.exists():
        raise ImportError(
            f"libfcct_b200.so is not built ({path}); run __graft_entry__.build() — "
            "the FCC-DCT has no CPU fallback"
        )
    L = ctypes.CDLL(str(path))
    sig = {
        "fcct_last_error": (c_char_p, []),
        "fcct_plan_create_executor": (c_int, [c_int, c_double, c_double, c_double, c_int, c_int, c_int, POINTER(c_void_p)]),
        "fcct_plan_create": (c_int, [c_int, c_double, c_double, c_double, c_int, c_int, c_int, POINTER(c_void_p)]),
        "fcct_plan_destroy": (c_int, [c_void_p]),
        "fcct_plan_info": (c_int, [c_void_p, POINTER(PlanInfo)]),
        "fcct_forward": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "fcct_inverse": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "fcct_inverse_checked": (c_int, [c_void_p, c_double, c_double, c_double, c_void_p, c_void_p, c_int64, c_void_p]),
        "fcct_forward_host": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "fcct_inverse_host": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "fcct_forward_real": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "fcct_inverse_real": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "fcct_forward_real_host": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "fcct_inverse_real_host": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "fcct_radix_permutation": (c_int, [c_int, POINTER(c_uint64)]),
        "fcct_dense_matrix": (c_int, [c_int, c_double, c_double, c_double, c_void_p, c_void_p]),
        "fcct_dense_matrix_host": (c_int, [c_int, c_double, c_double, c_double, c_int, c_void_p]),
        "fcct_skew_nodes": (c_int, [c_int, c_double, c_double, c_double, c_void_p, c_void_p]),
        "fcct_plan_kernel": (c_int, [c_void_p, POINTER(c_double)]),
        "fcct_plan_basis": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64), POINTER(c_int32), POINTER(c_double)]),
        "fcct_plan_child": (c_int, [c_void_p, c_int, POINTER(c_int), POINTER(c_double), POINTER(c_double), POINTER(c_double), POINTER(c_int)]),
        "fcct_factorization_residual": (c_int, [c_void_p, POINTER(c_double)]),
        "fcct_plan_perturbed_basis": (c_int, [c_void_p, c_double, POINTER(c_void_p)]),
        "fcct_shard_range": (c_int, [c_int64, c_int, c_int, POINTER(c_int64), POINTER(c_int64)]),
        "fcct_debug_dmma_probe": (c_int, [c_void_p, c_void_p, c_void_p]),
        "fcct_store_open": (c_int, [ctypes.c_char_p, POINTER(c_void_p)]),
        "fcct_parse_params": (c_int, [ctypes.c_char_p, POINTER(c_double), POINTER(c_double), POINTER(c_double)]),
        "fcct_encode_params": (c_int, [c_double, c_double, c_double, ctypes.c_char_p, c_int64]),
        "fcct_export_nodes_csv": (c_int, [c_int, c_double, c_double, c_double, ctypes.c_char_p]),
        "fcct_export_geometry": (c_int, [ctypes.c_char_p]),
        "fcct_export_spectrum": (c_int, [c_int, c_double, c_double, c_double, c_void_p, ctypes.c_char_p]),
        "fcct_load_spectrum_csv": (c_int, [ctypes.c_char_p, POINTER(c_int), POINTER(c_double), POINTER(c_double), POINTER(c_double), c_void_p, c_int64]),
        "fcct_grid_load": (c_int, [ctypes.c_char_p, POINTER(c_int), c_void_p, c_int64, ctypes.c_char_p, c_int64]),
        "fcct_grid_save": (c_int, [ctypes.c_char_p, c_int, c_void_p, ctypes.c_char_p]),
        "fcct_synthetic_sword": (c_int, [c_int, c_void_p]),
        "fcct_occupancy_checksum": (c_int, [c_void_p, c_int64, POINTER(ctypes.c_uint64)]),
        "fcct_store_close": (c_int, [c_void_p]),
        "fcct_store_warm": (c_int, [c_void_p, c_int, c_double, c_double, c_double]),
        "fcct_store_stats": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int), POINTER(c_int)]),
        "fcct_store_path": (c_int, [c_void_p, c_int, c_double, c_double, c_double, ctypes.c_char_p, c_int]),
        "fcct_plan_create_from_store": (c_int, [c_void_p, c_int, c_double, c_double, c_double, c_int, c_int, POINTER(c_void_p)]),
        "fcct_debug_emulate_v2": (c_int, [c_int, c_double, c_double, c_double, c_int, c_void_p, c_void_p, c_int64]),
        "fcct_debug_emulate_orbit_fft": (c_int, [c_int, c_double, c_double, c_double, c_int, c_void_p, c_void_p, c_int64]),
        "fcct_debug_emulate_orbit16": (c_int, [c_int, c_double, c_double, c_double, c_int, c_void_p, c_void_p, c_int64]),
        "fcct_debug_emulate_orbit_pat": (c_int, [c_int, c_double, c_double, c_double, c_int, c_void_p, c_void_p, c_int64, POINTER(c_int64)]),
        "fcct_debug_emulate_orbit_big": (c_int, [c_int, c_double, c_double, c_double, c_int, c_void_p, c_void_p, c_int64]),
        "fcct_debug_v2_stats": (c_int, [c_int, c_double, c_double, c_double, c_int, POINTER(c_int64)]),
        "fcct_debug_v2_entry_slots": (c_int, [c_int, c_double, c_double, c_double, c_int, c_int, POINTER(c_int32), c_int64, POINTER(c_int64)]),
        "fcct_debug_v2_stage_stats": (c_int, [c_int, c_double, c_double, c_double, c_int, POINTER(c_int64), POINTER(c_int)]),
        "fcct_debug_timing": (c_int, [c_void_p, c_int, c_void_p, POINTER(c_int)]),
        "fcct_condition_estimate": (c_int, [c_int, c_double, c_double, c_double, POINTER(c_double)]),
        "fcct_basis_change": (c_int, [c_int, c_double, c_double, c_double, c_int, POINTER(c_int64), POINTER(c_int64), POINTER(c_int32), POINTER(c_double)]),
        "fcct_plan_tree_stats": (c_int, [c_int, c_double, c_double, c_double, POINTER(c_int64), POINTER(c_int64), POINTER(c_double), POINTER(c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


# Symbols include/fcct_gpu.h declares (checked by the CPU test suite).
HEADER_SYMBOLS = [
    "fcct_last_error",
    "fcct_plan_create",
    "fcct_plan_create_executor",
    "fcct_plan_destroy",
    "fcct_plan_info",
    "fcct_forward",
    "fcct_inverse",
    "fcct_inverse_checked",
    "fcct_forward_host",
    "fcct_inverse_host",
    "fcct_forward_real",
    "fcct_inverse_real",
    "fcct_forward_real_host",
    "fcct_inverse_real_host",
    "fcct_radix_permutation",
    "fcct_dense_matrix",
    "fcct_dense_matrix_host",
    "fcct_skew_nodes",
    "fcct_plan_kernel",
    "fcct_plan_basis",
    "fcct_plan_child",
    "fcct_factorization_residual",
    "fcct_plan_perturbed_basis",
    "fcct_shard_range",
    "fcct_basis_change",
    "fcct_condition_estimate",
    "fcct_plan_tree_stats",
    "fcct_parse_params",
    "fcct_encode_params",
    "fcct_export_nodes_csv",
    "fcct_export_geometry",
    "fcct_export_spectrum",
    "fcct_load_spectrum_csv",
    "fcct_grid_load",
    "fcct_grid_save",
    "fcct_synthetic_sword",
    "fcct_occupancy_checksum",
    "fcct_store_open",
    "fcct_store_close",
    "fcct_store_warm",
    "fcct_store_stats",
    "fcct_store_path",
    "fcct_plan_create_from_store",
]
