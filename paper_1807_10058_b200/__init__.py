"""B200-native FCC-lattice cosine transform (arXiv 1807.10058).

Drop-in for the hot path of the reference `fcct` library: plan creation,
forward / inverse, direct (dense, DMMA GEMM) and fast (radix-2x2x2
factorization) variants, executed by hand-written sm_100a kernels behind the C
ABI in include/fcct_gpu.h. See DESIGN.md.
"""
from .fcct import (  # noqa: F401
    DegenerateNodes,
    DenseTransform,
    ErrorCategory,
    FcctError,
    IllConditioned,
    IoFailure,
    Kind,
    MalformedFile,
    OddSize,
    PlanStore,
    SignalTensor,
    SizeMismatch,
    SkewParams,
    Spectrum,
    TransformPlan,
    basis_change,
    build_plan,
    dense_transform,
    encode_param,
    factorization_residual,
    fast_apply,
    inverse_apply,
    naive_apply,
    parse_param,
    parse_params,
    plan_tree_stats,
    radix_permutation,
    shard_range,
    skew_nodes,
    with_perturbed_basis,
)
