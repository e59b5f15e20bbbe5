"""Measured fp64 error floor of the fast path at large n vs the FFT/orbit oracle."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1807_10058_b200 import SignalTensor, SkewParams, Spectrum, build_plan, fast_apply, inverse_apply  # noqa: E402

CANON = SkewParams.canonical()
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
for n in [int(a) for a in sys.argv[1:]] or [16, 32, 64]:
    t = time.time()
    route = oracle.OrbitRoute(n, (CANON.r, CANON.s, CANON.t))
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (1, n**3)) + 1j * rng.uniform(-1, 1, (1, n**3))
    y_ref = route.forward(x)
    t0 = time.time()
    plan = build_plan(n, CANON)
    tb = time.time() - t0
    y = fast_apply(plan, SignalTensor(n, torch.from_numpy(x).cuda())).values.cpu().numpy()
    xb = inverse_apply(plan, Spectrum(n, CANON, torch.from_numpy(y_ref).cuda())).data.cpu().numpy()
    back = inverse_apply(plan, Spectrum(n, CANON, torch.from_numpy(y).cuda())).data.cpu().numpy()
    print(f"n={n} plan {tb:.1f}s fwd {rel(y, y_ref):.2e} inv {rel(xb, route.inverse(y_ref)):.2e} "
          f"roundtrip {rel(back, x):.2e} (oracle setup {t0 - t:.1f}s) tree_nnz {plan.info.tree_nnz}", flush=True)
