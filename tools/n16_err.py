"""Relative forward error of n = 16 plans against the orbit-route oracle, per executor (argv: r s t)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1807_10058_b200 import SignalTensor, SkewParams, build_plan, fast_apply  # noqa: E402

p = SkewParams(*(float(a) for a in sys.argv[1:4])) if len(sys.argv) > 3 else SkewParams.canonical()
oracle.build()
rng = np.random.default_rng(31)
x = rng.uniform(-1, 1, (7, 4096)) + 1j * rng.uniform(-1, 1, (7, 4096))
ref = oracle.OrbitRoute(16, (p.r, p.s, p.t)).forward(x)
plan = build_plan(16, p)
y = fast_apply(plan, SignalTensor(16, torch.from_numpy(x).cuda())).values.cpu().numpy()
print(os.environ.get("FCCT_PIPELINE", "default"), "executor", plan.info.executor, "cond", plan.info.condition,
      "rel", np.linalg.norm(y - ref) / np.linalg.norm(ref))
