"""Small driver for ncu captures: one forward + one inverse launch of a plan."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1807_10058_b200 import SkewParams, build_plan, dense_transform, _capi  # noqa: E402
from paper_1807_10058_b200.fcct import _raise  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--blocks", type=int, default=65536)
ap.add_argument("--method", default="fast")
ap.add_argument("--precision", default="f64")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--real", action="store_true", help="real samples in and out (fcct_forward_real / fcct_inverse_real)")
a = ap.parse_args()
p = SkewParams.canonical()
plan = build_plan(a.n, p, precision=a.precision) if a.method == "fast" else dense_transform(a.n, p, precision=a.precision)._plan
dt = torch.complex64 if a.precision == "f32" else torch.complex128
x = torch.randn(a.blocks, a.n**3, dtype=dt, device="cuda")
y = torch.empty_like(x)
L = _capi.lib()
if a.real:
    x = torch.randn(a.blocks, a.n**3, dtype=torch.float32 if a.precision == "f32" else torch.float64, device="cuda")
for _ in range(a.reps):
    if a.real:
        _raise(L.fcct_forward_real(plan._h, x.data_ptr(), y.data_ptr(), a.blocks, None))
        _raise(L.fcct_inverse_real(plan._h, y.data_ptr(), x.data_ptr(), a.blocks, None))
    else:
        _raise(L.fcct_forward(plan._h, x.data_ptr(), y.data_ptr(), a.blocks, None))
        _raise(L.fcct_inverse(plan._h, y.data_ptr(), x.data_ptr(), a.blocks, None))
torch.cuda.synchronize()
print("ok")
