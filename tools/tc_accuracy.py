"""fp32 direct transform accuracy: tcgen05 3xTF32 (executor 8) against the SIMT
FFMA kernel (n = 6 has no 128-wide tiling -> SIMT; so compare on n = 8 via the
fp64 oracle), forward and round trip, relative L2."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import oracle
from paper_1807_10058_b200 import SkewParams, SignalTensor, Spectrum, dense_transform, naive_apply, inverse_apply
P = SkewParams.canonical()
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for n, b in [(4, 300), (8, 130), (8, 2000)]:
    rng = np.random.default_rng(5)
    x = (rng.uniform(-1, 1, (b, n**3)) + 1j * rng.uniform(-1, 1, (b, n**3)))
    y_ref = oracle.forward_dense(n, (P.r, P.s, P.t), x)
    d32 = dense_transform(n, P, precision="f32"); d64 = dense_transform(n, P)
    xt = torch.from_numpy(x).to(torch.complex64).cuda()
    y = naive_apply(d32, SignalTensor(n, xt)).values
    back = inverse_apply(d32, Spectrum(n, P, y)).data
    # inverse alone on the exact spectrum (rounded to complex64)
    yr = torch.from_numpy(y_ref).to(torch.complex64).cuda()
    xi = inverse_apply(d32, Spectrum(n, P, yr)).data
    x64 = inverse_apply(d64, Spectrum(n, P, yr.to(torch.complex128))).data
    print(f"n={n} b={b} exec={d32._plan.info.executor} fwd {rel(y.cpu().numpy(), y_ref):.2e} inv(y_ref) {rel(xi.cpu().numpy(), x):.2e} "
          f"inv64(y_ref as c64) {rel(x64.cpu().numpy(), x):.2e} roundtrip {rel(back.cpu().numpy(), x):.2e}")
