"""Small-batch workload for compute-sanitizer (memcheck / racecheck / synccheck):
every executor of the fast plan and the direct GEMMs, forward and inverse, two
back-to-back calls on one stream (programmatic dependent launch overlaps the
second call's prologue with the first's tail) and calls on two streams sharing a
plan (plan scratch handed over by events). Each result is checked against the
first call's, so a race that corrupts data also fails the run.

  compute-sanitizer --tool racecheck python tools/sanitize.py [--quick]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1807_10058_b200 import SignalTensor, SkewParams, Spectrum, build_plan, dense_transform, fast_apply
from paper_1807_10058_b200 import inverse_apply, naive_apply

quick = "--quick" in sys.argv
P = SkewParams.canonical()
dev = torch.device("cuda:0")
cases = [(4, "orbit", 37), (8, "orbit", 37), (8, "orbit-phased", 19), (8, "pipeline2", 19), (16, "orbit", 5),
         (16, "orbit", 1200), (16, "orbit-two-pass", 5), (16, "two-level", 4), (32, "orbit", 1), (32, "orbit-streamed", 1),
         (8, "tile", 9), (8, "global", 9)]
if not quick:
    cases += [(64, "orbit", 1), (16, "global", 2)]


def rnd(n, b, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.rand((b, n**3), generator=g, dtype=torch.float64) * 2 - 1
    y = torch.rand((b, n**3), generator=g, dtype=torch.float64) * 2 - 1
    return torch.complex(x, y).to(dev)


failures = 0
for n, ex, b in cases:
    plan = build_plan(n, P, executor=ex)
    x = rnd(n, b, n + b)
    y0 = fast_apply(plan, SignalTensor(n, x)).values
    y1 = fast_apply(plan, SignalTensor(n, x)).values  # back to back on one stream
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        y2 = fast_apply(plan, SignalTensor(n, x)).values  # second stream, same plan scratch
        x2 = inverse_apply(plan, Spectrum(n, P, y2)).data
    s2.synchronize()
    xb = inverse_apply(plan, Spectrum(n, P, y0)).data
    torch.cuda.synchronize()
    ok = torch.equal(y0, y1) and torch.equal(y0, y2) and torch.equal(xb, x2)
    err = float((xb - x).abs().max())
    print(f"n={n:2d} {ex:13s} batch={b:3d} executor={plan.info.executor} repeat-equal={ok} roundtrip={err:.1e}")
    failures += (not ok) or err > 1e-9
for n, prec in [(4, "f64"), (8, "f64"), (8, "f32"), (2, "f64")]:
    # tcgen05 direct plans (executors 8, 9) share a per-plan slice workspace across
    # calls and streams; n = 2 runs the DMMA GEMM
    dt = dense_transform(n, P, precision=prec)
    x = rnd(n, 333, 5)
    if prec == "f32":
        x = x.to(torch.complex64)
    y = naive_apply(dt, SignalTensor(n, x)).values
    y1 = naive_apply(dt, SignalTensor(n, x)).values
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        y2 = naive_apply(dt, SignalTensor(n, x)).values
        x2 = inverse_apply(dt, Spectrum(n, P, y2)).data
    s2.synchronize()
    xb = inverse_apply(dt, Spectrum(n, P, y)).data
    torch.cuda.synchronize()
    ok = torch.equal(y, y1) and torch.equal(y, y2) and torch.equal(xb, x2)
    err = float((xb - x).abs().max())
    print(f"n={n:2d} direct {prec} executor={dt._plan.info.executor} repeat-equal={ok} roundtrip={err:.1e}")
    failures += (not ok) or err > (1e-4 if prec == "f32" else 1e-9)
print("FAILURES", failures)
sys.exit(1 if failures else 0)
