"""Per-stage clock64 breakdown of the fp64 fast pipeline (CTA 0), profiling aid."""
import ctypes
import os
import sys
from pathlib import Path

os.environ["FCCT_DEBUG_TIMING"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1807_10058_b200 import SkewParams, _capi, build_plan  # noqa: E402
from paper_1807_10058_b200.fcct import _raise  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
plan = build_plan(n, SkewParams.canonical())
x = torch.randn(blocks, n**3, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
L = _capi.lib()
for inv in (0, 1):
    fn = L.fcct_inverse if inv else L.fcct_forward
    for _ in range(3):
        _raise(fn(plan._h, x.data_ptr(), y.data_ptr(), blocks, None))
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (18 + 16 * 16))()
    ns = ctypes.c_int()
    _raise(L.fcct_debug_timing(plan._h, inv, buf, ctypes.byref(ns)))
    t = np.array(buf[:], dtype=np.float64)
    S = ns.value
    comp = t[1 : 1 + S]
    store = t[9 : 9 + S]
    tot = t[0] + comp.sum() + store.sum()
    print(("inverse" if inv else "forward"), "total Mcycles (CTA 0)", round(tot / 1e6, 3), f"load={100 * t[0] / tot:.1f}%",
          " ".join(f"s{i}=({100 * comp[i] / tot:.1f}% + {100 * store[i] / tot:.1f}%)" for i in range(S)))
    if len(sys.argv) > 3:  # per-warp compute-phase cycles per tile (CTA 0)
        tiles = (blocks + 16 * 148 - 1) // (16 * 148)
        for i in range(S):
            w = t[18 + 16 * i: 18 + 16 * i + 16] / tiles
            print(f"   s{i} per-warp compute cyc/tile: min {w.min():.0f} mean {w.mean():.0f} max {w.max():.0f}  stage {comp[i] / tiles:.0f}")
