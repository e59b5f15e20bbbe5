"""Per-stage DMMA work of the compiled v2 pipeline (CPU only): total per tile,
busiest warp, busiest SM sub-partition (its tensor-pipe bound in cycles = x16)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1807_10058_b200 import _capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = _capi.lib()
for inv in (0, 1):
    out = (ctypes.c_int64 * 128)()
    ns = ctypes.c_int()
    assert L.fcct_debug_v2_stage_stats(n, 0.125, 0.0, 0.375, inv, out, ctypes.byref(ns)) == 0
    tot = sum(out[4 * s + 1] for s in range(ns.value))
    bound = sum(out[4 * s + 3] for s in range(ns.value)) * 16
    print(("inverse" if inv else "forward"), f"DMMA/tile {tot}  SMSP-bound cycles/tile {bound} (ideal {tot * 4})")
    for s in range(ns.value):
        k, t, mx, sp = out[4 * s: 4 * s + 4]
        ld, ldi, st, sti = out[64 + 4 * s: 68 + 4 * s]
        print(f"  stage {s} {'mix' if k else 'sparse':6s} dmma {t:5d}  max/warp {mx:4d}  max/smsp {sp:5d} -> {sp * 16:6d} cyc (ideal {t * 4})"
              f"  A-load wf/mtile {ld}/{ldi}  store wf/mtile {st}/{sti}")
