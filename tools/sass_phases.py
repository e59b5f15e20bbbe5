"""Aggregates ncu per-instruction stall samples (source page, SASS view) into
code regions split at barrier instructions. Usage: sass_phases.py <csv> [kernel index]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
# the file holds one or more kernels: "Kernel Name" row then header row then instructions
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "hdr": None, "ins": []}
        blocks.append(cur)
    elif cur is not None and cur["hdr"] is None:
        cur["hdr"] = r
    elif cur is not None and len(r) > 3:
        cur["ins"].append(r)
b = blocks[kidx]
h = b["hdr"]
ci = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
total = sum(int(r[ci]) for r in b["ins"])
print(b["name"][:120], "total samples", total)
region, acc, ops, start = 0, Counter(), Counter(), None
def flush(reg, acc, ops, start, end):
    s = sum(acc.values())
    if s < 0.005 * total:
        return
    top = ", ".join(f"{k[6:]} {v}" for k, v in acc.most_common(5))
    mix = ", ".join(f"{k} {v}" for k, v in ops.most_common(6))
    print(f"region {reg:2d} [{start}..{end}] {100.0 * s / total:5.1f}%  stalls: {top}\n           ops: {mix}")
for r in b["ins"]:
    src = r[1].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    if start is None:
        start = r[0][-5:]
    for i in stall_cols:
        v = int(r[i] or 0)
        if v:
            acc[h[i]] += v
    ops[op.split(".")[0]] += int(r[h.index("Instructions Executed")] or 0)
    if op.startswith("BAR") or op.startswith("SYNCS"):
        flush(region, acc, ops, start, r[0][-5:])
        region, acc, ops, start = region + 1, Counter(), Counter(), None
flush(region, acc, ops, start, "end")
