"""Generates the committed golden fixtures under tests/golden/.

* weyl_s4_expected.json — the 24 expected group matrices, extracted verbatim
  from the reference's own unit test (proj/tests/unit/test_weyl_s4.cpp:15-28).
* vectors.npz — seeded inputs (the reference tests' mt19937 streams,
  test_transform.cpp:14-21) and the oracle's forward/inverse outputs at n = 4
  and n = 8, plus the reference-faithful basis factor B_4 (canonical). The
  oracle is pinned against the reference's known-answer tests in
  tests/test_oracle_pins.py; these fixtures freeze its outputs so later
  changes to either side are caught.

Run from the repo root (needs /root/reference for the group table only):
    python tests/golden/make_golden.py
"""
import json
import re
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle  # noqa: E402

HERE = Path(__file__).resolve().parent
REF_TEST = Path("/root/reference/proj/tests/unit/test_weyl_s4.cpp")
CANON = (0.125, 0.0, 0.375)


def group_table():
    text = REF_TEST.read_text()
    block = text[text.index("kExpectedElements"): text.index("};", text.index("kExpectedElements"))]
    rows = re.findall(r"\{([-0-9,\s]+)\}", block)
    mats = [[int(v) for v in r.split(",")] for r in rows if r.count(",") == 8]
    assert len(mats) == 24
    return mats


def main():
    if REF_TEST.exists():
        (HERE / "weyl_s4_expected.json").write_text(
            json.dumps({"source": "proj/tests/unit/test_weyl_s4.cpp:15-28", "elements": group_table()}, indent=1)
        )
    oracle.build()
    out = {}
    for n, seed in ((4, 44), (8, 48)):
        x = oracle.random_signal(n, seed)
        y = oracle.forward_dense(n, CANON, x)
        out[f"x_n{n}"] = x
        out[f"y_n{n}"] = y
        out[f"xinv_n{n}"] = oracle.inverse_dense(n, CANON, y)
    out["B4_ref"] = oracle.RefPlan(4, CANON).basis_dense()
    out["perm4"] = oracle.radix_permutation(4)
    np.savez_compressed(HERE / "vectors.npz", **out)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
