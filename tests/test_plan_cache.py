"""Plan cache (PlanStore) — CPU tests of the reference-compatible `.fccplan`
store: layout (plan_cache.hpp:11-27), keys (plan_cache.cpp:74-88,213-220),
load-or-build statistics and corruption handling (plan_cache.cpp:222-282;
test_plan_cache.cpp), and the byte format parsed independently here."""
import os
import struct
from pathlib import Path

import numpy as np

from oracle import oracle
from paper_1807_10058_b200 import PlanStore, SkewParams

CANON = SkewParams.canonical()


def parse_fccplan(path):
    """Independent reader of the reference layout (plan_cache.hpp:11-27)."""
    b = Path(path).read_bytes()
    assert b[:8] == b"FCCPLAN1"
    ver, kind = struct.unpack_from("<IB", b, 8)
    (n,) = struct.unpack_from("<Q", b, 13)
    off = 21
    strs = []
    for _ in range(3):
        (ln,) = struct.unpack_from("<I", b, off)
        strs.append(b[off + 4: off + 4 + ln].decode())
        off += 4 + ln
    out = {"version": ver, "kind": kind, "n": n, "params": strs}
    N = n**3
    if kind == 0:
        (dim,) = struct.unpack_from("<Q", b, off)
        off += 8
        out["dense"] = np.frombuffer(b, dtype=np.complex128, count=dim * dim, offset=off).reshape(dim, dim)
        off += 16 * dim * dim
    else:
        out["kernel"] = np.frombuffer(b, dtype=np.complex128, count=64, offset=off).reshape(8, 8)
        off += 16 * 64
        out["perm"] = np.frombuffer(b, dtype=np.uint64, count=N, offset=off)
        off += 8 * N
        (nnz,) = struct.unpack_from("<Q", b, off)
        off += 8
        rec = np.frombuffer(b, dtype=np.dtype([("r", "<u8"), ("c", "<u8"), ("re", "<f8"), ("im", "<f8")]), count=nnz,
                            offset=off)
        off += 32 * nnz
        B = np.zeros((N, N), complex)
        B[rec["r"].astype(int), rec["c"].astype(int)] = rec["re"] + 1j * rec["im"]
        out["B"] = B
        out["order"] = list(zip(rec["c"].tolist(), rec["r"].tolist()))
    assert off == len(b), "trailing bytes"
    return out


def test_store_layout_keys_and_stats(tmp_path):
    st = PlanStore(tmp_path)
    st.warm(8, CANON)
    files = sorted(os.listdir(tmp_path))
    assert len(files) == 585  # an n = 8 tree is 585 files
    assert all(f.endswith(".fccplan") for f in files)
    assert Path(st.path_for(8, CANON)).name == "n8_r1d8_s0_t3d8.fccplan"
    assert PlanStore.cache_key(8, CANON) == "n8_r1/8_s0_t3/8"
    s = st.stats()
    assert (s.hits, s.misses, s.rebuilt) == (0, 585, 0)
    st2 = PlanStore(tmp_path)
    st2.warm(8, CANON)
    s2 = st2.stats()
    assert (s2.hits, s2.misses, s2.rebuilt) == (585, 0, 0)


def test_store_format_matches_reference_layout(tmp_path):
    st = PlanStore(tmp_path)
    st.warm(4, CANON)
    root = parse_fccplan(st.path_for(4, CANON))
    assert root["version"] == 1 and root["kind"] == 1 and root["n"] == 4
    assert root["params"] == ["1/8", "0", "3/8"]
    assert np.abs(root["kernel"] - oracle.dense_transform(2, (0.125, 0.0, 0.375))).max() < 1e-15
    assert np.array_equal(root["perm"], oracle.radix_permutation(4))
    ref = oracle.RefPlan(4, (0.125, 0.0, 0.375)).basis_dense()
    assert np.count_nonzero(root["B"]) == 245
    assert np.abs(root["B"] - ref).max() < 1e-11
    assert root["order"] == sorted(root["order"])  # Eigen compressed-column order
    leaf = parse_fccplan(st.path_for(1, CANON.child(0, 0, 0).child(1, 1, 0)))
    assert leaf["kind"] == 0 and leaf["n"] == 1 and abs(leaf["dense"][0, 0] - 1) < 1e-15


def test_store_rebuilds_corrupt_entries(tmp_path, capfd):
    st = PlanStore(tmp_path)
    st.warm(4, CANON)
    victim = Path(st.path_for(2, CANON.child(1, 0, 1)))
    good = victim.read_bytes()
    victim.write_bytes(good[:40])  # truncated
    st2 = PlanStore(tmp_path)
    st2.warm(4, CANON)
    s = st2.stats()
    assert s.rebuilt == 1 and s.hits == 72 and s.misses == 0
    assert "warning: rebuilding plan cache entry" in capfd.readouterr().err
    assert victim.read_bytes() == good  # rebuilt in place, deterministic
    # header mismatch (wrong n) is also caught
    Path(st.path_for(4, CANON)).write_bytes(Path(st.path_for(2, CANON.child(1, 0, 1))).read_bytes())
    st3 = PlanStore(tmp_path)
    st3.warm(4, CANON)
    assert st3.stats().rebuilt == 1
