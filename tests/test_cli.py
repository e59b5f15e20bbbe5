"""CLI parity: the `fcct` binary built from csrc/cli.cpp
over the C ABI, case by case after the reference's tests/cli/test_cli.cpp —
same subcommands, flags, outputs and exit codes (0 ok, 1 usage, 2 math, 3 io).
Commands that transform data need the GPU and are marked so."""
import json
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1807_10058_b200 import _build, load_grid, load_spectrum_csv, synthetic_sword, occupancy_checksum

_build.build()  # the library and the CLI binary next to it
CLI = str(_build.CLI)


def run(args, cwd, env=None):
    e = dict(os.environ)
    e.pop("FCCT_CACHE_DIR", None)
    if env:
        e.update(env)
    p = subprocess.run([CLI, *args], cwd=cwd, capture_output=True, text=True, env=e, timeout=600)
    return p.returncode, p.stdout, p.stderr


def body_lines(text, skip):
    return len([l for l in text.splitlines() if l]) - skip


def test_zeros_emits_one_row_per_node(tmp_path):
    rc, out, err = run(["zeros", "--n", "8"], tmp_path)
    assert rc == 0
    assert out.startswith("i,j,k,x,y,z\n") and body_lines(out, 1) == 512
    assert "512 nodes" in err
    rc, _, _ = run(["zeros", "--n", "4", "--params", "0.21,0.055,2/5", "--out", str(tmp_path / "z.csv")], tmp_path)
    assert rc == 0 and body_lines((tmp_path / "z.csv").read_text(), 1) == 64


def test_degenerate_offsets_exit_with_math_code(tmp_path):
    rc, _, err = run(["zeros", "--n", "2", "--params", "0,0,0"], tmp_path)
    assert rc == 2 and "error:" in err
    rc, _, err = run(["zeros", "--n", "2", "--params", "1/8,0"], tmp_path)
    assert rc == 2 and "error:" in err


def test_usage_problems_exit_with_code_1(tmp_path):
    assert run([], tmp_path)[0] == 1
    assert run(["zeros"], tmp_path)[0] == 1  # --n is required
    assert run(["zeros", "--n", "8", "--wat"], tmp_path)[0] == 1
    assert run(["zeros", "--n", "0"], tmp_path)[0] == 1
    assert run(["zeros", "--n", "eight"], tmp_path)[0] == 1
    assert run(["transform", "--input", "a", "--out", "b", "--method", "wrong"], tmp_path)[0] == 1
    assert run(["transform", "--input", "a", "--out", "b", "--threads", "65"], tmp_path)[0] == 1
    assert run(["verify", "--n-max", "17"], tmp_path)[0] == 1
    assert run(["sword", "--n", "4", "--out", "x.json"], tmp_path)[0] == 1
    assert run(["nosuch"], tmp_path)[0] == 1
    rc, out, _ = run(["--help"], tmp_path)
    assert rc == 0 and "transform" in out
    assert run(["zeros", "--help"], tmp_path)[0] == 0


def test_missing_input_exits_with_io_code(tmp_path):
    rc, _, err = run(["transform", "--input", str(tmp_path / "nope.json"), "--out", str(tmp_path / "out.csv")], tmp_path)
    assert rc == 3 and "error:" in err
    (tmp_path / "bad.csv").write_text("i,j,k,x,y,z,re,im,magnitude\n")
    rc, _, _ = run(["transform", "--direction", "inverse", "--input", str(tmp_path / "bad.csv"), "--out",
                    str(tmp_path / "o.json")], tmp_path)
    assert rc == 3


def test_plan_caching_reports_loads_on_second_run(tmp_path):
    cache = str(tmp_path / "cache")

    def counts(out):
        m = re.search(r"loaded=(\d+) built=(\d+) rebuilt=(\d+) cache_files=(\d+)", out)
        return tuple(int(x) for x in m.groups())

    rc, out, _ = run(["plan", "--n", "4", "--cache-dir", cache], tmp_path)
    assert rc == 0
    c1 = counts(out)
    assert c1[0] == 0 and c1[1] > 0 and c1[2] == 0 and c1[3] == c1[1]
    rc, out, _ = run(["plan", "--n", "4"], tmp_path, env={"FCCT_CACHE_DIR": cache})
    c2 = counts(out)
    assert rc == 0 and c2[0] == c1[1] and c2[1] == 0 and c2[2] == 0
    assert out.startswith("plan n=4 params=1/8,0,3/8: ")
    rc, _, err = run(["plan", "--n", "4"], tmp_path)
    assert rc == 1 and "cache-dir" in err


def test_geometry_prints_the_fourteen_shifts(tmp_path):
    rc, out, _ = run(["geometry"], tmp_path)
    assert rc == 0 and out.startswith("dx,dy,dz\n") and body_lines(out, 1) == 14


def test_sword_writes_the_solid(tmp_path):
    rc, _, err = run(["sword", "--n", "16", "--out", str(tmp_path / "s.json")], tmp_path)
    assert rc == 0 and "checksum=4168761945289145573" in err
    g = load_grid(tmp_path / "s.json")
    assert g.metadata == {"solid": "sword"} and np.array_equal(g.values, synthetic_sword(16).values)
    rc, _, _ = run(["sword", "--n", "8", "--out", str(tmp_path / "s.f64")], tmp_path)
    assert rc == 0 and occupancy_checksum(load_grid(tmp_path / "s.f64")) == 15946957412154716965


@pytest.mark.gpu
def test_forward_and_inverse_round_trip_through_files(tmp_path):
    solid, spec, back = tmp_path / "solid.json", tmp_path / "spec.csv", tmp_path / "back.json"
    assert run(["sword", "--n", "8", "--out", str(solid)], tmp_path)[0] == 0
    rc, _, err = run(["transform", "--input", str(solid), "--out", str(spec), "--threads", "2"], tmp_path)
    assert rc == 0 and "forward fast n=8 done" in err
    rc, _, err = run(["transform", "--direction", "inverse", "--input", str(spec), "--out", str(back)], tmp_path)
    assert rc == 0 and "inverse fast n=8 done" in err
    a, b = load_grid(solid), load_grid(back)
    assert b.n == a.n and np.abs(a.values - b.values).max() < 1e-12  # reference bar: 1e-8
    # --n / --params cross-checks (fcct.cpp:86-91,110-121)
    assert run(["transform", "--input", str(solid), "--out", str(spec), "--n", "4"], tmp_path)[0] == 1
    assert run(["transform", "--direction", "inverse", "--input", str(spec), "--out", str(back), "--params",
                "1/4,0,3/8"], tmp_path)[0] == 1


@pytest.mark.gpu
def test_naive_and_fast_spectra_agree_through_the_cli(tmp_path, oracle_mod):
    solid = tmp_path / "solid.json"
    assert run(["sword", "--n", "8", "--out", str(solid)], tmp_path)[0] == 0
    assert run(["transform", "--input", str(solid), "--out", str(tmp_path / "f.csv"), "--method", "fast"], tmp_path)[0] == 0
    assert run(["transform", "--input", str(solid), "--out", str(tmp_path / "n.csv"), "--method", "naive"], tmp_path)[0] == 0
    a = load_spectrum_csv(tmp_path / "f.csv").values.numpy()
    b = load_spectrum_csv(tmp_path / "n.csv").values.numpy()
    assert np.abs(a - b).max() / np.abs(b).max() < 1e-12  # reference bar: 1e-10
    ref = oracle_mod.forward_dense(8, (0.125, 0.0, 0.375), load_grid(solid).values.astype(np.complex128)[None])[0]
    assert np.linalg.norm(a - ref) / np.linalg.norm(ref) <= 1e-12


@pytest.mark.gpu
def test_verify_passes_clean_and_fails_the_negative_control(tmp_path):
    report = tmp_path / "report.json"
    rc, _, err = run(["verify", "--n-max", "4", "--out", str(report)], tmp_path)
    assert rc == 0, err
    doc = json.loads(report.read_text())
    assert doc["all_passed"] is True and len(doc["checks"]) >= 10 and doc["n_max"] == 4
    names = [c["name"] for c in doc["checks"]]
    assert names[:3] == ["group_structure", "evaluation_routes_agree", "coordinate_identities"]
    assert {"factorization_residual", "fast_matches_dense", "round_trip", "basis_sparsity"} <= set(names)
    assert "n=4: nnz/n^3=3.828125" in doc["checks"][names.index("basis_sparsity")]["detail"]  # 245 / 64
    rc, _, err = run(["verify", "--n-max", "2", "--perturb-b"], tmp_path)
    assert rc == 2 and "FAIL factorization_residual" in err


@pytest.mark.gpu
def test_bench_writes_one_csv_row_per_size_and_method(tmp_path):
    rc, out, _ = run(["bench", "--sizes", "2,4", "--repeats", "2"], tmp_path)
    assert rc == 0
    lines = out.splitlines()
    assert lines[0] == "n,method,plan_seconds,apply_seconds"
    assert sum(",fast," in l for l in lines) == 2 and sum(",naive," in l for l in lines) == 2
    assert run(["bench", "--sizes", "2,x"], tmp_path)[0] == 1
    assert run(["bench", "--sizes", "0"], tmp_path)[0] == 1
