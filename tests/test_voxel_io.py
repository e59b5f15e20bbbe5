"""I/O either side of the path, CPU only: grid
files, spectrum CSV interchange, node / geometry exports and the synthetic
sword, mirroring the reference's tests/unit/test_voxel_io.cpp case by case
plus byte-exact CSV checks against the oracle's node coordinates."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_1807_10058_b200 import (
    DegenerateNodes,
    ErrorCategory,
    IoFailure,
    MalformedFile,
    SizeMismatch,
    SkewParams,
    Spectrum,
    VoxelGrid,
    export_geometry,
    export_nodes_csv,
    export_spectrum,
    grid_from_signal,
    load_grid,
    load_spectrum_csv,
    occupancy_checksum,
    save_grid,
    synthetic_sword,
    z_transform,
)
from paper_1807_10058_b200 import _capi

CANON = SkewParams.canonical()


def sample_grid(n):  # test_voxel_io.cpp:29-38
    vals = 0.5 * np.arange(n**3, dtype=np.float64) - 3.25
    return VoxelGrid(n, vals, {"source": "unit-test", "unit": "none"})


def g17(v):
    return "%.17g" % v


def expected_rows(n, p, values=None):
    """CSV rows built from the oracle's node coordinates (real_coords,
    chebyshev.cpp:87-97) and Python's %.17g — independent of the product."""
    nodes = oracle.skew_nodes(n, (p.r, p.s, p.t))
    rows = []
    for a in range(n**3):
        x, y, z = nodes[a, 3], nodes[a, 4], nodes[a, 5]
        xt = 0.5 * (x + z)
        zt = (x - z) / complex(0.0, 2.0)
        i, j, k = a // (n * n), (a // n) % n, a % n
        row = f"{i},{j},{k},{g17(xt.real)},{g17(y.real)},{g17(zt.real)}"
        if values is not None:
            v = complex(values[a])
            row += f",{g17(v.real)},{g17(v.imag)},{g17(abs(v))}"
        rows.append(row)
    return rows


def test_format_follows_extension(tmp_path):
    g = sample_grid(2)
    for name, is_json in [("grid.json", True), ("grid.raw", False), ("grid.f64", False), ("grid", False)]:
        save_grid(g, tmp_path / name)
        assert os.path.exists(tmp_path / (name + ".json")) == (not is_json)
        if is_json:
            json.loads((tmp_path / name).read_text())


def test_json_grid_round_trip(tmp_path):
    g = sample_grid(3)
    save_grid(g, tmp_path / "grid.json")
    back = load_grid(tmp_path / "grid.json")
    assert back.n == 3 and np.array_equal(back.values, g.values) and back.metadata == g.metadata
    doc = json.loads((tmp_path / "grid.json").read_text())
    assert doc["n"] == 3 and doc["values"] == g.values.tolist()
    # layout of nlohmann::json::dump(): compact, sorted keys, integral doubles as x.0
    text = (tmp_path / "grid.json").read_text()
    assert text.startswith('{"metadata":{"source":"unit-test","unit":"none"},"n":3,"values":[-3.25,-2.75,')
    assert text.endswith("]}\n")


def test_json_doubles_round_trip_exactly(tmp_path):
    rng = np.random.default_rng(3)
    vals = np.concatenate([rng.standard_normal(20) * 10.0 ** rng.integers(-30, 30, 20),
                           [0.0, -0.0, 1.0, 1e15, 1e16, 1e-4, 1e-5, 123456789012345678.0, 5e-324, 1.7976931348623157e308]])
    vals = np.resize(vals, 27)
    save_grid(VoxelGrid(3, vals), tmp_path / "g.json")
    back = load_grid(tmp_path / "g.json")
    assert np.array_equal(back.values.view(np.uint64), vals.view(np.uint64))
    assert json.loads((tmp_path / "g.json").read_text())["values"] == vals.tolist()


def test_raw_grid_round_trip_bit_for_bit(tmp_path):
    g = sample_grid(4)
    save_grid(g, tmp_path / "grid.f64")
    assert (tmp_path / "grid.f64.json").exists()
    assert (tmp_path / "grid.f64").read_bytes() == g.values.astype("<f8").tobytes()
    back = load_grid(tmp_path / "grid.f64")
    assert back.n == 4 and np.array_equal(back.values, g.values) and back.metadata == g.metadata


def test_grid_structural_errors(tmp_path):
    (tmp_path / "bad.json").write_text("{ not json")
    with pytest.raises(MalformedFile):
        load_grid(tmp_path / "bad.json")
    (tmp_path / "short.json").write_text('{"n": 2, "values": [1.0, 2.0]}')
    with pytest.raises(SizeMismatch) as e:
        load_grid(tmp_path / "short.json")
    assert e.value.category == ErrorCategory.io
    (tmp_path / "no_n.json").write_text('{"values": []}')
    with pytest.raises(MalformedFile):
        load_grid(tmp_path / "no_n.json")
    (tmp_path / "float_n.json").write_text('{"n": 2.0, "values": []}')
    with pytest.raises(MalformedFile):
        load_grid(tmp_path / "float_n.json")
    (tmp_path / "big_n.json").write_text('{"n": 5000, "values": []}')
    with pytest.raises(MalformedFile):
        load_grid(tmp_path / "big_n.json")
    (tmp_path / "strval.json").write_text('{"n": 1, "values": ["x"]}')
    with pytest.raises(MalformedFile):
        load_grid(tmp_path / "strval.json")
    (tmp_path / "meta.json").write_text('{"n": 1, "values": [1], "metadata": {"a": 1}}')
    with pytest.raises(MalformedFile):
        load_grid(tmp_path / "meta.json")
    (tmp_path / "orphan.f64").write_bytes(b"xxxxxxxx")
    with pytest.raises(MalformedFile):
        load_grid(tmp_path / "orphan.f64")
    save_grid(sample_grid(2), tmp_path / "trunc.f64")
    with open(tmp_path / "trunc.f64", "r+b") as f:
        f.truncate(3 * 8)
    with pytest.raises(SizeMismatch) as e:
        load_grid(tmp_path / "trunc.f64")
    assert e.value.category == ErrorCategory.io
    with pytest.raises(IoFailure):
        load_grid(tmp_path / "missing.json")
    with pytest.raises(IoFailure):
        save_grid(sample_grid(2), tmp_path / "no_dir" / "g.json")


def test_complexification_round_trips_exactly():
    g = sample_grid(3)
    s = z_transform(g)
    assert s.n == 3 and s.data.numel() == 27
    assert torch.equal(s.data, torch.from_numpy(g.values))
    back = grid_from_signal(s)
    assert np.array_equal(back.values, g.values)
    c = grid_from_signal(type(s)(3, torch.complex(s.data, torch.ones_like(s.data))))
    assert np.array_equal(c.values, g.values)
    with pytest.raises(SizeMismatch):
        z_transform(VoxelGrid(3, np.zeros(26)))


def test_sword_is_binary_with_frozen_occupancy():
    with pytest.raises(ValueError):
        synthetic_sword(4)
    s8 = synthetic_sword(8)
    assert s8.n == 8 and s8.metadata["solid"] == "sword"
    assert set(np.unique(s8.values)) <= {0.0, 1.0} and s8.values.sum() == 10.0
    assert occupancy_checksum(s8) == 15946957412154716965  # test_voxel_io.cpp:136
    s16 = synthetic_sword(16)
    assert s16.values.sum() == 64.0
    assert occupancy_checksum(s16) == 4168761945289145573  # test_voxel_io.cpp:142
    assert 0 < s16.values.sum() / s16.size() < 0.5
    for n in (9, 31, 64):
        s = synthetic_sword(n)
        assert 0 < s.values.mean() < 0.5


def test_occupancy_checksum_sees_pattern_only():
    g = VoxelGrid(2, np.array([0, 1, 0, 0, 1, 0, 0, 0], dtype=np.float64))
    base = occupancy_checksum(g)
    assert occupancy_checksum(VoxelGrid(2, g.values * 7.5)) == base
    moved = g.values.copy()
    moved[[0, 1]] = moved[[1, 0]]
    assert occupancy_checksum(VoxelGrid(2, moved)) != base
    # FNV-1a 64 restated here
    h = 14695981039346656037
    for v in g.values:
        h ^= ord("1") if v != 0 else ord("0")
        h = (h * 1099511628211) % 2**64
    assert base == h


def test_spectrum_export_and_reload(tmp_path):
    vals = np.array([complex(1.0 + 0.25 * i, -0.125 * i) for i in range(8)])
    spec = Spectrum(2, CANON, torch.from_numpy(vals))
    export_spectrum(spec, tmp_path / "spec.csv")
    lines = (tmp_path / "spec.csv").read_text().split("\n")
    assert lines[0] == "# n=2 params=1/8,0,3/8"
    assert lines[1] == "i,j,k,x,y,z,re,im,magnitude"
    assert [l for l in lines[2:] if l] == expected_rows(2, CANON, vals)
    back = load_spectrum_csv(tmp_path / "spec.csv")
    assert back.n == 2 and back.params == CANON
    assert np.array_equal(back.values.numpy(), vals)


@pytest.mark.parametrize("n,p", [(4, CANON), (8, CANON), (4, SkewParams(0.21, 0.055, 0.4)), (3, CANON)])
def test_spectrum_csv_byte_exact_vs_oracle_coordinates(tmp_path, n, p):
    rng = np.random.default_rng(n)
    vals = rng.standard_normal(n**3) + 1j * rng.standard_normal(n**3)
    vals[0] = 0.0
    export_spectrum(Spectrum(n, p, torch.from_numpy(vals)), tmp_path / "s.csv")
    text = (tmp_path / "s.csv").read_text()
    header = f"# n={n} params={p.encode()}\ni,j,k,x,y,z,re,im,magnitude\n"
    assert text == header + "\n".join(expected_rows(n, p, vals)) + "\n"
    back = load_spectrum_csv(tmp_path / "s.csv")
    assert back.params == p and np.array_equal(back.values.numpy(), vals)


def test_spectrum_export_large_parallel_path(tmp_path):
    n = 32  # 32768 rows: formatted by several threads, order preserved
    rng = np.random.default_rng(7)
    vals = rng.standard_normal(n**3) + 1j * rng.standard_normal(n**3)
    export_spectrum(Spectrum(n, CANON, torch.from_numpy(vals)), tmp_path / "big.csv")
    lines = (tmp_path / "big.csv").read_text().splitlines()
    assert len(lines) == 2 + n**3
    assert [tuple(map(int, l.split(",")[:3])) for l in lines[2::997]] == [
        (a // (n * n), (a // n) % n, a % n) for a in range(0, n**3, 997)
    ]
    back = load_spectrum_csv(tmp_path / "big.csv")
    assert np.array_equal(back.values.numpy(), vals)


def test_spectrum_export_argument_checks(tmp_path):
    with pytest.raises(SizeMismatch):
        export_spectrum(Spectrum(2, CANON, torch.zeros(7, dtype=torch.complex128)), tmp_path / "x.csv")
    with pytest.raises(ValueError):
        export_spectrum(Spectrum(2, CANON, torch.zeros(8, dtype=torch.complex128)), tmp_path / "x.csv",
                        params=SkewParams(0.1, 0.2, 0.3))
    with pytest.raises(DegenerateNodes):
        export_spectrum(Spectrum(2, SkewParams(0, 0, 0), torch.zeros(8, dtype=torch.complex128)), tmp_path / "x.csv")


def _write(path, *lines):
    path.write_text("".join(l + "\n" for l in lines))
    return path


HDR = "# n=2 params=1/8,0,3/8"
COLS = "i,j,k,x,y,z,re,im,magnitude"


def test_spectrum_reload_rejects_broken_files(tmp_path):
    with pytest.raises(MalformedFile):
        load_spectrum_csv(_write(tmp_path / "a.csv", COLS))
    with pytest.raises(SizeMismatch) as e:
        load_spectrum_csv(_write(tmp_path / "b.csv", HDR, COLS, "0,0,0,0,0,0,1,0,1"))
    assert e.value.category == ErrorCategory.io
    with pytest.raises(MalformedFile, match="repeats"):
        load_spectrum_csv(_write(tmp_path / "c.csv", "# n=1 params=1/8,0,3/8", COLS, "0,0,0,0,0,0,1,0,1",
                                 "0,0,0,0,0,0,1,0,1"))
    with pytest.raises(IoFailure):
        load_spectrum_csv(tmp_path / "nope.csv")
    with pytest.raises(MalformedFile, match="lacks params"):
        load_spectrum_csv(_write(tmp_path / "d.csv", "# n=2", COLS))
    with pytest.raises(MalformedFile, match="cannot parse spectrum header"):
        load_spectrum_csv(_write(tmp_path / "e.csv", "# n=2 params=1/8,0", COLS))
    with pytest.raises(MalformedFile, match="out of range"):
        load_spectrum_csv(_write(tmp_path / "f.csv", "# n=0 params=1/8,0,3/8", COLS))
    with pytest.raises(MalformedFile, match="column header"):
        load_spectrum_csv(_write(tmp_path / "g.csv", HDR, "i,j,k"))
    with pytest.raises(MalformedFile, match="too few columns"):
        load_spectrum_csv(_write(tmp_path / "h.csv", HDR, COLS, "0,0,0,0,0,0,1,0"))
    with pytest.raises(MalformedFile, match="index out of range"):
        load_spectrum_csv(_write(tmp_path / "i.csv", HDR, COLS, "0,0,2,0,0,0,1,0,1"))
    with pytest.raises(MalformedFile, match="cannot parse spectrum row"):
        load_spectrum_csv(_write(tmp_path / "j.csv", HDR, COLS, "0,0,0,0,0,0,abc,0,1"))
    with pytest.raises(MalformedFile, match="cannot parse spectrum row"):
        load_spectrum_csv(_write(tmp_path / "k.csv", HDR, COLS, "x,0,0,0,0,0,1,0,1"))
    # the reference checks for a repeated node before it parses the values
    with pytest.raises(MalformedFile, match="repeats"):
        load_spectrum_csv(_write(tmp_path / "l.csv", HDR, COLS, "0,0,0,0,0,0,1,0,1", "0,0,0,0,0,0,zz,0,1"))
    # first error in row order wins
    with pytest.raises(MalformedFile, match="too few"):
        load_spectrum_csv(_write(tmp_path / "m.csv", HDR, COLS, "0,0,0", "0,0,9,0,0,0,1,0,1"))


def test_spectrum_reload_tolerates_blank_lines_and_any_row_order(tmp_path):
    rows = [f"{a // 4},{(a // 2) % 2},{a % 2},0,0,0,{a}.5,-{a},0" for a in range(8)]
    rows = rows[::-1]
    rows.insert(3, "")
    f = _write(tmp_path / "ok.csv", HDR, COLS, *rows)
    back = load_spectrum_csv(f)
    assert np.array_equal(back.values.numpy(), np.array([complex(a + 0.5, -a) for a in range(8)]))


def test_geometry_lists_the_fourteen_shifts(tmp_path):
    export_geometry(tmp_path / "geo.csv")
    lines = (tmp_path / "geo.csv").read_text().splitlines()
    assert lines[0] == "dx,dy,dz" and len(lines) == 15
    g = oracle.group()
    expect = sorted({tuple(int(x) for x in w @ e) for e in np.eye(3, dtype=int) for w in g})
    assert [tuple(map(int, l.split(","))) for l in lines[1:]] == expect


@pytest.mark.parametrize("n,p", [(1, CANON), (4, CANON), (8, CANON), (5, SkewParams(0.37, 0.61, 0.085))])
def test_nodes_csv_byte_exact(tmp_path, n, p):
    export_nodes_csv(n, p, tmp_path / "z.csv")
    assert (tmp_path / "z.csv").read_text() == "i,j,k,x,y,z\n" + "\n".join(expected_rows(n, p)) + "\n"


def test_nodes_csv_degenerate_and_stdout(capfd):
    with pytest.raises(DegenerateNodes):
        export_nodes_csv(2, SkewParams(0.0, 0.0, 0.0))
    with pytest.raises(ValueError):
        export_nodes_csv(0, CANON)
    export_nodes_csv(1, CANON)
    assert capfd.readouterr().out.startswith("i,j,k,x,y,z\n0,0,0,")


def test_params_text_through_the_c_abi():
    import ctypes
    L = _capi.lib()
    r, s, t = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    for text, want in [("1/8,0,3/8", (0.125, 0.0, 0.375)), ("0.25, 1e-1,-3/4", (0.25, 0.1, -0.75))]:
        assert L.fcct_parse_params(text.encode(), ctypes.byref(r), ctypes.byref(s), ctypes.byref(t)) == 0
        assert (r.value, s.value, t.value) == want
    for bad in ["1/8,0", "1/8,0,3/8,1", "a,0,0", "1/0,0,0", "1/8x,0,0", ",0,0"]:
        assert L.fcct_parse_params(bad.encode(), ctypes.byref(r), ctypes.byref(s), ctypes.byref(t)) == _capi.INVALID_ARGUMENT
    buf = ctypes.create_string_buffer(64)
    assert L.fcct_encode_params(0.125, 0.0, 0.375, buf, 64) == 0 and buf.value == b"1/8,0,3/8"
    assert L.fcct_encode_params(0.1, -0.5, 3.0, buf, 64) == 0 and buf.value == b"1/10,-1/2,3"
    assert L.fcct_encode_params(0.125, 0.0, 0.375, buf, 4) == _capi.INVALID_ARGUMENT
