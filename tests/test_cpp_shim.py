"""The C++ shim (include/fcct_b200.hpp, the reference's transform.hpp names over
the C ABI) compiles and links against libfcct_b200.so (CPU), and a program
written against it passes the reference's transform checks and matches the
oracle on the GPU."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "shim_test.cpp"


def build_shim_test(tmp: Path) -> Path:
    from paper_1807_10058_b200 import _build

    _build.build()
    exe = tmp / "shim_test"
    subprocess.run(["g++", "-O2", "-std=c++20", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}", str(SRC),
                    "-o", str(exe), f"-L{_build.LIB_DIR}", "-lfcct_b200", f"-Wl,-rpath,{_build.LIB_DIR}"], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    exe = build_shim_test(tmp_path)
    assert exe.exists()


@pytest.mark.gpu
def test_shim_program_on_gpu(cuda, oracle_mod, tmp_path):
    exe = build_shim_test(tmp_path)
    out = tmp_path / "xy.bin"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    data = np.fromfile(out, dtype=np.complex128).reshape(2, 4, 512)
    x, y = data
    y_ref = oracle_mod.forward_dense(8, (0.125, 0.0, 0.375), x)
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) <= 1e-12
