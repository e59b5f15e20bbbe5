"""In-tree build of the CUDA library (sm_100a) behind the C ABI.

The shared object lands in paper_1807_10058_b200/_lib/ so it travels with the
repository snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libfcct_b200.so"
CLI = LIB_DIR / "fcct"  # command-line front end (csrc/cli.cpp), a client of the C ABI
SOURCES = ["kernels.cu", "gemm_tc.cu", "host_stage.cpp", "orbit_fft.cu", "orbit_fft_host.cpp", "orbit16.cu", "orbit16_host.cpp", "orbit_pat.cu", "orbit_pat_host.cpp", "orbit_big.cu", "orbit_big_host.cpp", "capi.cpp", "plan.cpp", "tiling.cpp", "plan_cache.cpp", "voxel_io.cpp"]
HEADERS = ["kernels.hpp", "host_stage.hpp", "orbit_fft.hpp", "orbit16.hpp", "orbit_pat.hpp", "orbit_dev.cuh", "orbit_big.hpp", "device.cuh", "plan.hpp", "tiling.hpp", "plan_cache.hpp", "voxel_io.hpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3",
    "-std=c++20",
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC,-O3",
    "-shared",
]
# FCCT_BUILD_AB=1: a tuning build whose library honours the FCCT_DEBUG_* / A/B
# environment switches (capi.cpp ab_env; tools/stage_timing.py). The product
# build never reads them.
if os.environ.get("FCCT_BUILD_AB") == "1":
    FLAGS.append("-DFCCT_AB_SWITCHES")


# FCCT_NVTX=1: NVTX ranges around the forward / inverse calls too (plan construction
# always carries one).
if os.environ.get("FCCT_NVTX") == "1":
    FLAGS.append("-DFCCT_NVTX")


STAMP = LIB_DIR / "build_flags.txt"


def _stale() -> bool:
    if not LIB.exists() or not STAMP.exists() or STAMP.read_text() != " ".join(FLAGS):
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "fcct_gpu.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def _cli_stale() -> bool:
    if not CLI.exists():
        return True
    t = CLI.stat().st_mtime
    return any(p.stat().st_mtime > t for p in [CSRC / "cli.cpp", LIB, PKG.parent / "include" / "fcct_gpu.h"])


def build_cli(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _cli_stale():
        return CLI
    tmp = CLI.with_suffix(".tmp")
    cmd = ["g++", "-O2", "-std=c++20", "-Wall", str(CSRC / "cli.cpp"), "-o", str(tmp), f"-L{LIB_DIR}", "-lfcct_b200",
           "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, CLI)
    return CLI


def build(force: bool = False, verbose: bool = False) -> Path:
    if force or _stale():
        LIB_DIR.mkdir(exist_ok=True)
        obj_dir = LIB_DIR / "obj"
        obj_dir.mkdir(exist_ok=True)
        # one translation unit per nvcc process, all in parallel, then one link
        compile_flags = [f for f in FLAGS if f != "-shared"]
        procs, objs = [], []
        for s in SOURCES:
            obj = obj_dir / (s + ".o")
            cmd = [NVCC, *compile_flags, "-c", str(CSRC / s), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd))
            procs.append((s, subprocess.Popen(cmd)))
            objs.append(str(obj))
        failed = [s for s, p in procs if p.wait() != 0]
        if failed:
            raise subprocess.CalledProcessError(1, f"nvcc {' '.join(failed)}")
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, *FLAGS, "-o", str(tmp), *objs]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
        STAMP.write_text(" ".join(FLAGS))
    build_cli(force=force, verbose=verbose)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
