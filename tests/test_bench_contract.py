"""The bench.py reference arm runs on CPU and prints the contract's JSON line."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.timeout(300)
def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "3",
         "--cpu-sample", "256"],
        check=True, capture_output=True, text=True, cwd=ROOT,
    )
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_own_arm_json_line():
    """bench.py's own arm on a small config: one JSON line with the contract's
    keys, the roofline and cpu_baseline objects, an e2e through host buffers,
    clocks sampled under load and a nonzero count of this repo's launches."""
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--config", "c1", "--steps", "3", "--warmup", "3",
         "--cpu-seconds", "0.5", "--cpu-sample", "64", "--e2e-blocks", "64", "--e2e-steps", "2"],
        check=True, capture_output=True, text=True, cwd=ROOT,
    )
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "clocks", "gpu_launches"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["value"] > 0
    assert "workload" in line["config"]
    roof = line["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in roof, key
    assert roof["bound"] in ("hbm", "tensor") and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    cpu = line["cpu_baseline"]
    assert cpu["value"] > 0 and cpu["kind"] in ("port", "reference") and cpu["cores"] >= 1
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0
    assert line["clocks"]["sm_max_mhz"] > 0


@pytest.mark.timeout(300)
def test_multi_rank_launcher_end_to_end_on_cpu():
    """`bench.py --gpus 2` outside torchrun starts two ranks itself
    (torch.distributed.run on 127.0.0.1); --emulate-cpu runs them over gloo on
    the host emulation of the compiled orbit-FFT tables. c5 is the strong-scaling
    config: the ragged 37-block volume is split 19 + 18 with no collective on the
    data path, and rank 0 prints one line with n_gpus = 2."""
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--emulate-cpu", "--config", "c5", "--blocks", "37",
         "--steps", "2", "--warmup", "3"],
        check=True, capture_output=True, text=True, cwd=ROOT, timeout=280,
    )
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["blocks_total"] == 37 and line["config"]["blocks_per_gpu_max"] == 19
    assert [tuple(s) for s in line["shards"]] == [(0, 19), (19, 37)]
    assert line["roundtrip_rel_err"] < 1e-12
    assert line["value"] > 0


def test_launcher_fails_loudly_without_enough_gpus():
    import torch

    if torch.cuda.device_count() >= 64:
        pytest.skip("this host has 64 GPUs")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "64", "--steps", "1"],
                       capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert r.returncode != 0
    assert "visible" in r.stderr


@pytest.mark.timeout(300)
def test_reference_arm_config_equals_own_arm_config():
    """The driver compares the two arms' `config` objects: both come from
    bench.workload() with the same arguments."""
    sys.path.insert(0, str(ROOT))
    import argparse

    import bench

    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1", "--steps", "1",
         "--warmup", "3"],
        check=True, capture_output=True, text=True, cwd=ROOT,
    )
    line = json.loads(out.stdout.strip().splitlines()[-1])
    args = argparse.Namespace(config="c1", n=None, precision=None, real_io=None, blocks=None, method="fast")
    assert line["config"] == bench.workload(args, 1)["config"]
    cpu = line["cpu_baseline"]
    assert cpu["cores"] == 1 and "threads=1" in cpu["sample"]
