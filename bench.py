#!/usr/bin/env python3
"""Benchmark of the B200 FCC-DCT hot path (BASELINE.json configs[1]).

Workload ("c2"): batched FCC-DCT n = 8 (N = n^3 = 512 points per block, the
reference's index set), 65,536 independent blocks per GPU,
fp64, inputs i.i.d. uniform[-1,1] (re and im) from a seed, one step = forward
then inverse (round trip) of every block through the fast (radix-2x2x2)
plan. Metric: transforms/s (one transform = one block forward OR inverse;
points/s = N x that), whole job over all ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU (torchrun, one process per GPU): blocks are sharded, 65,536 per
rank (weak scaling), no collective on the data path; the timed region is
bracketed by barriers and the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_DEFAULT = 8
BLOCKS_PER_GPU = 65536
METRIC = "FCC-DCT transforms/s and points/s (fp64) vs HBM/FP64-TC roofline, 1–8 GPU"
FP64_PEAK_TFLOPS = 37.17  # measured DMMA peak on this pool's B200 (profiles/r01_fp_peaks.txt)
FP32_PEAK_TFLOPS = 72.4  # measured FFMA peak (profiles/r01_fp_peaks.txt)
# dense TF32 tensor-core peak: the fallback B200_PROFILING.md states (MEASURED_PEAKS.json
# has no TF32 figure; its measured bf16 burst / 2 = 805 TF/s is reported beside it)
TF32_PEAK_TFLOPS = 1100.0
# dense INT8 tensor-core peak, the B200_PROFILING.md fallback (fp8 / int8 4.5 PFLOP/s dense)
INT8_PEAK_TOPS = 4500.0


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(smax), "reasons": sorted(reasons), "samples": len(sm)}


def profiled_traffic(cfg_name: str, f32: bool, executor: int):
    """dram__bytes_read.sum + dram__bytes_write.sum of one forward call of the
    dominant kernel(s) from the committed `ncu --set full` captures; None when
    the run is not a captured configuration.
    c2 fp64 (tools/prof_run.py, 65,536 blocks): profiles/r01_orbit_fft_ws_raw.csv
    (orbit-FFT executor) or profiles/r01_pipeline2_raw.csv (stage pipeline).
    c3 (16,384 blocks, real f64 input): the single-pass kernel's forward launch from
    profiles/r02_orbit_pat_raw.csv (`prof_run.py --n 16 --real`); on the two-pass
    executor the forward base change from profiles/r01_orbit16_passA_raw.csv plus the
    forward cube FFT from profiles/r01_orbit16_raw.csv (z is complex128 either way)."""
    parts = {
        ("c2", 2): [("r01_pipeline2_raw.csv", None)],
        ("c2", 5): [("r01_orbit_fft_ws_raw.csv", None)],
        ("c3", 6): [("r01_orbit16_passA_raw.csv", "orbit16_base_kernel<0, 2, 0>"),
                    ("r01_orbit16_raw.csv", "fft_cube_kernel<16, 1,")],
        ("c3", 10): [("r02_orbit_pat_raw.csv", "orbit_pat_kernel<0, 2, 0>")],
    }.get((cfg_name, executor))
    if f32 or parts is None:
        return None
    try:
        import csv

        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for fname, kernel in parts:
            rows = list(csv.reader(open(Path(__file__).resolve().parent / "profiles" / fname)))
            hdr, units = rows[0], rows[1]
            ki = hdr.index("Kernel Name")
            vals = next(r for r in rows[2:] if kernel is None or kernel in r[ki])
            for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(name)
                tot += float(vals[i]) * scale[units[i]]
        return tot
    except (OSError, ValueError, KeyError, IndexError, StopIteration):
        return None


def launches_per_call(info):  # noqa: C901
    """Kernels one forward / one inverse call launches on each executor
    (fcct_plan_info_t.executor): orbit-FFT 1; two-pass n = 16: base change +
    cube FFT (+ un-permute on the inverse); large n: S pass + 3 line passes;
    two-level: root pass + 8 children + permutation; stage pipelines and the
    direct GEMM: 1 (global multi-pass: one per stage, ~levels * 2 + 1)."""
    ex = info.executor
    if ex == 6:
        return (2, 3)
    if ex == 7:
        return (4, 4)
    if ex == 4:
        return (10, 10)
    if ex == 3:
        k = 2 * info.levels + 1
        return (k, k)
    if ex == 9:  # input slicing + the int8 GEMM
        return (2, 2)
    return (1, 1)


def cpu_baseline_run(n: int, mode: str = "batched", method: str = "fast", blocks: int = 1, threads: int = 1,
                     fanout: int = 1, repeats: int = 5, min_seconds: float = 0.0, reps: int = 1) -> dict:
    """One run of oracle/cpu_baseline.cpp (built on this host with -march=native)."""
    from oracle import oracle  # CPU baseline / reference arm only

    exe = oracle.cpu_baseline_path()
    out = subprocess.run(
        [str(exe), "--n", str(n), "--mode", mode, "--method", method, "--blocks", str(blocks), "--threads",
         str(threads), "--fanout", str(fanout), "--repeats", str(repeats), "--min-seconds", str(min_seconds),
         "--reps", str(reps)],
        check=True, capture_output=True, text=True,
    )
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_baseline(config: str, n: int, method: str, sample: int, min_seconds: float) -> dict:
    """The reference path timed on this host's cores, beside the GPU number
    (BASELINE.md "CPU baseline plan"). value = transforms/s (forward + inverse
    per transform pair, like the GPU metric)."""
    threads = os.cpu_count() or 1
    if n > 16:
        r = cpu_baseline_run(n, "fftroute", repeats=3, min_seconds=min_seconds)
        return {
            "value": 2e6 / (r["forward_us"] + r["inverse_us"]), "unit": "transforms/s", "cores": 1, "kind": "port",
            "sample": (f"one n={n} transform, forward + inverse, median of {r['repeats']} calls: the FFT-route oracle "
                       "(D x = n^3 IFFT3(S x); inverse S^-1 FFT3(y)/n^3 with S's orbit blocks), NOT the reference "
                       "path, which cannot build an n = 64 plan (~137 GB of dense child LUs, SURVEY.md 0.6)"),
            "us_per_forward": r["forward_us"], "us_per_inverse": r["inverse_us"], "route": "fft",
        }
    # mode 1: one vector per call (fcct bench protocol), threads = 1 and the reference's threads = 8 fan-out
    rows = {}
    for tag, fan in (("threads1", 1), ("fanout8", 8)):
        if method == "direct" and fan > 1:
            continue  # the dense path has no fan-out
        if method == "direct" and n > 8:
            continue  # a fresh 4096^2 LU per inverse call: minutes per call (transform.cpp:158-169)
        r = cpu_baseline_run(n, "faithful", method, fanout=fan, repeats=5)
        rows[tag] = {"us_per_forward": r["forward_us"], "us_per_inverse": r["inverse_us"],
                     "transforms_per_s": 2e6 / (r["forward_us"] + r["inverse_us"]), "cores": fan,
                     "inner_loop": r["inner"]}
    if config == "c1":
        best = rows["threads1"]
        return {
            "value": best["transforms_per_s"], "unit": "transforms/s", "cores": 1, "kind": "port",
            "sample": (f"one n={n} vector per call, {method} path, threads=1, the fcct bench protocol "
                       f"(tools/fcct.cpp:508-521: warm-up, median of 5 repeats of a {best['inner_loop']}-call inner "
                       "loop), reference-faithful C++ restatement (oracle/cpu_baseline.cpp, -O3 -march=native)"),
            "us_per_forward": best["us_per_forward"], "us_per_inverse": best["us_per_inverse"], "mode1": rows,
        }
    # mode 2: batched, all cores
    r = cpu_baseline_run(n, "batched", method, blocks=sample, threads=threads, min_seconds=min_seconds)
    return {
        "value": 2 * sample / (r["forward_s"] + r["inverse_s"]), "unit": "transforms/s", "cores": threads,
        "kind": "port",
        "sample": (f"{sample} blocks of n={n}, forward then inverse, {method} path, repeated {r.get('reps', 1)}x "
                   f"(>= {min_seconds:g} s of CPU work), one block per call, std::thread over blocks; "
                   "reference-faithful C++ restatement (oracle/cpu_baseline.cpp, -O3 -march=native)"
                   + ("; the direct inverse reuses one LU factored at plan time (the reference refactors per "
                      "call, transform.cpp:158-169: a lower bound on its time)" if method == "direct" else "")),
        "mode1": rows,
    }


CONFIGS = {
    # BASELINE.json configs restated on the reference's n^3 index set
    "c1": dict(n=4, blocks=1, scaling="weak", desc="single FCC-DCT n=4 (64 points), i.i.d. U[-1,1] re/im (latency config)"),
    "c2": dict(n=8, blocks=65536, scaling="weak", desc="batched FCC-DCT n=8, 65,536 blocks per GPU, i.i.d. U[-1,1] re/im"),
    "c3": dict(n=16, blocks=16384, scaling="weak",
               desc="batched FCC-DCT n=16, 16,384 blocks per GPU, 8 seeded Gaussian blobs (sigma U[0.05,0.3] x extent) + N(0,0.01) noise at the FCC node coordinates"),
    "c4": dict(n=64, blocks=1, scaling="weak", desc="single FCC-DCT n=64 (262,144 points), i.i.d. U[-1,1] re/im"),
    "c5": dict(n=8, blocks=185193, scaling="strong",
               desc="whole volume: 57^3 = 185,193 n=8 FCC blocks (~512^3 CC equivalent), 4-octave seeded Perlin noise in [0,1], sharded across GPUs"),
}


def node_real_coords(n, dev):
    """Real coordinates ((x+z)/2, Re y, (x-z)/(2i)) of the canonical skew nodes
    (real_coords, chebyshev.cpp:87-97), from the device-generated node set."""
    from paper_1807_10058_b200 import SkewParams, skew_nodes

    nodes = skew_nodes(n, SkewParams.canonical(), device=dev)
    x, y, z = nodes[:, 3], nodes[:, 4], nodes[:, 5]
    return torch_stack_real([(0.5 * (x + z)).real, y.real, ((x - z) / 2j).real])


def torch_stack_real(cols):
    import torch

    return torch.stack(cols, dim=1)


def gaussian_blobs(n, blocks, gen, dev, dtype):
    import torch

    pos = node_real_coords(n, dev).to(dtype)  # [N, 3]
    lo, hi = pos.min(0).values, pos.max(0).values
    ext = (hi - lo).max()
    out = torch.zeros((blocks, n**3), dtype=dtype, device=dev)
    for _ in range(8):
        c = lo + (hi - lo) * torch.rand((blocks, 3), generator=gen, device=dev, dtype=dtype)
        sig = ext * (0.05 + 0.25 * torch.rand((blocks, 1), generator=gen, device=dev, dtype=dtype))
        amp = torch.rand((blocks, 1), generator=gen, device=dev, dtype=dtype)
        d2 = ((pos[None, :, :] - c[:, None, :]) ** 2).sum(-1)
        out += amp * torch.exp(-0.5 * d2 / sig**2)
    out += 0.1 * torch.randn((blocks, n**3), generator=gen, device=dev, dtype=dtype)
    return out


def perlin_volume(n, b0, b1, side, gen_seed, dev, dtype):
    """4-octave gradient noise in [0,1] at block-local positions
    (bx + (i+1/2)/n, by + (j+1/2)/n, bz + (k+1/2)/n) of blocks [b0, b1) of a side^3 volume."""
    import torch

    g = torch.Generator(device="cpu").manual_seed(gen_seed)
    perm = torch.randperm(256, generator=g)
    perm = torch.cat([perm, perm]).to(dev)
    grads = torch.nn.functional.normalize(torch.randn((256, 3), generator=g), dim=1).to(dev, dtype)
    bid = torch.arange(b0, b1, device=dev)
    bx, by, bz = bid // (side * side), (bid // side) % side, bid % side
    ii = torch.arange(n, device=dev, dtype=dtype)
    off = (ii + 0.5) / n
    P = torch.stack(torch.meshgrid(off, off, off, indexing="ij"), dim=-1).reshape(-1, 3)  # [N, 3]
    pts = torch.stack([bx, by, bz], dim=1).to(dtype)[:, None, :] + P[None, :, :]  # [B, N, 3]

    def fade(t):
        return t * t * t * (t * (t * 6 - 15) + 10)

    def noise(p):
        pi = torch.floor(p).long()
        pf = p - pi
        u = fade(pf)
        res = 0
        for dx in (0, 1):
            for dy in (0, 1):
                for dz in (0, 1):
                    h = perm[(perm[(perm[(pi[..., 0] + dx) & 255] + pi[..., 1] + dy) & 255] + pi[..., 2] + dz) & 255]
                    d = pf - torch.tensor([dx, dy, dz], device=dev, dtype=dtype)
                    dot = (grads[h] * d).sum(-1)
                    w = (u[..., 0] if dx else 1 - u[..., 0]) * (u[..., 1] if dy else 1 - u[..., 1]) * (
                        u[..., 2] if dz else 1 - u[..., 2])
                    res = res + w * dot
        return res

    field = 0
    amp, freq, norm = 1.0, 1.0 / 8.0, 0.0
    for _ in range(4):
        field = field + amp * noise(pts * freq)
        norm += amp
        amp *= 0.5
        freq *= 2.0
    return (0.5 + 0.5 * field / norm).clamp(0, 1)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def launch_ranks(args) -> int:
    """`bench.py --gpus N` (N > 1) outside torchrun: start N ranks, one per GPU,
    with torch.distributed.run on 127.0.0.1 and the same arguments."""
    if not args.emulate_cpu:
        import torch

        visible = torch.cuda.device_count()
        if visible < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {visible} CUDA device(s) are visible", file=sys.stderr)
            return 1
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def workload(args, world: int) -> dict:
    """The configuration both arms measure (BASELINE.json configs restated on the
    reference's n^3 index set); the JSON `config` object is built
    here so the reference arm's equals the B200 arm's."""
    cfg = CONFIGS[args.config]
    n = args.n if args.n is not None else cfg["n"]
    precision = args.precision or ("f32" if args.config == "c5" else "f64")
    f32 = precision == "f32"
    esize = 8 if f32 else 16
    real_io = bool(args.real_io) if args.real_io is not None else args.config in ("c3", "c5")
    in_esize = esize // 2 if real_io else esize
    per_gpu = args.blocks if args.blocks is not None else cfg["blocks"]
    total = per_gpu if cfg["scaling"] == "strong" else per_gpu * world
    per_rank_max = -(-total // world)
    N = n**3
    subset = (f"; {args.blocks} blocks per GPU (a subset of the config's {cfg['blocks']:,}, labelled as such)"
              if args.blocks is not None and args.blocks != cfg["blocks"] else "")
    config = {
        "workload": f"{args.config}: {cfg['desc']}; n={n} (N={N} points/block), {args.method} path, "
                    f"forward then inverse per step{subset}",
        "blocks_total": total,
        "blocks_per_gpu_max": per_rank_max,
        "points_per_block": N,
        "params": "canonical (1/8, 0, 3/8)",
        "precision": precision,
        "io": ("real samples in and out (z_transform / grid_from_signal fused into the device pipeline)"
               if real_io else "complex in and out"),
        "input": cfg["desc"] + " (seeded, generated on device)",
        "l2": (f"inputs larger than L2 ({per_rank_max * N * in_esize / 2**20:.0f} MiB per array vs 126 MB L2), "
               "no flush needed" if per_rank_max * N * in_esize > 126e6 else
               f"input {per_rank_max * N * in_esize / 2**20:.1f} MiB is L2-resident (single-transform latency config)"),
        "parallelism": f"batch-sharded dp{world}, no collective on the data path",
    }
    return dict(cfg=cfg, n=n, N=N, precision=precision, f32=f32, esize=esize, real_io=real_io, in_esize=in_esize,
                per_gpu=per_gpu, total=total, config=config)


def reference_arm(args):
    """--impl reference: the reference's CPU path (the oracle port; the reference
    itself needs Eigen3 and cannot be built) on this host's cores,
    rank 0 only, each step a bounded sample of the same workload."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    w = workload(args, world)
    n = w["n"]
    threads = os.cpu_count() or 1
    if n > 16 or args.config == "c1":
        sample = 1
        vals = []
        for i in range(args.warmup + args.steps):
            res = cpu_baseline(args.config, n, args.method, 1, 0.0)
            if i >= args.warmup:
                vals.append(res["value"])
    else:
        # one plan build, warmup + steps timed passes over the sample (the reference arm's steps)
        sample = min(args.cpu_sample, max(1, (2**25 if args.method == "fast" else 2**17) // n**3))
        r = cpu_baseline_run(n, "batched", args.method, blocks=sample, threads=threads, reps=args.warmup + args.steps)
        vals = [2 * sample / t for t in r["rep_s"][args.warmup:]]
        res = {"cores": threads, "kind": "port",
               "sample": f"{sample} blocks of n={n} per step, forward then inverse, {args.method} path, one block "
                         "per call (the reference API), std::thread over blocks; reference-faithful C++ "
                         "restatement (oracle/cpu_baseline.cpp, -O3 -march=native)"}
    v = statistics.median(vals)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": "transforms/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * 2 * (sample if n <= 16 and args.config != "c1" else 1) / v,
        "higher_is_better": True,
        "scaling": w["cfg"]["scaling"],
        "vs_baseline": None,
        "dtype": w["precision"],
        "data": "synthetic",
        "config": w["config"],
        "points_per_s": v * n**3,
        "cpu_baseline": {"value": v, "unit": "transforms/s", "cores": res["cores"], "kind": res["kind"],
                         "sample": res["sample"]},
        "e2e": {"value": v, "unit": "transforms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def emulated_arm(args):
    """--emulate-cpu: the multi-rank launcher end to end without a GPU (gloo).
    Each rank transforms its shard through the host emulation of the orbit-FFT
    executor's compiled tables (the exact kernel indexing); timing is wall clock,
    max over ranks. Test infrastructure for the launcher, not a measurement."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1807_10058_b200 import _capi, shard_range

    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    w = workload(args, world)
    n, N = w["n"], w["N"]
    b0, b1 = shard_range(w["total"], rank, world)
    rng = np.random.default_rng(1234 + rank)
    x = rng.uniform(-1, 1, (b1 - b0, N)) + 1j * rng.uniform(-1, 1, (b1 - b0, N))
    y, z = np.zeros_like(x), np.zeros_like(x)
    L = _capi.lib()

    def step():
        if b1 > b0:
            assert L.fcct_debug_emulate_orbit_fft(n, 0.125, 0.0, 0.375, 0, x.ctypes.data, y.ctypes.data, b1 - b0) == 0
            assert L.fcct_debug_emulate_orbit_fft(n, 0.125, 0.0, 0.375, 1, y.ctypes.data, z.ctypes.data, b1 - b0) == 0

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    ms = 1e3 * (time.perf_counter() - t0)
    err = float(np.linalg.norm(z - x) / max(np.linalg.norm(x), 1e-300))
    shards = [(b0, b1)]
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        e = torch.tensor([err], dtype=torch.float64)
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
        err = e.item()
        gathered = [None] * world
        dist.all_gather_object(gathered, (b0, b1))
        shards = gathered
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    value = 2.0 * w["total"] * args.steps / (ms / 1e3)
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "transforms/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": w["cfg"]["scaling"], "vs_baseline": None, "dtype": w["precision"], "data": "synthetic",
        "config": w["config"], "emulated": "CPU host emulation of the orbit-FFT tables over gloo (launcher test)",
        "shards": shards, "roundtrip_rel_err": err, "gpu_launches": 0,
    }), flush=True)


def b200_arm(args):
    import torch
    import torch.distributed as dist

    from paper_1807_10058_b200 import SkewParams, build_plan, dense_transform, shard_range

    world, rank, local = dist_env()
    visible = torch.cuda.device_count()
    if visible < max(1, world) or visible == 0:
        raise SystemExit(f"bench.py: {world} rank(s) need {world} CUDA device(s), {visible} visible")
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device(f"cuda:{local if world > 1 else 0}")
    torch.cuda.set_device(dev)
    w = workload(args, world)
    cfg, n, N, f32 = w["cfg"], w["n"], w["N"], w["f32"]
    esize, in_esize, real_io, total = w["esize"], w["in_esize"], w["real_io"], w["total"]
    cdt = torch.complex64 if f32 else torch.complex128
    rdt = torch.float32 if f32 else torch.float64
    p = SkewParams.canonical()
    b0, b1 = shard_range(total, rank, world)
    blocks = b1 - b0

    if args.method == "fast":
        plan = build_plan(n, p, precision=w["precision"], executor=args.executor)
    else:
        plan = dense_transform(n, p, precision=w["precision"])._plan
    info = plan.info

    # seeded synthetic input, resident in HBM before the timed region
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    # real fields (c3, c5) enter and leave as real samples: z_transform / grid_from_signal
    # fused into the device pipelines, as the reference CLI uses them (fcct.cpp:95-129)
    if args.config == "c3":
        x = gaussian_blobs(n, blocks, g, dev, rdt)
    elif args.config == "c5":
        side = round(total ** (1.0 / 3.0))
        x = perlin_volume(n, b0, b1, side, 5, dev, rdt)
    else:
        x = torch.complex(torch.rand((blocks, N), generator=g, device=dev, dtype=rdt) * 2 - 1,
                          torch.rand((blocks, N), generator=g, device=dev, dtype=rdt) * 2 - 1).to(cdt)
    if not x.is_complex() and not real_io:
        x = x.to(cdt)
    if x.is_complex() and real_io:
        x = x.real.contiguous()
    y = torch.empty((blocks, N), dtype=cdt, device=dev)
    z = torch.empty_like(x)
    fwd_fn = "fcct_forward_real" if real_io else "fcct_forward"
    inv_fn = "fcct_inverse_real" if real_io else "fcct_inverse"
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    from paper_1807_10058_b200 import _capi
    from paper_1807_10058_b200.fcct import _raise

    L = _capi.lib()

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        _raise(getattr(L, fwd_fn)(plan._h, x.data_ptr(), y.data_ptr(), blocks, sh))
        if ev is not None:
            ev[1].record(stream)
        _raise(getattr(L, inv_fn)(plan._h, y.data_ptr(), z.data_ptr(), blocks, sh))
        if ev is not None:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    # correctness guard on the benchmarked data (size-independent property)
    err = (torch.linalg.norm(z - x) / torch.linalg.norm(x)).item()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index) as clk:
        start.record(stream)
        for i in range(args.steps):
            step(evs[i])
        end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(end)
    fwd_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    inv_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    per_rank_ms = [ms]
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        per_rank_ms = [float(v.item()) for v in gathered]
        ms = max(per_rank_ms)
    value = 2.0 * total * args.steps / (ms / 1e3)

    # e2e: the reference-facing host-buffer API (H2D + transform + D2H in every
    # call), from pinned and from pageable host memory (staged by the library)
    def e2e_run(pinned: bool):
        eb = max(1, min(blocks, args.e2e_blocks))
        xh = x[:eb].cpu()
        yh = torch.empty((eb, N), dtype=cdt)
        zh = torch.empty_like(xh)
        if pinned:
            xh, yh, zh = xh.pin_memory(), yh.pin_memory(), zh.pin_memory()
        fwd_host = getattr(L, fwd_fn + "_host")
        inv_host = getattr(L, inv_fn + "_host")
        for _ in range(2):
            _raise(fwd_host(plan._h, xh.data_ptr(), yh.data_ptr(), eb, sh))
            _raise(inv_host(plan._h, yh.data_ptr(), zh.data_ptr(), eb, sh))
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            _raise(fwd_host(plan._h, xh.data_ptr(), yh.data_ptr(), eb, sh))
            _raise(inv_host(plan._h, yh.data_ptr(), zh.data_ptr(), eb, sh))
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        ok = bool(torch.allclose(zh.to(x.dtype), x[:eb].cpu(), rtol=0, atol=1e-4 if f32 else 1e-9))
        return {
            "value": 2.0 * eb * world * args.e2e_steps / (ems / 1e3),
            "unit": "transforms/s",
            "h2d_bytes_per_step": eb * N * (in_esize + esize),
            "d2h_bytes_per_step": eb * N * (esize + in_esize),
            "blocks_per_step": eb,
            "host_memory": "pinned (cudaHostAlloc)" if pinned else "pageable (staged through pinned bounce buffers)",
            "roundtrip_ok": ok,
        }

    e2e = e2e_pageable = None
    if not args.no_e2e:
        e2e = e2e_run(pinned=True)
        e2e_pageable = e2e_run(pinned=False)
    launches = args.steps * sum(launches_per_call(info))

    if world > 1:
        lt = torch.tensor([launches, blocks], device=dev, dtype=torch.int64)
        lg = [torch.zeros_like(lt) for _ in range(world)]
        dist.all_gather(lg, lt)
        per_rank = [{"rank": r, "gpu_launches": int(v[0]), "blocks": int(v[1]), "ms": per_rank_ms[r]}
                    for r, v in enumerate(lg)]
    else:
        per_rank = [{"rank": 0, "gpu_launches": launches, "blocks": blocks, "ms": ms}]
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel (the forward pipeline launch)
    flops_fwd = info.flops_forward * blocks
    # algorithmic bytes of one forward launch: the data once in and once out, plus
    # the plan tables streamed once (about half of table_bytes, which counts both
    # directions) — negligible for batched configs, dominant for a single n = 64
    data_bytes = float(N * (in_esize + esize) * blocks)
    table_bytes_fwd = float(info.table_bytes_forward) if info.executor in (3, 7) else 0.0
    bytes_fwd = data_bytes + table_bytes_fwd
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6488.0)
    # the roofline of the pipe that executes the plan: the FP64 tensor pipe for
    # the DMMA executors (fp32 plans there keep fp64 arithmetic, complex64 I/O)
    on_fp64_pipe = (not f32) or info.executor in (2, 4, 5, 6, 7, 10)
    on_tcgen05 = info.executor in (8, 9)
    peak_tf = (TF32_PEAK_TFLOPS if info.executor == 8 else INT8_PEAK_TOPS) if on_tcgen05 else (
        FP64_PEAK_TFLOPS if on_fp64_pipe else FP32_PEAK_TFLOPS)
    exec_flops = ((w["real_io"] and info.exec_flops_forward_real) or info.exec_flops_forward or info.flops_forward) * blocks
    achieved_tf = exec_flops / (fwd_ms / 1e3) / 1e12
    achieved_gbs = bytes_fwd / (fwd_ms / 1e3) / 1e9
    t_hbm, t_pipe = bytes_fwd / (hbm * 1e9), exec_flops / (peak_tf * 1e12)
    hbm_bound = t_hbm >= t_pipe
    # frac: the kernel against its OWN work (executed flops, algorithmic bytes)
    roof = {
        "bound": "hbm" if hbm_bound else "tensor",
        "achieved": achieved_gbs if hbm_bound else achieved_tf,
        "peak": hbm if hbm_bound else peak_tf,
        "unit": "GB/s" if hbm_bound else "TFLOP/s",
        "frac": max(t_hbm, t_pipe) / (fwd_ms / 1e3),
        "traffic": args.traffic if args.traffic is not None else profiled_traffic(args.config, f32, info.executor),
        "kernel": KERNELS[info.executor],
        "executed_flops_per_launch": exec_flops,
        "algorithmic_flops_per_launch": flops_fwd,
        "algorithmic_bytes_per_launch": bytes_fwd,
        "table_bytes_per_launch": table_bytes_fwd,
        "achieved_tflops_executed": achieved_tf,
        "achieved_gbs": achieved_gbs,
        "hbm_frac": achieved_gbs / hbm,
        "hbm_peak_gbs": hbm,
        "pipe_peak_tflops": peak_tf,
        "t_star_algorithmic_over_t": max(t_hbm, flops_fwd / (peak_tf * 1e12)) / (fwd_ms / 1e3),
        "peak_source": (("dense TF32 tensor-core peak 1.1 PFLOP/s, the B200_PROFILING.md fallback (no measured TF32 "
                         "figure; MEASURED_PEAKS.json bf16 burst / 2 = %.0f TF/s)" % (peaks.get("bf16_tflops", 0) / 2))
                        if info.executor == 8 else
                        "dense INT8 tensor-core peak 4.5 POPS, the B200_PROFILING.md fallback (executed = 28 int8 slice "
                        "products per algorithmic fp64 op; TOPS)" if info.executor == 9 else
                        ("measured DMMA m8n8k4 f64 peak" if on_fp64_pipe else "measured FFMA fp32 peak")
                        + " (tools/peak_fp.cu, profiles/r01_fp_peaks.txt)") + "; HBM: MEASURED_PEAKS.json hbm_gbs (burst)",
        "fwd_ms": fwd_ms,
        "inv_ms": inv_ms,
        "note": ("frac = max(algorithmic bytes / HBM peak, executed flops / pipe peak) / forward launch time: the "
                 "kernel against its own work. t_star_algorithmic_over_t uses SURVEY.md 8(d)'s tree flop count "
                 "instead (the orbit-FFT executors issue fewer flops than the tree, so that ratio can exceed frac)"),
    }
    if info.executor == 6 and roof["traffic"] is not None:
        roof["traffic_note"] = ("two kernels per forward call: the base change writes z (complex128, orbit order) "
                                "and the cube FFT reads it back, 2 x 16 B per point by design on top of the "
                                "algorithmic bytes")
    cpu = None
    if not args.no_cpu:
        sample = min(args.cpu_sample, max(1, (2**24 if args.method == "fast" else 2**16) // N))
        cpu = cpu_baseline(args.config, n, args.method, sample, args.cpu_seconds)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "transforms/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": cfg["scaling"],
        "vs_baseline": None,
        "dtype": w["precision"],
        "data": "synthetic",
        "config": w["config"],
        "points_per_s": value * N,
        "roundtrip_rel_err": err,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_pageable": e2e_pageable if not args.no_e2e else None,
        "gpu_launches": launches,
        "gpu_launches_per_rank": per_rank,
        "clocks": clk.summary(),
        "plan": {"tree_nnz": info.tree_nnz, "tree_nnz_inv": info.tree_nnz_inv, "table_bytes": info.table_bytes,
                 "flops_forward_per_block": info.flops_forward, "flops_inverse_per_block": info.flops_inverse,
                 "exec_flops_forward_per_block": info.exec_flops_forward, "executor": info.executor},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


KERNELS = {0: "gemm_f64_kernel / gemm_f32_kernel (direct)", 1: "pipeline_kernel (tile interpreter)",
           2: "pipeline2_kernel (FP64 tensor pipe)", 3: "gstage_* kernels (global multi-pass)",
           4: "root pass + 8 x pipeline2_kernel (two-level, FP64 tensor pipe)",
           5: "orbit_fft_ws_kernel (S_n on the FP64 tensor pipe + radix-2 FFT, warp-specialised)",
           6: "orbit16_base_kernel + fft_cube_kernel (two-pass orbit-FFT: S_n on the FP64 tensor pipe, then the n^3 FFT)",
           7: "orbit_big_s_kernel + line_fft_kernel (large-n orbit-FFT: S_n then three line-FFT passes)",
           8: "gemm_tf32x3_kernel (direct, tcgen05.mma kind::tf32 x3 split, TMEM accumulator, TMA tensor maps)",
           9: "ozaki_slice_kernel + gemm_ozaki_kernel (direct fp64, tcgen05.mma kind::i8 on 7 int8 slices, TMEM)",
           10: "orbit_pat_kernel (single pass: the block resident in shared memory, constant-operator DMMA base change "
               "over the block's own orbits + the n^3 FFT)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--blocks", type=int, default=None, help="blocks per GPU (weak) / in total (strong)")
    ap.add_argument("--method", default="fast", choices=["fast", "direct"])
    ap.add_argument("--precision", default=None, choices=["f64", "f32"])
    ap.add_argument("--cpu-sample", type=int, default=65536)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="minimum CPU work of the cpu_baseline leg")
    ap.add_argument("--real-io", type=int, default=None, help="1/0: real samples in and out (default: c3 and c5)")
    ap.add_argument("--e2e-blocks", type=int, default=65536)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--emulate-cpu", action="store_true", help="launcher test without a GPU (gloo, host emulation)")
    ap.add_argument("--executor", default="auto", help="force a fast executor (fcct.EXECUTORS; A/B runs)")
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes per launch (from profiles/)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        sys.exit(launch_ranks(args))
    if world and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} under a world of {world} ranks", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        reference_arm(args)
    elif args.emulate_cpu:
        emulated_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
