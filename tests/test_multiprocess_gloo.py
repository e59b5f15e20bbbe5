"""World-size-2 tests of the multi-GPU batch scheduler on CPU (gloo).

The B200 path shards independent blocks across ranks with no collective on
the data path; bench.py times each rank and reduces the
elapsed time with a MAX all-reduce. Here two gloo ranks run the same
sharding, transform their shards through the host emulation of the compiled
DMMA stage tables (the exact kernel indexing, no GPU), and the gathered result
must equal the single-process result bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_SIZE = 4
TOTAL = 37  # ragged: not divisible by the world size


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _emulate(x, n=N_SIZE, inverse=0):
    from paper_1807_10058_b200 import _capi

    y = np.zeros_like(x)
    if len(x):
        st = _capi.lib().fcct_debug_emulate_v2(n, 0.125, 0.0, 0.375, inverse, x.ctypes.data, y.ctypes.data, len(x))
        assert st == 0
    return y


def _inputs():
    rng = np.random.default_rng(2024)
    return rng.uniform(-1, 1, (TOTAL, N_SIZE**3)) + 1j * rng.uniform(-1, 1, (TOTAL, N_SIZE**3))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_1807_10058_b200 import shard_range

        w, r, _ = bench.dist_env()
        assert (w, r) == (world, rank)
        b0, b1 = shard_range(TOTAL, rank, world)
        x = np.ascontiguousarray(_inputs()[b0:b1])
        y = _emulate(x)
        back = _emulate(np.ascontiguousarray(y), inverse=1)
        parts = [None] * world
        dist.all_gather_object(parts, (b0, b1, y, back))
        # max-over-ranks timing reduction as bench.py does it
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            q.put((parts, t.item()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharded_transform_matches_single_process():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == float(world)
    parts.sort(key=lambda t: t[0])
    assert parts[0][0] == 0 and parts[-1][1] == TOTAL
    y = np.concatenate([p[2] for p in parts])
    back = np.concatenate([p[3] for p in parts])
    x = _inputs()
    assert np.array_equal(y, _emulate(x))  # sharding does not change a bit
    assert np.linalg.norm(back - x) / np.linalg.norm(x) < 1e-13
