"""N > 1 path of bench.py on CPU (gloo, world_size 2): replicas only, max-over-ranks timing,
whole-job value; the reference arm runs on rank 0 only. No GPU needed."""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local_ms = 100.0 * (rank + 1)  # rank 1 is the slow one
    value, ms = bench.replica_aggregate(5, local_ms, world, bench.torch_reduce_max("cpu"))
    q.put((rank, value, ms))
    dist.destroy_process_group()


def test_replica_aggregation_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    for rank, value, ms in res:
        assert ms == 200.0                       # max over ranks
        assert abs(value - 2 * 5 / 0.2) < 1e-9   # all ranks' evaluations / slowest rank's time


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_bench_self_launches_n_ranks():
    """`bench.py --gpus 2` with WORLD_SIZE unset starts 2 replica ranks itself;
    --mock replaces the GPU evaluation by a per-rank sleep (rank 1 slower): n_gpus = 2 and the
    time is the max over ranks."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--mock",
                        "--steps", "5", "--warmup", "0"], env=env, capture_output=True, text=True,
                       timeout=180)
    assert r.returncode == 0, r.stderr[-2000:]
    import json
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["mock"] is True
    assert line["max_ms"] >= line["local_ms"] and line["max_ms"] >= 5 * 20.0  # rank 1: 20 ms/step
    assert abs(line["value"] - 2 * 5 / (line["max_ms"] * 1e-3)) < 1e-6 * line["value"]
