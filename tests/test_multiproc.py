"""N > 1 host logic of bench.py on CPU with gloo, world_size 2 (the GPU path runs one replica per
rank with no data-path collective; the only collective is the max-over-ranks timing reduction).
DESIGN.md §10: replicas only."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = bench.max_over_ranks(10.0 * (rank + 1), world, torch.device("cpu"))
        Pb = bench.replica_problem("c1", rank)
        q.put((rank, t, Pb.seed, float(Pb.u[0][0]), Pb.n, bench.aggregate_rate(world, 5, t)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_max_over_ranks_and_replicas():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    (r0, t0, s0, u0, n0, v0), (r1, t1, s1, u1, n1, v1) = res
    assert t0 == t1 == 20.0                      # every rank sees the slowest rank's time
    assert v0 == v1 == 2 * 5 / 0.020            # whole-job throughput: world * steps / max time
    assert n0 == n1 and s1 == s0 + 1000 and u0 != u1   # same shapes, independent problem per rank


def test_single_rank_helpers():
    assert bench.max_over_ranks(3.5, 1, None) == 3.5
    Pb0 = bench.replica_problem("c2", 0)
    Pb1 = bench.replica_problem("c2", 1)
    assert Pb0.stencil == Pb1.stencil and Pb0.n == Pb1.n
    assert not np.array_equal(Pb0.u[0], Pb1.u[0])


def test_reference_arm_under_torchrun_prints_once():
    # bench.py --impl reference under torchrun with 2 ranks: rank 0 times the oracle and prints one
    # JSON line, rank 1 exits 0 without work
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", "bench.py", "--impl", "reference",
           "--gpus", "2", "--config", "c1", "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    assert lines[0]["value"] > 0 and lines[0]["e2e"]["h2d_bytes_per_step"] == 0
