"""The N > 1 plumbing of bench.py on CPU: world_size-2 gloo process groups.

job_rate is the timing reduction of bench.py --replicas (MAX over ranks of the device
time, SUM of the work); the default N > 1 path is the slab-distributed solve, whose host
logic tests/test_dist_gloo.py covers.  The reference arm runs on rank 0 alone.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench

    # rank r measured (r + 1) * 10 ms for 100 * (r + 1) units of work
    t, rate = bench.job_rate(10.0 * (rank + 1), 100.0 * (rank + 1), world)
    q.put((rank, t, rate))
    torch.distributed.destroy_process_group()


def test_job_rate_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, t, rate in out:
        assert t == 20.0  # MAX over ranks
        assert rate == pytest.approx(300.0 / 0.020)  # SUM of work / max time


def test_job_rate_single_rank():
    sys.path.insert(0, ROOT)
    import bench

    t, rate = bench.job_rate(4.0, 8.0, 1)
    assert t == 4.0 and rate == pytest.approx(2000.0)


def test_reference_arm_torchrun_world2():
    """bench.py --impl reference under torchrun: rank 0 prints one JSON line, rank 1 exits 0."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--cells", "8"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
