"""The multi-GPU pipelined hand-off's IPC path, on one B200 without waiting kernels.

Two processes (gloo for the host plumbing) each own one z-slab of the n=32 lattice
and map the other's cell buffer with CUDA IPC (rd_gpu_slab_ipc_handle /
rd_gpu_slab_open_peer), exactly as the ranks of a multi-GPU run do.  The sweeps
are serialised on the host (the upstream rank's kernel finishes before the
downstream rank launches), so no kernel ever waits on a kernel of the other
process (B200_PROFILING.md), yet every boundary cell crosses the process
boundary through the peer store of the sweep kernel.  The two slab sweeps must
reproduce the single-GPU forward and backward passes bit for bit.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    sys.path.insert(0, ROOT)
    try:
        from paper_2102_03515_b200 import rd
        from paper_2102_03515_b200.dist import DeviceOps, SlabPlan, TorchComm

        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ctx = rd.Context(0, s.cuda_stream)
            n, rho = 32, 2.0 ** -10
            ops = DeviceOps(n, rho, "smooth", ctx=ctx)
            plan = SlabPlan(ops.sides, 2, 1)
            ops.localize(plan, rank)
            TorchComm().link_slabs(ops, 1)
            L = plan.sides[0]
            P = L * L
            g = torch.Generator().manual_seed(7)
            xin_full = torch.rand(L ** 3, generator=g, dtype=torch.float64).cuda()
            f_full = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
            f_full.copy_(torch.from_numpy(ops.sys.f()))
            lo, hi = plan.owned(0, rank)
            g0, g1 = plan.ghost(0, rank)
            xin = xin_full[g0 * P:g1 * P].clone()
            f = f_full[g0 * P:g1 * P].clone()
            outs = {}
            for fwd in (True, False):
                xout = ops.vec(0)
                first = 0 if fwd else 1  # the upstream rank of this pass runs first
                for who in (first, 1 - first):
                    if rank == who:
                        ops.sweep_pipelined(0, fwd, f, xin, xout)
                        ops.ctx.synchronize()
                    dist.barrier()
                outs[fwd] = xout[(lo - g0) * P:(hi - g0) * P].cpu()
            ref = {}
            if rank == 0:
                for fwd in (True, False):
                    y = torch.empty_like(xin_full)
                    ops.h.level_sweep(0, fwd, f_full, xin_full, y)
                    ref[fwd] = y.cpu()
            for fwd in (True, False):
                parts = [torch.empty(plan.owned(0, r)[1] * P - plan.owned(0, r)[0] * P, dtype=torch.float64)
                         for r in range(2)]
                if rank == 0:
                    parts[0].copy_(outs[fwd])
                    dist.recv(parts[1], 1)
                    got = torch.cat(parts).numpy()
                    q.put((fwd, bool(np.array_equal(got, ref[fwd].numpy())),
                           float(np.abs(got - ref[fwd].numpy()).max())))
                else:
                    dist.send(outs[fwd], 0)
            s.synchronize()
    except Exception:
        import traceback

        q.put(("error", traceback.format_exc(), 0.0))
    finally:
        dist.destroy_process_group()


def test_pipelined_ipc_two_processes():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[0] != "error", r[1]
    assert all(ok for (_, ok, _) in res), res
    for p in procs:
        assert p.exitcode == 0
