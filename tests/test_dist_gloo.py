"""The distributed (z-slab) solve of dist.py on CPU: world_size-2 gloo process groups.

Each rank runs DistSolver with the oracle-backed HostOps (tests/dist_host_ops.py),
so the host logic -- slab plan, halo planes, the exact smoother hand-off between
ranks, the gather of the coarse levels onto rank 0, the rank-ordered dot sums --
is checked against the single-process oracle:
  * exact mode: the distributed V-cycle equals the oracle's amg_apply bit for bit;
    the PCG takes the oracle's iteration count and its solution agrees to 1e-10;
  * block mode: a different (processor-block) preconditioner, still converging in
    about as many iterations.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, n, rho, target, mode, gather_rows):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        from paper_2102_03515_b200.dist import DistSolver, TorchComm
        from dist_host_ops import HostOps

        ops = HostOps(n, rho, target)
        comm = TorchComm()
        s = DistSolver(comm, ops, gather_rows=gather_rows, mode=mode)
        z = ops.vec(0)
        s.apply(ops.f_local, z)
        zfull = s.gather_solution(s.own(0, z))
        res = s.pcg(1e-8, 500)
        xfull = s.gather_solution(res.x_local)
        out = dict(rank=rank, G=s.G, cuts=s.plan.cuts, it=res.iterations, conv=res.converged,
                   hist=list(res.residual_history))
        if rank == 0:
            out["z"] = zfull.numpy().copy()
            out["x"] = xfull.numpy().copy()
        q.put(out)
    except Exception as e:  # surface the failure in the parent
        import traceback

        q.put(dict(rank=rank, error=traceback.format_exc() + repr(e)))
    finally:
        torch.distributed.destroy_process_group()


def _run(world, n, rho, target, mode, gather_rows):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, n, rho, target, mode, gather_rows))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted((q.get(timeout=600) for _ in procs), key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=120)
    for o in outs:
        assert "error" not in o, o["error"]
    for p in procs:
        assert p.exitcode == 0
    return outs


@pytest.fixture(scope="module")
def oracle_ref(O):
    n, rho = 16, 1.0 / 256.0
    mesh = O.build_structured_cube(n)
    sys_ = O.build_system(mesh, rho, "smooth")
    h = O.build_amg(sys_.A)
    z = h.apply(sys_.f)
    res = O.pcg(sys_.A, "amg", sys_.f, 1e-8, 500, hierarchy=h)
    return dict(n=n, rho=rho, z=z, x=res.x, it=res.iterations)


def test_exact_world2_matches_oracle(oracle_ref):
    ref = oracle_ref
    outs = _run(2, ref["n"], ref["rho"], "smooth", "exact", gather_rows=100)
    o0 = outs[0]
    assert o0["G"] == 2 and o0["cuts"] == [0, 8, 15]  # levels 0, 1 cut at z = 8 / 4; 4^3 gathered
    # the V-cycle is the single-process V-cycle, bit for bit
    assert np.array_equal(o0["z"], ref["z"])
    # PCG: same iteration count, the same scalars on every rank, solution within 1e-10
    assert all(o["it"] == ref["it"] for o in outs) and all(o["conv"] for o in outs)
    assert outs[0]["hist"] == outs[1]["hist"]
    err = np.abs(o0["x"] - ref["x"]).max() / np.abs(ref["x"]).max()
    assert err <= 1e-10, err


def test_exact_world2_one_distributed_level(oracle_ref):
    ref = oracle_ref
    outs = _run(2, ref["n"], ref["rho"], "smooth", "exact", gather_rows=4096)
    assert outs[0]["G"] == 1  # only level 0 cut; levels 1.. gathered onto rank 0
    assert np.array_equal(outs[0]["z"], ref["z"])
    assert outs[0]["it"] == ref["it"]


def test_block_world2_converges(oracle_ref):
    ref = oracle_ref
    outs = _run(2, ref["n"], ref["rho"], "smooth", "block", gather_rows=100)
    o0 = outs[0]
    assert all(o["conv"] for o in outs)
    assert abs(o0["it"] - ref["it"]) <= 2  # processor-block SGS: a different preconditioner
    assert not np.array_equal(o0["z"], ref["z"])
    err = np.abs(o0["x"] - ref["x"]).max() / np.abs(ref["x"]).max()
    assert err <= 1e-6, err  # both solve A x = f to rtol 1e-8


def test_slab_plan_alignment():
    sys.path.insert(0, ROOT)
    from paper_2102_03515_b200.dist import SlabPlan, choose_dist_levels

    p = SlabPlan([127, 64, 32, 16, 8, 4], 8, 2)
    assert all(c % 4 == 0 for c in p.cuts[:-1])
    for l in range(3):
        owned = [p.owned(l, r) for r in range(8)]
        assert owned[0][0] == 0 and owned[-1][1] == p.sides[l]
        assert all(owned[r][1] == owned[r + 1][0] for r in range(7))
    # C2 with a 262,144-row gather threshold: only level 0 is cut
    sides = [127, 64, 32, 16, 8, 4]
    rows = [127 ** 3, 64 ** 3, 32 ** 3, 16 ** 3, 8 ** 3, 4 ** 3]
    assert choose_dist_levels(sides, rows, [True] * 6, 8, 262144) == 1
    # by cost (>= 65,536 rows per rank): 2 and 4 ranks cut levels 0-1, 8 ranks level 0 only
    assert choose_dist_levels(sides, rows, [True] * 6, 2) == 2
    assert choose_dist_levels(sides, rows, [True] * 6, 4) == 2
    assert choose_dist_levels(sides, rows, [True] * 6, 8) == 1
    # C4 (n = 256) on 8 ranks: levels 0 and 1 (level 1: 2,097,152 / 8 = 262,144 rows per rank)
    s4 = [255, 128, 64, 32, 16, 8, 4]
    r4 = [s ** 3 for s in s4]
    assert choose_dist_levels(s4, r4, [True] * 7, 8) == 2
    with pytest.raises(ValueError):
        SlabPlan([7, 4, 2], 8, 1)
