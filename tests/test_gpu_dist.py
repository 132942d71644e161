"""The distributed (z-slab) solve on one B200: ranks emulated as threads (ThreadComm).

Each virtual rank has its own rd context and CUDA stream and runs the product
path (DeviceOps: row blocks, slab smoother, PCG updates through the C-ABI);
planes move between ranks through stream events, so no kernel ever waits on a
kernel of another rank (B200_PROFILING.md: waiting ranks must not share a GPU).
Checked against the single-GPU path, which the parity suite pins to the oracle:
  * exact mode: the V-cycle equals rd_gpu_amg_apply bit for bit; the PCG takes
    the same iteration count and agrees to 1e-10 (dots reduce in another order);
  * block mode: converges in about as many iterations.
"""
import os
import sys
import threading

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def _run_ranks(world, n, rho, target, mode, gather_rows, solve=True, release=False):
    import torch

    from paper_2102_03515_b200 import rd
    from paper_2102_03515_b200.dist import DeviceOps, DistSolver, ThreadComm

    hub = ThreadComm.hub(world)
    outs = [None] * world
    errs = []

    def body(rank):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = rd.Context(0, s.cuda_stream)
                ops = DeviceOps(n, rho, target, ctx=ctx)
                solver = DistSolver(ThreadComm(hub, rank), ops, gather_rows=gather_rows, mode=mode,
                                    release_replicated=release)
                z = ops.vec(0)
                solver.apply(ops.f_local, z)
                zf = solver.gather_solution(solver.own(0, z))
                out = dict(G=solver.G, cuts=solver.plan.cuts, launches0=ctx.launch_count,
                           kept=(ops.sys is not None, ops.h is not None), pool=ctx.pool_bytes())
                if solve:
                    res = solver.pcg(1e-8, 500)
                    xf = solver.gather_solution(res.x_local)
                    out.update(it=res.iterations, conv=res.converged, hist=res.residual_history,
                               rerun=res.exact_rerun)
                    if rank == 0:
                        out["x"] = xf.cpu().numpy()
                if rank == 0:
                    out["z"] = zf.cpu().numpy()
                s.synchronize()
                outs[rank] = out
        except Exception:
            import traceback

            errs.append(traceback.format_exc())

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not errs, errs[0]
    return outs


def _single(n, rho, target):
    from paper_2102_03515_b200 import rd

    mesh = rd.build_structured_cube(n)
    sys_ = rd.build_system(mesh, rho, target)
    h = rd.build_amg(sys_.A)
    f = sys_.f()
    z = h.apply(f)
    res = rd.pcg(sys_.A, "amg", f, 1e-8, 500, hierarchy=h)
    return dict(z=z, x=res.x, it=res.iterations)


@pytest.mark.parametrize("mode", ["exact", "pipelined"])
@pytest.mark.parametrize("world,gather_rows,G", [(2, 600, 2), (4, 600, 2), (3, 100000, 1)])
def test_exact_slabs_match_single_gpu(world, gather_rows, G, mode):
    """exact: planes handed on between sweeps; pipelined: the sweep kernels write the
    boundary cells into the next slab's buffer (all slabs in one cooperative launch)."""
    n, rho = 32, 2.0 ** -10
    ref = _single(n, rho, "smooth")
    outs = _run_ranks(world, n, rho, "smooth", mode, gather_rows)
    o0 = outs[0]
    assert o0["G"] == G
    assert np.array_equal(o0["z"], ref["z"])  # the V-cycle, bit for bit
    assert all(o["it"] == ref["it"] and o["conv"] for o in outs)
    assert all(o["hist"] == o0["hist"] for o in outs)
    err = np.abs(o0["x"] - ref["x"]).max() / np.abs(ref["x"]).max()
    assert err <= 1e-10, err


@pytest.mark.parametrize("mode", ["exact", "pipelined"])
def test_replicated_setup_released_after_localisation(mode):
    """release_replicated: the whole-box system goes on every rank and the hierarchy on ranks
    > 0 once the row blocks and slab smoothers exist; the solve is unchanged."""
    n, rho = 32, 2.0 ** -10
    ref = _single(n, rho, "smooth")
    outs = _run_ranks(2, n, rho, "smooth", mode, 600, release=True)
    assert outs[0]["kept"] == (False, True) and outs[1]["kept"] == (False, False)
    assert all(o["pool"][0] > 0 and o["pool"][1] >= o["pool"][0] for o in outs)
    assert np.array_equal(outs[0]["z"], ref["z"])
    assert all(o["it"] == ref["it"] and o["conv"] for o in outs)
    err = np.abs(outs[0]["x"] - ref["x"]).max() / np.abs(ref["x"]).max()
    assert err <= 1e-10, err


def test_block_slabs_converge():
    n, rho = 32, 2.0 ** -10
    ref = _single(n, rho, "smooth")
    outs = _run_ranks(4, n, rho, "smooth", "block", 600)
    o0 = outs[0]
    assert all(o["conv"] for o in outs)
    assert abs(o0["it"] - ref["it"]) <= 2
    err = np.abs(o0["x"] - ref["x"]).max() / np.abs(ref["x"]).max()
    assert err <= 1e-6, err


@pytest.mark.parametrize("mode,world", [("exact", 2), ("pipelined", 2), ("pipelined", 4)])
def test_exact_slabs_c2_vcycle(mode, world):
    """C2 (n=128, ball target): slabs of 64 / 63 planes (a partial last tile), the
    level-0 V-cycle through the slab kernels equals the single-GPU V-cycle bit for bit."""
    n, rho = 128, 2.0 ** -14
    from paper_2102_03515_b200 import rd

    mesh = rd.build_structured_cube(n)
    sys_ = rd.build_system(mesh, rho, "ball")
    h = rd.build_amg(sys_.A)
    zref = h.apply(sys_.f())
    del h, sys_, mesh
    outs = _run_ranks(world, n, rho, "ball", mode, 262144, solve=False)
    assert outs[0]["G"] == 1 and outs[0]["cuts"][0] == 0 and outs[0]["cuts"][-1] == 127
    assert np.array_equal(outs[0]["z"], zref)


def test_pipelined_slabs_c2_solve():
    """C2 solved on 2 pipelined slabs: the single-GPU iteration count and solution (1e-10)."""
    n, rho = 128, 2.0 ** -14
    ref = _single(n, rho, "ball")
    outs = _run_ranks(2, n, rho, "ball", "pipelined", 262144)
    o0 = outs[0]
    assert all(o["conv"] and o["it"] == ref["it"] for o in outs)
    assert np.array_equal(o0["z"], ref["z"])
    err = np.abs(o0["x"] - ref["x"]).max() / np.abs(ref["x"]).max()
    assert err <= 1e-10, err
