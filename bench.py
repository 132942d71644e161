#!/usr/bin/env python
"""Benchmark of the B200-native AMG-PCG solve path (BASELINE.json configs[1] = C2).

Workload (C2): unit cube, n = 128 cells per side (127^3 = 2,048,383 interior dofs,
30.3M nnz), rho = h^2 = 2^-14, ball target (64-point rule), fp64 AMG-PCG to
rtol 1e-8 from a zero initial guess.  Synthetic and seeded: the mesh is generated,
not loaded.

One *step* = one pass of the whole hot path over that input:
    build_system (device assembly of rho*K + M and f)  ->  build_amg (device setup)
    ->  pcg with the AMG V-cycle (device-resident).
`value` = DOF * PCG iterations / step time (inputs resident in HBM: the device
mesh is built before the timed region), aggregated over ranks.  `e2e` = the same
metric through the C-ABI with HOST buffers: the pinned host TetMesh is uploaded
(rd_gpu_mesh_create), assembled, solved, and u read back, every step.

--impl reference times the CPU oracle port (oracle/, the reference cannot be built
here: no Eigen) on the host cores for the same config and metric.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEFAULT = 128
RHO_EXP = -14  # rho = h^2 = 2^-14 at n = 128
TARGET = "ball"
TOL = 1e-8
METRIC = "AMG-PCG DOF*iters/s (C2: n=128, 2.05M dofs, fp64, rho=h^2, rtol 1e-8)"
UNIT = "DOF*iters/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cells", "--n", dest="n", type=int, default=N_DEFAULT, help="cells per cube side")
    p.add_argument("--target", default=TARGET)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the C4 / C5 single-GPU runs")
    p.add_argument("--profile", action="store_true", help="short run for ncu: 1 step, no extras")
    p.add_argument("--mode", default="exact", choices=["pipelined", "exact", "block"],
                   help="N > 1: smoother hand-off between slabs: pipelined = the sweep kernels write the "
                        "boundary cells into the next GPU's memory (NVLink, CUDA IPC); exact = planes handed on "
                        "over NCCL between sweeps (both the single-GPU sweep bit for bit); block = concurrent "
                        "processor-block SGS (a different preconditioner)")
    p.add_argument("--gather-rows", dest="gather_rows", type=int, default=None,
                   help="N > 1: levels with at most this many rows run whole on rank 0 (default: by "
                        "cost, a level is cut while every rank gets >= 65536 of its rows)")
    p.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of slabs")
    p.add_argument("--dist", action="store_true", help="run the slab-distributed path even at N = 1")
    return p.parse_args()


def workload_config(n, n_dofs, target):
    """The workload both arms name (identical dicts, so the driver's same-config check holds)."""
    return {"workload": f"C2: build_system + build_amg + pcg, n={n} ({n_dofs} dofs), rho=h^2, {target} target, "
                        f"rtol {TOL}",
            "n": n, "n_dofs": n_dofs, "rho": rho_for(n), "target": target, "tol": TOL,
            "l2": "inputs exceed L2 (device mesh 255 MB, A 364 MB > 126 MB L2 at n=128); no flush"}


def rho_for(n):
    return 1.0 / (n * n)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_profile_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def job_rate(elapsed_ms, work, world, device=None):
    """Whole-job throughput: the slowest rank's device time (MAX) over all ranks' work (SUM).
    Used by the --replicas mode (independent solves per rank, no data-path collective);
    the default N > 1 path is the slab-distributed solve of run_dist."""
    import torch

    t = torch.tensor([float(elapsed_ms)], dtype=torch.float64, device=device)
    wk = torch.tensor([float(work)], dtype=torch.float64, device=device)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(wk, op=torch.distributed.ReduceOp.SUM)
    return float(t.item()), float(wk.item()) / (float(t.item()) / 1e3)


# ---------------------------------------------------------------------------- ours, N > 1
def run_dist(args, rank, world, local_rank):
    """N > 1: the C2 solve cut into z-slabs across the ranks (dist.py):
    one step = build_system + build_amg (replicated) + slab localisation + the distributed
    PCG (NCCL halo planes, rank-ordered dot sums, coarse levels on rank 0).  The total work
    is fixed as N grows: strong scaling."""
    import torch

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)  # rd kernels, torch copies and NCCL waits all order on it
    with torch.cuda.stream(stream):
        return _run_dist(args, rank, world, local_rank, dev, stream)


def rank_memory(ctx, comm, last, make_solver):
    """Pool bytes in use per rank with a distributed solver alive whose replicated setup objects
    were released after localisation (rank 0 keeps the hierarchy for the coarse levels, the
    other ranks their slabs only), and the peak the replicated setup reserved.  Measured on one
    extra, untimed setup (the timed steps keep the setup objects: releasing them costs ~1 ms)."""
    import gc

    last.clear()
    gc.collect()
    solver = make_solver()
    gc.collect()
    used, reserved = ctx.pool_bytes()
    del solver
    return {"used_bytes_per_rank": comm.allgather_int(int(used)),
            "reserved_bytes_per_rank": comm.allgather_int(int(reserved)),
            "note": "steady state after localisation; the setup itself is still replicated (peak = reserved)"}


def _run_dist(args, rank, world, local_rank, dev, stream):
    import torch

    from paper_2102_03515_b200 import rd
    from paper_2102_03515_b200.dist import DeviceOps, DistSolver, TorchComm

    ctx = rd.Context(local_rank, stream.cuda_stream)
    comm = TorchComm()
    n = args.n
    rho = rho_for(n)
    mesh = rd.build_structured_cube(n, ctx)
    ctx.synchronize()
    last = {}

    phase_ev = []  # (start, after setup, after solve) events per timed step, on the rd stream

    def step():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        ops = DeviceOps(n, rho, args.target, ctx=ctx, device=local_rank, mesh=mesh)
        solver = DistSolver(comm, ops, gather_rows=args.gather_rows, mode=args.mode)
        ev[1].record(stream)
        res = solver.pcg(TOL, 500)
        ev[2].record(stream)
        phase_ev.append(ev)
        last.update(ops=ops, solver=solver, res=res)
        return ops.rows[0], res

    def barrier():
        torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    phase_ev.clear()
    clocks = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = ctx.launch_count
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    its = []
    for _ in range(args.steps):
        ndofs, res = step()
        assert res.converged
        its.append(res.iterations)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count - l0
    # every rank solved the same system: the job's work is counted once (strong scaling)
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    value = float(ndofs) * sum(its) / (elapsed_ms / 1e3)
    # setup (replicated build_system + build_amg + slab localisation + neighbour linking) and
    # the distributed pcg, each the max over ranks of its per-step mean
    ph = torch.tensor([sum(e[0].elapsed_time(e[1]) for e in phase_ev) / len(phase_ev),
                       sum(e[1].elapsed_time(e[2]) for e in phase_ev) / len(phase_ev)], dtype=torch.float64,
                      device=dev)
    torch.distributed.all_reduce(ph, op=torch.distributed.ReduceOp.MAX)
    solver = last["solver"]
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated Kuhn lattice, ball target, seeded)",
        "config": workload_config(n, ndofs, args.target),
        "parallelism": f"z-slabs x{world} ({args.mode} smoother hand-off), {solver.G} distributed level(s), "
                       f"coarse tail on rank 0; setup replicated on every rank",
        "slab_cuts": solver.plan.cuts,
        "iterations": its[0],
        "phases_ms": {"setup_replicated": float(ph[0]), "distributed_pcg": float(ph[1])},
        "clocks": clk,
        "gpu_launches": launches,
        "exchanges_per_iteration": {"halo_planes": "1 per face before SpMV/residual/restriction/"
                                                   "prolongation/smoother", "dot_bytes": 16 * world,
                                    "plane_bytes": 8 * (n - 1) ** 2},
    }
    # the dominant kernel on this rank: its level-0 slab forward sweep, timed alone
    ops = last["ops"]
    lo, hi = solver.plan.owned(0, rank)
    P = (n - 1) ** 2
    rows = (hi - lo) * P
    f = ops.f_local
    xin = torch.rand_like(f)
    xo = torch.empty_like(f)
    for _ in range(3):
        ops.sweep(0, True, f, xin, xo, None)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    R = 20
    for _ in range(R):
        ops.sweep(0, True, f, xin, xo, None)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / R
    Zs = ops.blkA[0].nnz
    by = 8 * Zs + 4 * (rows + 1) + 24 * rows
    peak, peak_kind = peaks()
    result["roofline"] = {"kernel": f"slab gs_sweep level 0 (rank 0: planes [{lo}, {hi}))", "bound": "hbm",
                          "achieved": by / (ms * 1e-3) / 1e9, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                          "frac": by / (ms * 1e-3) / 1e9 / peak, "traffic": None, "bytes_per_launch": by,
                          "launch_ms": ms}
    # per-rank memory in steady state (one extra, untimed setup whose replicated objects are released)
    del ops, f, xin, xo
    solver = None
    result["memory"] = rank_memory(ctx, comm, last, lambda: DistSolver(
        comm, DeviceOps(n, rho, args.target, ctx=ctx, device=local_rank, mesh=mesh),
        gather_rows=args.gather_rows, mode=args.mode, release_replicated=True))
    # e2e: the same distributed solve, u gathered on rank 0 and read back to pinned host memory
    u_host = torch.empty(ndofs, dtype=torch.float64).pin_memory()

    def e2e_step():
        nd, res = step()
        full = last["solver"].gather_solution(res.x_local)
        if rank == 0:
            u_host.copy_(full)
        return res.iterations

    e2e_step()
    barrier()
    torch.cuda.synchronize()
    a.record(stream)
    e2e_its = [e2e_step() for _ in range(args.steps)]
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = float(t.item())
    result["e2e"] = {"value": float(ndofs) * sum(e2e_its) / (e2e_ms / 1e3), "unit": UNIT,
                     "ms_per_step": e2e_ms / args.steps, "h2d_bytes_per_step": 0,
                     "d2h_bytes_per_step": int(8 * ndofs),
                     "path": "device-generated mesh -> distributed solve -> u gathered on rank 0 -> pinned host"}
    return result


# ---------------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2102_03515_b200 import rd

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = rd.Context(local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    n = args.n
    rho = rho_for(n)
    mesh = rd.build_structured_cube(n, ctx)
    ctx.synchronize()
    u_dev = None

    def step():
        nonlocal u_dev
        s = rd.build_system(mesh, rho, args.target)
        if u_dev is None:
            u_dev = torch.empty(s.n_dofs, dtype=torch.float64, device=dev)
        out = rd.solve_system_amg(s.A, s.f_ptr, TOL, u=u_dev)
        return s.n_dofs, out

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    ctx.synchronize()

    # ---------------- timed region: K steps, inputs resident in HBM
    clocks = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = ctx.launch_count
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    its, ndofs, setup_s, solve_s = [], 0, [], []
    for _ in range(args.steps):
        ndofs, out = step()
        its.append(out.iterations)
        setup_s.append(out.setup_seconds)
        solve_s.append(out.solve_seconds)
        assert out.converged
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count - l0
    elapsed_ms, value = job_rate(e0.elapsed_time(e1), float(ndofs) * sum(its), world, dev)
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated Kuhn lattice, ball target, seeded)",
        "config": workload_config(n, ndofs, args.target),
        "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
        "iterations": its[0],
        "phases_ms": {"setup_host_clock": 1e3 * statistics.mean(setup_s), "pcg_host_clock": 1e3 * statistics.mean(solve_s)},
        "pcg_dof_iters_per_s": float(ndofs) * statistics.mean(its) / statistics.mean(solve_s),
        "clocks": clk,
        "gpu_launches": launches,
    }
    if args.profile:
        return result

    # ---------------- the BASELINE error gate on the solution just computed (assembly.cpp:312-331)
    s_err = rd.build_system(mesh, rho, args.target)
    result["errors"] = {"l2_u_minus_target": float(np.sqrt(rd.l2_error_target_squared(s_err, u_dev, args.target))),
                        "rule": "64-point subdivision" if args.target in ("ball", "box") else "degree 5"}
    del s_err

    # ---------------- dominant kernels, timed live with events on the library stream
    s = rd.build_system(mesh, rho, args.target)
    h = rd.build_amg(s.A)
    N, Z = s.n_dofs, s.A.nnz
    x = torch.rand(N, dtype=torch.float64, device=dev)
    y = torch.empty(N, dtype=torch.float64, device=dev)
    ctx.synchronize()
    R = 20

    def timed(fn):
        for _ in range(3):
            fn()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(R):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / R

    gs_ms = timed(lambda: h.level_sweep(0, True, s.f_ptr, x, y))
    level_sweeps = []
    for l in range(h.num_levels - 1):
        Al = h.level(l)
        xl = torch.rand(Al.rows, dtype=torch.float64, device=dev)
        fl = torch.rand(Al.rows, dtype=torch.float64, device=dev)
        yl = torch.empty(Al.rows, dtype=torch.float64, device=dev)
        fw = timed(lambda: h.level_sweep(l, True, fl, xl, yl))
        bw = timed(lambda: h.level_sweep(l, False, fl, xl, yl))
        level_sweeps.append({"level": l, "rows": Al.rows, "nnz": Al.nnz, "fwd_ms": fw, "bwd_ms": bw})
    spmv_ms = timed(lambda: rd.lib().rd_gpu_spmv(ctx.h, s.A.h, rd._ptr(x), rd._ptr(y)))
    # the V-cycle / PCG SpMV on the prepared level-0 matrix: the lattice stencil kernel (no CSR read)
    A0 = h.level(0)
    st_ms = timed(lambda: rd.lib().rd_gpu_spmv(ctx.h, A0.h, rd._ptr(x), rd._ptr(y)))
    structured = h.structured(0)
    uniform = h.uniform(0)
    # SURVEY.md 8(d) algorithmic bytes of a GS sweep (the CSR formulation: values, columns, row
    # pointers, f, x in, x out).  The structured kernel moves far less (uniform stencil: the row
    # is held in registers, ~24 B/row move) -- the DRAM traffic in `traffic` shows it -- so the
    # sweep is bounded by its wavefront depth, reported alongside as dag_steps / us_per_step.
    gs_bytes = 12 * Z + 28 * N + 4
    L0 = round(N ** (1.0 / 3.0))
    dag_steps = 3 * (L0 - 1) + 1
    spmv_bytes = 12 * Z + 20 * N + 4
    peak, peak_kind = peaks()
    traffic = load_profile_traffic()
    gs_gbs = gs_bytes / (gs_ms * 1e-3) / 1e9
    its0 = its[0]
    # level-0 sweeps per step: 4 per V-cycle, V-cycles = iterations + 1
    share = (4 * (its0 + 1) * gs_ms) / (elapsed_ms / args.steps)
    result["roofline"] = {
        "kernel": "gs_sweep level 0 (" + ("structured lattice kernel" if structured else "generic sync-free kernel") + ")",
        "bound": "hbm", "achieved": gs_gbs, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
        "frac": gs_gbs / peak, "traffic": traffic.get("gs_sweep"),
        "bytes_per_launch": gs_bytes, "launch_ms": gs_ms, "share_of_step_est": share,
        "stencil": "uniform (in registers)" if uniform else ("packed stream" if structured else "CSR"),
        "dag_steps": dag_steps, "us_per_step": 1e3 * gs_ms / dag_steps,
    }
    # per kernel class: algorithmic bytes / measured time, vs measured and spec HBM
    nl = h.num_levels
    lv = [(h.level(l).rows, h.level(l).nnz, h.level(l, "P").nnz if l + 1 < nl else 0) for l in range(nl)]
    vc_bytes = sum(60 * Z_ + 168 * N_ + 24 * ZP + 20 * lv[l + 1][0] for l, (N_, Z_, ZP) in enumerate(lv[:-1]))
    vc_bytes += 8 * lv[-1][0] ** 2
    zr = torch.rand(N, dtype=torch.float64, device=dev)
    zz = torch.empty(N, dtype=torch.float64, device=dev)
    vcycle_ms = timed(lambda: h.apply(zr, zz))
    it_bytes = vc_bytes + 12 * Z + 92 * N
    it_ms = 1e3 * statistics.mean(solve_s) / max(1, its0)
    SPEC_HBM = 8000.0

    def cls(bytes_, ms):
        gbs = bytes_ / (ms * 1e-3) / 1e9
        return {"bytes": bytes_, "ms": ms, "achieved_gbs": gbs, "frac_measured": gbs / peak, "frac_spec": gbs / SPEC_HBM}

    result["roofline_classes"] = {
        "spmv": cls(spmv_bytes, spmv_ms), "gs_sweep_level0": cls(gs_bytes, gs_ms),
        "vcycle": cls(vc_bytes, vcycle_ms),
        "pcg_iteration": dict(cls(it_bytes, it_ms), note="solve_seconds / iterations (includes the host loop)"),
        "ceiling_dof_iters_per_s": peak * 1e9 / (it_bytes / N),
    }
    result["kernels"] = {
        "spmv": {"bytes_per_launch": spmv_bytes, "launch_ms": spmv_ms,
                 "achieved_gbs": spmv_bytes / (spmv_ms * 1e-3) / 1e9,
                 "frac": spmv_bytes / (spmv_ms * 1e-3) / 1e9 / peak, "traffic": traffic.get("spmv")},
        "gs_sweep_level0": {"bytes_per_launch": gs_bytes, "launch_ms": gs_ms, "achieved_gbs": gs_gbs,
                            "frac": gs_gbs / peak},
        "spmv_stencil_level0": {"source": h.stencil_source(0), "launch_ms": st_ms,
                                "moved_bytes_per_launch": 16 * N,
                                "moved_gbs": 16 * N / (st_ms * 1e-3) / 1e9,
                                "frac_moved": 16 * N / (st_ms * 1e-3) / 1e9 / peak,
                                "csr_algorithmic_gbs": spmv_bytes / (st_ms * 1e-3) / 1e9},
        "levels": h.num_levels,
        "level_sweeps": level_sweeps,
        "structured_levels": [bool(h.structured(l)) for l in range(h.num_levels - 1)],
        "uniform_levels": [bool(h.uniform(l)) for l in range(h.num_levels - 1)],
    }
    del h, s

    # ---------------- e2e through the C-ABI with host buffers
    if not args.no_e2e:
        xyz, tets, bnd = mesh.download()
        pxyz = torch.from_numpy(xyz).pin_memory()
        ptets = torch.from_numpy(tets).pin_memory()
        pbnd = torch.from_numpy(bnd).pin_memory()
        u_host = torch.empty(ndofs, dtype=torch.float64).pin_memory()

        def e2e_step():
            # one C-ABI call: mesh upload (overlapping the provisional lattice-path solve, every
            # array checked before the result stands), build_system, build_amg + pcg, u back to
            # pinned host memory
            out = rd.solve_host_mesh(pxyz.numpy(), ptets.numpy(), pbnd.numpy(), rho, args.target, TOL,
                                     u=u_host, ctx=ctx)
            return out.iterations

        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        torch.cuda.synchronize()
        if os.environ.get("RD_BENCH_VERBOSE"):  # host-timed probe steps, outside the timed window
            for _ in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                e2e_step()
                torch.cuda.synchronize()
                print(f"e2e step {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_its = [e2e_step() for _ in range(args.steps)]
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms, e2e_value = job_rate(a.elapsed_time(b), float(ndofs) * sum(e2e_its), world, dev)
        result["e2e"] = {"value": e2e_value, "unit": UNIT,
                         "ms_per_step": e2e_ms / args.steps,
                         "h2d_bytes_per_step": int(xyz.nbytes + tets.nbytes + bnd.nbytes),
                         "d2h_bytes_per_step": int(8 * ndofs),
                         "path": "rd_gpu_solve_host_mesh(pinned host TetMesh -> build_system -> build_amg + "
                                 "pcg -> u in pinned host memory; the solve starts on generated lattice "
                                 "vertices while vertices, flags and tets upload, all three checked "
                                 "against the upload before the result stands)"}

    # ---------------- the other BASELINE sizes on this GPU (C4 n=256, C5 n=512 = 133M dofs):
    # one timed solve each after a warm-up, same path; reported beside the C2 headline
    if rank == 0 and world == 1 and not args.no_extra:
        result["other_configs"] = other_configs(ctx, stream)
    # ---------------- CPU baseline (rank 0, N = 1): the oracle port on the host cores
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(n, args.target)
    return result


def other_configs(ctx, stream):
    import torch

    from paper_2102_03515_b200 import rd

    out = []
    for name, n, target in (("C4", 256, "smooth"), ("C5", 512, "ball")):
        try:
            rho = rho_for(n)
            mesh = rd.build_structured_cube(n, ctx)
            u = None
            for rep in range(2):  # warm-up, then the timed step
                ctx.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                s = rd.build_system(mesh, rho, target)
                if u is None:
                    u = torch.empty(s.n_dofs, dtype=torch.float64, device=stream.device)
                o = rd.solve_system_amg(s.A, s.f_ptr, TOL, u=u)
                b.record(stream)
                torch.cuda.synchronize()
                ms = a.elapsed_time(b)
                nd = s.n_dofs
                del s
            out.append({"config": name, "n": n, "n_dofs": nd, "target": target, "rho": rho, "iterations": o.iterations,
                        "ms_per_step": ms, "value": nd * o.iterations / (ms / 1e3), "unit": UNIT,
                        "phases_ms": {"setup": 1e3 * o.setup_seconds, "pcg": 1e3 * o.solve_seconds}})
            del mesh, u
        except Exception as e:  # reported, never fatal for the headline line
            out.append({"config": name, "error": str(e)[:200]})
    out += generic_legs(ctx, stream)
    return out


def generic_legs(ctx, stream, n=N_DEFAULT):
    """The C2 workload on the paths the lattice fast paths do not take (SURVEY.md 8(a) generic
    kernels): (1) jittered interior coordinates -- Kuhn lattice, non-uniform geometry, per-cell
    values, packed-stencil sweeps; (2) renumbered vertices + shuffled tets -- no lattice anywhere:
    vertex->tet CSR assembly, MIS coarsening, Gustavson Galerkin, the sync-free Gauss-Seidel.
    One timed build_system + solve each after a warm-up, plus each level's forward sweep."""
    import numpy as np
    import torch

    from paper_2102_03515_b200 import rd

    rho, target = rho_for(n), TARGET
    xyz, tets, b = rd.build_structured_cube(n, ctx).download()
    rng = np.random.default_rng(5)
    xj = xyz.copy()
    xj[b == 0] += rng.uniform(-0.2, 0.2, size=(int((b == 0).sum()), 3)) / n
    rng = np.random.default_rng(7)
    pv = rng.permutation(xyz.shape[0])
    inv = np.empty_like(pv)
    inv[pv] = np.arange(pv.size)
    tr = inv[tets][rng.permutation(tets.shape[0])].astype(np.int32)
    legs = [("C2_jittered", "jittered interior coordinates (+-0.2 h, seeded): lattice pattern, per-cell geometry",
             (xj, tets, b)),
            ("C2_renumbered", "renumbered vertices + shuffled tets (seeded): no lattice, every generic kernel",
             (np.ascontiguousarray(xyz[pv]), np.ascontiguousarray(tr), np.ascontiguousarray(b[pv])))]
    out = []
    for name, what, arrays in legs:
        try:
            mesh = rd.mesh_from_arrays(*arrays, ctx=ctx)
            u = None
            for rep in range(2):
                ctx.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                s = rd.build_system(mesh, rho, target)
                if u is None:
                    u = torch.empty(s.n_dofs, dtype=torch.float64, device=stream.device)
                o = rd.solve_system_amg(s.A, s.f_ptr, TOL, u=u)
                e.record(stream)
                torch.cuda.synchronize()
                ms = a.elapsed_time(e)
            h = rd.build_amg(s.A)
            levels = []
            for l in range(h.num_levels - 1):
                A = h.level(l)
                x = torch.rand(A.rows, dtype=torch.float64, device=stream.device)
                f = torch.rand(A.rows, dtype=torch.float64, device=stream.device)
                y = torch.empty_like(x)
                h.level_sweep(l, True, f, x, y)
                ctx.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(3):
                    h.level_sweep(l, True, f, x, y)
                e.record(stream)
                torch.cuda.synchronize()
                levels.append({"level": l, "rows": A.rows, "nnz": A.nnz, "stencil": h.stencil_source(l),
                               "fwd_sweep_ms": a.elapsed_time(e) / 3})
            out.append({"config": name, "what": what, "n": n, "n_dofs": s.n_dofs, "target": target, "rho": rho,
                        "lattice_mesh": mesh.lattice_n, "iterations": o.iterations, "ms_per_step": ms,
                        "value": s.n_dofs * o.iterations / (ms / 1e3), "unit": UNIT,
                        "phases_ms": {"setup": 1e3 * o.setup_seconds, "pcg": 1e3 * o.solve_seconds},
                        "levels": levels})
            del s, h, mesh, u
        except Exception as ex:  # reported, never fatal for the headline line
            out.append({"config": name, "error": str(ex)[:200]})
    out.append(adaptive_leg(ctx, stream))
    return out


def adaptive_leg(ctx, stream, budget=200000, rho=1e-2):
    """rdbench adapt's loop (rdbench.cpp:99-104: box target, budget 200,000 dofs)
    from build_structured_cube(8) on the device -- per level build_system (generic assembly on the
    bisected mesh), AMG setup + PCG, estimator, error norms, H^-1 dual norm, Dorfler marking and
    newest-vertex bisection.  One warm-up run, then one timed run (CUDA events)."""
    import torch

    from paper_2102_03515_b200 import rd

    try:
        init = rd.build_structured_cube(8, ctx)
        rd.adaptive_solve(init, "box", rho, budget, tol=TOL)
        ctx.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        res = rd.adaptive_solve(init, "box", rho, budget, tol=TOL)
        e.record(stream)
        torch.cuda.synchronize()
        h = res.history
        return {"config": "adaptive_box", "what": "adaptive_solve(cube(8), box, rho=1e-2, budget 200000, AMG tol "
                "1e-8, theta 0.5): every level on the generic path", "levels": len(h), "final_dofs": h[-1]["dofs"],
                "ms_total": a.elapsed_time(e), "iterations": [r["iterations"] for r in h],
                "dofs": [r["dofs"] for r in h], "seconds_per_level": [round(r["seconds"], 5) for r in h],
                "eta": [h[0]["eta"], h[-1]["eta"]]}
    except Exception as ex:  # reported, never fatal for the headline line
        return {"config": "adaptive_box", "error": str(ex)[:200]}


def host_info():
    """CPU model and RAM of the host the CPU baseline ran on."""
    model, mem_gb = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem_gb = round(int(line.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "ram_gib": mem_gb}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(n, target):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O

    O.build()
    cores = host_threads()
    O.set_num_threads(cores)
    r = O.pipeline(n, rho_for(n), target, 0, TOL)
    out = {"value": r["n_dofs"] * r["iterations"] / r["total_s"], "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"one full C2 step on the CPU oracle (n={n}: build_system + build_amg + pcg, "
                     f"{r['iterations']} iterations), {r['total_s']:.1f} s; SGS/setup serial as in the reference",
           "phases_s": {"build": r["build_s"], "setup": r["setup_s"], "solve": r["solve_s"]},
           "host": host_info()}
    if cores > 1 and not os.environ.get("RD_BENCH_NO_CPU1"):  # threads = 1 as well
        O.set_num_threads(1)
        r1 = O.pipeline(n, rho_for(n), target, 0, TOL)
        out["single_thread"] = {"value": r1["n_dofs"] * r1["iterations"] / r1["total_s"], "total_s": r1["total_s"],
                                "phases_s": {"build": r1["build_s"], "setup": r1["setup_s"], "solve": r1["solve_s"]}}
        O.set_num_threads(cores)
    return out


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O

    O.build()
    cores = host_threads()
    O.set_num_threads(cores)
    n = args.n
    for _ in range(args.warmup):  # CPU warm-up on a small case (threads, page cache)
        O.pipeline(16, rho_for(16), args.target, 0, TOL)
    t0 = time.perf_counter()
    runs = [O.pipeline(n, rho_for(n), args.target, 0, TOL) for _ in range(args.steps)]
    el = time.perf_counter() - t0
    work = sum(r["n_dofs"] * r["iterations"] for r in runs)
    value = work / el
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated Kuhn lattice, ball target, seeded)",
        "config": workload_config(n, runs[0]["n_dofs"], args.target),
        "iterations": runs[0]["iterations"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{args.steps} full C2 steps (reference rdsolve not buildable here: no Eigen; "
                                   f"the oracle/ C++ port with -O3 -ffp-contract=off, {cores} threads)",
                         "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phases_s": {k: statistics.mean(r[k] for r in runs) for k in ("build_s", "setup_s", "solve_s")},
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "reference":
        # the CPU reference arm runs on rank 0 alone; the other ranks exit without work
        if rank != 0:
            return
    use_pg = args.impl == "ours" and (world > 1 or args.dist)
    if use_pg:
        import socket

        import torch

        if world == 1:  # a one-rank group for --dist at N = 1
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(port))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
            # NCCL_DEBUG=VERSION prints "NCCL version ..." on stdout, which must carry one JSON line only
            if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
                os.environ["NCCL_DEBUG"] = "WARN"
        torch.distributed.init_process_group(backend=backend)
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    elif (world > 1 and not args.replicas) or args.dist:
        res = run_dist(args, rank, world, local_rank)
    else:
        res = run_ours(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    if use_pg:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
