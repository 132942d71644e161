"""Distributed (z-slab) AMG-PCG solve over torch.distributed -- SURVEY.md §8(e).

The reference solves on one host with a thread pool (parallel.cpp:12-73); it
has no distributed solver.  This module shards the north-star solve across
ranks, one GPU per rank, the way §8(e) lays out:

* **Partition.**  Every distributed level's lattice is cut into z-slabs; a slab
  is a contiguous row range (z is the slowest lattice index).  The cuts sit on
  multiples of 2^G at level 0 (G = number of distributed levels), so level l's
  cut is the level-0 cut >> l and every coarse (all-even) point lies in the slab
  of its fine twin.  Each rank keeps its slab plus one ghost
  plane per side ("local vectors", planes [g0, g1)).
* **Per-rank device work** (``DeviceOps``, the rd_gpu C-ABI): row blocks of
  A_l, P_l, Pt_l (the same row sums in the same order as the single-GPU SpMV),
  the slab smoother, the fused PCG vector updates.
* **Exchanges per PCG iteration** (``TorchComm``: NCCL over NVLink, or gloo on
  CPU): one plane per face before every SpMV / residual / restriction /
  prolongation / smoother pass that reads a neighbour's rows; the inner products
  all-gathered (16 bytes per iteration) and summed in rank order, so every rank
  holds the same scalars; levels too small to pay for their exchanges gathered onto rank 0
  (``rd_gpu_amg_apply_from``) and the correction scattered back.
* **Smoother.**  ``mode="exact"`` hands the Gauss-Seidel wavefront from rank to
  rank (the upstream ghost plane is the neighbour's *fresh* values): the
  V-cycle is the single-GPU V-cycle bit for bit, and the PCG differs only by the
  order of the dot-product reductions.  ``mode="block"`` relaxes all slabs at
  once with the neighbours' *old* values (processor-block symmetric GS, a
  different preconditioner; SURVEY.md §8(e) option ii).

Setup in this round is replicated (every rank builds the whole system and
hierarchy with the single-GPU kernels, then keeps its row blocks); the solve is
distributed.  ``ThreadComm`` runs several ranks in one process on one device
(one thread and one stream per rank, plane hand-off through stream events, no
kernel ever waits on another), which is how the GPU tests exercise the
multi-rank path on a single B200.
"""
from __future__ import annotations

import math
import queue
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

__all__ = ["SlabPlan", "choose_dist_levels", "TorchComm", "ThreadComm", "DeviceOps", "DistSolver", "DistResult",
           "NotSpdError"]


class NotSpdError(RuntimeError):
    """pcg / preconditioner lost positive definiteness (linalg.cpp:71,81-82,88-89)."""


# ------------------------------------------------------------------ partition
class SlabPlan:
    """z-slab ownership of levels 0..G (G = dist_levels; level G is gathered on rank 0)."""

    def __init__(self, sides, world: int, dist_levels: int):
        self.sides = [int(s) for s in sides]
        self.world = int(world)
        self.G = int(dist_levels)
        if not 1 <= self.G < len(self.sides):
            raise ValueError("slab plan: need 1 <= dist_levels < number of levels")
        align = 1 << self.G
        L0 = self.sides[0]
        self.cuts = [0] + [int(round(r * L0 / self.world / align)) * align for r in range(1, self.world)] + [L0]
        for l in range(self.G + 1):
            for r in range(self.world):
                lo, hi = self.owned(l, r)
                if hi <= lo:
                    raise ValueError(f"slab plan: rank {r} owns no plane of level {l} (side {self.sides[l]}, "
                                     f"{self.world} ranks, cuts on multiples of {align})")

    def owned(self, l: int, r: int):
        lo = self.cuts[r] >> l
        hi = self.sides[l] if r == self.world - 1 else self.cuts[r + 1] >> l
        return lo, hi

    def ghost(self, l: int, r: int):
        lo, hi = self.owned(l, r)
        return max(lo - 1, 0), min(hi + 1, self.sides[l])


MIN_ROWS_PER_RANK = 65536  # below this a level's slab work no longer pays for its exchanges


def choose_dist_levels(sides, rows, structured, world: int, gather_rows: int | None = None) -> int:
    """Distribute the leading lattice levels (at least level 0), as many as the 2^G-aligned cuts
    allow.  gather_rows=None: by cost -- a level is cut while every rank's share has at least
    MIN_ROWS_PER_RANK rows (its per-sweep plane exchanges and hand-off waits are then small
    against the slab's own sweep); otherwise levels with more than `gather_rows` rows are cut."""
    nl = len(rows)
    G = 1
    keep = (lambda r: r // world >= MIN_ROWS_PER_RANK) if gather_rows is None else (lambda r: r > gather_rows)
    while G < nl - 1 and keep(rows[G]) and structured[G]:
        G += 1
    while G >= 1:
        try:
            SlabPlan(sides, world, G)
            return G
        except ValueError:
            G -= 1
    raise ValueError(f"cannot cut a side-{sides[0]} lattice into {world} slabs")


# ------------------------------------------------------------------ communication
class TorchComm:
    """torch.distributed process group: NCCL (device tensors) or gloo (CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange(self, ops):
        """ops: list of ("send" | "recv", peer, tensor); posted as one batch."""
        if not ops:
            return
        d = self.dist
        p2p = [d.P2POp(d.isend if k == "send" else d.irecv, t, peer, self.group) for (k, peer, t) in ops]
        for w in d.batch_isend_irecv(p2p):
            w.wait()

    def allgather_scalars(self, t: torch.Tensor):
        """t: 1-element float64 tensor on this rank's device -> list of floats in rank order."""
        out = torch.empty(self.world, dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t.reshape(1), group=self.group)
        return out.tolist()

    def allgather_into(self, t: torch.Tensor, out: torch.Tensor):
        """t: 1-element float64 tensor -> out[world] in rank order, on the stream (NCCL for
        device tensors): the scalar never visits the host."""
        self.dist.all_gather_into_tensor(out, t.reshape(1), group=self.group)

    def link_slabs(self, ops, G):
        """Map the neighbours' slab cell buffers (CUDA IPC over NVLink) for the pipelined hand-off.

        Every rank runs every level's collective whatever fails locally (an export or a
        peer mapping), and the outcome is reduced once at the end, so a failure on some
        ranks can never leave the others waiting in a different collective."""
        ok = True
        for l in range(G):
            try:
                mine = (ops.ipc_handle(l), ops.slab_g0(l))
            except Exception:  # noqa: BLE001
                mine = None
            allh = [None] * self.world
            self.dist.all_gather_object(allh, mine, group=self.group)
            if not ok or any(h is None for h in allh):
                ok = False
                continue
            try:
                if self.rank + 1 < self.world:
                    ops.open_peer(l, 0, *allh[self.rank + 1])
                if self.rank > 0:
                    ops.open_peer(l, 1, *allh[self.rank - 1])
            except Exception:  # noqa: BLE001
                ok = False
        if not all(self.allgather_int(1 if ok else 0)):
            raise RuntimeError("slab cell buffers could not be mapped for the pipelined hand-off")

    def pipelined_sweep(self, ops, l, fwd, f, xin, xout):
        ops.sweep_pipelined(l, fwd, f, xin, xout)

    def allgather_int(self, v: int):
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.int64, device=dev)
        out = torch.empty(self.world, dtype=torch.int64, device=dev)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.tolist()


class _ThreadHub:
    def __init__(self, world: int):
        self.world = world
        self.boxes = {}
        self.lock = threading.Lock()
        self.bar = threading.Barrier(world)
        self.vals = [None] * world

    def box(self, src, dst):
        with self.lock:
            return self.boxes.setdefault((src, dst), queue.Queue())


class ThreadComm:
    """Ranks as threads of one process on one device (tests and single-GPU emulation).

    A send stages the plane into a fresh buffer on the sender's stream and posts it
    with a CUDA event; the receiver's stream waits on that event before copying.
    Only the host threads block; no kernel waits on another rank's kernel.
    """

    def __init__(self, hub: _ThreadHub, rank: int):
        self.hub = hub
        self.rank = rank
        self.world = hub.world

    @staticmethod
    def hub(world: int) -> _ThreadHub:
        return _ThreadHub(world)

    def exchange(self, ops):
        for (k, peer, t) in ops:
            if k == "send":
                buf = t.clone()
                ev = None
                if buf.is_cuda:
                    ev = torch.cuda.Event()
                    ev.record()
                self.hub.box(self.rank, peer).put((buf, ev))
        for (k, peer, t) in ops:
            if k == "recv":
                buf, ev = self.hub.box(peer, self.rank).get(timeout=600)
                if ev is not None:
                    torch.cuda.current_stream().wait_event(ev)
                t.copy_(buf)
                if buf.is_cuda:
                    # buf was allocated on the sender's stream: without this the caching
                    # allocator hands the block back to the sender's stream as soon as buf
                    # is dropped here, before this stream's copy has run
                    buf.record_stream(torch.cuda.current_stream())

    def _allgather(self, v):
        self.hub.vals[self.rank] = v
        self.hub.bar.wait(timeout=600)
        out = list(self.hub.vals)
        self.hub.bar.wait(timeout=600)
        return out

    def allgather_scalars(self, t: torch.Tensor):
        return self._allgather(float(t.reshape(-1)[0].item()))

    def allgather_into(self, t: torch.Tensor, out: torch.Tensor):
        """Every rank's scalar into out[world] on this rank's stream (event-ordered copies)."""
        ev = None
        if t.is_cuda:
            # a snapshot: the sender's stream may overwrite t (the next dot) before a
            # receiver's stream copies it; record_stream keeps the snapshot's block from
            # being reused until every receiver's copy has run
            t = t.clone()
            ev = torch.cuda.Event()
            ev.record()
        entries = self._allgather((t, ev))
        for k, (tk, ek) in enumerate(entries):
            if ek is not None:
                torch.cuda.current_stream().wait_event(ek)
                tk.record_stream(torch.cuda.current_stream())
            out[k:k + 1].copy_(tk.reshape(1))

    def allgather_int(self, v: int):
        return self._allgather(int(v))

    def link_slabs(self, ops, G):
        for l in range(G):
            allo = self._allgather(ops)
            nxt = allo[self.rank + 1] if self.rank + 1 < self.world else None
            prv = allo[self.rank - 1] if self.rank > 0 else None
            ops.link(l, nxt, prv)

    def pipelined_sweep(self, ops, l, fwd, f, xin, xout):
        """All ranks' slabs of level l in ONE cooperative launch on rank 0's stream (kernels
        that wait on one another must not be separate launches on one GPU)."""
        ev = torch.cuda.Event()
        ev.record()
        entries = self._allgather((ops, f, xin, xout, ev))
        if self.rank == 0:
            cur = torch.cuda.current_stream()
            for e in entries:
                cur.wait_event(e[4])
            ops.sweep_multi(l, fwd, [(e[0], e[1], e[2], e[3]) for e in entries])
            done = torch.cuda.Event()
            done.record()
            self.hub.done = done
        self.hub.bar.wait(timeout=600)
        if self.rank != 0:
            torch.cuda.current_stream().wait_event(self.hub.done)
        self.hub.bar.wait(timeout=600)


# ------------------------------------------------------------------ device work (the product path)
class DeviceOps:
    """One rank's device work through the rd_gpu C-ABI (sm_100a kernels).

    Builds the whole system and hierarchy with the single-GPU path (replicated
    setup), then keeps the rank's row blocks and slab smoothers.  Every call is
    stream-ordered on the rd context's stream, which is torch's current stream
    when the context is created here, so torch copies and NCCL waits order with it.
    """

    def __init__(self, n: int, rho: float, target: str = "ball", seed: int = 0, ctx=None, device: int = 0,
                 mesh=None):
        from . import rd

        self.rd = rd
        self.device = torch.device("cuda", device)
        if ctx is None and mesh is None:
            # order with torch's current stream (handle 0 = the legacy default stream: cudaStreamLegacy)
            ctx = rd.Context(device, torch.cuda.current_stream(self.device).cuda_stream or 1)
        self.ctx = ctx or mesh.ctx
        self.mesh_owned = mesh is None
        self.mesh = mesh if mesh is not None else rd.build_structured_cube(n, self.ctx)
        self.sys = rd.build_system(self.mesh, rho, target, seed)
        self.A = self.sys.A
        self.h = rd.build_amg(self.A)
        nl = self.h.num_levels
        self.rows = [self.h.level(l).rows for l in range(nl)]
        self.sides = [_icbrt(r) for r in self.rows]
        self.structured = [self.sides[l] ** 3 == self.rows[l] and (l == nl - 1 or self.h.structured(l))
                           for l in range(nl)]

    # -- setup
    def localize(self, plan: SlabPlan, rank: int, release_replicated: bool = False):
        """Keep this rank's row blocks, slab smoothers and load-vector slab.  With
        `release_replicated` the whole-box objects of the replicated setup are dropped afterwards
        (everything on ranks > 0; rank 0 keeps the hierarchy, whose coarse levels it runs): the
        steady-state footprint of a rank is then its slabs, not the whole problem."""
        rd, lib, C = self.rd, self.rd.lib(), __import__("ctypes")
        self.plan, self.rank = plan, rank
        self.blkA, self.blkP, self.blkPt, self.slab = [], [], [], []

        def rowblock(M, r0, r1, c0, c1):
            h = C.c_void_p()
            self.ctx.check(lib.rd_gpu_csr_rowblock(self.ctx.h, M.h, r0, r1, c0, c1, C.byref(h)))
            return rd.Csr(h, self.ctx)

        for l in range(plan.G):
            if not self.structured[l]:
                raise ValueError(f"distributed level {l} is not a lattice level")
            P0 = plan.sides[l] ** 2
            P1 = plan.sides[l + 1] ** 2
            lo, hi = plan.owned(l, rank)
            g0, g1 = plan.ghost(l, rank)
            clo, chi = plan.owned(l + 1, rank)
            cg0, cg1 = plan.ghost(l + 1, rank)
            self.blkA.append(rowblock(self.h.level(l, "A"), lo * P0, hi * P0, g0 * P0, g1 * P0))
            self.blkP.append(rowblock(self.h.level(l, "P"), lo * P0, hi * P0, cg0 * P1, cg1 * P1))
            self.blkPt.append(rowblock(self.h.level(l, "Pt"), clo * P1, chi * P1, g0 * P0, g1 * P0))
            s = C.c_void_p()
            self.ctx.check(lib.rd_gpu_slab_create(self.ctx.h, self.h.level(l, "A").h, lo, hi, C.byref(s)))
            self.slab.append(_Slab(s))
        # local load vector
        lo, hi = plan.owned(0, rank)
        g0, _ = plan.ghost(0, rank)
        P0 = plan.sides[0] ** 2
        f_all = torch.empty(self.rows[0], dtype=torch.float64, device=self.device)
        self.ctx.check(lib.rd_gpu_copy(self.ctx.h, C.c_void_p(f_all.data_ptr()), C.c_void_p(self.sys.f_ptr),
                                       8 * self.rows[0]))
        self.f_local = self.vec(0)
        self.f_local[(lo - g0) * P0:(hi - g0) * P0].copy_(f_all[lo * P0:hi * P0])
        del f_all
        if release_replicated:
            self.sys = self.A = None  # K, M, A, f of the whole box (build_amg keeps its own A)
            if rank != 0:
                self.h = None  # the coarse tail runs on rank 0 only
            if self.mesh_owned:
                self.mesh = None

    # -- vectors
    def vec(self, l: int, full: bool = False) -> torch.Tensor:
        if full:
            return torch.zeros(self.rows[l], dtype=torch.float64, device=self.device)
        g0, g1 = self.plan.ghost(l, self.rank)
        return torch.zeros((g1 - g0) * self.plan.sides[l] ** 2, dtype=torch.float64, device=self.device)

    def scalar(self) -> torch.Tensor:
        return torch.zeros(1, dtype=torch.float64, device=self.device)

    # -- kernels
    def spmv(self, M, x, y):
        self.ctx.check(self.rd.lib().rd_gpu_spmv(self.ctx.h, M.h, _p(x), _p(y)))

    def residual(self, M, r, z, res):
        self.ctx.check(self.rd.lib().rd_gpu_residual(self.ctx.h, M.h, _p(r), _p(z), _p(res)))

    def prolong_add(self, M, zc, z):
        self.ctx.check(self.rd.lib().rd_gpu_prolong_add(self.ctx.h, M.h, _p(zc), _p(z)))

    def sweep(self, l, fwd, f, xin, xout, in_plane):
        self.ctx.check(self.rd.lib().rd_gpu_slab_sweep(self.slab[l].h, 1 if fwd else 0, _p(f), _p(xin), _p(xout),
                                                       _p(in_plane)))

    # -- pipelined hand-off (peer cells)
    def slab_g0(self, l):
        return self.plan.ghost(l, self.rank)[0]

    def ipc_handle(self, l) -> bytes:
        import ctypes

        buf = ctypes.create_string_buffer(64)
        self.ctx.check(self.rd.lib().rd_gpu_slab_ipc_handle(self.slab[l].h, buf))
        return buf.raw

    def open_peer(self, l, which, handle: bytes, peer_g0: int):
        import ctypes

        buf = ctypes.create_string_buffer(bytes(handle), 64)
        self.ctx.check(self.rd.lib().rd_gpu_slab_open_peer(self.slab[l].h, int(which), buf, int(peer_g0)))

    def link(self, l, nxt, prv):
        self.ctx.check(self.rd.lib().rd_gpu_slab_link(self.slab[l].h, nxt.slab[l].h if nxt else None,
                                                      prv.slab[l].h if prv else None))

    def sweep_pipelined(self, l, fwd, f, xin, xout):
        self.ctx.check(self.rd.lib().rd_gpu_slab_sweep_pipelined(self.slab[l].h, 1 if fwd else 0, _p(f), _p(xin),
                                                                 _p(xout)))

    def sweep_multi(self, l, fwd, entries):
        """entries: [(ops_q, f_q, xin_q, xout_q)] of every slab of level l, in rank order."""
        import ctypes

        n = len(entries)
        P = ctypes.c_void_p * n
        sl = P(*[e[0].slab[l].h for e in entries])
        fs = P(*[e[1].data_ptr() for e in entries])
        xi = P(*[(e[2].data_ptr() if e[2] is not None else None) for e in entries])
        xo = P(*[e[3].data_ptr() for e in entries])
        self.ctx.check(self.rd.lib().rd_gpu_slab_sweep_multi(n, sl, 1 if fwd else 0, fs, xi, xo))

    def dot(self, a, b, out):
        self.ctx.check(self.rd.lib().rd_gpu_dot_async(self.ctx.h, a.numel(), _p(a), _p(b), _p(out)))

    def xr(self, alpha, p, ap, x, r):
        self.ctx.check(self.rd.lib().rd_gpu_pcg_update_xr(self.ctx.h, p.numel(), float(alpha), _p(p), _p(ap), _p(x),
                                                          _p(r)))

    def pupd(self, beta, z, p):
        self.ctx.check(self.rd.lib().rd_gpu_pcg_update_p(self.ctx.h, p.numel(), float(beta), _p(z), _p(p)))

    def coarse(self, level, r, z):
        self.ctx.check(self.rd.lib().rd_gpu_amg_apply_from(self.h.h, int(level), _p(r), _p(z)))

    # -- the PCG scalars on the device (rd_pcg_state, 80 bytes = 10 doubles)
    def pcg_state(self) -> torch.Tensor:
        return torch.zeros(10, dtype=torch.float64, device=self.device)

    def pcg_begin(self, parts, st):
        self.ctx.check(self.rd.lib().rd_gpu_pcg_dist_begin(self.ctx.h, parts.numel(), _p(parts), _p(st)))

    def pcg_alpha(self, parts, st):
        self.ctx.check(self.rd.lib().rd_gpu_pcg_dist_alpha(self.ctx.h, parts.numel(), _p(parts), _p(st)))

    def pcg_xr(self, st, p, ap, x, r):
        self.ctx.check(self.rd.lib().rd_gpu_pcg_dist_xr(self.ctx.h, p.numel(), _p(st), _p(p), _p(ap), _p(x), _p(r)))

    def pcg_check(self, parts, st, tol, hist):
        self.ctx.check(self.rd.lib().rd_gpu_pcg_dist_check(self.ctx.h, parts.numel(), _p(parts), _p(st), float(tol),
                                                           _p(hist), hist.numel()))

    def pcg_p(self, st, z, p):
        self.ctx.check(self.rd.lib().rd_gpu_pcg_dist_p(self.ctx.h, p.numel(), _p(st), _p(z), _p(p)))

    def set_exact(self, exact: bool):
        self.ctx.check(self.rd.lib().rd_gpu_ctx_set_exact_sweeps(self.ctx.h, 1 if exact else 0))

    def check(self) -> int:
        """Device errors of the asynchronous calls so far (0, or RD_GS_SPECULATION_MISS, ...)."""
        rc = self.check_raw()
        if rc not in (0, self.rd.RD_GS_SPECULATION_MISS):
            self.ctx.check(rc)
        return rc

    def check_raw(self) -> int:
        """The status of rd_gpu_synchronize, never raised here (collective callers raise together)."""
        return int(self.rd.lib().rd_gpu_synchronize(self.ctx.h))


class _Slab:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            from . import rd

            if self.h and not rd._closing:
                rd.lib().rd_gpu_slab_free(self.h)
        except Exception:
            pass
        self.h = None


def _state(st: torch.Tensor) -> dict:
    """Host copy of an rd_pcg_state (8 doubles, then done / status / iterations as int32)."""
    a = st.detach().cpu().numpy()
    iv = a.view(np.int32)
    return {"rz": float(a[0]), "rz0": float(a[1]), "pap": float(a[2]), "rz_next": float(a[3]),
            "alpha": float(a[4]), "beta": float(a[5]), "rel": float(a[6]),
            "done": int(iv[16]), "status": int(iv[17]), "iterations": int(iv[18])}


def _p(t):
    import ctypes

    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _icbrt(n: int) -> int:
    r = int(round(n ** (1.0 / 3.0)))
    for c in (r - 1, r, r + 1):
        if c >= 0 and c ** 3 == n:
            return c
    return r


# ------------------------------------------------------------------ the solver
@dataclass
class DistResult:
    x_local: torch.Tensor  # owned rows of the solution (level-0 slab)
    iterations: int
    converged: bool
    residual_history: list = field(default_factory=list)
    exact_rerun: bool = False


class DistSolver:
    """Slab-distributed AMG-PCG (linalg.cpp:64-102 with amg_precond, amg.cpp:119-145)."""

    def __init__(self, comm, ops, gather_rows: int | None = None, mode: str = "exact",
                 dist_levels: int | None = None, release_replicated: bool = False):
        if mode not in ("exact", "block", "pipelined"):
            raise ValueError("mode must be 'exact', 'block' or 'pipelined'")
        self.comm, self.ops, self.mode = comm, ops, mode
        self.rank, self.world = comm.rank, comm.world
        G = dist_levels or choose_dist_levels(ops.sides, ops.rows, ops.structured, self.world, gather_rows)
        self.plan = SlabPlan(ops.sides, self.world, G)
        self.G = G
        try:
            ops.localize(self.plan, self.rank, release_replicated=release_replicated)
        except TypeError:  # an ops class without the option (the host ops of the CPU tests)
            ops.localize(self.plan, self.rank)
        if mode == "pipelined":
            # peer mapping of the neighbours' cell buffers; if any rank cannot map (no P2P
            # path, IPC unavailable) every rank falls back to the NCCL plane hand-off
            ok = 1
            try:
                comm.link_slabs(ops, G)
            except Exception as e:  # noqa: BLE001 -- reported through the fallback
                self.link_error = repr(e)
                ok = 0
            if not all(comm.allgather_int(ok)):
                self.mode = "exact"
        R = self.rank
        pl = self.plan
        self.r = [None] + [ops.vec(l) for l in range(1, G + 1)]
        self.z = [ops.vec(l) for l in range(G + 1)]
        self.t = [ops.vec(l) for l in range(G)]
        self.res = [ops.vec(l) for l in range(G)]
        self.inplane = [ops.vec(l)[: pl.sides[l] ** 2].clone() for l in range(G)]
        if R == 0:
            self.rG = ops.vec(G, full=True)
            self.zG = ops.vec(G, full=True)
        self.bar_ = ops.scalar()

    # -- local-vector views
    def _P(self, l):
        return self.plan.sides[l] ** 2

    def own(self, l, v):
        lo, hi = self.plan.owned(l, self.rank)
        g0, _ = self.plan.ghost(l, self.rank)
        P = self._P(l)
        return v[(lo - g0) * P:(hi - g0) * P]

    def plane(self, l, v, z):
        g0, _ = self.plan.ghost(l, self.rank)
        P = self._P(l)
        return v[(z - g0) * P:(z - g0 + 1) * P]

    # -- exchanges
    def halo(self, l, v, lower=True, upper=True):
        """Fill v's lower / upper ghost plane from the neighbours' owned boundary planes."""
        R, W = self.rank, self.world
        lo, hi = self.plan.owned(l, R)
        ops = []
        if lower:
            if R + 1 < W:
                ops.append(("send", R + 1, self.plane(l, v, hi - 1)))
            if R > 0:
                ops.append(("recv", R - 1, self.plane(l, v, lo - 1)))
        if upper:
            if R > 0:
                ops.append(("send", R - 1, self.plane(l, v, lo)))
            if R + 1 < W:
                ops.append(("recv", R + 1, self.plane(l, v, hi)))
        self.comm.exchange(ops)

    # -- smoother
    def sweep(self, l, fwd, f, xin, xout):
        R, W = self.rank, self.world
        lo, hi = self.plan.owned(l, R)
        up = R - 1 if fwd else R + 1      # rank upstream of the sweep
        down = R + 1 if fwd else R - 1
        has_up, has_down = 0 <= up < W, 0 <= down < W
        if self.mode == "block":
            if xin is not None:
                self.halo(l, xin, lower=True, upper=True)
            in_plane = None
            if has_up and xin is not None:
                in_plane = self.plane(l, xin, lo - 1 if fwd else hi)
            self.ops.sweep(l, fwd, f, xin, xout, in_plane)
            return
        if xin is not None:  # old values of the downstream ghost plane
            self.halo(l, xin, lower=not fwd, upper=fwd)
        if self.mode == "pipelined":  # the kernels hand the wavefront on through peer memory
            self.comm.pipelined_sweep(self.ops, l, fwd, f, xin, xout)
            return
        in_plane = None
        if has_up:
            in_plane = self.inplane[l]
            self.comm.exchange([("recv", up, in_plane)])
        self.ops.sweep(l, fwd, f, xin, xout, in_plane)
        if has_down:
            self.comm.exchange([("send", down, self.plane(l, xout, hi - 1 if fwd else lo))])

    # -- V-cycle
    def vcycle(self, l, r, z):
        """z = V_l(r) on local vectors of level l (owned rows of r valid)."""
        ops, G = self.ops, self.G
        if l == G:
            self._coarse(r, z)
            return
        t, res = self.t[l], self.res[l]
        self.sweep(l, True, r, None, t)
        self.sweep(l, False, r, t, z)
        self.halo(l, z)
        ops.residual(self.blk("A", l), self.own(l, r), z, self.own(l, res))
        self.halo(l, res, lower=True, upper=False)
        rc, zc = self.r[l + 1], self.z[l + 1]
        ops.spmv(self.blk("Pt", l), res, self.own(l + 1, rc))
        self.vcycle(l + 1, rc, zc)
        if l + 1 < G:
            self.halo(l + 1, zc, lower=False, upper=True)
        ops.prolong_add(self.blk("P", l), zc, self.own(l, z))
        self.sweep(l, True, r, z, t)
        self.sweep(l, False, r, t, z)

    def blk(self, which, l):
        return {"A": self.ops.blkA, "P": self.ops.blkP, "Pt": self.ops.blkPt}[which][l]

    def _coarse(self, r, z):
        """Gather level G on rank 0, run its V-cycle tail, send each rank its planes + upper ghost."""
        G, R, W, pl = self.G, self.rank, self.world, self.plan
        P = self._P(G)
        if R == 0:
            ops = []
            for q in range(1, W):
                qlo, qhi = pl.owned(G, q)
                ops.append(("recv", q, self.rG[qlo * P:qhi * P]))
            self.comm.exchange(ops)
            lo, hi = pl.owned(G, 0)
            self.rG[lo * P:hi * P].copy_(self.own(G, r))
            self.ops.coarse(G, self.rG, self.zG)
            ops = []
            for q in range(1, W):
                qlo, qhi = pl.owned(G, q)
                ops.append(("send", q, self.zG[qlo * P:min(qhi + 1, pl.sides[G]) * P]))
            self.comm.exchange(ops)
            g0, g1 = pl.ghost(G, 0)
            z.copy_(self.zG[g0 * P:g1 * P])
        else:
            self.comm.exchange([("send", 0, self.own(G, r))])
            lo, hi = pl.owned(G, R)
            g0, _ = pl.ghost(G, R)
            top = min(hi + 1, pl.sides[G])
            self.comm.exchange([("recv", 0, z[(lo - g0) * P:(top - g0) * P])])

    def apply(self, r, z):
        """amg_apply on the level-0 slab (r, z: local vectors)."""
        self.vcycle(0, r, z)

    # -- PCG
    def pcg(self, tol: float = 1e-8, max_iter: int = 500) -> DistResult:
        err, res = None, None
        try:
            res = self._pcg(tol, max_iter)
        except NotSpdError as e:  # raised on every rank at once (the scalars are replicated)
            err = e
        # the raw device status goes through the collective first, so a device error on
        # one rank is raised on every rank together instead of stranding the others
        rcs = self.comm.allgather_int(self.ops.check_raw())
        miss = 0x5EC  # RD_GS_SPECULATION_MISS (rd.py): rerun with exact sweeps
        bad = [c for c in rcs if c not in (0, miss)]
        if bad:
            raise RuntimeError(f"distributed pcg: device error {bad[0]} on rank {rcs.index(bad[0])}")
        if any(rcs):
            # a speculative sweep somewhere left the division fast path (possibly behind the
            # error it caused): rerun the whole solve with exact sweeps on every rank
            self.ops.set_exact(True)
            try:
                res = self._pcg(tol, max_iter)
                if self.ops.check():
                    raise RuntimeError("distributed pcg: device error in the exact rerun")
            finally:
                self.ops.set_exact(False)
            res.exact_rerun = True
            return res
        if err is not None:
            raise err
        return res

    def _pcg(self, tol, max_iter):
        """linalg.cpp:64-102 with every scalar on the device: the local dot partials are
        all-gathered (NCCL) into `parts` and summed in rank order by the state kernels;
        alpha / beta never leave the device.  The host reads the 80-byte state once per
        iteration, after the next iteration's halo + A p + x / r update are already queued
        (no-ops once converged), so the GPU does not idle across the round trip."""
        ops, comm = self.ops, self.comm
        f = ops.f_local
        x = ops.vec(0)
        r = f.clone()
        z, p, Ap = ops.vec(0), ops.vec(0), ops.vec(0)
        s = ops.scalar()
        parts = torch.zeros(self.world, dtype=torch.float64, device=s.device)
        st = ops.pcg_state()
        hist = torch.zeros(max(max_iter, 1), dtype=torch.float64, device=s.device)
        own = lambda v: self.own(0, v)  # noqa: E731
        out = DistResult(own(x), 0, False, [])
        self.apply(r, z)
        ops.dot(own(r), own(z), s)
        comm.allgather_into(s, parts)
        ops.pcg_begin(parts, st)
        hs = _state(st)
        if hs["status"]:
            raise NotSpdError("pcg: preconditioner not positive definite")
        if hs["done"]:
            out.converged = True
            return out
        p.copy_(z)

        def ap_xr():
            self.halo(0, p)
            ops.spmv(self.blk("A", 0), p, own(Ap))
            ops.dot(own(p), own(Ap), s)
            comm.allgather_into(s, parts)
            ops.pcg_alpha(parts, st)
            ops.pcg_xr(st, own(p), own(Ap), own(x), own(r))

        if max_iter >= 1:
            ap_xr()
        for it in range(1, max_iter + 1):
            self.apply(r, z)
            ops.dot(own(r), own(z), s)
            comm.allgather_into(s, parts)
            ops.pcg_check(parts, st, tol, hist)
            ops.pcg_p(st, own(z), own(p))
            if it < max_iter:
                ap_xr()  # the next iteration's first half, queued before the state read
            hs = _state(st)
            if hs["status"] == 1:
                raise NotSpdError("pcg: operator not positive definite (p'Ap <= 0)")
            if hs["status"]:
                raise NotSpdError("pcg: preconditioner not positive definite")
            out.iterations = hs["iterations"]
            if hs["done"]:
                out.converged = True
                break
        out.residual_history = [float(v) for v in hist[: out.iterations].cpu().tolist()]
        return out

    def gather_solution(self, x_local: torch.Tensor):
        """Rank 0 receives every rank's owned rows: the whole level-0 solution (others: None)."""
        R, W, pl = self.rank, self.world, self.plan
        P = self._P(0)
        if R == 0:
            full = self.ops.vec(0, full=True)
            lo, hi = pl.owned(0, 0)
            full[lo * P:hi * P].copy_(x_local)
            ops = []
            for q in range(1, W):
                qlo, qhi = pl.owned(0, q)
                ops.append(("recv", q, full[qlo * P:qhi * P]))
            self.comm.exchange(ops)
            return full
        self.comm.exchange([("send", 0, x_local)])
        return None
