"""TEST INFRASTRUCTURE ONLY: the per-rank work of dist.DistSolver on the CPU.

``HostOps`` implements the interface of ``paper_2102_03515_b200.dist.DeviceOps``
with numpy over the CPU oracle's matrices, so the distributed host logic (slab
plan, halo planes, the rank-to-rank smoother hand-off, the gather onto rank 0,
the PCG scalars) runs under a gloo process group on a machine without a GPU.
Arithmetic follows the reference (linalg.cpp:19-33 row sums from 0 in column
order, amg.cpp:67-88 relax(i)), so an exact-mode distributed V-cycle must equal
the oracle's single-process V-cycle bit for bit.  The product path never uses
this module (DeviceOps runs the sm_100a kernels).
"""
from __future__ import annotations

import numpy as np
import torch


class _Blk:
    def __init__(self, rows, cols, rp, ci, v):
        self.rows, self.cols = rows, cols
        cnt = np.diff(rp)
        k = int(cnt.max()) if rows else 0
        self.V = np.zeros((rows, max(k, 1)))
        self.CI = np.zeros((rows, max(k, 1)), np.int64)
        for i in range(rows):
            s, e = rp[i], rp[i + 1]
            self.V[i, : e - s] = v[s:e]
            self.CI[i, : e - s] = ci[s:e]
        self.rp, self.ci, self.v = rp, ci, v

    def matvec(self, x):
        y = np.zeros(self.rows)  # +0, then += v x in column order (padding adds +-0: exact)
        for k in range(self.V.shape[1]):
            y = y + self.V[:, k] * x[self.CI[:, k]]
        return y


def _rowblock(M, r0, r1, c0, c1):
    rp = M.rp[r0:r1 + 1] - M.rp[r0]
    ci = M.ci[M.rp[r0]:M.rp[r1]]
    v = M.v[M.rp[r0]:M.rp[r1]]
    assert ci.size == 0 or (ci.min() >= c0 and ci.max() < c1), "row block column outside its range"
    return _Blk(r1 - r0, c1 - c0, rp, ci - c0, v)


class HostOps:
    def __init__(self, n: int, rho: float, target: str = "smooth", seed: int = 0):
        import pyoracle as O

        self.O = O
        mesh = O.build_structured_cube(n)
        self.sys = O.build_system(mesh, rho, target, seed)
        self.A = self.sys.A
        self.h = O.build_amg(self.A)
        nl = self.h.num_levels
        self.rows = [self.h.level(l, "A").rows for l in range(nl)]
        self.sides = [round(r ** (1 / 3)) for r in self.rows]
        self.structured = [self.sides[l] ** 3 == self.rows[l] for l in range(nl)]

    def localize(self, plan, rank):
        self.plan, self.rank = plan, rank
        self.blkA, self.blkP, self.blkPt, self.slab = [], [], [], []
        for l in range(plan.G):
            P0, P1 = plan.sides[l] ** 2, plan.sides[l + 1] ** 2
            lo, hi = plan.owned(l, rank)
            g0, g1 = plan.ghost(l, rank)
            clo, chi = plan.owned(l + 1, rank)
            cg0, cg1 = plan.ghost(l + 1, rank)
            A = self.h.level(l, "A")
            self.blkA.append(_rowblock(A, lo * P0, hi * P0, g0 * P0, g1 * P0))
            self.blkP.append(_rowblock(self.h.level(l, "P"), lo * P0, hi * P0, cg0 * P1, cg1 * P1))
            self.blkPt.append(_rowblock(self.h.level(l, "Pt"), clo * P1, chi * P1, g0 * P0, g1 * P0))
            self.slab.append((lo, hi, g0, g1, P0, self.blkA[-1]))
        lo, hi = plan.owned(0, rank)
        g0, _ = plan.ghost(0, rank)
        P0 = plan.sides[0] ** 2
        self.f_local = self.vec(0)
        self.f_local[(lo - g0) * P0:(hi - g0) * P0] = torch.from_numpy(self.sys.f[lo * P0:hi * P0].copy())

    def vec(self, l, full=False):
        if full:
            return torch.zeros(self.rows[l], dtype=torch.float64)
        g0, g1 = self.plan.ghost(l, self.rank)
        return torch.zeros((g1 - g0) * self.plan.sides[l] ** 2, dtype=torch.float64)

    def scalar(self):
        return torch.zeros(1, dtype=torch.float64)

    def spmv(self, M, x, y):
        y.numpy()[:] = M.matvec(x.numpy())

    def residual(self, M, r, z, res):
        res.numpy()[:] = r.numpy() - M.matvec(z.numpy())

    def prolong_add(self, M, zc, z):
        z.numpy()[:] = z.numpy() + M.matvec(zc.numpy())

    def sweep(self, l, fwd, f, xin, xout, in_plane):
        lo, hi, g0, g1, P, B = self.slab[l]
        x = xin.numpy().copy() if xin is not None else np.zeros(xout.numel())
        up = lo - 1 if fwd else hi
        if g0 <= up < g1:
            x[(up - g0) * P:(up - g0 + 1) * P] = in_plane.numpy() if in_plane is not None else 0.0
        fv = f.numpy()
        off = (lo - g0) * P
        order = range(B.rows) if fwd else range(B.rows - 1, -1, -1)
        rp, ci, v = B.rp, B.ci, B.v
        xs = x.tolist()
        for i in order:
            g = off + i
            s = float(fv[g])
            d = 0.0
            for k in range(rp[i], rp[i + 1]):
                c = int(ci[k])
                if c == g:
                    d = float(v[k])
                else:
                    s -= float(v[k]) * xs[c]
            if d == 0.0:
                raise RuntimeError("sgs_sweep: zero diagonal")
            xs[g] = s / d
        xo = xout.numpy()
        xo[off:off + B.rows] = np.asarray(xs[off:off + B.rows])

    def dot(self, a, b, out):
        out[0] = self.O.dot(a.numpy(), b.numpy())

    def xr(self, alpha, p, ap, x, r):
        x.numpy()[:] = x.numpy() + alpha * p.numpy()
        r.numpy()[:] = r.numpy() - alpha * ap.numpy()

    def pupd(self, beta, z, p):
        p.numpy()[:] = z.numpy() + beta * p.numpy()

    def coarse(self, level, r, z):
        z.numpy()[:] = self.h.apply_from(level, r.numpy())

    # -- rd_pcg_state on the host: same layout and arithmetic as dist.cu's dpcg_* kernels
    def pcg_state(self):
        return torch.zeros(10, dtype=torch.float64)

    @staticmethod
    def _st(st):
        a = st.numpy()
        return a, a.view(np.int32)

    @staticmethod
    def _rank_sum(parts):
        s = 0.0
        for v in parts.numpy().tolist():
            s = s + v
        return s

    def pcg_begin(self, parts, st):
        a, iv = self._st(st)
        rz = self._rank_sum(parts)
        a[0] = a[1] = rz
        iv[16] = iv[17] = iv[18] = 0
        if rz < 0.0:
            iv[17] = 2
        elif rz == 0.0:
            iv[16] = 1

    def pcg_alpha(self, parts, st):
        a, iv = self._st(st)
        if iv[16] or iv[17]:
            return
        pap = self._rank_sum(parts)
        a[2] = pap
        if not pap > 0.0:
            iv[17] = 1
            return
        a[4] = a[0] / pap

    def pcg_xr(self, st, p, ap, x, r):
        a, iv = self._st(st)
        if iv[16] or iv[17]:
            return
        self.xr(float(a[4]), p, ap, x, r)

    def pcg_check(self, parts, st, tol, hist):
        a, iv = self._st(st)
        if iv[16] or iv[17]:
            return
        rzn = self._rank_sum(parts)
        a[3] = rzn
        if rzn < 0.0:
            iv[17] = 2
            return
        rel = float(np.sqrt(np.float64(rzn) / np.float64(a[1])))
        it = int(iv[18]) + 1
        iv[18] = it
        a[6] = rel
        if it - 1 < hist.numel():
            hist[it - 1] = rel
        if rel <= tol:
            iv[16] = 1
            return
        a[5] = rzn / a[0]
        a[0] = rzn

    def pcg_p(self, st, z, p):
        a, iv = self._st(st)
        if iv[16] or iv[17]:
            return
        self.pupd(float(a[5]), z, p)

    def set_exact(self, exact):
        pass

    def check(self):
        return 0

    def check_raw(self):
        return 0
