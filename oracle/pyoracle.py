"""TEST INFRASTRUCTURE ONLY -- ctypes view of the CPU parity oracle (liboracle.so).

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs.  The product package never imports this module.

Every function mirrors a reference entry point (paths relative to
/root/reference/proj) and returns numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

TARGETS = {"smooth": 0, "box": 1, "nonzero_bc": 2, "ball": 3, "sine_random": 4,
           "zero": 5, "one": 6, "quadratic": 7}

_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_pd = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_pi = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_pu8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


def build():
    """Compile the oracle (make) if the shared object is missing or stale."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    L = C.CDLL(_LIB_PATH)
    sig = {
        "or_last_error": (C.c_char_p, []),
        "or_set_num_threads": (None, [_I]),
        "or_num_threads": (_I, []),
        "or_build_structured_cube": (_I, [_I, C.POINTER(_P)]),
        "or_mesh_free": (None, [_P]),
        "or_mesh_new": (_I, [_I, _pd, _I, _pi, _pu8, C.POINTER(_P)]),
        "or_mesh_info": (None, [_P, C.POINTER(_I), C.POINTER(_I)]),
        "or_mesh_get": (None, [_P, _pd, _pi, _pu8, _pu8, _pi]),
        "or_tet_volume": (_D, [_P, _I]),
        "or_rule_size": (_I, [_I]),
        "or_rule_get": (None, [_I, _pd, _pd]),
        "or_target_eval": (_I, [_I, _I, C.c_uint64, _I, _pd, _pd]),
        "or_pseudo_random_vec": (None, [_I, C.c_uint64, _pd]),
        "or_build_system": (_I, [_P, _D, _I, C.c_uint64, C.POINTER(_P)]),
        "or_system_free": (None, [_P]),
        "or_system_n_dofs": (_I, [_P]),
        "or_system_csr": (_P, [_P, _I]),
        "or_system_get_f": (None, [_P, _pd]),
        "or_system_get_dofmap": (None, [_P, _pi, _pi]),
        "or_assemble_full": (_I, [_P, _I, C.POINTER(_P)]),
        "or_assemble_load": (_I, [_P, _I, C.c_uint64, _pd]),
        "or_csr_new": (_I, [_I, _I, C.c_int64, _pi, _pi, _pd, C.POINTER(_P)]),
        "or_from_triplets": (_I, [_I, _I, C.c_int64, _pi, _pi, _pd, C.POINTER(_P)]),
        "or_csr_free": (None, [_P]),
        "or_csr_info": (None, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(C.c_int64)]),
        "or_csr_get": (None, [_P, _pi, _pi, _pd]),
        "or_spmv": (_I, [_P, _I, _pd, _pd]),
        "or_dense_cholesky_solve": (_I, [_I, _pd, _pd, _pd]),
        "or_dot": (_D, [_I, _pd, _pd]),
        "or_coarsen_redblack": (_I, [_P, _pu8, C.POINTER(_P)]),
        "or_galerkin_coarse": (_I, [_P, _P, C.POINTER(_P)]),
        "or_sgs_sweep": (_I, [_P, _pd, _pd, _pd]),
        "or_build_amg": (_I, [_P, _I, _I, C.POINTER(_P)]),
        "or_amg_free": (None, [_P]),
        "or_amg_num_levels": (_I, [_P]),
        "or_amg_level_csr": (_P, [_P, _I, _I]),
        "or_amg_level_flags": (_I, [_P, _I, _pu8]),
        "or_amg_apply": (_I, [_P, _I, _pd, _pd]),
        "or_amg_apply_from": (_I, [_P, _I, _I, _pd, _pd]),
        "or_pcg": (_I, [_P, _I, _P, _pd, _D, _I, _pd, C.POINTER(_I), C.POINTER(_I), _pd]),
        "or_solve_system_amg": (_I, [_P, _D, _pd, C.POINTER(_I), C.POINTER(_I), C.POINTER(_D), C.POINTER(_D)]),
        "or_pipeline": (_I, [_I, _D, _I, C.c_uint64, _D, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I),
                             C.POINTER(_D), C.POINTER(_D), C.POINTER(_D)]),
        "or_l2_error_manufactured": (_I, [_P, _P, _pd, _D, C.POINTER(_D)]),
        "or_l2_error_target_squared": (_I, [_P, _P, _pd, _I, _I, C.c_uint64, C.POINTER(_D)]),
        "or_target_dual_norm": (_I, [_P, _pd, C.POINTER(_D)]),
        "or_h1_semi_error_manufactured": (_I, [_P, _P, _pd, _D, C.POINTER(_D)]),
        "or_error_norms_target": (_I, [_P, _P, _pd, _I, _I, C.c_uint64, C.POINTER(_D), C.POINTER(_D)]),
        "or_target_grad": (_I, [_I, _I, C.c_uint64, _I, _pd, _pd]),
        "or_partition_geometric": (_I, [_P, _P, _I, _pi, _pi, _pi]),
        "or_bddc_create": (_I, [_P, _P, _I, C.POINTER(_P)]),
        "or_bddc_free": (None, [_P]),
        "or_bddc_info": (None, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
        "or_bddc_interface": (None, [_P, _pi]),
        "or_bddc_coarse": (None, [_P, _pd]),
        "or_bddc_sub_info": (None, [_P, _I, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
        "or_bddc_sub_get": (None, [_P, _I, _pi, _pi, _pi, _pd, _pd, _pd, _pd]),
        "or_bddc_op": (_I, [_P, _I, _I, _pd, _pd, _pd]),
        "or_bddc_solve": (_I, [_P, _P, _I, _D, _I, _pd, C.POINTER(_I), C.POINTER(_I), _pd]),
        "or_estimate": (_I, [_P, _P, _pd, _I, C.c_uint64, _pd, C.POINTER(_D)]),
        "or_mark_dorfler": (_I, [_I, _pd, _D, _pi, C.POINTER(_I)]),
        "or_bisect_marked": (_I, [_P, _I, _pi, C.POINTER(_P)]),
        "or_uniform_refine": (_I, [_P, C.POINTER(_P)]),
        "or_adaptive_solve": (_I, [_P, _I, C.c_uint64, _D, _I, _D, _D, _I, C.POINTER(_I), _pi, _pd, C.POINTER(_P),
                                   _pd, _I]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc):
    if rc == 0:
        return
    msg = lib().or_last_error().decode()
    if rc == 1:
        raise OracleInvalidArgument(msg)
    raise OracleError(msg)


def set_num_threads(n: int):
    lib().or_set_num_threads(int(n))


# ---------------------------------------------------------------- containers
@dataclass
class Csr:
    rows: int
    cols: int
    rp: np.ndarray
    ci: np.ndarray
    v: np.ndarray

    @property
    def nnz(self):
        return int(self.ci.size)

    def dense(self):
        D = np.zeros((self.rows, self.cols))
        for r in range(self.rows):
            s, e = self.rp[r], self.rp[r + 1]
            D[r, self.ci[s:e]] = self.v[s:e]
        return D

    def handle(self):
        h = _P()
        _check(lib().or_csr_new(self.rows, self.cols, self.nnz, np.ascontiguousarray(self.rp, np.int32),
                                np.ascontiguousarray(self.ci, np.int32),
                                np.ascontiguousarray(self.v, np.float64), C.byref(h)))
        return _Handle(h, lib().or_csr_free)

    @staticmethod
    def from_dense(D):
        D = np.asarray(D, dtype=np.float64)
        rp = [0]
        ci, v = [], []
        for r in range(D.shape[0]):
            for c in range(D.shape[1]):
                if D[r, c] != 0.0:
                    ci.append(c)
                    v.append(D[r, c])
            rp.append(len(ci))
        return Csr(D.shape[0], D.shape[1], np.array(rp, np.int32), np.array(ci, np.int32), np.array(v, np.float64))


class _Handle:
    def __init__(self, h, free):
        self.h = h
        self._free = free

    def __del__(self):
        if self.h and self._free is not None:
            self._free(self.h)
            self.h = None


def _csr_from_handle(h) -> Csr:
    rows, cols, nnz = _I(), _I(), C.c_int64()
    lib().or_csr_info(h, C.byref(rows), C.byref(cols), C.byref(nnz))
    rp = np.zeros(rows.value + 1, np.int32)
    ci = np.zeros(max(nnz.value, 1), np.int32)
    v = np.zeros(max(nnz.value, 1), np.float64)
    lib().or_csr_get(h, rp, ci, v)
    return Csr(rows.value, cols.value, rp, ci[: nnz.value].copy(), v[: nnz.value].copy())


# ---------------------------------------------------------------- mesh
@dataclass
class Mesh:
    n: int
    xyz: np.ndarray
    tets: np.ndarray
    boundary: np.ndarray
    refinement_edge: np.ndarray
    generation: np.ndarray
    _h: object = None


def build_structured_cube(n: int) -> Mesh:
    """mesh.cpp:29-65."""
    h = _P()
    _check(lib().or_build_structured_cube(int(n), C.byref(h)))
    hh = _Handle(h, lib().or_mesh_free)
    nv, nt = _I(), _I()
    lib().or_mesh_info(h, C.byref(nv), C.byref(nt))
    xyz = np.zeros((max(nv.value, 1), 3))
    tets = np.zeros((max(nt.value, 1), 4), np.int32)
    b = np.zeros(max(nv.value, 1), np.uint8)
    re = np.zeros(max(nt.value, 1), np.uint8)
    gen = np.zeros(max(nt.value, 1), np.int32)
    lib().or_mesh_get(h, xyz, tets, b, re, gen)
    return Mesh(n, xyz[: nv.value], tets[: nt.value], b[: nv.value], re[: nt.value], gen[: nt.value], hh)


def _mesh_from_handle(h, n: int = -1) -> Mesh:
    hh = _Handle(h, lib().or_mesh_free)
    nv, nt = _I(), _I()
    lib().or_mesh_info(h, C.byref(nv), C.byref(nt))
    xyz = np.zeros((max(nv.value, 1), 3))
    tets = np.zeros((max(nt.value, 1), 4), np.int32)
    b = np.zeros(max(nv.value, 1), np.uint8)
    re = np.zeros(max(nt.value, 1), np.uint8)
    gen = np.zeros(max(nt.value, 1), np.int32)
    lib().or_mesh_get(h, xyz, tets, b, re, gen)
    return Mesh(n, xyz[: nv.value], tets[: nt.value], b[: nv.value], re[: nt.value], gen[: nt.value], hh)


def mesh_from_arrays(xyz, tets, boundary) -> Mesh:
    """A hand-built TetMesh (e.g. test_assembly.cpp:23-33's reference tet)."""
    xyz = np.ascontiguousarray(xyz, np.float64)
    tets = np.ascontiguousarray(tets, np.int32)
    boundary = np.ascontiguousarray(boundary, np.uint8)
    h = _P()
    _check(lib().or_mesh_new(xyz.shape[0], xyz, tets.shape[0], tets, boundary, C.byref(h)))
    return Mesh(-1, xyz, tets, boundary, np.full(tets.shape[0], 3, np.uint8), np.zeros(tets.shape[0], np.int32),
                _Handle(h, lib().or_mesh_free))


def tet_volume(mesh: Mesh, t: int) -> float:
    return lib().or_tet_volume(mesh._h.h, int(t))


def rule(rule_id: int):
    """quadrature.cpp: 0 centroid, 1 degree-2, 2 degree-5 (14 pt), 3 subdivision64."""
    n = lib().or_rule_size(rule_id)
    pts = np.zeros((n, 4))
    w = np.zeros(n)
    lib().or_rule_get(rule_id, pts, w)
    return pts, w


def target_eval(kind: str, xyz, n: int = 0, seed: int = 0) -> np.ndarray:
    xyz = np.ascontiguousarray(np.atleast_2d(xyz), np.float64)
    out = np.zeros(xyz.shape[0])
    _check(lib().or_target_eval(TARGETS[kind], int(n), int(seed), xyz.shape[0], xyz, out))
    return out


def pseudo_random_vec(n: int, seed: int) -> np.ndarray:
    """tests/oracles.hpp:97-108."""
    out = np.zeros(max(n, 1))
    lib().or_pseudo_random_vec(int(n), int(seed), out)
    return out[:n]


# ---------------------------------------------------------------- system
@dataclass
class FemSystem:
    rho: float
    K: Csr
    M: Csr
    A: Csr
    f: np.ndarray
    vertex_to_dof: np.ndarray
    dof_to_vertex: np.ndarray
    _h: object = None

    @property
    def n_dofs(self):
        return int(self.f.size)


def build_system(mesh: Mesh, rho: float, target: str = "smooth", seed: int = 0) -> FemSystem:
    """assembly.cpp:225-238."""
    h = _P()
    _check(lib().or_build_system(mesh._h.h, float(rho), TARGETS[target], int(seed), C.byref(h)))
    hh = _Handle(h, lib().or_system_free)
    nd = lib().or_system_n_dofs(h)
    K = _csr_from_handle(lib().or_system_csr(h, 0))
    M = _csr_from_handle(lib().or_system_csr(h, 1))
    A = _csr_from_handle(lib().or_system_csr(h, 2))
    f = np.zeros(max(nd, 1))
    lib().or_system_get_f(h, f)
    v2d = np.zeros(mesh.xyz.shape[0], np.int32)
    d2v = np.zeros(max(nd, 1), np.int32)
    lib().or_system_get_dofmap(h, v2d, d2v)
    return FemSystem(rho, K, M, A, f[:nd], v2d, d2v[:nd], hh)


def assemble_full(mesh: Mesh, which: str) -> Csr:
    h = _P()
    _check(lib().or_assemble_full(mesh._h.h, 0 if which == "K" else 1, C.byref(h)))
    hh = _Handle(h, lib().or_csr_free)
    return _csr_from_handle(hh.h)


def assemble_load(mesh: Mesh, target: str, seed: int = 0) -> np.ndarray:
    nd = int((mesh.boundary == 0).sum())
    f = np.zeros(max(nd, 1))
    _check(lib().or_assemble_load(mesh._h.h, TARGETS[target], int(seed), f))
    return f[:nd]


# ---------------------------------------------------------------- linalg
def from_triplets(rows, cols, trips) -> Csr:
    ti = np.array([t[0] for t in trips], np.int32)
    tj = np.array([t[1] for t in trips], np.int32)
    tv = np.array([t[2] for t in trips], np.float64)
    if ti.size == 0:
        ti = np.zeros(1, np.int32)[:0]
    h = _P()
    _check(lib().or_from_triplets(int(rows), int(cols), len(trips), np.ascontiguousarray(ti),
                                  np.ascontiguousarray(tj), np.ascontiguousarray(tv), C.byref(h)))
    hh = _Handle(h, lib().or_csr_free)
    return _csr_from_handle(hh.h)


def spmv(A: Csr, x) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(max(A.rows, 1))
    ah = A.handle()
    _check(lib().or_spmv(ah.h, x.size, x if x.size else np.zeros(1), y))
    return y[: A.rows]


def dot(a, b) -> float:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return lib().or_dot(a.size, a, b)


def dense_cholesky_solve(A, b) -> np.ndarray:
    A = np.ascontiguousarray(A, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    x = np.zeros(b.size)
    _check(lib().or_dense_cholesky_solve(b.size, A, b, x))
    return x


# ---------------------------------------------------------------- amg
def coarsen_redblack(A: Csr):
    flags = np.zeros(max(A.rows, 1), np.uint8)
    h = _P()
    ah = A.handle()
    _check(lib().or_coarsen_redblack(ah.h, flags, C.byref(h)))
    hh = _Handle(h, lib().or_csr_free)
    return flags[: A.rows], _csr_from_handle(hh.h)


def galerkin_coarse(A: Csr, P: Csr) -> Csr:
    h = _P()
    ah, ph = A.handle(), P.handle()
    _check(lib().or_galerkin_coarse(ah.h, ph.h, C.byref(h)))
    hh = _Handle(h, lib().or_csr_free)
    return _csr_from_handle(hh.h)


def sgs_sweep(A: Csr, f, u) -> np.ndarray:
    f = np.ascontiguousarray(f, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    out = np.zeros(max(A.rows, 1))
    ah = A.handle()
    _check(lib().or_sgs_sweep(ah.h, f if f.size else np.zeros(1), u if u.size else np.zeros(1), out))
    return out[: A.rows]


class AmgHierarchy:
    """amg.hpp:13-24 / amg.cpp:90-117."""

    def __init__(self, A: Csr, coarsest_threshold: int = 64, smoothing_steps: int = 1):
        h = _P()
        ah = A.handle()
        _check(lib().or_build_amg(ah.h, int(coarsest_threshold), int(smoothing_steps), C.byref(h)))
        self._h = _Handle(h, lib().or_amg_free)
        self.n = A.rows

    @property
    def num_levels(self):
        return lib().or_amg_num_levels(self._h.h)

    def level(self, l: int, which: str = "A"):
        p = lib().or_amg_level_csr(self._h.h, int(l), {"A": 0, "P": 1, "Pt": 2}[which])
        return None if not p else _csr_from_handle(p)

    def flags(self, l: int):
        A = self.level(l, "A")
        f = np.zeros(max(A.rows, 1), np.uint8)
        if lib().or_amg_level_flags(self._h.h, int(l), f) != 0:
            return None
        return f[: A.rows]

    def apply(self, r) -> np.ndarray:
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(max(r.size, 1))
        _check(lib().or_amg_apply(self._h.h, r.size, r if r.size else np.zeros(1), z))
        return z[: r.size]

    def apply_from(self, level: int, r) -> np.ndarray:
        """The V-cycle entered at `level` (amg.cpp:121-132): the coarse tail of a distributed cycle."""
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(max(r.size, 1))
        _check(lib().or_amg_apply_from(self._h.h, int(level), r.size, r if r.size else np.zeros(1), z))
        return z[: r.size]


def build_amg(A: Csr, coarsest_threshold: int = 64, smoothing_steps: int = 1) -> AmgHierarchy:
    return AmgHierarchy(A, coarsest_threshold, smoothing_steps)


@dataclass
class PcgResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_history: np.ndarray


def pcg(A: Csr, precond="amg", f=None, tol=1e-8, max_iter=500, hierarchy: AmgHierarchy | None = None) -> PcgResult:
    """linalg.cpp:64-102; precond in {'identity','jacobi','amg'}."""
    f = np.ascontiguousarray(f, np.float64)
    kind = {"identity": 0, "jacobi": 1, "amg": 2}[precond]
    if kind == 2 and hierarchy is None:
        hierarchy = build_amg(A)
    x = np.zeros(max(f.size, 1))
    hist = np.zeros(max(max_iter, 1))
    it, conv = _I(), _I()
    ah = A.handle()
    _check(lib().or_pcg(ah.h, kind, hierarchy._h.h if hierarchy is not None else None,
                        f if f.size else np.zeros(1), float(tol), int(max_iter), x, C.byref(it), C.byref(conv), hist))
    return PcgResult(x[: f.size], it.value, bool(conv.value), hist[: it.value].copy())


@dataclass
class SolveOutcome:
    u: np.ndarray
    iterations: int
    converged: bool
    setup_seconds: float
    solve_seconds: float


def solve_system_amg(sys: FemSystem, tol: float = 1e-8) -> SolveOutcome:
    """bench.cpp:185-241, PrecondKind::amg branch (:215-225)."""
    u = np.zeros(max(sys.n_dofs, 1))
    it, conv = _I(), _I()
    ts, tv = _D(), _D()
    _check(lib().or_solve_system_amg(sys._h.h, float(tol), u, C.byref(it), C.byref(conv), C.byref(ts), C.byref(tv)))
    return SolveOutcome(u[: sys.n_dofs], it.value, bool(conv.value), ts.value, tv.value)


def pipeline(n: int, rho: float, target: str = "ball", seed: int = 0, tol: float = 1e-8) -> dict:
    """Mesh + build_system, build_amg, pcg on the CPU, timed in C++ (bench.cpp:193-224)."""
    it, conv, nd = _I(), _I(), _I()
    tb, ts, tv = _D(), _D(), _D()
    _check(lib().or_pipeline(int(n), float(rho), TARGETS[target], int(seed), float(tol), C.byref(it), C.byref(conv),
                             C.byref(nd), C.byref(tb), C.byref(ts), C.byref(tv)))
    return {"iterations": it.value, "converged": bool(conv.value), "n_dofs": nd.value, "build_s": tb.value,
            "setup_s": ts.value, "solve_s": tv.value, "total_s": tb.value + ts.value + tv.value}


def l2_error_manufactured(mesh: Mesh, sys: FemSystem, coeffs, rho_exact: float) -> float:
    out = _D()
    _check(lib().or_l2_error_manufactured(mesh._h.h, sys._h.h, np.ascontiguousarray(coeffs, np.float64),
                                          float(rho_exact), C.byref(out)))
    return out.value


def h1_semi_error_manufactured(mesh: Mesh, sys: FemSystem, coeffs, rho_exact: float) -> float:
    out = _D()
    _check(lib().or_h1_semi_error_manufactured(mesh._h.h, sys._h.h, np.ascontiguousarray(coeffs, np.float64),
                                               float(rho_exact), C.byref(out)))
    return out.value


def l2_error_target_squared(mesh: Mesh, sys: FemSystem, coeffs, target: str, n: int = 0, seed: int = 0) -> float:
    """assembly.cpp:312-331: squared L2 distance of the P1 field to the target, the target's rule."""
    out = _D()
    _check(lib().or_l2_error_target_squared(mesh._h.h, sys._h.h, np.ascontiguousarray(coeffs, np.float64),
                                            TARGETS[target], int(n), int(seed), C.byref(out)))
    return out.value


def error_norms_target(mesh: Mesh, sys: FemSystem, coeffs, target: str, n: int = 0, seed: int = 0):
    """assembly.cpp:265-310 with the target field as the exact function: (||u_h - u_bar||_L2,
    ||grad(u_h - u_bar)||_L2), degree-5 rule; grad(u_bar) from Target::grad."""
    l2, h1 = _D(), _D()
    _check(lib().or_error_norms_target(mesh._h.h, sys._h.h, np.ascontiguousarray(coeffs, np.float64),
                                       TARGETS[target], int(n), int(seed), C.byref(l2), C.byref(h1)))
    return l2.value, h1.value


def target_grad(kind: str, xyz, n: int = 0, seed: int = 0) -> np.ndarray:
    """The exact gradient of a target field at points xyz [npts, 3]."""
    xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
    out = np.zeros_like(xyz)
    _check(lib().or_target_grad(TARGETS[kind], int(n), int(seed), xyz.shape[0], xyz, out))
    return out


def target_dual_norm(sys: FemSystem, coeffs) -> float:
    """bench.cpp:55-63: ||f - M u||_{H^-1} via K (dense LLT for n <= 2000, else AMG-PCG at 1e-11)."""
    out = _D()
    _check(lib().or_target_dual_norm(sys._h.h, np.ascontiguousarray(coeffs, np.float64), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- adaptivity (§8(f)3)
def estimate(mesh: Mesh, sys: FemSystem, coeffs, target: str, seed: int = 0):
    """adapt.cpp:35-124 -> (per_tet, global)."""
    per = np.zeros(max(mesh.tets.shape[0], 1))
    g = _D()
    _check(lib().or_estimate(mesh._h.h, sys._h.h, np.ascontiguousarray(coeffs, np.float64), TARGETS[target],
                             int(seed), per, C.byref(g)))
    return per[: mesh.tets.shape[0]], g.value


def mark_dorfler(eta, theta: float) -> np.ndarray:
    """adapt.cpp:126-150 -> marked tet ids in marking order."""
    eta = np.ascontiguousarray(eta, np.float64)
    out = np.zeros(max(eta.size, 1), np.int32)
    k = _I()
    _check(lib().or_mark_dorfler(eta.size, eta if eta.size else np.zeros(1), float(theta), out, C.byref(k)))
    return out[: k.value]


def bisect_marked(mesh: Mesh, marked) -> Mesh:
    """mesh.cpp:67-145."""
    mk = np.ascontiguousarray(marked, np.int32).reshape(-1)
    h = _P()
    _check(lib().or_bisect_marked(mesh._h.h, mk.size, mk if mk.size else np.zeros(1, np.int32), C.byref(h)))
    return _mesh_from_handle(h)


def uniform_refine(mesh: Mesh) -> Mesh:
    """mesh.cpp:147-156."""
    h = _P()
    _check(lib().or_uniform_refine(mesh._h.h, C.byref(h)))
    return _mesh_from_handle(h)


def adaptive_solve(mesh: Mesh, target: str, rho: float, dof_budget: int, tol: float = 1e-8, theta: float = 0.5,
                   seed: int = 0, cap: int = 256, coeffs_cap: int = 1 << 22):
    """adapt.cpp:152-205 with the AMG solver -> (history rows, final mesh, final coefficients)."""
    k = _I()
    hi = np.zeros(3 * cap, np.int32)
    hd = np.zeros(3 * cap)
    fm = _P()
    co = np.zeros(coeffs_cap)
    _check(lib().or_adaptive_solve(mesh._h.h, TARGETS[target], int(seed), float(rho), int(dof_budget), float(tol),
                                   float(theta), cap, C.byref(k), hi, hd, C.byref(fm), co, coeffs_cap))
    rows = [dict(level=int(hi[3 * i]), dofs=int(hi[3 * i + 1]), iterations=int(hi[3 * i + 2]), eta=float(hd[3 * i]),
                 err_l2_sq=float(hd[3 * i + 1]), err_hm1_sq=float(hd[3 * i + 2])) for i in range(min(k.value, cap))]
    final = _mesh_from_handle(fm)
    return rows, final, co[: rows[-1]["dofs"]].copy()


# ---------------------------------------------------------------- BDDC (§8(f)4)
def partition_geometric(mesh: Mesh, sys: FemSystem, p: int):
    """bddc.cpp:45-111 -> (owner per tet, dof_subdomains list per dof)."""
    nt, nd = mesh.tets.shape[0], sys.n_dofs
    owner = np.zeros(max(nt, 1), np.int32)
    cnt = np.zeros(max(nd, 1), np.int32)
    subs = np.zeros(max(8 * nd, 1), np.int32)
    _check(lib().or_partition_geometric(mesh._h.h, sys._h.h, int(p), owner, cnt, subs))
    return owner[:nt], [list(subs[8 * d:8 * d + cnt[d]]) for d in range(nd)]


class Bddc:
    """bddc.hpp BddcOperator (the oracle's restatement)."""

    def __init__(self, mesh: Mesh, sys: FemSystem, p: int):
        h = _P()
        _check(lib().or_bddc_create(mesh._h.h, sys._h.h, int(p), C.byref(h)))
        self._h = _Handle(h, lib().or_bddc_free)
        self.n_dofs = sys.n_dofs
        ni, npr, pp = _I(), _I(), _I()
        lib().or_bddc_info(h, C.byref(ni), C.byref(npr), C.byref(pp))
        self.n_interface, self.n_primal, self.p = ni.value, npr.value, pp.value
        self.interface_dofs = np.zeros(max(ni.value, 1), np.int32)
        lib().or_bddc_interface(h, self.interface_dofs)
        self.interface_dofs = self.interface_dofs[: ni.value]

    def coarse_matrix(self):
        out = np.zeros(max(self.n_primal ** 2, 1))
        lib().or_bddc_coarse(self._h.h, out)
        return out[: self.n_primal ** 2].reshape(self.n_primal, self.n_primal)

    def sub(self, s: int) -> dict:
        nI, nB, nc = _I(), _I(), _I()
        lib().or_bddc_sub_info(self._h.h, int(s), C.byref(nI), C.byref(nB), C.byref(nc))
        nB_, nc_ = nB.value, nc.value
        b = np.zeros(max(nB_, 1), np.int32)
        bi = np.zeros(max(nB_, 1), np.int32)
        pi = np.zeros(max(nc_, 1), np.int32)
        sc = np.zeros(max(nB_, 1))
        Cm = np.zeros(max(nc_ * nB_, 1))
        Ph = np.zeros(max(nc_ * nB_, 1))
        S = np.zeros(max(nB_ * nB_, 1))
        lib().or_bddc_sub_get(self._h.h, int(s), b, bi, pi, sc, Cm, Ph, S)
        return dict(nI=nI.value, nB=nB_, ncon=nc_, boundary=b[:nB_], boundary_index=bi[:nB_], primal_index=pi[:nc_],
                    scaling=sc[:nB_], C=Cm[:nc_ * nB_].reshape(nc_, nB_), Phi=Ph[:nc_ * nB_].reshape(nB_, nc_),
                    S=S[:nB_ * nB_].reshape(nB_, nB_))

    def _op(self, which, x, f=None, n_out=None):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(max(n_out, 1))
        fv = np.ascontiguousarray(f if f is not None else np.zeros(max(self.n_dofs, 1)), np.float64)
        _check(lib().or_bddc_op(self._h.h, which, x.size, x if x.size else np.zeros(1), fv, out))
        return out[:n_out]

    def schur_apply(self, x):
        return self._op(0, x, n_out=self.n_interface)

    def reduce_rhs(self, f):
        return self._op(1, f, n_out=self.n_interface)

    def expand_solution(self, uC, f):
        return self._op(2, uC, f=f, n_out=self.n_dofs)

    def apply(self, r):
        return self._op(3, r, n_out=self.n_interface)


def bddc_solve(mesh: Mesh, sys: FemSystem, p: int, tol: float = 1e-8, max_iter: int = 500) -> PcgResult:
    """bddc.cpp:440-456."""
    u = np.zeros(max(sys.n_dofs, 1))
    hist = np.zeros(max(max_iter, 1))
    it, conv = _I(), _I()
    _check(lib().or_bddc_solve(mesh._h.h, sys._h.h, int(p), float(tol), int(max_iter), u, C.byref(it), C.byref(conv),
                               hist))
    return PcgResult(u[: sys.n_dofs], it.value, bool(conv.value), hist[: it.value].copy())
