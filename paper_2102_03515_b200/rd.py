"""Host-side mirror of the reference rd:: API over the rd_gpu C-ABI (include/rd_gpu.h).

Names, argument meaning and error behaviour follow the reference library
(/root/reference/proj/include/rd/*.hpp); every call runs the sm_100a kernels in
``_build/librd_gpu.so``.  There is no CPU fallback: importing this module on a
machine without the built library raises, and every compute call without a
CUDA device raises :class:`RdCudaError`.

Error mapping: RD_EINVAL -> ValueError (std::invalid_argument),
RD_ENOTSPD / RD_EZERODIAG / RD_EDEGENERATE -> RuntimeError subclasses
(std::runtime_error), CUDA failures -> RdCudaError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RD_GPU_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("RD_GPU_LIB") or os.path.join(_HERE, "_build", "librd_gpu.so")

RD_OK, RD_EINVAL, RD_ERUNTIME, RD_ENOTSPD, RD_EZERODIAG, RD_ECUDA, RD_ENCCL, RD_EDEGENERATE = range(8)
RD_GS_SPECULATION_MISS = 0x5EC  # rd_gpu_synchronize after asynchronous speculative sweeps: rerun exactly

TARGETS = {"smooth": 0, "box": 1, "nonzero_bc": 2, "ball": 3, "sine_random": 4, "zero": 5, "one": 6,
           "quadratic": 7}


class RdError(RuntimeError):
    pass


class RdInvalidArgument(RdError, ValueError):
    pass


class RdNotSpdError(RdError):
    pass


class RdZeroDiagonalError(RdError):
    pass


class RdDegenerateTetError(RdError):
    pass


class RdCudaError(RdError):
    pass


class RdSpeculationMiss(RdError):
    """An asynchronous speculative lattice sweep left the division fast path: rerun exactly."""


_EXC = {RD_EINVAL: RdInvalidArgument, RD_ENOTSPD: RdNotSpdError, RD_EZERODIAG: RdZeroDiagonalError,
        RD_EDEGENERATE: RdDegenerateTetError, RD_ECUDA: RdCudaError, RD_GS_SPECULATION_MISS: RdSpeculationMiss}

_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_lib = None
_closing = False  # set at interpreter exit: handles are then leaked to the process teardown


def _at_exit():
    global _closing
    _closing = True


import atexit  # noqa: E402

atexit.register(_at_exit)


def library_path() -> str:
    return LIB_PATH


def lib():
    """Load librd_gpu.so; raise if it was not built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"rd_gpu CUDA library missing at {LIB_PATH}: run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    sig = {
        "rd_gpu_version": (C.c_char_p, []),
        "rd_gpu_ctx_create": (_I, [_I, _P, C.POINTER(_P)]),
        "rd_gpu_ctx_destroy": (None, [_P]),
        "rd_gpu_last_error": (C.c_char_p, [_P]),
        "rd_gpu_ctx_stream": (_P, [_P]),
        "rd_gpu_synchronize": (_I, [_P]),
        "rd_gpu_launch_count": (C.c_int64, [_P]),
        "rd_gpu_pool_bytes": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "rd_gpu_copy": (_I, [_P, _P, _P, C.c_size_t]),
        "rd_gpu_build_structured_cube": (_I, [_P, _I, C.POINTER(_P)]),
        "rd_gpu_mesh_create": (_I, [_P, _I, _P, _I, _P, _P, C.POINTER(_P)]),
        "rd_gpu_mesh_free": (None, [_P]),
        "rd_gpu_mesh_info": (_I, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
        "rd_gpu_mesh_download": (_I, [_P, _P, _P, _P]),
        "rd_gpu_build_system": (_I, [_P, _P, _D, _P, C.POINTER(_P)]),
        "rd_gpu_system_free": (None, [_P]),
        "rd_gpu_system_n_dofs": (_I, [_P]),
        "rd_gpu_system_matrix": (_P, [_P, _I]),
        "rd_gpu_system_load": (_P, [_P]),
        "rd_gpu_system_dofmap": (_I, [_P, _P, _P]),
        "rd_gpu_csr_create": (_I, [_P, _I, _I, C.c_int64, _P, _P, _P, C.POINTER(_P)]),
        "rd_gpu_csr_free": (None, [_P]),
        "rd_gpu_csr_info": (_I, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(C.c_int64)]),
        "rd_gpu_csr_download": (_I, [_P, _P, _P, _P]),
        "rd_gpu_spmv": (_I, [_P, _P, _P, _P]),
        "rd_gpu_dot": (_I, [_P, _I, _P, _P, _P]),
        "rd_gpu_coarsen_redblack": (_I, [_P, _P, _P, C.POINTER(_P)]),
        "rd_gpu_galerkin_coarse": (_I, [_P, _P, _P, C.POINTER(_P)]),
        "rd_gpu_sgs_sweep": (_I, [_P, _P, _P, _P, _P]),
        "rd_gpu_amg_setup": (_I, [_P, _P, _I, _I, C.POINTER(_P)]),
        "rd_gpu_amg_free": (None, [_P]),
        "rd_gpu_amg_num_levels": (_I, [_P]),
        "rd_gpu_amg_level_matrix": (_P, [_P, _I, _I]),
        "rd_gpu_amg_level_flags": (_I, [_P, _I, _P]),
        "rd_gpu_amg_level_structured": (_I, [_P, _I]),
        "rd_gpu_amg_apply": (_I, [_P, _P, _P]),
        "rd_gpu_amg_level_sweep": (_I, [_P, _I, _I, _P, _P, _P]),
        "rd_gpu_pcg": (_I, [_P, _P, _P, _P, _D, _I, _P, _P, _P]),
        "rd_gpu_solve_system_amg": (_I, [_P, _P, _P, _D, _P, _P]),
        "rd_gpu_solve_host_mesh": (_I, [_P, _I, _P, _I, _P, _P, _D, _P, _D, _P, _P, _P]),
        "rd_gpu_error_norms": (_I, [_P, _P, _P, _P, _D, C.POINTER(_D), C.POINTER(_D)]),
        "rd_gpu_l2_error_target_squared": (_I, [_P, _P, _P, _P, _P, C.POINTER(_D)]),
        "rd_gpu_error_norms_target": (_I, [_P, _P, _P, _P, _P, C.POINTER(_D), C.POINTER(_D)]),
        "rd_gpu_target_dual_norm": (_I, [_P, _P, _P, C.POINTER(_D)]),
        # distributed (z-slab) pieces, dist.py
        "rd_gpu_ctx_set_exact_sweeps": (_I, [_P, _I]),
        "rd_gpu_csr_rowblock": (_I, [_P, _P, _I, _I, _I, _I, C.POINTER(_P)]),
        "rd_gpu_residual": (_I, [_P, _P, _P, _P, _P]),
        "rd_gpu_prolong_add": (_I, [_P, _P, _P, _P]),
        "rd_gpu_dot_async": (_I, [_P, _I, _P, _P, _P]),
        "rd_gpu_pcg_update_xr": (_I, [_P, C.c_int64, _D, _P, _P, _P, _P]),
        "rd_gpu_pcg_update_p": (_I, [_P, C.c_int64, _D, _P, _P]),
        "rd_gpu_mesh_tags": (_I, [_P, _P, _P]),
        "rd_gpu_mesh_set_tags": (_I, [_P, _P, _P]),
        "rd_gpu_bisect_marked": (_I, [_P, _P, _I, _P, _P]),
        "rd_gpu_uniform_refine": (_I, [_P, _P, _P]),
        "rd_gpu_estimate": (_I, [_P, _P, _P, _P, _P, _P, _P]),
        "rd_gpu_mark_dorfler": (_I, [_P, _I, _P, _D, _P, _P]),
        "rd_gpu_adaptive_solve": (_I, [_P, _P, _P, _D, _I, _D, _D, _P, _I, _P, _P, _P, _I]),
        "rd_gpu_partition_geometric": (_I, [_P, _P, _P, _I, _P]),
        "rd_gpu_bddc_create": (_I, [_P, _P, _P, _I, _P]),
        "rd_gpu_bddc_free": (None, [_P]),
        "rd_gpu_bddc_info": (_I, [_P, _P, _P]),
        "rd_gpu_bddc_interface_dofs": (_I, [_P, _P]),
        "rd_gpu_bddc_coarse_matrix": (_I, [_P, _P]),
        "rd_gpu_bddc_schur_apply": (_I, [_P, _P, _P]),
        "rd_gpu_bddc_reduce_rhs": (_I, [_P, _P, _P]),
        "rd_gpu_bddc_expand": (_I, [_P, _P, _P, _P]),
        "rd_gpu_bddc_apply": (_I, [_P, _P, _P]),
        "rd_gpu_linop_bddc_schur": (_I, [_P, _P]),
        "rd_gpu_linop_bddc": (_I, [_P, _P]),
        "rd_gpu_bddc_solve": (_I, [_P, _P, _P, _I, _D, _I, _P, _P, _P]),
        "rd_gpu_linop_identity": (_I, [_P]),
        "rd_gpu_linop_csr": (_I, [_P, _P]),
        "rd_gpu_linop_amg": (_I, [_P, _P]),
        "rd_gpu_jacobi_create": (_I, [_P, _P, _P]),
        "rd_gpu_jacobi_free": (None, [_P]),
        "rd_gpu_linop_jacobi": (_I, [_P, _P]),
        "rd_gpu_linop_apply": (_I, [_P, _LinOp, C.c_int64, _P, _P]),
        "rd_gpu_pcg_linop": (_I, [_P, C.c_int64, _LinOp, _LinOp, _P, _D, _I, _P, _P, _P]),
        "rd_gpu_pcg_dist_begin": (_I, [_P, _I, _P, _P]),
        "rd_gpu_pcg_dist_alpha": (_I, [_P, _I, _P, _P]),
        "rd_gpu_pcg_dist_xr": (_I, [_P, C.c_int64, _P, _P, _P, _P, _P]),
        "rd_gpu_pcg_dist_check": (_I, [_P, _I, _P, _P, _D, _P, _I]),
        "rd_gpu_pcg_dist_p": (_I, [_P, C.c_int64, _P, _P, _P]),
        "rd_gpu_amg_apply_from": (_I, [_P, _I, _P, _P]),
        "rd_gpu_slab_create": (_I, [_P, _P, _I, _I, C.POINTER(_P)]),
        "rd_gpu_slab_free": (None, [_P]),
        "rd_gpu_slab_info": (_I, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
        "rd_gpu_slab_sweep": (_I, [_P, _I, _P, _P, _P, _P]),
        "rd_gpu_slab_link": (_I, [_P, _P, _P]),
        "rd_gpu_slab_ipc_handle": (_I, [_P, _P]),
        "rd_gpu_slab_open_peer": (_I, [_P, _I, _P, _I]),
        "rd_gpu_slab_sweep_pipelined": (_I, [_P, _I, _P, _P, _P]),
        "rd_gpu_slab_sweep_multi": (_I, [_I, _P, _I, _P, _P, _P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class _PcgReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int)]


# rd_linop (include/rd_gpu.h): y = op(x) on device vectors, on the context's stream
_LINOP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


class _LinOp(C.Structure):
    _fields_ = [("apply", _LINOP_FN), ("user", C.c_void_p)]


class _SolveOutcome(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("setup_seconds", C.c_double),
                ("solve_seconds", C.c_double)]


class _Target(C.Structure):
    _fields_ = [("kind", C.c_int), ("seed", C.c_uint64)]


class _AdaptLevel(C.Structure):
    _fields_ = [("level", C.c_int), ("dofs", C.c_int), ("iterations", C.c_int), ("eta", C.c_double),
                ("err_l2_sq", C.c_double), ("err_hm1_sq", C.c_double), ("seconds", C.c_double)]


def _ptr(x):
    """Raw pointer of a numpy array (host), a torch tensor (data_ptr) or an int."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return C.c_void_p(x.ctypes.data)
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    if isinstance(x, int):
        return C.c_void_p(x)
    raise TypeError(f"unsupported buffer type {type(x)!r}")


# ------------------------------------------------------------------ context
class Context:
    """rd_ctx: one device, one stream."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = _P()
        rc = lib().rd_gpu_ctx_create(int(device), C.c_void_p(stream) if stream else None, C.byref(h))
        if rc != RD_OK:
            raise _EXC.get(rc, RdError)(lib().rd_gpu_last_error(None).decode())
        self.h = h
        self.device = device

    def check(self, rc):
        if rc != RD_OK:
            raise _EXC.get(rc, RdError)(lib().rd_gpu_last_error(self.h).decode())

    @property
    def stream(self) -> int:
        return lib().rd_gpu_ctx_stream(self.h) or 0

    @property
    def launch_count(self) -> int:
        return int(lib().rd_gpu_launch_count(self.h))

    def pool_bytes(self):
        """(used, reserved) bytes of the library's memory pool on this context's device."""
        u, r = C.c_uint64(0), C.c_uint64(0)
        self.check(lib().rd_gpu_pool_bytes(self.h, C.byref(u), C.byref(r)))
        return int(u.value), int(r.value)

    def synchronize(self):
        self.check(lib().rd_gpu_synchronize(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None) and not _closing:
                lib().rd_gpu_ctx_destroy(self.h)
        except Exception:
            pass
        self.h = None


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ------------------------------------------------------------------ CSR
class Csr:
    """SpMat (types.hpp:14): int32 row_ptr/col_idx, fp64 values, resident in HBM."""

    def __init__(self, h, ctx: Context, owner=None, owned=True):
        self.h = h
        self.ctx = ctx
        self._owner = owner  # keeps a borrowed view's parent alive
        self._owned = owned
        r, c, z = _I(), _I(), C.c_int64()
        lib().rd_gpu_csr_info(h, C.byref(r), C.byref(c), C.byref(z))
        self.rows, self.cols, self.nnz = r.value, c.value, z.value

    @staticmethod
    def from_arrays(rows, cols, rp, ci, v, ctx: Context | None = None) -> "Csr":
        ctx = ctx or default_context()
        rp = np.ascontiguousarray(rp, np.int32)
        ci = np.ascontiguousarray(ci, np.int32)
        v = np.ascontiguousarray(v, np.float64)
        h = _P()
        ctx.check(lib().rd_gpu_csr_create(ctx.h, int(rows), int(cols), int(ci.size), _ptr(rp),
                                          _ptr(ci) if ci.size else None, _ptr(v) if v.size else None, C.byref(h)))
        return Csr(h, ctx)

    @staticmethod
    def from_scipy_like(A, ctx: Context | None = None) -> "Csr":
        return Csr.from_arrays(A.rows, A.cols, A.rp, A.ci, A.v, ctx)

    def download(self):
        rp = np.zeros(self.rows + 1, np.int32)
        ci = np.zeros(max(self.nnz, 1), np.int32)
        v = np.zeros(max(self.nnz, 1), np.float64)
        self.ctx.check(lib().rd_gpu_csr_download(self.h, _ptr(rp), _ptr(ci), _ptr(v)))
        return rp, ci[: self.nnz], v[: self.nnz]

    def dense(self):
        rp, ci, v = self.download()
        D = np.zeros((self.rows, self.cols))
        for r in range(self.rows):
            D[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
        return D

    def __del__(self):
        try:
            if getattr(self, "h", None) and self._owned and not _closing:
                lib().rd_gpu_csr_free(self.h)
        except Exception:
            pass
        self.h = None


def from_triplets(rows, cols, trips, ctx: Context | None = None) -> Csr:
    """linalg.cpp:11-17 semantics (duplicates summed in insertion order, zeros pruned), staged on
    the host only to build the input matrix of a test; every compute call then runs on the device."""
    acc: dict = {}
    order = []
    for (i, j, val) in trips:
        if not (0 <= i < rows and 0 <= j < cols):
            raise ValueError("from_triplets: index out of range")
        if (i, j) not in acc:
            acc[(i, j)] = val
            order.append((i, j))
        else:
            acc[(i, j)] = acc[(i, j)] + val
    keys = sorted(k for k in order if acc[k] != 0.0)
    rp = np.zeros(rows + 1, np.int32)
    for (i, _) in keys:
        rp[i + 1] += 1
    rp = np.cumsum(rp).astype(np.int32)
    ci = np.array([k[1] for k in keys], np.int32)
    v = np.array([acc[k] for k in keys], np.float64)
    return Csr.from_arrays(rows, cols, rp, ci, v, ctx)


# ------------------------------------------------------------------ mesh / system
class TetMesh:
    """mesh.hpp:13-24, resident in HBM."""

    def __init__(self, h, ctx: Context):
        self.h = h
        self.ctx = ctx
        nv, nt, ln = _I(), _I(), _I()
        lib().rd_gpu_mesh_info(h, C.byref(nv), C.byref(nt), C.byref(ln))
        self.n_vertices, self.n_tets, self.lattice_n = nv.value, nt.value, ln.value

    def download(self):
        xyz = np.zeros((max(self.n_vertices, 1), 3))
        tets = np.zeros((max(self.n_tets, 1), 4), np.int32)
        b = np.zeros(max(self.n_vertices, 1), np.uint8)
        self.ctx.check(lib().rd_gpu_mesh_download(self.h, _ptr(xyz), _ptr(tets), _ptr(b)))
        return xyz[: self.n_vertices], tets[: self.n_tets], b[: self.n_vertices]

    def tags(self):
        """mesh.hpp:17-20: (refinement_edge u8[n_tets], generation i32[n_tets])."""
        re = np.zeros(max(self.n_tets, 1), np.uint8)
        gen = np.zeros(max(self.n_tets, 1), np.int32)
        self.ctx.check(lib().rd_gpu_mesh_tags(self.h, _ptr(re), _ptr(gen)))
        return re[: self.n_tets], gen[: self.n_tets]

    def set_tags(self, refinement_edge, generation):
        re = np.ascontiguousarray(refinement_edge, np.uint8)
        gen = np.ascontiguousarray(generation, np.int32)
        self.ctx.check(lib().rd_gpu_mesh_set_tags(self.h, _ptr(re), _ptr(gen)))

    def __del__(self):
        try:
            if getattr(self, "h", None) and not _closing:
                lib().rd_gpu_mesh_free(self.h)
        except Exception:
            pass
        self.h = None


def build_structured_cube(n: int, ctx: Context | None = None) -> TetMesh:
    """mesh.hpp:36 / mesh.cpp:29-65 on the device."""
    ctx = ctx or default_context()
    h = _P()
    ctx.check(lib().rd_gpu_build_structured_cube(ctx.h, int(n), C.byref(h)))
    return TetMesh(h, ctx)


def mesh_from_arrays(xyz, tets, boundary, ctx: Context | None = None) -> TetMesh:
    """Upload a host rd::TetMesh."""
    ctx = ctx or default_context()
    xyz = np.ascontiguousarray(xyz, np.float64)
    tets = np.ascontiguousarray(tets, np.int32)
    boundary = np.ascontiguousarray(boundary, np.uint8)
    h = _P()
    ctx.check(lib().rd_gpu_mesh_create(ctx.h, xyz.shape[0], _ptr(xyz), tets.shape[0], _ptr(tets), _ptr(boundary),
                                       C.byref(h)))
    return TetMesh(h, ctx)


class FemSystem:
    """assembly.hpp:24-31: K, M, A = rho*K + M, f and the dof map, resident in HBM."""

    def __init__(self, h, ctx: Context, mesh: TetMesh, rho: float):
        self.h = h
        self.ctx = ctx
        self.mesh = mesh
        self.rho = rho
        self.n_dofs = lib().rd_gpu_system_n_dofs(h)

    # K, M, A are views created on access: each holds the system alive, and the
    # system holds no reference back (no cycle, so the device memory is released
    # as soon as the last user drops it, not at the next cyclic GC).
    def _view(self, which: int) -> Csr:
        return Csr(lib().rd_gpu_system_matrix(self.h, which), self.ctx, owner=self, owned=False)

    K = property(lambda self: self._view(0))
    M = property(lambda self: self._view(1))
    A = property(lambda self: self._view(2))

    @property
    def f_ptr(self) -> int:
        """Device pointer of the load vector."""
        return lib().rd_gpu_system_load(self.h) or 0

    def f(self) -> np.ndarray:
        """Download the load vector."""
        out = np.zeros(max(self.n_dofs, 1))
        if self.n_dofs:
            self.ctx.check(lib().rd_gpu_copy(self.ctx.h, _ptr(out), C.c_void_p(self.f_ptr), 8 * self.n_dofs))
        return out[: self.n_dofs]

    def dofmap(self):
        v2d = np.zeros(max(self.mesh.n_vertices, 1), np.int32)
        d2v = np.zeros(max(self.n_dofs, 1), np.int32)
        self.ctx.check(lib().rd_gpu_system_dofmap(self.h, _ptr(v2d), _ptr(d2v)))
        return v2d[: self.mesh.n_vertices], d2v[: self.n_dofs]

    def __del__(self):
        try:
            if getattr(self, "h", None) and not _closing:
                lib().rd_gpu_system_free(self.h)
        except Exception:
            pass
        self.h = None


def build_system(mesh: TetMesh, rho: float, target: str = "smooth", seed: int = 0) -> FemSystem:
    """assembly.hpp:48 / assembly.cpp:225-238 on the device."""
    ctx = mesh.ctx
    t = _Target(TARGETS[target], int(seed))
    h = _P()
    ctx.check(lib().rd_gpu_build_system(ctx.h, mesh.h, float(rho), C.byref(t), C.byref(h)))
    return FemSystem(h, ctx, mesh, rho)


def error_norms(sys: FemSystem, coeffs, rho_exact: float):
    """assembly.hpp:59-61 l2_error / h1_semi_error against rd::manufactured_exact(rho_exact)
    (target.cpp:45-58), on the device.  `coeffs`: interior dof values (host array or device pointer)."""
    ctx = sys.ctx
    if isinstance(coeffs, np.ndarray) or isinstance(coeffs, (list, tuple)):
        coeffs = np.ascontiguousarray(coeffs, np.float64)
        if coeffs.size != sys.n_dofs:
            raise RdInvalidArgument("error_norms: coefficient vector size mismatch")
    l2, h1 = _D(), _D()
    ctx.check(lib().rd_gpu_error_norms(ctx.h, sys.mesh.h, sys.h, _ptr(coeffs) if sys.n_dofs else None,
                                       float(rho_exact), C.byref(l2), C.byref(h1)))
    return l2.value, h1.value


def l2_error_target_squared(sys: FemSystem, coeffs, target: str, seed: int = 0) -> float:
    """assembly.hpp:62 / assembly.cpp:312-331 on the device: squared L2 distance of the P1 field
    with interior coefficients `coeffs` to the target field (the target's own quadrature rule)."""
    ctx = sys.ctx
    if isinstance(coeffs, np.ndarray) or isinstance(coeffs, (list, tuple)):
        coeffs = np.ascontiguousarray(coeffs, np.float64)
        if coeffs.size != sys.n_dofs:
            raise RdInvalidArgument("l2_error_target_squared: coefficient vector size mismatch")
    t = _Target(TARGETS[target], int(seed))
    out = _D()
    ctx.check(lib().rd_gpu_l2_error_target_squared(ctx.h, sys.mesh.h, sys.h, _ptr(coeffs) if sys.n_dofs else None,
                                                   C.byref(t), C.byref(out)))
    return out.value


def error_norms_target(sys: FemSystem, coeffs, target: str, seed: int = 0):
    """assembly.hpp:59-61 l2_error / h1_semi_error with the target field as the exact function
    (value and gradient), on the device: (||u_h - u_bar||_L2, ||grad(u_h - u_bar)||_L2)."""
    ctx = sys.ctx
    if isinstance(coeffs, np.ndarray) or isinstance(coeffs, (list, tuple)):
        coeffs = np.ascontiguousarray(coeffs, np.float64)
        if coeffs.size != sys.n_dofs:
            raise RdInvalidArgument("error_norms_target: coefficient vector size mismatch")
    t = _Target(TARGETS[target], int(seed))
    l2, h1 = _D(), _D()
    ctx.check(lib().rd_gpu_error_norms_target(ctx.h, sys.mesh.h, sys.h, _ptr(coeffs) if sys.n_dofs else None,
                                              C.byref(t), C.byref(l2), C.byref(h1)))
    return l2.value, h1.value


def target_dual_norm(sys: FemSystem, coeffs) -> float:
    """bench.cpp:55-63 on the device: ||f - M u||_{H^-1} = sqrt(r . K^-1 r)."""
    ctx = sys.ctx
    if isinstance(coeffs, np.ndarray) or isinstance(coeffs, (list, tuple)):
        coeffs = np.ascontiguousarray(coeffs, np.float64)
        if coeffs.size != sys.n_dofs:
            raise RdInvalidArgument("target_dual_norm: coefficient vector size mismatch")
    out = _D()
    ctx.check(lib().rd_gpu_target_dual_norm(ctx.h, sys.h, _ptr(coeffs) if sys.n_dofs else None, C.byref(out)))
    return out.value


# ------------------------------------------------------------------ kernels
def spmv(A: Csr, x) -> np.ndarray:
    """linalg.hpp:30 -- y = A x."""
    x = np.ascontiguousarray(x, np.float64)
    if x.size != A.cols:
        raise RdInvalidArgument("spmv: dimension mismatch")
    y = np.zeros(max(A.rows, 1))
    A.ctx.check(lib().rd_gpu_spmv(A.ctx.h, A.h, _ptr(x), _ptr(y)))
    return y[: A.rows]


def dot(a, b, ctx: Context | None = None) -> float:
    ctx = ctx or default_context()
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    out = np.zeros(1)
    ctx.check(lib().rd_gpu_dot(ctx.h, a.size, _ptr(a), _ptr(b), _ptr(out)))
    return float(out[0])


def coarsen_redblack(A: Csr):
    """amg.hpp:29 -- (coarse flags, P)."""
    flags = np.zeros(max(A.rows, 1), np.uint8)
    h = _P()
    A.ctx.check(lib().rd_gpu_coarsen_redblack(A.ctx.h, A.h, _ptr(flags), C.byref(h)))
    return flags[: A.rows], Csr(h, A.ctx)


def galerkin_coarse(A: Csr, P: Csr) -> Csr:
    """amg.hpp:31 -- prune(P^T A P)."""
    if A.cols != P.rows:
        raise RdInvalidArgument("galerkin_coarse: dims")
    h = _P()
    A.ctx.check(lib().rd_gpu_galerkin_coarse(A.ctx.h, A.h, P.h, C.byref(h)))
    return Csr(h, A.ctx)


def sgs_sweep(A: Csr, f, u) -> np.ndarray:
    """amg.hpp:34 -- one forward then one backward Gauss-Seidel pass."""
    f = np.ascontiguousarray(f, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    out = np.zeros(max(A.rows, 1))
    A.ctx.check(lib().rd_gpu_sgs_sweep(A.ctx.h, A.h, _ptr(f), _ptr(u), _ptr(out)))
    return out[: A.rows]


class AmgHierarchy:
    """amg.hpp:13-24 (levels of A, P, Pt, coarse flags; coarsest LLT) built on the device."""

    def __init__(self, A: Csr, coarsest_threshold: int = 64, smoothing_steps: int = 1):
        self.ctx = A.ctx
        h = _P()
        self.ctx.check(lib().rd_gpu_amg_setup(self.ctx.h, A.h, int(coarsest_threshold), int(smoothing_steps),
                                              C.byref(h)))
        self.h = h
        self.n = A.rows

    @property
    def num_levels(self) -> int:
        return lib().rd_gpu_amg_num_levels(self.h)

    def level(self, l: int, which: str = "A") -> Csr | None:
        p = lib().rd_gpu_amg_level_matrix(self.h, int(l), {"A": 0, "P": 1, "Pt": 2}[which])
        return Csr(p, self.ctx, owner=self, owned=False) if p else None

    def flags(self, l: int):
        A = self.level(l)
        f = np.zeros(max(A.rows, 1), np.uint8)
        rc = lib().rd_gpu_amg_level_flags(self.h, int(l), _ptr(f))
        if rc != RD_OK:
            return None
        return f[: A.rows]

    def structured(self, l: int) -> bool:
        return lib().rd_gpu_amg_level_structured(self.h, int(l)) >= 1

    def uniform(self, l: int) -> bool:
        """Level l's lattice stencil is the same in every row (kept in registers by the smoother)."""
        return lib().rd_gpu_amg_level_structured(self.h, int(l)) == 2

    def stencil_source(self, l: int) -> str:
        """How level l's smoother gets its stencil: generic / packed / uniform / class."""
        return ["generic", "packed", "uniform", "class"][lib().rd_gpu_amg_level_structured(self.h, int(l))]

    def apply(self, r, z=None):
        """amg.hpp:39 amg_apply: one V-cycle, zero initial guess.  Host arrays in -> host array out;
        device buffers (torch tensors / pointers) are used in place and left stream-ordered."""
        if isinstance(r, np.ndarray) or not hasattr(r, "data_ptr"):
            r = np.ascontiguousarray(r, np.float64)
            if r.size != self.n:
                raise RdInvalidArgument("amg_apply: dimension mismatch")
            out = np.zeros(max(self.n, 1))
            self.ctx.check(lib().rd_gpu_amg_apply(self.h, _ptr(r), _ptr(out)))
            return out[: self.n]
        self.ctx.check(lib().rd_gpu_amg_apply(self.h, _ptr(r), _ptr(z)))
        return z

    def level_sweep(self, l: int, forward: bool, f, xin, xout):
        """One GS pass on level l with the V-cycle's kernel (device buffers, stream-ordered)."""
        self.ctx.check(lib().rd_gpu_amg_level_sweep(self.h, int(l), 1 if forward else 0, _ptr(f), _ptr(xin),
                                                    _ptr(xout)))

    def __del__(self):
        try:
            if getattr(self, "h", None) and not _closing:
                lib().rd_gpu_amg_free(self.h)
        except Exception:
            pass
        self.h = None


def build_amg(A: Csr, coarsest_threshold: int = 64, smoothing_steps: int = 1) -> AmgHierarchy:
    return AmgHierarchy(A, coarsest_threshold, smoothing_steps)


@dataclass
class PcgResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_history: np.ndarray


def pcg(A: Csr, precond="amg", f=None, tol: float = 1e-8, max_iter: int = 500,
        hierarchy: AmgHierarchy | None = None) -> PcgResult:
    """linalg.hpp:46-49 with amg_precond(h), the identity, Jacobi, or any LinOp."""
    f = np.ascontiguousarray(f, np.float64)
    if isinstance(precond, LinOp):
        return pcg_linop(A, precond, f, tol, max_iter)
    if precond == "jacobi":
        return pcg_linop(A, jacobi_precond(A), f, tol, max_iter)
    if precond == "amg" and hierarchy is None:
        hierarchy = build_amg(A)
    if precond not in ("amg", "identity"):
        raise RdInvalidArgument(f"unsupported preconditioner {precond!r} on the device path")
    x = np.zeros(max(A.rows, 1))
    hist = np.zeros(max(max_iter, 1))
    rep = _PcgReport()
    A.ctx.check(lib().rd_gpu_pcg(A.ctx.h, A.h, hierarchy.h if precond == "amg" else None, _ptr(f), float(tol),
                                 int(max_iter), _ptr(x), C.byref(rep), _ptr(hist)))
    return PcgResult(x[: A.rows], rep.iterations, bool(rep.converged), hist[: rep.iterations].copy())


# ------------------------------------------------------------------ LinOp (linalg.hpp:11)
class LinOp:
    """rd::LinOp: a fixed linear map y = op(x), applied on the device (rd_linop).  Built-ins come
    from identity_precond / spmv_op / amg_precond / jacobi_precond; `LinOp.from_device_fn(fn, n)`
    wraps a Python callable fn(x, y) on device tensors (torch, on the current stream)."""

    def __init__(self, st: _LinOp, keep=()):
        self._st = st
        self._keep = keep  # objects the operator borrows (matrix, hierarchy, callback)

    def __call__(self, x, ctx: "Context | None" = None):
        """y = op(x): host array in -> host array out (device tensors are used in place)."""
        ctx = ctx or self._ctx()
        if isinstance(x, np.ndarray) or not hasattr(x, "data_ptr"):
            x = np.ascontiguousarray(x, np.float64)
            y = np.zeros(max(x.size, 1))
            ctx.check(lib().rd_gpu_linop_apply(ctx.h, self._st, x.size, _ptr(x), _ptr(y)))
            return y[: x.size]
        y = x.new_empty(x.shape)
        ctx.check(lib().rd_gpu_linop_apply(ctx.h, self._st, x.numel(), _ptr(x), _ptr(y)))
        return y

    def _ctx(self):
        for k in self._keep:
            if hasattr(k, "ctx"):
                return k.ctx
        return default_context()

    @staticmethod
    def from_device_fn(fn, ctx: "Context | None" = None) -> "LinOp":
        """fn(x, y): torch float64 device tensors of n entries; write y = op(x) on the current
        stream (the context's stream is made current around the call)."""
        import torch

        ctx = ctx or default_context()

        def tramp(user, hctx, n, x, y):
            try:
                s = torch.cuda.ExternalStream(lib().rd_gpu_ctx_stream(ctx.h) or 0)
                with torch.cuda.stream(s):
                    xt = _device_view(x, n)
                    yt = _device_view(y, n)
                    fn(xt, yt)
                return RD_OK
            except Exception:  # noqa: BLE001 - an exception cannot cross the C frame
                return RD_ERUNTIME

        cb = _LINOP_FN(tramp)
        op = LinOp(_LinOp(cb, None), keep=(cb, ctx))
        return op


def _device_view(ptr, n):
    """A float64 torch tensor over n doubles of device memory at ptr (no copy)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr or 0), False),
                                    "version": 2}

    return torch.as_tensor(_Arr(), device="cuda")


def identity_precond() -> LinOp:
    """linalg.hpp:39 identity_precond()."""
    st = _LinOp()
    lib().rd_gpu_linop_identity(C.byref(st))
    return LinOp(st)


def spmv_op(A: Csr) -> LinOp:
    """[&A](x) { return spmv(A, x); } (linalg.cpp:104-106)."""
    st = _LinOp()
    A.ctx.check(lib().rd_gpu_linop_csr(A.h, C.byref(st)))
    return LinOp(st, keep=(A,))


def amg_precond(h: "AmgHierarchy") -> LinOp:
    """amg.hpp:42 amg_precond(h): one V-cycle per application."""
    st = _LinOp()
    h.ctx.check(lib().rd_gpu_linop_amg(h.h, C.byref(st)))
    return LinOp(st, keep=(h,))


class _Jacobi:
    def __init__(self, A: Csr):
        self.ctx = A.ctx
        h = _P()
        self.ctx.check(lib().rd_gpu_jacobi_create(self.ctx.h, A.h, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None) and not _closing:
                lib().rd_gpu_jacobi_free(self.h)
        except Exception:
            pass
        self.h = None


def jacobi_precond(A: Csr) -> LinOp:
    """linalg.hpp:40 jacobi_precond(A): r ./ diag(A); RdNotSpdError on a non-positive diagonal."""
    j = _Jacobi(A)
    st = _LinOp()
    A.ctx.check(lib().rd_gpu_linop_jacobi(j.h, C.byref(st)))
    return LinOp(st, keep=(j, A))


def pcg_linop(apply_A, apply_P: LinOp, f, tol: float = 1e-8, max_iter: int = 500,
              ctx: "Context | None" = None) -> PcgResult:
    """linalg.hpp:46-49 pcg(apply_A, apply_P, f, tol, max_iter); apply_A may be a Csr (the SpMat
    overload).  f: host array (x returned on the host)."""
    if isinstance(apply_A, Csr):
        apply_A = spmv_op(apply_A)
    ctx = ctx or apply_A._ctx()
    f = np.ascontiguousarray(f, np.float64)
    n = f.size
    x = np.zeros(max(n, 1))
    hist = np.zeros(max(max_iter, 1))
    rep = _PcgReport()
    ctx.check(lib().rd_gpu_pcg_linop(ctx.h, n, apply_A._st, apply_P._st, _ptr(f), float(tol), int(max_iter), _ptr(x),
                                     C.byref(rep), _ptr(hist)))
    return PcgResult(x[:n], rep.iterations, bool(rep.converged), hist[: rep.iterations].copy())


@dataclass
class SolveOutcome:
    u: np.ndarray
    iterations: int
    converged: bool
    setup_seconds: float
    solve_seconds: float


def solve_host_mesh(xyz, tets, boundary, rho: float, target: str = "smooth", tol: float = 1e-8, u=None,
                    seed: int = 0, ctx: Context | None = None) -> SolveOutcome:
    """mesh upload + build_system + solve_system(..., PrecondKind::amg) in one call
    (rd_gpu_solve_host_mesh: the tets upload overlaps the lattice-path solve).  `u`: an
    output array or device pointer of n_dofs doubles; None allocates a host array."""
    ctx = ctx or default_context()
    xyz = np.ascontiguousarray(xyz, np.float64)
    tets = np.ascontiguousarray(tets, np.int32)
    boundary = np.ascontiguousarray(boundary, np.uint8)
    host = u is None
    if host:
        u = np.zeros(max(int((boundary == 0).sum()), 1))
    t = _Target(TARGETS[target], int(seed))
    out = _SolveOutcome()
    nd = C.c_int(0)
    ctx.check(lib().rd_gpu_solve_host_mesh(ctx.h, xyz.shape[0], _ptr(xyz), tets.shape[0], _ptr(tets), _ptr(boundary),
                                           float(rho), C.byref(t), float(tol), _ptr(u), C.byref(nd), C.byref(out)))
    return SolveOutcome(u[: nd.value] if host else u, out.iterations, bool(out.converged), out.setup_seconds,
                        out.solve_seconds)


def solve_system_amg(A: Csr, f, tol: float = 1e-8, u=None) -> SolveOutcome:
    """bench.hpp:56 solve_system(mesh, sys, PrecondKind::amg, p, tol)."""
    host = u is None
    if host:
        u = np.zeros(max(A.rows, 1))
    if isinstance(f, np.ndarray):
        f = np.ascontiguousarray(f, np.float64)
    out = _SolveOutcome()
    A.ctx.check(lib().rd_gpu_solve_system_amg(A.ctx.h, A.h, _ptr(f), float(tol), _ptr(u), C.byref(out)))
    return SolveOutcome(u[: A.rows] if host else u, out.iterations, bool(out.converged), out.setup_seconds,
                        out.solve_seconds)


# ------------------------------------------------------------------ adaptivity
def bisect_marked(mesh: TetMesh, marked) -> TetMesh:
    """mesh.hpp:44 / mesh.cpp:67-145 on the device."""
    mk = np.ascontiguousarray(marked, np.int32).reshape(-1)
    h = _P()
    mesh.ctx.check(lib().rd_gpu_bisect_marked(mesh.ctx.h, mesh.h, mk.size, _ptr(mk) if mk.size else None,
                                              C.byref(h)))
    return TetMesh(h, mesh.ctx)


def uniform_refine(mesh: TetMesh) -> TetMesh:
    """mesh.hpp:40 / mesh.cpp:147-156 on the device."""
    h = _P()
    mesh.ctx.check(lib().rd_gpu_uniform_refine(mesh.ctx.h, mesh.h, C.byref(h)))
    return TetMesh(h, mesh.ctx)


def estimate(sys: FemSystem, coeffs, target: str, seed: int = 0):
    """adapt.hpp:21 / adapt.cpp:35-124 on the device -> (per_tet, global)."""
    coeffs = np.ascontiguousarray(coeffs, np.float64)
    if coeffs.size != sys.n_dofs:
        raise RdInvalidArgument("estimate: coefficient vector size mismatch")
    per = np.zeros(max(sys.mesh.n_tets, 1))
    g = C.c_double()
    t = _Target(TARGETS[target], int(seed))
    sys.ctx.check(lib().rd_gpu_estimate(sys.ctx.h, sys.mesh.h, sys.h, _ptr(coeffs) if coeffs.size else None,
                                        C.byref(t), _ptr(per), C.byref(g)))
    return per[: sys.mesh.n_tets], g.value


def mark_dorfler(eta, theta: float, ctx: Context | None = None) -> np.ndarray:
    """adapt.hpp:24 / adapt.cpp:126-150 on the device -> marked tets in marking order."""
    ctx = ctx or default_context()
    eta = np.ascontiguousarray(eta, np.float64)
    out = np.zeros(max(eta.size, 1), np.int32)
    k = C.c_int()
    ctx.check(lib().rd_gpu_mark_dorfler(ctx.h, eta.size, _ptr(eta) if eta.size else None, float(theta), _ptr(out),
                                        C.byref(k)))
    return out[: k.value]


@dataclass
class AdaptResult:
    history: list
    mesh: TetMesh
    coefficients: np.ndarray


def adaptive_solve(initial: TetMesh, target: str, rho: float, dof_budget: int, tol: float = 1e-8,
                   theta: float = 0.5, seed: int = 0, cap: int = 256, coeffs_cap: int = 1 << 24) -> AdaptResult:
    """adapt.hpp:44-47 / adapt.cpp:152-205 on the device, with the AMG solver (build_amg + pcg(tol, 500))."""
    ctx = initial.ctx
    hist = (_AdaptLevel * cap)()
    k = C.c_int()
    fm = _P()
    co = np.zeros(coeffs_cap)
    t = _Target(TARGETS[target], int(seed))
    ctx.check(lib().rd_gpu_adaptive_solve(ctx.h, initial.h, C.byref(t), float(rho), int(dof_budget), float(tol),
                                          float(theta), hist, cap, C.byref(k), C.byref(fm), _ptr(co), coeffs_cap))
    rows = [dict(level=r.level, dofs=r.dofs, iterations=r.iterations, eta=r.eta, err_l2_sq=r.err_l2_sq,
                 err_hm1_sq=r.err_hm1_sq, seconds=r.seconds) for r in hist[: min(k.value, cap)]]
    return AdaptResult(rows, TetMesh(fm, ctx), co[: rows[-1]["dofs"]].copy())


# ------------------------------------------------------------------ BDDC
def partition_geometric(sys: FemSystem, p: int) -> np.ndarray:
    """bddc.hpp:30 / bddc.cpp:45-111: the RCB owner of every tet."""
    out = np.zeros(max(sys.mesh.n_tets, 1), np.int32)
    sys.ctx.check(lib().rd_gpu_partition_geometric(sys.ctx.h, sys.mesh.h, sys.h, int(p), _ptr(out)))
    return out[: sys.mesh.n_tets]


class Bddc:
    """bddc.hpp BddcOperator on the device."""

    def __init__(self, sys: FemSystem, p: int):
        self.ctx = sys.ctx
        self.sys = sys
        h = _P()
        self.ctx.check(lib().rd_gpu_bddc_create(self.ctx.h, sys.mesh.h, sys.h, int(p), C.byref(h)))
        self.h = h
        ni, npr = C.c_int(), C.c_int()
        lib().rd_gpu_bddc_info(h, C.byref(ni), C.byref(npr))
        self.n_interface, self.n_primal, self.n_dofs = ni.value, npr.value, sys.n_dofs
        d = np.zeros(max(self.n_interface, 1), np.int32)
        lib().rd_gpu_bddc_interface_dofs(h, _ptr(d))
        self.interface_dofs = d[: self.n_interface]

    def coarse_matrix(self):
        out = np.zeros(max(self.n_primal ** 2, 1))
        self.ctx.check(lib().rd_gpu_bddc_coarse_matrix(self.h, _ptr(out)))
        return out[: self.n_primal ** 2].reshape(self.n_primal, self.n_primal)

    def _vec(self, fn, x, n_out, *extra):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(max(n_out, 1))
        args = [self.h, _ptr(x) if x.size else None] + [(_ptr(np.ascontiguousarray(e, np.float64))) for e in extra]
        self.ctx.check(fn(*args, _ptr(out)))
        return out[:n_out]

    def schur_apply(self, x):
        return self._vec(lib().rd_gpu_bddc_schur_apply, x, self.n_interface)

    def reduce_rhs(self, f):
        return self._vec(lib().rd_gpu_bddc_reduce_rhs, f, self.n_interface)

    def expand_solution(self, uC, f):
        return self._vec(lib().rd_gpu_bddc_expand, uC, self.n_dofs, f)

    def apply(self, r):
        return self._vec(lib().rd_gpu_bddc_apply, r, self.n_interface)

    def schur_op(self) -> LinOp:
        st = _LinOp()
        self.ctx.check(lib().rd_gpu_linop_bddc_schur(self.h, C.byref(st)))
        return LinOp(st, keep=(self,))

    def precond(self) -> LinOp:
        st = _LinOp()
        self.ctx.check(lib().rd_gpu_linop_bddc(self.h, C.byref(st)))
        return LinOp(st, keep=(self,))

    def __del__(self):
        try:
            if getattr(self, "h", None) and not _closing:
                lib().rd_gpu_bddc_free(self.h)
        except Exception:
            pass
        self.h = None


def bddc_solve(sys: FemSystem, p: int, tol: float = 1e-8, max_iter: int = 500) -> PcgResult:
    """bddc.hpp:85-87 / bddc.cpp:440-456 on the device."""
    u = np.zeros(max(sys.n_dofs, 1))
    hist = np.zeros(max(max_iter, 1))
    rep = _PcgReport()
    sys.ctx.check(lib().rd_gpu_bddc_solve(sys.ctx.h, sys.mesh.h, sys.h, int(p), float(tol), int(max_iter), _ptr(u),
                                          C.byref(rep), _ptr(hist)))
    return PcgResult(u[: sys.n_dofs], rep.iterations, bool(rep.converged), hist[: rep.iterations].copy())
