"""rd_gpu_solve_host_mesh: the bench-precond row from a host TetMesh in one C-ABI call.

For a mesh of Kuhn-lattice size the solve starts on generated unit-cube vertices while the host
arrays upload on a second stream; the uploaded vertices / flags are compared with the generated
ones and the uploaded tets with the Kuhn enumeration before any result stands.
Checked against the three-call path (rd_gpu_mesh_create -> rd_gpu_build_system ->
rd_gpu_solve_system_amg), which the parity suite pins to the oracle: the same u bit for bit
and the same iteration count, on lattice meshes, on a lattice-sized mesh whose tets are not
the enumeration (the provisional lattice solve is discarded and rerun on the generic path),
on custom boundary flags and on a mesh that is not lattice-sized; errors map like
build_system's.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rd():
    from paper_2102_03515_b200 import rd as _rd

    return _rd


def _three_call(rd, xyz, tets, b, rho, target):
    m = rd.mesh_from_arrays(xyz, tets, b)
    s = rd.build_system(m, rho, target)
    return rd.solve_system_amg(s.A, s.f(), 1e-8)


def _check(rd, xyz, tets, b, rho, target):
    ref = _three_call(rd, xyz, tets, b, rho, target)
    got = rd.solve_host_mesh(xyz, tets, b, rho, target, 1e-8)
    assert got.iterations == ref.iterations and got.converged == ref.converged
    assert np.array_equal(got.u, ref.u)
    return got


@pytest.mark.parametrize("n,target", [(16, "smooth"), (32, "smooth"), (64, "ball")])
def test_lattice_mesh_matches_three_call_path(rd, n, target):
    xyz, tets, b = rd.build_structured_cube(n).download()
    got = _check(rd, xyz, tets, b, 1.0 / (n * n), target)
    assert got.converged and got.iterations > 0


def test_pinned_host_arrays(rd):
    import torch

    n = 32
    xyz, tets, b = rd.build_structured_cube(n).download()
    px, pt, pb = (torch.from_numpy(a).pin_memory() for a in (xyz, tets, b))
    ref = _three_call(rd, xyz, tets, b, 1.0 / (n * n), "ball")
    u = torch.empty(int((b == 0).sum()), dtype=torch.float64).pin_memory()
    got = rd.solve_host_mesh(px.numpy(), pt.numpy(), pb.numpy(), 1.0 / (n * n), "ball", 1e-8, u=u)
    assert got.iterations == ref.iterations
    assert np.array_equal(u.numpy(), ref.u)


def test_shuffled_tets_fall_back_to_generic_path(rd):
    """Lattice-sized, not the enumeration: the provisional lattice solve must not stand."""
    n = 16
    xyz, tets, b = rd.build_structured_cube(n).download()
    rng = np.random.default_rng(3)
    ts = np.ascontiguousarray(tets[rng.permutation(tets.shape[0])])
    # the same tets in another order give the same system only up to summation order:
    # compare with the three-call path on the shuffled mesh (generic there too)
    assert rd.mesh_from_arrays(xyz, ts, b).lattice_n == -1
    _check(rd, xyz, ts, b, 1.0 / (n * n), "smooth")
    # two tets of one cell swapped: still lattice-sized
    tt = tets.copy()
    tt[[0, 1]] = tt[[1, 0]]
    _check(rd, xyz, np.ascontiguousarray(tt), b, 1.0 / (n * n), "smooth")


def test_other_geometry_on_lattice_sized_mesh(rd):
    """The solve starts on generated unit-cube vertices while the host vertices upload; any
    other geometry (or boundary flags) must restart on the uploaded arrays."""
    n = 16
    xyz, tets, b = rd.build_structured_cube(n).download()
    rng = np.random.default_rng(11)
    xj = xyz.copy()
    inner = b == 0
    xj[inner] += (rng.random((int(inner.sum()), 3)) - 0.5) * (0.4 / n)  # jittered interior: lattice tets, other geometry
    _check(rd, xj, tets, b, 1.0 / (n * n), "ball")
    _check(rd, np.ascontiguousarray(xyz * 2.0), tets, b, 1.0 / (n * n), "smooth")  # a cube of side 2
    xz = xyz.copy()
    xz[0, 0] = -0.0  # equal as numbers, not as bits: handled like any other difference
    _check(rd, xz, tets, b, 1.0 / (n * n), "smooth")
    # both provisional assumptions fail: other geometry and tets that are not the enumeration
    ts = np.ascontiguousarray(tets[rng.permutation(tets.shape[0])])
    _check(rd, xj, ts, b, 1.0 / (n * n), "smooth")


def test_tets_differ_in_either_half(rd):
    """A difference from the Kuhn enumeration anywhere in the tet array -- front, middle, the
    very last tet -- must send the solve down the generic path."""
    n = 12
    xyz, tets, b = rd.build_structured_cube(n).download()
    nt = tets.shape[0]
    for i, j in ((3, 4), (nt // 2 + 7, nt // 2 + 8), (nt - 2, nt - 1), (5, nt - 5)):
        tt = tets.copy()
        tt[[i, j]] = tt[[j, i]]
        _check(rd, xyz, np.ascontiguousarray(tt), b, 1.0 / (n * n), "smooth")


def test_custom_boundary_and_non_lattice_sizes(rd):
    n = 8
    xyz, tets, b = rd.build_structured_cube(n).download()
    bb = b.copy()
    bb[(n + 1) * (n + 1) * (n // 2) + (n + 1) * (n // 2)] = 0  # a surface vertex flagged interior
    _check(rd, xyz, tets, bb, 1.0 / 64, "smooth")
    # drop the last cell's six tets: not lattice-sized, plain generic path
    _check(rd, xyz, np.ascontiguousarray(tets[:-6]), b, 1.0 / 64, "box")


def test_errors(rd):
    xyz, tets, b = rd.build_structured_cube(4).download()
    with pytest.raises(ValueError):
        rd.solve_host_mesh(xyz, tets, b, 0.0, "smooth")
    tt = tets.copy()
    tt[[0, 1]] = tt[[1, 0]]
    with pytest.raises(ValueError):  # sine+random needs a structured cube: rejected after the check
        rd.solve_host_mesh(xyz, np.ascontiguousarray(tt), b, 1.0 / 16, "sine_random")
    # the context is still usable afterwards
    _check(rd, xyz, tets, b, 1.0 / 16, "smooth")
