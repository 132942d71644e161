"""Device parity: every sm_100a kernel called through the C-ABI against the CPU oracle.

Bars (BASELINE.json north star):
  * mesh, dof map, CSR patterns, C/F splittings, P, Galerkin operators: bit-exact;
  * fp64 values on integer/indicator paths (K, M, A, SpMV, GS sweeps, ball/box loads): bit-exact;
  * loads of sin targets: CUDA sin vs glibc sin -> <= 4 ulp (tolerance 1e-15 relative);
  * PCG: iteration counts equal, solutions within 1e-10 relative (dot products are
    reduced in a different -- deterministic -- order than Eigen's SSE2 dot).
"""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rd():
    from paper_2102_03515_b200 import rd as _rd

    _rd.default_context()
    return _rd


def assert_csr_equal(dev, ref, what=""):
    rp, ci, v = dev.download()
    assert dev.rows == ref.rows and dev.cols == ref.cols, what
    assert np.array_equal(rp, ref.rp), f"{what}: row_ptr"
    assert np.array_equal(ci, ref.ci), f"{what}: col_idx"
    assert np.array_equal(v, ref.v), f"{what}: values differ (max {np.abs(v - ref.v).max() if v.size else 0})"


def to_dev(rd, A):
    return rd.Csr.from_arrays(A.rows, A.cols, A.rp, A.ci, A.v)


# ------------------------------------------------------------------ mesh / assembly
@pytest.mark.parametrize("n", [1, 2, 4, 7, 8])
def test_mesh_bit_exact(rd, O, n):
    dm = rd.build_structured_cube(n)
    om = O.build_structured_cube(n)
    xyz, tets, b = dm.download()
    assert np.array_equal(xyz, om.xyz) and np.array_equal(tets, om.tets) and np.array_equal(b, om.boundary)


def test_mesh_rejects_nonpositive(rd):
    with pytest.raises(ValueError):
        rd.build_structured_cube(0)


@pytest.mark.parametrize("target", ["smooth", "ball", "box", "sine_random", "quadratic", "one", "zero", "nonzero_bc"])
@pytest.mark.parametrize("n", [3, 8])
def test_build_system_parity(rd, O, n, target):
    rho = 1.0 / (n * n)
    ds = rd.build_system(rd.build_structured_cube(n), rho, target)
    os_ = O.build_system(O.build_structured_cube(n), rho, target)
    assert_csr_equal(ds.K, os_.K, "K")
    assert_csr_equal(ds.M, os_.M, "M")
    assert_csr_equal(ds.A, os_.A, "A")
    v2d, d2v = ds.dofmap()
    assert np.array_equal(v2d, os_.vertex_to_dof) and np.array_equal(d2v, os_.dof_to_vertex)
    f = ds.f()
    if target in ("smooth", "sine_random", "nonzero_bc"):
        # CUDA sin vs glibc sin: ulp-level only
        assert np.abs(f - os_.f).max() <= 1e-15 * np.abs(os_.f).max() + 1e-300
    else:
        assert np.array_equal(f, os_.f), np.abs(f - os_.f).max()


def test_build_system_c2_pattern_n32(rd, O):
    ds = rd.build_system(rd.build_structured_cube(32), 2.0 ** -10, "ball")
    os_ = O.build_system(O.build_structured_cube(32), 2.0 ** -10, "ball")
    assert_csr_equal(ds.A, os_.A, "A")
    assert np.array_equal(ds.f(), os_.f)


def _sys_equal(ds, os_, exact_f=True):
    assert_csr_equal(ds.K, os_.K, "K")
    assert_csr_equal(ds.M, os_.M, "M")
    assert_csr_equal(ds.A, os_.A, "A")
    f = ds.f()
    if exact_f:
        assert np.array_equal(f, os_.f), np.abs(f - os_.f).max()
    else:
        assert np.abs(f - os_.f).max() <= 1e-15 * np.abs(os_.f).max() + 1e-300


@pytest.mark.parametrize("target", ["ball", "smooth"])
def test_uploaded_mesh_lattice_and_generic_paths(rd, O, target):
    """The Kuhn-lattice assembly (adjacency by formula) and the generic one
    (vertex->tet CSR, searched pattern) against the oracle on the same arrays."""
    n, rho = 8, 1.0 / 64
    exact = target == "ball"
    xyz, tets, b = rd.build_structured_cube(n).download()
    # (a) the cube as host arrays: detected as a lattice
    dm = rd.mesh_from_arrays(xyz, tets, b)
    assert dm.lattice_n == n
    _sys_equal(rd.build_system(dm, rho, target), O.build_system(O.mesh_from_arrays(xyz, tets, b), rho, target), exact)
    # (b) jittered interior coordinates: still a lattice, non-uniform geometry
    rng = np.random.default_rng(5)
    xj = xyz.copy()
    xj[b == 0] += rng.uniform(-0.2, 0.2, size=(int((b == 0).sum()), 3)) / n
    dm = rd.mesh_from_arrays(xj, tets, b)
    assert dm.lattice_n == n
    _sys_equal(rd.build_system(dm, rho, target), O.build_system(O.mesh_from_arrays(xj, tets, b), rho, target), exact)
    # (c) shuffled tet order: not the enumeration -> generic path
    perm = rng.permutation(tets.shape[0])
    ts = np.ascontiguousarray(tets[perm])
    dm = rd.mesh_from_arrays(xyz, ts, b)
    assert dm.lattice_n == -1
    _sys_equal(rd.build_system(dm, rho, target), O.build_system(O.mesh_from_arrays(xyz, ts, b), rho, target), exact)
    # (d) a surface vertex flagged interior: lattice mesh, generic fallback
    bb = b.copy()
    bb[(n + 1) * (n + 1) * (n // 2) + (n + 1) * (n // 2)] = 0  # x = 0 face, centre
    dm = rd.mesh_from_arrays(xyz, tets, bb)
    assert dm.lattice_n == n
    _sys_equal(rd.build_system(dm, rho, target), O.build_system(O.mesh_from_arrays(xyz, tets, bb), rho, target), exact)


@pytest.mark.parametrize("n", [30, 32])
def test_indicator_support_culling(rd, O, n):
    """Box and ball loads skip the quadrature loop on tets strictly inside or
    outside the support; the box faces lie on lattice planes when 4 | n."""
    for target in ("box", "ball"):
        ds = rd.build_system(rd.build_structured_cube(n), 1.0 / (n * n), target)
        os_ = O.build_system(O.build_structured_cube(n), 1.0 / (n * n), target)
        assert np.array_equal(ds.f(), os_.f), target


def test_build_system_rejects_rho(rd):
    with pytest.raises(ValueError):
        rd.build_system(rd.build_structured_cube(2), 0.0, "smooth")


def test_reference_tet_assembly(rd, O):  # test_assembly.cpp:41-62 on a hand-built mesh
    xyz = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [2, 2, 2]]
    tets = [[0, 1, 2, 3]]
    bnd = [0, 0, 0, 0, 1]
    ds = rd.build_system(rd.mesh_from_arrays(xyz, tets, bnd), 1.0, "one")
    K = ds.K.dense()
    assert K[0, 0] == pytest.approx(0.5, rel=1e-14) and K[1, 1] == pytest.approx(1 / 6, rel=1e-14)
    M = ds.M.dense()
    assert M[0, 0] == pytest.approx(1 / 60, rel=1e-14) and M[0, 1] == pytest.approx(1 / 120, rel=1e-14)


# ------------------------------------------------------------------ SpMV
@pytest.mark.parametrize("n", [4, 16, 33])
def test_spmv_bit_exact(rd, O, n):
    os_ = O.build_system(O.build_structured_cube(n), 1e-3, "smooth")
    A = to_dev(rd, os_.A)
    x = O.pseudo_random_vec(A.rows, 7)
    assert np.array_equal(rd.spmv(A, x), O.spmv(os_.A, x))


def test_spmv_hand_cases(rd, O):  # test_linalg.cpp:47-71
    I3 = rd.from_triplets(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0)])
    x = np.array([3.0, -1.0, 2.0])
    assert np.array_equal(rd.spmv(I3, x), x)
    A = rd.from_triplets(2, 2, [(0, 0, 2.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 2.0)])
    assert list(rd.spmv(A, np.ones(2))) == [3.0, 3.0]
    with pytest.raises(ValueError):
        rd.spmv(A, np.ones(5))


def test_spmv_irregular_rows(rd, O):  # rows longer than one staging chunk
    rng = np.random.default_rng(0)
    n = 300
    trips = []
    for i in range(n):
        k = 1 + (i * 37) % 700 if i % 50 == 0 else 1 + i % 9
        cols = rng.choice(n, size=min(k, n), replace=False)
        trips += [(i, int(c), float(rng.standard_normal())) for c in cols]
    Ao = O.from_triplets(n, n, trips)
    A = to_dev(rd, Ao)
    x = rng.standard_normal(n)
    assert np.array_equal(rd.spmv(A, x), O.spmv(Ao, x))


# ------------------------------------------------------------------ coarsening / Galerkin
def test_coarsen_hand_cases(rd):  # test_amg.cpp:36-60
    t = []
    for i in range(5):
        t.append((i, i, 2.0))
        if i + 1 < 5:
            t += [(i, i + 1, -1.0), (i + 1, i, -1.0)]
    flags, P = rd.coarsen_redblack(rd.from_triplets(5, 5, t))
    assert list(flags) == [1, 0, 1, 0, 1]
    D = P.dense()
    assert D[1, 0] == 0.5 and D[1, 1] == 0.5 and D[4, 2] == 1.0
    flags, P = rd.coarsen_redblack(rd.from_triplets(3, 3, [(0, 0, 1.0), (1, 1, 2.0), (2, 2, 3.0)]))
    assert list(flags) == [1, 1, 1] and np.array_equal(P.dense(), np.eye(3))


@pytest.mark.parametrize("n", [4, 8, 16])
def test_coarsen_galerkin_bit_exact(rd, O, n):
    os_ = O.build_system(O.build_structured_cube(n), 1e-2, "smooth")
    A = to_dev(rd, os_.A)
    flags, P = rd.coarsen_redblack(A)
    oflags, oP = O.coarsen_redblack(os_.A)
    assert np.array_equal(flags, oflags)
    assert_csr_equal(P, oP, "P")
    assert_csr_equal(rd.galerkin_coarse(A, P), O.galerkin_coarse(os_.A, oP), "Ac")


def test_galerkin_hand_case(rd):  # test_amg.cpp:83-99
    A = rd.from_triplets(2, 2, [(0, 0, 2.0), (0, 1, -1.0), (1, 0, -1.0), (1, 1, 2.0)])
    P = rd.from_triplets(2, 1, [(0, 0, 1.0), (1, 0, 0.5)])
    assert rd.galerkin_coarse(A, P).dense()[0, 0] == pytest.approx(1.5, rel=1e-14)


def test_coarsen_nonsymmetric_pattern(rd, O):
    rng = np.random.default_rng(3)
    n = 60
    trips = [(i, i, 4.0) for i in range(n)]
    for _ in range(150):
        i, j = rng.integers(0, n, 2)
        if i != j:
            trips.append((int(i), int(j), -0.1))
    Ao = O.from_triplets(n, n, trips)
    flags, P = rd.coarsen_redblack(to_dev(rd, Ao))
    of, oP = O.coarsen_redblack(Ao)
    assert np.array_equal(flags, of)
    assert_csr_equal(P, oP, "P")


# ------------------------------------------------------------------ Gauss-Seidel
def test_sgs_hand_cases(rd):  # test_amg.cpp:109-126
    A = rd.from_triplets(2, 2, [(0, 0, 2.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 2.0)])
    u = rd.sgs_sweep(A, np.ones(2), np.zeros(2))
    assert u[0] == pytest.approx(0.375, rel=1e-15) and u[1] == pytest.approx(0.25, rel=1e-15)
    D = rd.from_triplets(2, 2, [(0, 0, 2.0), (1, 1, 4.0)])
    u = rd.sgs_sweep(D, np.array([2.0, 2.0]), np.zeros(2))
    assert u[0] == 1.0 and u[1] == 0.5


def test_sgs_zero_diagonal_raises(rd):  # amg.cpp:82
    A = rd.from_triplets(2, 2, [(0, 1, 1.0), (1, 0, 1.0), (1, 1, 2.0)])
    with pytest.raises(rd.RdZeroDiagonalError):
        rd.sgs_sweep(A, np.ones(2), np.zeros(2))


@pytest.mark.parametrize("n", [3, 8, 17, 32])
def test_sgs_bit_exact(rd, O, n):
    os_ = O.build_system(O.build_structured_cube(n), 2.0 ** -8, "smooth")
    A = to_dev(rd, os_.A)
    f = O.pseudo_random_vec(A.rows, 1)
    u = O.pseudo_random_vec(A.rows, 2)
    assert np.array_equal(rd.sgs_sweep(A, f, u), O.sgs_sweep(os_.A, f, u))


@pytest.mark.parametrize("n,target", [(65, "smooth"), (128, "ball")])
def test_sgs_bit_exact_large(rd, O, n, target):
    """The structured lattice kernel at the BASELINE sizes (many tiles, halo traffic)."""
    O.set_num_threads(8)
    ds = rd.build_system(rd.build_structured_cube(n), 1.0 / (n * n), target)
    A = ds.A
    rp, ci, v = A.download()
    Ao = O.Csr(A.rows, A.cols, rp, ci, v)
    f = O.pseudo_random_vec(A.rows, 3)
    u = O.pseudo_random_vec(A.rows, 4)
    assert np.array_equal(rd.sgs_sweep(A, f, u), O.sgs_sweep(Ao, f, u))


@pytest.mark.parametrize("scale", [1e-300, 1e300])
def test_sgs_speculation_fallback(rd, O, scale):
    """Row sums far outside the division fast path (|s| < 2^-969, or quotients
    near overflow) make the speculative lattice sweep flag itself; the call is
    rerun with exact sweeps and must still match the reference bit for bit."""
    n = 16
    os_ = O.build_system(O.build_structured_cube(n), 1.0 / (n * n), "smooth")
    A = to_dev(rd, os_.A)
    f = O.pseudo_random_vec(A.rows, 21) * scale
    u = np.zeros(A.rows)
    assert np.array_equal(rd.sgs_sweep(A, f, u), O.sgs_sweep(os_.A, f, u))
    h = rd.build_amg(A, 64)
    oh = O.build_amg(os_.A, 64)
    assert np.array_equal(h.apply(f), oh.apply(f))


def test_structured_levels_detected(rd, O):
    os_ = O.build_system(O.build_structured_cube(32), 2.0 ** -10, "smooth")
    h = rd.build_amg(to_dev(rd, os_.A))
    assert [h.structured(l) for l in range(h.num_levels - 1)] == [True] * (h.num_levels - 1)


def test_sgs_random_sparse_bit_exact(rd, O):
    rng = np.random.default_rng(5)
    n = 500
    trips = [(i, i, 10.0 + rng.random()) for i in range(n)]
    for _ in range(3000):
        i, j = rng.integers(0, n, 2)
        if i != j:
            trips.append((int(i), int(j), float(rng.standard_normal())))
    Ao = O.from_triplets(n, n, trips)
    f, u = rng.standard_normal(n), rng.standard_normal(n)
    assert np.array_equal(rd.sgs_sweep(to_dev(rd, Ao), f, u), O.sgs_sweep(Ao, f, u))


# ------------------------------------------------------------------ hierarchy / V-cycle
@pytest.mark.parametrize("n,thr", [(4, 16), (6, 8), (16, 64), (32, 64)])
def test_hierarchy_bit_exact(rd, O, n, thr):
    os_ = O.build_system(O.build_structured_cube(n), 1.0 / (n * n), "ball")
    oh = O.build_amg(os_.A, thr)
    dh = rd.build_amg(to_dev(rd, os_.A), thr)
    assert dh.num_levels == oh.num_levels
    for l in range(oh.num_levels):
        assert_csr_equal(dh.level(l), oh.level(l), f"A_{l}")
        if l + 1 < oh.num_levels:
            assert np.array_equal(dh.flags(l), oh.flags(l))
            assert_csr_equal(dh.level(l, "P"), oh.level(l, "P"), f"P_{l}")
            assert_csr_equal(dh.level(l, "Pt"), oh.level(l, "Pt"), f"Pt_{l}")


@pytest.mark.parametrize("n,jitter,thr", [(16, 0.0, 64), (16, 0.2, 64), (24, 0.2, 64), (13, 0.0, 64), (64, 0.0, 64),
                                          (10, 0.1, 1), (5, 0.0, 1), (3, 0.0, 4), (12, 0.0, 8)])
def test_hierarchy_lattice_levels(rd, O, n, jitter, thr):
    """Lattice levels take the closed-form C/F split, P, P^T and the fused Galerkin
    product; non-uniform geometry (jitter), odd and even level sides (high-face F
    points with a single C neighbour) and hierarchies down to one coarse point."""
    xyz, tets, b = O.build_structured_cube(n).xyz, O.build_structured_cube(n).tets, O.build_structured_cube(n).boundary
    if jitter:
        rng = np.random.default_rng(11)
        xyz = xyz.copy()
        xyz[b == 0] += rng.uniform(-jitter, jitter, size=(int((b == 0).sum()), 3)) / n
    os_ = O.build_system(O.mesh_from_arrays(xyz, tets, b), 1.0 / (n * n), "ball")
    oh = O.build_amg(os_.A, thr)
    dh = rd.build_amg(to_dev(rd, os_.A), thr)
    assert dh.num_levels == oh.num_levels
    for l in range(oh.num_levels):
        assert_csr_equal(dh.level(l), oh.level(l), f"A_{l}")
        if l + 1 < oh.num_levels:
            assert np.array_equal(dh.flags(l), oh.flags(l))
            assert_csr_equal(dh.level(l, "P"), oh.level(l, "P"), f"P_{l}")
            assert_csr_equal(dh.level(l, "Pt"), oh.level(l, "Pt"), f"Pt_{l}")
    r = O.pseudo_random_vec(os_.A.rows, 3)
    assert np.array_equal(dh.apply(r), oh.apply(r))


@pytest.mark.parametrize("n,rho", [(9, 1.0), (16, 2.0 ** -8), (33, 1e-6)])
def test_hierarchy_from_device_assembly(rd, O, n, rho):
    """A from the lattice assembly carries its lattice facts (no detection pass);
    the hierarchy built on it is the oracle's, level by level."""
    ds = rd.build_system(rd.build_structured_cube(n), rho, "ball")
    os_ = O.build_system(O.build_structured_cube(n), rho, "ball")
    oh = O.build_amg(os_.A, 64)
    dh = rd.build_amg(ds.A, 64)
    assert dh.num_levels == oh.num_levels
    for l in range(oh.num_levels):
        assert_csr_equal(dh.level(l), oh.level(l), f"A_{l}")
        if l + 1 < oh.num_levels:
            assert_csr_equal(dh.level(l, "P"), oh.level(l, "P"), f"P_{l}")
            assert_csr_equal(dh.level(l, "Pt"), oh.level(l, "Pt"), f"Pt_{l}")
            assert dh.structured(l)


@pytest.mark.parametrize("variant", ["random_zeros", "cancelled_coarse_entry"])
def test_hierarchy_lattice_explicit_zeros(rd, O, variant):
    """Explicit zero values on a lattice pattern: the fine level stays a lattice
    (the split is pattern based) and the Galerkin product prunes exact zeros.  In
    the second variant (identity plus one coupling -1/2 between fine points 2I and
    2I + e_x) the coarse entry (I, I + e_x) cancels to exactly zero, so level 1
    loses the 15-point pattern and continues on the generic path."""
    os_ = O.build_system(O.build_structured_cube(17), 2.0 ** -8, "ball")
    A = os_.A
    L = 16
    rows = np.repeat(np.arange(A.rows), np.diff(A.rp))
    if variant == "random_zeros":
        v = A.v.copy()
        rng = np.random.default_rng(4)
        v[(rows != A.ci) & (rng.random(v.size) < 0.3)] = 0.0
    else:
        v = np.where(rows == A.ci, 1.0, 0.0)
        a = (4 * L + 4) * L + 4
        for i, j in ((a, a + 1), (a + 1, a)):
            k = A.rp[i] + int(np.searchsorted(A.ci[A.rp[i]:A.rp[i + 1]], j))
            assert A.ci[k] == j
            v[k] = -0.5
    Az = O.Csr(A.rows, A.cols, A.rp, A.ci, v)
    oh = O.build_amg(Az, 8)
    dh = rd.build_amg(to_dev(rd, Az), 8)
    assert dh.num_levels == oh.num_levels
    for l in range(oh.num_levels):
        assert_csr_equal(dh.level(l), oh.level(l), f"A_{l}")
        if l + 1 < oh.num_levels:
            assert np.array_equal(dh.flags(l), oh.flags(l))
            assert_csr_equal(dh.level(l, "P"), oh.level(l, "P"), f"P_{l}")
            assert_csr_equal(dh.level(l, "Pt"), oh.level(l, "Pt"), f"Pt_{l}")
    assert dh.structured(0)
    assert dh.structured(1) == (variant == "random_zeros")
    r = O.pseudo_random_vec(A.rows, 5)
    assert np.array_equal(dh.apply(r), oh.apply(r))


@pytest.mark.parametrize("n,thr", [(3, 1000), (4, 16), (16, 64), (32, 64)])
def test_amg_apply_bit_exact(rd, O, n, thr):
    os_ = O.build_system(O.build_structured_cube(n), 1e-4, "smooth")
    oh = O.build_amg(os_.A, thr)
    dh = rd.build_amg(to_dev(rd, os_.A), thr)
    r = O.pseudo_random_vec(os_.A.rows, 9)
    assert np.array_equal(dh.apply(r), oh.apply(r))


def test_vcycle_symmetric_positive(rd, O):  # test_amg.cpp:139-151
    os_ = O.build_system(O.build_structured_cube(4), 1e-2, "smooth")
    h = rd.build_amg(to_dev(rd, os_.A), 16)
    for s in range(3):
        r1, r2 = O.pseudo_random_vec(os_.A.rows, 10 + s), O.pseudo_random_vec(os_.A.rows, 20 + s)
        assert r2 @ h.apply(r1) == pytest.approx(r1 @ h.apply(r2), rel=1e-11)


def test_empty_hierarchy(rd):  # test_amg.cpp:204-210
    A = rd.Csr.from_arrays(0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0))
    h = rd.build_amg(A)
    assert h.num_levels == 1


# ------------------------------------------------------------------ PCG / solve_system
def test_pcg_hand_cases(rd, O):  # test_linalg.cpp:96-139
    A1 = rd.from_triplets(1, 1, [(0, 0, 2.0)])
    r = rd.pcg(A1, "identity", np.array([4.0]), 1e-12, 10)
    assert r.converged and r.iterations == 1 and r.x[0] == pytest.approx(2.0, rel=1e-14)
    t = []
    for i in range(40):
        t.append((i, i, 4.0 + 0.01 * i))
        if i + 1 < 40:
            t += [(i, i + 1, -1.0), (i + 1, i, -1.0)]
        if i + 3 < 40:
            t += [(i, i + 3, -0.5), (i + 3, i, -0.5)]
    B = rd.from_triplets(40, 40, t)
    r = rd.pcg(B, "identity", np.ones(40), 1e-14, 2)
    assert not r.converged and r.iterations == 2
    r = rd.pcg(B, "identity", np.zeros(40), 1e-10, 10)
    assert r.converged and r.iterations == 0 and np.linalg.norm(r.x) == 0.0
    with pytest.raises(rd.RdNotSpdError):
        rd.pcg(rd.from_triplets(2, 2, [(0, 0, 1.0), (1, 1, -1.0)]), "identity", np.ones(2), 1e-10, 10)


@pytest.mark.parametrize("max_iter", [0, -3])
@pytest.mark.parametrize("precond", ["identity", "amg"])
def test_pcg_max_iter_nonpositive(rd, O, max_iter, precond):  # linalg.cpp:66,77: the loop never runs
    ds = rd.build_system(rd.build_structured_cube(8), 1.0, "smooth")
    os_ = O.build_system(O.build_structured_cube(8), 1.0, "smooth")
    r = rd.pcg(ds.A, precond, ds.f(), 1e-8, max_iter)
    ref = O.pcg(os_.A, precond, os_.f, 1e-8, max_iter)
    assert r.iterations == ref.iterations == 0 and not r.converged and not ref.converged
    assert np.all(r.x == 0.0) and np.all(ref.x == 0.0)


@pytest.mark.parametrize("n,rho,target", [(8, 1.0, "smooth"), (8, 1e-12, "smooth"), (16, 2.0 ** -8, "ball"),
                                          (32, 2.0 ** -10, "smooth"), (32, 1e-2, "sine_random"),
                                          (32, 2.0 ** -10, "box")])
def test_solve_system_parity(rd, O, n, rho, target):
    ds = rd.build_system(rd.build_structured_cube(n), rho, target)
    os_ = O.build_system(O.build_structured_cube(n), rho, target)
    out = rd.solve_system_amg(ds.A, ds.f(), 1e-8)
    ref = O.solve_system_amg(os_, 1e-8)
    assert out.converged and ref.converged
    assert out.iterations == ref.iterations
    assert np.abs(out.u - ref.u).max() <= 1e-10 * np.abs(ref.u).max()


@pytest.mark.parametrize("n,rho", [(8, 1.0), (16, 2.0 ** -8), (32, 2.0 ** -10)])
def test_error_norms_manufactured(rd, O, n, rho):
    """assembly.cpp:265-310 on the device: the converged solution of the smooth target
    against rd::manufactured_exact(rho).  CUDA sin/cos vs glibc and a different order of
    the final sum over tets: agreement to 1e-12 relative."""
    om = O.build_structured_cube(n)
    os_ = O.build_system(om, rho, "smooth")
    ref = O.solve_system_amg(os_, 1e-10)
    l2o = O.l2_error_manufactured(om, os_, ref.u, rho)
    h1o = O.h1_semi_error_manufactured(om, os_, ref.u, rho)
    ds = rd.build_system(rd.build_structured_cube(n), rho, "smooth")
    l2, h1 = rd.error_norms(ds, ref.u, rho)
    assert abs(l2 - l2o) <= 1e-12 * l2o and abs(h1 - h1o) <= 1e-12 * h1o
    # zero field: the norms of the exact solution itself
    l2z, h1z = rd.error_norms(ds, np.zeros(ds.n_dofs), rho)
    assert abs(l2z - O.l2_error_manufactured(om, os_, np.zeros(ds.n_dofs), rho)) <= 1e-12 * l2z
    assert abs(h1z - O.h1_semi_error_manufactured(om, os_, np.zeros(ds.n_dofs), rho)) <= 1e-12 * h1z
    with pytest.raises(ValueError):
        rd.error_norms(ds, ref.u, -1.0)


@pytest.mark.parametrize("rho", [1.0, 1e-2, 1e-4, 1e-6, 2.0 ** -12])
def test_c3_rho_sweep_n64(rd, O, rho):  # BASELINE config 3 at full size
    O.set_num_threads(8)
    ds = rd.build_system(rd.build_structured_cube(64), rho, "sine_random")
    os_ = O.build_system(O.build_structured_cube(64), rho, "sine_random")
    assert_csr_equal(ds.A, os_.A, "A")
    out = rd.solve_system_amg(ds.A, ds.f(), 1e-8)
    ref = O.solve_system_amg(os_, 1e-8)
    assert abs(out.iterations - ref.iterations) <= 0, (out.iterations, ref.iterations)
    assert np.abs(out.u - ref.u).max() <= 1e-10 * np.abs(ref.u).max()


def test_pcg_history_matches(rd, O):
    os_ = O.build_system(O.build_structured_cube(16), 1e-3, "smooth")
    A = to_dev(rd, os_.A)
    r = rd.pcg(A, "amg", os_.f, 1e-10, 100)
    ro = O.pcg(os_.A, "amg", os_.f, 1e-10, 100)
    assert r.iterations == ro.iterations
    assert np.allclose(r.residual_history, ro.residual_history, rtol=1e-9, atol=0)


def test_degenerate_meshes(rd):  # test_bench.cpp:185-195: n=1 has no dofs
    ds = rd.build_system(rd.build_structured_cube(1), 1.0, "smooth")
    assert ds.n_dofs == 0
    out = rd.solve_system_amg(ds.A, np.zeros(0), 1e-8)
    assert out.converged and out.iterations == 0
    ds = rd.build_system(rd.build_structured_cube(2), 1.0, "smooth")
    assert ds.n_dofs == 1
    out = rd.solve_system_amg(ds.A, ds.f(), 1e-8)
    assert out.converged


def test_c2_full_solve(rd, O):  # BASELINE config 2 at full size: n=128, rho=h^2, ball target
    """The bench workload end to end against the oracle: A bit for bit, iteration count equal,
    solution within 1e-10 relative, every smoothed level on a structured kernel."""
    O.set_num_threads(8)
    n, rho = 128, 2.0 ** -14
    ds = rd.build_system(rd.build_structured_cube(n), rho, "ball")
    os_ = O.build_system(O.build_structured_cube(n), rho, "ball")
    assert_csr_equal(ds.A, os_.A, "A")
    assert np.array_equal(ds.f(), os_.f)
    out = rd.solve_system_amg(ds.A, ds.f(), 1e-8)
    ref = O.solve_system_amg(os_, 1e-8)
    assert out.converged and ref.converged and out.iterations == ref.iterations == 5
    assert np.abs(out.u - ref.u).max() <= 1e-10 * np.abs(ref.u).max()
    h = rd.build_amg(ds.A)
    assert [h.stencil_source(l) for l in range(h.num_levels - 1)][:2] == ["uniform", "class"]


@pytest.mark.parametrize("n,rho,target", [(16, 2.0 ** -8, "ball"), (16, 1e-2, "sine_random"), (16, 2.0 ** -8, "smooth"),
                                          (12, 1.0, "box"), (8, 1.0, "quadratic")])
def test_l2_error_target_squared(rd, O, n, rho, target):
    """assembly.cpp:312-331 on the device (the BASELINE error gate ||u - u_bar||_L2 for every
    target) against the oracle on the oracle's converged solution: 1e-12 relative."""
    om = O.build_structured_cube(n)
    os_ = O.build_system(om, rho, target)
    ref = O.solve_system_amg(os_, 1e-10)
    want = O.l2_error_target_squared(om, os_, ref.u, target, n)
    ds = rd.build_system(rd.build_structured_cube(n), rho, target)
    got = rd.l2_error_target_squared(ds, ref.u, target)
    assert abs(got - want) <= 1e-12 * want, (got, want)
    z = np.zeros(ds.n_dofs)
    assert abs(rd.l2_error_target_squared(ds, z, target) - O.l2_error_target_squared(om, os_, z, target, n)) <= \
        1e-12 * O.l2_error_target_squared(om, os_, z, target, n)


@pytest.mark.parametrize("n,rho,target", [(4, 1.0, "box"), (8, 1e-2, "smooth"), (8, 1.0, "ball"),
                                          (13, 1e-3, "ball"), (16, 2.0 ** -8, "ball"), (16, 1e-4, "sine_random")])
def test_target_dual_norm(rd, O, n, rho, target):
    """bench.cpp:55-63 on the device: dense LLT of K for n_dofs <= 2000 (n=4: the one-CTA
    shared-memory factorization; n=8, 13: the cooperative whole-GPU one -- both the oracle's
    operation order, agreement to rounding in the final dot), AMG(K)-PCG to 1e-11 above (n=16:
    the generic, non-lattice K hierarchy)."""
    om = O.build_structured_cube(n)
    os_ = O.build_system(om, rho, target)
    u = O.solve_system_amg(os_, 1e-10).u
    want = O.target_dual_norm(os_, u)
    ds = rd.build_system(rd.build_structured_cube(n), rho, target)
    got = rd.target_dual_norm(ds, u)
    tol = 1e-12 if (n - 1) ** 3 <= 2000 else 1e-8
    assert abs(got - want) <= tol * want, (got, want)


@pytest.mark.parametrize("target", ["smooth", "sine_random", "ball", "box", "quadratic", "nonzero_bc"])
@pytest.mark.parametrize("n", [8, 13])
def test_error_norms_target_parity(rd, O, n, target):
    """assembly.cpp:265-310 with the target field as the exact function (value and gradient,
    oracle Target::grad) on the device against the oracle, for the solution and for a
    pseudo-random field; CUDA sin/cos vs glibc -> 1e-12 relative."""
    rho = 1e-2
    om = O.build_structured_cube(n)
    os_ = O.build_system(om, rho, target)
    u = O.solve_system_amg(os_, 1e-8).u
    ds = rd.build_system(rd.build_structured_cube(n), rho, target)
    for coeffs in (u, O.pseudo_random_vec(os_.n_dofs, 11)):
        want = O.error_norms_target(om, os_, coeffs, target, n, 0)
        got = rd.error_norms_target(ds, coeffs, target)
        for g, w in zip(got, want):
            assert abs(g - w) <= 1e-12 * max(w, 1e-300), (target, got, want)


def _goldens():
    import json as _json
    return _json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                        "baseline_configs.json")))["cases"]


@pytest.mark.parametrize("case", _goldens(), ids=lambda c: c["name"])
def test_baseline_config_goldens(rd, case):
    """BASELINE configs C1, C2 and the C3 rho sweep against the committed oracle goldens
    (tools/make_goldens.py): iteration count equal, residual history / solution / error gates
    within the north star's 1e-10."""
    n, rho, target = case["n"], case["rho"], case["target"]
    ds = rd.build_system(rd.build_structured_cube(n), rho, target)
    out = rd.pcg(ds.A, "amg", ds.f(), 1e-8, 500)
    assert out.converged and out.iterations == case["iterations"]
    assert np.allclose(out.residual_history, case["residual_history"], rtol=1e-9, atol=0)
    u = out.x
    assert abs(np.linalg.norm(u) - case["u_norm2"]) <= 1e-10 * case["u_norm2"]
    for i, v in case["u_samples"].items():
        assert abs(u[int(i)] - v) <= 1e-10 * np.abs(u).max()
    l2 = math.sqrt(rd.l2_error_target_squared(ds, u, target))
    assert abs(l2 - case["l2_u_minus_target"]) <= 1e-10 * case["l2_u_minus_target"]
    # the gates with the target as the exact function: ||u - u_bar|| (degree 5), ||grad(u - u_bar)||
    l2d5, h1 = rd.error_norms_target(ds, u, target)
    assert abs(l2d5 - case["l2_deg5_u_minus_target"]) <= 1e-10 * case["l2_deg5_u_minus_target"]
    assert abs(h1 - case["h1_u_minus_target"]) <= 1e-10 * case["h1_u_minus_target"]
    if target == "smooth":  # the same gate through manufactured_exact(0)
        _, h1m = rd.error_norms(ds, u, 0.0)
        assert h1m == h1


@pytest.mark.parametrize("n,target", [(256, "smooth"), (512, "ball")])
def test_full_size_properties(rd, n, target):
    """C4 (n=256) and C5 (n=512, 133M dofs) on one B200, where the oracle cannot follow:
    size-independent properties -- convergence to rtol 1e-8 in the C2-like iteration count, a
    true residual ||f - A u|| consistent with it, every smoothed level structured, and for the
    smooth target the O(h^2) error decay against the C1 golden."""
    rho = 1.0 / n ** 2
    mesh = rd.build_structured_cube(n)
    ds = rd.build_system(mesh, rho, target)
    import torch
    u = torch.empty(ds.n_dofs, dtype=torch.float64, device="cuda")
    out = rd.solve_system_amg(ds.A, ds.f_ptr, 1e-8, u=u)
    assert out.converged and 2 <= out.iterations <= 8
    f = torch.empty_like(u)
    rd.lib().rd_gpu_copy(ds.ctx.h, rd._ptr(f), rd.C.c_void_p(ds.f_ptr), 8 * ds.n_dofs)
    Au = torch.empty_like(u)
    ds.ctx.check(rd.lib().rd_gpu_spmv(ds.ctx.h, ds.A.h, rd._ptr(u), rd._ptr(Au)))
    ds.ctx.synchronize()
    rel = float(torch.linalg.norm(f - Au) / torch.linalg.norm(f))
    assert rel < 1e-6, rel
    l2 = math.sqrt(rd.l2_error_target_squared(ds, u, target))
    if target == "smooth":
        c1 = next(c for c in _goldens() if c["name"] == "C1")
        ratio = c1["l2_u_minus_target"] / l2
        assert 30 < ratio < 130, ratio  # h: 1/32 -> 1/256, rho = h^2 coupled: ~(h1/h2)^2 = 64
    else:
        assert 0.0 < l2 < 0.1


@pytest.mark.parametrize("n,thr,m", [(16, 64, 2), (32, 64, 3), (32, 512, 2), (33, 64, 2), (64, 64, 0)])
def test_amg_apply_smoothing_steps(rd, O, n, thr, m):
    """build_amg(A, threshold, m) with m != 1 (amg.cpp:90-132: m symmetric sweeps before and
    after the coarse correction; m = 0 skips smoothing): the structured levels, the one-CTA
    coarse tail and the generic path (n = 33: side 32 levels) against the oracle, bit for bit."""
    os_ = O.build_system(O.build_structured_cube(n), 1.0 / n ** 2, "ball")
    oh = O.build_amg(os_.A, thr, m)
    ds = rd.build_system(rd.build_structured_cube(n), 1.0 / n ** 2, "ball")
    dh = rd.build_amg(ds.A, thr, m)
    r = O.pseudo_random_vec(os_.A.rows, 5)
    assert np.array_equal(dh.apply(r), oh.apply(r))


@pytest.mark.parametrize("n", [64, 129])
def test_repeated_solves_bit_identical(rd, n):
    """The solve loop's kernels overlap (programmatic dependent launch: a kernel's blocks are
    scheduled while its predecessor drains) and the sweep's tiles hand values on through memory:
    any race there would make runs differ.  Ten full build + setup + solve runs, bit for bit."""
    mesh = rd.build_structured_cube(n)
    ref = None
    for k in range(10):
        s = rd.build_system(mesh, 1.0 / n ** 2, "ball")
        out = rd.solve_system_amg(s.A, s.f(), 1e-8)
        if ref is None:
            ref = (out.u.copy(), out.iterations)
        else:
            assert out.iterations == ref[1]
            assert np.array_equal(out.u, ref[0]), f"run {k} differs from run 0"
