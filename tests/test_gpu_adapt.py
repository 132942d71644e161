"""§8(f)3 on the B200: the adaptive loop's kernels against the oracle (oracle/rd_oracle.cpp,
itself pinned by the reference's test_adapt.cpp / test_mesh.cpp cases in test_oracle_adapt.py).

Bars:
  * bisect_marked / uniform_refine: the refined mesh bit for bit (vertex coordinates, boundary
    flags, tets, refinement tags, generations) -- integer and exact-midpoint work;
  * mark_dorfler: the marked list exactly, on the same indicators;
  * estimate: per-tet indicators and the global value bit for bit on indicator targets (box: no
    transcendental functions), within 1e-13 where CUDA sin meets glibc sin (smooth);
  * adaptive_solve: every level's dof count and PCG iteration count equal, the estimate and
    error columns within 1e-8 (the solve agrees to 1e-10), the final mesh identical.  Run on a
    mesh with jittered interior vertices so that no two indicators tie by symmetry: with exact
    ties a 1e-12 difference in the solution could reorder tied tets around the Dorfler cut.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rd():
    from paper_2102_03515_b200 import rd as _rd

    _rd.default_context()
    return _rd


def same_mesh(dm, om):
    xyz, tets, b = dm.download()
    re, gen = dm.tags()
    assert np.array_equal(tets, om.tets), "tets"
    assert np.array_equal(xyz, om.xyz), "vertex coordinates"
    assert np.array_equal(b, om.boundary), "boundary flags"
    assert np.array_equal(re, om.refinement_edge), "refinement tags"
    assert np.array_equal(gen, om.generation), "generations"


def jittered_cube(rd, O, n, amp, seed):
    om = O.build_structured_cube(n)
    xyz = om.xyz.copy()
    r = O.pseudo_random_vec(3 * xyz.shape[0], seed).reshape(-1, 3)
    inner = om.boundary == 0
    xyz[inner] += amp / n * r[inner]
    return rd.mesh_from_arrays(xyz, om.tets, om.boundary), O.mesh_from_arrays(xyz, om.tets, om.boundary)


# ------------------------------------------------------------------ bisection
def test_bisect_single_and_all(rd, O):  # test_mesh.cpp:92-116
    dm, om = rd.build_structured_cube(2), O.build_structured_cube(2)
    same_mesh(dm, om)
    same_mesh(rd.bisect_marked(dm, []), O.bisect_marked(om, []))
    same_mesh(rd.bisect_marked(dm, [5]), O.bisect_marked(om, [5]))
    allm = list(range(om.tets.shape[0]))
    same_mesh(rd.bisect_marked(dm, allm), O.bisect_marked(om, allm))
    with pytest.raises(rd.RdInvalidArgument):
        rd.bisect_marked(rd.build_structured_cube(1), [6])
    with pytest.raises(rd.RdInvalidArgument):
        rd.bisect_marked(rd.build_structured_cube(1), [-1])


def test_uniform_refine(rd, O):  # test_mesh.cpp:73-90, 143-150
    dm, om = rd.build_structured_cube(1), O.build_structured_cube(1)
    for _ in range(2):
        dm, om = rd.uniform_refine(dm), O.uniform_refine(om)
        same_mesh(dm, om)
    assert dm.n_tets == 8 * 48


def test_repeated_selective_bisection(rd, O):  # test_mesh.cpp:124-141, every sweep vs the oracle
    dm, om = rd.build_structured_cube(2), O.build_structured_cube(2)
    for sweep in range(10):
        marks = list(range(0, om.tets.shape[0], 3))
        dm, om = rd.bisect_marked(dm, marks), O.bisect_marked(om, marks)
        same_mesh(dm, om)
    assert dm.n_tets == om.tets.shape[0] > 1000


def test_bisect_larger_random_marks(rd, O):
    """A few thousand tets, seeded random marks with duplicates, three rounds: the midpoint map
    grows and is rehashed on the device."""
    dm, om = rd.build_structured_cube(6), O.build_structured_cube(6)
    rng = np.random.default_rng(7)
    for _ in range(3):
        nt = om.tets.shape[0]
        marks = rng.integers(0, nt, size=nt // 4)
        dm, om = rd.bisect_marked(dm, marks), O.bisect_marked(om, marks)
        same_mesh(dm, om)


# ------------------------------------------------------------------ marking
def test_dorfler_hand_cases(rd):  # test_adapt.cpp:105-137
    assert list(rd.mark_dorfler([3.0, 0.0, 0.0, 0.0], 0.5)) == [0]
    assert sorted(rd.mark_dorfler([2.0, 2.0, 1.0], 0.8)) == [0, 1]
    assert list(rd.mark_dorfler([2.0, 2.0, 1.0], 0.8)) == [0, 1]  # ties: ascending tet order
    assert sorted(rd.mark_dorfler([1.0, 0.0, 2.0, 0.0, 0.5], 1.0)) == [0, 2, 4]
    assert len(rd.mark_dorfler([3.0, 2.0, 2.0, 1.0], 0.6)) == 1
    assert len(rd.mark_dorfler([], 0.5)) == 0
    for bad in (0.0, 1.5):
        with pytest.raises(rd.RdInvalidArgument):
            rd.mark_dorfler([1.0], bad)


@pytest.mark.parametrize("theta", [0.3, 0.5, 0.9, 1.0])
def test_dorfler_matches_oracle(rd, O, theta):
    rng = np.random.default_rng(3)
    eta = rng.random(20000) ** 3
    eta[rng.integers(0, eta.size, 500)] = 0.0
    eta[100:200] = eta[99]  # a run of ties
    assert np.array_equal(rd.mark_dorfler(eta, theta), O.mark_dorfler(eta, theta))


# ------------------------------------------------------------------ estimator
@pytest.mark.parametrize("n,rho,target,exact", [(4, 1e-2, "box", True), (6, 1e-3, "box", True),
                                                (4, 1e-2, "smooth", False), (5, 0.5, "nonzero_bc", False)])
def test_estimate_matches_oracle(rd, O, n, rho, target, exact):
    dm, om = rd.build_structured_cube(n), O.build_structured_cube(n)
    ds, os_ = rd.build_system(dm, rho, target), O.build_system(om, rho, target)
    u = O.dense_cholesky_solve(os_.A.dense(), os_.f) if os_.n_dofs <= 2000 else O.pcg(os_.A, "amg", os_.f, 1e-10).x
    dp, dg = rd.estimate(ds, u, target)
    op, og = O.estimate(om, os_, u, target)
    if exact:
        assert np.array_equal(dp, op) and dg == og
    else:
        assert np.allclose(dp, op, rtol=1e-13, atol=0) and dg == pytest.approx(og, rel=1e-13)


def test_estimate_on_bisected_mesh(rd, O):
    """Non-lattice meshes (the generic path): an adapted mesh from a few bisection rounds."""
    dm, om = rd.build_structured_cube(3), O.build_structured_cube(3)
    for k in range(3):
        marks = list(range(k, om.tets.shape[0], 5))
        dm, om = rd.bisect_marked(dm, marks), O.bisect_marked(om, marks)
    ds, os_ = rd.build_system(dm, 1e-2, "box"), O.build_system(om, 1e-2, "box")
    u = O.dense_cholesky_solve(os_.A.dense(), os_.f)
    dp, dg = rd.estimate(ds, u, "box")
    op, og = O.estimate(om, os_, u, "box")
    assert np.array_equal(dp, op) and dg == og


def test_zero_target_zero_indicator(rd):  # test_adapt.cpp:57-64
    ds = rd.build_system(rd.build_structured_cube(3), 0.01, "zero")
    per, g = rd.estimate(ds, np.zeros(ds.n_dofs), "zero")
    assert g == 0.0 and np.abs(per).max() == 0.0


# ------------------------------------------------------------------ the loop
def test_adaptive_solve_matches_oracle(rd, O):
    dm, om = jittered_cube(rd, O, 4, 0.15, 11)
    res = rd.adaptive_solve(dm, "box", 1e-2, 1500, tol=1e-10)
    orows, ofinal, ocoeffs = O.adaptive_solve(om, "box", 1e-2, 1500, tol=1e-10)
    assert len(res.history) == len(orows) >= 3
    for d, o in zip(res.history, orows):
        assert (d["level"], d["dofs"], d["iterations"]) == (o["level"], o["dofs"], o["iterations"])
        for k in ("eta", "err_l2_sq", "err_hm1_sq"):
            assert d[k] == pytest.approx(o[k], rel=1e-8), k
    same_mesh(res.mesh, ofinal)
    assert np.abs(res.coefficients - ocoeffs).max() <= 1e-9 * np.abs(ocoeffs).max()


def test_adaptive_solve_properties(rd):  # test_adapt.cpp:139-161 on the device
    res = rd.adaptive_solve(rd.build_structured_cube(4), "box", 1e-2, 800, tol=1e-10)
    h = res.history
    assert len(h) >= 2 and h[-1]["dofs"] >= 800
    assert all(h[l]["dofs"] > h[l - 1]["dofs"] and h[l]["level"] == l for l in range(1, len(h)))
    assert h[-1]["eta"] < h[0]["eta"] and h[-1]["err_l2_sq"] < h[0]["err_l2_sq"]
    assert res.coefficients.size == h[-1]["dofs"]
    one = rd.adaptive_solve(rd.build_structured_cube(4), "box", 1e-2, 5)
    assert len(one.history) == 1 and one.history[0]["dofs"] == 27 and one.mesh.n_tets == 384
    with pytest.raises(rd.RdInvalidArgument):
        rd.adaptive_solve(rd.build_structured_cube(4), "box", 1e-2, 800, theta=0.0)
