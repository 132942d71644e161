"""§8(f)3 oracle pins: the reference's own adaptivity and bisection test cases
(tests/test_adapt.cpp, tests/test_mesh.cpp:73-150) re-expressed against the CPU restatement
(oracle/rd_oracle.cpp: estimate, mark_dorfler, bisect_marked, uniform_refine, adaptive_solve).
The device path (tests/test_gpu_adapt.py) is then checked against this oracle."""
import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


@pytest.fixture(scope="module")
def O():
    import pyoracle

    pyoracle.build()
    return pyoracle


# ------------------------------------------------------------------ helpers (tests/oracles.hpp)
def mesh_conforming(m) -> bool:  # oracles.hpp:32-62
    faces = {}
    for t in m.tets:
        for f in range(4):
            key = tuple(sorted(int(t[v]) for v in range(4) if v != f))
            faces[key] = faces.get(key, 0) + 1
    for key, count in faces.items():
        if count > 2:
            return False
        if count == 1:
            x = m.xyz[list(key)]
            if not any(np.all(np.abs(x[:, c] - p) <= 1e-12) for c in range(3) for p in (0.0, 1.0)):
                return False
    return True


def total_volume(O, m) -> float:
    return sum(O.tet_volume(m, t) for t in range(m.tets.shape[0]))


def boundary_flags_consistent(m) -> bool:  # test_mesh.cpp:22-31
    on = np.any((np.abs(m.xyz) <= 1e-12) | (np.abs(m.xyz - 1.0) <= 1e-12), axis=1)
    return bool(np.array_equal(on, m.boundary != 0))


def tags_valid(m) -> bool:
    return bool(np.all((m.refinement_edge >= 1) & (m.refinement_edge <= 3)))


def min_dihedral_degrees(m) -> float:  # oracles.hpp:71-94
    best = 180.0
    for tet in m.tets:
        for a in range(4):
            for b in range(a + 1, 4):
                rest = [v for v in range(4) if v not in (a, b)]
                pa, pb = m.xyz[tet[a]], m.xyz[tet[b]]
                pc, pd = m.xyz[tet[rest[0]]], m.xyz[tet[rest[1]]]
                e = (pb - pa) / np.linalg.norm(pb - pa)
                u = (pc - pa) - np.dot(pc - pa, e) * e
                v = (pd - pa) - np.dot(pd - pa, e) * e
                best = min(best, math.degrees(math.atan2(np.linalg.norm(np.cross(u, v)), np.dot(u, v))))
    return best


def h_max(m) -> float:
    h = 0.0
    for t in m.tets:
        for a in range(4):
            for b in range(a + 1, 4):
                h = max(h, float(np.linalg.norm(m.xyz[t[a]] - m.xyz[t[b]])))
    return h


# ------------------------------------------------------------------ bisection (test_mesh.cpp)
def test_uniform_refinement_eight_children(O):  # test_mesh.cpp:73-90
    fine = O.uniform_refine(O.build_structured_cube(1))
    assert fine.tets.shape[0] == 48 and fine.xyz.shape[0] == 27
    assert total_volume(O, fine) == pytest.approx(1.0, rel=1e-13)
    assert mesh_conforming(fine) and boundary_flags_consistent(fine) and tags_valid(fine)
    assert h_max(fine) == pytest.approx(math.sqrt(3.0) / 2.0, rel=1e-13)
    finer = O.uniform_refine(fine)
    assert finer.tets.shape[0] == 8 * 48 and mesh_conforming(finer)
    assert h_max(finer) == pytest.approx(math.sqrt(3.0) / 4.0, rel=1e-13)


def test_empty_marking_is_identity(O):  # test_mesh.cpp:92-97
    m = O.build_structured_cube(2)
    out = O.bisect_marked(m, [])
    assert out.tets.shape == m.tets.shape and out.xyz.shape == m.xyz.shape


def test_single_mark_closes_conformally(O):  # test_mesh.cpp:99-108
    m = O.build_structured_cube(2)
    out = O.bisect_marked(m, [5])
    assert out.tets.shape[0] > m.tets.shape[0] and out.xyz.shape[0] > m.xyz.shape[0]
    assert mesh_conforming(out) and boundary_flags_consistent(out) and tags_valid(out)
    assert total_volume(O, out) == pytest.approx(1.0, rel=1e-13)


def test_mark_everything_doubles(O):  # test_mesh.cpp:110-116
    m = O.build_structured_cube(2)
    out = O.bisect_marked(m, range(m.tets.shape[0]))
    assert out.tets.shape[0] == 2 * m.tets.shape[0] and mesh_conforming(out)
    assert np.all(out.generation == 1)


def test_mark_rejects_out_of_range(O):  # test_mesh.cpp:118-122
    m = O.build_structured_cube(1)
    for bad in ([6], [-1]):
        with pytest.raises(O.OracleError):
            O.bisect_marked(m, bad)


def test_repeated_selective_bisection(O):  # test_mesh.cpp:124-141
    m = O.build_structured_cube(2)
    assert min_dihedral_degrees(m) > 30.0
    for _ in range(10):
        m = O.bisect_marked(m, range(0, m.tets.shape[0], 3))
        assert mesh_conforming(m) and tags_valid(m)
        assert total_volume(O, m) == pytest.approx(1.0, rel=1e-12)
    assert boundary_flags_consistent(m)
    assert min_dihedral_degrees(m) > 10.0
    assert all(O.tet_volume(m, t) > 0.0 for t in range(m.tets.shape[0]))


def test_generation_counts_children(O):  # test_mesh.cpp:143-150
    m = O.build_structured_cube(1)
    assert np.all(O.bisect_marked(m, range(6)).generation == 1)
    assert np.all(O.uniform_refine(m).generation == 3)


# ------------------------------------------------------------------ estimator / marking (test_adapt.cpp)
def test_zero_target_zero_indicator(O):  # test_adapt.cpp:57-64 (zero field: zero coefficients, zero target)
    m = O.build_structured_cube(3)
    s = O.build_system(m, 0.01, "zero")
    per, g = O.estimate(m, s, np.zeros(s.n_dofs), "zero")
    assert g == 0.0 and np.abs(per).max() == 0.0


def test_indicator_nonnegative_localized(O):  # test_adapt.cpp:66-80
    m = O.build_structured_cube(4)
    s = O.build_system(m, 1e-2, "box")
    u = O.dense_cholesky_solve(s.A.dense(), s.f)
    per, g = O.estimate(m, s, u, "box")
    assert per.size == m.tets.shape[0] and np.all(per >= 0.0)
    assert g == pytest.approx(math.sqrt(float(np.sum(per * per))), rel=1e-13) and g > 0.0


def test_estimator_brackets_energy_error(O):  # test_adapt.cpp:82-103
    rho = 1e-2
    coarse = O.build_structured_cube(4)
    sc = O.build_system(coarse, rho, "smooth")
    uc = O.dense_cholesky_solve(sc.A.dense(), sc.f)
    _, g = O.estimate(coarse, sc, uc, "smooth")
    fine = O.uniform_refine(coarse)
    sf = O.build_system(fine, rho, "smooth")
    uf = O.pcg(sf.A, "amg", sf.f, 1e-12, 500).x
    err_sq = float(uf @ sf.f - uc @ sc.f)
    assert err_sq > 0.0
    err = math.sqrt(err_sq)
    assert err / 20.0 < g < err * 20.0


def test_dorfler_hand_cases(O):  # test_adapt.cpp:105-137
    assert list(O.mark_dorfler([3.0, 0.0, 0.0, 0.0], 0.5)) == [0]
    mk = list(O.mark_dorfler([2.0, 2.0, 1.0], 0.8))
    assert sorted(mk) == [0, 1]
    assert sorted(O.mark_dorfler([1.0, 0.0, 2.0, 0.0, 0.5], 1.0)) == [0, 2, 4]
    assert len(O.mark_dorfler([3.0, 2.0, 2.0, 1.0], 0.6)) == 1
    for bad in (0.0, 1.5):
        with pytest.raises(O.OracleError):
            O.mark_dorfler([1.0], bad)


# ------------------------------------------------------------------ the loop
def test_adaptive_loop_reaches_budget(O):  # test_adapt.cpp:139-152
    rows, final, coeffs = O.adaptive_solve(O.build_structured_cube(4), "box", 1e-2, 800, tol=1e-10)
    assert len(rows) >= 2
    for l in range(1, len(rows)):
        assert rows[l]["dofs"] > rows[l - 1]["dofs"] and rows[l]["level"] == l
    assert rows[-1]["dofs"] >= 800
    assert rows[-1]["eta"] < rows[0]["eta"] and rows[-1]["err_l2_sq"] < rows[0]["err_l2_sq"]
    assert coeffs.size == rows[-1]["dofs"]
    assert mesh_conforming(final)


def test_budget_below_initial_single_level(O):  # test_adapt.cpp:154-161
    init = O.build_structured_cube(4)
    rows, final, _ = O.adaptive_solve(init, "box", 1e-2, 5)
    assert len(rows) == 1 and rows[0]["dofs"] == 27 and final.tets.shape[0] == init.tets.shape[0]


def test_history_errors_against_target(O):  # test_adapt.cpp:163-175
    init = O.build_structured_cube(4)
    rows, _, coeffs = O.adaptive_solve(init, "box", 0.1, 20)
    assert len(rows) == 1
    s = O.build_system(init, 0.1, "box")
    assert rows[0]["err_l2_sq"] == pytest.approx(O.l2_error_target_squared(init, s, coeffs, "box"), rel=1e-10)
    assert rows[0]["err_hm1_sq"] == pytest.approx(O.target_dual_norm(s, coeffs) ** 2, rel=1e-8)
