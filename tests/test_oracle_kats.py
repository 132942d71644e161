"""Pins the CPU oracle against the reference's own known-answer tests.

The reference (rdsolve) cannot be compiled here (no Eigen), so every hand
case, dense-oracle check and property the reference's doctest suites hold for
the solve path is re-expressed here against the oracle restatement.  Each test
cites the reference test it mirrors (paths relative to /root/reference/proj).
"""
import json
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def path_laplacian(O, n):  # test_amg.cpp:16-27
    t = []
    for i in range(n):
        t.append((i, i, 2.0))
        if i + 1 < n:
            t.append((i, i + 1, -1.0))
            t.append((i + 1, i, -1.0))
    return O.from_triplets(n, n, t)


def band_spd(O, n):  # test_linalg.cpp:19-34
    t = []
    for i in range(n):
        t.append((i, i, 4.0 + 0.01 * i))
        if i + 1 < n:
            t += [(i, i + 1, -1.0), (i + 1, i, -1.0)]
        if i + 3 < n:
            t += [(i, i + 3, -0.5), (i + 3, i, -0.5)]
    return O.from_triplets(n, n, t)


def interior_matrix(O, n, rho):  # test_amg.cpp:29-32
    return O.build_system(O.build_structured_cube(n), rho, "smooth").A


# ------------------------------------------------------------------ mesh
def test_structured_cube_n1(O):  # test_mesh.cpp:41-53
    m = O.build_structured_cube(1)
    assert m.xyz.shape[0] == 8 and m.tets.shape[0] == 6
    vol = sum(O.tet_volume(m, t) for t in range(6))
    assert vol == pytest.approx(1.0, rel=1e-14)
    assert int((m.boundary == 0).sum()) == 0
    assert (m.refinement_edge == 3).all()


def test_structured_cube_n4(O):  # test_mesh.cpp:55-66
    m = O.build_structured_cube(4)
    assert m.xyz.shape[0] == 125 and m.tets.shape[0] == 384
    assert sum(O.tet_volume(m, t) for t in range(384)) == pytest.approx(1.0, rel=1e-13)
    assert int((m.boundary == 0).sum()) == 27
    e = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    hmax = max(np.linalg.norm(m.xyz[t[a]] - m.xyz[t[b]]) for t in m.tets for a, b in e)
    assert hmax == pytest.approx(math.sqrt(3.0) / 4.0, rel=1e-13)
    on = ((np.abs(m.xyz) <= 1e-12) | (np.abs(m.xyz - 1) <= 1e-12)).any(axis=1)
    assert (on == (m.boundary != 0)).all()


def test_structured_cube_rejects_nonpositive(O):  # test_mesh.cpp:68-71
    for n in (0, -3):
        with pytest.raises(ValueError):
            O.build_structured_cube(n)


def test_mesh_faces_conform(O):  # oracles.hpp:32-62 on n=2
    m = O.build_structured_cube(2)
    faces = {}
    for t in m.tets:
        for f in range(4):
            key = tuple(sorted(int(t[v]) for v in range(4) if v != f))
            faces[key] = faces.get(key, 0) + 1
    for key, cnt in faces.items():
        assert cnt <= 2
        if cnt == 1:
            pts = m.xyz[list(key)]
            assert any(np.all(np.abs(pts[:, c] - p) <= 1e-12) for c in range(3) for p in (0.0, 1.0))


# ------------------------------------------------------------------ quadrature
def _rule_integral(pts, w, vol, e):
    return vol * sum(w[q] * np.prod([pts[q, c] ** e[c] for c in range(4)]) for q in range(len(w)))


def _bary(vol, e):
    return 6.0 * vol * np.prod([math.factorial(k) for k in e]) / math.factorial(sum(e) + 3)


def test_rules_weights_points(O):  # test_quadrature.cpp:28-60
    sizes = {0: 1, 1: 4, 2: 14, 3: 64}
    for rid, size in sizes.items():
        pts, w = O.rule(rid)
        assert len(w) == size
        assert (w > 0).all() and w.sum() == pytest.approx(1.0, rel=1e-14)
        assert (pts >= 0).all()
        assert np.allclose(pts.sum(axis=1), 1.0, rtol=0, atol=1e-14)


def test_rule_exactness(O):  # test_quadrature.cpp:62-99
    pts, w = O.rule(2)
    for e in [(5, 0, 0, 0), (3, 2, 0, 0), (2, 2, 1, 0), (1, 1, 1, 2), (0, 4, 1, 0), (2, 1, 1, 1)]:
        assert _rule_integral(pts, w, 0.8, e) == pytest.approx(_bary(0.8, e), rel=1e-12)
    pts, w = O.rule(1)
    for e in [(2, 0, 0, 0), (1, 1, 0, 0), (0, 1, 1, 0), (0, 0, 0, 2)]:
        assert _rule_integral(pts, w, 1 / 6, e) == pytest.approx(_bary(1 / 6, e), rel=1e-13)
    pts, w = O.rule(3)
    assert np.all(w == 1.0 / 64.0)
    for e in [(1, 0, 0, 0), (0, 0, 1, 0)]:
        assert _rule_integral(pts, w, 0.25, e) == pytest.approx(_bary(0.25, e), rel=1e-13)


# ------------------------------------------------------------------ targets
def test_targets(O):  # test_targets.cpp:12-40
    assert O.target_eval("smooth", [0.5, 0.5, 0.5])[0] == pytest.approx(1.0, rel=1e-14)
    assert abs(O.target_eval("smooth", [0.0, 0.3, 0.7])[0]) < 1e-14
    s = math.sin(math.pi * 0.3)
    assert O.target_eval("smooth", [0.3, 0.3, 0.3])[0] == pytest.approx(s ** 3, rel=1e-14)
    box = O.target_eval("box", [[0.5, 0.5, 0.5], [0.1, 0.1, 0.1], [0.25, 0.5, 0.5], [0.26, 0.74, 0.5],
                                [0.5, 0.5, 0.75]])
    assert list(box) == [1.0, 0.0, 0.0, 1.0, 0.0]
    nz = O.target_eval("nonzero_bc", [[0, 0, 0], [0.5, 0.5, 0.5]])
    assert nz[0] == pytest.approx(1.0, rel=1e-14) and nz[1] == pytest.approx(2.0, rel=1e-14)


def test_ball_and_random_targets(O):  # BASELINE configs 2 and 3
    ball = O.target_eval("ball", [[0.5, 0.5, 0.5], [0.75, 0.5, 0.5], [0.74, 0.5, 0.5], [0.1, 0.1, 0.1]])
    assert list(ball) == [1.0, 0.0, 1.0, 0.0]
    n = 4
    r = O.pseudo_random_vec((n + 1) ** 3, 0)
    m = O.build_structured_cube(n)
    # at every vertex the P1 interpolant reproduces the (boundary-zeroed) nodal value
    vals = O.target_eval("sine_random", m.xyz, n=n, seed=0)
    sine = O.target_eval("smooth", m.xyz)
    rz = np.where(m.boundary != 0, 0.0, r)
    assert np.allclose(vals - sine, 0.1 * rz, rtol=0, atol=1e-15)


def test_splitmix_generator(O):  # oracles.hpp:97-108
    v = O.pseudo_random_vec(1000, 7)
    assert (v >= -1).all() and (v < 1).all()
    assert np.array_equal(v, O.pseudo_random_vec(1000, 7))


# ------------------------------------------------------------------ assembly
def _ref_tet(O):  # test_assembly.cpp:23-33
    return O.mesh_from_arrays([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], [[0, 1, 2, 3]], [0, 0, 0, 0])


def test_reference_tet_stiffness(O):  # test_assembly.cpp:41-50
    K = O.assemble_full(_ref_tet(O), "K").dense()
    assert K[0, 0] == pytest.approx(0.5, rel=1e-14)
    assert K[1, 1] == pytest.approx(1 / 6, rel=1e-14)
    assert np.allclose(K.sum(axis=1), 0.0, atol=1e-14)
    assert np.allclose(K, K.T)


def test_reference_tet_mass(O):  # test_assembly.cpp:52-62
    M = O.assemble_full(_ref_tet(O), "M").dense()
    v = 1 / 6
    for i in range(4):
        assert M[i, i] == pytest.approx(v / 10, rel=1e-14)
        for j in range(4):
            if i != j:
                assert M[i, j] == pytest.approx(v / 20, rel=1e-14)
    assert M.sum() == pytest.approx(v, rel=1e-14)


def test_full_mass_and_stiffness_sums(O):  # test_assembly.cpp:64-71
    m = O.build_structured_cube(3)
    assert O.assemble_full(m, "M").dense().sum() == pytest.approx(1.0, rel=1e-12)
    assert np.allclose(O.assemble_full(m, "K").dense().sum(axis=1), 0.0, atol=1e-12)


def test_interior_spd_symmetric(O):  # test_assembly.cpp:73-83
    s = O.build_system(O.build_structured_cube(3), 1e-3, "smooth")
    for X in (s.K, s.M, s.A):
        D = X.dense()
        assert np.abs(D - D.T).max() <= 1e-14
        np.linalg.cholesky(D)
        O.dense_cholesky_solve(D, np.ones(D.shape[0]))


def test_affine_in_rho(O):  # test_assembly.cpp:85-94
    m = O.build_structured_cube(3)
    s1, s2 = O.build_system(m, 0.25, "smooth"), O.build_system(m, 1.25, "smooth")
    assert np.abs(s2.A.dense() - s1.A.dense() - s1.K.dense()).max() < 1e-13
    assert np.abs(s1.A.dense() - 0.25 * s1.K.dense() - s1.M.dense()).max() < 1e-13


def test_rejects_nonpositive_rho(O):  # test_assembly.cpp:96-100
    with pytest.raises(ValueError):
        O.build_system(O.build_structured_cube(2), 0.0, "smooth")


def test_zero_and_constant_loads(O):  # test_assembly.cpp:102-124
    m = O.build_structured_cube(3)
    assert np.linalg.norm(O.assemble_load(m, "zero")) == 0.0
    f = O.assemble_load(m, "one")
    s = O.build_system(m, 1.0, "smooth")
    exp = np.zeros(f.size)
    for t in range(m.tets.shape[0]):
        for v in m.tets[t]:
            d = s.vertex_to_dof[v]
            if d >= 0:
                exp[d] += O.tet_volume(m, t) / 4
    assert np.allclose(f, exp, rtol=1e-13, atol=0)


def test_polynomial_load(O):  # test_assembly.cpp:126-154 (independent per-element loop)
    m = O.build_structured_cube(2)
    f = O.assemble_load(m, "quadratic")
    s = O.build_system(m, 1.0, "smooth")
    pts, w = O.rule(2)
    exp = np.zeros(f.size)
    for t in range(m.tets.shape[0]):
        V = m.xyz[m.tets[t]]
        X = pts @ V
        vol = O.tet_volume(m, t)
        u = X[:, 0] * X[:, 1] + 2 * X[:, 2]
        for lv, v in enumerate(m.tets[t]):
            d = s.vertex_to_dof[v]
            if d >= 0:
                exp[d] += vol * np.sum(w * u * pts[:, lv])
    assert np.abs(f - exp).max() < 1e-13


def test_errors_vanish_and_interpolation_order(O):  # test_assembly.cpp:330-356
    m = O.build_structured_cube(3)
    s = O.build_system(m, 1.0, "smooth")
    z = np.zeros(s.n_dofs)
    # exact solution of rho = infinity-ish is not available; the zero field against
    # the zero function uses l2 with the closed form scaled to zero via huge rho
    errs = []
    for n in (4, 8):
        mm = O.build_structured_cube(n)
        ss = O.build_system(mm, 1.0, "smooth")
        c = 1.0 / (3.0 * math.pi ** 2 + 1.0)
        xyz = mm.xyz[ss.dof_to_vertex]
        coeff = c * np.sin(math.pi * xyz[:, 0]) * np.sin(math.pi * xyz[:, 1]) * np.sin(math.pi * xyz[:, 2])
        errs.append(O.l2_error_manufactured(mm, ss, coeff, 1.0))
    assert 3.0 < errs[0] / errs[1] < 5.0
    assert O.l2_error_manufactured(m, s, z, 1.0) > 0


# ------------------------------------------------------------------ linalg
def test_from_triplets(O):  # test_linalg.cpp:38-45
    A = O.from_triplets(2, 2, [(0, 0, 1.0), (0, 0, 2.0), (1, 1, 5.0), (0, 1, 0.0)])
    assert A.nnz == 2
    D = A.dense()
    assert D[0, 0] == 3.0 and D[1, 1] == 5.0 and D[0, 1] == 0.0


def test_spmv_hand_and_dense(O):  # test_linalg.cpp:47-66
    I3 = O.from_triplets(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0)])
    x = np.array([3.0, -1.0, 2.0])
    assert np.array_equal(O.spmv(I3, x), x)
    A = O.from_triplets(2, 2, [(0, 0, 2.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 2.0)])
    assert list(O.spmv(A, np.ones(2))) == [3.0, 3.0]
    B = band_spd(O, 50)
    x = O.pseudo_random_vec(50, 7)
    assert np.linalg.norm(O.spmv(B, x) - B.dense() @ x) < 1e-13


def test_spmv_dimension_mismatch(O):  # test_linalg.cpp:68-71
    with pytest.raises(ValueError):
        O.spmv(band_spd(O, 4), np.ones(5))


def test_dense_cholesky(O):  # test_linalg.cpp:80-94
    x = O.dense_cholesky_solve(np.array([[4.0, 2.0], [2.0, 3.0]]), np.array([2.0, 1.0]))
    assert x[0] == pytest.approx(0.5, rel=1e-14) and abs(x[1]) < 1e-14
    with pytest.raises(RuntimeError):
        O.dense_cholesky_solve(np.array([[1.0, 2.0], [2.0, 1.0]]), np.ones(2))


def test_pcg_cases(O):  # test_linalg.cpp:96-139
    A1 = O.from_triplets(1, 1, [(0, 0, 2.0)])
    r = O.pcg(A1, "identity", np.array([4.0]), 1e-12, 10)
    assert r.converged and r.iterations == 1 and r.x[0] == pytest.approx(2.0, rel=1e-14)
    B = band_spd(O, 40)
    f = O.pseudo_random_vec(40, 3)
    r = O.pcg(B, "jacobi", f, 1e-12, 200)
    assert r.converged and np.abs(r.x - np.linalg.solve(B.dense(), f)).max() < 1e-9
    assert len(r.residual_history) == r.iterations and r.residual_history[-1] <= 1e-12
    r = O.pcg(B, "identity", np.ones(40), 1e-14, 2)
    assert not r.converged and r.iterations == 2
    r = O.pcg(band_spd(O, 8), "identity", np.zeros(8), 1e-10, 10)
    assert r.converged and r.iterations == 0 and np.linalg.norm(r.x) == 0.0
    with pytest.raises(RuntimeError):
        O.pcg(O.from_triplets(2, 2, [(0, 0, 1.0), (1, 1, -1.0)]), "identity", np.ones(2), 1e-10, 10)


def test_pcg_permutation_invariance(O):  # test_linalg.cpp:141-159
    n = 12
    A = band_spd(O, n)
    perm = [(5 * i + 3) % n for i in range(n)]
    t = []
    for r in range(n):
        for k in range(A.rp[r], A.rp[r + 1]):
            t.append((perm[r], perm[A.ci[k]], A.v[k]))
    B = O.from_triplets(n, n, t)
    f = O.pseudo_random_vec(n, 11)
    g = np.zeros(n)
    for i in range(n):
        g[perm[i]] = f[i]
    x = O.pcg(A, "jacobi", f, 1e-13, 100).x
    y = O.pcg(B, "jacobi", g, 1e-13, 100).x
    for i in range(n):
        assert y[perm[i]] == pytest.approx(x[i], rel=1e-8)


# ------------------------------------------------------------------ amg
def test_coarsen_path_graph(O):  # test_amg.cpp:36-52
    flags, P = O.coarsen_redblack(path_laplacian(O, 5))
    assert list(flags) == [1, 0, 1, 0, 1]
    D = P.dense()
    assert D.shape == (5, 3)
    assert D[0, 0] == 1.0 and D[1, 0] == 0.5 and D[1, 1] == 0.5 and D[2, 1] == 1.0 and D[4, 2] == 1.0


def test_coarsen_diagonal(O):  # test_amg.cpp:54-60
    flags, P = O.coarsen_redblack(O.from_triplets(3, 3, [(0, 0, 1.0), (1, 1, 2.0), (2, 2, 3.0)]))
    assert list(flags) == [1, 1, 1]
    assert np.array_equal(P.dense(), np.eye(3))


def test_coarse_set_independent_maximal(O):  # test_amg.cpp:62-81
    A = interior_matrix(O, 4, 1e-2)
    flags, P = O.coarsen_redblack(A)
    for i in range(A.rows):
        nb = [A.ci[k] for k in range(A.rp[i], A.rp[i + 1]) if A.ci[k] != i]
        if flags[i]:
            assert not any(flags[j] for j in nb)
        else:
            assert any(flags[j] for j in nb)
    assert np.allclose(P.dense().sum(axis=1), 1.0, rtol=1e-13)


def test_galerkin_hand_case(O):  # test_amg.cpp:83-90
    A = O.from_triplets(2, 2, [(0, 0, 2.0), (0, 1, -1.0), (1, 0, -1.0), (1, 1, 2.0)])
    P = O.from_triplets(2, 1, [(0, 0, 1.0), (1, 0, 0.5)])
    Ac = O.galerkin_coarse(A, P)
    assert Ac.rows == 1 and Ac.dense()[0, 0] == pytest.approx(1.5, rel=1e-14)


def test_galerkin_identity(O):  # test_amg.cpp:92-99
    A = path_laplacian(O, 7)
    I7 = O.from_triplets(7, 7, [(i, i, 1.0) for i in range(7)])
    assert np.array_equal(O.galerkin_coarse(A, I7).dense(), A.dense())


def test_galerkin_dense_triple_product(O):  # test_amg.cpp:101-107
    A = interior_matrix(O, 4, 1e-4)
    _, P = O.coarsen_redblack(A)
    Ac = O.galerkin_coarse(A, P)
    ref = P.dense().T @ A.dense() @ P.dense()
    assert np.abs(Ac.dense() - ref).max() < 1e-12


def test_sgs_hand_sweep(O):  # test_amg.cpp:109-117
    A = O.from_triplets(2, 2, [(0, 0, 2.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 2.0)])
    u = O.sgs_sweep(A, np.ones(2), np.zeros(2))
    assert u[0] == pytest.approx(0.375, rel=1e-15) and u[1] == pytest.approx(0.25, rel=1e-15)


def test_gs_exact_on_diagonal(O):  # test_amg.cpp:119-126
    A = O.from_triplets(2, 2, [(0, 0, 2.0), (1, 1, 4.0)])
    u = O.sgs_sweep(A, np.array([2.0, 2.0]), np.zeros(2))
    assert u[0] == 1.0 and u[1] == 0.5


def test_vcycle_linear(O):  # test_amg.cpp:128-137
    A = interior_matrix(O, 4, 1e-6)
    h = O.build_amg(A, 16)
    r1, r2 = O.pseudo_random_vec(A.rows, 1), O.pseudo_random_vec(A.rows, 2)
    lhs = h.apply(2.0 * r1 - 3.0 * r2)
    rhs = 2.0 * h.apply(r1) - 3.0 * h.apply(r2)
    assert np.abs(lhs - rhs).max() < 1e-12


def test_vcycle_symmetric_positive(O):  # test_amg.cpp:139-151
    A = interior_matrix(O, 4, 1e-2)
    h = O.build_amg(A, 16)
    for s in range(5):
        r1, r2 = O.pseudo_random_vec(A.rows, 10 + s), O.pseudo_random_vec(A.rows, 20 + s)
        assert r2 @ h.apply(r1) == pytest.approx(r1 @ h.apply(r2), rel=1e-11)
        assert r1 @ h.apply(r1) > 0


def test_error_propagation_contracts(O):  # test_amg.cpp:153-160
    A = interior_matrix(O, 3, 1.0)
    h = O.build_amg(A, 4)
    e = O.pseudo_random_vec(A.rows, 5)
    e0 = np.linalg.norm(e)
    for _ in range(50):
        e = e - h.apply(O.spmv(A, e))
    assert np.linalg.norm(e) < 1e-6 * e0


def test_single_level_exact_inverse(O):  # test_amg.cpp:162-170
    A = interior_matrix(O, 3, 0.5)
    h = O.build_amg(A, 1000)
    assert h.num_levels == 1
    r = O.pseudo_random_vec(A.rows, 9)
    assert np.abs(h.apply(r) - np.linalg.solve(A.dense(), r)).max() < 1e-10


def test_levels_shrink_galerkin_identity(O):  # test_amg.cpp:172-185
    A = interior_matrix(O, 6, 1e-4)
    h = O.build_amg(A, 8)
    assert h.num_levels >= 2
    for l in range(1, h.num_levels):
        assert h.level(l).rows < h.level(l - 1).rows
    for l in range(h.num_levels - 1):
        P, Al = h.level(l, "P").dense(), h.level(l).dense()
        assert np.abs(h.level(l + 1).dense() - P.T @ Al @ P).max() < 1e-12


def test_rho_robust_counts_n8(O):  # test_amg.cpp:187-202
    m = O.build_structured_cube(8)

    def iters(rho):
        s = O.build_system(m, rho, "smooth")
        r = O.pcg(s.A, "amg", s.f, 1e-8, 200)
        assert r.converged
        return r.iterations

    a, b = iters(1.0), iters(1e-12)
    assert a <= 30 and b <= 30 and b <= a + 2


def test_empty_system(O):  # test_amg.cpp:204-210
    A = O.Csr(0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0))
    h = O.build_amg(A)
    assert h.apply(np.zeros(0)).size == 0


# ------------------------------------------------------------------ end to end
def test_backends_agree_n5(O):  # test_bench.cpp:171-183 (AMG vs dense)
    m = O.build_structured_cube(5)
    for rho in (1.0, 1e-6):
        s = O.build_system(m, rho, "smooth")
        ref = np.linalg.solve(s.A.dense(), s.f)
        out = O.solve_system_amg(s, 1e-10)
        assert out.converged and np.abs(out.u - ref).max() < 1e-6


def test_criterion5_amg_robustness(O):  # acceptance.cpp:149-178 (n in {8,16} here; 32 in the slow set)
    rhos = [1.0, 1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12]
    for n in (8, 16):
        m = O.build_structured_cube(n)
        its = {}
        for rho in rhos:
            out = O.solve_system_amg(O.build_system(m, rho, "smooth"))
            assert out.converged and out.iterations <= 30
            its[rho] = out.iterations
        assert its[1e-12] <= its[1.0] + 2


def test_criterion3_l2_error(O):  # acceptance.cpp:116-131
    m = O.build_structured_cube(16)
    s = O.build_system(m, 1.0, "smooth")
    out = O.solve_system_amg(s)
    err = O.l2_error_manufactured(m, s, out.u, 1.0)
    assert 2.2924e-4 / 2 <= err <= 2.2924e-4 * 2


def test_appendix_a_hierarchy(O):  # SURVEY.md Appendix A table (n = 32)
    with open(os.path.join(GOLDEN, "appendix_a.json")) as fh:
        gold = json.load(fh)["32"]
    A = O.build_system(O.build_structured_cube(32), 2.0 ** -10, "smooth").A
    h = O.build_amg(A)
    assert [h.level(l).rows for l in range(h.num_levels)] == gold["rows"]
    assert [h.level(l).nnz for l in range(h.num_levels)] == gold["nnzA"]
    assert [h.level(l, "P").nnz for l in range(h.num_levels - 1)] == gold["nnzP"]
    # C = the all-even lattice points at level 0 (Appendix A)
    m = 31
    idx = np.arange(A.rows)
    a, b, c = idx % m, (idx // m) % m, idx // (m * m)
    even = ((a % 2 == 0) & (b % 2 == 0) & (c % 2 == 0)).astype(np.uint8)
    assert np.array_equal(h.flags(0), even)


def test_l2_error_target_squared_kats(O):
    """assembly.cpp:312-331 restated: exact integrals of the target against the zero field."""
    n = 4
    m = O.build_structured_cube(n)
    for target, want in [("zero", 0.0), ("one", 1.0), ("quadratic", 35.0 / 18.0)]:
        s = O.build_system(m, 1.0, target)
        got = O.l2_error_target_squared(m, s, np.zeros(s.n_dofs), target)
        assert abs(got - want) <= 1e-13 * max(1.0, want), (target, got, want)
    # the P1 interpolant of a linear field is exact: zero distance up to rounding
    s = O.build_system(m, 1.0, "one")
    assert O.l2_error_target_squared(m, s, np.ones(s.n_dofs), "one") > 0.0  # boundary nodes are 0


def test_oracle_reproduces_c1_golden(O):
    """The committed goldens (tools/make_goldens.py) are the oracle's own answers: C1 re-run."""
    g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                    "baseline_configs.json")))["cases"]
    c1 = next(c for c in g if c["name"] == "C1")
    m = O.build_structured_cube(c1["n"])
    s = O.build_system(m, c1["rho"], c1["target"])
    r = O.pcg(s.A, "amg", s.f, 1e-8, 500)
    assert r.iterations == c1["iterations"]
    assert [float(v) for v in r.residual_history] == c1["residual_history"]
    assert float(np.linalg.norm(r.x)) == c1["u_norm2"]
    assert math.sqrt(O.l2_error_target_squared(m, s, r.x, "smooth")) == c1["l2_u_minus_target"]
    l2d5, h1 = O.error_norms_target(m, s, r.x, "smooth", c1["n"], 0)
    assert l2d5 == c1["l2_deg5_u_minus_target"] and h1 == c1["h1_u_minus_target"]


def _fd_grad(O, kind, pts, n, h=1e-7):
    fd = np.zeros_like(pts)
    for d in range(3):
        e = np.zeros(3)
        e[d] = h
        fd[:, d] = (O.target_eval(kind, pts + e, n, 0) - O.target_eval(kind, pts - e, n, 0)) / (2 * h)
    return fd


@pytest.mark.parametrize("kind", ["smooth", "nonzero_bc", "sine_random", "quadratic", "ball", "one"])
def test_target_gradient_matches_finite_differences(O, kind):
    """The exact gradients behind the error gates (oracle Target::grad) against central
    differences of the target evaluator, at points inside Kuhn tets (away from faces, where the
    random part's P1 gradient jumps)."""
    n = 8
    rng = np.random.default_rng(3)
    cells = rng.integers(0, n, (200, 3))
    xi = rng.uniform(0.0, 1.0, (200, 3))
    srt = -np.sort(-xi, axis=1)  # keep points 1e-3 away from every tet face of the cell
    gaps = np.concatenate([1 - srt[:, :1], srt[:, :-1] - srt[:, 1:], srt[:, -1:]], axis=1)
    keep = gaps.min(axis=1) > 1e-3
    pts = ((cells + xi) / n)[keep]
    g = O.target_grad(kind, pts, n)
    fd = _fd_grad(O, kind, pts, n)
    assert np.abs(g - fd).max() <= 1e-6 * max(1.0, np.abs(g).max())


def test_error_norms_target_smooth_is_manufactured_zero(O):
    """||grad(u - u_bar)|| of the smooth target is h1_semi_error with
    manufactured_exact(0) (c = 1 exactly), and ||u - u_bar|| its l2_error -- bit for bit."""
    m = O.build_structured_cube(8)
    s = O.build_system(m, 1e-2, "smooth")
    u = O.solve_system_amg(s, 1e-8).u
    l2, h1 = O.error_norms_target(m, s, u, "smooth", 8, 0)
    assert h1 == O.h1_semi_error_manufactured(m, s, u, 0.0)
    assert l2 == O.l2_error_manufactured(m, s, u, 0.0)


def test_error_norms_target_zero_field(O):
    """Against the zero field the gates are the target's own norms: ||grad sin^3||_L2 =
    pi sqrt(3/8) on the unit cube (degree-5 rule, so to quadrature accuracy), and the sine+random
    target's differs by its random part's gradient."""
    n = 8
    m = O.build_structured_cube(n)
    s_smooth = O.build_system(m, 1.0, "smooth")
    l2s, h1s = O.error_norms_target(m, s_smooth, np.zeros(s_smooth.n_dofs), "smooth", n, 0)
    assert abs(h1s - math.pi * math.sqrt(3.0 / 8.0)) < 1e-6
    assert abs(l2s - math.sqrt(1.0 / 8.0)) < 1e-6
    s = O.build_system(m, 1.0, "sine_random")
    l2z, h1z = O.error_norms_target(m, s, np.zeros(s.n_dofs), "sine_random", n, 0)
    assert h1z > 0 and abs(h1z - h1s) > 1e-3
