"""§8(f)4 BDDC on the B200 (paper_2102_03515_b200/csrc/bddc.cu) against the oracle restatement
(oracle/rd_oracle.cpp, pinned by the reference's test_bddc.cpp in test_oracle_bddc.py).

Bars: the partition, interface set and primal count exactly (integer work); the operators
(schur_apply, reduce_rhs, expand_solution, bddc_apply, the coarse matrix) within 1e-10 relative
(the local factorizations are cuSOLVER's, the oracle's are dense left-looking ones -- both
differ in order from Eigen's, so this row is pinned to rounding); bddc_solve: iteration counts
equal, solutions within 1e-8.  Plus the reference's own properties on the device."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rd():
    from paper_2102_03515_b200 import rd as _rd

    _rd.default_context()
    return _rd


def both(rd, O, n, rho, target="smooth"):
    dm, om = rd.build_structured_cube(n), O.build_structured_cube(n)
    return dm, om, rd.build_system(dm, rho, target), O.build_system(om, rho, target)


@pytest.mark.parametrize("n,p", [(4, 2), (4, 4), (4, 8), (6, 3), (6, 8), (8, 5)])
def test_partition_and_interface(rd, O, n, p):
    dm, om, ds, os_ = both(rd, O, n, 0.1)
    owner_d = rd.partition_geometric(ds, p)
    owner_o, _ = O.partition_geometric(om, os_, p)
    assert np.array_equal(owner_d, owner_o)
    bd, bo = rd.Bddc(ds, p), O.Bddc(om, os_, p)
    assert np.array_equal(bd.interface_dofs, bo.interface_dofs) and bd.n_primal == bo.n_primal


@pytest.mark.parametrize("n,p,rho", [(4, 2, 0.05), (4, 4, 1e-2), (6, 8, 1e-4), (8, 4, 1.0)])
def test_operators_match_oracle(rd, O, n, p, rho):
    dm, om, ds, os_ = both(rd, O, n, rho)
    bd, bo = rd.Bddc(ds, p), O.Bddc(om, os_, p)
    nc = bd.n_interface
    rel = lambda a, b: np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)  # noqa: E731
    cm_d, cm_o = bd.coarse_matrix(), bo.coarse_matrix()
    assert cm_d.shape == cm_o.shape and (cm_o.size == 0 or rel(cm_d, cm_o) < 1e-10)
    for k in range(3):
        x = O.pseudo_random_vec(nc, 11 + k)
        assert rel(bd.schur_apply(x), bo.schur_apply(x)) < 1e-10
        assert rel(bd.apply(x), bo.apply(x)) < 1e-10
    assert rel(bd.reduce_rhs(os_.f), bo.reduce_rhs(os_.f)) < 1e-10
    uC = O.pseudo_random_vec(nc, 7)
    assert rel(bd.expand_solution(uC, os_.f), bo.expand_solution(uC, os_.f)) < 1e-10


def test_schur_matches_dense_elimination(rd, O):  # test_bddc.cpp:112-123 on the device
    dm, om, ds, os_ = both(rd, O, 4, 0.05)
    bd = rd.Bddc(ds, 2)
    A = os_.A.dense()
    iface = set(int(d) for d in bd.interface_dofs)
    interior = [d for d in range(A.shape[0]) if d not in iface]
    Cd = list(bd.interface_dofs)
    S = A[np.ix_(Cd, Cd)] - A[np.ix_(Cd, interior)] @ np.linalg.solve(A[np.ix_(interior, interior)],
                                                                     A[np.ix_(interior, Cd)])
    for k in range(3):
        x = O.pseudo_random_vec(bd.n_interface, 31 + k)
        assert np.abs(bd.schur_apply(x) - S @ x).max() < 1e-10
    assert np.linalg.norm(bd.schur_apply(np.zeros(bd.n_interface))) == 0.0


def test_preconditioner_symmetric_positive(rd, O):  # test_bddc.cpp:202-214
    dm, om, ds, os_ = both(rd, O, 4, 1e-4)
    bd = rd.Bddc(ds, 4)
    for k in range(3):
        r1 = O.pseudo_random_vec(bd.n_interface, 300 + k)
        r2 = O.pseudo_random_vec(bd.n_interface, 400 + k)
        assert r2 @ bd.apply(r1) == pytest.approx(r1 @ bd.apply(r2), rel=1e-10)
        assert r1 @ bd.apply(r1) > 0.0


@pytest.mark.parametrize("n,p,rho", [(4, 2, 1.0), (4, 4, 1e-6), (8, 4, 1e-2), (8, 8, 1e-4), (12, 8, 2.0 ** -7),
                                     (16, 8, 1.0)])
def test_bddc_solve_matches_oracle(rd, O, n, p, rho):
    dm, om, ds, os_ = both(rd, O, n, rho)
    r = rd.bddc_solve(ds, p, 1e-8, 500)
    ref = O.bddc_solve(om, os_, p, 1e-8, 500)
    assert r.converged and ref.converged and r.iterations == ref.iterations
    assert np.abs(r.x - ref.x).max() <= 1e-8 * np.abs(ref.x).max()
    # (histories agree to 1e-6 relative above the rounding floor, where they are noise)
    assert np.allclose(r.residual_history, ref.residual_history, rtol=1e-6, atol=1e-13)


def test_pipeline_without_interface(rd):  # test_bddc.cpp:245-253
    ds = rd.build_system(rd.build_structured_cube(2), 0.1, "smooth")
    r = rd.bddc_solve(ds, 2, 1e-10, 50)
    u = rd.solve_system_amg(ds.A, ds.f(), 1e-12).u
    assert np.abs(r.x - u).max() < 1e-9


def test_bddc_linops_in_pcg(rd, O):
    """pcg(schur_op(op), bddc_precond(op), g) through the LinOp C-ABI (bddc.cpp:449)."""
    dm, om, ds, os_ = both(rd, O, 8, 1e-2)
    bd = rd.Bddc(ds, 4)
    g = bd.reduce_rhs(os_.f)
    res = rd.pcg_linop(bd.schur_op(), bd.precond(), g, 1e-8, 500, ctx=ds.ctx)
    ref = rd.bddc_solve(ds, 4, 1e-8, 500)
    assert res.iterations == ref.iterations
    u = bd.expand_solution(res.x, os_.f)
    assert np.abs(u - ref.x).max() <= 1e-10 * np.abs(ref.x).max()


def test_bddc_rejects(rd):
    ds = rd.build_system(rd.build_structured_cube(2), 0.1, "smooth")
    for p in (1, 10 ** 6):
        with pytest.raises(rd.RdInvalidArgument):
            rd.partition_geometric(ds, p)
