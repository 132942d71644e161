"""The operator-callback PCG (rd::LinOp, linalg.hpp:11, 39-49; amg.hpp:42) on the device.

rd_gpu_pcg_linop takes any pair of rd_linop operators.  Built-ins (spmv(A, .), amg_precond,
jacobi_precond, identity_precond) run fused; anything else goes through its callback.  Bars:
  * built-in A + amg_precond / identity: bit-identical to rd_gpu_pcg (the same kernels);
  * jacobi_precond: the reference's hand cases (test_linalg.cpp:106-159) and the oracle's
    Jacobi PCG (iterations equal, solution and history within 1e-10);
  * callbacks: the same iterations as the fused path, solutions within 1e-10 (the dot after a
    callback reduces in another deterministic order than the fused SpMV epilogue);
  * errors: a non-positive diagonal and a failing callback raise, like the reference.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rd():
    from paper_2102_03515_b200 import rd as _rd

    _rd.default_context()
    return _rd


def band_triplets(n):  # test_linalg.cpp:19-34
    t = []
    for i in range(n):
        t.append((i, i, 4.0 + 0.01 * i))
        if i + 1 < n:
            t += [(i, i + 1, -1.0), (i + 1, i, -1.0)]
        if i + 3 < n:
            t += [(i, i + 3, -0.5), (i + 3, i, -0.5)]
    return t


@pytest.mark.parametrize("n,rho,target", [(8, 1.0, "ball"), (16, 2.0 ** -8, "smooth"), (33, 1e-2, "sine_random")])
def test_linop_amg_matches_pcg(rd, n, rho, target):
    """pcg(sys.A, amg_precond(h), sys.f, tol, 500) (bench.cpp:218) through LinOps == rd_gpu_pcg."""
    s = rd.build_system(rd.build_structured_cube(n), rho, target)
    h = rd.build_amg(s.A)
    f = s.f()
    ref = rd.pcg(s.A, "amg", f, 1e-8, 500, hierarchy=h)
    out = rd.pcg_linop(s.A, rd.amg_precond(h), f, 1e-8, 500)
    assert out.converged and out.iterations == ref.iterations
    assert np.array_equal(out.x, ref.x)
    assert np.array_equal(out.residual_history, ref.residual_history)
    out2 = rd.pcg_linop(rd.spmv_op(s.A), rd.amg_precond(h), f, 1e-8, 500)
    assert np.array_equal(out2.x, ref.x)
    ident = rd.pcg(s.A, "identity", f, 1e-8, 500)
    out3 = rd.pcg_linop(s.A, rd.identity_precond(), f, 1e-8, 500)
    assert out3.iterations == ident.iterations and np.array_equal(out3.x, ident.x)


def test_jacobi_hand_cases(rd, O):  # test_linalg.cpp:106-116, 141-159
    A = rd.from_triplets(40, 40, band_triplets(40))
    f = O.pseudo_random_vec(40, 3)
    r = rd.pcg_linop(A, rd.jacobi_precond(A), f, 1e-12, 200)
    dense = np.zeros((40, 40))
    for i, j, v in band_triplets(40):
        dense[i, j] += v
    assert r.converged and np.abs(r.x - np.linalg.solve(dense, f)).max() < 1e-9
    assert len(r.residual_history) == r.iterations and r.residual_history[-1] <= 1e-12
    oa = O.from_triplets(40, 40, band_triplets(40))
    ref = O.pcg(oa, "jacobi", f, 1e-12, 200)
    assert r.iterations == ref.iterations
    assert np.abs(r.x - ref.x).max() <= 1e-10 * np.abs(ref.x).max()
    assert np.allclose(r.residual_history, ref.residual_history, rtol=1e-10, atol=0)
    # symmetric permutation invariance
    n = 12
    perm = [(5 * i + 3) % n for i in range(n)]
    t = band_triplets(n)
    A = rd.from_triplets(n, n, t)
    B = rd.from_triplets(n, n, [(perm[i], perm[j], v) for i, j, v in t])
    f = O.pseudo_random_vec(n, 11)
    g = np.zeros(n)
    for i in range(n):
        g[perm[i]] = f[i]
    x = rd.pcg(A, "jacobi", f, 1e-13, 100).x
    y = rd.pcg(B, "jacobi", g, 1e-13, 100).x
    for i in range(n):
        assert y[perm[i]] == pytest.approx(x[i], rel=1e-8)


@pytest.mark.parametrize("n,rho,target", [(8, 1.0, "smooth"), (16, 2.0 ** -8, "ball")])
def test_jacobi_system_parity(rd, O, n, rho, target):
    """bench.cpp:205-207 (PrecondKind::jacobi) against the oracle's Jacobi PCG."""
    ds = rd.build_system(rd.build_structured_cube(n), rho, target)
    os_ = O.build_system(O.build_structured_cube(n), rho, target)
    r = rd.pcg(ds.A, "jacobi", ds.f(), 1e-8, 500)
    ref = O.pcg(os_.A, "jacobi", os_.f, 1e-8, 500)
    assert r.converged and r.iterations == ref.iterations
    assert np.abs(r.x - ref.x).max() <= 1e-10 * np.abs(ref.x).max()
    # the preconditioner alone is r ./ diag(A), exactly
    d = ref_diag(os_.A)
    v = O.pseudo_random_vec(os_.A.rows, 5)
    assert np.array_equal(rd.jacobi_precond(ds.A)(v), v / d)


def ref_diag(A):
    d = np.zeros(A.rows)
    for i in range(A.rows):
        for k in range(A.rp[i], A.rp[i + 1]):
            if A.ci[k] == i:
                d[i] = A.v[k]
    return d


def test_jacobi_rejects_nonpositive_diagonal(rd):  # linalg.cpp:57-61
    with pytest.raises(rd.RdNotSpdError):
        rd.jacobi_precond(rd.from_triplets(2, 2, [(0, 0, 1.0), (1, 1, -1.0)]))
    with pytest.raises(rd.RdNotSpdError):  # a missing diagonal entry reads as 0
        rd.jacobi_precond(rd.from_triplets(2, 2, [(0, 0, 1.0), (0, 1, 0.5), (1, 0, 0.5)]))


def test_callback_operators(rd):
    """A user LinOp (a Python callable on device tensors) as the operator and as the
    preconditioner: the loop calls it through the C ABI on the context's stream."""
    from paper_2102_03515_b200.rd import lib

    s = rd.build_system(rd.build_structured_cube(16), 2.0 ** -8, "ball")
    h = rd.build_amg(s.A)
    f = s.f()
    ref = rd.pcg(s.A, "amg", f, 1e-8, 500, hierarchy=h)
    ctx = s.A.ctx
    calls = {"A": 0, "P": 0}

    def apply_A(x, y):
        calls["A"] += 1
        ctx.check(lib().rd_gpu_spmv(ctx.h, s.A.h, x.data_ptr(), y.data_ptr()))

    def apply_P(x, y):
        calls["P"] += 1
        ctx.check(lib().rd_gpu_amg_apply(h.h, x.data_ptr(), y.data_ptr()))

    A_op = rd.LinOp.from_device_fn(apply_A, ctx)
    P_op = rd.LinOp.from_device_fn(apply_P, ctx)
    out = rd.pcg_linop(A_op, P_op, f, 1e-8, 500, ctx=ctx)
    assert out.converged and out.iterations == ref.iterations
    assert np.abs(out.x - ref.x).max() <= 1e-10 * np.abs(ref.x).max()
    assert calls["P"] >= ref.iterations + 1 and calls["A"] >= ref.iterations
    # a callback error surfaces as the call's error
    def broken(x, y):
        raise ValueError("boom")

    with pytest.raises(rd.RdError):
        rd.pcg_linop(rd.LinOp.from_device_fn(broken, ctx), P_op, f, 1e-8, 500, ctx=ctx)
    # and an operator applied on its own
    v = np.linspace(-1.0, 1.0, s.A.rows)
    assert np.array_equal(rd.spmv_op(s.A)(v), rd.spmv(s.A, v))
    assert np.array_equal(rd.amg_precond(h)(v), h.apply(v))
