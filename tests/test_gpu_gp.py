"""GPU: conjugate gradients and the GP posterior mean (csrc/gp.cu) against
the reference's own gp.cpp (oracle/_ref) -- ports of test_gp.cpp:38-189.

Finding (reproduced here with the reference itself on the same inputs): the
reference's monotonicity restart (gp.cpp:100-111: restart from the current
iterate whenever |r| grows) fires on about every other iteration for the
smooth kernels of test_gp.cpp, because CG residuals are not monotone; the
solves then stall (e.g. matern32 N=500: 2000 iterations, 999 restarts,
residual 0.50). Most reference GP tests therefore miss their own assertions.
Each case is ported twice:
  * parity: the default (reference rule) reproduces the reference's
    diagnostics and iterates on the same inputs;
  * intent: restartOnIncrease=False (additive option, textbook CG) meets the
    reference test's own assertions (convergence, 1e-6 vs a direct solve,
    fast vs dense pipeline 1e-4, ...).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cloud(fkt, x):
    return fkt.PointCloud.from_array(x)


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _same_run(res, dr, x_ref, xtol):
    """Same reference-rule trajectory: flags and counts equal (restarts may
    differ by a few roundoff-borderline decisions: the rule compares |r|
    across iterations, and MVMs equal to ~1e-14 flip near-ties), iterates
    close."""
    assert res.diagnostics.converged == dr["converged"]
    assert res.diagnostics.iterations == dr["iterations"]
    assert abs(res.diagnostics.restarts - dr["restarts"]) <= max(3, dr["iterations"] // 100)
    assert _rel(res.x, x_ref) <= xtol


def test_noise_dominated_solve(fkt, ref):  # test_gp.cpp:38-50
    # The zero kernel is a user lambda the GPU path cannot run: a Gaussian on
    # points 1000x apart with K(0) = 0 has off-diagonal values < 1e-40. The
    # reference's "one iteration" claim is false for a diagonal operator with
    # distinct entries (the reference needs 16); with Jacobi it is one.
    x, b = fkt.synthCloud("cube", 50, 2, 10)
    x = x * 1000.0
    noise = 0.5 + 0.01 * np.arange(50)
    op = fkt.NoisyOperator(_cloud(fkt, x), fkt.makeKernel("gaussian"), noise, diagonal=0.0)
    assert op.kernelDiagonal() == 0.0
    res = fkt.cgSolve(op, b, 1e-12, 100)
    xr, dr = ref.cg_solve(x, "gaussian", {}, noise, b, 1e-12, 100, diagonal=0.0)
    assert res.diagnostics.converged and dr["converged"]
    assert abs(res.diagnostics.iterations - dr["iterations"]) <= 1
    np.testing.assert_allclose(res.x, b / noise, rtol=1e-10)
    pre = fkt.cgSolve(op, b, 1e-12, 100, True)
    assert pre.diagnostics.converged and pre.diagnostics.iterations == 1
    np.testing.assert_allclose(pre.x, b / noise, rtol=1e-12)


def test_zero_rhs_returns_zero(fkt):  # :52-61
    x = fkt.synthCloud("cube", 20, 2, 11, with_weights=False)
    op = fkt.NoisyOperator(_cloud(fkt, x), fkt.makeKernel("gaussian"), np.full(20, 0.1))
    for restart in (True, False):
        res = fkt.cgSolve(op, np.zeros(20), 1e-10, 50, restartOnIncrease=restart)
        assert res.diagnostics.converged and res.diagnostics.iterations == 0 and np.all(res.x == 0.0)


def test_cg_dense_system(fkt, ref):  # :63-85
    x, b = fkt.synthCloud("cube", 500, 3, 12)
    k = fkt.makeKernel("matern32")
    noise = np.full(500, 0.01)
    op = fkt.NoisyOperator(_cloud(fkt, x), k, noise)
    # parity with the reference rule (which stalls here)
    res = fkt.cgSolve(op, b, 1e-10, 2000)
    xr, dr = ref.cg_solve(x, "matern32", {}, noise, b, 1e-10, 2000)
    _same_run(res, dr, xr, 1e-3)
    # the test's intent with textbook CG
    cg = fkt.cgSolve(op, b, 1e-10, 2000, restartOnIncrease=False)
    assert cg.diagnostics.converged and cg.diagnostics.finalResidual <= 1e-10 and cg.diagnostics.restarts == 0
    r = np.sqrt(((x[:, None, :] - x[None, :, :]) ** 2).sum(-1))
    A = k(r.ravel()).reshape(500, 500) + np.diag(noise)
    assert _rel(cg.x, np.linalg.solve(A, b)) < 1e-6


def test_cg_flags_non_convergence(fkt, ref):  # :87-97
    x, b = fkt.synthCloud("cube", 200, 2, 13)
    noise = np.full(200, 1e-12)
    res = fkt.cgSolve(fkt.NoisyOperator(_cloud(fkt, x), fkt.makeKernel("gaussian"), noise), b, 1e-14, 3)
    assert not res.diagnostics.converged and res.diagnostics.iterations <= 3
    _, dr = ref.cg_solve(x, "gaussian", {}, noise, b, 1e-14, 3)
    assert dr["iterations"] == res.diagnostics.iterations and not dr["converged"]
    assert res.diagnostics.restarts == dr["restarts"]


def test_jacobi_preconditioning(fkt, ref):  # :99-113
    x, b = fkt.synthCloud("cube", 300, 2, 14)
    noise = 0.05 * (1.0 + (np.arange(300) % 7))
    op = fkt.NoisyOperator(_cloud(fkt, x), fkt.makeKernel("exponential"), noise)
    for jac in (False, True):
        res = fkt.cgSolve(op, b, 1e-10, 2000, jac)
        xr, dr = ref.cg_solve(x, "exponential", {}, noise, b, 1e-10, 2000, jacobi=jac)
        _same_run(res, dr, xr, 1e-3)
    plain = fkt.cgSolve(op, b, 1e-10, 2000, False, restartOnIncrease=False)
    pre = fkt.cgSolve(op, b, 1e-10, 2000, True, restartOnIncrease=False)
    assert plain.diagnostics.converged and pre.diagnostics.converged
    assert pre.diagnostics.iterations <= plain.diagnostics.iterations
    np.testing.assert_allclose(pre.x, plain.x, rtol=1e-6, atol=1e-8 * np.abs(plain.x).max())


def test_gp_constant_targets(fkt, ref):  # :115-123
    train = fkt.synthCloud("cube", 200, 2, 15, with_weights=False)
    test = fkt.synthCloud("cube", 60, 2, 115, with_weights=False)
    pred = fkt.gpPosteriorMean(_cloud(fkt, train), np.full(200, 3.25), np.full(200, 0.1), fkt.makeKernel("matern32"),
                               _cloud(fkt, test))
    np.testing.assert_allclose(pred.mean, 3.25, rtol=1e-10)
    assert pred.diagnostics.iterations == 0 and pred.diagnostics.converged
    mr, _ = ref.gp_posterior_mean(train, np.full(200, 3.25), np.full(200, 0.1), "matern32", {}, test)
    assert np.array_equal(pred.mean, mr)


def test_gp_interpolates_coincident_points(fkt, ref):  # :125-139
    train = fkt.synthCloud("cube", 120, 2, 16, with_weights=False)
    test = train[7:8].copy()
    y = np.sin(3.0 * train[:, 0])
    noise = np.full(120, 1e-8)
    k = fkt.makeKernel("matern32")
    pred = fkt.gpPosteriorMean(_cloud(fkt, train), y, noise, k, _cloud(fkt, test),
                               fkt.GpOptions(cgTolerance=1e-12, cgMaxIterations=5000))
    mr, dr = ref.gp_posterior_mean(train, y, noise, "matern32", {}, test, tol=1e-12, maxit=5000)
    assert pred.diagnostics.converged == dr["converged"] and pred.diagnostics.iterations == dr["iterations"]
    assert abs(pred.mean[0] - mr[0]) <= 1e-3 * abs(mr[0])
    cg = fkt.gpPosteriorMean(_cloud(fkt, train), y, noise, k, _cloud(fkt, test),
                             fkt.GpOptions(cgTolerance=1e-12, cgMaxIterations=5000, restartOnIncrease=False))
    assert abs(cg.mean[0] - y[7]) <= 1e-4 * abs(y[7])


def test_fast_pipeline_and_dense_pipeline(fkt, ref):  # :141-173
    rng = np.random.default_rng(17)
    train = fkt.synthCloud("cube", 900, 2, 17, with_weights=False)
    test = fkt.synthCloud("cube", 400, 2, 117, with_weights=False)
    y = np.sin(4.0 * train[:, 0]) * np.cos(2.0 * train[:, 1]) + 0.05 * rng.standard_normal(900)
    noise = np.full(900, 0.01)
    k = fkt.makeKernel("matern32")

    def opts(dense, restart):
        return fkt.GpOptions(fkt=fkt.FktOptions(p=6, leafCapacity=256), cgTolerance=1e-10, cgMaxIterations=4000,
                             dense=dense, restartOnIncrease=restart)

    # parity with the reference's (stalled) pipelines
    for dense in (False, True):
        p = fkt.gpPosteriorMean(_cloud(fkt, train), y, noise, k, _cloud(fkt, test), opts(dense, True))
        mr, dr = ref.gp_posterior_mean(train, y, noise, "matern32", {}, test, p=6, leaf=256, tol=1e-10, maxit=4000,
                                       dense=dense)
        assert p.diagnostics.iterations == dr["iterations"] and p.diagnostics.converged == dr["converged"]
        assert _rel(p.mean, mr) <= 1e-3
    # The test's intent with converged CG: the fast pipeline tracks the dense
    # one up to the FKT truncation error amplified by the solve (noise 0.01 ->
    # condition number ~1e5). At p = 6, theta = 0.75 that is ~1e-2, not the
    # test's 1e-4 (the FKT MVM itself is reference-identical, tests/
    # test_gpu_parity.py); raising p / lowering theta closes the gap.
    pd = fkt.gpPosteriorMean(_cloud(fkt, train), y, noise, k, _cloud(fkt, test), opts(True, False))
    pf = fkt.gpPosteriorMean(_cloud(fkt, train), y, noise, k, _cloud(fkt, test), opts(False, False))
    hi = fkt.GpOptions(fkt=fkt.FktOptions(p=12, theta=0.4, leafCapacity=256), cgTolerance=1e-10, cgMaxIterations=4000,
                       restartOnIncrease=False)
    ph = fkt.gpPosteriorMean(_cloud(fkt, train), y, noise, k, _cloud(fkt, test), hi)
    assert pf.diagnostics.converged and pd.diagnostics.converged and ph.diagnostics.converged
    e6, e12 = _rel(pf.mean, pd.mean), _rel(ph.mean, pd.mean)
    assert e6 < 2e-2 and e12 < 1e-4 and e12 < e6 / 10, (e6, e12)


def test_restarts_with_fast_plan(fkt, ref):  # :175-189
    x, b = fkt.synthCloud("sphere", 400, 3, 18)
    noise = np.full(400, 0.05)
    pl = fkt.plan(_cloud(fkt, x), fkt.makeKernel("exponential"), fkt.FktOptions(leafCapacity=64))
    op = fkt.NoisyOperator(pl, noise)
    res = fkt.cgSolve(op, b, 1e-11, 1000)
    xr, dr = ref.cg_solve(x, "exponential", {}, noise, b, 1e-11, 1000, plan={"p": 4, "theta": 0.75, "leaf": 64})
    _same_run(res, dr, xr, 1e-3)
    cg = fkt.cgSolve(op, b, 1e-11, 1000, restartOnIncrease=False)
    assert cg.diagnostics.converged and cg.diagnostics.restarts == 0


def test_gp_errors(fkt):
    x = fkt.synthCloud("cube", 30, 2, 1, with_weights=False)
    k = fkt.makeKernel("matern32")
    with pytest.raises(fkt.DimensionMismatchError):
        fkt.NoisyOperator(_cloud(fkt, x), k, np.ones(29))
    op = fkt.NoisyOperator(_cloud(fkt, x), k, np.ones(30))
    with pytest.raises(fkt.DimensionMismatchError):
        fkt.cgSolve(op, np.ones(31), 1e-10, 10)
    with pytest.raises(fkt.InvalidArgument):
        fkt.cgSolve(op, np.ones(30), 0.0, 10)
    with pytest.raises(fkt.DimensionMismatchError):
        fkt.gpPosteriorMean(_cloud(fkt, x), np.ones(30), np.ones(30), k, _cloud(fkt, np.zeros((4, 3))))
    np.testing.assert_allclose(op.apply(np.ones(30)), fkt.denseMultiply(_cloud(fkt, x), k, np.ones(30)) + 1.0)


def test_device_cg_at_scale(fkt):
    """N = 200k through the FKT plan: textbook device CG converges and its
    solution satisfies the system through an independent plan multiply."""
    x, b = fkt.synthCloud("cube", 200000, 3, 21)
    noise = np.full(200000, 0.5)
    pl = fkt.plan(_cloud(fkt, x), fkt.makeKernel("matern32", {"sigma": 1.0, "rho": 0.05}),
                  fkt.FktOptions(p=6, theta=0.5, leafCapacity=512))
    op = fkt.NoisyOperator(pl, noise)
    res = fkt.cgSolve(op, b, 1e-8, 500, restartOnIncrease=False)
    assert res.diagnostics.converged
    assert _rel(op.apply(res.x), b) <= 2e-8
