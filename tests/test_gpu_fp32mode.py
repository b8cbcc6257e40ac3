"""The fp32 mode (FistaOptions(fp32_forward=True), fp32 X on the single-pass
kernel: X beta with fp32 products and fp64 reductions, the logistic loss in
single precision in the gather) against the fp64 oracle at the north star's
fp32-mode tolerance 1e-5, on ragged shapes (rows not a multiple of the
4-row tile, column slices with padding), node mode, squared hinge, and the
exact mode as the control (1e-9 there)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _instance(engine, rng, n, p, loss, k, M, lam2):
    X = rng.standard_normal((n, p)).astype(np.float32)
    if loss == "squared_error":
        b = np.zeros(p)
        b[:: max(1, p // k)][:k] = 1.0
        y = X.astype(np.float64) @ b + 0.5 * rng.standard_normal(n)
    else:
        y = rng.choice([-1.0, 1.0], n)
    inst = engine.ProblemInstance(X, y, engine.LossKind(loss), k, M, lam2, dtype="fp32")
    L = engine.lipschitz_constant(inst, method="lanczos")
    return X, y, inst, L


@pytest.mark.parametrize("n,p,loss,node", [
    (1001, 700, "squared_error", False),
    (4003, 2500, "logistic", False),
    (2999, 3100, "squared_hinge", False),
    (2501, 1800, "squared_error", True),
    (3001, 2200, "logistic", True),
])
def test_fp32_mode_vs_oracle(engine, oracle, n, p, loss, node):
    rng = np.random.default_rng(n + p)
    k, M, lam2 = 8, 2.0, 0.3
    X, y, inst, L = _instance(engine, rng, n, p, loss, k, M, lam2)
    f1, f0 = ((3, 17), (5, 40, 41)) if node else ((), ())
    nd = engine.NodeState(fixed_one=f1, fixed_zero=f0) if node else None
    iters = 30
    ref = oracle.fista(X.astype(np.float64), y, loss, k, M, lam2, L=L, max_iter=iters, gap_tol=1e-300,
                       fixed_one=f1, fixed_zero=f0)
    for fp32_forward, tol in ((False, 1e-9), (True, 1e-5)):
        rep = engine.solve_relaxation(inst, nd, opts=engine.FistaOptions(
            lipschitz=L, max_iterations=iters, gap_tolerance=1e-300, engine_path="single_pass",
            fp32_forward=fp32_forward))
        assert rep.stats["single_pass"] and rep.iterations == iters
        assert rep.primal_value == pytest.approx(ref["primal_value"], rel=tol)
        assert rep.dual_bound == pytest.approx(ref["dual_bound"], rel=max(tol, 1e-9), abs=1e-9)
        scale = max(1.0, float(np.max(np.abs(ref["beta"]))))
        np.testing.assert_allclose(rep.beta, ref["beta"], rtol=0, atol=tol * 10 * scale)
        if node:
            assert np.all(rep.beta[list(f0)] == 0.0)


def test_fp32_mode_is_ignored_for_fp64_x(engine):
    rng = np.random.default_rng(5)
    X = rng.standard_normal((800, 500))
    y = rng.standard_normal(800)
    inst = engine.ProblemInstance(X, y, engine.LossKind.SQUARED_ERROR, 5, 1.0, 0.5)
    L = engine.lipschitz_constant(inst, method="lanczos")
    o = lambda f: engine.FistaOptions(lipschitz=L, max_iterations=20, gap_tolerance=1e-300,
                                      engine_path="single_pass", fp32_forward=f)
    a, b = engine.solve_relaxation(inst, opts=o(False)), engine.solve_relaxation(inst, opts=o(True))
    assert a.primal_value == b.primal_value and np.array_equal(a.beta, b.beta)
