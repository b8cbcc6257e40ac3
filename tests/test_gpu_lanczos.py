"""The package's device Lanczos estimate of lambda_max(X^T X)
(``lipschitz_constant(instance, method="lanczos")``, spectral.py) against
scipy / LAPACK eigenvalues of the same matrices, at 1e-12 relative; the
reference's power iteration (model.py:283-327) stays the default."""

import numpy as np
import pytest

from paper_2502_09502_b200 import data as mydata

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,scale,dtype", [("C1", 1.0, "fp64"), ("C2", 0.25, "fp64"),
                                              ("C3", 0.1, "fp32"), ("C4", 0.5, "fp32")])
def test_lanczos_matches_lapack(engine, name, scale, dtype):
    import scipy.sparse.linalg as sla
    cd = mydata.make_config(name, scale=scale)
    inst = engine.ProblemInstance(cd.X, cd.y, engine.LossKind(cd.loss), cd.k, cd.M, cd.lambda2,
                                  dtype=dtype)
    X = np.asarray(cd.X, dtype=np.float64)
    G = X.T @ X
    if cd.p <= 5000:
        lam_ref = float(np.linalg.eigvalsh(G)[-1])
    else:
        lam_ref = float(sla.eigsh(G, k=1, which="LA", tol=1e-15, return_eigenvectors=False)[0])
    from paper_2502_09502_b200.model import lanczos_lambda_max
    lam = lanczos_lambda_max(inst)
    assert lam == pytest.approx(lam_ref, rel=1e-12)
    curv = {"squared_error": 2.0, "logistic": 0.25}[cd.loss]
    assert engine.lipschitz_constant(inst, method="lanczos") == pytest.approx(curv * lam * 1.01,
                                                                              rel=1e-15)


def test_lanczos_zero_matrix_and_power_default(engine):
    X = np.zeros((50, 20))
    inst = engine.ProblemInstance(X, np.zeros(50), engine.LossKind.SQUARED_ERROR, 3, 1.0, 1.0)
    assert engine.lipschitz_constant(inst, method="lanczos") == 0.0
    with pytest.raises(engine.InvalidInputError):
        engine.lipschitz_constant(inst, method="bogus")
    # the reference clamps L = max(L, 1e-12) (fista.py:101): an all-zero X solves
    rep = engine.solve_relaxation(inst, opts=engine.FistaOptions(max_iterations=5))
    assert np.all(rep.beta == 0.0)
    assert rep.primal_value == 0.0
