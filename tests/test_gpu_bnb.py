"""Branch-and-bound on the batched engine vs the spec's examples and an
enumeration oracle (oracle/bnb_oracle.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inst(X, y, k, M, lam2):
    from paper_2502_09502_b200 import LossKind, ProblemInstance
    return ProblemInstance(np.asarray(X, dtype=np.float64), np.asarray(y, dtype=np.float64),
                           LossKind.SQUARED_ERROR, k, M, lam2)


def test_beam_search_spec_example():
    # X = I2, y = (3, 1), lambda2 = 1, M = 10, k = 1 -> support {first}, 1.5, 5.5
    from paper_2502_09502_b200.bnb import beam_search_incumbent
    beta, obj = beam_search_incumbent(_inst(np.eye(2), [3.0, 1.0], 1, 10.0, 1.0), beam_width=2)
    assert np.flatnonzero(beta).tolist() == [0]
    assert beta[0] == pytest.approx(1.5, rel=1e-9)
    assert obj == pytest.approx(5.5, rel=1e-9)


def test_branching_spec_example():
    # incumbent (1.5, 0.5), k = 2 -> the first coordinate
    from paper_2502_09502_b200.bnb import select_branching_variable
    from paper_2502_09502_b200 import NodeState
    inst = _inst(np.eye(2), [3.0, 1.0], 2, 10.0, 1.0)
    assert select_branching_variable(inst, None, np.array([1.5, 0.5])) == 0
    assert select_branching_variable(inst, NodeState(fixed_one=(0, 1)), np.array([1.5, 0.5])) is None


def test_certify_one_dimensional():
    # X = [[1]], y = (1), k = 1, M = 2, lambda2 = 1 -> optimal 0.5, one node
    from paper_2502_09502_b200.bnb import CertificateStatus, certify
    cert = certify(_inst([[1.0]], [1.0], 1, 2.0, 1.0))
    assert cert.status is CertificateStatus.OPTIMAL
    assert cert.incumbent_objective == pytest.approx(0.5, rel=1e-9)
    assert cert.nodes_explored == 1
    assert cert.global_lower_bound <= cert.incumbent_objective + 1e-9


def test_certify_k_equals_p_is_one_node():
    # k = p, M large -> the root relaxation is integral
    from paper_2502_09502_b200.bnb import CertificateStatus, certify
    rng = np.random.default_rng(5)
    X = rng.standard_normal((30, 6))
    y = X @ rng.standard_normal(6) + 0.1 * rng.standard_normal(30)
    cert = certify(_inst(X, y, 6, 100.0, 0.5))
    assert cert.status is CertificateStatus.OPTIMAL
    assert cert.nodes_explored == 1


@pytest.mark.parametrize("seed", range(20))
def test_certify_matches_enumeration(seed):
    # 20 random instances p=8, n=20, k=2 -> enumeration optimum, Optimal
    from oracle.bnb_oracle import best_subset
    from paper_2502_09502_b200.bnb import BnBOptions, CertificateStatus, certify
    rng = np.random.default_rng(100 + seed)
    X = rng.standard_normal((20, 8))
    bt = np.zeros(8)
    bt[rng.choice(8, 2, replace=False)] = rng.choice([-1.0, 1.0], 2) * rng.uniform(0.5, 1.5, 2)
    y = X @ bt + 0.3 * rng.standard_normal(20)
    k, M, lam2 = 2, 20.0, 0.3
    obj, beta, S = best_subset(X, y, k, lam2, M)
    cert = certify(_inst(X, y, k, M, lam2), BnBOptions(gap_tolerance=1e-7, batch_size=8))
    assert cert.status is CertificateStatus.OPTIMAL
    assert cert.incumbent_objective == pytest.approx(obj, rel=1e-7, abs=1e-9)
    assert tuple(np.flatnonzero(np.abs(cert.incumbent_beta) > 1e-9)) == S
    # soundness: the certified bound never exceeds the true optimum
    assert cert.global_lower_bound <= obj + 1e-7 * abs(obj)


@pytest.mark.parametrize("seed", range(4))
def test_certify_logistic_matches_enumeration(seed):
    """Logistic loss: leaf and node refits are iterative (no closed form), so
    the certificate must stay sound when a refit is inexact: the
    certified bound never exceeds the enumeration optimum, and an OPTIMAL
    status comes with the optimal objective."""
    from oracle.bnb_oracle import best_subset_logistic
    from paper_2502_09502_b200 import LossKind, ProblemInstance
    from paper_2502_09502_b200.bnb import BnBOptions, CertificateStatus, certify
    rng = np.random.default_rng(300 + seed)
    X = rng.standard_normal((40, 7))
    bt = np.zeros(7)
    bt[rng.choice(7, 2, replace=False)] = rng.choice([-1.0, 1.0], 2) * 1.5
    y = np.where(rng.random(40) < 1.0 / (1.0 + np.exp(-(X @ bt))), 1.0, -1.0)
    k, M, lam2 = 2, 3.0, 0.2
    obj, beta, S = best_subset_logistic(X, y, k, lam2, M)
    inst = ProblemInstance(X, y, LossKind.LOGISTIC, k, M, lam2)
    cert = certify(inst, BnBOptions(gap_tolerance=1e-6, batch_size=8))
    assert cert.global_lower_bound <= obj + 1e-7 * abs(obj)
    assert cert.incumbent_objective >= obj - 1e-7 * abs(obj)     # a feasible point
    if cert.status is CertificateStatus.OPTIMAL:
        assert cert.incumbent_objective == pytest.approx(obj, rel=1e-5)
    assert cert.status in (CertificateStatus.OPTIMAL, CertificateStatus.GAP_LIMIT)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_refit_ridge_kernel_matches_numpy(dtype):
    """l0_refit_ridge (csrc/refit.cu): batched exact ridge refits on supports
    of mixed sizes (1..48, padded), vs numpy's solve on the same (fp64-upcast)
    columns; objectives |y - X_S b|^2 + l2 |b|^2 at 1e-10."""
    import numpy as np
    from paper_2502_09502_b200 import LossKind, ProblemInstance
    from paper_2502_09502_b200.bnb import _refit
    rng = np.random.default_rng(7)
    n, p, lam2 = 700, 120, 0.37
    X = rng.standard_normal((n, p))
    if dtype == "fp32":
        X = X.astype(np.float32)
    y = rng.standard_normal(n) * 3.0
    inst = ProblemInstance(X, y, LossKind.SQUARED_ERROR, 48, 1e6, lam2, dtype=dtype)
    sizes = [1, 2, 5, 8, 13, 31, 48, 0, 7]
    supports = [tuple(sorted(rng.choice(p, size=k, replace=False).tolist())) for k in sizes]
    betas, objs = _refit(inst, supports, 10)
    X64 = X.astype(np.float64)
    for S, beta, obj in zip(supports, betas, objs):
        XS = X64[:, list(S)]
        b = np.linalg.solve(XS.T @ XS + lam2 * np.eye(len(S)), XS.T @ y) if S else np.zeros(0)
        ref = np.zeros(p)
        ref[list(S)] = b
        np.testing.assert_allclose(beta, ref, rtol=1e-9, atol=1e-11)
        r = y - XS @ b
        assert obj == pytest.approx(float(r @ r + lam2 * b @ b), rel=1e-10)
