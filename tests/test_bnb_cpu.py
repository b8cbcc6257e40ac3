"""Host-side logic of the branch-and-bound module and its enumeration oracle
(no GPU): cadence rules, leaf detection, the oracle against brute force."""

import itertools

import numpy as np

from oracle.bnb_oracle import best_subset, ridge_objective


def test_beam_cadence_matches_spec():
    # every node at depth <= 3, then every 5th depth
    from paper_2502_09502_b200.bnb import _beam_due
    assert [d for d in range(12) if _beam_due(d)] == [0, 1, 2, 3, 5, 10]


def test_leaf_detection():
    from paper_2502_09502_b200.bnb import _is_leaf
    from paper_2502_09502_b200.model import NodeState

    class Inst:
        k, p = 2, 4
    assert _is_leaf(Inst, NodeState(fixed_one=(0, 1)))
    assert _is_leaf(Inst, NodeState(fixed_one=(0,), fixed_zero=(1, 2, 3)))
    assert not _is_leaf(Inst, NodeState(fixed_one=(0,), fixed_zero=(1,)))


def test_oracle_spec_examples():
    # X = I2, y = (3, 1), lambda2 = 1, k = 1 -> support {first}, 1.5, 5.5
    obj, beta, S = best_subset(np.eye(2), np.array([3.0, 1.0]), 1, 1.0, 10.0)
    assert S == (0,) and abs(beta[0] - 1.5) < 1e-12 and abs(obj - 5.5) < 1e-12
    # X = [[1]], y = (1), k = 1, lambda2 = 1 -> 0.5
    obj, _, _ = best_subset(np.array([[1.0]]), np.array([1.0]), 1, 1.0, 2.0)
    assert abs(obj - 0.5) < 1e-12


def test_oracle_against_brute_force_grid():
    """The ridge-per-support oracle equals a brute-force minimisation over
    supports with a dense coefficient grid search refinement (tiny case)."""
    rng = np.random.default_rng(0)
    X = rng.standard_normal((12, 4))
    y = rng.standard_normal(12)
    obj, beta, S = best_subset(X, y, 2, 0.5)
    for m in range(3):
        for sup in itertools.combinations(range(4), m):
            o, b = ridge_objective(X, y, sup, 0.5)
            assert o >= obj - 1e-12
            # stationarity of the per-support ridge solution
            if sup:
                Xs = X[:, list(sup)]
                g = 2 * Xs.T @ (Xs @ b[list(sup)] - y) + 2 * 0.5 * b[list(sup)]
                assert np.max(np.abs(g)) < 1e-9
