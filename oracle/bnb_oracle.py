"""Enumeration oracle for the branch-and-bound module.

TEST INFRASTRUCTURE ONLY: used by tests/ to check certify / beam search
against the exact k-sparse optimum on small instances; never imported by the
engine.  Parity is anchored on the spec's own examples.

Squared-error loss, box |b| <= M assumed inactive at the ridge solution
(checked): the optimum over a support S is the ridge solution
(X_S^T X_S + lambda2 I) b = X_S^T y.
"""

import itertools

import numpy as np


def ridge_objective(X, y, S, lam2):
    if not S:
        return float(y @ y), np.zeros(X.shape[1])
    Xs = X[:, list(S)]
    b = np.linalg.solve(Xs.T @ Xs + lam2 * np.eye(len(S)), Xs.T @ y)
    r = Xs @ b - y
    beta = np.zeros(X.shape[1])
    beta[list(S)] = b
    return float(r @ r + lam2 * b @ b), beta


def best_subset(X, y, k, lam2, M=np.inf, fixed_one=(), fixed_zero=()):
    """Exact min ||X b - y||^2 + lam2 ||b||^2 over ||b||_0 <= k (ridge per
    support; raises if the box binds).  Returns (objective, beta, support)."""
    p = X.shape[1]
    free = [j for j in range(p) if j not in set(fixed_one) | set(fixed_zero)]
    best = (np.inf, None, None)
    for m in range(0, k - len(fixed_one) + 1):
        for extra in itertools.combinations(free, m):
            S = tuple(sorted(tuple(fixed_one) + extra))
            obj, beta = ridge_objective(X, y, S, lam2)
            if np.max(np.abs(beta), initial=0.0) > M:
                raise ValueError("box constraint binds; oracle assumes it inactive")
            if obj < best[0] - 1e-12:
                best = (obj, beta, S)
    return best
