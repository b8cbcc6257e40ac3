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


def logistic_objective(X, y, S, lam2, M):
    """min_b sum log(1 + exp(-y X_S b)) + lam2 |b|^2, |b| <= M (model.py:167-169
    loss; SPEC.md:294-357 node problem) by L-BFGS-B to high accuracy."""
    from scipy.optimize import minimize
    p = X.shape[1]
    if not S:
        return float(np.sum(np.logaddexp(0.0, np.zeros(X.shape[0])))), np.zeros(p)
    Xs = X[:, list(S)]

    def f(b):
        m = -y * (Xs @ b)
        val = np.sum(np.logaddexp(0.0, m)) + lam2 * b @ b
        s = 1.0 / (1.0 + np.exp(-m))
        grad = Xs.T @ (-y * s) + 2.0 * lam2 * b
        return val, grad

    res = minimize(f, np.zeros(len(S)), jac=True, method="L-BFGS-B",
                   bounds=[(-M, M)] * len(S), options={"ftol": 1e-15, "gtol": 1e-12,
                                                       "maxiter": 10000})
    beta = np.zeros(p)
    beta[list(S)] = res.x
    return float(res.fun), beta


def best_subset_logistic(X, y, k, lam2, M):
    """Exact k-sparse logistic optimum by enumeration of supports."""
    p = X.shape[1]
    best = (np.inf, None, None)
    for m in range(0, k + 1):
        for S in itertools.combinations(range(p), m):
            obj, beta = logistic_objective(X, y, S, lam2, M)
            if obj < best[0] - 1e-12:
                best = (obj, beta, tuple(S))
    return best
