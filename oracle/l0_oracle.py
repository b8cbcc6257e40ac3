"""CPU oracle for the dual-bound engine — TEST INFRASTRUCTURE ONLY.

This module is the checker the B200 engine is compared against.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import it; the product package never does.

It restates, function by function, the reference's algorithm for the hot path
(``/root/reference/pkg/src/l0cert``):

=====================  ======================================================
oracle function        reference it follows
=====================  ======================================================
``huber``              prox.py:27-32
``hprox``              prox.py:35-43  (and the inline copies prox.py:70-73, 88-91)
``pava``               prox.py:46-98  (C restatement in oracle/pava.c)
``prox_conj``          prox.py:101-116 (``_prox_gstar_core``)
``prox_g``             prox.py:144-151
``prox_conj_node``     prox.py:166-187
``prox_g_node``        prox.py:190-201
``envelope_free``      perspective.py:76-111 (``_g_value_free``)
``envelope``           perspective.py:114-132 (``g_value``)
``topk_sum``           perspective.py:135-140 (``_topsum``)
``envelope_conj``      perspective.py:143-159 (``g_conjugate``)
``loss_value``         model.py:159-181 (solver-grade branches)
``loss_grad``          model.py:184-205 (solver-grade branches)
``loss_conj_neg``      model.py:221-280 (solver-grade branches)
``lambda_max_power``   model.py:283-306
``lipschitz``          model.py:309-327
``fenchel_bound``      perspective.py:162-190 and fista.py:150-157
``fista``              fista.py:76-222 (``solve_relaxation``)
``pava_closed_form``   SURVEY.md Appendix A.3 — the parallel single-pool
                       characterisation the GPU kernel implements; checked
                       here against ``pava`` so the GPU design is pinned to the
                       reference's sequential sweep.
=====================  ======================================================

Pinning: ``tests/test_oracle_golden.py`` checks every function above against
golden vectors produced by running the reference itself in the build container
(``tests/golden/make_golden.py``) — bitwise where the reference's own arithmetic
order is reproduced (prox, g, losses, the FISTA trajectory at the same BLAS),
otherwise to 1e-13 relative.

Losses are plain strings: ``"squared_error"``, ``"logistic"``,
``"squared_hinge"`` (the reference's ``LossKind`` values).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time
from typing import Callable, Optional, Sequence

import numpy as np
import scipy.special as _scipy_special

SQUARED_ERROR = "squared_error"
LOGISTIC = "logistic"
SQUARED_HINGE = "squared_hinge"
POISSON = "poisson"              # bound-grade (values, conjugates, bounds only)
GAMMA = "gamma"
SOLVER_LOSSES = (SQUARED_ERROR, LOGISTIC, SQUARED_HINGE)

LIPSCHITZ_SAFETY = 1.01          # model.py:32
POWER_TOL = 1e-7                 # model.py:34
POWER_MAX_ITER = 500             # model.py:35
DOMAIN_SLACK = 1e-12             # model.py:39
FEAS_RTOL = 1e-9                 # perspective.py:23
ZERO_ATOL = 1e-9                 # perspective.py:25
CURVATURE = {SQUARED_ERROR: 2.0, LOGISTIC: 0.25, SQUARED_HINGE: 2.0}  # model.py:309-313

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libl0oracle.so")
_lib = None


def build_c_oracle(force: bool = False) -> str:
    """Compile oracle/pava.c (gcc) into oracle/_build/libl0oracle.so."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load_lib():
    global _lib
    if _lib is None:
        try:
            build_c_oracle()
        except Exception:  # gcc missing: the pure-Python sweep below is used
            return None
        lib = ctypes.CDLL(_LIB_PATH)
        lib.l0o_pava.restype = ctypes.c_int64
        lib.l0o_pava.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
            ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
        ]
        _lib = lib
    return _lib


# ----------------------------------------------------------------------------
# scalar Huber pieces
# ----------------------------------------------------------------------------

def huber(x, M):
    """H_M(x) — prox.py:27-32."""
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    res = np.where(a <= M, 0.5 * x * x, M * a - 0.5 * M * M)
    return float(res) if res.ndim == 0 else res


def hprox(x, w, M):
    """argmin_v (v-x)^2/2 + w H_M(v) for x >= 0 — prox.py:35-43."""
    x = np.asarray(x, dtype=np.float64)
    res = np.where(x <= M * (1.0 + w), x / (1.0 + w), x - w * M)
    return float(res) if res.ndim == 0 else res


# ----------------------------------------------------------------------------
# PAVA
# ----------------------------------------------------------------------------

def _pava_python(xs, k, rho, M):
    # pure-Python stack sweep, same arithmetic as oracle/pava.c
    p = len(xs)
    out = np.empty(p)
    wsum, msum, cnt, val, last = [], [], [], [], []
    for j in range(p):
        w = rho if j < k else 0.0
        x = float(xs[j])
        wsum.append(w)
        msum.append(x)
        cnt.append(1.0)
        val.append(x / (1.0 + w) if x <= M * (1.0 + w) else x - w * M)
        last.append(j)
        while len(val) > 1 and val[-1] > val[-2]:
            wsum[-2] += wsum[-1]
            msum[-2] += msum[-1]
            cnt[-2] += cnt[-1]
            last[-2] = last[-1]
            for arr in (wsum, msum, cnt, val, last):
                arr.pop()
            mean = msum[-1] / cnt[-1]
            wavg = wsum[-1] / cnt[-1]
            val[-1] = mean / (1.0 + wavg) if mean <= M * (1.0 + wavg) else mean - wavg * M
    start = 0
    for b, end in enumerate(last):
        out[start:end + 1] = val[b]
        start = end + 1
    return out, np.asarray(last, dtype=np.int64)


def pava(xs, k: int, rho: float, M: float, want_pools: bool = False):
    """Stack PAVA of prox.py:46-98 on magnitudes sorted non-increasingly.

    Returns the pooled values, and with ``want_pools`` also the inclusive end
    index of every pool (the reference's ``last`` stack).
    """
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    p = xs.shape[0]
    lib = _load_lib()
    if lib is None:
        out, ends = _pava_python(xs, k, rho, M)
    else:
        out = np.empty(p)
        ends = np.empty(max(p, 1), dtype=np.int64)
        nb = lib.l0o_pava(xs.ctypes.data, p, int(k), float(rho), float(M),
                          out.ctypes.data, ends.ctypes.data)
        if nb < 0:
            raise MemoryError("oracle PAVA allocation failed")
        ends = ends[:nb].copy()
    return (out, ends) if want_pools else out


def merged_pool(ends) -> Optional[tuple]:
    """The single non-singleton pool (a*, c*) of a PAVA result, or None."""
    start = 0
    found = None
    for end in np.asarray(ends):
        if end > start:
            if found is not None:
                raise AssertionError("more than one merged pool")
            found = (int(start), int(end))
        start = int(end) + 1
    return found


def pava_closed_form(xs, k: int, rho: float, M: float):
    """Parallel single-pool characterisation.

    Head values hprox(x_j, rho, M) (j < k) and tail values x_j (j >= k) are
    each non-increasing, so PAVA merges at most one pool and it straddles
    k-1 | k.  With S(a, c) = sum x_a..x_c and N = c - a + 1 the pool value is
    V(a, c) = hprox(S/N, rho (k-a) / N, M);

      c(a) = smallest c >= k with c = p-1 or x_{c+1} <= V(a, c)
      a*   = largest a <= k-1 with a = 0 or hprox(x_{a-1}) >= V(a, c(a))

    This is the GPU kernel's algorithm, written sequentially.  Sums are taken
    as (head part a..k-1) + (tail prefix k..c), as on the device.
    Returns (values, (a*, c*) or None).
    """
    xs = np.asarray(xs, dtype=np.float64)
    p = xs.shape[0]
    out = xs.copy()
    if k <= 0:
        return out, None
    if k >= p:
        return hprox(xs, rho, M), None
    head_vals = hprox(xs[:k], rho, M)
    out[:k] = head_vals
    if not (xs[k] > head_vals[k - 1]):
        return out, None
    tail_prefix = np.cumsum(xs[k:])              # T[c-k] = x_k + ... + x_c

    def pool_value(a, c, head_sum):
        n_el = float(c - a + 1)
        s = head_sum + tail_prefix[c - k]
        w = (rho * (k - a)) / n_el
        m = s / n_el
        return m / (1.0 + w) if m <= M * (1.0 + w) else m - w * M

    def c_of(a, head_sum):
        lo, hi = k, p - 1                         # predicate monotone in c
        while lo < hi:
            mid = (lo + hi) // 2
            if xs[mid + 1] <= pool_value(a, mid, head_sum):
                hi = mid
            else:
                lo = mid + 1
        return lo

    head_sum = 0.0
    best = None
    for a in range(k - 1, -1, -1):
        head_sum = head_sum + xs[a]
        c = c_of(a, head_sum)
        v = pool_value(a, c, head_sum)
        if a == 0 or head_vals[a - 1] >= v:
            best = (a, c, v)
            break
    a, c, v = best
    out[a:c + 1] = v
    return out, (a, c)


# ----------------------------------------------------------------------------
# prox of rho g* and of g / rho
# ----------------------------------------------------------------------------

def sort_order(mu) -> np.ndarray:
    """Stable descending order of |mu| — prox.py:111."""
    return np.argsort(-np.abs(mu), kind="stable")


def prox_conj(mu, rho: float, k: int, M: float, instrument: bool = False):
    """prox of rho * TopSum_k(H_M(.)) — prox.py:101-116 (``_prox_gstar_core``).

    With ``instrument`` also returns (order, pool) where pool is the merged
    (a*, c*) in sorted positions or None.
    """
    mu = np.asarray(mu, dtype=np.float64)
    p = mu.shape[0]
    if k == 0 or p == 0:
        res = mu.copy()
        return (res, None, None) if instrument else res
    sgn = np.sign(mu)
    mag = np.abs(mu)
    if k >= p:
        res = sgn * hprox(mag, rho, M)
        return (res, None, None) if instrument else res
    order = np.argsort(-mag, kind="stable")
    vals, ends = pava(mag[order], k, rho, M, want_pools=True)
    res = np.empty(p)
    res[order] = vals
    res *= sgn
    if instrument:
        return res, order, merged_pool(ends)
    return res


def prox_g(mu, rho: float, k: int, M: float):
    """prox of g / rho through the extended Moreau identity — prox.py:144-151."""
    mu = np.asarray(mu, dtype=np.float64)
    return mu - prox_conj(rho * mu, rho, k, M) / rho


def prox_conj_node(mu, rho, free, fixed_one, k_rem, M):
    """Node-masked prox of the conjugate — prox.py:166-187 (validated inputs)."""
    mu = np.asarray(mu, dtype=np.float64)
    free = np.asarray(sorted(free), dtype=np.int64)
    fone = np.asarray(sorted(fixed_one), dtype=np.int64)
    res = mu.copy()
    if fone.size:
        part = mu[fone]
        res[fone] = np.sign(part) * hprox(np.abs(part), rho, M)
    if free.size:
        res[free] = prox_conj(mu[free], rho, int(min(k_rem, free.size)), M)
    return res


def prox_g_node(mu, rho, free, fixed_one, k_rem, M):
    """prox_g under a node; fixed-out coordinates exactly 0 — prox.py:190-201."""
    mu = np.asarray(mu, dtype=np.float64)
    res = mu - prox_conj_node(rho * mu, rho, free, fixed_one, k_rem, M) / rho
    keep = np.zeros(mu.shape[0], dtype=bool)
    both = sorted(set(int(i) for i in free) | set(int(i) for i in fixed_one))
    if both:
        keep[np.asarray(both, dtype=np.int64)] = True
    res[~keep] = 0.0
    return res


# ----------------------------------------------------------------------------
# envelope g and its conjugate
# ----------------------------------------------------------------------------

def envelope_free(mag, k: int, M: float) -> float:
    """g over unrestricted coordinates — perspective.py:76-111."""
    mag = np.asarray(mag, dtype=np.float64)
    p = mag.shape[0]
    if p == 0:
        return 0.0
    total = float(mag.sum())
    if float(mag.max()) > M * (1.0 + FEAS_RTOL):
        return math.inf
    if total > k * M * (1.0 + FEAS_RTOL):
        return math.inf
    if k == 0:
        return 0.0
    kk = min(k, p)
    top = np.sort(mag)[::-1][:kk]            # the kk largest, descending
    before = np.concatenate(([0.0], np.cumsum(top[:-1])))
    left = total - before
    slots = kk - np.arange(kk)
    avg = left / slots
    hit = np.flatnonzero(avg >= top)
    j = int(hit[0]) if hit.size else kk - 1
    head = top[:j]
    return float(0.5 * (head @ head + slots[j] * avg[j] * avg[j]))


def envelope(beta, k: int, M: float, fixed_one=(), fixed_zero=()) -> float:
    """g(beta) with an optional node restriction — perspective.py:114-132."""
    beta = np.asarray(beta, dtype=np.float64)
    if not fixed_one and not fixed_zero:
        return envelope_free(np.abs(beta), k, M)
    acc = 0.0
    if fixed_zero:
        if np.any(np.abs(beta[np.asarray(fixed_zero, dtype=np.int64)]) > ZERO_ATOL):
            return math.inf
    if fixed_one:
        part = beta[np.asarray(fixed_one, dtype=np.int64)]
        if np.any(np.abs(part) > M * (1.0 + FEAS_RTOL)):
            return math.inf
        acc += 0.5 * float(part @ part)
    free = free_indices(beta.shape[0], fixed_one, fixed_zero)
    return acc + envelope_free(np.abs(beta[free]), k - len(fixed_one), M)


def free_indices(p: int, fixed_one=(), fixed_zero=()) -> np.ndarray:
    mask = np.ones(p, dtype=bool)
    fixed = list(fixed_one) + list(fixed_zero)
    if fixed:
        mask[np.asarray(fixed, dtype=np.int64)] = False
    return np.flatnonzero(mask)


def topk_sum(vals, k: int) -> float:
    """Sum of the k largest entries — perspective.py:135-140."""
    vals = np.asarray(vals, dtype=np.float64)
    if k <= 0 or vals.size == 0:
        return 0.0
    if k >= vals.size:
        return float(vals.sum())
    return float(np.partition(vals, vals.size - k)[vals.size - k:].sum())


def envelope_conj(alpha, k: int, M: float, fixed_one=(), fixed_zero=()) -> float:
    """g*(alpha) = TopSum_k(H_M(alpha)) (node aware) — perspective.py:143-159."""
    alpha = np.asarray(alpha, dtype=np.float64)
    H = huber(alpha, M)
    H = np.atleast_1d(H)
    if not fixed_one and not fixed_zero:
        return topk_sum(H, k)
    acc = 0.0
    if fixed_one:
        acc += float(H[np.asarray(fixed_one, dtype=np.int64)].sum())
    free = free_indices(alpha.shape[0], fixed_one, fixed_zero)
    return acc + topk_sum(H[free], k - len(fixed_one))


# ----------------------------------------------------------------------------
# losses (solver-grade only: the engine's scope)
# ----------------------------------------------------------------------------

def _expit(t):
    # logistic sigmoid 1/(1+exp(-t)); scipy.special.expit is the function the
    # reference calls (model.py:15, :193) — a pinned third-party routine
    return _scipy_special.expit(t)


def loss_value(kind: str, u, y) -> float:
    """F(u) — model.py:159-172."""
    u = np.asarray(u, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if kind == SQUARED_ERROR:
        d = u - y
        return float(d @ d)
    if kind == LOGISTIC:
        return float(np.sum(np.logaddexp(0.0, -y * u)))
    if kind == SQUARED_HINGE:
        h = np.maximum(0.0, 1.0 - y * u)
        return float(h @ h)
    if kind == POISSON:                                   # model.py:174-175
        return float(np.sum(np.exp(u) - y * u))
    if kind == GAMMA:                                     # model.py:176-177
        return float(np.sum(y * np.exp(-u) + u))
    raise ValueError(kind)


def loss_grad(kind: str, u, y) -> np.ndarray:
    """grad F(u) — model.py:184-195."""
    u = np.asarray(u, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if kind == SQUARED_ERROR:
        return 2.0 * (u - y)
    if kind == LOGISTIC:
        return -y * _expit(-y * u)
    if kind == SQUARED_HINGE:
        return -2.0 * y * np.maximum(0.0, 1.0 - y * u)
    if kind == POISSON:                                   # model.py:196-197 (_gradient_any)
        return np.exp(u) - y
    if kind == GAMMA:                                     # model.py:198-199
        return 1.0 - y * np.exp(-u)
    raise ValueError(kind)


def _xlogx(r):
    # r log r with 0 log 0 = 0: scipy.special.xlogy(r, r) as in model.py:223
    return _scipy_special.xlogy(r, r)


def loss_conj_neg(kind: str, zeta, y) -> float:
    """F*(-zeta), +inf outside the domain — model.py:221-253."""
    zeta = np.asarray(zeta, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if kind == SQUARED_ERROR:
        return float(0.25 * (zeta @ zeta) - y @ zeta)
    if kind == LOGISTIC:
        r = zeta / y
        if np.any(r < -DOMAIN_SLACK) or np.any(r > 1.0 + DOMAIN_SLACK):
            return math.inf
        r = np.clip(r, 0.0, 1.0)
        return float(np.sum(_xlogx(r) + _xlogx(1.0 - r)))
    if kind == SQUARED_HINGE:
        z = -y * zeta
        if np.any(z > DOMAIN_SLACK):
            return math.inf
        z = np.minimum(z, 0.0)
        return float(np.sum(z + 0.25 * z * z))
    if kind == POISSON:                                   # model.py:259-264
        z = y - zeta
        if np.any(z < -DOMAIN_SLACK):
            return math.inf
        z = np.maximum(z, 0.0)
        return float(np.sum(_xlogx(z) - z))
    if kind == GAMMA:                                     # model.py:266-273
        z = (1.0 + zeta) / y
        if np.any(z < -DOMAIN_SLACK):
            return math.inf
        z = np.maximum(z, 0.0)
        return float(np.sum(y * (_xlogx(z) - z)))
    raise ValueError(kind)


# ----------------------------------------------------------------------------
# Lipschitz constant
# ----------------------------------------------------------------------------

class PowerIterationError(RuntimeError):
    def __init__(self, msg, iteration):
        super().__init__(msg)
        self.iteration = iteration


def power_start(p: int, seed: int = 0) -> np.ndarray:
    """Unit start vector of model.py:286-288."""
    v = np.random.default_rng(seed).standard_normal(p)
    return v / np.linalg.norm(v)


def lambda_max_power(X, tol=POWER_TOL, max_iter=POWER_MAX_ITER, seed=0) -> float:
    """Power iteration on X^T X — model.py:283-306."""
    v = power_start(X.shape[1], seed)
    prev = math.inf
    for _ in range(max_iter):
        w = X @ v
        lam = float(w @ w)
        if lam == 0.0:
            return 0.0
        v = X.T @ w
        nrm = np.linalg.norm(v)
        if nrm == 0.0:
            return 0.0
        v = v / nrm
        if abs(lam - prev) <= tol * lam:
            return lam
        prev = lam
    raise PowerIterationError("power iteration did not converge", max_iter)


def lipschitz(kind: str, X) -> float:
    """curvature * lambda_max * 1.01 — model.py:316-327."""
    return CURVATURE[kind] * lambda_max_power(X) * LIPSCHITZ_SAFETY


# ----------------------------------------------------------------------------
# Fenchel bound and the restarted FISTA driver
# ----------------------------------------------------------------------------

def fenchel_bound(X, y, kind, k, M, lam2, beta, fixed_one=(), fixed_zero=()) -> float:
    """Safe lower bound at beta — perspective.py:162-190 / fista.py:150-157."""
    u = X @ np.asarray(beta, dtype=np.float64)
    return _dual_at(X, y, kind, k, M, lam2, u, fixed_one, fixed_zero)


def _dual_at(X, y, kind, k, M, lam2, u, fixed_one, fixed_zero) -> float:
    zeta = -loss_grad(kind, u, y)
    fstar = loss_conj_neg(kind, zeta, y)
    if not np.isfinite(fstar):
        return -math.inf
    v = X.T @ zeta
    two = 2.0 * lam2
    return float(-fstar - two * envelope_conj(v / two, k, M, fixed_one, fixed_zero))


TERMINATIONS = ("converged", "iteration_limit", "time_limit",
                "primal_below_incumbent", "dual_above_incumbent")


def fista(X, y, kind: str, k: int, M: float, lam2: float, L: Optional[float] = None,
          fixed_one: Sequence[int] = (), fixed_zero: Sequence[int] = (),
          parent_bound: float = -math.inf, warm: Optional[np.ndarray] = None,
          max_iter: int = 100_000, gap_tol: float = 1e-6, time_limit: float = math.inf,
          early_primal: Optional[float] = None, early_dual: Optional[float] = None,
          bci: int = 10, restart: bool = True,
          trace: Optional[Callable[[dict], None]] = None,
          stop_on_gap: bool = True,
          on_iteration: Optional[Callable[[int, np.ndarray, float, bool], None]] = None,
          on_prox: Optional[Callable[[int, np.ndarray, Optional[tuple]], None]] = None) -> dict:
    """Restarted FISTA on the perspective relaxation — fista.py:76-222.

    Same operation order as the reference (three X passes per iteration, the
    dual at t == 1 and every ``bci``).  ``stop_on_gap=False`` is the engine's
    fixed-iteration extension (the reference has no such switch; with it left
    True the behaviour is the reference's).  ``on_iteration(t, beta, obj,
    restarted)`` is a test hook that sees every iterate; ``on_prox(t, order,
    pool, sorted_keys)`` sees the prox's stable descending order (coordinate ids of the free
    coordinates, prox.py:111) and merged PAVA pool (a*, c*) or None
    (prox.py:46-98) at every iteration.
    """
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    p = X.shape[1]
    fixed_one = tuple(sorted(int(j) for j in fixed_one))
    fixed_zero = tuple(sorted(int(j) for j in fixed_zero))
    restricted = bool(fixed_one or fixed_zero)
    two = 2.0 * lam2
    if L is None:
        L = lipschitz(kind, X)
    L = max(L, 1e-12)
    rho = L / two

    cur_t = [0]

    def _conj(mu_free, kk, ids=None):
        if on_prox is None:
            return prox_conj(mu_free, rho, kk, M)
        res, order, pool = prox_conj(mu_free, rho, kk, M, instrument=True)
        keys = None
        if order is not None:
            keys = np.abs(mu_free)[order]
            if ids is not None:
                order = ids[order]
        on_prox(cur_t[0], order, pool, keys)
        return res

    if not restricted:
        def step(gam):
            return gam - _conj(rho * gam, k, np.arange(p)) / rho
    else:
        free = free_indices(p, fixed_one, fixed_zero)
        fone = np.asarray(fixed_one, dtype=np.int64)
        k_rem = min(k - len(fixed_one), free.size)
        zero_mask = np.ones(p, dtype=bool)
        zero_mask[free] = False
        if fone.size:
            zero_mask[fone] = False

        def step(gam):
            mu = rho * gam
            shrunk = mu.copy()
            if fone.size:
                part = mu[fone]
                shrunk[fone] = np.sign(part) * hprox(np.abs(part), rho, M)
            if free.size:
                shrunk[free] = _conj(mu[free], k_rem, free)
            res = gam - shrunk / rho
            res[zero_mask] = 0.0
            return res

    beta = np.zeros(p) if warm is None else np.asarray(warm, dtype=np.float64).copy()
    beta_prev = beta.copy()
    t0 = time.perf_counter()
    u = X @ beta
    obj = loss_value(kind, u, y) + two * envelope(beta, k, M, fixed_one, fixed_zero)
    phi = 1
    restarts = 0
    best = parent_bound
    term = "iteration_limit"
    it = 0
    for t in range(1, max_iter + 1):
        it = t
        cur_t[0] = t
        gam = beta + (phi / (phi + 3.0)) * (beta - beta_prev)
        grad = X.T @ loss_grad(kind, X @ gam, y)
        gam -= grad / L
        nxt = step(gam)
        u = X @ nxt
        obj_new = loss_value(kind, u, y) + two * envelope(nxt, k, M, fixed_one, fixed_zero)
        if not np.isfinite(obj_new):
            raise PowerIterationError("composite objective became non-finite", t)
        did_restart = restart and obj_new >= obj
        if did_restart:
            phi = 1
            restarts += 1
        else:
            phi += 1
        beta_prev, beta = beta, nxt
        obj = obj_new
        if on_iteration is not None:
            on_iteration(t, beta, obj, did_restart)
        if t == 1 or t % bci == 0:
            best = max(best, _dual_at(X, y, kind, k, M, lam2, u, fixed_one, fixed_zero))
            gap = obj - best
            if trace is not None:
                trace({"iteration": t, "primal": obj, "dual": best, "gap": gap,
                       "restarted": did_restart})
            if stop_on_gap and gap <= gap_tol:
                term = "converged"
                break
            if early_dual is not None and best >= early_dual:
                term = "dual_above_incumbent"
                break
        if early_primal is not None and obj < early_primal:
            term = "primal_below_incumbent"
            break
        if time.perf_counter() - t0 > time_limit:
            term = "time_limit"
            break
    if not np.isfinite(best):
        best = _dual_at(X, y, kind, k, M, lam2, X @ beta, fixed_one, fixed_zero)
    gap = obj - best
    if term == "iteration_limit" and gap <= gap_tol:
        term = "converged"
    return {"beta": beta, "primal_value": obj, "dual_bound": best, "gap": gap,
            "iterations": it, "restarts": restarts, "termination": term,
            "wall_time": time.perf_counter() - t0}
