"""Synthetic inputs for the engine's parity cases and benchmark configs.

Host-side harness code (input generation is not on the hot path).  The
generator reproduces the reference's synthetic protocol bit for bit so that
the GPU engine and the CPU oracle see identical inputs:

* ``true_support``  — /root/reference/pkg/src/l0cert/data.py:63-73
* ``ar1_rows``      — data.py:76-85 (AR(1) rows, Toeplitz correlation sigma^|i-j|),
  evaluated in place on the Gaussian draw: every element is still
  ``sigma*x_{j-1} + c*w_j`` with the same two roundings, so the bits agree
  with the reference while peak memory halves.
* ``synthetic``     — data.py:88-115 (``generate_synthetic``: beta*, SNR noise
  with the reference's "variance" reading, labels)
* ``standardize``   — data.py:224-242

``make_config(name)`` builds the five BASELINE configs.
"""

from __future__ import annotations

import dataclasses
import math
from typing import Optional, Tuple

import numpy as np

__all__ = [
    "true_support", "ar1_rows", "synthetic", "standardize", "ConfigData",
    "make_config", "CONFIGS", "random_nodes",
]


def true_support(p: int, k_true: int) -> np.ndarray:
    """0-based equally spaced support — data.py:63-73."""
    if p % k_true == 0:
        pos = np.arange(1, k_true + 1) * (p // k_true)
    else:
        pos = np.unique(np.round(np.arange(1, k_true + 1) * p / k_true).astype(np.int64))
        pos = np.clip(pos, 1, p)
    return pos - 1


def ar1_rows(n: int, p: int, sigma: float, rng: np.random.Generator,
             dtype=np.float64) -> np.ndarray:
    """Rows ~ N(0, Toeplitz(sigma^|i-j|)) by the AR(1) recursion — data.py:76-85.

    The recursion runs in place on the Gaussian draw (float64 arithmetic);
    ``dtype=np.float32`` rounds the finished matrix once, as the fp32 configs
    specify ("X cast to fp32").
    """
    X = rng.standard_normal((n, p))
    if sigma != 0.0:
        c = np.sqrt(1.0 - sigma * sigma)
        col_prev = X[:, 0]
        tmp = np.empty(n)
        for j in range(1, p):
            col = X[:, j]
            np.multiply(col, c, out=tmp)          # c * w_j
            np.multiply(col_prev, sigma, out=col)  # sigma * x_{j-1}
            np.add(col, tmp, out=col)
            col_prev = col
    if dtype != np.float64:
        X = X.astype(dtype)
    return X


def synthetic(n: int, p: int, k_true: int, sigma: float = 0.5, snr: float = 5.0,
              seed: int = 0, task: str = "regression", snr_scale: str = "variance"):
    """(X, y, beta_true) of ``generate_synthetic`` — data.py:88-115."""
    rng = np.random.default_rng(seed)
    X = ar1_rows(n, p, sigma, rng)
    beta_true = np.zeros(p)
    beta_true[true_support(p, k_true)] = 1.0
    signal = X @ beta_true
    scale = np.linalg.norm(signal) / snr
    noise_std = np.sqrt(scale) if snr_scale == "variance" else scale
    eps = rng.normal(0.0, noise_std, n) if noise_std > 0 else np.zeros(n)
    if task == "regression":
        y = signal + eps
    else:
        prob = np.clip(signal + eps, 0.0, 1.0)
        y = np.where(rng.random(n) < prob, 1.0, -1.0)
    return X, y, beta_true


def standardize(X) -> Tuple[np.ndarray, np.ndarray]:
    """Centre columns, scale to unit norm, drop constant ones — data.py:224-242.

    Returns (X_std, kept_columns)."""
    X = np.asarray(X, dtype=np.float64)
    means = X.mean(axis=0)
    centered = X - means
    norms = np.linalg.norm(centered, axis=0)
    scale = np.abs(X).max(axis=0)
    keep = norms > 1e-12 * np.maximum(1.0, scale)
    kept = np.nonzero(keep)[0]
    return centered[:, kept] / norms[kept], kept


@dataclasses.dataclass
class ConfigData:
    name: str
    X: np.ndarray            # host matrix (float64, or float32 for the fp32 configs)
    y: np.ndarray            # float64 labels
    loss: str                # "squared_error" | "logistic"
    k: int
    M: float
    lambda2: float
    iterations: Optional[int]    # fixed iteration count (None: run to the gap)
    rel_gap: Optional[float]     # relative gap target (C2)
    dtype: str                   # "fp64" | "fp32"
    beta_true: Optional[np.ndarray] = None
    nodes: Optional[list] = None  # [(fixed_zero, fixed_one)] for C4
    note: str = ""

    @property
    def n(self) -> int:
        return self.X.shape[0]

    @property
    def p(self) -> int:
        return self.X.shape[1]


def random_nodes(p: int, count: int, seed: int = 1, max_zero: int = 8, max_one: int = 4):
    """C4's seeded node sets: per node nz ~ U{0..8},
    no ~ U{0..4}, disjoint indices drawn without replacement."""
    rng = np.random.default_rng(seed)
    nodes = []
    for _ in range(count):
        nz = int(rng.integers(0, max_zero + 1))
        no = int(rng.integers(0, max_one + 1))
        idx = rng.choice(p, nz + no, replace=False)
        nodes.append((tuple(sorted(int(i) for i in idx[:nz])),
                      tuple(sorted(int(i) for i in idx[nz:]))))
    return nodes


def _c1(scale: float = 1.0, literal: bool = False) -> ConfigData:
    n, p = int(2000 * scale), int(1000 * scale)
    if literal:
        # the reference pipeline verbatim: y from the raw X, then standardize X
        X, y, bt = synthetic(n, p, 10, sigma=0.5, snr=5.0, seed=0)
        Xs, _ = standardize(X)
        note = "literal reference pipeline (degenerate: gap hits 0 at t=10)"
    else:
        rng = np.random.default_rng(0)
        Xs, _ = standardize(ar1_rows(n, p, 0.5, rng))
        bt = np.zeros(p)
        bt[true_support(p, 10)] = 1.0
        sig = Xs @ bt
        eps = rng.normal(0.0, math.sqrt(np.linalg.norm(sig) / 5.0), n)
        y = sig + eps
        note = "y drawn from the standardised X (well-posed)"
    return ConfigData("C1" + ("-literal" if literal else ""), np.ascontiguousarray(Xs), y,
                      "squared_error", 10, 2.0, 1.0, 1000, None, "fp64", bt, note=note)


def _c2(scale: float = 1.0) -> ConfigData:
    n = p = int(16000 * scale)
    X, y, bt = synthetic(n, p, 20, sigma=0.7, snr=5.0, seed=0)
    return ConfigData("C2", X, y, "squared_error", 20, 2.0, 0.1, None, 1e-6, "fp64", bt)


def _c3(scale: float = 1.0) -> ConfigData:
    n, p = int(50000 * scale), int(20000 * scale)
    rng = np.random.default_rng(0)
    X = ar1_rows(n, p, 0.5, rng, dtype=np.float32)
    bt = np.zeros(p)
    bt[true_support(p, 15)] = 1.0
    eta = X.astype(np.float64) @ bt
    prob = 1.0 / (1.0 + np.exp(-eta))
    y = np.where(rng.random(n) < prob, 1.0, -1.0)
    return ConfigData("C3", X, y, "logistic", 15, 3.0, 0.01, 2000, None, "fp32", bt,
                      note="labels ~ Bernoulli(sigmoid(x.beta*)) (builder recipe)")


def _c4(scale: float = 1.0, nodes: int = 512) -> ConfigData:
    n, p = int(20000 * scale), int(5000 * scale)
    X, y, bt = synthetic(n, p, 10, sigma=0.5, snr=5.0, seed=0)
    return ConfigData("C4", X.astype(np.float32), y, "squared_error", 10, 2.0, 0.5, 500,
                      None, "fp32", bt, nodes=random_nodes(p, nodes, seed=1))


def _c5(scale: float = 1.0, block_rows: int = 100_000) -> ConfigData:
    n, p = int(1_000_000 * scale), int(10_000 * min(1.0, scale * 10))
    X = np.empty((n, p), dtype=np.float32)
    for b, r0 in enumerate(range(0, n, block_rows)):
        r1 = min(n, r0 + block_rows)
        X[r0:r1] = ar1_rows(r1 - r0, p, 0.5, np.random.default_rng([0, b]), dtype=np.float32)
    bt = np.zeros(p)
    bt[true_support(p, 25)] = 1.0
    sig = X.astype(np.float64) @ bt if n * p <= 2e8 else _rowblock_matvec(X, bt)
    eps = np.random.default_rng([0, 1 << 20]).normal(0.0, math.sqrt(np.linalg.norm(sig) / 5.0), n)
    return ConfigData("C5", X, sig + eps, "squared_error", 25, 2.0, 0.1, 1000, None, "fp32", bt)


def _rowblock_matvec(X, v, block=50_000):
    out = np.empty(X.shape[0])
    for r0 in range(0, X.shape[0], block):
        out[r0:r0 + block] = X[r0:r0 + block].astype(np.float64) @ v
    return out


CONFIGS = {"C1": _c1, "C1-literal": lambda scale=1.0: _c1(scale, literal=True),
           "C2": _c2, "C3": _c3, "C4": _c4, "C5": _c5}


def make_config(name: str, scale: float = 1.0, **kw) -> ConfigData:
    """Build config ``name`` (C1, C1-literal, C2, C3, C4, C5) at ``scale``
    (scale < 1 shrinks n and p proportionally for parity tests)."""
    return CONFIGS[name](scale=scale, **kw) if kw else CONFIGS[name](scale=scale)
