"""lambda_max(X^T X) by Lanczos on the device — the robust companion of the
reference's power iteration (model.py:283-327).

The reference estimates lambda_max with a power iteration capped at 500 steps
(tol 1e-7); on slowly separating spectra (BASELINE C2, C3, C5) it stops
without converging and ``lipschitz_constant`` raises NumericalError
(SURVEY.md §3.5).  Lanczos with full reorthogonalisation converges on the same
matrices in a few dozen X^T X products: the top Ritz value of the Krylov space
rises monotonically to lambda_max.

Every product is one pair of the engine's device passes (``l0_matvec`` /
``l0_rmatvec``, or an all-reduced sum of them over row shards); the
recurrence coefficients stay on the device, and the host only reads the
tridiagonal matrix every ``check_every`` steps to test convergence.
"""

from __future__ import annotations

import math
from typing import Callable, Optional

import numpy as np

from .errors import NumericalError


def lanczos_lambda_max(normal_op: Callable, p: int, device, tol: float = 1e-13,
                       max_steps: int = 300, check_every: int = 8, seed: int = 0,
                       allreduce: Optional[Callable] = None) -> float:
    """Largest eigenvalue of the PSD operator ``normal_op`` (v -> X^T X v on
    CUDA float64 vectors of length p).

    ``allreduce`` (in place, sum over ranks) turns per-shard products into the
    global X^T X v; every rank then runs the same recurrence bit for bit.
    Starts from the reference's seed-0 unit vector (model.py:286-288).
    Converged when the top Ritz value changes by <= tol (relative) over
    ``check_every`` steps, or on an invariant subspace.
    """
    import torch
    steps = int(min(max_steps, p))
    v0 = np.random.default_rng(seed).standard_normal(p)
    v0 /= np.linalg.norm(v0)
    V = torch.empty((steps + 1, p), dtype=torch.float64, device=device)
    V[0] = torch.from_numpy(v0).to(device)
    alpha = torch.zeros(steps, dtype=torch.float64, device=device)
    beta = torch.zeros(steps, dtype=torch.float64, device=device)
    prev = -math.inf
    theta = 0.0
    for j in range(steps):
        w = normal_op(V[j])
        if allreduce is not None:
            allreduce(w)
        a = torch.dot(w, V[j])
        alpha[j] = a
        # full reorthogonalisation against the whole basis, twice (classical
        # Gram-Schmidt): keeps the Ritz values free of ghost copies
        B = V[:j + 1]
        w = w - B.T @ (B @ w)
        w = w - B.T @ (B @ w)
        b = torch.linalg.vector_norm(w)
        beta[j] = b
        V[j + 1] = w / b
        last = j == steps - 1
        if (j + 1) % check_every == 0 or last or j < 2:
            al = alpha[:j + 1].cpu().numpy()
            be = beta[:j + 1].cpu().numpy()
            if not np.all(np.isfinite(al)) or not np.all(np.isfinite(be)):
                raise NumericalError("Lanczos recurrence became non-finite", iteration=j + 1)
            T = np.diag(al) + np.diag(be[:-1], 1) + np.diag(be[:-1], -1)
            theta = float(np.linalg.eigvalsh(T)[-1]) if j >= 0 else 0.0
            if theta <= 0.0 and al.max(initial=0.0) <= 0.0:
                return 0.0                      # X == 0 (the reference returns 0 too)
            scale = max(abs(theta), 1e-300)
            if be[-1] <= 1e-14 * scale:        # invariant subspace: theta is exact
                return theta
            if j >= 2 and abs(theta - prev) <= tol * scale:
                return theta
            prev = theta
    raise NumericalError(f"Lanczos did not converge within {steps} steps", iteration=steps)


def engine_normal_op(dp) -> Callable:
    """v -> X^T (X v) through the engine's device passes of problem ``dp``."""
    import torch
    from . import _device, native
    lib = native.lib()
    u = torch.empty(dp.n, dtype=torch.float64, device=dp.X.device)

    def op(v):
        v = v.contiguous()
        out = torch.empty(dp.p, dtype=torch.float64, device=dp.X.device)
        s = _device.stream_handle()
        native.check(lib.l0_matvec(dp.handle, v.data_ptr(), u.data_ptr(), s))
        native.check(lib.l0_rmatvec(dp.handle, u.data_ptr(), out.data_ptr(), s))
        return out
    return op
