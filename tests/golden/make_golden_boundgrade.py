"""Golden vectors for the bound-grade losses (Poisson, gamma): values,
conjugates (inside and outside the domain) and safe lower bounds, produced by
the reference itself.  Build container only:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_boundgrade.py
"""

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

from l0cert import model as rmodel  # noqa: E402
from l0cert import perspective as rpersp  # noqa: E402

OUT = {}
idx = 0
for loss in ("poisson", "gamma"):
    kind = rmodel.LossKind(loss)
    for n, seed in ((1, 1), (7, 2), (60, 3)):
        rng = np.random.default_rng(seed)
        p = max(2, n // 3)
        X = rng.standard_normal((n, p)) * 0.5
        y = rng.poisson(2.0, n).astype(np.float64) if loss == "poisson" else rng.gamma(2.0, 1.5, n)
        beta = rng.standard_normal(p) * 0.3
        u = X @ beta
        zeta = -rmodel._gradient_any(kind, u, y)
        zeta_bad = zeta.copy()
        zeta_bad[0] = (y[0] + 5.0) if loss == "poisson" else (-1.0 - 5.0)   # outside the domain
        inst = rmodel.ProblemInstance(X=X, y=y, loss=kind, k=1, M=2.0, lambda2=0.4)
        node = rmodel.NodeState(fixed_zero=(p - 1,)) if p > 2 else None
        pre = f"bg/{idx}/"
        OUT[pre + "X"] = X
        OUT[pre + "y"] = y
        OUT[pre + "beta"] = beta
        OUT[pre + "u"] = u
        OUT[pre + "zeta"] = zeta
        OUT[pre + "zeta_bad"] = zeta_bad
        OUT[pre + "kind"] = np.array(["poisson", "gamma"].index(loss))
        OUT[pre + "value"] = np.array(rmodel.loss_value(kind, u, y))
        OUT[pre + "conj"] = np.array(rmodel.loss_conjugate_at_neg(kind, zeta, y))
        OUT[pre + "conj_bad"] = np.array(rmodel.loss_conjugate_at_neg(kind, zeta_bad, y))
        OUT[pre + "bound"] = np.array(rpersp.safe_lower_bound(inst, beta, None))
        OUT[pre + "bound_node"] = np.array(rpersp.safe_lower_bound(inst, beta, node) if node else np.nan)
        OUT[pre + "node_zero"] = np.array(p - 1 if node else -1)
        idx += 1
OUT["n_bg"] = np.array(idx)
np.savez_compressed(os.path.join(HERE, "boundgrade.npz"), **OUT)
print("wrote", idx, "bound-grade cases")
