"""Batched fp64 safe lower bound: one
l0_safe_lower_bound_batched call for a batch of branch-and-bound nodes vs the
reference's per-node safe_lower_bound (perspective.py:162-190) -- its golden
bounds at 1e-12, the oracle's fenchel_bound (oracle/l0_oracle.py) at 1e-11 on
larger batches (fp64 and fp32 storage, > 64 nodes: two node tiles, split-K
transpose), and the engine's own per-node call."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOSSES = ["squared_error", "logistic", "squared_hinge"]


def test_batched_bound_golden(engine, golden):
    data, meta = golden
    for i in range(meta["n_lip"]):
        X, y = data[f"lip/{i}/X"], data[f"lip/{i}/y"]
        kind_i, k, M, lam2 = data[f"lip/{i}/args"]
        inst = engine.ProblemInstance(X, y, engine.LossKind(LOSSES[int(kind_i)]), int(k), float(M), float(lam2))
        betas = data[f"lip/{i}/betas"]
        nodes = [engine.NodeState(fixed_one=(0,), fixed_zero=(1, 2)) if h else None
                 for h in data[f"lip/{i}/nodes"]]
        got = engine.safe_lower_bound_batched(inst, betas, nodes)
        for g, ref in zip(got, data[f"lip/{i}/bounds"]):
            assert g == pytest.approx(float(ref), rel=1e-12, abs=1e-12)


def _random_nodes(rng, p, k, count):
    nodes = []
    for j in range(count):
        if j % 5 == 0:
            nodes.append(None)
            continue
        idx = rng.choice(p, size=rng.integers(0, 9) + rng.integers(0, 5), replace=False)
        n1 = min(int(rng.integers(0, 5)), len(idx), k)
        nodes.append((tuple(int(v) for v in idx[:n1]), tuple(int(v) for v in idx[n1:])))
    return nodes


@pytest.mark.parametrize("loss,dtype,n,p,count", [
    ("squared_error", "fp64", 900, 300, 70),
    ("logistic", "fp64", 700, 260, 20),
    ("squared_error", "fp32", 1200, 500, 96),
    ("squared_hinge", "fp32", 500, 333, 9),
])
def test_batched_bound_vs_oracle(engine, oracle, loss, dtype, n, p, count):
    rng = np.random.default_rng(n + p + count)
    X = rng.standard_normal((n, p))
    if dtype == "fp32":
        X = X.astype(np.float32)
    y = rng.standard_normal(n) if loss == "squared_error" else rng.choice([-1.0, 1.0], n)
    k, M, lam2 = 7, 1.5, 0.4
    inst = engine.ProblemInstance(X, y, engine.LossKind(loss), k, M, lam2, dtype=dtype)
    spec = _random_nodes(rng, p, k, count)
    nodes = [None if s is None else engine.NodeState(fixed_one=s[0], fixed_zero=s[1]) for s in spec]
    betas = rng.standard_normal((count, p)) * 0.3
    got = engine.safe_lower_bound_batched(inst, betas, nodes)
    X64 = X.astype(np.float64)
    for j, s in enumerate(spec):
        f1, f0 = ((), ()) if s is None else s
        ref = oracle.fenchel_bound(X64, y, loss, k, M, lam2, betas[j], fixed_one=f1, fixed_zero=f0)
        assert got[j] == pytest.approx(ref, rel=1e-11, abs=1e-11), j
        if j % 7 == 0:
            single = engine.safe_lower_bound(inst, betas[j], nodes[j])
            assert got[j] == pytest.approx(single, rel=1e-12, abs=1e-12), j


def test_batched_bound_validation(engine):
    rng = np.random.default_rng(3)
    X, y = rng.standard_normal((20, 6)), rng.standard_normal(20)
    inst = engine.ProblemInstance(X, y, engine.LossKind.SQUARED_ERROR, 2, 1.0, 0.5)
    assert engine.safe_lower_bound_batched(inst, np.zeros((0, 6)), []) == []
    with pytest.raises(engine.InvalidInputError):
        engine.safe_lower_bound_batched(inst, np.zeros((2, 5)), [None, None])
    bad = np.zeros((1, 6))
    bad[0, 3] = np.nan
    with pytest.raises(engine.InvalidInputError):
        engine.safe_lower_bound_batched(inst, bad, [None])
    with pytest.raises(engine.InfeasibleNodeError):
        engine.safe_lower_bound_batched(inst, np.zeros((1, 6)), [engine.NodeState(fixed_one=(0, 1, 2))])
