"""Pin the CPU oracle (oracle/l0_oracle.py) to the reference.

Every case compares the oracle against outputs the reference itself produced
(tests/golden/make_golden.py).  Operator-level cases are bitwise: the oracle
reproduces the reference's operation order.  Trajectories are compared with
BLAS limited to one thread, as when the fixture was generated.
"""

import math

import numpy as np
import pytest
import threadpoolctl

from paper_2502_09502_b200 import data as mydata

LOSSES = ["squared_error", "logistic", "squared_hinge"]


def _cases(golden, prefix, count_key):
    data, meta = golden
    return [(data, i) for i in range(meta[count_key])]


def test_prox_bitwise(golden, oracle):
    data, meta = golden
    for i in range(meta["n_prox"]):
        mu = data[f"prox/{i}/mu"]
        rho, k, M = data[f"prox/{i}/args"]
        k = int(k)
        got = oracle.prox_conj(mu, rho, k, M)
        assert np.array_equal(got, data[f"prox/{i}/gstar"]), i
        src = data[f"prox/{i}/gamma"] if f"prox/{i}/gamma" in data else mu
        assert np.array_equal(oracle.prox_g(src, rho, k, M), data[f"prox/{i}/g"]), i


def test_node_prox_bitwise(golden, oracle):
    data, meta = golden
    for i in range(meta["n_node"]):
        mu = data[f"node/{i}/mu"]
        rho, k_rem, M = data[f"node/{i}/args"]
        free = data[f"node/{i}/free"].tolist()
        fone = data[f"node/{i}/fone"].tolist()
        got = oracle.prox_conj_node(mu, rho, free, fone, int(k_rem), M)
        assert np.array_equal(got, data[f"node/{i}/gstar"]), i
        got = oracle.prox_g_node(mu, rho, free, fone, int(k_rem), M)
        assert np.array_equal(got, data[f"node/{i}/g"]), i


def test_envelope_bitwise(golden, oracle):
    data, meta = golden
    n_inf = 0
    for i in range(meta["n_env"]):
        k, M = data[f"env/{i}/args"]
        fone = tuple(data[f"env/{i}/fone"].tolist())
        fzero = tuple(data[f"env/{i}/fzero"].tolist())
        g = oracle.envelope(data[f"env/{i}/beta"], int(k), M, fone, fzero)
        ref = float(data[f"env/{i}/g"])
        n_inf += math.isinf(ref)
        assert g == ref or (math.isinf(g) and math.isinf(ref)), i
        gs = oracle.envelope_conj(data[f"env/{i}/alpha"], int(k), M, fone, fzero)
        assert gs == float(data[f"env/{i}/gstar"]), i
    assert 0 < n_inf < meta["n_env"]  # both classes exercised


def test_losses_bitwise(golden, oracle):
    data, meta = golden
    for i in range(meta["n_loss"]):
        kind = LOSSES[int(data[f"loss/{i}/kind"])]
        u, y = data[f"loss/{i}/u"], data[f"loss/{i}/y"]
        assert oracle.loss_value(kind, u, y) == float(data[f"loss/{i}/value"])
        assert np.array_equal(oracle.loss_grad(kind, u, y), data[f"loss/{i}/grad"])
        zeta = -oracle.loss_grad(kind, u, y)
        assert oracle.loss_conj_neg(kind, zeta, y) == float(data[f"loss/{i}/conj"])
        bad = oracle.loss_conj_neg(kind, data[f"loss/{i}/zeta_bad"], y)
        ref = float(data[f"loss/{i}/conj_bad"])
        assert bad == ref or (math.isinf(bad) and math.isinf(ref))


def test_lipschitz_and_safe_bound(golden, oracle):
    data, meta = golden
    with threadpoolctl.threadpool_limits(1):
        for i in range(meta["n_lip"]):
            X, y = data[f"lip/{i}/X"], data[f"lip/{i}/y"]
            kind_i, k, M, lam2 = data[f"lip/{i}/args"]
            kind = LOSSES[int(kind_i)]
            L_ref = float(data[f"lip/{i}/L"])
            if math.isnan(L_ref):
                with pytest.raises(oracle.PowerIterationError):
                    oracle.lipschitz(kind, X)
            else:
                assert oracle.lipschitz(kind, X) == pytest.approx(L_ref, rel=1e-13)
            for beta, has_node, ref in zip(data[f"lip/{i}/betas"], data[f"lip/{i}/nodes"],
                                           data[f"lip/{i}/bounds"]):
                fo, fz = ((0,), (1, 2)) if has_node else ((), ())
                b = oracle.fenchel_bound(X, y, kind, int(k), M, lam2, beta, fo, fz)
                assert b == pytest.approx(float(ref), rel=1e-13, abs=1e-13)


def _traj_inputs(golden, name):
    data, meta = golden
    spec = meta["cases"][name]
    if spec["gen"] == "inline":
        X, y = data[f"traj/{name}/X"], data[f"traj/{name}/y"]
    else:
        cd = mydata.make_config(spec["config"], scale=spec["scale"])
        import hashlib
        digest = hashlib.sha256(np.ascontiguousarray(cd.X).tobytes()).digest()
        assert digest == bytes(data[f"traj/{name}/xsha"]), "generator drifted from the fixture"
        X, y = cd.X.astype(np.float64), cd.y
    return spec, X, y


TRAJ = ["spec_1d", "spec_2x2", "spec_y0", "c1", "c1_default_tol", "c1_literal", "c1_norestart",
        "c2_small", "c3_small", "c3_small_bci7", "c4_node0", "c4_node1", "c4_node2",
        "c4_node_warm", "c4_primal_cut", "c4_dual_cut"]


def oracle_solve(oracle, spec, X, y, L, p):
    opts = dict(spec["opts"])
    node = spec.get("node")
    fz, fo, pb = (), (), -math.inf
    if node:
        fz, fo = tuple(node[0]), tuple(node[1])
        if len(node) > 2:
            pb = node[2]
    warm = None
    if spec.get("warm_seed") is not None:
        warm = np.random.default_rng(spec["warm_seed"]).standard_normal(p) * 0.05
        warm[list(fz)] = 0.0
    rec = []
    rep = oracle.fista(X, y, spec["loss"], spec["k"], spec["M"], spec["lambda2"], L=L,
                       fixed_one=fo, fixed_zero=fz, parent_bound=pb, warm=warm,
                       max_iter=opts.get("max_iterations", 100000),
                       gap_tol=opts.get("gap_tolerance", 1e-6),
                       early_primal=opts.get("early_primal_cutoff"),
                       early_dual=opts.get("early_dual_cutoff"),
                       bci=opts.get("bound_check_interval", 10),
                       restart=opts.get("restart", True), trace=rec.append)
    return rep, rec


@pytest.mark.parametrize("name", TRAJ)
def test_trajectory_matches_reference(golden, oracle, name):
    data, meta = golden
    spec, X, y = _traj_inputs(golden, name)
    primal, dual, gap, iters, restarts, L = data[f"traj/{name}/scalars"]
    with threadpoolctl.threadpool_limits(1):
        rep, rec = oracle_solve(oracle, spec, X, y, float(L), X.shape[1])
    trace = data[f"traj/{name}/trace"]
    assert rep["termination"] == spec["termination"]
    assert rep["iterations"] == int(iters)
    assert rep["restarts"] == int(restarts)
    assert len(rec) == trace.shape[0]
    for r, ref in zip(rec, trace):
        assert r["iteration"] == int(ref[0])
        assert r["primal"] == pytest.approx(ref[1], rel=1e-13)
        assert r["dual"] == pytest.approx(ref[2], rel=1e-12, abs=1e-12)
        assert r["restarted"] == bool(ref[4])
    assert rep["primal_value"] == pytest.approx(primal, rel=1e-13)
    np.testing.assert_allclose(rep["beta"], data[f"traj/{name}/beta"], rtol=0, atol=1e-12)
