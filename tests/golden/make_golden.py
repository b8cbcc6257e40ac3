"""Generate the golden fixtures that pin the CPU oracle to the reference.

Run in the BUILD container only (it imports the reference from
/root/reference, which does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It executes the reference's own functions (``l0cert.prox``, ``perspective``,
``model``, ``fista``) on seeded inputs and stores inputs + outputs in
``tests/golden/golden.npz``.  Matrices of the trajectory cases are NOT stored;
they are regenerated from their seeds by ``paper_2502_09502_b200.data`` (which
reproduces ``l0cert.data`` bit for bit — checked here) and identified by a
SHA-256 of their bytes, so the fixture stays small.
"""

import hashlib
import json
import math
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import l0cert  # noqa: E402  (the reference)
from l0cert import data as rdata  # noqa: E402
from l0cert import fista as rfista  # noqa: E402
from l0cert import model as rmodel  # noqa: E402
from l0cert import perspective as rpersp  # noqa: E402
from l0cert import prox as rprox  # noqa: E402

from paper_2502_09502_b200 import data as mydata  # noqa: E402

OUT = {}
META = {"cases": {}}


def put(key, val):
    OUT[key] = np.asarray(val)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def lanczos_L(X, loss):
    """Injected step constant: curvature * lambda_max(X^T X) * 1.01, lambda_max
    by ARPACK with a fixed start vector (bitwise reproducible)."""
    from scipy.sparse.linalg import LinearOperator, eigsh
    n, p = X.shape
    op = LinearOperator((p, p), matvec=lambda v: X.T @ (X @ v), dtype=np.float64)
    v0 = np.ones(p) / math.sqrt(p)
    lam = float(eigsh(op, k=1, which="LA", v0=v0, tol=1e-12, return_eigenvectors=False)[0])
    curv = {"squared_error": 2.0, "logistic": 0.25, "squared_hinge": 2.0}[loss]
    return curv * lam * 1.01


def mu_sample(rng, p, kind):
    if kind == "normal":
        mu = rng.standard_normal(p) * rng.choice([0.1, 1.0, 5.0])
    elif kind == "ties":
        base = rng.standard_normal(max(1, p // 3))
        mu = rng.choice(base, p) * rng.choice([-1.0, 1.0], p)
    elif kind == "sparse":
        mu = rng.standard_normal(p) * 1e-3
        hot = rng.choice(p, max(1, p // 10), replace=False)
        mu[hot] = rng.standard_normal(hot.size) * 20.0
    elif kind == "zeros":
        mu = rng.standard_normal(p)
        mu[rng.random(p) < 0.4] = 0.0
    else:  # rounded values: many exact ties
        mu = np.round(rng.standard_normal(p) * 4.0) / 4.0
    return mu


def gen_prox():
    rng = np.random.default_rng(12345)
    sizes = [1, 2, 3, 5, 8, 13, 20, 50, 200, 1000, 4000]
    kinds = ["normal", "ties", "sparse", "zeros", "rounded"]
    idx = 0
    for p in sizes:
        reps = 12 if p <= 50 else 4
        for r in range(reps):
            kind = kinds[(idx + r) % len(kinds)]
            mu = mu_sample(rng, p, kind)
            k = int(rng.integers(1, p + 1)) if r % 3 else int(min(p, rng.integers(1, 26)))
            rho = float(rng.choice([0.1, 1.0, 10.0, 3.7, 9680.5]))
            M = float(rng.choice([0.5, 2.0, 10.0]))
            put(f"prox/{idx}/mu", mu)
            put(f"prox/{idx}/args", [rho, k, M])
            put(f"prox/{idx}/gstar", rprox.prox_gstar(mu, rho, k, M))
            put(f"prox/{idx}/g", rprox.prox_g(mu, rho, k, M))
            idx += 1
    # FISTA-like inputs: large rho, a few dominant coordinates
    for r in range(10):
        p = int(rng.choice([100, 1000, 3000]))
        gamma = rng.standard_normal(p) * 1e-2
        hot = rng.choice(p, 30, replace=False)
        gamma[hot] = rng.standard_normal(30) * 2.0
        rho = float(rng.choice([50.0, 9680.5, 1.5e5]))
        k = int(rng.integers(5, 26))
        M = 2.0
        mu = rho * gamma
        put(f"prox/{idx}/mu", mu)
        put(f"prox/{idx}/args", [rho, k, M])
        put(f"prox/{idx}/gstar", rprox.prox_gstar(mu, rho, k, M))
        put(f"prox/{idx}/g", rprox.prox_g(gamma, rho, k, M))
        put(f"prox/{idx}/gamma", gamma)
        idx += 1
    META["n_prox"] = idx


def gen_node_prox():
    rng = np.random.default_rng(777)
    idx = 0
    for p in [1, 3, 6, 10, 50, 300]:
        for r in range(8):
            mu = mu_sample(rng, p, ["normal", "ties", "zeros", "rounded"][r % 4])
            perm = rng.permutation(p)
            n1 = int(rng.integers(0, min(p, 4) + 1))
            n0 = int(rng.integers(0, p - n1 + 1)) if r % 2 else int(rng.integers(0, min(p - n1, 8) + 1))
            fone = sorted(int(i) for i in perm[:n1])
            fzero = sorted(int(i) for i in perm[n1:n1 + n0])
            free = sorted(set(range(p)) - set(fone) - set(fzero))
            k = int(rng.integers(n1, p + 1)) if p > n1 else n1
            k_rem = k - n1
            rho = float(rng.choice([0.1, 1.0, 10.0, 250.0]))
            M = float(rng.choice([0.5, 2.0, 10.0]))
            put(f"node/{idx}/mu", mu)
            put(f"node/{idx}/args", [rho, k_rem, M])
            put(f"node/{idx}/free", np.asarray(free, dtype=np.int64))
            put(f"node/{idx}/fone", np.asarray(fone, dtype=np.int64))
            put(f"node/{idx}/fzero", np.asarray(fzero, dtype=np.int64))
            put(f"node/{idx}/gstar", rprox.prox_gstar_node(mu, rho, free, fone, k_rem, M))
            put(f"node/{idx}/g", rprox.prox_g_node(mu, rho, free, fone, k_rem, M))
            idx += 1
    META["n_node"] = idx


def gen_envelope():
    rng = np.random.default_rng(4242)
    idx = 0
    for p in [1, 2, 4, 10, 30, 200, 2000]:
        for r in range(8):
            k = int(rng.integers(1, p + 1))
            M = float(rng.choice([0.5, 2.0, 10.0]))
            if r % 4 == 0:      # random, often infeasible
                beta = rng.standard_normal(p) * M
            elif r % 4 == 1:    # prox output: on the domain boundary
                beta = rprox.prox_g(rng.standard_normal(p) * 3.0, float(rng.choice([0.5, 5.0])), k, M)
            elif r % 4 == 2:    # sparse feasible
                beta = np.zeros(p)
                sup = rng.choice(p, min(k, p), replace=False)
                beta[sup] = rng.uniform(-M, M, sup.size)
            else:               # spread mass with ties
                beta = np.round(rng.uniform(-M, M, p) * 2) / 2 * (k / p)
            fone, fzero = (), ()
            if r >= 4 and p >= 3:
                perm = rng.permutation(p)
                n1 = int(rng.integers(0, min(k, 2) + 1))
                n0 = int(rng.integers(0, 3))
                fone = tuple(sorted(int(i) for i in perm[:n1]))
                fzero = tuple(sorted(int(i) for i in perm[n1:n1 + n0]))
                if r % 2:
                    beta[list(fzero)] = 0.0
            params = rpersp.EnvelopeParams(k=k, M=M, fixed_one=fone, fixed_zero=fzero)
            alpha = rng.standard_normal(p) * float(rng.choice([0.3, 3.0]))
            put(f"env/{idx}/beta", beta)
            put(f"env/{idx}/alpha", alpha)
            put(f"env/{idx}/args", [k, M])
            put(f"env/{idx}/fone", np.asarray(fone, dtype=np.int64))
            put(f"env/{idx}/fzero", np.asarray(fzero, dtype=np.int64))
            put(f"env/{idx}/g", rpersp.g_value(beta, params))
            put(f"env/{idx}/gstar", rpersp.g_conjugate(alpha, params))
            idx += 1
    META["n_env"] = idx


def gen_losses():
    rng = np.random.default_rng(99)
    idx = 0
    for loss in ("squared_error", "logistic", "squared_hinge"):
        kind = rmodel.LossKind(loss)
        for n in [1, 5, 100, 5000]:
            for r in range(3):
                u = rng.standard_normal(n) * float(rng.choice([0.5, 3.0, 40.0]))
                if loss == "squared_error":
                    y = rng.standard_normal(n) * 2.0
                else:
                    y = rng.choice([-1.0, 1.0], n)
                zeta = -rmodel.loss_gradient(kind, u, y)
                zeta_bad = zeta + (rng.standard_normal(n) * 0.7 if r == 2 else 0.0)
                put(f"loss/{idx}/u", u)
                put(f"loss/{idx}/y", y)
                put(f"loss/{idx}/kind", ["squared_error", "logistic", "squared_hinge"].index(loss))
                put(f"loss/{idx}/value", rmodel.loss_value(kind, u, y))
                put(f"loss/{idx}/grad", rmodel.loss_gradient(kind, u, y))
                put(f"loss/{idx}/conj", rmodel.loss_conjugate_at_neg(kind, zeta, y))
                put(f"loss/{idx}/zeta_bad", zeta_bad)
                put(f"loss/{idx}/conj_bad", rmodel.loss_conjugate_at_neg(kind, zeta_bad, y))
                idx += 1
    META["n_loss"] = idx


def gen_lipschitz_and_bounds():
    rng = np.random.default_rng(5)
    idx = 0
    for (n, p, loss) in [(1, 1, "squared_error"), (2, 2, "squared_error"), (30, 10, "logistic"),
                         (60, 40, "squared_error"), (40, 60, "squared_hinge"), (200, 50, "logistic")]:
        X = rng.standard_normal((n, p))
        if n == p == 2:
            X = np.diag([1.0, 2.0])
        y = rng.standard_normal(n) if loss == "squared_error" else rng.choice([-1.0, 1.0], n)
        k = max(1, p // 4)
        inst = rmodel.ProblemInstance(X=X, y=y, loss=rmodel.LossKind(loss), k=k, M=2.0, lambda2=0.3)
        try:
            L = rmodel.lipschitz_constant(inst)
        except l0cert.NumericalError:
            L = float("nan")
        put(f"lip/{idx}/X", X)
        put(f"lip/{idx}/y", y)
        put(f"lip/{idx}/args", [["squared_error", "logistic", "squared_hinge"].index(loss), k, 2.0, 0.3])
        put(f"lip/{idx}/L", L)
        bounds = []
        betas = []
        nodes = []
        for r in range(4):
            beta = rng.standard_normal(p) * 0.5
            node = None
            if r >= 2 and p >= 4:
                node = rmodel.NodeState(fixed_one=(0,), fixed_zero=(1, 2))
            bounds.append(rpersp.safe_lower_bound(inst, beta, node))
            betas.append(beta)
            nodes.append(node is not None)
        put(f"lip/{idx}/betas", np.asarray(betas))
        put(f"lip/{idx}/nodes", np.asarray(nodes))
        put(f"lip/{idx}/bounds", np.asarray(bounds))
        idx += 1
    META["n_lip"] = idx


def run_ref_solve(X, y, loss, k, M, lam2, L, node=None, warm=None, **opts):
    inst = rmodel.ProblemInstance(X=X, y=y, loss=rmodel.LossKind(loss), k=k, M=M, lambda2=lam2)
    rec = []
    o = rfista.FistaOptions(lipschitz=L, trace_hook=rec.append, **opts)
    rep = rfista.solve_relaxation(inst, node=node, warm_start=warm, opts=o)
    trace = np.asarray([[r["iteration"], r["primal"], r["dual"], r["gap"], float(r["restarted"])]
                        for r in rec]).reshape(-1, 5)
    return rep, trace


def store_traj(name, rep, trace, L, spec):
    put(f"traj/{name}/beta", rep.beta)
    put(f"traj/{name}/scalars", [rep.primal_value, rep.dual_bound, rep.gap, rep.iterations,
                                 rep.restarts, L])
    put(f"traj/{name}/trace", trace)
    META["cases"][name] = dict(spec, termination=rep.termination.value)
    print(f"  {name}: it={rep.iterations} restarts={rep.restarts} term={rep.termination.value} "
          f"primal={rep.primal_value:.12g} dual={rep.dual_bound:.12g}")


def gen_trajectories():
    # SPEC.md:269-272 known answers
    for name, X, y, k, M in [("spec_1d", np.array([[1.0]]), np.array([1.0]), 1, 2.0),
                             ("spec_2x2", np.eye(2), np.array([1.0, 1.0]), 2, 10.0),
                             ("spec_y0", np.eye(3), np.zeros(3), 2, 2.0)]:
        inst = rmodel.ProblemInstance(X=X, y=y, loss=rmodel.LossKind.SQUARED_ERROR, k=k, M=M, lambda2=1.0)
        L = rmodel.lipschitz_constant(inst)
        rep, trace = run_ref_solve(X, y, "squared_error", k, M, 1.0, L)
        put(f"traj/{name}/X", X)
        put(f"traj/{name}/y", y)
        store_traj(name, rep, trace, L, {"gen": "inline", "loss": "squared_error", "k": k, "M": M,
                                         "lambda2": 1.0, "opts": {}})

    def cfg_case(name, cfg_name, scale, opts, node_spec=None, warm_seed=None, extra=None):
        cd = mydata.make_config(cfg_name, scale=scale)
        X = cd.X.astype(np.float64)
        L = lanczos_L(X, cd.loss)
        node = None
        if node_spec is not None:
            node = rmodel.NodeState(fixed_one=node_spec[1], fixed_zero=node_spec[0],
                                    parent_bound=node_spec[2] if len(node_spec) > 2 else -np.inf)
        warm = None
        if warm_seed is not None:
            warm = np.random.default_rng(warm_seed).standard_normal(cd.p) * 0.05
            if node is not None:
                warm[list(node.fixed_zero)] = 0.0
        rep, trace = run_ref_solve(X, cd.y, cd.loss, cd.k, cd.M, cd.lambda2, L, node=node,
                                   warm=warm, **opts)
        put(f"traj/{name}/xsha", np.frombuffer(bytes.fromhex(sha(cd.X)), dtype=np.uint8))
        spec = {"gen": "config", "config": cfg_name, "scale": scale, "loss": cd.loss, "k": cd.k,
                "M": cd.M, "lambda2": cd.lambda2, "opts": opts, "node": node_spec,
                "warm_seed": warm_seed}
        if extra:
            spec.update(extra)
        store_traj(name, rep, trace, L, spec)

    cfg_case("c1", "C1", 1.0, {"max_iterations": 1000, "gap_tolerance": 1e-300})
    cfg_case("c1_default_tol", "C1", 1.0, {"max_iterations": 1000})
    cfg_case("c1_literal", "C1-literal", 1.0, {"max_iterations": 1000})
    cfg_case("c1_norestart", "C1", 0.5, {"max_iterations": 300, "gap_tolerance": 1e-300,
                                         "restart": False})
    cfg_case("c2_small", "C2", 1.0 / 16, {"max_iterations": 2000})
    cfg_case("c3_small", "C3", 1.0 / 20, {"max_iterations": 300, "gap_tolerance": 1e-300})
    cfg_case("c3_small_bci7", "C3", 1.0 / 20, {"max_iterations": 120, "gap_tolerance": 1e-300,
                                               "bound_check_interval": 7})
    nodes = mydata.random_nodes(250, 3, seed=1)
    for i, (fz, fo) in enumerate(nodes):
        cfg_case(f"c4_node{i}", "C4", 0.05, {"max_iterations": 200, "gap_tolerance": 1e-300},
                 node_spec=(fz, fo))
    cfg_case("c4_node_warm", "C4", 0.05, {"max_iterations": 150}, node_spec=((3, 7), (11,), -1e9),
             warm_seed=3)
    cfg_case("c4_primal_cut", "C4", 0.05, {"max_iterations": 400, "early_primal_cutoff": 17700.0},
             node_spec=((), (5,)))
    cfg_case("c4_dual_cut", "C4", 0.05, {"max_iterations": 400, "early_dual_cutoff": 17300.0})


def main():
    import threadpoolctl
    with threadpoolctl.threadpool_limits(1):
        # the generator must reproduce l0cert.data bit for bit
        inst = rdata.generate_synthetic(rdata.SyntheticParams(n=300, p=120, k_true=7, sigma=0.6, seed=3))
        X, y, _ = mydata.synthetic(300, 120, 7, sigma=0.6, seed=3)
        assert np.array_equal(inst.X, X) and np.array_equal(inst.y, y)
        assert np.array_equal(rdata.standardize(X)[0], mydata.standardize(X)[0])
        print("prox"); gen_prox()
        print("node prox"); gen_node_prox()
        print("envelope"); gen_envelope()
        print("losses"); gen_losses()
        print("lipschitz/bounds"); gen_lipschitz_and_bounds()
        print("trajectories"); gen_trajectories()
    META["blas_threads"] = 1
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **OUT)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(META, fh, indent=1, sort_keys=True)
    print("wrote", len(OUT), "arrays")


if __name__ == "__main__":
    main()
