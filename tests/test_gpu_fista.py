"""Trajectory-level parity of the B200 solve_relaxation.

Every case runs the drop-in API on the GPU and compares with the reference's
own trajectory (golden fixture, same injected L) and with the CPU oracle:

* before the plateau (relative gap >= 1e-6): objective within 1e-12 and dual
  bound within 1e-9 relative at every bound check (fp64 and fp32-storage
  modes), final beta within 1e-9 * max|beta|, identical iteration count and
  termination;
* on the plateau the reference's own restart/stop tests compare ulp-equal
  objectives (it disagrees with itself between BLAS thread
  counts), so values must agree to within the runs' gaps, beta to 1e-6, and
  the stopping iteration may differ;
* identical support {|beta_j| > 1e-9 M} always.
"""

import math

import numpy as np
import pytest

from paper_2502_09502_b200 import data as mydata

pytestmark = pytest.mark.gpu


def _instance(engine, golden, name, dtype="fp64"):
    data, meta = golden
    spec = meta["cases"][name]
    if spec["gen"] == "inline":
        X, y = data[f"traj/{name}/X"], data[f"traj/{name}/y"]
    else:
        cd = mydata.make_config(spec["config"], scale=spec["scale"])
        X, y = cd.X, cd.y
        if dtype == "fp64":
            X = X.astype(np.float64)
    inst = engine.ProblemInstance(X, y, engine.LossKind(spec["loss"]), spec["k"], spec["M"],
                                  spec["lambda2"], dtype=dtype)
    return spec, inst


def _solve(engine, spec, inst, L, **extra):
    opts = dict(spec["opts"])
    node = None
    if spec.get("node"):
        nz = spec["node"]
        node = engine.NodeState(fixed_one=tuple(nz[1]), fixed_zero=tuple(nz[0]),
                                parent_bound=nz[2] if len(nz) > 2 else -np.inf)
    warm = None
    if spec.get("warm_seed") is not None:
        warm = np.random.default_rng(spec["warm_seed"]).standard_normal(inst.p) * 0.05
        warm[list(node.fixed_zero)] = 0.0
    rec = []
    o = engine.FistaOptions(lipschitz=L, trace_hook=rec.append, **opts, **extra)
    rep = engine.solve_relaxation(inst, node=node, warm_start=warm, opts=o)
    return rep, rec


PLATEAU = 1e-6   # relative gap below which restart tests may flip


def _rel(gap, primal):
    return abs(gap) / max(1.0, abs(primal))


def _close_or_within_gap(ours, ref, gap_o, gap_r, rtol):
    """Pre-plateau: relative agreement.  On the plateau both runs are within
    their own gaps of the optimum, so they agree to max(gap)."""
    if math.isinf(ref) or math.isinf(ours):
        assert ours == ref
        return
    slack = max(abs(gap_o), abs(gap_r)) + rtol * max(1.0, abs(ref))
    assert abs(ours - ref) <= slack, (ours, ref, slack)


def _compare(rep, rec, trace, scalars, ref_beta, spec, dual_rtol=1e-9):
    """Plateau-aware parity: once the relative gap is
    below 1e-6 the reference's own restart/stop decisions compare ulp-equal
    objectives and flip between BLAS thread counts; before that everything
    must agree (objective 1e-12, bound 1e-9 relative, beta 1e-9)."""
    primal, dual, gap, iters, restarts, L = scalars
    plateau = _rel(gap, primal) <= PLATEAU and _rel(rep.gap, rep.primal_value) <= PLATEAU
    same_stop = rep.termination.value == spec["termination"] and rep.iterations == int(iters)
    if not same_stop:
        assert plateau, (rep.termination, rep.iterations, spec["termination"], int(iters),
                         rep.gap, gap)
    common = min(len(rec), trace.shape[0])
    if same_stop:
        assert len(rec) == trace.shape[0]
    for r, ref in zip(rec[:common], trace[:common]):
        assert r["iteration"] == int(ref[0])
        if not math.isfinite(ref[2]):
            assert not math.isfinite(r["dual"])
            assert r["primal"] == pytest.approx(ref[1], rel=1e-12, abs=1e-12)
        elif _rel(ref[3], ref[1]) >= PLATEAU:
            assert r["primal"] == pytest.approx(ref[1], rel=1e-12, abs=1e-12)
            assert r["dual"] == pytest.approx(ref[2], rel=dual_rtol, abs=1e-9)
        else:
            _close_or_within_gap(r["primal"], ref[1], r["gap"], ref[3], 1e-12)
            _close_or_within_gap(r["dual"], ref[2], r["gap"], ref[3], dual_rtol)
    if plateau:
        _close_or_within_gap(rep.primal_value, primal, rep.gap, gap, 1e-12)
        _close_or_within_gap(rep.dual_bound, dual, rep.gap, gap, dual_rtol)
    else:
        assert rep.primal_value == pytest.approx(primal, rel=1e-12, abs=1e-12)
        if math.isfinite(dual):
            assert rep.dual_bound == pytest.approx(dual, rel=dual_rtol, abs=1e-9)
    scale = max(1.0, float(np.max(np.abs(ref_beta))))
    # post-plateau restart flips move beta transiently (survey: <= 2.4e-7 relative)
    tol = 1e-6 if plateau else 1e-9
    np.testing.assert_allclose(rep.beta, ref_beta, rtol=0, atol=tol * scale)
    M = spec["M"]
    assert np.array_equal(np.abs(rep.beta) > 1e-9 * M, np.abs(ref_beta) > 1e-9 * M)


TRAJ = ["spec_1d", "spec_2x2", "spec_y0", "c1", "c1_default_tol", "c1_literal", "c1_norestart",
        "c2_small", "c3_small", "c3_small_bci7", "c4_node0", "c4_node1", "c4_node2",
        "c4_node_warm", "c4_primal_cut", "c4_dual_cut"]


@pytest.mark.parametrize("name", TRAJ)
def test_trajectory_vs_reference(engine, golden, name):
    data, _ = golden
    spec, inst = _instance(engine, golden, name)
    scalars = data[f"traj/{name}/scalars"]
    rep, rec = _solve(engine, spec, inst, float(scalars[5]))
    _compare(rep, rec, data[f"traj/{name}/trace"], scalars, data[f"traj/{name}/beta"], spec)


@pytest.mark.parametrize("name", ["c3_small", "c4_node0", "c4_node_warm"])
def test_fp32_storage_mode_matches(engine, golden, name):
    """fp32 X storage + fp64 arithmetic reproduces the fp64 solve on the
    fp64-widened matrix (the golden was produced on X32.astype(float64))."""
    data, meta = golden
    if meta["cases"][name]["gen"] != "config":
        pytest.skip("inline case")
    spec, inst = _instance(engine, golden, name, dtype="fp32")
    scalars = data[f"traj/{name}/scalars"]
    rep, rec = _solve(engine, spec, inst, float(scalars[5]))
    _compare(rep, rec, data[f"traj/{name}/trace"], scalars, data[f"traj/{name}/beta"], spec)


def test_spec_known_answers(engine):
    SE = engine.LossKind.SQUARED_ERROR
    inst = engine.ProblemInstance(np.array([[1.0]]), np.array([1.0]), SE, 1, 2.0, 1.0)
    rep = engine.solve_relaxation(inst)
    assert rep.primal_value == pytest.approx(0.5, abs=1e-6) and rep.gap <= 1e-6
    inst = engine.ProblemInstance(np.eye(2), np.array([1.0, 1.0]), SE, 2, 10.0, 1.0)
    rep = engine.solve_relaxation(inst)
    assert rep.primal_value == pytest.approx(1.0, abs=1e-6)
    np.testing.assert_allclose(rep.beta, [0.5, 0.5], atol=1e-6)
    inst = engine.ProblemInstance(np.eye(3), np.zeros(3), SE, 2, 2.0, 1.0)
    rep = engine.solve_relaxation(inst)
    assert rep.iterations == 1 and np.all(rep.beta == 0.0) and rep.gap == 0.0


def test_lockstep_iterates_vs_oracle(engine, oracle):
    """beta_t after exactly t iterations equals the oracle's beta_t (pre-plateau)."""
    cd = mydata.make_config("C1", scale=0.5)
    L = 2.0 * 1.01 * float(np.linalg.eigvalsh(cd.X.T @ cd.X)[-1])
    inst = engine.ProblemInstance(cd.X, cd.y, engine.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
    seen = {}

    def keep(t, beta, obj, restarted):
        seen[t] = (beta.copy(), obj, restarted)

    oracle.fista(cd.X, cd.y, cd.loss, cd.k, cd.M, cd.lambda2, L=L, max_iter=40, gap_tol=1e-300,
                 on_iteration=keep)
    for t in (1, 2, 3, 7, 15, 40):
        rep = engine.solve_relaxation(inst, opts=engine.FistaOptions(
            lipschitz=L, max_iterations=t, gap_tolerance=1e-300))
        ref_beta, ref_obj, _ = seen[t]
        assert rep.iterations == t
        assert rep.primal_value == pytest.approx(ref_obj, rel=1e-12)
        np.testing.assert_allclose(rep.beta, ref_beta, rtol=0, atol=1e-10 * np.max(np.abs(ref_beta)))


def test_numerical_error_on_bad_step(engine, oracle):
    """A step constant far below the true L drives the loss to overflow:
    NumericalError carrying the iteration (fista.py:167-172)."""
    # checked against the reference: NumericalError(iteration=1)
    X = 1e155 * np.eye(3)
    y = np.ones(3)
    with pytest.raises(oracle.PowerIterationError) as ref_err:
        oracle.fista(X, y, "squared_error", 2, 2.0, 1.0, L=1e155, max_iter=50)
    inst = engine.ProblemInstance(X, y, engine.LossKind.SQUARED_ERROR, 2, 2.0, 1.0)
    with pytest.raises(engine.NumericalError) as err:
        engine.solve_relaxation(inst, opts=engine.FistaOptions(lipschitz=1e155, max_iterations=50))
    assert err.value.iteration == ref_err.value.iteration == 1


def test_invalid_predictions_raise(engine):
    """Non-finite predictions surface as InvalidInputError (model.py:152-156, :215)."""
    # checked against the reference: X @ beta overflows -> InvalidInputError
    X = 1e308 * np.eye(3)
    inst = engine.ProblemInstance(X, np.ones(3), engine.LossKind.SQUARED_ERROR, 2, 2.0, 1.0)
    with pytest.raises(engine.InvalidInputError):
        engine.solve_relaxation(inst, opts=engine.FistaOptions(lipschitz=1e308, max_iterations=5))


def test_time_limit_and_hook_exception(engine):
    cd = mydata.make_config("C1", scale=0.5)
    inst = engine.ProblemInstance(cd.X, cd.y, engine.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
    rep = engine.solve_relaxation(inst, opts=engine.FistaOptions(
        lipschitz=1e4, max_iterations=10**6, gap_tolerance=1e-300, time_limit=0.05))
    assert rep.termination is engine.Termination.TIME_LIMIT
    assert rep.iterations > 0 and math.isfinite(rep.dual_bound)

    class Stop(Exception):
        pass

    def hook(r):
        if r["iteration"] >= 20:
            raise Stop()

    with pytest.raises(Stop):
        engine.solve_relaxation(inst, opts=engine.FistaOptions(lipschitz=1e4, trace_hook=hook,
                                                                gap_tolerance=1e-300))


def test_solver_validation_errors(engine):
    SE = engine.LossKind.SQUARED_ERROR
    inst = engine.ProblemInstance(np.eye(3), np.ones(3), SE, 2, 2.0, 1.0)
    with pytest.raises(engine.InvalidInputError):
        engine.solve_relaxation(inst, warm_start=np.zeros(2), opts=engine.FistaOptions(lipschitz=2.0))
    with pytest.raises(engine.InfeasibleNodeError):
        engine.solve_relaxation(inst, node=engine.NodeState(fixed_one=(0, 1, 2)),
                                opts=engine.FistaOptions(lipschitz=2.0))
    with pytest.raises(engine.InvalidInputError):
        engine.FistaOptions(gap_tolerance=0.0)
    pois = engine.ProblemInstance(np.eye(2), np.ones(2), engine.LossKind.POISSON, 1, 1.0, 1.0)
    with pytest.raises(engine.UnsupportedOperationError):
        engine.solve_relaxation(pois)


@pytest.mark.parametrize("n,p,sigma,k", [(800, 12000, 0.7, 20), (500, 20000, 0.5, 15),
                                         (300, 40000, 0.7, 30)])
def test_wide_problems_vs_oracle(engine, oracle, n, p, sigma, k):
    """Wide X: the windowed prox sorts several windows at t=1 (pool end ~0.4 p)
    and must reproduce the oracle's full-sort trajectory."""
    X, y, _ = mydata.synthetic(n, p, k, sigma=sigma, snr=5.0, seed=7)
    s = np.linalg.svd(X, compute_uv=False)[0]
    L = 2.0 * 1.01 * s * s
    inst = engine.ProblemInstance(X, y, engine.LossKind.SQUARED_ERROR, k, 2.0, 0.1)
    pools = []
    orig = oracle.prox_conj

    def spy(mu, rho, kk, M, instrument=False):
        r, order, pool = orig(mu, rho, kk, M, instrument=True)
        pools.append(pool)
        return r

    oracle.prox_conj = spy
    try:
        ref = oracle.fista(X, y, "squared_error", k, 2.0, 0.1, L=L, max_iter=25, gap_tol=1e-300)
    finally:
        oracle.prox_conj = orig
    assert pools[0] is not None
    rep = engine.solve_relaxation(inst, opts=engine.FistaOptions(lipschitz=L, max_iterations=25,
                                                                 gap_tolerance=1e-300))
    assert rep.iterations == 25
    assert rep.primal_value == pytest.approx(ref["primal_value"], rel=1e-12)
    assert rep.dual_bound == pytest.approx(ref["dual_bound"], rel=1e-9)
    np.testing.assert_allclose(rep.beta, ref["beta"], rtol=0, atol=1e-10 * np.max(np.abs(ref["beta"])))
    assert rep.stats["topk_fallbacks"] >= 0


@pytest.mark.parametrize("case", ["C1", "C2s", "C3s", "C4node", "C5s"])
def test_single_pass_engine_matches_two_pass(engine, case):
    """The fused single-pass kernel (K3 -> KF -> KR) and the two-pass engine
    (K2 -> K3 -> K1) run the same algorithm; pre-plateau they agree to
    summation-order rounding."""
    node = None
    dtype = "fp64"
    if case == "C1":
        cd = mydata.make_config("C1", scale=0.5)
    elif case == "C2s":
        cd = mydata.make_config("C2", scale=1 / 8)
    elif case == "C3s":
        cd = mydata.make_config("C3", scale=1 / 10)
        dtype = "fp32"
    elif case == "C5s":
        cd = mydata.make_config("C5", scale=0.02)
        dtype = "fp32"
    else:
        cd = mydata.make_config("C4", scale=0.1)
        dtype = "fp32"
        fz, fo = cd.nodes[5]
        node = engine.NodeState(fixed_one=fo, fixed_zero=fz)
    X = cd.X if dtype == "fp32" else cd.X.astype(np.float64)
    inst = engine.ProblemInstance(X, cd.y, engine.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=dtype)
    curv = 0.25 if cd.loss == "logistic" else 2.0
    L = curv * 1.01 * float(np.linalg.norm(X.astype(np.float64), 2) ** 2)
    res = {}
    for path in ("two_pass", "single_pass"):
        rec = []
        res[path] = (engine.solve_relaxation(inst, node=node, opts=engine.FistaOptions(
            lipschitz=L, max_iterations=40, gap_tolerance=1e-300, engine_path=path,
            trace_hook=rec.append)), rec)
    (a, ra), (b, rb) = res["two_pass"], res["single_pass"]
    assert b.stats["single_pass"] and not a.stats["single_pass"]
    assert a.iterations == b.iterations == 40
    assert b.primal_value == pytest.approx(a.primal_value, rel=1e-12)
    assert b.dual_bound == pytest.approx(a.dual_bound, rel=1e-9)
    for x, y in zip(ra, rb):
        assert y["primal"] == pytest.approx(x["primal"], rel=1e-12)
    np.testing.assert_allclose(b.beta, a.beta, rtol=0, atol=1e-10 * max(1.0, np.max(np.abs(a.beta))))


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,dtype,loss", [
    (1001, 3001, "fp64", "squared_error"),    # LIN, 1-row x 3072-column tiles (6 vectors per thread), no
                                              # cluster; odd n: y / u_{t-1} loaded per row; odd p: padded columns
    (7, 5, "fp64", "squared_error"),          # one partial tile, one CTA per cluster
    (301, 20000, "fp64", "logistic"),         # 16-CTA (non-portable) clusters, 3 vectors per thread
    (300, 20001, "fp64", "squared_error"),    # LIN, 1-row tiles in clusters of 8, 5 vectors per thread
    (1000, 1500, "fp64", "squared_error"),    # LIN, 2-row tiles, no cluster
    (999, 5003, "fp32", "logistic"),          # fp32 X, odd n, partial last tile; SPEC kernel, no cluster
    (640, 11000, "fp32", "logistic"),         # SPEC kernel (one vector + conditional K2), clusters of 2
    (777, 9001, "fp32", "squared_error"),     # LIN kernel on fp32 X, clusters of 2, 5 vectors per thread
    (2048, 9000, "fp64", "logistic"),         # 8-CTA clusters, last CTA's slice partly past p
    (1500, 4100, "fp64", "squared_hinge"),    # the third solver-grade loss through the gather warps
])
def test_single_pass_edge_shapes(engine, n, p, dtype, loss):
    """kf_fused_s on ragged shapes (odd rows, partial last tile, slices past p,
    every cluster size the plan can pick) against the two-pass engine."""
    rng = np.random.default_rng(n * 7 + p)
    X = rng.standard_normal((n, p))
    if dtype == "fp32":
        X = X.astype(np.float32)
    beta_true = np.zeros(p)
    beta_true[:: max(1, p // 5)] = 1.0
    u = X.astype(np.float64) @ beta_true
    if loss in ("logistic", "squared_hinge"):
        y = np.where(rng.random(n) < 1.0 / (1.0 + np.exp(-u)), 1.0, -1.0)
    else:
        y = u + rng.standard_normal(n)
    k = min(5, p)
    inst = engine.ProblemInstance(X, y, engine.LossKind(loss), k, 2.0, 0.5, dtype=dtype)
    curv = 0.25 if loss == "logistic" else 2.0
    L = curv * 1.01 * float(np.linalg.norm(X.astype(np.float64), 2) ** 2)
    res = {}
    for path in ("two_pass", "single_pass"):
        rec = []
        res[path] = (engine.solve_relaxation(inst, opts=engine.FistaOptions(
            lipschitz=L, max_iterations=30, gap_tolerance=1e-300, engine_path=path,
            trace_hook=rec.append)), rec)
    (a, ra), (b, rb) = res["two_pass"], res["single_pass"]
    assert b.stats["single_pass"] and not a.stats["single_pass"]
    assert b.stats["cluster_size"] == {3001: 1, 5: 1, 20000: 16, 20001: 8, 1500: 1, 5003: 1,
                                          11000: 2, 9001: 2, 9000: 8, 4100: 4}[p]
    assert a.iterations == b.iterations == 30
    assert b.primal_value == pytest.approx(a.primal_value, rel=1e-12)
    assert b.dual_bound == pytest.approx(a.dual_bound, rel=1e-9, abs=1e-12)
    for x, y_ in zip(ra, rb):
        assert y_["primal"] == pytest.approx(x["primal"], rel=1e-12)
    np.testing.assert_allclose(b.beta, a.beta, rtol=0, atol=1e-10 * max(1.0, np.max(np.abs(a.beta))))


@pytest.mark.gpu
def test_k3_variants_agree(engine, monkeypatch):
    """The windowed K3 (pinned, L0_FULL_SORT=0), the full key sort (pinned, =1)
    and the automatic switch (unset: window first, full sort once a chunk's
    pools keep reaching past the window) run the same exact prox: identical
    trajectories on a C3-like problem whose PAVA pool spans most of p."""
    cd = mydata.make_config("C3", scale=1 / 10)
    inst = engine.ProblemInstance(cd.X, cd.y, engine.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype="fp32")
    L = 0.25 * 1.01 * float(np.linalg.norm(cd.X.astype(np.float64), 2) ** 2)
    res = {}
    for mode in ("0", "1", None):
        if mode is None:
            monkeypatch.delenv("L0_FULL_SORT", raising=False)
        else:
            monkeypatch.setenv("L0_FULL_SORT", mode)
        rec = []
        res[mode] = (engine.solve_relaxation(inst, opts=engine.FistaOptions(
            lipschitz=L, max_iterations=60, gap_tolerance=1e-300, chunk_iterations=4,
            trace_hook=rec.append)), rec)
    a, ra = res["0"]
    for mode in ("1", None):
        b, rb = res[mode]
        assert b.iterations == a.iterations == 60
        assert b.restarts == a.restarts
        assert b.primal_value == pytest.approx(a.primal_value, rel=1e-12)
        assert b.dual_bound == pytest.approx(a.dual_bound, rel=1e-9)
        for x, y_ in zip(ra, rb):
            assert y_["primal"] == pytest.approx(x["primal"], rel=1e-12)
        np.testing.assert_allclose(b.beta, a.beta, rtol=0, atol=1e-10 * max(1.0, np.max(np.abs(a.beta))))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["C3", "C5", "C2", "hinge", "time_limit"])
def test_single_pass_kernel_variants_agree(engine, monkeypatch, case):
    """The one-vector single-pass kernels -- LIN (squared error: both momentum
    candidates and X^T zeta from A_t = X^T grad F(u_t) by linearity) and SPEC
    (non-linear loss on fp32 X: the no-restart candidate, plus X^T zeta in the
    two-vector kernel of bound-check iterations; restarts and bound-only passes
    through the conditional K2 launch) -- against the three-vector
    kernel they replace (L0_FZ_LIN=0 / L0_FZ_SPEC=0) and the two-pass engine:
    same iterations, restarts and termination, values to summation order."""
    kw = {}
    if case in ("C3", "time_limit"):
        cd = mydata.make_config("C3", scale=1 / 10)
        X, curv, var = cd.X, 0.25, "L0_FZ_SPEC"
    elif case == "hinge":
        cd = mydata.make_config("C3", scale=1 / 12)
        cd.loss = "squared_hinge"
        X, curv, var = cd.X, 2.0, "L0_FZ_SPEC"
    elif case == "C5":
        cd = mydata.make_config("C5", scale=1 / 200)
        X, curv, var = cd.X, 2.0, "L0_FZ_LIN"
    else:
        cd = mydata.make_config("C2", scale=1 / 8)
        X, curv, var = cd.X, 2.0, "L0_FZ_LIN"
    L = curv * 1.01 * float(np.linalg.norm(X.astype(np.float64), 2) ** 2)
    # the small squared-error problems reach their round-off plateau (where
    # restart decisions compare ulp-equal objectives) within ~100 iterations
    iters = 150 if var == "L0_FZ_SPEC" else 60
    if var == "L0_FZ_LIN":
        L *= 0.55   # over-long steps: the momentum overshoots and the restart rule fires early
    res = {}
    modes = ("two_pass", "0", "1") + (("k2z",) if var == "L0_FZ_SPEC" else ())
    for mode in modes:
        monkeypatch.setenv(var, "0" if mode == "0" else "1")
        # "k2z": SPEC without the two-vector bound-check kernel (X^T zeta from the conditional K2)
        monkeypatch.setenv("L0_FZ_SPEC2", "0" if mode == "k2z" else "1")
        # a fresh instance per variant: the plan is fixed when the device problem is created
        inst = engine.ProblemInstance(X, cd.y, engine.LossKind(cd.loss), cd.k, cd.M, cd.lambda2,
                                      dtype=cd.dtype)
        rec = []
        if case == "time_limit":
            # the stop request between chunks re-runs the fused tail (KR and,
            # for SPEC, the conditional transpose launch)
            kw = dict(time_limit=0.0, chunk_iterations=3, bound_check_interval=1000)
        rep = engine.solve_relaxation(inst, opts=engine.FistaOptions(
            lipschitz=L, max_iterations=iters, gap_tolerance=1e-300,
            engine_path="two_pass" if mode == "two_pass" else "single_pass", trace_hook=rec.append, **kw))
        res[mode] = (rep, rec)
        assert rep.stats["single_pass"] == (mode != "two_pass")
    a, ra = res["two_pass"]
    if case == "time_limit":
        for mode in modes[1:]:
            b, _ = res[mode]
            assert b.termination == engine.Termination.TIME_LIMIT
            assert np.isfinite(b.dual_bound) and b.dual_bound <= b.primal_value + 1e-9 * abs(b.primal_value)
        return
    assert a.restarts > 0 or case == "hinge"
    for mode in modes[1:]:
        b, rb = res[mode]
        assert b.iterations == a.iterations == iters
        assert b.restarts == a.restarts and b.termination == a.termination
        assert b.primal_value == pytest.approx(a.primal_value, rel=1e-12)
        assert b.dual_bound == pytest.approx(a.dual_bound, rel=1e-9)
        assert len(rb) == len(ra)
        for x, y_ in zip(ra, rb):
            assert y_["primal"] == pytest.approx(x["primal"], rel=1e-12)
            assert y_["dual"] == pytest.approx(x["dual"], rel=1e-9)
            assert y_["restarted"] == x["restarted"]
        np.testing.assert_allclose(b.beta, a.beta, rtol=0, atol=1e-10 * max(1.0, np.max(np.abs(a.beta))))


@pytest.mark.gpu
@pytest.mark.parametrize("stop", ["converged", "primal_cutoff", "dual_cutoff", "iteration_limit_check",
                                  "warm_node"])
def test_single_pass_stopping_rules(engine, stop):
    """Termination paths of the single-pass engine (K3 bound checks, the
    objective's cutoffs, the final bound pass) against the two-pass engine."""
    cd = mydata.make_config("C2", scale=1 / 8)
    inst = engine.ProblemInstance(cd.X, cd.y, engine.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
    L = 2.0 * 1.01 * float(np.linalg.norm(cd.X, 2) ** 2)
    base = engine.solve_relaxation(inst, opts=engine.FistaOptions(lipschitz=L, max_iterations=60,
                                                                  gap_tolerance=1e-300))
    kw = {"lipschitz": L}
    if stop == "converged":
        kw.update(max_iterations=5000, gap_tolerance=1e-4 * abs(base.primal_value))
    elif stop == "primal_cutoff":
        kw.update(max_iterations=5000, early_primal_cutoff=base.primal_value * (1 + 1e-3))
    elif stop == "dual_cutoff":
        kw.update(max_iterations=5000, early_dual_cutoff=base.dual_bound * (1 - 1e-3))
    elif stop == "warm_node":
        kw.update(max_iterations=5000, gap_tolerance=1e-4 * abs(base.primal_value))
    else:
        kw.update(max_iterations=37, gap_tolerance=1e-300)   # stops between bound checks
    node, warm = None, None
    if stop == "warm_node":   # a branch-and-bound child warm-started from its parent's iterate
        order = np.argsort(-np.abs(base.beta))
        node = engine.NodeState(fixed_one=(int(order[0]),), fixed_zero=(int(order[1]), int(order[-1])),
                                parent_bound=base.dual_bound)
        warm = base.beta.copy()
        warm[[int(order[1]), int(order[-1])]] = 0.0
    res = {}
    for path in ("two_pass", "single_pass"):
        rec = []
        res[path] = (engine.solve_relaxation(inst, node=node, warm_start=warm, opts=engine.FistaOptions(
            engine_path=path, trace_hook=rec.append, **kw)), rec)
    (a, ra), (b, rb) = res["two_pass"], res["single_pass"]
    assert b.stats["single_pass"] and not a.stats["single_pass"]
    assert b.termination == a.termination
    assert a.termination.value == {"converged": "converged", "primal_cutoff": "primal_below_incumbent",
                                   "dual_cutoff": "dual_above_incumbent",
                                   "iteration_limit_check": "iteration_limit", "warm_node": "converged"}[stop]
    assert b.iterations == a.iterations
    assert b.primal_value == pytest.approx(a.primal_value, rel=1e-12)
    assert b.dual_bound == pytest.approx(a.dual_bound, rel=1e-9)
    assert len(ra) == len(rb)
    for x, y_ in zip(ra, rb):
        assert y_["iteration"] == x["iteration"]
        assert y_["primal"] == pytest.approx(x["primal"], rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_single_pass_time_limit(engine, dtype):
    """The host-side time limit on the single-pass engine: the solve stops
    between graph replays with TIME_LIMIT and a finite bound from the final
    bound pass at the last iterate (fista.py:204-209), weakly dual."""
    cd = mydata.make_config("C2", scale=1 / 8)
    X = cd.X.astype(np.float32) if dtype == "fp32" else cd.X
    inst = engine.ProblemInstance(X, cd.y, engine.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2, dtype=dtype)
    L = 2.0 * 1.01 * float(np.linalg.norm(X.astype(np.float64), 2) ** 2)
    rep = engine.solve_relaxation(inst, opts=engine.FistaOptions(
        lipschitz=L, max_iterations=10 ** 7, gap_tolerance=1e-300, time_limit=0.05,
        engine_path="single_pass"))
    assert rep.stats["single_pass"]
    assert rep.termination.value == "time_limit"
    assert 0 < rep.iterations < 10 ** 7
    assert np.isfinite(rep.dual_bound) and np.isfinite(rep.primal_value)
    assert rep.dual_bound <= rep.primal_value * (1 + 1e-12)
