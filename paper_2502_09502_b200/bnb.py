"""Branch-and-bound certification on top of the batched dual-bound engine.

The reference specifies this module (``bnb``) but ships no
code for it; SURVEY.md §8(f) ranks it first among the callers of the hot path.
Behaviour follows the spec:

* ``beam_search_incumbent``: supports grown one feature at a time from the
  node's fixed-one set, each candidate refit on the box-constrained
  ridge-regularised loss (squared error: the exact ridge solution when the
  box does not bind; otherwise projected gradient descent with a fixed
  budget), the ``beam_width`` best kept;
* ``select_branching_variable``: among the incumbent's unfixed nonzeros, the
  coordinate whose zeroing (no refit) raises the composite loss most;
* ``certify``: best-first search keyed by the parent bound (ties: deeper
  first, then insertion order), safe-bound pruning with the spec's 1e-8
  absolute + 1e-9 relative tolerance, children inherit the parent's bound.

B200 specifics: open nodes are evaluated in batches through
``solve_relaxation_batched`` (the spec's optional parallel mode: one stale
incumbent per batch, which keeps pruning sound) with ``early_primal_cutoff``
and ``early_dual_cutoff`` at the incumbent; every node's bound in the
certificate is then the fp64 ``safe_lower_bound`` at its final iterate (the
batched contraction is 3xTF32); the incumbent refits are batched exact ridge
solves on the GPU and the screening gradients ``X^T grad F`` use the engine's
transpose kernel.
"""

from __future__ import annotations

import dataclasses
import heapq
import math
import time
from dataclasses import dataclass, field
from enum import Enum
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .errors import InfeasibleNodeError, UnsupportedOperationError
from .fista import FistaOptions, Termination, solve_relaxation_batched
from .model import LossKind, NodeState, ProblemInstance, is_solver_grade, lipschitz_constant
from . import native
from .perspective import safe_lower_bound, safe_lower_bound_batched

__all__ = ["BnBOptions", "Certificate", "CertificateStatus", "beam_search_incumbent",
           "select_branching_variable", "certify"]

_CURV = {LossKind.SQUARED_ERROR: 2.0, LossKind.LOGISTIC: 0.25, LossKind.SQUARED_HINGE: 2.0}


class CertificateStatus(Enum):
    OPTIMAL = "optimal"
    GAP_LIMIT = "gap_limit"
    TIME_LIMIT = "time_limit"
    NODE_LIMIT = "node_limit"


@dataclass
class Certificate:
    """SPEC.md:306-309."""
    incumbent_beta: np.ndarray
    incumbent_objective: float
    global_lower_bound: float
    gap_absolute: float
    gap_relative: float
    nodes_explored: int
    wall_time: float
    status: CertificateStatus
    log: List[dict] = field(default_factory=list, repr=False)


@dataclass
class BnBOptions:
    gap_tolerance: float = 1e-4           # relative gap for OPTIMAL
    time_limit: float = math.inf
    node_limit: int = 100_000
    beam_width: int = 4
    batch_size: int = 64                  # open nodes per batched relaxation call
    refit_iterations: int = 300           # projected-gradient budget per candidate support
    prune_abs: float = 1e-8
    prune_rel: float = 1e-9
    relaxation: FistaOptions = field(default_factory=lambda: FistaOptions(max_iterations=2000))


# ---------------------------------------------------------------------------
# device helpers (torch on the engine's device; small per-support problems)
# ---------------------------------------------------------------------------
def _dev(instance: ProblemInstance):
    return instance.device_problem()


def _loss_and_grad(loss: LossKind, u, y):
    import torch
    if loss is LossKind.SQUARED_ERROR:
        r = u - y
        return (r * r).sum(-1), 2.0 * r
    if loss is LossKind.LOGISTIC:
        m = -y * u
        return torch.nn.functional.softplus(m).sum(-1), -y * torch.sigmoid(m)
    if loss is LossKind.SQUARED_HINGE:
        h = torch.clamp(1.0 - y * u, min=0.0)
        return (h * h).sum(-1), -2.0 * y * h
    raise UnsupportedOperationError(f"{loss.value} is not solver-grade")


_REFIT_MAX_S = 48   # csrc/refit.cu kRefitMaxS


def _refit(instance: ProblemInstance, supports: Sequence[Tuple[int, ...]], iters: int):
    """min F(X_S b) + l2 |b|^2, |b| <= M, for every support at once: squared
    error solves the ridge problems exactly on the device (l0_refit_ridge:
    batched Gram + Cholesky, one launch) and keeps them where the box does not
    bind; the rest (binding box, other losses) runs accelerated projected
    gradient.  Returns (list of dense betas, objectives)."""
    import torch
    dp = _dev(instance)
    p = instance.p
    C = len(supports)
    s = max(1, max(len(S) for S in supports))
    if instance.loss is LossKind.SQUARED_ERROR and s <= _REFIT_MAX_S:
        from . import _device
        sup = np.full((C, s), -1, dtype=np.int32)
        for c, S in enumerate(supports):
            sup[c, :len(S)] = S
        sup_d = torch.from_numpy(sup).to(dp.X.device)
        bd = torch.empty((C, s), dtype=torch.float64, device=dp.X.device)
        od = torch.empty(C, dtype=torch.float64, device=dp.X.device)
        if getattr(dp, "_yty", None) is None:
            dp._yty = float(torch.dot(dp.y, dp.y))
        native.check(native.lib().l0_refit_ridge(dp.handle, sup_d.data_ptr(), C, s, float(instance.lambda2),
                                                 dp._yty, bd.data_ptr(), od.data_ptr(),
                                                 _device.stream_handle()))
        bh, objs = bd.cpu().numpy(), od.cpu().numpy()
        viol = [c for c in range(C) if np.any(np.abs(bh[c]) > float(instance.M))]
        betas = []
        for c, S in enumerate(supports):
            beta = np.zeros(p)
            if S:
                beta[list(S)] = bh[c, :len(S)]
            betas.append(beta)
        if viol:   # the box binds: projected gradient from the clamped ridge point
            vb, vo = _refit_pg(instance, [supports[c] for c in viol], iters,
                               start=[np.clip(bh[c], -float(instance.M), float(instance.M)) for c in viol])
            for i, c in enumerate(viol):
                betas[c], objs[c] = vb[i], vo[i]
        return betas, objs
    return _refit_pg(instance, supports, iters)


def _refit_pg(instance: ProblemInstance, supports: Sequence[Tuple[int, ...]], iters: int, start=None):
    """Projected gradient descent of min F(X_S b) + l2 |b|^2, |b| <= M, for
    every support at once (squared error: exact ridge first, as the start)."""
    import torch
    dp = _dev(instance)
    p = instance.p
    C = len(supports)
    s = max(1, max(len(S) for S in supports))
    idx = torch.zeros((C, s), dtype=torch.long, device=dp.X.device)
    mask = torch.zeros((C, s), dtype=torch.float64, device=dp.X.device)
    for c, S in enumerate(supports):
        if S:
            idx[c, :len(S)] = torch.tensor(S, device=dp.X.device)
            mask[c, :len(S)] = 1.0
    n = dp.n
    Xs = dp.X[:, :p].index_select(1, idx.reshape(-1)).T.reshape(C, s, n).to(torch.float64)
    Xs = Xs * mask[:, :, None]                               # (C, s, n), padded columns zero
    y = dp.y[None, :]
    lam2, M = float(instance.lambda2), float(instance.M)
    L = _CURV[instance.loss] * (Xs * Xs).sum(dim=(1, 2)) + 2.0 * lam2 + 1e-12   # >= curvature
    b = torch.zeros((C, s), dtype=torch.float64, device=dp.X.device)
    todo = torch.ones(C, dtype=torch.bool, device=dp.X.device)
    if start is not None:
        for c, b0 in enumerate(start):
            b[c, :len(b0)] = torch.from_numpy(np.asarray(b0[:s], dtype=np.float64))
    elif instance.loss is LossKind.SQUARED_ERROR:
        # exact ridge solution per support; projected gradient only where the box binds
        G = torch.einsum("csn,ctn->cst", Xs, Xs) + lam2 * torch.eye(s, dtype=torch.float64,
                                                                     device=dp.X.device)
        G = G + torch.diag_embed(1.0 - mask)              # padded coordinates: identity rows
        rhs = torch.einsum("csn,n->cs", Xs, dp.y)
        b = torch.linalg.solve(G, rhs[:, :, None])[:, :, 0] * mask
        todo = (b.abs() > M).any(dim=1)
        b = torch.clamp(b, -M, M)
    if bool(todo.any()):
        # accelerated projected gradient (FISTA on the box) from the current point
        bt = b[todo]
        bp = bt.clone()
        Xt, Lt, mt = Xs[todo], L[todo], mask[todo]
        for it in range(iters):
            z = bt + ((it - 1.0) / (it + 2.0) if it > 0 else 0.0) * (bt - bp)
            u = torch.einsum("csn,cs->cn", Xt, z)
            _, g = _loss_and_grad(instance.loss, u, y)
            grad = torch.einsum("csn,cn->cs", Xt, g) + 2.0 * lam2 * z
            bp, bt = bt, torch.clamp(z - grad / Lt[:, None], -M, M) * mt
        b[todo] = bt
    u = torch.einsum("csn,cs->cn", Xs, b)
    f, _ = _loss_and_grad(instance.loss, u, y)
    obj = f + lam2 * (b * b).sum(-1)
    betas = []
    bh = b.cpu().numpy()
    for c, S in enumerate(supports):
        beta = np.zeros(p)
        if S:
            beta[list(S)] = bh[c, :len(S)]
        betas.append(beta)
    return betas, obj.cpu().numpy()


def _objective(instance: ProblemInstance, beta: np.ndarray) -> float:
    """F(X beta) + lambda2 |beta|^2 (the MIP objective)."""
    import torch
    dp = _dev(instance)
    u = dp.matvec(beta)
    f, _ = _loss_and_grad(instance.loss, u, dp.y)
    return float(f) + float(instance.lambda2) * float(np.dot(beta, beta))


def beam_search_incumbent(instance: ProblemInstance, node: Optional[NodeState] = None,
                          beam_width: int = 4, refit_iterations: int = 300):
    """a feasible solution with support >= fixed_one, disjoint
    from fixed_zero, at most k nonzeros and |beta| <= M.  Candidate features of
    a support are screened by |X^T grad F| at its refit (the engine's transpose
    kernel) before the batched refits."""
    node = node or NodeState()
    k, p = int(instance.k), instance.p
    f1 = tuple(sorted(node.fixed_one))
    if len(f1) > k:
        raise InfeasibleNodeError("|fixed_one| exceeds k")
    banned = set(node.fixed_zero) | set(f1)
    betas, objs = _refit(instance, [f1], refit_iterations)
    beam = [(float(objs[0]), f1, betas[0])]
    best = beam[0]
    dp = _dev(instance)
    for _ in range(k - len(f1)):
        cands = set()
        for obj, S, beta in beam:
            import torch
            u = dp.matvec(beta)
            _, g = _loss_and_grad(instance.loss, u, dp.y)
            score = np.abs(dp.rmatvec(g).cpu().numpy())
            if banned or S:
                score[list(banned | set(S))] = -1.0
            order = np.argsort(-score, kind="stable")[:beam_width]
            for j in order:
                if score[j] >= 0:
                    cands.add(tuple(sorted(S + (int(j),))))
        if not cands:
            break
        cands = sorted(cands)
        betas, objs = _refit(instance, cands, refit_iterations)
        scored = sorted(zip(objs.tolist(), range(len(cands))), key=lambda t: (t[0], t[1]))[:beam_width]
        beam = [(o, cands[i], betas[i]) for o, i in scored]
        if beam[0][0] < best[0]:
            best = beam[0]
    return best[2], best[0]


def select_branching_variable(instance: ProblemInstance, node: Optional[NodeState],
                              incumbent_beta: np.ndarray) -> Optional[int]:
    """the unfixed incumbent nonzero whose zeroing raises
    F(X beta) + lambda2 |beta|^2 most (no refit); None = node complete."""
    import torch
    node = node or NodeState()
    fixed = set(node.fixed_one) | set(node.fixed_zero)
    cand = [int(j) for j in np.flatnonzero(incumbent_beta) if int(j) not in fixed]
    if not cand:
        return None
    dp = _dev(instance)
    beta = np.asarray(incumbent_beta, dtype=np.float64)
    u = dp.matvec(beta)
    cols = dp.X[:, cand].to(torch.float64).T                   # (c, n)
    bj = torch.tensor(beta[cand], device=u.device)
    uz = u[None, :] - bj[:, None] * cols
    f, _ = _loss_and_grad(instance.loss, uz, dp.y[None, :])
    reg = float(instance.lambda2) * (float(np.dot(beta, beta)) - bj * bj)
    inc = (f + reg).cpu().numpy()
    return cand[int(np.argmax(inc))]        # first index on ties (stable)


def _beam_due(depth: int) -> bool:
    """every node at depth <= 3, then every 5th depth."""
    return depth <= 3 or depth % 5 == 0


def certify(instance: ProblemInstance, opts: Optional[BnBOptions] = None) -> Certificate:
    """SPEC.md:331-336, with open nodes evaluated in batches on the B200."""
    opts = opts or BnBOptions()
    if not is_solver_grade(instance.loss):
        raise UnsupportedOperationError(f"{instance.loss.value} is bound-grade")
    t0 = time.perf_counter()
    L = opts.relaxation.lipschitz if opts.relaxation.lipschitz is not None else lipschitz_constant(instance)
    inc_beta, inc_obj = beam_search_incumbent(instance, None, opts.beam_width, opts.refit_iterations)
    heap: list = []
    counter = 0

    def push(bound, node):
        nonlocal counter
        heapq.heappush(heap, (bound, -node.depth, counter, node))
        counter += 1

    push(-math.inf, NodeState())
    explored = 0
    log: List[dict] = []
    status = None

    def pruned(bound):
        return bound >= inc_obj - (opts.prune_abs + opts.prune_rel * abs(inc_obj))

    # bounds of nodes closed without being pruned (a leaf whose convex solve
    # did not reach the incumbent, a node with nothing left to branch on):
    # they stay in the global bound so the certificate remains sound
    unresolved: List[float] = []

    def glb():
        return min([inc_obj] + [b for b, _, _, _ in heap] + unresolved)

    while heap:
        if time.perf_counter() - t0 > opts.time_limit:
            status = CertificateStatus.TIME_LIMIT
            break
        if explored >= opts.node_limit:
            status = CertificateStatus.NODE_LIMIT
            break
        lb = glb()
        if inc_obj - lb <= opts.gap_tolerance * max(abs(inc_obj), 1e-12):
            status = CertificateStatus.OPTIMAL
            break
        batch = []
        while heap and len(batch) < min(opts.batch_size, opts.node_limit - explored):
            bound, _, _, node = heapq.heappop(heap)
            if pruned(bound):
                log.append({"node": None, "bound": bound, "decision": "prune(parent bound)"})
                continue
            if _is_leaf(instance, node):
                # every free coordinate must stay zero: the node is the convex
                # problem on its fixed-one support (the relaxation solver's prox
                # leaves ulp residues there that its envelope rejects, as the
                # reference's does) -> refit until its safe bound closes the
                # node; a node that stays open keeps its bound in glb()
                explored += 1
                b, o, lb_leaf = _solve_leaf(instance, node, bound, opts, inc_obj)
                if o < inc_obj:
                    inc_beta, inc_obj = b, o
                closed = pruned(lb_leaf)
                if not closed:
                    unresolved.append(lb_leaf)
                log.append({"depth": node.depth, "fixed_one": node.fixed_one,
                            "fixed_zero": node.fixed_zero, "bound": lb_leaf,
                            "decision": "leaf" if closed else "leaf (open)"})
                continue
            batch.append((bound, node))
        if not batch:
            continue
        # incumbents first (SPEC order), then the relaxations against them
        for _, node in batch:
            if node.depth > 0 and _beam_due(node.depth) and len(node.fixed_one) <= instance.k:
                b, o = beam_search_incumbent(instance, node, opts.beam_width, opts.refit_iterations)
                if o < inc_obj:
                    inc_beta, inc_obj = b, o
        ropts = dataclasses.replace(opts.relaxation, lipschitz=L, early_primal_cutoff=inc_obj,
                                    early_dual_cutoff=inc_obj, trace_hook=None)
        # fixed batch size (padding repeats the last node): one batched engine
        # (X split into TF32 operands once) serves the whole search
        nodes = [n for _, n in batch]
        nodes += [nodes[-1]] * (max(opts.batch_size, 1) - len(nodes))
        reps = solve_relaxation_batched(instance, nodes, opts=ropts)[:len(batch)]
        explored += len(batch)
        # the certificate uses the fp64 Fenchel bound at each node's final
        # iterate (perspective.py:162-190), all nodes of the batch in one
        # engine call (two fp64 multi-right-hand-side X passes): the batched
        # engine's own bound carries 3xTF32 rounding and only steers its
        # stopping tests
        safes = safe_lower_bound_batched(instance, np.stack([rep.beta for rep in reps]),
                                         [node for _, node in batch])
        for (pbound, node), rep, safe in zip(batch, reps, safes):
            bound = max(pbound, safe) if math.isfinite(safe) else pbound
            entry = {"depth": node.depth, "fixed_one": node.fixed_one, "fixed_zero": node.fixed_zero,
                     "bound": bound, "termination": rep.termination.value}
            if pruned(bound):
                entry["decision"] = "prune"
                log.append(entry)
                continue
            # branch on the node's own feasible point (its relaxation, projected
            # onto k largest free coordinates, refit) -- else the incumbent
            b_node, o_node = _node_point(instance, node, rep.beta, opts)
            if o_node < inc_obj:
                inc_beta, inc_obj = b_node, o_node
            j = select_branching_variable(instance, node, b_node)
            if j is None:
                # the node's feasible point uses only fixed coordinates: branch
                # on the relaxation's largest free coordinate instead
                j = _relaxation_branch(instance, node, rep.beta)
            if j is None:
                # nothing free is active: closed only if its bound prunes it
                # against the (possibly just improved) incumbent
                if pruned(bound):
                    entry["decision"] = "complete"
                else:
                    unresolved.append(bound)
                    entry["decision"] = "complete (open)"
                log.append(entry)
                continue
            entry["decision"] = f"branch {j}"
            log.append(entry)
            # children inherit the parent's relaxation beta, projected onto
            # their fixed-zero pattern, as warm start
            warm = np.asarray(rep.beta, dtype=np.float64)
            if len(node.fixed_one) + 1 <= instance.k:
                push(bound, NodeState(fixed_one=node.fixed_one + (j,), fixed_zero=node.fixed_zero,
                                      depth=node.depth + 1, parent_bound=bound, warm_start=warm))
            w0 = warm.copy()
            w0[j] = 0.0
            push(bound, NodeState(fixed_one=node.fixed_one, fixed_zero=node.fixed_zero + (j,),
                                  depth=node.depth + 1, parent_bound=bound, warm_start=w0))
    unresolved[:] = [b for b in unresolved if not pruned(b)]
    lb = glb()
    if status is None:
        status = CertificateStatus.OPTIMAL
    gap = max(0.0, inc_obj - lb)
    rel = gap / max(abs(inc_obj), 1e-12)
    if status is CertificateStatus.OPTIMAL and rel > opts.gap_tolerance:
        status = CertificateStatus.GAP_LIMIT
    return Certificate(incumbent_beta=inc_beta, incumbent_objective=inc_obj, global_lower_bound=lb,
                       gap_absolute=gap, gap_relative=rel, nodes_explored=explored,
                       wall_time=time.perf_counter() - t0, status=status, log=log)


def _solve_leaf(instance: ProblemInstance, node: NodeState, bound: float, opts: BnBOptions,
                inc_obj: float):
    """Leaf node: the convex problem on the fixed-one support.  Squared error
    refits exactly (ridge); other losses (or a binding box) refit by projected
    gradient with a growing budget until the fp64 safe bound at the refit is
    within the pruning tolerance of its objective.  Returns (beta, objective,
    bound); the bound is sound whether or not the refit converged."""
    S = tuple(node.fixed_one)
    iters = max(1, opts.refit_iterations)
    best_b, best_o, best_lb = None, math.inf, bound
    for _ in range(6):
        b, o = _refit(instance, [S], iters)
        if float(o[0]) < best_o:
            best_b, best_o = b[0], float(o[0])
        best_lb = max(best_lb, safe_lower_bound(instance, b[0], node))
        ub = min(inc_obj, best_o)
        if best_lb >= ub - (opts.prune_abs + opts.prune_rel * abs(ub)):
            break
        iters *= 4
    return best_b, best_o, best_lb


def _relaxation_branch(instance: ProblemInstance, node: NodeState, relax_beta) -> Optional[int]:
    """The free coordinate with the largest |relaxation beta| (None if all zero)."""
    beta = np.abs(np.asarray(relax_beta, dtype=np.float64))
    free = np.ones(instance.p, dtype=bool)
    free[list(node.fixed_one) + list(node.fixed_zero)] = False
    beta[~free] = 0.0
    if len(node.fixed_one) >= int(instance.k) or not np.any(beta > 0.0):
        return None
    return int(np.argmax(beta))


def _is_leaf(instance: ProblemInstance, node: NodeState) -> bool:
    """No free coordinate may become nonzero: |fixed_one| = k or nothing free."""
    free = instance.p - len(node.fixed_one) - len(node.fixed_zero)
    return len(node.fixed_one) >= int(instance.k) or free == 0


def _node_point(instance: ProblemInstance, node: NodeState, relax_beta, opts: BnBOptions):
    """A feasible point of the node: fixed_one plus the largest |relaxation|
    free coordinates up to k, refit."""
    beta = np.asarray(relax_beta, dtype=np.float64)
    k = int(instance.k)
    f1 = list(node.fixed_one)
    free = np.ones(instance.p, dtype=bool)
    free[list(node.fixed_one) + list(node.fixed_zero)] = False
    room = max(0, k - len(f1))
    cand = np.flatnonzero(free & (beta != 0.0))
    order = cand[np.argsort(-np.abs(beta[cand]), kind="stable")][:room]
    S = tuple(sorted(f1 + [int(j) for j in order]))
    betas, objs = _refit(instance, [S], opts.refit_iterations)
    return betas[0], float(objs[0])
