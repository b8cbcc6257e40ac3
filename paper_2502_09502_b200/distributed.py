"""Multi-GPU partitioning of the dual-bound engine.

One process per GPU (torch.distributed for the plumbing):

* **Row sharding** (C5, also usable for C2/C3): rank r holds the contiguous
  rows ``row_range(n, world, r)`` of X and y.  Every iteration the engine
  all-reduces, over its own NCCL communicator (graph-captured inside
  ``l0_fista_solve``), one buffer [X_r^T grad F | X_r^T zeta | F* terms] and the
  loss pair; prox, envelope, restart and bound are computed redundantly and
  identically on every rank (NCCL gives every rank the same reduced bits).
* **Node sharding** (C4): X is replicated, the branch-and-bound nodes are
  dealt round-robin to the ranks, no collective except gathering reports.

Host logic here is backend-agnostic where it can be (partitioning, the id
exchange, the distributed power iteration) so it is exercised by the gloo
tests on CPU; the device work goes through libl0b200.so.
"""

from __future__ import annotations

import ctypes
import math
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import native
from .errors import InvalidInputError, NumericalError, UnsupportedOperationError

__all__ = ["row_range", "shard_nodes", "broadcast_bytes", "nccl_unique_id", "power_iteration",
           "ShardedProblem", "solve_relaxation_sharded", "solve_nodes_sharded",
           "assert_replicated"]


def row_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced block of rows of rank ``rank`` (first n % world
    ranks get one extra row)."""
    if world < 1 or not (0 <= rank < world):
        raise InvalidInputError("bad world/rank")
    base, extra = divmod(n, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def shard_nodes(nodes: Sequence, world: int, rank: int) -> List[int]:
    """Indices of the nodes solved by ``rank`` (round-robin, deterministic)."""
    return list(range(rank, len(nodes), world))


def broadcast_bytes(payload: Optional[bytes], src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string from ``src`` over torch.distributed."""
    import torch.distributed as dist
    box = [payload]
    dist.broadcast_object_list(box, src=src, group=group)
    return box[0]


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, everybody receives it)."""
    buf = ctypes.create_string_buffer(128)
    lib = native._lib if native._lib is not None else native.load_library()
    rc = lib.l0_nccl_unique_id(buf)
    if rc != native.OK:
        raise RuntimeError("ncclGetUniqueId failed: " + (lib.l0_last_error() or b"").decode())
    return buf.raw


def power_iteration(matvec: Callable, rmatvec: Callable, allreduce: Callable, v0: np.ndarray,
                    tol: float = 1e-7, max_iter: int = 500) -> Tuple[float, int]:
    """Power iteration on X^T X for row-sharded X (model.py:283-306):
    lambda = sum_r ||X_r v||^2 and v <- sum_r X_r^T (X_r v), normalised.
    ``allreduce`` sums an array over the ranks (identity on one rank)."""
    v = np.asarray(v0, dtype=np.float64)
    prev = math.inf
    for it in range(max_iter):
        w = matvec(v)
        lam = float(allreduce(np.array([float(np.dot(w, w))]))[0])
        if lam == 0.0:
            return 0.0, it + 1
        v = allreduce(np.asarray(rmatvec(w), dtype=np.float64))
        nrm = float(np.linalg.norm(v))
        if nrm == 0.0:
            return 0.0, it + 1
        v = v / nrm
        if abs(lam - prev) <= tol * lam:
            return lam, it + 1
        prev = lam
    raise NumericalError(f"power iteration did not converge within {max_iter} iterations",
                         iteration=max_iter)


def _torch_allreduce(group=None):
    import torch
    import torch.distributed as dist

    def red(arr):
        t = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64))
        backend = dist.get_backend(group)
        if backend == "nccl":
            t = t.cuda()
        dist.all_reduce(t, group=group)
        return t.cpu().numpy()
    return red


class ShardedProblem:
    """This rank's rows of a row-sharded ProblemInstance, on its GPU, with the
    engine's NCCL communicator attached."""

    def __init__(self, X_local, y_local, loss, k: int, M: float, lambda2: float,
                 n_global: int, dtype: str = "fp64", group=None, emulate: bool = False):
        import torch.distributed as dist
        from .model import ProblemInstance
        self.instance = ProblemInstance(X_local, y_local, loss, k, M, lambda2, dtype=dtype)
        self.n_global = int(n_global)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        dp = self.instance.device_problem()
        lib = native.lib()
        if emulate or self.world == 1:
            native.check(lib.l0_problem_set_comm(dp.handle, None, 1, 0))
        else:
            uid = nccl_unique_id() if self.rank == 0 else None
            uid = broadcast_bytes(uid, src=0, group=group)
            native.check(lib.l0_problem_set_comm(dp.handle, uid, self.world, self.rank))

    @property
    def p(self) -> int:
        return self.instance.p

    def lipschitz(self, method: str = "power") -> float:
        """curvature * lambda_max(X^T X) * 1.01 over all ranks (model.py:316-327);
        ``method="lanczos"``: device Lanczos on the all-reduced X^T X v."""
        from .model import _CURVATURE, LIPSCHITZ_SAFETY
        dp = self.instance.device_problem()
        if method == "lanczos":
            from .spectral import engine_normal_op, lanczos_lambda_max
            red = None
            if self.world > 1:
                import torch.distributed as dist
                red = lambda t: dist.all_reduce(t, group=self.group)
            lam = lanczos_lambda_max(engine_normal_op(dp), self.p, dp.X.device, allreduce=red)
            return _CURVATURE[self.instance.loss] * lam * LIPSCHITZ_SAFETY
        v0 = np.random.default_rng(0).standard_normal(self.p)
        v0 /= np.linalg.norm(v0)
        red = _torch_allreduce(self.group) if self.world > 1 else (lambda a: a)
        lam, _ = power_iteration(lambda v: dp.matvec(v).cpu().numpy(),
                                 lambda w: dp.rmatvec(w).cpu().numpy(), red, v0)
        return _CURVATURE[self.instance.loss] * lam * LIPSCHITZ_SAFETY


def assert_replicated(beta, group=None, atol: float = 0.0) -> None:
    """Every rank holds the same iterate (replicated state invariant)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    t = torch.as_tensor(np.asarray(beta, dtype=np.float64))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    ref = t.clone()
    dist.broadcast(ref, src=0, group=group)
    diff = (t - ref).abs().max().reshape(1)
    dist.all_reduce(diff, op=dist.ReduceOp.MAX, group=group)
    if float(diff.item()) > atol:
        raise AssertionError(f"iterates differ across ranks by {float(diff.item())}")


def solve_relaxation_sharded(problem: ShardedProblem, node=None, warm_start=None, opts=None):
    """solve_relaxation over a row-sharded X; every rank returns the same report."""
    from .fista import FistaOptions, solve_relaxation
    opts = opts or FistaOptions()
    if opts.lipschitz is None:
        import dataclasses
        opts = dataclasses.replace(opts, lipschitz=problem.lipschitz())
    return solve_relaxation(problem.instance, node=node, warm_start=warm_start, opts=opts)


def solve_nodes_sharded(instance, nodes: Sequence, opts=None, group=None, batched: bool = True):
    """Node sharding: this rank solves its round-robin share of ``nodes`` on
    the replicated X -- as ONE batched call (``solve_relaxation_batched``: the
    share's X passes run as tcgen05 contractions), or node by node with
    ``batched=False``.  Returns {node index: report} on this rank plus, gathered
    from every rank, {node index: (primal, dual, gap, iterations, restarts,
    termination)} as the second element."""
    import torch.distributed as dist
    from .fista import solve_relaxation, solve_relaxation_batched
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    idx = shard_nodes(nodes, world, rank)
    mine = {}
    if idx and batched:
        reps = solve_relaxation_batched(instance, [nodes[i] for i in idx], opts=opts)
        mine = dict(zip(idx, reps))
    else:
        for i in idx:
            mine[i] = solve_relaxation(instance, node=nodes[i], opts=opts)
    summary = {i: (r.primal_value, r.dual_bound, r.gap, r.iterations, r.restarts,
                   r.termination.value) for i, r in mine.items()}
    if world == 1:
        return mine, summary
    gathered = [None] * world
    dist.all_gather_object(gathered, summary, group=group)
    out = {}
    for part in gathered:
        out.update(part)
    return mine, out
