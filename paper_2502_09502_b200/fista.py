"""Restarted FISTA on the perspective relaxation — drop-in for l0cert.fista.

``solve_relaxation(instance, node=None, warm_start=None, opts=None)`` keeps the
signature, options, report, trace-hook records and exceptions of
/root/reference/pkg/src/l0cert/fista.py:35-222.  The whole loop runs on the
B200: one C-ABI call (``l0_fista_solve``) replays CUDA graphs of K2 (transpose
pass + gradient step), K3 (bound check, sort, PAVA, scatter, envelope) and K1
(forward pass, loss, objective, restart) with the control state resident on
the device; the host only reads the state between graph replays.

Differences a caller can observe (documented in DESIGN.md):
* ``time_limit`` is checked between graph replays (~16 ms of work apart), not after
  every iteration;
* ``trace_hook`` is called with the same records, in order, but in batches;
* engine-only options: ``gap_tolerance_rel``, ``stop_on_gap``,
  ``chunk_iterations``, ``profile`` (defaults reproduce the reference).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, Optional

import numpy as np

from . import native
from .errors import InvalidInputError, NumericalError, UnsupportedOperationError
from .model import NodeState, ProblemInstance, is_solver_grade, lipschitz_constant
from .perspective import EnvelopeParams

__all__ = ["FistaOptions", "Termination", "RelaxationReport", "solve_relaxation",
           "solve_relaxation_batched"]


class Termination(Enum):
    CONVERGED = "converged"
    ITERATION_LIMIT = "iteration_limit"
    TIME_LIMIT = "time_limit"
    PRIMAL_BELOW_INCUMBENT = "primal_below_incumbent"
    DUAL_ABOVE_INCUMBENT = "dual_above_incumbent"


@dataclass
class FistaOptions:
    max_iterations: int = 100_000
    gap_tolerance: float = 1e-6
    time_limit: float = np.inf
    early_primal_cutoff: Optional[float] = None
    early_dual_cutoff: Optional[float] = None
    bound_check_interval: int = 10
    restart: bool = True
    lipschitz: Optional[float] = None
    trace_hook: Optional[Callable[[dict], None]] = None
    # ---- engine extensions (defaults = reference behaviour) ----
    gap_tolerance_rel: float = 0.0      # also stop at gap <= rel * |primal|
    stop_on_gap: bool = True            # False: fixed-iteration runs
    chunk_iterations: int = 0           # iterations per CUDA graph replay (0: auto)
    profile: bool = False               # time the kernels with CUDA events
    engine_path: str = "auto"           # "auto" | "two_pass" | "single_pass"
    # fp32 mode for fp32 X (BASELINE C3 / C5: "fp32 X with fp64 reductions"):
    # the single-pass kernel's X beta in fp32 products, reduced in fp64;
    # results within ~1e-6 relative of the fp64 path (north star: 1e-5)
    fp32_forward: bool = False

    def __post_init__(self):
        if self.gap_tolerance <= 0:
            raise InvalidInputError("gap_tolerance must be positive")
        if self.bound_check_interval < 1:
            raise InvalidInputError("bound_check_interval must be >= 1")
        if self.max_iterations < 1:
            raise InvalidInputError("max_iterations must be >= 1")
        if self.engine_path not in ("auto", "two_pass", "single_pass"):
            raise InvalidInputError("engine_path must be 'auto', 'two_pass' or 'single_pass'")


@dataclass
class RelaxationReport:
    beta: np.ndarray
    primal_value: float
    dual_bound: float
    gap: float
    iterations: int
    restarts: int
    termination: Termination
    wall_time: float = field(default=0.0)
    # engine metrics (not in the reference report)
    stats: dict = field(default_factory=dict, repr=False)


_TERM = {i: Termination(v) for i, v in enumerate(native.TERMINATIONS)}


def _opt(x) -> float:
    return math.nan if x is None else float(x)


def _native_opts(opts: FistaOptions, L: float):
    o = native.FistaOpts()
    o.max_iterations = int(opts.max_iterations)
    o.gap_tolerance = float(opts.gap_tolerance)
    o.time_limit = float(opts.time_limit)
    o.early_primal_cutoff = _opt(opts.early_primal_cutoff)
    o.early_dual_cutoff = _opt(opts.early_dual_cutoff)
    o.bound_check_interval = int(opts.bound_check_interval)
    o.restart = 1 if opts.restart else 0
    o.lipschitz = float(L)
    o.gap_tolerance_rel = float(opts.gap_tolerance_rel)
    o.stop_on_gap = 1 if opts.stop_on_gap else 0
    o.chunk_iterations = int(opts.chunk_iterations)
    o.profile = 1 if opts.profile else 0
    o.engine_path = {"auto": 0, "two_pass": 1, "single_pass": 2}[opts.engine_path]
    o.fp32_forward = 1 if opts.fp32_forward else 0
    return o


def solve_relaxation_batched(instance: ProblemInstance, nodes, opts: Optional[FistaOptions] = None,
                             return_device: bool = False):
    """Solve the relaxations of many branch-and-bound nodes on one shared X
    (the engine's batched mode): per node exactly
    ``solve_relaxation(instance, node, opts=opts)`` from a cold start, with the
    two X passes of every iteration run as tcgen05 tensor-core contractions
    over all nodes (3xTF32, fp32-class rounding: results agree with the
    per-node solve to ~1e-5 relative).  ``nodes`` is a sequence of NodeState
    (or None for the root).  Returns one RelaxationReport per node."""
    opts = opts or FistaOptions()
    if not is_solver_grade(instance.loss):
        raise UnsupportedOperationError(
            f"{instance.loss.value} is bound-grade; the relaxation solver needs a "
            "Lipschitz-smooth gradient")
    if opts.trace_hook is not None:
        raise UnsupportedOperationError("trace_hook is not available in batched mode")
    nodes = list(nodes)
    if not nodes:
        return []
    params = [EnvelopeParams.for_instance(instance, nd) for nd in nodes]   # InfeasibleNodeError (fista.py:97)
    L = opts.lipschitz if opts.lipschitz is not None else lipschitz_constant(instance)

    import torch
    from . import _device
    lib = native.load()
    dp = instance.device_problem()
    handle, _ws, _fin = dp.batch(len(nodes))
    o = _native_opts(opts, L)
    # every node's index lists in one int64 buffer; the Node structs point into it
    arr = (native.Node * len(nodes))()
    lists = [(tuple(nd.fixed_one), tuple(nd.fixed_zero)) if nd is not None else ((), ()) for nd in nodes]
    flat = np.fromiter((j for f1, f0 in lists for j in (*f1, *f0)), dtype=np.int64,
                       count=sum(len(f1) + len(f0) for f1, f0 in lists))
    keep = [flat]
    base = flat.ctypes.data
    pos = 0
    for i, (nd, (f1, f0)) in enumerate(zip(nodes, lists)):
        a = arr[i]
        a.h_fixed_one = ctypes.cast(base + 8 * pos, ctypes.POINTER(ctypes.c_int64))
        a.n_fixed_one = len(f1)
        a.h_fixed_zero = ctypes.cast(base + 8 * (pos + len(f1)), ctypes.POINTER(ctypes.c_int64))
        a.n_fixed_zero = len(f0)
        a.parent_bound = float(nd.parent_bound) if nd is not None else -math.inf
        pos += len(f1) + len(f0)
    p = instance.p
    # warm starts (NodeState.warm_start; fista.py:130-137): beta_0 per node and
    # g(beta_0) for the initial objective; cold nodes start at 0 with g = 0
    # g(beta_0) of the warm starts is evaluated by the engine (kb_g0)
    warm = g0 = None
    if any(nd is not None and getattr(nd, "warm_start", None) is not None for nd in nodes):
        warm = torch.zeros((len(nodes), p), dtype=torch.float64, device=dp.X.device)
        for i, nd in enumerate(nodes):
            ws = getattr(nd, "warm_start", None) if nd is not None else None
            if ws is None:
                continue
            w = _device.to_cuda_f64(ws)
            if tuple(w.shape) != (p,):
                raise InvalidInputError("warm start has the wrong dimension")
            warm[i].copy_(w)
    beta_out = torch.empty((len(nodes), p), dtype=torch.float64, device=dp.X.device)
    reps = (native.Report * len(nodes))()
    rc = lib.l0_batch_solve(handle, int(instance.k), float(instance.M), float(instance.lambda2),
                            ctypes.byref(o), ctypes.cast(arr, ctypes.c_void_p),
                            _device.ptr(warm), g0.ctypes.data_as(ctypes.c_void_p) if g0 is not None else None,
                            beta_out.data_ptr(), ctypes.cast(reps, ctypes.c_void_p), _device.stream_handle())
    if rc == native.NUMERICAL:
        bad = next((r for r in reps if r.status == native.NUMERICAL), None)
        raise NumericalError(native.last_error(),
                             iteration=int(bad.error_iteration) if bad is not None else None)
    native.check(rc)
    betas = beta_out.unbind(0) if return_device else beta_out.cpu().numpy()
    out = []
    for i, r in enumerate(reps):
        out.append(RelaxationReport(
            beta=betas[i], primal_value=float(r.primal_value), dual_bound=float(r.dual_bound),
            gap=float(r.gap), iterations=int(r.iterations), restarts=int(r.restarts),
            termination=_TERM[int(r.termination)], wall_time=float(r.wall_time),
            stats={"gpu_launches": int(r.gpu_launches), "batched": len(nodes),
                   "lipschitz": float(L), "prox_full_passes": int(r.prox_full_passes),
                   **({"gemm_t_ms": r.k2_ms, "prox_ms": r.k3_ms, "gemm_f_ms": r.k1_ms,
                       "profiled_iterations": int(r.k1_count)} if opts.profile else {})}))
    return out


def solve_relaxation(instance: ProblemInstance, node: Optional[NodeState] = None,
                     warm_start=None, opts: Optional[FistaOptions] = None,
                     return_device: bool = False) -> RelaxationReport:
    """Solve the (node-restricted) perspective relaxation on the B200
    (fista.py:76-222).  ``return_device=True`` leaves ``report.beta`` as a CUDA
    tensor instead of copying it to a numpy array."""
    opts = opts or FistaOptions()
    if not is_solver_grade(instance.loss):
        raise UnsupportedOperationError(
            f"{instance.loss.value} is bound-grade; the relaxation solver needs a "
            "Lipschitz-smooth gradient")
    p = instance.p
    EnvelopeParams.for_instance(instance, node)          # InfeasibleNodeError (fista.py:97)
    L = opts.lipschitz if opts.lipschitz is not None else lipschitz_constant(instance)

    import torch
    from . import _device
    lib = native.load()
    dp = instance.device_problem()

    if warm_start is None and node is not None and node.warm_start is not None:
        warm_start = node.warm_start
    warm = None
    if warm_start is not None:
        warm = _device.to_cuda_f64(warm_start)
        if tuple(warm.shape) != (p,):
            raise InvalidInputError("warm start has the wrong dimension")

    o = native.FistaOpts()
    o.max_iterations = int(opts.max_iterations)
    o.gap_tolerance = float(opts.gap_tolerance)
    o.time_limit = float(opts.time_limit)
    o.early_primal_cutoff = _opt(opts.early_primal_cutoff)
    o.early_dual_cutoff = _opt(opts.early_dual_cutoff)
    o.bound_check_interval = int(opts.bound_check_interval)
    o.restart = 1 if opts.restart else 0
    o.lipschitz = float(L)
    o.gap_tolerance_rel = float(opts.gap_tolerance_rel)
    o.stop_on_gap = 1 if opts.stop_on_gap else 0
    o.chunk_iterations = int(opts.chunk_iterations)
    o.profile = 1 if opts.profile else 0
    o.engine_path = {"auto": 0, "two_pass": 1, "single_pass": 2}[opts.engine_path]
    o.fp32_forward = 1 if opts.fp32_forward else 0

    nd = None
    keep = []
    if node is not None:
        nd = native.Node()
        f1 = np.ascontiguousarray(node.fixed_one, dtype=np.int64)
        f0 = np.ascontiguousarray(node.fixed_zero, dtype=np.int64)
        keep += [f1, f0]
        nd.h_fixed_one = f1.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        nd.n_fixed_one = f1.size
        nd.h_fixed_zero = f0.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        nd.n_fixed_zero = f0.size
        nd.parent_bound = float(node.parent_bound)

    hook = opts.trace_hook
    raised = []

    def _cb(rec_ptr, _user):
        r = rec_ptr.contents
        try:
            hook({"iteration": int(r.iteration), "primal": float(r.primal),
                  "dual": float(r.dual), "gap": float(r.gap), "restarted": bool(r.restarted)})
        except BaseException as exc:  # re-raised after the engine unwinds
            raised.append(exc)
            return 1
        return 0

    cb = native.TRACE_CB(_cb) if hook is not None else native.TRACE_CB()
    beta_out = torch.empty(p, dtype=torch.float64, device=dp.X.device)
    rep = native.Report()
    rc = lib.l0_fista_solve(dp.handle, int(instance.k), float(instance.M),
                            float(instance.lambda2), ctypes.byref(o),
                            ctypes.byref(nd) if nd is not None else None,
                            _device.ptr(warm), beta_out.data_ptr(), ctypes.byref(rep), cb, None,
                            _device.stream_handle())
    if raised:
        raise raised[0]
    if rc == native.NUMERICAL:
        raise NumericalError(native.last_error(), iteration=int(rep.error_iteration))
    native.check(rc)
    beta = beta_out if return_device else beta_out.cpu().numpy()
    stats = {"gpu_launches": int(rep.gpu_launches), "topk_fallbacks": int(rep.topk_fallbacks),
             "prox_full_passes": int(rep.prox_full_passes),
             "single_pass": bool(rep.single_pass), "cluster_size": int(rep.cluster_size),
             "lipschitz": float(L)}
    if opts.profile:
        stats.update(k1_ms=rep.k1_ms, k2_ms=rep.k2_ms, k3_ms=rep.k3_ms, k1_count=rep.k1_count,
                     k2_count=rep.k2_count, k3_count=rep.k3_count)
    return RelaxationReport(beta=beta, primal_value=float(rep.primal_value),
                            dual_bound=float(rep.dual_bound), gap=float(rep.gap),
                            iterations=int(rep.iterations), restarts=int(rep.restarts),
                            termination=_TERM[int(rep.termination)],
                            wall_time=float(rep.wall_time), stats=stats)
