"""The perspective envelope g, its conjugate and the safe Fenchel bound —
drop-in for l0cert.perspective (/root/reference/pkg/src/l0cert/perspective.py:17-190).

g_value / g_conjugate / safe_lower_bound run on the B200 (l0_g_value,
l0_g_conjugate, l0_safe_lower_bound); validation and +inf conventions are the
reference's.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from . import native
from .errors import InfeasibleNodeError, InvalidInputError, UnsupportedOperationError
from .model import LossKind, NodeState, ProblemInstance

__all__ = ["EnvelopeParams", "g_value", "g_conjugate", "safe_lower_bound", "safe_lower_bound_batched"]

_FEAS_RTOL = 1e-9   # perspective.py:23
_ZERO_ATOL = 1e-9   # perspective.py:25


@dataclass(frozen=True)
class EnvelopeParams:
    """Budget k and box bound M, optionally restricted to a search node
    (perspective.py:28-73)."""

    k: int
    M: float
    fixed_one: Tuple[int, ...] = ()
    fixed_zero: Tuple[int, ...] = ()

    def __post_init__(self):
        if self.k < 0:
            raise InvalidInputError("k must be nonnegative")
        if not (self.M > 0 and np.isfinite(self.M)):
            raise InvalidInputError("M must be a positive finite real")
        if set(self.fixed_one) & set(self.fixed_zero):
            raise InvalidInputError("fixed_one and fixed_zero must be disjoint")
        if self.k_remaining < 0:
            raise InfeasibleNodeError(
                f"|fixed_one| = {len(self.fixed_one)} exceeds the budget k = {self.k}")

    @property
    def k_remaining(self) -> int:
        return self.k - len(self.fixed_one)

    @property
    def restricted(self) -> bool:
        return bool(self.fixed_one or self.fixed_zero)

    @classmethod
    def for_instance(cls, instance: ProblemInstance,
                     node: Optional[NodeState] = None) -> "EnvelopeParams":
        if node is None:
            return cls(k=instance.k, M=instance.M)
        return cls(k=instance.k, M=instance.M, fixed_one=node.fixed_one,
                   fixed_zero=node.fixed_zero)

    def free_indices(self, p: int) -> np.ndarray:
        keep = np.ones(p, dtype=bool)
        fixed = list(self.fixed_one) + list(self.fixed_zero)
        if fixed:
            keep[np.asarray(fixed, dtype=np.int64)] = False
        return np.flatnonzero(keep)

    def node_classes(self, p: int):
        """Device uint8 class vector (free / fixed-one / fixed-zero) or None."""
        if not self.restricted:
            return None
        from . import _device
        return _device.node_class_array(p, self.free_indices(p), self.fixed_one, native.FIXED_ZERO)


def g_value(beta, params: EnvelopeParams) -> float:
    """Exact envelope value g(beta); +inf signals infeasibility (perspective.py:114-132)."""
    import torch
    from . import _device
    lib = native.load()
    bd = _device.to_cuda_f64(beta)
    p = bd.numel()
    cls = params.node_classes(p)
    fone = None
    if params.restricted and params.fixed_one:
        fone = torch.tensor(list(params.fixed_one), dtype=torch.int32, device=bd.device)
    kf = params.k_remaining if params.restricted else params.k
    buf, nb = _device.ops_workspace(p)
    out = ctypes.c_double()
    native.check(lib.l0_g_value(bd.data_ptr(), p, int(kf), float(params.M), _device.ptr(cls),
                                _device.ptr(fone), len(params.fixed_one) if fone is not None else 0,
                                ctypes.byref(out), buf.data_ptr(), nb, _device.stream_handle()))
    return float(out.value)


def g_conjugate(alpha, params: EnvelopeParams) -> float:
    """g*(alpha) = TopSum_k(H_M(alpha)), node-aware (perspective.py:143-159)."""
    from . import _device
    lib = native.load()
    ad = _device.to_cuda_f64(alpha)
    p = ad.numel()
    cls = params.node_classes(p)
    kf = params.k_remaining if params.restricted else params.k
    buf, nb = _device.ops_workspace(p)
    out = ctypes.c_double()
    native.check(lib.l0_g_conjugate(ad.data_ptr(), p, int(kf), float(params.M), _device.ptr(cls),
                                    ctypes.byref(out), buf.data_ptr(), nb,
                                    _device.stream_handle()))
    return float(out.value)


def safe_lower_bound(instance: ProblemInstance, beta_hat, node: Optional[NodeState] = None) -> float:
    """Weak-duality lower bound -F*(-zeta) - 2 l2 g*(X^T zeta / 2 l2), zeta = -grad F(X beta_hat)
    (perspective.py:162-190)."""
    if instance.loss is LossKind.MULTINOMIAL:
        raise UnsupportedOperationError("multinomial instances have no vector-coefficient bound")
    if instance.loss not in (LossKind.SQUARED_ERROR, LossKind.LOGISTIC, LossKind.SQUARED_HINGE,
                             LossKind.POISSON, LossKind.GAMMA):
        raise UnsupportedOperationError(
            f"{instance.loss.value}: the B200 engine evaluates bounds for vector GLM losses")
    from . import _device
    bd = _device.to_cuda_f64(beta_hat)
    import torch
    if not bool(torch.isfinite(bd).all()):
        raise InvalidInputError("beta_hat contains non-finite entries")
    params = EnvelopeParams.for_instance(instance, node)
    dp = instance.device_problem()
    cls = params.node_classes(instance.p)
    kf = params.k_remaining if params.restricted else params.k
    out = ctypes.c_double()
    native.check(native.lib().l0_safe_lower_bound(dp.handle, bd.data_ptr(), int(kf),
                                                  float(instance.M), float(instance.lambda2),
                                                  _device.ptr(cls), ctypes.byref(out),
                                                  _device.stream_handle()))
    return float(out.value)


_bb_ws = None


def safe_lower_bound_batched(instance: ProblemInstance, betas, nodes: Sequence[Optional[NodeState]]):
    """safe_lower_bound (perspective.py:162-190) of len(nodes) search nodes in
    one engine call: row j of ``betas`` (len(nodes) x p) is node j's point.
    fp64 throughout (l0_safe_lower_bound_batched); each value equals the
    per-node bound up to the summation order of the two X passes.  Returns a
    list of floats (-inf where F*(-zeta) is +inf)."""
    global _bb_ws
    if instance.loss is LossKind.MULTINOMIAL:
        raise UnsupportedOperationError("multinomial instances have no vector-coefficient bound")
    if instance.loss not in (LossKind.SQUARED_ERROR, LossKind.LOGISTIC, LossKind.SQUARED_HINGE,
                             LossKind.POISSON, LossKind.GAMMA):
        raise UnsupportedOperationError(
            f"{instance.loss.value}: the B200 engine evaluates bounds for vector GLM losses")
    nodes = list(nodes)
    nb = len(nodes)
    if nb == 0:
        return []
    from . import _device
    import torch
    bd = _device.to_cuda_f64(betas)
    if bd.ndim != 2 or bd.shape[0] != nb or bd.shape[1] != instance.p:
        raise InvalidInputError(f"betas must be {nb} x {instance.p}")
    if not bool(torch.isfinite(bd).all()):
        raise InvalidInputError("beta_hat contains non-finite entries")
    params = [EnvelopeParams.for_instance(instance, nd) for nd in nodes]
    kf = np.array([pr.k_remaining if pr.restricted else pr.k for pr in params], dtype=np.int64)
    cls = None
    if any(pr.restricted for pr in params):
        host = np.zeros((nb, instance.p), dtype=np.uint8)
        for j, pr in enumerate(params):
            if pr.fixed_one:
                host[j, np.asarray(pr.fixed_one, dtype=np.int64)] = native.FIXED_ONE
            if pr.fixed_zero:
                host[j, np.asarray(pr.fixed_zero, dtype=np.int64)] = native.FIXED_ZERO
        cls = torch.from_numpy(host).to(_device.device())
    dp = instance.device_problem()
    lib = native.lib()
    need = ctypes.c_uint64()
    native.check(lib.l0_safe_lower_bound_batched_workspace(dp.handle, nb, ctypes.byref(need)))
    if _bb_ws is None:
        _bb_ws = _device.Workspace()
    ws = _bb_ws.get(need.value)
    out = np.empty(nb, dtype=np.float64)
    native.check(lib.l0_safe_lower_bound_batched(
        dp.handle, bd.data_ptr(), nb, kf.ctypes.data_as(ctypes.c_void_p), float(instance.M),
        float(instance.lambda2), _device.ptr(cls), out.ctypes.data_as(ctypes.c_void_p),
        ws.data_ptr(), need.value, _device.stream_handle()))
    return [float(v) for v in out]
