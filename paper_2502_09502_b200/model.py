"""Problem instances and GLM losses — drop-in for l0cert.model.

Same names, fields, validation and error behaviour as
/root/reference/pkg/src/l0cert/model.py:19-327; the numerical work (losses,
gradients, conjugates, power iteration) runs on the B200 through
libl0b200.so.  Engine extensions (keyword-only, defaults keep the reference
behaviour):

* ``ProblemInstance(..., dtype="fp32")`` keeps X in fp32 storage (arithmetic
  stays fp64), the fp32 mode of the BASELINE configs;
* ``X`` may be a torch tensor (CUDA-resident data is used in place).

Solver-grade losses (squared error, logistic, squared hinge) are what the
engine solves; the bound-grade Poisson and gamma losses are evaluated on the
GPU for values, conjugates and safe bounds (the solver rejects them, as the
reference does); multinomial (matrix predictions) raises
UnsupportedOperationError.
"""

from __future__ import annotations

import ctypes
import os
import math
import weakref
from dataclasses import dataclass, field
from enum import Enum
from typing import Any, Optional, Tuple

import numpy as np

from . import native
from .errors import InvalidInputError, NumericalError, UnsupportedOperationError

__all__ = [
    "LossKind", "ProblemInstance", "NodeState", "is_solver_grade", "loss_value",
    "loss_gradient", "loss_conjugate_at_neg", "lipschitz_constant",
]

LIPSCHITZ_SAFETY = 1.01      # model.py:32
_POWER_TOL = 1e-7            # model.py:34
_POWER_MAX_ITER = 500        # model.py:35
_DOMAIN_SLACK = 1e-12        # model.py:39


class LossKind(Enum):
    SQUARED_ERROR = "squared_error"
    LOGISTIC = "logistic"
    SQUARED_HINGE = "squared_hinge"
    POISSON = "poisson"
    GAMMA = "gamma"
    MULTINOMIAL = "multinomial"


_SOLVER_GRADE = (LossKind.SQUARED_ERROR, LossKind.LOGISTIC, LossKind.SQUARED_HINGE)
_PM_ONE = (LossKind.LOGISTIC, LossKind.SQUARED_HINGE)
_CURVATURE = {LossKind.SQUARED_ERROR: 2.0, LossKind.LOGISTIC: 0.25,
              LossKind.SQUARED_HINGE: 2.0}   # model.py:309-313


def is_solver_grade(loss: LossKind) -> bool:
    return loss in _SOLVER_GRADE


_ENGINE_LOSSES = _SOLVER_GRADE + (LossKind.POISSON, LossKind.GAMMA)


def _engine_loss(loss: LossKind) -> int:
    """Engine code of a loss the kernels evaluate: the solver-grade ones and,
    for values, conjugates and bounds only, Poisson and gamma.  Multinomial
    (matrix predictions) stays host-side unsupported."""
    if loss not in _ENGINE_LOSSES:
        raise UnsupportedOperationError(
            f"{loss.value}: the B200 engine evaluates squared_error, logistic, squared_hinge "
            "(solver-grade) and poisson, gamma (bound-grade)")
    return native.LOSS_CODES[loss.value]


def _host_vector(v) -> np.ndarray:
    try:
        import torch
        if isinstance(v, torch.Tensor):
            return v.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(v, dtype=np.float64)


def _check_labels(loss: LossKind, y: np.ndarray) -> None:
    """model.py:59-72 (solver-grade and bound-grade label domains)."""
    if not np.all(np.isfinite(y)):
        raise InvalidInputError("labels contain non-finite entries")
    if loss in _PM_ONE:
        if not np.all(np.abs(y) == 1.0):
            raise InvalidInputError(f"{loss.value} labels must be +/-1")
    elif loss is LossKind.GAMMA:
        if not np.all(y > 0):
            raise InvalidInputError("gamma labels must be positive")
    elif loss is LossKind.MULTINOMIAL:
        if y.ndim != 2:
            raise InvalidInputError("multinomial labels must be an (n, K) indicator matrix")
        if not (np.all((y == 0) | (y == 1)) and np.all(y.sum(axis=1) == 1)):
            raise InvalidInputError("multinomial labels must be one-hot rows")


def _padded_finite(Xt, lib) -> bool:
    """All n x stride(0) elements under a strided device view are finite
    (the engine reads the padding columns with beta = 0 there)."""
    import torch
    from . import _device
    if Xt.stride(0) == Xt.shape[1]:
        return True
    full = Xt.as_strided((Xt.shape[0], Xt.stride(0)), (Xt.stride(0), 1))
    buf, nb = _device.ops_workspace(1)
    ok = ctypes.c_int32()
    code = native.F64 if Xt.dtype == torch.float64 else native.F32
    native.check(lib.l0_all_finite(full.data_ptr(), code, full.shape[0], full.shape[1],
                                   full.stride(0), ctypes.byref(ok), buf.data_ptr(), nb,
                                   _device.stream_handle()))
    return bool(ok.value)


class DeviceProblem:
    """X, y resident in HBM plus the engine's problem handle and workspace."""

    def __init__(self, X, y: np.ndarray, loss: LossKind, dtype: str):
        import torch
        from . import _device
        lib = native.load()
        dev = _device.device()
        tdt = torch.float64 if dtype == "fp64" else torch.float32
        if isinstance(X, torch.Tensor):
            Xt = X.detach()
        else:
            Xt = torch.from_numpy(np.ascontiguousarray(X))
        n, p = Xt.shape
        align = 32
        ld = ((p + align - 1) // align) * align
        if not isinstance(X, torch.Tensor) and Xt.dtype == tdt:
            # pageable host array: multi-threaded pinned staging overlapped with the DMA
            es = Xt.element_size()
            Xd = (torch.empty if ld == p else torch.zeros)((n, ld), dtype=tdt, device=dev)
            native.check(lib.l0_upload_rows(Xd.data_ptr(), ld * es, Xt.data_ptr(), p * es, p * es,
                                            n, min(8, os.cpu_count() or 8),   # tools/upload_bw.py: 8 > 12 > 16
                                            _device.stream_handle()))
        elif (Xt.device.type == "cuda" and Xt.dtype == tdt and Xt.dim() == 2 and Xt.stride(1) == 1
              and Xt.stride(0) >= p and Xt.stride(0) % align == 0 and n > 0
              and (Xt.storage_offset() + n * Xt.stride(0)) * Xt.element_size()
              <= Xt.untyped_storage().nbytes()
              and _padded_finite(Xt, lib)):
            # a device view whose rows already carry finite padding (e.g. the
            # [:, :p] view of an (n, ld) buffer): used in place, no copy
            ld = int(Xt.stride(0))
            Xd = Xt.as_strided((n, ld), (ld, 1))
        elif ld == p and Xt.dtype == tdt and Xt.is_contiguous():
            Xd = Xt.to(dev, non_blocking=Xt.is_pinned()) if Xt.device.type != "cuda" else Xt
        else:
            Xd = torch.zeros((n, ld), dtype=tdt, device=dev)
            Xd[:, :p].copy_(Xt.to(dev) if Xt.device.type != "cuda" else Xt)
        self.X = Xd
        self.y = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).to(dev)
        self.n, self.p, self.ld = int(n), int(p), int(ld)
        self.dtype_code = native.F64 if dtype == "fp64" else native.F32
        self.loss_code = native.LOSS_CODES[loss.value]
        handle = ctypes.c_void_p()
        native.check(lib.l0_problem_create(Xd.data_ptr(), self.dtype_code, self.n, self.p,
                                           self.ld, self.y.data_ptr(), self.loss_code,
                                           ctypes.byref(handle)))
        self.handle = handle
        self._finalizer = weakref.finalize(self, lib.l0_problem_destroy, handle)
        nb = ctypes.c_uint64()
        native.check(lib.l0_problem_workspace_bytes(handle, ctypes.byref(nb)))
        self.ws = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
        native.check(lib.l0_problem_set_workspace(handle, self.ws.data_ptr(), nb.value))

    def batch(self, n_nodes: int):
        """Batched-node engine for ``n_nodes`` nodes on this X (cached; the
        workspace holds X split into TF32 hi/lo operands, 4 x n x p fp32)."""
        import torch
        cache = self.__dict__.setdefault("_batches", {})
        if n_nodes in cache:
            return cache[n_nodes]
        for old in list(cache):          # keep one batch engine resident
            cache.pop(old)[2]()
        lib = native.load()
        handle = ctypes.c_void_p()
        native.check(lib.l0_batch_create(self.handle, int(n_nodes), ctypes.byref(handle)))
        fin = weakref.finalize(self, lib.l0_batch_destroy, handle)
        nb = ctypes.c_uint64()
        native.check(lib.l0_batch_workspace_bytes(handle, ctypes.byref(nb)))
        ws = torch.empty(int(nb.value), dtype=torch.uint8, device=self.X.device)
        native.check(lib.l0_batch_set_workspace(handle, ws.data_ptr(), nb.value))
        cache[n_nodes] = (handle, ws, fin)
        return cache[n_nodes]

    def matvec(self, v):
        import torch
        from . import _device
        out = torch.empty(self.n, dtype=torch.float64, device=self.X.device)
        vd = _device.to_cuda_f64(v)
        native.check(native.lib().l0_matvec(self.handle, vd.data_ptr(), out.data_ptr(),
                                            _device.stream_handle()))
        return out

    def rmatvec(self, r):
        import torch
        from . import _device
        out = torch.empty(self.p, dtype=torch.float64, device=self.X.device)
        rd = _device.to_cuda_f64(r)
        native.check(native.lib().l0_rmatvec(self.handle, rd.data_ptr(), out.data_ptr(),
                                             _device.stream_handle()))
        return out


@dataclass
class ProblemInstance:
    """Minimise ``f(X beta, y) + lambda2 ||beta||^2`` s.t. ``||beta||_0 <= k``,
    ``||beta||_inf <= M`` (model.py:75-116)."""

    X: Any
    y: Any
    loss: LossKind
    k: int
    M: float
    lambda2: float
    beta_true: Optional[np.ndarray] = field(default=None, repr=False)
    dtype: str = field(default="fp64", repr=False, kw_only=True)

    def __post_init__(self):
        if self.dtype not in ("fp64", "fp32"):
            raise InvalidInputError("dtype must be 'fp64' or 'fp32'")
        is_t = False
        try:
            import torch
            is_t = isinstance(self.X, torch.Tensor)
        except ImportError:  # pragma: no cover
            pass
        if not is_t:
            self.X = np.ascontiguousarray(self.X, dtype=np.float64 if self.dtype == "fp64"
                                          else np.float32)
        self.y = _host_vector(self.y)
        if len(self.X.shape) != 2:
            raise InvalidInputError("X must be a 2-d matrix")
        n, p = self.X.shape
        if self.y.shape[0] != n:
            raise InvalidInputError(f"X has {n} rows but y has {self.y.shape[0]} entries")
        if not self._x_finite():
            raise InvalidInputError("X contains non-finite entries")
        if not (1 <= self.k <= p):
            raise InvalidInputError(f"k must satisfy 1 <= k <= p, got k={self.k}, p={p}")
        if not (self.M > 0 and np.isfinite(self.M)):
            raise InvalidInputError("M must be a positive finite real")
        if not (self.lambda2 > 0 and np.isfinite(self.lambda2)):
            raise InvalidInputError("lambda2 must be a positive finite real")
        _check_labels(self.loss, self.y)
        self._dev = None
        self._dev_src = None

    def _x_finite(self) -> bool:
        if isinstance(self.X, np.ndarray):
            return bool(np.all(np.isfinite(self.X)))
        import torch
        X = self.X
        if X.device.type != "cuda":
            return bool(torch.isfinite(X).all())
        from . import _device
        buf, nb = _device.ops_workspace(1)
        ok = ctypes.c_int32()
        code = native.F64 if X.dtype == torch.float64 else native.F32
        Xc = X if X.dtype in (torch.float64, torch.float32) else X.to(torch.float64)
        native.check(native.load().l0_all_finite(Xc.data_ptr(), code, Xc.shape[0], Xc.shape[1],
                                                 Xc.stride(0), ctypes.byref(ok), buf.data_ptr(),
                                                 nb, _device.stream_handle()))
        return bool(ok.value)

    @property
    def n(self) -> int:
        return self.X.shape[0]

    @property
    def p(self) -> int:
        return self.X.shape[1]

    def device_problem(self) -> DeviceProblem:
        """The HBM-resident copy of (X, y) used by every engine call (built once).

        X (and y) are treated as immutable after the first engine call, as the
        reference treats its private float64 copy (model.py:92): in-place
        edits of the host array are not seen; assign a new array to ``X`` (a
        new object re-uploads) or call ``release_device()``."""
        # keyed by the array object itself (a reference, not its id: a new
        # array cannot reuse a freed id while the old one is held here)
        if self._dev is None or self._dev_src is not self.X:
            if not is_solver_grade(self.loss):
                _engine_loss(self.loss)
            self._dev = DeviceProblem(self.X, self.y, self.loss, self.dtype)
            self._dev_src = self.X
        return self._dev

    def release_device(self) -> None:
        self._dev = None
        self._dev_src = None


@dataclass
class NodeState:
    """Search-tree node (model.py:119-149): fixed sets, parent bound, warm start."""

    fixed_one: Tuple[int, ...] = ()
    fixed_zero: Tuple[int, ...] = ()
    depth: int = 0
    parent_bound: float = -np.inf
    warm_start: Optional[np.ndarray] = None

    def __post_init__(self):
        self.fixed_one = tuple(sorted(int(j) for j in self.fixed_one))
        self.fixed_zero = tuple(sorted(int(j) for j in self.fixed_zero))
        if set(self.fixed_one) & set(self.fixed_zero):
            raise InvalidInputError("fixed_one and fixed_zero must be disjoint")

    def free_indices(self, p: int) -> np.ndarray:
        keep = np.ones(p, dtype=bool)
        fixed = list(self.fixed_one) + list(self.fixed_zero)
        if fixed:
            keep[np.asarray(fixed, dtype=np.int64)] = False
        return np.flatnonzero(keep)

    def is_trivial(self) -> bool:
        return not self.fixed_one and not self.fixed_zero


def _finite_vector(u, name):
    u = _host_vector(u) if not _is_cuda_tensor(u) else u
    if _is_cuda_tensor(u):
        import torch
        if not bool(torch.isfinite(u).all()):
            raise InvalidInputError(f"{name} contains non-finite entries")
        return u
    if not np.all(np.isfinite(u)):
        raise InvalidInputError(f"{name} contains non-finite entries")
    return u


def _is_cuda_tensor(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor) and x.device.type == "cuda"
    except ImportError:  # pragma: no cover
        return False


def loss_value(loss: LossKind, u, y) -> float:
    """F(u) at linear predictions u (model.py:159-181)."""
    code = _engine_loss(loss)
    from . import _device
    u = _finite_vector(u, "u")
    yh = _host_vector(y)
    _check_labels(loss, yh)
    ud, yd = _device.to_cuda_f64(u), _device.to_cuda_f64(yh)
    buf, nb = _device.ops_workspace(1)
    val = ctypes.c_double()
    bad = ctypes.c_int32()
    native.check(native.load().l0_loss_value(code, ud.data_ptr(), yd.data_ptr(), ud.numel(),
                                             ctypes.byref(val), None, ctypes.byref(bad),
                                             buf.data_ptr(), nb, _device.stream_handle()))
    return float(val.value)


def loss_gradient(loss: LossKind, u, y):
    """grad F(u), solver-grade losses only (model.py:208-218)."""
    if not is_solver_grade(loss):
        raise UnsupportedOperationError(
            f"{loss.value} is bound-grade: gradients are not exposed because no "
            "global Lipschitz constant exists for the solver to rely on")
    import torch
    from . import _device
    u = _finite_vector(u, "u")
    yh = _host_vector(y)
    _check_labels(loss, yh)
    ud, yd = _device.to_cuda_f64(u), _device.to_cuda_f64(yh)
    grad = torch.empty_like(ud)
    buf, nb = _device.ops_workspace(1)
    val = ctypes.c_double()
    bad = ctypes.c_int32()
    native.check(native.load().l0_loss_value(native.LOSS_CODES[loss.value], ud.data_ptr(),
                                             yd.data_ptr(), ud.numel(), ctypes.byref(val),
                                             grad.data_ptr(), ctypes.byref(bad), buf.data_ptr(),
                                             nb, _device.stream_handle()))
    return _device.like_input(u, grad)


def loss_conjugate_at_neg(loss: LossKind, zeta, y) -> float:
    """F*(-zeta); +inf outside the domain, never an error (model.py:226-280)."""
    code = _engine_loss(loss)
    from . import _device
    zh = zeta if _is_cuda_tensor(zeta) else _host_vector(zeta)
    if _is_cuda_tensor(zh):
        import torch
        if bool(torch.isnan(zh).any()):
            raise InvalidInputError("zeta contains NaN entries")
    elif np.any(np.isnan(zh)):
        raise InvalidInputError("zeta contains NaN entries")
    yh = _host_vector(y)
    _check_labels(loss, yh)
    zd, yd = _device.to_cuda_f64(zh), _device.to_cuda_f64(yh)
    buf, nb = _device.ops_workspace(1)
    out = ctypes.c_double()
    native.check(native.load().l0_loss_conjugate(code, zd.data_ptr(), yd.data_ptr(), zd.numel(),
                                                 ctypes.byref(out), buf.data_ptr(), nb,
                                                 _device.stream_handle()))
    return float(out.value)


def power_iteration_lambda_max(instance: ProblemInstance, tol=_POWER_TOL,
                               max_iter=_POWER_MAX_ITER, seed=0) -> float:
    """lambda_max(X^T X) by power iteration from the reference's seed-0 start
    (model.py:283-306), both passes on the device."""
    from . import _device
    dp = instance.device_problem()
    v = np.random.default_rng(seed).standard_normal(instance.p)
    v /= np.linalg.norm(v)
    vd = _device.to_cuda_f64(v)
    lam = ctypes.c_double()
    its = ctypes.c_int64()
    rc = native.lib().l0_power_iteration(dp.handle, vd.data_ptr(), float(tol), int(max_iter),
                                         ctypes.byref(lam), ctypes.byref(its),
                                         _device.stream_handle())
    if rc == native.NUMERICAL:
        raise NumericalError(f"power iteration did not converge within {max_iter} iterations",
                             iteration=max_iter)
    native.check(rc)
    return float(lam.value)


def lanczos_lambda_max(instance: ProblemInstance, tol: float = 1e-13, max_steps: int = 300) -> float:
    """lambda_max(X^T X) by device Lanczos with full reorthogonalisation
    (spectral.py): converges where the reference's 500-step power iteration
    does not."""
    from .spectral import engine_normal_op, lanczos_lambda_max as _lanczos
    dp = instance.device_problem()
    return _lanczos(engine_normal_op(dp), instance.p, dp.X.device, tol=tol, max_steps=max_steps)


def lipschitz_constant(instance: ProblemInstance, *, method: str = "power") -> float:
    """curvature * lambda_max(X^T X) * 1.01 (model.py:316-327).

    ``method="power"`` (default) is the reference's estimator, failing the same
    way (NumericalError after 500 steps); ``method="lanczos"`` is the engine's
    robust extension (same curvature and 1.01 safety factor)."""
    if not is_solver_grade(instance.loss):
        raise UnsupportedOperationError(
            f"{instance.loss.value} has no global gradient Lipschitz constant")
    if method == "power":
        lam = power_iteration_lambda_max(instance)
    elif method == "lanczos":
        lam = lanczos_lambda_max(instance)
    else:
        raise InvalidInputError("method must be 'power' or 'lanczos'")
    return _CURVATURE[instance.loss] * lam * LIPSCHITZ_SAFETY
