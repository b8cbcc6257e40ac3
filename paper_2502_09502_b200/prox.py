"""Exact proximal operators of the top-k Huber penalty — drop-in for l0cert.prox.

Signatures, validation and error behaviour follow
/root/reference/pkg/src/l0cert/prox.py:17-201; the computation is the B200
kernel (stable radix sort of |mu|, closed-form single-pool PAVA, scatter) via
``l0_prox`` in libl0b200.so.  Inputs may be numpy arrays (numpy returned) or
torch tensors (CUDA tensors returned).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import native
from .errors import InfeasibleNodeError, InvalidInputError

__all__ = ["huber", "huber_prox", "prox_gstar", "prox_g", "prox_gstar_node", "prox_g_node"]


def _elementwise(x, w, M, prox: int):
    import torch
    from . import _device
    native.load()
    scalar = not _device.is_torch(x) and np.ndim(x) == 0
    xd = _device.to_cuda_f64(np.atleast_1d(x) if scalar else x)
    out = torch.empty_like(xd)
    native.check(native.lib().l0_huber(xd.data_ptr(), xd.numel(), float(w), float(M), prox,
                                       out.data_ptr(), _device.stream_handle()))
    if scalar:
        return float(out.cpu()[0])
    return _device.like_input(x, out)


def huber(x, M):
    """H_M(x): x^2/2 for |x| <= M, M|x| - M^2/2 beyond (prox.py:27-32)."""
    return _elementwise(x, 0.0, M, 0)


def huber_prox(x, w, M):
    """argmin_v (v - x)^2/2 + w H_M(v) for x >= 0 (prox.py:35-43)."""
    return _elementwise(x, w, M, 1)


def _validated(mu, rho, k, M):
    """prox.py:119-131"""
    from . import _device
    if _device.is_torch(mu):
        import torch
        if mu.dim() != 1:
            raise InvalidInputError("mu must be a 1-d vector")
        if not bool(torch.isfinite(mu).all()):
            raise InvalidInputError("mu contains non-finite entries")
        p = mu.shape[0]
    else:
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        if mu.ndim != 1:
            raise InvalidInputError("mu must be a 1-d vector")
        if not np.all(np.isfinite(mu)):
            raise InvalidInputError("mu contains non-finite entries")
        p = mu.shape[0]
    if not (rho > 0 and np.isfinite(rho)):
        raise InvalidInputError("rho must be a positive finite real")
    if not (M > 0 and np.isfinite(M)):
        raise InvalidInputError("M must be a positive finite real")
    if not (1 <= k <= p):
        raise InvalidInputError(f"k must satisfy 1 <= k <= p, got k={k}, p={p}")
    return mu


def prox_engine(mu, rho: float, k: int, M: float, g_mode: int, node_class=None,
                want_perm: bool = False):
    """Run ``l0_prox``.  Returns (out_tensor, perm_tensor_or_None, (a*, c*))."""
    import torch
    from . import _device
    lib = native.load()
    md = _device.to_cuda_f64(mu)
    p = md.numel()
    out = torch.empty_like(md)
    perm = torch.empty(p, dtype=torch.int32, device=md.device) if want_perm else None
    pool = (ctypes.c_int64 * 2)(-1, -1)
    if p == 0:
        return out, perm, (-1, -1)
    buf, nb = _device.ops_workspace(p)
    native.check(lib.l0_prox(md.data_ptr(), p, float(rho), int(k), float(M),
                             _device.ptr(node_class), int(g_mode), out.data_ptr(),
                             _device.ptr(perm), pool, buf.data_ptr(), nb,
                             _device.stream_handle()))
    return out, perm, (int(pool[0]), int(pool[1]))


def prox_gstar(mu, rho, k, M):
    """Exact prox of rho * TopSum_k(H_M(.)) (prox.py:134-141)."""
    mu = _validated(mu, rho, k, M)
    out, _, _ = prox_engine(mu, float(rho), int(k), float(M), 0)
    from . import _device
    return _device.like_input(mu, out)


def prox_g(mu, rho, k, M):
    """prox of g/rho through the extended Moreau identity (prox.py:144-151)."""
    mu = _validated(mu, rho, k, M)
    out, _, _ = prox_engine(mu, float(rho), int(k), float(M), 1)
    from . import _device
    return _device.like_input(mu, out)


def _node_index_arrays(p, free_set, fixed_one_set):
    """prox.py:154-163"""
    free = np.asarray(sorted(free_set), dtype=np.int64)
    fone = np.asarray(sorted(fixed_one_set), dtype=np.int64)
    if free.size and (free[0] < 0 or free[-1] >= p):
        raise InvalidInputError("free_set index out of range")
    if fone.size and (fone[0] < 0 or fone[-1] >= p):
        raise InvalidInputError("fixed_one_set index out of range")
    if np.intersect1d(free, fone).size:
        raise InvalidInputError("free_set and fixed_one_set must be disjoint")
    return free, fone


def _node_call(mu, rho, free_set, fixed_one_set, k_remaining, M, g_mode):
    from . import _device
    if _device.is_torch(mu):
        import torch
        md = _device.to_cuda_f64(mu)
        if not bool(torch.isfinite(md).all()):
            raise InvalidInputError("mu contains non-finite entries")
        p = md.numel()
    else:
        md = np.ascontiguousarray(mu, dtype=np.float64)
        if not np.all(np.isfinite(md)):
            raise InvalidInputError("mu contains non-finite entries")
        p = md.shape[0]
    if not (rho > 0 and np.isfinite(rho)):
        raise InvalidInputError("rho must be a positive finite real")
    if k_remaining < 0:
        raise InfeasibleNodeError(f"remaining cardinality budget is negative ({k_remaining})")
    free, fone = _node_index_arrays(p, free_set, fixed_one_set)
    native.load()
    cls = _device.node_class_array(p, free, fone, native.FIXED_ZERO)
    out, _, _ = prox_engine(md, float(rho), int(min(k_remaining, free.size)), float(M), g_mode,
                            node_class=cls)
    return _device.like_input(mu, out)


def prox_gstar_node(mu, rho, free_set, fixed_one_set, k_remaining, M):
    """Node-masked prox of the conjugate (prox.py:166-187): fixed-in coordinates
    take the elementwise Huber prox, free ones compete for the remaining budget,
    fixed-out ones pass through."""
    return _node_call(mu, rho, free_set, fixed_one_set, k_remaining, M, 0)


def prox_g_node(mu, rho, free_set, fixed_one_set, k_remaining, M):
    """Node-masked prox of g/rho (prox.py:190-201); fixed-out coordinates are 0."""
    return _node_call(mu, rho, free_set, fixed_one_set, k_remaining, M, 1)
