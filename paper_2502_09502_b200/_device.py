"""Device plumbing: torch owns every device buffer the engine touches."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import native


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_cuda_f64(x, name: str = "array") -> torch.Tensor:
    """A contiguous float64 CUDA tensor holding x (numpy, torch or scalar)."""
    if is_torch(x):
        t = x.detach()
        if t.device.type != "cuda":
            t = t.to(device(), non_blocking=t.is_pinned())
        return t.to(torch.float64).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to(device())


def like_input(x, t: torch.Tensor):
    """Return the engine result in the caller's array type (numpy in, numpy out)."""
    if is_torch(x):
        return t
    return t.cpu().numpy()


class Workspace:
    """Grow-only device scratch buffer (one per thread of use)."""

    def __init__(self):
        self._buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self._buf is None or self._buf.numel() < nbytes:
            self._buf = torch.empty(int(nbytes), dtype=torch.uint8, device=device())
        return self._buf


_ops_ws = Workspace()


def ops_workspace(length: int):
    nb = ctypes.c_uint64()
    native.check(native.lib().l0_ops_workspace_bytes(int(length), ctypes.byref(nb)))
    buf = _ops_ws.get(nb.value)
    return buf, nb.value


def node_class_array(p: int, free, fixed_one, default: int) -> torch.Tensor:
    """uint8 class per coordinate (0 free, 1 fixed-one, 2 fixed-zero)."""
    cls = np.full(p, default, dtype=np.uint8)
    if len(free):
        cls[np.asarray(free, dtype=np.int64)] = native.FREE
    if len(fixed_one):
        cls[np.asarray(fixed_one, dtype=np.int64)] = native.FIXED_ONE
    return torch.from_numpy(cls).to(device())
