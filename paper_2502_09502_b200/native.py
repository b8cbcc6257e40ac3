"""ctypes binding of libl0b200.so (include/l0cert_b200.h).

The product path has no fallback: if the library is missing or no CUDA device
is present, ``load()`` raises.  ``lib()`` returns the loaded handle.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (InfeasibleNodeError, InvalidInputError, L0CertError, NumericalError,
                     UnsupportedOperationError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libl0b200.so")

OK, INVALID, NUMERICAL, INFEASIBLE, UNSUPPORTED, CUDA_ERR, ABORTED = range(7)
F64, F32 = 0, 1
LOSS_CODES = {"squared_error": 0, "logistic": 1, "squared_hinge": 2, "poisson": 3, "gamma": 4}
TERMINATIONS = ("converged", "iteration_limit", "time_limit", "primal_below_incumbent",
                "dual_above_incumbent")
FREE, FIXED_ONE, FIXED_ZERO = 0, 1, 2

c_i32, c_i64, c_u64, c_f64, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                    ctypes.c_double, ctypes.c_void_p)


class FistaOpts(ctypes.Structure):
    _fields_ = [("max_iterations", c_i64), ("gap_tolerance", c_f64), ("time_limit", c_f64),
                ("early_primal_cutoff", c_f64), ("early_dual_cutoff", c_f64),
                ("bound_check_interval", c_i32), ("restart", c_i32), ("lipschitz", c_f64),
                ("gap_tolerance_rel", c_f64), ("stop_on_gap", c_i32),
                ("chunk_iterations", c_i32), ("profile", c_i32), ("engine_path", c_i32),
                ("fp32_forward", c_i32)]


class Node(ctypes.Structure):
    _fields_ = [("h_fixed_one", ctypes.POINTER(c_i64)), ("n_fixed_one", c_i64),
                ("h_fixed_zero", ctypes.POINTER(c_i64)), ("n_fixed_zero", c_i64),
                ("parent_bound", c_f64)]


class Report(ctypes.Structure):
    _fields_ = [("primal_value", c_f64), ("dual_bound", c_f64), ("gap", c_f64),
                ("iterations", c_i64), ("restarts", c_i64), ("termination", c_i32),
                ("status", c_i32), ("error_iteration", c_i64), ("wall_time", c_f64),
                ("gpu_launches", c_i64), ("topk_fallbacks", c_i64), ("k1_ms", c_f64),
                ("k2_ms", c_f64), ("k3_ms", c_f64), ("k1_count", c_i64), ("k2_count", c_i64),
                ("k3_count", c_i64), ("prox_full_passes", c_i64), ("single_pass", c_i32),
                ("cluster_size", c_i32)]


class TraceRecord(ctypes.Structure):
    _fields_ = [("iteration", c_f64), ("primal", c_f64), ("dual", c_f64), ("gap", c_f64),
                ("restarted", c_f64)]


TRACE_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(TraceRecord), c_vp)

# name -> (restype, argtypes)
_PROTOS = {
    "l0_last_error": (ctypes.c_char_p, []),
    "l0_abi_version": (c_i32, []),
    "l0_problem_create": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, c_vp, c_i32, ctypes.POINTER(c_vp)]),
    "l0_problem_workspace_bytes": (c_i32, [c_vp, ctypes.POINTER(c_u64)]),
    "l0_problem_set_workspace": (c_i32, [c_vp, c_vp, c_u64]),
    "l0_problem_destroy": (c_i32, [c_vp]),
    "l0_problem_set_comm": (c_i32, [c_vp, c_vp, c_i32, c_i32]),
    "l0_nccl_unique_id": (c_i32, [c_vp]),
    "l0_fista_solve": (c_i32, [c_vp, c_i64, c_f64, c_f64, ctypes.POINTER(FistaOpts),
                               ctypes.POINTER(Node), c_vp, c_vp, ctypes.POINTER(Report), TRACE_CB,
                               c_vp, c_vp]),
    "l0_debug_probe": (c_i32, [c_vp, ctypes.POINTER(c_i64)]),
    "l0_problem_set_prox_record": (c_i32, [c_vp, c_vp, c_i32, c_i32]),
    "l0_upload_rows": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i32, c_vp]),
    "l0_debug_scratch": (c_i32, [c_vp, c_vp, c_i64]),
    "l0_matvec": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "l0_rmatvec": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "l0_power_iteration": (c_i32, [c_vp, c_vp, c_f64, c_i64, ctypes.POINTER(c_f64),
                                   ctypes.POINTER(c_i64), c_vp]),
    "l0_safe_lower_bound": (c_i32, [c_vp, c_vp, c_i64, c_f64, c_f64, c_vp,
                                    ctypes.POINTER(c_f64), c_vp]),
    "l0_safe_lower_bound_batched_workspace": (c_i32, [c_vp, c_i64, ctypes.POINTER(c_u64)]),
    "l0_safe_lower_bound_batched": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_f64, c_f64, c_vp, c_vp, c_vp,
                                            c_u64, c_vp]),
    "l0_standardize_stats": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "l0_standardize_apply": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "l0_refit_ridge": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_f64, c_f64, c_vp, c_vp, c_vp]),
    "l0_ops_workspace_bytes": (c_i32, [c_i64, ctypes.POINTER(c_u64)]),
    "l0_prox": (c_i32, [c_vp, c_i64, c_f64, c_i64, c_f64, c_vp, c_i32, c_vp, c_vp,
                        ctypes.POINTER(c_i64), c_vp, c_u64, c_vp]),
    "l0_g_value": (c_i32, [c_vp, c_i64, c_i64, c_f64, c_vp, c_vp, c_i64, ctypes.POINTER(c_f64),
                           c_vp, c_u64, c_vp]),
    "l0_g_conjugate": (c_i32, [c_vp, c_i64, c_i64, c_f64, c_vp, ctypes.POINTER(c_f64), c_vp,
                               c_u64, c_vp]),
    "l0_huber": (c_i32, [c_vp, c_i64, c_f64, c_f64, c_i32, c_vp, c_vp]),
    "l0_loss_value": (c_i32, [c_i32, c_vp, c_vp, c_i64, ctypes.POINTER(c_f64), c_vp,
                              ctypes.POINTER(c_i32), c_vp, c_u64, c_vp]),
    "l0_loss_conjugate": (c_i32, [c_i32, c_vp, c_vp, c_i64, ctypes.POINTER(c_f64), c_vp, c_u64,
                                  c_vp]),
    "l0_all_finite": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, ctypes.POINTER(c_i32), c_vp,
                              c_u64, c_vp]),
    "l0_batch_create": (c_i32, [c_vp, c_i64, ctypes.POINTER(c_vp)]),
    "l0_batch_workspace_bytes": (c_i32, [c_vp, ctypes.POINTER(c_u64)]),
    "l0_batch_set_workspace": (c_i32, [c_vp, c_vp, c_u64]),
    "l0_batch_solve": (c_i32, [c_vp, c_i64, c_f64, c_f64, ctypes.POINTER(FistaOpts),
                               c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "l0_batch_destroy": (c_i32, [c_vp]),
    "l0_tc_gemm_workspace_bytes": (c_u64, [c_i64, c_i64, c_i64]),
    "l0_tc_gemm_3xtf32": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, c_vp, c_i32, c_i64, c_i64,
                                  c_vp, c_i64, c_i32, ctypes.POINTER(c_i32), c_vp, c_u64, c_vp]),
    "l0_tc_gemm_3xf16": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, c_vp, c_i32, c_i64, c_i64,
                                 c_vp, c_i64, c_i32, ctypes.POINTER(c_i32), c_vp, c_u64, c_vp]),
}

EXPORTED = tuple(_PROTOS)

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """dlopen the engine library and bind every prototype (no GPU needed)."""
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the B200 engine first "
            "(python -m paper_2502_09502_b200.build)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def load() -> ctypes.CDLL:
    """The engine library, checked to run on a CUDA device.  Raises loudly."""
    global _lib
    with _lock:
        if _lib is None:
            import torch
            if not torch.cuda.is_available():
                raise RuntimeError("the B200 engine needs a CUDA device; none is visible")
            _lib = load_library()
            torch.cuda.init()
    return _lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load()


def last_error() -> str:
    msg = lib().l0_last_error()
    return msg.decode() if msg else ""


def check(rc: int, iteration=None) -> None:
    """Map an l0_status to the reference's exception classes (errors.py)."""
    if rc == OK:
        return
    msg = last_error()
    if rc == INVALID:
        raise InvalidInputError(msg)
    if rc == NUMERICAL:
        raise NumericalError(msg, iteration=iteration)
    if rc == INFEASIBLE:
        raise InfeasibleNodeError(msg)
    if rc == UNSUPPORTED:
        raise UnsupportedOperationError(msg)
    raise L0CertError(f"engine failure ({rc}): {msg}")
