"""Thin ctypes binding of libpcdn.so with the C-ABI's names (include/pcdn.h).

Argument marshalling only: torch tensors supply device pointers and streams; every step of
the PCDN path runs in the library's CUDA kernels.  There is no CPU fallback: if the library
is missing, importing the bindings raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PCDN_LIB (A/B measurements of prebuilt variants): another build of the same library, e.g. under scratch/
LIB_PATH = os.environ.get("PCDN_LIB") or os.path.join(HERE, "libpcdn.so")

PCDN_OK, PCDN_ERR_INVALID, PCDN_BUDGET, PCDN_ERR_NUMERIC, PCDN_ERR_CUDA, PCDN_ERR_NOMEM = 0, 1, 2, 3, 4, 5
PCDN_LOSS_LOGISTIC, PCDN_LOSS_L2SVM, PCDN_LOSS_SQUARED = 0, 1, 2
STATUS_NAMES = {0: "PCDN_OK", 1: "PCDN_ERR_INVALID", 2: "PCDN_BUDGET", 3: "PCDN_ERR_NUMERIC",
                4: "PCDN_ERR_CUDA", 5: "PCDN_ERR_NOMEM"}


class PCDNError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class pcdn_step_info(C.Structure):
    _fields_ = [("q", C.c_int32), ("reserved", C.c_int32), ("alpha", C.c_double), ("Delta", C.c_double),
                ("lhs", C.c_double), ("rhs", C.c_double), ("F", C.c_double), ("bundle_nnz", C.c_int64),
                ("n_touched", C.c_int64)]


class pcdn_solve_info(C.Structure):
    _fields_ = [("status", C.c_int32), ("outer_iters", C.c_int32), ("steps", C.c_int64),
                ("null_steps", C.c_int64), ("nnz_processed", C.c_int64), ("touched_total", C.c_int64),
                ("positions", C.c_int64), ("kernel_launches", C.c_int64), ("F", C.c_double),
                ("gap", C.c_double), ("t_wall_ms", C.c_double), ("t_step_kernel_ms", C.c_double),
                ("t_gpu_ms", C.c_double), ("alg_bytes", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class pcdn_shard_decision(C.Structure):
    _fields_ = [("q", C.c_int32), ("next", C.c_int32), ("alpha", C.c_double), ("lhs", C.c_double),
                ("rhs", C.c_double), ("Delta", C.c_double), ("F", C.c_double)]


P = C.c_void_p
I64 = C.c_int64
# name -> (restype, argtypes), exactly the functions declared in include/pcdn.h
SIGNATURES = {
    "pcdn_workspace_bytes": (C.c_size_t, [I64, I64, I64]),
    "pcdn_create": (C.c_int, [I64, I64, I64, P, P, P, P, P, P, P, C.c_double, C.c_int, P, C.c_size_t, P,
                              C.POINTER(P)]),
    "pcdn_set_armijo": (C.c_int, [P, C.c_double, C.c_double, C.c_double, C.c_int]),
    "pcdn_set_reference": (C.c_int, [P, C.c_double]),
    "pcdn_bundle_step": (C.c_int, [P, P, I64, C.POINTER(pcdn_step_info), P, P, P]),
    "pcdn_last_touched": (C.c_int, [P, P, P, I64, C.POINTER(I64)]),
    "pcdn_solve": (C.c_int, [P, I64, C.c_double, C.c_uint64, C.c_int32, C.POINTER(pcdn_solve_info)]),
    "pcdn_objective": (C.c_int, [P, C.c_int, C.POINTER(C.c_double)]),
    "pcdn_get_w": (C.c_int, [P, P]),
    "pcdn_set_w": (C.c_int, [P, P]),
    "pcdn_get_z": (C.c_int, [P, P]),
    "pcdn_reset": (C.c_int, [P]),
    "pcdn_permutation": (C.c_int, [P, C.c_uint64, I64, P]),
    "pcdn_set_trace": (C.c_int, [P, P, P, I64]),
    "pcdn_set_debug": (C.c_int, [P, C.c_int]),
    "pcdn_set_launch": (C.c_int, [P, C.c_int, C.c_int, C.c_int]),
    "pcdn_set_resident_cap": (C.c_int, [P, C.c_int]),
    "pcdn_set_l2_persist": (C.c_int, [P, C.c_int]),
    "pcdn_set_elastic": (C.c_int, [P, C.c_double]),
    "pcdn_set_targets": (C.c_int, [P, C.c_void_p]),
    "pcdn_set_scdn": (C.c_int, [P, C.c_int]),
    "pcdn_shard_gh": (C.c_int, [P, C.c_void_p, C.c_int64, C.c_void_p]),
    "pcdn_shard_direction": (C.c_int, [P, C.c_void_p, C.c_int64, C.c_void_p]),
    "pcdn_shard_line_search": (C.c_int, [P, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    "pcdn_shard_decide": (C.c_int, [P, C.c_void_p, C.c_int, C.POINTER(pcdn_shard_decision)]),
    "pcdn_shard_commit": (C.c_int, [P, C.c_void_p, C.c_int64]),
    "pcdn_shard_loss": (C.c_int, [P, C.c_void_p]),
    "pcdn_shard_objective": (C.c_int, [P, C.c_void_p, C.POINTER(C.c_double)]),
    "pcdn_set_profile": (C.c_int, [P, C.c_int]),
    "pcdn_phase_cycles": (C.c_int, [P, P, C.POINTER(C.c_int32)]),
    "pcdn_warp_timeline": (C.c_int, [P, P]),
    "pcdn_last_error": (C.c_char_p, [P]),
    "pcdn_destroy": (None, [P]),
    "pcdn_train_host": (C.c_int, [I64, I64, I64, P, P, P, P, P, P, P, C.c_double, C.c_int, I64, C.c_double,
                                  C.c_double, C.c_uint64, C.c_int32, P, P, C.POINTER(pcdn_solve_info)]),
    "pcdn_version": (C.c_char_p, []),
}

_lib = None


def lib():
    """Load libpcdn.so (built by paper_1306_4080_b200.build / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1306_4080_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(ctx, status, ok=(PCDN_OK,)):
    if status in ok:
        return status
    msg = lib().pcdn_last_error(ctx).decode() if ctx else ""
    raise PCDNError(status, msg)
