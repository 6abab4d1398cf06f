"""ctypes mirrors of the plain structs shared by both C-ABIs
(include/pathtrack_b200.h, include/pathtrack_inputs.h).  Loads no library."""
from __future__ import annotations

import ctypes as C

PT_OK = 0
PT_E_INVAL = -1
PT_E_CUDA = -2
PT_E_RANK = -3
PT_E_NODEVICE = -4
PT_E_TIMEOUT = -5
PT_E_NOMEM = -6


class SystemDesc(C.Structure):
    _fields_ = [
        ("n_vars", C.c_int32),
        ("n_eqs", C.c_int32),
        ("n_terms", C.c_int32),
        ("eq_ptr", C.POINTER(C.c_int32)),
        ("term_ptr", C.POINTER(C.c_int32)),
        ("var", C.POINTER(C.c_int32)),
        ("exp", C.POINTER(C.c_int32)),
        ("coef", C.POINTER(C.c_double)),
    ]


class StepParams(C.Structure):
    _fields_ = [
        ("max_step", C.c_double),
        ("min_step", C.c_double),
        ("max_steps", C.c_int32),
        ("pred_degree", C.c_int32),
        ("newton_max_iter", C.c_int32),
        ("reserved", C.c_int32),
        ("newton_tol", C.c_double),
    ]


class PathStats(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("failure_kind", C.c_int32),
        ("steps", C.c_int32),
        ("accepted", C.c_int32),
        ("newton_iters", C.c_int32),
        ("start_iters", C.c_int32), ("solves", C.c_int32), ("flags", C.c_int32),
        ("final_residual", C.c_double),
        ("final_update", C.c_double),
        ("t_end", C.c_double),
    ]


class TraceEvent(C.Structure):
    _fields_ = [
        ("t", C.c_double),
        ("ok", C.c_int32),
        ("iters", C.c_int32),
        ("residual", C.c_double),
        ("update", C.c_double),
    ]


_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pathtrack_b200 error {code}: {msg}")
        self.code = code


def dptr(a) -> C.POINTER(C.c_double):
    return a.ctypes.data_as(_dp)


def iptr(a) -> C.POINTER(C.c_int32):
    return a.ctypes.data_as(C.POINTER(C.c_int32))
