"""ctypes binding of the C-ABI in include/pathtrack_b200.h.

The shared library is built in-tree (``make`` at the repo root, or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
importing this module raises, and every compute call on a machine without an
sm_100 device returns PT_E_NODEVICE.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpathtrack_b200.so")

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
        ("start_iters", C.c_int32), ("solves", C.c_int32), ("reserved", C.c_int32),
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

# name -> (restype, argtypes); every symbol declared in include/pathtrack_b200.h
PROTOTYPES = {
    "pt_default_params": (C.c_int, [C.c_int, C.POINTER(StepParams)]),
    "pt_device_count": (C.c_int, []),
    "pt_plan_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(SystemDesc), C.POINTER(SystemDesc), _dp, C.c_int32,
                                 C.POINTER(_vp)]),
    "pt_plan_destroy": (None, [_vp]),
    "pt_plan_info": (C.c_int64, [_vp, C.c_int32]),
    "pt_plan_set_engine": (C.c_int, [_vp, C.c_int32]),
    "pt_plan_set_trace": (C.c_int, [_vp, C.c_int32]),
    "pt_plan_work": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp]),
    "pt_fp64_peak": (C.c_int, [C.c_int, _dp, _dp]),
    "pt_plan_profile": (C.c_int, [_vp, _dp, C.c_int32]),
    "pt_plan_batch_profile": (C.c_int, [_vp, C.c_int32, _dp, C.c_int32]),
    "pt_plan_mgs_timeline": (C.c_int, [_vp, _dp, C.c_int32]),
    "pt_microbench": (C.c_int, [C.c_int, C.c_int32, _dp]),
    "pt_plan_get_trace": (C.c_int, [_vp, C.POINTER(TraceEvent), C.c_int32, C.POINTER(C.c_int32)]),
    "pt_track_path": (C.c_int, [_vp, _dp, C.POINTER(StepParams), _dp, C.POINTER(PathStats)]),
    "pt_track_path_device": (C.c_int, [_vp, _vp, C.POINTER(StepParams), _vp, _vp, _vp]),
    "pt_track_batch": (C.c_int, [_vp, C.c_int32, _dp, C.POINTER(StepParams), _dp, C.POINTER(PathStats)]),
    "pt_track_batch_device": (C.c_int, [_vp, C.c_int32, _vp, C.POINTER(StepParams), _vp, _vp, _vp]),
    "pt_eval_homotopy": (C.c_int, [_vp, _dp, C.c_double, _dp, _dp, _dp]),
    "pt_lstsq": (C.c_int, [C.c_int, C.c_int, C.c_int32, C.c_int32, _dp, _dp, _dp]),
    "pt_arith_device": (C.c_int, [C.c_int, C.c_int, C.c_int32, C.c_int64, _dp, _dp, _dp]),
    "pt_arith_host": (C.c_int, [C.c_int, C.c_int32, C.c_int64, _dp, _dp, _dp]),
    "pt_last_error": (C.c_char_p, []),
    "pt_version": (C.c_char_p, []),
    "pt_gen_cyclic": (C.c_int, [C.c_int32, C.c_int, C.POINTER(_vp)]),
    "pt_gen_augment": (C.c_int, [_vp, C.c_int32, C.c_uint64, C.c_int, C.POINTER(_vp)]),
    "pt_gen_chandra": (C.c_int, [C.c_int32, C.c_double, C.c_int, C.POINTER(_vp)]),
    "pt_gen_random_dense": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_int, C.POINTER(_vp)]),
    "pt_gen_total_degree": (C.c_int, [C.c_int32, C.c_int32, C.c_int, C.POINTER(_vp)]),
    "pt_sysbuf_desc": (C.c_int, [_vp, C.POINTER(SystemDesc)]),
    "pt_sysbuf_free": (None, [_vp]),
    "pt_gen_gamma": (C.c_int, [C.c_uint64, C.c_int, _dp]),
    "pt_gen_unit_complex": (C.c_int, [C.c_double, C.c_int, _dp]),
}


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pathtrack_b200 error {code}: {msg}")
        self.code = code


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "the tracker has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(code: int) -> int:
    if code != PT_OK:
        raise NativeError(code, (lib.pt_last_error() or b"").decode())
    return code


def dptr(a) -> C.POINTER(C.c_double):
    return a.ctypes.data_as(_dp)


def iptr(a) -> C.POINTER(C.c_int32):
    return a.ctypes.data_as(C.POINTER(C.c_int32))
