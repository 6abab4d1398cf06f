"""ctypes binding of the C-ABI in include/pathtrack_b200.h.

The shared library is built in-tree (``make`` at the repo root, or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
importing this module raises, and every compute call on a machine without an
sm_100 device returns PT_E_NODEVICE.
"""
from __future__ import annotations

import ctypes as C
import os

from ._abi import *  # noqa: F401,F403  (structs, error codes, pointer helpers)
from ._abi import NativeError, PathStats, StepParams, SystemDesc, TraceEvent, _dp, _vp, dptr, iptr  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
# PT_LIB_PATH: A/B experiments only (tools/); the product loads the in-tree library
LIB_PATH = os.environ.get("PT_LIB_PATH") or os.path.join(_HERE, "libpathtrack_b200.so")


# name -> (restype, argtypes); every symbol declared in include/pathtrack_b200.h
PROTOTYPES = {
    "pt_default_params": (C.c_int, [C.c_int, C.POINTER(StepParams)]),
    "pt_device_count": (C.c_int, []),
    "pt_plan_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(SystemDesc), C.POINTER(SystemDesc), _dp, C.c_int32,
                                 C.POINTER(_vp)]),
    "pt_plan_destroy": (None, [_vp]),
    "pt_plan_info": (C.c_int64, [_vp, C.c_int32]),
    "pt_plan_set_engine": (C.c_int, [_vp, C.c_int32]),
    "pt_plan_set_arith": (C.c_int, [_vp, C.c_int32]),
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
    "pt_eval_bench": (C.c_int, [_vp, _dp, C.c_double, C.c_int32, _dp]),
    "pt_lstsq": (C.c_int, [C.c_int, C.c_int, C.c_int32, C.c_int32, _dp, _dp, _dp]),
    "pt_arith_device": (C.c_int, [C.c_int, C.c_int, C.c_int32, C.c_int64, _dp, _dp, _dp]),
    "pt_arith_device_mode": (C.c_int, [C.c_int, C.c_int, C.c_int32, C.c_int32, C.c_int64, _dp, _dp, _dp]),
    "pt_arith_host": (C.c_int, [C.c_int, C.c_int32, C.c_int64, _dp, _dp, _dp]),
    "pt_last_error": (C.c_char_p, []),
    "pt_version": (C.c_char_p, []),
}


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

