"""ctypes binding of the host-only inputs library (include/pathtrack_inputs.h,
libpt_inputs.so): synthetic systems, system / solution files, hex limbs,
Pieri minors.  Loading it never loads the CUDA tracker library, so the
reference arm of bench.py and the CPU oracle tests can build the same inputs
without touching the product."""
from __future__ import annotations

import ctypes as C
import os

from ._abi import NativeError, SystemDesc, _dp, _vp, dptr, iptr  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpt_inputs.so")

_i32p = C.POINTER(C.c_int32)
_cpp = C.POINTER(C.c_void_p)  # char** (malloc'ed text, released with pt_text_free)

# name -> (restype, argtypes); every symbol declared in include/pathtrack_inputs.h
PROTOTYPES = {
    "pt_inputs_last_error": (C.c_char_p, []),
    "pt_text_free": (None, [C.c_void_p]),
    "pt_hex_encode_limb": (C.c_int, [C.c_double, C.c_char_p]),
    "pt_hex_decode_limb": (C.c_int, [C.c_char_p, C.c_int32, _dp]),
    "pt_hex_limbs": (C.c_int, [_dp, C.c_int32, _cpp]),
    "pt_parse_hex_limbs": (C.c_int, [C.c_char_p, C.c_int32, _dp, C.c_int32, _i32p]),
    "pt_system_parse": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_vp)]),
    "pt_system_serialize": (C.c_int, [C.POINTER(SystemDesc), C.c_int, _cpp]),
    "pt_solutions_write": (C.c_int, [C.c_int32, C.c_int, C.c_int32, _dp, _dp, _dp, _dp, _cpp]),
    "pt_solutions_read": (C.c_int, [C.c_char_p, C.c_int, C.c_int32, _i32p, _i32p, _dp, _dp, _dp, _dp]),
    "pt_gen_cyclic": (C.c_int, [C.c_int32, C.c_int, C.POINTER(_vp)]),
    "pt_gen_augment": (C.c_int, [_vp, C.c_int32, C.c_uint64, C.c_int, C.POINTER(_vp)]),
    "pt_gen_chandra": (C.c_int, [C.c_int32, C.c_double, C.c_int, C.POINTER(_vp)]),
    "pt_gen_random_dense": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_int, C.POINTER(_vp)]),
    "pt_gen_total_degree": (C.c_int, [C.c_int32, C.c_int32, C.c_int, C.POINTER(_vp)]),
    "pt_sysbuf_desc": (C.c_int, [_vp, C.POINTER(SystemDesc)]),
    "pt_sysbuf_from_desc": (C.c_int, [C.POINTER(SystemDesc), C.c_int, C.POINTER(_vp)]),
    "pt_sysbuf_stack": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "pt_sysbuf_free": (None, [_vp]),
    "pt_gen_gamma": (C.c_int, [C.c_uint64, C.c_int, _dp]),
    "pt_gen_unit_complex": (C.c_int, [C.c_double, C.c_int, _dp]),
    "pt_cyclic_degree": (C.c_int, [C.c_int32, _i32p, _i32p, _i32p, _i32p]),
    "pt_pieri_events": (C.c_int, [C.c_int32, C.c_int32, _i32p, _i32p]),
    "pt_pieri_planes": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_int, _dp]),
    "pt_pieri_minor": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _dp, C.c_int, C.POINTER(_vp)]),
    "pt_pieri_det": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _dp, _dp, C.c_int, _dp]),
    "pt_pieri_linear_start": (C.c_int, [C.c_int32, C.c_int32, _dp, C.c_int, _dp]),
    "pt_pieri_special": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _dp, C.c_int, _dp]),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(code: int) -> int:
    if code != 0:
        raise NativeError(code, (lib.pt_inputs_last_error() or b"").decode())
    return code


def take_text(p: C.c_void_p) -> str:
    """Copy a malloc'ed C string returned through char** and free it."""
    try:
        return C.string_at(p.value).decode()
    finally:
        lib.pt_text_free(p)
