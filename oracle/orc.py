"""TEST INFRASTRUCTURE -- ctypes wrapper of the CPU oracle (never the product).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module.

Two builds of the same SPEC-following tracker (oracle/orc_tracker.hpp):
  * liborc.so           arithmetic restated in oracle/orc_arith.hpp
  * _ref/liborc_ref.so  arithmetic from the UNMODIFIED reference headers
                        (/root/reference/proj/include, built by `make ref`)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED = os.path.join(HERE, "liborc.so")
REFERENCE = os.path.join(HERE, "_ref", "liborc_ref.so")


class SystemDesc(C.Structure):  # same layout as pt_system_desc
    _fields_ = [("n_vars", C.c_int32), ("n_eqs", C.c_int32), ("n_terms", C.c_int32),
                ("eq_ptr", C.POINTER(C.c_int32)), ("term_ptr", C.POINTER(C.c_int32)),
                ("var", C.POINTER(C.c_int32)), ("exp", C.POINTER(C.c_int32)), ("coef", C.POINTER(C.c_double))]


class StepParams(C.Structure):
    _fields_ = [("max_step", C.c_double), ("min_step", C.c_double), ("max_steps", C.c_int32),
                ("pred_degree", C.c_int32), ("newton_max_iter", C.c_int32), ("reserved", C.c_int32),
                ("newton_tol", C.c_double)]


class PathStats(C.Structure):
    _fields_ = [("status", C.c_int32), ("failure_kind", C.c_int32), ("steps", C.c_int32),
                ("accepted", C.c_int32), ("newton_iters", C.c_int32), ("start_iters", C.c_int32), ("solves", C.c_int32), ("reserved", C.c_int32),
                ("final_residual", C.c_double), ("final_update", C.c_double), ("t_end", C.c_double)]


class TraceEvent(C.Structure):
    _fields_ = [("t", C.c_double), ("ok", C.c_int32), ("iters", C.c_int32), ("residual", C.c_double),
                ("update", C.c_double)]


_dp = C.POINTER(C.c_double)


def build(ref: bool = False) -> None:
    """Compile the oracle in place (restatement always; ref only where
    /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE] + (["ref"] if ref else []), check=True)


class Oracle:
    def __init__(self, variant: str = "auto"):
        if variant == "auto":
            variant = "reference" if os.path.exists(REFERENCE) else "restatement"
        path = REFERENCE if variant == "reference" else RESTATED
        if not os.path.exists(path):
            if variant == "restatement":
                build()
            else:
                raise FileNotFoundError(path)
        self.path = path
        self.variant = variant
        lib = C.CDLL(path)
        lib.orc_track_path.argtypes = [C.c_int, C.POINTER(SystemDesc), C.POINTER(SystemDesc), _dp, C.c_int, _dp,
                                       C.POINTER(StepParams), _dp, C.POINTER(PathStats), C.POINTER(TraceEvent),
                                       C.c_int, C.POINTER(C.c_int)]
        lib.orc_eval_homotopy.argtypes = [C.c_int, C.POINTER(SystemDesc), C.POINTER(SystemDesc), _dp, C.c_int, _dp,
                                          C.c_double, _dp, _dp, _dp]
        lib.orc_lstsq.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        lib.orc_arith.argtypes = [C.c_int, C.c_int, C.c_long, _dp, _dp, _dp]
        lib.orc_track_batch.argtypes = [C.c_int, C.POINTER(SystemDesc), C.POINTER(SystemDesc), _dp, C.c_int, C.c_int,
                                        _dp, C.POINTER(StepParams), _dp, C.POINTER(PathStats), C.c_int]
        if variant == "reference":
            lib.orc_ref_hex_limbs.argtypes = [_dp, C.c_int, C.c_char_p, C.c_int]
            lib.orc_ref_parse_hex_limbs.argtypes = [C.c_char_p, C.c_int, _dp, C.c_int, C.POINTER(C.c_int)]
        lib.orc_set_threads.argtypes = [C.c_int]
        lib.orc_variant.restype = C.c_char_p
        lib.orc_last_error.restype = C.c_char_p
        self.lib = lib

    # ---- helpers -----------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"oracle error {rc}: {self.lib.orc_last_error().decode()}")

    @staticmethod
    def _desc(sysm):
        """sysm: object with n_vars, eq_ptr, term_ptr, var, exp, coef (numpy)."""
        keep = [np.ascontiguousarray(getattr(sysm, k), dtype=np.int32) for k in ("eq_ptr", "term_ptr", "var", "exp")]
        keep = [a if a.size else np.zeros(1, np.int32) for a in keep]
        coef = np.ascontiguousarray(sysm.coef, dtype=np.float64)
        d = SystemDesc(sysm.n_vars, int(keep[0].size - 1), int(keep[1].size - 1),
                       *[a.ctypes.data_as(C.POINTER(C.c_int32)) for a in keep], coef.ctypes.data_as(_dp))
        return d, (keep, coef)

    def set_threads(self, n: int) -> None:
        self.lib.orc_set_threads(int(n))

    def max_threads(self) -> int:
        return int(self.lib.orc_max_threads())

    # ---- API ---------------------------------------------------------------
    def track_path(self, prec: int, g, f, gamma, k, start, params, trace_cap: int = 0):
        gd, kg = self._desc(g)
        fd, kf = self._desc(f)
        gamma = np.ascontiguousarray(gamma, dtype=np.float64)
        start = np.ascontiguousarray(start, dtype=np.float64)
        end = np.zeros_like(start)
        st = PathStats()
        sp = StepParams(params.max_step, params.min_step, params.max_steps, params.pred_degree,
                        params.newton_max_iter, 0, params.newton_tol)
        tr = (TraceEvent * max(trace_cap, 1))()
        tl = C.c_int(0)
        self._check(self.lib.orc_track_path(int(prec), C.byref(gd), C.byref(fd), gamma.ctypes.data_as(_dp), int(k),
                                            start.ctypes.data_as(_dp), C.byref(sp), end.ctypes.data_as(_dp),
                                            C.byref(st), tr if trace_cap else None, trace_cap, C.byref(tl)))
        return end, st, list(tr[: min(tl.value, trace_cap)]) if trace_cap else []

    def track_batch(self, prec: int, g, f, gamma, k, starts, params, threads: int):
        """Independent paths on a pool of `threads` host threads, one
        single-threaded tracker per path (the batch CPU baseline)."""
        gd, kg = self._desc(g)
        fd, kf = self._desc(f)
        gamma = np.ascontiguousarray(gamma, dtype=np.float64)
        starts = np.ascontiguousarray(starts, dtype=np.float64)
        P = starts.shape[0]
        ends = np.zeros_like(starts)
        stats = (PathStats * max(P, 1))()
        sp = StepParams(params.max_step, params.min_step, params.max_steps, params.pred_degree,
                        params.newton_max_iter, 0, params.newton_tol)
        self._check(self.lib.orc_track_batch(int(prec), C.byref(gd), C.byref(fd), gamma.ctypes.data_as(_dp), int(k),
                                             P, starts.ctypes.data_as(_dp), C.byref(sp), ends.ctypes.data_as(_dp),
                                             stats, int(threads)))
        return ends, list(stats[:P])

    def ref_hex_limbs(self, limbs) -> str:
        """The reference's hex_limbs (hexio.cpp) -- reference variant only."""
        a = np.ascontiguousarray(np.atleast_1d(limbs), dtype=np.float64)
        buf = C.create_string_buffer(32 + 17 * a.size)
        self._check(self.lib.orc_ref_hex_limbs(a.ctypes.data_as(_dp), a.size, buf, len(buf)))
        return buf.value.decode()

    def ref_parse_hex_limbs(self, text: str):
        """The reference's parse_hex_limbs; None when it throws."""
        raw = text.encode()
        out = np.zeros(64)
        cnt = C.c_int()
        if self.lib.orc_ref_parse_hex_limbs(raw, len(raw), out.ctypes.data_as(_dp), 64, C.byref(cnt)) != 0:
            return None
        return out[: cnt.value].copy()

    def eval_homotopy(self, prec: int, g, f, gamma, k, x, t):
        gd, kg = self._desc(g)
        fd, kf = self._desc(f)
        L = (1, 2, 4)[int(prec)]
        n, N = g.n_vars, int(np.asarray(g.eq_ptr).size - 1)
        gamma = np.ascontiguousarray(gamma, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        h = np.zeros((2, L, N))
        J = np.zeros((2, L, N * n))
        r = np.zeros(1)
        self._check(self.lib.orc_eval_homotopy(int(prec), C.byref(gd), C.byref(fd), gamma.ctypes.data_as(_dp), int(k),
                                               x.ctypes.data_as(_dp), C.c_double(t), h.ctypes.data_as(_dp),
                                               J.ctypes.data_as(_dp), r.ctypes.data_as(_dp)))
        return h, J, float(r[0])

    def lstsq(self, prec: int, A, b):
        L = (1, 2, 4)[int(prec)]
        A = np.ascontiguousarray(A, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        N = b.shape[-1]
        n = A.shape[-1] // N
        x = np.zeros((2, L, n))
        rc = self.lib.orc_lstsq(int(prec), N, n, A.ctypes.data_as(_dp), b.ctypes.data_as(_dp), x.ctypes.data_as(_dp))
        if rc == -3:
            return None
        self._check(rc)
        return x

    def arith(self, prec: int, op: int, a, b):
        L = (1, 2, 4)[int(prec)]
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.zeros_like(a)
        self._check(self.lib.orc_arith(int(prec), int(op), a.size // (2 * L), a.ctypes.data_as(_dp),
                                       b.ctypes.data_as(_dp), out.ctypes.data_as(_dp)))
        return out
