"""Inputs of the tracker: precision modes, polynomial systems, step-control
parameters, the synthetic generators and the system / solution file formats.

Host-only: everything here goes through libpt_inputs.so
(include/pathtrack_inputs.h) and never loads the CUDA tracker library, so the
CPU oracle and the reference arm of bench.py build exactly the same inputs.

  PrecisionMode                multiprec.hpp:27
  PolynomialSystem             SPEC.md:133-136 (canonical form :150)
  parse_system / serialize_system   SPEC.md:147-159 (grammar :197)
  read_solutions / write_solutions
  StepControlParams
  cyclic_system / augment_with_linear / cyclic_degree
  hex_encode_limb / hex_decode_limb / hex_limbs / parse_hex_limbs
                               proj/include/pathtrack/hexio.hpp:16-24
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _inputs as inp
from ._abi import StepParams, SystemDesc, dptr, iptr


class PrecisionMode(enum.IntEnum):  # multiprec.hpp:27
    D = 0
    DD = 1
    QD = 2

    @property
    def limbs(self) -> int:
        return (1, 2, 4)[int(self)]

    @staticmethod
    def parse(text: str) -> "PrecisionMode":  # precision.cpp:22-27
        m = {"d": PrecisionMode.D, "dd": PrecisionMode.DD, "qd": PrecisionMode.QD}
        if text not in m:
            raise ValueError(f"unknown precision mode '{text}' (expected d, dd, or qd)")
        return m[text]


def limbs_from_complex(z, prec: PrecisionMode) -> np.ndarray:
    """complex128 vector -> (2, L, n) limbs with the value in limb 0."""
    z = np.asarray(z, dtype=np.complex128).reshape(-1)
    out = np.zeros((2, prec.limbs, z.size))
    out[0, 0] = z.real
    out[1, 0] = z.imag
    return out


def complex_from_limbs(a: np.ndarray) -> np.ndarray:
    """(2, L, n) limbs -> complex128 (sum of limbs rounded to binary64)."""
    a = np.asarray(a)
    return a[0].sum(axis=0) + 1j * a[1].sum(axis=0)


@dataclass
class PolynomialSystem:
    """Canonical distributed form, pt_system_desc layout."""

    n_vars: int
    eq_ptr: np.ndarray
    term_ptr: np.ndarray
    var: np.ndarray
    exp: np.ndarray
    coef: np.ndarray  # (2, L, n_terms)
    prec: PrecisionMode

    @property
    def n_eqs(self) -> int:
        return int(self.eq_ptr.size - 1)

    @property
    def n_terms(self) -> int:
        return int(self.term_ptr.size - 1)

    def desc(self) -> SystemDesc:
        for name in ("eq_ptr", "term_ptr", "var", "exp"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.int32))
        self.coef = np.ascontiguousarray(self.coef, dtype=np.float64)
        d = SystemDesc()
        d.n_vars, d.n_eqs, d.n_terms = self.n_vars, self.n_eqs, self.n_terms
        d.eq_ptr = iptr(self.eq_ptr)
        d.term_ptr = iptr(self.term_ptr)
        d.var = iptr(self.var if self.var.size else np.zeros(1, np.int32))
        d.exp = iptr(self.exp if self.exp.size else np.ones(1, np.int32))
        d.coef = dptr(self.coef)
        return d

    def terms(self, i: int):
        """(support [(var, exp)], complex128 coefficient) of equation i."""
        out = []
        for t in range(self.eq_ptr[i], self.eq_ptr[i + 1]):
            sup = [(int(self.var[q]), int(self.exp[q])) for q in range(self.term_ptr[t], self.term_ptr[t + 1])]
            c = self.coef[0, :, t].sum() + 1j * self.coef[1, :, t].sum()
            out.append((sup, c))
        return out

    @staticmethod
    def _from_sysbuf(buf, prec: PrecisionMode) -> "PolynomialSystem":
        d = SystemDesc()
        inp.check(inp.lib.pt_sysbuf_desc(buf, C.byref(d)))
        T = d.n_terms
        V = d.term_ptr[T] if T > 0 else 0
        arr = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy() if n > 0 else np.zeros(0, np.int32)
        sysm = PolynomialSystem(
            n_vars=d.n_vars,
            eq_ptr=arr(d.eq_ptr, d.n_eqs + 1),
            term_ptr=arr(d.term_ptr, T + 1),
            var=arr(d.var, V),
            exp=arr(d.exp, V),
            coef=np.ctypeslib.as_array(d.coef, shape=(2 * prec.limbs * max(T, 1),)).copy()[: 2 * prec.limbs * T]
            .reshape(2, prec.limbs, T),
            prec=prec,
        )
        inp.lib.pt_sysbuf_free(buf)
        return sysm

    @staticmethod
    def from_terms(n_vars: int, equations, prec: PrecisionMode) -> "PolynomialSystem":
        """Build from [[(support, coef), ...], ...] with support [(var, exp), ...]
        (var ascending, exp >= 1) and coef a complex number or a (2, L) limb
        array.  Term order is kept as given."""
        L = prec.limbs
        eq_ptr, term_ptr, var, exp, coefs = [0], [0], [], [], []
        for eq in equations:
            for sup, c in eq:
                for v, e in sup:
                    var.append(v)
                    exp.append(e)
                term_ptr.append(len(var))
                cl = np.zeros((2, L))
                if np.ndim(c) == 0:
                    cl[0, 0], cl[1, 0] = complex(c).real, complex(c).imag
                else:
                    cl[:] = np.asarray(c, dtype=np.float64).reshape(2, L)
                coefs.append(cl)
            eq_ptr.append(len(term_ptr) - 1)
        coef = np.stack(coefs, axis=-1) if coefs else np.zeros((2, L, 0))
        return PolynomialSystem(n_vars, np.array(eq_ptr, np.int32), np.array(term_ptr, np.int32),
                                np.array(var, np.int32), np.array(exp, np.int32), coef, prec)


def _gen(fn, *args, prec: PrecisionMode) -> PolynomialSystem:
    buf = C.c_void_p()
    inp.check(fn(*args, int(prec), C.byref(buf)))
    return PolynomialSystem._from_sysbuf(buf, prec)


def cyclic_system(n: int, prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """Cyclic n-roots, Eq. (5)."""
    return _gen(inp.lib.pt_gen_cyclic, n, prec=prec)


def augment_with_linear(n_cyclic: int, dim: int, seed: int,
                        prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """cyclic-n plus `dim` random affine slices, Eq. (6)."""
    fb = C.c_void_p()
    inp.check(inp.lib.pt_gen_cyclic(n_cyclic, int(prec), C.byref(fb)))
    out = C.c_void_p()
    rc = inp.lib.pt_gen_augment(fb, dim, C.c_uint64(seed), int(prec), C.byref(out))
    inp.lib.pt_sysbuf_free(fb)
    inp.check(rc)
    return PolynomialSystem._from_sysbuf(out, prec)


def chandrasekhar(n: int, c: float = 0.51234, prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """Discretised Chandrasekhar H-equation (BASELINE config 2)."""
    return _gen(inp.lib.pt_gen_chandra, n, C.c_double(c), prec=prec)


def random_dense(n: int, degree: int, n_monomials: int, seed: int,
                 prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """n equations on one shared random support (BASELINE configs 3 and 5)."""
    return _gen(inp.lib.pt_gen_random_dense, n, degree, n_monomials, C.c_uint64(seed), prec=prec)


def total_degree_start(n: int, degree: int, prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """g_i = x_i^degree - 1."""
    return _gen(inp.lib.pt_gen_total_degree, n, degree, prec=prec)


def gamma_from_seed(seed: int, prec: PrecisionMode) -> np.ndarray:
    """Rng(seed).unit<R>() (rng.hpp:38-41) as 2L limbs."""
    out = np.zeros(2 * prec.limbs)
    inp.check(inp.lib.pt_gen_gamma(C.c_uint64(seed), int(prec), dptr(out)))
    return out


def unit_complex(theta: float, prec: PrecisionMode) -> np.ndarray:
    """unit_complex<R>(theta) (complex.hpp:141-148) as 2L limbs."""
    out = np.zeros(2 * prec.limbs)
    inp.check(inp.lib.pt_gen_unit_complex(C.c_double(theta), int(prec), dptr(out)))
    return out


@dataclass
class StepControlParams:  # SPEC.md:448-451 + NewtonParams SPEC.md:357-359
    max_step: float = 0.1
    min_step: float = 1e-6
    max_steps: int = 500
    pred_degree: int = 4
    newton_max_iter: int = 6
    newton_tol: float = 1e-20

    @staticmethod
    def defaults(prec: PrecisionMode) -> "StepControlParams":
        """SPEC defaults (pt_default_params restated; tests pin the two equal):
        tolerance RealTraits<R>::newton_tolerance (multiprec.hpp:391,404,418),
        6 iterations, dt_max 0.1, h_min 1e-6, predictor degree 4, max steps
        500 / 500 / 1500."""
        return StepControlParams(0.1, 1e-6, 1500 if prec == PrecisionMode.QD else 500, 4, 6,
                                 (1e-8, 1e-20, 1e-44)[int(prec)])

    def native(self) -> StepParams:
        return StepParams(self.max_step, self.min_step, self.max_steps, self.pred_degree,
                          self.newton_max_iter, 0, self.newton_tol)


# ---------------------------------------------------------------------------
# system and solution files
# ---------------------------------------------------------------------------
def parse_system(text: str, prec: PrecisionMode) -> PolynomialSystem:
    """parse_system: canonical form, duplicates merged in
    `prec`, zeros dropped.  Raises ValueError("line L, column C: ...")."""
    buf = C.c_void_p()
    rc = inp.lib.pt_system_parse(text.encode(), int(prec), C.byref(buf))
    if rc != 0:
        raise ValueError((inp.lib.pt_inputs_last_error() or b"").decode())
    return PolynomialSystem._from_sysbuf(buf, prec)


def serialize_system(s: PolynomialSystem) -> str:
    """serialize_system: hex-limb coefficients, so
    parse_system(serialize_system(s)) == s bit for bit (canonical s)."""
    d = s.desc()
    out = C.c_void_p()
    inp.check(inp.lib.pt_system_serialize(C.byref(d), int(s.prec), C.byref(out)))
    return inp.take_text(out)


def canonical(s: PolynomialSystem) -> PolynomialSystem:
    """The canonical form of a caller-built system."""
    d = s.desc()
    buf = C.c_void_p()
    inp.check(inp.lib.pt_sysbuf_from_desc(C.byref(d), int(s.prec), C.byref(buf)))
    return PolynomialSystem._from_sysbuf(buf, s.prec)


@dataclass
class Solution:
    point: np.ndarray   # (2, L, n) limbs
    t: float
    residual: float
    update: float


def write_solutions(solutions: List[Solution], prec: PrecisionMode) -> str:
    """Solutions file: one record per point (t, n hex-limb components,
    residual and update norm)."""
    L = prec.limbs
    n = solutions[0].point.shape[-1] if solutions else 0
    pts = np.ascontiguousarray(np.stack([s.point.reshape(2, L, n) for s in solutions]) if solutions
                               else np.zeros((0, 2, L, 0)))
    t = np.array([s.t for s in solutions], dtype=np.float64)
    r = np.array([s.residual for s in solutions], dtype=np.float64)
    u = np.array([s.update for s in solutions], dtype=np.float64)
    out = C.c_void_p()
    z = np.zeros(1)
    inp.check(inp.lib.pt_solutions_write(n, int(prec), len(solutions), dptr(t if t.size else z),
                                         dptr(pts if pts.size else z), dptr(r if r.size else z),
                                         dptr(u if u.size else z), C.byref(out)))
    return inp.take_text(out)


def read_solutions(text: str, prec: PrecisionMode) -> List[Solution]:
    cnt, n = C.c_int32(), C.c_int32()
    raw = text.encode()
    rc = inp.lib.pt_solutions_read(raw, int(prec), 0, C.byref(cnt), C.byref(n), None, None, None, None)
    if rc != 0:
        raise ValueError((inp.lib.pt_inputs_last_error() or b"").decode())
    P, N, L = cnt.value, n.value, prec.limbs
    pts = np.zeros((max(P, 1), 2, L, max(N, 1)))  # stride 2 L N when N > 0
    t, r, u = np.zeros(max(P, 1)), np.zeros(max(P, 1)), np.zeros(max(P, 1))
    rc = inp.lib.pt_solutions_read(raw, int(prec), P, C.byref(cnt), C.byref(n), dptr(t), dptr(pts), dptr(r), dptr(u))
    if rc != 0:
        raise ValueError((inp.lib.pt_inputs_last_error() or b"").decode())
    return [Solution(pts[p, :, :, :N].copy(), float(t[p]), float(r[p]), float(u[p])) for p in range(P)]


# ---------------------------------------------------------------------------
# hex limbs (hexio.hpp:16-24)
# ---------------------------------------------------------------------------
def hex_encode_limb(value: float) -> str:
    buf = C.create_string_buffer(17)
    inp.check(inp.lib.pt_hex_encode_limb(float(value), buf))
    return buf.value.decode()


def hex_decode_limb(text: str) -> float:
    out = np.zeros(1)
    raw = text.encode()
    rc = inp.lib.pt_hex_decode_limb(raw, len(raw), dptr(out))
    if rc != 0:
        raise ValueError((inp.lib.pt_inputs_last_error() or b"").decode())
    return float(out[0])


def hex_limbs(limbs) -> str:
    a = np.ascontiguousarray(np.atleast_1d(limbs), dtype=np.float64)
    out = C.c_void_p()
    inp.check(inp.lib.pt_hex_limbs(dptr(a), a.size, C.byref(out)))
    return inp.take_text(out)


def parse_hex_limbs(text: str) -> np.ndarray:
    raw = text.encode()
    cnt = C.c_int32()
    rc = inp.lib.pt_parse_hex_limbs(raw, len(raw), None, 0, C.byref(cnt))
    if rc != 0:
        raise ValueError((inp.lib.pt_inputs_last_error() or b"").decode())
    out = np.zeros(cnt.value)
    inp.check(inp.lib.pt_parse_hex_limbs(raw, len(raw), dptr(out), cnt.value, C.byref(cnt)))
    return out


# ---------------------------------------------------------------------------
# cyclic n-roots facts (Table 5)
# ---------------------------------------------------------------------------
@dataclass
class CyclicDegreeFact:
    n: int
    m: int
    l: int
    dim: int
    degree: int


def cyclic_degree(n: int) -> Optional[CyclicDegreeFact]:
    """cyclic_degree: n = l m^2 with m >= 2 maximal, l squarefree."""
    m, l, dim, deg = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    rc = inp.lib.pt_cyclic_degree(n, C.byref(m), C.byref(l), C.byref(dim), C.byref(deg))
    if rc < 0:
        inp.check(rc)
    if rc == 0:
        return None
    return CyclicDegreeFact(n, m.value, l.value, dim.value, deg.value)


def stack_systems(a: PolynomialSystem, b: PolynomialSystem) -> PolynomialSystem:
    """Equations of a followed by those of b."""
    if a.prec != b.prec or a.n_vars != b.n_vars:
        raise ValueError("systems must share precision and variables")
    ba, bb = _to_sysbuf(a), _to_sysbuf(b)
    out = C.c_void_p()
    try:
        inp.check(inp.lib.pt_sysbuf_stack(ba, bb, C.byref(out)))
    finally:
        inp.lib.pt_sysbuf_free(ba)
        inp.lib.pt_sysbuf_free(bb)
    return PolynomialSystem._from_sysbuf(out, a.prec)


def _to_sysbuf(s: PolynomialSystem) -> C.c_void_p:
    """A pt_sysbuf copy of s (canonical form)."""
    d = s.desc()
    buf = C.c_void_p()
    inp.check(inp.lib.pt_sysbuf_from_desc(C.byref(d), int(s.prec), C.byref(buf)))
    return buf
