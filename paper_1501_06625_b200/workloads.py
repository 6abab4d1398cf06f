"""The BASELINE.json configurations as ready-to-track homotopies.

  C1 cyclic-16 monodromy leg, DD, Backelin witness start   (configs[0])
  C2 Chandrasekhar H n=64, D/DD/QD, start x = 1            (configs[1])
  C3 random dense n=96 degree 4, M monomials, DD/QD        (configs[2])
  C4 cyclic-256 monodromy leg, QD                          (configs[3])
  C5 batch of random dense n=32 (M=512) paths, DD          (configs[4])

Definitions follow SURVEY.md 8(d) / Appendix C; seeds are pinned here so
every test and bench line tracks the same path.  Inputs the reference does not
ship (Backelin witness points) are generated in closed form:
x_{a m + b} = omega^a r_b with omega = e^{2 pi i/m}, prod r_b = 1, and r
chosen on the slice L (root #0 of a degree-m polynomial, roots ordered by
(real, imag)); the tracker's t=0 Newton pass polishes it to working precision.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .systems import (
    PolynomialSystem,
    PrecisionMode,
    StepControlParams,
    augment_with_linear,
    chandrasekhar,
    gamma_from_seed,
    limbs_from_complex,
    random_dense,
    total_degree_start,
    unit_complex,
)


@dataclass
class Workload:
    name: str
    prec: PrecisionMode
    g: PolynomialSystem
    f: PolynomialSystem
    gamma: np.ndarray
    k: int
    starts: np.ndarray  # (P, 2, L, n)
    params: StepControlParams

    @property
    def start(self) -> np.ndarray:
        return self.starts[0]

    @property
    def n(self) -> int:
        return self.g.n_vars

    @property
    def N(self) -> int:
        return self.g.n_eqs


def backelin_witness(aug: PolynomialSystem, m: int, dim: int) -> np.ndarray:
    """Point on the Backelin component of cyclic-(m^2) lying on the affine
    slices stored as the last `dim` equations of `aug` (complex128)."""
    n = m * m
    N = aug.n_eqs
    omega = np.exp(2j * np.pi * np.arange(m) / m)
    M = np.zeros((dim, m), dtype=np.complex128)
    rhs = np.zeros(dim, dtype=np.complex128)
    for row in range(dim):
        terms = aug.terms(N - dim + row)
        c = np.zeros(n + 1, dtype=np.complex128)
        for sup, coef in terms:
            c[0 if not sup else sup[0][0] + 1] += coef
        rhs[row] = -c[0]
        for b in range(m):
            M[row, b] = sum(c[a * m + b + 1] * omega[a] for a in range(m))
    r0 = np.linalg.lstsq(M, rhs, rcond=None)[0]
    v = np.linalg.svd(M)[2].conj()[-1]
    poly = np.array([1.0 + 0j])
    for b in range(m):
        poly = np.polymul(poly, np.array([v[b], r0[b]]))
    poly = poly.copy()
    poly[-1] -= 1.0
    roots = np.roots(poly)
    roots = sorted(roots, key=lambda z: (round(z.real, 12), round(z.imag, 12)))
    r = r0 + roots[0] * v
    x = np.zeros(n, dtype=np.complex128)
    for a in range(m):
        for b in range(m):
            x[a * m + b] = omega[a] * r[b]
    return x


def backelin_component_key(m: int):
    """Invariant of a Backelin component of cyclic-(m^2): on the family
    x_{a m + b} = omega^a r_b the product r_0 ... r_{m-1} = x_0 ... x_{m-1} is
    an m-th root of unity fixed along the component (prod x = (prod r)^m = 1
    splits the family into m components {prod r = zeta}); a monodromy endpoint
    with a different value has jumped to another component."""

    def key(point: np.ndarray) -> complex:
        z = point[0].sum(axis=0)[:m] + 1j * point[1].sum(axis=0)[:m]
        return complex(np.prod(z))

    return key


def cyclic4_witness(slice_row: np.ndarray, family: int = 1) -> list:
    """cyclic4_witness: family 1 (a, 1/a, -a, -1/a) or
    family 2 (a, -1/a, -a, 1/a) substituted into the affine slice
    c_0 + c_1 x_0 + ... + c_4 x_3 = 0 gives (c_1 - c_3 s) a^2 + c_0 a +
    (c_2 s - c_4) ... written out below; both roots are returned (complex128
    points satisfying cyclic-4 and the slice to working precision before the
    tracker's t = 0 Newton polish).  Raises ValueError on a degenerate quadratic."""
    c0, c1, c2, c3, c4 = [complex(v) for v in slice_row]
    s = 1.0 if family == 1 else -1.0
    # x = (a, s/a, -a, -s/a):  c0 + c1 a + c2 s/a - c3 a - c4 s/a = 0
    #   -> (c1 - c3) a^2 + c0 a + s (c2 - c4) = 0
    qa, qb, qc = c1 - c3, c0, s * (c2 - c4)
    if abs(qa) < 1e-14 and abs(qc) < 1e-14:
        raise ValueError("degenerate slice for the cyclic-4 witness: resample L")
    roots = np.roots([qa, qb, qc]) if abs(qa) >= 1e-14 else np.array([-qc / qb])
    # a = 0 is not a point of the family (x_1 = s/a): it appears only when the slice has c2 = c4
    return [np.array([a, s / a, -a, -s / a], dtype=np.complex128) for a in roots if abs(a) > 1e-14]


def slice_rows(aug: PolynomialSystem, dim: int) -> np.ndarray:
    """The last `dim` affine equations of `aug` as rows (c_0, c_1, ..., c_n)."""
    n, N = aug.n_vars, aug.n_eqs
    out = np.zeros((dim, n + 1), dtype=np.complex128)
    for r in range(dim):
        for sup, coef in aug.terms(N - dim + r):
            out[r, 0 if not sup else sup[0][0] + 1] += coef
    return out


def cyclic_leg(m: int, prec: PrecisionMode, seed_l: int = 1, seed_k: int = 2, seed_gamma: int = 3) -> Workload:
    """Monodromy leg h = alpha (1-t) (f, L) + t (f, K), k = 1."""
    n = m * m
    dim = m - 1
    g = augment_with_linear(n, dim, seed_l, prec)
    f = augment_with_linear(n, dim, seed_k, prec)
    x0 = backelin_witness(g, m, dim)
    params = StepControlParams.defaults(prec)
    return Workload(f"cyclic{n}-{prec.name.lower()}", prec, g, f, gamma_from_seed(seed_gamma, prec), 1,
                    limbs_from_complex(x0, prec)[None], params)


def chandra(n: int = 64, prec: PrecisionMode = PrecisionMode.DD, c: float = 0.51234,
            seed_gamma: int = 1) -> Workload:
    g = total_degree_start(n, 2, prec)
    f = chandrasekhar(n, c, prec)
    start = limbs_from_complex(np.ones(n), prec)
    return Workload(f"chandra{n}-{prec.name.lower()}", prec, g, f, gamma_from_seed(seed_gamma, prec), 2,
                    start[None], StepControlParams.defaults(prec))


def random_system(n: int = 96, degree: int = 4, n_monomials: int = 65536, prec: PrecisionMode = PrecisionMode.DD,
                  seed: int = 7, seed_gamma: int = 11, n_paths: int = 1) -> Workload:
    g = total_degree_start(n, degree, prec)
    f = random_dense(n, degree, n_monomials, seed, prec)
    starts = total_degree_starts(n, degree, n_paths, prec)
    return Workload(f"rand{n}-d{degree}-m{n_monomials}-{prec.name.lower()}", prec, g, f,
                    gamma_from_seed(seed_gamma, prec), 2, starts, StepControlParams.defaults(prec))


def total_degree_starts(n: int, degree: int, n_paths: int, prec: PrecisionMode) -> np.ndarray:
    """Start points of g_i = x_i^d - 1: path p picks the degree-th root of
    unity number (p // d^i) % d on coordinate i (base-d digits of p); the
    roots are unit_complex<R>(2 pi j / d) so |x_i| = 1 in working precision."""
    L = prec.limbs
    roots = np.stack([unit_complex(2.0 * np.pi * j / degree, prec).reshape(2, L) for j in range(degree)])
    if degree >= 1:
        roots[0] = 0.0
        roots[0, 0, 0] = 1.0  # the root 1 exactly
    out = np.zeros((n_paths, 2, L, n))
    for p in range(n_paths):
        q = p
        for i in range(n):
            out[p, :, :, i] = roots[q % degree]
            q //= degree
    return out


def batch(n: int = 32, n_monomials: int = 512, n_paths: int = 8192, prec: PrecisionMode = PrecisionMode.DD,
          seed: int = 5, seed_gamma: int = 9) -> Workload:
    w = random_system(n, 4, n_monomials, prec, seed, seed_gamma, n_paths)
    w.name = f"batch{n_paths}-rand{n}-m{n_monomials}-{prec.name.lower()}"
    return w


def by_name(name: str, prec: Optional[PrecisionMode] = None) -> Workload:
    p = prec if prec is not None else PrecisionMode.DD
    if name == "cyclic16":
        return cyclic_leg(4, p)
    if name == "cyclic256":
        return cyclic_leg(16, prec if prec is not None else PrecisionMode.QD)
    if name == "chandra64":
        return chandra(64, p)
    if name == "rand96":
        return random_system(96, 4, 65536, p)
    if name == "batch32":
        return batch(prec=p)
    raise KeyError(name)
