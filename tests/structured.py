"""Randomly STRUCTURED square systems for the tracker parity tests
(tests/test_gpu_random.py on the device, tests/test_oracle_tracker.py for the
oracle against the reference-header build): ragged equations, exponents 1-4,
constant terms, monomials shared between equations, variables absent from
whole equations, DD / QD coefficients with every limb populated."""
import numpy as np

import paper_1501_06625_b200 as pt
from paper_1501_06625_b200 import PolynomialSystem, PrecisionMode as PM
from paper_1501_06625_b200 import workloads as W


def full_limbs(z, prec, rng):
    """A complex coefficient with all L limbs populated and canonical
    (|c_{i+1}| < 2^-54 |c_i| < ulp(c_i) / 2)."""
    L = prec.limbs
    cl = np.zeros((2, L))
    cl[0, 0], cl[1, 0] = z.real, z.imag
    for i in range(1, L):
        cl[:, i] = cl[:, i - 1] * 2.0 ** -54 * rng.uniform(-1, 1, 2)
    return cl


def random_structured(n, prec, seed):
    rng = np.random.default_rng(seed)
    pool = []  # monomials shared between equations
    for _ in range(max(2, n)):
        k = int(rng.integers(1, min(n, 4) + 1))
        vs = sorted(rng.choice(n, size=k, replace=False).tolist())
        pool.append([(v, int(rng.integers(1, 5))) for v in vs])
    eqs = []
    for i in range(n):
        terms = []
        absent = int(rng.integers(0, n)) if n > 2 and rng.uniform() < 0.5 else -1
        for _ in range(int(rng.integers(1, 15))):
            if rng.uniform() < 0.4:
                sup = pool[int(rng.integers(0, len(pool)))]
            else:
                k = int(rng.integers(1, min(n, 5) + 1))
                vs = sorted(rng.choice(n, size=k, replace=False).tolist())
                sup = [(v, int(rng.integers(1, 5))) for v in vs]
            if any(v == absent for v, _ in sup):
                continue
            terms.append((sup, full_limbs(complex(*rng.uniform(-1, 1, 2)), prec, rng)))
        terms.append(([(i, 1)], full_limbs(complex(*rng.uniform(0.5, 1, 2)), prec, rng)))  # x_i itself
        if rng.uniform() < 0.7:
            terms.append(([], full_limbs(complex(*rng.uniform(-1, 1, 2)), prec, rng)))  # constant term
        eqs.append(terms)
    return PolynomialSystem.from_terms(n, eqs, prec)


def case(n, prec, seed, max_steps):
    f = random_structured(n, prec, seed)
    deg = 3
    g = pt.total_degree_start(n, deg, prec)
    gamma = pt.gamma_from_seed(seed + 1000, prec)
    params = pt.StepControlParams.defaults(prec)
    params.max_steps = max_steps
    starts = W.total_degree_starts(n, deg, 6, prec)
    return f, g, gamma, params, starts


CASES = [(1, PM.D, 1), (2, PM.DD, 2), (3, PM.QD, 3), (5, PM.D, 4), (6, PM.DD, 5), (7, PM.DD, 6),
         (9, PM.QD, 7), (12, PM.D, 8), (13, PM.DD, 9), (17, PM.DD, 10), (20, PM.D, 11), (24, PM.DD, 12)]


def max_steps(prec):
    return 40 if prec == PM.QD else 120
