"""Random normalized DD / QD operands for the arithmetic parity tests."""
import numpy as np

OPS = {"add": 0, "sub": 1, "mul": 2, "mul_d": 3, "div": 4, "sqrt": 5, "renorm": 6, "cmul": 7, "cadd": 8,
       "conj_mul": 9, "norm_sqr": 10, "modulus_double": 11, "powi": 12, "unit_complex": 13, "cscale": 14,
       "cpowi": 15}


def random_operands(prec: int, count: int, seed: int, positive=False, small_int=False, oracle=None):
    """(count, 2, L) limbs: leading limb with spread exponents, lower limbs
    scaled below ulp/2 and renormalised through `oracle` when given."""
    L = (1, 2, 4)[prec]
    rng = np.random.default_rng(seed)
    out = np.zeros((count, 2, L))
    for c in range(2):
        hi = rng.uniform(-1, 1, count) * np.exp2(rng.integers(-30, 30, count))
        if positive:
            hi = np.abs(hi)
        out[:, c, 0] = hi
        scale = np.abs(hi)
        for l in range(1, L):
            scale = scale * 2.0 ** -53
            out[:, c, l] = rng.uniform(-1, 1, count) * scale
    # sprinkle exact zeros, ones, ties and cancellations
    k = count // 16
    out[:k, :, 1:] = 0.0
    out[k:2 * k, 0, 0] = 1.0
    out[2 * k:3 * k, :, :] = 0.0
    if small_int:
        out[:, 0, 0] = rng.integers(0, 6, count)
        out[:, 0, 1:] = 0
    if oracle is not None and L > 1:
        for c in range(2):
            flat = np.zeros((count, 2, L))
            flat[:, 0] = out[:, c]
            r = oracle.arith(prec, OPS["renorm"], flat, flat)
            out[:, c] = r[:, 0]
    return out
