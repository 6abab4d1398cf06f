"""CPU: the host-only inputs library (libpt_inputs.so) -- hex limbs pinned
against the reference's hexio.cpp, system files (parse_system /
serialize_system), solution files and
cyclic_degree (Table 5, acceptance criterion 1)."""
import numpy as np
import pytest

import paper_1501_06625_b200 as pt
from paper_1501_06625_b200 import PrecisionMode as PM
from conftest import assert_bits_equal

PRECS = [PM.D, PM.DD, PM.QD]


# ---------------------------------------------------------------------------
# hex limbs (hexio.hpp:16-24)
# ---------------------------------------------------------------------------
def _edge_doubles(rng, count):
    v = rng.uniform(-1, 1, count) * np.exp2(rng.integers(-1074, 1023, count).astype(float))
    extra = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 1.7976931348623157e308, 1.0, -2.5])
    return np.concatenate([v, extra])


def test_hex_limb_round_trip_bit_exact():
    rng = np.random.default_rng(1)
    vals = _edge_doubles(rng, 2000)
    for v in vals:
        s = pt.hex_encode_limb(v)
        assert len(s) == 16 and s == s.lower()
        assert np.float64(pt.hex_decode_limb(s)).view(np.uint64) == np.float64(v).view(np.uint64)
    assert pt.hex_encode_limb(1.0) == "3ff0000000000000"  # hexio.hpp:13 example
    assert pt.hex_limbs([2.0, 0.0]) == "#(4000000000000000 0000000000000000)"
    assert pt.hex_decode_limb("3FF0000000000000") == 1.0  # either case


@pytest.mark.parametrize("bad", ["3ff", "3ff00000000000000", "3ff000000000000g"])
def test_hex_decode_rejects(bad):
    with pytest.raises(ValueError):
        pt.hex_decode_limb(bad)


@pytest.mark.parametrize("bad", ["", "#()", "(3ff0000000000000)", "#(3ff0000000000000", "#(3ff00000000)",
                                 "#(3ff000000000000x)", "#(   )"])
def test_parse_hex_limbs_rejects(bad):
    with pytest.raises(ValueError):
        pt.parse_hex_limbs(bad)


def test_hex_matches_reference_hexio(ref_oracle):
    """Pinned against the UNMODIFIED reference hexio.cpp (oracle/_ref)."""
    rng = np.random.default_rng(2)
    vals = _edge_doubles(rng, 500)
    for k in (1, 2, 4):
        for i in range(0, vals.size - k, 7):
            limbs = vals[i:i + k]
            s = pt.hex_limbs(limbs)
            assert s == ref_oracle.ref_hex_limbs(limbs)
            assert_bits_equal(pt.parse_hex_limbs(s), ref_oracle.ref_parse_hex_limbs(s), "parse")
    for text in ["#(3ff0000000000000  4000000000000000)", "#( 3ff0000000000000)", "#(3FF0000000000000)",
                 "#()", "#(3ff00000000)", "#(zz00000000000000)", "#(3ff0000000000000"]:
        ours = None
        try:
            ours = pt.parse_hex_limbs(text)
        except ValueError:
            pass
        ref = ref_oracle.ref_parse_hex_limbs(text)
        assert (ours is None) == (ref is None), text
        if ref is not None:
            assert_bits_equal(ours, ref, text)


# ---------------------------------------------------------------------------
# system files
# ---------------------------------------------------------------------------
def test_parse_spec_examples():
    s = pt.parse_system("vars: x0 x1\nx0 + x1;\n", PM.D)
    assert s.n_eqs == 1 and s.terms(0) == [([(0, 1)], 1 + 0j), ([(1, 1)], 1 + 0j)]
    s = pt.parse_system("vars: x0 x1\nx0*x1 + x1*x0;\n", PM.DD)  # merge rule
    assert s.terms(0) == [([(0, 1), (1, 1)], 2 + 0j)]
    cyc3 = "vars: x0 x1 x2\nx0 + x1 + x2;\nx0*x1 + x1*x2 + x2*x0;\nx0*x1*x2 - 1;\n"
    s = pt.parse_system(cyc3, PM.D)
    assert [len(s.terms(i)) for i in range(3)] == [3, 3, 2]  # Eq. (5) at n = 3
    ref = pt.cyclic_system(3, PM.D)
    assert [s.terms(i) for i in range(3)] == [ref.terms(i) for i in range(3)]  # same values (the text's
    # "- 1" is the complex negation of 1, whose imaginary part is -0: equal, not bit-equal, to the generator's)


@pytest.mark.parametrize("prec", PRECS, ids=lambda p: p.name)
def test_cyclic_round_trip(prec):
    c = pt.cyclic_system(4, prec)
    back = pt.parse_system(pt.serialize_system(c), prec)
    for name in ("eq_ptr", "term_ptr", "var", "exp"):
        assert np.array_equal(getattr(back, name), getattr(c, name)), name
    assert_bits_equal(back.coef, c.coef, "coef")


@pytest.mark.parametrize("prec", PRECS, ids=lambda p: p.name)
def test_random_system_round_trip_bit_exact(prec):
    """Multi-limb coefficients (random DD / QD values, exponents > 1) survive
    serialize -> parse bit for bit, and parse is idempotent."""
    rng = np.random.default_rng(int(prec) + 10)
    L = prec.limbs
    eqs = []
    for _ in range(5):
        eq = []
        for _ in range(7):
            k = int(rng.integers(0, 4))
            vs = sorted(rng.choice(6, size=k, replace=False).tolist())
            sup = [(v, int(rng.integers(1, 4))) for v in vs]
            c = np.zeros((2, L))
            c[:, 0] = rng.uniform(-1, 1, 2)
            for l in range(1, L):
                c[:, l] = c[:, 0] * 2.0 ** (-53 * l) * rng.uniform(-0.5, 0.5, 2)
            eq.append((sup, c))
        eqs.append(eq)
    s = pt.canonical(pt.PolynomialSystem.from_terms(6, eqs, prec))
    text = pt.serialize_system(s)
    back = pt.parse_system(text, prec)
    assert_bits_equal(back.coef, s.coef, "coef")
    assert np.array_equal(back.var, s.var) and np.array_equal(back.exp, s.exp)
    assert pt.serialize_system(back) == text


def test_decimal_coefficients_in_working_precision():
    s = pt.parse_system("vars: x\n0.1*x + (1.5 - 2.25*i);\n", PM.DD)
    c = s.coef
    # the DD value of 0.1 is accurate to ~1e-32 (not just the binary64 0.1)
    from fractions import Fraction
    got = Fraction(float(c[0, 0, 1])) + Fraction(float(c[0, 1, 1]))
    assert abs(got - Fraction(1, 10)) < Fraction(1, 10 ** 31)
    assert complex(c[0, 0, 0], c[1, 0, 0]) == 1.5 - 2.25j
    d = pt.parse_system("vars: x\n0.1*x;\n", PM.D)
    assert d.coef[0, 0, 0] == 0.1


@pytest.mark.parametrize("text,where", [
    ("x0 + x1;", "vars"),                              # no header
    ("vars: x0 x1\n;\n", "empty polynomial"),          # empty-term polynomial
    ("vars: x0 x1\nx0 + x2;\n", "out of range"),       # variable index out of range
    ("vars: x0 x1\n", "empty polynomial list"),
    ("vars: x0 x1\nx0 + * x1;\n", "line 2, column"),   # syntax error with position
    ("vars: x0 x1\nx0 + x1\n", "missing ';'"),
    ("vars: x0 x0\nx0;\n", "duplicate"),
    ("vars: x0\nx0^0;\n", "exponent"),
])
def test_parse_errors(text, where):
    with pytest.raises(ValueError) as e:
        pt.parse_system(text, PM.DD)
    assert where in str(e.value)


def test_empty_term_polynomial_rejected_on_reparse():
    s = pt.parse_system("vars: x0\nx0 - x0;\nx0;\n", PM.D)  # first equation cancels to zero
    assert s.terms(0) == []
    text = pt.serialize_system(s)
    assert pt.parse_system(text, PM.D).terms(0) == []  # "0" is the zero polynomial, not an empty one
    with pytest.raises(ValueError):
        pt.parse_system(text.replace("0;", ";", 1), PM.D)


# ---------------------------------------------------------------------------
# solution files
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("prec", PRECS, ids=lambda p: p.name)
def test_solutions_round_trip(prec):
    rng = np.random.default_rng(5)
    L = prec.limbs
    sols = []
    for r in range(4):
        x = np.zeros((2, L, 6))
        x[:, 0] = rng.uniform(-2, 2, (2, 6))
        for l in range(1, L):
            x[:, l] = x[:, 0] * 2.0 ** (-53 * l) * rng.uniform(-0.5, 0.5, (2, 6))
        sols.append(pt.Solution(x, float(rng.uniform()), float(rng.uniform() * 1e-20), float(rng.uniform())))
    text = pt.write_solutions(sols, prec)
    back = pt.read_solutions(text, prec)
    assert len(back) == 4
    for a, b in zip(sols, back):
        assert_bits_equal(b.point, a.point, "point")
        assert_bits_equal(np.array([b.t, b.residual, b.update]), np.array([a.t, a.residual, a.update]), "diag")
    assert pt.read_solutions(pt.write_solutions([], prec), prec) == []


@pytest.mark.parametrize("bad", ["", "solutions 1 dim 1 precision dd\n",
                                 "solutions 1 dim 1 precision dd\nsolution 0 t #(0) residual #(0) update #(0)\n",
                                 "solutions 1 dim 1 precision d\nsolution 0 t #(3ff0000000000000) residual "
                                 "#(0000000000000000) update #(0000000000000000)\nx0 #(3ff0000000000000)\n"])
def test_solutions_errors(bad):
    with pytest.raises(ValueError):
        pt.read_solutions(bad, PM.DD)


# ---------------------------------------------------------------------------
# cyclic_degree (acceptance criterion 1: all 20 pairs of Table 5)
# ---------------------------------------------------------------------------
# PAPER.md:803-806 (Table 5), verbatim
TABLE5 = {16: 4, 32: 4, 48: 4, 64: 8, 80: 4, 96: 4, 128: 8, 144: 12, 160: 4, 176: 4, 192: 8, 208: 4, 240: 4,
          256: 16, 272: 4, 288: 12, 304: 4, 320: 8, 336: 4, 352: 4}


def test_cyclic_degree_table5():
    import time
    t0 = time.perf_counter()
    for n, d in TABLE5.items():
        f = pt.cyclic_degree(n)
        assert f is not None and f.degree == d and f.dim == f.m - 1 and f.l * f.m ** 2 == n, (n, f)
    assert time.perf_counter() - t0 < 1.0
    assert pt.cyclic_degree(15) is None and pt.cyclic_degree(7) is None
