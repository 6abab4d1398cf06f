// orc_arith.hpp -- TEST INFRASTRUCTURE (CPU oracle), not product code.
//
// Plain-C++ restatement of the reference scalar layer, used by the oracle
// tracker when it is built without /root/reference (e.g. on the GPU box).
// Public names match the reference API so oracle code compiles unchanged
// against either this file or the unmodified reference headers
// (oracle/Makefile, target _ref/).  Each routine cites the reference line it
// restates; tests/test_oracle_arith.py pins this file bit-for-bit against the
// reference build.
//
// Must be compiled with -ffp-contract=off (FMA contraction changes bits,
// SURVEY.md finding 0.4).
#pragma once

#include <array>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

static_assert(FLT_EVAL_METHOD == 0, "oracle needs strict binary64 evaluation");

namespace orc {

// ---- error-free building blocks (multiprec.hpp:39-83) ----------------------
// sum and exact rounding error of a+b (Knuth), multiprec.hpp:39-44
inline double sum_err(double a, double b, double& err) {
  const double s = a + b;
  const double b_virtual = s - a;
  const double a_virtual = s - b_virtual;
  err = (a - a_virtual) + (b - b_virtual);
  return s;
}
// Dekker's variant for |a| >= |b|, multiprec.hpp:47-51
inline double sum_err_ordered(double a, double b, double& err) {
  const double s = a + b;
  err = b - (s - a);
  return s;
}
// product and exact rounding error, multiprec.hpp:71-75 (the FMA form; the
// split form of :61-68 yields the same exact error term)
inline double prod_err(double a, double b, double& err) {
  const double p = a * b;
  err = std::fma(a, b, -p);
  return p;
}

// ---- double-double (multiprec.hpp:91-189) ----------------------------------
struct DoubleDouble {
  double hi = 0.0;
  double lo = 0.0;
  constexpr DoubleDouble() = default;
  constexpr DoubleDouble(double h) : hi(h) {}
  constexpr DoubleDouble(double h, double l) : hi(h), lo(l) {}
};

namespace detail {
// renormalise (h, l); non-finite leading limb wins, multiprec.hpp:102-107
inline DoubleDouble dd_fix(double h, double l) {
  if (!std::isfinite(h)) return DoubleDouble(h, 0.0);
  double e;
  const double s = sum_err_ordered(h, l, e);
  return DoubleDouble(s, e);
}
}  // namespace detail

inline DoubleDouble operator-(DoubleDouble a) { return DoubleDouble(-a.hi, -a.lo); }

// multiprec.hpp:115-123 (accurate sum: both limb pairs through two_sum)
inline DoubleDouble operator+(DoubleDouble a, DoubleDouble b) {
  double err_hi, err_lo;
  double top = sum_err(a.hi, b.hi, err_hi);
  const double low = sum_err(a.lo, b.lo, err_lo);
  err_hi += low;
  top = sum_err_ordered(top, err_hi, err_hi);
  err_hi += err_lo;
  return detail::dd_fix(top, err_hi);
}
inline DoubleDouble operator-(DoubleDouble a, DoubleDouble b) { return a + (-b); }

// multiprec.hpp:127-132
inline DoubleDouble operator*(DoubleDouble a, DoubleDouble b) {
  double err;
  const double p = prod_err(a.hi, b.hi, err);
  const double cross = (a.hi * b.lo + a.lo * b.hi) + a.lo * b.lo;
  err += cross;
  return detail::dd_fix(p, err);
}
// multiprec.hpp:134-141
inline DoubleDouble operator*(DoubleDouble a, double b) {
  double err;
  const double p = prod_err(a.hi, b, err);
  err += a.lo * b;
  return detail::dd_fix(p, err);
}
inline DoubleDouble operator*(double a, DoubleDouble b) { return b * a; }

// three binary64 quotient estimates with full-precision residuals,
// multiprec.hpp:145-155
inline DoubleDouble operator/(DoubleDouble a, DoubleDouble b) {
  const double q1 = a.hi / b.hi;
  if (!std::isfinite(q1)) return DoubleDouble(q1, 0.0);
  DoubleDouble rem = a - b * q1;
  const double q2 = rem.hi / b.hi;
  rem = rem - b * q2;
  const double q3 = rem.hi / b.hi;
  double e;
  const double s = sum_err_ordered(q1, q2, e);
  return DoubleDouble(s, e) + DoubleDouble(q3);
}
inline DoubleDouble& operator+=(DoubleDouble& a, DoubleDouble b) { return a = a + b; }
inline DoubleDouble& operator-=(DoubleDouble& a, DoubleDouble b) { return a = a - b; }
inline DoubleDouble& operator*=(DoubleDouble& a, DoubleDouble b) { return a = a * b; }
inline bool operator==(DoubleDouble a, DoubleDouble b) { return a.hi == b.hi && a.lo == b.lo; }
inline double to_double(DoubleDouble a) { return a.hi; }
inline bool is_finite(DoubleDouble a) { return std::isfinite(a.hi); }
inline DoubleDouble renormalize(DoubleDouble a) { return detail::dd_fix(a.hi, a.lo); }

// Newton refinement of the binary64 reciprocal root, multiprec.hpp:176-189
inline DoubleDouble sqrt(DoubleDouble a) {
  if (a.hi == 0.0 && a.lo == 0.0) return DoubleDouble(0.0, 0.0);
  if (a.hi < 0.0) throw std::domain_error("sqrt of negative double-double");
  const double inv_root = 1.0 / std::sqrt(a.hi);
  const double half_inv = 0.5 * inv_root;
  DoubleDouble root(a.hi * inv_root);
  for (int round = 0; round < 2; ++round) {
    const DoubleDouble resid = a - root * root;
    root += DoubleDouble(resid.hi * half_inv);
  }
  return root;
}

// ---- quad-double (multiprec.hpp:196-372) -----------------------------------
struct QuadDouble {
  std::array<double, 4> c{0.0, 0.0, 0.0, 0.0};
  constexpr QuadDouble() = default;
  constexpr QuadDouble(double x) : c{x, 0.0, 0.0, 0.0} {}
  constexpr QuadDouble(double a, double b, double d, double e) : c{a, b, d, e} {}
};

namespace detail {

// five-limb to four-limb compression with the zero-tests of
// multiprec.hpp:209-250.  Written as a small state machine over the output
// position instead of the reference's nested ifs; the sequence of two_sum
// calls it performs is the same.
inline QuadDouble qd_pack5(double c0, double c1, double c2, double c3, double c4) {
  if (!std::isfinite(c0)) return QuadDouble(c0, 0.0, 0.0, 0.0);
  // bottom-up compression
  double carry = sum_err(c3, c4, c4);
  carry = sum_err(c2, carry, c3);
  carry = sum_err(c1, carry, c2);
  c0 = sum_err(c0, carry, c1);
  // top-down sweep: 'out[pos]' is the limb being filled; a zero error term
  // means the limb absorbed the addend completely and the slot is reused.
  double out[4] = {c0, c1, 0.0, 0.0};
  const double rest[3] = {c2, c3, c4};
  int pos = (out[1] != 0.0) ? 1 : 0;
  for (int r = 0; r < 3; ++r) {
    if (pos == 3) {  // all four limbs busy: fold the remaining addend
      out[3] += rest[r];
      break;
    }
    double e;
    out[pos] = sum_err(out[pos], rest[r], e);
    out[pos + 1] = e;
    if (e != 0.0) ++pos;
  }
  return QuadDouble(out[0], out[1], out[2], out[3]);
}

// multiprec.hpp:256-279: order addends by decreasing magnitude (stable),
// two compensation sweeps, fold the tail, compress.
template <std::size_t Cap>
inline QuadDouble qd_collapse(std::array<double, Cap>& v, int k) {
  for (int i = 1; i < k; ++i) {  // stable insertion by |.|
    const double x = v[i];
    int j = i;
    while (j > 0 && std::fabs(v[j - 1]) < std::fabs(x)) {
      v[j] = v[j - 1];
      --j;
    }
    v[j] = x;
  }
  if (!std::isfinite(v[0])) return QuadDouble(v[0], 0.0, 0.0, 0.0);
  for (int sweep = 0; sweep < 2; ++sweep)
    for (int i = k - 1; i > 0; --i) v[i - 1] = sum_err(v[i - 1], v[i], v[i]);
  double tail = 0.0;
  for (int i = k - 1; i >= 4; --i) tail += v[i];
  return qd_pack5(k > 0 ? v[0] : 0.0, k > 1 ? v[1] : 0.0, k > 2 ? v[2] : 0.0, k > 3 ? v[3] : 0.0,
                  tail);
}

}  // namespace detail

inline QuadDouble operator-(const QuadDouble& a) {
  return QuadDouble(-a.c[0], -a.c[1], -a.c[2], -a.c[3]);
}
// multiprec.hpp:290-293
inline QuadDouble operator+(const QuadDouble& a, const QuadDouble& b) {
  std::array<double, 8> v{a.c[0], a.c[1], a.c[2], a.c[3], b.c[0], b.c[1], b.c[2], b.c[3]};
  return detail::qd_collapse(v, 8);
}
inline QuadDouble operator-(const QuadDouble& a, const QuadDouble& b) { return a + (-b); }
// multiprec.hpp:297-312: exact pair products down to order 3, three plain
// products of order 4, in the reference's (i outer, j inner) order.
inline QuadDouble operator*(const QuadDouble& a, const QuadDouble& b) {
  std::array<double, 23> v;
  int n = 0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; i + j < 4; ++j) {
      double e;
      v[n++] = prod_err(a.c[i], b.c[j], e);
      v[n++] = e;
    }
  v[n++] = a.c[1] * b.c[3];
  v[n++] = a.c[2] * b.c[2];
  v[n++] = a.c[3] * b.c[1];
  return detail::qd_collapse(v, n);
}
// multiprec.hpp:314-323
inline QuadDouble operator*(const QuadDouble& a, double b) {
  std::array<double, 8> v;
  for (int i = 0; i < 4; ++i) v[2 * i] = prod_err(a.c[i], b, v[2 * i + 1]);
  return detail::qd_collapse(v, 8);
}
inline QuadDouble operator*(double a, const QuadDouble& b) { return b * a; }
// five quotient digits, multiprec.hpp:327-337
inline QuadDouble operator/(const QuadDouble& a, const QuadDouble& b) {
  const double first = a.c[0] / b.c[0];
  if (!std::isfinite(first)) return QuadDouble(first, 0.0, 0.0, 0.0);
  std::array<double, 5> digits;
  QuadDouble rem = a;
  for (int i = 0; i < 5; ++i) {
    digits[i] = rem.c[0] / b.c[0];
    rem = rem - b * digits[i];
  }
  return detail::qd_collapse(digits, 5);
}
inline QuadDouble& operator+=(QuadDouble& a, const QuadDouble& b) { return a = a + b; }
inline QuadDouble& operator-=(QuadDouble& a, const QuadDouble& b) { return a = a - b; }
inline QuadDouble& operator*=(QuadDouble& a, const QuadDouble& b) { return a = a * b; }
inline bool operator==(const QuadDouble& a, const QuadDouble& b) { return a.c == b.c; }
inline double to_double(const QuadDouble& a) { return a.c[0]; }
inline bool is_finite(const QuadDouble& a) { return std::isfinite(a.c[0]); }
inline QuadDouble renormalize(const QuadDouble& a) {
  std::array<double, 4> v{a.c[0], a.c[1], a.c[2], a.c[3]};
  return detail::qd_collapse(v, 4);
}
// reciprocal-root iteration then one multiply, multiprec.hpp:364-372
inline QuadDouble sqrt(const QuadDouble& a) {
  if (a.c[0] == 0.0 && a.c[1] == 0.0 && a.c[2] == 0.0 && a.c[3] == 0.0) return QuadDouble();
  if (a.c[0] < 0.0) throw std::domain_error("sqrt of negative quad-double");
  QuadDouble y(1.0 / std::sqrt(a.c[0]));
  const QuadDouble one(1.0);
  for (int it = 0; it < 3; ++it) y = y + y * ((one - a * (y * y)) * 0.5);
  return a * y;
}

inline double to_double(double a) { return a; }
inline bool is_finite(double a) { return std::isfinite(a); }
inline double renormalize(double a) { return a; }

// ---- traits (multiprec.hpp:383-429) ----------------------------------------
template <class Real>
struct RealTraits;
template <>
struct RealTraits<double> {
  static constexpr int limbs = 1;
  static constexpr double epsilon = 0x1p-52;
  static constexpr double newton_tolerance = 1e-8;
  static std::array<double, 1> components(double a) { return {a}; }
  static double from_components(const double* l, int n) { return n > 0 ? l[0] : 0.0; }
};
template <>
struct RealTraits<DoubleDouble> {
  static constexpr int limbs = 2;
  static constexpr double epsilon = 0x1p-104;
  static constexpr double newton_tolerance = 1e-20;
  static std::array<double, 2> components(DoubleDouble a) { return {a.hi, a.lo}; }
  static DoubleDouble from_components(const double* l, int n) {
    DoubleDouble r;
    for (int i = 0; i < n && i < 2; ++i) r += DoubleDouble(l[i]);
    return r;
  }
};
template <>
struct RealTraits<QuadDouble> {
  static constexpr int limbs = 4;
  static constexpr double epsilon = 0x1p-209;
  static constexpr double newton_tolerance = 1e-44;
  static std::array<double, 4> components(const QuadDouble& a) {
    return {a.c[0], a.c[1], a.c[2], a.c[3]};
  }
  static QuadDouble from_components(const double* l, int n) {
    std::array<double, 4> v{0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < n && i < 4; ++i) v[i] = l[i];
    return detail::qd_collapse(v, n < 4 ? n : 4);
  }
};

// square-and-multiply, multiprec.hpp:431-441
template <class Real>
Real powi(Real base, unsigned e) {
  Real acc(1.0);
  for (; e != 0; e >>= 1) {
    if (e & 1u) acc = acc * base;
    base = base * base;
  }
  return acc;
}

// ---- complex (complex.hpp:10-148) ------------------------------------------
template <class Real>
struct Complex {
  Real re{};
  Real im{};
  constexpr Complex() = default;
  constexpr Complex(Real r) : re(r) {}
  constexpr Complex(Real r, Real i) : re(r), im(i) {}
};
template <class Real>
inline Complex<Real> operator-(const Complex<Real>& a) {
  return Complex<Real>(-a.re, -a.im);
}
template <class Real>
inline Complex<Real> operator+(const Complex<Real>& a, const Complex<Real>& b) {
  return Complex<Real>(a.re + b.re, a.im + b.im);
}
template <class Real>
inline Complex<Real> operator-(const Complex<Real>& a, const Complex<Real>& b) {
  return Complex<Real>(a.re - b.re, a.im - b.im);
}
// textbook product, complex.hpp:35-38
template <class Real>
inline Complex<Real> operator*(const Complex<Real>& a, const Complex<Real>& b) {
  const Real rr = a.re * b.re, ii = a.im * b.im, ri = a.re * b.im, ir = a.im * b.re;
  return Complex<Real>(rr - ii, ri + ir);
}
template <class Real>
inline Complex<Real> operator*(const Complex<Real>& a, const Real& s) {
  return Complex<Real>(a.re * s, a.im * s);
}
template <class Real>
inline Complex<Real> operator*(const Real& s, const Complex<Real>& a) {
  return a * s;
}
template <class Real>
inline Complex<Real> conj(const Complex<Real>& a) {
  return Complex<Real>(a.re, -a.im);
}
template <class Real>
inline Real norm_sqr(const Complex<Real>& a) {
  return a.re * a.re + a.im * a.im;
}
// binary64 modulus of the leading limbs, complex.hpp:113-116
template <class Real>
inline double modulus_double(const Complex<Real>& a) {
  return std::hypot(to_double(a.re), to_double(a.im));
}
// tan-half-angle unit point, complex.hpp:141-148
template <class Real>
inline Complex<Real> unit_complex(double theta) {
  const double t = std::tan(0.5 * theta);
  if (!std::isfinite(t)) return Complex<Real>(Real(-1.0), Real(0.0));
  const Real tt = Real(t) * Real(t);
  const Real den = Real(1.0) + tt;
  return Complex<Real>((Real(1.0) - tt) / den, (Real(t) + Real(t)) / den);
}

}  // namespace orc
