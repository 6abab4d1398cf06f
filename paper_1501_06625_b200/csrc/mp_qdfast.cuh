// mp_qdfast.cuh -- the TOLERANCE-PARITY quad-double arithmetic (fast QD mode).
//
// Included by mp.cuh.  Active only in translation units compiled with
// -DPT_QD_FAST (kern_qd_fast.cu; host code with -DPT_QD_FAST_HOST for the
// CPU accuracy tests): the QD operations r_add / r_mul / r_mul_d / r_div /
// r_sqrt then use these classic quad-double algorithms (Hida, Li & Bailey,
// "Algorithms for quad-double precision floating point arithmetic",
// ARITH-15, 2001: sloppy addition, the O(eps^4)-truncated product, long
// division, Newton reciprocal square root) instead of the reference's
// 8- / 23-addend distill (multiprec.hpp:256-337) and 3-iteration full-QD
// square root (multiprec.hpp:364-372).  Every result is a valid quad-double
// within a few units of 2^-209 of the exact value, but the LIMBS DIFFER from
// the reference: the fast mode promises tolerance parity (end points within
// 1e-55 relative, scaled by the condition estimate, identical step / Newton
// counts barring documented ties), never bit parity.  The default build and
// every bitwise parity test keep the reference sequences.
//
// GPU shape: no sorting network, no data-dependent branches on the common
// path (the renormalisation's zero tests only fire on exact cancellation),
// 3-5x fewer FP64 instructions than the distill forms, and a square root
// whose Newton steps run in increasing precision (binary64 seed -> one
// double-double step -> one quad-double step: 53 -> 106 -> 212 bits).
#pragma once

namespace ptk {
namespace qdfast {

PT_HD void three_sum(double& a, double& b, double& c) {
  double t1, t2, t3;
  t1 = two_sum(a, b, t2);
  a = two_sum(c, t1, t3);
  b = two_sum(t2, t3, c);
}
PT_HD void three_sum2(double& a, double& b, double c) {
  double t1, t2, t3;
  t1 = two_sum(a, b, t2);
  a = two_sum(c, t1, t3);
  b = add64(t2, t3);
}

// renormalisation of a 5-term overlapping expansion (QD library renorm,
// quick_two_sum form); the zero tests only branch on exact cancellation
PT_HD qd renorm5(double c0, double c1, double c2, double c3, double c4) {
  if (!finite(c0)) return {{c0, c1, c2, c3}};
  double s0, s1, s2 = 0.0, s3 = 0.0;
  s0 = quick_two_sum(c3, c4, c4);
  s0 = quick_two_sum(c2, s0, c3);
  s0 = quick_two_sum(c1, s0, c2);
  c0 = quick_two_sum(c0, s0, c1);
  s0 = c0;
  s1 = c1;
  if (s1 != 0.0) {
    s1 = quick_two_sum(s1, c2, s2);
    if (s2 != 0.0) {
      s2 = quick_two_sum(s2, c3, s3);
      if (s3 != 0.0)
        s3 = add64(s3, c4);
      else
        s2 = quick_two_sum(s2, c4, s3);
    } else {
      s1 = quick_two_sum(s1, c3, s2);
      if (s2 != 0.0)
        s2 = quick_two_sum(s2, c4, s3);
      else
        s1 = quick_two_sum(s1, c4, s2);
    }
  } else {
    s0 = quick_two_sum(s0, c2, s1);
    if (s1 != 0.0) {
      s1 = quick_two_sum(s1, c3, s2);
      if (s2 != 0.0)
        s2 = quick_two_sum(s2, c4, s3);
      else
        s1 = quick_two_sum(s1, c4, s2);
    } else {
      s0 = quick_two_sum(s0, c3, s1);
      if (s1 != 0.0)
        s1 = quick_two_sum(s1, c4, s2);
      else
        s0 = quick_two_sum(s0, c4, s1);
    }
  }
  return {{s0, s1, s2, s3}};
}
PT_HD qd renorm4(double c0, double c1, double c2, double c3) { return renorm5(c0, c1, c2, c3, 0.0); }

// a + b: limb-wise two_sums, error propagation by three-sums, renormalise
PT_HD qd add(const qd& a, const qd& b) {
  double s0, s1, s2, s3, t0, t1, t2, t3;
  s0 = two_sum(a.c[0], b.c[0], t0);
  s1 = two_sum(a.c[1], b.c[1], t1);
  s2 = two_sum(a.c[2], b.c[2], t2);
  s3 = two_sum(a.c[3], b.c[3], t3);
  s1 = two_sum(s1, t0, t0);
  three_sum(s2, t0, t1);
  three_sum2(s3, t0, t2);
  t0 = add64(add64(t0, t1), t3);
  return renorm5(s0, s1, s2, s3, t0);
}

// a * b, terms of order eps^4 and below dropped (the O(eps^3) ones summed
// in binary64): 6 exact products, 4 plain ones
PT_HD qd mul(const qd& a, const qd& b) {
  double p0, p1, p2, p3, p4, p5, q0, q1, q2, q3, q4, q5, t0, t1, s0, s1, s2;
  p0 = two_prod(a.c[0], b.c[0], q0);
  p1 = two_prod(a.c[0], b.c[1], q1);
  p2 = two_prod(a.c[1], b.c[0], q2);
  p3 = two_prod(a.c[0], b.c[2], q3);
  p4 = two_prod(a.c[1], b.c[1], q4);
  p5 = two_prod(a.c[2], b.c[0], q5);
  three_sum(p1, p2, q0);   // (p1, p2, q0): order eps
  three_sum(p2, q1, q2);   // six-three sum of p2, q1, q2, p3, p4, p5
  three_sum(p3, p4, p5);
  s0 = two_sum(p2, p3, t0);
  s1 = two_sum(q1, p4, t1);
  s2 = add64(q2, p5);
  s1 = two_sum(s1, t0, t0);
  s2 = add64(s2, add64(t0, t1));
  s1 = add64(s1, add64(add64(add64(add64(add64(add64(add64(mul64(a.c[0], b.c[3]), mul64(a.c[1], b.c[2])),
                                                             mul64(a.c[2], b.c[1])),
                                                       mul64(a.c[3], b.c[0])),
                                                 q0),
                                           q3),
                                     q4),
                               q5));
  return renorm5(p0, p1, s0, s1, s2);
}

PT_HD qd mul_d(const qd& a, double b) {
  double p0, p1, p2, p3, q0, q1, q2, s0, s1, s2, s3, s4;
  p0 = two_prod(a.c[0], b, q0);
  p1 = two_prod(a.c[1], b, q1);
  p2 = two_prod(a.c[2], b, q2);
  p3 = mul64(a.c[3], b);
  s0 = p0;
  s1 = two_sum(q0, p1, s2);
  three_sum(s2, q1, p2);
  three_sum2(q1, q2, p3);
  s3 = q1;
  s4 = add64(q2, p2);
  return renorm5(s0, s1, s2, s3, s4);
}

PT_HD qd neg(const qd& a) { return {{-a.c[0], -a.c[1], -a.c[2], -a.c[3]}}; }

// a / b by long division: five binary64 quotient digits, four exact-ish
// remainder updates, one renormalisation
PT_HD qd div(const qd& a, const qd& b) {
  const double q0 = div64(a.c[0], b.c[0]);
  if (!finite(q0)) return {{q0, 0.0, 0.0, 0.0}};
  qd r = add(a, neg(mul_d(b, q0)));
  const double q1 = div64(r.c[0], b.c[0]);
  r = add(r, neg(mul_d(b, q1)));
  const double q2 = div64(r.c[0], b.c[0]);
  r = add(r, neg(mul_d(b, q2)));
  const double q3 = div64(r.c[0], b.c[0]);
  r = add(r, neg(mul_d(b, q3)));
  const double q4 = div64(r.c[0], b.c[0]);
  return renorm5(q0, q1, q2, q3, q4);
}

// 1/sqrt(a) for a > 0: binary64 seed, one Newton step y += y (1 - a y^2)/2
// in double-double on the two leading limbs (106 bits), one in quad-double
// (212 bits)
PT_HD qd rsqrt(const qd& a) {
  const double y0 = div64(1.0, sqrt64(a.c[0]));
  // double-double step: e = 1 - (a0 + a1) y0^2, y1 = y0 + y0 e / 2
  double ylo;
  const double y2 = two_prod(y0, y0, ylo);  // y0^2 = y2 + ylo exactly
  double e0, e1;
  const double ay = two_prod(a.c[0], y2, e0);  // a0 y2 = ay + e0
  e1 = fma64(a.c[0], ylo, fma64(a.c[1], y2, e0));
  double r1;
  const double r0 = two_sum(1.0, -ay, r1);
  const double corr = mul64(mul64(y0, 0.5), add64(r0, sub64(r1, e1)));
  double y1lo;
  const double y1 = quick_two_sum(y0, corr, y1lo);
  // quad-double step on the full a: y2 = y1 + y1 (1 - a y1^2) / 2
  const qd y{{y1, y1lo, 0.0, 0.0}};
  const qd one{{1.0, 0.0, 0.0, 0.0}};
  const qd r = add(one, neg(mul(a, mul(y, y))));
  return add(y, mul_d(mul(y, r), 0.5));
}

PT_HD qd sqrt(const qd& a) {
  if (a.c[0] == 0.0 && a.c[1] == 0.0 && a.c[2] == 0.0 && a.c[3] == 0.0) return {{0.0, 0.0, 0.0, 0.0}};
  if (a.c[0] < 0.0) return {{bitsd(0x7ff8000000000000ull), 0.0, 0.0, 0.0}};
  return mul(a, rsqrt(a));
}

}  // namespace qdfast
}  // namespace ptk
