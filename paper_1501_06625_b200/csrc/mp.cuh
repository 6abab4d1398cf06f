// mp.cuh -- complex double / double-double / quad-double arithmetic for the
// B200 tracker, usable from host and device code.
//
// Every operation reproduces the operation sequence of the reference scalar
// library bit for bit (IEEE binary64, round-to-nearest-even):
//   error-free transforms      /root/reference/proj/include/pathtrack/multiprec.hpp:36-85
//   DoubleDouble               multiprec.hpp:91-189
//   QuadDouble + qd_distill    multiprec.hpp:196-372
//   powi                       multiprec.hpp:431-441
//   Complex<Real>              /root/reference/proj/include/pathtrack/complex.hpp:10-116
//   modulus_double (std::hypot of the leading limbs)  complex.hpp:113-116
//
// Device code uses the explicit-rounding intrinsics (__dadd_rn, __dmul_rn,
// __fma_rn, __ddiv_rn, __dsqrt_rn) so that nvcc can never contract a*b+c into
// an FMA; host code must be compiled with -ffp-contract=off.  The two_prod
// error term uses one FMA, which is bit-identical to the reference's Dekker
// split (both produce the exact product error).
//
// Data layout on the device is structure-of-arrays: a complex vector of length
// S in precision with L limbs occupies 2*L*S doubles, re limb l at [l*S + i],
// im limb l at [(L+l)*S + i] (see load_c / store_c below).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define PT_HD __host__ __device__ __forceinline__
#define PT_HDI __host__ __device__ inline
// QD operations are hundreds of instructions each: compile them once and call
// them, instead of inlining a 23-way sort at every use site.
#if defined(PT_QD_INLINE) && PT_QD_INLINE
#define PT_QDOP __host__ __device__ __forceinline__
#else
#define PT_QDOP static __host__ __device__ __noinline__
#endif
#else
#define PT_HD inline
#define PT_HDI inline
#define PT_QDOP inline
#endif

// Tolerance-parity QD mode (mp_qdfast.cuh): device code of kern_qd_fast.cu,
// or host code built with -DPT_QD_FAST_HOST (CPU accuracy tests only).
#if defined(PT_QD_FAST) && (defined(__CUDA_ARCH__) || defined(PT_QD_FAST_HOST))
#define PT_QD_FAST_ON 1
#else
#define PT_QD_FAST_ON 0
#endif

namespace ptk {

#if defined(PT_COUNT_FP64) && !defined(__CUDA_ARCH__)
// host-only instrumentation (tools/count_fp64.cpp): FP64 arithmetic
// instructions executed, i.e. the roofline work unit of DESIGN.md section 4
inline unsigned long long g_fp64 = 0;
#define PT_TICK() (++::ptk::g_fp64)
#else
#define PT_TICK() ((void)0)
#endif

// ---------------------------------------------------------------------------
// binary64 primitives with pinned rounding
// ---------------------------------------------------------------------------
PT_HD double add64(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  PT_TICK();
  return a + b;
#endif
}
PT_HD double sub64(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  PT_TICK();
  return a - b;
#endif
}
PT_HD double mul64(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  PT_TICK();
  return a * b;
#endif
}
PT_HD double fma64(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  PT_TICK();
  return std::fma(a, b, c);
#endif
}
PT_HD double div64(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  PT_TICK();
  return a / b;
#endif
}
PT_HD double sqrt64(double a) {
#if defined(__CUDA_ARCH__)
  return __dsqrt_rn(a);
#else
  PT_TICK();
  return std::sqrt(a);
#endif
}
PT_HD uint64_t dbits(double x) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return b;
#endif
}
PT_HD double bitsd(uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(b));
#else
  double x;
  std::memcpy(&x, &b, 8);
  return x;
#endif
}
// |x| as an unsigned key: same order as fabs() for all non-NaN values, +0 == -0.
// Keeps the qd_distill sort compares on the integer pipe instead of FP64.
PT_HD uint64_t mag(double x) { return dbits(x) & 0x7fffffffffffffffull; }
PT_HD bool finite(double x) { return (dbits(x) & 0x7ff0000000000000ull) != 0x7ff0000000000000ull; }
PT_HD double fabs_(double x) { return bitsd(mag(x)); }
// |a| < |b| as the reference writes it (std::fabs compare; false with NaN)
PT_HD bool fabs_cmp_lt(double a, double b) {
#if defined(__CUDA_ARCH__)
  return ::fabs(a) < ::fabs(b);
#else
  return std::fabs(a) < std::fabs(b);
#endif
}
PT_HD int clz32(unsigned x) {
#if defined(__CUDA_ARCH__)
  return __clz(x);
#else
  return x ? __builtin_clz(x) : 32;
#endif
}

// Error-free transforms (multiprec.hpp:39-83).
PT_HD double two_sum(double a, double b, double& e) {
  double s = add64(a, b);
  double bb = sub64(s, a);
  e = add64(sub64(a, sub64(s, bb)), sub64(b, bb));
  return s;
}
PT_HD double quick_two_sum(double a, double b, double& e) {  // requires |a| >= |b|
  double s = add64(a, b);
  e = sub64(b, sub64(s, a));
  return s;
}
PT_HD double two_prod(double a, double b, double& e) {
  double p = mul64(a, b);
  e = fma64(a, b, -p);
  return p;
}

// glibc 2.39 hypot (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel with
// the Borges correction).  std::hypot is what modulus_double calls
// (complex.hpp:115) and it is NOT correctly rounded, so the device has to
// replicate the library's exact sequence to keep the Newton norm tests
// bit-identical.  Verified against glibc on 4e7 random inputs (0 mismatches).
PT_HD double hypot_kernel(double ax, double ay) {
  double t1, t2;
  double h = sqrt64(add64(mul64(ax, ax), mul64(ay, ay)));
  if (h <= mul64(2.0, ay)) {
    double d = sub64(h, ay);
    t1 = mul64(ax, sub64(mul64(2.0, d), ax));
    t2 = mul64(sub64(d, mul64(2.0, sub64(ax, ay))), d);
  } else {
    double d = sub64(h, ax);
    t1 = mul64(mul64(2.0, d), sub64(ax, mul64(2.0, ay)));
    t2 = add64(mul64(sub64(mul64(4.0, d), ay), ay), mul64(d, d));
  }
  return sub64(h, div64(add64(t1, t2), mul64(2.0, h)));
}
PT_HDI double glibc_hypot(double x, double y) {
  if (!finite(x) || !finite(y)) {
    bool xinf = mag(x) == 0x7ff0000000000000ull, yinf = mag(y) == 0x7ff0000000000000ull;
    if (xinf || yinf) return bitsd(0x7ff0000000000000ull);
    return add64(x, y);
  }
  x = fabs_(x);
  y = fabs_(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  if (ax > 0x1p+511) {
    if (ay <= mul64(ax, 0x1p-54)) return add64(ax, ay);
    return div64(hypot_kernel(mul64(ax, 0x1p-600), mul64(ay, 0x1p-600)), 0x1p-600);
  }
  if (ay < 0x1p-459) {
    if (ax >= div64(ay, 0x1p-54)) return add64(ax, ay);
    return mul64(hypot_kernel(div64(ax, 0x1p-600), div64(ay, 0x1p-600)), 0x1p-600);
  }
  if (ay <= mul64(ax, 0x1p-54)) return add64(ax, ay);
  return hypot_kernel(ax, ay);
}

// ---------------------------------------------------------------------------
// Real types.  Layout-compatible with the reference structs
// (DoubleDouble = {hi, lo}; QuadDouble = std::array<double,4>).
// ---------------------------------------------------------------------------
struct dd {
  double hi, lo;
};
struct qd {
  double c[4];
};

template <class R>
struct limbs_of;
template <>
struct limbs_of<double> {
  static constexpr int L = 1;
};
template <>
struct limbs_of<dd> {
  static constexpr int L = 2;
};
template <>
struct limbs_of<qd> {
  static constexpr int L = 4;
};

// ----- double -----
PT_HD double r_from(double x, double*) { return x; }
PT_HD double r_add(double a, double b) { return add64(a, b); }
PT_HD double r_sub(double a, double b) { return sub64(a, b); }
PT_HD double r_neg(double a) { return -a; }
PT_HD double r_mul(double a, double b) { return mul64(a, b); }
PT_HD double r_mul_d(double a, double b) { return mul64(a, b); }
PT_HD double r_div(double a, double b) { return div64(a, b); }
PT_HD double r_sqrt(double a) { return sqrt64(a); }
PT_HD double r_hi(double a) { return a; }
PT_HD bool r_is_zero(double a) { return a == 0.0; }
PT_HD double r_limb(double a, int) { return a; }
PT_HD void r_set_limb(double& a, int, double v) { a = v; }

// ----- double-double (multiprec.hpp:91-189) -----
// multiprec.hpp:102-107 returns {h, 0} for a non-finite h; the device does
// the same with integer masks (dd_norm below), so non-finite DD values match
// the reference too (NaN payloads aside: the GPU's FP64 units produce the
// canonical NaN, x86 propagates the operand's payload).
// -DPT_DD_FAST_NONFINITE drops the non-finite fix-up (round-1 behaviour).
PT_HD dd dd_norm(double h, double l) {  // multiprec.hpp:102-107
  double e;
  double s = quick_two_sum(h, l, e);
#if defined(__CUDA_ARCH__) && defined(PT_DD_FAST_NONFINITE)
  return {s, e};
#elif defined(__CUDA_ARCH__)
  // {h, 0} for a non-finite h, branch- and predicate-free: an all-ones mask
  // from h's exponent field on the integer pipe (it depends on h only, so
  // it is ready long before s and e), then AND / AND-OR on the bit patterns.
  // A predicated select here made ptxas serialise independent DD chains
  // (round 1); the mask form keeps them interleaved and is bit-identical to
  // the reference, non-finite values included.
  const unsigned hw = (unsigned)__double2hiint(h);
  const int t = (int)((hw & 0x7ff00000u) - 0x7ff00000u);          // 0 iff h is inf / NaN
  const long long m = (long long)((t | -t) >> 31);                  // all ones iff h is finite
  const long long sb = __double_as_longlong(s), hb = __double_as_longlong(h);
  return {__longlong_as_double((sb & m) | (hb & ~m)), __longlong_as_double(__double_as_longlong(e) & m)};
#else
  if (!finite(h)) return {h, 0.0};
  return {s, e};
#endif
}
PT_HD dd r_from(double x, dd*) { return {x, 0.0}; }
PT_HD dd r_neg(dd a) { return {-a.hi, -a.lo}; }
PT_HD dd r_add(dd a, dd b) {  // multiprec.hpp:115-123
  double s2, t2;
  double s1 = two_sum(a.hi, b.hi, s2);
  double t1 = two_sum(a.lo, b.lo, t2);
  s2 = add64(s2, t1);
  s1 = quick_two_sum(s1, s2, s2);
  s2 = add64(s2, t2);
  return dd_norm(s1, s2);
}
PT_HD dd r_sub(dd a, dd b) { return r_add(a, r_neg(b)); }
PT_HD dd r_mul(dd a, dd b) {  // multiprec.hpp:127-132
  double e;
  double p = two_prod(a.hi, b.hi, e);
  e = add64(e, add64(add64(mul64(a.hi, b.lo), mul64(a.lo, b.hi)), mul64(a.lo, b.lo)));
  return dd_norm(p, e);
}
PT_HD dd r_mul_d(dd a, double b) {  // multiprec.hpp:134-139
  double e;
  double p = two_prod(a.hi, b, e);
  e = add64(e, mul64(a.lo, b));
  return dd_norm(p, e);
}
PT_HD dd r_div(dd a, dd b) {  // multiprec.hpp:145-155
  double q1 = div64(a.hi, b.hi);
  dd r = r_sub(a, r_mul_d(b, q1));
  double q2 = div64(r.hi, b.hi);
  r = r_sub(r, r_mul_d(b, q2));
  double q3 = div64(r.hi, b.hi);
  double e;
  double s = quick_two_sum(q1, q2, e);
  const dd out = r_add(dd{s, e}, dd{q3, 0.0});
  const bool f = finite(q1);  // non-finite first quotient: {q1, 0} (branch-free select)
  return {f ? out.hi : q1, f ? out.lo : 0.0};
}
// Negative argument: the reference throws std::domain_error
// (multiprec.hpp:178); the device returns NaN instead (never reached on the
// tracker path, whose sqrt arguments are sums of squares).
PT_HD dd r_sqrt(dd a) {  // multiprec.hpp:176-189
  if (a.hi == 0.0 && a.lo == 0.0) return {0.0, 0.0};
  if (a.hi < 0.0) return {bitsd(0x7ff8000000000000ull), 0.0};
  double x = div64(1.0, sqrt64(a.hi));
  double half_x = mul64(0.5, x);
  dd s{mul64(a.hi, x), 0.0};
  dd r = r_sub(a, r_mul(s, s));
  s = r_add(s, dd{mul64(r.hi, half_x), 0.0});
  r = r_sub(a, r_mul(s, s));
  s = r_add(s, dd{mul64(r.hi, half_x), 0.0});
  return s;
}
PT_HD double r_hi(dd a) { return a.hi; }
PT_HD bool r_is_zero(dd a) { return a.hi == 0.0 && a.lo == 0.0; }
PT_HD double r_limb(const dd& a, int l) { return l == 0 ? a.hi : a.lo; }
PT_HD void r_set_limb(dd& a, int l, double v) {
  if (l == 0)
    a.hi = v;
  else
    a.lo = v;
}

}  // namespace ptk
#include "mp_qdfast.cuh"
namespace ptk {

// ----- quad-double (multiprec.hpp:196-372) -----
// qd_renorm5, multiprec.hpp:209-250.  Branch structure kept verbatim: the
// zero tests decide which limbs absorb the tail, and changing them changes bits.
PT_HDI qd qd_renorm5(double c0, double c1, double c2, double c3, double c4) {
  if (!finite(c0)) return {{c0, 0.0, 0.0, 0.0}};
  double s0, s1, s2 = 0.0, s3 = 0.0;
  s0 = two_sum(c3, c4, c4);
  s0 = two_sum(c2, s0, c3);
  s0 = two_sum(c1, s0, c2);
  c0 = two_sum(c0, s0, c1);
  s0 = c0;
  s1 = c1;
  if (s1 != 0.0) {
    s1 = two_sum(s1, c2, s2);
    if (s2 != 0.0) {
      s2 = two_sum(s2, c3, s3);
      if (s3 != 0.0)
        s3 = add64(s3, c4);
      else
        s2 = two_sum(s2, c4, s3);
    } else {
      s1 = two_sum(s1, c3, s2);
      if (s2 != 0.0)
        s2 = two_sum(s2, c4, s3);
      else
        s1 = two_sum(s1, c4, s2);
    }
  } else {
    s0 = two_sum(s0, c2, s1);
    if (s1 != 0.0) {
      s1 = two_sum(s1, c3, s2);
      if (s2 != 0.0)
        s2 = two_sum(s2, c4, s3);
      else
        s1 = two_sum(s1, c4, s2);
    } else {
      s0 = two_sum(s0, c3, s1);
      if (s1 != 0.0)
        s1 = two_sum(s1, c4, s2);
      else
        s0 = two_sum(s0, c4, s1);
    }
  }
  return {{s0, s1, s2, s3}};
}

// qd_distill, multiprec.hpp:256-279, with K a compile-time constant so the
// addend array lives in registers.  The reference orders addends by a stable
// insertion sort on |m| (descending, ties keep input order); any stable sort
// yields the same permutation.  Variants (PT_QD_SORT), all comparing
//   4 (default) odd-even transposition: K rounds of adjacent compare-exchanges
//     swapping only on strict fabs(a) < fabs(b) (the reference's compare, one
//     DSETP), branch-free, constant depth -- lowest latency and highest
//     throughput measured on B200 (tools/qd_sort_bench.cu: QD mul 3.3k cycles
//     dependent, 5.6 T FP64 instr/s; the integer-key variant 3: 5.0k, 3.6 T);
//   3 the same network comparing magnitudes as integers on the FP64 bits;
//   2 insertion position by mask; 1 plain insertion; 0 insertion with a
//     warp-uniform early exit (integer keys).
#ifndef PT_QD_MUL_LEVELS
#define PT_QD_MUL_LEVELS 1
#endif
#ifndef PT_QD_SORT
#define PT_QD_SORT 4
#endif
template <int K>
PT_HD void qd_sort(double (&m)[K]) {
#if PT_QD_SORT == 2
  // Insertion position by mask: all compares of the sorted prefix against v
  // are independent; pos = 1 + index of the highest prefix entry with
  // |m[j]| >= |v| (stable: ties stay in front); then an independent shift.
  // Same permutation as the reference's insertion sort, constant depth per
  // element instead of a chain as long as the move.
#pragma unroll
  for (int i = 1; i < K; ++i) {
    const double v = m[i];
    const uint64_t av = mag(v);
    if (mag(m[i - 1]) >= av) continue;  // already in place: the common case
    unsigned keep = 0;  // bit j: m[j] stays in front of v
#pragma unroll
    for (int j = 0; j < i - 1; ++j) keep |= (mag(m[j]) >= av ? 1u : 0u) << j;
    const int pos = 32 - clz32(keep);  // 0 when every prefix entry moves
#pragma unroll
    for (int j = i; j >= 1; --j) m[j] = (j > pos) ? m[j - 1] : (j == pos ? v : m[j]);
    if (pos == 0) m[0] = v;
  }
#elif PT_QD_SORT == 4
  // odd-even transposition with the reference's own comparison,
  // fabs(m[i]) < fabs(m[i+1]) (one DSETP with |.| operand modifiers on the
  // otherwise idle FP64 pipe instead of 64-bit integer compares on the ALU
  // pipe); NaN never swaps, exactly as it blocks the reference's insertion.
#pragma unroll
  for (int r = 0; r < K; ++r) {
#pragma unroll
    for (int i = r & 1; i + 1 < K; i += 2) {
      const double a = m[i], b = m[i + 1];
      const bool sw = fabs_cmp_lt(a, b);
      m[i] = sw ? b : a;
      m[i + 1] = sw ? a : b;
    }
  }
#elif PT_QD_SORT == 3
  // odd-even transposition sort: K rounds of adjacent compare-exchanges that
  // swap only on strict |m[i]| < |m[i+1]| (stable), so the permutation equals
  // the reference's stable insertion sort; constant depth K, no branches.
#pragma unroll
  for (int r = 0; r < K; ++r) {
#pragma unroll
    for (int i = r & 1; i + 1 < K; i += 2) {
      const double a = m[i], b = m[i + 1];
      const bool sw = mag(a) < mag(b);
      m[i] = sw ? b : a;
      m[i + 1] = sw ? a : b;
    }
  }
#else
#pragma unroll
  for (int i = 1; i < K; ++i) {
    const double v = m[i];
    const uint64_t av = mag(v);
    if (mag(m[i - 1]) >= av) continue;  // already in place: the common case
    bool moving = true;
#pragma unroll
    for (int j = i - 1; j >= 0; --j) {
#if defined(__CUDA_ARCH__) && PT_QD_SORT == 0
      // leave once no lane of the warp still moves
      if (!__any_sync(__activemask(), moving)) break;
#elif !defined(__CUDA_ARCH__)
      if (!moving) break;
#endif
      const bool c = moving && (mag(m[j]) < av);
      m[j + 1] = c ? m[j] : (moving ? v : m[j + 1]);
      moving = c;
    }
    if (moving) m[0] = v;
  }
#endif
}

// qd_distill after the sort: two two_sum sweeps, tail, renorm5 (multiprec.hpp:269-278)
template <int K>
PT_HD qd qd_distill_sorted(double (&m)[K]) {
  if (!finite(m[0])) return {{m[0], 0.0, 0.0, 0.0}};
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
    for (int i = K - 1; i >= 1; --i) m[i - 1] = two_sum(m[i - 1], m[i], m[i]);
  }
  double tail = 0.0;
#pragma unroll
  for (int i = K - 1; i >= 4; --i) tail = add64(tail, m[i]);
  const double c0 = K > 0 ? m[0] : 0.0;
  const double c1 = K > 1 ? m[K > 1 ? 1 : 0] : 0.0;
  const double c2 = K > 2 ? m[K > 2 ? 2 : 0] : 0.0;
  const double c3 = K > 3 ? m[K > 3 ? 3 : 0] : 0.0;
  return qd_renorm5(c0, c1, c2, c3, tail);
}

template <int K>
PT_HD qd qd_distill(double (&m)[K]) {
  qd_sort<K>(m);
  return qd_distill_sorted<K>(m);
}

// Stable odd-even transposition on G values (descending |.|, strict swaps).
template <int G>
PT_HD void oe_sort(double (&g)[G]) {
#pragma unroll
  for (int r = 0; r < G; ++r) {
#pragma unroll
    for (int i = r & 1; i + 1 < G; i += 2) {
      const double a = g[i], b = g[i + 1];
      const bool sw = fabs_cmp_lt(a, b);
      g[i] = sw ? b : a;
      g[i + 1] = sw ? a : b;
    }
  }
}

PT_HD qd r_from(double x, qd*) { return {{x, 0.0, 0.0, 0.0}}; }
PT_HD qd r_neg(const qd& a) { return {{-a.c[0], -a.c[1], -a.c[2], -a.c[3]}}; }
PT_QDOP qd r_add(qd a, qd b) {  // multiprec.hpp:290-293
#if PT_QD_FAST_ON
  return qdfast::add(a, b);
#endif
  double m[8] = {a.c[0], a.c[1], a.c[2], a.c[3], b.c[0], b.c[1], b.c[2], b.c[3]};
  return qd_distill<8>(m);
}
PT_HD qd r_sub(qd a, qd b) { return r_add(a, r_neg(b)); }
PT_QDOP qd r_mul(qd a, qd b) {  // multiprec.hpp:297-312
#if PT_QD_FAST_ON
  return qdfast::mul(a, b);
#endif
  double m[23];
  int k = 0;
#pragma unroll
  for (int i = 0; i <= 3; ++i) {
#pragma unroll
    for (int j = 0; j + i <= 3; ++j) {
      double e;
      m[k++] = two_prod(a.c[i], b.c[j], e);
      m[k++] = e;
    }
  }
  m[20] = mul64(a.c[1], b.c[3]);
  m[21] = mul64(a.c[2], b.c[2]);
  m[22] = mul64(a.c[3], b.c[1]);
#if PT_QD_MUL_LEVELS
  // Short left operand (a = (a0, 0, 0, 0): coefficients built from doubles,
  // Rng::box / complex_from): every addend with index >= 8 is a product with
  // a zero limb, i.e. +-0, and all indices >= 8 follow 0..7.  The stable sort
  // is then the stable sort of m[0..7] (its zeros sink to its end in index
  // order) followed by m[8..22] unchanged.
  if (a.c[1] == 0.0 && a.c[2] == 0.0 && a.c[3] == 0.0) {
    double s8[8] = {m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7]};
    oe_sort<8>(s8);
    double s[23] = {s8[0], s8[1], s8[2],  s8[3],  s8[4],  s8[5],  s8[6],  s8[7],  m[8],  m[9],  m[10], m[11],
                    m[12], m[13], m[14], m[15], m[16], m[17], m[18], m[19], m[20], m[21], m[22]};
    return qd_distill_sorted<23>(s);
  }
  // Fast path, same permutation: group the 23 addends by "level" i+j of
  // p_ij = fl(a_i b_j) (level i+j+1 for its error e_ij and for the three
  // plain products), each group listed in input order:
  //   G0 {p00}  G1 {e00 p01 p10}  G2 {e01 p02 e10 p11 p20}
  //   G3 {e02 p03 e11 p12 e20 p21 p30}  G4 {e03 e12 e21 e30 x13 x22 x31}.
  // Sort each group stably (55 compare-exchanges instead of 253).  If every
  // element of each group is STRICTLY larger in magnitude than every element
  // of the next (4 checks on the sorted groups' ends), the concatenation is
  // the stable sort of all 23 -- exactly the reference's insertion-sort
  // permutation.  Otherwise (zeros, short or non-canonical operands, NaN)
  // the full network sorts the original array.
  double g1[3] = {m[1], m[2], m[8]};
  double g2[5] = {m[3], m[4], m[9], m[10], m[14]};
  double g3[7] = {m[5], m[6], m[11], m[12], m[15], m[16], m[18]};
  double g4[7] = {m[7], m[13], m[17], m[19], m[20], m[21], m[22]};
  oe_sort<3>(g1);
  oe_sort<5>(g2);
  oe_sort<7>(g3);
  oe_sort<7>(g4);
  const bool levels = fabs_cmp_lt(g1[0], m[0]) && fabs_cmp_lt(g2[0], g1[2]) && fabs_cmp_lt(g3[0], g2[4]) &&
                      fabs_cmp_lt(g4[0], g3[6]);
  if (levels) {
    double s[23] = {m[0],  g1[0], g1[1], g1[2], g2[0], g2[1], g2[2], g2[3], g2[4], g3[0], g3[1], g3[2],
                    g3[3], g3[4], g3[5], g3[6], g4[0], g4[1], g4[2], g4[3], g4[4], g4[5], g4[6]};
    return qd_distill_sorted<23>(s);
  }
#endif
  return qd_distill<23>(m);
}
PT_QDOP qd r_mul_d(qd a, double b) {  // multiprec.hpp:314-323
#if PT_QD_FAST_ON
  return qdfast::mul_d(a, b);
#endif
  double m[8];
#pragma unroll
  for (int i = 0; i <= 3; ++i) {
    double e;
    m[2 * i] = two_prod(a.c[i], b, e);
    m[2 * i + 1] = e;
  }
#if PT_QD_MUL_LEVELS
  // Same permutation, cheaper (cf. r_mul): addends m = p0 e0 p1 e1 p2 e2 p3 e3.
  //  * exact products (all e_i == 0, e.g. b = 0.5) with |p0|>|p1|>|p2|>|p3|>0:
  //    the stable sort is p0 p1 p2 p3 then the four zeros in index order;
  //  * else level groups {p0} {e0 p1} {e1 p2} {e2 p3} {e3}, each sorted stably,
  //    valid when every group is strictly larger than the next.
  if (m[1] == 0.0 && m[3] == 0.0 && m[5] == 0.0 && m[7] == 0.0 && fabs_cmp_lt(m[2], m[0]) &&
      fabs_cmp_lt(m[4], m[2]) && fabs_cmp_lt(m[6], m[4]) && m[6] != 0.0) {
    double s[8] = {m[0], m[2], m[4], m[6], m[1], m[3], m[5], m[7]};
    return qd_distill_sorted<8>(s);
  }
  {
    double g1[2] = {m[1], m[2]}, g2[2] = {m[3], m[4]}, g3[2] = {m[5], m[6]};
    oe_sort<2>(g1);
    oe_sort<2>(g2);
    oe_sort<2>(g3);
    if (fabs_cmp_lt(g1[0], m[0]) && fabs_cmp_lt(g2[0], g1[1]) && fabs_cmp_lt(g3[0], g2[1]) &&
        fabs_cmp_lt(m[7], g3[1])) {
      double s[8] = {m[0], g1[0], g1[1], g2[0], g2[1], g3[0], g3[1], m[7]};
      return qd_distill_sorted<8>(s);
    }
  }
#endif
  return qd_distill<8>(m);
}
PT_QDOP qd r_div(qd a, qd b) {  // multiprec.hpp:327-337
#if PT_QD_FAST_ON
  return qdfast::div(a, b);
#endif
  double q0 = div64(a.c[0], b.c[0]);
  if (!finite(q0)) return {{q0, 0.0, 0.0, 0.0}};
  double q[5];
  qd r = a;
#pragma unroll 1
  for (int i = 0; i < 5; ++i) {
    double qi = div64(r.c[0], b.c[0]);
    r = r_sub(r, r_mul_d(b, qi));
#pragma unroll
    for (int j = 0; j < 5; ++j)
      if (j == i) q[j] = qi;
  }
  return qd_distill<5>(q);
}
PT_QDOP qd r_sqrt(qd a) {  // multiprec.hpp:364-372
#if PT_QD_FAST_ON
  return qdfast::sqrt(a);
#endif
  if (a.c[0] == 0.0 && a.c[1] == 0.0 && a.c[2] == 0.0 && a.c[3] == 0.0) return {{0.0, 0.0, 0.0, 0.0}};
  if (a.c[0] < 0.0) return {{bitsd(0x7ff8000000000000ull), 0.0, 0.0, 0.0}};
  qd x{{div64(1.0, sqrt64(a.c[0])), 0.0, 0.0, 0.0}};
  const qd one{{1.0, 0.0, 0.0, 0.0}};
#pragma unroll 1
  for (int i = 0; i < 3; ++i) x = r_add(x, r_mul(x, r_mul_d(r_sub(one, r_mul(a, r_mul(x, x))), 0.5)));
  return r_mul(a, x);
}
PT_HD double r_hi(const qd& a) { return a.c[0]; }
PT_HD bool r_is_zero(const qd& a) { return a.c[0] == 0.0 && a.c[1] == 0.0 && a.c[2] == 0.0 && a.c[3] == 0.0; }
PT_HD double r_limb(const qd& a, int l) { return a.c[l]; }
PT_HD void r_set_limb(qd& a, int l, double v) { a.c[l] = v; }
PT_QDOP qd qd_renormalize(qd a) {  // multiprec.hpp:283-286
#if PT_QD_FAST_ON
  return qdfast::renorm4(a.c[0], a.c[1], a.c[2], a.c[3]);
#endif
  double m[4] = {a.c[0], a.c[1], a.c[2], a.c[3]};
  return qd_distill<4>(m);
}

template <class R>
PT_HD R rconst(double x) {
  return r_from(x, static_cast<R*>(nullptr));
}

// r = sqrt(x) and inv = 1/r, the pair every MGS normalisation needs
// (r_kk = sqrt(norm^2), q_k = a_k * (1/r_kk)).  Reference
// sequence: sqrt, then one division.  Fast QD mode: one reciprocal square
// root y ~ 1/sqrt(x) (mp_qdfast.cuh) gives both, r = x y and inv = y -- no
// division on the column chain (tolerance parity).
template <class R>
PT_HD void r_sqrt_inv(const R& x, R& r, R& inv) {
  r = r_sqrt(x);
  inv = r_div(rconst<R>(1.0), r);
}
#if PT_QD_FAST_ON
template <>
PT_HD void r_sqrt_inv<qd>(const qd& x, qd& r, qd& inv) {
  if (!(x.c[0] > 0.0) || !finite(x.c[0])) {  // zero, negative, NaN, inf: the plain forms
    r = r_sqrt(x);
    inv = r_div(rconst<qd>(1.0), r);
    return;
  }
  inv = qdfast::rsqrt(x);
  r = qdfast::mul(x, inv);
}
#endif

// Binary exponentiation, multiprec.hpp:431-441.  Starts from one and
// multiplies result*base exactly like the reference (1*base is not elided:
// for QD it can renormalise non-canonical limbs).  The final squaring of the
// reference is dead and skipped.
template <class T>
PT_HD T powi_generic(T base, unsigned e, T one) {
  T result = one;
  while (e) {
    if (e & 1u) result = result * base;
    e >>= 1;
    if (e) base = base * base;
  }
  return result;
}

// ---------------------------------------------------------------------------
// Complex (complex.hpp:10-116)
// ---------------------------------------------------------------------------
template <class R>
struct cplx {
  R re, im;
};

template <class R>
PT_HD cplx<R> c_zero() {
  return {rconst<R>(0.0), rconst<R>(0.0)};
}
template <class R>
PT_HD cplx<R> c_one() {
  return {rconst<R>(1.0), rconst<R>(0.0)};
}
template <class R>
PT_HD cplx<R> c_add(const cplx<R>& a, const cplx<R>& b) {
  return {r_add(a.re, b.re), r_add(a.im, b.im)};
}
template <class R>
PT_HD cplx<R> c_sub(const cplx<R>& a, const cplx<R>& b) {
  return {r_sub(a.re, b.re), r_sub(a.im, b.im)};
}
template <class R>
PT_HD cplx<R> c_neg(const cplx<R>& a) {
  return {r_neg(a.re), r_neg(a.im)};
}
// complex.hpp:36-38: {a.re*b.re - a.im*b.im, a.re*b.im + a.im*b.re}
template <class R>
PT_HD cplx<R> c_mul(const cplx<R>& a, const cplx<R>& b) {
  return {r_sub(r_mul(a.re, b.re), r_mul(a.im, b.im)), r_add(r_mul(a.re, b.im), r_mul(a.im, b.re))};
}
// complex.hpp:41-43: Complex * Real
template <class R>
PT_HD cplx<R> c_scale(const cplx<R>& a, const R& s) {
  return {r_mul(a.re, s), r_mul(a.im, s)};
}
// conj(a) * b with the reference's operator sequence (complex.hpp:96-98, 36-38)
template <class R>
PT_HD cplx<R> c_conj_mul(const cplx<R>& a, const cplx<R>& b) {
  const R nim = r_neg(a.im);
  return {r_sub(r_mul(a.re, b.re), r_mul(nim, b.im)), r_add(r_mul(a.re, b.im), r_mul(nim, b.re))};
}
// complex.hpp:101-103
template <class R>
PT_HD R c_norm_sqr(const cplx<R>& a) {
  return r_add(r_mul(a.re, a.re), r_mul(a.im, a.im));
}
// complex.hpp:113-116
template <class R>
PT_HD double c_mod_double(const cplx<R>& a) {
  return glibc_hypot(r_hi(a.re), r_hi(a.im));
}
template <class R>
PT_HD bool c_is_zero(const cplx<R>& a) {
  return r_is_zero(a.re) && r_is_zero(a.im);
}

// operator sugar so powi_generic reads like the reference
template <class R>
PT_HD cplx<R> operator*(const cplx<R>& a, const cplx<R>& b) {
  return c_mul(a, b);
}
template <class R>
PT_HD cplx<R> c_powi(const cplx<R>& base, unsigned e) {
  return powi_generic(base, e, c_one<R>());
}
struct rwrap_dd {
  dd v;
};
PT_HD rwrap_dd operator*(rwrap_dd a, rwrap_dd b) { return {r_mul(a.v, b.v)}; }
struct rwrap_qd {
  qd v;
};
PT_HD rwrap_qd operator*(const rwrap_qd& a, const rwrap_qd& b) { return {r_mul(a.v, b.v)}; }
PT_HD double r_powi(double b, unsigned e) { return powi_generic(b, e, 1.0); }
PT_HD dd r_powi(dd b, unsigned e) { return powi_generic(rwrap_dd{b}, e, rwrap_dd{{1.0, 0.0}}).v; }
PT_HD qd r_powi(const qd& b, unsigned e) {
  return powi_generic(rwrap_qd{b}, e, rwrap_qd{{{1.0, 0.0, 0.0, 0.0}}}).v;
}

// ---------------------------------------------------------------------------
// SoA load / store of complex entries.  Stride S = vector (or matrix) length.
// ---------------------------------------------------------------------------
template <class R>
PT_HD cplx<R> load_c(const double* p, long S, long i) {
  constexpr int L = limbs_of<R>::L;
  cplx<R> v;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    r_set_limb(v.re, l, p[l * S + i]);
    r_set_limb(v.im, l, p[(L + l) * S + i]);
  }
  return v;
}
template <class R>
PT_HD void store_c(double* p, long S, long i, const cplx<R>& v) {
  constexpr int L = limbs_of<R>::L;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    p[l * S + i] = r_limb(v.re, l);
    p[(L + l) * S + i] = r_limb(v.im, l);
  }
}
template <class R>
PT_HD R load_r(const double* p, long S, long i) {
  constexpr int L = limbs_of<R>::L;
  R v;
#pragma unroll
  for (int l = 0; l < L; ++l) r_set_limb(v, l, p[l * S + i]);
  return v;
}
template <class R>
PT_HD void store_r(double* p, long S, long i, const R& v) {
  constexpr int L = limbs_of<R>::L;
#pragma unroll
  for (int l = 0; l < L; ++l) p[l * S + i] = r_limb(v, l);
}

// unit_complex, complex.hpp:141-148: e^{i theta} via tan(theta/2).  Host only
// (tan is libm's; gamma is built once on the host and shipped as limbs).
template <class R>
inline cplx<R> unit_complex_host(double theta) {
  double t = std::tan(0.5 * theta);
  if (!std::isfinite(t)) return {rconst<R>(-1.0), rconst<R>(0.0)};
  R tr = rconst<R>(t);
  R tt = r_mul(tr, tr);
  R den = r_add(rconst<R>(1.0), tt);
  return {r_div(r_sub(rconst<R>(1.0), tt), den), r_div(r_add(tr, tr), den)};
}

}  // namespace ptk
