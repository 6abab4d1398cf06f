// work.hpp -- algorithmic work model of the tracked path.
//
// Counts the emulated real operations one evaluation / one least-squares
// solve / one prediction performs, straight from the compiled plan, and turns
// them into FP64 arithmetic instructions of the reference algorithms with the
// per-operation costs measured by tools/count_fp64.cpp on the operation-exact
// host build of mp.cuh (multiprec.hpp sequences; negations and compares are
// not counted).  This is the numerator of roofline.achieved in bench.py.
#pragma once

#include <cstdint>

#include "plan.hpp"

namespace ptwork {

struct OpCount {
  double radd = 0, rmul = 0, rdiv = 0, rsqrt = 0, hypot = 0;
  void cmul(double k = 1) {
    rmul += 4 * k;
    radd += 2 * k;
  }
  void cadd(double k = 1) { radd += 2 * k; }
  void cscale(double k = 1) { rmul += 2 * k; }
  void add(const OpCount& o, double k = 1) {
    radd += k * o.radd;
    rmul += k * o.rmul;
    rdiv += k * o.rdiv;
    rsqrt += k * o.rsqrt;
    hypot += k * o.hypot;
  }
};

// FP64 instructions per emulated real op {add/sub, mul, div, sqrt, hypot}
// (tools/count_fp64.cpp; QD values are averages over random operands since
// qd_distill / qd_renorm5 are data dependent).
inline void fp64_costs(int L, double c[5]) {
  static const double D[5] = {1.0, 1.0, 1.0, 1.0, 19.15};
  static const double DD[5] = {20.0, 11.0, 80.0, 108.0, 19.15};
  static const double QD[5] = {128.36, 343.0, 1407.0, 4622.98, 19.15};
  const double* s = L == 1 ? D : (L == 2 ? DD : QD);
  for (int i = 0; i < 5; ++i) c[i] = s[i];
}

inline double fp64_instructions(const OpCount& o, int L) {
  double c[5];
  fp64_costs(L, c);
  return o.radd * c[0] + o.rmul * c[1] + o.rdiv * c[2] + o.rsqrt * c[3] + o.hypot * c[4];
}

inline int powi_muls(unsigned e) {  // popcount + (bit length - 1): multiprec.hpp:431-441 minus the dead squaring
  if (e == 0) return 0;
  int pc = 0, bl = 0;
  for (unsigned v = e; v; v >>= 1) {
    pc += v & 1u;
    ++bl;
  }
  return pc + bl - 1;
}

// one evaluate_homotopy: weights, monomials, slot sums, combine, norms
inline OpCount eval_work(const ptplan::HostPlan& P, int relax_k) {
  OpCount o;
  o.radd += 1;
  o.rmul += 2 * powi_muls((unsigned)relax_k) + 2;
  for (size_t q = 0; q < P.mono_size.size(); ++q) {
    const int m = P.mono_size[q];
    if (m == 2) o.cmul(1);
    if (m >= 3) o.cmul(3 * m - 5);
    if (P.mono_flags[q] & 1) {
      int npow = 0;
      for (int k = 0; k < m; ++k) {
        const int e = P.mono_exp[P.mono_vbeg[q] + k];
        if (e >= 2) {
          o.cmul(powi_muls((unsigned)(e - 1)));
          o.cscale(1);
          ++npow;
        }
      }
      o.cmul(npow - 1);
      o.cmul(1 + m);
    }
  }
  for (const auto& tk : P.tasks) {
    auto sum = [&](int beg, int cnt) {
      if (cnt <= 0) return;
      for (int r = 0; r < cnt; ++r)
        if (P.ctr_ws[beg + r] >= 0) o.cmul(1);
      o.cadd(cnt - 1);
    };
    sum(tk.g_beg, tk.g_cnt);
    if (tk.f_cnt >= 0) sum(tk.f_beg, tk.f_cnt);
    const bool any = tk.g_cnt > 0 || tk.f_cnt > 0;
    if (any) {
      o.cmul(1);
      o.cscale(1);
      o.cadd(1);
    }
    if (tk.col == P.n) o.hypot += 1;
  }
  return o;
}

// one least_squares_solve on [J | -h] plus the update x += dx
inline OpCount solve_work(int N, int n) {
  OpCount o;
  for (int k = 0; k < n; ++k) {
    o.rmul += 2.0 * N;
    o.radd += N + (N - 1);
    o.rsqrt += 1;
    o.rdiv += 1;
    o.cscale(N);
    const int cols = n - k;  // j = k+1..n
    o.cmul((double)cols * N);
    o.cadd((double)cols * (N - 1));
    const int updated = (k == n - 1) ? cols - 1 : cols;
    o.cmul((double)updated * N);
    o.cadd((double)updated * N);
  }
  o.cmul(0.5 * n * (n - 1));
  o.cadd(0.5 * n * (n - 1));
  o.cscale(n);
  o.hypot += n;
  o.cadd(n);
  return o;
}

// one prediction of degree d over n coordinates
inline OpCount predict_work(int n, int d) {
  OpCount o;
  const double tri = 0.5 * d * (d + 1);
  o.radd += tri + d;
  o.rdiv += tri;
  o.cadd(n * (tri + d));
  o.cscale(n * (tri + d));
  return o;
}

}  // namespace ptwork
