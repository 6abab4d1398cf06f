// inputs.hpp -- shared internals of the host-only inputs library
// (libpt_inputs.so: gen.cpp, sysio.cpp, pieri.cpp).  No CUDA.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pathtrack_inputs.h"
#include "mp.cuh"

struct pt_sysbuf {
  int32_t n_vars = 0, n_eqs = 0, L = 1;
  std::vector<int32_t> eq_ptr, term_ptr, var, exp;
  std::vector<double> coef;  // [2][L][n_terms]
};

namespace ptgen {

inline thread_local std::string g_err;
inline int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

using Support = std::vector<std::pair<int, int>>;  // (var, exp), var ascending

struct Term {
  Support sup;
  double c[8];  // re limbs then im limbs (2L used)
};

class Rng {  // rng.hpp:14-45
 public:
  explicit Rng(uint64_t seed) : g_(seed) {}
  uint64_t bits() { return g_(); }
  double uniform01() { return static_cast<double>(g_() >> 11) * 0x1p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  double angle() { return 2.0 * std::numbers::pi * uniform01(); }

 private:
  std::mt19937_64 g_;
};

inline int limbs(pt_prec p) { return p == PT_D ? 1 : (p == PT_DD ? 2 : 4); }

// canonical form: terms sorted lexicographically by support
inline pt_sysbuf* emit(int n, std::vector<std::vector<Term>>& eqs, int L) {
  auto* s = new pt_sysbuf;
  s->n_vars = n;
  s->n_eqs = (int)eqs.size();
  s->L = L;
  s->eq_ptr.push_back(0);
  s->term_ptr.push_back(0);
  std::vector<const Term*> all;
  for (auto& e : eqs) {
    std::stable_sort(e.begin(), e.end(), [](const Term& a, const Term& b) { return a.sup < b.sup; });
    for (auto& t : e) {
      for (auto& ve : t.sup) {
        s->var.push_back(ve.first);
        s->exp.push_back(ve.second);
      }
      s->term_ptr.push_back((int)s->var.size());
      all.push_back(&t);
    }
    s->eq_ptr.push_back((int)all.size());
  }
  const long T = (long)all.size();
  s->coef.assign((size_t)2 * L * T, 0.0);
  for (long t = 0; t < T; ++t)
    for (int q = 0; q < 2 * L; ++q) s->coef[(size_t)q * T + t] = all[t]->c[q];
  return s;
}

template <class R>
void put(Term& t, const ptk::cplx<R>& v) {
  constexpr int L = ptk::limbs_of<R>::L;
  for (int l = 0; l < L; ++l) {
    t.c[l] = ptk::r_limb(v.re, l);
    t.c[L + l] = ptk::r_limb(v.im, l);
  }
}
inline Term make_term(Support sup, double re, double im, int L) {
  Term t;
  t.sup = std::move(sup);
  std::memset(t.c, 0, sizeof t.c);
  t.c[0] = re;
  t.c[L] = im;
  return t;
}


// Canonical form of parsed / caller-built systems: terms sorted
// lexicographically by support (stable), duplicate supports merged by
// coefficient addition in the working precision (complex.hpp operator+,
// in term order), zero coefficients dropped.
template <class R>
void merge_terms(std::vector<Term>& e) {
  constexpr int L = ptk::limbs_of<R>::L;
  std::stable_sort(e.begin(), e.end(), [](const Term& a, const Term& b) { return a.sup < b.sup; });
  std::vector<Term> out;
  auto get = [&](const Term& t) {
    ptk::cplx<R> v;
    for (int l = 0; l < L; ++l) {
      ptk::r_set_limb(v.re, l, t.c[l]);
      ptk::r_set_limb(v.im, l, t.c[L + l]);
    }
    return v;
  };
  for (const Term& t : e) {
    if (!out.empty() && out.back().sup == t.sup) {
      put<R>(out.back(), ptk::c_add(get(out.back()), get(t)));
    } else {
      out.push_back(t);
    }
  }
  e.clear();
  for (const Term& t : out)
    if (!ptk::c_is_zero(get(t))) e.push_back(t);
}
inline void canonicalize(std::vector<std::vector<Term>>& eqs, int L) {
  for (auto& e : eqs) {
    if (L == 1) merge_terms<double>(e);
    else if (L == 2) merge_terms<ptk::dd>(e);
    else merge_terms<ptk::qd>(e);
  }
}
// equations of a buffer as term lists
inline std::vector<std::vector<Term>> terms_of(const pt_sysbuf& s) {
  std::vector<std::vector<Term>> eqs(s.n_eqs);
  const long T = (long)s.term_ptr.size() - 1;
  for (int i = 0; i < s.n_eqs; ++i)
    for (int t = s.eq_ptr[i]; t < s.eq_ptr[i + 1]; ++t) {
      Term tm;
      for (int q = s.term_ptr[t]; q < s.term_ptr[t + 1]; ++q) tm.sup.push_back({s.var[q], s.exp[q]});
      std::memset(tm.c, 0, sizeof tm.c);
      for (int q = 0; q < 2 * s.L; ++q) tm.c[q] = s.coef[(size_t)q * T + t];
      eqs[i].push_back(tm);
    }
  return eqs;
}

}  // namespace ptgen
