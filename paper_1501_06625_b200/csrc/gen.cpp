// gen.cpp -- synthetic systems for the BASELINE.json configurations (host).
//
// Not on the hot path: these build the inputs both the CUDA tracker and the
// CPU oracle consume, so every test and bench line sees identical systems.
//   cyclic n-roots          SPEC.md:529-537, PAPER.md:726-734 (Eq. 5)
//   augment_with_linear     SPEC.md:547-555 (Eq. 6)
//   Chandrasekhar H
//   random dense degree-d
//   total-degree start      g_i = x_i^d - 1
// Randomness follows pathtrack::Rng (rng.hpp:14-45): std::mt19937_64,
// uniform01 = (bits >> 11) * 2^-53, box<R> = (uniform(-1,1), uniform(-1,1)),
// unit<R> = unit_complex<R>(2*pi*uniform01).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <numbers>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pathtrack_b200.h"
#include "mp.cuh"

struct pt_sysbuf {
  int32_t n_vars = 0, n_eqs = 0, L = 1;
  std::vector<int32_t> eq_ptr, term_ptr, var, exp;
  std::vector<double> coef;  // [2][L][n_terms]
};

namespace ptgen {

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
pt_sysbuf* emit(int n, std::vector<std::vector<Term>>& eqs, int L) {
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
Term make_term(Support sup, double re, double im, int L) {
  Term t;
  t.sup = std::move(sup);
  std::memset(t.c, 0, sizeof t.c);
  t.c[0] = re;
  t.c[L] = im;
  return t;
}

template <class R>
pt_sysbuf* chandra(int n, double c) {
  constexpr int L = ptk::limbs_of<R>::L;
  using namespace ptk;
  const R two_n = rconst<R>(2.0 * n);
  std::vector<R> mu(n);
  for (int i = 0; i < n; ++i) mu[i] = r_div(rconst<R>(2.0 * i + 1.0), two_n);  // (i+1/2)/n
  const R cc = rconst<R>(c);
  std::vector<std::vector<Term>> eqs(n);
  for (int i = 0; i < n; ++i) {
    // 2n x_i - 2n - sum_j c*mu_i/(mu_i+mu_j) x_i x_j
    eqs[i].push_back(make_term({}, -2.0 * n, 0.0, L));
    eqs[i].push_back(make_term({{i, 1}}, 2.0 * n, 0.0, L));
    for (int j = 0; j < n; ++j) {
      R w = r_neg(r_div(r_mul(cc, mu[i]), r_add(mu[i], mu[j])));
      Support sup = (i == j) ? Support{{i, 2}} : (i < j ? Support{{i, 1}, {j, 1}} : Support{{j, 1}, {i, 1}});
      Term t;
      t.sup = sup;
      std::memset(t.c, 0, sizeof t.c);
      put<R>(t, cplx<R>{w, rconst<R>(0.0)});
      eqs[i].push_back(t);
    }
  }
  return emit(n, eqs, L);
}

}  // namespace ptgen

using namespace ptgen;

template <class R>
static void unit_out(double theta, double* out) {
  constexpr int L = ptk::limbs_of<R>::L;
  auto u = ptk::unit_complex_host<R>(theta);
  for (int l = 0; l < L; ++l) {
    out[l] = ptk::r_limb(u.re, l);
    out[L + l] = ptk::r_limb(u.im, l);
  }
}


extern "C" {

int pt_gen_cyclic(int32_t n, pt_prec prec, pt_sysbuf** out) {
  if (n < 2 || !out) return PT_E_INVAL;
  const int L = limbs(prec);
  std::vector<std::vector<Term>> eqs(n);
  for (int i = 1; i < n; ++i) {  // f_i: sum_tau prod_{k<i} x_{(tau+k) mod n}
    for (int tau = 0; tau < n; ++tau) {
      std::vector<int> vs;
      for (int k = 0; k < i; ++k) vs.push_back((tau + k) % n);
      std::sort(vs.begin(), vs.end());
      Support sup;
      for (int v : vs) sup.push_back({v, 1});
      eqs[i - 1].push_back(make_term(sup, 1.0, 0.0, L));
    }
  }
  Support all;
  for (int v = 0; v < n; ++v) all.push_back({v, 1});
  eqs[n - 1].push_back(make_term(all, 1.0, 0.0, L));
  eqs[n - 1].push_back(make_term({}, -1.0, 0.0, L));
  *out = emit(n, eqs, L);
  return PT_OK;
}

// dim random affine rows c_0 + sum_j c_{j+1} x_j, coefficients Rng::box
// drawn row by row, constant first.
int pt_gen_augment(const pt_sysbuf* f, int32_t dim, uint64_t seed, pt_prec prec, pt_sysbuf** out) {
  if (!f || !out || dim < 0) return PT_E_INVAL;
  const int L = limbs(prec);
  if (L != f->L) return PT_E_INVAL;
  const int n = f->n_vars;
  std::vector<std::vector<Term>> eqs(f->n_eqs + dim);
  const long T = (long)f->term_ptr.size() - 1;
  for (int i = 0; i < f->n_eqs; ++i) {
    for (int t = f->eq_ptr[i]; t < f->eq_ptr[i + 1]; ++t) {
      Term tm;
      for (int q = f->term_ptr[t]; q < f->term_ptr[t + 1]; ++q) tm.sup.push_back({f->var[q], f->exp[q]});
      std::memset(tm.c, 0, sizeof tm.c);
      for (int q = 0; q < 2 * L; ++q) tm.c[q] = f->coef[(size_t)q * T + t];
      eqs[i].push_back(tm);
    }
  }
  Rng rng(seed);
  for (int r = 0; r < dim; ++r) {
    auto& e = eqs[f->n_eqs + r];
    for (int q = 0; q <= n; ++q) {
      const double re = rng.uniform(-1.0, 1.0);
      const double im = rng.uniform(-1.0, 1.0);
      e.push_back(make_term(q == 0 ? Support{} : Support{{q - 1, 1}}, re, im, L));
    }
  }
  *out = emit(n, eqs, L);
  return PT_OK;
}

int pt_gen_chandra(int32_t n, double c, pt_prec prec, pt_sysbuf** out) {
  if (n < 1 || !out) return PT_E_INVAL;
  switch (prec) {
    case PT_D: *out = chandra<double>(n, c); break;
    case PT_DD: *out = chandra<ptk::dd>(n, c); break;
    case PT_QD: *out = chandra<ptk::qd>(n, c); break;
    default: return PT_E_INVAL;
  }
  return PT_OK;
}

// n equations sharing one random support of n_monomials distinct monomials
// of total degree `degree` (variables drawn with replacement via bits() % n)
// plus a constant; coefficients Rng::box, equation by equation, constant
// first then monomials in canonical order.
int pt_gen_random_dense(int32_t n, int32_t degree, int32_t n_monomials, uint64_t seed, pt_prec prec,
                        pt_sysbuf** out) {
  if (n < 1 || degree < 1 || n_monomials < 1 || !out) return PT_E_INVAL;
  const int L = limbs(prec);
  Rng rng(seed);
  std::set<Support> seen;
  std::vector<Support> sups;
  long guard = 0;
  while ((int)sups.size() < n_monomials) {
    if (++guard > 100L * n_monomials + 1000) return PT_E_INVAL;  // support space too small
    std::map<int, int> ex;
    for (int d = 0; d < degree; ++d) ex[(int)(rng.bits() % (uint64_t)n)] += 1;
    Support s(ex.begin(), ex.end());
    if (seen.insert(s).second) sups.push_back(s);
  }
  std::sort(sups.begin(), sups.end());
  std::vector<std::vector<Term>> eqs(n);
  for (int i = 0; i < n; ++i) {
    const double re0 = rng.uniform(-1.0, 1.0), im0 = rng.uniform(-1.0, 1.0);
    eqs[i].push_back(make_term({}, re0, im0, L));
    for (auto& s : sups) {
      const double re = rng.uniform(-1.0, 1.0), im = rng.uniform(-1.0, 1.0);
      eqs[i].push_back(make_term(s, re, im, L));
    }
  }
  *out = emit(n, eqs, L);
  return PT_OK;
}

int pt_gen_total_degree(int32_t n, int32_t degree, pt_prec prec, pt_sysbuf** out) {
  if (n < 1 || degree < 1 || !out) return PT_E_INVAL;
  const int L = limbs(prec);
  std::vector<std::vector<Term>> eqs(n);
  for (int i = 0; i < n; ++i) {
    eqs[i].push_back(make_term({}, -1.0, 0.0, L));
    eqs[i].push_back(make_term({{i, degree}}, 1.0, 0.0, L));
  }
  *out = emit(n, eqs, L);
  return PT_OK;
}

int pt_sysbuf_desc(const pt_sysbuf* s, pt_system_desc* d) {
  if (!s || !d) return PT_E_INVAL;
  d->n_vars = s->n_vars;
  d->n_eqs = s->n_eqs;
  d->n_terms = (int32_t)s->term_ptr.size() - 1;
  d->eq_ptr = s->eq_ptr.data();
  d->term_ptr = s->term_ptr.data();
  d->var = s->var.data();
  d->exp = s->exp.data();
  d->coef = s->coef.data();
  return PT_OK;
}

void pt_sysbuf_free(pt_sysbuf* s) { delete s; }

int pt_gen_unit_complex(double theta, pt_prec prec, double* out) {
  if (!out) return PT_E_INVAL;
  switch (prec) {
    case PT_D: unit_out<double>(theta, out); break;
    case PT_DD: unit_out<ptk::dd>(theta, out); break;
    case PT_QD: unit_out<ptk::qd>(theta, out); break;
    default: return PT_E_INVAL;
  }
  return PT_OK;
}

int pt_gen_gamma(uint64_t seed, pt_prec prec, double* out) {
  Rng rng(seed);
  return pt_gen_unit_complex(rng.angle(), prec, out);
}

}  // extern "C"
