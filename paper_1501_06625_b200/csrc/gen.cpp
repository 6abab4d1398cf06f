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
#include <cstdlib>
#include <vector>

#include "inputs.hpp"

namespace ptgen {

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

const char* pt_inputs_last_error(void) { return g_err.c_str(); }
void pt_text_free(char* text) { std::free(text); }

int pt_sysbuf_from_desc(const pt_system_desc* d, pt_prec prec, pt_sysbuf** out) {
  if (!d || !out || d->n_vars < 0 || d->n_eqs < 0 || d->n_terms < 0) return fail(PT_E_INVAL, "bad system descriptor");
  pt_sysbuf tmp;
  tmp.n_vars = d->n_vars;
  tmp.n_eqs = d->n_eqs;
  tmp.L = limbs(prec);
  tmp.eq_ptr.assign(d->eq_ptr, d->eq_ptr + d->n_eqs + 1);
  tmp.term_ptr.assign(d->term_ptr, d->term_ptr + d->n_terms + 1);
  const int V = tmp.term_ptr.back();
  tmp.var.assign(d->var, d->var + V);
  tmp.exp.assign(d->exp, d->exp + V);
  tmp.coef.assign(d->coef, d->coef + (size_t)2 * tmp.L * d->n_terms);
  for (int q = 0; q < V; ++q)
    if (tmp.var[q] < 0 || tmp.var[q] >= d->n_vars || tmp.exp[q] < 1) return fail(PT_E_INVAL, "bad term support");
  auto eqs = terms_of(tmp);
  canonicalize(eqs, tmp.L);
  *out = emit(d->n_vars, eqs, tmp.L);
  return PT_OK;
}

int pt_sysbuf_stack(const pt_sysbuf* a, const pt_sysbuf* b, pt_sysbuf** out) {
  if (!a || !b || !out || a->n_vars != b->n_vars || a->L != b->L) return fail(PT_E_INVAL, "cannot stack systems");
  auto ea = terms_of(*a), eb = terms_of(*b);
  ea.insert(ea.end(), eb.begin(), eb.end());
  *out = emit(a->n_vars, ea, a->L);
  return PT_OK;
}

// Table 5: n = l m^2, m >= 2 maximal, l squarefree;
// dimension m - 1, degree m.
int pt_cyclic_degree(int32_t n, int32_t* m, int32_t* l, int32_t* dim, int32_t* degree) {
  if (n < 1) return fail(PT_E_INVAL, "n must be >= 1");
  int best = 1;
  for (int q = 2; (long)q * q <= n; ++q)
    if (n % (q * q) == 0) best = q;
  if (best < 2) return 0;
  int rest = n / (best * best);
  for (int q = 2; (long)q * q <= rest; ++q)
    if (rest % (q * q) == 0) return 0;  // unreachable for maximal m, kept for clarity
  if (m) *m = best;
  if (l) *l = rest;
  if (dim) *dim = best - 1;
  if (degree) *degree = best;
  return 1;
}

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
