// pieri.cpp -- Pieri homotopy inputs (PAPER.md 4.1, Eqs. 7-8).
//
// X_k is the n x p localization pattern of stage k (n = m + p): column j
// (0-based) has its pivot 1 at row j, zeros above, and variables at rows
// j+1 .. j+m introduced rightmost column first, top to bottom (the paper's
// n = 4 sequence x_{3,2}, x_{4,2}, x_{2,1}, x_{3,1} generalised, SPEC.md
// "DESIGN DECISIONS"); stage k holds the first k of those m p variables.
//
//   minor_expand(A, X_k)   det([A | X_k]) by Laplace expansion over the X
//                          columns: sum over p-row subsets R of
//                          (-1)^(sum R + sum Xcols) det(X_k[R,:]) det(A[R^c,:]),
//                          det(X_k[R,:]) expanded by permutations (entries 1,
//                          0 or one variable), the complementary m x m minors
//                          of A by complex Gaussian elimination in the
//                          working precision; canonical form afterwards.
//   choose_special_matrix  first S_X (standard basis columns, then sums of
//                          two basis vectors), deterministic order, with
//                          det([S_X | X_k(x0)]) == 0 and a nonzero cofactor
//                          of the new variable at the start point x0.
#include <cmath>
#include <type_traits>
#include <cstdlib>
#include <vector>

#include "inputs.hpp"

using namespace ptgen;

namespace {

int n_of(int m, int p) { return m + p; }

void events(int m, int p, std::vector<int>& rows, std::vector<int>& cols) {
  rows.clear();
  cols.clear();
  for (int j = p - 1; j >= 0; --j)
    for (int r = j + 1; r <= j + m; ++r) {
      rows.push_back(r);
      cols.push_back(j);
    }
}

// X_k entry kinds: -1 zero, -2 one, v >= 0 variable v
std::vector<int> pattern(int m, int p, int k) {
  const int n = n_of(m, p);
  std::vector<int> X((size_t)n * p, -1);
  for (int j = 0; j < p; ++j) X[(size_t)j * n + j] = -2;
  std::vector<int> rows, cols;
  events(m, p, rows, cols);
  for (int v = 0; v < k; ++v) X[(size_t)cols[v] * n + rows[v]] = v;
  return X;
}

template <class R>
using C = ptk::cplx<R>;

template <class R>
C<R> ld(const double* a, long S, long i) {
  return ptk::load_c<R>(a, S, i);
}

template <class R>
C<R> cdiv(const C<R>& a, const C<R>& b) {  // a conj(b) / |b|^2
  using namespace ptk;
  const R d = c_norm_sqr(b);
  const C<R> num = c_mul(a, C<R>{b.re, r_neg(b.im)});
  return {r_div(num.re, d), r_div(num.im, d)};
}

// determinant of a k x k complex matrix (column-major, row stride k) by
// Gaussian elimination with partial pivoting on modulus_double
template <class R>
C<R> det(std::vector<C<R>> M, int k) {
  using namespace ptk;
  C<R> d = c_one<R>();
  for (int c = 0; c < k; ++c) {
    int piv = c;
    double best = -1.0;
    for (int r = c; r < k; ++r) {
      const double v = c_mod_double(M[(size_t)c * k + r]);
      if (v > best) {
        best = v;
        piv = r;
      }
    }
    if (!(best > 0.0)) return c_zero<R>();
    if (piv != c) {
      for (int j = 0; j < k; ++j) std::swap(M[(size_t)j * k + c], M[(size_t)j * k + piv]);
      d = c_neg(d);
    }
    const C<R> pv = M[(size_t)c * k + c];
    d = c_mul(d, pv);
    for (int r = c + 1; r < k; ++r) {
      const C<R> f = cdiv(M[(size_t)c * k + r], pv);
      if (c_is_zero(f)) continue;
      for (int j = c + 1; j < k; ++j) M[(size_t)j * k + r] = c_sub(M[(size_t)j * k + r], c_mul(f, M[(size_t)j * k + c]));
    }
  }
  return d;
}

// numeric [A | X_k(x)] (n x n, column-major); A: n x m SoA (S = n m)
template <class R>
std::vector<C<R>> full_matrix(int m, int p, int k, const double* A, const double* x, const std::vector<int>* Xpat = nullptr) {
  using namespace ptk;
  const int n = n_of(m, p);
  std::vector<C<R>> M((size_t)n * n);
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < n; ++r) M[(size_t)c * n + r] = ld<R>(A, (long)n * m, (long)c * n + r);
  const std::vector<int> X = Xpat ? *Xpat : pattern(m, p, k);
  for (int j = 0; j < p; ++j)
    for (int r = 0; r < n; ++r) {
      const int e = X[(size_t)j * n + r];
      M[(size_t)(m + j) * n + r] = e == -1 ? c_zero<R>() : (e == -2 ? c_one<R>() : ld<R>(x, k, e));
    }
  return M;
}

template <class R>
int minor_expand(int m, int p, int k, const double* A, pt_sysbuf** out) {
  using namespace ptk;
  constexpr int L = limbs_of<R>::L;
  const int n = n_of(m, p);
  const std::vector<int> X = pattern(m, p, k);
  std::vector<Term> terms;
  std::vector<int> Rr(p), perm(p);
  // p-row subsets in lexicographic order
  for (int i = 0; i < p; ++i) Rr[i] = i;
  const int xcol_sum = [&] {
    int s = 0;
    for (int c = m; c < n; ++c) s += c + 1;
    return s;
  }();
  while (true) {
    // det(X[R,:]) by permutations: list of (sign, variables)
    std::vector<std::pair<int, std::vector<int>>> xt;
    for (int i = 0; i < p; ++i) perm[i] = i;
    do {
      int sgn = 1;
      for (int a = 0; a < p; ++a)
        for (int b = a + 1; b < p; ++b)
          if (perm[a] > perm[b]) sgn = -sgn;
      std::vector<int> vars;
      bool zero = false;
      for (int a = 0; a < p && !zero; ++a) {
        const int e = X[(size_t)perm[a] * n + Rr[a]];
        if (e == -1) zero = true;
        else if (e >= 0) vars.push_back(e);
      }
      if (!zero) xt.push_back({sgn, vars});
    } while (std::next_permutation(perm.begin(), perm.end()));
    if (!xt.empty()) {
      int rsum = 0;
      std::vector<char> inR(n, 0);
      for (int a = 0; a < p; ++a) {
        rsum += Rr[a] + 1;
        inR[Rr[a]] = 1;
      }
      // complementary minor of A: rows not in R, all m columns
      std::vector<C<R>> Am((size_t)m * m);
      int rr = 0;
      for (int r = 0; r < n; ++r) {
        if (inR[r]) continue;
        for (int c = 0; c < m; ++c) Am[(size_t)c * m + rr] = ld<R>(A, (long)n * m, (long)c * n + r);
        ++rr;
      }
      C<R> am = m > 0 ? det<R>(Am, m) : c_one<R>();
      if (((rsum + xcol_sum) & 1) != 0) am = c_neg(am);
      for (auto& [sgn, vars] : xt) {
        Term t;
        std::memset(t.c, 0, sizeof t.c);
        std::sort(vars.begin(), vars.end());
        for (int v : vars) t.sup.push_back({v, 1});
        put<R>(t, sgn > 0 ? am : c_neg(am));
        terms.push_back(t);
      }
    }
    // next subset
    int i = p - 1;
    while (i >= 0 && Rr[i] == n - p + i) --i;
    if (i < 0) break;
    ++Rr[i];
    for (int j = i + 1; j < p; ++j) Rr[j] = Rr[j - 1] + 1;
  }
  std::vector<std::vector<Term>> eqs(1, terms);
  canonicalize(eqs, L);
  *out = emit(k, eqs, L);
  return PT_OK;
}

template <class R>
void store(const C<R>& v, double* out) {
  constexpr int L = ptk::limbs_of<R>::L;
  for (int l = 0; l < L; ++l) {
    out[l] = ptk::r_limb(v.re, l);
    out[L + l] = ptk::r_limb(v.im, l);
  }
}

template <class R>
int special(int m, int p, int k, const double* x, double* S) {
  using namespace ptk;
  constexpr int L = limbs_of<R>::L;
  const int n = n_of(m, p);
  std::vector<int> rows, cols;
  events(m, p, rows, cols);
  const int nv = k - 1, vr = rows[nv], vc = cols[nv];  // the new variable's entry of X
  // candidate columns: e_i, then e_i + e_j (i < j)
  std::vector<std::vector<int>> cand;
  for (int i = 0; i < n; ++i) cand.push_back({i});
  const size_t nbasis = cand.size();
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) cand.push_back({i, j});
  std::vector<double> Sbuf((size_t)2 * L * n * m);
  auto build = [&](const std::vector<int>& pick) {
    std::fill(Sbuf.begin(), Sbuf.end(), 0.0);
    for (int c = 0; c < m; ++c)
      for (int r : cand[pick[c]]) Sbuf[(size_t)c * n + r] = 1.0;  // re limb 0 of entry (r, c)
  };
  std::vector<int> X = pattern(m, p, k);
  for (int phase = 0; phase < 2; ++phase) {
    const int lo = 0, hi = phase == 0 ? (int)nbasis : (int)cand.size();
    std::vector<int> pick(m);
    for (int c = 0; c < m; ++c) pick[c] = lo + c;
    if (hi - lo < m) continue;
    while (true) {
      bool fresh = phase == 0 || pick[m - 1] >= (int)nbasis;  // phase 1: at least one sum column
      if (fresh) {
        build(pick);
        const C<R> d0 = det<R>(full_matrix<R>(m, p, k, Sbuf.data(), x, &X), n);
        // cofactor of entry (vr, vc) of X: replace that column by e_vr
        std::vector<int> Xd = X;
        for (int r = 0; r < n; ++r) Xd[(size_t)vc * n + r] = -1;
        Xd[(size_t)vc * n + vr] = -2;
        const C<R> d1 = det<R>(full_matrix<R>(m, p, k, Sbuf.data(), x, &Xd), n);
        if (c_mod_double(d0) <= 1e-12 && c_mod_double(d1) > 1e-6) {
          std::copy(Sbuf.begin(), Sbuf.end(), S);
          return PT_OK;
        }
      }
      int i = m - 1;
      while (i >= 0 && pick[i] == hi - m + i) --i;
      if (i < 0) break;
      ++pick[i];
      for (int j = i + 1; j < m; ++j) pick[j] = pick[j - 1] + 1;
    }
  }
  return fail(PT_E_INVAL, "choose_special_matrix: no qualifying S_X (search exhausted)");
}

template <class R>
int det_at(int m, int p, int k, const double* A, const double* x, double* out) {
  store<R>(det<R>(full_matrix<R>(m, p, k, A, x), n_of(m, p)), out);
  return PT_OK;
}

// Stage 1: det([A | X_1(v)]) = a v + b is linear in its one variable:
// v = -b / a with b = det at v = 0, a = det at v = 1 minus b.
template <class R>
int linear_start(int m, int p, const double* A, double* out) {
  using namespace ptk;
  constexpr int L = limbs_of<R>::L;
  double x0[2 * L] = {}, x1[2 * L] = {};
  x1[0] = 1.0;
  const int n = n_of(m, p);
  const C<R> b = det<R>(full_matrix<R>(m, p, 1, A, x0), n);
  const C<R> a = c_sub(det<R>(full_matrix<R>(m, p, 1, A, x1), n), b);
  if (c_is_zero(a)) return fail(PT_E_INVAL, "first Pieri stage is degenerate (zero linear coefficient)");
  store<R>(c_neg(cdiv(b, a)), out);
  return PT_OK;
}

template <class F>
int by_prec(pt_prec prec, F&& f) {
  switch (prec) {
    case PT_D: return f((double*)nullptr);
    case PT_DD: return f((ptk::dd*)nullptr);
    case PT_QD: return f((ptk::qd*)nullptr);
  }
  return fail(PT_E_INVAL, "bad precision");
}

bool bad_mp(int m, int p) { return m < 1 || p < 1 || m + p > 64; }

}  // namespace

extern "C" {

int pt_pieri_events(int32_t m, int32_t p, int32_t* rows, int32_t* cols) {
  if (bad_mp(m, p) || !rows || !cols) return fail(PT_E_INVAL, "need m, p >= 1, m + p <= 64");
  std::vector<int> r, c;
  events(m, p, r, c);
  for (size_t e = 0; e < r.size(); ++e) {
    rows[e] = r[e];
    cols[e] = c[e];
  }
  return PT_OK;
}

int pt_pieri_planes(int32_t m, int32_t p, int32_t count, uint64_t seed, pt_prec prec, double* out) {
  if (bad_mp(m, p) || count < 0 || !out) return fail(PT_E_INVAL, "bad Pieri plane arguments");
  const int L = limbs(prec), n = m + p;
  const long S = (long)n * m;
  Rng rng(seed);
  for (int i = 0; i < count; ++i) {
    double* A = out + (size_t)i * 2 * L * S;
    std::fill(A, A + 2 * L * S, 0.0);
    for (long e = 0; e < S; ++e) {  // column by column: entry (r, c) at c n + r
      A[e] = rng.uniform(-1.0, 1.0);
      A[L * S + e] = rng.uniform(-1.0, 1.0);
    }
  }
  return PT_OK;
}

int pt_pieri_minor(int32_t m, int32_t p, int32_t k, const double* A, pt_prec prec, pt_sysbuf** out) {
  if (bad_mp(m, p) || k < 0 || k > m * p || !A || !out) return fail(PT_E_INVAL, "bad Pieri minor arguments");
  return by_prec(prec, [&](auto* tag) {
    using R = std::remove_pointer_t<decltype(tag)>;
    return minor_expand<R>(m, p, k, A, out);
  });
}

int pt_pieri_det(int32_t m, int32_t p, int32_t k, const double* A, const double* x, pt_prec prec, double* out) {
  if (bad_mp(m, p) || k < 0 || k > m * p || !A || (k > 0 && !x) || !out)
    return fail(PT_E_INVAL, "bad Pieri det arguments");
  return by_prec(prec, [&](auto* tag) {
    using R = std::remove_pointer_t<decltype(tag)>;
    return det_at<R>(m, p, k, A, x, out);
  });
}

int pt_pieri_linear_start(int32_t m, int32_t p, const double* A, pt_prec prec, double* x) {
  if (bad_mp(m, p) || !A || !x) return fail(PT_E_INVAL, "bad Pieri start arguments");
  return by_prec(prec, [&](auto* tag) {
    using R = std::remove_pointer_t<decltype(tag)>;
    return linear_start<R>(m, p, A, x);
  });
}

int pt_pieri_special(int32_t m, int32_t p, int32_t k, const double* x, pt_prec prec, double* S) {
  if (bad_mp(m, p) || k < 1 || k > m * p || !x || !S) return fail(PT_E_INVAL, "bad special-matrix arguments");
  return by_prec(prec, [&](auto* tag) {
    using R = std::remove_pointer_t<decltype(tag)>;
    return special<R>(m, p, k, x, S);
  });
}

}  // extern "C"
