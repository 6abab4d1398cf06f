// orc_tracker.hpp -- TEST INFRASTRUCTURE (CPU oracle), not product code.
//
// CPU restatement of the single-path tracker the reference specifies but does
// not implement (SURVEY.md finding 0.2).  It follows /root/reference/SPEC.md:
//   polysys   SPEC.md:124-202   (homotopy_weights :174-182)
//   evaldiff  SPEC.md:204-279   (reverse mode :231-239, Table 1 = PAPER.md:458-497)
//   linalg    SPEC.md:281-350   (MGS :296-304, lstsq :314-322, max_modulus :323-331)
//   newton    SPEC.md:352-393   (Fig. 2 = PAPER.md:290-321)
//   predictor SPEC.md:395-441
//   tracker   SPEC.md:443-504   (Fig. 3 = PAPER.md:374-407)
// The scalar arithmetic comes either from orc_arith.hpp (restatement) or, for
// the _ref build, from the unmodified reference headers.
//
// Every place where SPEC.md leaves an order or a tie-break to the implementer
// is pinned here and in DESIGN.md section 3 ("Pinned semantics"); the CUDA
// path implements the same pins, which is what makes the comparison bitwise.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
// --impl reference) may load this code.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <vector>

#ifdef ORC_USE_REFERENCE
#include <vector>  // complex.hpp:156 uses std::vector without including it
#include "pathtrack/complex.hpp"
#include "pathtrack/multiprec.hpp"
namespace A = pathtrack;
#else
#include "orc_arith.hpp"
namespace A = orc;
#endif

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc_track {

struct SystemDesc {  // same layout as pt_system_desc (include/pathtrack_b200.h)
  int32_t n_vars, n_eqs, n_terms;
  const int32_t* eq_ptr;
  const int32_t* term_ptr;
  const int32_t* var;
  const int32_t* exp;
  const double* coef;  // [2][L][n_terms]
};

struct StepParams {  // same layout as pt_step_params
  double max_step, min_step;
  int32_t max_steps, pred_degree, newton_max_iter, reserved;
  double newton_tol;
};

struct PathStats {  // same layout as pt_path_stats
  int32_t status, failure_kind, steps, accepted, newton_iters, start_iters, solves, reserved;
  double final_residual, final_update, t_end;
};

struct TraceEvent {  // same layout as pt_trace_event
  double t;
  int32_t ok, iters;
  double residual, update;
};

enum { ST_SUCCESS = 0, ST_FAIL = 1 };
enum { FK_NONE = 0, FK_START = 1, FK_MAX_STEPS = 2, FK_MIN_STEP = 3 };
enum { NW_OK = 0, NW_RESIDUAL_INCREASE = 1, NW_ITERATION_BUDGET = 2, NW_LINEAR_SOLVE = 3 };

// ---------------------------------------------------------------------------
// Canonical fixed-shape summation ("fixed reduction tree").
// P partials (P a power of two): partial p = c[p] + c[p+P] + ... left to
// right; then for off = P/2 .. 1: partial[p] += partial[p+off] for p < off
// whenever p+off < K (empty partials are skipped, never added as zeros).
// K == 0 is handled by the caller (structural zero).
// ---------------------------------------------------------------------------
inline int pow2ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
inline int width_eval(int K) { return std::min(256, std::max(32, pow2ceil((K + 15) / 16))); }
inline int width_mgs(int N) { return std::min(256, std::max(32, pow2ceil((N + 1) / 2))); }

template <class T, class Get>
T canon_sum(int K, int P, Get get) {
  std::vector<T> part(std::min(P, K));
  for (int p = 0; p < P && p < K; ++p) {
    T acc = get(p);
    for (int r = p + P; r < K; r += P) acc = acc + get(r);
    part[p] = acc;
  }
  for (int off = P / 2; off >= 1; off /= 2)
    for (int p = 0; p < off; ++p)
      if (p + off < K) part[p] = part[p] + part[p + off];
  return part[0];
}

// NaN-propagating max of binary64 norms (pinned reading of max_modulus,
// empty -> 0, any NaN -> NaN).
inline double nan_max(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return std::numeric_limits<double>::quiet_NaN();
  return b > a ? b : a;
}

template <class R>
struct Tracker {
  using C = A::Complex<R>;
  static constexpr int L = A::RealTraits<R>::limbs;

  struct Mono {
    std::vector<int> v, e;
    bool pow = false;
  };
  struct Term {
    int mono;  // -1: constant term
    C coef;
  };
  struct Contrib {
    int term;  // index into the equation's term list
    int k;     // -1: monomial value; >= 0: partial w.r.t. the k-th support variable
  };

  int n = 0, N = 0;
  std::vector<Mono> monos;
  std::vector<std::vector<Term>> eq[2];
  // slot lists: sl[s][i][j], j in [0, n] (j == n is the value slot)
  std::vector<std::vector<std::vector<Contrib>>> sl[2];
  std::vector<char> shared;  // equation i identical in g and f
  C gamma;
  int relax_k = 2;
  double sqrt_eps = std::sqrt(A::RealTraits<R>::epsilon);

  static R real_from_limbs(const double* p, long stride, long i) {
    double l[4];
    for (int q = 0; q < L; ++q) l[q] = p[q * stride + i];
    return limbs_to_real(l);
  }
  static R real_sqrt(const R& v) {
    if constexpr (L == 1) {
      return std::sqrt(v);
    } else {
      return A::sqrt(v);
    }
  }
  static R limbs_to_real(const double* l) {
    if constexpr (L == 1) {
      return l[0];
    } else if constexpr (L == 2) {
      return R(l[0], l[1]);
    } else {
      return R(l[0], l[1], l[2], l[3]);
    }
  }
  static void real_to_limbs(const R& r, double* out) {
    auto c = A::RealTraits<R>::components(r);
    for (int q = 0; q < L; ++q) out[q] = c[q];
  }
  static C load_c(const double* p, long S, long i) {
    return C(real_from_limbs(p, S, i), real_from_limbs(p + (long)L * S, S, i));
  }
  static void store_c(double* p, long S, long i, const C& v) {
    double l[4];
    real_to_limbs(v.re, l);
    for (int q = 0; q < L; ++q) p[q * S + i] = l[q];
    real_to_limbs(v.im, l);
    for (int q = 0; q < L; ++q) p[(L + q) * S + i] = l[q];
  }

  // compile_plan: deduplicate supports, build per-slot
  // contribution lists in term order.
  void build(const SystemDesc& g, const SystemDesc& f, const double* gamma_limbs, int k) {
    n = g.n_vars;
    N = g.n_eqs;
    relax_k = k;
    gamma = C(limbs_to_real(gamma_limbs), limbs_to_real(gamma_limbs + L));
    std::map<std::pair<std::vector<int>, std::vector<int>>, int> index;
    const SystemDesc* sys[2] = {&g, &f};
    for (int s = 0; s < 2; ++s) {
      const SystemDesc& d = *sys[s];
      eq[s].assign(N, {});
      sl[s].assign(N, std::vector<std::vector<Contrib>>(n + 1));
      for (int i = 0; i < N; ++i) {
        for (int t = d.eq_ptr[i]; t < d.eq_ptr[i + 1]; ++t) {
          Term term;
          term.coef = load_c(d.coef, d.n_terms, t);
          std::vector<int> vv(d.var + d.term_ptr[t], d.var + d.term_ptr[t + 1]);
          std::vector<int> ee(d.exp + d.term_ptr[t], d.exp + d.term_ptr[t + 1]);
          if (vv.empty()) {
            term.mono = -1;
          } else {
            auto key = std::make_pair(vv, ee);
            auto it = index.find(key);
            if (it == index.end()) {
              Mono m;
              m.v = vv;
              m.e = ee;
              for (int x : ee) m.pow = m.pow || x >= 2;
              it = index.emplace(key, (int)monos.size()).first;
              monos.push_back(m);
            }
            term.mono = it->second;
          }
          const int ti = (int)eq[s][i].size();
          eq[s][i].push_back(term);
          sl[s][i][n].push_back({ti, -1});
          for (int q = 0; q < (int)vv.size(); ++q) sl[s][i][vv[q]].push_back({ti, q});
        }
      }
    }
    shared.assign(N, 0);
    for (int i = 0; i < N; ++i) {
      const auto &a = eq[0][i], &b = eq[1][i];
      bool same = a.size() == b.size();
      for (size_t t = 0; same && t < a.size(); ++t) {
        same = a[t].mono == b[t].mono && bits_equal(a[t].coef, b[t].coef);
      }
      shared[i] = same;
    }
  }

  static bool bits_equal(const C& a, const C& b) {
    double x[8], y[8];
    real_to_limbs(a.re, x);
    real_to_limbs(a.im, x + L);
    real_to_limbs(b.re, y);
    real_to_limbs(b.im, y + L);
    return std::memcmp(x, y, sizeof(double) * 2 * L) == 0;
  }

  // eval_monomial_derivatives with the Table 1 scheme
  // (PAPER.md:458-497), 3m-5 products for m >= 3:
  //   F[0] = y0, F[k] = F[k-1]*y[k] (k = 1..m-2); value = F[m-2]*y[m-1];
  //   d[m-1] = F[m-2]; B = y[m-1];
  //   for k = m-2..1: d[k] = F[k-1]*B; B = y[k]*B;   d[0] = B.
  // m == 1: value = y0, d0 = 1.  m == 2: value = y0*y1, d0 = y1, d1 = y0.
  // Exponents: Cf = prod_{e_k>=2} y_k^(e_k-1) (powi, ascending
  // k, first factor is the initial value); value *= Cf; d[k] *= Cf, then
  // d[k] *= Real(e_k) when e_k >= 2.
  void eval_mono(const Mono& m, const std::vector<C>& x, C* out /* value, d0..d{m-1} */) const {
    const int sz = (int)m.v.size();
    C* d = out + 1;
    auto y = [&](int k) -> const C& { return x[m.v[k]]; };
    if (sz == 1) {
      out[0] = y(0);
      d[0] = C(R(1.0), R(0.0));
    } else if (sz == 2) {
      out[0] = y(0) * y(1);
      d[0] = y(1);
      d[1] = y(0);
    } else {
      std::vector<C> F(sz - 1);
      F[0] = y(0);
      for (int k = 1; k <= sz - 2; ++k) F[k] = F[k - 1] * y(k);
      out[0] = F[sz - 2] * y(sz - 1);
      d[sz - 1] = F[sz - 2];
      C B = y(sz - 1);
      for (int k = sz - 2; k >= 1; --k) {
        d[k] = F[k - 1] * B;
        B = y(k) * B;
      }
      d[0] = B;
    }
    if (m.pow) {
      C cf;
      bool have = false;
      for (int k = 0; k < sz; ++k) {
        if (m.e[k] < 2) continue;
        C pk = A::powi(y(k), (unsigned)(m.e[k] - 1));
        cf = have ? cf * pk : pk;
        have = true;
      }
      out[0] = out[0] * cf;
      for (int k = 0; k < sz; ++k) {
        d[k] = d[k] * cf;
        if (m.e[k] >= 2) d[k] = d[k] * R((double)m.e[k]);
      }
    }
  }

  // homotopy_weights: wS = gamma*(1-t)^k, wT = t^k.
  void weights(double t, C& wS, R& wT) const {
    const R omt = R(1.0) - R(t);
    const R a = A::powi(omt, (unsigned)relax_k);
    wT = A::powi(R(t), (unsigned)relax_k);
    wS = gamma * a;
  }

  // evaluate_homotopy into the least-squares system
  // [J | -h] (column-major, N x (n+1)); returns max_modulus(h).
  // h_slot = wS*Sg + Sf*wT; a slot with no contributions in either system is
  // an exact zero; a side with no contributions enters as zero.
  double eval_homotopy(const std::vector<C>& x, double t, std::vector<C>& Amat) const {
    // monomial table
    std::vector<long> off(monos.size() + 1, 0);
    for (size_t q = 0; q < monos.size(); ++q) off[q + 1] = off[q] + 1 + (long)monos[q].v.size();
    std::vector<C> mv(off.back());
#pragma omp parallel for schedule(dynamic, 8)
    for (long q = 0; q < (long)monos.size(); ++q) eval_mono(monos[q], x, mv.data() + off[q]);
    C wS;
    R wT;
    weights(t, wS, wT);
    Amat.assign((size_t)N * (n + 1), C());
    std::vector<double> hmod(N, 0.0);
#pragma omp parallel for schedule(dynamic, 4) collapse(2)
    for (int i = 0; i < N; ++i) {
      for (int j = 0; j <= n; ++j) {
        C S[2];
        bool have[2] = {false, false};
        const int ns = shared[i] ? 1 : 2;
        for (int s = 0; s < ns; ++s) {
          const auto& lst = sl[s][i][j];
          const int K = (int)lst.size();
          if (K == 0) continue;
          have[s] = true;
          const auto& terms = eq[s][i];
          S[s] = canon_sum<C>(K, width_eval(K), [&](int r) -> C {
            const Contrib& cb = lst[r];
            const Term& tm = terms[cb.term];
            if (tm.mono < 0) return tm.coef;  // constant term: coefficient itself
            return tm.coef * mv[off[tm.mono] + 1 + cb.k];
          });
        }
        if (shared[i]) {
          S[1] = S[0];
          have[1] = have[0];
        }
        C h;
        if (have[0] || have[1]) {
          const C zero(R(0.0), R(0.0));
          const C& sg = have[0] ? S[0] : zero;
          const C& sf = have[1] ? S[1] : zero;
          h = wS * sg + sf * wT;
        } else {
          h = C(R(0.0), R(0.0));
        }
        if (j == n) {
          Amat[(size_t)n * N + i] = -h;
          hmod[i] = A::modulus_double(h);
        } else {
          Amat[(size_t)j * N + i] = h;
        }
      }
    }
    double r = 0.0;
    for (int i = 0; i < N; ++i) r = nan_max(r, hmod[i]);
    return r;
  }

  // least_squares_solve via column-sweep MGS on [A | b].
  // Pinned: norm^2 and q^H a are canonical sums of width width_mgs(N);
  // r_kk = sqrt(norm^2); rank test: !(r_kk > sqrt(eps) * max_{k'<=k} r_k'k')
  // in binary64; q_k = a_k * (1/r_kk); a_j -= r_kj * q_k;
  // back substitution x_k = (y_k - sum_{j=n-1..k+1} r_kj x_j) * (1/r_kk),
  // subtracting in descending j.
  bool lstsq(std::vector<C>& Amat, std::vector<C>& dx) const {
    const int P = width_mgs(N);
    std::vector<C> Rm((size_t)n * (n + 1));
    std::vector<R> inv(n);
    double maxnorm = 0.0;
    bool ok = true;
    // one parallel region per factorisation (a fork/join per column cost more
    // than the columns of a 64 x 64 system): column k is normalised by one
    // thread, the updates j > k are shared; every column's arithmetic is the
    // same single-thread sequence, so the result does not depend on the team
#pragma omp parallel if ((long)N * n >= 1024)
    for (int k = 0; k < n; ++k) {
      C* ak = &Amat[(size_t)k * N];
#pragma omp single
      {
        const R nrm2 = canon_sum<R>(N, P, [&](int i) { return A::norm_sqr(ak[i]); });
        const R rkk = real_sqrt(nrm2);
        const double d = A::to_double(rkk);
        maxnorm = d > maxnorm ? d : maxnorm;
        if (!(d > sqrt_eps * maxnorm)) {
          ok = false;
        } else {
          inv[k] = R(1.0) / rkk;
          for (int i = 0; i < N; ++i) ak[i] = ak[i] * inv[k];
          Rm[(size_t)k * (n + 1) + k] = C(rkk, R(0.0));
        }
      }  // implicit barrier: ok, q_k and inv[k] visible to the team
      if (!ok) break;
#pragma omp for schedule(static)
      for (int j = k + 1; j <= n; ++j) {
        C* aj = &Amat[(size_t)j * N];
        const C rkj = canon_sum<C>(N, P, [&](int i) { return A::conj(ak[i]) * aj[i]; });
        Rm[(size_t)k * (n + 1) + j] = rkj;
        if (j < n || k < n - 1)
          for (int i = 0; i < N; ++i) aj[i] = aj[i] - rkj * ak[i];
      }  // implicit barrier
    }
    if (!ok) return false;
    dx.assign(n, C());
    for (int k = n - 1; k >= 0; --k) {
      C acc = Rm[(size_t)k * (n + 1) + n];
      for (int j = n - 1; j > k; --j) acc = acc - Rm[(size_t)k * (n + 1) + j] * dx[j];
      dx[k] = acc * inv[k];
    }
    return true;
  }

  struct NewtonOutcome {
    bool ok;
    int kind, iters;
    double residual, update;
    int solves;
  };

  // newton_correct, Fig. 2.
  NewtonOutcome newton(std::vector<C>& x, double t, const StepParams& P) const {
    NewtonOutcome o{false, NW_ITERATION_BUDGET, 0, -1.0, -1.0, 0};
    double last = std::numeric_limits<double>::infinity();
    std::vector<C> Amat, dx;
    for (int it = 1; it <= P.newton_max_iter; ++it) {
      o.iters = it;
      const double r = eval_homotopy(x, t, Amat);
      o.residual = r;
      if (r > last) {
        o.kind = NW_RESIDUAL_INCREASE;
        return o;
      }
      if (r < P.newton_tol) {
        o.ok = true;
        o.kind = NW_OK;
        return o;
      }
      if (!lstsq(Amat, dx)) {
        o.kind = NW_LINEAR_SOLVE;
        return o;
      }
      ++o.solves;
      double u = 0.0;
      for (int i = 0; i < n; ++i) u = nan_max(u, A::modulus_double(dx[i]));
      o.update = u;
      for (int i = 0; i < n; ++i) x[i] = x[i] + dx[i];
      if (u < P.newton_tol) {
        o.ok = true;
        o.kind = NW_OK;
        return o;
      }
      last = r;
    }
    o.kind = NW_ITERATION_BUDGET;
    return o;
  }

  // predict: Newton divided differences over the last
  // d+1 accepted points (t oldest..newest), Horner evaluation at tau.
  //   D[j] <- (D[j] - D[j-1]) * (1 / (R(t_j) - R(t_{j-l}))), j = d..l, l = 1..d
  //   p = D[d]; p = D[j] + p * (R(tau) - R(t_j)), j = d-1..0
  void predict(const std::vector<double>& ht, const std::vector<std::vector<C>>& hx, double tau,
               std::vector<C>& out) const {
    const int d = (int)ht.size() - 1;
    std::vector<R> inv((size_t)(d + 1) * (d + 1));
    for (int l = 1; l <= d; ++l)
      for (int j = d; j >= l; --j) inv[(size_t)l * (d + 1) + j] = R(1.0) / (R(ht[j]) - R(ht[j - l]));
    std::vector<R> dt(d + 1);
    for (int j = 0; j <= d; ++j) dt[j] = R(tau) - R(ht[j]);
    out.assign(n, C());
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
      C D[9];
      for (int j = 0; j <= d; ++j) D[j] = hx[j][i];
      for (int l = 1; l <= d; ++l)
        for (int j = d; j >= l; --j) D[j] = (D[j] - D[j - 1]) * inv[(size_t)l * (d + 1) + j];
      C p = D[d];
      for (int j = d - 1; j >= 0; --j) p = D[j] + p * dt[j];
      out[i] = p;
    }
  }

  // track_path, Fig. 3 with SPEC.md:466-495 decisions.
  void track(const std::vector<C>& start, const StepParams& P, std::vector<C>& end, PathStats& st,
             std::vector<TraceEvent>* trace) const {
    std::memset(&st, 0, sizeof st);
    std::vector<C> x = start;
    NewtonOutcome o = newton(x, 0.0, P);  // start validation
    st.start_iters = o.iters;
    st.newton_iters = o.iters;
    st.solves = o.solves;
    st.final_residual = o.residual;
    st.final_update = o.update;
    if (!o.ok) {
      st.status = ST_FAIL;
      st.failure_kind = FK_START;
      st.t_end = 0.0;
      end = x;
      return;
    }
    const int cap = P.pred_degree + 1;
    std::vector<double> ht{0.0};
    std::vector<std::vector<C>> hx{x};
    double tacc = 0.0, dt = P.max_step;
    int succ = 0, steps = 0, accepted = 0;
    std::vector<C> xp;
    while (tacc < 1.0) {
      if (steps > P.max_steps) {
        st.status = ST_FAIL;
        st.failure_kind = FK_MAX_STEPS;
        break;
      }
      const double tsum = tacc + dt;
      const double ttrial = tsum < 1.0 ? tsum : 1.0;  // std::min(1.0, t + dt)
      predict(ht, hx, ttrial, xp);
      o = newton(xp, ttrial, P);
      st.newton_iters += o.iters;
      st.solves += o.solves;
      st.final_residual = o.residual;
      st.final_update = o.update;
      if (trace) trace->push_back({ttrial, o.ok ? 1 : 0, o.iters, o.residual, o.update});
      ++steps;
      if (o.ok) {
        tacc = ttrial;
        x = xp;
        ht.push_back(ttrial);
        hx.push_back(x);
        if ((int)ht.size() > cap) {
          ht.erase(ht.begin());
          hx.erase(hx.begin());
        }
        ++accepted;
        ++succ;
        if (succ > 2) {
          const double two = 2.0 * dt;
          dt = P.max_step < two ? P.max_step : two;  // std::min(2*dt, max)
        }
      } else {
        succ = 0;
        dt = dt / 2.0;
        if (dt < P.min_step) {
          st.status = ST_FAIL;
          st.failure_kind = FK_MIN_STEP;
          break;
        }
      }
    }
    st.steps = steps;
    st.accepted = accepted;
    st.t_end = tacc;
    end = x;
  }
};

}  // namespace orc_track
