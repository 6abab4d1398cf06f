// pathtrack_b200.hpp -- header-only C++ adapter from the reference's types
// (pathtrack::Complex<Real>, pathtrack::Point<Real>, RealTraits<Real>;
// /root/reference/proj/include/pathtrack/{multiprec,complex}.hpp) to the
// C-ABI in pathtrack_b200.h.  This is the binding a maintainer adds next to
// the reference headers: include it after "pathtrack/complex.hpp" and call
// pathtrack::b200::track_path(...) where SPEC.md:466 calls track_path(...).
//
// Limbs cross the ABI exactly as RealTraits<Real>::components() returns them
// (multiprec.hpp:393,406,421) and come back through from_components(), so a
// Point<DoubleDouble> round-trips bit for bit.  Errors are rethrown with the
// reference's exception classes: std::invalid_argument for bad input,
// std::runtime_error for device problems (precision.cpp:39-43 style).
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "pathtrack_b200.h"

namespace pathtrack::b200 {

template <class Real>
constexpr pt_prec prec_of() {
  constexpr int L = RealTraits<Real>::limbs;
  return L == 1 ? PT_D : (L == 2 ? PT_DD : PT_QD);
}

inline void check(int rc) {
  if (rc == PT_OK) return;
  const std::string msg = std::string("pathtrack_b200: ") + pt_last_error();
  if (rc == PT_E_INVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// SoA limb buffer of a Point<Real>: re limbs then im limbs (pathtrack_b200.h)
template <class Real>
std::vector<double> to_limbs(const Point<Real>& x) {
  constexpr int L = RealTraits<Real>::limbs;
  const size_t n = x.size();
  std::vector<double> out(2 * L * n);
  for (size_t i = 0; i < n; ++i) {
    auto re = RealTraits<Real>::components(x[i].re);
    auto im = RealTraits<Real>::components(x[i].im);
    for (int l = 0; l < L; ++l) {
      out[l * n + i] = re[l];
      out[(L + l) * n + i] = im[l];
    }
  }
  return out;
}

template <class Real>
Point<Real> from_limbs(const std::vector<double>& v, size_t n) {
  constexpr int L = RealTraits<Real>::limbs;
  Point<Real> x(n);
  double re[4], im[4];
  for (size_t i = 0; i < n; ++i) {
    for (int l = 0; l < L; ++l) {
      re[l] = v[l * n + i];
      im[l] = v[(L + l) * n + i];
    }
    // limbs are already a valid expansion: rebuild without re-rounding
    if constexpr (L == 1) {
      x[i] = Complex<Real>(re[0], im[0]);
    } else if constexpr (L == 2) {
      x[i] = Complex<Real>(Real(re[0], re[1]), Real(im[0], im[1]));
    } else {
      x[i] = Complex<Real>(Real(re[0], re[1], re[2], re[3]), Real(im[0], im[1], im[2], im[3]));
    }
  }
  return x;
}

// One polynomial system in the canonical form of SPEC.md:129-136,150.
template <class Real>
struct System {
  int n_vars = 0;
  std::vector<int32_t> eq_ptr{0, 0}, term_ptr{0}, var, exp;  // one open equation: [start, running end]
  std::vector<Complex<Real>> coef;

  // add one term (support: (var, exp) with var ascending) to the last equation
  void term(const std::vector<std::pair<int, int>>& support, const Complex<Real>& c) {
    for (auto [v, e] : support) {
      var.push_back(v);
      exp.push_back(e);
    }
    term_ptr.push_back((int32_t)var.size());
    coef.push_back(c);
    eq_ptr.back() = (int32_t)coef.size();
  }
  void next_equation() { eq_ptr.push_back((int32_t)coef.size()); }

  // pt_system_desc view; `limbs` keeps the SoA coefficient buffer alive
  pt_system_desc desc(std::vector<double>& limbs) const {
    limbs = to_limbs<Real>(coef);
    pt_system_desc d{};
    d.n_vars = n_vars;
    d.n_eqs = (int32_t)eq_ptr.size() - 1;
    d.n_terms = (int32_t)coef.size();
    d.eq_ptr = eq_ptr.data();
    d.term_ptr = term_ptr.data();
    d.var = var.data();
    d.exp = exp.data();
    d.coef = limbs.data();
    return d;
  }
};

template <class Real>
struct TrackOutcome {
  bool success = false;
  Point<Real> end;
  pt_path_stats stats{};
};

// make_homotopy + compile_plan on one device.
template <class Real>
class Homotopy {
 public:
  Homotopy(const System<Real>& g, const System<Real>& f, const Complex<Real>& gamma, int k = 2, int device = 0)
      : n_(g.n_vars) {
    std::vector<double> gl, fl;
    const pt_system_desc gd = g.desc(gl), fd = f.desc(fl);
    std::vector<double> gam = to_limbs<Real>(Point<Real>{gamma});
    check(pt_plan_create(device, prec_of<Real>(), &gd, &fd, gam.data(), k, &plan_));
  }
  ~Homotopy() { pt_plan_destroy(plan_); }
  Homotopy(const Homotopy&) = delete;
  Homotopy& operator=(const Homotopy&) = delete;

  // track_path
  TrackOutcome<Real> track_path(const Point<Real>& start, const pt_step_params* params = nullptr) const {
    pt_step_params p{};
    if (!params) {
      check(pt_default_params(prec_of<Real>(), &p));
      params = &p;
    }
    std::vector<double> in = to_limbs<Real>(start), out(in.size());
    TrackOutcome<Real> o;
    check(pt_track_path(plan_, in.data(), params, out.data(), &o.stats));
    o.success = o.stats.status == PT_PATH_SUCCESS;
    o.end = from_limbs<Real>(out, n_);
    return o;
  }

  // Many independent paths (one tracker per path), one CTA
  // per path on the device (pt_track_batch): outcome p belongs to starts[p].
  std::vector<TrackOutcome<Real>> track_batch(const std::vector<Point<Real>>& starts,
                                              const pt_step_params* params = nullptr) const {
    pt_step_params p{};
    if (!params) {
      check(pt_default_params(prec_of<Real>(), &p));
      params = &p;
    }
    std::vector<double> in;
    for (const auto& s : starts) {
      const std::vector<double> l = to_limbs<Real>(s);
      in.insert(in.end(), l.begin(), l.end());
    }
    std::vector<double> out(in.size());
    std::vector<pt_path_stats> st(starts.size());
    if (!starts.empty()) check(pt_track_batch(plan_, (int32_t)starts.size(), in.data(), params, out.data(), st.data()));
    std::vector<TrackOutcome<Real>> res(starts.size());
    const size_t per = starts.empty() ? 0 : in.size() / starts.size();
    for (size_t q = 0; q < starts.size(); ++q) {
      res[q].stats = st[q];
      res[q].success = st[q].status == PT_PATH_SUCCESS;
      res[q].end = from_limbs<Real>(std::vector<double>(out.begin() + q * per, out.begin() + (q + 1) * per), n_);
    }
    return res;
  }

  // QD only: opt into the tolerance-parity arithmetic (pt_plan_set_arith).
  void set_fast_arithmetic(bool fast) { check(pt_plan_set_arith(plan_, fast ? PT_ARITH_FAST : PT_ARITH_REFERENCE)); }

  pt_plan* plan() const { return plan_; }

 private:
  pt_plan* plan_ = nullptr;
  size_t n_;
};

}  // namespace pathtrack::b200
