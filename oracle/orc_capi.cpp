// orc_capi.cpp -- TEST INFRASTRUCTURE (CPU oracle), not product code.
//
// extern "C" entry points of the CPU oracle, loaded with ctypes by tests/,
// __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference).
// Argument layouts are the product's C-ABI layouts (include/pathtrack_b200.h)
// so the same host buffers feed both sides.
#include <cfenv>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <atomic>
#include <thread>
#include <vector>

#include "orc_tracker.hpp"
#ifdef ORC_USE_REFERENCE
#include "pathtrack/hexio.hpp"
#endif

using namespace orc_track;

namespace {

thread_local std::string g_err;

// assert_ieee_environment (reference precision.cpp:37-44), restated
volatile double v_one = 1.0;
volatile double v_eps = 0x1p-53;
bool ieee_ok() {
  if (std::fegetround() != FE_TONEAREST) return false;
  double sum = v_one + v_eps;
  if (sum != 1.0) return false;
  double tie = v_one + 3.0 * v_eps;
  return tie > 1.0;
}

template <class R>
int run_track(const SystemDesc* g, const SystemDesc* f, const double* gamma, int k, const double* start,
              const StepParams* P, double* end, PathStats* st, TraceEvent* trace, int trace_cap,
              int* trace_len) {
  Tracker<R> T;
  T.build(*g, *f, gamma, k);
  std::vector<typename Tracker<R>::C> x0(T.n), x1;
  for (int i = 0; i < T.n; ++i) x0[i] = Tracker<R>::load_c(start, T.n, i);
  std::vector<TraceEvent> tr;
  T.track(x0, *P, x1, *st, trace ? &tr : nullptr);
  for (int i = 0; i < T.n; ++i) Tracker<R>::store_c(end, T.n, i, x1[i]);
  if (trace) {
    const int m = (int)tr.size() < trace_cap ? (int)tr.size() : trace_cap;
    std::memcpy(trace, tr.data(), sizeof(TraceEvent) * m);
    if (trace_len) *trace_len = (int)tr.size();
  }
  return 0;
}

template <class R>
int run_eval(const SystemDesc* g, const SystemDesc* f, const double* gamma, int k, const double* x,
             double t, double* h, double* J, double* rmax) {
  Tracker<R> T;
  T.build(*g, *f, gamma, k);
  const int n = T.n, N = T.N;
  std::vector<typename Tracker<R>::C> xv(n), Amat;
  for (int i = 0; i < n; ++i) xv[i] = Tracker<R>::load_c(x, n, i);
  const double r = T.eval_homotopy(xv, t, Amat);
  if (rmax) *rmax = r;
  for (int i = 0; i < N; ++i) Tracker<R>::store_c(h, N, i, -Amat[(size_t)n * N + i]);
  for (long q = 0; q < (long)N * n; ++q) Tracker<R>::store_c(J, (long)N * n, q, Amat[q]);
  return 0;
}

template <class R>
int run_lstsq(int N, int n, const double* Ain, const double* b, double* x) {
  Tracker<R> T;
  T.n = n;
  T.N = N;
  std::vector<typename Tracker<R>::C> Amat((size_t)N * (n + 1)), dx;
  for (long q = 0; q < (long)N * n; ++q) Amat[q] = Tracker<R>::load_c(Ain, (long)N * n, q);
  for (int i = 0; i < N; ++i) Amat[(size_t)n * N + i] = Tracker<R>::load_c(b, N, i);
  if (!T.lstsq(Amat, dx)) return -3;
  for (int i = 0; i < n; ++i) Tracker<R>::store_c(x, n, i, dx[i]);
  return 0;
}

template <class R>
R rd(const double* p) {
  return Tracker<R>::limbs_to_real(p);
}
template <class R>
void wr(const R& v, double* p) {
  Tracker<R>::real_to_limbs(v, p);
}

template <class R>
int run_arith(int op, long count, const double* a, const double* b, double* out) {
  using C = A::Complex<R>;
  constexpr int L = A::RealTraits<R>::limbs;
  for (long i = 0; i < count; ++i) {
    const double* pa = a + i * 2 * L;
    const double* pb = b + i * 2 * L;
    double* po = out + i * 2 * L;
    const R ar = rd<R>(pa), br = rd<R>(pb);
    const C ac(rd<R>(pa), rd<R>(pa + L)), bc(rd<R>(pb), rd<R>(pb + L));
    C oc;
    switch (op) {
      case 0: wr<R>(ar + br, po); break;
      case 1: wr<R>(ar - br, po); break;
      case 2: wr<R>(ar * br, po); break;
      case 3: wr<R>(ar * pb[0], po); break;
      case 4: wr<R>(ar / br, po); break;
      case 5: wr<R>(Tracker<R>::real_sqrt(ar), po); break;
      case 6: wr<R>(A::renormalize(ar), po); break;
      case 7: oc = ac * bc; wr<R>(oc.re, po); wr<R>(oc.im, po + L); break;
      case 8: oc = ac + bc; wr<R>(oc.re, po); wr<R>(oc.im, po + L); break;
      case 9: oc = A::conj(ac) * bc; wr<R>(oc.re, po); wr<R>(oc.im, po + L); break;
      case 10: wr<R>(A::norm_sqr(ac), po); break;
      case 11: po[0] = A::modulus_double(ac); break;
      case 12: wr<R>(A::powi(ar, (unsigned)pb[0]), po); break;
      case 13: oc = A::unit_complex<R>(pa[0]); wr<R>(oc.re, po); wr<R>(oc.im, po + L); break;
      case 14: oc = ac * br; wr<R>(oc.re, po); wr<R>(oc.im, po + L); break;
      case 15: oc = A::powi(ac, (unsigned)pb[0]); wr<R>(oc.re, po); wr<R>(oc.im, po + L); break;
      default: return -1;
    }
  }
  return 0;
}

template <class F>
int guarded(F&& f) {
  try {
    if (!ieee_ok()) {
      g_err = "binary64 environment is not round-to-nearest";
      return -1;
    }
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Batch baseline: a pool of `threads` host threads
// over independent paths (one tracker per path), each tracker
// single-threaded inside (its OpenMP regions run on 1 thread).
template <class R>
int run_batch(const SystemDesc* g, const SystemDesc* f, const double* gamma, int k, int n_paths,
              const double* starts, const StepParams* P, double* ends, PathStats* st, int threads) {
  std::atomic<int> next{0};
  std::atomic<int> bad{0};
  auto worker = [&]() {
#ifdef _OPENMP
    omp_set_num_threads(1);
#endif
    try {
      Tracker<R> T;
      T.build(*g, *f, gamma, k);
      const long PS = 2L * Tracker<R>::L * T.n;
      std::vector<typename Tracker<R>::C> x0(T.n), x1;
      for (int p = next++; p < n_paths; p = next++) {
        for (int i = 0; i < T.n; ++i) x0[i] = Tracker<R>::load_c(starts + p * PS, T.n, i);
        T.track(x0, *P, x1, st[p], nullptr);
        for (int i = 0; i < T.n; ++i) Tracker<R>::store_c(ends + p * PS, T.n, i, x1[i]);
      }
    } catch (...) {
      bad = 1;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < (threads > 0 ? threads : 1); ++t) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  return bad ? -1 : 0;
}

}  // namespace

extern "C" {

int orc_track_batch(int prec, const SystemDesc* g, const SystemDesc* f, const double* gamma, int k, int n_paths,
                    const double* starts, const StepParams* P, double* ends, PathStats* st, int threads) {
  return guarded([&] {
    switch (prec) {
      case 0: return run_batch<double>(g, f, gamma, k, n_paths, starts, P, ends, st, threads);
      case 1: return run_batch<A::DoubleDouble>(g, f, gamma, k, n_paths, starts, P, ends, st, threads);
      case 2: return run_batch<A::QuadDouble>(g, f, gamma, k, n_paths, starts, P, ends, st, threads);
    }
    return -1;
  });
}

#ifdef ORC_USE_REFERENCE
// The reference's own hex I/O (proj/src/hexio.cpp), for pinning the product's
// restatement (libpt_inputs.so).  Exceptions become -1 + orc_last_error().
int orc_ref_hex_limbs(const double* limbs, int count, char* out, int cap) {
  return guarded([&] {
    const std::string s = pathtrack::hex_limbs(std::span<const double>(limbs, (size_t)count));
    if ((int)s.size() + 1 > cap) throw std::invalid_argument("output buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  });
}
int orc_ref_parse_hex_limbs(const char* text, int len, double* out, int cap, int* count) {
  return guarded([&] {
    const std::vector<double> v = pathtrack::parse_hex_limbs(std::string_view(text, (size_t)len));
    *count = (int)v.size();
    for (int i = 0; i < (int)v.size() && i < cap; ++i) out[i] = v[i];
    return 0;
  });
}
#endif

const char* orc_variant(void) {
#ifdef ORC_USE_REFERENCE
  return "reference-headers";
#else
  return "restatement";
#endif
}

const char* orc_last_error(void) { return g_err.c_str(); }

void orc_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : 1);
#else
  (void)n;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int orc_track_path(int prec, const SystemDesc* g, const SystemDesc* f, const double* gamma, int k,
                   const double* start, const StepParams* P, double* end, PathStats* st, TraceEvent* trace,
                   int trace_cap, int* trace_len) {
  return guarded([&] {
    switch (prec) {
      case 0: return run_track<double>(g, f, gamma, k, start, P, end, st, trace, trace_cap, trace_len);
      case 1:
        return run_track<A::DoubleDouble>(g, f, gamma, k, start, P, end, st, trace, trace_cap, trace_len);
      case 2:
        return run_track<A::QuadDouble>(g, f, gamma, k, start, P, end, st, trace, trace_cap, trace_len);
    }
    return -1;
  });
}

int orc_eval_homotopy(int prec, const SystemDesc* g, const SystemDesc* f, const double* gamma, int k,
                      const double* x, double t, double* h, double* J, double* rmax) {
  return guarded([&] {
    switch (prec) {
      case 0: return run_eval<double>(g, f, gamma, k, x, t, h, J, rmax);
      case 1: return run_eval<A::DoubleDouble>(g, f, gamma, k, x, t, h, J, rmax);
      case 2: return run_eval<A::QuadDouble>(g, f, gamma, k, x, t, h, J, rmax);
    }
    return -1;
  });
}

int orc_lstsq(int prec, int N, int n, const double* Amat, const double* b, double* x) {
  return guarded([&] {
    switch (prec) {
      case 0: return run_lstsq<double>(N, n, Amat, b, x);
      case 1: return run_lstsq<A::DoubleDouble>(N, n, Amat, b, x);
      case 2: return run_lstsq<A::QuadDouble>(N, n, Amat, b, x);
    }
    return -1;
  });
}

// Bulk scalar operations for the arithmetic parity tests.  Element i of a, b,
// out occupies 2L doubles (re limbs, then im limbs; reals use the first L).
int orc_arith(int prec, int op, long count, const double* a, const double* b, double* out) {
  return guarded([&] {
    switch (prec) {
      case 0: return run_arith<double>(op, count, a, b, out);
      case 1: return run_arith<A::DoubleDouble>(op, count, a, b, out);
      case 2: return run_arith<A::QuadDouble>(op, count, a, b, out);
    }
    return -1;
  });
}

}  // extern "C"
