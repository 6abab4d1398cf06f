// Compile-and-link check of include/pathtrack_b200.hpp against the reference
// headers (or the oracle restatement with the same public names).  Without a
// device pt_plan_create must throw (no CPU fallback); with one it tracks the
// 1-variable homotopy of SPEC.md:472 and prints the end point.
#include <cstdio>
#include <vector>
#ifdef USE_REFERENCE_HEADERS
#include "pathtrack/complex.hpp"
#else
#include "orc_arith.hpp"
namespace pathtrack { using namespace orc; template <class R> using Point = std::vector<orc::Complex<R>>; }
#endif
#include "pathtrack_b200.hpp"

using namespace pathtrack;
int main() {
  using R = DoubleDouble;
  b200::System<R> g, f;
  g.n_vars = f.n_vars = 1;
  g.term({}, Complex<R>(R(-1.0)));
  g.term({{0, 1}}, Complex<R>(R(1.0)));
  f.term({}, Complex<R>(R(-2.0)));
  f.term({{0, 1}}, Complex<R>(R(1.0)));
  {  // the canonical-form view the C-ABI receives (one equation, two terms)
    std::vector<double> limbs;
    const pt_system_desc d = g.desc(limbs);
    if (d.n_eqs != 1 || d.n_terms != 2 || d.eq_ptr[0] != 0 || d.eq_ptr[1] != 2 || d.term_ptr[2] != 1) return 4;
  }
  Point<R> x0{Complex<R>(R(1.0))};
  auto rt = b200::from_limbs<R>(b200::to_limbs<R>(x0), 1);
  if (!(rt[0].re.hi == 1.0 && rt[0].re.lo == 0.0)) return 3;
  try {
    b200::Homotopy<R> h(g, f, Complex<R>(R(0.6), R(0.8)), 2);
    auto o = h.track_path(x0);
    std::printf("device: success=%d x=%.17g steps=%d\n", (int)o.success, o.end[0].re.hi, o.stats.steps);
    // the batch entry: three copies of the start, the same end point bits each time
    const auto b = h.track_batch(std::vector<Point<R>>(3, x0));
    for (const auto& ob : b)
      if (!ob.success || ob.end[0].re.hi != o.end[0].re.hi || ob.end[0].re.lo != o.end[0].re.lo ||
          ob.stats.steps != o.stats.steps)
        return 5;
    std::printf("batch: %zu paths, all equal to the single path\n", b.size());
    return o.success && o.end[0].re.hi == 2.0 ? 0 : 1;
  } catch (const std::runtime_error& e) {
    std::printf("no device: %s\n", e.what());
    return pt_device_count() == 0 ? 0 : 2;
  }
}
