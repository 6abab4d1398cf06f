// count_fp64.cpp -- FP64 arithmetic instructions per emulated operation of
// the reference algorithms, measured on the host build of csrc/mp.cuh (which
// replays multiprec.hpp / complex.hpp operation for operation).  Negation and
// comparisons are not counted (sign flips are free operand modifiers on the
// device).  Output feeds DESIGN.md section 4 and csrc/work.hpp.
//   g++ -std=c++20 -O2 -ffp-contract=off -DPT_COUNT_FP64 tools/count_fp64.cpp && ./a.out
#include <cstdio>
#include <random>

#include "../paper_1501_06625_b200/csrc/mp.cuh"

using namespace ptk;

template <class R>
R rnd(std::mt19937_64& g) {
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  R r = rconst<R>(u(g) * 4.0);
  for (int l = 1; l < limbs_of<R>::L; ++l) r_set_limb(r, l, u(g) * std::ldexp(1.0, -53 * l) * r_hi(r));
  if constexpr (limbs_of<R>::L == 4) r = qd_renormalize(r);
  if constexpr (limbs_of<R>::L == 2) r = dd_norm(r_hi(r), r_limb(r, 1));
  return r;
}

template <class R>
void run(const char* name) {
  std::mt19937_64 g(1);
  const int T = 20000;
  auto avg = [&](auto&& f) {
    unsigned long long c0 = g_fp64;
    for (int i = 0; i < T; ++i) f();
    return double(g_fp64 - c0) / T;
  };
  volatile double sink = 0;
  double add = avg([&] { R a = rnd<R>(g), b = rnd<R>(g); unsigned long long c = g_fp64; R r = r_add(a, b); sink = r_hi(r); (void)c; });
  // subtract the operand construction cost measured separately
  double mk = avg([&] { R a = rnd<R>(g), b = rnd<R>(g); sink = r_hi(a) + r_hi(b); });
  double mul = avg([&] { R a = rnd<R>(g), b = rnd<R>(g); sink = r_hi(r_mul(a, b)); });
  double muld = avg([&] { R a = rnd<R>(g), b = rnd<R>(g); sink = r_hi(r_mul_d(a, r_hi(b))); });
  double dv = avg([&] { R a = rnd<R>(g), b = rnd<R>(g); sink = r_hi(r_div(a, b)); });
  double sq = avg([&] { R a = rnd<R>(g), b = rnd<R>(g); a = r_is_zero(a) ? b : a; if (r_hi(a) < 0) a = r_neg(a); sink = r_hi(r_sqrt(a)) + r_hi(b); });
  double hy = avg([&] { R a = rnd<R>(g), b = rnd<R>(g); sink = glibc_hypot(r_hi(a), r_hi(b)); });
  std::printf("%s add %.2f mul %.2f mul_d %.2f div %.2f sqrt %.2f hypot %.2f (cmul %.2f cadd %.2f)\n", name,
              add - mk, mul - mk, muld - mk, dv - mk, sq - mk, hy - mk, 4 * (mul - mk) + 2 * (add - mk),
              2 * (add - mk));
}

int main() {
  run<double>("d ");
  run<dd>("dd");
  run<qd>("qd");
}
