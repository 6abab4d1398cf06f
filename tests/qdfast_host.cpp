// Host build of the tolerance-parity QD arithmetic (mp_qdfast.cuh) for the
// CPU accuracy tests (tests/test_qdfast.py): the same source the fast device
// kernels compile, through mp.cuh's host path with PT_QD_FAST_HOST.
#include "../paper_1501_06625_b200/csrc/mp.cuh"

using namespace ptk;

extern "C" int qdf_arith(int op, long count, const double* a, const double* b, double* out) {
  for (long i = 0; i < count; ++i) {
    const qd x{{a[4 * i], a[4 * i + 1], a[4 * i + 2], a[4 * i + 3]}};
    const qd y{{b[4 * i], b[4 * i + 1], b[4 * i + 2], b[4 * i + 3]}};
    qd r{};
    switch (op) {
      case 0: r = r_add(x, y); break;
      case 1: r = r_sub(x, y); break;
      case 2: r = r_mul(x, y); break;
      case 3: r = r_mul_d(x, y.c[0]); break;
      case 4: r = r_div(x, y); break;
      case 5: r = r_sqrt(x); break;
      case 6: {  // r_sqrt_inv: out = 1/sqrt(x) (the MGS pair's inverse)
        qd s;
        r_sqrt_inv(x, s, r);
        break;
      }
      default: return -1;
    }
    for (int l = 0; l < 4; ++l) out[4 * i + l] = r.c[l];
  }
  return 0;
}
