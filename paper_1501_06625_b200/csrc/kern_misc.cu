// kern_misc.cu -- microbenchmark kernels behind pt_fp64_peak / pt_microbench
// (the measured peaks and latencies DESIGN.md sections 4-5 are sized with).
#include "kernels.cuh"

namespace ptdev {

// FP64-pipe peak: kPeakChains (kernel_set.hpp) independent DFMA chains per thread.
__global__ void __launch_bounds__(256) k_fp64_peak(double* out, int iters) {
  double a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = 1e-3 * (threadIdx.x + c);
  const double b = 0.9999999, d = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = __fma_rn(a[c], b, d);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Latency microbenchmarks (one thread): dependent chains of the primitive and
// emulated operations, in SM cycles per operation.
__global__ void k_latency(double* out, double seed) {
  const int T = 256;
  long long c0, c1;
  double a = seed, b = 1.0000001;
  c0 = clock64();
  for (int i = 0; i < T; ++i) a = __dadd_rn(a, b);
  c1 = clock64();
  out[0] = (double)(c1 - c0) / T;
  out[10] = a;
  dd x{seed, 0.0}, y{1.0000001, 1e-20};
  c0 = clock64();
  for (int i = 0; i < T; ++i) x = r_add(x, y);
  c1 = clock64();
  out[1] = (double)(c1 - c0) / T;
  c0 = clock64();
  for (int i = 0; i < T; ++i) x = r_mul(x, y);
  c1 = clock64();
  out[2] = (double)(c1 - c0) / T;
  out[11] = x.hi;
  qd q{{seed, 1e-17, 1e-34, 1e-51}}, w{{1.0000001, 1e-20, 1e-37, 1e-54}};
  c0 = clock64();
  for (int i = 0; i < T / 8; ++i) q = r_add(q, w);
  c1 = clock64();
  out[3] = (double)(c1 - c0) / (T / 8);
  c0 = clock64();
  for (int i = 0; i < T / 8; ++i) q = r_mul(q, w);
  c1 = clock64();
  out[4] = (double)(c1 - c0) / (T / 8);
  out[12] = q.c[0];
  cplx<dd> z{{seed, 0}, {0.5, 0}}, u{{0.9999, 1e-20}, {0.01, 0}};
  c0 = clock64();
  for (int i = 0; i < T; ++i) z = c_mul(z, u);
  c1 = clock64();
  out[5] = (double)(c1 - c0) / T;
  out[13] = z.re.hi;
  double h = seed;
  c0 = clock64();
  for (int i = 0; i < T; ++i) h = glibc_hypot(h, 0.5) * 0.5;
  c1 = clock64();
  out[6] = (double)(c1 - c0) / T;
  out[14] = h;
}

// MGS building blocks on one warp (group width 1, N = 64), in cycles:
// out[0] group_tree<cplx<dd>>, [1] mgs_project, [2] c_conj_mul, [3] dd sqrt, [4] dd div
__global__ void k_mgs_pieces(double* out) {
  __shared__ Smem<dd> sh;
  __shared__ double col[4 * 64], rcol[4 * 65], invb[2];
  const int lane = threadIdx.x;
  const Group g{1, lane, 1};
  for (int i = lane; i < 4 * 64; i += 32) col[i] = 1.0 + 1e-3 * i;
  __syncwarp();
  cplx<dd> q[kMaxElems];
  for (int r = 0; r < 2; ++r) q[r] = cplx<dd>{{0.5 + 1e-4 * lane, 1e-20}, {0.25, 0}};
  DevPlan P{};
  P.n = 64;
  P.N = 64;
  P.P_mgs = 32;
  P.mgs_gw = 1;
  OwnedCol c{ColRef{col, 64}, ColRef{rcol, 65}, invb, 1, 0};
  int phase = 0;
  cplx<dd> acc{{1.0 + lane, 0}, {0.5, 0}};
  long long t0 = clock64();
  cplx<dd> t = group_tree(acc, g, 32, 64, sh.tree);
  __syncwarp();
  long long t1 = clock64();
  mgs_project<dd, true>(P, g, 0, sh, phase, q, c, 3, 10);
  __syncwarp();
  long long t2 = clock64();
  cplx<dd> z = c_conj_mul(q[0], q[1]);
  long long t3 = clock64();
  dd sq = r_sqrt(z.re);
  long long t4 = clock64();
  dd dv = r_div(dd{1.0, 0.0}, sq);
  long long t5 = clock64();
  if (lane == 0) {
    out[0] = (double)(t1 - t0);
    out[1] = (double)(t2 - t1);
    out[2] = (double)(t3 - t2);
    out[3] = (double)(t4 - t3);
    out[4] = (double)(t5 - t4);
    out[15] = t.re.hi + dv.hi + col[5];
  }
}

// Grid barrier cost: every CTA crosses `iters` GridTeam barriers.
__global__ void k_barrier(unsigned long long* ctl, int iters, double* out) {
  __shared__ int flag;
  const GridTeam team{ctl, (int)gridDim.x, (int)blockIdx.x, nullptr};
  const unsigned long long t0 = gtimer();
  for (int i = 0; i < iters; ++i)
    if (!team.sync(&flag)) break;
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (double)(gtimer() - t0) / iters;
}

// Flag ping-pong between CTA 0 and CTA gridDim.x-1 (release/acquire through L2).
__global__ void k_pingpong(unsigned long long* flags, int iters, double* out) {
  if (threadIdx.x != 0) return;
  const bool ping = blockIdx.x == 0, pong = blockIdx.x == gridDim.x - 1;
  if (!ping && !pong) return;
  const unsigned long long t0 = gtimer();
  for (int i = 1; i <= iters; ++i) {
    if (ping) {
      st_release(flags, i);
      while (ld_acquire(flags + 32) != (unsigned long long)i) {
      }
    } else {
      while (ld_acquire(flags) != (unsigned long long)i) {
      }
      st_release(flags + 32, i);
    }
  }
  if (ping) out[0] = (double)(gtimer() - t0) / iters / 2;  // one-way ns
}


}  // namespace ptdev

const ptdev::MiscKernels ptdev::kmisc = {(const void*)&ptdev::k_fp64_peak, (const void*)&ptdev::k_latency,
                                         (const void*)&ptdev::k_mgs_pieces, (const void*)&ptdev::k_barrier,
                                         (const void*)&ptdev::k_pingpong};
