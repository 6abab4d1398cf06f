// Critical-chain microbenchmarks of the single-path kernels on one warp:
// backsub_warp_e<dd,2> on a synthetic 64x65 R, and the pieces of its step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -o chain_bench_bin chain_bench.cu
#include <cstdio>
#include "../paper_1501_06625_b200/csrc/device.cuh"
using namespace ptdev;

__global__ void k_bs(DevPlan P, Work W, double* out, int reps) {
  long long t0 = clock64();
  double u = 0;
  for (int r = 0; r < reps; ++r) u += backsub_warp_e<dd, 2>(P, W);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / reps; out[1] = u; }
}

// one backsub-like step chain without memory: x = acc*inv; shfl; acc -= cur*x
__global__ void k_step(double* out, int steps) {
  const int lane = threadIdx.x & 31;
  cplx<dd> acc{{1.0 + lane, 1e-20}, {0.5, 0}}, cur{{0.25, 1e-19}, {0.125 * lane, 0}};
  dd inv{0.999, 1e-18};
  long long t0 = clock64();
  for (int j = 0; j < steps; ++j) {
    cplx<dd> x = c_scale(acc, inv);
    x = shfl0(x, j & 31);
    acc = c_sub(acc, c_mul(cur, x));
  }
  long long t1 = clock64();
  if (lane == 0) { out[2] = (double)(t1 - t0) / steps; out[3] = acc.re.hi; }
  // same without the shuffle
  t0 = clock64();
  for (int j = 0; j < steps; ++j) {
    cplx<dd> x = c_scale(acc, inv);
    acc = c_sub(acc, c_mul(cur, x));
  }
  t1 = clock64();
  if (lane == 0) { out[4] = (double)(t1 - t0) / steps; out[5] = acc.re.hi; }
  // dd add chain, dd mul chain, complex dd mul chain
  dd a{1.0 + lane, 1e-20}, b{1e-3, 1e-21};
  t0 = clock64();
  for (int j = 0; j < steps; ++j) a = r_add(a, b);
  t1 = clock64();
  if (lane == 0) { out[6] = (double)(t1 - t0) / steps; out[7] = a.hi; }
  t0 = clock64();
  for (int j = 0; j < steps; ++j) a = r_mul(a, inv);
  t1 = clock64();
  if (lane == 0) { out[8] = (double)(t1 - t0) / steps; out[9] = a.hi; }
  t0 = clock64();
  for (int j = 0; j < steps; ++j) cur = c_mul(cur, acc);
  t1 = clock64();
  if (lane == 0) { out[10] = (double)(t1 - t0) / steps; out[11] = cur.re.hi; }
  // warp tree of complex dd (5 shuffle levels)
  cplx<dd> v = acc;
  t0 = clock64();
  for (int j = 0; j < steps; ++j) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const cplx<dd> o = shfl_down_r(v, off);
      v = pick(lane < off, c_add(v, o), v);
    }
  }
  t1 = clock64();
  if (lane == 0) { out[12] = (double)(t1 - t0) / steps; out[13] = v.re.hi; }
}

// WarpMgs::project<2> (DD, N = 64) on `active` warps of one CTA at once
__global__ void k_proj(DevPlan P, Work W, double* out, int active, int reps) {
  __shared__ Smem<dd> sh;
  extern __shared__ double dyn[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const BlockTeam team{W.ctl, 1, 0, nullptr};
  const WarpMgs<dd, BlockTeam> m{P, W, team, sh, dyn, ColMap{1, 4}, lane, w, P.N, P.n, (long)P.N * (P.n + 1),
                                 (long)P.n * (P.n + 1), 2L * 2 * P.N, 1ull, 0x1p-52};
  for (int i = threadIdx.x; i < 8 * 4 * 64; i += blockDim.x) dyn[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  if (w >= active) return;
  cplx<dd> q[2], a[2];
  for (int r = 0; r < 2; ++r) q[r] = cplx<dd>{{0.5 + 1e-4 * lane, 1e-20}, {0.25, 0}};
  double* col = dyn + w * 4 * 64;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) m.template project<2>(3, 10, q, a, col);
  long long t1 = clock64();
  if (lane == 0) out[16 + w] = (double)(t1 - t0) / reps;
}

int main() {
  const int n = 64, L = 2;
  DevPlan P{};
  P.n = n; P.N = n;
  Work W{};
  double *Rm, *inv, *x, *dx, *out;
  cudaMalloc(&Rm, 2 * L * n * (n + 1) * 8);
  cudaMalloc(&inv, L * n * 8);
  cudaMalloc(&x, 2 * L * n * 8);
  cudaMalloc(&dx, 2 * L * n * 8);
  cudaMalloc(&out, 64 * 8);
  cudaMemset(Rm, 0, 2 * L * n * (n + 1) * 8);
  cudaMemset(inv, 0, L * n * 8);
  cudaMemset(x, 0, 2 * L * n * 8);
  W.Rm = Rm; W.inv = inv; W.x = x; W.dx = dx;
  k_bs<<<1, 32>>>(P, W, out, 2);
  k_bs<<<1, 32>>>(P, W, out, 4);
  k_step<<<1, 32>>>(out, 64);
  k_step<<<1, 32>>>(out, 64);
  cudaMalloc(&W.ctl, 64);
  P.P_mgs = 32;
  cudaFuncSetAttribute(k_proj, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  double pr[3];
  for (int ai = 0; ai < 3; ++ai) {
    const int act = ai == 0 ? 1 : (ai == 1 ? 4 : 8);
    k_proj<<<1, 256, 64 * 1024>>>(P, W, out, act, 4);
    k_proj<<<1, 256, 64 * 1024>>>(P, W, out, act, 16);
    cudaDeviceSynchronize();
    cudaMemcpy(&pr[ai], out + 16, 8, cudaMemcpyDeviceToHost);
  }
  printf("{\"project_dd_n64_cycles_1_4_8_warps\": [%.0f, %.0f, %.0f]}\n", pr[0], pr[1], pr[2]);
  cudaError_t e = cudaDeviceSynchronize();
  double h[16];
  cudaMemcpy(h, out, 128, cudaMemcpyDeviceToHost);
  printf("{\"err\": \"%s\", \"backsub_dd_n64_cycles\": %.0f, \"step_with_shfl\": %.1f, \"step_no_shfl\": %.1f, "
         "\"dd_add\": %.1f, \"dd_mul\": %.1f, \"cdd_mul\": %.1f, \"tree5_cdd\": %.1f}\n",
         cudaGetErrorString(e), h[0], h[2], h[4], h[6], h[8], h[10], h[12]);
}
