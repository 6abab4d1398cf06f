// QD op latency/throughput for the exact-sort variants (identical results).
// nvcc -DPT_QD_SORT={0,1,2,3} -DPT_QD_INLINE={0,1} ...
// prints cycles/op (1 thread, dependent chain) and the full-grid throughput
#include <cstdio>
#include "../paper_1501_06625_b200/csrc/mp.cuh"
using namespace ptk;
__global__ void lat(double* out, double seed) {
  qd q{{seed, 1e-17, 1e-34, 1e-51}}, w{{1.0000001, 1e-20, 1e-37, 1e-54}};
  long long c0 = clock64();
  for (int i = 0; i < 64; ++i) q = r_mul(q, w);
  long long c1 = clock64();
  for (int i = 0; i < 64; ++i) q = r_add(q, w);
  long long c2 = clock64();
  cplx<qd> z{q, w}, u{w, q};
  for (int i = 0; i < 16; ++i) z = c_mul(z, u);
  long long c3 = clock64();
  out[0] = (c1 - c0) / 64.0; out[1] = (c2 - c1) / 64.0; out[3] = (c3 - c2) / 16.0;
  out[2] = q.c[0] + z.re.c[1];
}
__global__ void thr(double* out, double seed, int iters) {
  qd q{{seed + threadIdx.x * 1e-9, 1e-17, 1e-34, 1e-51}}, w{{1.0000001, 1e-20, 1e-37, 1e-54}};
  qd q2 = q;
  for (int i = 0; i < iters; ++i) { q = r_mul(q, w); q2 = r_add(q2, w); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = q.c[0] + q2.c[0];
}
int main() {
  double* d; cudaMalloc(&d, 1 << 24);
  lat<<<1, 1>>>(d, 1.25); cudaDeviceSynchronize(); lat<<<1, 1>>>(d, 1.25);
  double h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks = 148 * 4, threads = 256, iters = 64;
  thr<<<blocks, threads>>>(d, 1.25, iters);
  cudaEventRecord(a); thr<<<blocks, threads>>>(d, 1.25, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)blocks * threads * iters;  // (mul + add) pairs
  printf("{\"variant\": %d, \"inline\": %d, \"qd_mul_cycles\": %.1f, \"qd_add_cycles\": %.1f, \"cqd_mul_cycles\": %.1f, \"pair_ns_per_op_gpu\": %.5f, \"fp64_instr_rate_T\": %.3f}\n",
         PT_QD_SORT, PT_QD_INLINE, h[0], h[1], h[3], ms * 1e6 / ops, ops * (343.0 + 128.36) / (ms * 1e-3) * 1e-12);
}
