// Stand-alone warp-MGS benchmark: the production mgs_warp<R, ClusterTeam> on a
// synthetic well-conditioned N x (n+1) complex matrix, one cluster of C CTAs,
// R repetitions; prints the per-column timeline medians recorded by the
// kernel (same instrumentation as tools/mgs_timeline.py) and ns per MGS.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -o mgs_bench_bin mgs_bench.cu
//   ./mgs_bench_bin [N] [C] [B] [reps]
#define PT_MGS_FINE 1
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "../paper_1501_06625_b200/csrc/device.cuh"
using namespace ptdev;
#ifndef MB_R
#define MB_R dd
#endif
using R = MB_R;

// I-cache polluter: a long straight-line body (QD arithmetic, ~tens of KB of
// code) run by every thread between two MGS sweeps when MB_POLLUTE is set
__device__ __noinline__ double pollute(double seed) {
  qd a{{seed, 1e-17, 1e-34, 1e-51}}, b{{1.0000001, 1e-20, 1e-37, 1e-54}};
  cplx<qd> z{a, b}, u{b, a};
#pragma unroll
  for (int i = 0; i < 6; ++i) z = c_add(c_mul(z, u), z);
  return z.re.c[0];
}

__global__ void __launch_bounds__(kThreads, 1) k_mgs(DevPlan P, Work W, double* A0, int reps, double* out, int probe) {
  __shared__ Smem<R> sh;
  __shared__ uint32_t s_flags[kMaxCols];
  extern __shared__ double dyn[];
  const ClusterTeam team{W.ctl, (int)cluster_nranks(), (int)cluster_rank(), s_flags};
  constexpr int L = limbs_of<R>::L;
  if (threadIdx.x == 0) {
    sh.mgs_seq = 0;
    uint64_t* bars = reinterpret_cast<uint64_t*>(dyn + mgs_warp_slots_doubles(L, P.N, P.n, team.nblocks) +
                                                 (long)P.n * mgs_warp_qs(L, P.N));
    for (int k = 0; k < P.n; ++k) mbar_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  team.sync(&sh.flag);
  const long SA = (long)P.N * (P.n + 1);
  unsigned long long t0 = 0;
  for (int r = 0; r < reps; ++r) {
    // fresh matrix (every CTA copies a slice)
    for (long q = team.block * kThreads + threadIdx.x; q < 2L * L * SA; q += (long)team.nblocks * kThreads)
      W.A[q] = A0[q];
    team.sync(&sh.flag);
    if (r == 1) t0 = gtimer();
    if (std::is_same<R, dd>::value && probe == 1 && team.block == 0 && threadIdx.x >= 192 && threadIdx.x < 224) {
#ifndef MB_NO_DD_PROBES
      // concurrent probe: warp 6 of CTA 0 (no columns) runs the isolated
      // projection loop on a private smem slot while the MGS runs
      const int lane = threadIdx.x & 31;
      const WarpMgs<R, ClusterTeam> m{P, W, team, sh, dyn, ColMap{team.nblocks, P.mgs_B}, lane, 6, P.N, P.n, SA,
                                      (long)P.n * (P.n + 1), 2L * L * P.N, 1ull, 0x1p-52, nullptr, nullptr};
      cplx<R> q[2], a[2];
      for (int rr = 0; rr < 2; ++rr) q[rr] = cplx<R>{{0.5 + 1e-4 * lane, 1e-20}, {0.25, 0}};
      double* scratch = dyn + 6 * 4 * 64;  // slot of warp 6 (no columns)
      long long c0 = clock64();
      for (int i = 0; i < 64; ++i) m.template project<2>(3, 10, q, a, scratch);
      long long c1 = clock64();
      if (lane == 0 && r == reps - 1) out[2] = (double)(c1 - c0) / 64 + (a[0].re.hi == 12345.0);
#endif
    } else
    mgs_warp<R, ClusterTeam>(P, W, team, sh, dyn, 1000ull + r, 0x1p-52);
    team.sync(&sh.flag);
    if (probe == 2) out[4 + (threadIdx.x & 3)] = pollute(1.0 + r);
    if (threadIdx.x == 0) ++sh.mgs_seq;
    team.sync(&sh.flag);
  }
  if (team.block == 0 && threadIdx.x == 0) out[0] = (double)(gtimer() - t0) / max(1, reps - 1);
  // the same projection code in isolation inside this kernel: warp 0 of CTA 0 alone
#ifndef MB_NO_DD_PROBES
  if (team.block == 0 && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const WarpMgs<R, ClusterTeam> m{P, W, team, sh, dyn, ColMap{team.nblocks, P.mgs_B}, lane, 0, P.N, P.n, SA,
                                    (long)P.n * (P.n + 1), 2L * L * P.N, 1ull, 0x1p-52, nullptr, nullptr};
    cplx<R> q[2], a[2];
    for (int r = 0; r < 2; ++r) q[r] = cplx<R>{{0.5 + 1e-4 * lane, 1e-20}, {0.25, 0}};
    long long c0 = clock64();
    for (int i = 0; i < 16; ++i) m.template project<2>(3, 10, q, a, dyn);
    long long c1 = clock64();
    if (lane == 0) out[1] = (double)(c1 - c0) / 16 + (a[0].re.hi == 12345.0);
  }
#endif
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 64, C = argc > 2 ? atoi(argv[2]) : 16, B = argc > 3 ? atoi(argv[3]) : 4;
  const int reps = argc > 4 ? atoi(argv[4]) : 4;
  const int n = N, L = limbs_of<R>::L;
  const long SA = (long)N * (n + 1);
  std::vector<double> hA(2L * L * SA, 0.0);
  srand(7);
  for (long q = 0; q < SA; ++q) {
    const int i = q % N, j = q / N;
    const double re = (double)rand() / RAND_MAX - 0.5 + (i == j ? 4.0 : 0.0);
    const double im = (double)rand() / RAND_MAX - 0.5;
    double sr = re, si = im;
    for (int l = 0; l < L; ++l) {  // limb l ~ 2^-53 l below the leading one
      hA[(long)l * SA + q] = sr;
      hA[(long)(L + l) * SA + q] = si;
      sr *= 1e-17;
      si *= 1e-17;
    }
  }
  if (const char* fn = getenv("MGS_MATRIX")) {  // [2L][N*(n+1)] doubles (SoA planes), e.g. chandra's [J | -h]
    FILE* fp = fopen(fn, "rb");
    if (fp) {
      const size_t got = fread(hA.data(), 8, hA.size(), fp);
      fclose(fp);
      printf("{\"matrix\": \"%s\", \"doubles\": %zu}\n", fn, got);
    }
  }
  DevPlan P{};
  P.n = n;
  P.N = N;
  P.P_mgs = std::min(256, std::max(32, [](int x) { int p = 1; while (p < x) p <<= 1; return p; }((N + 1) / 2)));
  P.mgs_warp = 2;
  P.mgs_B = B;
  P.mgs_smem = 1;
  Work W{};
  double *A, *A0, *Rm, *inv, *rmaxp, *out, *qg;
  unsigned long long *flags, *ctl, *prof;
  cudaMalloc(&A, hA.size() * 8);
  cudaMalloc(&A0, hA.size() * 8);
  cudaMalloc(&Rm, 2L * L * n * (n + 1) * 8);
  cudaMalloc(&inv, L * n * 8);
  cudaMalloc(&rmaxp, (n + 1) * 8);
  cudaMalloc(&out, 64);
  cudaMalloc(&qg, (size_t)n * mgs_warp_qs(L, N) * 8);
  cudaMalloc(&flags, (n + 1) * 8);
  cudaMalloc(&ctl, 64 * 8);
  cudaMalloc(&prof, (8 + 14 * (n + 2)) * 8);
  cudaMemset(ctl, 0, 64 * 8);
  cudaMemset(prof, 0, (8 + 14 * (n + 2)) * 8);
  cudaMemcpy(A0, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice);
  W.A = A; W.Rm = Rm; W.inv = inv; W.rmaxp = rmaxp; W.flags = flags; W.ctl = ctl; W.prof = prof; W.qg = qg;
  const size_t dyn = mgs_warp_bytes(L, N, n, C, true);
  cudaFuncSetAttribute(k_mgs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  cudaFuncSetAttribute(k_mgs, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = dyn;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int probe = argc > 5 ? atoi(argv[5]) : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_mgs, P, W, A0, reps, out, probe);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  double ns = 0, iso = 0, conc = 0;
  cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&iso, out + 1, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&conc, out + 2, 8, cudaMemcpyDeviceToHost);
  std::vector<unsigned long long> t(6 * (n + 2));
  cudaMemcpy(t.data(), prof + 8, t.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<double> wl, pr, no, col;
  for (int j = 2; j < n; ++j) {
    wl.push_back((double)(t[6 * j + 2] - t[6 * j + 1]));
    pr.push_back((double)(t[6 * j + 3] - t[6 * j + 2]));
    no.push_back((double)(t[6 * j + 4] - t[6 * j + 3]));
    col.push_back((double)(t[6 * j + 5] - t[6 * (j - 1) + 5]));
  }
  if (getenv("MGS_DUMP")) {
    for (size_t q = 0; q < pr.size(); ++q) printf("%d:%.0f/%.0f ", (int)q + 2, pr[q], no[q]);
    printf("\n");
  }
  std::vector<unsigned long long> fine(8 * (n + 2));
  cudaMemcpy(fine.data(), prof + 8 + 6 * (n + 2), fine.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<double> st[5];
  for (int j = 2; j < n; ++j)
    for (int q = 0; q < 5; ++q) st[q].push_back((double)(fine[8 * j + q + 1] - fine[8 * j + q]));
  auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v.empty() ? 0.0 : v[v.size() / 2]; };
  printf("{\"err\": \"%s\", \"N\": %d, \"C\": %d, \"B\": %d, \"ns_per_mgs\": %.0f, \"wait_load_cyc\": %.0f, "
         "\"project_cyc\": %.0f, \"normalize_cyc\": %.0f, \"column_ns\": %.0f, \"isolated_project_cyc\": %.0f, \"concurrent_probe_cyc\": %.0f}\n",
         cudaGetErrorString(e), N, C, B, ns, med(wl), med(pr), med(no), med(col), iso, conc);
  printf("{\"fine_cycles\": {\"load_col\": %.0f, \"conj_mul\": %.0f, \"tree\": %.0f, \"bcast\": %.0f, \"axpy\": %.0f}}\n",
         med(st[0]), med(st[1]), med(st[2]), med(st[3]), med(st[4]));
  return 0;
}
