// device.cuh -- the device-resident tracker: evaluation/differentiation,
// MGS least squares, predictor and step control for one path, written once
// and instantiated for
//   * GridTeam: one path spread over a cooperative persistent grid (one CTA
//     per SM); phases are separated by a grid barrier and the MGS columns are
//     pipelined with per-column release/acquire flags (no host round trip);
//   * BlockTeam: one path per CTA (batch mode); barriers are __syncthreads.
//
// Pinned semantics (must equal oracle/orc_tracker.hpp):
//   - canonical sums: partial p = c[p] + c[p+P] + ..., then off = P/2..1,
//     partial[p] += partial[p+off] if p+off < K; P = width_eval(K) for
//     evaluation slots, width_mgs(N) for MGS norms and dots;
//   - monomials: Table 1 reverse mode, 3m-5 products;
//   - h = wS*Sg + Sf*wT, wS = gamma*(1-t)^k, wT = t^k;
//   - MGS q_k = a_k * (1/r_kk), a_j -= r_kj*q_k, rank test in binary64;
//   - back substitution subtracting r_kj*x_j for j = n-1 down to k+1;
//   - Newton Fig. 2, tracker Fig. 3 with SPEC.md:492-495.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/pathtrack_b200.h"
#include "mp.cuh"
#include "plan.hpp"

namespace ptdev {

using namespace ptk;

constexpr int kThreads = 256;  // every tracker CTA
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRowsPerThread = 4;  // n <= 1024
constexpr int kMaxDegree = 8;
constexpr double kTimeoutNs = 20e9;

enum { CTL_BAR_COUNT = 0, CTL_BAR_GEN = 1, CTL_ABORT = 2, CTL_RANK = 3, CTL_QUEUE = 4, CTL_WORDS = 8 };
enum { NW_OK = 0, NW_RESIDUAL_INCREASE = 1, NW_ITERATION_BUDGET = 2, NW_LINEAR_SOLVE = 3, NW_ABORT = 4 };

struct DevPlan {
  int n, N, M;
  int P_mgs;
  const int32_t* mono_size;
  const int32_t* mono_vbeg;
  const int32_t* mono_out;
  const int32_t* mono_flags;
  const int32_t* mono_var;
  const int32_t* mono_exp;
  long ws_len;
  const ptplan::SlotTask* tasks;
  int class_beg[5];
  const int32_t* ctr_coef;
  const int32_t* ctr_ws;
  const double* coef;
  long n_coef;
  const double* gamma;  // 2L limbs
  int relax_k;
};

// One path's workspace.  All arrays are complex SoA unless noted.
struct Work {
  double* x;      // [2L][n] working point
  double* hist;   // [cap][2L][n] accepted points (ring)
  double* ws;     // [2L][ws_len] monomial values / partials
  double* A;      // [2L][N*(n+1)] least-squares matrix [J | -h], column-major
  double* Rm;     // [2L][n*(n+1)] R factor, (k,j) at j*n + k; column n = Q^H b
  double* inv;    // [L][n] 1/r_kk (real)
  double* rmaxp;  // [n] prefix max of binary64 r_kk
  double* hmod;   // [N] |h_i| in binary64
  double* scal;   // [8] 0: update norm u
  double* dx;     // [2L][n] last Newton update
  unsigned long long* flags;  // [n+1] MGS column-ready flags (epoch values)
  unsigned long long* ctl;    // [CTL_WORDS] barrier / abort / rank-fail
};

// ---------------------------------------------------------------------------
// synchronisation helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

struct GridTeam {
  unsigned long long* ctl;
  int nblocks, block;
  static constexpr bool kGrid = true;
  // Sense-free generation barrier; returns false once any CTA has aborted.
  __device__ bool sync(int* s_flag) const {
    __syncthreads();
    if (threadIdx.x == 0) {
      int abort = 0;
      const unsigned long long gen = ld_acquire(ctl + CTL_BAR_GEN);
      __threadfence();
      const unsigned long long arrived = atomicAdd(ctl + CTL_BAR_COUNT, 1ull);
      if (arrived == (unsigned long long)(nblocks - 1)) {
        atomicExch(ctl + CTL_BAR_COUNT, 0ull);
        __threadfence();
        st_release(ctl + CTL_BAR_GEN, gen + 1);
      } else {
        const unsigned long long t0 = gtimer();
        while (ld_acquire(ctl + CTL_BAR_GEN) == gen) {
          if (ld_acquire(ctl + CTL_ABORT)) {
            abort = 1;
            break;
          }
          if ((double)(gtimer() - t0) > kTimeoutNs) {
            atomicExch(ctl + CTL_ABORT, 1ull);
            abort = 1;
            break;
          }
          __nanosleep(32);
        }
      }
      __threadfence();
      if (ld_acquire(ctl + CTL_ABORT)) abort = 1;
      *s_flag = abort;
    }
    __syncthreads();
    return *s_flag == 0;
  }
};

struct BlockTeam {
  unsigned long long* ctl;
  int nblocks, block;  // 1, 0
  static constexpr bool kGrid = false;
  __device__ bool sync(int*) const {
    __syncthreads();
    return true;
  }
};

// Wait for column flag == epoch (one thread spins, the group then syncs).
__device__ __forceinline__ bool wait_flag(const unsigned long long* flag, unsigned long long epoch,
                                          unsigned long long* ctl) {
  const unsigned long long t0 = gtimer();
  while (ld_acquire(flag) != epoch) {
    if (ld_acquire(ctl + CTL_ABORT)) return false;
    if ((double)(gtimer() - t0) > kTimeoutNs) {
      atomicExch(ctl + CTL_ABORT, 1ull);
      return false;
    }
    __nanosleep(20);
  }
  __threadfence();
  return true;
}

// ---------------------------------------------------------------------------
// shuffles and group reductions of reals / complex values
// ---------------------------------------------------------------------------
__device__ __forceinline__ double shfl_down_r(double v, int off) { return __shfl_down_sync(0xffffffffu, v, off); }
__device__ __forceinline__ dd shfl_down_r(dd v, int off) {
  return {__shfl_down_sync(0xffffffffu, v.hi, off), __shfl_down_sync(0xffffffffu, v.lo, off)};
}
__device__ __forceinline__ qd shfl_down_r(const qd& v, int off) {
  qd r;
#pragma unroll
  for (int l = 0; l < 4; ++l) r.c[l] = __shfl_down_sync(0xffffffffu, v.c[l], off);
  return r;
}
template <class R>
__device__ __forceinline__ cplx<R> shfl_down_r(const cplx<R>& v, int off) {
  return {shfl_down_r(v.re, off), shfl_down_r(v.im, off)};
}
__device__ __forceinline__ double add_v(double a, double b) { return add64(a, b); }
__device__ __forceinline__ dd add_v(dd a, dd b) { return r_add(a, b); }
__device__ __forceinline__ qd add_v(const qd& a, const qd& b) { return r_add(a, b); }
template <class R>
__device__ __forceinline__ cplx<R> add_v(const cplx<R>& a, const cplx<R>& b) {
  return c_add(a, b);
}

// A "group" is gw consecutive warps of a CTA (gw in {1,2,4,8}) that owns one
// canonical sum of width Pw <= 32*gw; thread p of the group holds partial p.
struct Group {
  int gw;      // warps
  int p;       // thread index within the group
  int bar_id;  // named barrier id (unused when gw == 1)
  __device__ void sync() const {
    if (gw == 1)
      __syncwarp();
    else
      named_bar(bar_id, 32 * gw);
  }
};

// Canonical tree over the partials held by threads p < min(Pw, K); the result
// is valid in thread p == 0.  sm: Pw scratch entries owned by this group.
template <class T>
__device__ T group_tree(T acc, const Group& g, int Pw, int K, T* sm) {
  if (Pw > 32) {
    if (g.p < Pw && g.p < K) sm[g.p] = acc;
    g.sync();
    for (int off = Pw / 2; off >= 32; off >>= 1) {
      if (g.p < off && g.p + off < K) sm[g.p] = add_v(sm[g.p], sm[g.p + off]);
      g.sync();
    }
    if (g.p < 32 && g.p < K) acc = sm[g.p];
  }
  if (g.p < 32) {
#pragma unroll 1
    for (int off = 16; off >= 1; off >>= 1) {
      T other = shfl_down_r(acc, off);
      if (g.p < off && g.p + off < K) acc = add_v(acc, other);
    }
  }
  return acc;
}

__device__ __forceinline__ double nan_max(double a, double b) {
  if (isnan(a) || isnan(b)) return bitsd(0x7ff8000000000000ull);
  return b > a ? b : a;
}

// block-wide NaN-propagating max; every thread gets the result
__device__ double block_nan_max(double v, double* s_red) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = nan_max(v, __shfl_xor_sync(0xffffffffu, v, off));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  double r = s_red[0];
  for (int w = 1; w < kWarps; ++w) r = nan_max(r, s_red[w]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ int pow2ceil_d(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
__device__ __forceinline__ int width_eval_d(int K) { return min(256, max(32, pow2ceil_d((K + 15) / 16))); }

// Shared-memory scratch of one CTA.
template <class R>
struct Smem {
  cplx<R> tree[kThreads];   // group tree partials
  cplx<R> bcast[kWarps][2]; // per-group broadcast slots (double-buffered)
  R rbcast[kWarps][2];
  int ibcast[kWarps][2];
  cplx<R> xbs[2];           // back-substitution broadcast
  double red[kWarps];
  int flag;
};

// ---------------------------------------------------------------------------
// (1) evaluation and differentiation
// ---------------------------------------------------------------------------
template <class R>
__device__ void weights(const DevPlan& P, double t, cplx<R>& wS, R& wT) {
  const R omt = r_sub(rconst<R>(1.0), rconst<R>(t));
  const R a = r_powi(omt, (unsigned)P.relax_k);
  wT = r_powi(rconst<R>(t), (unsigned)P.relax_k);
  const cplx<R> gam = load_c<R>(P.gamma, 1, 0);
  wS = c_scale(gam, a);
}

// Reverse-mode value + partials of every monomial.
// Prefix products F[j] are parked in the slot of partial j+1 and consumed by
// the backward sweep, so the workspace is the only scratch.
template <class R>
__device__ void eval_monomials(const DevPlan& P, const Work& W, int tid, int nthreads) {
  const long S = P.ws_len;
  for (int q = tid; q < P.M; q += nthreads) {
    const int m = P.mono_size[q];
    const int vb = P.mono_vbeg[q];
    const long out = P.mono_out[q];
    auto Y = [&](int k) { return load_c<R>(W.x, P.n, P.mono_var[vb + k]); };
    auto put = [&](int p, const cplx<R>& v) { store_c<R>(W.ws, S, out + 32L * p, v); };
    auto get = [&](int p) { return load_c<R>(W.ws, S, out + 32L * p); };
    if (m == 1) {
      put(0, Y(0));
      put(1, c_one<R>());
    } else if (m == 2) {
      const cplx<R> y0 = Y(0), y1 = Y(1);
      put(0, c_mul(y0, y1));
      put(1, y1);
      put(2, y0);
    } else {
      cplx<R> F = Y(0);
      put(2, F);
      for (int k = 1; k <= m - 2; ++k) {
        F = c_mul(F, Y(k));
        put(k + 2, F);
      }
      put(0, c_mul(F, Y(m - 1)));
      cplx<R> B = Y(m - 1);
      for (int k = m - 2; k >= 1; --k) {
        put(k + 1, c_mul(get(k + 1), B));
        B = c_mul(Y(k), B);
      }
      put(1, B);
    }
    if (P.mono_flags[q] & 1) {  // exponents >= 2
      cplx<R> cf = c_one<R>();
      bool have = false;
      for (int k = 0; k < m; ++k) {
        const int e = P.mono_exp[vb + k];
        if (e < 2) continue;
        const cplx<R> pk = c_powi(Y(k), (unsigned)(e - 1));
        cf = have ? c_mul(cf, pk) : pk;
        have = true;
      }
      put(0, c_mul(get(0), cf));
      for (int k = 0; k < m; ++k) {
        cplx<R> d = c_mul(get(1 + k), cf);
        const int e = P.mono_exp[vb + k];
        if (e >= 2) d = c_scale(d, rconst<R>((double)e));
        put(1 + k, d);
      }
    }
  }
}

// Canonical sum of one contribution list by a group; valid at g.p == 0.
template <class R>
__device__ cplx<R> slot_sum(const DevPlan& P, const Work& W, const Group& g, int beg, int K, cplx<R>* sm) {
  const int Pw = width_eval_d(K);
  cplx<R> acc = c_zero<R>();
  if (g.p < Pw && g.p < K) {
    for (int r = g.p; r < K; r += Pw) {
      const int ci = P.ctr_coef[beg + r];
      const int wi = P.ctr_ws[beg + r];
      const cplx<R> c = load_c<R>(P.coef, P.n_coef, ci);
      const cplx<R> v = wi < 0 ? c : c_mul(c, load_c<R>(W.ws, P.ws_len, wi));
      acc = (r == g.p) ? v : c_add(acc, v);
    }
  }
  return group_tree(acc, g, Pw, K, sm);
}

template <class R, class Team>
__device__ void eval_slots(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, double t) {
  cplx<R> wS;
  R wT;
  weights<R>(P, t, wS, wT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long SA = (long)P.N * (P.n + 1);
  for (int c = 0; c < 4; ++c) {
    const int gw = 8 >> c;
    const int gpc = kWarps / gw;
    const int gi = warp / gw;
    Group g{gw, (warp % gw) * 32 + lane, 1 + gi};
    cplx<R>* sm = sh.tree + gi * 32 * gw;
    const int ngroups = team.nblocks * gpc;
    const int beg = P.class_beg[c], end = P.class_beg[c + 1];
    for (int ti = beg + team.block * gpc + gi; ti < end; ti += ngroups) {
      const ptplan::SlotTask tk = P.tasks[ti];
      const cplx<R> Sg = slot_sum<R>(P, W, g, tk.g_beg, tk.g_cnt, sm);
      cplx<R> Sf;
      bool have_f;
      if (tk.f_cnt < 0) {
        Sf = Sg;
        have_f = tk.g_cnt > 0;
      } else {
        Sf = slot_sum<R>(P, W, g, tk.f_beg, tk.f_cnt, sm);
        have_f = tk.f_cnt > 0;
      }
      if (g.p == 0) {
        const bool have_g = tk.g_cnt > 0;
        cplx<R> h = c_zero<R>();
        if (have_g || have_f) {
          const cplx<R> zero = c_zero<R>();
          h = c_add(c_mul(wS, have_g ? Sg : zero), c_scale(have_f ? Sf : zero, wT));
        }
        if (tk.col == P.n) {
          store_c<R>(W.A, SA, (long)P.n * P.N + tk.row, c_neg(h));
          W.hmod[tk.row] = c_mod_double(h);
        } else {
          store_c<R>(W.A, SA, (long)tk.col * P.N + tk.row, h);
        }
      }
      g.sync();  // protect the group scratch before the next task
    }
  }
}

// ---------------------------------------------------------------------------
// (2) MGS least squares on [J | -h]
// ---------------------------------------------------------------------------
template <class R>
__device__ R group_bcast_r(const Group& g, int gi, R v, Smem<R>& sh, int& phase) {
  if (g.p == 0) sh.rbcast[gi][phase] = v;
  g.sync();
  R r = sh.rbcast[gi][phase];
  phase ^= 1;
  return r;
}
template <class R>
__device__ cplx<R> group_bcast_c(const Group& g, int gi, const cplx<R>& v, Smem<R>& sh, int& phase) {
  if (g.p == 0) sh.bcast[gi][phase] = v;
  g.sync();
  cplx<R> r = sh.bcast[gi][phase];
  phase ^= 1;
  return r;
}

// Normalise column k (already projected against q_0..q_{k-1}) and publish it.
// Returns false on rank deficiency (flag still published so nobody hangs).
template <class R, class Team>
__device__ bool mgs_normalize(const DevPlan& P, const Work& W, const Team& team, const Group& g, int gi,
                              Smem<R>& sh, int& phase, int k, unsigned long long epoch, double sqrt_eps) {
  const int N = P.N, Pm = P.P_mgs;
  const long SA = (long)N * (P.n + 1);
  const double* colk = W.A + (long)k * N;
  R acc = rconst<R>(0.0);
  if (g.p < Pm && g.p < N) {
    for (int i = g.p; i < N; i += Pm) {
      const R v = c_norm_sqr(load_c<R>(colk, SA, i));
      acc = (i == g.p) ? v : r_add(acc, v);
    }
  }
  R* rsm = reinterpret_cast<R*>(sh.tree + (gi * 32 * g.gw));
  const R nrm2 = group_tree(acc, g, Pm, N, rsm);
  int ok = 0;
  R inv = rconst<R>(0.0);
  if (g.p == 0) {
    const R rkk = r_sqrt(nrm2);
    const double d = r_hi(rkk);
    const double prev = k > 0 ? W.rmaxp[k - 1] : 0.0;
    const double mx = d > prev ? d : prev;
    ok = d > sqrt_eps * mx;
    W.rmaxp[k] = mx;
    if (ok) {
      inv = r_div(rconst<R>(1.0), rkk);
      store_r<R>(W.inv, P.n, k, inv);
      store_c<R>(W.Rm, (long)P.n * (P.n + 1), (long)k * P.n + k, cplx<R>{rkk, rconst<R>(0.0)});
    }
    sh.ibcast[gi][phase] = ok;
  }
  inv = group_bcast_r<R>(g, gi, inv, sh, phase);
  ok = sh.ibcast[gi][phase ^ 1];
  if (ok) {
    double* ck = W.A + (long)k * N;
    for (int i = g.p; i < N; i += 32 * g.gw) store_c<R>(ck, SA, i, c_scale(load_c<R>(ck, SA, i), inv));
  }
  g.sync();
  if (g.p == 0) {
    if (!ok) atomicExch(W.ctl + CTL_RANK, epoch);
    __threadfence();
    st_release(W.flags + k, epoch);
  }
  return ok != 0;
}

template <class R, class Team>
__device__ void mgs_project(const DevPlan& P, const Work& W, const Group& g, int gi, Smem<R>& sh, int& phase,
                            int k, int j) {
  const int N = P.N, n = P.n, Pm = P.P_mgs;
  const long SA = (long)N * (n + 1);
  const double* qk = W.A + (long)k * N;
  double* aj = W.A + (long)j * N;
  cplx<R> acc = c_zero<R>();
  if (g.p < Pm && g.p < N) {
    for (int i = g.p; i < N; i += Pm) {
      const cplx<R> v = c_conj_mul(load_c<R>(qk, SA, i), load_c<R>(aj, SA, i));
      acc = (i == g.p) ? v : c_add(acc, v);
    }
  }
  cplx<R>* sm = sh.tree + gi * 32 * g.gw;
  cplx<R> rkj = group_tree(acc, g, Pm, N, sm);
  if (g.p == 0) store_c<R>(W.Rm, (long)n * (n + 1), (long)j * n + k, rkj);
  rkj = group_bcast_c<R>(g, gi, rkj, sh, phase);
  if (j < n || k < n - 1) {
    for (int i = g.p; i < N; i += 32 * g.gw)
      store_c<R>(aj, SA, i, c_sub(load_c<R>(aj, SA, i), c_mul(rkj, load_c<R>(qk, SA, i))));
  }
  g.sync();
}

// Column-pipelined right-looking MGS.  Column j is owned
// by group j mod G; the owner of column k+1 normalises it as soon as q_k has
// been applied, so the sqrt/reciprocal chain overlaps the bulk updates.
template <class R, class Team>
__device__ void mgs(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, unsigned long long epoch,
                    double sqrt_eps) {
  const int n = P.n;
  const int gm = P.P_mgs / 32;
  const int gpc = kWarps / gm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gi = warp / gm;
  const Group g{gm, (warp % gm) * 32 + lane, 1 + gi};
  const int G = team.nblocks * gpc;
  const int me = team.block * gpc + gi;
  int phase = 0;
  bool alive = true;
  if (me > n) return;  // owns no column
  const int last_owned = me + ((n - me) / G) * G;
  if (me == 0) alive = mgs_normalize<R, Team>(P, W, team, g, gi, sh, phase, 0, epoch, sqrt_eps);
  for (int k = 0; k < n && alive && k < last_owned; ++k) {
    if (k % G != me) {
      if (g.p == 0) sh.ibcast[gi][phase] = wait_flag(W.flags + k, epoch, W.ctl) ? 1 : 0;
      g.sync();
      const int okw = sh.ibcast[gi][phase];
      phase ^= 1;
      if (!okw) return;
      if (ld_acquire(W.ctl + CTL_RANK) == epoch) return;
    }
    // first owned column > k
    int j = k + 1 + ((me - (k + 1)) % G + G) % G;
    for (; j <= n; j += G) {
      mgs_project<R, Team>(P, W, g, gi, sh, phase, k, j);
      if (j == k + 1 && j < n) {
        if (!mgs_normalize<R, Team>(P, W, team, g, gi, sh, phase, j, epoch, sqrt_eps)) alive = false;
      }
    }
  }
}

// Back substitution R dx = y, dx_k = (y_k - sum_{j>k} r_kj dx_j) * (1/r_kk),
// column-oriented (one CTA); then u = max|dx| and x += dx.
template <class R>
__device__ double backsub_update(const DevPlan& P, const Work& W, Smem<R>& sh) {
  const int n = P.n;
  const long SR = (long)n * (n + 1);
  cplx<R> acc[kMaxRowsPerThread];
#pragma unroll
  for (int r = 0; r < kMaxRowsPerThread; ++r) {
    const int i = threadIdx.x + r * kThreads;
    if (i < n) acc[r] = load_c<R>(W.Rm, SR, (long)n * n + i);
  }
  for (int j = n - 1; j >= 0; --j) {
    const int owner = j % kThreads, orow = j / kThreads;
    if ((int)threadIdx.x == owner) {
      cplx<R> a;
#pragma unroll
      for (int r = 0; r < kMaxRowsPerThread; ++r)
        if (r == orow) a = acc[r];
      const cplx<R> xj = c_scale(a, load_r<R>(W.inv, n, j));
#pragma unroll
      for (int r = 0; r < kMaxRowsPerThread; ++r)
        if (r == orow) acc[r] = xj;  // row j finished: acc now holds dx_j
      sh.xbs[j & 1] = xj;
    }
    __syncthreads();
    const cplx<R> xj = sh.xbs[j & 1];
#pragma unroll
    for (int r = 0; r < kMaxRowsPerThread; ++r) {
      const int i = threadIdx.x + r * kThreads;
      if (i < j) acc[r] = c_sub(acc[r], c_mul(load_c<R>(W.Rm, SR, (long)j * n + i), xj));
    }
  }
  double u = 0.0;
#pragma unroll
  for (int r = 0; r < kMaxRowsPerThread; ++r) {
    const int i = threadIdx.x + r * kThreads;
    if (i < n) {
      u = nan_max(u, c_mod_double(acc[r]));
      store_c<R>(W.dx, n, i, acc[r]);
      store_c<R>(W.x, n, i, c_add(load_c<R>(W.x, n, i), acc[r]));
    }
  }
  return block_nan_max(u, sh.red);
}

// ---------------------------------------------------------------------------
// (3) predictor -- one CTA
// ---------------------------------------------------------------------------
struct History {
  double t[kMaxDegree + 1];
  int count, next, cap;
  __device__ int slot(int j) const { return (next - count + j + 2 * cap) % cap; }  // j-th oldest
};

template <class R>
__device__ void predict(const DevPlan& P, const Work& W, const History& H, double tau) {
  const int n = P.n, d = H.count - 1;
  const long HS = 2L * limbs_of<R>::L * n;
  for (int i = threadIdx.x; i < n; i += kThreads) {
    cplx<R> D[kMaxDegree + 1];
    for (int j = 0; j <= d; ++j) D[j] = load_c<R>(W.hist + (long)H.slot(j) * HS, n, i);
    for (int l = 1; l <= d; ++l) {
      for (int j = d; j >= l; --j) {
        const R inv = r_div(rconst<R>(1.0), r_sub(rconst<R>(H.t[H.slot(j)]), rconst<R>(H.t[H.slot(j - l)])));
        D[j] = c_scale(c_sub(D[j], D[j - 1]), inv);
      }
    }
    cplx<R> p = D[d];
    for (int j = d - 1; j >= 0; --j)
      p = c_add(D[j], c_scale(p, r_sub(rconst<R>(tau), rconst<R>(H.t[H.slot(j)]))));
    store_c<R>(W.x, n, i, p);
  }
}

template <class R>
__device__ void push_history(const DevPlan& P, const Work& W, History& H, double t) {
  const int n = P.n;
  const long HS = 2L * limbs_of<R>::L * n;
  double* dst = W.hist + (long)H.next * HS;
  for (int i = threadIdx.x; i < n; i += kThreads) store_c<R>(dst, n, i, load_c<R>(W.x, n, i));
  H.t[H.next] = t;
  H.next = (H.next + 1) % H.cap;
  H.count = H.count < H.cap ? H.count + 1 : H.cap;
}

// ---------------------------------------------------------------------------
// Newton (Fig. 2) and the tracker (Fig. 3)
// ---------------------------------------------------------------------------
template <class R>
__device__ __forceinline__ double kSqrtEps();
template <>
__device__ __forceinline__ double kSqrtEps<double>() {
  return 0x1p-26;  // sqrt(2^-52)
}
template <>
__device__ __forceinline__ double kSqrtEps<dd>() {
  return 0x1p-52;  // sqrt(2^-104)
}
template <>
__device__ __forceinline__ double kSqrtEps<qd>() {
  return 0x1.6a09e667f3bcdp-105;  // sqrt(2^-209) rounded to binary64
}

struct NewtonOut {
  int ok, kind, iters;
  double residual, update;
  int solves;
};

template <class R, class Team>
__device__ NewtonOut newton(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh,
                            const pt_step_params& sp, double t, unsigned long long& epoch) {
  NewtonOut o{0, NW_ITERATION_BUDGET, 0, -1.0, -1.0, 0};
  const double sqrt_eps = kSqrtEps<R>();
  double last = bitsd(0x7ff0000000000000ull);
  const int tid = team.block * kThreads + threadIdx.x, nth = team.nblocks * kThreads;
  for (int it = 1; it <= sp.newton_max_iter; ++it) {
    o.iters = it;
    eval_monomials<R>(P, W, tid, nth);
    if (!team.sync(&sh.flag)) return {0, NW_ABORT, it, -1.0, -1.0, 0};
    eval_slots<R, Team>(P, W, team, sh, t);
    if (!team.sync(&sh.flag)) return {0, NW_ABORT, it, -1.0, -1.0, 0};
    double r = 0.0;
    for (int i = threadIdx.x; i < P.N; i += kThreads) r = nan_max(r, W.hmod[i]);
    r = block_nan_max(r, sh.red);
    o.residual = r;
    if (r > last) {
      o.kind = NW_RESIDUAL_INCREASE;
      return o;
    }
    if (r < sp.newton_tol) {
      o.ok = 1;
      o.kind = NW_OK;
      return o;
    }
    ++epoch;
    mgs<R, Team>(P, W, team, sh, epoch, sqrt_eps);
    if (!team.sync(&sh.flag)) return {0, NW_ABORT, it, -1.0, -1.0, 0};
    if (ld_acquire(W.ctl + CTL_RANK) == epoch) {
      o.kind = NW_LINEAR_SOLVE;
      return o;
    }
    if (team.block == 0) {
      const double u = backsub_update<R>(P, W, sh);
      if (threadIdx.x == 0) W.scal[0] = u;
    }
    if (!team.sync(&sh.flag)) return {0, NW_ABORT, it, -1.0, -1.0, 0};
    const double u = *(volatile double*)(W.scal);
    ++o.solves;
    o.update = u;
    if (u < sp.newton_tol) {
      o.ok = 1;
      o.kind = NW_OK;
      return o;
    }
    last = r;
  }
  return o;
}

struct TrackIO {
  const double* start;  // [2L][n]
  double* end;          // [2L][n]
  pt_path_stats* stats;
  pt_trace_event* trace;
  int trace_cap;
  int* trace_len;
};

template <class R, class Team>
__device__ void track_path(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh,
                           const pt_step_params& sp, const TrackIO& io, unsigned long long epoch_base) {
  const int n = P.n;
  unsigned long long epoch = epoch_base;
  const bool leader = team.block == 0;
  pt_path_stats st{};
  if (leader)
    for (int i = threadIdx.x; i < n; i += kThreads) store_c<R>(W.x, n, i, load_c<R>(io.start, n, i));
  if (!team.sync(&sh.flag)) return;
  NewtonOut o = newton<R, Team>(P, W, team, sh, sp, 0.0, epoch);
  if (o.kind == NW_ABORT) return;
  st.start_iters = o.iters;
  st.newton_iters = o.iters;
  st.solves = o.solves;
  st.final_residual = o.residual;
  st.final_update = o.update;
  History H;
  H.count = 0;
  H.next = 0;
  H.cap = sp.pred_degree + 1;
  int ntrace = 0;
  if (!o.ok) {
    st.status = PT_PATH_FAIL;
    st.failure_kind = PT_FAIL_START;
    st.t_end = 0.0;
    if (leader)
      for (int i = threadIdx.x; i < n; i += kThreads) store_c<R>(io.end, n, i, load_c<R>(W.x, n, i));
  } else {
    if (leader) push_history<R>(P, W, H, 0.0);
    else H.count = 1;
    double tacc = 0.0, dt = sp.max_step;
    int succ = 0, steps = 0, accepted = 0;
    while (tacc < 1.0) {
      if (steps > sp.max_steps) {
        st.status = PT_PATH_FAIL;
        st.failure_kind = PT_FAIL_MAX_STEPS;
        break;
      }
      const double tsum = add64(tacc, dt);
      const double ttrial = tsum < 1.0 ? tsum : 1.0;
      if (leader) predict<R>(P, W, H, ttrial);
      if (!team.sync(&sh.flag)) return;
      o = newton<R, Team>(P, W, team, sh, sp, ttrial, epoch);
      if (o.kind == NW_ABORT) return;
      st.newton_iters += o.iters;
      st.solves += o.solves;
      st.final_residual = o.residual;
      st.final_update = o.update;
      if (leader && threadIdx.x == 0 && io.trace && ntrace < io.trace_cap)
        io.trace[ntrace] = pt_trace_event{ttrial, o.ok, o.iters, o.residual, o.update};
      ++ntrace;
      ++steps;
      if (o.ok) {
        tacc = ttrial;
        if (leader) {
          __syncthreads();
          push_history<R>(P, W, H, ttrial);
        }
        ++accepted;
        ++succ;
        if (succ > 2) {
          const double two = mul64(2.0, dt);
          dt = sp.max_step < two ? sp.max_step : two;
        }
      } else {
        succ = 0;
        dt = div64(dt, 2.0);
        if (dt < sp.min_step) {
          st.status = PT_PATH_FAIL;
          st.failure_kind = PT_FAIL_MIN_STEP;
          break;
        }
      }
    }
    st.steps = steps;
    st.accepted = accepted;
    st.t_end = tacc;
    if (leader) {
      __syncthreads();
      const long HS = 2L * limbs_of<R>::L * n;
      const double* newest = W.hist + (long)H.slot(H.count - 1) * HS;
      for (int i = threadIdx.x; i < n; i += kThreads) store_c<R>(io.end, n, i, load_c<R>(newest, n, i));
    }
  }
  if (leader && threadIdx.x == 0) {
    *io.stats = st;
    if (io.trace_len) *io.trace_len = ntrace;
  }
}

}  // namespace ptdev
