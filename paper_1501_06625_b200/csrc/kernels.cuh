// kernels.cuh -- every __global__ kernel of the tracker library.
//
//   k_track_grid<R>     one path, cooperative persistent grid (GridTeam)
//   k_track_cluster<R>  one path, one thread-block cluster (ClusterTeam)
//   k_track_batch<R>    many paths, one CTA per path, atomic path queue
//   k_eval<R>           evaluate_homotopy only (parity tests)
//   k_lstsq<R>          least_squares_solve only (parity tests)
//   k_arith<R>          bulk scalar ops (arithmetic parity tests)
// Instantiated once per precision in kern_{d,dd,qd}.cu (separate TUs so the
// three ptxas runs proceed in parallel); tracker.cu launches them through
// the KernelSet tables (kernel_set.hpp).
#pragma once

#include "device.cuh"
#include "kernel_set.hpp"

namespace ptdev {
// Per-path workspace layout (element counts); slice b of a batch starts at
// b * dslice doubles / b * uslice u64 words.
struct Layout {
  long x, hist, ws, A, Rm, inv, rmaxp, hmod, scal, dx, qg;  // double offsets
  long dslice;
  long flags, ctl, prof;  // u64 offsets
  long uslice;
};

inline Layout make_layout(int L, int n, int N, long ws_len) {
  Layout o{};
  long d = 0;
  auto take = [&](long cnt) {
    long at = d;
    d += (cnt + 31) & ~31L;  // 256-byte aligned sub-arrays
    return at;
  };
  o.x = take(2L * L * n);
  o.hist = take((long)(kMaxDegree + 1) * 2 * L * n);
  o.ws = take(2L * L * ws_len);
  o.A = take(2L * L * N * (n + 1));
  o.Rm = take(2L * L * n * (n + 1));
  o.inv = take((long)L * n);
  o.rmaxp = take(n);
  o.hmod = take(N);
  o.scal = take(8);
  o.dx = take(2L * L * n);
  o.qg = take((long)n * mgs_warp_qs(L, N));
  o.dslice = d;
  long u = 0;
  o.flags = u;
  u += (n + 1 + 31) & ~31L;
  o.ctl = u;
  u += 32;
  o.prof = u;
  u += kProfSlots + 14 * (n + 2) + 32;  // + per-column fine markers (PT_MGS_FINE builds)
  o.uslice = u;
  return o;
}

__host__ __device__ inline Work carve(double* dbase, unsigned long long* ubase, const Layout& o, long b) {
  double* d = dbase + b * o.dslice;
  unsigned long long* u = ubase + b * o.uslice;
  Work W;
  W.x = d + o.x;
  W.hist = d + o.hist;
  W.ws = d + o.ws;
  W.A = d + o.A;
  W.Rm = d + o.Rm;
  W.inv = d + o.inv;
  W.rmaxp = d + o.rmaxp;
  W.hmod = d + o.hmod;
  W.scal = d + o.scal;
  W.dx = d + o.dx;
  W.qg = d + o.qg;
  W.flags = u + o.flags;
  W.ctl = u + o.ctl;
  W.prof = u + o.prof;
  return W;
}

// kern_dd.cu (-DPT_DD_FAST_NONFINITE) and kern_dd_exact.cu instantiate the same
// templates with different device bodies: the kernels live in an inline
// namespace per variant, so the two host stubs are distinct symbols (one
// weak symbol would silently serve both kernel sets).
#if defined(PT_DD_FAST_NONFINITE)
#define PT_KVARIANT kv_fastnf
#elif defined(PT_QD_FAST)
#define PT_KVARIANT kv_qdfast
#else
#define PT_KVARIANT kv_exact
#endif
inline namespace PT_KVARIANT {
// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// Per-launch CTA prologue: MGS sweep counter and, for the mbarrier exchange
// of the warp MGS, one receive barrier per column (phase = sweep parity).
// The caller's team barrier publishes the initialisation.
template <class R>
__device__ void cta_prologue(const DevPlan& P, Smem<R>& sh, double* dyn_smem, int nblocks) {
  if (threadIdx.x == 0) {
    sh.mgs_seq = 0;
    if (P.mgs_warp == 2) {
      constexpr int L = limbs_of<R>::L;
      uint64_t* bars = reinterpret_cast<uint64_t*>(dyn_smem + mgs_warp_slots_doubles(L, P.N, P.n, nblocks) +
                                                   (long)P.n * mgs_warp_qs(L, P.N));
      for (int k = 0; k < P.n; ++k) mbar_init(bars + k, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
}

// CTAs per SM of the cooperative grid engine (k_track_grid, k_eval): two in
// D / DD (128 registers, twice the warps to hide the L2 latency of the slot
// sums: rand-96 DD evaluation 1.03 -> 0.90 ms, a 3-step prefix 39.5 -> 34.2
// ms), one in QD (at 128 registers the QD chains spill: cyclic-256 QD
// evaluation 19.4 -> 24.7 ms).
template <class R>
constexpr int kGridCtasPerSm = limbs_of<R>::L == 4 ? 1 : 2;
template <class R>
__global__ void __launch_bounds__(kThreads, kGridCtasPerSm<R>)
    k_track_grid(DevPlan P, Work W, pt_step_params sp, TrackIO io, unsigned long long epoch_base) {
  __shared__ Smem<R> sh;
  extern __shared__ double dyn_smem[];
  const GridTeam team{W.ctl, (int)gridDim.x, (int)blockIdx.x, nullptr};
  cta_prologue<R>(P, sh, dyn_smem, (int)gridDim.x);
  __syncthreads();
  track_path<R, GridTeam>(P, W, team, sh, P.dyn_smem ? dyn_smem : nullptr, sp, io, epoch_base);
}

// One path on one thread-block cluster (launched with a cluster dimension
// attribute, grid == cluster): barrier.cluster + DSMEM column exchange.
template <class R>
__global__ void __launch_bounds__(kThreads, 1)
    k_track_cluster(DevPlan P, Work W, pt_step_params sp, TrackIO io, unsigned long long epoch_base) {
  __shared__ Smem<R> sh;
  __shared__ uint32_t s_flags[kMaxCols];
  extern __shared__ double dyn_smem[];
  for (int i = threadIdx.x; i < kMaxCols; i += kThreads) s_flags[i] = 0;
  const ClusterTeam team{W.ctl, (int)cluster_nranks(), (int)cluster_rank(), s_flags};
  cta_prologue<R>(P, sh, dyn_smem, team.nblocks);
  team.sync(&sh.flag);
  track_path<R, ClusterTeam>(P, W, team, sh, P.dyn_smem ? dyn_smem : nullptr, sp, io, epoch_base);
  team.sync(&sh.flag);  // keep every CTA's shared memory alive until all DSMEM reads are done
}

// Batch CTAs per SM: two paths share an SM in D / DD (128 registers per
// thread suffice there); QD keeps the whole register file for one path.
#ifndef PT_BATCH_CTAS
#define PT_BATCH_CTAS 2
#endif
template <class R>
constexpr int kBatchCtasPerSm = limbs_of<R>::L == 4 ? 1 : PT_BATCH_CTAS;

template <class R>
__global__ void __launch_bounds__(kThreads, kBatchCtasPerSm<R>)
    k_track_batch(DevPlan P, double* dbase, unsigned long long* ubase, Layout lay, pt_step_params sp,
                  const double* starts, double* ends, pt_path_stats* stats, int n_paths,
                  unsigned long long* queue, unsigned long long epoch_base, int retrack) {
  __shared__ Smem<R> sh;
  __shared__ int s_path;
  __shared__ uint32_t s_flags[kMaxCols];
  extern __shared__ double dyn_smem[];
  for (int i = threadIdx.x; i < kMaxCols; i += kThreads) s_flags[i] = 0;
  const Work W = carve(dbase, ubase, lay, blockIdx.x);
  const BlockTeam team{W.ctl, 1, 0, s_flags};
  if (threadIdx.x < CTL_WORDS) W.ctl[threadIdx.x] = 0ull;  // this CTA's slice: abort / rank words of the last launch
  cta_prologue<R>(P, sh, dyn_smem, 1);
  __syncthreads();
  const long PS = 2L * limbs_of<R>::L * P.n;
  for (;;) {
    if (threadIdx.x == 0) s_path = (int)atomicAdd(queue, 1ull);
    // MGS column flags are compared on the low 31 bits of the epoch: clear
    // them per path so they only have to be unique within one path
    for (int i = threadIdx.x; i < kMaxCols; i += kThreads) s_flags[i] = 0;
    __syncthreads();
    const int p = s_path;
    __syncthreads();
    if (p >= n_paths) break;
    // exact re-track launch: only the paths whose fast run met a non-finite value
    if (retrack && !(((volatile const pt_path_stats*)(stats + p))->flags & PT_STAT_NONFINITE)) continue;
    TrackIO io{starts + p * PS, ends + p * PS, stats + p, nullptr, 0, nullptr, 0};
    track_path<R, BlockTeam>(P, W, team, sh, P.dyn_smem ? dyn_smem : nullptr, sp, io,
                             epoch_base + ((unsigned long long)p << 16));
    // watchdog abort (the stats of path p say PT_FAIL_ABORT): this CTA's
    // exchange state is no longer trustworthy -- stop taking paths, tell the host
    if (ld_acquire(W.ctl + CTL_ABORT)) {
      if (threadIdx.x == 0) atomicOr(queue + 1, 1ull);
      break;
    }
  }
}

template <class R>
__global__ void __launch_bounds__(kThreads, kGridCtasPerSm<R>)
    k_eval(DevPlan P, Work W, const double* x, double t, double* h, double* J, double* rmax) {
  __shared__ Smem<R> sh;
  const GridTeam team{W.ctl, (int)gridDim.x, (int)blockIdx.x, nullptr};
  const int n = P.n, N = P.N;
  if (team.block == 0)
    for (int i = threadIdx.x; i < n; i += kThreads) store_c<R>(W.x, n, i, load_c<R>(x, n, i));
  if (!team.sync(&sh.flag)) return;
  eval_monomials<R>(P, W, W.x, team.block * kThreads + threadIdx.x, team.nblocks * kThreads);
  if (!team.sync(&sh.flag)) return;
  eval_slots<R, GridTeam>(P, W, team, sh, t);
  if (!team.sync(&sh.flag)) return;
  const long SA = (long)N * (n + 1), SJ = (long)N * n;
  const long tid = (long)team.block * kThreads + threadIdx.x, nth = (long)team.nblocks * kThreads;
  if (J)
    for (long q = tid; q < SJ; q += nth) store_c<R>(J, SJ, q, load_c<R>(W.A, SA, q));
  if (h)
    for (long i = tid; i < N; i += nth) store_c<R>(h, N, i, c_neg(load_c<R>(W.A, SA, (long)n * N + i)));
  if (team.block == 0) {
    double r = 0.0;
    for (int i = threadIdx.x; i < N; i += kThreads) r = nan_max(r, W.hmod[i]);
    r = block_nan_max(r, sh.red);
    if (threadIdx.x == 0 && rmax) *rmax = r;
  }
}

template <class R>
__global__ void __launch_bounds__(kThreads, 1) k_lstsq(DevPlan P, Work W, unsigned long long epoch, int* status) {
  __shared__ Smem<R> sh;
  extern __shared__ double dyn_smem[];
  const GridTeam team{W.ctl, (int)gridDim.x, (int)blockIdx.x, nullptr};
  cta_prologue<R>(P, sh, dyn_smem, (int)gridDim.x);
  __syncthreads();
  mgs<R, GridTeam>(P, W, team, sh, P.mgs_smem ? dyn_smem : nullptr, nullptr, epoch, kSqrtEps<R>());
  if (!team.sync(&sh.flag)) {
    if (team.block == 0 && threadIdx.x == 0) *status = PT_E_TIMEOUT;
    return;
  }
  if (ld_acquire(W.ctl + CTL_RANK) == epoch) {
    if (team.block == 0 && threadIdx.x == 0) *status = PT_E_RANK;
    return;
  }
  if (team.block == 0) {
    backsub_update<R>(P, W, sh);
    if (threadIdx.x == 0) *status = 0;
  }
}

template <class R>
__device__ R arith_rd(const double* p) {
  R v;
#pragma unroll
  for (int l = 0; l < limbs_of<R>::L; ++l) r_set_limb(v, l, p[l]);
  return v;
}
template <class R>
__host__ __device__ inline void arith_one(int op, const double* pa, const double* pb, double* po) {
  constexpr int L = limbs_of<R>::L;
  auto rd = [](const double* p) {
    R v;
    for (int l = 0; l < L; ++l) r_set_limb(v, l, p[l]);
    return v;
  };
  auto wr = [](const R& v, double* p) {
    for (int l = 0; l < L; ++l) p[l] = r_limb(v, l);
  };
  const R ar = rd(pa), br = rd(pb);
  const cplx<R> ac{rd(pa), rd(pa + L)}, bc{rd(pb), rd(pb + L)};
  cplx<R> oc;
  switch (op) {
    case 0: wr(r_add(ar, br), po); break;
    case 1: wr(r_sub(ar, br), po); break;
    case 2: wr(r_mul(ar, br), po); break;
    case 3: wr(r_mul_d(ar, pb[0]), po); break;
    case 4: wr(r_div(ar, br), po); break;
    case 5: wr(r_sqrt(ar), po); break;
    case 6:
      if constexpr (L == 4) {
        wr(qd_renormalize(ar), po);
      } else if constexpr (L == 2) {
        wr(dd_norm(r_limb(ar, 0), r_limb(ar, 1)), po);
      } else {
        wr(ar, po);
      }
      break;
    case 7: oc = c_mul(ac, bc); wr(oc.re, po); wr(oc.im, po + L); break;
    case 8: oc = c_add(ac, bc); wr(oc.re, po); wr(oc.im, po + L); break;
    case 9: oc = c_conj_mul(ac, bc); wr(oc.re, po); wr(oc.im, po + L); break;
    case 10: wr(c_norm_sqr(ac), po); break;
    case 11: po[0] = c_mod_double(ac); break;
    case 12: wr(r_powi(ar, (unsigned)pb[0]), po); break;
    case 14: oc = c_scale(ac, br); wr(oc.re, po); wr(oc.im, po + L); break;
    case 15: oc = c_powi(ac, (unsigned)pb[0]); wr(oc.re, po); wr(oc.im, po + L); break;
    default: break;
  }
}

template <class R>
__global__ void k_arith(int op, long count, const double* a, const double* b, double* out) {
  constexpr int L = limbs_of<R>::L;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x)
    arith_one<R>(op, a + i * 2 * L, b + i * 2 * L, out + i * 2 * L);
}

}  // inline namespace PT_KVARIANT
}  // namespace ptdev
