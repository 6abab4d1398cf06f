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

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "../../include/pathtrack_b200.h"
#include "mp.cuh"
#include "plan.hpp"

namespace ptdev {

using namespace ptk;

// every tracker CTA.  (Measured on the batch: 4 x 128-thread CTAs per SM
// instead of 2 x 256 cut the barrier stalls but almost doubled the
// instruction-cache stalls -- 4 CTAs in 4 different phases -- and ran 27 %
// slower.)
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRowsPerThread = 2;  // n <= 512
constexpr int kMaxDegree = 8;
constexpr double kTimeoutNs = 20e9;
constexpr int kMaxCols = 520;  // n + 1 <= 513 MGS columns (shared flag arrays)

enum { CTL_BAR_COUNT = 0, CTL_BAR_GEN = 1, CTL_ABORT = 2, CTL_RANK = 3, CTL_QUEUE = 4, CTL_NONFINITE = 5, CTL_WORDS = 8 };
enum { NW_OK = 0, NW_RESIDUAL_INCREASE = 1, NW_ITERATION_BUDGET = 2, NW_LINEAR_SOLVE = 3, NW_ABORT = 4 };

struct DevPlan {
  int n, N, M;
  int mono_long;  // leading monomials (size >= kMonoSplit) evaluated by lane pairs
  int P_mgs;   // canonical width of the MGS sums
  int mgs_gw;  // warps per MGS group (>= P_mgs/32; one element per thread when N <= 256)
  const int32_t* mono_size;
  const int32_t* mono_vbeg;
  const int32_t* mono_out;
  const int32_t* mono_flags;
  const int32_t* mono_var;
  const int32_t* mono_exp;
  long ws_len;
  const ptplan::SlotTask* tasks;
  int class_beg[6];
  const int32_t* ctr_coef;
  const int32_t* ctr_ws;
  const double* coef;
  long n_coef;
  const double* gamma;  // 2L limbs
  int relax_k;
  int mgs_smem;  // 1: MGS keeps owned columns in dynamic shared memory
  int dyn_smem;  // 1: the launch has dynamic shared memory (x copy, split scratch, staged R)
  int mgs_warp;  // 1: warp-per-column MGS + one-warp back substitution (mgs_warp.cuh, N <= 128)
  int mgs_B;     // warp MGS: consecutive columns per CTA block (divides kWarps)
  int bs_smem;   // warp back substitution stages R in CTA 0's dynamic shared memory
  int x_smem;    // monomial evaluation reads x from a per-CTA shared-memory copy
  int mgs_batch; // batch (BlockTeam, N <= 64): column-item MGS on a padded shared-memory matrix (mgs_batch)
  // batch only (BlockTeam): lane tasks as warp bundles over lane-interleaved
  // contribution streams (plan.hpp Bundle); bundles == nullptr: unbundled
  const ptplan::Bundle* bundles;
  int n_bundles;
  const int32_t* splits;  // split groups: (task_beg, ntasks, D, scratch base) x n_splits
  int n_splits;
  int scratch_units;      // 32-lane complex rows of split scratch (dynamic smem after the x copy)
  const ptplan::SlotTask* btasks;
  const int32_t* s_ws;
  const double* s_coef;
  long s_len;
  int s_hi;  // the stream holds only the leading limb of re / im (the others are +0.0)
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
  double* qg;     // [n][2L*N + 2] warp-MGS messages staged for the TMA multicast
  unsigned long long* flags;  // [n+1] MGS column-ready flags (epoch values)
  unsigned long long* ctl;    // [CTL_WORDS] barrier / abort / rank-fail
  unsigned long long* prof;   // [kProfSlots] phase time accumulators (ns, block 0)
};

// Phase timers: block 0 / thread 0 accumulates globaltimer deltas.
enum { PROF_MONO = 0, PROF_SLOTS = 1, PROF_MGS = 2, PROF_BACKSUB = 3, PROF_PREDICT = 4, PROF_ITERS = 5, kProfSlots = 8 };
// W.prof[kProfSlots + 6*j + {0..5}]: owner of column j, last MGS of the launch (debugging aid):
// globaltimer + clock64 when q_{j-1} was seen, clock64 after q loaded / projected / published, globaltimer at publish
struct PhaseClock {
  unsigned long long t;
  bool on;
  __device__ PhaseClock(bool enable) : t(0), on(enable) {
    if (on) t = gtimer_raw();
  }
  __device__ static unsigned long long gtimer_raw() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
  }
  __device__ void lap(unsigned long long* acc) {
    if (!on) return;
    const unsigned long long now = gtimer_raw();
    *acc += now - t;
    t = now;
  }
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
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ unsigned long long atom_add_release(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

// Wait until the flag word carries (epoch << 1) | bit; returns the bit
// (1 = the column failed the rank test), or -1 on abort / watchdog.
__device__ __forceinline__ int wait_flag(const unsigned long long* flag, unsigned long long epoch,
                                         unsigned long long* ctl) {
  const unsigned long long t0 = gtimer();
  unsigned int spins = 0;
  for (;;) {
    // relaxed polling (an acquire load would invalidate L1 on every poll),
    // one acquire fence once the flag is seen
    const unsigned long long v = ld_relaxed(flag);
    if ((v >> 1) == epoch) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      return (int)(v & 1ull);
    }
    if ((++spins & 255u) == 0) {
      if (ld_acquire(ctl + CTL_ABORT)) return -1;
      if ((double)(gtimer() - t0) > kTimeoutNs) {
        atomicExch(ctl + CTL_ABORT, 1ull);
        return -1;
      }
    }
  }
}

// --- shared-memory (DSMEM) primitives for the cluster engine ---------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_release_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cluster_u32(uint32_t cta_addr) {
  uint32_t v;
  asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(cta_addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nranks() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

// A team runs one path.  Besides a barrier it provides the MGS column
// exchange: publish(k) after the owner group has normalised column k,
// wait(k) before a consumer reads q_k, and q_src(k) = where q_k can be read.
//
// GridTeam: cooperative persistent grid; q_k is copied to the global matrix
// and announced by a release flag in global memory (through L2).
struct GridTeam {
  unsigned long long* ctl;
  int nblocks, block;
  static constexpr bool kGrid = true;
  static constexpr bool kQInGlobal = true;
  uint32_t* sflags;  // unused
  // Generation barrier; returns false once any CTA has aborted.
  __device__ bool sync(int* s_flag) const {
    __syncthreads();
    if (threadIdx.x == 0) {
      int abort = 0;
      const unsigned long long gen = ld_acquire(ctl + CTL_BAR_GEN);
      const unsigned long long arrived = atom_add_release(ctl + CTL_BAR_COUNT, 1ull);
      if (arrived == (unsigned long long)(nblocks - 1)) {
        atomicExch(ctl + CTL_BAR_COUNT, 0ull);
        st_release(ctl + CTL_BAR_GEN, gen + 1);
      } else {
        const unsigned long long t0 = gtimer();
        unsigned int spins = 0;
        while (ld_relaxed(ctl + CTL_BAR_GEN) == gen) {
          if ((++spins & 255u) == 0) {
            if (ld_acquire(ctl + CTL_ABORT)) {
              abort = 1;
              break;
            }
            if ((double)(gtimer() - t0) > kTimeoutNs) {
              atomicExch(ctl + CTL_ABORT, 1ull);
              abort = 1;
              break;
            }
          }
        }
      }
      __threadfence();
      *s_flag = abort;
    }
    __syncthreads();
    return *s_flag == 0;
  }
  __device__ void publish(unsigned long long* flags, int k, unsigned long long epoch, int fail) const {
    st_release(flags + k, (epoch << 1) | (unsigned long long)fail);
  }
  __device__ int wait(const unsigned long long* flags, int k, unsigned long long epoch) const {
    return wait_flag(flags + k, epoch, ctl);
  }
};

// ClusterTeam: one thread-block cluster (<= 16 CTAs) runs the path.  Barrier
// = barrier.cluster; q_k stays in the owner CTA's shared memory and is read
// through DSMEM; the owner pushes a release flag into every CTA's shared
// flag array, so consumers poll locally.
struct ClusterTeam {
  unsigned long long* ctl;
  int nblocks, block;
  static constexpr bool kGrid = false;
  static constexpr bool kQInGlobal = false;
  uint32_t* sflags;  // [n+1] per CTA (shared memory)
  __device__ bool sync(int*) const {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    return true;
  }
  __device__ void publish(unsigned long long*, int k, unsigned long long epoch, int fail) const {
    const uint32_t v = ((uint32_t)(epoch & 0x7fffffffull) << 1) | (uint32_t)fail;
    const uint32_t local = smem_u32(sflags + k);
    asm volatile("fence.acq_rel.cluster;" ::: "memory");  // one release fence, then relaxed remote flag stores
    for (int r = 0; r < nblocks; ++r)
      asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"r"(mapa_u32(local, (uint32_t)r)), "r"(v)
                   : "memory");
  }
  __device__ int wait(const unsigned long long*, int k, unsigned long long epoch) const {
    const uint32_t want = (uint32_t)(epoch & 0x7fffffffull);
    const uint32_t a = smem_u32(sflags + k);
    const unsigned long long t0 = gtimer();
    unsigned int spins = 0;
    for (;;) {
      uint32_t v;
      asm volatile("ld.relaxed.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
      if ((v >> 1) == want) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        return (int)(v & 1u);
      }
      if (++spins > 512u) __nanosleep(20);
      // Watchdog: a stalled exchange sets CTL_ABORT and gives up; every other
      // waiter sees the flag and gives up too, all CTAs still reach the next
      // cluster barrier (no CTA exits early, no __trap poisoning the context)
      // and newton() reports NW_ABORT after it.
      if ((spins & 1023u) == 0 && (ld_acquire(ctl + CTL_ABORT) || (double)(gtimer() - t0) > kTimeoutNs)) {
        atomicExch(ctl + CTL_ABORT, 1ull);
        return -1;
      }
    }
  }
};

struct BlockTeam {
  unsigned long long* ctl;
  int nblocks, block;  // 1, 0
  static constexpr bool kGrid = false;
  static constexpr bool kQInGlobal = false;
  uint32_t* sflags;  // [n+1] shared memory
  __device__ bool sync(int*) const {
    __syncthreads();
    return true;
  }
  __device__ void publish(unsigned long long*, int k, unsigned long long epoch, int fail) const {
    __threadfence_block();
    *(volatile uint32_t*)(sflags + k) = ((uint32_t)(epoch & 0x7fffffffull) << 1) | (uint32_t)fail;
  }
  // Flags are cleared at the start of every path (k_track_batch), so the low
  // 31 bits of the epoch only have to be unique within one path.
  __device__ int wait(const unsigned long long*, int k, unsigned long long epoch) const {
    const uint32_t want = (uint32_t)(epoch & 0x7fffffffull);
    const unsigned long long t0 = gtimer();
    for (unsigned int spins = 1;; ++spins) {
      const uint32_t v = *(volatile uint32_t*)(sflags + k);
      if ((v >> 1) == want) {
        __threadfence_block();
        return (int)(v & 1u);
      }
      if ((spins & 1023u) == 0 && (ld_acquire(ctl + CTL_ABORT) || (double)(gtimer() - t0) > kTimeoutNs)) {
        atomicExch(ctl + CTL_ABORT, 1ull);
        return -1;
      }
    }
  }
};

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
__device__ __forceinline__ double shfl0(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ dd shfl0(dd v, int src) {
  return {__shfl_sync(0xffffffffu, v.hi, src), __shfl_sync(0xffffffffu, v.lo, src)};
}
__device__ __forceinline__ qd shfl0(const qd& v, int src) {
  qd r;
#pragma unroll
  for (int l = 0; l < 4; ++l) r.c[l] = __shfl_sync(0xffffffffu, v.c[l], src);
  return r;
}
template <class R>
__device__ __forceinline__ cplx<R> shfl0(const cplx<R>& v, int src) {
  return {shfl0(v.re, src), shfl0(v.im, src)};
}

__device__ __forceinline__ double add_v(double a, double b) { return add64(a, b); }
__device__ __forceinline__ dd add_v(dd a, dd b) { return r_add(a, b); }
__device__ __forceinline__ qd add_v(const qd& a, const qd& b) { return r_add(a, b); }
template <class R>
__device__ __forceinline__ cplx<R> add_v(const cplx<R>& a, const cplx<R>& b) {
  return c_add(a, b);
}

// branch-free select (keeps independent chains in one basic block)
__device__ __forceinline__ double pick(bool c, double a, double b) { return c ? a : b; }
__device__ __forceinline__ dd pick(bool c, dd a, dd b) { return {c ? a.hi : b.hi, c ? a.lo : b.lo}; }
__device__ __forceinline__ qd pick(bool c, const qd& a, const qd& b) {
  qd r;
#pragma unroll
  for (int l = 0; l < 4; ++l) r.c[l] = c ? a.c[l] : b.c[l];
  return r;
}
template <class R>
__device__ __forceinline__ cplx<R> pick(bool c, const cplx<R>& a, const cplx<R>& b) {
  return {pick(c, a.re, b.re), pick(c, a.im, b.im)};
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
__device__ __forceinline__ T group_tree(T acc, const Group& g, int Pw, int K, T* sm) {
  if (Pw > 32) {
    if (g.p < Pw && g.p < K) sm[g.p] = acc;
    g.sync();
    for (int off = Pw / 2; off >= 32; off >>= 1) {
      if (g.p < off && g.p + off < K) sm[g.p] = add_v(sm[g.p], sm[g.p + off]);
      g.sync();
    }
    if (g.p < 32 && g.p < K) acc = sm[g.p];
  }
  // Warp levels: every warp of the group runs them (only warp 0's lanes
  // p < off, p + off < K add), so the shuffles are in provably converged
  // code -- under a lane-dependent branch nvcc falls back to the slow
  // WARPSYNC.COLLECTIVE shuffle emulation.
  __syncwarp();
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    T other = shfl_down_r(acc, off);
    acc = pick(g.p < off && g.p + off < K, add_v(acc, other), acc);
  }
  return acc;
}

__device__ __forceinline__ double nan_max(double a, double b) {
  if (isnan(a) || isnan(b)) return bitsd(0x7ff8000000000000ull);
  return b > a ? b : a;
}

// block-wide NaN-propagating max; every thread gets the result
__device__ inline double block_nan_max(double v, double* s_red) {
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
  double pmax[kMaxCols];    // MGS prefix max of r_kk (cluster / block teams)
  int flag;
  int mgs_seq;              // MGS sweeps completed by this CTA in this launch (mbarrier phase parity)
  int bundle_next;          // batch: next bundle to claim (reset before every evaluation)
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

// Exponents >= 2: Cf = prod y_k^(e_k-1), value *= Cf,
// partial k *= Cf, then *= e_k when e_k >= 2.
template <class R>
__device__ __forceinline__ void mono_exponents(const DevPlan& P, const Work& W, const double* xs, int q, int m, int vb,
                                               long out) {
  const long S = P.ws_len;
  auto Y = [&](int k) { return load_c<R>(xs, P.n, P.mono_var[vb + k]); };
  auto put = [&](int p, const cplx<R>& v) { store_c<R>(W.ws, S, out + 32L * p, v); };
  auto get = [&](int p) { return load_c<R>(W.ws, S, out + 32L * p); };
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

// Long monomials (size >= kMonoSplit, the first P.mono_long in device order)
// are evaluated by a PAIR of lanes: the even lane runs the prefix chain
// F_s = F_{s-1} y_s, the odd lane the suffix chain B_j = y_j B_{j+1}, one
// multiplication each per step, and each partial d_k = F_{k-1} B_{k+1} is
// formed by the lane whose operand arrives last, reading the other operand
// parked (by the partner, at an earlier step or earlier in this step) in the
// slot of d_k.  Every product has exactly the operands and operand order of
// the single-thread sweep, so the bits are the same; the dependent chain is
// m-1 products instead of 2m-4.
// QD only: a QD multiply is issue bound, so the pair halves the chain; a DD
// multiply is latency bound and the pair's barriers cost more than they save.
template <class R>
constexpr int kMonoSplit = limbs_of<R>::L == 4 ? 8 : (1 << 30);

template <class R>
__device__ __forceinline__ void mono_pair(const DevPlan& P, const Work& W, const double* xs, int q, bool fwd,
                                          unsigned pmask) {
  const long S = P.ws_len;
  const int m = P.mono_size[q];
  const int vb = P.mono_vbeg[q];
  const long out = P.mono_out[q];
  auto Y = [&](int k) { return load_c<R>(xs, P.n, P.mono_var[vb + k]); };
  auto put = [&](int p, const cplx<R>& v) { store_c<R>(W.ws, S, out + 32L * p, v); };
  auto get = [&](int p) { return load_c<R>(W.ws, S, out + 32L * p); };
  // chain values: F_s (fwd lane), B_{m-1-s} (bwd lane).  Both lanes run one
  // instruction stream (operands chosen by select), so the pair never diverges.
  cplx<R> c = Y(fwd ? 0 : m - 1);
  for (int s = 0; s <= m - 2; ++s) {
    if (s > 0) {
      const cplx<R> y = Y(fwd ? s : m - 1 - s);
      c = c_mul(pick(fwd, c, y), pick(fwd, y, c));  // F_{s-1} y_s  |  y_j B_{j+1}
    }
    // the partial this chain value feeds: F_s = F_{k-1} with k = s+1;
    // B_{m-1-s} = B_{k+1} with k = m-2-s.  F ready at step a = k-1, B at b = m-2-k.
    const int k = fwd ? s + 1 : m - 2 - s;
    const int a = k - 1, b = m - 2 - k;
    const bool edge = fwd ? k == m - 1 : k == 0;  // d_{m-1} = F_{m-2}, d_0 = B_1
    const bool mine_later = fwd ? a > b : a <= b;  // this lane forms d_k in phase 2
    const int slot = fwd ? (edge ? m : k + 1) : (edge ? 1 : k + 1);
    if (edge || !mine_later) put(slot, c);  // final partial, or park the operand
    __syncwarp(pmask);
    // phase 2: in the first half of the steps neither lane forms a partial
    // (both park); from the middle on both do (fwd the upper, bwd the lower
    // half of the partials) -- the same condition in both lanes of the pair
    if (2 * s >= m - 3) {
      const bool later = !edge && mine_later;
      const cplx<R> o = later ? get(k + 1) : c;  // the partner's parked operand
      const cplx<R> d = c_mul(pick(fwd, c, o), pick(fwd, o, c));  // d_k = F_{k-1} * B_{k+1}
      if (later) put(k + 1, d);
    }
    // no second barrier: phase 2 writes the slot of d_k, which the partner
    // parked earlier and never touches again
  }
  if (fwd) put(0, c_mul(c, Y(m - 1)));  // value = F_{m-2} * y_{m-1}
  __syncwarp(pmask);
  if (fwd && (P.mono_flags[q] & 1)) mono_exponents<R>(P, W, xs, q, m, vb, out);
}

// xs: x (2L planes of n) -- a per-CTA shared-memory copy when P.x_smem, else W.x.
// The single-thread sweeps prefetch the next factor (and, backwards, the
// parked prefix product) one step ahead, so the chain of products does not
// wait on an index load and a value load per step.
template <class R>
__device__ __noinline__ void eval_monomials(const DevPlan& P, const Work& W, const double* xs, int tid, int nthreads) {
  const long S = P.ws_len;
  {  // long monomials: lane pairs (tid, tid^1) are in the same warp
    const int pair = tid >> 1, npairs = nthreads >> 1;
    const unsigned pmask = 3u << (threadIdx.x & 30);
    for (int q = pair; q < P.mono_long; q += npairs) mono_pair<R>(P, W, xs, q, (tid & 1) == 0, pmask);
  }
  for (int q = P.mono_long + tid; q < P.M; q += nthreads) {
    const int m = P.mono_size[q];
    const int vb = P.mono_vbeg[q];
    const long out = P.mono_out[q];
    auto Y = [&](int k) { return load_c<R>(xs, P.n, P.mono_var[vb + k]); };
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
      cplx<R> yn = Y(1);
      for (int k = 1; k <= m - 2; ++k) {
        const cplx<R> y = yn;
        yn = Y(k + 1);  // k + 1 <= m - 1: the last one is y_{m-1}
        F = c_mul(F, y);
        put(k + 2, F);
      }
      put(0, c_mul(F, yn));
      cplx<R> B = yn;  // y_{m-1}
      cplx<R> yk = Y(m - 2), fk = get(m - 1);
      for (int k = m - 2; k >= 1; --k) {
        const cplx<R> y = yk, f = fk;
        if (k > 1) {
          yk = Y(k - 1);
          fk = get(k);
        }
        put(k + 1, c_mul(f, B));
        B = c_mul(y, B);
      }
      put(1, B);
    }
    if (P.mono_flags[q] & 1) mono_exponents<R>(P, W, xs, q, m, vb, out);
  }
}

// One contribution: coef * (monomial value or partial), or the coefficient
// itself for a constant term (wi < 0).  Branch-free so unrolled copies
// interleave.
template <class R>
__device__ __forceinline__ cplx<R> contrib(const DevPlan& P, const Work& W, int ci, int wi) {
  const cplx<R> c = load_c<R>(P.coef, P.n_coef, ci);
  const cplx<R> m = load_c<R>(W.ws, P.ws_len, wi < 0 ? 0 : wi);
  return pick(wi < 0, c, c_mul(c, m));
}

// Canonical sum of one contribution list by a group; valid at g.p == 0.
// Partial p = c[p] + c[p+Pw] + ... is accumulated in order, kU contributions
// per round: their index and value loads and products are independent, so
// the L2 round trips overlap and only the additions stay sequential.
template <class R>
__device__ __forceinline__ cplx<R> slot_sum(const DevPlan& P, const Work& W, const Group& g, int beg, int K, cplx<R>* sm) {
  constexpr int kU = limbs_of<R>::L == 4 ? 2 : 4;
  const int Pw = width_eval_d(K);
  cplx<R> acc = c_zero<R>();
  if (g.p < Pw && g.p < K) {
    int r = g.p;
    acc = contrib<R>(P, W, P.ctr_coef[beg + r], P.ctr_ws[beg + r]);
    r += Pw;
    for (; r + (kU - 1) * Pw < K; r += kU * Pw) {
      int ci[kU], wi[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        ci[u] = P.ctr_coef[beg + r + u * Pw];
        wi[u] = P.ctr_ws[beg + r + u * Pw];
      }
      cplx<R> v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = contrib<R>(P, W, ci[u], wi[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u) acc = c_add(acc, v[u]);
    }
    for (; r < K; r += Pw) acc = c_add(acc, contrib<R>(P, W, P.ctr_coef[beg + r], P.ctr_ws[beg + r]));
  }
  return group_tree(acc, g, Pw, K, sm);
}

// Canonical width-32 sums of K <= 512 contributions by ONE lane (lane tasks):
// leaves are the partials p = c[p] + c[p+32] + ... (each summed in order),
// merged by the levels off = 16 .. 1, an empty right subtree (least index
// p + off >= K) skipped.  No shuffles, no idle lanes.
// K <= KMAX: all contributions in registers, levels off = 4, 2, 1 only.
template <class R, int KMAX>
__device__ __forceinline__ cplx<R> lane_sum(const DevPlan& P, const Work& W, int beg, int K) {
  cplx<R> part[KMAX];
#pragma unroll
  for (int r = 0; r < KMAX; ++r) {
    if (r < K) part[r] = contrib<R>(P, W, P.ctr_coef[beg + r], P.ctr_ws[beg + r]);
  }
#pragma unroll
  for (int off = KMAX / 2; off >= 1; off >>= 1) {
#pragma unroll
    for (int p = 0; p < off; ++p)
      if (p + off < K) part[p] = c_add(part[p], part[p + off]);
  }
  return part[0];
}

// K > KMAX: the tree rolled (code size: a fully unrolled 32-leaf tree of
// complex DD products is ~10k instructions per copy and thrashed the
// instruction cache of the batch kernel -- ncu: 26 % of its stall samples
// were no_instruction).  The width-32 canonical tree splits into the
// subtrees Q(c) of the leaves = c mod 8,
//   Q(c) = (L_c + L_{c+16}) + (L_{c+8} + L_{c+24})       (levels off = 16, 8)
// merged by the levels off = 4, 2, 1:
//   ((Q0 + Q4) + (Q2 + Q6)) + ((Q1 + Q5) + (Q3 + Q7)).
// Iteration u = 0..7 computes Q(brev3(u)) (four independent leaf sums, the
// ILP of the body) and folds it into a three-level stack; a merge whose right
// subtree starts at a leaf index >= K is skipped ("p + off < K").  The loop
// structure is warp-uniform (u), only the K tests are per lane.
__host__ __device__ constexpr int brev3(int u) { return ((u & 1) << 2) | (u & 2) | ((u & 4) >> 2); }

// General form: the subtree of the canonical width-P tree over the leaves
// p = c + D t (t < W = P / D, 4 <= W <= 32) -- D = 1 is the whole tree; the
// batch splits long sums over D lanes and merges the D subtrees with the
// levels off = D/2 .. 1 afterwards (tree_combine).  The leaves t0 + mG
// (G = W / 4, m = 0..3) form Q(t0) (levels off = W/2, W/4 of the subtree);
// the Q's are merged in bit-reversed order t0 = brev(u) through a stack of up
// to three levels, each merge skipped when its right subtree's least leaf
// index is >= K.
__device__ __forceinline__ int brev_g(int u, int G) {
  return G == 8 ? brev3(u) : (G == 4 ? (((u & 1) << 1) | ((u & 2) >> 1)) : (G == 2 ? u : 0));
}

template <class R, class Get>
__device__ __forceinline__ cplx<R> lane_tree_g(int K, int P, int D, int c, const Get& get) {
  cplx<R> A = c_zero<R>(), B = c_zero<R>(), C = c_zero<R>(), q = c_zero<R>();
  if (c >= K) return q;  // the subtree is empty
  const int G = P / (4 * D);
#pragma unroll 1
  for (int u = 0; u < G; ++u) {
    const int t0 = brev_g(u, G);
    const int p0 = c + D * t0;
    q = c_zero<R>();
    if (p0 < K) {  // Q(t0) exists: leaves p0 + m D G, summed round by round (c[p], c[p+P], ...)
      const int dg = D * G;
      cplx<R> l[4] = {c_zero<R>(), c_zero<R>(), c_zero<R>(), c_zero<R>()};
#pragma unroll 1
      for (int r0 = 0; p0 + r0 < K; r0 += P) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int r = p0 + m * dg + r0;
          if (r < K) {
            const cplx<R> v = get(r);
            l[m] = r0 == 0 ? v : c_add(l[m], v);
          }
        }
      }
      cplx<R> x = l[0], y = l[1];
      if (p0 + 2 * dg < K) x = c_add(x, l[2]);  // off = W/2 of the subtree
      if (p0 + 3 * dg < K) y = c_add(y, l[3]);
      q = p0 + dg < K ? c_add(x, y) : x;        // off = W/4
    }
    if (G == 1) break;
    if ((u & 1) == 0) {
      A = q;
    } else {
      if (c + D * t0 < K) A = c_add(A, q);  // right subtree {u}
      if (G >= 4) {
        if ((u & 2) == 0) {
          B = A;
        } else {
          if (c + D * brev_g(u - 1, G) < K) B = c_add(B, A);
          if (G == 8) {
            if ((u & 4) == 0)
              C = B;
            else if (c + D * brev_g(u - 3, G) < K)
              C = c_add(C, B);
          }
        }
      }
    }
  }
  return G == 1 ? q : (G == 2 ? A : (G == 4 ? B : C));
}

// Merge the D subtree sums v[c] (c < D) with the levels off = D/2 .. 1.
template <class R>
__device__ __forceinline__ cplx<R> tree_combine(cplx<R> (&v)[8], int D, int K) {
#pragma unroll
  for (int off = 4; off >= 1; off >>= 1) {
    if (off < D) {
#pragma unroll
      for (int c = 0; c < off; ++c)
        if (c + off < K) v[c] = c_add(v[c], v[c + off]);
    }
  }
  return v[0];
}

template <class R, class Get>
__device__ __forceinline__ cplx<R> lane_canon32_g(int K, const Get& get) {
  return lane_tree_g<R>(K, 32, 1, 0, get);
}

template <class R>
__device__ __forceinline__ cplx<R> lane_canon32(const DevPlan& P, const Work& W, int beg, int K) {
  return lane_canon32_g<R>(K, [&](int r) { return contrib<R>(P, W, P.ctr_coef[beg + r], P.ctr_ws[beg + r]); });
}

// Contribution streams of the batch bundles (plan.hpp Bundle): entry `at`
// = pos*32 + lane.  The index and the 2L coefficient limbs are coalesced
// across the warp; the workspace entry is the same for every lane when the
// bundle's slots share their support (a broadcast).
template <class R, bool HI>
__device__ __forceinline__ cplx<R> s_contrib(const DevPlan& P, const Work& W, long at) {
  const int wi = P.s_ws[at];
  cplx<R> c;
  if constexpr (HI) {  // binary64 coefficients: rebuild the +0.0 lower limbs (same operand bits)
    c.re = r_from(P.s_coef[at], static_cast<R*>(nullptr));
    c.im = r_from(P.s_coef[P.s_len * 32 + at], static_cast<R*>(nullptr));
  } else {
    c = load_c<R>(P.s_coef, P.s_len * 32, at);
  }
  const cplx<R> m = load_c<R>(W.ws, P.ws_len, wi < 0 ? 0 : wi);
  return pick(wi < 0, c, c_mul(c, m));
}

// lane_canon32 over a stream (contribution r of this lane at (s0 + r)*32 + lane).
// HI: the stream holds only the leading limb of re / im (DevPlan::s_hi) --
// a template parameter, not a branch in the loop (the branch cost registers
// and spills in the hot loop: 11 % on C5).
template <class R, bool HI>
__device__ __forceinline__ cplx<R> lane_tree_s(const DevPlan& P, const Work& W, long s0, int lane, int K, int D,
                                               int c) {
  return lane_tree_g<R>(K, K > 0 ? width_eval_d(K) : 32, D, c,
                        [&](int r) { return s_contrib<R, HI>(P, W, (s0 + r) * 32 + lane); });
}

template <class R>
__device__ __forceinline__ void slot_store(const DevPlan& P, const Work& W, const ptplan::SlotTask& tk,
                                           const cplx<R>& Sg, const cplx<R>& Sf, bool have_f, const cplx<R>& wS,
                                           const R& wT) {
  const long SA = (long)P.N * (P.n + 1);
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

// The batch's lane tasks: warp w runs its bundles (plan.hpp Bundle), lane l
// the l-th slot of each.  Own register-allocation unit (the unrolled trees).
// The batch's lane tasks: warps claim bundles (plan.hpp Bundle) from a
// shared counter, largest first; lane l runs the l-th slot of a bundle.  A
// split bundle (D > 1) computes only the subtree c of its slots' sums and
// parks it in shared scratch; after one CTA barrier the D subtrees of each
// split group are merged (tree_combine) and stored.  Own register-allocation
// unit; one copy of the tree for g and f (instruction cache).
template <class R, bool HI>
__device__ __noinline__ void eval_bundles(const DevPlan& P, const Work& W, const cplx<R> wS, const R wT, int* next,
                                          double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int L = limbs_of<R>::L;
  const long SS = (long)P.scratch_units * 32;  // complex entries of the scratch (plane stride)
  for (;;) {
    int b = 0;
    if (lane == 0) b = atomicAdd(next, 1);  // largest bundles first: greedy list scheduling over the warps
    b = __shfl_sync(0xffffffffu, b, 0);
    if (b >= P.n_bundles) break;
    const ptplan::Bundle B = P.bundles[b];
    const int D = B.dc >> 8, c = B.dc & 255;
    if (lane < B.ntasks) {
      const ptplan::SlotTask tk = P.btasks[B.task_beg + lane];
      cplx<R> Sg = c_zero<R>(), Sf = c_zero<R>();
#pragma unroll 1
      for (int side = 0; side < 2; ++side) {
        const int K = side ? tk.f_cnt : tk.g_cnt;
        const cplx<R> v = lane_tree_s<R, HI>(P, W, side ? B.sf : B.sg, lane, K, D, c);
        if (side)
          Sf = v;
        else
          Sg = v;
      }
      if (D == 1) {
        bool have_f;
        if (tk.f_cnt < 0) {
          Sf = Sg;
          have_f = tk.g_cnt > 0;
        } else {
          have_f = tk.f_cnt > 0;
        }
        slot_store<R>(P, W, tk, Sg, Sf, have_f, wS, wT);
      } else {
        store_c<R>(scratch, SS, (long)(B.split + c) * 32 + lane, Sg);
        store_c<R>(scratch, SS, (long)(B.split + D + c) * 32 + lane, Sf);
      }
    }
  }
  if (P.n_splits == 0) return;
  __syncthreads();  // every split subtree parked
  for (int gi = warp; gi < P.n_splits; gi += kWarps) {
    const int32_t* sp = P.splits + 4 * gi;  // task_beg, ntasks, D, scratch base
    if (lane >= sp[1]) continue;
    const ptplan::SlotTask tk = P.btasks[sp[0] + lane];
    const int D = sp[2], base = sp[3];
    cplx<R> v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = c < D ? load_c<R>(scratch, SS, (long)(base + c) * 32 + lane) : c_zero<R>();
    const cplx<R> Sg = tree_combine<R>(v, D, tk.g_cnt);
    cplx<R> Sf;
    bool have_f;
    if (tk.f_cnt < 0) {
      Sf = Sg;
      have_f = tk.g_cnt > 0;
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        v[c] = c < D ? load_c<R>(scratch, SS, (long)(base + D + c) * 32 + lane) : c_zero<R>();
      Sf = tree_combine<R>(v, D, tk.f_cnt);
      have_f = tk.f_cnt > 0;
    }
    slot_store<R>(P, W, tk, Sg, Sf, have_f, wS, wT);
  }
  (void)L;
}

template <class R, class Team>
__device__ __noinline__ void eval_slots(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, double t,
                                       double* scratch = nullptr) {
  __syncwarp();  // whole warps call this: converged entry (no WARPSYNC.COLLECTIVE fallback for its shuffles)
  cplx<R> wS;
  R wT;
  weights<R>(P, t, wS, wT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (P.bundles != nullptr) {  // batch: lane tasks in warp bundles over coalesced streams
    if (P.s_hi)
      eval_bundles<R, true>(P, W, wS, wT, &sh.bundle_next, scratch);
    else
      eval_bundles<R, false>(P, W, wS, wT, &sh.bundle_next, scratch);
  } else {  // lane tasks: one slot per lane (canonical width 32, K <= lane_k)
    constexpr int KM = limbs_of<R>::L == 4 ? 4 : 8;
    const int beg = P.class_beg[0], end = P.class_beg[1];
    const int nth = team.nblocks * kThreads;
    for (int ti = beg + team.block * kThreads + threadIdx.x; ti < end; ti += nth) {
      const ptplan::SlotTask tk = P.tasks[ti];
      cplx<R> Sg = c_zero<R>(), Sf;
      if (tk.g_cnt > 0) Sg = tk.g_cnt <= KM ? lane_sum<R, KM>(P, W, tk.g_beg, tk.g_cnt) : lane_canon32<R>(P, W, tk.g_beg, tk.g_cnt);
      bool have_f;
      if (tk.f_cnt < 0) {
        Sf = Sg;
        have_f = tk.g_cnt > 0;
      } else {
        Sf = c_zero<R>();
        if (tk.f_cnt > 0) Sf = tk.f_cnt <= KM ? lane_sum<R, KM>(P, W, tk.f_beg, tk.f_cnt) : lane_canon32<R>(P, W, tk.f_beg, tk.f_cnt);
        have_f = tk.f_cnt > 0;
      }
      slot_store<R>(P, W, tk, Sg, Sf, have_f, wS, wT);
    }
  }
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {  // rolled: one copy of the group sums (instruction cache)
    const int gw = 8 >> c;
    if (gw > kWarps) continue;  // 128-thread batch CTAs: the host never leaves 8-warp tasks for them
    const int gpc = kWarps / gw;
    const int gi = warp / gw;
    Group g{gw, (warp % gw) * 32 + lane, 1 + gi};
    cplx<R>* sm = sh.tree + gi * 32 * gw;
    const int ngroups = team.nblocks * gpc;
    const int beg = P.class_beg[c + 1], end = P.class_beg[c + 2];
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
      if (g.p == 0) slot_store<R>(P, W, tk, Sg, Sf, have_f, wS, wT);
      g.sync();  // protect the group scratch before the next task
    }
  }
}

// ---------------------------------------------------------------------------
// (2) MGS least squares on [J | -h]
// ---------------------------------------------------------------------------
template <class R>
__device__ __forceinline__ R group_bcast_r(const Group& g, int gi, R v, Smem<R>& sh, int& phase) {
  if (g.p == 0) sh.rbcast[gi][phase] = v;
  g.sync();
  R r = sh.rbcast[gi][phase];
  phase ^= 1;
  return r;
}
template <class R>
__device__ __forceinline__ cplx<R> group_bcast_c(const Group& g, int gi, const cplx<R>& v, Smem<R>& sh, int& phase) {
  if (g.p == 0) sh.bcast[gi][phase] = v;
  g.sync();
  cplx<R> r = sh.bcast[gi][phase];
  phase ^= 1;
  return r;
}

// Column storage during MGS: owned columns live in shared memory (SoA, stride
// N) when they fit, else in place in the global matrix (stride N*(n+1)).
struct ColRef {
  double* p;
  long S;
};

template <class R>
__device__ __forceinline__ cplx<R> ldcg_c(const double* p, long S, long i) {
  constexpr int L = limbs_of<R>::L;
  cplx<R> v;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    r_set_limb(v.re, l, __ldcg(p + l * S + i));
    r_set_limb(v.im, l, __ldcg(p + (L + l) * S + i));
  }
  return v;
}

// complex entry i of an SoA vector in another CTA's shared memory (DSMEM);
// base = shared::cluster address of element 0
template <class R>
__device__ __forceinline__ cplx<R> ldsc_c(uint32_t base, long S, long i) {
  constexpr int L = limbs_of<R>::L;
  cplx<R> v;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    double a, b;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(a) : "r"(base + (uint32_t)(8 * (l * S + i))));
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(b) : "r"(base + (uint32_t)(8 * ((L + l) * S + i))));
    r_set_limb(v.re, l, a);
    r_set_limb(v.im, l, b);
  }
  return v;
}

constexpr int kMaxElems = 4;  // ceil(N / P_mgs) <= 4  (N <= 1024)

// Where one owned column keeps its data while the factorisation runs.
struct OwnedCol {
  ColRef a;       // the column itself (becomes q_j)
  ColRef r;       // R column j: r_kj at index k (k <= j)
  double* inv;    // 1/r_jj (L limbs, stride 1 in shared memory / n in global)
  long inv_S;
  int inv_i;
};

// Shared-memory layout of the MGS staging area of one CTA (dynamic smem):
// [cols][2L][N] columns, then [cols][2L][n+1] R columns, then [cols][L] inverses.
__host__ __device__ inline size_t mgs_stage_doubles(int L, int N, int n, int cols) {
  return (size_t)cols * (2 * L * (size_t)N + 2 * L * (size_t)(n + 1) + L);
}

// Normalise column j (already projected against q_0..q_{j-1}) and publish it.
// prev = max_{k<j} r_kk (binary64).  Returns false on rank deficiency (the
// flag is still published, with the failure bit, so nobody hangs).
// S: the owned column, its R column and inverse live in this CTA's shared
// memory (tell nvcc, so it emits LDS/STS instead of generic loads).
template <bool S>
__device__ __forceinline__ void assume_shared(const OwnedCol& c) {
  if constexpr (S) {
    if (!__isShared(c.a.p) || !__isShared(c.r.p) || !__isShared(c.inv)) __builtin_unreachable();
  }
}

// Canonical width-Pm sum of the group's element values v[r] (element
// i = g.p + r*32*gw).  With 32*gw == Pm thread p owns partial p and adds its
// elements in order; with 32*gw > Pm (then every thread holds at most one
// element and N > Pm) element p + m*Pm is held by thread p + m*Pm and handed
// to thread p through shared memory, so partial p = c[p] + c[p+Pm] + ... in
// the same order either way.
template <class T>
__device__ __forceinline__ T mgs_reduce(const T* v, const Group& g, int Pm, int N, T* sm) {
  const int TT = 32 * g.gw;
  T acc = v[0];
  if (TT == Pm) {
#pragma unroll
    for (int r = 1; r < kMaxElems; ++r)
      if (g.p + r * Pm < N) acc = add_v(acc, v[r]);
  } else {
    if (g.p >= Pm && g.p < N) sm[g.p - Pm] = v[0];
    g.sync();
    if (g.p < Pm)
      for (int m = 1; g.p + m * Pm < N; ++m) acc = add_v(acc, sm[(m - 1) * Pm + g.p]);
  }
  return group_tree(acc, g, Pm, N, sm);
}

template <class R, class Team, bool S>
__device__ __forceinline__ bool mgs_normalize(const DevPlan& P, const Work& W, const Team& team, const Group& g, int gi, Smem<R>& sh,
                              int& phase, const OwnedCol& c, bool q_to_global, double* pmax_sm, int j, double prev,
                              unsigned long long epoch, double sqrt_eps) {
  assume_shared<S>(c);
  const int N = P.N, Pm = P.P_mgs, TT = 32 * g.gw;
  const long SA = (long)N * (P.n + 1);
  R v[kMaxElems];
#pragma unroll
  for (int r = 0; r < kMaxElems; ++r) {
    const int i = g.p + r * TT;
    v[r] = i < N ? c_norm_sqr(load_c<R>(c.a.p, c.a.S, i)) : rconst<R>(0.0);
  }
  R* rsm = reinterpret_cast<R*>(sh.tree + (gi * 32 * g.gw));
  const R nrm2 = mgs_reduce(v, g, Pm, N, rsm);
  int ok = 0;
  R inv = rconst<R>(0.0);
  if (g.p == 0) {
    R rjj, inv1;
    r_sqrt_inv(nrm2, rjj, inv1);
    const double d = r_hi(rjj);
    const double mx = d > prev ? d : prev;
    ok = d > sqrt_eps * mx;
    if (!ptk::finite(d)) atomicExch(W.ctl + CTL_NONFINITE, 1ull);  // see pt_path_stats.flags
    if (pmax_sm)
      pmax_sm[j] = mx;
    else
      W.rmaxp[j] = mx;
    if (ok) {
      inv = inv1;
      store_r<R>(c.inv, c.inv_S, c.inv_i, inv);
      store_c<R>(c.r.p, c.r.S, j, cplx<R>{rjj, rconst<R>(0.0)});
    }
    sh.ibcast[gi][phase] = ok;
  }
  inv = group_bcast_r<R>(g, gi, inv, sh, phase);
  ok = sh.ibcast[gi][phase ^ 1];
  if (ok) {
    double* gj = W.A + (long)j * N;
#pragma unroll
    for (int r = 0; r < kMaxElems; ++r) {
      const int i = g.p + r * TT;
      if (i < N) {
        const cplx<R> q = c_scale(load_c<R>(c.a.p, c.a.S, i), inv);
        store_c<R>(c.a.p, c.a.S, i, q);
        if (q_to_global && c.a.p != gj) store_c<R>(gj, SA, i, q);
      }
    }
  }
  g.sync();
  if (g.p == 0) {
    if (!ok) atomicExch(W.ctl + CTL_RANK, epoch);
    team.publish(W.flags, j, epoch, !ok);  // release: cumulative over the group's writes (bar.sync above)
  }
  return ok != 0;
}

// r_kj = q_k^H a_j (canonical width P_mgs), a_j -= r_kj q_k.  q: this thread's
// elements of q_k (rows p + r*P_mgs).
template <class R, bool S>
__device__ __forceinline__ void mgs_project(const DevPlan& P, const Group& g, int gi, Smem<R>& sh, int& phase, const cplx<R>* q,
                            const OwnedCol& c, int k, int j) {
  assume_shared<S>(c);
  const int N = P.N, n = P.n, Pm = P.P_mgs, TT = 32 * g.gw;
  cplx<R> v[kMaxElems];
#pragma unroll
  for (int r = 0; r < kMaxElems; ++r) {
    const int i = g.p + r * TT;
    v[r] = i < N ? c_conj_mul(q[r], load_c<R>(c.a.p, c.a.S, i)) : c_zero<R>();
  }
  cplx<R>* sm = sh.tree + gi * 32 * g.gw;
  cplx<R> rkj = mgs_reduce(v, g, Pm, N, sm);
  if (g.p == 0) store_c<R>(c.r.p, c.r.S, k, rkj);
  rkj = group_bcast_c<R>(g, gi, rkj, sh, phase);
  if (j < n || k < n - 1) {
#pragma unroll
    for (int r = 0; r < kMaxElems; ++r) {
      const int i = g.p + r * TT;
      if (i < N) store_c<R>(c.a.p, c.a.S, i, c_sub(load_c<R>(c.a.p, c.a.S, i), c_mul(rkj, q[r])));
    }
  }
}

// Column-pipelined right-looking MGS.  Column j is owned
// by group j mod G (group id = block + nblocks * group-in-CTA, so
// consecutive columns sit on different SMs).  The owner keeps its columns,
// their R entries and 1/r_jj in shared memory for the whole factorisation
// (flushed to global at the end, so no release fence ever waits on them),
// normalises column k+1 as soon as q_k has been applied (look-ahead) and
// publishes q_{k+1} with a flag.  Consumers read q_k once (L2 for the grid
// team, DSMEM for the cluster team, local smem for the block team).
template <class R, class Team, bool S>
__device__ __forceinline__ void mgs_run(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, double* colsm,
                                        double* pmax_sm, unsigned long long epoch, double sqrt_eps) {
  constexpr int L = limbs_of<R>::L;
  if constexpr (S) {
    if (!__isShared(colsm)) __builtin_unreachable();
  }
  const int N = P.N, n = P.n, Pm = P.P_mgs;
  const long SA = (long)N * (n + 1), SR = (long)n * (n + 1);
  const int gm = P.mgs_gw;
  const int TT = 32 * gm;
  const int gpc = kWarps / gm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gi = warp / gm;
  const Group g{gm, (warp % gm) * 32 + lane, 1 + gi};
  const int nb = team.nblocks;
  const int G = nb * gpc;
  const int me = team.block + nb * gi;
  if (me > n) return;  // owns no column
  const int cols = (n + 1 + nb - 1) / nb;
  double* rbase = colsm ? colsm + (size_t)cols * 2 * L * N : nullptr;
  double* ibase = colsm ? rbase + (size_t)cols * 2 * L * (n + 1) : nullptr;
  auto own = [&](int j) -> OwnedCol {
    if (colsm) {
      const int slot = j / nb;
      return OwnedCol{ColRef{colsm + (long)slot * 2 * L * N, (long)N},
                      ColRef{rbase + (long)slot * 2 * L * (n + 1), (long)(n + 1)}, ibase + (long)slot * L, 1, 0};
    }
    return OwnedCol{ColRef{W.A + (long)j * N, SA}, ColRef{W.Rm + (long)j * n, SR}, W.inv, (long)n, j};
  };
  if (colsm) {  // stage the owned columns (each thread its own rows: no sync needed)
    for (int j = me; j <= n; j += G) {
      const ColRef c = own(j).a;
#pragma unroll
      for (int r = 0; r < kMaxElems; ++r) {
        const int i = g.p + r * TT;
        if (i < N) store_c<R>(c.p, c.S, i, ldcg_c<R>(W.A + (long)j * N, SA, i));
      }
    }
  }
  int phase = 0;
  bool alive = true;
  const int last_owned = me + ((n - me) / G) * G;
  // q_k travels through global memory (grid team, or no shared staging),
  // else it is read from the owner CTA's shared memory (local or DSMEM)
  const bool q_global = Team::kQInGlobal || colsm == nullptr;
  const bool pmax_shared = !Team::kQInGlobal && pmax_sm != nullptr;
  double* pmx = pmax_shared ? pmax_sm : nullptr;
  if (me == 0)
    alive = mgs_normalize<R, Team, S>(P, W, team, g, gi, sh, phase, own(0), q_global, pmx, 0, 0.0, epoch, sqrt_eps);
  for (int k = 0; k < n && alive && k < last_owned; ++k) {
    const bool mine = (k % G == me);
    if (!mine) {
      if (g.p == 0) sh.ibcast[gi][phase] = team.wait(W.flags, k, epoch);
      g.sync();
      const int st = sh.ibcast[gi][phase];
      phase ^= 1;
      if (st != 0) return;  // rank failure of column k, or abort
    }
    const bool next_mine = ((k + 1) % G == me) && k + 1 < n;
    unsigned long long* dbg = (W.prof && next_mine && g.p == 0) ? W.prof + kProfSlots + 6 * (k + 1) : nullptr;
    if (dbg) {
      dbg[0] = gtimer();
      dbg[1] = clock64();
    }
    cplx<R> q[kMaxElems];
    double prev = 0.0;
    {
      const double* qp;
      const double* pm;
      long qS;
      if (mine) {
        const ColRef ck = own(k).a;
        qp = ck.p;
        qS = ck.S;
        pm = pmx ? pmx + k : W.rmaxp + k;
      } else if (q_global) {
        qp = W.A + (long)k * N;
        qS = SA;
        pm = pmx ? nullptr : W.rmaxp + k;
      } else {
        const double* loc = colsm + (long)(k / nb) * 2 * L * N;
        qp = loc;  // nb == 1: local shared memory; else read below through DSMEM
        qS = N;
        pm = nb == 1 ? pmx + k : cooperative_groups::this_cluster().map_shared_rank(pmx + k, k % nb);
      }
      const bool remote = !mine && !q_global && nb > 1;
      if (next_mine && g.p == 0) {
        if (pmx && !mine && q_global)  // cluster/block team without shared staging
          pm = nb == 1 ? pmx + k : cooperative_groups::this_cluster().map_shared_rank(pmx + k, k % nb);
        prev = (pmx || mine) ? *(volatile const double*)pm : __ldcg(pm);
      }
      const uint32_t qremote = remote ? mapa_u32(smem_u32(qp), (uint32_t)(k % nb)) : 0u;
#pragma unroll
      for (int r = 0; r < kMaxElems; ++r) {
        const int i = g.p + r * TT;
        if (i < N) {
          if (remote)
            q[r] = ldsc_c<R>(qremote, qS, i);
          else
            q[r] = (!mine && q_global && Team::kGrid) ? ldcg_c<R>(qp, qS, i) : load_c<R>(qp, qS, i);
        }
      }
      if (dbg) dbg[2] = clock64() + (unsigned long long)(r_hi(q[0].re) == 12345.0);  // after the loads land
    }
    int j = k + 1 + ((me - (k + 1)) % G + G) % G;  // first owned column > k
    for (; j <= n; j += G) {
      const OwnedCol c = own(j);
      mgs_project<R, S>(P, g, gi, sh, phase, q, c, k, j);
      if (j == k + 1 && j < n) {
        if (dbg) dbg[3] = clock64();
        if (!mgs_normalize<R, Team, S>(P, W, team, g, gi, sh, phase, c, q_global, pmx, j, prev, epoch, sqrt_eps))
          alive = false;
        if (dbg) {
          dbg[4] = clock64();
          dbg[5] = gtimer();
        }
      }
    }
  }
  if (colsm && alive) {  // flush R columns and inverses of the owned columns
    for (int j = me; j <= n; j += G) {
      const OwnedCol c = own(j);
      const int rows = j < n ? j + 1 : n;
      for (int k = g.p; k < rows; k += 32 * g.gw)
        store_c<R>(W.Rm + (long)j * n, SR, k, load_c<R>(c.r.p, c.r.S, k));
      if (j < n && g.p == 0) store_r<R>(W.inv, n, j, load_r<R>(c.inv, 1, 0));
    }
  }
}

template <class R, class Team>
__device__ __noinline__ void mgs(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, double* colsm,
                                 double* pmax_sm, unsigned long long epoch, double sqrt_eps) {
  __syncwarp();  // whole warps call this: converged entry (no WARPSYNC.COLLECTIVE fallback for its shuffles)
  if (colsm)
    mgs_run<R, Team, true>(P, W, team, sh, colsm, pmax_sm, epoch, sqrt_eps);
  else
    mgs_run<R, Team, false>(P, W, team, sh, colsm, pmax_sm, epoch, sqrt_eps);
}

// Back substitution R dx = y, dx_k = (y_k - sum_{j>k} r_kj dx_j) * (1/r_kk),
// column-oriented in one CTA with the next column of R prefetched one step
// ahead (L2 latency off the dependency chain); then u = max|dx|, x += dx.
// Component-split back substitution for n <= kThreads / 2 (the group-MGS
// path, i.e. QD): thread 2i handles the real, 2i+1 the imaginary part of row
// i, so each thread does half of every complex product on the chain.  The
// operations are the complex ones, split: c_mul(a, b) = (a.re b.re - a.im
// b.im, a.re b.im + a.im b.re) with r_sub(p, q) = r_add(p, -q), c_scale and
// c_sub component-wise -- the same bits.  Operands are chosen by select so
// both threads of a pair run one instruction stream.
template <class R>
__device__ __noinline__ double backsub_split(const DevPlan& P, const Work& W, Smem<R>& sh) {
  __syncwarp();  // whole warps call this: converged entry (no WARPSYNC.COLLECTIVE fallback for its shuffles)
  constexpr int L = limbs_of<R>::L;
  const int n = P.n;
  const long SR = (long)n * (n + 1);
  const int i = threadIdx.x >> 1;
  const bool im = threadIdx.x & 1;
  const bool row = i < n;
  auto comp = [&](const cplx<R>& z) { return im ? z.im : z.re; };
  R acc = rconst<R>(0.0), inv = rconst<R>(0.0);
  cplx<R> cur = c_zero<R>();
  if (row) {
    acc = comp(load_c<R>(W.Rm, SR, (long)n * n + i));
    inv = load_r<R>(W.inv, n, i);
    cur = load_c<R>(W.Rm, SR, (long)(n - 1) * n + i);  // R column storage covers rows 0..n-1
  }
  for (int j = n - 1; j >= 0; --j) {
    if (i == j) {
      acc = r_mul(acc, inv);  // row j finished: this component of dx_j
      if (im)
        sh.xbs[j & 1].im = acc;
      else
        sh.xbs[j & 1].re = acc;
    }
    const cplx<R> nxt = row ? load_c<R>(W.Rm, SR, (long)(j > 0 ? j - 1 : 0) * n + i) : c_zero<R>();
    __syncthreads();
    const cplx<R> xj = sh.xbs[j & 1];
    if (i < j) {
      const R p1 = r_mul(cur.re, im ? xj.im : xj.re);
      const R p2 = r_mul(cur.im, im ? xj.re : xj.im);
      const R m = r_add(p1, im ? p2 : r_neg(p2));
      acc = r_sub(acc, m);
    }
    cur = nxt;
  }
  double u = 0.0;
  const double other = __shfl_xor_sync(0xffffffffu, r_hi(acc), 1);
  if (row) {
    if (!im) u = glibc_hypot(r_hi(acc), other);  // modulus_double of dx_i
#pragma unroll
    for (int l = 0; l < L; ++l) W.dx[(im ? L + l : l) * (long)n + i] = r_limb(acc, l);
    R xv;
#pragma unroll
    for (int l = 0; l < L; ++l) r_set_limb(xv, l, W.x[(im ? L + l : l) * (long)n + i]);
    const R xs = r_add(xv, acc);
#pragma unroll
    for (int l = 0; l < L; ++l) W.x[(im ? L + l : l) * (long)n + i] = r_limb(xs, l);
  }
  return block_nan_max(u, sh.red);
}

template <class R>
__device__ __noinline__ double backsub_update(const DevPlan& P, const Work& W, Smem<R>& sh) {
  __syncwarp();  // whole warps call this: converged entry (no WARPSYNC.COLLECTIVE fallback for its shuffles)
  if (P.n <= kThreads / 2) return backsub_split<R>(P, W, sh);
  const int n = P.n;
  const long SR = (long)n * (n + 1);
  cplx<R> acc[kMaxRowsPerThread], cur[kMaxRowsPerThread], nxt[kMaxRowsPerThread];
  R inv[kMaxRowsPerThread];
#pragma unroll
  for (int r = 0; r < kMaxRowsPerThread; ++r) {
    const int i = threadIdx.x + r * kThreads;
    if (i < n) {
      acc[r] = load_c<R>(W.Rm, SR, (long)n * n + i);
      inv[r] = load_r<R>(W.inv, n, i);
      if (i < n - 1) cur[r] = load_c<R>(W.Rm, SR, (long)(n - 1) * n + i);
    }
  }
  for (int j = n - 1; j >= 0; --j) {
    const int owner = j % kThreads, orow = j / kThreads;
    if ((int)threadIdx.x == owner) {
#pragma unroll
      for (int r = 0; r < kMaxRowsPerThread; ++r)
        if (r == orow) {
          acc[r] = c_scale(acc[r], inv[r]);  // row j finished: acc now holds dx_j
          sh.xbs[j & 1] = acc[r];
        }
    }
#pragma unroll
    for (int r = 0; r < kMaxRowsPerThread; ++r) {
      const int i = threadIdx.x + r * kThreads;
      if (i < j - 1) nxt[r] = load_c<R>(W.Rm, SR, (long)(j - 1) * n + i);
    }
    __syncthreads();
    const cplx<R> xj = sh.xbs[j & 1];
#pragma unroll
    for (int r = 0; r < kMaxRowsPerThread; ++r) {
      const int i = threadIdx.x + r * kThreads;
      if (i < j) acc[r] = c_sub(acc[r], c_mul(cur[r], xj));
      cur[r] = nxt[r];
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

}  // namespace ptdev

#include "mgs_warp.cuh"
#include "mgs_batch.cuh"

namespace ptdev {

// ---------------------------------------------------------------------------
// (3) predictor -- one CTA
// ---------------------------------------------------------------------------
struct History {
  double t[kMaxDegree + 1];
  int count, next, cap;
  __device__ int slot(int j) const { return (next - count + j + 2 * cap) % cap; }  // j-th oldest
};

template <class R>
__device__ __noinline__ void predict(const DevPlan& P, const Work& W, const History& H, double tau) {
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
__device__ __noinline__ void push_history(const DevPlan& P, const Work& W, History& H, double t) {
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
  int nonfinite;  // max|h|, max|dx| or an MGS diagonal was inf / NaN (pt_path_stats.flags)
};

template <class R, class Team>
__device__ NewtonOut newton(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, double* colsm,
                            const pt_step_params& sp, double t, unsigned long long& epoch) {
  NewtonOut o{0, NW_ITERATION_BUDGET, 0, -1.0, -1.0, 0, 0};
  const double sqrt_eps = kSqrtEps<R>();
  double last = bitsd(0x7ff0000000000000ull);
  const int tid = team.block * kThreads + threadIdx.x, nth = team.nblocks * kThreads;
  PhaseClock pc(team.block == 0 && threadIdx.x == 0 && W.prof != nullptr);
  for (int it = 1; it <= sp.newton_max_iter; ++it) {
    o.iters = it;
    if (pc.on) W.prof[PROF_ITERS] += 1;
    const double* xs = W.x;
    if (P.x_smem) {  // every CTA stages x in its dynamic shared memory (free during evaluation)
      constexpr int L = limbs_of<R>::L;
      for (int i = threadIdx.x; i < 2 * L * P.n; i += kThreads) colsm[i] = W.x[i];
      __syncthreads();
      xs = colsm;
    }
    if (threadIdx.x == 0) sh.bundle_next = 0;  // published by the team barrier below
    eval_monomials<R>(P, W, xs, tid, nth);
    if (!team.sync(&sh.flag)) return {0, NW_ABORT, it, -1.0, -1.0, 0, 0};
    pc.lap(W.prof + PROF_MONO);
    // split-bundle scratch: the batch's dynamic smem after the x copy
    eval_slots<R, Team>(P, W, team, sh, t, colsm ? colsm + ((2L * limbs_of<R>::L * P.n + 31) & ~31L) : nullptr);
    if (!team.sync(&sh.flag)) return {0, NW_ABORT, it, -1.0, -1.0, 0, 0};
    pc.lap(W.prof + PROF_SLOTS);
    double r = 0.0;
    for (int i = threadIdx.x; i < P.N; i += kThreads) r = nan_max(r, W.hmod[i]);
    r = block_nan_max(r, sh.red);
    o.residual = r;
    o.nonfinite |= !ptk::finite(r);
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
    pc.lap(W.prof + PROF_SLOTS);
    if (P.mgs_batch) {  // set for the batch kernel (BlockTeam) only
      if constexpr (std::is_same<Team, BlockTeam>::value) mgs_batch<R>(P, W, colsm, epoch, sqrt_eps);
    } else if (P.mgs_warp) {
      mgs_warp<R, Team>(P, W, team, sh, colsm, epoch, sqrt_eps);
    } else {
      mgs<R, Team>(P, W, team, sh, P.mgs_smem ? colsm : nullptr, Team::kQInGlobal ? nullptr : sh.pmax, epoch, sqrt_eps);
    }
    if (!team.sync(&sh.flag)) return {0, NW_ABORT, it, -1.0, -1.0, 0, 0};
    pc.lap(W.prof + PROF_MGS);
    if (threadIdx.x == 0) ++sh.mgs_seq;  // read again only after the next team barrier
    // a watchdog inside the MGS exchange (cluster / block teams) set CTL_ABORT
    // before its CTA arrived at the barrier above: every CTA sees it here
    if (!Team::kGrid && ld_acquire(W.ctl + CTL_ABORT)) return {0, NW_ABORT, it, -1.0, -1.0, 0, 0};
    o.nonfinite |= ld_acquire(W.ctl + CTL_NONFINITE) != 0ull;
    if (ld_acquire(W.ctl + CTL_RANK) == epoch) {
      o.kind = NW_LINEAR_SOLVE;
      return o;
    }
    if (P.mgs_warp || P.mgs_batch) {
      if (team.block == 0) {
        const double u = backsub_warp<R>(P, W, P.bs_smem ? colsm : nullptr, sh);
        if (threadIdx.x == 0) W.scal[0] = u;
      }
    } else if (team.block == 0) {
      const double u = backsub_update<R>(P, W, sh);
      if (threadIdx.x == 0) W.scal[0] = u;
    }
    if (!team.sync(&sh.flag)) return {0, NW_ABORT, it, -1.0, -1.0, 0, 0};
    pc.lap(W.prof + PROF_BACKSUB);
    const double u = *(volatile double*)(W.scal);
    ++o.solves;
    o.update = u;
    o.nonfinite |= !ptk::finite(u);
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
  int retrack;          // exact re-track launch: run only if stats->flags has PT_STAT_NONFINITE
};

template <class R, class Team>
__device__ void track_path(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, double* colsm,
                           const pt_step_params& sp, const TrackIO& io, unsigned long long epoch_base) {
  const int n = P.n;
  // exact re-track launch (DD): only paths whose fast run met a non-finite
  // value run again; every CTA reads the same word, so all leave together
  if (io.retrack && !(((volatile const pt_path_stats*)io.stats)->flags & PT_STAT_NONFINITE)) return;
  unsigned long long epoch = epoch_base;
  const bool leader = team.block == 0;
  pt_path_stats st{};
  if (leader)
    for (int i = threadIdx.x; i < n; i += kThreads) store_c<R>(W.x, n, i, load_c<R>(io.start, n, i));
  // Watchdog abort (stalled barrier / exchange): the path is reported as
  // failed with PT_FAIL_ABORT -- never left with stale statistics.
  auto aborted = [&](int iters) {
    if (leader && threadIdx.x == 0) {
      pt_path_stats a{};
      a.status = PT_PATH_FAIL;
      a.failure_kind = PT_FAIL_ABORT;
      a.newton_iters = st.newton_iters + iters;
      a.final_residual = bitsd(0x7ff8000000000000ull);
      a.final_update = bitsd(0x7ff8000000000000ull);
      *io.stats = a;
      if (io.trace_len) *io.trace_len = 0;
    }
  };
  if (!team.sync(&sh.flag)) return aborted(0);
  NewtonOut o = newton<R, Team>(P, W, team, sh, colsm, sp, 0.0, epoch);
  if (o.kind == NW_ABORT) return aborted(o.iters);
  int nonfinite = o.nonfinite;
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
      PhaseClock pc(leader && threadIdx.x == 0 && W.prof != nullptr);
      if (leader) predict<R>(P, W, H, ttrial);
      if (!team.sync(&sh.flag)) return aborted(0);
      pc.lap(W.prof + PROF_PREDICT);
      o = newton<R, Team>(P, W, team, sh, colsm, sp, ttrial, epoch);
      if (o.kind == NW_ABORT) return aborted(o.iters);
      st.newton_iters += o.iters;
      st.solves += o.solves;
      nonfinite |= o.nonfinite;
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
  if (leader) {  // a non-finite end point counts too (NaN-propagating check over the limbs)
    __syncthreads();  // io.end was written with another thread-to-entry mapping
    int bad = 0;
    for (int q = threadIdx.x; q < 2 * limbs_of<R>::L * n; q += kThreads) bad |= !ptk::finite(io.end[q]);
    bad = __syncthreads_or(bad);
    nonfinite |= bad;
  }
  if (leader && threadIdx.x == 0) {
    st.flags = nonfinite ? PT_STAT_NONFINITE : 0;
    *io.stats = st;
    if (io.trace_len) *io.trace_len = ntrace;
  }
}

}  // namespace ptdev
