// mgs_warp.cuh -- warp-per-column MGS least squares and one-warp back
// substitution for the single-path engines (N <= 128).
//
// Same arithmetic as the oracle (oracle/orc_tracker.hpp Tracker::lstsq,
// SPEC.md:296-322,339) and as mgs_run in device.cuh, bit for bit:
//   r_kk = sqrt(canon_sum |a_k|^2), rank test in binary64 against the prefix
//   max, q_k = a_k * (1/r_kk), r_kj = canon_sum conj(q_k) a_j,
//   a_j -= r_kj q_k (skipped for the last update of column n), and the
//   column-oriented back substitution subtracting r_kj x_j in descending j.
//
// Why a separate path: the single path is latency bound -- the chain
// q_k -> project a_{k+1} -> normalise -> q_{k+1} is strictly sequential, so
// the time per column is the latency of one projection plus one
// normalisation.  Here one warp owns a column and lane l holds rows
// l + 32 r (r < E), which is exactly the canonical partial layout for
// width_mgs(N) in {32, 64}: partial p = c[p] + c[p+P] + ... sits in lane
// p mod 32, the off >= 32 tree level is lane-local and the remaining five
// levels are warp shuffles.  No shared-memory tree, no named barriers; the
// only cross-warp traffic is q_k itself (local smem, DSMEM or L2 by team)
// and one flag per column.
//
// Column ownership: columns are dealt to the G = C * kWarps warps in blocks
// of B consecutive columns per CTA (B | kWarps), so B - 1 of every B steps
// of the critical chain hand q_k to a warp of the same CTA (shared memory),
// and the trailing updates are spread over all CTAs.  Warp (c, w) owns
// columns base(c, w) + m G, m = 0, 1, ...  (slot m of its smem column area).
#pragma once

#include <type_traits>

namespace ptdev {

constexpr int kWarpMgsMaxN = 128;

#ifndef PT_MGS_WARP_INLINE
#define PT_MGS_WARP_INLINE __noinline__
#endif  // E <= 4 elements per lane, width_mgs(N) <= 64

struct ColMap {
  int C, B;  // CTAs in the team, columns per CTA block
  __device__ __forceinline__ int G() const { return C * kWarps; }
  __device__ __forceinline__ int base(int c, int w) const { return ((w / B) * C + c) * B + (w % B); }
  // owner of column j: CTA, warp, CTA-local column slot
  __device__ __forceinline__ void owner(int j, int& c, int& w, int& ls) const {
    const int r0 = j % G(), b = r0 / B;
    c = b % C;
    w = (b / C) * B + r0 % B;
    ls = (j / G()) * kWarps + w;
  }
};

// width_mgs(N) as a function of E = ceil(N/32): 32 for N <= 64, 64 for N <= 128
template <int E>
constexpr int kCanonP = E <= 2 ? 32 : 64;

// Canonical width-P sum (P = width_mgs(N) in {32, 64}) of the values v[r]
// of rows lane + 32 r; the result is valid in lane 0.
template <class T, int E>
__device__ __forceinline__ T warp_canon(const T (&v)[E], int lane, int N, int P) {
  T acc = v[0];
  if (N >= 32 * E) {  // every row present (warp-uniform): no per-level selects
    if (P == 32) {
#pragma unroll
      for (int r = 1; r < E; ++r) acc = add_v(acc, v[r]);
    } else {
      if constexpr (E > 2) acc = add_v(acc, v[2]);
      if constexpr (E > 1) {
        T a1 = v[1];
        if constexpr (E > 3) a1 = add_v(a1, v[3]);
        acc = add_v(acc, a1);
      }
    }
    __syncwarp();
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc = add_v(acc, shfl_down_r(acc, off));  // lanes >= off: unused
    return acc;
  }
  if (P == 32) {  // compile-time at every call site (kCanonP<E>)
#pragma unroll
    for (int r = 1; r < E; ++r) acc = pick(lane + 32 * r < N, add_v(acc, v[r]), acc);
  } else {  // P == 64 (65 <= N <= 128): partial l = c[l] + c[l+64], partial l+32 = c[l+32] + c[l+96]
    if constexpr (E > 2) acc = pick(lane + 64 < N, add_v(acc, v[2]), acc);
    if constexpr (E > 1) {
      T a1 = v[1];
      if constexpr (E > 3) a1 = pick(lane + 96 < N, add_v(a1, v[3]), a1);
      acc = add_v(acc, a1);  // off = 32 level: l + 32 < 65 <= N always
    }
  }
  __syncwarp();
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const T o = shfl_down_r(acc, off);
    acc = pick(lane < off && lane + off < N, add_v(acc, o), acc);
  }
  return acc;
}

// --- mbarrier / st.async primitives (q_k push into every CTA that needs it) --
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, int parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for phase `parity` of a receive barrier.  Watchdog: a stalled
// exchange (or an abort raised by another waiter) sets CTL_ABORT and returns
// false; the caller abandons the sweep and newton() reports NW_ABORT after
// the team barrier (no __trap: the CUDA context stays usable).
__device__ __forceinline__ bool mbar_wait(uint64_t* b, int parity, unsigned long long* ctl) {
  if (mbar_try(b, parity)) return true;
  const unsigned long long t0 = gtimer();
  for (unsigned int spins = 1;; ++spins) {
    if (mbar_try(b, parity)) return true;
    if ((spins & 1023u) == 0 && (ld_acquire(ctl + CTL_ABORT) || (double)(gtimer() - t0) > kTimeoutNs)) {
      atomicExch(ctl + CTL_ABORT, 1ull);
      return false;
    }
  }
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// One TMA bulk copy global -> the same shared-memory offset of every CTA in
// `mask`, each completing `bytes` on its own copy of the barrier.
__device__ __forceinline__ void bulk_multicast(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

// Dynamic shared memory of the warp MGS, per CTA (doubles / u64 words):
//   [column slots: S * kWarps * 2L*N][Q buffer: n * QS][n mbarriers]
// Q buffer row k = the message of column k: q_k (2L planes of N), pmax_k, pad.
// The Q buffer exists only in the mbarrier exchange (cluster / block teams);
// the grid team exchanges q_k through L2 with release/acquire flags.
__host__ __device__ inline long mgs_warp_qs(int L, int N) { return 2L * L * N + 2; }  // even: 16-byte rows
__host__ __device__ inline size_t mgs_warp_slots_doubles(int L, int N, int n, int C) {
  const int G = C * kWarps;
  const int slots = (n + 1 + G - 1) / G;
  return (size_t)slots * kWarps * 2 * L * (size_t)N;
}
__host__ __device__ inline size_t mgs_warp_bytes(int L, int N, int n, int C, bool mbar) {
  size_t d = mgs_warp_slots_doubles(L, N, n, C);
  if (mbar) d += (size_t)n * mgs_warp_qs(L, N) + n;  // + one 8-byte mbarrier per column
  return d * 8;
}

template <class R, class Team>
struct WarpMgs {
  static constexpr int L = limbs_of<R>::L;
  const DevPlan& P;
  // Work and Team by value in the single-path engines: through references
  // every store to shared or global memory may alias them, so their pointers
  // would be reloaded (from the kernel's stack) on the critical chain after
  // each store.  The batch kernel (BlockTeam, 128 registers per thread) keeps
  // references: there the extra ~30 registers cost more in spills.
  static constexpr bool kByValue = !std::is_same<Team, BlockTeam>::value;
  std::conditional_t<kByValue, const Work, const Work&> W;
  std::conditional_t<kByValue, const Team, const Team&> team;
  Smem<R>& sh;
  double* colsm;  // this CTA's dynamic smem (layout above)
  ColMap cm;
  int lane, w, N, n;
  long SA, SR, CS;
  unsigned long long epoch;
  double sqrt_eps;

  double* qb;     // Q buffer (mbarrier exchange)
  uint64_t* bb;   // receive barriers

  __device__ double* slot_ptr(int ls) const { return colsm + (long)ls * CS; }
  __device__ double* qbuf() const { return qb; }
  __device__ uint64_t* bars() const { return bb; }

  // rows >= N read as zero (their lanes compute ignored values, branch-free)
  template <int E>
  __device__ __forceinline__ void load_col(const double* p, long S, cplx<R> (&a)[E]) const {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane + 32 * r;
      a[r] = i < N ? load_c<R>(p, S, i) : c_zero<R>();
    }
  }
  template <int E>
  __device__ __forceinline__ void store_col(double* p, long S, const cplx<R> (&a)[E]) const {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane + 32 * r;
      if (i < N) store_c<R>(p, S, i, a[r]);
    }
  }

  // largest column owned by CTA d (-1: none)
  __device__ int maxcol(int d) const {
    const int G = cm.G();
    int mx = -1;
    for (int ww = 0; ww < kWarps; ++ww) {
      const int b = cm.base(d, ww);
      if (b <= n) mx = max(mx, b + ((n - b) / G) * G);
    }
    return mx;
  }

  // Hand q_j to its consumers (mbarrier exchange).  Warps of this CTA read
  // q_j from the owner's column slot after a local arrive on bar[j]; every
  // other CTA that owns a column > j receives the message (q_j, pmax_j) by
  // one TMA multicast from its global staging row W.qg[j] -- the copy runs on
  // the L2 -> SM path, so the producer SM's shared-memory port stays free
  // for the critical next column.  lane_maxcol: lane d < C holds maxcol(d).
  template <int E>
  __device__ void handoff(int j, const cplx<R> (&a)[E], double pmax, int lane_maxcol) const {
    const long QS = mgs_warp_qs(L, N);
    const unsigned need = __ballot_sync(0xffffffffu, lane < team.nblocks && lane_maxcol > j);
    const unsigned remote = need & ~(1u << team.block);
    double* msg = W.qg + (long)j * QS;
    // this CTA's consumers read the owner's slot (stored by the caller): release
    // them first -- the global staging and its proxy fence are for remote CTAs only
    __syncwarp();
    if (lane == 0 && ((need >> team.block) & 1u)) mbar_arrive_local(bars() + j);
    if (remote) {
      store_col(msg, N, a);
      if (lane == 0) msg[2 * L * N] = pmax;
      asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> async-proxy (TMA) reads
      __syncwarp();
      if (lane == 0) bulk_multicast(qbuf() + (long)j * QS, msg, (uint32_t)(QS * 8), bars() + j, (uint16_t)remote);
    }
  }

  // Normalise column j (values a, already projected against q_0..q_{j-1}),
  // then hand q_j to the consumers.  prev = max_{k<j} binary64 r_kk.  With
  // the mbarrier exchange a rank failure does not stop the sweep (every
  // receive barrier must complete its phase): the column is still scaled
  // and pushed, CTL_RANK records the failure and the Newton step fails.
  template <int E, bool MB>
  __device__ bool normalize(int j, cplx<R> (&a)[E], double* col, double prev, int lane_maxcol,
                            unsigned long long* dbg = nullptr) const {
    R v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = c_norm_sqr(a[r]);  // rows >= N never enter the sum
    const R nrm2 = warp_canon(v, lane, N, kCanonP<E>);
    int ok = 0;
    R inv = rconst<R>(0.0);
    double mx = 0.0;
    if (lane == 0) {
      R rjj;
      r_sqrt_inv(nrm2, rjj, inv);
      const double d = r_hi(rjj);
      mx = d > prev ? d : prev;
      ok = d > sqrt_eps * mx;
      if (!ptk::finite(d)) atomicExch(W.ctl + CTL_NONFINITE, 1ull);  // see pt_path_stats.flags
      if constexpr (Team::kQInGlobal)
        W.rmaxp[j] = mx;
      else
        sh.pmax[j] = mx;
      if (ok) {
        store_r<R>(W.inv, n, j, inv);
        store_c<R>(W.Rm, SR, (long)j * n + j, cplx<R>{rjj, rconst<R>(0.0)});
      } else {
        atomicExch(W.ctl + CTL_RANK, epoch);
      }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    inv = shfl0(inv, 0);  // converged: shuffles never sit under a data-dependent branch
    if (MB || ok) {
#pragma unroll
      for (int r = 0; r < E; ++r) a[r] = c_scale(a[r], inv);
      store_col(col, N, a);
      if constexpr (Team::kQInGlobal) store_col(W.A + (long)j * N, SA, a);
    }
    if (dbg) dbg[4] = clock64() + (unsigned long long)(r_hi(a[0].re) == 12345.0);
    if constexpr (MB) {
      handoff(j, a, mx, lane_maxcol);
    } else {
      __syncwarp();
      if (lane == 0) team.publish(W.flags, j, epoch, !ok);
    }
    return ok != 0;
  }

  // r_kj = q_k^H a_j, a_j -= r_kj q_k; leaves the updated a_j in a.
  template <int E>
  // reg: the column lives in `a` (registers) and is neither loaded nor stored
  __device__ void project(int k, int j, const cplx<R> (&q)[E], cplx<R> (&a)[E], double* col, bool reg = false) const {
#ifdef PT_MGS_FINE  // stage clocks of the critical projection (tools/mgs_bench.cu only)
    unsigned long long* fd = (j == k + 1 && lane == 0) ? W.prof + kProfSlots + 6 * (n + 2) + 8 * j : nullptr;
#define PT_FINE(i, dep) \
  if (fd) fd[i] = clock64() + (unsigned long long)(r_hi(dep) == 12345.0);
#else
#define PT_FINE(i, dep)
#endif
    PT_FINE(0, q[0].re)
    if (!reg) load_col(col, N, a);
    PT_FINE(1, a[0].re)
    cplx<R> v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = c_conj_mul(q[r], a[r]);  // rows >= N never enter the sum
    PT_FINE(2, v[E - 1].im)
    cplx<R> rkj = warp_canon(v, lane, N, kCanonP<E>);
    PT_FINE(3, rkj.re)
    const cplx<R> r0 = rkj;
    rkj = shfl0(rkj, 0);
    PT_FINE(4, rkj.im)
    if (j < n || k < n - 1) {
#pragma unroll
      for (int r = 0; r < E; ++r) a[r] = c_sub(a[r], c_mul(rkj, q[r]));  // rows >= N: ignored garbage
      PT_FINE(5, a[E - 1].im)
      if (!reg) store_col(col, N, a);
    }
    if (lane == 0) store_c<R>(W.Rm, SR, (long)j * n + k, r0);  // off the chain
#undef PT_FINE
  }

  template <int E, bool MB>
  __device__ void run() const {
    if (!__isShared(colsm)) __builtin_unreachable();  // LDS/STS, not generic accesses
    const int c = team.block, G = cm.G();
    const int base = cm.base(c, w);
    const int par = sh.mgs_seq & 1;
    const int lane_maxcol = (MB && lane < team.nblocks) ? maxcol(lane) : -1;
    if constexpr (MB) {  // arm the receive barriers of the columns this CTA consumes but does not own
      if (w == kWarps - 1) {
        const int mc = maxcol(c);
        const uint32_t bytes = (uint32_t)(mgs_warp_qs(L, N) * 8);
        for (int k = lane; k < n && k < mc; k += 32) {
          int oc, ow, ols;
          cm.owner(k, oc, ow, ols);
          if (oc != c) mbar_expect(bars() + k, bytes);
        }
      }
    }
    if (base > n) return;  // owns no column
    // The first owned column (slot 0) stays in registers until it is
    // normalised (its slot then receives q for this CTA's consumers); the
    // others are staged in shared memory (each lane its own rows).
    cplx<R> ar[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane + 32 * r;
      ar[r] = i < N ? ldcg_c<R>(W.A + (long)base * N, SA, i) : c_zero<R>();
    }
    for (int j = base + G, m = 1; j <= n; j += G, ++m) {
      double* col = slot_ptr(m * kWarps + w);
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const int i = lane + 32 * r;
        if (i < N) store_c<R>(col, N, i, ldcg_c<R>(W.A + (long)j * N, SA, i));
      }
    }
    __syncwarp();
    cplx<R> a[E], q[E];
    if (base == 0) {
      if (!normalize<E, MB>(0, ar, slot_ptr(w), 0.0, lane_maxcol) && !MB) return;
    }
    const int last = base + ((n - base) / G) * G;
    const long QS = mgs_warp_qs(L, N);
    // owner of column k, tracked incrementally (no integer division on the chain):
    // r0 = k mod G, rb = r0 mod B, kc = (r0 / B) mod C, bc = r0 / (B C), slot = k / G
    int r0 = 0, rb = 0, kc = 0, bc = 0, kslot = 0;
    int jn = base;  // smallest owned column > k
    int mfirst = 0;
    for (int k = 0; k < n && k < last; ++k) {
      if (k > 0) {
        if (++r0 == G) {
          r0 = rb = kc = bc = 0;
          ++kslot;
        } else if (++rb == cm.B) {
          rb = 0;
          if (++kc == cm.C) {
            kc = 0;
            ++bc;
          }
        }
      }
      if (jn <= k) {
        jn += G;
        ++mfirst;
      }
      const int kw = bc * cm.B + rb, kls = kslot * kWarps + kw;
      const bool mine = kc == c && kw == w;
      const bool next_mine = jn == k + 1 && k + 1 < n;
      // timeline of the critical chain (tools/mgs_timeline.py): the owner of
      // column k+1 records when it starts waiting for q_k, has it, has
      // projected and normalised column k+1, and has pushed q_{k+1}
      unsigned long long* dbg = (next_mine && lane == 0) ? W.prof + kProfSlots + 6 * (k + 1) : nullptr;
      if (dbg) {
        dbg[0] = gtimer();
        dbg[1] = clock64();
      }
      double prev = 0.0;
      if (mine) {
        load_col(slot_ptr(kls), N, q);
      } else if constexpr (MB) {
        if (!__all_sync(0xffffffffu, mbar_wait(bars() + k, par, W.ctl))) return;  // watchdog abort
        if (kc == c) {  // the owner's slot in this CTA
          load_col(slot_ptr(kls), N, q);
          if (next_mine && lane == 0) prev = sh.pmax[k];
        } else {
          const double* msg = qbuf() + (long)k * QS;
          load_col(msg, N, q);
          if (next_mine && lane == 0) prev = msg[2 * L * N];
        }
      } else {
        int st = 0;
        if (lane == 0) st = team.wait(W.flags, k, epoch);
        st = __shfl_sync(0xffffffffu, st, 0);
        __syncwarp();
        if (st != 0) return;  // rank failure of column k, or abort
        if (kc == c) {  // this CTA's shared memory (the flag acquire ordered the owner's stores)
          load_col(slot_ptr(kls), N, q);
          if (next_mine && lane == 0) prev = Team::kQInGlobal ? *(volatile double*)(W.rmaxp + k) : sh.pmax[k];
        } else if constexpr (Team::kQInGlobal) {
#pragma unroll
          for (int r = 0; r < E; ++r) {
            const int i = lane + 32 * r;
            q[r] = i < N ? ldcg_c<R>(W.A + (long)k * N, SA, i) : c_zero<R>();
          }
          if (next_mine && lane == 0) prev = __ldcg(W.rmaxp + k);
        } else {
          const uint32_t qa = mapa_u32(smem_u32(slot_ptr(kls)), (uint32_t)kc);
#pragma unroll
          for (int r = 0; r < E; ++r) {
            const int i = lane + 32 * r;
            q[r] = i < N ? ldsc_c<R>(qa, N, i) : c_zero<R>();
          }
          if (next_mine && lane == 0) {
            double pv;
            asm volatile("ld.shared::cluster.f64 %0, [%1];"
                         : "=d"(pv)
                         : "r"(mapa_u32(smem_u32(sh.pmax + k), (uint32_t)kc)));
            prev = pv;
          }
        }
      }
      if (dbg) dbg[2] = clock64() + (unsigned long long)(r_hi(q[0].re) == 12345.0);  // after the loads land
      // owned columns > k, smallest (the look-ahead column k+1) first
      int m = mfirst;
      for (int j = jn; j <= n; j += G, ++m) {
        double* col = slot_ptr(m * kWarps + w);
        if (m == 0) {  // the register-resident column
          project(k, j, q, ar, col, true);
          if (j == k + 1 && j < n) {
            if (dbg) dbg[3] = clock64() + (unsigned long long)(r_hi(ar[0].re) == 12345.0);
            if (!normalize<E, MB>(j, ar, col, prev, lane_maxcol, dbg) && !MB) return;
            if (dbg) dbg[5] = gtimer();
          } else if (j == n && k == n - 1) {
            store_col(col, N, ar);  // column n (Q^H b lives in R; keep the slot coherent)
          }
          continue;
        }
        project(k, j, q, a, col);
        if (j == k + 1 && j < n) {
          if (dbg) dbg[3] = clock64() + (unsigned long long)(r_hi(a[0].re) == 12345.0);
          if (!normalize<E, MB>(j, a, col, prev, lane_maxcol, dbg) && !MB) return;
          if (dbg) dbg[5] = gtimer();
        }
      }
    }
  }
};

// one register-allocation unit per E (a QD E = 4 body must not make the
// E = 2 body spill)
template <class R, class Team, int E>
__device__ PT_MGS_WARP_INLINE void mgs_warp_e(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, double* colsm,
                                        unsigned long long epoch, double sqrt_eps) {
  __syncwarp();  // whole warps call this: converged entry (no WARPSYNC.COLLECTIVE fallback for its shuffles)
  constexpr int L = limbs_of<R>::L;
  double* qb = colsm + mgs_warp_slots_doubles(L, P.N, P.n, team.nblocks);
  uint64_t* bb = reinterpret_cast<uint64_t*>(qb + (long)P.n * mgs_warp_qs(L, P.N));
  const WarpMgs<R, Team> m{P,    W, team, sh, colsm, ColMap{team.nblocks, P.mgs_B}, (int)(threadIdx.x & 31),
                           (int)(threadIdx.x >> 5), P.N, P.n, (long)P.N * (P.n + 1), (long)P.n * (P.n + 1),
                           2L * L * P.N, epoch, sqrt_eps, qb, bb};
  if (P.mgs_warp == 2)
    m.template run<E, true>();
  else
    m.template run<E, false>();
}

template <class R, class Team>
__device__ __forceinline__ void mgs_warp(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, double* colsm,
                                         unsigned long long epoch, double sqrt_eps) {
  if (P.N <= 32)
    mgs_warp_e<R, Team, 1>(P, W, team, sh, colsm, epoch, sqrt_eps);
  else if (P.N <= 64)
    mgs_warp_e<R, Team, 2>(P, W, team, sh, colsm, epoch, sqrt_eps);
  else
    mgs_warp_e<R, Team, 4>(P, W, team, sh, colsm, epoch, sqrt_eps);
}

// Blocked back substitution R dx = y by the warps of one CTA (n <= 256):
// warp b owns the rows 32b .. 32b+31 (one per lane).  For b = top block down
// to 0: warp b solves its diagonal block sequentially (x_j = acc_j * (1/r_jj),
// shuffle, acc_i -= r_ij x_j for its rows i < j -- a one-element chain per
// step), publishes its x's in shared memory, and after one CTA barrier every
// warp a < b applies them to its rows in descending j.  Every row therefore
// subtracts r_ij x_j in exactly the oracle's order j = n-1 .. i+1.  Then
// u = max|dx| and x += dx.  Returns u (valid in every thread of the CTA).
template <class R>
__device__ __noinline__ double backsub_blocked(const DevPlan& P, const Work& W, const double* Rs, const double* invs,
                                               Smem<R>& sh, cplx<R>* xs) {
  __syncwarp();  // whole warps call this: converged entry (no WARPSYNC.COLLECTIVE fallback for its shuffles)
  const int n = P.n, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long SR = (long)n * (n + 1);
  const int nb = (n + 31) >> 5;
  const int i = 32 * w + lane;
  const bool row = w < nb && i < n;
  cplx<R> acc = row ? load_c<R>(Rs, SR, (long)n * n + i) : c_zero<R>();
  const R inv = row ? load_r<R>(invs, n, i) : rconst<R>(0.0);
  for (int b = nb - 1; b >= 0; --b) {
    const int j0 = 32 * b, jtop = min(n, j0 + 32) - 1;
    if (w == b) {  // diagonal block: the sequential chain
      const long long tb0 = clock64();
      // R column j is stored for every row 0..n-1 (entries below the diagonal
      // are unused), so the prefetch needs no guard; lanes past row n-1 read
      // up to 31 - 2n doubles past the last plane, inside the tail padding of
      // the staged copy (backsub_stage_doubles) or of the Rm / inv arrays
      // (make_layout), and never use the value
      cplx<R> cur = load_c<R>(Rs, SR, (long)jtop * n + i);
#pragma unroll 4
      for (int j = jtop; j >= j0; --j) {
        const int jl = j - j0;
        const cplx<R> nxt = load_c<R>(Rs, SR, (long)(j > 0 ? j - 1 : 0) * n + i);
        const cplx<R> xs_l = c_scale(acc, inv);  // meaningful in lane jl: dx_j
        acc = pick(lane == jl, xs_l, acc);
        const cplx<R> xj = shfl0(xs_l, jl);
        acc = pick(lane < jl, c_sub(acc, c_mul(cur, xj)), acc);
        cur = nxt;
      }
      if (row) xs[i] = acc;  // the block's x's, one store per lane after the chain
      (void)tb0;
    }
    __syncthreads();
    if (w < b && row) {  // apply block b's x's, descending j (products independent, subtractions in order)
#pragma unroll 4
      for (int j = jtop; j >= j0; --j) acc = c_sub(acc, c_mul(load_c<R>(Rs, SR, (long)j * n + i), xs[j]));
    }
  }
  double u = 0.0;
  if (row) {
    u = c_mod_double(acc);
    store_c<R>(W.dx, n, i, acc);
    store_c<R>(W.x, n, i, c_add(load_c<R>(W.x, n, i), acc));
  }
  return block_nan_max(u, sh.red);
}

// doubles of CTA 0's shared-memory copy of R (2L planes of n(n+1)) and 1/r_kk,
// plus 32 doubles of tail padding for the unguarded prefetch of the lanes past
// row n-1 in backsub_blocked (n < 16: up to 31 - 2n - Ln doubles past the copy)
__host__ __device__ inline size_t backsub_stage_doubles(int L, int n) {
  return (size_t)2 * L * n * (n + 1) + (size_t)L * n + 32;
}

// Back substitution of the warp MGS, run by CTA 0 after the MGS barrier: all
// its warps copy R (written by the column owners through L2) into shared
// memory with independent coalesced loads, then run the blocked solve on
// shared-memory reads.  stage == nullptr: R is read from global.
template <class R>
__device__ __forceinline__ double backsub_warp_body(const DevPlan& P, const Work& W, double* stage, Smem<R>& sh) {
  constexpr int L = limbs_of<R>::L;
  const int n = P.n;
  const double* Rs = W.Rm;
  const double* invs = W.inv;
  if (stage) {
    const long nr = 2L * L * n * (n + 1), ni = (long)L * n;
    // 16-byte loads, 8 in flight per thread (a dependent load->store loop
    // would pay one L2 round trip per element: ~23 us for a 64x65 DD R)
    const double2* src = reinterpret_cast<const double2*>(W.Rm);
    double2* dst = reinterpret_cast<double2*>(stage);
    const long nv = nr / 2;  // nr = 2L n(n+1) is even
    constexpr int U = 8;
    for (long q0 = threadIdx.x; q0 < nv; q0 += (long)U * blockDim.x) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long q = q0 + (long)u * blockDim.x;
        if (q < nv) v[u] = __ldcg(src + q);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long q = q0 + (long)u * blockDim.x;
        if (q < nv) dst[q] = v[u];
      }
    }
    for (long q = threadIdx.x; q < ni; q += blockDim.x) stage[nr + q] = __ldcg(W.inv + q);
    __syncthreads();
    Rs = stage;
    invs = stage + nr;
  }
  return backsub_blocked<R>(P, W, Rs, invs, sh, sh.tree);  // sh.tree: kThreads complex >= n x's
}

template <class R>
__device__ __noinline__ double backsub_warp(const DevPlan& P, const Work& W, double* stage, Smem<R>& sh) {
  const long long tb0 = clock64();
  const double u = backsub_warp_body<R>(P, W, stage, sh);
  if (threadIdx.x == 0 && W.prof) {  // debugging aid: cycles inside the back substitution (CTA 0)
    W.prof[6] += (unsigned long long)(clock64() - tb0);
    W.prof[7] += (unsigned long long)P.n;
  }
  return u;
}

}  // namespace ptdev
