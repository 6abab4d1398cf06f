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

namespace ptdev {

constexpr int kWarpMgsMaxN = 128;  // E <= 4 elements per lane, width_mgs(N) <= 64

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

// Canonical width-P sum (P = width_mgs(N) in {32, 64}) of the values v[r]
// of rows lane + 32 r; the result is valid in lane 0.
template <class T, int E>
__device__ __forceinline__ T warp_canon(const T (&v)[E], int lane, int N, int P) {
  T acc = v[0];
  if (P == 32) {
#pragma unroll
    for (int r = 1; r < E; ++r)
      if (lane + 32 * r < N) acc = add_v(acc, v[r]);
  } else {  // P == 64 (65 <= N <= 128): partial l = c[l] + c[l+64], partial l+32 = c[l+32] + c[l+96]
    if constexpr (E > 2) {
      if (lane + 64 < N) acc = add_v(acc, v[2]);
    }
    if constexpr (E > 1) {
      T a1 = v[1];
      if constexpr (E > 3) {
        if (lane + 96 < N) a1 = add_v(a1, v[3]);
      }
      acc = add_v(acc, a1);  // off = 32 level: l + 32 < 65 <= N always
    }
  }
  __syncwarp();
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const T o = shfl_down_r(acc, off);
    if (lane < off && lane + off < N) acc = add_v(acc, o);
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
// Wait for phase `parity` of a receive barrier; a stalled exchange traps
// (cluster barriers cannot be abandoned) after the watchdog time.
__device__ __forceinline__ void mbar_wait(uint64_t* b, int parity, unsigned long long* ctl) {
  if (mbar_try(b, parity)) return;
  const unsigned long long t0 = gtimer();
  for (unsigned int spins = 1;; ++spins) {
    if (mbar_try(b, parity)) return;
    if ((spins & 1023u) == 0 && (double)(gtimer() - t0) > kTimeoutNs) {
      atomicExch(ctl + CTL_ABORT, 1ull);
      __trap();
    }
  }
}
__device__ __forceinline__ void st_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
               "r"(rbar)
               : "memory");
}

// Dynamic shared memory of the warp MGS, per CTA (doubles / u64 words):
//   [column slots: S * kWarps * 2L*N][Q buffer: n * QS][n mbarriers]
// Q buffer row k = the message of column k: q_k (2L planes of N) + pmax_k.
// The Q buffer exists only in the mbarrier exchange (cluster / block teams);
// the grid team exchanges q_k through L2 with release/acquire flags.
__host__ __device__ inline long mgs_warp_qs(int L, int N) { return 2L * L * N + 1; }
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
  const Work& W;
  const Team& team;
  Smem<R>& sh;
  double* colsm;  // this CTA's dynamic smem (layout above)
  ColMap cm;
  int lane, w, N, n;
  long SA, SR, CS;
  unsigned long long epoch;
  double sqrt_eps;

  __device__ double* slot_ptr(int ls) const { return colsm + (long)ls * CS; }
  __device__ double* qbuf() const { return colsm + mgs_warp_slots_doubles(L, N, n, team.nblocks); }
  __device__ uint64_t* bars() const { return reinterpret_cast<uint64_t*>(qbuf() + (long)n * mgs_warp_qs(L, N)); }

  template <int E>
  __device__ __forceinline__ void load_col(const double* p, long S, cplx<R> (&a)[E]) const {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane + 32 * r;
      if (i < N) a[r] = load_c<R>(p, S, i);
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

  // Push the message of column j (q_j in a, pmax in lane 0) into the Q buffer
  // of every CTA that owns a column > j, the CTA of column j+1 first.
  // need: bit d set iff CTA d owns a column > j (lane-parallel ballot).
  template <int E>
  __device__ void push(int j, const cplx<R> (&a)[E], double pmax, int lane_maxcol) const {
    const unsigned need = __ballot_sync(0xffffffffu, lane < team.nblocks && lane_maxcol > j);
    int c1, w1, l1;
    cm.owner(j + 1 <= n ? j + 1 : j, c1, w1, l1);
    const long QS = mgs_warp_qs(L, N);
    const uint32_t qloc = smem_u32(qbuf() + (long)j * QS), bloc = smem_u32(bars() + j);
    unsigned rest = need;
    for (int it = 0; rest; ++it) {
      const int d = (it == 0 && (rest >> c1) & 1u) ? c1 : __ffs(rest) - 1;
      rest &= ~(1u << d);
      const uint32_t rq = mapa_u32(qloc, (uint32_t)d), rb = mapa_u32(bloc, (uint32_t)d);
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const int i = lane + 32 * r;
        if (i < N) {
#pragma unroll
          for (int l = 0; l < L; ++l) {
            st_async(rq + 8u * (uint32_t)(l * N + i), r_limb(a[r].re, l), rb);
            st_async(rq + 8u * (uint32_t)((L + l) * N + i), r_limb(a[r].im, l), rb);
          }
        }
      }
      if (lane == 0) st_async(rq + 8u * (uint32_t)(2 * L * N), pmax, rb);
    }
  }

  // Normalise column j (values a, already projected against q_0..q_{j-1}),
  // then hand q_j to the consumers.  prev = max_{k<j} binary64 r_kk.  With
  // the mbarrier exchange a rank failure does not stop the sweep (every
  // receive barrier must complete its phase): the column is still scaled
  // and pushed, CTL_RANK records the failure and the Newton step fails.
  template <int E, bool MB>
  __device__ bool normalize(int j, cplx<R> (&a)[E], double* col, double prev, int lane_maxcol) const {
    R v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = (lane + 32 * r < N) ? c_norm_sqr(a[r]) : rconst<R>(0.0);
    const R nrm2 = warp_canon(v, lane, N, P.P_mgs);
    int ok = 0;
    R inv = rconst<R>(0.0);
    double mx = 0.0;
    if (lane == 0) {
      const R rjj = r_sqrt(nrm2);
      const double d = r_hi(rjj);
      mx = d > prev ? d : prev;
      ok = d > sqrt_eps * mx;
      if constexpr (!MB) {
        if constexpr (Team::kQInGlobal)
          W.rmaxp[j] = mx;
        else
          sh.pmax[j] = mx;
      }
      inv = r_div(rconst<R>(1.0), rjj);
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
    if constexpr (MB) {
      push(j, a, mx, lane_maxcol);
    } else {
      __syncwarp();
      if (lane == 0) team.publish(W.flags, j, epoch, !ok);
    }
    return ok != 0;
  }

  // r_kj = q_k^H a_j, a_j -= r_kj q_k; leaves the updated a_j in a.
  template <int E>
  __device__ void project(int k, int j, const cplx<R> (&q)[E], cplx<R> (&a)[E], double* col) const {
    load_col(col, N, a);
    cplx<R> v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = (lane + 32 * r < N) ? c_conj_mul(q[r], a[r]) : c_zero<R>();
    cplx<R> rkj = warp_canon(v, lane, N, P.P_mgs);
    if (lane == 0) store_c<R>(W.Rm, SR, (long)j * n + k, rkj);
    rkj = shfl0(rkj, 0);
    if (j < n || k < n - 1) {
#pragma unroll
      for (int r = 0; r < E; ++r)
        if (lane + 32 * r < N) a[r] = c_sub(a[r], c_mul(rkj, q[r]));
      store_col(col, N, a);
    }
  }

  template <int E, bool MB>
  __device__ void run() const {
    const int c = team.block, G = cm.G();
    const int base = cm.base(c, w);
    const int par = sh.mgs_seq & 1;
    const int lane_maxcol = (MB && lane < team.nblocks) ? maxcol(lane) : -1;
    if constexpr (MB) {  // arm this CTA's receive barriers for the columns it consumes
      if (threadIdx.x == 0) {
        const int mc = maxcol(c);
        const uint32_t bytes = (uint32_t)(mgs_warp_qs(L, N) * 8);
        for (int k = 0; k < n && k < mc; ++k) mbar_expect(bars() + k, bytes);
      }
    }
    if (base > n) return;  // owns no column
    // stage the owned columns in shared memory (each lane its own rows)
    for (int j = base, m = 0; j <= n; j += G, ++m) {
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
      load_col(slot_ptr(w), N, a);
      if (!normalize<E, MB>(0, a, slot_ptr(w), 0.0, lane_maxcol) && !MB) return;
    }
    const int last = base + ((n - base) / G) * G;
    const long QS = mgs_warp_qs(L, N);
    for (int k = 0; k < n && k < last; ++k) {
      int kc, kw, kls;
      cm.owner(k, kc, kw, kls);
      const bool mine = kc == c && kw == w;
      const bool next_mine = (k + 1) % G == base && k + 1 < n;
      double prev = 0.0;
      if (mine) {
        load_col(slot_ptr(kls), N, q);
      } else if constexpr (MB) {
        mbar_wait(bars() + k, par, W.ctl);
        const double* msg = qbuf() + (long)k * QS;
        load_col(msg, N, q);
        if (next_mine && lane == 0) prev = msg[2 * L * N];
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
            if (i < N) q[r] = ldcg_c<R>(W.A + (long)k * N, SA, i);
          }
          if (next_mine && lane == 0) prev = __ldcg(W.rmaxp + k);
        } else {
          const uint32_t qa = mapa_u32(smem_u32(slot_ptr(kls)), (uint32_t)kc);
#pragma unroll
          for (int r = 0; r < E; ++r) {
            const int i = lane + 32 * r;
            if (i < N) q[r] = ldsc_c<R>(qa, N, i);
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
      // owned columns > k, smallest (the look-ahead column k+1) first
      int m = k + 1 <= base ? 0 : (k + 1 - base + G - 1) / G;
      for (int j = base + m * G; j <= n; j += G, ++m) {
        double* col = slot_ptr(m * kWarps + w);
        project(k, j, q, a, col);
        if (j == k + 1 && j < n)
          if (!normalize<E, MB>(j, a, col, prev, lane_maxcol) && !MB) return;
      }
    }
  }
};

// one register-allocation unit per E (a QD E = 4 body must not make the
// E = 2 body spill)
template <class R, class Team, int E>
__device__ __noinline__ void mgs_warp_e(const DevPlan& P, const Work& W, const Team& team, Smem<R>& sh, double* colsm,
                                        unsigned long long epoch, double sqrt_eps) {
  const WarpMgs<R, Team> m{P,    W, team, sh, colsm, ColMap{team.nblocks, P.mgs_B}, (int)(threadIdx.x & 31),
                           (int)(threadIdx.x >> 5), P.N, P.n, (long)P.N * (P.n + 1), (long)P.n * (P.n + 1),
                           2L * limbs_of<R>::L * P.N, epoch, sqrt_eps};
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

// Back substitution R dx = y by one warp, rows lane + 32 r, column-oriented
// with column j-1 of R prefetched while column j is applied; then
// u = max|dx|, x += dx.  Returns u in every lane.
template <class R, int E>
__device__ __noinline__ double backsub_warp_e(const DevPlan& P, const Work& W) {
  const int n = P.n, lane = threadIdx.x & 31;
  const long SR = (long)n * (n + 1);
  cplx<R> acc[E], cur[E], nxt[E];
  R inv[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int i = lane + 32 * r;
    if (i < n) {
      acc[r] = load_c<R>(W.Rm, SR, (long)n * n + i);
      inv[r] = load_r<R>(W.inv, n, i);
      if (i < n - 1) cur[r] = load_c<R>(W.Rm, SR, (long)(n - 1) * n + i);
    }
  }
  for (int j = n - 1; j >= 0; --j) {
    const int ol = j & 31, orow = j >> 5;
    cplx<R> xj = c_zero<R>();
#pragma unroll
    for (int r = 0; r < E; ++r)
      if (r == orow && lane == ol) {
        acc[r] = c_scale(acc[r], inv[r]);  // row j finished: dx_j
        xj = acc[r];
      }
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane + 32 * r;
      if (i < j - 1) nxt[r] = load_c<R>(W.Rm, SR, (long)(j - 1) * n + i);
    }
    xj = shfl0(xj, ol);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane + 32 * r;
      if (i < j) acc[r] = c_sub(acc[r], c_mul(cur[r], xj));
      cur[r] = nxt[r];
    }
  }
  double u = 0.0;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int i = lane + 32 * r;
    if (i < n) {
      u = nan_max(u, c_mod_double(acc[r]));
      store_c<R>(W.dx, n, i, acc[r]);
      store_c<R>(W.x, n, i, c_add(load_c<R>(W.x, n, i), acc[r]));
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) u = nan_max(u, __shfl_xor_sync(0xffffffffu, u, off));
  return u;
}

template <class R>
__device__ __forceinline__ double backsub_warp(const DevPlan& P, const Work& W) {
  if (P.n <= 32) return backsub_warp_e<R, 1>(P, W);
  if (P.n <= 64) return backsub_warp_e<R, 2>(P, W);
  return backsub_warp_e<R, 4>(P, W);
}

}  // namespace ptdev
