// mgs_batch.cuh -- the batch kernel's MGS least squares (one CTA per path,
// N <= 64), a throughput design for many paths per SM.
//
// Same arithmetic as the oracle (oracle/orc_tracker.hpp Tracker::lstsq,
// SPEC.md:296-322,339) and as the other MGS variants, bit for bit: r_kk =
// sqrt(canon_sum |a_k|^2), rank test in binary64 against the prefix max,
// q_k = a_k * (1/r_kk), r_kj = canon_sum conj(q_k) a_j, a_j -= r_kj q_k
// (skipped for the last update of column n); width_mgs(N) = 32, leaf
// p = c[p] + c[p+32].
//
// Work split (no CTA barrier inside the factorisation):
//  * warp 0 is the CRITICAL warp: for j = 1 .. n-1 it applies the last
//    projection q_{j-1} to column j and normalises it (lane = row, the
//    canonical tree as five shuffle levels, warp_canon), then publishes q_j --
//    the latency chain of the factorisation runs on one warp only;
//  * warps 1 .. 7 run the trailing projections as COLUMN ITEMS of 8 lanes:
//    lane c of an item holds rows c + 8m + 32e, i.e. the leaves = c mod 8 of
//    the canonical tree; it reduces them in registers (levels off = 16, 8)
//    and the item finishes with three shuffle levels (off = 4, 2, 1) -- every
//    lane busy on products, no 32-lane tree per column.  Item s owns the
//    columns 2 + s + 28 m (the right-hand side n included), the four items
//    of a warp own consecutive columns and step through k in lockstep.
// Hand-offs through shared memory flags (cleared per factorisation): qready[k]
// (1 = q_k published, 2 = rank failure: everybody stops, as the oracle
// returns at the first failing column) and cstep[j] = projections applied to
// column j by its item, which the critical warp waits for (j - 1 of them)
// before it takes column j over.
// Shared memory: 2L planes of (n+1) padded columns (stride bm_stride(N) =
// 8 mod 16 doubles: the two items of a half-warp hit distinct banks), then
// the two flag arrays.  R and 1/r_kk go to global (W.Rm, W.inv) for the back
// substitution, as in the other variants.
#pragma once

namespace ptdev {

constexpr int kBmLanes = 8;  // lanes per column item
constexpr int kBmMaxN = 64;
constexpr int kBmItems = (kWarps - 1) * (32 / kBmLanes);
__host__ __device__ inline int bm_stride(int N) { return ((N + 7) / 16) * 16 + 8; }
__host__ __device__ inline size_t bm_smem_doubles(int L, int N, int n) {
  return (size_t)2 * L * (n + 1) * bm_stride(N) + (size_t)(n + 1);  // + 2 (n+1) u32 flags
}

// Canonical width-32 sum over the leaves held by the 8 lanes of an item:
// v[m + 4e] = value of row c + 8m + 32e (rows >= N are ignored).  Valid in
// lane c == 0 of the item.  All 32 lanes of the warp execute it.
template <class T, int E2>
__device__ __forceinline__ T bm_tree(const T (&v)[4 * E2], int c, int N) {
  T leaf[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    leaf[m] = v[m];
    if constexpr (E2 == 2) leaf[m] = pick(c + 8 * m + 32 < N, add_v(leaf[m], v[m + 4]), leaf[m]);
  }
  leaf[0] = pick(c + 16 < N, add_v(leaf[0], leaf[2]), leaf[0]);  // off = 16
  leaf[1] = pick(c + 24 < N, add_v(leaf[1], leaf[3]), leaf[1]);
  leaf[0] = pick(c + 8 < N, add_v(leaf[0], leaf[1]), leaf[0]);   // off = 8
  __syncwarp();
#pragma unroll
  for (int off = 4; off >= 1; off >>= 1) {  // off = 4, 2, 1 inside the item
    const T o = shfl_down_r(leaf[0], off);
    leaf[0] = pick(c < off && c + off < N, add_v(leaf[0], o), leaf[0]);
  }
  return leaf[0];
}

// Poll a shared-memory flag until it is nonzero (watchdog: CTL_ABORT after
// kTimeoutNs, then 2 = "stop" is returned like a rank failure).
__device__ __forceinline__ uint32_t bm_wait_nonzero(const volatile uint32_t* f, unsigned long long* ctl) {
  uint32_t v = *f;
  if (v) {
    __threadfence_block();
    return v;
  }
  const unsigned long long t0 = gtimer();
  for (unsigned int spins = 1;; ++spins) {
    v = *f;
    if (v) {
      __threadfence_block();
      return v;
    }
    if ((spins & 1023u) == 0 && (ld_acquire(ctl + CTL_ABORT) || (double)(gtimer() - t0) > kTimeoutNs)) {
      atomicExch(ctl + CTL_ABORT, 1ull);
      return 2u;
    }
  }
}
__device__ __forceinline__ bool bm_wait_value(const volatile uint32_t* f, uint32_t want, unsigned long long* ctl) {
  if (*f == want) {
    __threadfence_block();
    return true;
  }
  const unsigned long long t0 = gtimer();
  for (unsigned int spins = 1;; ++spins) {
    if (*f == want) {
      __threadfence_block();
      return true;
    }
    if ((spins & 1023u) == 0 && (ld_acquire(ctl + CTL_ABORT) || (double)(gtimer() - t0) > kTimeoutNs)) {
      atomicExch(ctl + CTL_ABORT, 1ull);
      return false;
    }
  }
}

template <class R, int E2>
struct BatchMgs {
  static constexpr int L = limbs_of<R>::L;
  const DevPlan& P;
  const Work& W;
  double* As;
  volatile uint32_t* qready;  // [n + 1]
  volatile uint32_t* cstep;   // [n + 1]
  int N, n, CS;
  long PL, SR;
  unsigned long long epoch;
  double sqrt_eps;

  __device__ cplx<R> ld(int j, int i) const { return load_c<R>(As + (long)j * CS, PL, i); }
  __device__ void st(int j, int i, const cplx<R>& v) const { store_c<R>(As + (long)j * CS, PL, i, v); }

  // ---- the critical warp (lane = row lane + 32 e) ----
  // normalise column j held in a[]; publish q_j.  Returns the rank-test outcome.
  __device__ bool crit_normalize(int j, cplx<R> (&a)[E2], double& pmax, int lane) const {
    R v[E2];
#pragma unroll
    for (int e = 0; e < E2; ++e) v[e] = c_norm_sqr(a[e]);  // rows >= N never enter the sum
    const R nrm2 = warp_canon(v, lane, N, 32);
    int ok = 0;
    R inv = rconst<R>(0.0);
    if (lane == 0) {
      R rjj;
      r_sqrt_inv(nrm2, rjj, inv);
      const double d = r_hi(rjj);
      pmax = d > pmax ? d : pmax;
      ok = d > sqrt_eps * pmax;
      if (!ptk::finite(d)) atomicExch(W.ctl + CTL_NONFINITE, 1ull);  // see pt_path_stats.flags
      if (ok) {
        store_r<R>(W.inv, n, j, inv);
        store_c<R>(W.Rm, SR, (long)j * n + j, cplx<R>{rjj, rconst<R>(0.0)});
      } else {
        atomicExch(W.ctl + CTL_RANK, epoch);
      }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    inv = shfl0(inv, 0);
    if (ok) {
#pragma unroll
      for (int e = 0; e < E2; ++e) {
        const int i = lane + 32 * e;
        if (i < N) st(j, i, c_scale(a[e], inv));
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      qready[j] = ok ? 1u : 2u;
    }
    return ok != 0;
  }

  __device__ void critical(int lane) const {
    double pmax = 0.0;
    cplx<R> a[E2], q[E2];
#pragma unroll
    for (int e = 0; e < E2; ++e) {
      const int i = lane + 32 * e;
      a[e] = i < N ? ld(0, i) : c_zero<R>();
    }
    if (!crit_normalize(0, a, pmax, lane)) return;
    if (n == 1) {  // the right-hand side is column 1 (items own columns >= 2): r_01 only
#pragma unroll
      for (int e = 0; e < E2; ++e) {
        const int i = lane + 32 * e;
        q[e] = i < N ? ld(0, i) : c_zero<R>();
        a[e] = i < N ? ld(1, i) : c_zero<R>();
      }
      cplx<R> v[E2];
#pragma unroll
      for (int e = 0; e < E2; ++e) v[e] = c_conj_mul(q[e], a[e]);
      const cplx<R> r01 = warp_canon(v, lane, N, 32);
      if (lane == 0) store_c<R>(W.Rm, SR, 1L * n + 0, r01);
      return;
    }
    for (int j = 1; j < n; ++j) {
      if (j >= 2 && !__all_sync(0xffffffffu, lane != 0 || bm_wait_value(cstep + j, (uint32_t)(j - 1), W.ctl))) {
        if (lane == 0) qready[j] = 2u;  // abort: release the items
        return;
      }
      __syncwarp();
#pragma unroll
      for (int e = 0; e < E2; ++e) {
        const int i = lane + 32 * e;
        q[e] = i < N ? ld(j - 1, i) : c_zero<R>();
        a[e] = i < N ? ld(j, i) : c_zero<R>();
      }
      cplx<R> v[E2];
#pragma unroll
      for (int e = 0; e < E2; ++e) v[e] = c_conj_mul(q[e], a[e]);
      cplx<R> rkj = warp_canon(v, lane, N, 32);
      if (lane == 0) store_c<R>(W.Rm, SR, (long)j * n + (j - 1), rkj);
      rkj = shfl0(rkj, 0);
#pragma unroll
      for (int e = 0; e < E2; ++e) a[e] = c_sub(a[e], c_mul(rkj, q[e]));
      if (!crit_normalize(j, a, pmax, lane)) return;
    }
  }

  // ---- the column items (warps 1 ..) ----
  __device__ void items(int warp, int lane) const {
    const int c = lane & 7, g = lane >> 3;
    const int first = 2 + (warp - 1) * 4;  // the warp's smallest column
    if (first > n) return;
    // last step any item of this warp needs: its largest column jl (column
    // j < n needs k <= j - 2, the right-hand side n needs k <= n - 1)
    const int jl = min(n, first + ((n - first) / kBmItems) * kBmItems + 3);
    const int kmax = jl == n ? n - 1 : jl - 2;
    cplx<R> q[4 * E2];
    for (int k = 0; k <= kmax; ++k) {
      // q_k: the critical warp publishes it (qready[0] after column 0)
      uint32_t st_k = 0;
      if (lane == 0) st_k = bm_wait_nonzero(qready + k, W.ctl);
      st_k = __shfl_sync(0xffffffffu, st_k, 0);
      if (st_k != 1u) return;  // rank failure or abort
#pragma unroll
      for (int e = 0; e < 4 * E2; ++e) {
        const int i = c + 8 * (e & 3) + 32 * (e >> 2);
        q[e] = i < N ? ld(k, i) : c_zero<R>();
      }
      for (int j0 = first; j0 <= n; j0 += kBmItems) {
        const int j = j0 + g;
        const bool need = j <= n && (j < n ? k <= j - 2 : true);
        if (!__any_sync(0xffffffffu, need)) continue;  // warp-uniform: no item of the warp has work
        const int jc = need ? j : j0;  // loads of a valid column (results discarded)
        cplx<R> a[4 * E2], v[4 * E2];
#pragma unroll
        for (int e = 0; e < 4 * E2; ++e) {
          const int i = c + 8 * (e & 3) + 32 * (e >> 2);
          a[e] = i < N ? ld(jc, i) : c_zero<R>();
          v[e] = c_conj_mul(q[e], a[e]);
        }
        cplx<R> rkj = bm_tree<cplx<R>, E2>(v, c, N);
        if (need && c == 0) store_c<R>(W.Rm, SR, (long)j * n + k, rkj);
        rkj = shfl0(rkj, lane & ~7);
        if (need && (j < n || k < n - 1)) {
#pragma unroll
          for (int e = 0; e < 4 * E2; ++e) {
            const int i = c + 8 * (e & 3) + 32 * (e >> 2);
            if (i < N) st(j, i, c_sub(a[e], c_mul(rkj, q[e])));
          }
        }
        __syncwarp();
        if (need && c == 0) {
          __threadfence_block();
          cstep[j] = (uint32_t)(k + 1);
        }
      }
    }
  }
};

template <class R, int E2>
__device__ __noinline__ void mgs_batch_e(const DevPlan& P, const Work& W, double* As, unsigned long long epoch,
                                         double sqrt_eps) {
  __syncwarp();  // whole warps call this: converged entry (no WARPSYNC.COLLECTIVE fallback for its shuffles)
  if (!__isShared(As)) __builtin_unreachable();
  constexpr int L = limbs_of<R>::L;
  const int N = P.N, n = P.n;
  const int CS = bm_stride(N);
  const long PL = (long)(n + 1) * CS;
  const long SA = (long)N * (n + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  volatile uint32_t* qready = reinterpret_cast<volatile uint32_t*>(As + 2L * L * PL);
  volatile uint32_t* cstep = qready + (n + 1);
  // stage [J | -h] (column-major, stride N) into the padded planes; clear the flags
  for (int j = warp; j <= n; j += kWarps)
    for (int i = lane; i < N; i += 32)
#pragma unroll
      for (int l = 0; l < 2 * L; ++l) As[l * PL + (long)j * CS + i] = __ldcg(W.A + l * SA + (long)j * N + i);
  for (int j = tid; j <= n; j += kThreads) {
    qready[j] = 0u;
    cstep[j] = 0u;
  }
  __syncthreads();
  const BatchMgs<R, E2> m{P, W, As, qready, cstep, N, n, CS, PL, (long)n * (n + 1), epoch, sqrt_eps};
  if (warp == 0)
    m.critical(lane);
  else
    m.items(warp, lane);
}

template <class R>
__device__ __forceinline__ void mgs_batch(const DevPlan& P, const Work& W, double* As, unsigned long long epoch,
                                          double sqrt_eps) {
  if (P.N <= 32)
    mgs_batch_e<R, 1>(P, W, As, epoch, sqrt_eps);
  else
    mgs_batch_e<R, 2>(P, W, As, epoch, sqrt_eps);
}

}  // namespace ptdev
