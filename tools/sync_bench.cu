// Cross-warp / cross-CTA hand-off latency on B200 (design input for the MGS
// q_k exchange).  Ping-pong of a 2 KB message (64 complex DD entries) between
// warp 0 of CTA 0 and warp 0 of CTA `peer` in one cluster, or between two
// warps of one CTA, with several mechanisms; prints ns per one-way hand-off.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_bench sync_bench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ uint32_t crank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_async2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}

constexpr int MSG = 256;  // doubles (2 KB)
constexpr int ITERS = 200;

// mode 0: flag in receiver smem, data pulled by the receiver via DSMEM (fence.acq_rel.cluster both sides)
// mode 1: st.async push of data into receiver smem + mbarrier complete_tx
// mode 2: same CTA, two warps: data in smem, volatile flag + __threadfence_block
// mode 3: same CTA, st.async to own CTA + mbarrier
__global__ void __cluster_dims__(2, 1, 1) k(int mode, double* out) {
  __shared__ __align__(16) double buf[2][ITERS % 2 + 2][MSG];
  __shared__ __align__(8) uint64_t bar[2][ITERS];
  __shared__ volatile uint32_t flag[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t me = crank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < ITERS; ++i) {
      mbar_init(&bar[0][i], 1);
      mbar_init(&bar[1][i], 1);
    }
    flag[0] = flag[1] = 0;
  }
  for (int i = threadIdx.x; i < 2 * MSG * 2; i += blockDim.x) (&buf[0][0][0])[i] = 1.0;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  csync();
  const bool cross = mode < 2;
  // roles: A = (cta 0, warp 0), B = cross ? (cta 1, warp 0) : (cta 0, warp 1)
  const bool isA = me == 0 && warp == 0;
  const bool isB = cross ? (me == 1 && warp == 0) : (me == 0 && warp == 1);
  if (mode == 1 || mode == 3) {
    // arm every barrier of my receive side: side index = 1 for B's buffer, 0 for A's
    if (lane == 0 && (isA || isB))
      for (int i = 0; i < ITERS; ++i) mbar_expect(&bar[isA ? 0 : 1][i], MSG * 8);
  }
  csync();
  unsigned long long t0 = gt();
  double acc = 0;
  if (isA || isB) {
    const int side = isA ? 0 : 1;  // my receive buffer
    const uint32_t peer = cross ? (me ^ 1u) : me;
    for (int i = 0; i < ITERS; ++i) {
      const bool send = (i & 1) == (isA ? 0 : 1);
      if (send) {
        double v[MSG / 32];
        for (int r = 0; r < MSG / 32; ++r) v[r] = acc + r;
        if (mode == 0) {
          // write to my own smem, release flag in the peer
          for (int r = 0; r < MSG / 32; ++r) buf[side][0][lane + 32 * r] = v[r];
          __syncwarp();
          if (lane == 0) {
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"r"(mapa(smem_u32((const void*)&flag[side ^ 1]), peer)),
                         "r"((uint32_t)i + 1)
                         : "memory");
          }
        } else if (mode == 1 || mode == 3) {
          const uint32_t rb = mapa(smem_u32(&bar[side ^ 1][i]), peer);
          const uint32_t rd = mapa(smem_u32(&buf[side ^ 1][0][0]), peer);
          for (int r = 0; r < MSG / 64; ++r)
            st_async2(rd + 8 * (2 * lane + 64 * r), v[2 * r], v[2 * r + 1], rb);
        } else {
          for (int r = 0; r < MSG / 32; ++r) buf[side][0][lane + 32 * r] = v[r];
          __syncwarp();
          if (lane == 0) {
            __threadfence_block();
            flag[side ^ 1] = (uint32_t)i + 1;
          }
        }
      } else {
        if (mode == 0) {
          if (lane == 0) {
            for (;;) {
              uint32_t f;
              asm volatile("ld.relaxed.cluster.shared::cta.u32 %0, [%1];" : "=r"(f) : "r"(smem_u32((const void*)&flag[side])) : "memory");
              if (f == (uint32_t)i + 1) break;
            }
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
          }
          __syncwarp();
          const uint32_t src = mapa(smem_u32(&buf[side ^ 1][0][0]), peer);
          for (int r = 0; r < MSG / 32; ++r) {
            double d;
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(d) : "r"(src + 8 * (lane + 32 * r)));
            acc += d;
          }
        } else if (mode == 1 || mode == 3) {
          mbar_wait(&bar[side][i], 0);
          for (int r = 0; r < MSG / 32; ++r) acc += buf[side][0][lane + 32 * r];
        } else {
          if (lane == 0)
            while (flag[side] != (uint32_t)i + 1) {
            }
          __syncwarp();
          __threadfence_block();
          for (int r = 0; r < MSG / 32; ++r) acc += buf[side ^ 1][0][lane + 32 * r];
        }
        acc = __shfl_sync(0xffffffffu, acc, 0) * 1e-3;
      }
    }
  }
  unsigned long long t1 = gt();
  if (isA && lane == 0) out[mode] = (double)(t1 - t0) / ITERS;
  if (isA && lane == 0) out[8 + mode] = acc;
  csync();
}

int main() {
  double* d;
  cudaMalloc(&d, 256);
  cudaMemset(d, 0, 256);
  for (int m = 0; m < 4; ++m) {
    k<<<2, 64>>>(m, d);
    k<<<2, 64>>>(m, d);
  }
  cudaError_t e = cudaDeviceSynchronize();
  double h[16];
  cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("{\"err\": \"%s\", \"ns_per_handoff\": {\"dsmem_pull_flag_fence\": %.1f, \"st_async_push_mbar\": %.1f, "
         "\"same_cta_volatile_flag\": %.1f, \"same_cta_st_async_mbar\": %.1f}}\n",
         cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
}
