// kernel_set.hpp -- per-precision tables of the tracker kernels.  Each
// precision's kernels are instantiated in their own translation unit
// (kern_d.cu, kern_dd.cu, kern_qd.cu); the host code in tracker.cu launches
// them through these untyped pointers (cudaLaunchKernelExC /
// cudaLaunchCooperativeKernel with argument arrays).
#pragma once

namespace ptdev {

struct KernelSet {
  const void* track_grid;     // k_track_grid<R>(DevPlan, Work, pt_step_params, TrackIO, u64 epoch)
  const void* track_cluster;  // k_track_cluster<R>(same)
  const void* track_batch;    // k_track_batch<R>(DevPlan, double*, u64*, Layout, pt_step_params, const double*,
                              //                  double*, pt_path_stats*, int, u64* queue, u64 epoch)
  const void* eval;           // k_eval<R>(DevPlan, Work, const double* x, double t, double* h, double* J, double* rmax)
  const void* lstsq;          // k_lstsq<R>(DevPlan, Work, u64 epoch, int* status)
  const void* arith;          // k_arith<R>(int op, long count, const double*, const double*, double*)
};
extern const KernelSet kset_d, kset_dd, kset_qd;
// dd with the reference's non-finite rule (kern_dd_exact.cu); kset_dd is the fast set
extern const KernelSet kset_dd_exact;
// qd in the tolerance-parity arithmetic (kern_qd_fast.cu, mp_qdfast.cuh)
extern const KernelSet kset_qd_fast;

struct MiscKernels {
  const void* fp64_peak;   // (double* out, int iters)
  const void* latency;     // (double* out, double seed)
  const void* mgs_pieces;  // (double* out)
  const void* barrier;     // (u64* ctl, int iters, double* out)
  const void* pingpong;    // (u64* flags, int iters, double* out)
};
extern const MiscKernels kmisc;
constexpr int kPeakChains = 8;  // independent DFMA chains per thread of k_fp64_peak

}  // namespace ptdev
