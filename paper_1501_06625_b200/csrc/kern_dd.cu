// kern_dd.cu -- the tracker kernels instantiated for R = ptk::dd (see kernels.cuh),
// compiled with -DPT_DD_FAST_NONFINITE (Makefile): dd_norm without the
// non-finite select; paths that meet a non-finite value are re-tracked by
// kern_dd_exact.cu (pt_path_stats.flags).
#include "kernels.cuh"

const ptdev::KernelSet ptdev::kset_dd = {
    (const void*)&ptdev::k_track_grid<ptk::dd>,  (const void*)&ptdev::k_track_cluster<ptk::dd>,
    (const void*)&ptdev::k_track_batch<ptk::dd>, (const void*)&ptdev::k_eval<ptk::dd>,
    (const void*)&ptdev::k_lstsq<ptk::dd>,       (const void*)&ptdev::k_arith<ptk::dd>};
