// kern_dd_exact.cu -- the tracker kernels for R = dd with the reference's
// non-finite rule in dd_norm (multiprec.hpp:102-107: {h, 0} for a non-finite
// h).  kern_dd.cu is compiled with -DPT_DD_FAST_NONFINITE (no select on the
// DD critical chain); these kernels (a) serve evaluate_homotopy /
// least_squares_solve / the arithmetic entry points and (b) re-track, on the
// same stream, every path whose fast run met a non-finite value
// (PT_STAT_NONFINITE, include/pathtrack_b200.h).
#include "kernels.cuh"

#if defined(PT_DD_FAST_NONFINITE)
#error "kern_dd_exact.cu must be compiled without PT_DD_FAST_NONFINITE"
#endif

const ptdev::KernelSet ptdev::kset_dd_exact = {
    (const void*)&ptdev::k_track_grid<ptk::dd>,  (const void*)&ptdev::k_track_cluster<ptk::dd>,
    (const void*)&ptdev::k_track_batch<ptk::dd>, (const void*)&ptdev::k_eval<ptk::dd>,
    (const void*)&ptdev::k_lstsq<ptk::dd>,       (const void*)&ptdev::k_arith<ptk::dd>};
