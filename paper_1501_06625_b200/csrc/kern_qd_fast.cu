// kern_qd_fast.cu -- the tracker kernels for R = qd in the tolerance-parity
// arithmetic (compiled with -DPT_QD_FAST, Makefile): the QD operations of
// mp.cuh run the classic quad-double algorithms of mp_qdfast.cuh and the MGS
// normalisations use one reciprocal square root (r_sqrt_inv).  Selected per
// plan by pt_plan_set_arith(PT_ARITH_FAST); kern_qd.cu stays the default,
// bit-identical set.
#include "kernels.cuh"

#if !defined(PT_QD_FAST)
#error "kern_qd_fast.cu must be compiled with -DPT_QD_FAST"
#endif

const ptdev::KernelSet ptdev::kset_qd_fast = {
    (const void*)&ptdev::k_track_grid<ptk::qd>,  (const void*)&ptdev::k_track_cluster<ptk::qd>,
    (const void*)&ptdev::k_track_batch<ptk::qd>, (const void*)&ptdev::k_eval<ptk::qd>,
    (const void*)&ptdev::k_lstsq<ptk::qd>,       (const void*)&ptdev::k_arith<ptk::qd>};
