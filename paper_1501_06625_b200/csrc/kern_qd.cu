// kern_qd.cu -- the tracker kernels instantiated for R = ptk::qd (see kernels.cuh).
#include "kernels.cuh"

const ptdev::KernelSet ptdev::kset_qd = {
    (const void*)&ptdev::k_track_grid<ptk::qd>,  (const void*)&ptdev::k_track_cluster<ptk::qd>,
    (const void*)&ptdev::k_track_batch<ptk::qd>, (const void*)&ptdev::k_eval<ptk::qd>,
    (const void*)&ptdev::k_lstsq<ptk::qd>,       (const void*)&ptdev::k_arith<ptk::qd>};
