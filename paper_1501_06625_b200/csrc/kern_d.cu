// kern_d.cu -- the tracker kernels instantiated for R = double (see kernels.cuh).
#include "kernels.cuh"

const ptdev::KernelSet ptdev::kset_d = {
    (const void*)&ptdev::k_track_grid<double>,  (const void*)&ptdev::k_track_cluster<double>,
    (const void*)&ptdev::k_track_batch<double>, (const void*)&ptdev::k_eval<double>,
    (const void*)&ptdev::k_lstsq<double>,       (const void*)&ptdev::k_arith<double>};
