// inst_d2.cu — resampling kernels for D = 2 (all m, both precisions).
#define NFFTB_INSTANTIATE_D
#include "dispatch.cuh"
NFFTB_DEFINE_D(kernels_d2, 2)
