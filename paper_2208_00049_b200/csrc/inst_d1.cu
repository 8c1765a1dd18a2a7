// inst_d1.cu — resampling kernels for D = 1 (all m, both precisions).
#define NFFTB_INSTANTIATE_D
#include "dispatch.cuh"
NFFTB_DEFINE_D(kernels_d1, 1)
