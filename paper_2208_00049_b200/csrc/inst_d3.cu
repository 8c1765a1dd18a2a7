// inst_d3.cu — resampling kernels for D = 3 (all m, both precisions).
#define NFFTB_INSTANTIATE_D
#include "dispatch.cuh"
NFFTB_DEFINE_D(kernels_d3, 3)
