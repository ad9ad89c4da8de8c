// tcgen05 GEMM kernel instantiations with 128-wide tiles (see gemm_tc.cu)
#define NNL_TC_INSTANTIATE 128
#include "gemm_tc.cu"
