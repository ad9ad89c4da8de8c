// tcgen05 GEMM kernel instantiations with 64-wide tiles (see gemm_tc.cu)
#define NNL_TC_INSTANTIATE 64
#include "gemm_tc.cu"
