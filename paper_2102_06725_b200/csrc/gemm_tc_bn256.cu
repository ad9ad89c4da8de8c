// tcgen05 GEMM kernel instantiations with 256-wide tiles (see gemm_tc.cu)
#define NNL_TC_INSTANTIATE 256
#include "gemm_tc.cu"
