// tcgen05 implicit GEMM (placeholder until the sm_100a kernel lands)
#include "gemm.cuh"
namespace nnl {
bool tc_eligible(const GemmProblem&, int) { return false; }
size_t tc_ws_bytes(const GemmProblem&) { return 0; }
int32_t tc_stat_rows(const GemmProblem&, int) { return 0; }
int tc_gemm(const GemmProblem&, int, void*, size_t, cudaStream_t) { return NNL_ERR_UNSUPPORTED; }
}  // namespace nnl
