// Streaming BatchNormalization kernels (bn_stream.cu), used by bn.cu for fp16
// activations with C % 8 == 0 and C <= 2048.
#pragma once
#include "common.cuh"

namespace nnl {

enum BnStreamMode { BNS_STATS_F = 0, BNS_APPLY_F = 1, BNS_STATS_B = 2, BNS_APPLY_B = 3 };

struct BnStreamArgs {
  int64_t rows;
  int32_t c;
  int32_t chunk_rows;  // filled by bn_stream_launch
  int64_t nchunks;     // filled by bn_stream_launch
  const __half* x;
  const __half* dy;
  __half* out;
  const float* gamma;
  const float* beta;
  const float* mu;
  const float* istd;
  const float* gsum;   // [2][C] gbeta, ggamma (APPLY_B)
  float* partials;     // [grid][2][C] (STATS_*, APPLY_B bias sums)
  // STATS_F centre K[c]: partials are sum(x-K), sum((x-K)^2) so a channel whose
  // |mean| >> std does not cancel; null -> K = x[0][c] (the first row)
  const float* shift;
  int relu;
  int acc;
  int batch_stat;
  // residual tail (BN -> Add2 -> ReLU):
  const __half* res;   // APPLY_F: y = relu(q(q(bn(x)) + res)), streamed
  const __half* gate;  // STATS_B / APPLY_B: gy *= (gate > 0), streamed
  __half* dres;        // STATS_B with gate: dres = q(0 + gated gy)
  // walk the chunks last to first: the tail of a tensor its producer has just
  // written (or the previous pass has just read) is still in the 126 MB L2
  int reverse;
};

bool bn_stream_ok(int64_t rows, int32_t c, const void* a, const void* b, const void* d);
// streamed tensors of a launch: x, plus dy (backward) or res, plus gate
int bn_stream_nt(int mode, const BnStreamArgs& a);
// number of partial rows the launch writes (its grid size)
int bn_stream_rows(int mode, int nt, int64_t rows, int32_t c);
int bn_stream_launch(int mode, const BnStreamArgs& a, cudaStream_t st);

}  // namespace nnl
