// Implicit-GEMM problem description shared by the SIMT and tcgen05 kernels.
//
//   D[m][n] = sum_k A(m,k) * B(n,k)      (f32 accumulation)
//
//   FPROP  (functions.py:187-194)  m=(b,p,q)  n=k_out  k=(r,s,c)   A=x gather, B=W[k_out][rsc]
//   DGRAD  (functions.py:208-209)  m=(b,h,w)  n=c      k=(r,s,ko)  A=dy gather, B=W[ko][r][s][c]
//   WGRAD  (functions.py:205-206)  m=k_out    n=(r,s,c) k=(b,p,q)  A=dy^T,      B=x gather
// Affine (functions.py:104-116) is the 1x1 / H=W=1 case with W stored (I,O).
#pragma once
#include "common.cuh"

namespace nnl {

enum GemmMode : int { kFprop = 0, kDgrad = 1, kWgrad = 2 };

struct ConvGeom {
  int32_t n, h, w, c, k, r, s, sh, sw, ph, pw, p, q;
  int32_t affine;  // weight stored (I,O): W[c][k] instead of W[k][c]
  // affine over an NHWC activation flattened in the reference's NCHW order:
  // physical feature f = hw*ac + ch  <->  weight row ch*ahw + hw
  int32_t ac, ahw;
};

__host__ __device__ __forceinline__ int64_t affine_row(const ConvGeom& g, int64_t f) {
  if (g.ahw == 1) return f;
  return (f % g.ac) * g.ahw + f / g.ac;
}

struct GemmProblem {
  int mode;
  ConvGeom g;
  int64_t M, N, K;
  const void* a;       // fprop: x; dgrad: dy; wgrad: dy
  const void* b;       // fprop/dgrad: w; wgrad: x
  const void* bias;    // fprop only (dtype), nullable
  void* out;           // dtype
  int acc;             // accumulate into out
  int out_trans;       // write D[m][n] at n*M + m (affine wgrad)
  int32_t* nonfinite;  // nullable
  void* bias_grad = nullptr;  // SIMT affine wgrad: also db[m] (+)= sum_k A(m, k)
  int acc_bias = 0;
  float* stats;        // fprop BN partials [rows][2][N] about stat_shift, nullable
  const float* stat_shift = nullptr;  // per-column centre K of the fprop statistics
  // dgrad with the following BN's backward statistics fused (TcArgs::bnx ...)
  const void* bnx = nullptr;
  const void* bn_gate = nullptr;
  const float *bn_mean = nullptr, *bn_istd = nullptr, *bn_gamma = nullptr, *bn_beta = nullptr;
  int bn_relu = 0, bn_canon = 0;
  void* bn_out = nullptr;
};

inline ConvGeom make_geom(const nnl_conv_shape& cs) {
  ConvGeom g;
  g.n = cs.n; g.h = cs.h; g.w = cs.w; g.c = cs.c; g.k = cs.k; g.r = cs.r; g.s = cs.s;
  g.sh = cs.stride_h; g.sw = cs.stride_w; g.ph = cs.pad_h; g.pw = cs.pad_w;
  g.p = cs.p; g.q = cs.q; g.affine = 0; g.ac = cs.c; g.ahw = 1;
  return g;
}

inline ConvGeom affine_geom(int64_t batch, int64_t in_f, int64_t in_c, int64_t out_f) {
  ConvGeom g;
  g.n = (int32_t)batch; g.h = 1; g.w = 1; g.c = (int32_t)in_f; g.k = (int32_t)out_f;
  g.r = 1; g.s = 1; g.sh = 1; g.sw = 1; g.ph = 0; g.pw = 0; g.p = 1; g.q = 1; g.affine = 1;
  g.ac = (int32_t)in_c;
  g.ahw = (int32_t)(in_f / in_c);
  return g;
}

inline void set_extent(GemmProblem& pb) {
  const ConvGeom& g = pb.g;
  int64_t npq = (int64_t)g.n * g.p * g.q;
  int64_t rsc = (int64_t)g.r * g.s * g.c;
  if (pb.mode == kFprop) { pb.M = npq; pb.N = g.k; pb.K = rsc; }
  if (pb.mode == kDgrad) { pb.M = (int64_t)g.n * g.h * g.w; pb.N = g.c; pb.K = (int64_t)g.r * g.s * g.k; }
  if (pb.mode == kWgrad) { pb.M = g.k; pb.N = rsc; pb.K = npq; }
}

// SIMT fallback (gemm_simt.cu)
int simt_gemm(const GemmProblem& pb, int dtype, void* ws, size_t ws_bytes, cudaStream_t st);
size_t simt_ws_bytes(const GemmProblem& pb);
// tcgen05 path (gemm_tc.cu): returns NNL_ERR_UNSUPPORTED when the shape is not eligible
int tc_gemm(const GemmProblem& pb, int dtype, void* ws, size_t ws_bytes, cudaStream_t st);
size_t tc_ws_bytes(const GemmProblem& pb);
bool tc_eligible(const GemmProblem& pb, int dtype);
int32_t tc_stat_rows(const GemmProblem& pb, int dtype);
// partial rows of a dgrad with fused BN-backward statistics (0: unsupported)
int32_t tc_bnb_rows(const GemmProblem& pb, int dtype);
// 3x3 / stride-1 weight gradients with shared halos (gemm_wgrad3.cu)
bool wgrad3_eligible(const GemmProblem& pb, int dtype);
size_t wgrad3_ws_bytes(const GemmProblem& pb);
int wgrad3_run(const GemmProblem& pb, void* ws, size_t ws_bytes, cudaStream_t st);
// the stem's wgrad over its x4 space-to-depth copy: f32 partials [splits][k][r2*64]
int wgrad_halo_x4(const void* x4, const void* dy, int n, int p, int q, int k, int r2,
                  float* partial, int max_splits, int* splits, cudaStream_t st);
// out[m*ldc + n] = q(prev + sum_s partial[s][m][n]) in fixed split order (gemm_tc.cu)
int tc_splitk_reduce(int M, int N, int splits, const float* partial, __half* out, int64_t ldc,
                     int acc, int32_t* nonfinite, cudaStream_t st);
// column sums of dy (bias gradient, functions.py:116,212): db[n] = q(prev + sum_m dy[m][n])
int bias_grad(int dtype, int64_t rows, int64_t cols, const void* dy, void* db, int acc,
              int32_t* nonfinite, void* ws, size_t ws_bytes, cudaStream_t st);
size_t bias_grad_ws_bytes(int64_t rows, int64_t cols);

}  // namespace nnl
