// C-ABI entry points for Convolution (functions.py:152-214) and Affine
// (functions.py:82-119).  Each call builds an implicit-GEMM problem and runs it
// on the tcgen05 kernel when the shape is eligible (fp16, 16-byte aligned
// rows), otherwise on the SIMT kernel (fp32 policy, odd channel counts).
#include "gemm.cuh"

using namespace nnl;

static int check_conv(const nnl_conv_shape* cs) {
  if (!cs) return fail(NNL_ERR_INVALID_ARGUMENT, "null conv shape");
  if (cs->n < 0 || cs->h <= 0 || cs->w <= 0 || cs->c <= 0 || cs->k <= 0 || cs->r <= 0 || cs->s <= 0)
    return fail(NNL_ERR_SHAPE_MISMATCH, "bad conv extents");
  if (cs->h + 2 * cs->pad_h < cs->r || cs->w + 2 * cs->pad_w < cs->s)
    return fail(NNL_ERR_KERNEL_TOO_LARGE, "window exceeds padded extent");
  if (cs->p != (cs->h + 2 * cs->pad_h - cs->r) / cs->stride_h + 1 ||
      cs->q != (cs->w + 2 * cs->pad_w - cs->s) / cs->stride_w + 1)
    return fail(NNL_ERR_SHAPE_MISMATCH, "output extent mismatch");
  return NNL_OK;
}

static int run_gemm(const GemmProblem& pb, int dtype, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (pb.M <= 0 || pb.N <= 0) return NNL_OK;
  if (g_tc_enabled && tc_eligible(pb, dtype)) {
    int rc = tc_gemm(pb, dtype, ws, ws_bytes, st);
    if (rc != NNL_ERR_UNSUPPORTED) return rc;
  }
  if (pb.stats) return fail(NNL_ERR_UNSUPPORTED, "BN statistics epilogue needs the tcgen05 path");
  return simt_gemm(pb, dtype, ws, ws_bytes, st);
}

static size_t gemm_ws(const GemmProblem& pb, int dtype) {
  size_t a = simt_ws_bytes(pb);
  size_t b = tc_eligible(pb, dtype) ? tc_ws_bytes(pb) : 0;
  return a > b ? a : b;
}

static GemmProblem conv_problem(const nnl_conv_shape* cs, int mode) {
  GemmProblem pb = {};
  pb.mode = mode;
  pb.g = make_geom(*cs);
  set_extent(pb);
  return pb;
}

// Stride-1 dgrad as a forward convolution (functions.py:208-209 restated):
// dx = conv(dy, W') with W'[c][r][s][k] = W[k][R-1-r][S-1-s][c] and padding
// R-1-p, so narrow output-channel layers (LeNet's conv2, K = 16) whose dgrad
// the tcgen05 plans do not take run on the forward path's tensor cores
// instead of the SIMT kernel.  Same sums per output (reduction order aside).
static bool dgrad_as_fprop(const nnl_conv_shape* cs, int dtype, GemmProblem& q) {
  if (dtype != NNL_F16 || !g_tc_enabled || cs->stride_h != 1 || cs->stride_w != 1 ||
      cs->pad_h > cs->r - 1 || cs->pad_w > cs->s - 1)
    return false;
  if (tc_eligible(conv_problem(cs, kDgrad), dtype)) return false;
  nnl_conv_shape f = *cs;
  f.h = cs->p; f.w = cs->q; f.c = cs->k; f.k = cs->c;
  f.pad_h = cs->r - 1 - cs->pad_h; f.pad_w = cs->s - 1 - cs->pad_w;
  f.p = cs->h; f.q = cs->w;
  q = conv_problem(&f, kFprop);
  return tc_eligible(q, dtype);
}

static size_t flip_bytes(const nnl_conv_shape* cs) {
  return ((size_t)cs->k * cs->c * cs->r * cs->s * 2 + 255) & ~(size_t)255;
}

__global__ void k_w_flip(int k, int c, int r, int s, const __half* __restrict__ w,
                         __half* __restrict__ wf) {
  pdl_wait();
  pdl_trigger();
  const int total = k * c * r * s;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    // wf[cc][rr][ss][kk] = w[kk][r-1-rr][s-1-ss][cc]
    const int kk = i % k, t = i / k;
    const int ss = t % s, t2 = t / s;
    const int rr = t2 % r, cc = t2 / r;
    wf[i] = w[(((int64_t)kk * r + (r - 1 - rr)) * s + (s - 1 - ss)) * c + cc];
  }
}

extern "C" {

size_t nnl_conv2d_workspace_size(const nnl_conv_shape* cs, int dtype, int pass) {
  if (check_conv(cs)) return 0;
  GemmProblem pb = conv_problem(cs, pass);
  size_t w = gemm_ws(pb, dtype);
  GemmProblem q;
  if (pass == kDgrad && dgrad_as_fprop(cs, dtype, q)) {
    const size_t f = flip_bytes(cs) + gemm_ws(q, dtype);
    if (f > w) w = f;
  }
  if (pass == kWgrad) {
    size_t b = bias_grad_ws_bytes((int64_t)cs->n * cs->p * cs->q, cs->k);
    if (b > w) w = b;
  }
  return w + 1024;
}

int32_t nnl_conv2d_stat_rows(const nnl_conv_shape* cs, int dtype) {
  if (check_conv(cs)) return 0;
  GemmProblem pb = conv_problem(cs, kFprop);
  if (!g_tc_enabled || !tc_eligible(pb, dtype)) return 0;
  return tc_stat_rows(pb, dtype);
}

int nnl_conv2d_fwd(const nnl_conv_shape* cs, int dtype, const void* x, const void* w,
                   const void* b, void* y, float* stat_partials, const float* stat_shift,
                   void* ws, size_t ws_bytes, void* stream) {
  int rc = check_conv(cs);
  if (rc) return rc;
  GemmProblem pb = conv_problem(cs, kFprop);
  pb.a = x; pb.b = w; pb.bias = b; pb.out = y; pb.stats = stat_partials;
  pb.stat_shift = stat_shift;
  return run_gemm(pb, dtype, ws, ws_bytes, as_stream(stream));
}

int nnl_conv2d_bwd_data(const nnl_conv_shape* cs, int dtype, const void* dy, const void* w,
                        void* dx, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_conv(cs);
  if (rc) return rc;
  GemmProblem pb = conv_problem(cs, kDgrad);
  pb.a = dy; pb.b = w; pb.out = dx; pb.acc = accumulate;
  GemmProblem q;
  if (dgrad_as_fprop(cs, dtype, q) && ws_bytes >= flip_bytes(cs) + gemm_ws(q, dtype)) {
    cudaStream_t st = as_stream(stream);
    __half* wf = reinterpret_cast<__half*>(ws);
    const int total = cs->k * cs->c * cs->r * cs->s;
    launch_k(k_w_flip, grid_for(total, 256), 256, 0, st, cs->k, cs->c, cs->r, cs->s,
             reinterpret_cast<const __half*>(w), wf);
    NNL_CHECK_LAUNCH();
    q.a = dy; q.b = wf; q.out = dx; q.acc = accumulate;
    return tc_gemm(q, dtype, reinterpret_cast<uint8_t*>(ws) + flip_bytes(cs),
                   ws_bytes - flip_bytes(cs), st);
  }
  return run_gemm(pb, dtype, ws, ws_bytes, as_stream(stream));
}

int32_t nnl_conv2d_bwd_data_bn_rows(const nnl_conv_shape* cs, int dtype) {
  if (check_conv(cs)) return 0;
  GemmProblem pb = conv_problem(cs, kDgrad);
  if (!g_tc_enabled || !tc_eligible(pb, dtype)) return 0;
  return tc_bnb_rows(pb, dtype);
}

int nnl_conv2d_bwd_data_bn(const nnl_conv_shape* cs, int dtype, const void* dy, const void* w,
                           void* dx, int accumulate, const nnl_bn_bwd_fuse* bf, void* ws,
                           size_t ws_bytes, void* stream) {
  int rc = check_conv(cs);
  if (rc) return rc;
  if (!bf || !bf->x || !bf->save_mean || !bf->save_istd || !bf->partials)
    return fail(NNL_ERR_INVALID_ARGUMENT, "incomplete BN-backward fusion descriptor");
  if (bf->relu && (bf->gate || !bf->gamma || !bf->beta))
    return fail(NNL_ERR_INVALID_ARGUMENT, "fused ReLU needs gamma/beta and no gate");
  GemmProblem pb = conv_problem(cs, kDgrad);
  if (!g_tc_enabled || !tc_eligible(pb, dtype) || tc_bnb_rows(pb, dtype) == 0)
    return fail(NNL_ERR_UNSUPPORTED, "BN-backward statistics epilogue not available");
  pb.a = dy; pb.b = w; pb.out = dx; pb.acc = accumulate;
  pb.stats = bf->partials;
  pb.bnx = bf->x; pb.bn_gate = bf->gate; pb.bn_mean = bf->save_mean; pb.bn_istd = bf->save_istd;
  pb.bn_gamma = bf->gamma; pb.bn_beta = bf->beta; pb.bn_relu = bf->relu;
  pb.bn_canon = bf->canonical; pb.bn_out = bf->out;
  return tc_gemm(pb, dtype, ws, ws_bytes, as_stream(stream));
}

int nnl_conv2d_bwd_weight(const nnl_conv_shape* cs, int dtype, const void* x, const void* dy,
                          void* dw, int acc_w, void* db, int acc_b, int32_t* nonfinite, void* ws,
                          size_t ws_bytes, void* stream) {
  int rc = check_conv(cs);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (dw) {
    GemmProblem pb = conv_problem(cs, kWgrad);
    pb.a = dy; pb.b = x; pb.out = dw; pb.acc = acc_w; pb.nonfinite = nonfinite;
    rc = run_gemm(pb, dtype, ws, ws_bytes, st);
    if (rc) return rc;
  }
  if (db) {
    rc = bias_grad(dtype, (int64_t)cs->n * cs->p * cs->q, cs->k, dy, db, acc_b, nonfinite, ws,
                   ws_bytes, st);
    if (rc) return rc;
  }
  return NNL_OK;
}

int nnl_affine_fwd(int dtype, int64_t batch, int64_t in_f, int64_t in_c, int64_t out_f, const void* x,
                   const void* w, const void* b, void* y, void* ws, size_t ws_bytes, void* stream) {
  GemmProblem pb = {};
  pb.mode = kFprop;
  pb.g = affine_geom(batch, in_f, in_c, out_f);
  set_extent(pb);
  pb.a = x; pb.b = w; pb.bias = b; pb.out = y;
  return run_gemm(pb, dtype, ws, ws_bytes, as_stream(stream));
}

int nnl_affine_bwd_data(int dtype, int64_t batch, int64_t in_f, int64_t in_c, int64_t out_f, const void* dy,
                        const void* w, void* dx, int accumulate, void* ws, size_t ws_bytes,
                        void* stream) {
  GemmProblem pb = {};
  pb.mode = kDgrad;
  pb.g = affine_geom(batch, in_f, in_c, out_f);
  set_extent(pb);
  pb.a = dy; pb.b = w; pb.out = dx; pb.acc = accumulate;
  return run_gemm(pb, dtype, ws, ws_bytes, as_stream(stream));
}

int nnl_affine_bwd_weight(int dtype, int64_t batch, int64_t in_f, int64_t in_c, int64_t out_f, const void* x,
                          const void* dy, void* dw, int acc_w, void* db, int acc_b,
                          int32_t* nonfinite, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  int rc;
  if (dw) {
    GemmProblem pb = {};
    pb.mode = kWgrad;
    pb.g = affine_geom(batch, in_f, in_c, out_f);
    set_extent(pb);
    pb.a = dy; pb.b = x; pb.out = dw; pb.acc = acc_w; pb.out_trans = 1; pb.nonfinite = nonfinite;
    if (db && !(g_tc_enabled && tc_eligible(pb, dtype))) {
      // the SIMT kernel takes the bias sums in the same pass (one launch)
      pb.bias_grad = db;
      pb.acc_bias = acc_b;
      return simt_gemm(pb, dtype, ws, ws_bytes, st);
    }
    rc = run_gemm(pb, dtype, ws, ws_bytes, st);
    if (rc) return rc;
  }
  if (db) {
    rc = bias_grad(dtype, batch, out_f, dy, db, acc_b, nonfinite, ws, ws_bytes, st);
    if (rc) return rc;
  }
  return NNL_OK;
}

}  // extern "C"

extern "C" size_t nnl_affine_workspace_size(int dtype, int64_t batch, int64_t in_f, int64_t out_f,
                                            int pass) {
  GemmProblem pb = {};
  pb.mode = pass;
  pb.g = affine_geom(batch, in_f, in_f, out_f);
  set_extent(pb);
  size_t w = gemm_ws(pb, dtype);
  if (pass == kWgrad) {
    size_t b = bias_grad_ws_bytes(batch, out_f);
    if (b > w) w = b;
  }
  return w + 1024;
}
