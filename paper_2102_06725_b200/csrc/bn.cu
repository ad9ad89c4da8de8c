// BatchNormalization (src/functions.py:363-441) on channel-innermost buffers
// [rows][C] (rows = N*H*W of an NHWC activation, or the batch of a 2-D input).
//
// Pipeline per call:
//   1. k_bn_partials   : one HBM pass, per-block f32 partial sums -> [R][2][C]
//                        (skipped in forward when the conv epilogue already
//                        produced the partials of the same rounded values)
//   2. k_bn_finalize_* : deterministic fixed-order f64 reduction of the R
//                        partial rows; mean/biased var/istd + running stats
//                        (fwd) or gbeta/ggamma + param grads (bwd)
//   3. k_bn_*_apply    : one HBM pass writing y (fwd, optional fused ReLU)
//                        or gx (bwd, optional fused ReLU gate)
// Op order in every f32 expression follows the reference line by line with
// explicit _rn intrinsics (no FMA contraction), so results differ from numpy
// only through the summation order of the statistics.
#include "common.cuh"

namespace nnl {

constexpr int kBnThreads = 256;

struct BnGeom {
  int vec;        // channels per thread (8 or 1)
  int groups;     // channel groups per row in one slab
  int lanes;      // rows processed concurrently by a block
  int slabs;      // grid.y
};

static BnGeom bn_geom(int32_t c, bool vec_ok) {
  BnGeom g;
  g.vec = (vec_ok && c % 8 == 0) ? 8 : 1;
  int total_groups = c / g.vec;
  g.groups = total_groups < kBnThreads ? total_groups : kBnThreads;
  g.lanes = kBnThreads / g.groups;
  g.slabs = (total_groups + g.groups - 1) / g.groups;
  return g;
}

template <typename T, int V>
struct VecLoad;
template <typename T>
struct VecLoad<T, 1> {
  static __device__ __forceinline__ void load(const T* p, float* out) { out[0] = Elem<T>::load(p); }
};
template <>
struct VecLoad<__half, 8> {
  static __device__ __forceinline__ void load(const __half* p, float* out) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __half22float2(h[j]);
      out[2 * j] = f.x;
      out[2 * j + 1] = f.y;
    }
  }
};
template <>
struct VecLoad<float, 8> {
  static __device__ __forceinline__ void load(const float* p, float* out) {
    float4 a = reinterpret_cast<const float4*>(p)[0];
    float4 b = reinterpret_cast<const float4*>(p)[1];
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
    out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
  }
};

// MODE 0: (sum x, sum x^2)                               -- forward statistics
// MODE 1: (sum gy, sum gy*xhat), gy gated by relu_out>0  -- backward reductions
template <typename T, int V, int MODE>
__global__ void __launch_bounds__(kBnThreads) k_bn_partials(
    int64_t rows, int32_t c, int groups, int lanes, int64_t rows_per_block,
    const T* __restrict__ x, const T* __restrict__ dy, const T* __restrict__ relu_out,
    const float* __restrict__ mu, const float* __restrict__ istd, float* __restrict__ partials) {
  __shared__ float red[kBnThreads * 8 * 2];
  const int tid = threadIdx.x;
  const int g = tid % groups;
  const int lane = tid / groups;
  const int c0 = (blockIdx.y * groups + g) * V;
  const bool active = lane < lanes && c0 < c;
  float s1[V], s2[V], m[V], is[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    s1[j] = 0.f;
    s2[j] = 0.f;
    if (MODE == 1 && active) {
      m[j] = mu[c0 + j];
      is[j] = istd[c0 + j];
    }
  }
  const int64_t r0 = blockIdx.x * rows_per_block;
  int64_t r1 = r0 + rows_per_block;
  if (r1 > rows) r1 = rows;
  if (active) {
    for (int64_t r = r0 + lane; r < r1; r += lanes) {
      float xv[V];
      VecLoad<T, V>::load(x + r * c + c0, xv);
      if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          s1[j] += xv[j];
          s2[j] = fmaf(xv[j], xv[j], s2[j]);
        }
      } else {
        float gv[V];
        VecLoad<T, V>::load(dy + r * c + c0, gv);
        if (relu_out) {
          float zv[V];
          VecLoad<T, V>::load(relu_out + r * c + c0, zv);
#pragma unroll
          for (int j = 0; j < V; ++j) gv[j] = __fmul_rn(gv[j], zv[j] > 0.f ? 1.f : 0.f);
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
          float xh = __fmul_rn(__fsub_rn(xv[j], m[j]), is[j]);
          s1[j] += gv[j];
          s2[j] += __fmul_rn(gv[j], xh);
        }
      }
    }
  }
  // block reduction over lanes in fixed order
  const int width = groups * V;
  if (lane < lanes) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      red[(lane * width + g * V + j) * 2 + 0] = s1[j];
      red[(lane * width + g * V + j) * 2 + 1] = s2[j];
    }
  }
  __syncthreads();
  for (int col = tid; col < width; col += kBnThreads) {
    int ch = blockIdx.y * groups * V + col;
    if (ch >= c) continue;
    float a = 0.f, b = 0.f;
    for (int l = 0; l < lanes; ++l) {
      a += red[(l * width + col) * 2 + 0];
      b += red[(l * width + col) * 2 + 1];
    }
    float* out = partials + (int64_t)blockIdx.x * 2 * c;
    out[ch] = a;
    out[c + ch] = b;
  }
}

// Fixed-order f64 reduction of partial rows [R][2][C]: block = 32 channel
// columns x 32 row lanes.
__device__ __forceinline__ void reduce_partials(const float* __restrict__ partials, int32_t R,
                                                int32_t c, int ch, double& a, double& b) {
  __shared__ double sa[32][33], sb[32][33];
  const int col = threadIdx.x & 31, lane = threadIdx.x >> 5;
  double x = 0.0, y = 0.0;
  if (ch < c) {
    for (int r = lane; r < R; r += 32) {
      x += (double)partials[(int64_t)r * 2 * c + ch];
      y += (double)partials[(int64_t)r * 2 * c + c + ch];
    }
  }
  sa[lane][col] = x;
  sb[lane][col] = y;
  __syncthreads();
  a = 0.0;
  b = 0.0;
  if (lane == 0) {
    for (int l = 0; l < 32; ++l) {
      a += sa[l][col];
      b += sb[l][col];
    }
  }
}

// forward: mean, biased var (functions.py:401-409), istd (:412)
__global__ void __launch_bounds__(1024) k_bn_finalize_fwd(
    const float* __restrict__ partials, int32_t R, int32_t c, int64_t count,
    float* __restrict__ running_mean, float* __restrict__ running_var, float eps, float momentum,
    float* __restrict__ save_mean, float* __restrict__ save_istd) {
  const int ch = blockIdx.x * 32 + (threadIdx.x & 31);
  double s1, s2;
  reduce_partials(partials, R, c, ch, s1, s2);
  if ((threadIdx.x >> 5) == 0 && ch < c) {
    double mean = s1 / (double)count;
    double var = s2 / (double)count - mean * mean;
    if (var < 0.0) var = 0.0;
    float mu = (float)mean, vb = (float)var;
    // m*mean + (1-m)*mu with m = f32(momentum), 1-m in f32 (functions.py:404-409)
    float m = momentum, one_m = __fsub_rn(1.0f, momentum);
    running_mean[ch] = __fadd_rn(__fmul_rn(m, running_mean[ch]), __fmul_rn(one_m, mu));
    running_var[ch] = __fadd_rn(__fmul_rn(m, running_var[ch]), __fmul_rn(one_m, vb));
    save_mean[ch] = mu;
    save_istd[ch] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(vb, eps)));
  }
}

__global__ void k_bn_eval_stats(int32_t c, const float* __restrict__ mean,
                                const float* __restrict__ var, float eps,
                                float* __restrict__ save_mean, float* __restrict__ save_istd) {
  int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch < c) {
    save_mean[ch] = mean[ch];
    save_istd[ch] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var[ch], eps)));
  }
}

// backward: gbeta = sum gy, ggamma = sum gy*xhat (functions.py:421-422)
__global__ void __launch_bounds__(1024) k_bn_finalize_bwd(
    const float* __restrict__ partials, int32_t R, int32_t c, float* __restrict__ gsum,
    float* __restrict__ dgamma, int acc_g, float* __restrict__ dbeta, int acc_b,
    int32_t* __restrict__ nonfinite) {
  const int ch = blockIdx.x * 32 + (threadIdx.x & 31);
  double s1, s2;
  reduce_partials(partials, R, c, ch, s1, s2);
  if ((threadIdx.x >> 5) == 0 && ch < c) {
    float gbeta = (float)s1, ggamma = (float)s2;
    gsum[ch] = gbeta;
    gsum[c + ch] = ggamma;
    int bad = 0;
    if (dgamma) {
      float v = acc_g ? __fadd_rn(dgamma[ch], ggamma) : ggamma;
      dgamma[ch] = v;
      bad |= !isfinite(v);
    }
    if (dbeta) {
      float v = acc_b ? __fadd_rn(dbeta[ch], gbeta) : gbeta;
      dbeta[ch] = v;
      bad |= !isfinite(v);
    }
    if (bad && nonfinite) atomicOr(nonfinite, 1);
  }
}

// y = q(gamma * ((x - mu) * istd) + beta), then ReLU on the stored value
template <typename T, int V>
__global__ void k_bn_fwd_apply(int64_t rows, int32_t c, const T* __restrict__ x,
                               const float* __restrict__ gamma, const float* __restrict__ beta,
                               const float* __restrict__ mu, const float* __restrict__ istd,
                               T* __restrict__ y, int fuse_relu) {
  const int64_t nvec = rows * c / V;
  const int cv = c / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % cv) * V;
    float xv[V];
    VecLoad<T, V>::load(x + i * V, xv);
    T out[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      float xh = __fmul_rn(__fsub_rn(xv[j], mu[c0 + j]), istd[c0 + j]);
      float v = __fadd_rn(__fmul_rn(gamma[c0 + j], xh), beta[c0 + j]);
      T q = Elem<T>::st(v);
      if (fuse_relu) {
        float f = Elem<T>::ld(q);
        q = Elem<T>::st((f > 0.f || f != f) ? f : 0.f);
      }
      out[j] = q;
    }
    if (V == 8 && sizeof(T) == 2) {
      *reinterpret_cast<uint4*>(y + i * V) = *reinterpret_cast<uint4*>(out);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) y[i * V + j] = out[j];
    }
  }
}

// gx = (g/n) * (n*gy - gbeta - xhat*ggamma), g = gamma*istd (functions.py:424-432)
// eval mode: gx = g * gy (functions.py:433-434)
template <typename T, int V>
__global__ void k_bn_bwd_apply(int64_t rows, int32_t c, const T* __restrict__ x,
                               const T* __restrict__ dy, const T* __restrict__ relu_out,
                               const float* __restrict__ gamma, const float* __restrict__ mu,
                               const float* __restrict__ istd, const float* __restrict__ gsum,
                               int batch_stat, T* __restrict__ dx, int acc) {
  const int64_t nvec = rows * c / V;
  const int cv = c / V;
  const float fn = (float)rows;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % cv) * V;
    float xv[V], gv[V], pv[V];
    VecLoad<T, V>::load(x + i * V, xv);
    VecLoad<T, V>::load(dy + i * V, gv);
    if (relu_out) {
      float zv[V];
      VecLoad<T, V>::load(relu_out + i * V, zv);
#pragma unroll
      for (int j = 0; j < V; ++j) gv[j] = __fmul_rn(gv[j], zv[j] > 0.f ? 1.f : 0.f);
    }
    if (acc) VecLoad<T, V>::load(dx + i * V, pv);
    T out[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int ch = c0 + j;
      float g = __fmul_rn(gamma[ch], istd[ch]);
      float r;
      if (batch_stat) {
        float xh = __fmul_rn(__fsub_rn(xv[j], mu[ch]), istd[ch]);
        float t = __fsub_rn(__fmul_rn(fn, gv[j]), gsum[ch]);
        t = __fsub_rn(t, __fmul_rn(xh, gsum[c + ch]));
        r = __fmul_rn(__fdiv_rn(g, fn), t);
      } else {
        r = __fmul_rn(g, gv[j]);
      }
      out[j] = Elem<T>::st(__fadd_rn(acc ? pv[j] : 0.f, r));
    }
    if (V == 8 && sizeof(T) == 2) {
      *reinterpret_cast<uint4*>(dx + i * V) = *reinterpret_cast<uint4*>(out);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) dx[i * V + j] = out[j];
    }
  }
}

static int64_t bn_blocks_x(int64_t rows, const BnGeom& g) {
  // ~4 blocks per SM in total, at least 8 rows per lane
  int64_t want = (148 * 4 + g.slabs - 1) / g.slabs;
  int64_t min_rows = (int64_t)g.lanes * 8;
  int64_t by_rows = (rows + min_rows - 1) / min_rows;
  if (want > by_rows) want = by_rows;
  if (want < 1) want = 1;
  return want;
}

struct BnWs {
  float* partials;
  float* gsum;
  int64_t bx;
};

static size_t bn_ws_bytes(int64_t rows, int32_t c) {
  BnGeom g = bn_geom(c, true);
  int64_t bx = bn_blocks_x(rows, g);
  BnGeom g1 = bn_geom(c, false);
  int64_t bx1 = bn_blocks_x(rows, g1);
  if (bx1 > bx) bx = bx1;
  return (size_t)(bx * 2 * c + 2 * c) * sizeof(float) + 256;
}

template <typename T, int MODE>
static int launch_partials(int64_t rows, int32_t c, const BnGeom& g, int64_t bx, const T* x,
                           const T* dy, const T* relu, const float* mu, const float* istd,
                           float* partials, cudaStream_t st) {
  int64_t rpb = (rows + bx - 1) / bx;
  dim3 grid((unsigned)bx, (unsigned)g.slabs);
  if (g.vec == 8)
    k_bn_partials<T, 8, MODE><<<grid, kBnThreads, 0, st>>>(rows, c, g.groups, g.lanes, rpb, x, dy,
                                                           relu, mu, istd, partials);
  else
    k_bn_partials<T, 1, MODE><<<grid, kBnThreads, 0, st>>>(rows, c, g.groups, g.lanes, rpb, x, dy,
                                                           relu, mu, istd, partials);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

static bool al16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace nnl

using namespace nnl;

extern "C" {

size_t nnl_bn_workspace_size(int64_t rows, int32_t c) { return bn_ws_bytes(rows, c); }

int nnl_bn_fwd_train(int dtype, int64_t rows, int32_t c, const void* x, const float* gamma,
                     const float* beta, float* running_mean, float* running_var, float eps,
                     float momentum, const float* stat_partials, int32_t n_partials,
                     float* save_mean, float* save_istd, void* y, int fuse_relu, void* ws,
                     size_t ws_bytes, void* stream) {
  if (rows <= 1) return fail(NNL_ERR_DEGENERATE_BATCH, "cannot take batch statistics over %lld element(s)", (long long)rows);
  cudaStream_t st = as_stream(stream);
  bool vec = al16(x) && al16(y);
  BnGeom g = bn_geom(c, vec);
  const float* parts = stat_partials;
  int32_t R = n_partials;
  if (!parts) {
    if (ws_bytes < bn_ws_bytes(rows, c)) return fail(NNL_ERR_INVALID_ARGUMENT, "bn workspace too small");
    int64_t bx = bn_blocks_x(rows, g);
    float* p = (float*)ws;
    int rc;
    NNL_DISPATCH_DTYPE(dtype, T, {
      rc = launch_partials<T, 0>(rows, c, g, bx, (const T*)x, nullptr, nullptr, nullptr, nullptr,
                                 p, st);
    });
    if (rc) return rc;
    parts = p;
    R = (int32_t)bx;
  }
  k_bn_finalize_fwd<<<(c + 31) / 32, 1024, 0, st>>>(parts, R, c, rows, running_mean, running_var,
                                                   eps, momentum, save_mean, save_istd);
  NNL_CHECK_LAUNCH();
  int64_t nvec = rows * c / g.vec;
  NNL_DISPATCH_DTYPE(dtype, T, {
    if (g.vec == 8)
      k_bn_fwd_apply<T, 8><<<grid_for(nvec, 256, 148 * 32), 256, 0, st>>>(
          rows, c, (const T*)x, gamma, beta, save_mean, save_istd, (T*)y, fuse_relu);
    else
      k_bn_fwd_apply<T, 1><<<grid_for(nvec, 256, 148 * 32), 256, 0, st>>>(
          rows, c, (const T*)x, gamma, beta, save_mean, save_istd, (T*)y, fuse_relu);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_bn_fwd_eval(int dtype, int64_t rows, int32_t c, const void* x, const float* gamma,
                    const float* beta, const float* mean, const float* var, float eps,
                    float* save_mean, float* save_istd, void* y, int fuse_relu, void* stream) {
  cudaStream_t st = as_stream(stream);
  k_bn_eval_stats<<<(c + 255) / 256, 256, 0, st>>>(c, mean, var, eps, save_mean, save_istd);
  NNL_CHECK_LAUNCH();
  if (rows * c <= 0) return NNL_OK;
  bool vec = al16(x) && al16(y) && c % 8 == 0;
  int V = vec ? 8 : 1;
  int64_t nvec = rows * c / V;
  NNL_DISPATCH_DTYPE(dtype, T, {
    if (V == 8)
      k_bn_fwd_apply<T, 8><<<grid_for(nvec, 256, 148 * 32), 256, 0, st>>>(
          rows, c, (const T*)x, gamma, beta, save_mean, save_istd, (T*)y, fuse_relu);
    else
      k_bn_fwd_apply<T, 1><<<grid_for(nvec, 256, 148 * 32), 256, 0, st>>>(
          rows, c, (const T*)x, gamma, beta, save_mean, save_istd, (T*)y, fuse_relu);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_bn_bwd(int dtype, int64_t rows, int32_t c, const void* x, const void* dy,
               const void* relu_out, const float* gamma, const float* save_mean,
               const float* save_istd, int batch_stat, void* dx, int acc_x, float* dgamma,
               int acc_g, float* dbeta, int acc_b, int32_t* nonfinite, void* ws, size_t ws_bytes,
               void* stream) {
  cudaStream_t st = as_stream(stream);
  if (ws_bytes < bn_ws_bytes(rows, c)) return fail(NNL_ERR_INVALID_ARGUMENT, "bn workspace too small");
  bool vec = al16(x) && al16(dy) && al16(relu_out) && al16(dx);
  BnGeom g = bn_geom(c, vec);
  int64_t bx = bn_blocks_x(rows, g);
  float* parts = (float*)ws;
  float* gsum = parts + bx * 2 * c;
  int rc;
  NNL_DISPATCH_DTYPE(dtype, T, {
    rc = launch_partials<T, 1>(rows, c, g, bx, (const T*)x, (const T*)dy, (const T*)relu_out,
                               save_mean, save_istd, parts, st);
  });
  if (rc) return rc;
  k_bn_finalize_bwd<<<(c + 31) / 32, 1024, 0, st>>>(parts, (int32_t)bx, c, gsum, dgamma, acc_g,
                                                   dbeta, acc_b, nonfinite);
  NNL_CHECK_LAUNCH();
  if (!dx) return NNL_OK;
  int64_t nvec = rows * c / g.vec;
  NNL_DISPATCH_DTYPE(dtype, T, {
    if (g.vec == 8)
      k_bn_bwd_apply<T, 8><<<grid_for(nvec, 256, 148 * 32), 256, 0, st>>>(
          rows, c, (const T*)x, (const T*)dy, (const T*)relu_out, gamma, save_mean, save_istd,
          gsum, batch_stat, (T*)dx, acc_x);
    else
      k_bn_bwd_apply<T, 1><<<grid_for(nvec, 256, 148 * 32), 256, 0, st>>>(
          rows, c, (const T*)x, (const T*)dy, (const T*)relu_out, gamma, save_mean, save_istd,
          gsum, batch_stat, (T*)dx, acc_x);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

}  // extern "C"
