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
#include "bn_stream.cuh"
#include "common.cuh"

namespace nnl {

constexpr int kBnThreads = 256;
constexpr int kUnroll = 4;  // rows loaded per thread before use (memory-level parallelism)

struct BnGeom {
  int vec;        // channels per thread (8 or 1)
  int groups;     // channel groups per row in one slab
  int lanes;      // rows processed concurrently by a block
  int slabs;      // grid.y
};

// vmax 8 for the forward kernels; 4 for the backward ones, whose per-channel
// state (9 constants + 2 loaded rows x unroll) would otherwise need ~180
// registers and drop the SM to one 256-thread block.
static BnGeom bn_geom(int32_t c, bool vec_ok, int vmax = 8) {
  BnGeom g;
  g.vec = (vec_ok && c % vmax == 0) ? vmax : 1;
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
struct VecLoad<__half, 4> {
  static __device__ __forceinline__ void load(const __half* p, float* out) {
    uint2 u = *reinterpret_cast<const uint2*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
    float2 a = __half22float2(h[0]), b = __half22float2(h[1]);
    out[0] = a.x; out[1] = a.y; out[2] = b.x; out[3] = b.y;
  }
};
template <>
struct VecLoad<float, 4> {
  static __device__ __forceinline__ void load(const float* p, float* out) {
    float4 a = *reinterpret_cast<const float4*>(p);
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
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

// The fused BN->ReLU gate (z > 0) is recomputed from x with the forward's
// exact op sequence, z = relu(q(gamma*((x-mu)*istd) + beta)), so backward
// never reads the ReLU output (2 B/element saved in each pass).
template <typename T>
__device__ __forceinline__ float relu_gate(float xh, float ga, float be) {
  return Elem<T>::ld(Elem<T>::st(__fadd_rn(__fmul_rn(ga, xh), be))) > 0.f ? 1.f : 0.f;
}

// MODE 0: (sum x-K, sum (x-K)^2), K = shift or x[0]     -- forward statistics
// MODE 1: (sum gy, sum gy*xhat), gy gated by the ReLU    -- backward reductions
template <typename T, int V, int MODE>
__global__ void __launch_bounds__(kBnThreads) k_bn_partials(
    int64_t rows, int32_t c, int groups, int lanes, int64_t rows_per_block,
    const T* __restrict__ x, const T* __restrict__ dy, int relu, const T* __restrict__ gate,
    const float* __restrict__ gamma, const float* __restrict__ beta,
    const float* __restrict__ mu, const float* __restrict__ istd, float* __restrict__ partials,
    const float* __restrict__ shift) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[kBnThreads * 8 * 2];
  const int tid = threadIdx.x;
  const int g = tid % groups;
  const int lane = tid / groups;
  const int c0 = (blockIdx.y * groups + g) * V;
  const bool active = lane < lanes && c0 < c;
  float s1[V], s2[V], m[V], is[V], ga[V], be[V], kc[V];
  if (MODE == 0 && active) {
    if (shift) {
#pragma unroll
      for (int j = 0; j < V; ++j) kc[j] = shift[c0 + j];
    } else {
      VecLoad<T, V>::load(x + c0, kc);  // centre on the first row
    }
  }
#pragma unroll
  for (int j = 0; j < V; ++j) {
    s1[j] = 0.f;
    s2[j] = 0.f;
    if (MODE == 1 && active) {
      m[j] = mu[c0 + j];
      is[j] = istd[c0 + j];
      ga[j] = relu ? gamma[c0 + j] : 0.f;
      be[j] = relu ? beta[c0 + j] : 0.f;
    }
  }
  const int64_t r0 = blockIdx.x * rows_per_block;
  int64_t r1 = r0 + rows_per_block;
  if (r1 > rows) r1 = rows;
  if (active) {
    for (int64_t rb = r0 + lane; rb < r1; rb += (int64_t)lanes * kUnroll) {
      float xv[kUnroll][V], gv[kUnroll][V];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t r = rb + (int64_t)u * lanes;
        if (r < r1) {
          VecLoad<T, V>::load(x + r * c + c0, xv[u]);
          if (MODE == 1) VecLoad<T, V>::load(dy + r * c + c0, gv[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t r = rb + (int64_t)u * lanes;
        if (r >= r1) break;
        if (MODE == 0) {
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const float d = __fsub_rn(xv[u][j], kc[j]);
            s1[j] += d;
            s2[j] = fmaf(d, d, s2[j]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const float xh = __fmul_rn(__fsub_rn(xv[u][j], m[j]), is[j]);
            float gy = relu ? __fmul_rn(gv[u][j], relu_gate<T>(xh, ga[j], be[j])) : gv[u][j];
            if (gate) gy = __fmul_rn(gy, Elem<T>::load(gate + r * c + c0 + j) > 0.f ? 1.f : 0.f);
            s1[j] += gy;
            s2[j] += __fmul_rn(gy, xh);
          }
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

// Fixed-order f64 reduction of partial rows [R][2][C]: block = 8 channel
// columns x 128 row lanes (1024 threads), so even C = 64 gets 8 blocks and
// each lane sums only R/128 rows.  Column index: blockIdx.x*8 + (tid & 7).
constexpr int kRedCols = 8, kRedLanes = 128;
__device__ __forceinline__ int red_channel() { return blockIdx.x * kRedCols + (threadIdx.x & 7); }
__device__ __forceinline__ bool red_leader() { return (threadIdx.x >> 3) == 0; }

__device__ __forceinline__ void reduce_partials(const float* __restrict__ partials, int32_t R,
                                                int32_t c, int ch, double& a, double& b) {
  // fixed order: row lanes -> the 4 lanes of a column inside a warp (xor 8, 16)
  // -> the 32 warps, serially (was 128 serial steps)
  __shared__ double sa[kRedLanes / 4][kRedCols + 1], sb[kRedLanes / 4][kRedCols + 1];
  const int col = threadIdx.x & 7, lane = threadIdx.x >> 3;
  double x = 0.0, y = 0.0;
  if (ch < c) {
    for (int r = lane; r < R; r += kRedLanes) {
      x += (double)partials[(int64_t)r * 2 * c + ch];
      y += (double)partials[(int64_t)r * 2 * c + c + ch];
    }
  }
  x += __shfl_xor_sync(0xffffffffu, x, 8);
  y += __shfl_xor_sync(0xffffffffu, y, 8);
  x += __shfl_xor_sync(0xffffffffu, x, 16);
  y += __shfl_xor_sync(0xffffffffu, y, 16);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) < 8) {
    sa[w][col] = x;
    sb[w][col] = y;
  }
  __syncthreads();
  a = 0.0;
  b = 0.0;
  if (lane == 0) {
    for (int l = 0; l < kRedLanes / 4; ++l) {
      a += sa[l][col];
      b += sb[l][col];
    }
  }
}

// forward: mean, biased var (functions.py:401-409), istd (:412).  The partials
// are sums of x-K and (x-K)^2 about a per-channel centre K (the caller's shift,
// else the first row of x), so mean = K + s1/n and var = s2/n - (s1/n)^2 keep
// their precision when |mean| >> std (the reference's np.var is two-pass).
// With `shift_out` the batch mean is stored there: the centre of the next call.
__global__ void __launch_bounds__(1024) k_bn_finalize_fwd(
    const float* __restrict__ partials, int32_t R, int32_t c, int64_t count,
    float* __restrict__ running_mean, float* __restrict__ running_var, float eps, float momentum,
    float* __restrict__ save_mean, float* __restrict__ save_istd, const float* shift_in,
    const void* x_row0, int x_f16, float* shift_out) {
  pdl_wait();
  pdl_trigger();
  const int ch = red_channel();
  double s1, s2;
  reduce_partials(partials, R, c, ch, s1, s2);
  if (red_leader() && ch < c) {
    double k = 0.0;
    if (shift_in) k = shift_in[ch];
    else if (x_row0) k = x_f16 ? (double)__half2float(((const __half*)x_row0)[ch])
                               : (double)((const float*)x_row0)[ch];
    const double d = s1 / (double)count;
    const double mean = k + d;
    double var = s2 / (double)count - d * d;
    if (var < 0.0) var = 0.0;
    if (shift_out) shift_out[ch] = (float)mean;
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
  const int ch = red_channel();
  double s1, s2;
  reduce_partials(partials, R, c, ch, s1, s2);
  if (red_leader() && ch < c) {
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

template <typename T, int V>
struct VecStore;
template <typename T>
struct VecStore<T, 1> {
  static __device__ __forceinline__ void store(T* p, const T* v) { p[0] = v[0]; }
};
template <>
struct VecStore<__half, 8> {
  static __device__ __forceinline__ void store(__half* p, const __half* v) {
    *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(v);
  }
};
template <>
struct VecStore<__half, 4> {
  static __device__ __forceinline__ void store(__half* p, const __half* v) {
    *reinterpret_cast<uint2*>(p) = *reinterpret_cast<const uint2*>(v);
  }
};
template <>
struct VecStore<float, 4> {
  static __device__ __forceinline__ void store(float* p, const float* v) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <>
struct VecStore<float, 8> {
  static __device__ __forceinline__ void store(float* p, const float* v) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

// Apply kernels use the same (row chunk x channel slab) decomposition as the
// reductions: each thread owns V channels for the whole launch, so the
// per-channel constants live in registers and the inner loop has no index
// division (the first version's int64 `i % C` per element cost 5x).

// y = q(gamma * ((x - mu) * istd) + beta), then ReLU on the stored value
template <typename T, int V>
__global__ void __launch_bounds__(kBnThreads) k_bn_fwd_apply(
    int64_t rows, int32_t c, int groups, int lanes, int64_t rows_per_block,
    const T* __restrict__ x, const float* __restrict__ gamma, const float* __restrict__ beta,
    const float* __restrict__ mu, const float* __restrict__ istd, T* __restrict__ y,
    int fuse_relu) {
  pdl_wait();
  pdl_trigger();
  const int g = threadIdx.x % groups, lane = threadIdx.x / groups;
  const int c0 = (blockIdx.y * groups + g) * V;
  if (lane >= lanes || c0 >= c) return;
  float m[V], is[V], ga[V], be[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    m[j] = mu[c0 + j];
    is[j] = istd[c0 + j];
    ga[j] = gamma[c0 + j];
    be[j] = beta[c0 + j];
  }
  const int64_t r0 = blockIdx.x * rows_per_block;
  const int64_t r1 = min(r0 + rows_per_block, rows);
  for (int64_t rb = r0 + lane; rb < r1; rb += (int64_t)lanes * kUnroll) {
    float xv[kUnroll][V];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t r = rb + (int64_t)u * lanes;
      if (r < r1) VecLoad<T, V>::load(x + r * c + c0, xv[u]);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t r = rb + (int64_t)u * lanes;
      if (r >= r1) break;
      __align__(16) T out[V];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float xh = __fmul_rn(__fsub_rn(xv[u][j], m[j]), is[j]);
        T q = Elem<T>::st(__fadd_rn(__fmul_rn(ga[j], xh), be[j]));
        if (fuse_relu) {
          const float f = Elem<T>::ld(q);
          q = Elem<T>::st((f > 0.f || f != f) ? f : 0.f);
        }
        out[j] = q;
      }
      VecStore<T, V>::store(y + r * c + c0, out);
    }
  }
}

// gx = (g/n) * (n*gy - gbeta - xhat*ggamma), g = gamma*istd (functions.py:424-432)
// eval mode: gx = g * gy (functions.py:433-434).  With `bias_part` the block
// also emits column sums of the ROUNDED gx: the gradient of the producing
// convolution's bias (functions.py:211-212), saving a separate pass.
template <typename T, int V>
__global__ void __launch_bounds__(kBnThreads) k_bn_bwd_apply(
    int64_t rows, int32_t c, int groups, int lanes, int64_t rows_per_block,
    const T* __restrict__ x, const T* __restrict__ dy, int relu, const T* __restrict__ gate,
    const float* __restrict__ gamma, const float* __restrict__ beta, const float* __restrict__ mu,
    const float* __restrict__ istd, const float* __restrict__ gsum, int batch_stat,
    T* __restrict__ dx, int acc, float* __restrict__ bias_part) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[kBnThreads * 8];
  const int g = threadIdx.x % groups, lane = threadIdx.x / groups;
  const int c0 = (blockIdx.y * groups + g) * V;
  const bool active = lane < lanes && c0 < c;
  const float fn = (float)rows;
  float m[V], is[V], gg[V], gn[V], gb[V], gy2[V], cs[V], ga[V], be[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    cs[j] = 0.f;
    if (active) {
      m[j] = mu[c0 + j];
      is[j] = istd[c0 + j];
      ga[j] = gamma[c0 + j];
      be[j] = relu ? beta[c0 + j] : 0.f;
      gg[j] = __fmul_rn(ga[j], is[j]);           // g = gamma * istd
      gn[j] = __fdiv_rn(gg[j], fn);              // g / n
      gb[j] = gsum[c0 + j];                      // gbeta
      gy2[j] = gsum[c + c0 + j];                 // ggamma
    }
  }
  if (active) {
    const int64_t r0 = blockIdx.x * rows_per_block;
    const int64_t r1 = min(r0 + rows_per_block, rows);
    for (int64_t rb = r0 + lane; rb < r1; rb += (int64_t)lanes * kUnroll) {
      float xv[kUnroll][V], gv[kUnroll][V];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t r = rb + (int64_t)u * lanes;
        if (r < r1) {
          VecLoad<T, V>::load(dy + r * c + c0, gv[u]);
          if (batch_stat || relu) VecLoad<T, V>::load(x + r * c + c0, xv[u]);
        }
      }
      if (relu) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const float xh = __fmul_rn(__fsub_rn(xv[u][j], m[j]), is[j]);
            gv[u][j] = __fmul_rn(gv[u][j], relu_gate<T>(xh, ga[j], be[j]));
          }
      }
      if (gate) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int64_t r = rb + (int64_t)u * lanes;
          if (r >= r1) break;
#pragma unroll
          for (int j = 0; j < V; ++j)
            gv[u][j] = __fmul_rn(gv[u][j],
                                 Elem<T>::load(gate + r * c + c0 + j) > 0.f ? 1.f : 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t r = rb + (int64_t)u * lanes;
        if (r >= r1) break;
        float pv[V];
        if (acc) VecLoad<T, V>::load(dx + r * c + c0, pv);
        __align__(16) T out[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
          float res;
          if (batch_stat) {
            const float xh = __fmul_rn(__fsub_rn(xv[u][j], m[j]), is[j]);
            float t = __fsub_rn(__fmul_rn(fn, gv[u][j]), gb[j]);
            t = __fsub_rn(t, __fmul_rn(xh, gy2[j]));
            res = __fmul_rn(gn[j], t);
          } else {
            res = __fmul_rn(gg[j], gv[u][j]);
          }
          out[j] = Elem<T>::st(__fadd_rn(acc ? pv[j] : 0.f, res));
          cs[j] += Elem<T>::ld(out[j]);
        }
        VecStore<T, V>::store(dx + r * c + c0, out);
      }
    }
  }
  if (!bias_part) return;
  const int width = groups * V;
  if (lane < lanes) {
#pragma unroll
    for (int j = 0; j < V; ++j) red[lane * width + g * V + j] = cs[j];
  }
  __syncthreads();
  for (int col = threadIdx.x; col < width; col += kBnThreads) {
    const int ch = blockIdx.y * groups * V + col;
    if (ch >= c) continue;
    float a = 0.f;
    for (int l = 0; l < lanes; ++l) a += red[l * width + col];
    float* out = bias_part + (int64_t)blockIdx.x * 2 * c;
    out[ch] = a;
    out[c + ch] = 0.f;
  }
}

// db = q(prev + sum of bias partials) (fixed-order f64 reduction)
template <typename T>
__global__ void __launch_bounds__(1024) k_bn_bias_finalize(const float* __restrict__ partials,
                                                           int32_t R, int32_t c, T* __restrict__ db,
                                                           int acc, int32_t* __restrict__ nonfinite) {
  pdl_wait();
  pdl_trigger();
  const int ch = red_channel();
  double s1, s2;
  reduce_partials(partials, R, c, ch, s1, s2);
  if (red_leader() && ch < c) {
    write_out(db + ch, (float)s1, acc != 0);
    if (nonfinite && !isfinite(Elem<T>::load(db + ch))) atomicOr(nonfinite, 1);
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
  int64_t bx = 1;
  for (int v : {8, 4, 1}) {
    const int64_t b = bn_blocks_x(rows, bn_geom(c, v > 1, v));
    if (b > bx) bx = b;
  }
  if (c % 8 == 0 && c <= 2048)
    for (int nt : {1, 2, 3}) {
      const int64_t b = bn_stream_rows(BNS_STATS_B, nt, rows, c);
      if (b > bx) bx = b;
    }
  return (size_t)(2 * bx * 2 * c + 2 * c) * sizeof(float) + 256;
}

template <typename T, int MODE>
static int launch_partials(int64_t rows, int32_t c, const BnGeom& g, int64_t bx, const T* x,
                           const T* dy, int relu, const T* gate, const float* gamma,
                           const float* beta,
                           const float* mu, const float* istd, float* partials, cudaStream_t st,
                           const float* shift = nullptr) {
  int64_t rpb = (rows + bx - 1) / bx;
  dim3 grid((unsigned)bx, (unsigned)g.slabs);
  if (g.vec == 8)
    launch_k(k_bn_partials<T, 8, MODE>, grid, kBnThreads, 0, st, rows, c, g.groups, g.lanes, rpb, x, dy,
                                                           relu, gate, gamma, beta, mu, istd, partials,
                                                           shift);
  else if (g.vec == 4)
    launch_k(k_bn_partials<T, 4, MODE>, grid, kBnThreads, 0, st, rows, c, g.groups, g.lanes, rpb, x, dy,
                                                           relu, gate, gamma, beta, mu, istd, partials,
                                                           shift);
  else
    launch_k(k_bn_partials<T, 1, MODE>, grid, kBnThreads, 0, st, rows, c, g.groups, g.lanes, rpb, x, dy,
                                                           relu, gate, gamma, beta, mu, istd, partials,
                                                           shift);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

static bool al16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace nnl

using namespace nnl;

extern "C" {

size_t nnl_bn_workspace_size(int64_t rows, int32_t c) { return bn_ws_bytes(rows, c); }

}  // extern "C"

template <typename T>
static int launch_fwd_apply(int64_t rows, int32_t c, const BnGeom& g, const T* x,
                            const float* gamma, const float* beta, const float* mu,
                            const float* istd, T* y, int fuse_relu, cudaStream_t st) {
  int64_t bx = bn_blocks_x(rows, g);
  int64_t rpb = (rows + bx - 1) / bx;
  dim3 grid((unsigned)bx, (unsigned)g.slabs);
  if (g.vec == 8)
    launch_k(k_bn_fwd_apply<T, 8>, grid, kBnThreads, 0, st, rows, c, g.groups, g.lanes, rpb, x, gamma,
                                                      beta, mu, istd, y, fuse_relu);
  else
    launch_k(k_bn_fwd_apply<T, 1>, grid, kBnThreads, 0, st, rows, c, g.groups, g.lanes, rpb, x, gamma,
                                                      beta, mu, istd, y, fuse_relu);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

static bool use_stream(int dtype, int64_t rows, int32_t c, const void* a, const void* b,
                       const void* d) {
  return dtype == NNL_F16 && bn_stream_ok(rows, c, a, b, d);
}

extern "C" {

int nnl_relu_bwd(int dtype, int64_t n, const void* x, const void* dy, void* dx, int accumulate,
                 void* stream);
int nnl_add2_fwd(int dtype, int64_t n, const void* a, const void* b, void* y, int fuse_relu,
                 void* stream);

// y = q(gamma*((x-mu)*istd)+beta); with `residual` the Add2 of the residual
// tail follows, y = q(y + residual) (Add2 forward), then the optional ReLU.
static int bn_apply_fwd(int dtype, int64_t rows, int32_t c, const void* x, const float* gamma,
                        const float* beta, const float* save_mean, const float* save_istd,
                        void* y, const void* residual, int fuse_relu, cudaStream_t st) {
  if (use_stream(dtype, rows, c, x, y, residual)) {
    BnStreamArgs a = {};
    a.rows = rows; a.c = c; a.x = (const __half*)x; a.out = (__half*)y; a.gamma = gamma;
    a.beta = beta; a.mu = save_mean; a.istd = save_istd; a.relu = fuse_relu;
    a.res = (const __half*)residual;
    a.reverse = 1;
    return bn_stream_launch(BNS_APPLY_F, a, st);
  }
  BnGeom g = bn_geom(c, al16(x) && al16(y));
  int rc = NNL_OK;
  NNL_DISPATCH_DTYPE(dtype, T, {
    rc = launch_fwd_apply<T>(rows, c, g, (const T*)x, gamma, beta, save_mean, save_istd, (T*)y,
                             residual ? 0 : fuse_relu, st);
  });
  if (rc || !residual) return rc;
  return nnl_add2_fwd(dtype, rows * c, y, residual, y, fuse_relu, st);  // in place, elementwise
}

int nnl_bn_fwd_train(int dtype, int64_t rows, int32_t c, const void* x, const float* gamma,
                     const float* beta, float* running_mean, float* running_var, float eps,
                     float momentum, const float* stat_partials, int32_t n_partials,
                     float* shift, float* save_mean, float* save_istd, void* y,
                     const void* residual, int fuse_relu, void* ws, size_t ws_bytes,
                     void* stream) {
  if (rows <= 1)
    return fail(NNL_ERR_DEGENERATE_BATCH, "cannot take batch statistics over %lld element(s)",
                (long long)rows);
  cudaStream_t st = as_stream(stream);
  const float* parts = stat_partials;
  int32_t R = n_partials;
  int rc = NNL_OK;
  if (!parts) {
    if (ws_bytes < bn_ws_bytes(rows, c))
      return fail(NNL_ERR_INVALID_ARGUMENT, "bn workspace too small");
    float* p = (float*)ws;
    if (use_stream(dtype, rows, c, x, nullptr, nullptr)) {
      BnStreamArgs a = {};
      a.rows = rows; a.c = c; a.x = (const __half*)x; a.partials = p;  // centre: x[0]
      rc = bn_stream_launch(BNS_STATS_F, a, st);
      R = bn_stream_rows(BNS_STATS_F, 1, rows, c);
    } else {
      BnGeom g = bn_geom(c, al16(x));
      const int64_t bx = bn_blocks_x(rows, g);
      NNL_DISPATCH_DTYPE(dtype, T, {
        rc = launch_partials<T, 0>(rows, c, g, bx, (const T*)x, nullptr, 0, nullptr, nullptr,
                                   nullptr, nullptr, nullptr, p, st);
      });
      R = (int32_t)bx;
    }
    if (rc) return rc;
    parts = p;
  }
  // producer partials are centred on `shift` (the value the convolution was
  // given); the partials pass above centres on x's first row
  launch_k(k_bn_finalize_fwd, (c + kRedCols - 1) / kRedCols, 1024, 0, st, 
      parts, R, c, rows, running_mean, running_var, eps, momentum, save_mean, save_istd,
      stat_partials ? shift : nullptr, stat_partials ? nullptr : x, dtype == NNL_F16, shift);
  NNL_CHECK_LAUNCH();
  if (!y) return NNL_OK;  // statistics only: the consumer applies them
  return bn_apply_fwd(dtype, rows, c, x, gamma, beta, save_mean, save_istd, y, residual,
                      fuse_relu, st);
}

int nnl_bn_fwd_eval(int dtype, int64_t rows, int32_t c, const void* x, const float* gamma,
                    const float* beta, const float* mean, const float* var, float eps,
                    float* save_mean, float* save_istd, void* y, const void* residual,
                    int fuse_relu, void* stream) {
  cudaStream_t st = as_stream(stream);
  launch_k(k_bn_eval_stats, (c + 255) / 256, 256, 0, st, c, mean, var, eps, save_mean, save_istd);
  NNL_CHECK_LAUNCH();
  if (rows * c <= 0) return NNL_OK;
  return bn_apply_fwd(dtype, rows, c, x, gamma, beta, save_mean, save_istd, y, residual,
                      fuse_relu, st);
}

int nnl_bn_bwd(int dtype, int64_t rows, int32_t c, const void* x, const void* dy,
               int fused_relu, const void* gate, void* dres, int acc_res, const float* gamma,
               const float* beta, const float* save_mean, const float* save_istd, int batch_stat,
               void* dx, int acc_x, float* dgamma, int acc_g, float* dbeta, int acc_b,
               void* conv_bias_grad, int acc_cb, int32_t* nonfinite, void* ws, size_t ws_bytes,
               void* stream) {
  cudaStream_t st = as_stream(stream);
  if (ws_bytes < bn_ws_bytes(rows, c))
    return fail(NNL_ERR_INVALID_ARGUMENT, "bn workspace too small");
  if (fused_relu && !beta) return fail(NNL_ERR_INVALID_ARGUMENT, "fused ReLU needs beta");
  if (fused_relu && gate)
    return fail(NNL_ERR_INVALID_ARGUMENT, "fused ReLU and residual gate are exclusive");
  const bool stream_ok =
      use_stream(dtype, rows, c, x, dy, dx) && use_stream(dtype, rows, c, gate, dres, nullptr);
  // the gated gradient is written once to dres and re-read by the apply pass
  const bool dres_first = stream_ok && gate && dres && !acc_res;
  BnGeom g = bn_geom(c, al16(x) && al16(dy) && al16(dx), 4);
  const int nt_stats = gate ? 3 : 2;
  const int64_t bx =
      stream_ok ? bn_stream_rows(BNS_STATS_B, nt_stats, rows, c) : bn_blocks_x(rows, g);
  float* parts = (float*)ws;
  float* gsum = parts + bx * 2 * c;
  float* bparts = gsum + 2 * c;
  int rc = NNL_OK;
  if (stream_ok) {
    BnStreamArgs a = {};
    a.rows = rows; a.c = c; a.x = (const __half*)x; a.dy = (const __half*)dy; a.gamma = gamma;
    a.beta = beta; a.mu = save_mean; a.istd = save_istd; a.relu = fused_relu; a.partials = parts;
    a.gate = (const __half*)gate;
    a.dres = dres_first ? (__half*)dres : nullptr;
    a.reverse = 1;  // dy's producer wrote it first to last; APPLY_B then re-reads
    rc = bn_stream_launch(BNS_STATS_B, a, st);  // from the start, still in L2
  } else {
    NNL_DISPATCH_DTYPE(dtype, T, {
      rc = launch_partials<T, 1>(rows, c, g, bx, (const T*)x, (const T*)dy, fused_relu,
                                 (const T*)gate, gamma, beta, save_mean, save_istd, parts, st);
    });
  }
  if (rc) return rc;
  launch_k(k_bn_finalize_bwd, (c + kRedCols - 1) / kRedCols, 1024, 0, st, 
      parts, (int32_t)bx, c, gsum, dgamma, acc_g, dbeta, acc_b, nonfinite);
  NNL_CHECK_LAUNCH();
  if (dx) {
    float* bp = conv_bias_grad ? bparts : nullptr;
    int32_t brows = (int32_t)bx;
    if (stream_ok) {
      BnStreamArgs a = {};
      a.rows = rows; a.c = c; a.x = (const __half*)x; a.out = (__half*)dx;
      a.gamma = gamma; a.beta = beta; a.mu = save_mean; a.istd = save_istd; a.gsum = gsum;
      a.partials = bp; a.relu = fused_relu; a.acc = acc_x; a.batch_stat = batch_stat;
      if (dres_first) {
        a.dy = (const __half*)dres;  // already gated
      } else {
        a.dy = (const __half*)dy;
        a.gate = (const __half*)gate;
      }
      rc = bn_stream_launch(BNS_APPLY_B, a, st);
      if (rc) return rc;
      brows = bn_stream_rows(BNS_APPLY_B, bn_stream_nt(BNS_APPLY_B, a), rows, c);
    } else {
      const int64_t rpb = (rows + bx - 1) / bx;
      dim3 grid((unsigned)bx, (unsigned)g.slabs);
      NNL_DISPATCH_DTYPE(dtype, T, {
        if (g.vec == 4)
          launch_k(k_bn_bwd_apply<T, 4>, grid, kBnThreads, 0, st, 
              rows, c, g.groups, g.lanes, rpb, (const T*)x, (const T*)dy, fused_relu,
              (const T*)gate, gamma, beta, save_mean, save_istd, gsum, batch_stat, (T*)dx, acc_x,
              bp);
        else
          launch_k(k_bn_bwd_apply<T, 1>, grid, kBnThreads, 0, st, 
              rows, c, g.groups, g.lanes, rpb, (const T*)x, (const T*)dy, fused_relu,
              (const T*)gate, gamma, beta, save_mean, save_istd, gsum, batch_stat, (T*)dx, acc_x,
              bp);
      });
      NNL_CHECK_LAUNCH();
    }
    if (bp) {
      NNL_DISPATCH_DTYPE(dtype, T, {
        launch_k(k_bn_bias_finalize<T>, (c + kRedCols - 1) / kRedCols, 1024, 0, st, 
            bp, brows, c, (T*)conv_bias_grad, acc_cb, nonfinite);
      });
      NNL_CHECK_LAUNCH();
    }
  }
  // the residual branch's gradient (Add2 backward after the ReLU gate)
  if (gate && dres && !dres_first)
    return nnl_relu_bwd(dtype, rows * c, gate, dy, dres, acc_res, st);
  return NNL_OK;
}

int nnl_bn_bwd_apply(int dtype, int64_t rows, int32_t c, const void* x, const void* gy,
                     const float* partials, int32_t nparts, const float* gamma,
                     const float* save_mean, const float* save_istd, int batch_stat,
                     void* dx, int acc_x, float* dgamma, int acc_g, float* dbeta, int acc_b,
                     void* conv_bias_grad, int acc_cb, int32_t* nonfinite, void* ws,
                     size_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (ws_bytes < bn_ws_bytes(rows, c))
    return fail(NNL_ERR_INVALID_ARGUMENT, "bn workspace too small");
  if (!partials || nparts <= 0) return fail(NNL_ERR_INVALID_ARGUMENT, "no statistics partials");
  if (!use_stream(dtype, rows, c, x, gy, dx))
    return fail(NNL_ERR_UNSUPPORTED, "bn_bwd_apply needs the streaming layout");
  const int64_t bx = bn_stream_rows(BNS_STATS_B, 2, rows, c);
  float* gsum = (float*)ws + bx * 2 * c;
  float* bparts = gsum + 2 * c;
  launch_k(k_bn_finalize_bwd, (c + kRedCols - 1) / kRedCols, 1024, 0, st, 
      partials, nparts, c, gsum, dgamma, acc_g, dbeta, acc_b, nonfinite);
  NNL_CHECK_LAUNCH();
  if (!dx) return NNL_OK;
  float* bp = conv_bias_grad ? bparts : nullptr;
  BnStreamArgs a = {};
  a.rows = rows; a.c = c; a.x = (const __half*)x; a.out = (__half*)dx; a.dy = (const __half*)gy;
  a.gamma = gamma; a.mu = save_mean; a.istd = save_istd; a.gsum = gsum;
  a.partials = bp; a.relu = 0; a.acc = acc_x; a.batch_stat = batch_stat;
  a.reverse = 1;  // the dgrad epilogue wrote gy first to last
  int rc = bn_stream_launch(BNS_APPLY_B, a, st);
  if (rc) return rc;
  if (bp) {
    const int32_t brows = bn_stream_rows(BNS_APPLY_B, bn_stream_nt(BNS_APPLY_B, a), rows, c);
    launch_k(k_bn_bias_finalize<__half>, (c + kRedCols - 1) / kRedCols, 1024, 0, st, 
        bp, brows, c, (__half*)conv_bias_grad, acc_cb, nonfinite);
    NNL_CHECK_LAUNCH();
  }
  return NNL_OK;
}

}  // extern "C"
