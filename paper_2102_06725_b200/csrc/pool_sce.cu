// MaxPooling (src/functions.py:217-291) and SoftmaxCrossEntropy
// (src/functions.py:320-360) on NHWC / row-major device buffers.
#include "common.cuh"

namespace nnl {

// ---- MaxPooling ------------------------------------------------------------
// Forward: scan the window in row-major order; the first maximum wins and the
// first NaN wins over everything (np.argmax, functions.py:265); positions
// outside the input read as -inf (functions.py:258-260).  The window-local
// index i*kw+j is kept as uint8 (the reference keeps a padded flat index;
// both identify the same element).
template <typename T>
__global__ void k_maxpool_fwd(nnl_pool_shape ps, const T* __restrict__ x, T* __restrict__ y,
                              uint8_t* __restrict__ arg) {
  const int64_t total = (int64_t)ps.n * ps.p * ps.q * ps.c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(i % ps.c);
    int64_t t = i / ps.c;
    int oq = (int)(t % ps.q);
    t /= ps.q;
    int op = (int)(t % ps.p);
    int b = (int)(t / ps.p);
    float best = -INFINITY;
    int bi = 0;
    bool have_nan = false;
    for (int di = 0; di < ps.kh; ++di) {
      int ih = op * ps.sh - ps.ph + di;
      for (int dj = 0; dj < ps.kw; ++dj) {
        int iw = oq * ps.sw - ps.pw + dj;
        float v = -INFINITY;
        if (ih >= 0 && ih < ps.h && iw >= 0 && iw < ps.w)
          v = Elem<T>::load(x + (((int64_t)b * ps.h + ih) * ps.w + iw) * ps.c + c);
        int idx = di * ps.kw + dj;
        if (have_nan) continue;
        if (v != v) {
          have_nan = true;
          best = v;
          bi = idx;
        } else if (idx == 0 || v > best) {
          best = v;
          bi = idx;
        }
      }
    }
    Elem<T>::store(y + i, best);
    arg[i] = (uint8_t)bi;
  }
}

// Backward in gather form: every input element sums, in raster order of the
// output windows (the order np.add.at visits them, functions.py:284-288), the
// gradients of the windows whose argmax is that element; then one rounding.
template <typename T>
__global__ void k_maxpool_bwd(nnl_pool_shape ps, const T* __restrict__ dy,
                              const uint8_t* __restrict__ arg, T* __restrict__ dx, int acc) {
  const int64_t total = (int64_t)ps.n * ps.h * ps.w * ps.c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(i % ps.c);
    int64_t t = i / ps.c;
    int iw = (int)(t % ps.w);
    t /= ps.w;
    int ih = (int)(t % ps.h);
    int b = (int)(t / ps.h);
    // windows p with p*sh - ph <= ih <= p*sh - ph + kh - 1
    int hp = ih + ps.ph;
    int wp = iw + ps.pw;
    int p_lo = hp - ps.kh + 1;
    p_lo = p_lo <= 0 ? 0 : (p_lo + ps.sh - 1) / ps.sh;
    int p_hi = hp / ps.sh;
    if (p_hi > ps.p - 1) p_hi = ps.p - 1;
    int q_lo = wp - ps.kw + 1;
    q_lo = q_lo <= 0 ? 0 : (q_lo + ps.sw - 1) / ps.sw;
    int q_hi = wp / ps.sw;
    if (q_hi > ps.q - 1) q_hi = ps.q - 1;
    float s = 0.f;
    for (int op = p_lo; op <= p_hi; ++op) {
      int di = hp - op * ps.sh;
      for (int oq = q_lo; oq <= q_hi; ++oq) {
        int dj = wp - oq * ps.sw;
        int64_t o = (((int64_t)b * ps.p + op) * ps.q + oq) * ps.c + c;
        if (arg[o] == di * ps.kw + dj) s = __fadd_rn(s, Elem<T>::load(dy + o));
      }
    }
    write_out(dx + i, s, acc != 0);
  }
}

// Vectorised variants (fp16, C % 8 == 0, < 2^31 elements): one thread owns 8
// channels of one pixel, 32-bit index math, 16-byte loads/stores.  Same
// semantics as the scalar kernels above.
__global__ void k_maxpool_fwd_h8(nnl_pool_shape ps, const uint4* __restrict__ x,
                                 uint4* __restrict__ y, uint2* __restrict__ arg) {
  const int cg = ps.c >> 3;
  const int total = ps.n * ps.p * ps.q * cg;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % cg;
    int t = i / cg;
    const int oq = t % ps.q;
    t /= ps.q;
    const int op = t % ps.p;
    const int b = t / ps.p;
    float best[8];
    uint8_t bi[8];
    bool nan[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { best[j] = -INFINITY; bi[j] = 0; nan[j] = false; }
    for (int di = 0; di < ps.kh; ++di) {
      const int ih = op * ps.sh - ps.ph + di;
      for (int dj = 0; dj < ps.kw; ++dj) {
        const int iw = oq * ps.sw - ps.pw + dj;
        const int idx = di * ps.kw + dj;
        float v[8];
        if (ih >= 0 && ih < ps.h && iw >= 0 && iw < ps.w) {
          uint4 u = x[((b * ps.h + ih) * ps.w + iw) * cg + g];
          const __half* h = reinterpret_cast<const __half*>(&u);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = __half2float(h[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = -INFINITY;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (nan[j]) continue;
          if (v[j] != v[j]) {
            nan[j] = true; best[j] = v[j]; bi[j] = (uint8_t)idx;
          } else if (idx == 0 || v[j] > best[j]) {
            best[j] = v[j]; bi[j] = (uint8_t)idx;
          }
        }
      }
    }
    uint4 o;
    __half* oh = reinterpret_cast<__half*>(&o);
#pragma unroll
    for (int j = 0; j < 8; ++j) oh[j] = __float2half_rn(best[j]);
    y[i] = o;
    uint2 a;
    a.x = bi[0] | (bi[1] << 8) | (bi[2] << 16) | ((uint32_t)bi[3] << 24);
    a.y = bi[4] | (bi[5] << 8) | (bi[6] << 16) | ((uint32_t)bi[7] << 24);
    arg[i] = a;
  }
}

__global__ void k_maxpool_bwd_h8(nnl_pool_shape ps, const uint4* __restrict__ dy,
                                 const uint2* __restrict__ arg, uint4* __restrict__ dx, int acc) {
  const int cg = ps.c >> 3;
  const int total = ps.n * ps.h * ps.w * cg;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % cg;
    int t = i / cg;
    const int iw = t % ps.w;
    t /= ps.w;
    const int ih = t % ps.h;
    const int b = t / ps.h;
    const int hp = ih + ps.ph, wp = iw + ps.pw;
    int p_lo = hp - ps.kh + 1;
    p_lo = p_lo <= 0 ? 0 : (p_lo + ps.sh - 1) / ps.sh;
    const int p_hi = min(hp / ps.sh, ps.p - 1);
    int q_lo = wp - ps.kw + 1;
    q_lo = q_lo <= 0 ? 0 : (q_lo + ps.sw - 1) / ps.sw;
    const int q_hi = min(wp / ps.sw, ps.q - 1);
    float s[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = 0.f;
    for (int op = p_lo; op <= p_hi; ++op) {
      const int di = hp - op * ps.sh;
      for (int oq = q_lo; oq <= q_hi; ++oq) {
        const int want = di * ps.kw + (wp - oq * ps.sw);
        const int o = ((b * ps.p + op) * ps.q + oq) * cg + g;
        const uint2 a = arg[o];
        const uint4 u = dy[o];
        const __half* h = reinterpret_cast<const __half*>(&u);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t word = j < 4 ? a.x : a.y;
          const int id = (word >> (8 * (j & 3))) & 0xff;
          if (id == want) s[j] = __fadd_rn(s[j], __half2float(h[j]));
        }
      }
    }
    uint4 prev = acc ? dx[i] : make_uint4(0, 0, 0, 0);
    __half* ph = reinterpret_cast<__half*>(&prev);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      ph[j] = __float2half_rn(__fadd_rn(acc ? __half2float(ph[j]) : 0.f, s[j]));
    dx[i] = prev;
  }
}

// ---- SoftmaxCrossEntropy ----------------------------------------------------
// One warp per row.  row_stats[3*b] = (max, log-sum-exp, log p[label]).
template <typename T>
__global__ void k_sce_rows(int64_t batch, int64_t classes, const T* __restrict__ logits,
                           const T* __restrict__ labels, float* __restrict__ row_stats,
                           int32_t* __restrict__ label_err) {
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= batch) return;
  const T* l = logits + row * classes;
  float mx = -INFINITY;
  for (int64_t j = lane; j < classes; j += 32) mx = fmaxf(mx, Elem<T>::load(l + j));
  mx = warp_max(mx);
  float s = 0.f;
  for (int64_t j = lane; j < classes; j += 32) s += expf(__fsub_rn(Elem<T>::load(l + j), mx));
  s = warp_sum(s);
  float logsum = logf(s);
  float lab = Elem<T>::load(labels + row);
  long long id = (long long)lab;
  bool ok = (lab == (float)id) && id >= 0 && id < classes;
  if (lane == 0) {
    float picked = 0.f;
    if (ok) {
      picked = __fsub_rn(__fsub_rn(Elem<T>::load(l + id), mx), logsum);
    } else if (label_err) {
      atomicOr(label_err, 1);
    }
    row_stats[3 * row + 0] = mx;
    row_stats[3 * row + 1] = logsum;
    row_stats[3 * row + 2] = picked;
  }
}

// loss = q(-(sum_b logp[b, t_b]) / B)  (functions.py:346; one block, fixed order)
template <typename T>
__global__ void k_sce_loss(int64_t batch, const float* __restrict__ row_stats, T* __restrict__ out) {
  __shared__ float part[32];
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < batch; i += blockDim.x) s += row_stats[3 * i + 2];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    float mean = __fdiv_rn(t, (float)batch);
    Elem<T>::store(out, -mean);
  }
}

// glogits = q(prev + (p - onehot) * (f32(gy) / B))  (functions.py:352-357)
template <typename T>
__global__ void k_sce_bwd(int64_t batch, int64_t classes, const T* __restrict__ logits,
                          const T* __restrict__ labels, const float* __restrict__ row_stats,
                          const T* __restrict__ gloss, T* __restrict__ g, int acc) {
  const float scale = __fdiv_rn(Elem<T>::load(gloss), (float)batch);
  const int64_t total = batch * classes;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = i / classes, j = i % classes;
    float mx = row_stats[3 * row], ls = row_stats[3 * row + 1];
    float p = expf(__fsub_rn(__fsub_rn(Elem<T>::load(logits + i), mx), ls));
    long long id = (long long)Elem<T>::load(labels + row);
    if (j == id) p = __fsub_rn(p, 1.0f);
    write_out(g + i, __fmul_rn(p, scale), acc != 0);
  }
}

}  // namespace nnl

using namespace nnl;

extern "C" {

int nnl_maxpool_fwd(int dtype, const nnl_pool_shape* ps, const void* x, void* y, uint8_t* argmax,
                    void* stream) {
  if (!ps) return fail(NNL_ERR_INVALID_ARGUMENT, "null pool shape");
  if (ps->kh * ps->kw > 255) return fail(NNL_ERR_UNSUPPORTED, "pool window > 255 elements");
  int64_t total = (int64_t)ps->n * ps->p * ps->q * ps->c;
  if (total <= 0) return NNL_OK;
  if (dtype == NNL_F16 && ps->c % 8 == 0 && (int64_t)ps->n * ps->h * ps->w * ps->c < (1ll << 31) &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
        reinterpret_cast<uintptr_t>(argmax)) & 15) == 0) {
    k_maxpool_fwd_h8<<<grid_for(total / 8, 256), 256, 0, as_stream(stream)>>>(
        *ps, (const uint4*)x, (uint4*)y, (uint2*)argmax);
    NNL_CHECK_LAUNCH();
    return NNL_OK;
  }
  NNL_DISPATCH_DTYPE(dtype, T, {
    k_maxpool_fwd<T><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(*ps, (const T*)x,
                                                                          (T*)y, argmax);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_maxpool_bwd(int dtype, const nnl_pool_shape* ps, const void* dy, const uint8_t* argmax,
                    void* dx, int accumulate, void* stream) {
  if (!ps) return fail(NNL_ERR_INVALID_ARGUMENT, "null pool shape");
  int64_t total = (int64_t)ps->n * ps->h * ps->w * ps->c;
  if (total <= 0) return NNL_OK;
  if (dtype == NNL_F16 && ps->c % 8 == 0 && total < (1ll << 31) &&
      ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx) |
        reinterpret_cast<uintptr_t>(argmax)) & 15) == 0) {
    k_maxpool_bwd_h8<<<grid_for(total / 8, 256), 256, 0, as_stream(stream)>>>(
        *ps, (const uint4*)dy, (const uint2*)argmax, (uint4*)dx, accumulate);
    NNL_CHECK_LAUNCH();
    return NNL_OK;
  }
  NNL_DISPATCH_DTYPE(dtype, T, {
    k_maxpool_bwd<T><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
        *ps, (const T*)dy, argmax, (T*)dx, accumulate);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_sce_fwd(int dtype, int64_t batch, int64_t classes, const void* logits, const void* labels,
                void* loss_out, float* row_stats, int32_t* label_err, void* stream) {
  if (batch <= 0 || classes <= 0) return fail(NNL_ERR_SHAPE_MISMATCH, "empty logits");
  NNL_DISPATCH_DTYPE(dtype, T, {
    int warps = 8;
    k_sce_rows<T><<<(int)((batch + warps - 1) / warps), warps * 32, 0, as_stream(stream)>>>(
        batch, classes, (const T*)logits, (const T*)labels, row_stats, label_err);
    NNL_CHECK_LAUNCH();
    k_sce_loss<T><<<1, 256, 0, as_stream(stream)>>>(batch, row_stats, (T*)loss_out);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_sce_bwd(int dtype, int64_t batch, int64_t classes, const void* logits, const void* labels,
                const float* row_stats, const void* gloss, void* glogits, int accumulate,
                void* stream) {
  int64_t total = batch * classes;
  if (total <= 0) return NNL_OK;
  NNL_DISPATCH_DTYPE(dtype, T, {
    k_sce_bwd<T><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
        batch, classes, (const T*)logits, (const T*)labels, row_stats, (const T*)gloss,
        (T*)glogits, accumulate);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

}  // extern "C"
