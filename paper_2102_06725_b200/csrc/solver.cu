// Multi-tensor solver and all-reduce bucket kernels.
//
//   nnl_multi_nonfinite   <- SgdSolver.check_inf_or_nan_grad (solver.py:115-117)
//   nnl_multi_scale_grad  <- SgdSolver.scale_grad            (solver.py:106-109)
//   nnl_multi_sgd_update  <- dynamic_step + update           (solver.py:100-104,132-155)
//   nnl_bucket_*          <- Communicator._reduce fold       (communicator.py:99-105)
//
// All of them walk a host-built chunk table (<=4096 elements per chunk) so one
// launch covers every parameter regardless of size spread (64 .. 2.4M).
#include "common.cuh"

namespace nnl {

template <typename F>
__device__ __forceinline__ void for_chunks(const nnl_chunk* __restrict__ chunks, int32_t n_chunks,
                                           F&& f) {
  for (int32_t ci = blockIdx.x; ci < n_chunks; ci += gridDim.x) {
    const nnl_chunk ch = chunks[ci];
    for (int32_t j = threadIdx.x; j < ch.len; j += blockDim.x) f(ci, ch.slot, ch.start + j);
  }
}

__device__ __forceinline__ float load_any(const void* p, int dtype, int64_t i) {
  return dtype == NNL_F16 ? __half2float(reinterpret_cast<const __half*>(p)[i])
                          : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void store_any(void* p, int dtype, int64_t i, float v) {
  if (dtype == NNL_F16)
    reinterpret_cast<__half*>(p)[i] = __float2half_rn(v);
  else
    reinterpret_cast<float*>(p)[i] = v;
}

__global__ void k_multi_nonfinite(const nnl_param_slot* __restrict__ slots,
                                  const nnl_chunk* __restrict__ chunks, int32_t n_chunks,
                                  int32_t* flag) {
  pdl_wait();
  pdl_trigger();
  int bad = 0;
  for_chunks(chunks, n_chunks, [&](int32_t, int32_t s, int64_t i) {
    bad |= !isfinite(load_any(slots[s].grad, slots[s].dtype, i));
  });
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void k_multi_scale(const nnl_param_slot* __restrict__ slots,
                              const nnl_chunk* __restrict__ chunks, int32_t n_chunks,
                              float factor) {
  pdl_wait();
  pdl_trigger();
  for_chunks(chunks, n_chunks, [&](int32_t, int32_t s, int64_t i) {
    const nnl_param_slot& p = slots[s];
    store_any(p.grad, p.dtype, i, __fmul_rn(load_any(p.grad, p.dtype, i), factor));
  });
}

__global__ void k_multi_sumsq(const nnl_param_slot* __restrict__ slots,
                              const nnl_chunk* __restrict__ chunks, int32_t n_chunks,
                              double* out) {
  pdl_wait();
  pdl_trigger();
  double acc = 0.0;
  for_chunks(chunks, n_chunks, [&](int32_t, int32_t s, int64_t i) {
    float g = load_any(slots[s].grad, slots[s].dtype, i);
    acc += (double)__fmul_rn(g, g);
  });
  acc = warp_sum_d(acc);
  __shared__ double part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    atomicAdd(out, t);
  }
}

// one parameter element of the update (solver.py:100-109 + Momentum/wd); g is the
// gradient as stored, returned: the (unscaled, re-rounded) gradient to store back
__device__ __forceinline__ float update_elem(float g, bool f16, bool scaled, float factor,
                                             float& m, float* mom, float lr, float momentum,
                                             float wd) {
  if (scaled) {
    // scale_grad rounds the unscaled gradient back into grad storage (R10)
    g = __fmul_rn(g, factor);
    if (f16) g = __half2float(__float2half_rn(g));
  }
  float gw = g;
  if (wd != 0.f) gw = __fadd_rn(gw, __fmul_rn(wd, m));
  float step = __fmul_rn(lr, gw);
  if (mom) {
    step = __fadd_rn(__fmul_rn(momentum, *mom), step);
    *mom = step;
  }
  m = __fsub_rn(m, step);
  return g;
}

// 4 elements per thread on 4-aligned chunks (16 B master / momentum accesses,
// 8 or 16 B grad / data accesses), scalar otherwise
__global__ void k_multi_update(const nnl_param_slot* __restrict__ slots,
                               const nnl_chunk* __restrict__ chunks, int32_t n_chunks, float lr,
                               float momentum, float wd, const nnl_scaler_state* scaler) {
  pdl_wait();
  pdl_trigger();
  float factor = 1.0f;
  if (scaler) {
    if (scaler->nonfinite) return;  // SkippedInfNan: bytes stay unchanged
    factor = (float)(1.0 / scaler->loss_scale);  // np.float32(1.0 / S)
  }
  const bool scaled = scaler != nullptr;
  for (int32_t ci = blockIdx.x; ci < n_chunks; ci += gridDim.x) {
    const nnl_chunk ch = chunks[ci];
    const nnl_param_slot& p = slots[ch.slot];
    const bool f16 = p.dtype == NNL_F16;
    if (((ch.start | ch.len) & 3) == 0) {
      for (int32_t j = threadIdx.x; j < ch.len / 4; j += blockDim.x) {
        const int64_t i = ch.start + 4 * (int64_t)j;
        float g[4];
        if (f16) {
          const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const __half*>(p.grad) + i);
          const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
          const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
          g[0] = a.x; g[1] = a.y; g[2] = b.x; g[3] = b.y;
        } else {
          const float4 v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.grad) + i);
          g[0] = v.x; g[1] = v.y; g[2] = v.z; g[3] = v.w;
        }
        float4 m4 = *reinterpret_cast<const float4*>(p.master + i);
        float m[4] = {m4.x, m4.y, m4.z, m4.w};
        float mo[4] = {0.f, 0.f, 0.f, 0.f};
        if (p.momentum) {
          const float4 o4 = *reinterpret_cast<const float4*>(p.momentum + i);
          mo[0] = o4.x; mo[1] = o4.y; mo[2] = o4.z; mo[3] = o4.w;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          g[e] = update_elem(g[e], f16, scaled, factor, m[e], p.momentum ? &mo[e] : nullptr, lr,
                             momentum, wd);
        if (p.momentum) *reinterpret_cast<float4*>(p.momentum + i) = make_float4(mo[0], mo[1], mo[2], mo[3]);
        *reinterpret_cast<float4*>(p.master + i) = make_float4(m[0], m[1], m[2], m[3]);
        if (f16) {
          const __half2 d0 = __floats2half2_rn(m[0], m[1]), d1 = __floats2half2_rn(m[2], m[3]);
          uint2 du;
          du.x = *reinterpret_cast<const uint32_t*>(&d0);
          du.y = *reinterpret_cast<const uint32_t*>(&d1);
          *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(p.data) + i) = du;
          if (scaled) {
            const __half2 g0 = __floats2half2_rn(g[0], g[1]), g1 = __floats2half2_rn(g[2], g[3]);
            uint2 gu;
            gu.x = *reinterpret_cast<const uint32_t*>(&g0);
            gu.y = *reinterpret_cast<const uint32_t*>(&g1);
            *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(p.grad) + i) = gu;
          }
        } else {
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.data) + i) =
              make_float4(m[0], m[1], m[2], m[3]);
          if (scaled)
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.grad) + i) =
                make_float4(g[0], g[1], g[2], g[3]);
        }
      }
    } else {
      for (int32_t j = threadIdx.x; j < ch.len; j += blockDim.x) {
        const int64_t i = ch.start + j;
        float m = p.master[i];
        float mo = p.momentum ? p.momentum[i] : 0.f;
        const float g = update_elem(load_any(p.grad, p.dtype, i), f16, scaled, factor, m,
                                    p.momentum ? &mo : nullptr, lr, momentum, wd);
        if (scaled) store_any(p.grad, p.dtype, i, g);
        if (p.momentum) p.momentum[i] = mo;
        p.master[i] = m;
        store_any(p.data, p.dtype, i, m);
      }
    }
  }
}

__global__ void k_scaler_finish(nnl_scaler_state* s) {
  pdl_wait();
  pdl_trigger();
  if (s->nonfinite) {
    s->loss_scale = s->loss_scale / s->scaling_factor;
    s->counter = 0;
    s->applied = 0;
  } else {
    if (s->counter > s->interval) {
      s->loss_scale = s->loss_scale * s->scaling_factor;
      s->counter = 0;
    }
    s->counter += 1;
    s->applied = 1;
  }
  s->nonfinite = 0;
}

// 4 elements per thread when the chunk, its bucket position and its start are
// 4-aligned (every chunk of a parameter whose size is a multiple of 4), else scalar
__global__ void k_bucket_pack(const nnl_param_slot* __restrict__ slots,
                              const nnl_chunk* __restrict__ chunks,
                              const int64_t* __restrict__ pos, int32_t n_chunks,
                              float* __restrict__ bucket) {
  pdl_wait();
  pdl_trigger();
  for (int32_t ci = blockIdx.x; ci < n_chunks; ci += gridDim.x) {
    const nnl_chunk ch = chunks[ci];
    const nnl_param_slot& p = slots[ch.slot];
    const int64_t b0 = pos[ci];
    if (((b0 | ch.start | ch.len) & 3) == 0) {
      float4* dst = reinterpret_cast<float4*>(bucket + b0);
      for (int32_t j = threadIdx.x; j < ch.len / 4; j += blockDim.x) {
        float4 v;
        if (p.dtype == NNL_F16) {
          const uint2 u = reinterpret_cast<const uint2*>(
              reinterpret_cast<const __half*>(p.grad) + ch.start)[j];
          const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
          const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
          v = make_float4(a.x, a.y, b.x, b.y);
        } else {
          v = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.grad) +
                                              ch.start)[j];
        }
        dst[j] = v;
      }
    } else {
      for (int32_t j = threadIdx.x; j < ch.len; j += blockDim.x)
        bucket[b0 + j] = load_any(p.grad, p.dtype, ch.start + j);
    }
  }
}

// g = q(sum / f32(n)) into the gradient storage (communicator.py:99-105), OR of
// non-finite results into the overflow flag
__global__ void k_bucket_unpack(const nnl_param_slot* __restrict__ slots,
                                const nnl_chunk* __restrict__ chunks,
                                const int64_t* __restrict__ pos, int32_t n_chunks,
                                const float* __restrict__ bucket, float world, int32_t* flag) {
  pdl_wait();
  pdl_trigger();
  int bad = 0;
  for (int32_t ci = blockIdx.x; ci < n_chunks; ci += gridDim.x) {
    const nnl_chunk ch = chunks[ci];
    const nnl_param_slot& p = slots[ch.slot];
    const int64_t b0 = pos[ci];
    if (((b0 | ch.start | ch.len) & 3) == 0) {
      const float4* src = reinterpret_cast<const float4*>(bucket + b0);
      for (int32_t j = threadIdx.x; j < ch.len / 4; j += blockDim.x) {
        const float4 s4 = src[j];
        const float v0 = __fdiv_rn(s4.x, world), v1 = __fdiv_rn(s4.y, world);
        const float v2 = __fdiv_rn(s4.z, world), v3 = __fdiv_rn(s4.w, world);
        if (p.dtype == NNL_F16) {
          const __half2 a = __floats2half2_rn(v0, v1), b = __floats2half2_rn(v2, v3);
          uint2 u;
          u.x = *reinterpret_cast<const uint32_t*>(&a);
          u.y = *reinterpret_cast<const uint32_t*>(&b);
          reinterpret_cast<uint2*>(reinterpret_cast<__half*>(p.grad) + ch.start)[j] = u;
          const float2 fa = __half22float2(a), fb = __half22float2(b);
          bad |= !isfinite(fa.x) | !isfinite(fa.y) | !isfinite(fb.x) | !isfinite(fb.y);
        } else {
          reinterpret_cast<float4*>(reinterpret_cast<float*>(p.grad) + ch.start)[j] =
              make_float4(v0, v1, v2, v3);
          bad |= !isfinite(v0) | !isfinite(v1) | !isfinite(v2) | !isfinite(v3);
        }
      }
    } else {
      for (int32_t j = threadIdx.x; j < ch.len; j += blockDim.x) {
        float v = __fdiv_rn(bucket[b0 + j], world);  // acc /= f32(n)
        store_any(p.grad, p.dtype, ch.start + j, v);
        bad |= !isfinite(load_any(p.grad, p.dtype, ch.start + j));
      }
    }
  }
  if (flag && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

static int chunk_grid(int32_t n_chunks) { return n_chunks < 148 * 8 ? (n_chunks > 0 ? n_chunks : 1) : 148 * 8; }

}  // namespace nnl

using namespace nnl;

extern "C" {

int nnl_multi_nonfinite(const nnl_param_slot* slots, const nnl_chunk* chunks, int32_t n_chunks,
                        int32_t* flag, void* stream) {
  if (n_chunks <= 0) return NNL_OK;
  launch_k(k_multi_nonfinite, chunk_grid(n_chunks), 256, 0, as_stream(stream), slots, chunks, n_chunks,
                                                                        flag);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_multi_scale_grad(const nnl_param_slot* slots, const nnl_chunk* chunks, int32_t n_chunks,
                         float factor, void* stream) {
  if (n_chunks <= 0) return NNL_OK;
  launch_k(k_multi_scale, chunk_grid(n_chunks), 256, 0, as_stream(stream), slots, chunks, n_chunks,
                                                                    factor);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_multi_sumsq(const nnl_param_slot* slots, const nnl_chunk* chunks, int32_t n_chunks,
                    double* out, void* stream) {
  if (n_chunks <= 0) return NNL_OK;
  launch_k(k_multi_sumsq, chunk_grid(n_chunks), 256, 0, as_stream(stream), slots, chunks, n_chunks,
                                                                    out);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_multi_sgd_update(const nnl_param_slot* slots, const nnl_chunk* chunks, int32_t n_chunks,
                         float lr, float momentum, float weight_decay, nnl_scaler_state* scaler,
                         void* stream) {
  if (n_chunks <= 0) return NNL_OK;
  launch_k(k_multi_update, chunk_grid(n_chunks), 256, 0, as_stream(stream), 
      slots, chunks, n_chunks, lr, momentum, weight_decay, scaler);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_scaler_finish(nnl_scaler_state* scaler, void* stream) {
  launch_k(k_scaler_finish, 1, 1, 0, as_stream(stream), scaler);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_bucket_pack(const nnl_param_slot* slots, const nnl_chunk* chunks, const int64_t* chunk_pos,
                    int32_t n_chunks, float* bucket, void* stream) {
  if (n_chunks <= 0) return NNL_OK;
  launch_k(k_bucket_pack, chunk_grid(n_chunks), 256, 0, as_stream(stream), slots, chunks, chunk_pos,
                                                                    n_chunks, bucket);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_bucket_unpack_mean(const nnl_param_slot* slots, const nnl_chunk* chunks,
                           const int64_t* chunk_pos, int32_t n_chunks, const float* bucket,
                           int32_t world, int32_t* nonfinite, void* stream) {
  if (n_chunks <= 0) return NNL_OK;
  launch_k(k_bucket_unpack, chunk_grid(n_chunks), 256, 0, as_stream(stream), 
      slots, chunks, chunk_pos, n_chunks, bucket, (float)world, nonfinite);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

}  // extern "C"
