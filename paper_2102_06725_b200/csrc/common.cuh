// Shared helpers for libnnl: status plumbing, dtype traits, rounding rules.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/nnl.h"

namespace nnl {

// ---- status plumbing ------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const char* fmt, ...);
void count_launch(int n = 1);
extern int g_tc_enabled;
extern int g_tc_pairs;

// ---- programmatic dependent launch (PDL) ---------------------------------
// Every libnnl kernel is launched with programmatic stream serialization, and
// every kernel begins with griddepcontrol.wait (the predecessor grid has
// completed and its writes are visible) followed by launch_dependents: the
// next kernel's CTAs are scheduled while this one drains, hiding the launch
// gap between consecutive kernels (also inside CUDA graphs).  NNL_PDL=0 or
// nnl_set_pdl(0) launches plainly; the waits then return at once.
extern int g_pdl;
int pdl_enabled();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
extern thread_local cudaError_t t_launch_err;

template <typename... K, typename... A>
inline void launch_k(void (*kernel)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  if (pdl_enabled()) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<K>(args)...);
  if (e != cudaSuccess) t_launch_err = e;
}

#define NNL_CHECK_LAUNCH()                                                      \
  do {                                                                          \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ == cudaSuccess && ::nnl::t_launch_err != cudaSuccess) {              \
      e_ = ::nnl::t_launch_err;                                                 \
      ::nnl::t_launch_err = cudaSuccess;                                        \
    }                                                                           \
    if (e_ != cudaSuccess)                                                      \
      return ::nnl::fail(NNL_ERR_CUDA, "%s:%d %s", __FILE__, __LINE__,          \
                         cudaGetErrorString(e_));                               \
    ::nnl::count_launch();                                                      \
  } while (0)

#define NNL_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      return ::nnl::fail(NNL_ERR_CUDA, "%s:%d %s", __FILE__, __LINE__,          \
                         cudaGetErrorString(e_));                               \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int grid_for(int64_t n, int threads, int max_blocks = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

// ---- numerics -----------------------------------------
// R1: every stored F16 value is q(f32) with RNE, overflow to inf, no FTZ.
__device__ __forceinline__ __half q16(float v) { return __float2half_rn(v); }

template <typename T>
struct Elem;
template <>
struct Elem<float> {
  static __device__ __forceinline__ float load(const float* p) { return *p; }
  static __device__ __forceinline__ float ld(float v) { return v; }
  static __device__ __forceinline__ float st(float v) { return v; }
  static __device__ __forceinline__ void store(float* p, float v) { *p = v; }
};
template <>
struct Elem<__half> {
  static __device__ __forceinline__ float load(const __half* p) { return __half2float(*p); }
  static __device__ __forceinline__ float ld(__half v) { return __half2float(v); }
  static __device__ __forceinline__ __half st(float v) { return __float2half_rn(v); }
  static __device__ __forceinline__ void store(__half* p, float v) { *p = __float2half_rn(v); }
};

// R2: write (q(v + 0)) or accumulate (q(prev + v)); "+0.0f" canonicalises -0
// exactly as numpy's `zeros + g` would before the quantizing write.
template <typename T>
__device__ __forceinline__ void write_out(T* p, float v, bool acc) {
  float prev = acc ? Elem<T>::load(p) : 0.0f;
  Elem<T>::store(p, __fadd_rn(prev, v));
}

__device__ __forceinline__ bool nonfinite_f(float v) { return !isfinite(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace nnl

#define NNL_DISPATCH_DTYPE(dtype, T, ...)                                       \
  do {                                                                          \
    if ((dtype) == NNL_F32) {                                                   \
      using T = float;                                                          \
      __VA_ARGS__;                                                              \
    } else if ((dtype) == NNL_F16) {                                            \
      using T = __half;                                                         \
      __VA_ARGS__;                                                              \
    } else {                                                                    \
      return ::nnl::fail(NNL_ERR_INVALID_ARGUMENT, "bad dtype %d", (int)(dtype)); \
    }                                                                           \
  } while (0)
