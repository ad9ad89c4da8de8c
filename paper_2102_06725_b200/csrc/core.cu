// Status plumbing + bandwidth kernels for storage/numerics and simple layers.
//
//   quantize / fill / accumulate / nonfinite  <- src/tensor.py:46-157
//   rng_uniform (SplitMix64)                  <- src/tensor.py:211-252
//   relu                                      <- src/functions.py:294-317
//   add2, gap                                 <- extensions (oracle/nnl_oracle.py)
#include <stdarg.h>

#include <atomic>

#include "common.cuh"

namespace nnl {

static thread_local std::string t_last_error;
static std::atomic<int64_t> g_launches{0};
int g_tc_enabled = 1;
// CTA-pair (cta_group::2) tiles for long-K GEMMs; NNL_TC_PAIRS=0 disables
int g_tc_pairs = -1;

void set_error(const std::string& msg) { t_last_error = msg; }

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_last_error = buf;
  return code;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

thread_local cudaError_t t_launch_err = cudaSuccess;
int g_pdl = -1;
int pdl_enabled() {
  if (g_pdl < 0) {
    const char* e = getenv("NNL_PDL");
    g_pdl = (e && e[0] == '0') ? 0 : 1;
  }
  return g_pdl;
}

// ---------------------------------------------------------------------------
// vectorised elementwise skeleton: 8 elements (16 B of fp16) per step when the
// pointers are 16-byte aligned, scalar otherwise.
template <typename T>
__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

__global__ void k_quantize_f16(int64_t n, const float* __restrict__ x, float* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __half2float(__float2half_rn(x[i]));
}

template <typename T>
__global__ void k_fill(int64_t n, T* __restrict__ dst, float v) {
  pdl_wait();
  pdl_trigger();
  T hv = Elem<T>::st(v);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = hv;
}

template <typename T>
__global__ void k_fill_dev(int64_t n, T* __restrict__ dst, const double* __restrict__ v) {
  pdl_wait();
  pdl_trigger();
  // NdArray.fill: np.float32(value) then quantize for F16 (tensor.py:125-131)
  T hv = Elem<T>::st(__double2float_rn(*v));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = hv;
}

template <typename T>
__global__ void k_accumulate(int64_t n, const T* __restrict__ src, T* __restrict__ dst, int acc) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    write_out(dst + i, Elem<T>::load(src + i), acc != 0);
}

__global__ void k_accumulate_h8(int64_t n8, const uint4* __restrict__ src, uint4* __restrict__ dst,
                                int acc) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 s = src[i];
    if (!acc) {
      // q(0 + g): only -0 -> +0 changes
      __half2* sh = reinterpret_cast<__half2*>(&s);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __half22float2(sh[j]);
        sh[j] = __floats2half2_rn(__fadd_rn(0.f, f.x), __fadd_rn(0.f, f.y));
      }
      dst[i] = s;
    } else {
      uint4 d = dst[i];
      __half2* sh = reinterpret_cast<__half2*>(&s);
      __half2* dh = reinterpret_cast<__half2*>(&d);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 a = __half22float2(dh[j]);
        float2 b = __half22float2(sh[j]);
        dh[j] = __floats2half2_rn(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
      }
      dst[i] = d;
    }
  }
}

template <typename T>
__global__ void k_nonfinite(int64_t n, const T* __restrict__ x, int32_t* flag) {
  pdl_wait();
  pdl_trigger();
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= nonfinite_f(Elem<T>::load(x + i));
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// SplitMix64 (tensor.py:217-222) and the counter stream (tensor.py:241-252)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4B7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void k_rng_uniform(uint64_t seed, uint64_t counter, int64_t n, double low, double high,
                              T* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const uint64_t base = seed * 0xBF58476D1CE4E5B9ull;
  const double span = __dsub_rn(high, low);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t bits = splitmix64(base + counter + (uint64_t)i);
    double u = __dmul_rn((double)(bits >> 11), 0x1p-53);
    double v = __dadd_rn(low, __dmul_rn(span, u));  // no FMA: numpy does mul then add
    Elem<T>::store(out + i, __double2float_rn(v));
  }
}

// ReLU (functions.py:307-314): np.maximum(x, 0) keeps NaN; bwd multiplies.
__device__ __forceinline__ float relu_f(float x) { return (x > 0.f || x != x) ? x : 0.f; }

template <typename T>
__global__ void k_relu_fwd(int64_t n, const T* __restrict__ x, T* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = Elem<T>::st(relu_f(Elem<T>::load(x + i)));
}

__global__ void k_relu_fwd_h8(int64_t n8, const uint4* __restrict__ x, uint4* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = x[i];
    __half* h = reinterpret_cast<__half*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j) h[j] = __float2half_rn(relu_f(__half2float(h[j])));
    y[i] = v;
  }
}

template <typename T>
__global__ void k_relu_bwd(int64_t n, const T* __restrict__ x, const T* __restrict__ dy,
                           T* __restrict__ dx, int acc) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float g = __fmul_rn(Elem<T>::load(dy + i), Elem<T>::load(x + i) > 0.f ? 1.f : 0.f);
    write_out(dx + i, g, acc != 0);
  }
}

__global__ void k_relu_bwd_h8(int64_t n8, const uint4* __restrict__ x, const uint4* __restrict__ dy,
                              uint4* __restrict__ dx, int acc) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 xv = x[i], gv = dy[i], pv = acc ? dx[i] : make_uint4(0, 0, 0, 0);
    const __half* xh = reinterpret_cast<const __half*>(&xv);
    const __half* gh = reinterpret_cast<const __half*>(&gv);
    __half* ph = reinterpret_cast<__half*>(&pv);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float g = __fmul_rn(__half2float(gh[j]), __half2float(xh[j]) > 0.f ? 1.f : 0.f);
      float prev = acc ? __half2float(ph[j]) : 0.f;
      ph[j] = __float2half_rn(__fadd_rn(prev, g));
    }
    dx[i] = pv;
  }
}

// Add2 (extension): y = q(a + b) [then ReLU on the stored value]
template <typename T>
__global__ void k_add2(int64_t n, const T* __restrict__ a, const T* __restrict__ b,
                       T* __restrict__ y, int fuse_relu) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = Elem<T>::ld(Elem<T>::st(__fadd_rn(Elem<T>::load(a + i), Elem<T>::load(b + i))));
    if (fuse_relu) v = relu_f(v);
    Elem<T>::store(y + i, v);
  }
}

__global__ void k_add2_h8(int64_t n8, const uint4* __restrict__ a, const uint4* __restrict__ b,
                          uint4* __restrict__ y, int fuse_relu) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 av = a[i], bv = b[i], o;
    const __half* ah = reinterpret_cast<const __half*>(&av);
    const __half* bh = reinterpret_cast<const __half*>(&bv);
    __half* oh = reinterpret_cast<__half*>(&o);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      __half s = __float2half_rn(__fadd_rn(__half2float(ah[j]), __half2float(bh[j])));
      oh[j] = fuse_relu ? __float2half_rn(relu_f(__half2float(s))) : s;
    }
    y[i] = o;
  }
}

// GlobalAveragePooling (extension): y[n,c] = q(sum_hw x / hw); NHWC input.
template <typename T>
__global__ void k_gap_fwd(int64_t n, int64_t hw, int64_t c, const T* __restrict__ x,
                          T* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  int64_t total = n * c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / c, ch = i % c;
    const T* p = x + b * hw * c + ch;
    float s = 0.f;
    for (int64_t j = 0; j < hw; ++j) s = __fadd_rn(s, Elem<T>::load(p + j * c));
    Elem<T>::store(y + i, __fdiv_rn(s, (float)hw));
  }
}

template <typename T>
__global__ void k_gap_bwd(int64_t n, int64_t hw, int64_t c, const T* __restrict__ dy,
                          T* __restrict__ dx, int acc) {
  pdl_wait();
  pdl_trigger();
  int64_t total = n * hw * c;
  const float fhw = (float)hw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t ch = i % c, b = i / (hw * c);
    write_out(dx + i, __fdiv_rn(Elem<T>::load(dy + b * c + ch), fhw), acc != 0);
  }
}

// fp16, c % 8 == 0: one thread per (image, 8 channels) computes q(0|prev + dy/hw)
// once per channel and writes the hw pixels as 16 B stores
__global__ void k_gap_bwd_h8(int n, int hw, int c, const __half* __restrict__ dy,
                             __half* __restrict__ dx, int acc) {
  pdl_wait();
  pdl_trigger();
  const int cg = c >> 3;
  const float fhw = (float)hw;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n * cg; t += gridDim.x * blockDim.x) {
    const int b = t / cg, g = t - b * cg;
    const uint4 u = *reinterpret_cast<const uint4*>(dy + (int64_t)b * c + g * 8);
    const __half* h = reinterpret_cast<const __half*>(&u);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __fdiv_rn(__half2float(h[j]), fhw);
    uint4* dst = reinterpret_cast<uint4*>(dx + (int64_t)b * hw * c + g * 8);
    for (int p = 0; p < hw; ++p) {
      __align__(16) __half o[8];
      uint4 pv = make_uint4(0, 0, 0, 0);
      if (acc) pv = dst[(int64_t)p * cg];
      const __half* ph = reinterpret_cast<const __half*>(&pv);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        o[j] = __float2half_rn(__fadd_rn(acc ? __half2float(ph[j]) : 0.f, v[j]));
      dst[(int64_t)p * cg] = *reinterpret_cast<const uint4*>(o);
    }
  }
}

// narrow-channel NCHW f32 -> NHWC (the network input, c = 3): one thread per
// pixel reads its c channel planes (coalesced across threads) and writes the c
// contiguous elements
template <typename T>
__global__ void k_import_narrow(int32_t n, int32_t c, int32_t hw, const float* __restrict__ src,
                                T* __restrict__ dst) {
  pdl_wait();
  pdl_trigger();
  const int total = n * hw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int b = i / hw, pix = i - b * hw;
    const float* s = src + (int64_t)b * c * hw + pix;
    T* d = dst + (int64_t)i * c;
    for (int ch = 0; ch < c; ++ch) Elem<T>::store(d + ch, __ldg(s + (int64_t)ch * hw));
  }
}

template <typename T>
__global__ void k_import(int32_t n, int32_t c, int32_t hw, const float* __restrict__ src,
                         T* __restrict__ dst) {
  pdl_wait();
  pdl_trigger();
  // 32-bit index math (the host guarantees n*c*hw < 2^31)
  const int total = n * c * hw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int ch = i % c;
    const int rest = i / c;
    const int pix = rest % hw;
    const int b = rest / hw;
    Elem<T>::store(dst + i, src[(b * c + ch) * hw + pix]);
  }
}

template <typename T>
__global__ void k_export(int32_t n, int32_t c, int32_t hw, const T* __restrict__ src,
                         float* __restrict__ dst) {
  pdl_wait();
  pdl_trigger();
  const int total = n * c * hw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int pix = i % hw;
    const int rest = i / hw;
    const int ch = rest % c;
    const int b = rest / c;
    dst[i] = Elem<T>::load(src + (b * hw + pix) * c + ch);
  }
}

__global__ void k_fold(int32_t k, const float* const* __restrict__ bufs, int64_t n,
                       float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = bufs[0][i];
    for (int r = 1; r < k; ++r) acc = __fadd_rn(acc, bufs[r][i]);
    out[i] = acc;
  }
}

}  // namespace nnl

using namespace nnl;

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

extern "C" {

const char* nnl_last_error(void) { return t_last_error.c_str(); }
int nnl_version(void) { return 1; }
int64_t nnl_launch_count(int reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}
int nnl_set_tc_enabled(int enabled) {
  int prev = g_tc_enabled;
  g_tc_enabled = enabled;
  return prev;
}
int nnl_set_tc_resident_b(int enabled) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NNL_TC_RESB");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  const int prev = v;
  if (enabled >= 0) v = enabled ? 1 : 0;
  return prev;
}
int nnl_set_tc_tile4(int enabled) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NNL_TILE4");
    v = e ? (e[0] == '0' ? 0 : e[0] == '2' ? 2 : 1) : 1;
  }
  const int prev = v;
  if (enabled >= 0) v = enabled > 2 ? 2 : enabled;
  return prev;
}
int nnl_conv2d_prep_reuse(int enabled) {
  static thread_local int v = 0;
  const int prev = v;
  if (enabled >= 0) v = enabled ? 1 : 0;
  return prev;
}
int nnl_set_tc_halo(int enabled) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NNL_HALO");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  const int prev = v;
  if (enabled >= 0) v = enabled ? 1 : 0;
  return prev;
}

int nnl_set_tc_epi_il(int enabled) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NNL_EPI_IL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  const int prev = v;
  if (enabled >= 0) v = enabled ? 1 : 0;
  return prev;
}
int nnl_set_tc_s2d4(int enabled) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NNL_S2D4");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  const int prev = v;
  if (enabled >= 0) v = enabled ? 1 : 0;
  return prev;
}
int nnl_set_pdl(int enabled) {
  const int prev = pdl_enabled();
  if (enabled >= 0) g_pdl = enabled ? 1 : 0;
  return prev;
}

int nnl_set_tc_pairs(int enabled) {
  if (g_tc_pairs < 0) {
    const char* e = getenv("NNL_TC_PAIRS");
    g_tc_pairs = (e && (e[0] == '0' || e[0] == '2')) ? e[0] - '0' : 1;
  }
  int prev = g_tc_pairs;
  if (enabled >= 0) g_tc_pairs = enabled > 2 ? 2 : enabled;
  return prev;
}

int nnl_quantize_f16(int64_t n, const float* x, float* y, void* stream) {
  if (n <= 0) return NNL_OK;
  launch_k(k_quantize_f16, grid_for(n, 256), 256, 0, as_stream(stream), n, x, y);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_fill(int dtype, int64_t n, void* dst, float value, void* stream) {
  if (n <= 0) return NNL_OK;
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_fill<T>, grid_for(n, 256), 256, 0, as_stream(stream), n, (T*)dst, value);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_fill_from_device(int dtype, int64_t n, void* dst, const double* value, void* stream) {
  if (n <= 0) return NNL_OK;
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_fill_dev<T>, grid_for(n, 256), 256, 0, as_stream(stream), n, (T*)dst, value);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_accumulate(int dtype, int64_t n, const void* src, void* dst, int accumulate,
                   void* stream) {
  if (n <= 0) return NNL_OK;
  if (dtype == NNL_F16 && n % 8 == 0 && al16(src) && al16(dst)) {
    launch_k(k_accumulate_h8, grid_for(n / 8, 256), 256, 0, as_stream(stream), 
        n / 8, (const uint4*)src, (uint4*)dst, accumulate);
  } else {
    NNL_DISPATCH_DTYPE(dtype, T, {
      launch_k(k_accumulate<T>, grid_for(n, 256), 256, 0, as_stream(stream), n, (const T*)src,
                                                                       (T*)dst, accumulate);
    });
  }
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_nonfinite(int dtype, int64_t n, const void* x, int32_t* flag, void* stream) {
  if (n <= 0) return NNL_OK;
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_nonfinite<T>, grid_for(n, 256), 256, 0, as_stream(stream), n, (const T*)x, flag);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_rng_uniform(uint64_t seed, uint64_t counter, int64_t n, double low, double high,
                    int dtype, void* out, void* stream) {
  if (!(low < high)) return fail(NNL_ERR_INVALID_RANGE, "empty range [%g, %g)", low, high);
  if (n <= 0) return NNL_OK;
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_rng_uniform<T>, grid_for(n, 256), 256, 0, as_stream(stream), seed, counter, n, low,
                                                                      high, (T*)out);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_relu_fwd(int dtype, int64_t n, const void* x, void* y, void* stream) {
  if (n <= 0) return NNL_OK;
  if (dtype == NNL_F16 && n % 8 == 0 && al16(x) && al16(y)) {
    launch_k(k_relu_fwd_h8, grid_for(n / 8, 256), 256, 0, as_stream(stream), n / 8, (const uint4*)x,
                                                                       (uint4*)y);
  } else {
    NNL_DISPATCH_DTYPE(dtype, T, {
      launch_k(k_relu_fwd<T>, grid_for(n, 256), 256, 0, as_stream(stream), n, (const T*)x, (T*)y);
    });
  }
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_relu_bwd(int dtype, int64_t n, const void* x, const void* dy, void* dx, int accumulate,
                 void* stream) {
  if (n <= 0) return NNL_OK;
  if (dtype == NNL_F16 && n % 8 == 0 && al16(x) && al16(dy) && al16(dx)) {
    launch_k(k_relu_bwd_h8, grid_for(n / 8, 256), 256, 0, as_stream(stream), 
        n / 8, (const uint4*)x, (const uint4*)dy, (uint4*)dx, accumulate);
  } else {
    NNL_DISPATCH_DTYPE(dtype, T, {
      launch_k(k_relu_bwd<T>, grid_for(n, 256), 256, 0, as_stream(stream), 
          n, (const T*)x, (const T*)dy, (T*)dx, accumulate);
    });
  }
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_add2_fwd(int dtype, int64_t n, const void* a, const void* b, void* y, int fuse_relu,
                 void* stream) {
  if (n <= 0) return NNL_OK;
  if (dtype == NNL_F16 && n % 8 == 0 && al16(a) && al16(b) && al16(y)) {
    launch_k(k_add2_h8, grid_for(n / 8, 256), 256, 0, as_stream(stream), 
        n / 8, (const uint4*)a, (const uint4*)b, (uint4*)y, fuse_relu);
  } else {
    NNL_DISPATCH_DTYPE(dtype, T, {
      launch_k(k_add2<T>, grid_for(n, 256), 256, 0, as_stream(stream), n, (const T*)a, (const T*)b,
                                                                 (T*)y, fuse_relu);
    });
  }
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_gap_fwd(int dtype, int64_t n, int64_t hw, int64_t c, const void* x, void* y,
                void* stream) {
  if (n * c <= 0) return NNL_OK;
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_gap_fwd<T>, grid_for(n * c, 256), 256, 0, as_stream(stream), n, hw, c, (const T*)x,
                                                                      (T*)y);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_gap_bwd(int dtype, int64_t n, int64_t hw, int64_t c, const void* dy, void* dx,
                int accumulate, void* stream) {
  if (n * c * hw <= 0) return NNL_OK;
  if (dtype == NNL_F16 && c % 8 == 0 && n * c < (1ll << 31) &&
      !((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx)) & 15)) {
    launch_k(k_gap_bwd_h8, grid_for(n * (c / 8), 256), 256, 0, as_stream(stream), 
        (int)n, (int)hw, (int)c, (const __half*)dy, (__half*)dx, accumulate);
    NNL_CHECK_LAUNCH();
    return NNL_OK;
  }
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_gap_bwd<T>, grid_for(n * hw * c, 256), 256, 0, as_stream(stream), 
        n, hw, c, (const T*)dy, (T*)dx, accumulate);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_import_f32(int dtype, int32_t n, int32_t c, int32_t hw, const float* src, void* dst,
                   void* stream) {
  int64_t total = (int64_t)n * c * hw;
  if (total <= 0) return NNL_OK;
  if (total >= (1ll << 31)) return fail(NNL_ERR_UNSUPPORTED, "import of >= 2^31 elements");
  NNL_DISPATCH_DTYPE(dtype, T, {
    if (c <= 4 && hw > 1)
      launch_k(k_import_narrow<T>, grid_for((int64_t)n * hw, 256), 256, 0, as_stream(stream), 
          n, c, hw, src, (T*)dst);
    else
      launch_k(k_import<T>, grid_for(total, 256), 256, 0, as_stream(stream), n, c, hw, src, (T*)dst);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_export_f32(int dtype, int32_t n, int32_t c, int32_t hw, const void* src, float* dst,
                   void* stream) {
  int64_t total = (int64_t)n * c * hw;
  if (total <= 0) return NNL_OK;
  if (total >= (1ll << 31)) return fail(NNL_ERR_UNSUPPORTED, "export of >= 2^31 elements");
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_export<T>, grid_for(total, 256), 256, 0, as_stream(stream), n, c, hw, (const T*)src, dst);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_fold_f32(int32_t k, const float* const* bufs_dev, int64_t n, float* out, void* stream) {
  if (n <= 0 || k <= 0) return NNL_OK;
  launch_k(k_fold, grid_for(n, 256), 256, 0, as_stream(stream), k, bufs_dev, n, out);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

}  // extern "C"
