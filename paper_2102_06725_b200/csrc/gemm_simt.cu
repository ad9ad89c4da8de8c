// SIMT implicit GEMM: the fp32 (TypeConfig.FLOAT) path and the fallback for
// shapes the tcgen05 kernel does not take (unaligned channel counts, tiny
// affine layers).  64x64 tile, BK=16, 4x4 micro-tile per thread, optional
// deterministic split-K over the reduction with f32 partials.
#include "gemm.cuh"

namespace nnl {

constexpr int kSB = 64, kSK = 16;

// affine problems are plain (permuted-row) matrices: no im2col index math
__device__ __forceinline__ int64_t affine_row32(const ConvGeom& g, int32_t f) {
  if (g.ahw == 1) return f;
  return (int64_t)(f % g.ac) * g.ahw + f / g.ac;
}

template <typename T>
__device__ __forceinline__ float fetch_a(const GemmProblem& pb, int64_t m, int64_t k) {
  const ConvGeom& g = pb.g;
  const T* a = (const T*)pb.a;
  if (g.affine) {
    // fprop: x[b][f]; dgrad: dy[b][o]; wgrad: dy[b = k][o = m]
    return pb.mode == kWgrad ? Elem<T>::load(a + k * g.k + m) : Elem<T>::load(a + m * pb.K + k);
  }
  if (pb.mode == kFprop) {
    int c = (int)(k % g.c);
    int64_t t = k / g.c;
    int s = (int)(t % g.s), r = (int)(t / g.s);
    int q = (int)(m % g.q);
    int64_t u = m / g.q;
    int p = (int)(u % g.p), b = (int)(u / g.p);
    int ih = p * g.sh - g.ph + r, iw = q * g.sw - g.pw + s;
    if (ih < 0 || ih >= g.h || iw < 0 || iw >= g.w) return 0.f;
    return Elem<T>::load(a + (((int64_t)b * g.h + ih) * g.w + iw) * g.c + c);
  } else if (pb.mode == kDgrad) {
    int ko = (int)(k % g.k);
    int64_t t = k / g.k;
    int s = (int)(t % g.s), r = (int)(t / g.s);
    int wq = (int)(m % g.w);
    int64_t u = m / g.w;
    int hh = (int)(u % g.h), b = (int)(u / g.h);
    int th = hh + g.ph - r, tw = wq + g.pw - s;
    if (th < 0 || tw < 0 || th % g.sh || tw % g.sw) return 0.f;
    th /= g.sh;
    tw /= g.sw;
    if (th >= g.p || tw >= g.q) return 0.f;
    return Elem<T>::load(a + (((int64_t)b * g.p + th) * g.q + tw) * g.k + ko);
  } else {  // wgrad: A(m=k_out, k=pix) = dy[pix][k_out]
    return Elem<T>::load(a + k * g.k + m);
  }
}

template <typename T>
__device__ __forceinline__ float fetch_b(const GemmProblem& pb, int64_t n, int64_t k) {
  const ConvGeom& g = pb.g;
  const T* b = (const T*)pb.b;
  if (g.affine) {
    if (pb.mode == kFprop) return Elem<T>::load(b + affine_row32(g, (int32_t)k) * g.k + n);
    if (pb.mode == kDgrad) return Elem<T>::load(b + affine_row32(g, (int32_t)n) * g.k + k);
    return Elem<T>::load(b + k * pb.N + n);  // wgrad: x[b = k][f = n]
  }
  if (pb.mode == kFprop) {
    return Elem<T>::load(b + n * pb.K + k);
  } else if (pb.mode == kDgrad) {
    if (g.affine) return Elem<T>::load(b + affine_row(g, n) * g.k + k);  // W[i=n][o=k]
    int ko = (int)(k % g.k);
    int64_t rs = k / g.k;
    return Elem<T>::load(b + ((int64_t)ko * g.r * g.s + rs) * g.c + n);
  } else {  // wgrad: B(n=(r,s,c), k=pix) = x gather
    int c = (int)(n % g.c);
    int64_t t = n / g.c;
    int s = (int)(t % g.s), r = (int)(t / g.s);
    int q = (int)(k % g.q);
    int64_t u = k / g.q;
    int p = (int)(u % g.p), bb = (int)(u / g.p);
    int ih = p * g.sh - g.ph + r, iw = q * g.sw - g.pw + s;
    if (ih < 0 || ih >= g.h || iw < 0 || iw >= g.w) return 0.f;
    return Elem<T>::load(b + (((int64_t)bb * g.h + ih) * g.w + iw) * g.c + c);
  }
}

template <typename T>
__device__ __forceinline__ void epilogue_store(const GemmProblem& pb, int64_t m, int64_t n, float v,
                                               int& bad) {
  if (pb.bias) v = __fadd_rn(v, Elem<T>::load((const T*)pb.bias + n));
  int64_t idx = pb.out_trans ? affine_row(pb.g, n) * pb.M + m : m * pb.N + n;
  T* o = (T*)pb.out;
  write_out(o + idx, v, pb.acc != 0);
  bad |= !isfinite(Elem<T>::load(o + idx));
}

template <typename T>
__global__ void __launch_bounds__(256) k_simt_gemm(GemmProblem pb, int64_t k_per_split,
                                                  float* __restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  __shared__ float As[kSK][kSB + 4];
  __shared__ float Bs[kSK][kSB + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.x * kSB, n0 = (int64_t)blockIdx.y * kSB;
  const int64_t k_begin = (int64_t)blockIdx.z * k_per_split;
  int64_t k_end = k_begin + k_per_split;
  if (k_end > pb.K) k_end = pb.K;
  float acc[4][4] = {};
  for (int64_t k0 = k_begin; k0 < k_end; k0 += kSK) {
    for (int e = threadIdx.x; e < kSB * kSK; e += 256) {
      int kk = e / kSB, mm = e % kSB;
      int64_t gk = k0 + kk;
      As[kk][mm] = (m0 + mm < pb.M && gk < k_end) ? fetch_a<T>(pb, m0 + mm, gk) : 0.f;
      Bs[kk][mm] = (n0 + mm < pb.N && gk < k_end) ? fetch_b<T>(pb, n0 + mm, gk) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kSK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = As[kk][ty * 4 + i];
        bv[i] = Bs[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  int bad = 0;
  if (pb.bias_grad && blockIdx.y == 0 && gridDim.z == 1) {
    // affine bias gradient db[o] = sum_b dy[b][o] (functions.py:116) = the row
    // sums of A, taken by the first N tile while the operands are hot
    for (int mm = threadIdx.x; mm < kSB; mm += blockDim.x) {
      const int64_t m = m0 + mm;
      if (m >= pb.M) continue;
      float s = 0.f;
      for (int64_t k = 0; k < pb.K; ++k) s += fetch_a<T>(pb, m, k);
      T* db = (T*)pb.bias_grad;
      write_out(db + m, s, pb.acc_bias != 0);
      bad |= !isfinite(Elem<T>::load(db + m));
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= pb.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t n = n0 + tx * 4 + j;
      if (n >= pb.N) continue;
      if (partial)
        partial[((int64_t)blockIdx.z * pb.M + m) * pb.N + n] = acc[i][j];
      else
        epilogue_store<T>(pb, m, n, acc[i][j], bad);
    }
  }
  if (pb.nonfinite && !partial && __syncthreads_or(bad) && threadIdx.x == 0)
    atomicOr(pb.nonfinite, 1);
}

// fixed-order split-K reduction + the same epilogue
template <typename T>
__global__ void k_splitk_reduce(GemmProblem pb, int splits, const float* __restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  int bad = 0;
  const int64_t total = pb.M * pb.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + i];
    epilogue_store<T>(pb, i / pb.N, i % pb.N, s, bad);
  }
  if (pb.nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(pb.nonfinite, 1);
}

// bias gradient: per-column f32 partial sums over row chunks, then fixed-order combine
// narrow outputs (cols <= 128): the block's threads tile (row lanes x cols),
// so a warp reads whole rows (coalesced) and the lane sums are combined in
// fixed order in shared memory
template <typename T>
__global__ void __launch_bounds__(256) k_colsum_partial_narrow(
    int64_t rows, int cols, int64_t rows_per_block, const T* __restrict__ x,
    float* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[256];
  const int lanes = 256 / cols;
  const int col = threadIdx.x % cols, lane = threadIdx.x / cols;
  const int64_t r0 = blockIdx.x * rows_per_block;
  int64_t r1 = r0 + rows_per_block;
  if (r1 > rows) r1 = rows;
  float s = 0.f;
  if (lane < lanes)
    for (int64_t r = r0 + lane; r < r1; r += lanes) s += Elem<T>::load(x + r * cols + col);
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < cols) {
    float t = 0.f;
    for (int l = 0; l < lanes; ++l) t += red[l * cols + threadIdx.x];
    part[blockIdx.x * (int64_t)cols + threadIdx.x] = t;
  }
}

template <typename T>
__global__ void k_colsum_partial(int64_t rows, int64_t cols, int64_t rows_per_block,
                                 const T* __restrict__ x, float* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  const int64_t col = blockIdx.y * (int64_t)blockDim.x + threadIdx.x;
  if (col >= cols) return;
  int64_t r0 = blockIdx.x * rows_per_block, r1 = r0 + rows_per_block;
  if (r1 > rows) r1 = rows;
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += Elem<T>::load(x + r * cols + col);
  part[blockIdx.x * cols + col] = s;
}

template <typename T>
__global__ void k_colsum_final(int64_t cols, int nparts, const float* __restrict__ part,
                               T* __restrict__ out, int acc, int32_t* flag) {
  pdl_wait();
  pdl_trigger();
  const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int bad = 0;
  if (col < cols) {
    double s = 0.0;
    for (int i = 0; i < nparts; ++i) s += (double)part[(int64_t)i * cols + col];
    write_out(out + col, (float)s, acc != 0);
    bad = !isfinite(Elem<T>::load(out + col));
  }
  if (flag && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

static int simt_splits(const GemmProblem& pb) {
  if (pb.bias_grad) return 1;  // the fused bias sums need the whole K range
  int64_t tiles = ((pb.M + kSB - 1) / kSB) * ((pb.N + kSB - 1) / kSB);
  // short reductions run in one pass: a split costs a partial round trip and a
  // second launch, more than the K loop it shortens
  if (pb.K <= 2048) return 1;
  int64_t want = (148 * 4 + tiles - 1) / tiles;
  int64_t max_by_k = (pb.K + 511) / 512;
  if (want > max_by_k) want = max_by_k;
  if (want > 64) want = 64;
  if (want < 1) want = 1;
  return (int)want;
}

size_t simt_ws_bytes(const GemmProblem& pb) {
  int sp = simt_splits(pb);
  return sp > 1 ? (size_t)sp * pb.M * pb.N * sizeof(float) : 0;
}

int simt_gemm(const GemmProblem& pb, int dtype, void* ws, size_t ws_bytes, cudaStream_t st) {
  int sp = simt_splits(pb);
  if (sp > 1 && ws_bytes < simt_ws_bytes(pb)) sp = 1;
  int64_t kps = (pb.K + sp - 1) / sp;
  kps = (kps + kSK - 1) / kSK * kSK;
  sp = (int)((pb.K + kps - 1) / kps);
  if (sp < 1) sp = 1;
  dim3 grid((unsigned)((pb.M + kSB - 1) / kSB), (unsigned)((pb.N + kSB - 1) / kSB), (unsigned)sp);
  float* partial = sp > 1 ? (float*)ws : nullptr;
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_simt_gemm<T>, grid, 256, 0, st, pb, kps > 0 ? kps : kSK, partial);
    NNL_CHECK_LAUNCH();
    if (partial) {
      launch_k(k_splitk_reduce<T>, grid_for(pb.M * pb.N, 256), 256, 0, st, pb, sp, partial);
      NNL_CHECK_LAUNCH();
    }
  });
  return NNL_OK;
}

size_t bias_grad_ws_bytes(int64_t rows, int64_t cols) {
  int64_t parts = rows < 256 ? 1 : 256;
  return (size_t)parts * cols * sizeof(float);
}

int bias_grad(int dtype, int64_t rows, int64_t cols, const void* dy, void* db, int acc,
              int32_t* nonfinite, void* ws, size_t ws_bytes, cudaStream_t st) {
  int64_t parts = rows < 256 ? 1 : 256;
  if (ws_bytes < (size_t)parts * cols * sizeof(float))
    return fail(NNL_ERR_INVALID_ARGUMENT, "bias-grad workspace too small");
  int64_t rpb = (rows + parts - 1) / parts;
  dim3 grid((unsigned)parts, (unsigned)((cols + 127) / 128));
  NNL_DISPATCH_DTYPE(dtype, T, {
    if (cols <= 128)
      launch_k(k_colsum_partial_narrow<T>, dim3((unsigned)parts), 256, 0, st, rows, (int)cols,
               rpb, (const T*)dy, (float*)ws);
    else
      launch_k(k_colsum_partial<T>, grid, 128, 0, st, rows, cols, rpb, (const T*)dy, (float*)ws);
    NNL_CHECK_LAUNCH();
    launch_k(k_colsum_final<T>, (unsigned)((cols + 127) / 128), 128, 0, st, 
        cols, (int)parts, (const float*)ws, (T*)db, acc, nonfinite);
    NNL_CHECK_LAUNCH();
  });
  return NNL_OK;
}

}  // namespace nnl
