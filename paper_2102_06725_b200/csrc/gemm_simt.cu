// SIMT implicit GEMM: the fp32 (TypeConfig.FLOAT) path and the fallback for
// shapes the tcgen05 kernel does not take (unaligned channel counts, tiny
// affine layers).  32x32 or 64x64 tiles, register-prefetched operand tiles,
// deterministic split-K over the reduction with f32 partials.
#include <cstdlib>

#include "gemm.cuh"

namespace nnl {

// The operand element (row, k) is fetched in two halves so that the integer
// divisions of the im2col index math run once per row (kernel start) and once
// per k-tile, not once per element: Part holds a decomposed index -- a flat
// offset plus, for convolutions, a (y, x, channel) triple.
struct Part {
  int64_t off;
  int y, x, c;
};

// A(m, k): fprop x gather | dgrad dy gather | wgrad dy^T (affine: x / dy / dy^T)
template <int MODE, bool AFF>
__device__ __forceinline__ Part row_a(const GemmProblem& pb, int64_t m) {
  const ConvGeom& g = pb.g;
  Part r = {0, 0, 0, 0};
  if constexpr (AFF) {
    r.off = MODE == kWgrad ? m : m * pb.K;
  } else if constexpr (MODE == kFprop) {
    const int mi = (int)m;  // 32-bit index math (SIMT problems are < 2^31 rows)
    const int q = mi % g.q, u = mi / g.q;
    const int p = u % g.p, b = u / g.p;
    r.off = (int64_t)b * g.h * g.w * g.c;
    r.y = p * g.sh - g.ph;
    r.x = q * g.sw - g.pw;
  } else if constexpr (MODE == kDgrad) {
    const int mi = (int)m;
    const int wq = mi % g.w, u = mi / g.w;
    const int hh = u % g.h, b = u / g.h;
    r.off = (int64_t)b * g.p * g.q * g.k;
    r.y = hh + g.ph;
    r.x = wq + g.pw;
  } else {
    r.off = m;
  }
  return r;
}

template <int MODE, bool AFF>
__device__ __forceinline__ Part kpart_a(const GemmProblem& pb, int64_t k) {
  const ConvGeom& g = pb.g;
  Part r = {0, 0, 0, 0};
  if constexpr (MODE == kWgrad) {
    r.off = k * g.k;  // dy[pix = k][k_out]
  } else if constexpr (AFF) {
    r.off = k;
  } else {  // fprop k = (r, s, c); dgrad k = (r, s, ko)
    const int cc = MODE == kFprop ? g.c : g.k, ki = (int)k;
    r.c = ki % cc;
    const int t = ki / cc;
    r.x = t % g.s;
    r.y = t / g.s;
  }
  return r;
}

template <typename T, int MODE, bool AFF>
__device__ __forceinline__ float load_a(const GemmProblem& pb, const Part& row, const Part& kp) {
  const ConvGeom& g = pb.g;
  const T* a = (const T*)pb.a;
  if constexpr (AFF || MODE == kWgrad) return Elem<T>::load(a + row.off + kp.off);
  if constexpr (MODE == kFprop) {
    const int ih = row.y + kp.y, iw = row.x + kp.x;
    if ((unsigned)ih >= (unsigned)g.h || (unsigned)iw >= (unsigned)g.w) return 0.f;
    return Elem<T>::load(a + row.off + ((int64_t)ih * g.w + iw) * g.c + kp.c);
  }
  int th = row.y - kp.y, tw = row.x - kp.x;  // dgrad: output pixel that tap (r, s) maps here
  if (th < 0 || tw < 0) return 0.f;
  if (g.sh > 1) {
    if (th % g.sh) return 0.f;
    th /= g.sh;
  }
  if (g.sw > 1) {
    if (tw % g.sw) return 0.f;
    tw /= g.sw;
  }
  if (th >= g.p || tw >= g.q) return 0.f;
  return Elem<T>::load(a + row.off + ((int64_t)th * g.q + tw) * g.k + kp.c);
}

// B(n, k): fprop W[k_out][rsc] | dgrad W[ko][r][s][c] | wgrad x gather
// (affine, W stored (I,O): fprop W[row(k)][n], dgrad W[row(n)][k], wgrad x[k][n])
__device__ __forceinline__ int64_t affine_row32(const ConvGeom& g, int32_t f) {
  if (g.ahw == 1) return f;
  return (int64_t)(f % g.ac) * g.ahw + f / g.ac;
}

template <int MODE, bool AFF>
__device__ __forceinline__ Part row_b(const GemmProblem& pb, int64_t n) {
  const ConvGeom& g = pb.g;
  Part r = {0, 0, 0, 0};
  if constexpr (AFF) {
    r.off = MODE == kDgrad ? affine_row32(g, (int32_t)n) * g.k : n;
  } else if constexpr (MODE == kFprop) {
    r.off = n * pb.K;
  } else if constexpr (MODE == kDgrad) {
    r.off = n;
  } else {  // wgrad n = (r, s, c)
    const int ni = (int)n;
    r.c = ni % g.c;
    const int t = ni / g.c;
    r.x = t % g.s;
    r.y = t / g.s;
  }
  return r;
}

template <int MODE, bool AFF>
__device__ __forceinline__ Part kpart_b(const GemmProblem& pb, int64_t k) {
  const ConvGeom& g = pb.g;
  Part r = {0, 0, 0, 0};
  if constexpr (AFF) {
    r.off = MODE == kFprop ? affine_row32(g, (int32_t)k) * g.k
                              : (MODE == kDgrad ? k : k * pb.N);
  } else if constexpr (MODE == kFprop) {
    r.off = k;
  } else if constexpr (MODE == kDgrad) {  // k = (rs, ko)
    const int ki = (int)k;
    const int ko = ki % g.k, rs = ki / g.k;
    r.off = ((int64_t)ko * g.r * g.s + rs) * g.c;
  } else {  // wgrad k = (b, p, q)
    const int ki = (int)k;
    const int q = ki % g.q, u = ki / g.q;
    const int p = u % g.p, b = u / g.p;
    r.off = (int64_t)b * g.h * g.w * g.c;
    r.y = p * g.sh - g.ph;
    r.x = q * g.sw - g.pw;
  }
  return r;
}

template <typename T, int MODE, bool AFF>
__device__ __forceinline__ float load_b(const GemmProblem& pb, const Part& row, const Part& kp) {
  const ConvGeom& g = pb.g;
  const T* b = (const T*)pb.b;
  if constexpr (AFF || MODE != kWgrad) return Elem<T>::load(b + row.off + kp.off);
  const int ih = kp.y + row.y, iw = kp.x + row.x;
  if ((unsigned)ih >= (unsigned)g.h || (unsigned)iw >= (unsigned)g.w) return 0.f;
  return Elem<T>::load(b + kp.off + ((int64_t)ih * g.w + iw) * g.c + row.c);
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

// TB x TB output tile, BK = 1024 / TB reduction steps per smem tile, 256
// threads with a (TB/16) x (TB/16) micro-tile each.  The next tile's operand
// elements are fetched into registers while the current tile is multiplied
// (one global round trip per tile instead of a load -> sync -> compute chain),
// and each operand is read in the order of its contiguous dimension
// (a_kfast / b_kfast) so that a warp's loads coalesce.  Split-K (grid.z)
// writes f32 partials that k_splitk_reduce sums in fixed split order.
// bias_grad (affine wgrad): the first N-tile column also sums the rows of A
// (db[m] = sum_k A(m, k), functions.py:116) from the staged tiles.
template <typename T, int TB, int MODE, bool AFF>
__global__ void __launch_bounds__(256) k_simt_gemm(GemmProblem pb, int64_t k_per_split,
                                                  float* __restrict__ partial) {
  constexpr int BK = 1024 / TB, MT = TB / 16, PER = TB * BK / 256;
  // operand order: x[b][f] / dy[b][o] and the NHWC gathers are k-contiguous,
  // dy^T is m-contiguous; B: W[k_out][rsc] (conv fprop) and affine W[i=n][o=k]
  // (dgrad) are k-contiguous, W[ko][rs][c], x[pix][c], affine W[row(k)][n] n-contiguous
  constexpr bool a_kfast = MODE != kWgrad;
  constexpr bool b_kfast = AFF ? MODE == kDgrad : MODE == kFprop;
  __shared__ float As[2][BK][TB + 1];
  __shared__ float Bs[2][BK][TB + 1];
  pdl_wait();
  pdl_trigger();
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.x * TB, n0 = (int64_t)blockIdx.y * TB;
  const int64_t k_begin = (int64_t)blockIdx.z * k_per_split;
  int64_t k_end = k_begin + k_per_split;
  if (k_end > pb.K) k_end = pb.K;
  const bool bias_cta = pb.bias_grad && blockIdx.y == 0;
  // element i of this thread's share of a tile: A/B row index (fixed for the
  // whole kernel) and k offset within the tile
  auto a_mm = [&](int i) { const int e = threadIdx.x + 256 * i; return a_kfast ? e / BK : e % TB; };
  auto a_kk = [&](int i) { const int e = threadIdx.x + 256 * i; return a_kfast ? e % BK : e / TB; };
  auto b_mm = [&](int i) { const int e = threadIdx.x + 256 * i; return b_kfast ? e / BK : e % TB; };
  auto b_kk = [&](int i) { const int e = threadIdx.x + 256 * i; return b_kfast ? e % BK : e / TB; };
  Part rowA[PER], rowB[PER];
  bool okA[PER], okB[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    okA[i] = m0 + a_mm(i) < pb.M;
    okB[i] = n0 + b_mm(i) < pb.N;
    rowA[i] = row_a<MODE, AFF>(pb, okA[i] ? m0 + a_mm(i) : 0);
    rowB[i] = row_b<MODE, AFF>(pb, okB[i] ? n0 + b_mm(i) : 0);
  }
  float ra[PER], rb[PER];
  auto fetch = [&](int64_t k0) {
    // k-fast order: every element of this thread shares one k (one decomposition)
    Part ka = {0, 0, 0, 0}, kb = {0, 0, 0, 0};
    if constexpr (a_kfast) ka = kpart_a<MODE, AFF>(pb, min(k0 + a_kk(0), pb.K - 1));
    if constexpr (b_kfast) kb = kpart_b<MODE, AFF>(pb, min(k0 + b_kk(0), pb.K - 1));
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int64_t gka = k0 + a_kk(i), gkb = k0 + b_kk(i);
      if constexpr (!a_kfast) ka = kpart_a<MODE, AFF>(pb, min(gka, pb.K - 1));
      if constexpr (!b_kfast) kb = kpart_b<MODE, AFF>(pb, min(gkb, pb.K - 1));
      ra[i] = (okA[i] && gka < k_end) ? load_a<T, MODE, AFF>(pb, rowA[i], ka) : 0.f;
      rb[i] = (okB[i] && gkb < k_end) ? load_b<T, MODE, AFF>(pb, rowB[i], kb) : 0.f;
    }
  };
  auto stage = [&](int buf) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = threadIdx.x + 256 * i;
      As[buf][a_kfast ? e % BK : e / TB][a_kfast ? e / BK : e % TB] = ra[i];
      Bs[buf][b_kfast ? e % BK : e / TB][b_kfast ? e / BK : e % TB] = rb[i];
    }
  };
  float acc[MT][MT] = {};
  float rowsum = 0.f;
  int buf = 0;
  if (k_begin < k_end) {
    fetch(k_begin);
    stage(0);
  }
  __syncthreads();
  for (int64_t k0 = k_begin; k0 < k_end; k0 += BK) {
    const bool more = k0 + BK < k_end;
    if (more) fetch(k0 + BK);
    if (bias_cta && threadIdx.x < TB) {
#pragma unroll 8
      for (int kk = 0; kk < BK; ++kk) rowsum += As[buf][kk][threadIdx.x];
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[MT], bv[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        av[i] = As[buf][kk][ty * MT + i];
        bv[i] = Bs[buf][kk][tx * MT + i];
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < MT; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) {
      stage(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  int bad = 0;
  if (bias_cta && threadIdx.x < TB && m0 + threadIdx.x < pb.M) {
    const int64_t m = m0 + threadIdx.x;
    if (partial) {
      partial[(int64_t)gridDim.z * pb.M * pb.N + (int64_t)blockIdx.z * pb.M + m] = rowsum;
    } else {
      T* db = (T*)pb.bias_grad;
      write_out(db + m, rowsum, pb.acc_bias != 0);
      bad |= !isfinite(Elem<T>::load(db + m));
    }
  }
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    int64_t m = m0 + ty * MT + i;
    if (m >= pb.M) continue;
#pragma unroll
    for (int j = 0; j < MT; ++j) {
      int64_t n = n0 + tx * MT + j;
      if (n >= pb.N) continue;
      if (partial)
        partial[((int64_t)blockIdx.z * pb.M + m) * pb.N + n] = acc[i][j];
      else
        epilogue_store<T>(pb, m, n, acc[i][j], bad);
    }
  }
  if (pb.nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(pb.nonfinite, 1);
}

// fixed-order split-K reduction + the same epilogue (and the fused bias sums)
template <typename T>
__global__ void k_splitk_reduce(GemmProblem pb, int splits, const float* __restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  int bad = 0;
  const int64_t total = pb.M * pb.N;
  const int64_t all = total + (pb.bias_grad ? pb.M : 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < all;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    if (i < total) {
      for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + i];
      epilogue_store<T>(pb, i / pb.N, i % pb.N, s, bad);
    } else {
      const int64_t m = i - total;
      const float* pbias = partial + (int64_t)splits * total;
      for (int z = 0; z < splits; ++z) s += pbias[(int64_t)z * pb.M + m];
      T* db = (T*)pb.bias_grad;
      write_out(db + m, s, pb.acc_bias != 0);
      bad |= !isfinite(Elem<T>::load(db + m));
    }
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

// one warp per column: lane l sums parts l, l+32, ... and the 32 lane sums are
// combined by a fixed shuffle tree (deterministic; a latency chain of
// nparts/32 loads instead of nparts)
template <typename T>
__global__ void k_colsum_final(int64_t cols, int nparts, const float* __restrict__ part,
                               T* __restrict__ out, int acc, int32_t* flag) {
  pdl_wait();
  pdl_trigger();
  const int64_t col = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  int bad = 0;
  double s = 0.0;
  if (col < cols)
    for (int i = lane; i < nparts; i += 32) s += (double)part[(int64_t)i * cols + col];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (col < cols && lane == 0) {
    write_out(out + col, (float)s, acc != 0);
    bad = !isfinite(Elem<T>::load(out + col));
  }
  if (flag && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// small problems (most of the fp32 / narrow-channel path: C1, C2) are
// latency bound: 32-wide tiles and split-K until ~2 CTAs per SM are busy
// NNL_SIMT_TB (32 | 64) / NNL_SIMT_SPLITS (cap) override the choices (probes)
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && e[0] ? atoi(e) : dflt;
}

static int simt_tile(const GemmProblem& pb) {
  static const int forced = env_int("NNL_SIMT_TB", 0);
  if (forced == 32 || forced == 64) return forced;
  const int64_t tiles64 = ((pb.M + 63) / 64) * ((pb.N + 63) / 64);
  return tiles64 >= 2 * 148 ? 64 : 32;
}

static int simt_splits(const GemmProblem& pb) {
  const int tb = simt_tile(pb), bk = 1024 / tb;
  const int64_t tiles = ((pb.M + tb - 1) / tb) * ((pb.N + tb - 1) / tb);
  int64_t want = (2 * 148 + tiles - 1) / tiles;
  const int64_t max_by_k = (pb.K + 2 * bk - 1) / (2 * bk);  // >= 2 smem tiles per split
  if (want > max_by_k) want = max_by_k;
  static const int cap = env_int("NNL_SIMT_SPLITS", 64);
  if (want > cap) want = cap;
  if (want > 64) want = 64;
  if (want < 1) want = 1;
  return (int)want;
}

static size_t simt_partial_floats(const GemmProblem& pb, int sp) {
  return (size_t)sp * pb.M * pb.N + (pb.bias_grad ? (size_t)sp * pb.M : 0);
}

size_t simt_ws_bytes(const GemmProblem& pb) {
  int sp = simt_splits(pb);
  // the bias-sum partials are sized for the largest M the same problem can ask
  GemmProblem q = pb;
  q.bias_grad = (void*)1;
  return sp > 1 ? simt_partial_floats(q, sp) * sizeof(float) : 0;
}

using SimtKernel = void (*)(GemmProblem, int64_t, float*);

template <typename T, int TB>
static SimtKernel simt_kernel_tb(int mode, bool affine) {
  if (affine)
    return mode == kFprop ? k_simt_gemm<T, TB, kFprop, true>
         : mode == kDgrad ? k_simt_gemm<T, TB, kDgrad, true> : k_simt_gemm<T, TB, kWgrad, true>;
  return mode == kFprop ? k_simt_gemm<T, TB, kFprop, false>
       : mode == kDgrad ? k_simt_gemm<T, TB, kDgrad, false> : k_simt_gemm<T, TB, kWgrad, false>;
}

template <typename T>
static SimtKernel simt_kernel(int tb, int mode, bool affine) {
  return tb == 64 ? simt_kernel_tb<T, 64>(mode, affine) : simt_kernel_tb<T, 32>(mode, affine);
}

int simt_gemm(const GemmProblem& pb, int dtype, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (pb.M >= INT32_MAX || pb.N >= INT32_MAX || pb.K >= INT32_MAX)
    return fail(NNL_ERR_UNSUPPORTED, "SIMT GEMM extents must be < 2^31");
  const int tb = simt_tile(pb), bk = 1024 / tb;
  int sp = simt_splits(pb);
  if (sp > 1 && ws_bytes < simt_partial_floats(pb, sp) * sizeof(float)) sp = 1;
  int64_t kps = (pb.K + sp - 1) / sp;
  kps = (kps + bk - 1) / bk * bk;
  if (kps < bk) kps = bk;
  sp = (int)((pb.K + kps - 1) / kps);
  if (sp < 1) sp = 1;
  dim3 grid((unsigned)((pb.M + tb - 1) / tb), (unsigned)((pb.N + tb - 1) / tb), (unsigned)sp);
  float* partial = sp > 1 ? (float*)ws : nullptr;
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(simt_kernel<T>(tb, pb.mode, pb.g.affine != 0), grid, 256, 0, st, pb, kps, partial);
    NNL_CHECK_LAUNCH();
    if (partial) {
      const int64_t outs = pb.M * pb.N + (pb.bias_grad ? pb.M : 0);
      launch_k(k_splitk_reduce<T>, grid_for(outs, 256), 256, 0, st, pb, sp, partial);
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
    launch_k(k_colsum_final<T>, (unsigned)((cols + 7) / 8), 256, 0, st,
        cols, (int)parts, (const float*)ws, (T*)db, acc, nonfinite);
    NNL_CHECK_LAUNCH();
  });
  return NNL_OK;
}

}  // namespace nnl
