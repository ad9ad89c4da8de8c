// tcgen05 implicit-GEMM for Convolution / Affine (functions.py:82-214) on B200.
//
//   D[128 x BN] tile accumulates in TMEM (fp32); operands are fp16 in 128-byte
//   swizzled shared memory, 64 K-elements per stage, fed either by TMA
//   (dense matrices: 1x1/stride-1 convs, affine, im2col'ed stems) or by a
//   cp.async gather (3x3 / strided convs: zero-filled padding rows).
//
//   warp 0 lane 0 : TMA producer            warp 1 lane 0 : tcgen05.mma issuer
//   warp 2        : TMEM alloc / dealloc    warps 4..7   : gather producers,
//                                                          then the epilogue
//
//   fprop  A = x gather (K-major)   B = W[k][rsc] (K-major, TMA)
//   dgrad  A = dy gather (K-major)  B = W[ko][rs*c] (MN-major, TMA)
//   wgrad  A = dy^T (MN-major, TMA) B = x gather (MN-major)
//
// Epilogue: bias add + one RNE rounding to fp16 (R1/R4), optional accumulate
// q(prev + acc) (R2), OR of non-finite outputs, per-tile BN statistics of the
// rounded outputs, or f32 split-K partials reduced in fixed order afterwards.
#include <cuda.h>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace nnl {
using namespace tc;

enum AMode { A_TMA_K = 0, A_TMA_MN = 1, A_GATHER_FPROP = 2, A_GATHER_DGRAD = 3 };
enum BMode { B_TMA_K = 0, B_TMA_MN = 1, B_GATHER_WGRAD = 2 };

constexpr int BM = 128, BK = 64, kThreads = 256;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGES = BN == 64 ? 4 : 3;
  static constexpr int TMEM_COLS = BN;
  static constexpr int PIPE = STAGES * (A_BYTES + B_BYTES);
  // barriers + tmem slot + row metadata (128 x 16 B) + stat scratch
  static constexpr int EXTRA = 256 + 128 * 16 + 4 * BN * 2 * 4;
  static constexpr int SMEM = PIPE + EXTRA + 1024;
};

struct TcArgs {
  int M, N;
  int num_kb, kb_per_split, tiles_n;
  ConvGeom g;
  const __half* gsrc;
  int cblk;           // 64-channel blocks per tap of the gathered tensor
  int b_kblk;         // B (MN-major TMA): k-blocks per tap (dgrad) or num_kb
  int b_tap_stride;   // B column offset per tap (dgrad: C) or 0
  void* out;
  int64_t ldc;
  int acc;
  const __half* bias;
  float* stats;
  int32_t* nonfinite;
  float* partial;
};

template <int BN, int AM, int BMD>
__global__ void __launch_bounds__(kThreads, 2)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const TcArgs a) {
  using C = Cfg<BN>;
  constexpr int S = C::STAGES;
  constexpr bool kGA = AM >= A_GATHER_FPROP;
  constexpr bool kGB = BMD == B_GATHER_WGRAD;
  constexpr bool kAmn = AM == A_TMA_MN;
  constexpr bool kBmn = BMD != B_TMA_K;
  constexpr uint32_t kTmaBytes = (kGA ? 0 : C::A_BYTES) + (kGB ? 0 : C::B_BYTES);
  constexpr uint32_t IDESC = idesc_f16(BN, kAmn, kBmn);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stA = smem;
  uint8_t* stB = smem + S * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::PIPE);
  uint64_t* empty = full + S;
  uint64_t* accf = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  int64_t* row_base = reinterpret_cast<int64_t*>(smem + C::PIPE + 256);
  int* row_h = reinterpret_cast<int*>(row_base + 128);
  int* row_w = row_h + 128;
  float* red = reinterpret_cast<float*>(row_w + 128);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_n = blockIdx.x % a.tiles_n, tile_m = blockIdx.x / a.tiles_n;
  const int m0 = tile_m * BM, n0 = tile_n * BN;
  const int split = blockIdx.y;
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(kb0 + a.kb_per_split, a.num_kb);
  const int nk = kb1 - kb0;
  const ConvGeom& g = a.g;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], (kTmaBytes ? 1u : 0u) + ((kGA || kGB) ? 128u : 0u));
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    if (!kGA) tma_prefetch(&tmA);
    if (!kGB) tma_prefetch(&tmB);
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  if (kGA && threadIdx.x >= 128) {
    const int r = threadIdx.x - 128;
    const int m = m0 + r;
    if (m < a.M) {
      if (AM == A_GATHER_FPROP) {
        int q = m % g.q, t = m / g.q;
        int p = t % g.p, n = t / g.p;
        int ih0 = p * g.sh - g.ph, iw0 = q * g.sw - g.pw;
        row_h[r] = ih0;
        row_w[r] = iw0;
        row_base[r] = (((int64_t)n * g.h + ih0) * g.w + iw0) * g.c;
      } else {
        int w = m % g.w, t = m / g.w;
        int h = t % g.h, n = t / g.h;
        row_h[r] = h + g.ph;
        row_w[r] = w + g.pw;
        row_base[r] = (int64_t)n * g.p * g.q;
      }
    } else {
      row_h[r] = AM == A_GATHER_FPROP ? -(1 << 28) : -(1 << 28);
      row_w[r] = 0;
      row_base[r] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (kTmaBytes && lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        const int kb = kb0 + i;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_tx(&full[s], kTmaBytes);
        if (AM == A_TMA_K) {
          tma_load_2d(stA + s * C::A_BYTES, &tmA, &full[s], kb * BK, m0);
        } else if (AM == A_TMA_MN) {
#pragma unroll
          for (int j = 0; j < BM / 64; ++j)
            tma_load_2d(stA + s * C::A_BYTES + j * 8192, &tmA, &full[s], m0 + 64 * j, kb * BK);
        }
        if (BMD == B_TMA_K) {
          tma_load_2d(stB + s * C::B_BYTES, &tmB, &full[s], kb * BK, n0);
        } else if (BMD == B_TMA_MN) {
          const int t = kb / a.b_kblk, kob = kb - t * a.b_kblk;
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_2d(stB + s * C::B_BYTES + j * 8192, &tmB, &full[s],
                        t * a.b_tap_stride + n0 + 64 * j, kob * BK);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t ab = smem_u32(stA + s * C::A_BYTES);
        const uint32_t bb = smem_u32(stB + s * C::B_BYTES);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t da = kAmn ? sdesc_sw128(ab + kk * 2048, 8192, 1024)
                                   : sdesc_sw128(ab + kk * 32, 16, 1024);
          const uint64_t db = kBmn ? sdesc_sw128(bb + kk * 2048, 8192, 1024)
                                   : sdesc_sw128(bb + kk * 32, 16, 1024);
          mma_f16(tmem, da, db, IDESC, (i | kk) != 0);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(accf);
    }
  } else if (warp >= 4) {
    const int tid = threadIdx.x - 128;
    if (kGA || kGB) {
      constexpr int LAG = S - 1;
      const int chunk = tid & 7;
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        const int kb = kb0 + i;
        mbar_wait(&empty[s], ph ^ 1);
        if (AM == A_GATHER_FPROP) {
          const int t = kb / a.cblk, cb = kb - t * a.cblk;
          const int r = t / g.s, sx = t - r * g.s;
          const int64_t toff = ((int64_t)r * g.w + sx) * g.c + cb * 64 + chunk * 8;
          uint8_t* dst = stA + s * C::A_BYTES;
#pragma unroll
          for (int i8 = 0; i8 < 8; ++i8) {
            const int row = (tid >> 3) + 16 * i8;
            const int ih = row_h[row] + r, iw = row_w[row] + sx;
            const bool ok = (unsigned)ih < (unsigned)g.h && (unsigned)iw < (unsigned)g.w;
            const __half* src = ok ? a.gsrc + row_base[row] + toff : a.gsrc;
            cp_async16(dst + row * 128 + ((chunk ^ (row & 7)) << 4), src, ok ? 16u : 0u);
          }
        } else if (AM == A_GATHER_DGRAD) {
          const int t = kb / a.cblk, kob = kb - t * a.cblk;
          const int r = t / g.s, sx = t - r * g.s;
          uint8_t* dst = stA + s * C::A_BYTES;
#pragma unroll
          for (int i8 = 0; i8 < 8; ++i8) {
            const int row = (tid >> 3) + 16 * i8;
            int th = row_h[row] - r, tw = row_w[row] - sx;
            bool ok = th >= 0 && tw >= 0;
            int oh = th, ow = tw;
            if (g.sh != 1) {
              ok = ok && (th % g.sh == 0);
              oh = th / g.sh;
            }
            if (g.sw != 1) {
              ok = ok && (tw % g.sw == 0);
              ow = tw / g.sw;
            }
            ok = ok && oh < g.p && ow < g.q;
            const __half* src =
                ok ? a.gsrc + (row_base[row] + (int64_t)oh * g.q + ow) * g.k + kob * 64 + chunk * 8
                   : a.gsrc;
            cp_async16(dst + row * 128 + ((chunk ^ (row & 7)) << 4), src, ok ? 16u : 0u);
          }
        } else if (BMD == B_GATHER_WGRAD) {
          const int64_t npq = (int64_t)g.n * g.p * g.q;
          int64_t base[4];
          int h0[4], w0[4];
#pragma unroll
          for (int i4 = 0; i4 < 4; ++i4) {
            const int row = (tid >> 3) + 16 * i4;
            const int64_t pix = (int64_t)kb * 64 + row;
            if (pix < npq) {
              const int q = (int)(pix % g.q);
              const int64_t t = pix / g.q;
              const int p = (int)(t % g.p), n = (int)(t / g.p);
              h0[i4] = p * g.sh - g.ph;
              w0[i4] = q * g.sw - g.pw;
              base[i4] = (((int64_t)n * g.h + h0[i4]) * g.w + w0[i4]) * g.c;
            } else {
              h0[i4] = -(1 << 28);
              w0[i4] = 0;
              base[i4] = 0;
            }
          }
          const int nblk_total = (int)((int64_t)g.r * g.s * g.c / 64);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) {
            const int cbg = (n0 >> 6) + j;
            const bool colok = cbg < nblk_total;
            const int t = cbg / a.cblk, cb = cbg - t * a.cblk;
            const int r = t / g.s, sx = t - r * g.s;
            const int64_t toff = ((int64_t)r * g.w + sx) * g.c + cb * 64 + chunk * 8;
            uint8_t* dst = stB + s * C::B_BYTES + j * 8192;
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4) {
              const int row = (tid >> 3) + 16 * i4;
              const int ih = h0[i4] + r, iw = w0[i4] + sx;
              const bool ok =
                  colok && (unsigned)ih < (unsigned)g.h && (unsigned)iw < (unsigned)g.w;
              const __half* src = ok ? a.gsrc + base[i4] + toff : a.gsrc;
              cp_async16(dst + row * 128 + ((chunk ^ (row & 7)) << 4), src, ok ? 16u : 0u);
            }
          }
        }
        cp_async_commit();
        if (i >= LAG) {
          cp_async_wait<LAG>();
          fence_proxy_async();
          mbar_arrive(&full[(i - LAG) % S]);
        }
      }
      cp_async_wait<0>();
      fence_proxy_async();
      for (int i = nk > LAG ? nk - LAG : 0; i < nk; ++i) mbar_arrive(&full[i % S]);
    }

    // ---------------- epilogue ----------------
    mbar_wait(accf, 0);
    tc_fence_after();
    const int wq = warp - 4;
    const int row = wq * 32 + lane;
    const int m = m0 + row;
    const bool mv = m < a.M;
    int bad = 0;
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)c, v);
      const int nb = n0 + c;
      const bool full_cols = nb + 32 <= a.N;
      if (a.partial) {
        if (mv) {
          float* dstp = a.partial + ((int64_t)split * a.M + m) * a.N + nb;
          if (full_cols && (a.N % 4 == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(dstp + j) =
                  make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                              __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
          } else {
            for (int j = 0; j < 32; ++j)
              if (nb + j < a.N) dstp[j] = __uint_as_float(v[j]);
          }
        }
        continue;
      }
      float f[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
      if (a.bias) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (nb + j < a.N) f[j] = __fadd_rn(f[j], __half2float(a.bias[nb + j]));
      }
      __half* dsth = reinterpret_cast<__half*>(a.out) + (int64_t)m * a.ldc + nb;
      __align__(16) __half hv[32];
      const bool vec = full_cols && (a.ldc % 8 == 0);
      if (mv) {
        if (a.acc) {
          if (vec) {
#pragma unroll
            for (int j = 0; j < 32; j += 8)
              *reinterpret_cast<uint4*>(hv + j) = *reinterpret_cast<const uint4*>(dsth + j);
          } else {
            for (int j = 0; j < 32; ++j) hv[j] = nb + j < a.N ? dsth[j] : __float2half(0.f);
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) hv[j] = __float2half_rn(__fadd_rn(__half2float(hv[j]), f[j]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) hv[j] = __float2half_rn(__fadd_rn(0.f, f[j]));
        }
        if (vec) {
#pragma unroll
          for (int j = 0; j < 32; j += 8)
            *reinterpret_cast<uint4*>(dsth + j) = *reinterpret_cast<const uint4*>(hv + j);
        } else {
          for (int j = 0; j < 32; ++j)
            if (nb + j < a.N) dsth[j] = hv[j];
        }
        if (a.nonfinite) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            bad |= (nb + j < a.N) && !isfinite(__half2float(hv[j]));
        }
      }
      if (a.stats) {
        // column sums over this warp's 32 rows of the ROUNDED outputs; the
        // halving exchange leaves column (c + lane) in every lane (31 shuffles)
        float s1[32], s2[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float x = (mv && nb + j < a.N) ? __half2float(hv[j]) : 0.f;
          s1[j] = x;
          s2[j] = x * x;
        }
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) {
          const bool up = (lane & st) != 0;
#pragma unroll
          for (int j = 0; j < st; ++j) {
            float send1 = up ? s1[j] : s1[j + st], keep1 = up ? s1[j + st] : s1[j];
            float send2 = up ? s2[j] : s2[j + st], keep2 = up ? s2[j + st] : s2[j];
            s1[j] = keep1 + __shfl_xor_sync(0xffffffffu, send1, st);
            s2[j] = keep2 + __shfl_xor_sync(0xffffffffu, send2, st);
          }
        }
        red[((wq * BN) + c + lane) * 2 + 0] = s1[0];
        red[((wq * BN) + c + lane) * 2 + 1] = s2[0];
      }
    }
    if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
    if (a.stats) {
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int col = tid; col < BN; col += 128) {
        if (n0 + col >= a.N) continue;
        float t1 = 0.f, t2 = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          t1 += red[(w * BN + col) * 2 + 0];
          t2 += red[(w * BN + col) * 2 + 1];
        }
        a.stats[((int64_t)tile_m * 2 + 0) * a.N + n0 + col] = t1;
        a.stats[((int64_t)tile_m * 2 + 1) * a.N + n0 + col] = t2;
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// out[m*ldc+n] = q(prev + bias + sum_s partial[s][m][n]), fixed split order
__global__ void k_tc_splitk_reduce(int M, int N, int splits, const float* __restrict__ partial,
                                   const __half* __restrict__ bias, __half* __restrict__ out,
                                   int64_t ldc, int acc, int32_t* nonfinite) {
  int bad = 0;
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / N, n = i % N;
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + i];
    if (bias) s = __fadd_rn(s, __half2float(bias[n]));
    __half* o = out + m * ldc + n;
    const float prev = acc ? __half2float(*o) : 0.f;
    const __half h = __float2half_rn(__fadd_rn(prev, s));
    *o = h;
    bad |= !isfinite(__half2float(h));
  }
  if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
}

// explicit im2col for convolutions whose channel count is not a multiple of
// 64 (the 3-channel stem): col[m][k] = x(pixel m, tap/channel k), zero pad to kp
__global__ void k_im2col(ConvGeom g, int64_t M, int kp, const __half* __restrict__ x,
                         __half* __restrict__ col) {
  const int rsc = g.r * g.s * g.c;
  const int64_t total = M * kp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % kp);
    const int64_t m = i / kp;
    __half v = __float2half(0.f);
    if (k < rsc) {
      const int c = k % g.c, t = k / g.c;
      const int sx = t % g.s, r = t / g.s;
      const int q = (int)(m % g.q);
      const int64_t u = m / g.q;
      const int p = (int)(u % g.p), n = (int)(u / g.p);
      const int ih = p * g.sh - g.ph + r, iw = q * g.sw - g.pw + sx;
      if ((unsigned)ih < (unsigned)g.h && (unsigned)iw < (unsigned)g.w)
        v = x[(((int64_t)n * g.h + ih) * g.w + iw) * g.c + c];
    }
    col[i] = v;
  }
}

__global__ void k_pad_rows(int rows, int cols, int kp, const __half* __restrict__ src,
                           __half* __restrict__ dst) {
  const int64_t total = (int64_t)rows * kp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % kp);
    const int64_t r = i / kp;
    dst[i] = k < cols ? src[r * cols + k] : __float2half(0.f);
  }
}

// ---------------------------------------------------------------------------
// host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

struct View {  // a row-major fp16 matrix [rows][cols] with a row stride
  const void* ptr = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;
};

static int make_tmap(CUtensorMap* tm, const View& v, int box_cols, int box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(NNL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(v.ptr) & 15) || (v.ld * 2) % 16)
    return fail(NNL_ERR_UNSUPPORTED, "TMA operand not 16-byte aligned");
  cuuint64_t dims[2] = {(cuuint64_t)v.cols, (cuuint64_t)v.rows};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(v.ptr), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NNL_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return NNL_OK;
}

struct Plan {
  bool ok = false;
  int amode = 0, bmode = 0, bn = 128;
  int M = 0, N = 0, K = 0;
  View A, B;
  bool im2col = false;   // A (fprop) or B (wgrad) is an explicit im2col matrix
  int kp = 0;            // padded reduction width of the im2col matrix
  bool pad_w = false;    // fprop im2col: weights padded to [k][kp]
  int cblk = 0, b_kblk = 0, b_tap_stride = 0;
  const void* gsrc = nullptr;
  int64_t ldc = 0;
  int splits = 1, kb_per_split = 0, num_kb = 0, tiles = 0;
  size_t ws_im2col = 0, ws_wpad = 0, ws_partial = 0;
};

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

static Plan make_plan(const GemmProblem& pb) {
  Plan pl;
  const ConvGeom& g = pb.g;
  const bool one = g.r == 1 && g.s == 1 && g.sh == 1 && g.sw == 1 && g.ph == 0 && g.pw == 0;
  const int64_t npq = (int64_t)g.n * g.p * g.q, nhw = (int64_t)g.n * g.h * g.w;
  const int64_t rsc = (int64_t)g.r * g.s * g.c;
  if (g.affine) {
    if (g.ahw != 1 || g.c % 8 || g.k % 8) return pl;
    const int64_t B = g.n, I = g.c, O = g.k;
    if (pb.mode == kFprop) {  // y[B][O] = x[B][I] . W[I][O]
      pl.M = (int)B; pl.N = (int)O; pl.K = (int)I;
      pl.amode = A_TMA_K; pl.A = {pb.a, B, I, I};
      pl.bmode = B_TMA_MN; pl.B = {pb.b, I, O, O};
      pl.ldc = O;
    } else if (pb.mode == kDgrad) {  // gx[B][I] = gy[B][O] . W[I][O]^T
      pl.M = (int)B; pl.N = (int)I; pl.K = (int)O;
      pl.amode = A_TMA_K; pl.A = {pb.a, B, O, O};
      pl.bmode = B_TMA_K; pl.B = {pb.b, I, O, O};
      pl.ldc = I;
    } else {  // gW[I][O] = x[B][I]^T . gy[B][O]
      pl.M = (int)I; pl.N = (int)O; pl.K = (int)B;
      pl.amode = A_TMA_MN; pl.A = {pb.b, B, I, I};
      pl.bmode = B_TMA_MN; pl.B = {pb.a, B, O, O};
      pl.ldc = O;
    }
  } else if (pb.mode == kFprop) {
    if (g.k % 8) return pl;
    pl.M = (int)npq; pl.N = g.k; pl.ldc = g.k;
    if (g.c % 64 == 0) {
      pl.K = (int)rsc;
      pl.bmode = B_TMA_K; pl.B = {pb.b, g.k, rsc, rsc};
      if (one) {
        pl.amode = A_TMA_K; pl.A = {pb.a, nhw, g.c, g.c};
      } else {
        pl.amode = A_GATHER_FPROP; pl.gsrc = pb.a; pl.cblk = g.c / 64;
      }
    } else {
      pl.im2col = true;
      pl.kp = (int)cdiv(rsc, 64) * 64;
      pl.K = pl.kp;
      pl.pad_w = true;
      pl.amode = A_TMA_K; pl.A = {nullptr, npq, pl.kp, pl.kp};
      pl.bmode = B_TMA_K; pl.B = {nullptr, g.k, pl.kp, pl.kp};
      pl.ws_im2col = (size_t)npq * pl.kp * 2;
      pl.ws_wpad = (size_t)g.k * pl.kp * 2;
    }
  } else if (pb.mode == kDgrad) {
    if (g.k % 64 || g.c % 8) return pl;
    pl.M = (int)nhw; pl.N = g.c; pl.K = (int)(g.r * g.s * g.k); pl.ldc = g.c;
    pl.bmode = B_TMA_MN; pl.B = {pb.b, g.k, rsc, rsc};
    pl.b_kblk = g.k / 64; pl.b_tap_stride = g.c;
    if (one) {
      pl.amode = A_TMA_K; pl.A = {pb.a, npq, g.k, g.k};
    } else {
      pl.amode = A_GATHER_DGRAD; pl.gsrc = pb.a; pl.cblk = g.k / 64;
    }
  } else {  // wgrad: dW[k][rsc] = dy^T . im2col(x)
    if (g.k % 8) return pl;
    pl.M = g.k; pl.N = (int)rsc; pl.K = (int)npq; pl.ldc = rsc;
    pl.amode = A_TMA_MN; pl.A = {pb.a, npq, g.k, g.k};
    if (g.c % 64 == 0) {
      if (one) {
        pl.bmode = B_TMA_MN; pl.B = {pb.b, nhw, g.c, g.c};
      } else {
        pl.bmode = B_GATHER_WGRAD; pl.gsrc = pb.b; pl.cblk = g.c / 64;
      }
    } else {
      pl.im2col = true;
      pl.kp = (int)cdiv(rsc, 64) * 64;
      pl.bmode = B_TMA_MN; pl.B = {nullptr, npq, pl.kp, pl.kp};
      pl.ws_im2col = (size_t)npq * pl.kp * 2;
    }
  }
  if (pl.bmode == B_TMA_MN && pl.b_kblk == 0) pl.b_kblk = 1 << 30;
  // tile width: 64 when the N extent is small or not a multiple of 128
  pl.bn = (pl.N <= 64 || (pl.bmode == B_TMA_MN && pl.b_tap_stride && pl.N % 128)) ? 64 : 128;
  pl.num_kb = (int)cdiv(pl.K, BK);
  const int tiles_m = (int)cdiv(pl.M, BM), tiles_n = (int)cdiv(pl.N, pl.bn);
  pl.tiles = tiles_m * tiles_n;
  // split the reduction when the tile grid cannot fill the machine
  int splits = 1;
  if (pl.tiles < 2 * 148 && pb.stats == nullptr) {
    splits = (int)cdiv(2 * 148, pl.tiles);
    int max_by_k = pl.num_kb / 4;
    if (splits > max_by_k) splits = max_by_k;
    if (splits > 128) splits = 128;
    if (splits < 1) splits = 1;
  }
  pl.kb_per_split = (int)cdiv(pl.num_kb, splits);
  pl.splits = (int)cdiv(pl.num_kb, pl.kb_per_split);
  if (pl.splits > 1) pl.ws_partial = (size_t)pl.splits * pl.M * pl.N * 4;
  pl.ok = pl.M > 0 && pl.N > 0 && pl.K > 0;
  return pl;
}

template <int BN, int AM, int BMD>
static int launch_tc(const Plan& pl, const CUtensorMap& ta, const CUtensorMap& tb, const TcArgs& args,
                     cudaStream_t st) {
  auto kern = k_tc_gemm<BN, AM, BMD>;
  static bool attr = false;
  if (!attr) {
    NNL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  Cfg<BN>::SMEM));
    attr = true;
  }
  dim3 grid((unsigned)pl.tiles, (unsigned)pl.splits);
  kern<<<grid, kThreads, Cfg<BN>::SMEM, st>>>(ta, tb, args);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

template <int BN>
static int dispatch_bn(const Plan& pl, const CUtensorMap& ta, const CUtensorMap& tb,
                       const TcArgs& args, cudaStream_t st) {
#define NNL_TC_CASE(AM, BMD) \
  if (pl.amode == AM && pl.bmode == BMD) return launch_tc<BN, AM, BMD>(pl, ta, tb, args, st);
  NNL_TC_CASE(A_TMA_K, B_TMA_K)
  NNL_TC_CASE(A_TMA_K, B_TMA_MN)
  NNL_TC_CASE(A_TMA_MN, B_TMA_MN)
  NNL_TC_CASE(A_GATHER_FPROP, B_TMA_K)
  NNL_TC_CASE(A_GATHER_DGRAD, B_TMA_MN)
  NNL_TC_CASE(A_TMA_MN, B_GATHER_WGRAD)
#undef NNL_TC_CASE
  return fail(NNL_ERR_UNSUPPORTED, "no tcgen05 kernel for mode %d/%d", pl.amode, pl.bmode);
}

bool tc_eligible(const GemmProblem& pb, int dtype) {
  if (dtype != NNL_F16) return false;
  return make_plan(pb).ok;
}

size_t tc_ws_bytes(const GemmProblem& pb) {
  Plan pl = make_plan(pb);
  if (!pl.ok) return 0;
  return pl.ws_im2col + pl.ws_wpad + pl.ws_partial + 3 * 256;
}

int32_t tc_stat_rows(const GemmProblem& pb, int dtype) {
  if (dtype != NNL_F16) return 0;
  GemmProblem q = pb;
  float dummy;
  q.stats = &dummy;  // stats disable split-K
  Plan pl = make_plan(q);
  if (!pl.ok || pb.mode != kFprop || pb.g.affine) return 0;
  return (int32_t)cdiv(pl.M, BM);
}

static inline uint8_t* align256(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
}

int tc_gemm(const GemmProblem& pb, int dtype, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (dtype != NNL_F16) return NNL_ERR_UNSUPPORTED;
  Plan pl = make_plan(pb);
  if (!pl.ok) return NNL_ERR_UNSUPPORTED;
  if (ws_bytes < tc_ws_bytes(pb)) return fail(NNL_ERR_INVALID_ARGUMENT, "tc workspace too small");
  const ConvGeom& g = pb.g;
  uint8_t* w = align256(reinterpret_cast<uint8_t*>(ws));
  __half* col = nullptr;
  __half* wpad = nullptr;
  float* partial = nullptr;
  if (pl.ws_im2col) { col = reinterpret_cast<__half*>(w); w = align256(w + pl.ws_im2col); }
  if (pl.ws_wpad) { wpad = reinterpret_cast<__half*>(w); w = align256(w + pl.ws_wpad); }
  if (pl.ws_partial) partial = reinterpret_cast<float*>(w);
  if (pl.im2col) {
    const __half* src = reinterpret_cast<const __half*>(pb.mode == kFprop ? pb.a : pb.b);
    int64_t total = (int64_t)pl.A.rows * 0 + (int64_t)g.n * g.p * g.q * pl.kp;
    k_im2col<<<grid_for(total, 256, 148 * 16), 256, 0, st>>>(g, (int64_t)g.n * g.p * g.q, pl.kp,
                                                              src, col);
    NNL_CHECK_LAUNCH();
    if (pb.mode == kFprop) pl.A.ptr = col; else pl.B.ptr = col;
  }
  if (pl.pad_w) {
    int64_t total = (int64_t)g.k * pl.kp;
    k_pad_rows<<<grid_for(total, 256), 256, 0, st>>>(g.k, (int)(g.r * g.s * g.c), pl.kp,
                                                      reinterpret_cast<const __half*>(pb.b), wpad);
    NNL_CHECK_LAUNCH();
    pl.B.ptr = wpad;
  }
  CUtensorMap ta, tb;
  memset(&ta, 0, sizeof(ta));
  memset(&tb, 0, sizeof(tb));
  int rc;
  if (pl.amode == A_TMA_K) {
    if ((rc = make_tmap(&ta, pl.A, 64, BM))) return rc;
  } else if (pl.amode == A_TMA_MN) {
    if ((rc = make_tmap(&ta, pl.A, 64, 64))) return rc;
  }
  if (pl.bmode == B_TMA_K) {
    if ((rc = make_tmap(&tb, pl.B, 64, pl.bn))) return rc;
  } else if (pl.bmode == B_TMA_MN) {
    if ((rc = make_tmap(&tb, pl.B, 64, 64))) return rc;
  }
  TcArgs args;
  memset(&args, 0, sizeof(args));
  args.M = pl.M; args.N = pl.N; args.num_kb = pl.num_kb; args.kb_per_split = pl.kb_per_split;
  args.tiles_n = (int)cdiv(pl.N, pl.bn);
  args.g = g;
  args.gsrc = reinterpret_cast<const __half*>(pl.gsrc);
  args.cblk = pl.cblk; args.b_kblk = pl.b_kblk; args.b_tap_stride = pl.b_tap_stride;
  args.out = pb.out; args.ldc = pl.ldc; args.acc = pb.acc;
  args.bias = reinterpret_cast<const __half*>(pb.bias);
  args.stats = pb.stats; args.nonfinite = pb.nonfinite;
  args.partial = pl.splits > 1 ? partial : nullptr;
  if (pl.splits > 1) {  // bias / accumulate / rounding happen in the reduction
    args.bias = nullptr; args.acc = 0; args.nonfinite = nullptr; args.stats = nullptr;
  }
  rc = pl.bn == 64 ? dispatch_bn<64>(pl, ta, tb, args, st) : dispatch_bn<128>(pl, ta, tb, args, st);
  if (rc) return rc;
  if (pl.splits > 1) {
    k_tc_splitk_reduce<<<grid_for((int64_t)pl.M * pl.N, 256), 256, 0, st>>>(
        pl.M, pl.N, pl.splits, partial, reinterpret_cast<const __half*>(pb.bias),
        reinterpret_cast<__half*>(pb.out), pl.ldc, pb.acc, pb.nonfinite);
    NNL_CHECK_LAUNCH();
  }
  return NNL_OK;
}

}  // namespace nnl
