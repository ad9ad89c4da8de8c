// Weight gradient of the 3x3 / stride-1 / pad-1 convolutions (functions.py:
// 196-206: gW = sum over (b, p, q) of dy x im2col(x)) with shared halos.
//
//   dW[k][r][s][c] = sum_pix dy[pix][k] * x[pix + (r - 1, s - 1)][c]
//
// The general wgrad path loads im2col(x) per filter tap, i.e. every input pixel
// crosses L2 -> SMEM nine times (the measured bound of that kernel).  Here the
// reduction runs over (8 x 8)-pixel tiles of dy, and for each tile ONE TMA box
// brings the (10 x 10)-pixel input halo of a 64-channel block into shared
// memory; the nine taps are nine descriptor views into it:
//
//   GEMM D[m = (tap, c)][n = k_out] += A[m][pix] * B[n][pix]
//   A = x halo views  (MN-major: channels contiguous, one 128 B row per pixel;
//                      the view of tap (r, s) starts (r * 10 + s) rows in; the
//                      8-pixel K groups of a view are image rows, SBO = 10 rows)
//   B = the dy tile   (MN-major: 64 output channels per 128 B pixel row)
//
// An M tile of 128 rows is a PAIR of taps (2j, 2j + 1): its two 64-row halves
// are the two taps' views, LBO apart -- so one CTA accumulates all nine taps
// (five 128 x 64 accumulators, 320 TMEM columns) from each halo.  The 128 B
// swizzle follows the absolute shared-memory address as the TMA wrote it, so
// views may start at any 128 B row (as for the fprop halo tiles, gemm_tc.cu).
//
// Work units are (channel block, output-channel block, split of the pixel
// tiles); splits write f32 partials [split][k][9c] that the fixed-order split
// reduction of gemm_tc.cu folds into one RNE rounding (R4), so the result does
// not depend on the schedule.
#include <cuda.h>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace nnl {
using namespace tc;

namespace {

constexpr int kPitch = 10;                       // halo row pitch (pixels)
constexpr int kHaloBytes = kPitch * 10 * 128;    // 12800
constexpr int kHaloStage = 13312;                // 1024-aligned
constexpr int kDyBytes = 64 * 128;               // 8 x 8 pixels x 64 channels
constexpr int kStageBytes = kHaloStage + 2 * kDyBytes;  // room for 128 output channels
constexpr int kStages = 6;
constexpr int kMT = 5;                           // tap-pair M tiles
constexpr int kTmemCols = 512;                   // 5 x 64 used
constexpr int kThreads = 256;
constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

struct W3Args {
  int c, k;              // channels of x / dy
  int tw, th, tiles;     // 8 x 8 tile grid per image, tiles in all
  int cblk, nblk;        // c / 64, k / 64
  int splits, tps;       // pixel-tile splits, tiles per split
  int units;
  int ntap;              // filter taps (9 for 3x3; 4 for the stem's 4x1 over x4)
  int ngroups;           // tap-pair M tiles split into groups (one pass each): NB = 128
  uint8_t mt0[3], mt1[3];  // group g covers tap-pair M tiles [mt0[g], mt1[g])
  uint16_t toff[16];     // tap t's view: toff[t] 128 B rows into the halo
  int hx, hy;            // halo box origin relative to the tile origin
  uint32_t halo_bytes;
  int hbw;               // halo box width (pixels) = its row pitch
  int64_t ld;            // row length of dW / the partials: ntap * c
  float* partial;        // [splits][k][ld] when splits > 1 (or force_partial)
  int force_partial;
  __half* out;           // dW [k][taps][c]
  int acc;
  int32_t* nonfinite;
  int dbg;               // probes (NNL_WG3_DBG): 1 = no MMAs, 2 = no operand loads
};

__device__ __forceinline__ void decode(const W3Args& a, int u, int& cb, int& nb, int& sp,
                                       int& grp) {
  // consecutive units share the pixel tiles (L2 reuse of x halos and dy tiles)
  grp = u % a.ngroups;
  u /= a.ngroups;
  cb = u % a.cblk;
  const int t = u / a.cblk;
  nb = t % a.nblk;
  sp = t / a.nblk;
}

}  // namespace

// NB output channels per unit (64, or 128 with the tap pairs split into two
// passes so that the accumulators fit the 512 TMEM columns)
template <int NB>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_wgrad3(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDy,
                const W3Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmDy);
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  pdl_wait();
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int per_img = a.tw * a.th;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        int cb, nb, sp, grp;
        decode(a, u, cb, nb, sp, grp);
        const int t0 = sp * a.tps, t1 = min(t0 + a.tps, a.tiles);
        for (int t = t0; t < t1; ++t, ++it) {
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          if (a.dbg & 2) {
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_arrive_tx(&full[s], a.halo_bytes + (NB / 64) * kDyBytes);
          const int img = t / per_img, r = t - img * per_img;
          const int ty = r / a.tw, tx = r - ty * a.tw;
          uint8_t* st = smem + s * kStageBytes;
          // the tile's input halo, 64 channels; out-of-image pixels read as zero
          // (the padding)
          tma_load_4d(st, &tmX, &full[s], cb * 64, tx * 8 + a.hx, ty * 8 + a.hy, img);
          // (8 x 8) dy tile; pixels past the image edge read as zero (no contribution)
#pragma unroll
          for (int h = 0; h < NB / 64; ++h)
            tma_load_4d(st + kHaloStage + h * kDyBytes, &tmDy, &full[s], nb * NB + 64 * h, tx * 8,
                        ty * 8, img);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t IDESC = idesc_f16(NB, true, true, 128);
    // all 24 descriptors of stage 0 built once (the issuing thread is otherwise
    // the bottleneck: ~10 integer ops per descriptor against a 48-cycle MMA);
    // stage s adds s * kStageBytes / 16 to the start-address field (< 2^14)
    const uint32_t base0 = smem_u32(smem);
    const uint32_t pitch = a.hbw;  // halo row pitch in pixels = the box width
    uint64_t dA[kMT][4], dB[4];
#pragma unroll
    for (int j = 0; j < kMT; ++j) {
      const int ta = min(2 * j, a.ntap - 1), tb = 2 * j + 1 < a.ntap ? 2 * j + 1 : ta;
      const uint32_t oa = (uint32_t)a.toff[ta] * 128, ob = (uint32_t)a.toff[tb] * 128;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)  // 16 pixels = tile rows 2kk, 2kk + 1
        dA[j][kk] = sdesc_sw128(base0 + oa + kk * 2 * pitch * 128, ob - oa, pitch * 128);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)  // MN-major dy tile: 64-channel chunks kDyBytes apart
      dB[kk] = sdesc_sw128(base0 + kHaloStage + (uint32_t)(kk * 2048), kDyBytes, 1024);
    int it = 0, ut = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++ut) {
      int cb, nb, sp, grp;
      decode(a, u, cb, nb, sp, grp);
      const int jlo = a.mt0[grp], jhi = a.mt1[grp];
      const int t0 = sp * a.tps, t1 = min(t0 + a.tps, a.tiles);
      mbar_wait(tempty, (ut & 1) ^ 1);
      tc_fence_after();
      for (int t = t0; t < t1; ++t, ++it) {
        const int s = it % kStages;
        mbar_wait(&full[s], (it / kStages) & 1);
        tc_fence_after();
        if (a.dbg == 1) {
          if (elect_one()) mbar_arrive(&empty[s]);
        } else if (elect_one()) {
          const uint64_t so = (uint64_t)((uint32_t)(s * kStageBytes) >> 4);
          const uint32_t acc0 = t > t0 ? 1u : 0u;
#pragma unroll
          for (int j = 0; j < kMT; ++j) {
            if (j < jlo || j >= jhi) continue;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_f16(tmem + (uint32_t)((j - jlo) * NB), dA[j][kk] + so, dB[kk] + so, IDESC,
                      kk ? 1u : acc0);
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(tfull);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int wq = warp - 4;  // TMEM lane quadrant
    const int64_t ld = a.ld;
    const bool to_partial = a.splits > 1 || a.force_partial;
    int ut = 0;
    int bad = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++ut) {
      int cb, nb, sp, grp;
      decode(a, u, cb, nb, sp, grp);
      mbar_wait(tfull, ut & 1);
      tc_fence_after();
      const int row = wq * 32 + lane;  // M row of each tap-pair tile
      const int c = cb * 64 + (row & 63);
#pragma unroll 1
      for (int j = a.mt0[grp]; j < a.mt1[grp]; ++j) {
        const int tap = 2 * j + (row >> 6);
#pragma unroll
        for (int h = 0; h < NB / 32; ++h) {
          uint32_t v[32];
          tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) +
                        (uint32_t)((j - a.mt0[grp]) * NB + h * 32), v);
          if (tap >= a.ntap) continue;
          const int n0 = nb * NB + h * 32;
          if (to_partial) {
            float* p = a.partial + ((int64_t)sp * a.k + n0) * ld + (int64_t)tap * a.c + c;
#pragma unroll
            for (int e = 0; e < 32; ++e) p[e * ld] = __uint_as_float(v[e]);
          } else {
            __half* o = a.out + (int64_t)n0 * ld + (int64_t)tap * a.c + c;
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const float prev = a.acc ? __half2float(o[e * ld]) : 0.f;
              const __half q = __float2half_rn(__fadd_rn(prev, __uint_as_float(v[e])));
              o[e * ld] = q;
              bad |= !isfinite(__half2float(q));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
    if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int tmap_nhwc(CUtensorMap* tm, const void* p, int c, int w, int h, int n, int bw, int bh) {
  static EncodeTiledFn enc = nullptr;
  if (!enc) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(NNL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    enc = reinterpret_cast<EncodeTiledFn>(fp);
  }
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(p), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NNL_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return NNL_OK;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct W3Plan {
  bool ok = false;
  int tw, th, tiles, cblk, nblk, splits, tps, units;
  int nb = 64, ngroups = 1;  // output block width; tap-pair groups (passes)
};

// NNL_WG3_NB=64 keeps 64-wide output blocks for every layer (probes)
int w3_nb128() {
  static int e = -1;
  if (e < 0) {
    const char* s = getenv("NNL_WG3_NB");
    e = (s && atoi(s) == 64) ? 0 : 1;
  }
  return e;
}

W3Plan plan_w3(const GemmProblem& pb) {
  W3Plan p;
  const ConvGeom& g = pb.g;
  if (pb.mode != kWgrad || g.affine || g.r != 3 || g.s != 3 || g.sh != 1 || g.sw != 1 ||
      g.ph != 1 || g.pw != 1 || g.p != g.h || g.q != g.w || g.c % 64 || g.k % 64 ||
      g.c > 4096 || g.k > 4096 || g.n <= 0)
    return p;
  // 8 x 8 tiles over a 7 x 7 map carry 30 % padding (and the halo 2x the input
  // pixels): the per-tap im2col path is as fast there (measured at 512 ch)
  static const int min_hw = getenv("NNL_WG3_MINHW") ? atoi(getenv("NNL_WG3_MINHW")) : 14;
  if (g.h < min_hw || g.w < min_hw) return p;
  if ((reinterpret_cast<uintptr_t>(pb.a) & 15) || (reinterpret_cast<uintptr_t>(pb.b) & 15))
    return p;
  p.tw = (g.w + 7) / 8;
  p.th = (g.h + 7) / 8;
  p.tiles = g.n * p.tw * p.th;
  p.cblk = g.c / 64;
  // 128 output channels per unit when they exist: the N = 128 MMA does twice
  // the work of N = 64 in 64 instead of 48 cycles (tools/mma_probe.cu); the
  // nine taps' 128-wide accumulators need two passes (tap pairs 0-2, 3-4) to
  // fit the 512 TMEM columns
  if (g.k % 128 == 0 && w3_nb128()) {
    p.nb = 128;
    p.ngroups = 2;
  }
  p.nblk = g.k / p.nb;
  const int pairs = p.ngroups * p.cblk * p.nblk, sms = sm_count();
  // one unit per CTA where the (channel block, output block) pairs leave room:
  // splits of the pixel tiles up to the SM count, at least 8 tiles each
  int splits = pairs >= sms ? 1 : sms / pairs;
  if (splits > p.tiles / 8) splits = p.tiles / 8;
  if (splits < 1) splits = 1;
  p.tps = (p.tiles + splits - 1) / splits;
  p.splits = (p.tiles + p.tps - 1) / p.tps;
  p.units = pairs * p.splits;
  p.ok = true;
  return p;
}

int w3_enabled() {
  static int e = -1;
  if (e < 0) {
    const char* s = getenv("NNL_WG3");
    e = (s && s[0] == '0') ? 0 : 1;
  }
  return e;
}

}  // namespace

size_t wgrad3_ws_bytes(const GemmProblem& pb) {
  if (!w3_enabled()) return 0;
  W3Plan p = plan_w3(pb);
  if (!p.ok || p.splits <= 1) return 0;
  return (size_t)p.splits * pb.g.k * 9 * pb.g.c * sizeof(float) + 256;
}

bool wgrad3_eligible(const GemmProblem& pb, int dtype) {
  return dtype == NNL_F16 && w3_enabled() && plan_w3(pb).ok;
}

template <int NB>
static int launch_w3_nb(const CUtensorMap& tx, const CUtensorMap& tdy, const W3Args& a,
                        cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    NNL_CUDA(cudaFuncSetAttribute(k_tc_wgrad3<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmem));
    attr = true;
  }
  static const int cap = getenv("NNL_WG_MAXGRID") ? atoi(getenv("NNL_WG_MAXGRID")) : 0;
  int grid = a.units < sm_count() ? a.units : sm_count();
  if (cap > 0 && grid > cap) grid = cap;
  launch_k(k_tc_wgrad3<NB>, dim3((unsigned)grid), dim3(kThreads), (size_t)kSmem, st, tx, tdy, a);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

static int launch_w3(const CUtensorMap& tx, const CUtensorMap& tdy, const W3Args& a, int nb,
                     cudaStream_t st) {
  return nb == 128 ? launch_w3_nb<128>(tx, tdy, a, st) : launch_w3_nb<64>(tx, tdy, a, st);
}

static W3Args base_args(const W3Plan& p, int c, int k) {
  W3Args a = {};
  a.c = c; a.k = k;
  a.tw = p.tw; a.th = p.th; a.tiles = p.tiles;
  a.cblk = p.cblk; a.nblk = p.nblk;
  a.splits = p.splits; a.tps = p.tps; a.units = p.units;
  a.ngroups = p.ngroups;
  const int mt = kMT;  // tap-pair M tiles of a 3x3 filter (set per caller below)
  if (p.ngroups == 2) {
    a.mt0[0] = 0; a.mt1[0] = 3;
    a.mt0[1] = 3; a.mt1[1] = (uint8_t)mt;
  } else {
    a.mt0[0] = 0; a.mt1[0] = (uint8_t)mt;
  }
  static const int dbg = getenv("NNL_WG3_DBG") ? atoi(getenv("NNL_WG3_DBG")) : 0;
  a.dbg = dbg;
  return a;
}

int wgrad3_run(const GemmProblem& pb, void* ws, size_t ws_bytes, cudaStream_t st) {
  W3Plan p = plan_w3(pb);
  if (!p.ok) return NNL_ERR_UNSUPPORTED;
  const ConvGeom& g = pb.g;
  if (ws_bytes < wgrad3_ws_bytes(pb)) return fail(NNL_ERR_INVALID_ARGUMENT, "wgrad3 workspace too small");
  CUtensorMap tx, tdy;
  memset(&tx, 0, sizeof(tx));
  memset(&tdy, 0, sizeof(tdy));
  int rc = tmap_nhwc(&tx, pb.b, g.c, g.w, g.h, g.n, kPitch, 10);
  if (rc) return rc;
  if ((rc = tmap_nhwc(&tdy, pb.a, g.k, g.q, g.p, g.n, 8, 8))) return rc;
  W3Args a = base_args(p, g.c, g.k);
  a.ntap = 9;
  for (int t = 0; t < 9; ++t) a.toff[t] = (uint16_t)((t / 3) * kPitch + t % 3);
  a.hx = -1; a.hy = -1;  // pad 1
  a.hbw = kPitch;
  a.halo_bytes = kHaloBytes;
  a.ld = 9LL * g.c;
  float* partial = nullptr;
  if (p.splits > 1)
    partial = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  a.partial = partial;
  a.out = reinterpret_cast<__half*>(pb.out);
  a.acc = pb.acc;
  a.nonfinite = p.splits > 1 ? nullptr : pb.nonfinite;
  if ((rc = launch_w3(tx, tdy, a, p.nb, st))) return rc;
  if (p.splits > 1)
    return tc_splitk_reduce(g.k, 9 * g.c, p.splits, partial, reinterpret_cast<__half*>(pb.out),
                            9LL * g.c, pb.acc, pb.nonfinite, st);
  return NNL_OK;
}

// The stem's weight gradient over its space-to-depth copy x4[n][p + r2 - 1][q][64]
// (gemm_tc.cu s2d_layout: an r2 x 1 convolution over 64 channels): the same
// halo kernel with r2 vertical taps, halo = 8 x (8 + r2 - 1) x4 pixels (rows
// 8 pixels apart, so a tap view starts 8 r rows in).  Writes f32 partials
// [splits][k][r2 * 64] (at most max_splits) for the caller's column-mapping
// reduction; returns the split count used in *splits.
int wgrad_halo_x4(const void* x4, const void* dy, int n, int p, int q, int k, int r2,
                  float* partial, int max_splits, int* splits, cudaStream_t st) {
  if (!w3_enabled() || q % 8 || k % 64 || r2 < 1 || r2 > 6 || max_splits < 1 ||
      (reinterpret_cast<uintptr_t>(x4) & 15) || (reinterpret_cast<uintptr_t>(dy) & 15))
    return NNL_ERR_UNSUPPORTED;
  W3Plan pl;
  pl.tw = q / 8;
  pl.th = (p + 7) / 8;
  pl.tiles = n * pl.tw * pl.th;
  pl.cblk = 1;
  pl.nblk = k / 64;
  int sp = sm_count() / pl.nblk;
  if (sp > pl.tiles / 8) sp = pl.tiles / 8;
  if (sp > max_splits) sp = max_splits;
  if (sp < 1) sp = 1;
  pl.tps = (pl.tiles + sp - 1) / sp;
  pl.splits = (pl.tiles + pl.tps - 1) / pl.tps;
  pl.units = pl.nblk * pl.splits;
  pl.ok = true;
  CUtensorMap tx, tdy;
  memset(&tx, 0, sizeof(tx));
  memset(&tdy, 0, sizeof(tdy));
  int rc = tmap_nhwc(&tx, x4, 64, q, p + r2 - 1, n, 8, 8 + r2 - 1);
  if (rc) return rc;
  if ((rc = tmap_nhwc(&tdy, dy, k, q, p, n, 8, 8))) return rc;
  W3Args a = base_args(pl, 64, k);
  a.mt1[0] = (uint8_t)((r2 + 1) / 2);
  a.ntap = r2;
  for (int t = 0; t < r2; ++t) a.toff[t] = (uint16_t)(t * 8);
  a.hx = 0; a.hy = 0;  // x4 rows are already shifted by the padding
  a.hbw = 8;
  a.halo_bytes = (uint32_t)(8 * (8 + r2 - 1) * 128);
  a.ld = (int64_t)r2 * 64;
  a.partial = partial;
  a.force_partial = 1;
  a.out = nullptr;
  a.nonfinite = nullptr;
  *splits = pl.splits;
  return launch_w3(tx, tdy, a, 64, st);
}

}  // namespace nnl
