// tcgen05 implicit-GEMM for Convolution / Affine (functions.py:82-214) on B200.
//
// Persistent, warp-specialised kernel (one CTA per SM, 384 threads):
//
//   warp 0 lane 0 : TMA producer              warp 1 lane 0 : tcgen05.mma issuer
//   warp 2        : TMEM alloc / dealloc      warp 3        : idle
//   warps 4..7    : cp.async gather producers (3x3 / strided convolutions)
//   warps 8..11   : epilogue (TMEM -> registers -> global)
//
// Each CTA walks work units (m-tile, n-tile, k-split) with stride gridDim.x.
// Operands are fp16 in 128-byte swizzled shared memory, 64 K-elements per
// stage, in a ring of STAGES buffers (full/empty mbarriers).  The fp32
// accumulator of a 128 x BN tile lives in TMEM; two accumulator buffers let
// the epilogue of tile t overlap the mainloop of tile t+1 (tmem_full /
// tmem_empty mbarriers).
//
//   fprop  A = x gather / TMA (K-major)   B = W[k][rsc]  (K-major, TMA)
//   dgrad  A = dy gather / TMA (K-major)  B = W[ko][rs*c] (MN-major, TMA)
//   wgrad  A = dy^T (MN-major, TMA)       B = x gather / TMA (MN-major)
//
// Epilogue: bias add + one RNE rounding to fp16 (R1/R4), optional accumulate
// q(prev + acc) (R2), OR of non-finite outputs, per-tile BN statistics of the
// rounded outputs, an output-row remap (1x1 stride-2 dgrad), or f32 split-K
// partials reduced in fixed order afterwards.
#include <cuda.h>

#include <cstdlib>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace nnl {
using namespace tc;

// A_IM2COL / B_IM2COL: TMA im2col mode (fprop + stride-1 dgrad A, wgrad B);
// the cp.async gathers remain for strided dgrad and as a debug path.
// A_GATHER_C4 / B_GATHER_C4: narrow-channel convolutions (the 3-channel stem)
// over a 4-channel padded copy of x, reduction index k = tap*4 + c, 16 taps per
// 64-wide k-block, gathered as 8 B pieces.
// A_IM2COL16 / B_IM2COL16: stride-2 narrow-channel convolutions (the stem)
// rewritten by space-to-depth as a stride-1 convolution over a 16-channel
// tensor; TMA im2col with 32-byte rows, one 16-wide K step per filter tap.
// A_TILE4 / A_TILE4MN / B_TILE4: spatial tiles.  A 128-row M tile (or a
// 64-pixel wgrad k-block) is a (bw x bh x bi) block of output pixels, and each
// filter tap's operand tile is ONE tiled 4D TMA box of the NHWC input shifted
// by the tap offset (out-of-range coordinates read as zero = the padding):
// plain tiled loads instead of per-pixel im2col rows (stride-1 convolutions
// whose grid the box tiles exactly).
enum AMode {
  A_TMA_K = 0, A_TMA_MN = 1, A_GATHER_FPROP = 2, A_GATHER_DGRAD = 3, A_IM2COL = 4,
  A_GATHER_C4 = 5, A_IM2COL16 = 6, A_TILE4 = 7, A_TILE4MN = 8, A_HALO = 9
};
// A_HALO: stride-1 convolutions over 64 channels (one channel block) -- the 3x3
// pad-1 layers and the stem's 4x1 convolution over x4: the (8 x 16)-pixel M tile's
// input halo (3x3: 10 x 18 pixels, a 10-pixel row pitch; stem: 8 x 19)
// is ONE tiled 4D TMA box per tile, and the nine taps are nine descriptor views
// into it (view (r, s) starts at halo pixel r*10 + s: SBO 1280 B, no base offset),
// so each input pixel crosses L2 -> SMEM once per tile instead of once per tap.
enum BMode {
  B_TMA_K = 0, B_TMA_MN = 1, B_GATHER_WGRAD = 2, B_IM2COL = 3, B_GATHER_C4 = 4, B_IM2COL16 = 5,
  B_TILE4 = 6
};

constexpr int BM = 128, BK = 64, kThreads = 384;

// CG = 2: a CTA pair (cluster of 2) computes a 256 x BN tile with
// tcgen05.mma.cta_group::2; each CTA holds its 128 rows of A and BN/2 columns
// of B, so one k-step moves (256 + BN) x 64 operand elements through L2 for
// 2 x 128 x BN outputs instead of 2 x (128 + BN) x 64.
// RB = 1: the whole B operand (all k-blocks of a single-N-tile GEMM, <= RES_MAX
// bytes) stays resident in shared memory for the CTA's lifetime; the ring then
// streams A only (weight-stationary narrow convolutions).
constexpr int RES_MAX = 64 * 1024;

// EP = 1 (fused BN-backward epilogue): each of the 8 epilogue warps keeps two
// 6 KB sets of TMA-loaded input tiles (x, gate, prev: 32 rows x 32 columns each)
template <int BN, int CG = 1, int RB = 0, int EP = 0, int HL = 0>
struct Cfg {
  // A_HALO: one halo box per stage -- 3x3: 18 rows x 10-pixel pitch, stem: 19 x 8 --
  // rounded up to the 1 KB swizzle-atom alignment of the next stage
  static constexpr int A_BYTES = HL ? (18 * 10 * 128 + 1023) / 1024 * 1024 : BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;  // this CTA's share of B
  static constexpr int STAGE_B = RB ? 0 : B_BYTES;      // B bytes per ring stage
  static constexpr int RES_BYTES = RB ? (HL ? 9 * B_BYTES : RES_MAX) : 0;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int RED_BYTES = 4 * BN * 2 * 4;
  static constexpr int BIAS_BYTES = BN * 4 * 5;  // bias + the fused BN-backward constants
  static constexpr int MAX_STAT_N = HL ? 64 : 2048;  // per-CTA BN statistics [2][N]
  static constexpr int STAT_BYTES = 2 * MAX_STAT_N * 4;
  // TMA-store staging: 8 x 4 KB (4 warps x 2 buffers, or 8 warps x 1)
  static constexpr int STG_BYTES = EP ? 8 * 2 * 6144 : (RB ? 8 * 2 * 4096 : 4 * 2 * 4096);
  static constexpr int FIXED =
      1024 + RED_BYTES + BIAS_BYTES + STAT_BYTES + STG_BYTES + 1024 + RES_BYTES;
  static constexpr int BUDGET = 232448;
  static constexpr int STAGES_FIT = (BUDGET - FIXED) / (A_BYTES + STAGE_B);
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int PIPE = STAGES * (A_BYTES + STAGE_B);
  static constexpr int SMEM = PIPE + FIXED;
  static_assert(STAGES >= 3 || (HL && STAGES >= 2), "pipeline too shallow");
};

// tensor maps of the fused BN-backward epilogue (EP = 1): the BN input x, the
// residual gate and the gated-gradient destination, 32 x 32 boxes, 64 B swizzle
struct EpiMaps {
  CUtensorMap x, g, o;
};

// n / d for 0 <= n < 2^31 as (umulhi(n, m) + n) >> s (Granlund-Montgomery with a
// rounded-up multiplier): the per-tile index math of the epilogue and the
// producers without the ~20-instruction runtime integer division
struct FDiv {
  uint32_t m, s;
};
__device__ __forceinline__ int fdiv(int n, FDiv d) {
  return (int)((__umulhi((uint32_t)n, d.m) + (uint32_t)n) >> d.s);
}

struct TcArgs {
  int64_t K;          // reduction length (B_GATHER_C4: pixels)
  // narrow-channel gathers: x4 is [n][h][c4_w4][4] with image column w at
  // c4_w4 column w + c4_off; reduction index k = (r * c4_s2 + s) * 4 + c
  int c4_s2, c4_w4, c4_off, c4_pair;
  int M, N;
  int num_kb, kb_per_split;
  int tiles_m, tiles_n, units;
  ConvGeom g;
  const __half* gsrc;
  int cblk;           // 64-channel blocks per tap of the gathered tensor
  int b_kblk;         // B (MN-major TMA): k-blocks per tap (dgrad) or "infinite"
  int b_tap_stride;   // B column offset per tap (dgrad: C) or 0
  void* out;
  int64_t ldc;
  int acc;
  int remap;          // output row m=(n,y,x) of an (rgh x rgw) grid -> dx pixel
  int rgh, rgw, rsh, rsw, ra, rb;  //   (n, y*rsh + ra, x*rsw + rb) of the H x W map
  // strided-dgrad parity class: k-block tap t uses im2col offsets tap_offw/h[t]
  // and weight tap tap_w[t] (ntap == 0: taps come from t = r*S + s)
  int ntap;
  uint8_t tap_w[16], tap_offw[16], tap_offh[16];
  // im2col TMA: GEMM rows (A) / reduction rows (B) enumerate an (gh x gw)
  // pixel grid per image; pixel (y, x) has window base (y*ish + ilh, x*isw + ilw)
  int gh, gw, ish, isw, ilh, ilw;
  int flip;           // dgrad: tap t of the im2col load uses weight tap R*S-1-t
  const __half* bias;
  float* stats;
  const float* stat_shift;  // per-column centre K of the fprop BN statistics (nullable)
  int32_t* nonfinite;
  float* partial;
  int tma_store;      // epilogue writes through the output tensor map (tmC)
  // spatial tiles (A_TILE4*, B_TILE4): box (sbw x sbh x sbi) pixels, tile grid
  // stw x sth (x fastest, then y, then image), sp_tiles boxes in all; tap
  // (r, s) of a box at (x0, y0, n0) reads input (x0 + s + slw, y0 + r + slh, n0);
  // the epilogue's output grid is sgw x sgh (A_TILE4: rows -> pixels, 4D store)
  int sbw, sbh, sbi, stw, sth, sp_tiles, slw, slh, sgw, sgh;
  int res_kb;         // resident-B k-blocks when they differ from num_kb (A_HALO: taps)
  int hl_pitch, hl_r, hl_s;  // A_HALO: halo row pitch (pixels) and filter taps R x S
  uint32_t hl_bytes;  // A_HALO: bytes of one halo box
  // fused BatchNormalization backward statistics (dgrad of the convolution
  // after a BN[+ReLU]): g = the rounded dgrad output; gy = g * gate with gate
  // = (bn_gate > 0) (residual tail) or (q(gamma*xhat + beta) > 0) (bn_relu),
  // xhat = (bnx - mean) * istd; writes q(gy) (bn_canon: q(0 + gy)) to bn_out
  // and per-CTA column sums (gy, gy*xhat) to stats (functions.py:418-422)
  const __half* bnx;
  const __half* bn_gate;
  const float *bn_mean, *bn_istd, *bn_gamma, *bn_beta;
  int bn_relu, bn_canon;
  __half* bn_out;
  // fast divisors: tiles_m * tiles_n, tiles_n, stw, sth, sbw, sbh, rgw, rgh
  FDiv fd_pers, fd_tn, fd_stw, fd_sth, fd_sbw, fd_sbh, fd_rgw, fd_rgh;
  int epi_il;         // allow tile-interleaved 8-warp epilogues (see k_tc_gemm)
};

// origin (x, y, image) of spatial box `tile`
__device__ __forceinline__ void sp_origin(const TcArgs& a, int tile, int& x0, int& y0, int& n0) {
  const int t2 = fdiv(tile, a.fd_stw), t3 = fdiv(t2, a.fd_sth);
  x0 = (tile - t2 * a.stw) * a.sbw;
  y0 = (t2 - t3 * a.sth) * a.sbh;
  n0 = t3 * a.sbi;
}

struct Unit {
  int tm, tn, split, kb0, nk;
};

__device__ __forceinline__ Unit decode_unit(const TcArgs& a, int u) {
  Unit w;
  const int per_split = a.tiles_m * a.tiles_n;
  w.split = fdiv(u, a.fd_pers);
  const int rem = u - w.split * per_split;
  w.tm = fdiv(rem, a.fd_tn);
  w.tn = rem - w.tm * a.tiles_n;
  w.kb0 = w.split * a.kb_per_split;
  w.nk = min(w.kb0 + a.kb_per_split, a.num_kb) - w.kb0;
  return w;
}

// One 16 B chunk of a narrow-channel reduction row: taps (r, s), (r, s+1)
// (s even) x 4 channels of the window based at (h0, w0) of the image whose
// first x4 pixel is nb.  Pair mode (even stride): the two pixels are one
// aligned 16 B load (x4 columns are shifted by c4_off so that every pair
// starts on an even column and never straddles the zero border); otherwise
// two 8 B loads.  Taps beyond the filter and out-of-image pixels read zero.
__device__ __forceinline__ void c4_chunk(uint8_t* dst, const TcArgs& a, const ConvGeom& g, int r,
                                         int s, int nb, int h0, int w0) {
  const int ih = h0 + r, col = w0 + s + a.c4_off;
  const bool okr = r < g.r && (unsigned)ih < (unsigned)g.h;
  const int64_t base = ((int64_t)nb + (int64_t)ih * a.c4_w4) * 4;
  if (a.c4_pair) {
    const bool ok = okr && (unsigned)col < (unsigned)a.c4_w4;
    cp_async16_ca(dst, ok ? a.gsrc + base + col * 4 : a.gsrc,
                  !ok ? 0u : (s + 1 < g.s ? 16u : 8u));
  } else {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const bool ok = okr && s + e < g.s && (unsigned)(col + e) < (unsigned)a.c4_w4;
      cp_async8(dst + 8 * e, ok ? a.gsrc + base + (col + e) * 4 : a.gsrc, ok ? 8u : 0u);
    }
  }
}

// EP = 1: the fused BN-backward statistics epilogue (TcArgs::bnx); a separate
// instantiation so the common epilogue keeps its register budget
template <int BN, int AM, int BMD, int CG, int RB, int EP>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, const __grid_constant__ EpiMaps em,
              const TcArgs a) {
  using C = Cfg<BN, CG, RB, EP, AM == A_HALO>;
  constexpr bool kSp = AM == A_TILE4 || AM == A_HALO;  // spatial pixel-box M tiles
  constexpr int S = C::STAGES;
  constexpr int BNL = BN / CG;  // B columns held by this CTA
  constexpr bool kGA = AM == A_GATHER_FPROP || AM == A_GATHER_DGRAD || AM == A_GATHER_C4;
  constexpr bool kGB = BMD == B_GATHER_WGRAD || BMD == B_GATHER_C4;
  constexpr bool kAmn = AM == A_TMA_MN || AM == A_TILE4MN;
  constexpr bool kBmn = BMD != B_TMA_K;
  constexpr uint32_t kTmaBytes = (kGA ? 0 : C::A_BYTES) + (kGB ? 0 : C::STAGE_B);
  static_assert(!RB || (CG == 1 && !kGB), "resident B: single CTA, TMA-fed B");
  constexpr uint32_t IDESC = idesc_f16(BN, kAmn, kBmn, 128 * CG);
  static_assert(CG == 1 || (!kGA && !kGB), "CTA pairs need TMA-fed operands");
  // TMA-fed tiles leave warps 4..7 free: they join the epilogue
  constexpr bool kEpi8 = !kGA && !kGB;
  constexpr int kEpi = kEpi8 ? 8 : 4, kEpiWarp0 = kEpi8 ? 4 : 8;
  // 4 KB TMA-store staging buffers per warp: two (store i drains while chunk
  // i + 1 is rounded) except for 8-warp epilogues of streamed-B tiles
  constexpr int kStgBufs = (kEpi8 && !RB) ? 1 : 2;
  // TMA-store chunk width: 64 columns (128 B rows, 128 B swizzle), or 32 (64 B
  // rows, 64 B swizzle) when eight warps share a 64-wide tile
  constexpr int CW = (kEpi8 && BN == 64) ? 32 : 64;
  // tile-interleaved 8-warp epilogue (single N tile, plain TMA-store outputs):
  // warps 4..7 take the even tiles (accumulator buffer 0) and warps 8..11 the
  // odd ones (buffer 1), each warp all BN columns of its 32 rows -- two tiles'
  // epilogues overlap per SM sub-partition and the per-tile index / barrier /
  // store-issue work is paid by four warps instead of eight
  const bool il = kEpi8 && EP == 0 && a.epi_il && a.tiles_n == 1 && a.tma_store && !a.acc;

  extern __shared__ uint8_t smem_raw[];
  // offset from the shared array itself (not via an integer cast), so that
  // every derived pointer stays in the shared address space (LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // [ A/B stage ring | TMA-store staging (1024-aligned) | barriers | red | bias | stats ]
  uint8_t* stA = smem;
  uint8_t* stB = smem + S * C::A_BYTES;      // ring B stages (RB: unused)
  uint8_t* resB = smem + C::PIPE;            // RB: all k-blocks of B
  uint8_t* stg = smem + C::PIPE + C::RES_BYTES;
  uint8_t* misc = stg + C::STG_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(misc);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* bfull = reinterpret_cast<uint64_t*>(misc + 512);  // RB: resident B landed
  // accumulate-mode epilogue: per epilogue warp, two prev-tile TMA loads in flight
  uint64_t* ebar = reinterpret_cast<uint64_t*>(misc + 256);  // [8 warps][2 buffers]
  float* red = reinterpret_cast<float*>(misc + 1024);
  float* bias_s = reinterpret_cast<float*>(misc + 1024 + C::RED_BYTES);
  float* stat_s = reinterpret_cast<float*>(misc + 1024 + C::RED_BYTES + C::BIAS_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ConvGeom& g = a.g;
  // CTA pair: rank 0 (the leader) owns the full/tempty barriers and issues the
  // MMAs; units are walked per pair
  const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
  const int pair = blockIdx.x / CG, npairs = gridDim.x / CG;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], (kTmaBytes ? 1u : 0u) + ((kGA || kGB) ? 128u : 0u));
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], (il ? 4 : kEpi) * CG);
    }
    mbar_init(bfull, 1);
    for (int b = 0; b < 16; ++b) mbar_init(&ebar[b], 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    if (!kGA) tma_prefetch(&tmA);
    if (!kGB) tma_prefetch(&tmB);
    if (a.tma_store) tma_prefetch(&tmC);
  }
  if (warp == 2) tmem_alloc_cg<CG>(tmem_slot, C::TMEM_COLS);
  // PDL: the set-up above overlapped the previous kernel's tail; from here on
  // its outputs are read
  pdl_wait();
  pdl_trigger();
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (kTmaBytes && lane == 0) {
      int it = 0;
      if (RB) {  // the whole B operand once (single N tile, no split)
        const int rkb = a.res_kb ? a.res_kb : a.num_kb;
        mbar_arrive_tx(bfull, (uint32_t)(rkb * C::B_BYTES));
        for (int kb = 0; kb < rkb; ++kb) {
          uint8_t* dst = resB + kb * C::B_BYTES;
          if (BMD == B_TMA_K) {
            tma_load_2d(dst, &tmB, bfull, kb * BK, 0);
          } else if (BMD == B_TMA_MN) {
            int t = kb / a.b_kblk;
            const int kob = kb - t * a.b_kblk;
            if (a.ntap) t = a.tap_w[t];
            else if (a.flip) t = g.r * g.s - 1 - t;
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(dst + j * 8192, &tmB, bfull, t * a.b_tap_stride + 64 * j, kob * BK);
          }
        }
      }
      for (int u = pair; u < a.units; u += npairs) {
        const Unit w = decode_unit(a, u);
        // this CTA's A rows and B columns of the (128*CG) x BN tile
        const int m0 = w.tm * (BM * CG) + rank * BM, n0 = w.tn * BN + rank * BNL;
        // im2col A: window base of the tile's first row pixel
        int a_x = 0, a_y = 0, a_n = 0;
        if (kSp) sp_origin(a, m0 / BM, a_x, a_y, a_n);
        if (AM == A_IM2COL || AM == A_IM2COL16) {
          a_x = m0 % a.gw;
          const int t = m0 / a.gw;
          a_y = t % a.gh;
          a_n = t / a.gh;
        }
        for (int i = 0; i < w.nk; ++i, ++it) {
          const int s = it % S;
          const uint32_t ph = (it / S) & 1;
          const int kb = w.kb0 + i;
          mbar_wait(&empty[s], ph ^ 1);
          // the leader's barrier counts both CTAs' bytes; the peer only loads
          if (rank == 0) mbar_arrive_tx(&full[s], AM == A_HALO ? a.hl_bytes : kTmaBytes * CG);
          const uint32_t fb = CG == 2 ? mapa_shared(&full[s], 0) : smem_u32(&full[s]);
          auto load2d = [&](void* dst, const CUtensorMap* tm, int c0, int c1) {
            if (CG == 2) tma_load_2d_cg2(dst, tm, fb, c0, c1);
            else tma_load_2d(dst, tm, &full[s], c0, c1);
          };
          auto loadi2c = [&](void* dst, const CUtensorMap* tm, int c, int w_, int h_, int n_,
                             uint16_t ow, uint16_t oh) {
            if (CG == 2) tma_load_im2col_cg2(dst, tm, fb, c, w_, h_, n_, ow, oh);
            else tma_load_im2col(dst, tm, &full[s], c, w_, h_, n_, ow, oh);
          };
          auto load4d = [&](void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3) {
            if (CG == 2) tma_load_4d_cg2(dst, tm, fb, c0, c1, c2, c3);
            else tma_load_4d(dst, tm, &full[s], c0, c1, c2, c3);
          };
          // A_TILE4MN / B_TILE4: this k-block's pixel box
          int kx0 = 0, ky0 = 0, kn0 = 0;
          if (AM == A_TILE4MN || BMD == B_TILE4) sp_origin(a, kb, kx0, ky0, kn0);
          if (AM == A_IM2COL) {
            const int t = kb / a.cblk, cb = kb - t * a.cblk;
            int r, sx;
            if (a.ntap) {
              r = a.tap_offh[t];
              sx = a.tap_offw[t];
            } else {
              r = t / g.s;
              sx = t - r * g.s;
            }
            loadi2c(stA + s * C::A_BYTES, &tmA, cb * 64, a_x * a.isw + a.ilw,
                    a_y * a.ish + a.ilh, a_n, (uint16_t)sx, (uint16_t)r);
          } else if (AM == A_IM2COL16) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {  // taps 4kb .. 4kb+3, 128 pixels x 32 B each
              const int t = kb * 4 + j;
              const int r = t / g.s, sx = t - r * g.s;
              loadi2c(stA + s * C::A_BYTES + j * 4096, &tmA, 0, a_x, a_y, a_n, (uint16_t)sx,
                      (uint16_t)r);
            }
          } else if (AM == A_HALO) {
            load4d(stA + s * C::A_BYTES, &tmA, 0, a_x + a.slw, a_y + a.slh, a_n);
          } else if (AM == A_TILE4) {
            const int t = kb / a.cblk, cb = kb - t * a.cblk;
            int r, sx;  // strided-dgrad class: the tap's dy offsets from the table
            if (a.ntap) { r = a.tap_offh[t]; sx = a.tap_offw[t]; }
            else { r = t / g.s; sx = t - r * g.s; }
            load4d(stA + s * C::A_BYTES, &tmA, cb * 64, a_x + sx + a.slw, a_y + r + a.slh, a_n);
          } else if (AM == A_TILE4MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              load4d(stA + s * C::A_BYTES + j * 8192, &tmA, m0 + 64 * j, kx0, ky0, kn0);
          } else if (AM == A_TMA_K) {
            load2d(stA + s * C::A_BYTES, &tmA, kb * BK, m0);
          } else if (AM == A_TMA_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              load2d(stA + s * C::A_BYTES + j * 8192, &tmA, m0 + 64 * j, kb * BK);
          }
          if (RB) {
            // B is resident
          } else if (BMD == B_TMA_K) {
            load2d(stB + s * C::B_BYTES, &tmB, kb * BK, n0);
          } else if (BMD == B_TMA_MN) {
            int t = kb / a.b_kblk;
            const int kob = kb - t * a.b_kblk;
            if (a.ntap) t = a.tap_w[t];
            else if (a.flip) t = g.r * g.s - 1 - t;
#pragma unroll
            for (int j = 0; j < BNL / 64; ++j)
              load2d(stB + s * C::B_BYTES + j * 8192, &tmB, t * a.b_tap_stride + n0 + 64 * j,
                     kob * BK);
          } else if (BMD == B_TILE4) {
            // 64 k-block pixels x 64 channels of tap (r, s) per 64-wide N block
#pragma unroll
            for (int j = 0; j < BNL / 64; ++j) {
              const int cbg = (n0 >> 6) + j;
              const int t = cbg / a.cblk, cb = cbg - t * a.cblk;
              const int r = t / g.s, sx = t - r * g.s;
              load4d(stB + s * C::B_BYTES + j * 8192, &tmB, cb * 64, kx0 + sx + a.slw,
                     ky0 + r + a.slh, kn0);
            }
          } else if (BMD == B_IM2COL16) {
            // 64 reduction pixels x 16 channels (32 B rows) per tap, BN/16 taps
            const int pix0 = kb * BK;
            const int bx = pix0 % a.gw, t0 = pix0 / a.gw;
            const int by = t0 % a.gh, bn_ = t0 / a.gh;
#pragma unroll
            for (int j = 0; j < BNL / 16; ++j) {
              const int t = (n0 >> 4) + j;
              const int r = t / g.s, sx = t - r * g.s;
              loadi2c(stB + s * C::B_BYTES + j * 2048, &tmB, 0, bx, by, bn_, (uint16_t)sx,
                      (uint16_t)r);
            }
          } else if (BMD == B_IM2COL) {
            // 64 reduction pixels x 64 channels of tap (r, s) per 64-wide N block
            const int pix0 = kb * BK;
            const int bx = pix0 % a.gw, t0 = pix0 / a.gw;
            const int by = t0 % a.gh, bn_ = t0 / a.gh;
#pragma unroll
            for (int j = 0; j < BNL / 64; ++j) {
              const int cbg = (n0 >> 6) + j;
              const int t = cbg / a.cblk, cb = cbg - t * a.cblk;
              const int r = t / g.s, sx = t - r * g.s;
              loadi2c(stB + s * C::B_BYTES + j * 8192, &tmB, cb * 64, bx * a.isw + a.ilw,
                      by * a.ish + a.ilh, bn_, (uint16_t)sx, (uint16_t)r);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp walks the loop (descriptors stay warp-uniform, in uniform
    // registers); one elected lane issues.  Descriptors are built once per
    // stage and advanced per 16-wide K step by adding to the address field.
    if (rank == 0) {
      int it = 0, t = 0;
      if (RB) {
        mbar_wait(bfull, 0);
        tc_fence_after();
      }
      // per-K16 address advance (in 16 B units) of the A and B descriptors
      constexpr uint32_t kDA = AM == A_IM2COL16 ? 4096 / 16 : kAmn ? 2048 / 16 : 32 / 16;
      constexpr uint32_t kDB = BMD == B_IM2COL16 ? 512 / 16 : kBmn ? 2048 / 16 : 32 / 16;
      for (int u = pair; u < a.units; u += npairs, ++t) {
        const Unit w = decode_unit(a, u);
        const int ab = t & 1;
        mbar_wait(&tempty[ab], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(ab * BN);
        for (int i = 0; i < w.nk; ++i, ++it) {
          const int s = it % S;
          const uint32_t ph = (it / S) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t abase = smem_u32(stA + s * C::A_BYTES);
          const uint32_t bbase = RB ? smem_u32(resB + (w.kb0 + i) * C::B_BYTES)
                                    : smem_u32(stB + s * C::B_BYTES);
          // A_IM2COL16: K step kk is tap kk's 128 x 32 B block (K-major,
          // 32 B swizzle); B_IM2COL16: 16 pixel rows of 32 B per K step,
          // taps (16-wide N blocks) 2 KB apart (MN-major, 32 B swizzle)
          const uint64_t da0 = AM == A_IM2COL16 ? sdesc_sw32(abase, 16, 256)
                               : kAmn ? sdesc_sw128(abase, 8192, 1024)
                                      : sdesc_sw128(abase, 16, 1024);
          const uint64_t db0 = BMD == B_IM2COL16 ? sdesc_sw32(bbase, 2048, 256)
                               : kBmn ? sdesc_sw128(bbase, 8192, 1024)
                                      : sdesc_sw128(bbase, 16, 1024);
          if (AM == A_HALO) {
            if (elect_one()) {
              for (int r = 0, tp = 0; r < a.hl_r; ++r)
              for (int sx = 0; sx < a.hl_s; ++sx, ++tp) {
                // the 128B swizzle follows the absolute shared-memory address (as the
                // TMA wrote it), so a view starting s rows into a swizzle atom needs
                // no base offset (measured: base offset s gives wrong products)
                const uint64_t ta = sdesc_sw128(
                    abase + (uint32_t)((r * a.hl_pitch + sx) * 128), 16,
                    (uint32_t)a.hl_pitch * 128u);
                const uint32_t tb = smem_u32(resB + tp * C::B_BYTES);
                const uint64_t tbd = kBmn ? sdesc_sw128(tb, 8192, 1024) : sdesc_sw128(tb, 16, 1024);
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                  mma_f16(d, ta + (uint64_t)(kk * kDA), tbd + (uint64_t)(kk * kDB), IDESC,
                          (tp | kk) != 0);
              }
              mma_commit(&empty[s]);
            }
          } else if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t da = da0 + (uint64_t)(kk * kDA);
              const uint64_t db = db0 + (uint64_t)(kk * kDB);
              if (CG == 2) mma_f16_cg2(d, da, db, IDESC, (i | kk) != 0);
              else mma_f16(d, da, db, IDESC, (i | kk) != 0);
            }
            if (CG == 2) mma_commit_cg2(&empty[s]);
            else mma_commit(&empty[s]);
          }
          __syncwarp();
        }
        if (elect_one()) {
          if (CG == 2) mma_commit_cg2(&tfull[ab]);
          else mma_commit(&tfull[ab]);
        }
        __syncwarp();
      }
    }
  } else if (!kEpi8 && warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ gather producers
    if (kGA || kGB) {
      constexpr int LAG = S - 1;
      const int tid = threadIdx.x - 128;
      const int chunk = tid & 7;
      int it = 0;
      for (int u = pair; u < a.units; u += npairs) {
        const Unit w = decode_unit(a, u);
        const int m0 = w.tm * BM, n0 = w.tn * BN;
        // per-row metadata of this tile's 8 A rows (fixed across its k-blocks)
        int64_t rbase[8];
        int rh[8], rw[8];
        int c4h = -(1 << 28), c4w = 0, c4n = 0;  // A_GATHER_C4: this thread's row = tid
        if (AM == A_GATHER_C4) {
          const int m = m0 + tid;
          if (m < a.M) {
            const int q = m % g.q, t = m / g.q;
            const int p = t % g.p;
            c4n = (t / g.p) * g.h * a.c4_w4;
            c4h = p * g.sh - g.ph;
            c4w = q * g.sw - g.pw;
          }
        } else if (kGA) {
#pragma unroll
          for (int i8 = 0; i8 < 8; ++i8) {
            const int m = m0 + (tid >> 3) + 16 * i8;
            if (m < a.M) {
              if (AM == A_GATHER_FPROP) {
                const int q = m % g.q, t = m / g.q;
                const int p = t % g.p, n = t / g.p;
                rh[i8] = p * g.sh - g.ph;
                rw[i8] = q * g.sw - g.pw;
                rbase[i8] = (((int64_t)n * g.h + rh[i8]) * g.w + rw[i8]) * g.c;
              } else {
                const int x = m % g.w, t = m / g.w;
                const int y = t % g.h, n = t / g.h;
                rh[i8] = y + g.ph;
                rw[i8] = x + g.pw;
                rbase[i8] = (int64_t)n * g.p * g.q;
              }
            } else {
              rh[i8] = -(1 << 28);
              rw[i8] = 0;
              rbase[i8] = 0;
            }
          }
        }
        for (int i = 0; i < w.nk; ++i, ++it) {
          const int s = it % S;
          const uint32_t ph = (it / S) & 1;
          const int kb = w.kb0 + i;
          mbar_wait(&empty[s], ph ^ 1);
          if (AM == A_GATHER_C4) {
            uint8_t* dst = stA + s * C::A_BYTES + tid * 128;
            const int rw = a.c4_s2 * 4;
            int r = (kb * 64) / rw, sl = ((kb * 64) % rw) >> 2;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              c4_chunk(dst + ((j ^ (tid & 7)) << 4), a, g, r, sl, c4n, c4h, c4w);
              sl += 2;
              if (sl == a.c4_s2) { sl = 0; ++r; }
            }
          } else if (BMD == B_GATHER_C4) {
            // reduction row (pixel) tid & 63; this thread fills 16 B chunks
            // 4*(tid>>6) .. +3 of every 64-column block of the tile
            const int row = tid & 63, half = tid >> 6;
            const int64_t pix = (int64_t)kb * 64 + row;
            int ph0 = -(1 << 28), pw0 = 0, pn = 0;
            if (pix < a.K) {
              const int q = (int)(pix % g.q);
              const int64_t tt = pix / g.q;
              const int p = (int)(tt % g.p);
              pn = (int)(tt / g.p) * g.h * a.c4_w4;
              ph0 = p * g.sh - g.ph;
              pw0 = q * g.sw - g.pw;
            }
            const int rw = a.c4_s2 * 4;
#pragma unroll
            for (int jb = 0; jb < BN / 64; ++jb) {
              uint8_t* dst = stB + s * C::B_BYTES + jb * 8192 + row * 128;
              const int k0 = n0 + jb * 64 + half * 32;
              int r = k0 / rw, sl = (k0 % rw) >> 2;
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const int j = half * 4 + jj;
                c4_chunk(dst + ((j ^ (row & 7)) << 4), a, g, r, sl, pn, ph0, pw0);
                sl += 2;
                if (sl == a.c4_s2) { sl = 0; ++r; }
              }
            }
          } else if (AM == A_GATHER_FPROP) {
            const int t = kb / a.cblk, cb = kb - t * a.cblk;
            const int r = t / g.s, sx = t - r * g.s;
            const int64_t toff = ((int64_t)r * g.w + sx) * g.c + cb * 64 + chunk * 8;
            uint8_t* dst = stA + s * C::A_BYTES;
#pragma unroll
            for (int i8 = 0; i8 < 8; ++i8) {
              const int row = (tid >> 3) + 16 * i8;
              const int ih = rh[i8] + r, iw = rw[i8] + sx;
              const bool ok = (unsigned)ih < (unsigned)g.h && (unsigned)iw < (unsigned)g.w;
              const __half* src = ok ? a.gsrc + rbase[i8] + toff : a.gsrc;
              cp_async16(dst + row * 128 + ((chunk ^ (row & 7)) << 4), src, ok ? 16u : 0u);
            }
          } else if (AM == A_GATHER_DGRAD) {
            const int t = kb / a.cblk, kob = kb - t * a.cblk;
            const int r = t / g.s, sx = t - r * g.s;
            uint8_t* dst = stA + s * C::A_BYTES;
#pragma unroll
            for (int i8 = 0; i8 < 8; ++i8) {
              const int row = (tid >> 3) + 16 * i8;
              const int th = rh[i8] - r, tw = rw[i8] - sx;
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
                  ok ? a.gsrc + (rbase[i8] + (int64_t)oh * g.q + ow) * g.k + kob * 64 + chunk * 8
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
          if (it >= LAG) {
            cp_async_wait<LAG>();
            fence_proxy_async();
            mbar_arrive(&full[(it - LAG) % S]);
          }
        }
      }
      cp_async_wait<0>();
      fence_proxy_async();
      for (int j = it > LAG ? it - LAG : 0; j < it; ++j) mbar_arrive(&full[j % S]);
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------ epilogue
    // kEpi8: warps 4..11, the first four on columns [0, BN/2), the others on
    // [BN/2, BN) (two warps per SM sub-partition hide each other's latency)
    const int ew = warp - kEpiWarp0;         // epilogue warp 0 .. kEpi - 1
    const int wq = warp & 3;                 // TMEM lane quarter
    const int grp = ew >> 2;                 // kEpi8: warp group 0 / 1
    const int c_lo = kEpi8 && !il ? grp * (BN / 2) : 0;
    const int c_hi = kEpi8 && !il ? c_lo + BN / 2 : BN;
    constexpr int kEpiThreads = 32 * kEpi;
    const int tid = threadIdx.x - 32 * kEpiWarp0;
    if (a.stats) {
      for (int j = tid; j < 2 * C::MAX_STAT_N; j += kEpiThreads) stat_s[j] = 0.f;
      named_sync(1, kEpiThreads);
    }
    int t = 0;
    uint32_t sb = 0;  // TMA-store staging buffer alternation (per warp)
    uint32_t ac = 0;  // accumulate mode: chunks processed by this warp (2 KB buffers)
    int staged_n0 = -1;  // N tile whose bias slice is in bias_s
    // BN statistics of a single-N-tile GEMM stored through TMA: each warp keeps its
    // columns' running sums in registers over all its tiles (fixed tile order) and
    // the four row-quarter warps are combined once at the end -- no per-tile barrier
    const bool reg_stats = a.stats && a.tma_store && a.tiles_n == 1;
    float racc[4][4] = {};
    // the leader's tempty barriers (the MMA waits on both CTAs' epilogues)
    const uint32_t te0 = CG == 2 ? mapa_shared(&tempty[0], 0) : smem_u32(&tempty[0]);
    if (il && (a.bias || a.stats)) {  // one N tile: its bias / centre slices once
      staged_n0 = 0;
      named_sync(2, kEpiThreads);
      for (int j = tid; j < BN; j += kEpiThreads) {
        const bool ok = j < a.N;
        if (a.bias) bias_s[j] = ok ? __half2float(a.bias[j]) : 0.f;
        if (a.bias) bias_s[2 * BN + j] = __fadd_rn(bias_s[j], 0.f);
        if (a.stats) bias_s[BN + j] = ok && a.stat_shift ? a.stat_shift[j] : 0.f;
      }
      named_sync(2, kEpiThreads);
    }
    for (int u = pair; u < a.units; u += npairs, ++t) {
      if (il && (t & 1) != grp) continue;
      const Unit w = decode_unit(a, u);
      const int m0 = w.tm * (BM * CG) + rank * BM, n0 = w.tn * BN;
      const int ab = t & 1;
      // bias / BN slices of this N tile (f32); fprop statistics: the centre K
      // of each column in bias_s[BN + j] (0 without a shift)
      if ((a.bias || EP == 1 || a.stats) && n0 != staged_n0) {
        staged_n0 = n0;
        named_sync(2, kEpiThreads);
        for (int j = tid; j < BN; j += kEpiThreads) {
          const bool ok = n0 + j < a.N;
          if (a.bias) bias_s[j] = ok ? __half2float(a.bias[n0 + j]) : 0.f;
          // EP = 0: the bias with -0 made +0 in bias_s[2 BN + j]: q(0 + (acc + b))
          // == q(acc + (b + 0)) for every acc and b, one add instead of two
          if (EP == 0 && a.bias) bias_s[2 * BN + j] = __fadd_rn(bias_s[j], 0.f);
          if (EP == 0 && a.stats) bias_s[BN + j] = ok && a.stat_shift ? a.stat_shift[n0 + j] : 0.f;
          if (EP == 1) {
            bias_s[BN + j] = ok ? a.bn_mean[n0 + j] : 0.f;
            bias_s[2 * BN + j] = ok ? a.bn_istd[n0 + j] : 0.f;
            bias_s[3 * BN + j] = ok && a.bn_gamma ? a.bn_gamma[n0 + j] : 0.f;
            bias_s[4 * BN + j] = ok && a.bn_beta ? a.bn_beta[n0 + j] : 0.f;
          }
        }
        named_sync(2, kEpiThreads);
      }
      const int row = wq * 32 + lane;
      const int m = m0 + row;
      int ex0 = 0, ey0 = 0, en0 = 0;
      if (kSp) sp_origin(a, m0 / BM, ex0, ey0, en0);
      // A_HALO tiles overhang the grid bottom: rows past the last image row are idle
      // tile row -> (bx, by, bi) of the pixel box (x fastest, then y, then image)
      const int rq = kSp ? fdiv(row, a.fd_sbw) : 0, rbi = kSp ? fdiv(rq, a.fd_sbh) : 0;
      const int rbx = row - rq * a.sbw, rby = rq - rbi * a.sbh;
      const bool mv = kSp ? (m0 / BM < a.sp_tiles && (AM != A_HALO || ey0 + rq < a.sgh))
                          : m < a.M;
      int64_t orow = m;
      if (kSp) orow = ((int64_t)(en0 + rbi) * a.sgh + ey0 + rby) * a.sgw + ex0 + rbx;
      // box coordinates of the warp's first row (its 32 rows are a sub-box)
      const int wrq = kSp ? fdiv(32 * wq, a.fd_sbw) : 0, wrb = kSp ? fdiv(wrq, a.fd_sbh) : 0;
      const int wcx = ex0 + 32 * wq - wrq * a.sbw, wcy = ey0 + wrq - wrb * a.sbh, wcn = en0 + wrb;
      if (a.remap && mv) {
        const int tt = fdiv(m, a.fd_rgw), x = m - tt * a.rgw;
        const int n = fdiv(tt, a.fd_rgh), y = tt - n * a.rgh;
        orow = ((int64_t)n * g.h + y * a.rsh + a.ra) * g.w + x * a.rsw + a.rb;
      }
      // accumulate mode through TMA: the previous values of each 32-column chunk
      // are TMA-loaded into the staging buffer (two 2 KB halves per warp,
      // alternating), updated in place to q(prev + acc) and TMA-stored; chunk
      // 0's load is issued before the accumulator is ready, chunk i+1's while
      // chunk i is processed
      const bool tacc = a.tma_store && a.acc;
      auto acc_load = [&](int cc, uint32_t k) {
        if (lane == 0) {
          uint8_t* bb = stg + ew * kStgBufs * 4096 + (k & 1) * 2048;
          bulk_wait_read<0>();  // this half's previous store has read it
          mbar_arrive_tx(&ebar[ew * 2 + (k & 1)], 2048);
          if (kSp) {
            tma_load_4d(bb, &tmC, &ebar[ew * 2 + (k & 1)], n0 + cc, wcx, wcy, wcn);
          } else {
            tma_load_2d(bb, &tmC, &ebar[ew * 2 + (k & 1)], n0 + cc, m0 + 32 * wq);
          }
        }
      };
      // EP = 1: the x / gate / prev tiles of each 32-column chunk, TMA-loaded into
      // one of this warp's two 6 KB sets (next chunk prefetched, first chunk before
      // the accumulator is ready)
      auto bnb_load = [&](int cc, uint32_t k) {
        if (lane == 0) {
          uint8_t* bb = stg + ew * 12288 + (k & 1) * 6144;
          uint64_t* bar = &ebar[ew * 2 + (k & 1)];
          bulk_wait_read<0>();  // this set's previous store has read it
          mbar_arrive_tx(bar, 2048u * (1u + (a.bn_gate ? 1u : 0u) + (a.acc ? 1u : 0u)));
          if (kSp) {
            const int cx = wcx, cy = wcy, cn = wcn;
            tma_load_4d(bb, &em.x, bar, n0 + cc, cx, cy, cn);
            if (a.bn_gate) tma_load_4d(bb + 2048, &em.g, bar, n0 + cc, cx, cy, cn);
            if (a.acc) tma_load_4d(bb + 4096, &tmC, bar, n0 + cc, cx, cy, cn);
          } else {
            tma_load_2d(bb, &em.x, bar, n0 + cc, m0 + 32 * wq);
            if (a.bn_gate) tma_load_2d(bb + 2048, &em.g, bar, n0 + cc, m0 + 32 * wq);
            if (a.acc) tma_load_2d(bb + 4096, &tmC, bar, n0 + cc, m0 + 32 * wq);
          }
        }
      };
      if (EP == 1) bnb_load(c_lo, ac);
      else if (tacc) acc_load(c_lo, ac);
      mbar_wait(&tfull[ab], (t >> 1) & 1);
      tc_fence_after();
      int bad = 0;
      // the accumulator buffer is handed back to the MMA warp as soon as this
      // warp's last TMEM load of the tile has completed (the rest of the
      // epilogue works from registers / shared memory)
      bool released = false;
      auto release_tmem = [&](bool last) {
        if (!last || released) return;
        released = true;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) mbar_arrive_cluster(te0 + 8 * ab);
          else mbar_arrive(&tempty[ab]);
        }
      };
      if (EP == 1) {
        // fused BN backward (TcArgs::bnx): row `lane`, 8 columns per 16 B piece;
        // g = q(prev + acc), gy = g * gate, out = q(gy) written over the x tile and
        // TMA-stored; column sums of (gy, gy*xhat) by shuffles, 16 columns at a time
        for (int c = c_lo; c < c_hi; c += 32, ++ac) {
          if (c + 32 < c_hi) bnb_load(c + 32, ac + 1);
          uint32_t v[32];
          tmem_ld32_nowait(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(ab * BN + c), v);
          tmem_wait_ld();
          release_tmem(c + 32 >= c_hi);
          uint8_t* bs = stg + ew * 12288 + (ac & 1) * 6144;
          mbar_wait(&ebar[ew * 2 + (ac & 1)], (ac >> 1) & 1);
          const int swz = (lane >> 1) & 3;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float s1[16], s2[16];
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const int j = 2 * h + jj;
              const int off = lane * 64 + ((j ^ swz) << 4);
              const uint4 xq = *reinterpret_cast<const uint4*>(bs + off);
              const uint4 gq = a.bn_gate ? *reinterpret_cast<const uint4*>(bs + 2048 + off)
                                         : make_uint4(0, 0, 0, 0);
              const uint4 pq = a.acc ? *reinterpret_cast<const uint4*>(bs + 4096 + off)
                                     : make_uint4(0, 0, 0, 0);
              const __half* xh8 = reinterpret_cast<const __half*>(&xq);
              const __half* gh8 = reinterpret_cast<const __half*>(&gq);
              const __half* ph8 = reinterpret_cast<const __half*>(&pq);
              __align__(16) __half o8[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int k = 8 * j + e;
                const float f = __uint_as_float(v[k]);
                const float g = __half2float(__float2half_rn(
                    __fadd_rn(a.acc ? __half2float(ph8[e]) : 0.f, f)));
                const float xh = __fmul_rn(__fsub_rn(__half2float(xh8[e]), bias_s[BN + c + k]),
                                           bias_s[2 * BN + c + k]);
                float gate = 1.f;
                if (a.bn_gate) {
                  gate = __half2float(gh8[e]) > 0.f ? 1.f : 0.f;
                } else if (a.bn_relu) {
                  const float z = __half2float(__float2half_rn(
                      __fadd_rn(__fmul_rn(bias_s[3 * BN + c + k], xh), bias_s[4 * BN + c + k])));
                  gate = z > 0.f ? 1.f : 0.f;
                }
                const float gy = __fmul_rn(g, gate);
                const bool ok = mv && n0 + c + k < a.N;
                s1[8 * jj + e] = ok ? gy : 0.f;
                s2[8 * jj + e] = ok ? __fmul_rn(gy, xh) : 0.f;
                o8[e] = __float2half_rn(a.bn_canon ? __fadd_rn(0.f, gy) : gy);
              }
              *reinterpret_cast<uint4*>(bs + off) = *reinterpret_cast<const uint4*>(o8);
            }
            if (a.stats) {
#pragma unroll
              for (int q = 0; q < 16; ++q) {
                s1[q] += __shfl_xor_sync(0xffffffffu, s1[q], 16);
                s2[q] += __shfl_xor_sync(0xffffffffu, s2[q], 16);
              }
#pragma unroll
              for (int st = 8; st >= 1; st >>= 1) {
                const bool up = (lane & st) != 0;
#pragma unroll
                for (int q = 0; q < st; ++q) {
                  const float send1 = up ? s1[q] : s1[q + st], keep1 = up ? s1[q + st] : s1[q];
                  const float send2 = up ? s2[q] : s2[q + st], keep2 = up ? s2[q + st] : s2[q];
                  s1[q] = keep1 + __shfl_xor_sync(0xffffffffu, send1, st);
                  s2[q] = keep2 + __shfl_xor_sync(0xffffffffu, send2, st);
                }
              }
              if (lane < 16) {
                red[((wq * BN) + c + 16 * h + lane) * 2 + 0] = s1[0];
                red[((wq * BN) + c + 16 * h + lane) * 2 + 1] = s2[0];
              }
            }
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            if (kSp) {
              tma_store_4d(&em.o, bs, n0 + c, wcx, wcy, wcn);
            } else {
              tma_store_2d(&em.o, bs, n0 + c, m0 + 32 * wq);
            }
            bulk_commit();
          }
        }
      } else if (tacc) {
        for (int c = c_lo; c < c_hi; c += 32, ++ac) {
          if (c + 32 < c_hi) acc_load(c + 32, ac + 1);
          uint32_t v[32];
          tmem_ld32_nowait(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(ab * BN + c), v);
          tmem_wait_ld();
          release_tmem(c + 32 >= c_hi);
          uint8_t* buf = stg + ew * kStgBufs * 4096 + (ac & 1) * 2048;
          mbar_wait(&ebar[ew * 2 + (ac & 1)], (ac >> 1) & 1);
          const int swz = (lane >> 1) & 3;  // 64 B rows, 64 B swizzle
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4* pp = reinterpret_cast<uint4*>(buf + lane * 64 + ((j ^ swz) << 4));
            const uint4 pv = *pp;
            const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w};
            uint32_t pk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int k = 8 * j + 2 * e;
              float f0 = __uint_as_float(v[k]), f1 = __uint_as_float(v[k + 1]);
              if (a.bias) {
                f0 = __fadd_rn(f0, bias_s[c + k]);
                f1 = __fadd_rn(f1, bias_s[c + k + 1]);
              }
              const float2 p2 = __half22float2(*reinterpret_cast<const __half2*>(&pw[e]));
              const __half2 h = __floats2half2_rn(__fadd_rn(p2.x, f0), __fadd_rn(p2.y, f1));
              pk[e] = mv ? *reinterpret_cast<const uint32_t*>(&h) : 0u;
            }
            if (a.nonfinite) {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                bad |= ((pk[e] & 0x7c00u) == 0x7c00u) | ((pk[e] & 0x7c000000u) == 0x7c000000u);
            }
            *pp = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            if (kSp) {
              tma_store_4d(&tmC, buf, n0 + c, wcx, wcy, wcn);
            } else {
              tma_store_2d(&tmC, buf, n0 + c, m0 + 32 * wq);
            }
            bulk_commit();
          }
        }
      } else if (a.tma_store) {
        // 64-column chunks: round into a 128B-swizzled 32 x 64 staging tile, TMA
        // store it (rows >= M and columns >= N are clipped by the tensor map),
        // and take the BN column sums from the staged (rounded) values.
        for (int c = c_lo; c < c_hi; c += CW) {
          uint32_t v[CW];
          const uint32_t tb = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(ab * BN + c);
          tmem_ld32_nowait(tb, v);
          if (CW == 64) tmem_ld32_nowait(tb + 32, v + 32);
          tmem_wait_ld();
          release_tmem(c + CW >= c_hi);
          uint8_t* buf = stg + (ew * kStgBufs + (sb % kStgBufs)) * 4096;
          ++sb;
          if (lane == 0) bulk_wait_read<kStgBufs - 1>();  // buf's previous store has read it
          __syncwarp();
          // row `lane`, 16 B piece j at the TMA swizzle position
          const int swz = CW == 64 ? (lane & 7) : ((lane >> 1) & 3);
#pragma unroll
          for (int j = 0; j < CW / 8; ++j) {  // piece j = columns c + 8j .. c + 8j + 7
            uint32_t pk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int k = 8 * j + 2 * e;
              // packed f32x2 add (FADD2): q(0 + (acc + b)) as q(acc + (b + 0))
              const float2 f = __fadd2_rn(
                  make_float2(__uint_as_float(v[k]), __uint_as_float(v[k + 1])),
                  a.bias ? *reinterpret_cast<const float2*>(&bias_s[2 * BN + c + k])
                         : make_float2(0.f, 0.f));
              const __half2 h = __floats2half2_rn(f.x, f.y);
              pk[e] = mv ? *reinterpret_cast<const uint32_t*>(&h) : 0u;
            }
            if (a.nonfinite) {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                bad |= ((pk[e] & 0x7c00u) == 0x7c00u) | ((pk[e] & 0x7c000000u) == 0x7c000000u);
            }
            *reinterpret_cast<uint4*>(buf + lane * (CW * 2) + ((j ^ swz) << 4)) =
                make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            if (kSp) {  // the warp's 32 rows are a sub-box of the pixel box
              tma_store_4d(&tmC, buf, n0 + c, wcx, wcy, wcn);
            } else {
              tma_store_2d(&tmC, buf, n0 + c, m0 + 32 * wq);
            }
            bulk_commit();
          }
          if (a.stats) {
            // sums of (y - K) over the warp's VALID rows (idle rows are staged
            // as zeros, which would otherwise count as -K)
            const uint32_t vrows = __ballot_sync(0xffffffffu, mv);
            // per column pair: s1 += y - K, s2 += (y - K)^2 with packed f32x2
            // FADD2 / FFMA2 (the same RN ops as the scalar FADD / contracted FFMA)
            auto acc2 = [](float2& s1, float2& s2, float2 x, float2 nk, bool ok) {
              float2 d = __fadd2_rn(x, nk);
              if (!ok) d = make_float2(0.f, 0.f);
              s1 = __fadd2_rn(s1, d);
              s2 = __ffma2_rn(d, d, s2);
            };
            if (CW == 64) {  // lane owns columns c + 2*lane, c + 2*lane + 1
              float2 s1 = make_float2(0.f, 0.f), s2 = make_float2(0.f, 0.f);
              const float2 nk = make_float2(-bias_s[BN + c + 2 * lane],
                                            -bias_s[BN + c + 2 * lane + 1]);
              const uint8_t* bp = buf + (lane & 3) * 4;
              if (vrows == 0xffffffffu) {  // two accumulator chains (even / odd rows)
                float2 t1 = make_float2(0.f, 0.f), t2 = make_float2(0.f, 0.f);
#pragma unroll 16
                for (int r = 0; r < 32; r += 2) {
                  acc2(s1, s2, __half22float2(*reinterpret_cast<const __half2*>(
                                   bp + r * 128 + (((lane >> 2) ^ (r & 7)) << 4))), nk, true);
                  acc2(t1, t2, __half22float2(*reinterpret_cast<const __half2*>(
                                   bp + (r + 1) * 128 + (((lane >> 2) ^ ((r + 1) & 7)) << 4))),
                       nk, true);
                }
                s1 = __fadd2_rn(s1, t1);
                s2 = __fadd2_rn(s2, t2);
              } else {
#pragma unroll 8
                for (int r = 0; r < 32; ++r)
                  acc2(s1, s2, __half22float2(*reinterpret_cast<const __half2*>(
                                   bp + r * 128 + (((lane >> 2) ^ (r & 7)) << 4))), nk,
                       (vrows >> r) & 1);
              }
              if (reg_stats) {
                float* ra = racc[(c - c_lo) / CW];
                ra[0] += s1.x; ra[1] += s2.x; ra[2] += s1.y; ra[3] += s2.y;
              } else {
                float* rp = red + ((wq * BN) + c + 2 * lane) * 2;
                rp[0] = s1.x;
                rp[1] = s2.x;
                rp[2] = s1.y;
                rp[3] = s2.y;
              }
            } else {
              // lane owns the column pair c + 2p, c + 2p + 1 (p = lane & 15) over
              // rows 16h .. 16h + 15 (h = lane >> 4), half2 loads; the upper half
              // walks its rows in (i ^ 1) order so the two halves of the warp read
              // the two different 64 B bank halves; halves combined by one shuffle
              const int p = lane & 15, h = lane >> 4;
              const float2 nk = make_float2(-bias_s[BN + c + 2 * p], -bias_s[BN + c + 2 * p + 1]);
              const uint8_t* bp = buf + (p & 3) * 4;
              float2 s1 = make_float2(0.f, 0.f), s2 = make_float2(0.f, 0.f);
              if (vrows == 0xffffffffu) {  // two accumulator chains (even / odd i)
                float2 t1 = make_float2(0.f, 0.f), t2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                  const int r = 16 * h + (i ^ h), r1 = 16 * h + ((i + 1) ^ h);
                  acc2(s1, s2, __half22float2(*reinterpret_cast<const __half2*>(
                                   bp + r * 64 + (((p >> 2) ^ ((r >> 1) & 3)) << 4))), nk, true);
                  acc2(t1, t2, __half22float2(*reinterpret_cast<const __half2*>(
                                   bp + r1 * 64 + (((p >> 2) ^ ((r1 >> 1) & 3)) << 4))), nk, true);
                }
                s1 = __fadd2_rn(s1, t1);
                s2 = __fadd2_rn(s2, t2);
              } else if (vrows) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const int r = 16 * h + (i ^ h);
                  acc2(s1, s2, __half22float2(*reinterpret_cast<const __half2*>(
                                   bp + r * 64 + (((p >> 2) ^ ((r >> 1) & 3)) << 4))), nk,
                       (vrows >> r) & 1);
                }
              }
              float s1a = s1.x, s1b = s1.y, s2a = s2.x, s2b = s2.y;
              s1a += __shfl_xor_sync(0xffffffffu, s1a, 16);
              s1b += __shfl_xor_sync(0xffffffffu, s1b, 16);
              s2a += __shfl_xor_sync(0xffffffffu, s2a, 16);
              s2b += __shfl_xor_sync(0xffffffffu, s2b, 16);
              if (reg_stats) {
                float* ra = racc[(c - c_lo) / CW];
                ra[0] += s1a; ra[1] += s2a; ra[2] += s1b; ra[3] += s2b;
              } else if (h == 0) {
                float* rp = red + ((wq * BN) + c + 2 * p) * 2;
                rp[0] = s1a;
                rp[1] = s2a;
                rp[2] = s1b;
                rp[3] = s2b;
              }
            }
          }
        }
      } else
      for (int c = c_lo; c < c_hi; c += 32) {
        uint32_t v[32];
        tmem_ld32_nowait(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(ab * BN + c), v);
        tmem_wait_ld();
        release_tmem(c + 32 >= c_hi);
        const int nb = n0 + c;
        const bool full_cols = nb + 32 <= a.N;
        if (a.partial) {
          if (mv) {
            float* dstp = a.partial + ((int64_t)w.split * a.M + m) * a.N + nb;
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
          for (int j = 0; j < 32; ++j) f[j] = __fadd_rn(f[j], bias_s[c + j]);
        }
        __half* dsth = reinterpret_cast<__half*>(a.out) + orow * a.ldc + nb;
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
            for (int j = 0; j < 32; ++j)
              hv[j] = __float2half_rn(__fadd_rn(__half2float(hv[j]), f[j]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) hv[j] = __float2half_rn(__fadd_rn(0.f, f[j]));
          }
        }
        // BN statistics of the rounded outputs, 16 columns at a time: column
        // sums over the warp's 32 rows (lanes l and l^16 add, then a halving
        // exchange leaves column c + 16h + (lane & 15) in lane; 31 shuffles)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!a.stats) break;
          float s1[16], s2[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int j = 16 * h + k;
            const float x = (mv && nb + j < a.N) ? __half2float(hv[j]) - bias_s[BN + c + j] : 0.f;
            s1[k] = x;
            s2[k] = x * x;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            s1[j] += __shfl_xor_sync(0xffffffffu, s1[j], 16);
            s2[j] += __shfl_xor_sync(0xffffffffu, s2[j], 16);
          }
#pragma unroll
          for (int st = 8; st >= 1; st >>= 1) {
            const bool up = (lane & st) != 0;
#pragma unroll
            for (int j = 0; j < st; ++j) {
              const float send1 = up ? s1[j] : s1[j + st], keep1 = up ? s1[j + st] : s1[j];
              const float send2 = up ? s2[j] : s2[j + st], keep2 = up ? s2[j + st] : s2[j];
              s1[j] = keep1 + __shfl_xor_sync(0xffffffffu, send1, st);
              s2[j] = keep2 + __shfl_xor_sync(0xffffffffu, send2, st);
            }
          }
          if (lane < 16) {
            red[((wq * BN) + c + 16 * h + lane) * 2 + 0] = s1[0];
            red[((wq * BN) + c + 16 * h + lane) * 2 + 1] = s2[0];
          }
        }
        if (mv) {
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
            for (int j = 0; j < 32; ++j) bad |= (nb + j < a.N) && !isfinite(__half2float(hv[j]));
          }
        }
      }
      release_tmem(true);  // (a warp with no columns in this tile)
      if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
      if (a.stats && !reg_stats) {
        named_sync(1, kEpiThreads);
        for (int col = tid; col < BN; col += kEpiThreads) {
          if (n0 + col >= a.N) continue;
          float t1 = 0.f, t2 = 0.f;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            t1 += red[(q * BN + col) * 2 + 0];
            t2 += red[(q * BN + col) * 2 + 1];
          }
          // per-CTA running sums, in this CTA's fixed tile order (deterministic)
          stat_s[n0 + col] += t1;
          stat_s[C::MAX_STAT_N + n0 + col] += t2;
        }
        named_sync(1, kEpiThreads);
      }
    }
    if (reg_stats) {  // combine the row-quarter warps: red[q][col] -> stat_s[col]
      // (tile-interleaved: group 0's quarters, then group 1's added -- fixed order)
      for (int pass = 0; pass < (il ? 2 : 1); ++pass) {
        if (!il || grp == pass)
          for (int k = 0; k * CW < c_hi - c_lo; ++k) {
            const int c = c_lo + k * CW;
            if (CW == 64) {
              float* rp = red + ((wq * BN) + c + 2 * lane) * 2;
              rp[0] = racc[k][0]; rp[1] = racc[k][1]; rp[2] = racc[k][2]; rp[3] = racc[k][3];
            } else if (lane < 16) {  // column pair c + 2 lane, c + 2 lane + 1
              float* rp = red + ((wq * BN) + c + 2 * lane) * 2;
              rp[0] = racc[k][0]; rp[1] = racc[k][1]; rp[2] = racc[k][2]; rp[3] = racc[k][3];
            }
          }
        named_sync(1, kEpiThreads);
        for (int col = tid; col < BN && col < a.N; col += kEpiThreads) {
          float t1 = 0.f, t2 = 0.f;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            t1 += red[(q * BN + col) * 2 + 0];
            t2 += red[(q * BN + col) * 2 + 1];
          }
          stat_s[col] = pass ? stat_s[col] + t1 : t1;
          stat_s[C::MAX_STAT_N + col] = pass ? stat_s[C::MAX_STAT_N + col] + t2 : t2;
        }
        named_sync(1, kEpiThreads);
      }
    }
    if (a.stats) {  // one partial row per CTA: stats[blockIdx.x][2][N]
      for (int col = tid; col < a.N; col += kEpiThreads) {
        a.stats[((int64_t)blockIdx.x * 2 + 0) * a.N + col] = stat_s[col];
        a.stats[((int64_t)blockIdx.x * 2 + 1) * a.N + col] = stat_s[C::MAX_STAT_N + col];
      }
    }
    if ((a.tma_store || EP == 1) && lane == 0) bulk_wait<0>();
  }
  __syncwarp();
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_cg<CG>(tmem, C::TMEM_COLS);
  }
}

#ifndef NNL_TC_INSTANTIATE  // helper kernels: host-side TU only
// out = q(prev + bias + sum_s partial[s][m][n]), 4 consecutive columns per
// thread (plain layout, N and ldc multiples of 4), float4 partial loads, 8 B
// stores.  P split groups per float4 column: thread group g sums splits g, g + P, ...
// in ascending order and the P group sums are added in ascending g -- a fixed
// association (deterministic, independent of the grid), with P loads in
// flight per output instead of one chain of `splits` dependent loads
template <int P>
__global__ void __launch_bounds__(256) k_tc_splitk_reduce4(
    int M, int N, int splits, const float* __restrict__ partial, const __half* __restrict__ bias,
    __half* __restrict__ out, int64_t ldc, int acc, int32_t* nonfinite) {
  pdl_wait();
  pdl_trigger();
  constexpr int COLS = 256 / P;
  __shared__ float4 red[P][COLS];
  const int g = threadIdx.x / COLS, cl = threadIdx.x % COLS;
  const int64_t total = (int64_t)M * N, total4 = total / 4;
  const int64_t t = (int64_t)blockIdx.x * COLS + cl;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (t < total4) {
#pragma unroll 4
    for (int z = g; z < splits; z += P) {
      const float4 p = *reinterpret_cast<const float4*>(partial + (int64_t)z * total + 4 * t);
      s.x += p.x; s.y += p.y; s.z += p.z; s.w += p.w;
    }
  }
  if (P > 1) {
    red[g][cl] = s;
    __syncthreads();
  }
  int bad = 0;
  if (g == 0 && t < total4) {
    if (P > 1) {
      s = red[0][cl];
#pragma unroll
      for (int q = 1; q < P; ++q) {
        const float4 r = red[q][cl];
        s.x += r.x; s.y += r.y; s.z += r.z; s.w += r.w;
      }
    }
    const int64_t i = 4 * t;
    const int64_t m = i / N, n = i % N;
    float v[4] = {s.x, s.y, s.z, s.w};
    if (bias) {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = __fadd_rn(v[e], __half2float(bias[n + e]));
    }
    uint2* o = reinterpret_cast<uint2*>(out + m * ldc + n);
    float pv[4] = {0.f, 0.f, 0.f, 0.f};
    if (acc) {
      const uint2 u = *o;
      const float2 a0 = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
      const float2 b0 = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
      pv[0] = a0.x; pv[1] = a0.y; pv[2] = b0.x; pv[3] = b0.y;
    }
    const __half2 h0 = __floats2half2_rn(__fadd_rn(pv[0], v[0]), __fadd_rn(pv[1], v[1]));
    const __half2 h1 = __floats2half2_rn(__fadd_rn(pv[2], v[2]), __fadd_rn(pv[3], v[3]));
    uint2 w;
    w.x = *reinterpret_cast<const uint32_t*>(&h0);
    w.y = *reinterpret_cast<const uint32_t*>(&h1);
    *o = w;
    const float2 c0 = __half22float2(h0), c1 = __half22float2(h1);
    bad = !isfinite(c0.x) | !isfinite(c0.y) | !isfinite(c1.x) | !isfinite(c1.y);
  }
  if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
}

// launch the grouped reduction: 8 groups once there are >= 16 splits
static int launch_reduce4(int M, int N, int splits, const float* partial, const __half* bias,
                          __half* out, int64_t ldc, int acc, int32_t* nonfinite, cudaStream_t st) {
  const int64_t total4 = (int64_t)M * N / 4;
  if (splits >= 16)
    launch_k(k_tc_splitk_reduce4<8>, (unsigned)((total4 + 31) / 32), 256, 0, st, M, N, splits,
             partial, bias, out, ldc, acc, nonfinite);
  else if (splits >= 4)
    launch_k(k_tc_splitk_reduce4<4>, (unsigned)((total4 + 63) / 64), 256, 0, st, M, N, splits,
             partial, bias, out, ldc, acc, nonfinite);
  else
    launch_k(k_tc_splitk_reduce4<1>, (unsigned)((total4 + 255) / 256), 256, 0, st, M, N, splits,
             partial, bias, out, ldc, acc, nonfinite);
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

// the general form: one column per thread, fixed split order; `trans` writes
// D[m][n] to out[n*ldc + m]
__global__ void k_tc_splitk_reduce(int M, int N, int splits, const float* __restrict__ partial,
                                   const __half* __restrict__ bias, __half* __restrict__ out,
                                   int64_t ldc, int acc, int trans, int c4, int c4_s2,
                                   int fr, int fs, int s2d, int32_t* nonfinite) {
  pdl_wait();
  pdl_trigger();
  int bad = 0;
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / N;
    int64_t n = i % N;
    if (s2d) {  // column (block tap, 16-slot) of the space-to-depth conv -> (r, s, c)
      const int tap = (int)(n >> 4), slot = (int)(n & 15);
      const int br = tap / c4_s2, bc = tap - br * c4_s2;
      const int sub = slot / c4, c = slot - sub * c4;
      const int r = 2 * br + (sub >> 1), sx = 2 * bc + (sub & 1);
      if (sub >= 4 || r >= fr || sx >= fs) continue;
      n = ((int64_t)r * fs + sx) * c4 + c;
    } else if (c4) {  // column (r, s, 4-channel slot) -> (r, s, channel); padding dropped
      const int rw = c4_s2 * 4;
      const int r = (int)(n / rw), sx = (int)(n % rw) >> 2, c = (int)(n & 3);
      if (c >= c4 || sx >= fs || r >= fr) continue;
      n = ((int64_t)r * fs + sx) * c4 + c;
    }
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + i];
    if (bias) s = __fadd_rn(s, __half2float(bias[n]));
    __half* o = out + (trans ? n * ldc + m : m * ldc + n);
    const float prev = acc ? __half2float(*o) : 0.f;
    const __half h = __float2half_rn(__fadd_rn(prev, s));
    *o = h;
    bad |= !isfinite(__half2float(h));
  }
  if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
}

// space-to-depth for stride-2 narrow convolutions: xs[n][bp][bq][(sr*2+sc)*c + ch]
// = x[n][2bp + sr - ph][2bq + sc - pw][ch] (zero outside x and in slots >= 4c)
__global__ void k_s2d(int nimg, int h, int w, int c, int ph, int pw, int hb, int wb,
                      const __half* __restrict__ x, uint4* __restrict__ xs) {
  pdl_wait();
  pdl_trigger();
  const int total = nimg * hb * wb;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int bq = i % wb, t = i / wb;
    const int bp = t % hb, n = t / hb;
    __align__(16) __half v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __float2half(0.f);
    for (int sub = 0; sub < 4; ++sub) {
      const int ih = 2 * bp + (sub >> 1) - ph, iw = 2 * bq + (sub & 1) - pw;
      if ((unsigned)ih < (unsigned)h && (unsigned)iw < (unsigned)w) {
        const __half* src = x + (((int64_t)n * h + ih) * w + iw) * c;
        for (int ch = 0; ch < c; ++ch) v[sub * c + ch] = src[ch];
      }
    }
    xs[2 * (int64_t)i] = reinterpret_cast<const uint4*>(v)[0];
    xs[2 * (int64_t)i + 1] = reinterpret_cast<const uint4*>(v)[1];
  }
}

// row-concatenated space-to-depth (the stem): x4[n][bp][q][bc*16 + (sr*2+sc)*c + ch]
// = x[n][2bp + sr - ph][2(q + bc) + sc - pw][ch] for block columns bc < 4, so the
// four block taps of one block row are one 64-channel (128 B) pixel and the
// stride-2 convolution becomes an R/2 x 1 stride-1 convolution over 64 channels
// (TMA im2col with 128 B rows instead of four 32 B rows per block row)
__global__ void k_s2d4(int nimg, int h, int w, int c, int ph, int pw, int hb, int q,
                       const __half* __restrict__ x, uint4* __restrict__ x4) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = (int64_t)nimg * hb * q * 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int bc = (int)(i & 3);
    const int64_t pix = i >> 2;
    const int qq = (int)(pix % q);
    const int64_t t = pix / q;
    const int bp = (int)(t % hb), n = (int)(t / hb);
    __align__(16) __half v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __float2half(0.f);
    for (int sub = 0; sub < 4; ++sub) {
      const int ih = 2 * bp + (sub >> 1) - ph, iw = 2 * (qq + bc) + (sub & 1) - pw;
      if ((unsigned)ih < (unsigned)h && (unsigned)iw < (unsigned)w) {
        const __half* src = x + (((int64_t)n * h + ih) * w + iw) * c;
        for (int ch = 0; ch < c; ++ch) v[sub * c + ch] = src[ch];
      }
    }
    x4[2 * i] = reinterpret_cast<const uint4*>(v)[0];
    x4[2 * i + 1] = reinterpret_cast<const uint4*>(v)[1];
  }
}

// k_s2d4 with the two input rows of a block row staged in shared memory
// (coalesced loads; one CTA per (image, block row)); 16 B stores
// RY x4 rows per CTA (2 RY input rows staged in shared memory, 16 B loads when
// the input rows are 16 B multiples), so each CTA's load latency is amortised
// over RY output rows
template <int C>
__global__ void __launch_bounds__(256) k_s2d4_rows(int h, int w, int ph, int pw, int hb, int q,
                                                   const __half* __restrict__ x,
                                                   uint4* __restrict__ x4) {
  constexpr int RY = 4;
  pdl_wait();
  pdl_trigger();
  extern __shared__ __half srow_all[];
  const int groups = (hb + RY - 1) / RY;
  const int Y0 = (blockIdx.x % groups) * RY, n = blockIdx.x / groups;
  const int rowh = w * C;
  const int ny = min(RY, hb - Y0);
  if ((rowh & 7) == 0) {
    const int row8 = rowh >> 3;
    uint4* s8 = reinterpret_cast<uint4*>(srow_all);
    for (int i = threadIdx.x; i < 2 * ny * row8; i += blockDim.x) {
      const int r = i / row8, j = i - r * row8;
      const int ih = 2 * Y0 + r - ph;
      s8[i] = (unsigned)ih < (unsigned)h
                  ? reinterpret_cast<const uint4*>(x + ((int64_t)n * h + ih) * rowh)[j]
                  : make_uint4(0u, 0u, 0u, 0u);
    }
  } else {
    for (int i = threadIdx.x; i < 2 * ny * rowh; i += blockDim.x) {
      const int r = i / rowh, j = i - r * rowh;
      const int ih = 2 * Y0 + r - ph;
      srow_all[i] = (unsigned)ih < (unsigned)h ? x[((int64_t)n * h + ih) * rowh + j]
                                               : __float2half(0.f);
    }
  }
  __syncthreads();
  for (int yy = 0; yy < ny; ++yy) {
  const __half* srow = srow_all + 2 * yy * rowh;
  const int Y = Y0 + yy;
  uint4* dst = x4 + ((int64_t)n * hb + Y) * q * 8;
  for (int i = threadIdx.x; i < q * 8; i += blockDim.x) {
    const int chunk = i & 7, qq = i >> 3;
    const int bc = chunk >> 1;
    __align__(16) __half v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __float2half(0.f);
    if (chunk & 1) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        constexpr int kBase = 8;
        const int slot = kBase + e, sub = slot / C, ch = slot - sub * C;
        if (sub < 4) {
          const int iw = 2 * (qq + bc) + (sub & 1) - pw;
          if ((unsigned)iw < (unsigned)w) v[e] = srow[(sub >> 1) * rowh + iw * C + ch];
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int sub = e / C, ch = e - sub * C;
        if (sub < 4) {
          const int iw = 2 * (qq + bc) + (sub & 1) - pw;
          if ((unsigned)iw < (unsigned)w) v[e] = srow[(sub >> 1) * rowh + iw * C + ch];
        }
      }
    }
    dst[i] = *reinterpret_cast<const uint4*>(v);
  }
  }
}

// W[k][r][s][c] -> w2[k][(br*s2 + bc)*16 + (sr*2+sc)*c + ch] (the space-to-depth filter)
__global__ void k_w_s2d(int k, int fr, int fs, int c, int r2, int s2, const __half* __restrict__ w,
                        __half* __restrict__ w2) {
  pdl_wait();
  pdl_trigger();
  const int kp = r2 * s2 * 16, total = k * kp;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int col = i % kp, row = i / kp;
    const int tap = col >> 4, slot = col & 15;
    const int br = tap / s2, bc = tap - br * s2;
    const int sub = slot / c, ch = slot - sub * c;
    const int r = 2 * br + (sub >> 1), sx = 2 * bc + (sub & 1);
    w2[i] = (sub < 4 && r < fr && sx < fs) ? w[(((int64_t)row * fr + r) * fs + sx) * c + ch]
                                           : __float2half(0.f);
  }
}

// x[n][h][w][c] (c <= 4) -> x4[n][h][w4][4]: image column w at w4 = w + off,
// zero channel and border padding
__global__ void k_pad_c4(int pix4, int w, int w4, int off, int c, const __half* __restrict__ x,
                         uint2* __restrict__ x4) {
  pdl_wait();
  pdl_trigger();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pix4; i += gridDim.x * blockDim.x) {
    const int col = i % w4 - off, nh = i / w4;
    __align__(8) __half v[4] = {__float2half(0.f), __float2half(0.f), __float2half(0.f),
                                __float2half(0.f)};
    if ((unsigned)col < (unsigned)w)
      for (int j = 0; j < c; ++j) v[j] = x[((int64_t)nh * w + col) * c + j];
    x4[i] = *reinterpret_cast<const uint2*>(v);
  }
}

// W[k][r][s][c] -> wp[k][kp] with wp[k][(r*s2 + s)*4 + c], zeros elsewhere
__global__ void k_pad_w_c4(int k, int fr, int fs, int s2, int c, int kp,
                           const __half* __restrict__ w, __half* __restrict__ wp) {
  pdl_wait();
  pdl_trigger();
  const int total = k * kp;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int col = i % kp, row = i / kp;
    const int r = col / (s2 * 4), sx = (col % (s2 * 4)) >> 2, ch = col & 3;
    wp[i] = (r < fr && sx < fs && ch < c) ? w[(((int64_t)row * fr + r) * fs + sx) * c + ch]
                                          : __float2half(0.f);
  }
}

// explicit im2col for convolutions whose channel count is not a multiple of
// 64 (the 3-channel stem): col[m][k] = x(pixel m, tap/channel k), zero pad to
// kp.  One thread per (row m, 8-wide k chunk), 32-bit index math, 16 B stores.
__global__ void k_im2col(ConvGeom g, int M, int kp, const __half* __restrict__ x,
                         __half* __restrict__ col) {
  pdl_wait();
  pdl_trigger();
  const int rsc = g.r * g.s * g.c;
  const int kc = kp >> 3;
  const int total = M * kc;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int j = i % kc, m = i / kc;
    const int q = m % g.q, u = m / g.q;
    const int p = u % g.p, n = u / g.p;
    const int ih0 = p * g.sh - g.ph, iw0 = q * g.sw - g.pw;
    const __half* xb = x + (int64_t)n * g.h * g.w * g.c;
    const int k = j * 8;
    int c = k % g.c, t = k / g.c;
    int sx = t % g.s, r = t / g.s;
    if ((g.c & 7) == 0) {  // the 8 columns are 8 channels of one tap: one 16 B load
      const int ih = ih0 + r, iw = iw0 + sx;
      uint4 u = make_uint4(0u, 0u, 0u, 0u);
      if (k < rsc && (unsigned)ih < (unsigned)g.h && (unsigned)iw < (unsigned)g.w)
        u = *reinterpret_cast<const uint4*>(xb + (ih * g.w + iw) * g.c + c);
      *reinterpret_cast<uint4*>(col + (int64_t)m * kp + j * 8) = u;
      continue;
    }
    __align__(16) __half v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      __half val = __float2half(0.f);
      if (k + e < rsc) {
        const int ih = ih0 + r, iw = iw0 + sx;
        if ((unsigned)ih < (unsigned)g.h && (unsigned)iw < (unsigned)g.w)
          val = xb[(ih * g.w + iw) * g.c + c];
      }
      v[e] = val;
      if (++c == g.c) {
        c = 0;
        if (++sx == g.s) { sx = 0; ++r; }
      }
    }
    *reinterpret_cast<uint4*>(col + (int64_t)m * kp + j * 8) = *reinterpret_cast<const uint4*>(v);
  }
}

__global__ void k_pad_rows(int rows, int cols, int kp, const __half* __restrict__ src,
                           __half* __restrict__ dst) {
  pdl_wait();
  pdl_trigger();
  const int total = rows * kp;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int k = i % kp, r = i / kp;
    dst[i] = k < cols ? src[(int64_t)r * cols + k] : __float2half(0.f);
  }
}

__global__ void k_zero16(int64_t n8, uint4* __restrict__ p) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}

#endif  // NNL_TC_INSTANTIATE

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

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct View {  // a row-major fp16 matrix [rows][cols] with a row stride
  const void* ptr = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;
};

// im2col-mode TMA view of an NHWC tensor (dims C, W, H, N innermost first)
struct Im2colView {
  const void* ptr = nullptr;
  int c = 0, w = 0, h = 0, n = 0;
  int lw = 0, lh = 0, uw = 0, uh = 0;  // bounding-box corners of the window bases
  int sw = 1, sh = 1;                  // traversal strides
  int pixels = 0;                      // pixels per load (tile rows)
  int cbox = 64;                       // channels per pixel per load
  int swz = 128;                       // smem swizzle of the loaded rows (128 or 32 B)
};

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                   cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  }
  return fn;
}

static int make_im2col_tmap(CUtensorMap* tm, const Im2colView& v) {
  EncodeIm2colFn enc = encode_im2col_fn();
  if (!enc) return fail(NNL_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  if (reinterpret_cast<uintptr_t>(v.ptr) & 15) return fail(NNL_ERR_UNSUPPORTED, "im2col base");
  cuuint64_t dims[4] = {(cuuint64_t)v.c, (cuuint64_t)v.w, (cuuint64_t)v.h, (cuuint64_t)v.n};
  cuuint64_t strides[3] = {(cuuint64_t)v.c * 2, (cuuint64_t)v.w * v.c * 2,
                           (cuuint64_t)v.h * v.w * v.c * 2};
  int lower[2] = {v.lw, v.lh}, upper[2] = {v.uw, v.uh};
  cuuint32_t es[4] = {1, (cuuint32_t)v.sw, (cuuint32_t)v.sh, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(v.ptr), dims, strides,
                   lower, upper, (cuuint32_t)v.cbox, (cuuint32_t)v.pixels, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   v.swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NNL_ERR_CUDA, "cuTensorMapEncodeIm2col failed (%d)", (int)r);
  return NNL_OK;
}

static bool use_tma_im2col() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NNL_TC_GATHER");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

static bool use_resident_b() { return nnl_set_tc_resident_b(-1) == 1; }

// 0: never, 1: cost heuristic, 2: whenever eligible (tuning)
static int cta_pair_policy() { return nnl_set_tc_pairs(-1); }

static bool use_tma_store() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NNL_TC_STORE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static int make_tmap(CUtensorMap* tm, const View& v, int box_cols, int box_rows,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(NNL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(v.ptr) & 15) || (v.ld * 2) % 16)
    return fail(NNL_ERR_UNSUPPORTED, "TMA operand not 16-byte aligned");
  cuuint64_t dims[2] = {(cuuint64_t)v.cols, (cuuint64_t)v.rows};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(v.ptr), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
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
  bool remap = false;    // 1x1 strided dgrad: rows scatter to (n, p*sh, q*sw)
  Im2colView im;         // A_IM2COL / B_IM2COL source
  int gh = 0, gw = 0, ish = 1, isw = 1, ilh = 0, ilw = 0, flip = 0;
  int rgh = 0, rgw = 0, rsh = 1, rsw = 1, ra = 0, rb = 0;
  int nclass = 0;        // strided dgrad: number of output parity classes
  int max_grid = 0;      // > 0: cap on the persistent grid (concurrent class GEMMs)
  int ntap = 0;
  uint8_t tap_w[16] = {}, tap_offw[16] = {}, tap_offh[16] = {};
  int cblk = 0, b_kblk = 0, b_tap_stride = 0;
  const void* gsrc = nullptr;
  int64_t ldc = 0;
  int splits = 1, kb_per_split = 0, num_kb = 0, tiles_m = 0, tiles_n = 0, units = 0;
  size_t ws_im2col = 0, ws_wpad = 0, ws_partial = 0;
  int cg = 1;            // 2: CTA-pair (cta_group::2) 256-row tiles
  bool resb = false;     // B resident in shared memory (weight-stationary)
  bool c4 = false;       // narrow-channel path over a 4-channel padded copy of x
  size_t ws_x4 = 0;
  int c4_s2 = 0, c4_w4 = 0, c4_off = 0, c4_pair = 0;
  bool s2d = false;      // stride-2 narrow conv as a stride-1 conv over a 16-channel
  ConvGeom g2;           //   space-to-depth tensor xs with geometry g2
  size_t ws_xs = 0;
  bool s2d4 = false;     //   ... or over the row-concatenated 64-channel x4 (k_s2d4)
  int s2 = 0;            // block-tap columns per block row of the column order
  // spatial tiles (A_TILE4 / A_TILE4MN / B_TILE4), see TcArgs
  bool sp = false;
  bool sp_cls = false;   // strided-dgrad class over spatial tiles: 4D store into the
                         // class's strided view of dx (pixel (ra, rb) + (rsh, rsw) steps)
  int sbw = 0, sbh = 0, sbi = 0, stw = 0, sth = 0, sp_tiles = 0, slw = 0, slh = 0;
  int sgw = 0, sgh = 0;
  bool halo = false;     // A_HALO (see the enum)
  int hl_pitch = 10, hl_r = 3, hl_s = 3;
  const void* sp_a = nullptr;  // tensor of the A boxes: dims (sp_ac, sgw, sgh, n)
  const void* sp_b = nullptr;  // wgrad B boxes: dims (sp_bc, bw_, bh_, n)
  int sp_ac = 0, sp_bc = 0, sp_bw = 0, sp_bh = 0, sp_n = 0;
};

static bool use_tile4() { return nnl_set_tc_tile4(-1) >= 1; }

static int halo_mode() { return nnl_set_tc_halo(-1); }

// 3x3 / stride 1 / pad 1 over one 64-channel block with a 64-wide output: the
// (8 x 16) pixel tiles of A_HALO (grid width a multiple of 8)
static bool halo_layout(const ConvGeom& g, int cin, int w, int h, const void* src, int cout,
                        Plan& pl) {
  if (!halo_mode() || g.r != 3 || g.s != 3 || g.sh != 1 || g.sw != 1 || g.ph != 1 ||
      g.pw != 1 || cin != 64 || cout != 64 || w % 8 || w > 256 || h > 256)
    return false;
  pl.halo = true; pl.sp = true;
  pl.amode = A_HALO; pl.cblk = 1;
  pl.sbw = 8; pl.sbh = 16; pl.sbi = 1;
  pl.stw = w / 8; pl.sth = (h + 15) / 16;
  pl.sp_tiles = pl.stw * pl.sth * g.n;
  pl.slw = -1; pl.slh = -1; pl.sgw = w; pl.sgh = h;
  pl.sp_a = src; pl.sp_ac = 64; pl.sp_bw = w; pl.sp_bh = h; pl.sp_n = g.n;
  pl.M = pl.sp_tiles * BM;
  return true;
}
// tile-interleaved 8-warp epilogues (env NNL_EPI_IL=0: column-split epilogues)
static int epi_il_env() { return nnl_set_tc_epi_il(-1); }
// accumulate-mode outputs through TMA load/store (env NNL_TMA_ACC=0: direct stores)
static bool use_tma_acc_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NNL_TMA_ACC");
    v = e && e[0] == '0' ? 0 : 1;
  }
  return v == 1;
}

static int pow2_div(int v, int cap) {
  int p = 1;
  while (p * 2 <= cap && v % (p * 2) == 0) p *= 2;
  return p;
}

// a (bw x bh x bi) pixel box of `rows` pixels that tiles the (w x h x n) grid
// exactly, with at least 4 pixels per box row group; false if none
static bool sp_box(int w, int h, int n, int rows, Plan& pl) {
  const int bw = pow2_div(w, rows);
  const int bh = pow2_div(h, rows / bw);
  const int bi = rows / (bw * bh);
  if (bw * bh < 4 || n % bi) return false;
  pl.sbw = bw; pl.sbh = bh; pl.sbi = bi;
  pl.stw = w / bw; pl.sth = h / bh;
  pl.sp_tiles = (w / bw) * (h / bh) * (n / bi);
  return true;
}

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// tiled 4D view of an NHWC fp16 tensor (dims C, W, H, N innermost first)
static int make_tmap4(CUtensorMap* tm, const void* ptr, int c, int w, int h, int n,
                      const int box[4], CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                      const int64_t* bstrides = nullptr) {  // byte strides of w, h, n
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(NNL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (c * 2) % 16)
    return fail(NNL_ERR_UNSUPPORTED, "TMA 4D operand not 16-byte aligned");
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
  if (bstrides)
    for (int i = 0; i < 3; ++i) strides[i] = (cuuint64_t)bstrides[i];
  cuuint32_t bx[4] = {(cuuint32_t)box[0], (cuuint32_t)box[1], (cuuint32_t)box[2],
                      (cuuint32_t)box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(ptr), dims, strides,
                   bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NNL_ERR_CUDA, "cuTensorMapEncodeTiled 4D failed (%d)", (int)r);
  return NNL_OK;
}

// tile width with the smallest (waves x per-tile time) cost.  A 128 x BN
// tile's k-step moves (128 + BN) x 64 operand elements through L2 -> SMEM,
// which bounds the mainloop (85 FLOP/B at BN = 256, 64 at 128: measured
// ~13 TB/s aggregate), so per-tile time ~ (128 + BN); ties go to the wider tile
static int pick_bn(const Plan& pl, bool tap_split_b) {
  if (pl.N <= 64) return 64;
  const int sms = num_sms();
  int best = 128;
  double best_cost = 1e30;
  for (int bn : {256, 128}) {
    if (bn == 256 && pl.N <= 128) continue;
    if (tap_split_b && pl.N % bn) continue;  // dgrad B tiles must not straddle taps
    const int64_t units = cdiv(pl.M, BM) * cdiv(pl.N, bn);
    const double cost = (double)cdiv(units, sms) * (128 + bn);
    if (cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  if (tap_split_b && pl.N % best) return 64;
  return best;
}

// Strided dgrad, output parity class (a, b): pixels (y*sh + a, x*sw + b) only
// receive taps r = a+ph (mod sh), s = b+pw (mod sw), reading dy at
// (y + (a+ph-r)/sh, x + (b+pw-s)/sw).  That is a stride-1 im2col GEMM over dy
// with 1..ceil(R/sh)*ceil(S/sw) taps: 9 taps of work in total instead of the
// 4x36 a zero-skipping-free gather would multiply.
static bool strided_class(const ConvGeom& g, int cls, Plan& pl) {
  const int a = cls / g.sw, b = cls % g.sw;
  int tr[16], dr[16], ts[16], ds[16], nr = 0, ns = 0;
  for (int r = 0; r < g.r && nr < 16; ++r) {
    const int x = a + g.ph - r;
    if (((x % g.sh) + g.sh) % g.sh == 0) { tr[nr] = r; dr[nr] = x / g.sh; ++nr; }
  }
  for (int s = 0; s < g.s && ns < 16; ++s) {
    const int x = b + g.pw - s;
    if (((x % g.sw) + g.sw) % g.sw == 0) { ts[ns] = s; ds[ns] = x / g.sw; ++ns; }
  }
  if (nr == 0 || ns == 0 || nr * ns > 16) return false;
  int dmr = dr[0], dms = ds[0];
  for (int i = 1; i < nr; ++i) dmr = dr[i] < dmr ? dr[i] : dmr;
  for (int j = 1; j < ns; ++j) dms = ds[j] < dms ? ds[j] : dms;
  pl.ntap = nr * ns;
  for (int i = 0; i < nr; ++i)
    for (int j = 0; j < ns; ++j) {
      const int t = i * ns + j;
      pl.tap_w[t] = (uint8_t)(tr[i] * g.s + ts[j]);
      pl.tap_offh[t] = (uint8_t)(dr[i] - dmr);
      pl.tap_offw[t] = (uint8_t)(ds[j] - dms);
    }
  const int gh = g.h > a ? (g.h - a + g.sh - 1) / g.sh : 0;
  const int gw = g.w > b ? (g.w - b + g.sw - 1) / g.sw : 0;
  pl.gh = gh; pl.gw = gw; pl.ish = 1; pl.isw = 1; pl.ilh = dmr; pl.ilw = dms;
  pl.rgh = gh; pl.rgw = gw; pl.rsh = g.sh; pl.rsw = g.sw; pl.ra = a; pl.rb = b;
  pl.remap = true;
  return gh > 0 && gw > 0;
}

static bool strided_ok(const ConvGeom& g) {
  for (int c = 0; c < g.sh * g.sw; ++c) {
    Plan tmp;
    if (!strided_class(g, c, tmp)) return false;
  }
  return g.sh * g.sw <= 16;
}

// narrow-channel layout: filter rows padded to an even tap count; with an even
// horizontal stride the x4 copy gets a column shift making tap pairs 16 B loads
static void c4_layout(const ConvGeom& g, Plan& pl) {
  pl.c4 = true;
  pl.c4_s2 = g.s + (g.s & 1);
  pl.c4_pair = g.sw % 2 == 0;
  pl.c4_off = pl.c4_pair ? (g.pw & 1) : 0;
  pl.c4_w4 = g.w + pl.c4_off;
  if (pl.c4_pair) pl.c4_w4 += pl.c4_w4 & 1;
  pl.kp = (int)cdiv((int64_t)g.r * pl.c4_s2 * 4, 64) * 64;
  pl.ws_x4 = (size_t)g.n * g.h * pl.c4_w4 * 8;
}

// space-to-depth eligibility: stride 2, <= 4 channels (4 sub-pixels x c <= 16
// slots), and a block filter whose taps fill whole 64-wide k-blocks
static bool s2d_ok(const ConvGeom& g) {
  const int r2 = (g.r + 1) / 2, s2 = (g.s + 1) / 2;
  return !g.affine && g.sh == 2 && g.sw == 2 && g.c <= 4 && (r2 * s2) % 4 == 0 && g.k % 8 == 0;
}

static bool use_s2d4() { return nnl_set_tc_s2d4(-1) == 1; }

static void s2d_layout(const ConvGeom& g, Plan& pl) {
  pl.s2d = true;
  ConvGeom v = g;
  v.r = (g.r + 1) / 2;
  v.s = (g.s + 1) / 2;
  v.h = g.p + v.r - 1;
  v.sh = v.sw = 1;
  v.ph = v.pw = 0;
  if (v.s <= 4 && use_s2d4()) {
    // x4[n][P + R2 - 1][Q][64]: an R2 x 1 convolution over 64 channels whose
    // reduction index (br, bc*16 + slot) is the s2d filter's with s2 = 4
    pl.s2d4 = true;
    pl.s2 = 4;
    v.s = 1;
    v.w = g.q;
    v.c = 64;
    pl.g2 = v;
    pl.kp = v.r * 64;
    pl.ws_xs = (size_t)g.n * v.h * v.w * 128;
    pl.im = {nullptr, 64, v.w, v.h, g.n, 0, 0, 0, -(v.r - 1), 1, 1, BM, 64, 128};
    pl.cblk = 1;
  } else {
    pl.s2 = v.s;
    v.w = g.q + v.s - 1;
    v.c = 16;
    pl.g2 = v;
    pl.kp = v.r * v.s * 16;
    pl.ws_xs = (size_t)g.n * v.h * v.w * 32;
    // im2col over xs: window bases (y, x) in [0, P) x [0, Q)
    pl.im = {nullptr, 16, v.w, v.h, g.n, 0, 0, -(v.s - 1), -(v.r - 1), 1, 1, BM, 16, 32};
  }
  pl.gh = g.p; pl.gw = g.q; pl.ish = 1; pl.isw = 1; pl.ilh = 0; pl.ilw = 0;
}

// NNL_WG_MAXGRID caps the persistent grid of weight-gradient GEMMs (probes of
// the side-stream overlap: fewer SMs for the off-critical-path wgrads)
static int wg_max_grid() {
  static const int v = getenv("NNL_WG_MAXGRID") ? atoi(getenv("NNL_WG_MAXGRID")) : 0;
  return v;
}

static Plan make_plan(const GemmProblem& pb, int cls = 0) {
  Plan pl;
  const ConvGeom& g = pb.g;
  const bool k1 = g.r == 1 && g.s == 1 && g.ph == 0 && g.pw == 0;
  const bool one = k1 && g.sh == 1 && g.sw == 1;
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
      } else if (!pb.bnx && halo_layout(g, g.c, g.q, g.p, pb.a, g.k, pl)) {
        // A_HALO: B = the nine taps' weights, resident
      } else if (use_tile4() && g.sh == 1 && g.sw == 1 && sp_box(g.q, g.p, g.n, BM, pl)) {
        pl.sp = true;
        pl.amode = A_TILE4; pl.cblk = g.c / 64;
        pl.slw = -g.pw; pl.slh = -g.ph; pl.sgw = g.q; pl.sgh = g.p;
        pl.sp_a = pb.a; pl.sp_ac = g.c; pl.sp_bw = g.w; pl.sp_bh = g.h; pl.sp_n = g.n;
        pl.M = pl.sp_tiles * BM;
      } else if (use_tma_im2col()) {
        pl.amode = A_IM2COL; pl.cblk = g.c / 64;
        pl.im = {pb.a, g.c, g.w, g.h, g.n, -g.pw, -g.ph, g.pw - (g.s - 1), g.ph - (g.r - 1),
                 g.sw, g.sh, BM};
        pl.gh = g.p; pl.gw = g.q; pl.ish = g.sh; pl.isw = g.sw; pl.ilh = -g.ph; pl.ilw = -g.pw;
      } else {
        pl.amode = A_GATHER_FPROP; pl.gsrc = pb.a; pl.cblk = g.c / 64;
      }
    } else if (s2d_ok(g) && use_tma_im2col()) {
      s2d_layout(g, pl);
      pl.K = pl.kp;
      pl.amode = pl.s2d4 ? A_IM2COL : A_IM2COL16;
      pl.bmode = B_TMA_K; pl.B = {nullptr, g.k, pl.kp, pl.kp};
      pl.ws_wpad = (size_t)g.k * pl.kp * 2;
      // the R2 x 1 convolution over x4 from one halo per (8 x 16)-pixel tile:
      // 8-pixel rows, so the tap views start on swizzle-atom boundaries
      if (pl.s2d4 && halo_mode() && g.k == 64 && g.q % 8 == 0 &&
          pl.g2.r + 15 <= 256) {
        pl.halo = true; pl.sp = true;
        pl.amode = A_HALO; pl.cblk = 1;
        pl.hl_pitch = 8; pl.hl_r = pl.g2.r; pl.hl_s = 1;
        pl.sbw = 8; pl.sbh = 16; pl.sbi = 1;
        pl.stw = g.q / 8; pl.sth = (g.p + 15) / 16;
        pl.sp_tiles = pl.stw * pl.sth * g.n;
        pl.slw = 0; pl.slh = 0; pl.sgw = g.q; pl.sgh = g.p;
        pl.sp_ac = 64; pl.sp_bw = pl.g2.w; pl.sp_bh = pl.g2.h; pl.sp_n = g.n;
        pl.M = pl.sp_tiles * BM;
      }
    } else if (g.c <= 4) {
      c4_layout(g, pl);
      pl.K = pl.kp;
      pl.amode = A_GATHER_C4;
      pl.bmode = B_TMA_K; pl.B = {nullptr, g.k, pl.kp, pl.kp};
      pl.ws_wpad = (size_t)g.k * pl.kp * 2;
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
    pl.N = g.c; pl.K = (int)(g.r * g.s * g.k); pl.ldc = g.c;
    pl.bmode = B_TMA_MN; pl.B = {pb.b, g.k, rsc, rsc};
    pl.b_kblk = g.k / 64; pl.b_tap_stride = g.c;
    if (k1) {
      // 1x1: dx(n, p*sh, q*sw) = dy(n,p,q) . W^T, every other input pixel is 0
      pl.M = (int)npq;
      pl.amode = A_TMA_K; pl.A = {pb.a, npq, g.k, g.k};
      pl.remap = !one;
      pl.rgh = g.p; pl.rgw = g.q; pl.rsh = g.sh; pl.rsw = g.sw;
    } else if ((g.sh > 1 || g.sw > 1) && use_tma_im2col() && strided_ok(g) &&
               strided_class(g, cls, pl)) {
      pl.nclass = g.sh * g.sw;
      pl.M = (int)((int64_t)g.n * pl.gh * pl.gw);
      pl.K = pl.ntap * g.k;
      pl.cblk = g.k / 64;
      // spatial tiles over the class grid (one tiled 4D dy box per tap, stored
      // through the class's strided 4D view of dx) when a pixel box tiles it and
      // the classes tile dx exactly; else TMA im2col rows + row-remapped stores
      if (use_tile4() && g.h == pl.gh * g.sh && g.w == pl.gw * g.sw && use_tma_store() &&
          (!pb.acc || use_tma_acc_env()) && !(reinterpret_cast<uintptr_t>(pb.out) & 15) &&
          g.c % 8 == 0 && sp_box(pl.gw, pl.gh, g.n, BM, pl)) {
        pl.sp = true; pl.sp_cls = true; pl.remap = false;
        pl.amode = A_TILE4;
        pl.slw = pl.ilw; pl.slh = pl.ilh; pl.sgw = pl.gw; pl.sgh = pl.gh;
        pl.sp_a = pb.a; pl.sp_ac = g.k; pl.sp_bw = g.q; pl.sp_bh = g.p; pl.sp_n = g.n;
        pl.M = pl.sp_tiles * BM;
      } else {
        pl.amode = A_IM2COL;
        pl.im = {pb.a, g.k, g.q, g.p, g.n, pl.ilw, pl.ilh, pl.gw - g.q + pl.ilw,
                 pl.gh - g.p + pl.ilh, 1, 1, BM};
      }
    } else if (!pb.bnx && halo_layout(g, g.k, g.w, g.h, pb.a, g.c, pl)) {
      pl.flip = 1;  // dgrad: tap t uses weight tap 8 - t (resident B)
    } else if (g.sh == 1 && g.sw == 1 && use_tile4() && sp_box(g.w, g.h, g.n, BM, pl)) {
      // stride-1 dgrad over spatial tiles of dx: tap t reads dy at
      // (x + s + pw-(S-1), y + r + ph-(R-1)) with weight tap R*S-1-t
      pl.sp = true;
      pl.amode = A_TILE4; pl.cblk = g.k / 64; pl.flip = 1;
      pl.slw = g.pw - (g.s - 1); pl.slh = g.ph - (g.r - 1); pl.sgw = g.w; pl.sgh = g.h;
      pl.sp_a = pb.a; pl.sp_ac = g.k; pl.sp_bw = g.q; pl.sp_bh = g.p; pl.sp_n = g.n;
      pl.M = pl.sp_tiles * BM;
    } else if (g.sh == 1 && g.sw == 1 && use_tma_im2col()) {
      // stride-1 dgrad is a convolution of dy with the flipped filter:
      // dx(y,x) = sum_{r',s'} dy(y + ph-(R-1) + r', x + pw-(S-1) + s') W[R-1-r'][S-1-s']
      pl.M = (int)nhw;
      pl.amode = A_IM2COL; pl.cblk = g.k / 64; pl.flip = 1;
      const int lw = g.pw - (g.s - 1), lh = g.ph - (g.r - 1);
      pl.im = {pb.a, g.k, g.q, g.p, g.n, lw, lh, lw + g.w - g.q, lh + g.h - g.p, 1, 1, BM};
      pl.gh = g.h; pl.gw = g.w; pl.ish = 1; pl.isw = 1; pl.ilh = lh; pl.ilw = lw;
    } else {
      pl.M = (int)nhw;
      pl.amode = A_GATHER_DGRAD; pl.gsrc = pb.a; pl.cblk = g.k / 64;
    }
  } else {  // wgrad: dW[k][rsc] = dy^T . im2col(x)
    if (g.k % 8) return pl;
    pl.M = g.k; pl.N = (int)rsc; pl.K = (int)npq; pl.ldc = rsc;
    pl.amode = A_TMA_MN; pl.A = {pb.a, npq, g.k, g.k};
    if (g.c % 64 == 0) {
      if (one) {
        pl.bmode = B_TMA_MN; pl.B = {pb.b, nhw, g.c, g.c};
      } else if (nnl_set_tc_tile4(-1) == 2 && g.sh == 1 && g.sw == 1 && g.k % 64 == 0 &&
                 sp_box(g.q, g.p, g.n, BK, pl)) {
        // k-blocks are 64-pixel boxes of the dy grid: A = dy^T boxes, B = the
        // tap-shifted x boxes (zero outside x)
        pl.sp = true;
        pl.amode = A_TILE4MN; pl.bmode = B_TILE4; pl.cblk = g.c / 64;
        pl.slw = -g.pw; pl.slh = -g.ph;
        pl.sp_a = pb.a; pl.sp_ac = g.k; pl.sgw = g.q; pl.sgh = g.p; pl.sp_n = g.n;
        pl.sp_b = pb.b; pl.sp_bc = g.c; pl.sp_bw = g.w; pl.sp_bh = g.h;
        pl.K = pl.sp_tiles * BK;
      } else if (use_tma_im2col()) {
        pl.bmode = B_IM2COL; pl.cblk = g.c / 64;
        pl.im = {pb.b, g.c, g.w, g.h, g.n, -g.pw, -g.ph, g.pw - (g.s - 1), g.ph - (g.r - 1),
                 g.sw, g.sh, 64};
        pl.gh = g.p; pl.gw = g.q; pl.ish = g.sh; pl.isw = g.sw; pl.ilh = -g.ph; pl.ilw = -g.pw;
      } else {
        pl.bmode = B_GATHER_WGRAD; pl.gsrc = pb.b; pl.cblk = g.c / 64;
      }
    } else if (s2d_ok(g) && use_tma_im2col()) {
      // columns in (block tap, 16-slot) order; the f32 reduction maps them back
      s2d_layout(g, pl);
      pl.im.pixels = 64;
      pl.N = pl.kp;
      pl.bmode = pl.s2d4 ? B_IM2COL : B_IM2COL16;
    } else if (g.c <= 4) {
      // columns in (r, s, 4-channel) order; the f32 reduction maps them back
      c4_layout(g, pl);
      pl.N = pl.kp;
      pl.bmode = B_GATHER_C4;
    } else {
      pl.im2col = true;
      pl.kp = (int)cdiv(rsc, 64) * 64;
      pl.bmode = B_TMA_MN; pl.B = {nullptr, npq, pl.kp, pl.kp};
      pl.ws_im2col = (size_t)npq * pl.kp * 2;
    }
  }
  if (pl.bmode == B_TMA_MN && pl.b_kblk == 0) pl.b_kblk = 1 << 30;
  pl.bn = pick_bn(pl, pl.bmode == B_TMA_MN && pl.b_tap_stride && !k1);
  // weight gradients (long, splittable reductions) with more than 128 output
  // channels: 256 x 256 CTA-pair tiles move the fewest operand bytes per FLOP
  // through L2 -> SMEM (the mainloop bound; measured 0-25 % faster per layer,
  // slower for single-CTA 128-row tiles).  NNL_WG_BN=128 restores the cost model.
  static const int wg_bn = getenv("NNL_WG_BN") ? atoi(getenv("NNL_WG_BN")) : 256;
  if (pb.mode == kWgrad && !pb.g.affine && pl.N > 128 && pl.M > BM && !pl.c4 && !pl.s2d &&
      pl.bmode != B_GATHER_WGRAD && wg_bn == 256)
    pl.bn = 256;
  if (pb.bnx && pl.bn > 128) pl.bn = 128;  // the fused BN-backward epilogue's smem budget
  if (pl.remap && pl.N % pl.bn) pl.bn = 64;
  pl.num_kb = pl.halo ? 1 : (int)cdiv(pl.K, BK);  // A_HALO: one ring stage per tile
  auto tile_and_split = [&](int cg) {
    pl.cg = cg;
    pl.tiles_m = (int)cdiv(pl.M, BM * cg);
    pl.tiles_n = (int)cdiv(pl.N, pl.bn);
    const int tiles = pl.tiles_m * pl.tiles_n;
    // split the reduction when the tile grid cannot fill the machine
    int splits = 1;
    const int sms = num_sms() / cg;  // concurrent work slots (CTAs or CTA pairs)
    if (tiles < sms && pb.stats == nullptr && !pl.remap && pl.amode != A_TILE4 && !pl.halo) {
      // wave-quantisation-aware choice: cost in k-block times of the busiest
      // slot (waves x (k-blocks per unit + epilogue)) plus the f32 partial
      // round trip of the fixed-order reduction (~0.26 us per k-block at
      // 128 x 256, partials at ~6 TB/s)
      int max_s = pl.num_kb / 4 < 4 * sms ? pl.num_kb / 4 : 4 * sms;
      while (max_s > 1 && (double)max_s * pl.M * pl.N * 4.0 > 256e6) --max_s;
      double best = 1e30;
      for (int s = 1; s <= (max_s > 1 ? max_s : 1); ++s) {
        const int64_t waves = cdiv((int64_t)tiles * s, sms);
        const int64_t per = cdiv(pl.num_kb, s);
        if (s > 1 && cdiv(pl.num_kb, per) < s) continue;  // empty splits
        const double red = s > 1 ? (double)s * pl.M * pl.N * 8.0 / 6e12 / 0.26e-6 : 0.0;
        const double cost = (double)waves * (per + 2) + red;
        if (cost < best) {
          best = cost;
          splits = s;
        }
      }
    }
    pl.kb_per_split = (int)cdiv(pl.num_kb, splits);
    pl.splits = (int)cdiv(pl.num_kb, pl.kb_per_split);
    pl.units = tiles * pl.splits;
  };
  tile_and_split(1);
  {
    // CTA pairs (256-row tiles, half the L2 operand traffic per output) pay off
    // once the k-loop is long enough for the mainloop, not the per-tile
    // epilogue, to bound the tile: 256-wide tiles with >= 16 k-blocks per unit
    const bool a_tma = pl.amode == A_TMA_K || pl.amode == A_TMA_MN || pl.amode == A_IM2COL ||
                       pl.amode == A_TILE4 || pl.amode == A_TILE4MN;
    const bool b_tma = pl.bmode == B_TMA_K || pl.bmode == B_TMA_MN || pl.bmode == B_IM2COL ||
                       pl.bmode == B_TILE4;
    // weight gradients always pair (measured: every ResNet-50 wgrad with
    // M > 128 output channels, 5-20 % faster; forward/dgrad tiles only when wide and long)
    const int pol = cta_pair_policy();
    const bool wg = pb.mode == kWgrad && !pb.g.affine;
    if (pol && a_tma && b_tma && pl.bn >= 128 && pl.M > BM && !pb.bnx &&
        (pol == 2 || wg || (pl.bn == 256 && pl.kb_per_split >= 16)))
      tile_and_split(2);
  }
  {
    // weight-stationary: one N tile, no split, all of B within RES_MAX
    const bool b_ok = pl.bmode == B_TMA_K || pl.bmode == B_TMA_MN;
    const bool a_ok = pl.amode == A_TMA_K || pl.amode == A_IM2COL || pl.amode == A_IM2COL16 ||
                      pl.amode == A_TILE4;
    pl.resb = pl.halo || (use_resident_b() && b_ok && a_ok && pl.cg == 1 && pl.tiles_n == 1 &&
                          !pb.bnx && pl.splits == 1 &&
                          (int64_t)pl.num_kb * pl.bn * BK * 2 <= RES_MAX);
  }
  if (pl.splits > 1 || ((pl.c4 || pl.s2d) && pb.mode == kWgrad)) {
    // the stem's halo wgrad (gemm_wgrad3.cu) splits its pixel tiles over every SM
    const int sp = (pl.s2d4 && pb.mode == kWgrad && pl.splits < num_sms()) ? num_sms()
                                                                            : pl.splits;
    pl.ws_partial = (size_t)sp * pl.M * pl.N * 4;
  }
  if (pb.mode == kWgrad && wg_max_grid() > 0) pl.max_grid = wg_max_grid();
  pl.ok = pl.M > 0 && pl.N > 0 && pl.K > 0;
  return pl;
}

static int plan_grid(const Plan& pl) {
  int pairs = num_sms() / pl.cg;
  if (pl.max_grid > 0 && pl.max_grid / pl.cg < pairs) pairs = pl.max_grid / pl.cg > 0 ? pl.max_grid / pl.cg : 1;
  return (pl.units < pairs ? pl.units : pairs) * pl.cg;
}

template <int BN, int AM, int BMD, int CG, int RB = 0, int EP = 0>
static int launch_tc(const Plan& pl, const CUtensorMap& ta, const CUtensorMap& tb,
                     const CUtensorMap& tc, const EpiMaps& em, const TcArgs& args,
                     cudaStream_t st) {
  auto kern = k_tc_gemm<BN, AM, BMD, CG, RB, EP>;
  using C = Cfg<BN, CG, RB, EP, AM == A_HALO>;
  static bool attr = false;
  if (!attr) {
    NNL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)plan_grid(pl));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (CG == 2) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 2;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {  // (common.cuh: programmatic dependent launch)
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  NNL_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, em, args));
  count_launch();
  return NNL_OK;
}

// The kernel instantiations of each tile width live in their own translation
// unit (gemm_tc_bn{64,128,256}.cu include this file with NNL_TC_INSTANTIATE)
// so that the ~90 variants compile in parallel; this TU holds the host side.
template <int BN>
int dispatch_bn(const Plan& pl, const CUtensorMap& ta, const CUtensorMap& tb,
                const CUtensorMap& tc, const EpiMaps& em, const TcArgs& args,
                cudaStream_t st) {
  if (args.bnx) {  // fused BN-backward statistics: dgrad modes, single-CTA tiles <= 128 wide
#define NNL_TC_BNB(AM, BMD)                                                    \
    if (pl.amode == AM && pl.bmode == BMD && pl.cg == 1 && !pl.resb)           \
      return launch_tc<BN, AM, BMD, 1, 0, 1>(pl, ta, tb, tc, em, args, st);
    if constexpr (BN <= 128) {
      NNL_TC_BNB(A_TMA_K, B_TMA_MN)
      NNL_TC_BNB(A_TILE4, B_TMA_MN)
      NNL_TC_BNB(A_IM2COL, B_TMA_MN)
    }
#undef NNL_TC_BNB
    return fail(NNL_ERR_UNSUPPORTED, "no fused BN-backward kernel for mode %d/%d", pl.amode,
                pl.bmode);
  }
#define NNL_TC_CASE(AM, BMD)                                                   \
  if (pl.amode == AM && pl.bmode == BMD && pl.cg == 1 && !pl.resb)             \
    return launch_tc<BN, AM, BMD, 1>(pl, ta, tb, tc, em, args, st);
#define NNL_TC_CASE_RB(AM, BMD)                                                \
  if (pl.amode == AM && pl.bmode == BMD && pl.cg == 1 && pl.resb)              \
    return launch_tc<BN, AM, BMD, 1, 1>(pl, ta, tb, tc, em, args, st);
#define NNL_TC_CASE2(AM, BMD)                                                  \
  if (pl.amode == AM && pl.bmode == BMD && pl.cg == 2)                         \
    return launch_tc<BN, AM, BMD, 2>(pl, ta, tb, tc, em, args, st);
  NNL_TC_CASE(A_TMA_K, B_TMA_K)
  NNL_TC_CASE(A_TMA_K, B_TMA_MN)
  NNL_TC_CASE(A_TMA_MN, B_TMA_MN)
  NNL_TC_CASE(A_GATHER_FPROP, B_TMA_K)
  NNL_TC_CASE(A_GATHER_DGRAD, B_TMA_MN)
  NNL_TC_CASE(A_TMA_MN, B_GATHER_WGRAD)
  NNL_TC_CASE(A_IM2COL, B_TMA_K)
  NNL_TC_CASE(A_IM2COL, B_TMA_MN)
  NNL_TC_CASE(A_TMA_MN, B_IM2COL)
  NNL_TC_CASE(A_GATHER_C4, B_TMA_K)
  NNL_TC_CASE(A_TMA_MN, B_GATHER_C4)
  NNL_TC_CASE(A_IM2COL16, B_TMA_K)
  NNL_TC_CASE(A_TMA_MN, B_IM2COL16)
  NNL_TC_CASE(A_TILE4, B_TMA_K)
  NNL_TC_CASE(A_TILE4, B_TMA_MN)
  NNL_TC_CASE(A_TILE4MN, B_TILE4)
  if constexpr (BN == 64) {
    NNL_TC_CASE_RB(A_HALO, B_TMA_K)
    NNL_TC_CASE_RB(A_HALO, B_TMA_MN)
  }
  NNL_TC_CASE_RB(A_TILE4, B_TMA_K)
  NNL_TC_CASE_RB(A_TILE4, B_TMA_MN)
  NNL_TC_CASE_RB(A_TMA_K, B_TMA_K)
  NNL_TC_CASE_RB(A_TMA_K, B_TMA_MN)
  NNL_TC_CASE_RB(A_IM2COL, B_TMA_K)
  NNL_TC_CASE_RB(A_IM2COL, B_TMA_MN)
  NNL_TC_CASE_RB(A_IM2COL16, B_TMA_K)
  if constexpr (BN >= 128) {
    NNL_TC_CASE2(A_TMA_K, B_TMA_K)
    NNL_TC_CASE2(A_TMA_K, B_TMA_MN)
    NNL_TC_CASE2(A_TMA_MN, B_TMA_MN)
    NNL_TC_CASE2(A_IM2COL, B_TMA_K)
    NNL_TC_CASE2(A_IM2COL, B_TMA_MN)
    NNL_TC_CASE2(A_TMA_MN, B_IM2COL)
    NNL_TC_CASE2(A_TILE4, B_TMA_K)
    NNL_TC_CASE2(A_TILE4, B_TMA_MN)
    NNL_TC_CASE2(A_TILE4MN, B_TILE4)
  }
#undef NNL_TC_CASE
#undef NNL_TC_CASE_RB
#undef NNL_TC_CASE2
  return fail(NNL_ERR_UNSUPPORTED, "no tcgen05 kernel for mode %d/%d cg %d", pl.amode, pl.bmode,
              pl.cg);
}

#ifdef NNL_TC_INSTANTIATE
template int dispatch_bn<NNL_TC_INSTANTIATE>(const Plan&, const CUtensorMap&, const CUtensorMap&,
                                             const CUtensorMap&, const EpiMaps&, const TcArgs&,
                                             cudaStream_t);
#else
extern template int dispatch_bn<64>(const Plan&, const CUtensorMap&, const CUtensorMap&,
                                    const CUtensorMap&, const EpiMaps&, const TcArgs&,
                                    cudaStream_t);
extern template int dispatch_bn<128>(const Plan&, const CUtensorMap&, const CUtensorMap&,
                                     const CUtensorMap&, const EpiMaps&, const TcArgs&,
                                     cudaStream_t);
extern template int dispatch_bn<256>(const Plan&, const CUtensorMap&, const CUtensorMap&,
                                     const CUtensorMap&, const EpiMaps&, const TcArgs&,
                                     cudaStream_t);

bool tc_eligible(const GemmProblem& pb, int dtype) {
  if (dtype != NNL_F16) return false;
  return make_plan(pb).ok;
}

size_t tc_ws_bytes(const GemmProblem& pb) {
  Plan pl = make_plan(pb);
  if (!pl.ok) return 0;
  if (wgrad3_eligible(pb, NNL_F16)) return wgrad3_ws_bytes(pb) + 4 * 256;
  size_t w = pl.ws_im2col + pl.ws_wpad + pl.ws_partial + pl.ws_x4 + pl.ws_xs;
  // strided dgrad: the parity-class GEMMs run concurrently, each in its own
  // slice of the workspace (class_ws)
  for (int cls = 1; cls < pl.nclass; ++cls) {
    Plan q = make_plan(pb, cls);
    w += q.ws_im2col + q.ws_wpad + q.ws_partial + q.ws_x4 + q.ws_xs + 4 * 256;
  }
  return w + 4 * 256;
}

int32_t tc_stat_rows(const GemmProblem& pb, int dtype) {
  if (dtype != NNL_F16) return 0;
  GemmProblem q = pb;
  float dummy;
  q.stats = &dummy;  // stats disable split-K
  Plan pl = make_plan(q);
  if (!pl.ok || pb.mode != kFprop || pb.g.affine || pl.N > Cfg<64>::MAX_STAT_N) return 0;
  // one partial row per persistent CTA
  return plan_grid(pl);
}

int32_t tc_bnb_rows(const GemmProblem& pb, int dtype) {
  if (dtype != NNL_F16 || pb.mode != kDgrad || pb.g.affine) return 0;
  GemmProblem q = pb;
  float dummy;
  q.stats = &dummy;  // no split-K
  q.bnx = &dummy;    // single-CTA tiles
  Plan pl = make_plan(q);
  if (!pl.ok || pl.remap || pl.nclass || pl.N > Cfg<64>::MAX_STAT_N || pl.N % 8) return 0;
  const bool mode_ok = (pl.amode == A_TMA_K && pl.bmode == B_TMA_MN) ||
                       (pl.amode == A_TILE4 && pl.bmode == B_TMA_MN) ||
                       (pl.amode == A_IM2COL && pl.bmode == B_TMA_MN);
  return mode_ok ? plan_grid(pl) : 0;
}

static inline uint8_t* align256(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
}

static int run_plan(const GemmProblem& pb, Plan pl, void* ws, cudaStream_t st);

int tc_splitk_reduce(int M, int N, int splits, const float* partial, __half* out, int64_t ldc,
                     int acc, int32_t* nonfinite, cudaStream_t st) {
  if (N % 4 || ldc % 4) return fail(NNL_ERR_INVALID_ARGUMENT, "split reduction needs N % 4 == 0");
  return launch_reduce4(M, N, splits, partial, nullptr, out, ldc, acc, nonfinite, st);
}

int tc_gemm(const GemmProblem& pb, int dtype, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (dtype != NNL_F16) return NNL_ERR_UNSUPPORTED;
  if (wgrad3_eligible(pb, dtype)) return wgrad3_run(pb, ws, ws_bytes, st);
  Plan p0 = make_plan(pb, 0);
  if (!p0.ok) return NNL_ERR_UNSUPPORTED;
  if (ws_bytes < tc_ws_bytes(pb)) return fail(NNL_ERR_INVALID_ARGUMENT, "tc workspace too small");
  if (!p0.nclass) return run_plan(pb, p0, ws, st);
  // strided dgrad: one GEMM per output parity class (1, 2, 2, 4 taps for 3x3 /
  // stride 2).  The classes write disjoint pixels, so they run CONCURRENTLY:
  // class c on its own stream (forked from / joined into `st` by events), its
  // persistent grid capped at its share of the SMs (by taps), its own slice of
  // the workspace -- one wave of all classes instead of four launches with four
  // tails.  NNL_CLASS_STREAMS=0 serialises them on `st`.
  static const bool conc = !(getenv("NNL_CLASS_STREAMS") && getenv("NNL_CLASS_STREAMS")[0] == '0');
  Plan pls[4];
  int taps = 0;
  const int ncls = p0.nclass < 4 ? p0.nclass : 4;
  for (int cls = 0; cls < ncls; ++cls) {
    pls[cls] = cls ? make_plan(pb, cls) : p0;
    taps += pls[cls].ntap > 0 ? pls[cls].ntap : 1;
  }
  // only when the classes are too small to fill the machine on their own (the
  // 14x14 -> 7x7 layer: 0.106 -> 0.084 ms); large classes lose more to the SM caps
  // than they save in tails (56x56: 0.148 -> 0.195 ms)
  int most = 0;
  for (int cls = 0; cls < ncls; ++cls) most = pls[cls].units > most ? pls[cls].units : most;
  if (!conc || p0.nclass > 4 || most >= 2 * num_sms()) {
    for (int cls = 0; cls < p0.nclass; ++cls) {
      const int rc = run_plan(pb, cls ? make_plan(pb, cls) : p0, ws, st);
      if (rc) return rc;
    }
    return NNL_OK;
  }
  static thread_local cudaStream_t aux[3] = {nullptr, nullptr, nullptr};
  static thread_local cudaEvent_t ev_fork = nullptr, ev_join[3] = {nullptr, nullptr, nullptr};
  if (!ev_fork) {
    NNL_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    for (int i = 0; i < 3; ++i) {
      NNL_CUDA(cudaStreamCreateWithFlags(&aux[i], cudaStreamNonBlocking));
      NNL_CUDA(cudaEventCreateWithFlags(&ev_join[i], cudaEventDisableTiming));
    }
  }
  NNL_CUDA(cudaEventRecord(ev_fork, st));
  uint8_t* w = reinterpret_cast<uint8_t*>(ws);
  size_t left = ws_bytes;
  for (int cls = 0; cls < ncls; ++cls) {
    Plan& pl = pls[cls];
    const int t = pl.ntap > 0 ? pl.ntap : 1;
    pl.max_grid = (num_sms() * t + taps - 1) / taps;
    cudaStream_t cs = cls ? aux[cls - 1] : st;
    if (cls) NNL_CUDA(cudaStreamWaitEvent(cs, ev_fork, 0));
    const int rc = run_plan(pb, pl, w, cs);
    if (rc) return rc;
    const size_t used =
        pl.ws_im2col + pl.ws_wpad + pl.ws_partial + pl.ws_x4 + pl.ws_xs + 4 * 256;
    if (used > left) return fail(NNL_ERR_INVALID_ARGUMENT, "tc workspace too small (classes)");
    w += used;
    left -= used;
  }
  for (int cls = 1; cls < ncls; ++cls) {
    NNL_CUDA(cudaEventRecord(ev_join[cls - 1], aux[cls - 1]));
    NNL_CUDA(cudaStreamWaitEvent(st, ev_join[cls - 1], 0));
  }
  return NNL_OK;
}

static int run_plan(const GemmProblem& pb, Plan pl, void* ws, cudaStream_t st) {
  const ConvGeom& g = pb.g;
  uint8_t* w = align256(reinterpret_cast<uint8_t*>(ws));
  __half* col = nullptr;
  __half* wpad = nullptr;
  float* partial = nullptr;
  __half* x4 = nullptr;
  __half* xs = nullptr;
  if (pl.ws_x4) { x4 = reinterpret_cast<__half*>(w); w = align256(w + pl.ws_x4); }
  if (pl.ws_xs) { xs = reinterpret_cast<__half*>(w); w = align256(w + pl.ws_xs); }
  if (pl.ws_im2col) { col = reinterpret_cast<__half*>(w); w = align256(w + pl.ws_im2col); }
  if (pl.ws_wpad) { wpad = reinterpret_cast<__half*>(w); w = align256(w + pl.ws_wpad); }
  if (pl.ws_partial) partial = reinterpret_cast<float*>(w);
  if (pl.im2col) {
    const __half* src = reinterpret_cast<const __half*>(pb.mode == kFprop ? pb.a : pb.b);
    const int64_t rows = (int64_t)g.n * g.p * g.q;
    if (rows * (pl.kp / 8) >= (1ll << 31)) return fail(NNL_ERR_UNSUPPORTED, "im2col too large");
    launch_k(k_im2col, grid_for(rows * (pl.kp / 8), 256, 148 * 16), 256, 0, st, g, (int)rows, pl.kp,
                                                                          src, col);
    NNL_CHECK_LAUNCH();
    if (pb.mode == kFprop) pl.A.ptr = col; else pl.B.ptr = col;
  }
  // the space-to-depth copy built by a forward stays valid in that workspace for
  // the weight gradient when the caller guarantees nothing else used it in between
  // (nnl_conv2d_prep_reuse, a per-node workspace)
  struct PrepKey {
    const void* xs; const void* src; int n, h, w, c, ph, pw;
  };
  static thread_local PrepKey last_prep = {};
  const __half* prep_src = reinterpret_cast<const __half*>(pb.mode == kFprop ? pb.a : pb.b);
  const PrepKey key = {xs, prep_src, g.n, g.h, g.w, g.c, g.ph, g.pw};
  const bool prep_hit = pl.s2d && pb.mode == kWgrad && nnl_conv2d_prep_reuse(-1) == 1 &&
                        memcmp(&key, &last_prep, sizeof(key)) == 0;
  if (pl.s2d && prep_hit) {  // one use per forward build
    pl.im.ptr = xs;
    pl.sp_a = xs;
    last_prep = PrepKey{};
  }
  if (pl.s2d && !prep_hit) {
    const __half* src = prep_src;
    if (pb.mode == kFprop) last_prep = key;
    else last_prep = PrepKey{};
    const int64_t pix = (int64_t)g.n * pl.g2.h * pl.g2.w;
    if (pix >= (1ll << 31)) return fail(NNL_ERR_UNSUPPORTED, "space-to-depth input too large");
    const bool rows = pl.s2d4 && g.w * g.c * 16 <= 48 * 1024;  // 4 rows x 2 input rows
#define NNL_S2D4_ROWS(CC)                                                                  \
    if (rows && g.c == CC)                                                                 \
      launch_k(k_s2d4_rows<CC>, g.n * ((pl.g2.h + 3) / 4), 256, g.w * g.c * 16, st,            \
          g.h, g.w, g.ph, g.pw, pl.g2.h, pl.g2.w, src, reinterpret_cast<uint4*>(xs));
    NNL_S2D4_ROWS(1) else NNL_S2D4_ROWS(2) else NNL_S2D4_ROWS(3) else NNL_S2D4_ROWS(4)
    else if (pl.s2d4)
      launch_k(k_s2d4, grid_for(pix * 4, 256, 148 * 16), 256, 0, st, 
          g.n, g.h, g.w, g.c, g.ph, g.pw, pl.g2.h, pl.g2.w, src, reinterpret_cast<uint4*>(xs));
    else
      launch_k(k_s2d, grid_for(pix, 256, 148 * 16), 256, 0, st, 
          g.n, g.h, g.w, g.c, g.ph, g.pw, pl.g2.h, pl.g2.w, src, reinterpret_cast<uint4*>(xs));
    NNL_CHECK_LAUNCH();
    pl.im.ptr = xs;
    pl.sp_a = xs;
    if (pb.mode == kFprop) {
      const int total = g.k * pl.kp;
      launch_k(k_w_s2d, grid_for(total, 256), 256, 0, st, g.k, g.r, g.s, g.c, pl.g2.r, pl.s2,
                                                     reinterpret_cast<const __half*>(pb.b), wpad);
      NNL_CHECK_LAUNCH();
      pl.B.ptr = wpad;
    }
  }
  if (pl.c4) {
    const __half* src = reinterpret_cast<const __half*>(pb.mode == kFprop ? pb.a : pb.b);
    const int64_t pix = (int64_t)g.n * g.h * pl.c4_w4;
    if (pix >= (1ll << 31)) return fail(NNL_ERR_UNSUPPORTED, "narrow-channel input too large");
    launch_k(k_pad_c4, grid_for(pix, 256, 148 * 16), 256, 0, st, 
        (int)pix, g.w, pl.c4_w4, pl.c4_off, g.c, src, reinterpret_cast<uint2*>(x4));
    NNL_CHECK_LAUNCH();
    pl.gsrc = x4;
    if (pb.mode == kFprop) {
      const int total = g.k * pl.kp;
      launch_k(k_pad_w_c4, grid_for(total, 256), 256, 0, st, g.k, g.r, g.s, pl.c4_s2, g.c, pl.kp,
                                                        reinterpret_cast<const __half*>(pb.b), wpad);
      NNL_CHECK_LAUNCH();
      pl.B.ptr = wpad;
    }
  }
  if (pl.pad_w) {
    const int total = g.k * pl.kp;
    launch_k(k_pad_rows, grid_for(total, 256), 256, 0, st, g.k, (int)(g.r * g.s * g.c), pl.kp,
                                                      reinterpret_cast<const __half*>(pb.b), wpad);
    NNL_CHECK_LAUNCH();
    pl.B.ptr = wpad;
  }
  if (pl.remap && !pb.acc && !pl.nclass) {  // 1x1 strided: unmapped pixels are exact zeros
    const int64_t n8 = (int64_t)g.n * g.h * g.w * g.c / 8;
    if ((g.c % 8) || (reinterpret_cast<uintptr_t>(pb.out) & 15))
      return fail(NNL_ERR_UNSUPPORTED, "strided dgrad output not 16 B aligned");
    launch_k(k_zero16, grid_for(n8, 256), 256, 0, st, n8, reinterpret_cast<uint4*>(pb.out));
    NNL_CHECK_LAUNCH();
  }
  CUtensorMap ta, tb;
  memset(&ta, 0, sizeof(ta));
  memset(&tb, 0, sizeof(tb));
  int rc;
  if (pl.amode == A_HALO) {  // pitch x (tile rows + R - 1) halo pixels per tile
    const int box[4] = {64, pl.hl_pitch, pl.sbh + pl.hl_r - 1, 1};
    if ((rc = make_tmap4(&ta, pl.sp_a, pl.sp_ac, pl.sp_bw, pl.sp_bh, pl.sp_n, box))) return rc;
  } else if (pl.amode == A_TILE4) {
    const int box[4] = {64, pl.sbw, pl.sbh, pl.sbi};
    if ((rc = make_tmap4(&ta, pl.sp_a, pl.sp_ac, pl.sp_bw, pl.sp_bh, pl.sp_n, box))) return rc;
  } else if (pl.amode == A_TILE4MN) {
    const int box[4] = {64, pl.sbw, pl.sbh, pl.sbi};
    if ((rc = make_tmap4(&ta, pl.sp_a, pl.sp_ac, pl.sgw, pl.sgh, pl.sp_n, box))) return rc;
  } else if (pl.amode == A_TMA_K) {
    if ((rc = make_tmap(&ta, pl.A, 64, BM))) return rc;
  } else if (pl.amode == A_TMA_MN) {
    if ((rc = make_tmap(&ta, pl.A, 64, 64))) return rc;
  } else if (pl.amode == A_IM2COL || pl.amode == A_IM2COL16) {
    if ((rc = make_im2col_tmap(&ta, pl.im))) return rc;
  }
  if (pl.bmode == B_TILE4) {
    const int box[4] = {64, pl.sbw, pl.sbh, pl.sbi};
    if ((rc = make_tmap4(&tb, pl.sp_b, pl.sp_bc, pl.sp_bw, pl.sp_bh, pl.sp_n, box))) return rc;
  } else if (pl.bmode == B_TMA_K) {
    if ((rc = make_tmap(&tb, pl.B, 64, pl.bn / pl.cg))) return rc;
  } else if (pl.bmode == B_TMA_MN) {
    if ((rc = make_tmap(&tb, pl.B, 64, 64))) return rc;
  } else if (pl.bmode == B_IM2COL || pl.bmode == B_IM2COL16) {
    if ((rc = make_im2col_tmap(&tb, pl.im))) return rc;
  }
  TcArgs args;
  memset(&args, 0, sizeof(args));
  auto fd = [](int d) {  // FDiv for 1 <= d < 2^31 (d <= 0: unused, zero)
    FDiv f = {0u, 0u};
    if (d <= 0) return f;
    uint32_t p = 0;
    while ((1ull << p) < (unsigned long long)d) ++p;
    f.m = (uint32_t)(((1ull << 32) * ((1ull << p) - (unsigned long long)d)) / (unsigned long long)d + 1);
    f.s = p;
    return f;
  };
  args.M = pl.M; args.N = pl.N; args.num_kb = pl.num_kb; args.kb_per_split = pl.kb_per_split;
  args.tiles_m = pl.tiles_m; args.tiles_n = pl.tiles_n; args.units = pl.units;
  args.g = pl.s2d ? pl.g2 : g;
  args.gsrc = reinterpret_cast<const __half*>(pl.gsrc);
  args.cblk = pl.cblk; args.b_kblk = pl.b_kblk; args.b_tap_stride = pl.b_tap_stride;
  args.out = pb.out; args.ldc = pl.ldc; args.acc = pb.acc; args.remap = pl.remap;
  args.gh = pl.gh; args.gw = pl.gw; args.ish = pl.ish; args.isw = pl.isw;
  args.ilh = pl.ilh; args.ilw = pl.ilw; args.flip = pl.flip;
  args.rgh = pl.rgh; args.rgw = pl.rgw; args.rsh = pl.rsh; args.rsw = pl.rsw;
  args.ra = pl.ra; args.rb = pl.rb; args.ntap = pl.ntap;
  memcpy(args.tap_w, pl.tap_w, sizeof(args.tap_w));
  memcpy(args.tap_offw, pl.tap_offw, sizeof(args.tap_offw));
  memcpy(args.tap_offh, pl.tap_offh, sizeof(args.tap_offh));
  args.bias = reinterpret_cast<const __half*>(pb.bias);
  args.stats = pb.stats; args.nonfinite = pb.nonfinite;
  args.stat_shift = pb.stats && !pb.bnx ? pb.stat_shift : nullptr;
  if (pb.bnx) {
    if (pl.remap || pl.nclass) return fail(NNL_ERR_UNSUPPORTED, "fused BN backward with remap");
    args.bnx = reinterpret_cast<const __half*>(pb.bnx);
    args.bn_gate = reinterpret_cast<const __half*>(pb.bn_gate);
    args.bn_mean = pb.bn_mean; args.bn_istd = pb.bn_istd;
    args.bn_gamma = pb.bn_gamma; args.bn_beta = pb.bn_beta;
    args.bn_relu = pb.bn_relu; args.bn_canon = pb.bn_canon;
    args.bn_out = reinterpret_cast<__half*>(pb.bn_out ? pb.bn_out : pb.out);
  }
  args.K = pl.K;
  args.sbw = pl.sbw; args.sbh = pl.sbh; args.sbi = pl.sbi; args.stw = pl.stw; args.sth = pl.sth;
  args.sp_tiles = pl.sp_tiles; args.slw = pl.slw; args.slh = pl.slh;
  args.sgw = pl.sgw; args.sgh = pl.sgh;
  args.fd_pers = fd(pl.tiles_m * pl.tiles_n); args.fd_tn = fd(pl.tiles_n);
  args.fd_stw = fd(pl.stw); args.fd_sth = fd(pl.sth);
  args.fd_sbw = fd(pl.sbw); args.fd_sbh = fd(pl.sbh);
  args.fd_rgw = fd(pl.rgw); args.fd_rgh = fd(pl.rgh);
  args.epi_il = epi_il_env();
  args.res_kb = pl.halo ? pl.hl_r * pl.hl_s : 0;
  args.hl_pitch = pl.hl_pitch; args.hl_r = pl.hl_r; args.hl_s = pl.hl_s;
  args.hl_bytes = (uint32_t)(pl.hl_pitch * (pl.sbh + pl.hl_r - 1) * 128);
  args.c4_s2 = pl.c4_s2; args.c4_w4 = pl.c4_w4; args.c4_off = pl.c4_off; args.c4_pair = pl.c4_pair;
  const bool to_partial = pl.splits > 1 || ((pl.c4 || pl.s2d) && pb.mode == kWgrad);
  args.partial = to_partial ? partial : nullptr;
  if (to_partial) {  // bias / accumulate / rounding happen in the reduction
    args.bias = nullptr; args.acc = 0; args.nonfinite = nullptr; args.stats = nullptr;
    if (pl.remap) return fail(NNL_ERR_UNSUPPORTED, "split-K with row remap");
  }
  CUtensorMap tc;
  memset(&tc, 0, sizeof(tc));
  EpiMaps em;
  memset(&em, 0, sizeof(em));
  if (!args.partial && !args.remap && !args.bnx && !(args.acc && args.stats) &&
      (!args.acc || use_tma_acc_env()) && use_tma_store() &&
      !(reinterpret_cast<uintptr_t>(pb.out) & 15) && (pl.ldc * 2) % 16 == 0) {
    View o;
    o.ptr = pb.out; o.rows = pl.M; o.cols = pl.N; o.ld = pl.ldc;
    // the kernel's chunk width (see CW): 32 columns when 8 epilogue warps share BN = 64
    const bool gather = pl.amode == A_GATHER_FPROP || pl.amode == A_GATHER_DGRAD ||
                        pl.amode == A_GATHER_C4 || pl.bmode == B_GATHER_WGRAD ||
                        pl.bmode == B_GATHER_C4;
    const bool cw32 = (!gather && pl.bn == 64) || args.acc;  // acc: 32-column chunks
    const CUtensorMapSwizzle sw = cw32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
    if (pl.amode == A_TILE4 || pl.amode == A_HALO) {  // 32-row sub-boxes over the output grid
      const int bw32 = pl.sbw < 32 ? pl.sbw : 32;
      const int bh32 = pl.sbh < 32 / bw32 ? pl.sbh : 32 / bw32;
      const int box[4] = {cw32 ? 32 : 64, bw32, bh32, 32 / (bw32 * bh32)};
      if (pl.sp_cls) {  // the class pixels (y*rsh + ra, x*rsw + rb) of dx as a 4D view
        const int64_t W = (int64_t)g.w, H = (int64_t)g.h, row = (int64_t)pl.N * 2;
        const int64_t bs[3] = {pl.rsw * row, pl.rsh * W * row, H * W * row};
        const uint8_t* base =
            reinterpret_cast<const uint8_t*>(pb.out) + ((int64_t)pl.ra * W + pl.rb) * row;
        if ((rc = make_tmap4(&tc, base, pl.N, pl.sgw, pl.sgh, pl.sp_n, box, sw, bs))) return rc;
      } else if ((rc = make_tmap4(&tc, pb.out, pl.N, pl.sgw, pl.sgh, pl.sp_n, box, sw))) {
        return rc;
      }
    } else if ((rc = make_tmap(&tc, o, cw32 ? 32 : 64, 32, sw))) {
      return rc;
    }
    args.tma_store = 1;
  }
  if (pl.sp_cls && !args.tma_store)
    return fail(NNL_ERR_UNSUPPORTED, "strided-dgrad spatial class needs the TMA-store epilogue");
  if (pb.bnx) {  // x / gate / prev / gated-output maps: 32 x 32 boxes, 64 B swizzle
    if ((pl.ldc * 2) % 16) return fail(NNL_ERR_UNSUPPORTED, "fused BN-backward: row stride");
    auto map = [&](CUtensorMap* m, const void* ptr) -> int {
      if (pl.amode == A_TILE4) {
        const int bw32 = pl.sbw < 32 ? pl.sbw : 32;
        const int bh32 = pl.sbh < 32 / bw32 ? pl.sbh : 32 / bw32;
        const int box[4] = {32, bw32, bh32, 32 / (bw32 * bh32)};
        return make_tmap4(m, ptr, pl.N, pl.sgw, pl.sgh, pl.sp_n, box, CU_TENSOR_MAP_SWIZZLE_64B);
      }
      View v;
      v.ptr = ptr; v.rows = pl.M; v.cols = pl.N; v.ld = pl.ldc;
      return make_tmap(m, v, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    };
    if ((rc = map(&em.x, pb.bnx))) return rc;
    if (pb.bn_gate && (rc = map(&em.g, pb.bn_gate))) return rc;
    if ((rc = map(&em.o, pb.bn_out ? pb.bn_out : pb.out))) return rc;
    if (pb.acc && (rc = map(&tc, pb.out))) return rc;
    args.tma_store = 0;
  }
  // the stem's weight gradient: halo tiles over x4 (gemm_wgrad3.cu) -- one x4
  // box per 8 x 8 pixel tile for all r2 taps instead of an im2col load per tap
  bool done = false;
  if (pl.s2d4 && pb.mode == kWgrad && to_partial && partial) {
    int used = 0;
    const int max_sp = (int)(pl.ws_partial / ((size_t)pl.M * pl.N * 4));
    rc = wgrad_halo_x4(pl.sp_a, pb.a, g.n, g.p, g.q, g.k, pl.g2.r, partial, max_sp, &used, st);
    if (rc == NNL_OK) {
      pl.splits = used;
      done = true;
    } else if (rc != NNL_ERR_UNSUPPORTED) {
      return rc;
    }
  }
  if (!done) {
    if (pl.bn == 64) rc = dispatch_bn<64>(pl, ta, tb, tc, em, args, st);
    else if (pl.bn == 128) rc = dispatch_bn<128>(pl, ta, tb, tc, em, args, st);
    else rc = dispatch_bn<256>(pl, ta, tb, tc, em, args, st);
    if (rc) return rc;
  }
  if (to_partial) {
    const bool mapped = (pl.c4 || pl.s2d) && pb.mode == kWgrad;
    const int c4 = mapped ? g.c : 0;
    if (!mapped && pl.N % 4 == 0 && pl.ldc % 4 == 0 &&
        !(reinterpret_cast<uintptr_t>(pb.out) & 7))
      return launch_reduce4(pl.M, pl.N, pl.splits, partial,
                            reinterpret_cast<const __half*>(pb.bias),
                            reinterpret_cast<__half*>(pb.out), pl.ldc, pb.acc, pb.nonfinite, st);
    else
      launch_k(k_tc_splitk_reduce, grid_for((int64_t)pl.M * pl.N, 256), 256, 0, st, 
          pl.M, pl.N, pl.splits, partial, reinterpret_cast<const __half*>(pb.bias),
          reinterpret_cast<__half*>(pb.out), pl.ldc, pb.acc, 0, c4,
          pl.s2d ? pl.s2 : pl.c4_s2, g.r, g.s, pl.s2d && pb.mode == kWgrad ? 1 : 0,
          pb.nonfinite);
    NNL_CHECK_LAUNCH();
  }
  return NNL_OK;
}

#endif  // NNL_TC_INSTANTIATE

}  // namespace nnl
