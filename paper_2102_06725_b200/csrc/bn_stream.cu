// Streaming BatchNormalization kernels (fp16, C % 8 == 0, C <= 2048).
//
// An NHWC activation is [rows][C] with rows contiguous, so a chunk of rows is
// one contiguous byte range: thread 0 streams chunks into a 3-stage shared
// memory ring with cp.async.bulk (mbarrier complete_tx), and all 256 threads
// consume them with 8 channels (16 B) per thread.  The bytes in flight live
// in shared memory instead of registers, which is what the register-heavy
// per-channel constants of BN backward otherwise starve.
//
//   STATS_F : (sum x-K, sum (x-K)^2) partial rows, K a per-channel centre
//             (the first row, or the caller's shift)   (functions.py:401-403)
//   APPLY_F : y = q(gamma*((x-mu)*istd)+beta) [+ReLU]   (functions.py:412-416)
//   STATS_B : (sum gy, sum gy*xhat), gy ReLU-gated      (functions.py:421-422)
//   APPLY_B : gx = (g/n)(n gy - gbeta - xhat ggamma)    (functions.py:424-434)
//             [+ conv-bias column sums of the rounded gx]
// f32 expressions keep the reference's op order with _rn intrinsics.
#include "bn_stream.cuh"
#include "tc_ptx.cuh"

namespace nnl {
using namespace tc;

enum BnMode { STATS_F = BNS_STATS_F, APPLY_F = BNS_APPLY_F, STATS_B = BNS_STATS_B,
              APPLY_B = BNS_APPLY_B };

constexpr int kThreads = 256;
constexpr int kChunkBytes = 16384;  // per streamed tensor per stage
// three-tensor launches keep two stages so that two CTAs still fit on an SM:
// the same grid and chunking as the two-tensor launch, hence the same partial
// sums (the fused residual tail is bit-identical to the unfused chain)
__host__ __device__ constexpr int stages(int nt) { return nt == 3 ? 2 : 3; }

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 t = __half22float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}

template <int MODE, int NT>
__global__ void __launch_bounds__(kThreads) k_bn_stream(const BnStreamArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int kStages = stages(NT);
  constexpr bool kGate = NT == 3;                   // backward, ReLU gate streamed
  constexpr bool kRes = MODE == APPLY_F && NT == 2;  // forward, residual streamed
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * NT * kChunkBytes);
  const int tid = threadIdx.x;
  const int groups = a.c >> 3;
  const int lanes = kThreads / groups;
  const int g = tid % groups, lane = tid / groups;
  const bool active = lane < lanes;
  const int c0 = g * 8;

  float m[8], is[8], ga[8], be[8], gn[8], gb[8], gy2[8], s1[8], s2[8], kc[8];
  if (MODE == STATS_F && active) {
    if (a.shift) {
#pragma unroll
      for (int j = 0; j < 8; ++j) kc[j] = a.shift[c0 + j];
    } else {
      unpack8(*reinterpret_cast<const uint4*>(a.x + c0), kc);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    s1[j] = 0.f;
    s2[j] = 0.f;
    if (MODE != STATS_F) {
      m[j] = a.mu[c0 + j];
      is[j] = a.istd[c0 + j];
      ga[j] = a.gamma[c0 + j];
      be[j] = a.beta ? a.beta[c0 + j] : 0.f;
    }
    if (MODE == APPLY_B) {
      const float fn = (float)a.rows;
      gn[j] = __fdiv_rn(__fmul_rn(ga[j], is[j]), fn);  // (gamma*istd)/n
      gb[j] = a.gsum[c0 + j];
      gy2[j] = a.gsum[a.c + c0 + j];
    }
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int s, int64_t chunk) {
    const int64_t r0 = (a.reverse ? a.nchunks - 1 - chunk : chunk) * a.chunk_rows;
    const int64_t nr = min((int64_t)a.chunk_rows, a.rows - r0);
    const uint32_t bytes = (uint32_t)(nr * a.c * 2);
    mbar_arrive_tx(&full[s], bytes * NT);
    bulk_load(smem + (s * NT + 0) * kChunkBytes, a.x + r0 * a.c, bytes, &full[s]);
    if (NT >= 2)
      bulk_load(smem + (s * NT + 1) * kChunkBytes, (kRes ? a.res : a.dy) + r0 * a.c, bytes,
                &full[s]);
    if (NT == 3) bulk_load(smem + (s * NT + 2) * kChunkBytes, a.gate + r0 * a.c, bytes, &full[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      const int64_t ch = blockIdx.x + (int64_t)s * gridDim.x;
      if (ch < a.nchunks) issue(s, ch);
    }
  }
  int it = 0;
  for (int64_t ch = blockIdx.x; ch < a.nchunks; ch += gridDim.x, ++it) {
    const int s = it % kStages;
    mbar_wait(&full[s], (it / kStages) & 1);
    const int64_t r0 = (a.reverse ? a.nchunks - 1 - ch : ch) * a.chunk_rows;
    const int nr = (int)min((int64_t)a.chunk_rows, a.rows - r0);
    const uint8_t* xs = smem + (s * NT + 0) * kChunkBytes;
    const uint8_t* gs = smem + (s * NT + 1) * kChunkBytes;
    const uint8_t* zs = smem + (s * NT + 2) * kChunkBytes;
    if (active) {
      for (int r = lane; r < nr; r += lanes) {
        float xv[8];
        unpack8(*reinterpret_cast<const uint4*>(xs + ((size_t)r * a.c + c0) * 2), xv);
        if (MODE == STATS_F) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float d = __fsub_rn(xv[j], kc[j]);
            s1[j] += d;
            s2[j] = fmaf(d, d, s2[j]);
          }
          continue;
        }
        float xh[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) xh[j] = __fmul_rn(__fsub_rn(xv[j], m[j]), is[j]);
        if (MODE == APPLY_F) {
          __align__(16) __half o[8];
          float rv[8];
          if (kRes) unpack8(*reinterpret_cast<const uint4*>(gs + ((size_t)r * a.c + c0) * 2), rv);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            __half q = __float2half_rn(__fadd_rn(__fmul_rn(ga[j], xh[j]), be[j]));
            if (kRes) q = __float2half_rn(__fadd_rn(__half2float(q), rv[j]));  // Add2: q(a + b)
            if (a.relu) {
              const float f = __half2float(q);
              q = __float2half_rn((f > 0.f || f != f) ? f : 0.f);
            }
            o[j] = q;
          }
          *reinterpret_cast<uint4*>(a.out + (r0 + r) * a.c + c0) =
              *reinterpret_cast<const uint4*>(o);
          continue;
        }
        float gv[8];
        unpack8(*reinterpret_cast<const uint4*>(gs + ((size_t)r * a.c + c0) * 2), gv);
        if (kGate) {  // ReLU after the residual add: gate on its stored output
          float zv[8];
          unpack8(*reinterpret_cast<const uint4*>(zs + ((size_t)r * a.c + c0) * 2), zv);
#pragma unroll
          for (int j = 0; j < 8; ++j) gv[j] = __fmul_rn(gv[j], zv[j] > 0.f ? 1.f : 0.f);
        } else if (a.relu) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float z = __half2float(__float2half_rn(__fadd_rn(__fmul_rn(ga[j], xh[j]), be[j])));
            gv[j] = __fmul_rn(gv[j], z > 0.f ? 1.f : 0.f);
          }
        }
        if (MODE == STATS_B) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            s1[j] += gv[j];
            s2[j] += __fmul_rn(gv[j], xh[j]);
          }
          if (kGate && a.dres) {  // the residual branch's gradient, q(0 + gy)
            __align__(16) __half o[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] = __float2half_rn(__fadd_rn(0.f, gv[j]));
            *reinterpret_cast<uint4*>(a.dres + (r0 + r) * a.c + c0) =
                *reinterpret_cast<const uint4*>(o);
          }
          continue;
        }
        // APPLY_B
        __half* dst = a.out + (r0 + r) * a.c + c0;
        float pv[8];
        if (a.acc) unpack8(*reinterpret_cast<const uint4*>(dst), pv);
        __align__(16) __half o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float res;
          if (a.batch_stat) {
            float t = __fsub_rn(__fmul_rn((float)a.rows, gv[j]), gb[j]);
            t = __fsub_rn(t, __fmul_rn(xh[j], gy2[j]));
            res = __fmul_rn(gn[j], t);
          } else {
            res = __fmul_rn(__fmul_rn(ga[j], is[j]), gv[j]);
          }
          o[j] = __float2half_rn(__fadd_rn(a.acc ? pv[j] : 0.f, res));
          s1[j] += __half2float(o[j]);  // conv-bias column sums of the rounded gx
        }
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(o);
      }
    }
    __syncthreads();  // stage s fully consumed
    if (tid == 0) {
      const int64_t nx = ch + (int64_t)kStages * gridDim.x;
      if (nx < a.nchunks) issue(s, nx);
    }
  }
  if (MODE == APPLY_F || (MODE == APPLY_B && !a.partials)) return;
  // fixed-order block reduction over lanes -> partials[blockIdx.x][2][C]
  float* red = reinterpret_cast<float*>(smem);
  __syncthreads();
  if (active) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      red[(lane * a.c + c0 + j) * 2 + 0] = s1[j];
      red[(lane * a.c + c0 + j) * 2 + 1] = s2[j];
    }
  }
  __syncthreads();
  for (int col = tid; col < a.c; col += kThreads) {
    float t1 = 0.f, t2 = 0.f;
    for (int l = 0; l < lanes; ++l) {
      t1 += red[(l * a.c + col) * 2 + 0];
      t2 += red[(l * a.c + col) * 2 + 1];
    }
    a.partials[(int64_t)blockIdx.x * 2 * a.c + col] = t1;
    a.partials[(int64_t)blockIdx.x * 2 * a.c + a.c + col] = MODE == APPLY_B ? 0.f : t2;
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

bool bn_stream_ok(int64_t rows, int32_t c, const void* a, const void* b, const void* d) {
  return c % 8 == 0 && c >= 8 && c <= 2048 && rows > 0 && aligned16(a) &&
         (!b || aligned16(b)) && (!d || aligned16(d));
}

int bn_stream_nt(int mode, const BnStreamArgs& a) {
  if (mode == STATS_B || mode == APPLY_B) return a.gate ? 3 : 2;
  return (mode == APPLY_F && a.res) ? 2 : 1;
}

int bn_stream_rows(int mode, int nt, int64_t rows, int32_t c) {
  (void)mode;
  // streamed-tensor smem: 1 tensor -> 4 blocks/SM, 2 or 3 tensors -> 2
  int grid = nt == 1 ? 148 * 4 : 148 * 2;
  const int64_t chunk_rows = kChunkBytes / (c * 2);
  const int64_t nchunks = (rows + chunk_rows - 1) / chunk_rows;
  if (grid > nchunks) grid = (int)nchunks;
  return grid;
}

int bn_stream_launch(int mode, const BnStreamArgs& in, cudaStream_t st) {
  BnStreamArgs a = in;
  const int nt = bn_stream_nt(mode, a);
  if (nt == 3 && a.relu) return fail(NNL_ERR_INVALID_ARGUMENT, "gate and fused ReLU both set");
  a.chunk_rows = kChunkBytes / (a.c * 2);
  a.nchunks = (a.rows + a.chunk_rows - 1) / a.chunk_rows;
  const int smem = stages(nt) * nt * kChunkBytes + 64;
  const int grid = bn_stream_rows(mode, nt, a.rows, a.c);
  static bool attr[4][4] = {};
#define NNL_BN_LAUNCH(M, NT)                                                               \
  if (mode == M && nt == NT) {                                                             \
    if (!attr[M][NT]) {                                                                    \
      NNL_CUDA(cudaFuncSetAttribute(k_bn_stream<M, NT>,                                    \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));   \
      attr[M][NT] = true;                                                                  \
    }                                                                                      \
    launch_k(k_bn_stream<M, NT>, grid, kThreads, smem, st, a);                                   \
    NNL_CHECK_LAUNCH();                                                                    \
    return NNL_OK;                                                                         \
  }
  NNL_BN_LAUNCH(STATS_F, 1)
  NNL_BN_LAUNCH(APPLY_F, 1)
  NNL_BN_LAUNCH(APPLY_F, 2)
  NNL_BN_LAUNCH(STATS_B, 2)
  NNL_BN_LAUNCH(STATS_B, 3)
  NNL_BN_LAUNCH(APPLY_B, 2)
  NNL_BN_LAUNCH(APPLY_B, 3)
#undef NNL_BN_LAUNCH
  return fail(NNL_ERR_INVALID_ARGUMENT, "bad bn stream mode");
}

}  // namespace nnl
