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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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

// The 3x3 window reduction of 8 fp16 channels (packed, exact: the values are
// fp16).  Fast path: m = NaN-propagating max of the window; the index is the
// first tap equal to m and the output that tap's bits (first max wins, so
// -0/+0 ties keep the first).  Windows with a NaN take the sequential rule
// (NaN wins, first NaN), functions.py:255-271.
__device__ __forceinline__ void pool9_k3(const uint4 (&u)[9], uint4& yo, uint2& a) {
  uint32_t best[4], idx[4];
  bool any_nan = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    auto word = [&](int k) -> uint32_t {
      return q == 0 ? u[k].x : q == 1 ? u[k].y : q == 2 ? u[k].z : u[k].w;
    };
    uint32_t mw = word(0);
    __half2 m = *reinterpret_cast<const __half2*>(&mw);
#pragma unroll
    for (int k = 1; k < 9; ++k) {
      const uint32_t vw = word(k);
      m = __hmax2_nan(m, *reinterpret_cast<const __half2*>(&vw));
    }
    const uint32_t mb = *reinterpret_cast<const uint32_t*>(&m);
    any_nan |= ((mb & 0x7c00u) == 0x7c00u && (mb & 0x03ffu)) ||
               ((mb & 0x7c000000u) == 0x7c000000u && (mb & 0x03ff0000u));
    uint32_t id = 0, val = 0;
#pragma unroll
    for (int k = 8; k >= 0; --k) {
      const uint32_t vw = word(k);
      const uint32_t eq = __heq2_mask(*reinterpret_cast<const __half2*>(&vw), m);
      id = ((uint32_t)k * 0x00010001u & eq) | (id & ~eq);
      val = (vw & eq) | (val & ~eq);
    }
    best[q] = val;
    idx[q] = id;
  }
  if (any_nan) {  // sequential rule, per lane
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t b = 0, id = 0, bnan = 0;
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const uint32_t v = q == 0 ? u[k].x : q == 1 ? u[k].y : q == 2 ? u[k].z : u[k].w;
        const uint32_t vnan = __vcmpgtu2(v & 0x7fff7fffu, 0x7c007c00u);
        if (k == 0) { b = v; bnan = vnan; continue; }
        const uint32_t gt = __hgt2_mask(*reinterpret_cast<const __half2*>(&v),
                                        *reinterpret_cast<const __half2*>(&b));
        const uint32_t upd = gt | (vnan & ~bnan);
        b = (v & upd) | (b & ~upd);
        id = ((uint32_t)k * 0x00010001u & upd) | (id & ~upd);
        bnan |= vnan;
      }
      best[q] = b;
      idx[q] = id;
    }
  }
  yo = make_uint4(best[0], best[1], best[2], best[3]);
  a.x = (idx[0] & 0xffu) | ((idx[0] >> 16) << 8) | ((idx[1] & 0xffu) << 16) | ((idx[1] >> 16) << 24);
  a.y = (idx[2] & 0xffu) | ((idx[2] >> 16) << 8) | ((idx[3] & 0xffu) << 16) | ((idx[3] >> 16) << 24);
}

// 3x3 stride-2 windows (the ResNet stem pool), fully unrolled: the nine 16 B
// window loads of a thread are independent and issued together (the generic
// loop above keeps one in flight), then reduced in row-major window order with
// the same first-max / NaN-wins rule (functions.py:255-271).
__global__ void __launch_bounds__(256) k_maxpool_fwd_k3s2(nnl_pool_shape ps,
                                                          const uint4* __restrict__ x,
                                                          uint4* __restrict__ y,
                                                          uint2* __restrict__ arg) {
  pdl_wait();
  pdl_trigger();
  const int cg = ps.c >> 3;
  const int total = ps.n * ps.p * ps.q * cg;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % cg;
    int t = i / cg;
    const int oq = t % ps.q;
    t /= ps.q;
    const int op = t % ps.p;
    const int b = t / ps.p;
    const int h0 = op * 2 - ps.ph, w0 = oq * 2 - ps.pw;
    uint4 u[9];
#pragma unroll
    for (int di = 0; di < 3; ++di)
#pragma unroll
      for (int dj = 0; dj < 3; ++dj) {
        const int ih = h0 + di, iw = w0 + dj;
        u[di * 3 + dj] = (unsigned)ih < (unsigned)ps.h && (unsigned)iw < (unsigned)ps.w
                             ? __ldg(x + ((int64_t)(b * ps.h + ih) * ps.w + iw) * cg + g)
                             : make_uint4(0xfc00fc00u, 0xfc00fc00u, 0xfc00fc00u, 0xfc00fc00u);
      }
    uint4 yo;
    uint2 a;
    pool9_k3(u, yo, a);
    y[i] = yo;
    arg[i] = a;
  }
}

// Same, one CTA per (image, output row): the three input rows of the windows
// are staged in shared memory with coalesced 16 B loads (adjacent output rows
// share one input row through L2), then each thread reduces windows from
// shared memory.  Used when three input rows fit in 48 KB.
__global__ void __launch_bounds__(256) k_maxpool_fwd_k3s2_rows(nnl_pool_shape ps,
                                                               const uint4* __restrict__ x,
                                                               uint4* __restrict__ y,
                                                               uint2* __restrict__ arg) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint4 rows[];
  const int cg = ps.c >> 3, rowv = ps.w * cg;
  const int op = blockIdx.x % ps.p, b = blockIdx.x / ps.p;
  const int h0 = op * 2 - ps.ph;
#pragma unroll 4
  for (int i = threadIdx.x; i < 3 * rowv; i += blockDim.x) {
    const int r = i / rowv, j = i - r * rowv;
    const int ih = h0 + r;
    rows[i] = (unsigned)ih < (unsigned)ps.h ? __ldg(x + (int64_t)(b * ps.h + ih) * rowv + j)
                                            : make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  // packed fp16 (exact: the values are fp16).  Fast path: m = NaN-propagating
  // max of the window; the index is the first tap equal to m and the output
  // that tap's bits (first max wins, so -0/+0 ties keep the first).  Windows
  // with a NaN take the sequential rule (NaN wins, first NaN).
  constexpr uint32_t kNegInf = 0xfc00fc00u;
  for (int i = threadIdx.x; i < ps.q * cg; i += blockDim.x) {
    const int g = i % cg, oq = i / cg;
    const int w0 = oq * 2 - ps.pw;
    uint4 u[9];
#pragma unroll
    for (int di = 0; di < 3; ++di) {
      const bool rin = (unsigned)(h0 + di) < (unsigned)ps.h;
      const uint4* rp = rows + di * rowv + g;
#pragma unroll
      for (int dj = 0; dj < 3; ++dj) {
        const int iw = w0 + dj;
        u[di * 3 + dj] = rin && (unsigned)iw < (unsigned)ps.w
                             ? rp[iw * cg] : make_uint4(kNegInf, kNegInf, kNegInf, kNegInf);
      }
    }
    uint4 yo;
    uint2 a;
    pool9_k3(u, yo, a);
    const int64_t oi = ((int64_t)(b * ps.p + op) * ps.q + oq) * cg + g;
    y[oi] = yo;
    arg[oi] = a;
  }
}

// BatchNormalization -> ReLU -> 3x3 / stride-2 max pool in one pass (the ResNet
// stem; engine fusion, clear_buffer=True): one CTA per (image, output row) stages
// the three input rows of x = the BN input, applied as the separate BN-apply
// pass would -- z = q(gamma * ((x - mean) * istd) + beta) with f32 RN steps
// (functions.py:412-416, bn_stream.cu APPLY_F) in packed f32x2 ops, then
// ReLU with NaN passing and -0 -> +0 -- and pools z with the same first-max /
// NaN-wins rule as the plain pool (pool9_k3).  z itself is never written: the
// pool's backward uses its argmax, BN's backward recomputes the gate from x.
__global__ void __launch_bounds__(256) k_bn_relu_maxpool_k3s2_rows(
    nnl_pool_shape ps, const uint4* __restrict__ x, const float* __restrict__ gamma,
    const float* __restrict__ beta, const float* __restrict__ mean,
    const float* __restrict__ istd, uint4* __restrict__ y, uint2* __restrict__ arg) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint4 rows[];
  const int cg = ps.c >> 3, rowv = ps.w * cg;
  // a thread's staged vectors are all of channel group threadIdx.x % cg (cg
  // divides the block and the row): its eight channels' constants in registers
  const int c8 = (threadIdx.x % cg) * 8;
  float2 nm[4], is2[4], ga2[4], be2[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int c = c8 + 2 * e;
    nm[e] = make_float2(-mean[c], -mean[c + 1]);
    is2[e] = make_float2(istd[c], istd[c + 1]);
    ga2[e] = make_float2(gamma[c], gamma[c + 1]);
    be2[e] = beta ? make_float2(beta[c], beta[c + 1]) : make_float2(0.f, 0.f);
  }
  const int op = blockIdx.x % ps.p, b = blockIdx.x / ps.p;
  const int h0 = op * 2 - ps.ph;
  // eight 16 B loads in flight per thread before any is used (one memory
  // latency per batch instead of one per element)
  constexpr int kB = 8;
  for (int i0 = threadIdx.x; i0 < 3 * rowv; i0 += kB * blockDim.x) {
    uint4 vb[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int i = i0 + k * blockDim.x;
      const int r = i / rowv, j = i - r * rowv;
      vb[k] = i < 3 * rowv && (unsigned)(h0 + r) < (unsigned)ps.h
                  ? __ldg(x + (int64_t)(b * ps.h + h0 + r) * rowv + j)
                  : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < kB; ++k) {
    const int i = i0 + k * blockDim.x;
    if (i >= 3 * rowv) break;
    const int r = i / rowv;
    const int ih = h0 + r;
    uint4 o = make_uint4(0, 0, 0, 0);
    if ((unsigned)ih < (unsigned)ps.h) {
      const uint4 v = vb[k];
      const uint32_t* vw = reinterpret_cast<const uint32_t*>(&v);
      uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 xv = __half22float2(*reinterpret_cast<const __half2*>(&vw[e]));
        const float2 xh = __fmul2_rn(__fadd2_rn(xv, nm[e]), is2[e]);
        const float2 zf = __fadd2_rn(__fmul2_rn(ga2[e], xh), be2[e]);
        const __half2 q = __floats2half2_rn(zf.x, zf.y);
        const uint32_t qw = *reinterpret_cast<const uint32_t*>(&q);
        // ReLU: keep q > 0 and NaN, everything else (negatives, -0) becomes +0
        const uint32_t keep = __hgt2_mask(q, __float2half2_rn(0.f)) |
                              __vcmpgtu2(qw & 0x7fff7fffu, 0x7c007c00u);
        ow[e] = qw & keep;
      }
    }
    rows[i] = o;
    }
  }
  __syncthreads();
  constexpr uint32_t kNegInf = 0xfc00fc00u;
  for (int i = threadIdx.x; i < ps.q * cg; i += blockDim.x) {
    const int g = i % cg, oq = i / cg;
    const int w0 = oq * 2 - ps.pw;
    uint4 u[9];
#pragma unroll
    for (int di = 0; di < 3; ++di) {
      const bool rin = (unsigned)(h0 + di) < (unsigned)ps.h;
      const uint4* rp = rows + di * rowv + g;
#pragma unroll
      for (int dj = 0; dj < 3; ++dj) {
        const int iw = w0 + dj;
        u[di * 3 + dj] = rin && (unsigned)iw < (unsigned)ps.w
                             ? rp[iw * cg] : make_uint4(kNegInf, kNegInf, kNegInf, kNegInf);
      }
    }
    uint4 yo;
    uint2 a;
    pool9_k3(u, yo, a);
    const int64_t oi = ((int64_t)(b * ps.p + op) * ps.q + oq) * cg + g;
    y[oi] = yo;
    arg[oi] = a;
  }
}

// Backward of the 3x3 / stride 2 / pad 1 pool: one thread per 2x2 input block
// (2a..2a+1, 2b..2b+1) x 8 channels.  Those four pixels are only reached by
// outputs (a..a+1, b..b+1): 4 dy + 4 index loads for 4 pixels, summed per
// pixel in ascending output order (np.add.at order, functions.py:284-288),
// f32, one rounding.
__global__ void __launch_bounds__(256) k_maxpool_bwd_k3s2p1(nnl_pool_shape ps,
                                                            const uint4* __restrict__ dy,
                                                            const uint2* __restrict__ arg,
                                                            uint4* __restrict__ dx, int acc) {
  pdl_wait();
  pdl_trigger();
  const int cg = ps.c >> 3;
  const int hb = (ps.h + 1) >> 1, wb = (ps.w + 1) >> 1;
  const int total = ps.n * hb * wb * cg;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % cg;
    int t = i / cg;
    const int bb = t % wb;
    t /= wb;
    const int ba = t % hb;
    const int n = t / hb;
    uint4 d[2][2];
    uint2 ix[2][2];
    bool ok[2][2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int op = ba + r, oq = bb + c;
        ok[r][c] = op < ps.p && oq < ps.q;
        const int64_t o = ((int64_t)(n * ps.p + op) * ps.q + oq) * cg + g;
        d[r][c] = ok[r][c] ? __ldg(dy + o) : make_uint4(0, 0, 0, 0);
        ix[r][c] = ok[r][c] ? __ldg(arg + o) : make_uint2(0xffffffffu, 0xffffffffu);
      }
#pragma unroll
    for (int ey = 0; ey < 2; ++ey)
#pragma unroll
      for (int ex = 0; ex < 2; ++ex) {
        const int ih = 2 * ba + ey, iw = 2 * bb + ex;
        if (ih >= ps.h || iw >= ps.w) continue;
        float s[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] = 0.f;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          if (r > ey) continue;  // even rows are only in window row a
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (c > ex) continue;
            // window offsets of (ih, iw) inside output (ba + r, bb + c)
            const uint32_t want = (uint32_t)((ih + 1 - 2 * (ba + r)) * 3 + (iw + 1 - 2 * (bb + c)));
            const __half* h = reinterpret_cast<const __half*>(&d[r][c]);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t word = j < 4 ? ix[r][c].x : ix[r][c].y;
              if (((word >> (8 * (j & 3))) & 0xffu) == want) s[j] = __fadd_rn(s[j], __half2float(h[j]));
            }
          }
        }
        const int64_t o = ((int64_t)(n * ps.h + ih) * ps.w + iw) * cg + g;
        uint4 prev = acc ? dx[o] : make_uint4(0, 0, 0, 0);
        __half* ph = reinterpret_cast<__half*>(&prev);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          ph[j] = __float2half_rn(__fadd_rn(acc ? __half2float(ph[j]) : 0.f, s[j]));
        dx[o] = prev;
      }
  }
}

__global__ void k_maxpool_bwd_h8(nnl_pool_shape ps, const uint4* __restrict__ dy,
                                 const uint2* __restrict__ arg, uint4* __restrict__ dx, int acc) {
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
    const int rows_bytes = 3 * ps->w * ps->c * 2;
    static const bool staged = getenv("NNL_POOL_ROWS") && getenv("NNL_POOL_ROWS")[0] == '1';
    if (staged && ps->kh == 3 && ps->kw == 3 && ps->sh == 2 && ps->sw == 2 &&
        rows_bytes <= 48 * 1024)
      launch_k(k_maxpool_fwd_k3s2_rows, ps->n * ps->p, 256, rows_bytes, as_stream(stream), 
          *ps, (const uint4*)x, (uint4*)y, (uint2*)argmax);
    else if (ps->kh == 3 && ps->kw == 3 && ps->sh == 2 && ps->sw == 2)
      launch_k(k_maxpool_fwd_k3s2, grid_for(total / 8, 256), 256, 0, as_stream(stream), 
          *ps, (const uint4*)x, (uint4*)y, (uint2*)argmax);
    else
      launch_k(k_maxpool_fwd_h8, grid_for(total / 8, 256), 256, 0, as_stream(stream), 
          *ps, (const uint4*)x, (uint4*)y, (uint2*)argmax);
    NNL_CHECK_LAUNCH();
    return NNL_OK;
  }
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_maxpool_fwd<T>, grid_for(total, 256), 256, 0, as_stream(stream), *ps, (const T*)x,
                                                                          (T*)y, argmax);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

int nnl_bn_relu_maxpool_ok(int dtype, const nnl_pool_shape* ps) {
  return ps && dtype == NNL_F16 && ps->c % 8 == 0 && ps->kh == 3 && ps->kw == 3 &&
         ps->sh == 2 && ps->sw == 2 && 3 * ps->w * ps->c * 2 <= 48 * 1024 &&
         256 % (ps->c / 8) == 0 &&
         (int64_t)ps->n * ps->h * ps->w * ps->c < (1ll << 31);
}

int nnl_bn_relu_maxpool_fwd(int dtype, const nnl_pool_shape* ps, const void* x,
                            const float* gamma, const float* beta, const float* save_mean,
                            const float* save_istd, void* y, uint8_t* argmax, void* stream) {
  if (!ps) return fail(NNL_ERR_INVALID_ARGUMENT, "null pool shape");
  const int rows_bytes = 3 * ps->w * ps->c * 2;
  if (!nnl_bn_relu_maxpool_ok(dtype, ps))
    return fail(NNL_ERR_UNSUPPORTED, "fused BN-ReLU-maxpool: fp16, C %% 8 == 0, 3x3 / stride 2");
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
        reinterpret_cast<uintptr_t>(argmax)) & 15) != 0)
    return fail(NNL_ERR_UNSUPPORTED, "fused BN-ReLU-maxpool: buffers not 16 B aligned");
  if ((int64_t)ps->n * ps->p * ps->q * ps->c <= 0) return NNL_OK;
  launch_k(k_bn_relu_maxpool_k3s2_rows, ps->n * ps->p, 256, rows_bytes, as_stream(stream),
           *ps, (const uint4*)x, gamma, beta, save_mean, save_istd, (uint4*)y, (uint2*)argmax);
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
    if (ps->kh == 3 && ps->kw == 3 && ps->sh == 2 && ps->sw == 2 && ps->ph == 1 && ps->pw == 1)
      launch_k(k_maxpool_bwd_k3s2p1, grid_for((int64_t)ps->n * ((ps->h + 1) / 2) * ((ps->w + 1) / 2) *
                                          (ps->c / 8), 256), 256, 0, as_stream(stream), *ps, (const uint4*)dy,
                                                          (const uint2*)argmax, (uint4*)dx,
                                                          accumulate);
    else
      launch_k(k_maxpool_bwd_h8, grid_for(total / 8, 256), 256, 0, as_stream(stream), 
          *ps, (const uint4*)dy, (const uint2*)argmax, (uint4*)dx, accumulate);
    NNL_CHECK_LAUNCH();
    return NNL_OK;
  }
  NNL_DISPATCH_DTYPE(dtype, T, {
    launch_k(k_maxpool_bwd<T>, grid_for(total, 256), 256, 0, as_stream(stream), 
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
    launch_k(k_sce_rows<T>, (int)((batch + warps - 1) / warps), warps * 32, 0, as_stream(stream), 
        batch, classes, (const T*)logits, (const T*)labels, row_stats, label_err);
    NNL_CHECK_LAUNCH();
    launch_k(k_sce_loss<T>, 1, 256, 0, as_stream(stream), batch, row_stats, (T*)loss_out);
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
    launch_k(k_sce_bwd<T>, grid_for(total, 256), 256, 0, as_stream(stream), 
        batch, classes, (const T*)logits, (const T*)labels, row_stats, (const T*)gloss,
        (T*)glogits, accumulate);
  });
  NNL_CHECK_LAUNCH();
  return NNL_OK;
}

}  // extern "C"
