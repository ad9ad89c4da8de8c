// Microbenchmark: issue rate of tcgen05.mma.cta_group::1.kind::f16 (M = 128,
// K = 16) from shared memory for N = 64 / 128 / 256, with no operand loads
// (fixed smem tiles), one CTA per SM.  Reports cycles per MMA and the implied
// dense fp16 throughput.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2102_06725_b200/csrc tools/mma_probe.cu -o /tmp/mma_probe -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace nnl::tc;

template <int N, bool MN, int NACC>
__global__ void __launch_bounds__(128, 1) k_probe(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  uint8_t* a = smem;                       // 128 x 64 fp16, SW128 K-major (16 KB)
  uint8_t* b = smem + 16384;               // N x 64 fp16, SW128 K-major
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;  // 1.0h
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t IDESC = idesc_f16(N, MN, MN);
  if (warp == 1) {
    // K-major: K16 step = +32 B; MN-major (64-row K blocks, 8 KB per 64 MN): +2 KB
    const uint64_t da0 = MN ? sdesc_sw128(smem_u32(a), 8192, 1024) : sdesc_sw128(smem_u32(a), 16, 1024);
    const uint64_t db0 = MN ? sdesc_sw128(smem_u32(b), 8192, 1024) : sdesc_sw128(smem_u32(b), 16, 1024);
    constexpr uint64_t step = MN ? 2048 / 16 : 2;
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_f16(tmem + (NACC > 1 ? (it % NACC) * (512 / NACC / 16 * 16) : (it & 1) * N), da0 + kk * step,
                  db0 + kk * step, IDESC, 1);
      }
      mma_commit(&done);
    }
    __syncwarp();
    mbar_wait(&done, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N, bool MN, int NACC>
static void run(int sms) {
  const int iters = 20000;
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int sm = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(k_probe<N, MN, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k_probe<N, MN, NACC><<<sms, 128, sm>>>(100, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_probe<N, MN, NACC><<<sms, 128, sm>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c = 0;
  cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
  const double mmas = 4.0 * iters;
  const double flop = 2.0 * 128 * N * 16 * mmas * sms;
  printf("%s nacc=%d N=%3d: %s  %.1f clk/MMA (SM0 clock64), %.3f ms, %.0f TF/s dense f16\n", MN ? "MN" : "K ", NACC, N,
         cudaGetErrorString(err), c / mmas, ms, flop / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, false, 1>(sms);
  run<128, false, 1>(sms);
  run<256, false, 1>(sms);
  run<64, true, 1>(sms);
  run<128, true, 1>(sms);
  run<256, true, 1>(sms);
  run<64, true, 5>(sms);
  run<128, true, 4>(sms);
  return 0;
}
