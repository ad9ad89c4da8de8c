// Microbenchmark: the MMA issue rate inside the warp-specialised pipeline shape
// of the libnnl GEMM kernels (producer warp -> full/empty mbarrier ring -> MMA
// warp issuing G MMAs per stage + tcgen05.commit), no operand loads, against
// the bare back-to-back rate (tools/mma_probe.cu).  Variants: MMAs per stage,
// whether 4 "epilogue" warps spin on an mbarrier meanwhile, and the mbarrier
// wait flavour.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2102_06725_b200/csrc tools/mma_pipe_probe.cu -o tools/mma_pipe_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace nnl::tc;

constexpr int S = 8;

template <int N, int G, bool SPIN>
__global__ void __launch_bounds__(256, 1) k_pipe(int stages_total, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[S], empty[S], done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (warp == 2) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    if ((threadIdx.x & 31) == 0) {
      for (int it = 0; it < stages_total; ++it) {
        const int s = it % S;
        mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
        mbar_arrive(&full[s]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t IDESC = idesc_f16(N, true, true);
    const uint64_t da0 = sdesc_sw128(smem_u32(smem), 8192, 1024);
    const uint64_t db0 = sdesc_sw128(smem_u32(smem) + 16384, 8192, 1024);
    long long t0 = clock64();
    for (int it = 0; it < stages_total; ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int g = 0; g < G; ++g)
          mma_f16(tmem + (uint32_t)((g / 4) % 5 * 64), da0 + (g % 4) * 128, db0 + (g % 4) * 128,
                  IDESC, 1);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&done);
    __syncwarp();
    mbar_wait(&done, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  } else if (warp >= 4 && SPIN) {
    mbar_wait(&done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N, int G, bool SPIN>
static void run(int sms) {
  const int stages_total = 2000;
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int sm = 32768 + 1024;
  cudaFuncSetAttribute(k_pipe<N, G, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k_pipe<N, G, SPIN><<<sms, 256, sm>>>(50, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_pipe<N, G, SPIN><<<sms, 256, sm>>>(stages_total, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c = 0;
  cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
  const double mmas = (double)G * stages_total;
  printf("N=%3d G=%2d spin=%d: %s  %.1f clk/MMA, %.3f ms, %.0f TF/s\n", N, G, (int)SPIN,
         cudaGetErrorString(err), c / mmas, ms, 2.0 * 128 * N * 16 * mmas * sms / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, 20, false>(sms);
  run<64, 20, true>(sms);
  run<64, 4, false>(sms);
  run<64, 4, true>(sms);
  run<128, 4, true>(sms);
  run<256, 4, true>(sms);
  run<64, 80, true>(sms);
  return 0;
}
