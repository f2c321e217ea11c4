// Microbenchmark: latency of n back-to-back N=32 SS MMAs + commit + mbarrier wait.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2501_06480_b200/csrc/fwa_sm100.cuh"
using namespace fwa::sm100;

__global__ void k(unsigned long long* out, int n) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  if (threadIdx.x < 32) {
    const uint64_t a = make_sdesc(smem_u32(s), 16384, 1024, 2), b = make_sdesc(smem_u32(s + 65536), 8192, 512, 4);
    constexpr uint32_t id = make_idesc_f16(false, 128, 32, true, true);
    uint32_t ph = 0;
    long long best = 1 << 30;
    for (int rep = 0; rep < 20; ++rep) {
      long long t0 = clock64();
      if (elect_one()) {
        for (int i = 0; i < n; ++i) mma_f16_ss(t + 256, desc_add(a, (i & 7) * 128), desc_add(b, (i & 7) * 64), id, i > 0);
        mma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, ph);
      ph ^= 1;
      long long dt = clock64() - t0;
      if (dt < best) best = dt;
    }
    if (threadIdx.x == 0) out[0] = best;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(t, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  for (int n : {1, 2, 4, 8, 16, 32}) {
    k<<<1, 128, 140000>>>(d, n);
    cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("n=%2d mma+commit+wait=%llu cycles\n", n, c);
  }
  return 0;
}
