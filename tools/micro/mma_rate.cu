// Microbenchmark: back-to-back tcgen05.mma issue rate (one CTA), SS vs TS, various N / majors.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2501_06480_b200/csrc/fwa_sm100.cuh"
using namespace fwa::sm100;

template <int MODE, int N>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(s), b = smem_u32(s + 32768);
    constexpr uint32_t id = make_idesc_f16(false, 128, N, MODE == 2, MODE == 2);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (MODE == 0 || MODE == 2)
          mma_f16_ss(t + 256, make_sdesc(a + j * 32, 16, 1024, 2), make_sdesc(b + j * 32, 16, 1024, 2), id, true);
        else
          mma_f16_ts(t + 256, t + j * 8, make_sdesc(b + j * 32, 16, 1024, 2), id, true);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[MODE * 8 + (N == 32 ? 0 : N == 64 ? 1 : N == 144 ? 2 : 3)] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(t, 512);
}

template <int MODE, int N>
void run(unsigned long long* d, int iters) {
  cudaFuncSetAttribute(k<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<MODE, N><<<1, 128, 70000>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[32];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  const int idx = MODE * 8 + (N == 32 ? 0 : N == 64 ? 1 : N == 144 ? 2 : 3);
  const double per = (double)c[idx] / (iters * 8.0);
  printf("mode=%s N=%3d err=%d cyc/mma(K=16)=%.1f ideal=%.1f\n",
         MODE == 0 ? "SS-K" : MODE == 1 ? "TS  " : "SS-MN", N, (int)e, per, N / 2.0);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 32 * 8);
  const int it = 4000;
  run<0, 32>(d, it); run<0, 64>(d, it); run<0, 144>(d, it); run<0, 256>(d, it);
  run<1, 32>(d, it); run<1, 64>(d, it); run<1, 144>(d, it); run<1, 256>(d, it);
  run<2, 32>(d, it); run<2, 64>(d, it); run<2, 144>(d, it); run<2, 256>(d, it);
  return 0;
}
