// Microbenchmark 4: N=32 SS MMAs (dV-like) with A/B walking over 96 KB of distinct data,
// optionally with 8 warps doing smem stores and/or tcgen05.ld concurrently.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2501_06480_b200/csrc/fwa_sm100.cuh"
using namespace fwa::sm100;

template <int MODE>  // bit3: tcgen05.fence::after_thread_sync every 8 MMAs; bit0: walk A/B over distinct data; bit1: smem store load; bit2: tmem ld load
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = i * 2654435761u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); done = 0; }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    long long t0 = clock64();
    const uint32_t p0 = smem_u32(s), b0 = smem_u32(s + 98304);
    for (int i = 0; i < iters; ++i) {
      const int w = (MODE & 1) ? (i % 12) : 0;
      if (MODE & 8) tc_fence_after();
      if (MODE & 16) tc_fence_before();
      const uint64_t a = make_sdesc(p0 + w * 8192, 16384, 1024, 2);
      const uint64_t b = make_sdesc(b0 + w * 8192, 8192, 512, 4);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_f16_ss(t + 320, a + ((kk * 2048) >> 4), b + ((kk * 1024) >> 4),
                     make_idesc_f16(false, 128, 32, true, true), 1);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (lane == 0) { out[MODE & 7] = clock64() - t0; done = 1; }
  } else if (warp >= 2) {
    uint32_t acc = 0;
    int it = 0;
    while (!done) {
      if (MODE & 2) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(s + 160000 + ((threadIdx.x * 16 + j * 4096 + it * 16) & 32767)) = make_uint4(acc, j, it, 1);
      }
      if (MODE & 4) {
        uint32_t v[16];
        tmem_ld16(t + ((uint32_t)((warp & 3) * 32) << 16) + (it & 7) * 16, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
      }
      ++it;
    }
    if (acc == 0x1234567) out[7] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(t, 512);
}

template <int MODE>
void run(unsigned long long* d) {
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  k<MODE><<<1, 320, 200000>>>(d, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[8];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  printf("fence_after=%d fence_before=%d walk=%d sts=%d tmemld=%d err=%d cyc/mma=%.1f\n", (MODE >> 3) & 1, (MODE >> 4) & 1, MODE & 1, (MODE >> 1) & 1, (MODE >> 2) & 1, (int)e,
         (double)c[MODE & 7] / 8000.0);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<1>(d); run<9>(d); run<17>(d); run<25>(d);
  return 0;
}
