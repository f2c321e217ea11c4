// Microbenchmark 3: back-to-back N=32 MMAs with the flat backward's real operand layouts.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2501_06480_b200/csrc/fwa_sm100.cuh"
using namespace fwa::sm100;

template <int MODE, int CEVERY = 0>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    const uint32_t p0 = smem_u32(s), b0 = smem_u32(s + 65536), k0 = smem_u32(s + 131072);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 0) {  // dV-like: A = P^T MN-major SW128 (LBO 16K), B = dO MN-major SW64
          if (elect_one())
            mma_f16_ss(t + 320, make_sdesc(p0 + kk * 2048, 16384, 1024, 2),
                       make_sdesc(b0 + kk * 16 * 64, 8192, 512, 4), make_idesc_f16(false, 128, 32, true, true), 1);
        } else if (MODE == 1) {  // dQ-like: A = dS K-major SW128, B = K MN-major SW64
          if (elect_one())
            mma_f16_ss(t + 288, make_sdesc(p0 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2),
                       make_sdesc(k0 + kk * 16 * 64, 9216, 512, 4), make_idesc_f16(false, 128, 32, false, true), 1);
        } else if (MODE == 2) {  // S-like: A = Q K-major SW64, B = K K-major SW64, N=144
          if (elect_one())
            mma_f16_ss(t, make_sdesc(b0 + (kk & 1) * 32, 16, 512, 4), make_sdesc(k0 + (kk & 1) * 32, 16, 512, 4),
                       make_idesc_f16(false, 128, 144, false, false), 1);
        } else {  // TS PV-like: A = P in TMEM, B = V MN-major SW64
          if (elect_one())
            mma_f16_ts(t + 320, t + kk * 8, make_sdesc(k0 + kk * 16 * 64, 9216, 512, 4),
                       make_idesc_f16(false, 128, 32, false, true), 1);
        }
        if (CEVERY > 0 && (kk + 1) % CEVERY == 0) {
          if (elect_one()) mma_commit(&bar2);
        }
        __syncwarp();
      }
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[MODE] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(t, 512);
}

template <int MODE, int CE = 0>
void run(unsigned long long* d, const char* name) {
  cudaFuncSetAttribute(k<MODE, CE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  k<MODE, CE><<<1, 128, 200000>>>(d, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[4];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  printf("%-10s commit_every=%d err=%d cyc/mma=%.1f\n", name, CE, (int)e, (double)c[MODE] / 8000.0);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<0>(d, "dV-like");
  run<1>(d, "dQ-like");
  run<2>(d, "S-like");
  run<3>(d, "PV-TS");
  run<0, 1>(d, "dV-like");
  run<0, 2>(d, "dV-like");
  run<0, 4>(d, "dV-like");
  run<0, 8>(d, "dV-like");
  run<3, 1>(d, "PV-TS");
  run<3, 4>(d, "PV-TS");
  return 0;
}
