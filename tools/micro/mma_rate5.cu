// Microbenchmark 5: cost of switching MMA shape / operand majorness / lane masks between MMAs.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2501_06480_b200/csrc/fwa_sm100.cuh"
using namespace fwa::sm100;

// MODE 0: 8 x dV-like (N=32, MN/MN)            MODE 1: 4 x dV-like + 4 x dQ-like (K/MN) alternating blocks
// MODE 2: 4 x S-like (N=144) + 4 x dV-like      MODE 3: 8 x dQ-like masked
// MODE 4: dV,dQ alternating every MMA            MODE 5: 8 x dV-like, D alternating between 2 regions
template <int MODE>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    const uint32_t p0 = smem_u32(s), b0 = smem_u32(s + 65536), k0 = smem_u32(s + 131072);
    constexpr uint32_t idMN = make_idesc_f16(false, 128, 32, true, true);
    constexpr uint32_t idQ = make_idesc_f16(false, 128, 32, false, true);
    constexpr uint32_t idS = make_idesc_f16(false, 128, 144, false, false);
    const uint64_t adv = make_sdesc(p0, 16384, 1024, 2), bdv = make_sdesc(b0, 8192, 512, 4);
    const uint64_t adq = make_sdesc(p0, 16, 1024, 2), bdq = make_sdesc(k0, 9216, 512, 4);
    const uint64_t as = make_sdesc(b0, 16, 512, 4), bs = make_sdesc(k0, 16, 512, 4);
    for (int i = 0; i < iters; ++i) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const bool dv = MODE == 0 || MODE == 5 || (MODE == 1 && kk < 4) || (MODE == 2 && kk >= 4) ||
                          (MODE == 4 && (kk & 1));
          const bool sl = MODE == 2 && kk < 4;
          if (sl)
            mma_f16_ss(t, as + ((kk & 1) * 2), bs + ((kk & 1) * 2), idS, 1);
          else if (dv)
            mma_f16_ss(t + 320 + (MODE == 5 ? (kk & 1) * 64 : 0), adv + kk * 128, bdv + kk * 64, idMN, 1);
          else
            mma_f16_ss_m(t + 288, adq + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4), bdq + kk * 64, idQ, 1,
                         MODE == 3 ? 0xffff0000u : 0u, 0, 0, 0);
        }
      }
      __syncwarp();
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

template <int MODE>
void run(unsigned long long* d, const char* name) {
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  k<MODE><<<148, 128, 200000>>>(d, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[8];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  printf("%-28s err=%d cyc/8mma=%.1f\n", name, (int)e, (double)c[MODE] / 1000.0);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<0>(d, "8 dV");
  run<1>(d, "4 dV + 4 dQ");
  run<2>(d, "4 S(N144) + 4 dV");
  run<3>(d, "8 dQ masked");
  run<4>(d, "dQ/dV alternating");
  run<5>(d, "8 dV, 2 D regions alt");
  return 0;
}
