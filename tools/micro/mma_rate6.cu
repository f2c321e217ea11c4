// Microbenchmark 6: the flat backward's per-block MMA sequence (L=144, d=32, 2 segments),
// issued back to back from one warp; cycles per block-equivalent.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2501_06480_b200/csrc/fwa_sm100.cuh"
using namespace fwa::sm100;

template <int MODE, int BULK = 0>  // 0 full sequence, 1 only dV/dK, 2 only dQ, 3 only S/dP
__global__ void k(unsigned long long* out, int iters, int klo, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bbar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 180224 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bbar, 1); fence_mbar_init(); done = 0; }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    const uint32_t p0 = smem_u32(s), ds0 = p0 + 49152, q0 = p0 + 98304, do0 = q0 + 8192, k0 = q0 + 16384;
    constexpr uint32_t idS = make_idesc_f16(false, 128, 144, false, false);
    constexpr uint32_t idMN = make_idesc_f16(false, 128, 32, true, true);
    constexpr uint32_t idQ = make_idesc_f16(false, 128, 32, false, true);
    for (int i = 0; i < iters; ++i) {
      const int k_hi = 8;
      if (elect_one()) {
        if (MODE == 0 || MODE == 3) {
#pragma unroll
          for (int sgm = 0; sgm < 2; ++sgm)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              mma_f16_ss_m(t, desc_add(make_sdesc(q0, 16, 512, 4), kk * 2), desc_add(make_sdesc(k0, 16, 512, 4), kk * 2),
                           idS, kk > 0, sgm ? 0xffffu : 0, 0, 0, 0);
              mma_f16_ss_m(t + 144, desc_add(make_sdesc(do0, 16, 512, 4), kk * 2), desc_add(make_sdesc(k0 + 9216, 16, 512, 4), kk * 2),
                           idS, kk > 0, sgm ? 0xffffu : 0, 0, 0, 0);
            }
        }
        if (MODE == 0 || MODE == 1) {
#pragma unroll
          for (int kt = 0; kt < 2; ++kt)
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_f16_ss_p(kk >= klo && kk < k_hi, t + 320 + kt * 32, desc_add(make_sdesc(p0, 16384, 1024, 2), (kt * 32768 + kk * 2048) >> 4),
                           desc_add(make_sdesc(do0, 8192, 512, 4), kk * 64), idMN, kk != klo);
#pragma unroll
          for (int kt = 0; kt < 2; ++kt)
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_f16_ss_p(kk >= klo && kk < k_hi, t + 448 + kt * 32, desc_add(make_sdesc(ds0, 16384, 1024, 2), (kt * 32768 + kk * 2048) >> 4),
                           desc_add(make_sdesc(q0, 8192, 512, 4), kk * 64), idMN, kk != klo);
        }
        if (MODE == 0 || MODE == 2) {
#pragma unroll
          for (int sgm = 0; sgm < 2; ++sgm)
#pragma unroll
            for (int kk = 0; kk < 9; ++kk)
              mma_f16_ss_m(t + 288, desc_add(make_sdesc(ds0, 16, 1024, 2), ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4),
                           desc_add(make_sdesc(k0, 9216, 512, 4), kk * 64), idQ, kk > 0, sgm ? 0xffffu : 0, 0, 0, 0);
        }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) { out[MODE] = clock64() - t0; done = 1; }
  } else if (BULK && threadIdx.x == 32) {
    // bulk global->smem copies (16 KB each) into a scratch region, back to back
    uint32_t ph = 0;
    uint64_t off = (uint64_t)blockIdx.x * 65536;
    while (!done) {
      // BULK copies of 4 KB in flight (the flat kernels keep ~16-48 KB of TMA loads in flight)
      mbar_arrive_expect_tx(&bbar, 4096 * BULK);
      for (int c = 0; c < BULK; ++c)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                     ::"r"(smem_u32(s + 180224 + (c % 4) * 4096)), "l"(gsrc + off + c * 4096), "r"(smem_u32(&bbar)) : "memory");
      mbar_wait(&bbar, ph);
      ph ^= 1;
      off = (off + 4096 * BULK) % (1ull << 30);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(t, 512);
}

template <int MODE, int BULK = 0>
void run(unsigned long long* d, const char* name, int klo, const uint8_t* g) {
  cudaFuncSetAttribute(k<MODE, BULK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  k<MODE, BULK><<<148, 128, 200000>>>(d, 500, klo, g);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[8];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  printf("%-14s bulk=%d err=%d cyc/block=%.1f\n", name, BULK, (int)e, (double)c[MODE] / 500.0);
}

int main(int argc, char** argv) {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int klo = argc > 1 ? atoi(argv[1]) : 0;  // runtime so predicates stay runtime
  uint8_t* g;
  cudaMalloc(&g, (1ull << 30) + 65536);
  run<0>(d, "full", klo, g);
  run<0, 1>(d, "full", klo, g);
  run<0, 4>(d, "full", klo, g);
  run<0, 12>(d, "full", klo, g);
  return 0;
}
