// Microbenchmark 7: the flat backward's per-block MMA sequence with the kernel's exact smem
// offsets and operand layouts (L=144, d=32, SW32 P/dS atoms), to compare with the in-kernel rate.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2501_06480_b200/csrc/fwa_sm100.cuh"
using namespace fwa::sm100;

template <int MODE>  // 0: kernel offsets; 1: compact; 2: + commits/waits per group; 3: 2 + runtime masks
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bars[8];
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 215040 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = i * 2654435761u & 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  if (threadIdx.x < 32) {
    const uint32_t base = smem_u32(s);
    const uint32_t p0 = base, ds0 = base + 36864;
    long long t0 = clock64();
    constexpr uint32_t idS = make_idesc_f16(false, 128, 144, false, false);
    constexpr uint32_t idMN = make_idesc_f16(false, 128, 32, true, true);
    constexpr uint32_t idQ = make_idesc_f16(false, 128, 32, false, true);
    for (int i = 0; i < iters; ++i) {
      const int st = i % 3, ks = i % 5;
      const uint32_t q0 = MODE == 0 ? base + 73728 + st * 16384 : base + 73728;
      const uint32_t do0 = q0 + 8192;
      const uint32_t k0 = MODE == 0 ? base + 122880 + ks * 9216 : base + 122880;
      const uint32_t v0 = MODE == 0 ? base + 168960 + ks * 9216 : base + 168960;
      const uint64_t aq = make_sdesc(q0, 16, 512, 4), ado = make_sdesc(do0, 16, 512, 4);
      const uint64_t bk = make_sdesc(k0, 16, 512, 4), bv = make_sdesc(v0, 16, 512, 4);
      const uint64_t ap = make_sdesc(p0, 4096, 256, 6), ads = make_sdesc(ds0, 4096, 256, 6);
      const uint64_t bdo = make_sdesc(do0, 8192, 512, 4), bq = make_sdesc(q0, 8192, 512, 4);
      const uint64_t adq = make_sdesc(ds0, 16, 256, 6), bkq = make_sdesc(k0, 9216, 512, 4);
      uint32_t mk0 = 0xffffu, mk1 = 0;
      if (MODE == 3) {   // runtime masks like blane_off
        const int lo = (i * 16) % 128, hi = 128;
        mk0 = lo >= 32 ? 0xffffffffu : (lo ? ((1u << lo) - 1u) : 0u);
        mk1 = hi > 0 ? 0u : 0xffffffffu;
      }
      if (MODE >= 2 && i > 0) {   // waits on barriers committed one block ago (complete)
        mbar_wait(&bars[0], (i - 1) & 1);
        mbar_wait(&bars[1], (i - 1) & 1);
        tc_fence_after();
      }
      if (elect_one()) {
#pragma unroll
        for (int sg = 0; sg < 2; ++sg) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            mma_f16_ss_m(t, desc_add(aq, kk * 2), desc_add(bk, kk * 2), idS, kk > 0, sg ? mk0 : 0, mk1, 0, 0);
        }
        if (MODE >= 2) mma_commit(&bars[2]);
#pragma unroll
        for (int sg = 0; sg < 2; ++sg) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            mma_f16_ss_m(t + 144, desc_add(ado, kk * 2), desc_add(bv, kk * 2), idS, kk > 0, sg ? 0xffffu : 0, 0, 0, 0);
        }
#pragma unroll
        for (int kt = 0; kt < 2; ++kt)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_f16_ss(t + 320 + kt * 32, desc_add(ap, (kt * 32768 + kk * 512) >> 4), desc_add(bdo, kk * 64), idMN, kk > 0);
#pragma unroll
        for (int kt = 0; kt < 2; ++kt)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_f16_ss(t + 448 + kt * 32, desc_add(ads, (kt * 32768 + kk * 512) >> 4), desc_add(bq, kk * 64), idMN, kk > 0);
#pragma unroll
        for (int sg = 0; sg < 2; ++sg)
#pragma unroll
          for (int kk = 0; kk < 9; ++kk)
            mma_f16_ss_m(t + 288, desc_add(adq, kk * 256), desc_add(bkq, kk * 64), idQ, kk > 0, sg ? mk0 : 0, mk1, 0, 0);
        if (MODE >= 2) {
          mma_commit(&bars[0]);
          mma_commit(&bars[1]);
          mma_commit(&bars[3]);
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
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 228352);
  k<MODE><<<148, 128, 228352>>>(d, 500);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[8];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  printf("%-16s err=%d cyc/block=%.1f\n", name, (int)e, (double)c[MODE] / 500.0);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<0>(d, "kernel offsets");
  run<2>(d, "+commit/wait");
  run<3>(d, "+runtime masks");
  return 0;
}
