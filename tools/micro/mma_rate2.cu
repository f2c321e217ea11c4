// Microbenchmark 2: N=32 PV-style MMAs (K=16 steps) — TS vs SS, masked vs not, with and
// without concurrent tcgen05.ld traffic from 8 other warps.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2501_06480_b200/csrc/fwa_sm100.cuh"
using namespace fwa::sm100;

__device__ __forceinline__ void ld32(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(addr));
}

// mode bit0: TS (else SS), bit1: masked, bit2: concurrent tcgen05.ld load, bit3: SS with MN-major B
__global__ void k(unsigned long long* out, int iters, int mode, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); done = 0; }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    const uint32_t a = smem_u32(s), b = smem_u32(s + 32768);
    const bool mn = mode & 8;
    const uint32_t id = make_idesc_f16(false, 128, 32, false, mn);
    const uint32_t m0 = (mode & 2) ? 0xffff0000u : 0, m1 = (mode & 2) ? 0xffffffffu : 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        const uint64_t bd = mn ? make_sdesc(b + j * 16 * 64, 9216, 512, 4) : make_sdesc(b + j * 32, 16, 512, 4);
        if (mode & 16) {
          if (mode & 1) mma_f16_ts(t + 256 + 80, t + 256 + j * 8, bd, id, j > 0);
          else mma_f16_ss(t + 256 + 80, make_sdesc(a + j * 32, 16, 1024, 2), bd, id, j > 0);
        } else if (mode & 1)
          mma_f16_ts_m(t + 256 + 80, t + 256 + j * 8, bd, id, j > 0, m0, m1, m1, m1);
        else
          mma_f16_ss_m(t + 256 + 80, make_sdesc(a + j * 32, 16, 1024, 2), bd, id, j > 0, m0, m1, m1, m1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
    done = 1;
  } else if (warp >= 2 && (mode & 4)) {
    uint32_t acc = 0;
    while (!done) {
      uint32_t v[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        ld32(t + ((uint32_t)((warp & 3) * 32) << 16) + c * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= v[j];
      }
    }
    if (acc == 0x12345) sink[0] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(t, 512);
}

int main() {
  unsigned long long* d;
  unsigned* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const int it = 2000;
  const char* names[] = {"SS", "TS", "SS+mask", "TS+mask", "SS+ldload", "TS+ldload", "SS+mask+ld", "TS+mask+ld",
                         "SSmn", "TSmn", "SSmn+mask", "TSmn+mask", "SSmn+ld", "TSmn+ld", "SSmn+m+ld", "TSmn+m+ld"};
  for (int mode : {0, 1, 2, 3, 16, 17, 20, 21, 24, 25}) {
    k<<<1, 320, 70000>>>(d, it, mode, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%-12s plain=%d err=%d cyc/mma=%.1f\n", names[mode & 15], mode >> 4, (int)e, (double)c / (it * 9.0));
  }
  return 0;
}
