// Microbenchmark: tcgen05.ld throughput per SM vs warps, MUFU ex2 rate, STS rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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

template <int MODE>
__global__ void k(unsigned long long* out, int iters, float* sink) {
  __shared__ uint32_t tbase;
  __shared__ uint32_t sbuf[4096];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  float facc = 0.f, x = lane * 0.001f;
  float fa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {  // TMEM loads: 4 x 32 cols then wait
      uint32_t v[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        ld32(t + ((warp >> 2) * 128 + c * 32) % 512, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= v[j];
      }
    } else if (MODE == 1) {  // ex2: 8 independent chains, input depends on i
      float xs = x + i * 1e-6f;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(xs + j * 0.01f));
        fa[j & 7] += y;
      }
    } else {  // STS 16B
#pragma unroll
      for (int j = 0; j < 8; ++j)
        reinterpret_cast<uint4*>(sbuf)[(threadIdx.x * 8 + j * 37 + i) & 1023] = make_uint4(acc, i, j, 1);
    }
  }
  for (int j = 0; j < 8; ++j) facc += fa[j];
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345 || facc == 1.2345f) sink[0] = facc + acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  unsigned long long* d;
  float* s;
  cudaMalloc(&d, 8 * 1024);
  cudaMalloc(&s, 64);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16}) {
      if (mode == 0) k<0><<<1, warps * 32>>>(d, iters, s);
      if (mode == 1) k<1><<<1, warps * 32>>>(d, iters, s);
      if (mode == 2) k<2><<<1, warps * 32>>>(d, iters, s);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long c;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      double per_iter = (double)c / iters;
      double bytes = mode == 0 ? warps * 32.0 * 128 * 4 : (mode == 1 ? warps * 32.0 * 32 : warps * 32.0 * 8 * 16);
      printf("mode=%d warps=%2d err=%d cyc/iter=%.1f  %s/cyc/SM=%.1f\n", mode, warps, (int)e, per_iter,
             mode == 0 ? "TMEM-B" : (mode == 1 ? "ex2" : "STS-B"), bytes / per_iter);
    }
  return 0;
}
