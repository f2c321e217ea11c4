// L2 vector-reduction throughput: red.global.add.v4.f32 with lanes one row apart (each
// lane its own sector, the flat backward's dBias pattern) vs lanes 16 B apart (a warp
// covers 512 contiguous bytes). Each CTA reduces into its own [rows][L] fp32 slice.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_rate red_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int L = 144, ROWS = 576;   // 4 heads x 144 query rows per CTA slice (332 KB)

template <bool ROWWISE>
__global__ void red_kernel(float* ws, int iters) {
  float4* slice = reinterpret_cast<float4*>(ws + (size_t)blockIdx.x * ROWS * L);
  const int t = threadIdx.x;   // 256 threads
  const float4 one = make_float4(1.f, 1.f, 1.f, 1.f);
  for (int it = 0; it < iters; ++it) {
    const int row0 = (it * 128) % ROWS;
    if (ROWWISE) {   // thread = row (t & 127), half the keys each (t >> 7): 18 float4
      const int r = row0 + (t & 127), h = t >> 7;
      float4* p = slice + (size_t)(r % ROWS) * (L / 4) + h * (L / 8);
#pragma unroll
      for (int c = 0; c < L / 8; ++c) atomicAdd(p + c, one);
    } else {   // 128 rows x 36 float4, consecutive threads on consecutive float4s
#pragma unroll 6
      for (int k = 0; k < 18; ++k) {
        const int item = t + k * 256;
        const int r = row0 + item / 36, c = item % 36;
        atomicAdd(slice + (size_t)(r % ROWS) * (L / 4) + c, one);
      }
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* ws;
  const size_t bytes = (size_t)sms * ROWS * L * 4;
  cudaMalloc(&ws, bytes);
  cudaMemset(ws, 0, bytes);
  const int iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) red_kernel<true><<<sms, 256>>>(ws, iters);
      else red_kernel<false><<<sms, 256>>>(ws, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double red_bytes = (double)sms * iters * 128 * L * 4;
      printf("%s: %.3f ms, %.2f TB/s of reduced fp32 (%.1f us per 16384 Swin-B units)\n",
             mode == 0 ? "row-per-lane" : "contiguous  ", ms, red_bytes / ms / 1e9,
             ms * 1e3 * (16384.0 * 144 * 144 * 4) / red_bytes);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
