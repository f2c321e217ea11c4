// fwa_window.cu — window partition/reverse (+cyclic shift), Swin bias/mask
// helpers, and the SplitMix64 device fill.
//
// window_partition / window_reverse follow the reference's index map
// (pkg/src/flashwin/windowing.py:44-70): windows row-major over (wr, wc),
// pixels row-major within the window; out[b*nW + wr*(W/k) + wc][r*k + c][:] =
// in[b][wr*k + r][wc*k + c][:]. The copy is bitwise (the kernel moves bytes),
// so partition∘reverse is the identity exactly (criterion 8, SPEC.md).
// One warp moves one pixel's C-channel row with the widest aligned vector.
#include <algorithm>

#include "fwa_common.cuh"

namespace fwa {
namespace {

// One warp per (window, pixel row r of the window): the k pixels of that row are one
// contiguous run on the window side and one (or, when the cyclic shift wraps, two) run(s)
// on the image side, so the warp does the index math once (32-bit, per run) and its lanes
// stream the run's 16-byte vectors coalesced. Each lane's (pixel, vector) position inside a
// run is advanced incrementally (no division per vector).
template <typename V>
__global__ void __launch_bounds__(256) window_copy_kernel(fwa_win_desc dsc, const V* __restrict__ in,
                                                          V* __restrict__ out, int reverse, int rowv,
                                                          int units) {
  const int k = dsc.window, H = dsc.height, W = dsc.width, shift = dsc.shift;
  const int nWc = W / k, nW = (H / k) * nWc, run = k * rowv;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  // lane's first vector: pixel pix0, vector c0 of that pixel
  const int pix0 = lane / rowv, c0 = lane - (lane / rowv) * rowv;
  for (int unit = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; unit < units; unit += nwarps) {
    const int win = unit / k, r = unit - win * k;
    const int b = win / nW, w = win - b * nW;
    const int wr = w / nWc, wc = w - wr * nWc;
    int y = wr * k + r + shift;
    if (y >= H) y -= H;
    const int x0 = wc * k + shift;
    const int64_t img_row = ((int64_t)b * H + y) * W;   // pixel index of (b, y, 0)
    const int64_t win_row = (int64_t)unit * k;          // window-major pixel of (win, r, 0)
    int pix = pix0, c = c0;
    // 4 vectors per lane in flight: all loads of a group before its stores
    for (int v = lane; v < run; v += 4 * 32) {
      int64_t src[4], dst[4];
      V val[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        int x = x0 + pix;
        if (x >= W) x -= W;
        const int64_t img = (img_row + x) * rowv + c;
        const int64_t wm = (win_row + pix) * rowv + c;
        src[t] = reverse ? wm : img;
        dst[t] = reverse ? img : wm;
        c += 32;
        while (c >= rowv) {
          c -= rowv;
          ++pix;
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (v + 32 * t < run) val[t] = in[src[t]];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (v + 32 * t < run) out[dst[t]] = val[t];
    }
  }
}

int launch_window(const fwa_win_desc* d, const void* in, void* out, cudaStream_t s, int reverse) {
  if (!d || !in || !out) return fail(FWA_ERR_SHAPE, "null window descriptor or pointer");
  if (d->batch < 1 || d->height < 1 || d->width < 1 || d->channels < 1 || d->window < 1)
    return fail(FWA_ERR_SHAPE, "window geometry extents must be >= 1");
  if (d->height % d->window || d->width % d->window)
    return fail(FWA_ERR_PARTITION, "window size " + std::to_string(d->window) +
                                       " must divide image " + std::to_string(d->height) + "x" +
                                       std::to_string(d->width));
  if (d->shift < 0 || d->shift >= d->window)
    return fail(FWA_ERR_INVALID_RANGE, "shift must satisfy 0 <= shift < window");
  const int eb = d->elem_bytes;
  if (eb != 1 && eb != 2 && eb != 4 && eb != 8)
    return fail(FWA_ERR_INVALID_RANGE, "elem_bytes must be 1, 2, 4 or 8");
  const int64_t row_bytes = (int64_t)d->channels * eb;
  const uintptr_t align = (uintptr_t)in | (uintptr_t)out;
  const int64_t total_bytes = d->batch * (int64_t)d->height * d->width * row_bytes;
  if (total_bytes == 0) return FWA_OK;
  const int threads = 256;
  const int64_t units64 = d->batch * (int64_t)(d->height / d->window) * (d->width / d->window) * d->window;
  if (units64 >= ((int64_t)1 << 31) || d->batch * (int64_t)d->height * d->width >= ((int64_t)1 << 31))
    return fail(FWA_ERR_CAPACITY, "window partition: more than 2^31 pixels per call");
  const int units = (int)units64;
  // a persistent grid of 8 warps per CTA, up to 16 CTAs per SM
  const unsigned grid = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((units + 7) / 8, (int64_t)device_sm_count() * 16));
  auto go = [&](auto vec) {
    using V = decltype(vec);
    const int rowv = (int)(row_bytes / sizeof(V));
    window_copy_kernel<V><<<grid, threads, 0, s>>>(*d, (const V*)in, (V*)out, reverse, rowv, units);
  };
  if (row_bytes % 16 == 0 && align % 16 == 0) go(uint4{});
  else if (row_bytes % 8 == 0 && align % 8 == 0) go(uint2{});
  else if (row_bytes % 4 == 0 && align % 4 == 0) go(uint32_t{});
  else if (row_bytes % 2 == 0 && align % 2 == 0) go(uint16_t{});
  else go(uint8_t{});
  count_launch();
  return check_cuda(cudaGetLastError(), "window_copy_kernel launch");
}

// ---- Swin relative-position bias (extension) --------------------------------
__device__ __forceinline__ int rel_index(int i, int j, int k) {
  const int yi = i / k, xi = i % k, yj = j / k, xj = j % k;
  return (yi - yj + k - 1) * (2 * k - 1) + (xi - xj + k - 1);
}

__global__ void bias_gather_kernel(const float* __restrict__ table, int k, int heads,
                                   float* __restrict__ bias) {
  const int L = k * k;
  const int64_t n = (int64_t)heads * L * L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int h = (int)(e / ((int64_t)L * L));
    const int r = (int)(e - (int64_t)h * L * L);
    const int i = r / L, j = r % L;
    bias[e] = table[(int64_t)rel_index(i, j, k) * heads + h];
  }
}

// dtable[t][h] = sum over (i,j) with rel_index(i,j)==t of dbias[h][i][j].
// For a fixed t = (dy, dx) offset the contributing (i, j) pairs are enumerated
// in a fixed order (i ascending), so the sum is deterministic.
__global__ void bias_scatter_kernel(const float* __restrict__ dbias, int k, int heads,
                                    float* __restrict__ dtable) {
  const int L = k * k;
  const int T = (2 * k - 1) * (2 * k - 1);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < T * heads; e += gridDim.x * blockDim.x) {
    const int t = e / heads, h = e % heads;
    const int dy = t / (2 * k - 1) - (k - 1), dx = t % (2 * k - 1) - (k - 1);
    float acc = 0.f;
    for (int yi = 0; yi < k; ++yi) {
      const int yj = yi - dy;
      if (yj < 0 || yj >= k) continue;
      for (int xi = 0; xi < k; ++xi) {
        const int xj = xi - dx;
        if (xj < 0 || xj >= k) continue;
        acc += dbias[((int64_t)h * L + yi * k + xi) * L + yj * k + xj];
      }
    }
    dtable[e] = acc;
  }
}

// Swin shifted-window mask: region id per pixel from the 3x3 slab split of
// the rolled image; mask[w][i][j] = (id(i) != id(j)) ? neg : 0.
__device__ __forceinline__ int region_1d(int p, int n, int k, int s) {
  return p < n - k ? 0 : (p < n - s ? 1 : 2);
}

__global__ void shift_mask_kernel(int H, int W, int k, int s, float neg, float* __restrict__ m) {
  const int L = k * k, nWc = W / k;
  const int64_t nW = (int64_t)(H / k) * nWc;
  const int64_t n = nW * L * L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = e / ((int64_t)L * L);
    const int r = (int)(e - w * L * L);
    const int i = r / L, j = r % L;
    const int wr = (int)(w / nWc), wc = (int)(w % nWc);
    const int yi = wr * k + i / k, xi = wc * k + i % k;
    const int yj = wr * k + j / k, xj = wc * k + j % k;
    const int ri = region_1d(yi, H, k, s) * 3 + region_1d(xi, W, k, s);
    const int rj = region_1d(yj, H, k, s) * 3 + region_1d(xj, W, k, s);
    m[e] = (ri != rj) ? neg : 0.f;
  }
}

// ---- SplitMix64 fill (tensor.py:118-138) ------------------------------------
__device__ __forceinline__ uint64_t splitmix_at(uint64_t state, uint64_t i) {
  uint64_t z = state + 0x9E3779B97F4A7C15ull * (i + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_uniform_kernel(uint64_t state, int64_t n, double lo, double hi,
                                    T* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double u = (double)(splitmix_at(state, (uint64_t)e) >> 11) * 0x1.0p-53;
    const float f = __double2float_rn(lo + (hi - lo) * u);  // f64 -> f32 (RNE)
    out[e] = DT<T>::from_f(f);                               // f32 -> dtype (RNE)
  }
}

unsigned grid_for(int64_t n, int threads) {
  return (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)device_sm_count() * 16));
}

}  // namespace
}  // namespace fwa

using namespace fwa;

extern "C" int fwa_window_partition(const fwa_win_desc* desc, const void* in, void* out,
                                    void* stream) {
  return launch_window(desc, in, out, (cudaStream_t)stream, 0);
}

extern "C" int fwa_window_reverse(const fwa_win_desc* desc, const void* in, void* out,
                                  void* stream) {
  return launch_window(desc, in, out, (cudaStream_t)stream, 1);
}

extern "C" int fwa_bias_gather(const float* table, int32_t window, int32_t heads, float* bias,
                               void* stream) {
  if (!table || !bias || window < 1 || heads < 1)
    return fail(FWA_ERR_SHAPE, "bias_gather: bad arguments");
  const int64_t n = (int64_t)heads * window * window * window * window;
  bias_gather_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(table, window, heads,
                                                                        bias);
  count_launch();
  return check_cuda(cudaGetLastError(), "bias_gather_kernel launch");
}

extern "C" int fwa_bias_scatter(const float* dbias, int32_t window, int32_t heads, float* dtable,
                                void* stream) {
  if (!dbias || !dtable || window < 1 || heads < 1)
    return fail(FWA_ERR_SHAPE, "bias_scatter: bad arguments");
  const int64_t n = (int64_t)(2 * window - 1) * (2 * window - 1) * heads;
  bias_scatter_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(dbias, window, heads,
                                                                         dtable);
  count_launch();
  return check_cuda(cudaGetLastError(), "bias_scatter_kernel launch");
}

extern "C" int fwa_shift_mask(int32_t height, int32_t width, int32_t window, int32_t shift,
                              float neg, float* mask, void* stream) {
  if (!mask || window < 1 || height < 1 || width < 1)
    return fail(FWA_ERR_SHAPE, "shift_mask: bad arguments");
  if (height % window || width % window)
    return fail(FWA_ERR_PARTITION, "window size must divide the image");
  if (shift < 1 || shift >= window)
    return fail(FWA_ERR_INVALID_RANGE, "shift_mask needs 0 < shift < window");
  const int64_t L = (int64_t)window * window;
  const int64_t n = (int64_t)(height / window) * (width / window) * L * L;
  shift_mask_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(height, width, window,
                                                                       shift, neg, mask);
  count_launch();
  return check_cuda(cudaGetLastError(), "shift_mask_kernel launch");
}

extern "C" int fwa_fill_uniform(uint64_t state, int64_t count, double lo, double hi,
                                int32_t dtype, void* out, void* stream) {
  if (count < 0 || (!out && count)) return fail(FWA_ERR_SHAPE, "fill_uniform: bad arguments");
  if (!(lo < hi)) return fail(FWA_ERR_INVALID_RANGE, "need lo < hi");
  if (count == 0) return FWA_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned g = grid_for(count, 256);
  switch (dtype) {
    case FWA_F32: fill_uniform_kernel<float><<<g, 256, 0, s>>>(state, count, lo, hi, (float*)out); break;
    case FWA_F16: fill_uniform_kernel<__half><<<g, 256, 0, s>>>(state, count, lo, hi, (__half*)out); break;
    case FWA_BF16:
      fill_uniform_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(state, count, lo, hi,
                                                           (__nv_bfloat16*)out);
      break;
    default: return fail(FWA_ERR_INVALID_RANGE, "unknown dtype");
  }
  count_launch();
  return check_cuda(cudaGetLastError(), "fill_uniform_kernel launch");
}
