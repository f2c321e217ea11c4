// fwa_generic.cu — generic SIMT window-attention kernels (any L, any d, f32/f16/bf16).
//
// This is the paper's Algorithm 1/2 (reference
// pkg/src/flashwin/flash.py:141-266) executed literally on one CTA: the score
// block S lives in shared memory, Q/K (and dO/V) are streamed in feature
// chunks of CW columns and accumulated into S, the row softmax runs in place,
// and O (or dQ/dK/dV) is streamed out chunk by chunk. It carries the fp32
// path (1e-5 relative, BASELINE configs[0]) and every shape the tcgen05
// kernel does not take (d not a multiple of 16, L > 256, ragged sizes). It is
// a GPU path; there is no CPU fallback anywhere in libfwa.
#include <math.h>

#include <algorithm>

#include "fwa_common.cuh"

namespace fwa {
namespace {

constexpr int kFwdThreads = 128;
constexpr int kBwdThreads = 256;
constexpr int CW = 32;  // feature-chunk width (the paper's C/r; result is r-invariant)

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int fwd_rows(int L) { return std::min(L, std::max(1, 8192 / L)); }
inline int bwd_rows(int L) { return std::min(L, std::max(1, 4096 / L)); }

// Row softmax of S rows [0, rows) in place (flash.py:127-130), after the
// scale (flash.py:171) and the optional additive bias/mask (extension).
__device__ __forceinline__ void softmax_rows_block(float* S, int rows, int i0, int L,
                                                   float scale, const float* bh,
                                                   const float* mw, int nthreads) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < rows; i += nthreads / 32) {
    float* Si = S + (size_t)i * L;
    const int gi = i0 + i;
    float mx = -INFINITY;
    for (int j = lane; j < L; j += 32) {
      float s = Si[j] * scale;
      if (bh) s += bh[(size_t)gi * L + j];
      if (mw) s += mw[(size_t)gi * L + j];
      Si[j] = s;
      mx = fmaxf(mx, s);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < L; j += 32) {
      const float p = expf(Si[j] - mx);
      Si[j] = p;
      sum += p;
    }
    sum = warp_sum(sum);
    for (int j = lane; j < L; j += 32) Si[j] = Si[j] / sum;
  }
}

template <typename T>
__device__ __forceinline__ void load_chunk(float* dst, int ld, const T* src, int rows,
                                           int d, int c0, int cw, int nthreads) {
  for (int e = threadIdx.x; e < rows * cw; e += nthreads) {
    const int r = e / cw, c = e - r * cw;
    dst[r * ld + c] = DT<T>::to_f(src[(size_t)r * d + c0 + c]);
  }
}

// ---------------------------------------------------------------------------
// Forward: one CTA per (unit, block of R query rows).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kFwdThreads)
fwd_generic_kernel(Geom g, int R, int nRB, const T* __restrict__ q, const T* __restrict__ k,
                   const T* __restrict__ v, const float* __restrict__ bias,
                   const float* __restrict__ mask, T* __restrict__ o) {
  extern __shared__ float sm[];
  const int L = g.L, d = g.d;
  const int64_t unit = blockIdx.x / nRB;
  const int rb = blockIdx.x % nRB;
  const int i0 = rb * R;
  const int rows = min(R, L - i0);
  float* S = sm;                       // [R][L]
  float* Qc = S + (size_t)R * L;       // [R][CW+1]
  float* Kc = Qc + (size_t)R * (CW + 1);  // [L][CW+1]; reused as Vc [L][CW]
  const size_t base = (size_t)unit * L * d;
  const T* qu = q + base + (size_t)i0 * d;
  const T* ku = k + base;
  const T* vu = v + base;
  T* ou = o + base + (size_t)i0 * d;

  for (int e = threadIdx.x; e < rows * L; e += kFwdThreads) S[e] = 0.f;
  // S = sum over feature chunks of Q_i K_i^T (flash.py:164-169)
  for (int c0 = 0; c0 < d; c0 += CW) {
    const int cw = min(CW, d - c0);
    __syncthreads();
    load_chunk(Qc, CW + 1, qu, rows, d, c0, cw, kFwdThreads);
    load_chunk(Kc, CW + 1, ku, L, d, c0, cw, kFwdThreads);
    __syncthreads();
    for (int e = threadIdx.x; e < rows * L; e += kFwdThreads) {
      const int i = e / L, j = e - i * L;
      const float* qi = Qc + i * (CW + 1);
      const float* kj = Kc + j * (CW + 1);
      float acc = 0.f;
      for (int c = 0; c < cw; ++c) acc = fmaf(qi[c], kj[c], acc);
      S[e] += acc;
    }
  }
  __syncthreads();
  const int h = (int)(unit % g.heads);
  const int64_t n = unit / g.heads;
  const float* bh = bias ? bias + (size_t)h * L * L : nullptr;
  const float* mw = mask ? mask + (size_t)(n % g.mask_windows) * L * L : nullptr;
  softmax_rows_block(S, rows, i0, L, g.scale, bh, mw, kFwdThreads);
  // O_i = P V_i per chunk (flash.py:174-180)
  float* Vc = Kc;
  for (int c0 = 0; c0 < d; c0 += CW) {
    const int cw = min(CW, d - c0);
    __syncthreads();
    load_chunk(Vc, CW, vu, L, d, c0, cw, kFwdThreads);
    __syncthreads();
    for (int e = threadIdx.x; e < rows * cw; e += kFwdThreads) {
      const int i = e / cw, c = e - i * cw;
      const float* Pi = S + (size_t)i * L;
      float acc = 0.f;
      for (int j = 0; j < L; ++j) acc = fmaf(Pi[j], Vc[j * CW + c], acc);
      ou[(size_t)i * d + c0 + c] = DT<T>::from_f(acc);
    }
  }
}

// ---------------------------------------------------------------------------
// Backward: persistent grid; one CTA owns whole units (so dK/dV accumulate
// in shared memory without atomics) and walks R-row query blocks.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kBwdThreads)
bwd_generic_kernel(Geom g, int R, const T* __restrict__ q, const T* __restrict__ k,
                   const T* __restrict__ v, const T* __restrict__ dout,
                   const float* __restrict__ bias, const float* __restrict__ mask,
                   T* __restrict__ dq, T* __restrict__ dk, T* __restrict__ dv,
                   float* __restrict__ dbias_ws) {
  extern __shared__ float sm[];
  const int L = g.L, d = g.d;
  float* dKa = sm;                          // [L][d]
  float* dVa = dKa + (size_t)L * d;         // [L][d]
  float* P = dVa + (size_t)L * d;           // [R][L]
  float* dP = P + (size_t)R * L;            // [R][L]
  float* A = dP + (size_t)R * L;            // [R][CW+1]
  float* B = A + (size_t)R * (CW + 1);      // [L][CW+1]
  const size_t LL = (size_t)L * L;
  float* my_ws = dbias_ws ? dbias_ws + (size_t)blockIdx.x * g.heads * LL : nullptr;
  if (my_ws) {
    for (size_t e = threadIdx.x; e < (size_t)g.heads * LL; e += kBwdThreads) my_ws[e] = 0.f;
  }

  for (int64_t unit = blockIdx.x; unit < g.units; unit += gridDim.x) {
    const size_t base = (size_t)unit * L * d;
    const int h = (int)(unit % g.heads);
    const int64_t n = unit / g.heads;
    const float* bh = bias ? bias + (size_t)h * LL : nullptr;
    const float* mw = mask ? mask + (size_t)(n % g.mask_windows) * LL : nullptr;
    float* wsh = my_ws ? my_ws + (size_t)h * LL : nullptr;
    __syncthreads();
    for (int e = threadIdx.x; e < 2 * L * d; e += kBwdThreads) dKa[e] = 0.f;  // dKa, dVa
    for (int i0 = 0; i0 < L; i0 += R) {
      const int rows = min(R, L - i0);
      const T* qb = q + base + (size_t)i0 * d;
      const T* dob = dout + base + (size_t)i0 * d;
      // Phase 1: recompute S, P (flash.py:215-225)
      __syncthreads();
      for (int e = threadIdx.x; e < rows * L; e += kBwdThreads) { P[e] = 0.f; dP[e] = 0.f; }
      for (int c0 = 0; c0 < d; c0 += CW) {
        const int cw = min(CW, d - c0);
        __syncthreads();
        load_chunk(A, CW + 1, qb, rows, d, c0, cw, kBwdThreads);
        load_chunk(B, CW + 1, k + base, L, d, c0, cw, kBwdThreads);
        __syncthreads();
        for (int e = threadIdx.x; e < rows * L; e += kBwdThreads) {
          const int i = e / L, j = e - i * L;
          float acc = 0.f;
          for (int c = 0; c < cw; ++c) acc = fmaf(A[i * (CW + 1) + c], B[j * (CW + 1) + c], acc);
          P[e] += acc;
        }
      }
      __syncthreads();
      softmax_rows_block(P, rows, i0, L, g.scale, bh, mw, kBwdThreads);
      // Phase 2: dP += dO_i V_i^T ; dV_i += P^T dO_i (flash.py:227-238)
      for (int c0 = 0; c0 < d; c0 += CW) {
        const int cw = min(CW, d - c0);
        __syncthreads();
        load_chunk(A, CW + 1, dob, rows, d, c0, cw, kBwdThreads);
        load_chunk(B, CW + 1, v + base, L, d, c0, cw, kBwdThreads);
        __syncthreads();
        for (int e = threadIdx.x; e < rows * L; e += kBwdThreads) {
          const int i = e / L, j = e - i * L;
          float acc = 0.f;
          for (int c = 0; c < cw; ++c) acc = fmaf(A[i * (CW + 1) + c], B[j * (CW + 1) + c], acc);
          dP[e] += acc;
        }
        for (int e = threadIdx.x; e < L * cw; e += kBwdThreads) {
          const int j = e / cw, c = e - j * cw;
          float acc = 0.f;
          for (int i = 0; i < rows; ++i) acc = fmaf(P[(size_t)i * L + j], A[i * (CW + 1) + c], acc);
          dVa[(size_t)j * d + c0 + c] += acc;
        }
      }
      __syncthreads();
      // dS = P * (dP - rowdot) (flash.py:133-138); dBias partial; dS *= scale
      {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int i = warp; i < rows; i += kBwdThreads / 32) {
          const float* Pi = P + (size_t)i * L;
          float* dPi = dP + (size_t)i * L;
          float rho = 0.f;
          for (int j = lane; j < L; j += 32) rho = fmaf(Pi[j], dPi[j], rho);
          rho = warp_sum(rho);
          for (int j = lane; j < L; j += 32) {
            const float ds = Pi[j] * (dPi[j] - rho);
            if (wsh) wsh[(size_t)(i0 + i) * L + j] += ds;
            dPi[j] = ds * g.scale;
          }
        }
      }
      // Phase 3: dQ_i = dS K_i ; dK_i += dS^T Q_i (flash.py:245-257)
      for (int c0 = 0; c0 < d; c0 += CW) {
        const int cw = min(CW, d - c0);
        __syncthreads();
        load_chunk(A, CW + 1, qb, rows, d, c0, cw, kBwdThreads);
        load_chunk(B, CW + 1, k + base, L, d, c0, cw, kBwdThreads);
        __syncthreads();
        for (int e = threadIdx.x; e < rows * cw; e += kBwdThreads) {
          const int i = e / cw, c = e - i * cw;
          const float* dSi = dP + (size_t)i * L;
          float acc = 0.f;
          for (int j = 0; j < L; ++j) acc = fmaf(dSi[j], B[j * (CW + 1) + c], acc);
          dq[base + (size_t)(i0 + i) * d + c0 + c] = DT<T>::from_f(acc);
        }
        for (int e = threadIdx.x; e < L * cw; e += kBwdThreads) {
          const int j = e / cw, c = e - j * cw;
          float acc = 0.f;
          for (int i = 0; i < rows; ++i) acc = fmaf(dP[(size_t)i * L + j], A[i * (CW + 1) + c], acc);
          dKa[(size_t)j * d + c0 + c] += acc;
        }
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < L * d; e += kBwdThreads) {
      dk[base + e] = DT<T>::from_f(dKa[e]);
      dv[base + e] = DT<T>::from_f(dVa[e]);
    }
  }
}

// dbias[e] = sum over CTAs c (fixed order) of ws[c][e]  — deterministic.
__global__ void dbias_reduce_kernel(const float* __restrict__ ws, int parts, size_t n,
                                    float* __restrict__ dbias) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < parts; ++p) acc += ws[(size_t)p * n + e];
    dbias[e] = acc;
  }
}

template <typename T>
int launch_fwd_generic_t(const Geom& g, const void* q, const void* k, const void* v,
                         const float* bias, const float* mask, void* o, cudaStream_t s) {
  const int R = fwd_rows(g.L);
  const int nRB = (g.L + R - 1) / R;
  const size_t smem = fwd_generic_smem(g);
  auto kern = fwd_generic_kernel<T>;
  int rc = FWA_OK;
  if ((rc = ensure_smem_attr((const void*)kern, (int)smem, "cudaFuncSetAttribute(fwd_generic)"))) return rc;
  const int64_t blocks = g.units * nRB;
  if (blocks <= 0) return FWA_OK;
  if (blocks > 0x7fffffffLL) return fail(FWA_ERR_CAPACITY, "too many units for one launch");
  kern<<<(unsigned)blocks, kFwdThreads, smem, s>>>(g, R, nRB, (const T*)q, (const T*)k,
                                                   (const T*)v, bias, mask, (T*)o);
  count_launch();
  return check_cuda(cudaGetLastError(), "fwd_generic_kernel launch");
}

template <typename T>
int launch_bwd_generic_t(const Geom& g, const void* q, const void* k, const void* v,
                         const void* dout, const float* bias, const float* mask, void* dq,
                         void* dk, void* dv, float* dbias, float* ws, cudaStream_t s) {
  const int R = bwd_rows(g.L);
  const size_t smem = bwd_generic_smem(g);
  auto kern = bwd_generic_kernel<T>;
  int rc = FWA_OK;
  if ((rc = ensure_smem_attr((const void*)kern, (int)smem, "cudaFuncSetAttribute(bwd_generic)"))) return rc;
  const int grid = bwd_generic_grid(g);
  if (g.units <= 0) return FWA_OK;
  kern<<<grid, kBwdThreads, smem, s>>>(g, R, (const T*)q, (const T*)k, (const T*)v,
                                       (const T*)dout, bias, mask, (T*)dq, (T*)dk, (T*)dv,
                                       dbias ? ws : nullptr);
  count_launch();
  rc = check_cuda(cudaGetLastError(), "bwd_generic_kernel launch");
  if (rc || !dbias) return rc;
  const size_t n = (size_t)g.heads * g.L * g.L;
  dbias_reduce_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, s>>>(
      ws, grid, n, dbias);
  count_launch();
  return check_cuda(cudaGetLastError(), "dbias_reduce_kernel launch");
}

}  // namespace

size_t fwd_generic_smem(const Geom& g) {
  const size_t R = fwd_rows(g.L);
  return sizeof(float) * (R * g.L + R * (CW + 1) + (size_t)g.L * (CW + 1));
}

size_t bwd_generic_smem(const Geom& g) {
  const size_t R = bwd_rows(g.L);
  return sizeof(float) * (2 * (size_t)g.L * g.d + 2 * R * g.L + R * (CW + 1) +
                          (size_t)g.L * (CW + 1));
}

bool bwd_generic_fits(const Geom& g) { return bwd_generic_smem(g) <= device_max_smem_optin(); }

int bwd_generic_grid(const Geom& g) {
  int per_sm = 1;
  const size_t smem = bwd_generic_smem(g);
  if (smem > 0) per_sm = std::max<int>(1, (int)(device_max_smem_optin() / smem));
  per_sm = std::min(per_sm, 2048 / kBwdThreads);
  const int64_t want = (int64_t)device_sm_count() * per_sm;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, g.units));
}

int launch_fwd_generic(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                       const float* bias, const float* mask, void* o, cudaStream_t s) {
  switch (dtype) {
    case FWA_F32: return launch_fwd_generic_t<float>(g, q, k, v, bias, mask, o, s);
    case FWA_F16: return launch_fwd_generic_t<__half>(g, q, k, v, bias, mask, o, s);
    case FWA_BF16: return launch_fwd_generic_t<__nv_bfloat16>(g, q, k, v, bias, mask, o, s);
  }
  return fail(FWA_ERR_INVALID_RANGE, "unknown dtype");
}

int launch_bwd_generic(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                       const void* dout, const float* bias, const float* mask, void* dq,
                       void* dk, void* dv, float* dbias, float* ws, cudaStream_t s) {
  switch (dtype) {
    case FWA_F32:
      return launch_bwd_generic_t<float>(g, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s);
    case FWA_F16:
      return launch_bwd_generic_t<__half>(g, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s);
    case FWA_BF16:
      return launch_bwd_generic_t<__nv_bfloat16>(g, q, k, v, dout, bias, mask, dq, dk, dv, dbias,
                                                 ws, s);
  }
  return fail(FWA_ERR_INVALID_RANGE, "unknown dtype");
}

}  // namespace fwa
