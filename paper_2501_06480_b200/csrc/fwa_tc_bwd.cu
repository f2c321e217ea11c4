// fwa_tc_bwd.cu — Flash Window Attention backward on tcgen05 + TMA (sm_100a).
//
// Algorithm 2 of the paper (reference flash.py:187-266) for
// f16/bf16, L <= 64, d in {16, 32, 64}. Same tile packing as the forward
// (two units per 128-row tile, 3-D TMA box (d, 64, 2), rows >= L zero-filled):
//
//   S  = Q K^T          tcgen05 SS, M=128 N=128 K=d  -> TMEM [0,128)
//   dP = dO V^T         tcgen05 SS, M=128 N=128 K=d  -> TMEM [128,256)
//   softmax warps (thread = query row = TMEM lane): P = softmax(scale*S),
//     rho = sum_j P dP, dS = scale * P (dP - rho)  (flash.py:133-138, :241-242);
//     P and dS go to shared memory as [query][key] SW128 tiles (the two
//     off-diagonal 64x64 blocks share one zero block).
//   dV = P^T dO         A = P read MN-major (the same bytes), B = dO MN-major
//   dK = dS^T Q         A = dS MN-major, B = Q MN-major
//   dQ = dS K           A = dS K-major, B = K MN-major
//   (gradient accumulators reuse TMEM [0, 3d) once S and dP are in registers)
//   Epilogue: tcgen05.ld of dV/dK/dQ rows, convert, stage into the tile's own
//   (now dead) Q/K/V smem slots, three TMA stores; the stage is released to the
//   producer only after the stores have read the staging.
//
// Q, K, V, dO are read once and dQ, dK, dV written once: 7*L*d elements per
// unit (the paper's schedule reloads Q and K: 9*L*d). No O or log-sum-exp is
// needed: P is recomputed on chip (FlashContext keeps only Q, K, V).
#include <cuda.h>
#include <math.h>

#include <algorithm>

#include "fwa_common.cuh"
#include "fwa_sm100.cuh"

namespace fwa {
namespace {

using namespace sm100;

constexpr int kThreads = 192;
constexpr int kTileRows = 128;
constexpr int kUnitRows = 64;
constexpr int kPBytes = 24 * 1024;  // [u0 | zero | u1] SW128 tile

template <int D>
struct BCfg {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTileBytes = kTileRows * kRowBytes;
  static constexpr int kStageBytes = 4 * kTileBytes;  // Q, K, V, dO
  static constexpr int kStages = D <= 16 ? 4 : 2;
  static constexpr int kCtasPerSm = D <= 32 ? 2 : 1;
  static constexpr uint32_t kSwz = D == 16 ? 6u : (D == 32 ? 4u : 2u);
  static constexpr int kSmem = kStages * kStageBytes + 2 * kPBytes + 256;
  static constexpr int kChunks = kRowBytes / 16;
  static constexpr uint32_t kTmemCols = 256;
  static constexpr uint32_t kTdP = 128, kTdV = 0, kTdK = D, kTdQ = 2 * D;
};

struct BwdBarriers {
  uint64_t full[4];
  uint64_t empty[4];
  uint64_t s_full, p_ready, ds_ready, grad_done, grad_free;
  uint32_t tmem_base;
};

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (DT<T>::id == FWA_BF16) {
    __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  } else {
    __half2 h2 = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  }
}

template <typename T, int D, int LK>
__global__ void __launch_bounds__(kThreads, BCfg<D>::kCtasPerSm)
bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
              const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
              const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dk,
              const __grid_constant__ CUtensorMap tm_dv, int n_tiles, int L_rt, float scale, unsigned int* err_flags) {
  using C = BCfg<D>;
  constexpr bool kBF16 = DT<T>::id == FWA_BF16;
  const int L = LK > 0 ? LK : L_rt;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sStage = smem;                                  // [stage][Q|K|V|dO]
  uint8_t* sP = smem + C::kStages * C::kStageBytes;
  uint8_t* sDS = sP + kPBytes;
  BwdBarriers* bars = reinterpret_cast<BwdBarriers*>(sDS + kPBytes);
  auto slot = [&](int st, int which) { return sStage + st * C::kStageBytes + which * C::kTileBytes; };
  // The swizzled layouts need a 1024-byte aligned base; the budget leaves no slack
  // for manual alignment (2 CTAs/SM), so verify it and report instead of computing garbage.
  if (smem_u32(smem) & 1023u) {
    if (threadIdx.x == 0 && err_flags) atomicOr(err_flags, 1u);
    return;
  }

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < 2 * kPBytes / 16; i += kThreads)
    reinterpret_cast<uint4*>(sP)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->p_ready, 128);
    mbar_init(&bars->ds_ready, 128);
    mbar_init(&bars->grad_done, 1);
    mbar_init(&bars->grad_free, 128);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_dq);
    tma_prefetch_desc(&tm_dk);
    tma_prefetch_desc(&tm_dv);
  }
  if (warp == 1) tmem_alloc(&bars->tmem_base, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const int n_local =
      n_tiles > (int)blockIdx.x ? (n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  griddep_launch_dependents();

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      griddep_wait();
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < n_local; ++i) {
        const int tile = blockIdx.x + i * gridDim.x;
        const int st = i % C::kStages;
        mbar_wait(&bars->empty[st], ((i / C::kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->full[st], C::kStageBytes);
        tma_load_3d(slot(st, 0), &tm_q, &bars->full[st], 0, 0, 2 * tile, pol);
        tma_load_3d(slot(st, 1), &tm_k, &bars->full[st], 0, 0, 2 * tile, pol);
        tma_load_3d(slot(st, 2), &tm_v, &bars->full[st], 0, 0, 2 * tile, pol);
        tma_load_3d(slot(st, 3), &tm_do, &bars->full[st], 0, 0, 2 * tile, pol);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_f16(kBF16, 128, 128, false, false);
      constexpr uint32_t idMN = make_idesc_f16(kBF16, 128, D, true, true);    // dV, dK
      constexpr uint32_t idQ = make_idesc_f16(kBF16, 128, D, false, true);    // dQ
      constexpr uint32_t sbo_row = 8 * C::kRowBytes;
      const uint32_t p0 = smem_u32(sP), ds0 = smem_u32(sDS);
      for (int i = 0; i < n_local; ++i) {
        const int st = i % C::kStages;
        const uint32_t q0 = smem_u32(slot(st, 0)), k0 = smem_u32(slot(st, 1));
        const uint32_t v0 = smem_u32(slot(st, 2)), do0 = smem_u32(slot(st, 3));
        mbar_wait(&bars->full[st], (i / C::kStages) & 1);
        if (i > 0) mbar_wait(&bars->grad_free, (i - 1) & 1);  // TMEM [0,256) free again
        tc_fence_after();
        // S = Q K^T, dP = dO V^T (both operands K-major, K = d)
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          mma_f16_ss(tmem, make_sdesc(q0 + kk * 32, 16, sbo_row, C::kSwz),
                     make_sdesc(k0 + kk * 32, 16, sbo_row, C::kSwz), idS, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          mma_f16_ss(tmem + C::kTdP, make_sdesc(do0 + kk * 32, 16, sbo_row, C::kSwz),
                     make_sdesc(v0 + kk * 32, 16, sbo_row, C::kSwz), idS, kk > 0);
        }
        mma_commit(&bars->s_full);
        // dV = P^T dO   (K = query rows; A = P read MN-major, B = dO MN-major)
        mbar_wait(&bars->p_ready, i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          mma_f16_ss(tmem + C::kTdV, make_sdesc(p0 + kk * 2048, 8192, 1024, 2),
                     make_sdesc(do0 + kk * 16 * C::kRowBytes, C::kTileBytes, sbo_row, C::kSwz),
                     idMN, kk > 0);
        }
        // dK = dS^T Q ; dQ = dS K
        mbar_wait(&bars->ds_ready, i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          mma_f16_ss(tmem + C::kTdK, make_sdesc(ds0 + kk * 2048, 8192, 1024, 2),
                     make_sdesc(q0 + kk * 16 * C::kRowBytes, C::kTileBytes, sbo_row, C::kSwz),
                     idMN, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          mma_f16_ss(tmem + C::kTdQ, make_sdesc(ds0 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, 2),
                     make_sdesc(k0 + kk * 16 * C::kRowBytes, C::kTileBytes, sbo_row, C::kSwz),
                     idQ, kk > 0);
        }
        mma_commit(&bars->grad_done);
      }
    }
  } else {
    // ============ softmax / dS / epilogue (warps 2..5; thread = row = TMEM lane) ============
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int ul = row >> 6;
    const uint32_t t_lane = (uint32_t)(q * 32) << 16;
    const uint32_t pswz = (uint32_t)(row & 7);
    const int prow_off = ul * 8192 + (row >> 3) * 1024 + (row & 7) * 128;
    const uint32_t oswz = (uint32_t)((row * C::kRowBytes) >> 7) & (C::kChunks - 1);
    const bool leader = (threadIdx.x == 64);
    const int p_chunks = LK > 0 ? (LK + 7) / 8 : 8;
    const float scale_log2 = scale * 1.4426950408889634f;
    for (int i = 0; i < n_local; ++i) {
      const int tile = blockIdx.x + i * gridDim.x;
      const int st = i % C::kStages;
      mbar_wait(&bars->s_full, i & 1);
      tc_fence_after();
      uint32_t s[64], dp[64];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (LK == 0 || g * 16 < LK) {
          tmem_ld16(tmem + t_lane + ul * 64 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&s[g * 16]));
          tmem_ld16(tmem + t_lane + C::kTdP + ul * 64 + g * 16,
                    *reinterpret_cast<uint32_t(*)[16]>(&dp[g * 16]));
        }
      }
      tmem_wait_ld();
      // P = softmax(scale * S) over the L valid keys (normalised: dV needs true P)
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if (j < L) mx = fmaxf(mx, __uint_as_float(s[j]));
      const float mxs = mx * scale_log2;
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const float p = j < L ? ex2(fmaf(__uint_as_float(s[j]), scale_log2, -mxs)) : 0.f;
        s[j] = __float_as_uint(p);
        sum += p;
      }
      const float inv = __frcp_rn(sum);
      // P (normalised) -> smem chunk by chunk; rho = sum_j P_j dP_j
      float rho = 0.f;
      uint8_t* prow = sP + prow_off;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int j = 8 * c + 2 * t;
          const float a = __uint_as_float(s[j]) * inv, b = __uint_as_float(s[j + 1]) * inv;
          s[j] = __float_as_uint(a);
          s[j + 1] = __float_as_uint(b);
          if (j < L) rho = fmaf(a, __uint_as_float(dp[j]), rho);
          if (j + 1 < L) rho = fmaf(b, __uint_as_float(dp[j + 1]), rho);
          w[t] = pack2<T>(a, b);
        }
        if (c < p_chunks)
          *reinterpret_cast<uint4*>(prow + ((c ^ pswz) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->p_ready);
      // dS = scale * P * (dP - rho)  (keys >= L forced to exactly 0)
      const float srho = scale * rho;
      uint8_t* dsrow = sDS + prow_off;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int j = 8 * c + 2 * t;
          const float a = __uint_as_float(s[j]) * fmaf(__uint_as_float(dp[j]), scale, -srho);
          const float b = __uint_as_float(s[j + 1]) * fmaf(__uint_as_float(dp[j + 1]), scale, -srho);
          w[t] = pack2<T>(j < L ? a : 0.f, j + 1 < L ? b : 0.f);
        }
        if (c < p_chunks)
          *reinterpret_cast<uint4*>(dsrow + ((c ^ pswz) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->ds_ready);
      // ---- epilogue: dV, dK (key rows: lane = key) and dQ (query rows), one at a time,
      // staged into this tile's V, K, Q slots (every MMA reading them has completed) ----
      mbar_wait(&bars->grad_done, i & 1);
      tc_fence_after();
#pragma unroll
      for (int which = 0; which < 3; ++which) {
        const uint32_t col = which == 0 ? C::kTdV : (which == 1 ? C::kTdK : C::kTdQ);
        uint8_t* dst = slot(st, which == 0 ? 2 : (which == 1 ? 1 : 0)) + row * C::kRowBytes;
        uint32_t gr[D];
#pragma unroll
        for (int g = 0; g < D / 16; ++g)
          tmem_ld16(tmem + t_lane + col + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&gr[g * 16]));
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          *reinterpret_cast<uint4*>(dst + ((c ^ oswz) << 4)) = make_uint4(
              pack2<T>(__uint_as_float(gr[8 * c]), __uint_as_float(gr[8 * c + 1])),
              pack2<T>(__uint_as_float(gr[8 * c + 2]), __uint_as_float(gr[8 * c + 3])),
              pack2<T>(__uint_as_float(gr[8 * c + 4]), __uint_as_float(gr[8 * c + 5])),
              pack2<T>(__uint_as_float(gr[8 * c + 6]), __uint_as_float(gr[8 * c + 7])));
      }
      tc_fence_before();
      mbar_arrive(&bars->grad_free);
      fence_proxy_async_smem();
      named_sync(1, 128);
      if (leader) {
        tma_store_3d(&tm_dq, slot(st, 0), 0, 0, 2 * tile);
        tma_store_3d(&tm_dk, slot(st, 1), 0, 0, 2 * tile);
        tma_store_3d(&tm_dv, slot(st, 2), 0, 0, 2 * tile);
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(&bars->empty[st]);   // stage may be refilled
      }
    }
    if (leader) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

template <typename T, int D, int LK>
int launch_bwd_t(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                 const void* dout, void* dq, void* dk, void* dv, cudaStream_t s) {
  CUtensorMap m[7];
  const void* ptrs[7] = {q, k, v, dout, dq, dk, dv};
  int rc;
  for (int i = 0; i < 7; ++i)
    if ((rc = get_units_map(&m[i], ptrs[i], dtype, g.units, g.L, g.d, kUnitRows, 2))) return rc;
  auto kern = bwd_tc_kernel<T, D, LK>;
  constexpr int smem = BCfg<D>::kSmem;
  static bool attr_done = false;
  if (!attr_done) {
    rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                    "cudaFuncSetAttribute(bwd_tc)");
    if (rc) return rc;
    attr_done = true;
  }
  const int n_tiles = (int)((g.units + 1) / 2);
  const int grid = std::max(1, std::min(n_tiles, device_sm_count() * BCfg<D>::kCtasPerSm));
  rc = check_cuda(launch_pdl(kern, dim3(grid), dim3(kThreads), smem, s, m[0], m[1], m[2], m[3],
                             m[4], m[5], m[6], n_tiles, (int)g.L, g.scale, device_flags_ptr()),
                  "bwd_tc_kernel launch");
  if (rc) return rc;
  count_launch();
  return FWA_OK;
}

template <typename T, int D>
int bwd_dispatch_l(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                   const void* dout, void* dq, void* dk, void* dv, cudaStream_t s) {
  if (g.L == 49) return launch_bwd_t<T, D, 49>(g, dtype, q, k, v, dout, dq, dk, dv, s);
  if (g.L == 64) return launch_bwd_t<T, D, 64>(g, dtype, q, k, v, dout, dq, dk, dv, s);
  return launch_bwd_t<T, D, 0>(g, dtype, q, k, v, dout, dq, dk, dv, s);
}

template <typename T>
int bwd_dispatch_d(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                   const void* dout, void* dq, void* dk, void* dv, cudaStream_t s) {
  switch (g.d) {
    case 16: return bwd_dispatch_l<T, 16>(g, dtype, q, k, v, dout, dq, dk, dv, s);
    case 32: return bwd_dispatch_l<T, 32>(g, dtype, q, k, v, dout, dq, dk, dv, s);
    case 64: return bwd_dispatch_l<T, 64>(g, dtype, q, k, v, dout, dq, dk, dv, s);
  }
  return fail(FWA_ERR_CAPACITY, "tcgen05 backward: unsupported head_dim");
}

}  // namespace

bool tc_bwd_supported(const Geom& g, int dtype, bool bias_or_mask) {
  if (bias_or_mask) return false;
  if (dtype != FWA_F16 && dtype != FWA_BF16) return false;
  if (g.L < 1 || g.L > kUnitRows) return false;
  if (g.d != 16 && g.d != 32 && g.d != 64) return false;
  return g.units <= ((int64_t)1 << 31);
}

size_t tc_bwd_smem(const Geom& g) {
  return g.d == 16 ? BCfg<16>::kSmem : g.d == 32 ? BCfg<32>::kSmem : BCfg<64>::kSmem;
}

int launch_bwd_tc(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                  const void* dout, void* dq, void* dk, void* dv, cudaStream_t s) {
  return dtype == FWA_BF16 ? bwd_dispatch_d<__nv_bfloat16>(g, dtype, q, k, v, dout, dq, dk, dv, s)
                           : bwd_dispatch_d<__half>(g, dtype, q, k, v, dout, dq, dk, dv, s);
}

}  // namespace fwa
