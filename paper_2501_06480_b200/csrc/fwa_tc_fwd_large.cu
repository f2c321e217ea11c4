// fwa_tc_fwd_large.cu — forward for large windows (64 < L <= 256, e.g. Swin-B 12x12,
// 16x16) on tcgen05 + TMA (sm_100a), f16/bf16, d in {16, 32, 64}, no bias/mask.
//
// Work item = (unit, query M-tile of 128 rows). K and V of a unit are TMA-loaded
// once (box (d, L_pad, 1); rows >= L are OOB zeros) and reused by its ceil(L/128)
// M-tiles; Q comes per M-tile (box (d, 128, 1)).
//   S = Q K^T     tcgen05 SS, M=128, N=L_pad (<= 256), K=d   -> TMEM [0, L_pad)
//   softmax       two passes over TMEM (row max, then ex2 / row sum); P (16-bit
//                 pairs) is stored over the S columns already consumed
//                 (P col c = keys 2c, 2c+1, written after keys >= 2c were read)
//   O = P V       tcgen05 TS (A = P in TMEM), N=d, K=L_pad  -> TMEM [O_col, O_col+d)
//                 with O_col = round_up(L_pad/2, 16): also inside consumed S columns
//   epilogue      1/rowsum, convert, swizzled staging, TMA store (rows >= L clipped)
// One item fits in 256 TMEM columns; the CTA (1 per SM) double-buffers items in its
// 512 columns, so the MMA warp computes S(i+2) while the softmax warps work on item
// i+1 and a separate epilogue warpgroup drains O(i): the softmax warps never wait on
// PV or on the store. Warps whose 32 rows are all >= L skip the math (warp-uniform)
// but still arrive on the barriers. HBM traffic: Q, K, V read once, O written once.
#include <cuda.h>
#include <math.h>

#include <algorithm>

#include "fwa_common.cuh"
#include "fwa_sm100.cuh"

namespace fwa {
namespace {

using namespace sm100;

constexpr int kThreads = 320;   // producer, MMA, 4 softmax warps, 4 epilogue warps
constexpr int kMRows = 128;

template <int D, int LP>
struct LCfg {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kQBytes = kMRows * kRowBytes;
  static constexpr int kKVBytes = LP * kRowBytes;          // one of K / V for a unit
  static constexpr int kMTiles = (LP + kMRows - 1) / kMRows;
  static constexpr int kKVStages = 2;
  static constexpr int kQStages = 3;
  static constexpr uint32_t kSwz = D == 16 ? 6u : (D == 32 ? 4u : 2u);
  // K/V tiles keep the 8-row swizzle atoms 1024-aligned
  static constexpr int kKVSlot = (kKVBytes + 1023) / 1024 * 1024;
  static constexpr int kSmem = 1024 + kKVStages * 2 * kKVSlot + kQStages * kQBytes + kQBytes + 1024 + 256;
  static constexpr int kChunks = kRowBytes / 16;
  // Each of the two TMEM buffers (256 columns) holds one item: S [0, LP), then P over the
  // consumed S columns [0, LP/2), then O at [kOCol, kOCol + d).
  static constexpr uint32_t kOCol = ((LP / 2 + 15) / 16) * 16;
  static_assert(kOCol + D <= 256, "O must fit in the consumed S columns");
  static_assert(kSmem <= 227 * 1024, "smem budget");
};

struct LBarriers {
  uint64_t kv_full[2], kv_empty[2], q_full[3], q_empty[3];
  uint64_t s_full[2], p_full[2], o_full[2], buf_free[2];
  uint32_t tmem_base;
};

template <typename T>
__device__ __forceinline__ uint32_t pack2l(float a, float b) {
  if constexpr (DT<T>::id == FWA_BF16) {
    __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  } else {
    __half2 h2 = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  }
}

template <typename T, int D, int LP>
__global__ void __launch_bounds__(kThreads, 1)
fwd_tc_large_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                    int n_units, int L, float scale_log2) {
  using C = LCfg<D, LP>;
  constexpr bool kBF16 = DT<T>::id == FWA_BF16;
  constexpr int NM = C::kMTiles;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;                                   // [kv stage] K
  uint8_t* sV = sK + C::kKVStages * C::kKVSlot;         // [kv stage] V
  uint8_t* sQ = sV + C::kKVStages * C::kKVSlot;         // [q stage] Q
  uint8_t* sO = sQ + C::kQStages * C::kQBytes;          // output staging
  float* sInv = reinterpret_cast<float*>(sO + C::kQBytes);   // [2 buffers][128 rows] 1/rowsum
  LBarriers* bars = reinterpret_cast<LBarriers*>(sO + C::kQBytes + 1024);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars->kv_full[s], 1);
      mbar_init(&bars->kv_empty[s], 1);
      mbar_init(&bars->s_full[s], 1);
      mbar_init(&bars->p_full[s], 128);
      mbar_init(&bars->o_full[s], 1);
      mbar_init(&bars->buf_free[s], 128);
    }
    for (int s = 0; s < 3; ++s) {
      mbar_init(&bars->q_full[s], 1);
      mbar_init(&bars->q_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_o);
  }
  if (warp == 1) tmem_alloc(&bars->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const int n_local =
      n_units > (int)blockIdx.x ? (n_units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int n_items = n_local * NM;
  griddep_launch_dependents();

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      griddep_wait();
      const uint64_t pol = policy_evict_first();
      int qi = 0;
      for (int i = 0; i < n_local; ++i) {
        const int unit = blockIdx.x + i * gridDim.x;
        const int kst = i & 1;
        mbar_wait(&bars->kv_empty[kst], ((i >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->kv_full[kst], 2 * C::kKVBytes);
        tma_load_3d(sK + kst * C::kKVSlot, &tm_k, &bars->kv_full[kst], 0, 0, unit, pol);
        tma_load_3d(sV + kst * C::kKVSlot, &tm_v, &bars->kv_full[kst], 0, 0, unit, pol);
        for (int m = 0; m < NM; ++m, ++qi) {
          const int qs = qi % C::kQStages;
          mbar_wait(&bars->q_empty[qs], ((qi / C::kQStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&bars->q_full[qs], C::kQBytes);
          tma_load_3d(sQ + qs * C::kQBytes, &tm_q, &bars->q_full[qs], 0, m * kMRows, unit, pol);
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: S(0), S(1), then [PV(it), S(it+2)] — S runs ahead of the softmax =====
    if (lane == 0 && n_items > 0) {
      constexpr uint32_t idS = make_idesc_f16(kBF16, 128, LP, false, false);
      constexpr uint32_t idO = make_idesc_f16(kBF16, 128, D, false, true);
      constexpr uint32_t sbo = 8 * C::kRowBytes;
      auto issue_S = [&](int it) {
        const int b = it & 1;
        const int i = it / NM;
        const int qs = it % C::kQStages;
        if (it % NM == 0) mbar_wait(&bars->kv_full[i & 1], (i >> 1) & 1);
        mbar_wait(&bars->q_full[qs], (it / C::kQStages) & 1);
        if (it >= 2) mbar_wait(&bars->buf_free[b], ((it >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t k0 = smem_u32(sK + (i & 1) * C::kKVSlot);
        const uint32_t q0 = smem_u32(sQ + qs * C::kQBytes);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_f16_ss(tmem + b * 256, make_sdesc(q0 + kk * 32, 16, sbo, C::kSwz),
                     make_sdesc(k0 + kk * 32, 16, sbo, C::kSwz), idS, kk > 0);
        mma_commit(&bars->s_full[b]);
        mma_commit(&bars->q_empty[qs]);
      };
      issue_S(0);
      if (n_items > 1) issue_S(1);
      for (int it = 0; it < n_items; ++it) {
        const int b = it & 1;
        const int i = it / NM;
        mbar_wait(&bars->p_full[b], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t v0 = smem_u32(sV + (i & 1) * C::kKVSlot);
#pragma unroll 4
        for (int kk = 0; kk < LP / 16; ++kk)
          mma_f16_ts(tmem + b * 256 + C::kOCol, tmem + b * 256 + kk * 8,
                     make_sdesc(v0 + kk * 16 * C::kRowBytes, C::kKVSlot, sbo, C::kSwz), idO, kk > 0);
        mma_commit(&bars->o_full[b]);
        if (it % NM == NM - 1) mma_commit(&bars->kv_empty[i & 1]);
        if (it + 2 < n_items) issue_S(it + 2);
      }
    }
  } else if (warp < 6) {
    // ===================== softmax (warps 2..5): back-to-back over items =====================
    const int qd = warp & 3;
    const int r_in = qd * 32 + lane;
    const uint32_t t_lane = (uint32_t)(qd * 32) << 16;
    for (int it = 0; it < n_items; ++it) {
      const int b = it & 1, m = it % NM;
      const uint32_t tb = tmem + t_lane + b * 256;
      const bool active = m * kMRows + qd * 32 < L;   // warp-uniform: any valid row?
      mbar_wait(&bars->s_full[b], (it >> 1) & 1);
      tc_fence_after();
      float inv = 0.f;
      if (active) {
        float mx = -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < LP; c0 += 64) {          // pass 1: row max
          uint32_t r[64];
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if (c0 + g * 16 < LP) tmem_ld16(tb + c0 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&r[g * 16]));
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 64; ++t)
            if (c0 + t < LP && c0 + t < L) mx = fmaxf(mx, __uint_as_float(r[t]));
        }
        const float mxs = mx * scale_log2;
        float sum = 0.f;
#pragma unroll
        for (int c0 = 0; c0 < LP; c0 += 64) {          // pass 2: exp2, P over consumed S cols
          uint32_t r[64];
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if (c0 + g * 16 < LP) tmem_ld16(tb + c0 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&r[g * 16]));
          tmem_wait_ld();
          uint32_t pk[32];
#pragma unroll
          for (int t = 0; t < 64; t += 2) {
            const int j = c0 + t;
            const float p0 = j < L ? ex2(fmaf(__uint_as_float(r[t]), scale_log2, -mxs)) : 0.f;
            const float p1 = j + 1 < L ? ex2(fmaf(__uint_as_float(r[t + 1]), scale_log2, -mxs)) : 0.f;
            sum += p0 + p1;
            pk[t >> 1] = pack2l<T>(p0, p1);
          }
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if (c0 + g * 16 < LP) tmem_st8(tb + c0 / 2 + g * 8, &pk[g * 8]);
        }
        tmem_wait_st();
        inv = __frcp_rn(sum);
      }
      sInv[b * 128 + r_in] = inv;
      tc_fence_before();
      mbar_arrive(&bars->p_full[b]);
    }
  } else {
    // ============ epilogue (warps 6..9): O rows -> 1/rowsum -> staging -> TMA store ============
    const int qd = warp & 3;
    const int r_in = qd * 32 + lane;
    const uint32_t t_lane = (uint32_t)(qd * 32) << 16;
    const uint32_t oswz = (uint32_t)((r_in * C::kRowBytes) >> 7) & (C::kChunks - 1);
    uint8_t* orow = sO + r_in * C::kRowBytes;
    const bool leader = (threadIdx.x == 192);
    for (int it = 0; it < n_items; ++it) {
      const int b = it & 1, m = it % NM;
      const int unit = blockIdx.x + (it / NM) * gridDim.x;
      const bool active = m * kMRows + qd * 32 < L;
      mbar_wait(&bars->o_full[b], (it >> 1) & 1);   // PV done => P (and sInv) were published
      tc_fence_after();
      uint32_t o[D];
      if (active) {
#pragma unroll
        for (int g = 0; g < D / 16; ++g)
          tmem_ld16(tmem + t_lane + b * 256 + C::kOCol + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&o[g * 16]));
        tmem_wait_ld();
      }
      const float inv = sInv[b * 128 + r_in];
      tc_fence_before();
      mbar_arrive(&bars->buf_free[b]);
      if (leader) bulk_wait_read<0>();
      named_sync(1, 128);
      if (active) {
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          *reinterpret_cast<uint4*>(orow + ((c ^ oswz) << 4)) = make_uint4(
              pack2l<T>(__uint_as_float(o[8 * c]) * inv, __uint_as_float(o[8 * c + 1]) * inv),
              pack2l<T>(__uint_as_float(o[8 * c + 2]) * inv, __uint_as_float(o[8 * c + 3]) * inv),
              pack2l<T>(__uint_as_float(o[8 * c + 4]) * inv, __uint_as_float(o[8 * c + 5]) * inv),
              pack2l<T>(__uint_as_float(o[8 * c + 6]) * inv, __uint_as_float(o[8 * c + 7]) * inv));
      }
      fence_proxy_async_smem();
      named_sync(2, 128);
      if (leader) {
        tma_store_3d(&tm_o, sO, 0, m * kMRows, unit);
        bulk_commit();
      }
    }
    if (leader) bulk_wait_read<0>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---- variant for d <= 32: 2 CTAs/SM, softmax warps also run the epilogue ----
constexpr int kThreads2 = 192;  // 2-CTA/SM variant (d <= 32)

template <int D, int LP>
struct LCfg2 {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kQBytes = kMRows * kRowBytes;
  static constexpr int kKVBytes = LP * kRowBytes;          // one of K / V for a unit
  static constexpr int kMTiles = (LP + kMRows - 1) / kMRows;
  static constexpr int kKVStages = 2;
  static constexpr int kQStages = 2;
  static constexpr uint32_t kSwz = D == 16 ? 6u : (D == 32 ? 4u : 2u);
  // K/V tiles must keep the 8-row swizzle atoms 1024-aligned
  static constexpr int kKVSlot = (kKVBytes + 1023) / 1024 * 1024;
  static constexpr int kSmem = 1024 + kKVStages * 2 * kKVSlot + kQStages * kQBytes + kQBytes + 256;
  static constexpr int kCtasPerSm = (2 * (kSmem + 1024) <= 228 * 1024) ? 2 : 1;
  static constexpr int kChunks = kRowBytes / 16;
  static constexpr uint32_t kOCol = ((LP / 2 + 15) / 16) * 16;
  static constexpr uint32_t kTmemCols = 256;
  static_assert(kOCol + D <= 256, "O must fit in the consumed S columns");
};

struct LBarriers2 {
  uint64_t kv_full[2], kv_empty[2], q_full[2], q_empty[2];
  uint64_t s_full, p_full, o_full, o_free;
  uint32_t tmem_base;
};

template <typename T>
__device__ __forceinline__ uint32_t pack2l_2(float a, float b) {
  if constexpr (DT<T>::id == FWA_BF16) {
    __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  } else {
    __half2 h2 = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  }
}

template <typename T, int D, int LP>
__global__ void __launch_bounds__(kThreads2, LCfg2<D, LP>::kCtasPerSm)
fwd_tc_large2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                    int n_units, int L, float scale_log2) {
  using C = LCfg2<D, LP>;
  constexpr bool kBF16 = DT<T>::id == FWA_BF16;
  constexpr int NM = C::kMTiles;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;                                   // [kv stage] K
  uint8_t* sV = sK + C::kKVStages * C::kKVSlot;         // [kv stage] V
  uint8_t* sQ = sV + C::kKVStages * C::kKVSlot;         // [q stage] Q
  uint8_t* sO = sQ + C::kQStages * C::kQBytes;          // staging
  LBarriers2* bars = reinterpret_cast<LBarriers2*>(sO + C::kQBytes);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars->kv_full[s], 1);
      mbar_init(&bars->kv_empty[s], 1);
      mbar_init(&bars->q_full[s], 1);
      mbar_init(&bars->q_empty[s], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->p_full, 128);
    mbar_init(&bars->o_full, 1);
    mbar_init(&bars->o_free, 128);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_o);
  }
  if (warp == 1) tmem_alloc(&bars->tmem_base, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const int n_local =
      n_units > (int)blockIdx.x ? (n_units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  griddep_launch_dependents();

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      griddep_wait();
      const uint64_t pol = policy_evict_first();
      int qi = 0;
      for (int i = 0; i < n_local; ++i) {
        const int unit = blockIdx.x + i * gridDim.x;
        const int kst = i & 1;
        mbar_wait(&bars->kv_empty[kst], ((i >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->kv_full[kst], 2 * C::kKVBytes);
        tma_load_3d(sK + kst * C::kKVSlot, &tm_k, &bars->kv_full[kst], 0, 0, unit, pol);
        tma_load_3d(sV + kst * C::kKVSlot, &tm_v, &bars->kv_full[kst], 0, 0, unit, pol);
        for (int m = 0; m < NM; ++m, ++qi) {
          const int qs = qi & 1;
          mbar_wait(&bars->q_empty[qs], ((qi >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&bars->q_full[qs], C::kQBytes);
          tma_load_3d(sQ + qs * C::kQBytes, &tm_q, &bars->q_full[qs], 0, m * kMRows, unit, pol);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_f16(kBF16, 128, LP, false, false);
      constexpr uint32_t idO = make_idesc_f16(kBF16, 128, D, false, true);
      constexpr uint32_t sbo = 8 * C::kRowBytes;
      int qi = 0;
      for (int i = 0; i < n_local; ++i) {
        const int kst = i & 1;
        mbar_wait(&bars->kv_full[kst], (i >> 1) & 1);
        const uint32_t k0 = smem_u32(sK + kst * C::kKVSlot);
        const uint32_t v0 = smem_u32(sV + kst * C::kKVSlot);
        for (int m = 0; m < NM; ++m, ++qi) {
          const int qs = qi & 1;
          mbar_wait(&bars->q_full[qs], (qi >> 1) & 1);
          if (qi > 0) mbar_wait(&bars->o_free, (qi - 1) & 1);   // epilogue pulled O(qi-1)
          tc_fence_after();
          const uint32_t q0 = smem_u32(sQ + qs * C::kQBytes);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_f16_ss(tmem, make_sdesc(q0 + kk * 32, 16, sbo, C::kSwz),
                       make_sdesc(k0 + kk * 32, 16, sbo, C::kSwz), idS, kk > 0);
          mma_commit(&bars->s_full);
          mma_commit(&bars->q_empty[qs]);
          mbar_wait(&bars->p_full, qi & 1);
          tc_fence_after();
#pragma unroll 4
          for (int kk = 0; kk < LP / 16; ++kk)
            mma_f16_ts(tmem + C::kOCol, tmem + kk * 8,
                       make_sdesc(v0 + kk * 16 * C::kRowBytes, C::kKVSlot, sbo, C::kSwz), idO,
                       kk > 0);
          mma_commit(&bars->o_full);
        }
        mma_commit(&bars->kv_empty[kst]);
      }
    }
  } else {
    // ===================== softmax + epilogue (warps 2..5) =====================
    const int qd = warp & 3;
    const int r_in = qd * 32 + lane;               // row within the M-tile = TMEM lane
    const uint32_t t_lane = (uint32_t)(qd * 32) << 16;
    const uint32_t oswz = (uint32_t)((r_in * C::kRowBytes) >> 7) & (C::kChunks - 1);
    uint8_t* orow = sO + r_in * C::kRowBytes;
    const bool leader = (threadIdx.x == 64);
    int qi = 0;
    for (int i = 0; i < n_local; ++i) {
      const int unit = blockIdx.x + i * gridDim.x;
      for (int m = 0; m < NM; ++m, ++qi) {
        const bool active = m * kMRows + qd * 32 < L;   // warp-uniform: any valid row?
        mbar_wait(&bars->s_full, qi & 1);
        tc_fence_after();
        float inv = 0.f;
        if (active) {
          // pass 1: row max over the L valid keys (64 columns per tcgen05.wait::ld)
          float mx = -INFINITY;
#pragma unroll
          for (int c0 = 0; c0 < LP; c0 += 64) {
            uint32_t r[64];
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (c0 + g * 16 < LP) tmem_ld16(tmem + t_lane + c0 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&r[g * 16]));
            tmem_wait_ld();
#pragma unroll
            for (int t = 0; t < 64; ++t)
              if (c0 + t < LP && c0 + t < L) mx = fmaxf(mx, __uint_as_float(r[t]));
          }
          const float mxs = mx * scale_log2;
          // pass 2: p = exp2(s*scale*log2e - max); P (16-bit pairs) over consumed S columns:
          // cols [c0/2, c0/2+32) hold keys [c0, c0+64), all already read
          float sum = 0.f;
#pragma unroll
          for (int c0 = 0; c0 < LP; c0 += 64) {
            uint32_t r[64];
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (c0 + g * 16 < LP) tmem_ld16(tmem + t_lane + c0 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&r[g * 16]));
            tmem_wait_ld();
            uint32_t pk[32];
#pragma unroll
            for (int t = 0; t < 64; t += 2) {
              const int j = c0 + t;
              const float p0 = j < L ? ex2(fmaf(__uint_as_float(r[t]), scale_log2, -mxs)) : 0.f;
              const float p1 = j + 1 < L ? ex2(fmaf(__uint_as_float(r[t + 1]), scale_log2, -mxs)) : 0.f;
              sum += p0 + p1;
              pk[t >> 1] = pack2l_2<T>(p0, p1);
            }
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (c0 + g * 16 < LP) tmem_st8(tmem + t_lane + c0 / 2 + g * 8, &pk[g * 8]);
          }
          tmem_wait_st();
          inv = __frcp_rn(sum);
        }
        tc_fence_before();
        mbar_arrive(&bars->p_full);
        // ---- epilogue ----
        mbar_wait(&bars->o_full, qi & 1);
        tc_fence_after();
        uint32_t o[D];
        if (active) {
#pragma unroll
          for (int g = 0; g < D / 16; ++g)
            tmem_ld16(tmem + t_lane + C::kOCol + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&o[g * 16]));
          tmem_wait_ld();
        }
        tc_fence_before();
        mbar_arrive(&bars->o_free);
        if (leader) bulk_wait_read<0>();
        named_sync(1, 128);
        if (active) {
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            *reinterpret_cast<uint4*>(orow + ((c ^ oswz) << 4)) = make_uint4(
                pack2l_2<T>(__uint_as_float(o[8 * c]) * inv, __uint_as_float(o[8 * c + 1]) * inv),
                pack2l_2<T>(__uint_as_float(o[8 * c + 2]) * inv, __uint_as_float(o[8 * c + 3]) * inv),
                pack2l_2<T>(__uint_as_float(o[8 * c + 4]) * inv, __uint_as_float(o[8 * c + 5]) * inv),
                pack2l_2<T>(__uint_as_float(o[8 * c + 6]) * inv, __uint_as_float(o[8 * c + 7]) * inv));
        }
        fence_proxy_async_smem();
        named_sync(2, 128);
        if (leader) {
          tma_store_3d(&tm_o, sO, 0, m * kMRows, unit);
          bulk_commit();
        }
      }
    }
    if (leader) bulk_wait_read<0>();  // smem reads done; the grid's completion flushes the writes
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

template <typename T, int D, int LP>
int launch_large_t(const Geom& g, int dtype, const void* q, const void* k, const void* v, void* o,
                   cudaStream_t s) {
  CUtensorMap mq, mk, mv, mo;
  int rc;
  if ((rc = get_units_map(&mq, q, dtype, g.units, g.L, g.d, kMRows, 1))) return rc;
  if ((rc = get_units_map(&mk, k, dtype, g.units, g.L, g.d, LP, 1))) return rc;
  if ((rc = get_units_map(&mv, v, dtype, g.units, g.L, g.d, LP, 1))) return rc;
  if ((rc = get_units_map(&mo, o, dtype, g.units, g.L, g.d, kMRows, 1))) return rc;
  const float sl2 = g.scale * 1.4426950408889634f;
  if constexpr (D >= 64) {
    // d = 64: one CTA per SM, items double-buffered in 512 TMEM columns
    using C = LCfg<D, LP>;
    auto kern = fwd_tc_large_kernel<T, D, LP>;
    if ((rc = ensure_smem_attr((const void*)kern, (int)(C::kSmem), "cudaFuncSetAttribute(fwd_tc_large)"))) return rc;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(g.units, (int64_t)device_sm_count()));
    rc = check_cuda(launch_pdl(kern, dim3(grid), dim3(kThreads), (size_t)C::kSmem, s, mq, mk, mv, mo,
                               (int)g.units, (int)g.L, sl2),
                    "fwd_tc_large_kernel launch");
  } else {
    // d <= 32: two CTAs per SM (more softmax warps per SM sub-partition)
    using C = LCfg2<D, LP>;
    auto kern = fwd_tc_large2_kernel<T, D, LP>;
    if ((rc = ensure_smem_attr((const void*)kern, (int)(C::kSmem), "cudaFuncSetAttribute(fwd_tc_large2)"))) return rc;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>(g.units, (int64_t)device_sm_count() * C::kCtasPerSm));
    rc = check_cuda(launch_pdl(kern, dim3(grid), dim3(kThreads2), (size_t)C::kSmem, s, mq, mk, mv,
                               mo, (int)g.units, (int)g.L, sl2),
                    "fwd_tc_large2_kernel launch");
  }
  if (rc) return rc;
  count_launch();
  return FWA_OK;
}

template <typename T, int D>
int large_dispatch_l(const Geom& g, int dtype, const void* q, const void* k, const void* v, void* o,
                     cudaStream_t s) {
  const int lp = (g.L + 15) / 16 * 16;
  switch (lp) {
    case 80: return launch_large_t<T, D, 80>(g, dtype, q, k, v, o, s);
    case 96: return launch_large_t<T, D, 96>(g, dtype, q, k, v, o, s);
    case 112: return launch_large_t<T, D, 112>(g, dtype, q, k, v, o, s);
    case 128: return launch_large_t<T, D, 128>(g, dtype, q, k, v, o, s);
    case 144: return launch_large_t<T, D, 144>(g, dtype, q, k, v, o, s);
    case 160: return launch_large_t<T, D, 160>(g, dtype, q, k, v, o, s);
    case 176: return launch_large_t<T, D, 176>(g, dtype, q, k, v, o, s);
    case 192: return launch_large_t<T, D, 192>(g, dtype, q, k, v, o, s);
    case 208: return launch_large_t<T, D, 208>(g, dtype, q, k, v, o, s);
    case 224: return launch_large_t<T, D, 224>(g, dtype, q, k, v, o, s);
    case 240: return launch_large_t<T, D, 240>(g, dtype, q, k, v, o, s);
    case 256: return launch_large_t<T, D, 256>(g, dtype, q, k, v, o, s);
  }
  return fail(FWA_ERR_CAPACITY, "tcgen05 large-window forward: unsupported L");
}

}  // namespace

bool tc_fwd_large_supported(const Geom& g, int dtype, bool has_bias, bool has_mask) {
  if (tc_fwd_flat_supported(g, dtype, has_bias, has_mask)) return true;
  if (has_bias || has_mask) return false;
  if (dtype != FWA_F16 && dtype != FWA_BF16) return false;
  if (g.L <= 64 || g.L > 256) return false;
  if (g.d != 16 && g.d != 32 && g.d != 64) return false;
  return g.units <= ((int64_t)1 << 31);
}

size_t tc_fwd_large_smem(const Geom& g) {
  if (tc_fwd_flat_supported(g, FWA_F16, false, false)) return tc_fwd_flat_smem(g);
  const int lp = (g.L + 15) / 16 * 16;
  const int row = g.d * 2;
  const int kv = (lp * row + 1023) / 1024 * 1024;
  if (g.d >= 64) return 1024 + 2 * 2 * kv + 4 * 128 * row + 1024 + 256;  // LCfg
  return 1024 + 2 * 2 * kv + 3 * 128 * row + 256;                       // LCfg2
}

int launch_fwd_tc_large(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                        const float* bias, const float* mask, void* o, cudaStream_t s) {
  if (tc_fwd_flat_supported(g, dtype, bias != nullptr, mask != nullptr))
    return launch_fwd_tc_flat(g, dtype, q, k, v, bias, mask, o, s);
  if (bias || mask) return fail(FWA_ERR_CAPACITY, "tcgen05 large-window forward: bias/mask need L % 16 == 0");
  const bool bf = dtype == FWA_BF16;
  switch (g.d) {
    case 16: return bf ? large_dispatch_l<__nv_bfloat16, 16>(g, dtype, q, k, v, o, s)
                       : large_dispatch_l<__half, 16>(g, dtype, q, k, v, o, s);
    case 32: return bf ? large_dispatch_l<__nv_bfloat16, 32>(g, dtype, q, k, v, o, s)
                       : large_dispatch_l<__half, 32>(g, dtype, q, k, v, o, s);
    case 64: return bf ? large_dispatch_l<__nv_bfloat16, 64>(g, dtype, q, k, v, o, s)
                       : large_dispatch_l<__half, 64>(g, dtype, q, k, v, o, s);
  }
  return fail(FWA_ERR_CAPACITY, "tcgen05 large-window forward: unsupported head_dim");
}

}  // namespace fwa
