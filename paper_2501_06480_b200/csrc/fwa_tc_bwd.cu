// fwa_tc_bwd.cu — Flash Window Attention backward on tcgen05 + TMA (sm_100a).
//
// Algorithm 2 of the paper (reference flash.py:187-266) for
// f16/bf16, L <= 64, d in {16, 32, 64}. Same tile packing as the forward
// (two units per 128-row tile, 3-D TMA box (d, 64, 2), rows >= L zero-filled):
//
//   S  = Q K^T          tcgen05 SS, M=128 N=128 K=d  -> TMEM [0,128)
//   dP = dO V^T         tcgen05 SS, M=128 N=128 K=d  -> TMEM [128,256)
//   (every MMA is issued once per unit with complementary disable-output-lane
//   masks, so both units share TMEM columns: S [0,64), dP [64,128))
//   softmax warps (thread = query row = TMEM lane): P = softmax(scale*S [+bias
//     +mask]), rho = sum_j P dP, dS = scale * P (dP - rho)  (flash.py:133-138,
//     :241-242); P and dS go to shared memory as [query][64 keys] SW128 tiles.
//     With dBias requested, P (dP - rho) is accumulated per CTA in TMEM [128,192)
//     (the grid is period-aligned so every tile of a CTA has the same heads) and
//     reduced over CTAs in a fixed order afterwards (deterministic).
//   dV = P^T dO         A = P read MN-major (the same bytes), B = dO MN-major
//   dK = dS^T Q         A = dS MN-major, B = Q MN-major
//   dQ = dS K           A = dS K-major, B = K MN-major
//   (gradient accumulators reuse the S/dP columns once they are in registers)
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
constexpr int kPBytes = 16 * 1024;  // [128 query rows][64 keys of the row's own unit], SW128

template <int D>
struct BCfg {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTileBytes = kTileRows * kRowBytes;
  static constexpr int kStageBytes = 4 * kTileBytes;  // Q, K, V, dO
  static constexpr int kStages = D <= 16 ? 4 : 2;
  static constexpr int kCtasPerSm = D <= 32 ? 2 : 1;
  static constexpr uint32_t kSwz = D == 16 ? 6u : (D == 32 ? 4u : 2u);
  // + 16 KB: the CTA's (bias + mask) * log2e rows as f16 (ADD variants)
  static constexpr int kSmem = kStages * kStageBytes + 3 * kPBytes + 256;
  static constexpr int kChunks = kRowBytes / 16;
  // TMEM (lane = tile row): S [0,64) | dP [64,128) | dBias acc [128,192) |
  // gradients dV, dK, dQ at [0,3d) when they fit in the S/dP columns, else [192,192+3d).
  static constexpr uint32_t kTdP = 64, kTdB = 128;
  static constexpr uint32_t kTg = 3 * D <= 128 ? 0 : 192;
  static constexpr uint32_t kTdV = kTg, kTdK = kTg + D, kTdQ = kTg + 2 * D;
  static constexpr uint32_t kTmemCols = kTg + 3 * D <= 256 ? 256 : 512;
};

struct BwdBarriers {
  uint64_t full[4];
  uint64_t empty[4];
  uint64_t s_full, p_ready, ds_ready, grad_done, grad_free;
  uint32_t tmem_base;
};

struct BwdAddArgs {
  const float* bias;   // [heads][L][L] or null
  const float* mask;   // [nW][L][L] or null
  float* dbias_ws;     // [grid][128][64] per-CTA dS partials (DBIAS) or null
  int heads;
  int mask_windows;
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

template <typename T, int D, int LK, bool ADD, bool DBIAS>
__global__ void __launch_bounds__(kThreads, BCfg<D>::kCtasPerSm)
bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
              const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
              const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dk,
              const __grid_constant__ CUtensorMap tm_dv, int n_tiles, int L_rt, float scale,
              BwdAddArgs add, LayoutArgs lay, unsigned int* err_flags) {
  using C = BCfg<D>;
  constexpr bool kBF16 = DT<T>::id == FWA_BF16;
  const int L = LK > 0 ? LK : L_rt;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sStage = smem;                                  // [stage][Q|K|V|dO]
  uint8_t* sP = smem + C::kStages * C::kStageBytes;
  uint8_t* sDS = sP + kPBytes;
  uint8_t* sAdd = sDS + kPBytes;  // [128 rows][64] f16, SW128-style chunk swizzle
  BwdBarriers* bars = reinterpret_cast<BwdBarriers*>(sAdd + kPBytes);
  auto slot = [&](int st, int which) { return sStage + st * C::kStageBytes + which * C::kTileBytes; };
  // The swizzled layouts need a 1024-byte aligned base; the budget leaves no slack
  // for manual alignment (2 CTAs/SM), so verify it and report instead of computing garbage.
  if (smem_u32(smem) & 1023u) {
    if (threadIdx.x == 0 && err_flags) atomicOr(err_flags, 1u);
    return;
  }

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // key chunks >= ceil(L/8) of P and dS are never written: they must read as zero
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
        constexpr int kUB = kUnitRows * C::kRowBytes;
        load_tile<kUB>(slot(st, 0), &tm_q, &bars->full[st], tile, lay.mode, lay.heads, pol);
        load_tile<kUB>(slot(st, 1), &tm_k, &bars->full[st], tile, lay.mode, lay.heads, pol);
        load_tile<kUB>(slot(st, 2), &tm_v, &bars->full[st], tile, lay.mode, lay.heads, pol);
        load_tile<kUB>(slot(st, 3), &tm_do, &bars->full[st], tile, lay.mode, lay.heads, pol);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (per unit, complementary lane masks) =====================
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_f16(kBF16, 128, 64, false, false);
      constexpr uint32_t idMN = make_idesc_f16(kBF16, 128, D, true, true);    // dV, dK
      constexpr uint32_t idQ = make_idesc_f16(kBF16, 128, D, false, true);    // dQ
      constexpr uint32_t sbo_row = 8 * C::kRowBytes;
      constexpr uint32_t kUnitBytes = kUnitRows * C::kRowBytes;  // 64 rows of one unit
      const uint32_t p0 = smem_u32(sP), ds0 = smem_u32(sDS);
      for (int i = 0; i < n_local; ++i) {
        const int st = i % C::kStages;
        const uint32_t q0 = smem_u32(slot(st, 0)), k0 = smem_u32(slot(st, 1));
        const uint32_t v0 = smem_u32(slot(st, 2)), do0 = smem_u32(slot(st, 3));
        mbar_wait(&bars->full[st], (i / C::kStages) & 1);
        if (i > 0) mbar_wait(&bars->grad_free, (i - 1) & 1);  // S/dP/gradient columns free
        tc_fence_after();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t lo = u ? ~0u : 0u, hi = u ? 0u : ~0u;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)   // S_u = Q K_u^T
            mma_f16_ss_m(tmem, make_sdesc(q0 + kk * 32, 16, sbo_row, C::kSwz),
                         make_sdesc(k0 + u * kUnitBytes + kk * 32, 16, sbo_row, C::kSwz), idS,
                         kk > 0, lo, lo, hi, hi);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)   // dP_u = dO V_u^T
            mma_f16_ss_m(tmem + C::kTdP, make_sdesc(do0 + kk * 32, 16, sbo_row, C::kSwz),
                         make_sdesc(v0 + u * kUnitBytes + kk * 32, 16, sbo_row, C::kSwz), idS,
                         kk > 0, lo, lo, hi, hi);
        }
        mma_commit(&bars->s_full);
        // dV_u = P_u^T dO_u : A = P read MN-major (M = key, K = query; atom 1 = unit-1 rows)
        mbar_wait(&bars->p_ready, i & 1);
        tc_fence_after();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t lo = u ? ~0u : 0u, hi = u ? 0u : ~0u;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_f16_ss_m(tmem + C::kTdV, make_sdesc(p0 + kk * 2048, 8192, 1024, 2),
                         make_sdesc(do0 + u * kUnitBytes + kk * 16 * C::kRowBytes, C::kTileBytes,
                                    sbo_row, C::kSwz),
                         idMN, kk > 0, lo, lo, hi, hi);
        }
        // dK_u = dS_u^T Q_u ; dQ_u = dS_u K_u
        mbar_wait(&bars->ds_ready, i & 1);
        tc_fence_after();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t lo = u ? ~0u : 0u, hi = u ? 0u : ~0u;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_f16_ss_m(tmem + C::kTdK, make_sdesc(ds0 + kk * 2048, 8192, 1024, 2),
                         make_sdesc(q0 + u * kUnitBytes + kk * 16 * C::kRowBytes, C::kTileBytes,
                                    sbo_row, C::kSwz),
                         idMN, kk > 0, lo, lo, hi, hi);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_f16_ss_m(tmem + C::kTdQ, make_sdesc(ds0 + kk * 32, 16, 1024, 2),
                         make_sdesc(k0 + u * kUnitBytes + kk * 16 * C::kRowBytes, C::kTileBytes,
                                    sbo_row, C::kSwz),
                         idQ, kk > 0, lo, lo, hi, hi);
        }
        mma_commit(&bars->grad_done);
      }
    }
  } else {
    // ============ softmax / dS / epilogue (warps 2..5; thread = row = TMEM lane) ============
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int ul = row >> 6;
    const int r_in = row & 63;
    const uint32_t t_lane = (uint32_t)(q * 32) << 16;
    const uint32_t pswz = (uint32_t)(row & 7);
    const int prow_off = (row >> 3) * 1024 + (row & 7) * 128;
    const uint32_t oswz = (uint32_t)((row * C::kRowBytes) >> 7) & (C::kChunks - 1);
    const bool leader = (threadIdx.x == 64);
    const int p_chunks = LK > 0 ? (LK + 7) / 8 : 8;
    const float scale_log2 = scale * 1.4426950408889634f;
    uint8_t* arow = sAdd + prow_off;
    if constexpr (ADD) {
      // Cooperative, coalesced fill of the CTA's two (bias + mask) * log2e tiles
      // (every tile of this CTA has the same (w, h) pair per slot): f16, swizzled rows.
      const int ct = threadIdx.x - 64;             // 0..127 within the softmax warps
      for (int i = ct; i < 2 * 64 * 64 / 2; i += 128)
        reinterpret_cast<uint32_t*>(sAdd)[i] = 0u;
      named_sync(3, 128);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int uu = 2 * (int)blockIdx.x + u;
        const int hd = uu % add.heads;
        const int w = (uu / add.heads) % add.mask_windows;
        const float* __restrict__ bt = add.bias ? add.bias + (size_t)hd * L * L : nullptr;
        const float* __restrict__ mt = add.mask ? add.mask + (size_t)w * L * L : nullptr;
        for (int e = ct; e < L * L; e += 128) {
          const float a = ((bt ? __ldg(bt + e) : 0.f) + (mt ? __ldg(mt + e) : 0.f)) * 1.4426950408889634f;
          const int r = u * 64 + e / L, j = e % L;
          uint8_t* dst = sAdd + (r >> 3) * 1024 + (r & 7) * 128 + ((((j >> 3) ^ (r & 7))) << 4) + (j & 7) * 2;
          *reinterpret_cast<__half*>(dst) = __float2half_rn(a);
        }
      }
      named_sync(3, 128);
    }
    if constexpr (DBIAS) {
      uint32_t z[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) z[j] = 0u;
#pragma unroll
      for (int g = 0; g < 4; ++g) tmem_st16(tmem + t_lane + C::kTdB + g * 16, z);
      tmem_wait_st();
    }
    for (int i = 0; i < n_local; ++i) {
      const int tile = blockIdx.x + i * gridDim.x;
      const int st = i % C::kStages;
      mbar_wait(&bars->s_full, i & 1);
      tc_fence_after();
      uint32_t s[64], dp[64];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (LK == 0 || g * 16 < LK) {
          tmem_ld16(tmem + t_lane + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&s[g * 16]));
          tmem_ld16(tmem + t_lane + C::kTdP + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&dp[g * 16]));
        }
      }
      tmem_wait_ld();
      // P = softmax(scale*S [+ bias + mask]) over the L valid keys (normalised: dV needs true P)
      float mx = -INFINITY;
      if constexpr (ADD) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (LK > 0 && 8 * c >= LK) break;
          const uint4 av = *reinterpret_cast<const uint4*>(arow + ((c ^ pswz) << 4));
          const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int j = 8 * c + 2 * t;
            const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&aw[t]));
            const float t0 = fmaf(__uint_as_float(s[j]), scale_log2, a.x);
            const float t1 = fmaf(__uint_as_float(s[j + 1]), scale_log2, a.y);
            s[j] = __float_as_uint(t0);
            s[j + 1] = __float_as_uint(t1);
            if (j < L) mx = fmaxf(mx, t0);
            if (j + 1 < L) mx = fmaxf(mx, t1);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
          if (j + 1 < L) {
            float m3;
            asm("max.f32 %0, %1, %2, %3;" : "=f"(m3) : "f"(mx), "f"(__uint_as_float(s[j])), "f"(__uint_as_float(s[j + 1])));
            mx = m3;
          } else if (j < L) {
            mx = fmaxf(mx, __uint_as_float(s[j]));
          }
        }
      }
      const float mxs = ADD ? mx : mx * scale_log2;
      const float sl2 = ADD ? 1.f : scale_log2;
      float2 sum2 = make_float2(0.f, 0.f);
      const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-mxs, -mxs);
#pragma unroll
      for (int j = 0; j < 64; j += 2) {
        // packed f32x2 math; a quarter of the exponentials on the FMA pipe (poly)
        const float2 a = __ffma2_rn(make_float2(__uint_as_float(s[j]), __uint_as_float(s[j + 1])), sc2, nm2);
        float2 p = (j & 7) == 6 ? ex2_poly2(a) : make_float2(ex2(a.x), ex2(a.y));
        if (j >= L) p.x = 0.f;
        if (j + 1 >= L) p.y = 0.f;
        s[j] = __float_as_uint(p.x);
        s[j + 1] = __float_as_uint(p.y);
        sum2 = __fadd2_rn(sum2, p);
      }
      const float inv = __frcp_rn(sum2.x + sum2.y);
      // P (normalised) -> smem chunk by chunk; rho = sum_j P_j dP_j
      float rho = 0.f;
      uint8_t* prow = sP + prow_off;
      float2 rho2 = make_float2(0.f, 0.f);
      const float2 inv2 = make_float2(inv, inv);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int j = 8 * c + 2 * t;
          const float2 pa = __fmul2_rn(make_float2(__uint_as_float(s[j]), __uint_as_float(s[j + 1])), inv2);
          s[j] = __float_as_uint(pa.x);
          s[j + 1] = __float_as_uint(pa.y);
          // keys >= L carry p = 0, so they add nothing to rho
          rho2 = __ffma2_rn(pa, make_float2(j < L ? __uint_as_float(dp[j]) : 0.f,
                                            j + 1 < L ? __uint_as_float(dp[j + 1]) : 0.f), rho2);
          w[t] = pack2<T>(pa.x, pa.y);
        }
        if (c < p_chunks)
          *reinterpret_cast<uint4*>(prow + ((c ^ pswz) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      rho = rho2.x + rho2.y;
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->p_ready);
      // dS = scale * P * (dP - rho)  (keys >= L forced to exactly 0); dBias += P (dP - rho)
      uint8_t* dsrow = sDS + prow_off;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (LK > 0 && g * 16 >= LK) break;
        uint32_t acc[16];
        if constexpr (DBIAS) {
          tmem_ld16(tmem + t_lane + C::kTdB + g * 16, *reinterpret_cast<uint32_t(*)[16]>(acc));
          tmem_wait_ld();
        }
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int c = 2 * g + h2;
          uint32_t w[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int j = 8 * c + 2 * t;
            const float a = j < L ? __uint_as_float(s[j]) * (__uint_as_float(dp[j]) - rho) : 0.f;
            const float b = j + 1 < L ? __uint_as_float(s[j + 1]) * (__uint_as_float(dp[j + 1]) - rho) : 0.f;
            if constexpr (DBIAS) {
              acc[8 * h2 + 2 * t] = __float_as_uint(__uint_as_float(acc[8 * h2 + 2 * t]) + a);
              acc[8 * h2 + 2 * t + 1] = __float_as_uint(__uint_as_float(acc[8 * h2 + 2 * t + 1]) + b);
            }
            w[t] = pack2<T>(a * scale, b * scale);
          }
          if (c < p_chunks)
            *reinterpret_cast<uint4*>(dsrow + ((c ^ pswz) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if constexpr (DBIAS) tmem_st16(tmem + t_lane + C::kTdB + g * 16, acc);
      }
      if constexpr (DBIAS) tmem_wait_st();
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
        constexpr int kUB = kUnitRows * C::kRowBytes;
        store_tile<kUB>(&tm_dq, slot(st, 0), tile, lay.mode, lay.heads);
        store_tile<kUB>(&tm_dk, slot(st, 1), tile, lay.mode, lay.heads);
        store_tile<kUB>(&tm_dv, slot(st, 2), tile, lay.mode, lay.heads);
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(&bars->empty[st]);   // stage may be refilled
      }
    }
    if constexpr (DBIAS) {
      // this CTA's dS partials: ws[cta][row][0..63] (reduced per head in fixed order later)
      float* wrow = add.dbias_ws + ((size_t)blockIdx.x * kTileRows + row) * 64;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint32_t acc[16];
        tmem_ld16(tmem + t_lane + C::kTdB + g * 16, *reinterpret_cast<uint32_t(*)[16]>(acc));
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 16; t += 4)
          *reinterpret_cast<float4*>(wrow + g * 16 + t) =
              make_float4(__uint_as_float(acc[t]), __uint_as_float(acc[t + 1]),
                          __uint_as_float(acc[t + 2]), __uint_as_float(acc[t + 3]));
      }
    }
    if (leader) bulk_wait_read<0>();  // smem reads done; the grid's completion flushes the writes
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

// dbias[h][i][j] = sum over (CTA c, slot u) with (2c+u) % heads == h of ws[c][64u + i][j].
// One warp per element: lane l sums c = l, l+32, ... in order, then a fixed shuffle tree —
// the same order every run (deterministic, no atomics).
// dbias[h][i][j] = sum over the tile slots t = 2c + u (CTA c, unit u) whose head is h. A block
// covers 32 consecutive (h, i, j) (threadIdx.x; j fastest, so a warp reads a contiguous row
// segment of each slot's [64][64] partial) x 8 slot groups (threadIdx.y: group g takes the
// head's slots g, g+8, g+16, ... in ascending order); the 8 group sums are then added in g
// order -- a fixed association, so the result is deterministic. (A warp per element
// gathering words 32 KB apart took 12 us for 7 MB at Swin-T stage 1.)
__global__ void __launch_bounds__(256) dbias_tc_reduce_kernel(const float* __restrict__ ws, int grid,
                                                              int heads, int L,
                                                              float* __restrict__ dbias) {
  __shared__ float part[8][33];
  const int n = heads * L * L;
  const int e = blockIdx.x * 32 + threadIdx.x;
  const int g = threadIdx.y;
  float acc = 0.f;
  if (e < n) {
    const int h = e / (L * L);
    const int r = e - h * L * L;
    const int i = r / L, j = r - (r / L) * L;
    const float* base = ws + (size_t)i * 64 + j;
#pragma unroll 4
    for (int t = h + g * heads; t < 2 * grid; t += 8 * heads) acc += base[(size_t)t * 64 * 64];
  }
  part[g][threadIdx.x] = acc;
  __syncthreads();
  if (g == 0 && e < n) {
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) sum += part[k][threadIdx.x];
    dbias[e] = sum;
  }
}

int bwd_period_tiles(const Geom& g, bool period_bias, bool has_mask) {
  if (!period_bias && !has_mask) return 1;
  const int64_t pu = (int64_t)g.heads * (has_mask ? g.mask_windows : 1);
  const int64_t pt = (pu % 2 == 0) ? pu / 2 : pu;
  return pt > (1 << 30) ? (1 << 30) : (int)pt;
}

template <int D>
int bwd_grid(const Geom& g, bool period_bias, bool has_mask) {
  const int n_tiles = (int)((g.units + 1) / 2);
  int grid = std::max(1, std::min(n_tiles, device_sm_count() * BCfg<D>::kCtasPerSm));
  if ((period_bias || has_mask) && n_tiles > grid) {
    const int pt = bwd_period_tiles(g, period_bias, has_mask);
    grid = (grid / pt) * pt;
  }
  return grid;
}

template <typename T, int D, int LK, bool ADD, bool DBIAS>
int launch_bwd_t(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                 const void* dout, const float* bias, const float* mask, void* dq, void* dk,
                 void* dv, float* dbias, float* ws, int layout, cudaStream_t s) {
  CUtensorMap m[7];
  int rc;
  if (layout == kUnits) {
    const void* ptrs[7] = {q, k, v, dout, dq, dk, dv};
    for (int i = 0; i < 7; ++i)
      if ((rc = get_units_map(&m[i], ptrs[i], dtype, g.units, g.L, g.d, kUnitRows, 2))) return rc;
  } else {  // q = qkv [N][L][3][h][d], dout = [N][L][h][d], dq = dqkv [N][L][3][h][d]
    const int64_t N = g.units / g.heads;
    const size_t hdb = (size_t)g.heads * g.d * 2;
    const uint8_t* qkv = static_cast<const uint8_t*>(q);
    uint8_t* dqkv = static_cast<uint8_t*>(dq);
    const void* src[7] = {qkv, qkv + hdb, qkv + 2 * hdb, dout, dqkv, dqkv + hdb, dqkv + 2 * hdb};
    for (int i = 0; i < 7; ++i)
      if ((rc = get_tokens_map(&m[i], src[i], dtype, N, g.L, i == 3 ? 1 : 3, g.heads, g.d,
                               kUnitRows)))
        return rc;
  }
  auto kern = bwd_tc_kernel<T, D, LK, ADD, DBIAS>;
  constexpr int smem = BCfg<D>::kSmem;
  if ((rc = ensure_smem_attr((const void*)kern, (int)(smem), "cudaFuncSetAttribute(bwd_tc)"))) return rc;
  const int n_tiles = (int)((g.units + 1) / 2);
  const int grid = bwd_grid<D>(g, ADD || DBIAS, mask != nullptr);
  BwdAddArgs add{bias, mask, ws, g.heads, mask ? g.mask_windows : 1};
  LayoutArgs lay{layout, g.heads};
  rc = check_cuda(launch_pdl(kern, dim3(grid), dim3(kThreads), smem, s, m[0], m[1], m[2], m[3],
                             m[4], m[5], m[6], n_tiles, (int)g.L, g.scale, add, lay,
                             device_flags_ptr()),
                  "bwd_tc_kernel launch");
  if (rc) return rc;
  count_launch();
  if (DBIAS) {
    const int n = g.heads * g.L * g.L;
    dbias_tc_reduce_kernel<<<(n + 31) / 32, dim3(32, 8), 0, s>>>(
        ws, grid, g.heads, g.L, dbias);
    count_launch();
    rc = check_cuda(cudaGetLastError(), "dbias_tc_reduce_kernel launch");
  }
  return rc;
}

template <typename T, int D, int LK>
int bwd_dispatch_flags(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                       const void* dout, const float* b, const float* m, void* dq, void* dk,
                       void* dv, float* db, float* ws, int lay, cudaStream_t s) {
  const bool add = b || m;
  if (db) {
    return add ? launch_bwd_t<T, D, LK, true, true>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s)
               : launch_bwd_t<T, D, LK, false, true>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s);
  }
  return add ? launch_bwd_t<T, D, LK, true, false>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s)
             : launch_bwd_t<T, D, LK, false, false>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s);
}

template <typename T, int D>
int bwd_dispatch_l(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                   const void* dout, const float* b, const float* m, void* dq, void* dk, void* dv,
                   float* db, float* ws, int lay, cudaStream_t s) {
  if (g.L == 49) return bwd_dispatch_flags<T, D, 49>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s);
  if (g.L == 64) return bwd_dispatch_flags<T, D, 64>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s);
  return bwd_dispatch_flags<T, D, 0>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s);
}

template <typename T>
int bwd_dispatch_d(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                   const void* dout, const float* b, const float* m, void* dq, void* dk, void* dv,
                   float* db, float* ws, int lay, cudaStream_t s) {
  switch (g.d) {
    case 16: return bwd_dispatch_l<T, 16>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s);
    case 32: return bwd_dispatch_l<T, 32>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s);
    case 64: return bwd_dispatch_l<T, 64>(g, dtype, q, k, v, dout, b, m, dq, dk, dv, db, ws, lay, s);
  }
  return fail(FWA_ERR_CAPACITY, "tcgen05 backward: unsupported head_dim");
}

}  // namespace

bool tc_bwd_supported(const Geom& g, int dtype, bool has_bias, bool has_mask, bool want_dbias) {
  if (dtype != FWA_F16 && dtype != FWA_BF16) return false;
  if (g.L < 1 || g.L > kUnitRows) return false;
  if (g.d != 16 && g.d != 32 && g.d != 64) return false;
  if (g.units > ((int64_t)1 << 31)) return false;
  if (has_bias || has_mask || want_dbias) {
    const int64_t n_tiles = (g.units + 1) / 2;
    const int cap = device_sm_count() * (g.d <= 32 ? 2 : 1);
    if (n_tiles > cap && bwd_period_tiles(g, has_bias || want_dbias, has_mask) > cap) return false;
  }
  return true;
}

size_t tc_bwd_smem(const Geom& g) {
  return g.d == 16 ? BCfg<16>::kSmem : g.d == 32 ? BCfg<32>::kSmem : BCfg<64>::kSmem;
}

int tc_bwd_tmem_cols(const Geom& g) {
  return g.d == 16 ? BCfg<16>::kTmemCols : g.d == 32 ? BCfg<32>::kTmemCols : BCfg<64>::kTmemCols;
}

size_t tc_bwd_workspace_bytes(const Geom& g, bool has_mask, bool want_dbias) {
  if (!want_dbias) return 0;
  int grid = 1;
  switch (g.d) {
    case 16: grid = bwd_grid<16>(g, true, has_mask); break;
    case 32: grid = bwd_grid<32>(g, true, has_mask); break;
    default: grid = bwd_grid<64>(g, true, has_mask); break;
  }
  return (size_t)grid * kTileRows * 64 * sizeof(float);
}

int launch_bwd_tc(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                  const void* dout, const float* bias, const float* mask, void* dq, void* dk,
                  void* dv, float* dbias, float* ws, cudaStream_t s, int layout) {
  return dtype == FWA_BF16
             ? bwd_dispatch_d<__nv_bfloat16>(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, layout, s)
             : bwd_dispatch_d<__half>(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, layout, s);
}

}  // namespace fwa
