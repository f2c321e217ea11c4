// fwa_tc_bwd_large.cu — backward for large windows (64 < L <= 256, L_pad*d <= 8192) on
// tcgen05 + TMA (sm_100a), f16/bf16, no bias/mask (those shapes take the generic kernel).
//
// One CTA (1 per SM, 512 TMEM columns) owns a whole unit at a time; its Q, K, V, dO
// are TMA-loaded once (box (d, L_pad, 1), rows >= L zero) into a 2-stage ring.
// For each 128-row query block qb:
//   S  = Q_qb K^T          -> TMEM [0, L_pad)             (SS, N = L_pad)
//   softmax warps: pass 1 row max, pass 2 p = exp2(.) in place + row sum,
//                  pass 3 P = p / l -> smem P [128 rows][L_pad keys] (SW128 K-major atoms)
//   dP = dO_qb V^T         -> TMEM [0, L_pad) (S consumed)
//   dV_kh += P^T dO_qb     (A = P read MN-major per 128-key half kh)  -> TMEM [256 + kh*d)
//   softmax warps: rho = sum_j P dP (pass 4), dS = scale P (dP - rho) -> smem (pass 5)
//   dK_kh += dS^T Q_qb     -> TMEM [256 + 2d + kh*d)
//   dQ_qb  = dS K          -> TMEM [0, d); epilogue stores it (TMA, rows >= L clipped)
// After the last qb the dK/dV halves are stored through the (now dead) Q/dO slots.
// HBM: Q, K, V, dO read once, dQ, dK, dV written once (7*L*d per unit).
#include <cuda.h>
#include <math.h>

#include <algorithm>

#include "fwa_common.cuh"
#include "fwa_sm100.cuh"

namespace fwa {
namespace {

using namespace sm100;

constexpr int kThreads = 192;
constexpr int kMRows = 128;

template <int D, int LP>
struct BLCfg {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kSlot = (LP * kRowBytes + 1023) / 1024 * 1024;  // one of Q/K/V/dO
  static constexpr int kStageBytes = 4 * kSlot;
  static constexpr int kNQ = (LP + kMRows - 1) / kMRows;              // query blocks = key halves
  static constexpr int kAtoms = (LP + 63) / 64;                         // 64-key SW128 atom columns
  static constexpr int kPBytes = 4 * 16384;                             // room for 4 atom cols (MN reads)
  static constexpr int kStageOut = kMRows * kRowBytes;                  // dQ staging
  static constexpr int kBase = kPBytes * 2 + kStageOut + 256 + 1024;
  static constexpr int kStages = (kBase + 2 * kStageBytes <= 227 * 1024) ? 2 : 1;
  static constexpr int kSmem = kBase + kStages * kStageBytes;
  static constexpr uint32_t kSwz = D == 16 ? 6u : (D == 32 ? 4u : 2u);
  static constexpr int kChunks = kRowBytes / 16;
  static constexpr uint32_t kTdV = 256, kTdK = 256 + 2 * D;             // + kh*D
  static constexpr int kOutRows = LP < kMRows ? LP : kMRows;            // dK/dV store box rows
  static_assert(256 + 4 * D <= 512, "TMEM budget");
  static_assert(kSmem <= 227 * 1024, "smem budget");
};

struct BLBarriers {
  uint64_t in_full[2], in_empty[2];
  uint64_t s_full, p_ready, dp_full, ds_ready, dq_full, s_free, grads_full, grads_free;
  uint32_t tmem_base;
};

template <typename T>
__device__ __forceinline__ uint32_t pk2(float a, float b) {
  if constexpr (DT<T>::id == FWA_BF16) {
    __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  } else {
    __half2 h2 = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  }
}
template <typename T>
__device__ __forceinline__ float2 up2(uint32_t w) {
  if constexpr (DT<T>::id == FWA_BF16) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
  } else {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
}

// byte offset of (row r, 8-key chunk c of atom column a) in a [128][LP] SW128 K-major tile
__device__ __forceinline__ int ptile_off(int a, int r, int c) {
  return a * 16384 + (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
}

template <typename T, int D, int LP>
__global__ void __launch_bounds__(kThreads, 1)
bwd_tc_large_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dk,
                    const __grid_constant__ CUtensorMap tm_dv, int n_units, int L, float scale) {
  using C = BLCfg<D, LP>;
  constexpr bool kBF16 = DT<T>::id == FWA_BF16;
  constexpr int NQ = C::kNQ;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sP = smem;
  uint8_t* sDS = sP + C::kPBytes;
  uint8_t* sIn = sDS + C::kPBytes;                          // [stage][Q|K|V|dO]
  uint8_t* sOut = sIn + C::kStages * C::kStageBytes;        // dQ staging
  BLBarriers* bars = reinterpret_cast<BLBarriers*>(sOut + C::kStageOut);
  auto slot = [&](int st, int w) { return sIn + st * C::kStageBytes + w * C::kSlot; };
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // P / dS rows of inactive (all >= L) warps and keys >= L must read as zero, and so
  // must the slot padding rows [L_pad, slot) that TMA never writes (the S MMA of the
  // last query block reads Q/dO rows up to 128*NQ).
  for (int i = threadIdx.x; i < 2 * C::kPBytes / 16; i += kThreads)
    reinterpret_cast<uint4*>(sP)[i] = make_uint4(0, 0, 0, 0);
  constexpr int kPad = C::kSlot - LP * C::kRowBytes;
  if constexpr (kPad > 0) {
    for (int i = threadIdx.x; i < C::kStages * 4 * (kPad / 16); i += kThreads) {
      const int sl = i / (kPad / 16), o = i % (kPad / 16);
      reinterpret_cast<uint4*>(sIn + sl * C::kSlot + LP * C::kRowBytes)[o] = make_uint4(0, 0, 0, 0);
    }
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars->in_full[s], 1);
      mbar_init(&bars->in_empty[s], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->p_ready, 128);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->ds_ready, 128);
    mbar_init(&bars->dq_full, 1);
    mbar_init(&bars->s_free, 128);
    mbar_init(&bars->grads_full, 1);
    mbar_init(&bars->grads_free, 128);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 1) tmem_alloc(&bars->tmem_base, 512);
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
      for (int i = 0; i < n_local; ++i) {
        const int unit = blockIdx.x + i * gridDim.x;
        const int st = i % C::kStages;
        mbar_wait(&bars->in_empty[st], ((i / C::kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->in_full[st], 4 * LP * C::kRowBytes);
        tma_load_3d(slot(st, 0), &tm_q, &bars->in_full[st], 0, 0, unit, pol);
        tma_load_3d(slot(st, 1), &tm_k, &bars->in_full[st], 0, 0, unit, pol);
        tma_load_3d(slot(st, 2), &tm_v, &bars->in_full[st], 0, 0, unit, pol);
        tma_load_3d(slot(st, 3), &tm_do, &bars->in_full[st], 0, 0, unit, pol);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_f16(kBF16, 128, LP, false, false);
      constexpr uint32_t idMN = make_idesc_f16(kBF16, 128, D, true, true);
      constexpr uint32_t idQ = make_idesc_f16(kBF16, 128, D, false, true);
      constexpr uint32_t sbo = 8 * C::kRowBytes;
      const uint32_t p0 = smem_u32(sP), ds0 = smem_u32(sDS);
      int it = 0;
      for (int i = 0; i < n_local; ++i) {
        const int st = i % C::kStages;
        const uint32_t q0 = smem_u32(slot(st, 0)), k0 = smem_u32(slot(st, 1));
        const uint32_t v0 = smem_u32(slot(st, 2)), do0 = smem_u32(slot(st, 3));
        mbar_wait(&bars->in_full[st], (i / C::kStages) & 1);
        for (int qb = 0; qb < NQ; ++qb, ++it) {
          const int kq = min(8, (L - qb * kMRows + 15) / 16);  // query k-steps with valid rows
          if (it > 0) mbar_wait(&bars->s_free, (it - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)   // S = Q_qb K^T
            mma_f16_ss(tmem, make_sdesc(q0 + qb * kMRows * C::kRowBytes + kk * 32, 16, sbo, C::kSwz),
                       make_sdesc(k0 + kk * 32, 16, sbo, C::kSwz), idS, kk > 0);
          mma_commit(&bars->s_full);
          mbar_wait(&bars->p_ready, it & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)   // dP = dO_qb V^T (S columns consumed)
            mma_f16_ss(tmem, make_sdesc(do0 + qb * kMRows * C::kRowBytes + kk * 32, 16, sbo, C::kSwz),
                       make_sdesc(v0 + kk * 32, 16, sbo, C::kSwz), idS, kk > 0);
          mma_commit(&bars->dp_full);
          if (qb == 0 && i > 0) {
            mbar_wait(&bars->grads_free, (i - 1) & 1);  // dK/dV of the previous unit pulled
            tc_fence_after();
          }
          for (int kh = 0; kh < NQ; ++kh)       // dV_kh += P^T dO_qb
            for (int kk = 0; kk < kq; ++kk)
              mma_f16_ss(tmem + C::kTdV + kh * D,
                         make_sdesc(p0 + kh * 2 * 16384 + kk * 2048, 16384, 1024, 2),
                         make_sdesc(do0 + (qb * kMRows + kk * 16) * C::kRowBytes, C::kSlot, sbo, C::kSwz),
                         idMN, (qb | kk) > 0);
          mbar_wait(&bars->ds_ready, it & 1);
          tc_fence_after();
          for (int kh = 0; kh < NQ; ++kh)       // dK_kh += dS^T Q_qb
            for (int kk = 0; kk < kq; ++kk)
              mma_f16_ss(tmem + C::kTdK + kh * D,
                         make_sdesc(ds0 + kh * 2 * 16384 + kk * 2048, 16384, 1024, 2),
                         make_sdesc(q0 + (qb * kMRows + kk * 16) * C::kRowBytes, C::kSlot, sbo, C::kSwz),
                         idMN, (qb | kk) > 0);
#pragma unroll 4
          for (int kk = 0; kk < LP / 16; ++kk)  // dQ_qb = dS K  -> TMEM [0, d)
            mma_f16_ss(tmem, make_sdesc(ds0 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2),
                       make_sdesc(k0 + kk * 16 * C::kRowBytes, C::kSlot, sbo, C::kSwz), idQ, kk > 0);
          mma_commit(&bars->dq_full);
        }
        mma_commit(&bars->grads_full);
      }
    }
  } else {
    // ============ softmax / dS / epilogues (warps 2..5; thread = row = TMEM lane) ============
    const int qd = warp & 3;
    const int r = qd * 32 + lane;          // row within the 128-row block
    const uint32_t t_lane = (uint32_t)(qd * 32) << 16;
    const uint32_t oswz = (uint32_t)((r * C::kRowBytes) >> 7) & (C::kChunks - 1);
    const bool leader = (threadIdx.x == 64);
    const float sl2 = scale * 1.4426950408889634f;
    int it = 0;
    for (int i = 0; i < n_local; ++i) {
      const int unit = blockIdx.x + i * gridDim.x;
      const int st = i % C::kStages;
      for (int qb = 0; qb < NQ; ++qb, ++it) {
        const bool active = qb * kMRows + qd * 32 < L;   // warp-uniform
        mbar_wait(&bars->s_full, it & 1);
        tc_fence_after();
        if (active) {
          float mx = -INFINITY;
#pragma unroll
          for (int c0 = 0; c0 < LP; c0 += 64) {       // pass 1: row max
            uint32_t v[64];
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (c0 + g * 16 < LP) tmem_ld16(tmem + t_lane + c0 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&v[g * 16]));
            tmem_wait_ld();
#pragma unroll
            for (int t = 0; t < 64; ++t)
              if (c0 + t < L) mx = fmaxf(mx, __uint_as_float(v[t]));
          }
          const float mxs = mx * sl2;
          float sum = 0.f;
#pragma unroll
          for (int c0 = 0; c0 < LP; c0 += 64) {       // pass 2: p in place, row sum
            uint32_t v[64];
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (c0 + g * 16 < LP) tmem_ld16(tmem + t_lane + c0 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&v[g * 16]));
            tmem_wait_ld();
#pragma unroll
            for (int t = 0; t < 64; ++t) {
              const float p = c0 + t < L ? ex2(fmaf(__uint_as_float(v[t]), sl2, -mxs)) : 0.f;
              sum += p;
              v[t] = __float_as_uint(p);
            }
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (c0 + g * 16 < LP) tmem_st16(tmem + t_lane + c0 + g * 16, &v[g * 16]);
          }
          tmem_wait_st();
          const float inv = __frcp_rn(sum);
#pragma unroll
          for (int c0 = 0; c0 < LP; c0 += 64) {       // pass 3: P = p / l -> smem
            uint32_t v[64];
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (c0 + g * 16 < LP) tmem_ld16(tmem + t_lane + c0 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&v[g * 16]));
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 8; ++c)
              if (c0 + 8 * c < LP)
                *reinterpret_cast<uint4*>(sP + ptile_off(c0 >> 6, r, c)) = make_uint4(
                    pk2<T>(__uint_as_float(v[8 * c]) * inv, __uint_as_float(v[8 * c + 1]) * inv),
                    pk2<T>(__uint_as_float(v[8 * c + 2]) * inv, __uint_as_float(v[8 * c + 3]) * inv),
                    pk2<T>(__uint_as_float(v[8 * c + 4]) * inv, __uint_as_float(v[8 * c + 5]) * inv),
                    pk2<T>(__uint_as_float(v[8 * c + 6]) * inv, __uint_as_float(v[8 * c + 7]) * inv));
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bars->p_ready);
        mbar_wait(&bars->dp_full, it & 1);
        tc_fence_after();
        if (active) {
          float rho = 0.f;
#pragma unroll
          for (int c0 = 0; c0 < LP; c0 += 64) {       // pass 4: rho = sum P dP
            uint32_t v[64];
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (c0 + g * 16 < LP) tmem_ld16(tmem + t_lane + c0 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&v[g * 16]));
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              if (c0 + 8 * c >= LP) break;
              const uint4 pw = *reinterpret_cast<const uint4*>(sP + ptile_off(c0 >> 6, r, c));
              const uint32_t pa[4] = {pw.x, pw.y, pw.z, pw.w};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float2 p = up2<T>(pa[t]);
                rho = fmaf(p.x, __uint_as_float(v[8 * c + 2 * t]), rho);
                rho = fmaf(p.y, __uint_as_float(v[8 * c + 2 * t + 1]), rho);
              }
            }
          }
          const float srho = scale * rho;
#pragma unroll
          for (int c0 = 0; c0 < LP; c0 += 64) {       // pass 5: dS = scale P (dP - rho) -> smem
            uint32_t v[64];
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (c0 + g * 16 < LP) tmem_ld16(tmem + t_lane + c0 + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&v[g * 16]));
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              if (c0 + 8 * c >= LP) break;
              const uint4 pw = *reinterpret_cast<const uint4*>(sP + ptile_off(c0 >> 6, r, c));
              const uint32_t pa[4] = {pw.x, pw.y, pw.z, pw.w};
              uint32_t w[4];
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float2 p = up2<T>(pa[t]);
                const int j = c0 + 8 * c + 2 * t;
                const float a = j < L ? p.x * fmaf(__uint_as_float(v[8 * c + 2 * t]), scale, -srho) : 0.f;
                const float b = j + 1 < L ? p.y * fmaf(__uint_as_float(v[8 * c + 2 * t + 1]), scale, -srho) : 0.f;
                w[t] = pk2<T>(a, b);
              }
              *reinterpret_cast<uint4*>(sDS + ptile_off(c0 >> 6, r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bars->ds_ready);
        // ---- dQ_qb epilogue ----
        mbar_wait(&bars->dq_full, it & 1);
        tc_fence_after();
        uint32_t g[D];
        if (active) {
#pragma unroll
          for (int q = 0; q < D / 16; ++q)
            tmem_ld16(tmem + t_lane + q * 16, *reinterpret_cast<uint32_t(*)[16]>(&g[q * 16]));
          tmem_wait_ld();
        }
        tc_fence_before();
        mbar_arrive(&bars->s_free);
        if (leader) bulk_wait_read<0>();
        named_sync(1, 128);
        if (active) {
          uint8_t* orow = sOut + r * C::kRowBytes;
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            *reinterpret_cast<uint4*>(orow + ((c ^ oswz) << 4)) = make_uint4(
                pk2<T>(__uint_as_float(g[8 * c]), __uint_as_float(g[8 * c + 1])),
                pk2<T>(__uint_as_float(g[8 * c + 2]), __uint_as_float(g[8 * c + 3])),
                pk2<T>(__uint_as_float(g[8 * c + 4]), __uint_as_float(g[8 * c + 5])),
                pk2<T>(__uint_as_float(g[8 * c + 6]), __uint_as_float(g[8 * c + 7])));
        }
        fence_proxy_async_smem();
        named_sync(2, 128);
        if (leader) {
          tma_store_3d(&tm_dq, sOut, 0, qb * kMRows, unit);
          bulk_commit();
        }
      }
      // ---- dK / dV of the unit (rows = keys), staged in the dead Q (dK) / dO (dV) slots ----
      mbar_wait(&bars->grads_full, i & 1);
      tc_fence_after();
      for (int kh = 0; kh < NQ; ++kh) {
        const bool act = kh * kMRows + qd * 32 < L;
        uint32_t gk[D], gv[D];
        if (act) {
#pragma unroll
          for (int q = 0; q < D / 16; ++q) {
            tmem_ld16(tmem + t_lane + C::kTdK + kh * D + q * 16, *reinterpret_cast<uint32_t(*)[16]>(&gk[q * 16]));
            tmem_ld16(tmem + t_lane + C::kTdV + kh * D + q * 16, *reinterpret_cast<uint32_t(*)[16]>(&gv[q * 16]));
          }
          tmem_wait_ld();
        }
        if (kh == NQ - 1) {
          tc_fence_before();
          mbar_arrive(&bars->grads_free);
        }
        if (leader) bulk_wait_read<0>();
        named_sync(1, 128);
        if (act && r < C::kOutRows) {
          uint8_t* rk = slot(st, 0) + r * C::kRowBytes;
          uint8_t* rv = slot(st, 3) + r * C::kRowBytes;
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c) {
            *reinterpret_cast<uint4*>(rk + ((c ^ oswz) << 4)) = make_uint4(
                pk2<T>(__uint_as_float(gk[8 * c]), __uint_as_float(gk[8 * c + 1])),
                pk2<T>(__uint_as_float(gk[8 * c + 2]), __uint_as_float(gk[8 * c + 3])),
                pk2<T>(__uint_as_float(gk[8 * c + 4]), __uint_as_float(gk[8 * c + 5])),
                pk2<T>(__uint_as_float(gk[8 * c + 6]), __uint_as_float(gk[8 * c + 7])));
            *reinterpret_cast<uint4*>(rv + ((c ^ oswz) << 4)) = make_uint4(
                pk2<T>(__uint_as_float(gv[8 * c]), __uint_as_float(gv[8 * c + 1])),
                pk2<T>(__uint_as_float(gv[8 * c + 2]), __uint_as_float(gv[8 * c + 3])),
                pk2<T>(__uint_as_float(gv[8 * c + 4]), __uint_as_float(gv[8 * c + 5])),
                pk2<T>(__uint_as_float(gv[8 * c + 6]), __uint_as_float(gv[8 * c + 7])));
          }
        }
        fence_proxy_async_smem();
        named_sync(2, 128);
        if (leader) {
          tma_store_3d(&tm_dk, slot(st, 0), 0, kh * kMRows, unit);
          tma_store_3d(&tm_dv, slot(st, 3), 0, kh * kMRows, unit);
          bulk_commit();
        }
      }
      if (leader) {
        bulk_wait_read<0>();
        mbar_arrive(&bars->in_empty[st]);   // the unit's slots may be refilled
      }
    }
    if (leader) bulk_wait_read<0>();  // smem reads done; the grid's completion flushes the writes
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template <typename T, int D, int LP>
int launch_bwd_large_t(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                       const void* dout, void* dq, void* dk, void* dv, cudaStream_t s) {
  using C = BLCfg<D, LP>;
  CUtensorMap m[7];
  const void* in[4] = {q, k, v, dout};
  int rc;
  for (int i = 0; i < 4; ++i)
    if ((rc = get_units_map(&m[i], in[i], dtype, g.units, g.L, g.d, LP, 1))) return rc;
  if ((rc = get_units_map(&m[4], dq, dtype, g.units, g.L, g.d, kMRows, 1))) return rc;
  if ((rc = get_units_map(&m[5], dk, dtype, g.units, g.L, g.d, C::kOutRows, 1))) return rc;
  if ((rc = get_units_map(&m[6], dv, dtype, g.units, g.L, g.d, C::kOutRows, 1))) return rc;
  auto kern = bwd_tc_large_kernel<T, D, LP>;
  if ((rc = ensure_smem_attr((const void*)kern, (int)(C::kSmem), "cudaFuncSetAttribute(bwd_tc_large)"))) return rc;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(g.units, device_sm_count()));
  rc = check_cuda(launch_pdl(kern, dim3(grid), dim3(kThreads), (size_t)C::kSmem, s, m[0], m[1],
                             m[2], m[3], m[4], m[5], m[6], (int)g.units, (int)g.L, g.scale),
                  "bwd_tc_large_kernel launch");
  if (rc) return rc;
  count_launch();
  return FWA_OK;
}

template <typename T, int D>
int bwd_large_l(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                const void* dout, void* dq, void* dk, void* dv, cudaStream_t s) {
  const int lp = (g.L + 15) / 16 * 16;
  if constexpr (D == 64) {
    switch (lp) {
      case 80: return launch_bwd_large_t<T, D, 80>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 96: return launch_bwd_large_t<T, D, 96>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 112: return launch_bwd_large_t<T, D, 112>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 128: return launch_bwd_large_t<T, D, 128>(g, dtype, q, k, v, dout, dq, dk, dv, s);
    }
  } else {
    switch (lp) {
      case 80: return launch_bwd_large_t<T, D, 80>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 96: return launch_bwd_large_t<T, D, 96>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 112: return launch_bwd_large_t<T, D, 112>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 128: return launch_bwd_large_t<T, D, 128>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 144: return launch_bwd_large_t<T, D, 144>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 160: return launch_bwd_large_t<T, D, 160>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 176: return launch_bwd_large_t<T, D, 176>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 192: return launch_bwd_large_t<T, D, 192>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 208: return launch_bwd_large_t<T, D, 208>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 224: return launch_bwd_large_t<T, D, 224>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 240: return launch_bwd_large_t<T, D, 240>(g, dtype, q, k, v, dout, dq, dk, dv, s);
      case 256: return launch_bwd_large_t<T, D, 256>(g, dtype, q, k, v, dout, dq, dk, dv, s);
    }
  }
  return fail(FWA_ERR_CAPACITY, "tcgen05 large-window backward: unsupported L");
}

}  // namespace

bool tc_bwd_large_supported(const Geom& g, int dtype, bool has_bias, bool has_mask, bool want_dbias) {
  if (tc_bwd_flat_supported(g, dtype, has_bias, has_mask, want_dbias)) return true;
  if (has_bias || has_mask || want_dbias) return false;
  if (dtype != FWA_F16 && dtype != FWA_BF16) return false;
  if (g.L <= 64 || g.L > 256) return false;
  const int lp = (g.L + 15) / 16 * 16;
  if (g.d != 16 && g.d != 32 && g.d != 64) return false;
  if (lp * g.d > 8192) return false;
  return g.units <= ((int64_t)1 << 31);
}

size_t tc_bwd_large_smem(const Geom& g) {
  if (tc_bwd_flat_supported(g, FWA_F16, false, false, false)) return tc_bwd_flat_smem(g);
  const int lp = (g.L + 15) / 16 * 16;
  const int row = g.d * 2;
  const int slot = (lp * row + 1023) / 1024 * 1024;
  const int base = 2 * 4 * 16384 + 128 * row + 256 + 1024;
  const int stages = (base + 2 * 4 * slot <= 227 * 1024) ? 2 : 1;
  return (size_t)base + stages * 4 * slot;
}

int launch_bwd_tc_large(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                        const void* dout, const float* bias, const float* mask, void* dq, void* dk,
                        void* dv, float* dbias, float* ws, cudaStream_t s) {
  if (tc_bwd_flat_supported(g, dtype, bias != nullptr, mask != nullptr, dbias != nullptr))
    return launch_bwd_tc_flat(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s);
  if (bias || mask || dbias)
    return fail(FWA_ERR_CAPACITY, "tcgen05 large-window backward: bias/mask not supported here");
  const bool bf = dtype == FWA_BF16;
  switch (g.d) {
    case 16: return bf ? bwd_large_l<__nv_bfloat16, 16>(g, dtype, q, k, v, dout, dq, dk, dv, s)
                       : bwd_large_l<__half, 16>(g, dtype, q, k, v, dout, dq, dk, dv, s);
    case 32: return bf ? bwd_large_l<__nv_bfloat16, 32>(g, dtype, q, k, v, dout, dq, dk, dv, s)
                       : bwd_large_l<__half, 32>(g, dtype, q, k, v, dout, dq, dk, dv, s);
    case 64: return bf ? bwd_large_l<__nv_bfloat16, 64>(g, dtype, q, k, v, dout, dq, dk, dv, s)
                       : bwd_large_l<__half, 64>(g, dtype, q, k, v, dout, dq, dk, dv, s);
  }
  return fail(FWA_ERR_CAPACITY, "tcgen05 large-window backward: unsupported head_dim");
}

}  // namespace fwa
