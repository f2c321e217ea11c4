// fwa_tc_fwd.cu — Flash Window Attention forward on tcgen05 + TMA (sm_100a).
//
// Algorithm 1 of the paper (reference flash.py:141-184) for
// f16/bf16, L <= 64, d in {16, 32, 64}, optionally with the Swin relative-position
// bias and shifted-window mask (ADD; fp32 rows kept in TMEM, see below), in the
// [N][h][L][d] layout or straight from the packed qkv-Linear output (kTokens):
//
//   * A tile = 128 rows = two (window, head) units, each padded to 64 rows.
//     TMA loads Q, K, V with a 3-D tensor map (d, L, units) and box (d, 64, 2):
//     rows L..63 are out of bounds and arrive as zeros, so L = 49 needs no
//     host padding, and the swizzled smem image is exactly the UMMA
//     K-major (Q, K) / MN-major (V) canonical layout.
//   * S = Q K^T: two tcgen05.mma chains (M=128, N=64, K=d), one per unit, with
//     complementary disable-output-lane masks, so both units' scores share TMEM
//     columns [0,64) (unit 0 in lanes 0-63, unit 1 in lanes 64-127).
//   * Softmax: 4 warps, one thread per row (TMEM lane = row): tcgen05.ld of the
//     row's own 64-column block, masked max over the L valid keys, ex2, row
//     sum; P (unnormalised, f16/bf16 pairs) is written back to TMEM with
//     tcgen05.st (columns [64,96)), so P never touches shared memory.
//   * O = P V: per unit a lane-masked tcgen05.mma with A from TMEM (M=128, N=d,
//     K=64) into TMEM (double-buffered O at [96, 96+2d)).
//   * Shared memory holds only the TMA ring (4 stages for d=32, 8 for d=16)
//     and one staging tile for the TMA store.
//   * Epilogue: tcgen05.ld, scale by 1/rowsum, convert, swizzled staging,
//     TMA store with the same 3-D map (rows >= L are clipped by the map).
//
// Warp roles (192 threads, 2 CTAs per SM, persistent over tiles):
//   warp 0: TMA producer, warp 1: TMEM allocator + MMA issuer,
//   warps 2-5: softmax + epilogue (warp w owns TMEM lanes 32*(w%4)..+31).
// The softmax warps are software-pipelined: iteration i runs softmax(i) and
// then the epilogue of tile i-1, whose P.V ran on the tensor core meanwhile;
// P (smem) and O (TMEM) are double-buffered for that. L = 49 and 64 are
// compile-time specialisations (no masking arithmetic); other L <= 64 run
// the runtime-L instance.
// HBM is touched once per tensor: Q, K, V read once, O written once.
#include <cuda.h>
#include <math.h>

#include <algorithm>
#include <mutex>

#include "fwa_common.cuh"
#include "fwa_sm100.cuh"

namespace fwa {
namespace {

using namespace sm100;

constexpr int kThreads = 192;
constexpr int kTileRows = 128;     // MMA M
constexpr int kUnitRows = 64;      // rows per packed unit

template <int D, bool ADD = false>
struct Cfg {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTileBytes = kTileRows * kRowBytes;            // one of Q/K/V per stage
  static constexpr int kStages = D <= 16 ? 8 : 4;
  // staging for the O tile; with bias/mask it also stages one unit's f16 add table
  // (64 x 64) once in the prologue, so it is at least 8 KB
  static constexpr int kStageO = (ADD && kTileRows * D * 2 < 8192) ? 8192 : kTileRows * D * 2;
  static constexpr int kCtasPerSm = D <= 32 ? 2 : 1;
  static constexpr uint32_t kSwz = D == 16 ? 6u : (D == 32 ? 4u : 2u);  // UMMA layout code
  static constexpr int kSmem = 1024 /*align slack*/ + kStages * 3 * kTileBytes + kStageO +
                               256 /*barriers*/;
  static constexpr int kChunks = kRowBytes / 16;  // 16-byte chunks per row
  // TMEM columns (lane = tile row; unit 0 rows are lanes 0-63, unit 1 rows 64-127):
  //   S [0,64) fp32 | P [64,96) 16-bit pairs | O0, O1 (d each) fp32.
  // Each unit's S/P/O occupy the SAME columns in its own 64 lanes: the MMAs for
  // unit 0 and unit 1 run with complementary disable-output-lane masks.
  static constexpr uint32_t kTmemP = 64, kTmemO0 = 96, kTmemO1 = 96 + D;
  // (bias + mask) * log2e rows of the CTA's two unit slots, fp32, loaded once (ADD)
  static constexpr uint32_t kTmemAdd = 96 + 2 * D;
  static constexpr uint32_t kTmemCols = (kTmemAdd + (ADD ? 64 : 0) <= 256) ? 256 : 512;
};

struct SmemBarriers {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t s_full, s_empty, p_full;
  uint64_t pv_done[2];
  uint32_t tmem_base;
};

// Additive bias/mask: the grid is a multiple of the (window mod nW, head) period
// of the tile sequence, so every tile of a CTA sees the same two (w, h) pairs and
// each thread keeps its row of (bias + mask) * log2(e) in registers (f16 pairs).
struct AddArgs {
  const float* bias;  // [heads][L][L] or null
  const float* mask;  // [nW][L][L] or null
  int heads;
  int mask_windows;
};

// LK > 0: compile-time window length (Swin 7x7 / 8x8); LK == 0: runtime L.
template <typename T, int D, int LK, bool ADD>
__global__ void __launch_bounds__(kThreads, Cfg<D, ADD>::kCtasPerSm)
fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
              const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
              int n_tiles, int L_rt, float scale_log2, AddArgs add, LayoutArgs lay) {
  using C = Cfg<D, ADD>;
  constexpr bool kBF16 = DT<T>::id == FWA_BF16;
  const int L = LK > 0 ? LK : L_rt;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::kStages * C::kTileBytes;
  uint8_t* sV = sK + C::kStages * C::kTileBytes;
  uint8_t* sO = sV + C::kStages * C::kTileBytes;   // 1 staging tile for the TMA store
  SmemBarriers* bars = reinterpret_cast<SmemBarriers*>(sO + C::kStageO);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->s_empty, 128);
    mbar_init(&bars->p_full, 128);
    mbar_init(&bars->pv_done[0], 1);
    mbar_init(&bars->pv_done[1], 1);
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
      n_tiles > (int)blockIdx.x ? (n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  // PDL: let the next kernel in the stream start its prologue; our own global
  // traffic starts only after the previous grid has fully completed.
  griddep_launch_dependents();
  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      griddep_wait();
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < n_local; ++i) {
        const int tile = blockIdx.x + i * gridDim.x;
        const int st = i % C::kStages;
        const uint32_t round = i / C::kStages;
        mbar_wait(&bars->empty[st], (round & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->full[st], 3 * C::kTileBytes);
        constexpr int kUB = kUnitRows * C::kRowBytes;
        load_tile<kUB>(sQ + st * C::kTileBytes, &tm_q, &bars->full[st], tile, lay.mode, lay.heads, pol);
        load_tile<kUB>(sK + st * C::kTileBytes, &tm_k, &bars->full[st], tile, lay.mode, lay.heads, pol);
        load_tile<kUB>(sV + st * C::kTileBytes, &tm_v, &bars->full[st], tile, lay.mode, lay.heads, pol);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0 && n_local > 0) {
      constexpr uint32_t idS = make_idesc_f16(kBF16, 128, 64, false, false);
      constexpr uint32_t idO = make_idesc_f16(kBF16, 128, D, false, true);
      constexpr uint32_t sbo_qk = 8 * C::kRowBytes;  // 8-row core-matrix group stride
      auto issue_S = [&](int i) {
        const int st = i % C::kStages;
        const uint32_t q0 = smem_u32(sQ + st * C::kTileBytes);
        const uint32_t k0 = smem_u32(sK + st * C::kTileBytes);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t lo = u ? ~0u : 0u, hi = u ? 0u : ~0u;  // unit u writes lanes 64u..64u+63
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t a = make_sdesc(q0 + kk * 32, 16, sbo_qk, C::kSwz);
            const uint64_t b = make_sdesc(k0 + u * 64 * C::kRowBytes + kk * 32, 16, sbo_qk, C::kSwz);
            mma_f16_ss_m(tmem, a, b, idS, kk > 0, lo, lo, hi, hi);
          }
        }
        mma_commit(&bars->s_full);
      };
      mbar_wait(&bars->full[0], 0);
      tc_fence_after();
      issue_S(0);
      for (int i = 0; i < n_local; ++i) {
        // S(i+1) as soon as softmax(i) has pulled S(i) into registers: it runs on the
        // tensor core while softmax(i) computes.
        if (i + 1 < n_local) {
          const int st1 = (i + 1) % C::kStages;
          mbar_wait(&bars->full[st1], ((i + 1) / C::kStages) & 1);
          mbar_wait(&bars->s_empty, i & 1);
          tc_fence_after();
          issue_S(i + 1);
        }
        const int st = i % C::kStages;
        const int ob = i & 1;
        // O(ob) = P V, P read from TMEM (TS form), once softmax has stored P(i)
        mbar_wait(&bars->p_full, i & 1);
        tc_fence_after();
        const uint32_t v0 = smem_u32(sV + st * C::kTileBytes);
        const uint32_t od = tmem + (ob ? C::kTmemO1 : C::kTmemO0);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t lo = u ? ~0u : 0u, hi = u ? 0u : ~0u;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t b = make_sdesc(v0 + (u * 64 + kk * 16) * C::kRowBytes, C::kTileBytes,
                                          8 * C::kRowBytes, C::kSwz);
            mma_f16_ts_m(od, tmem + C::kTmemP + kk * 8, b, idO, kk > 0, lo, lo, hi, hi);
          }
        }
        mma_commit(&bars->pv_done[ob]);
        mma_commit(&bars->empty[st]);
      }
    }
  } else {
    // ============ softmax(i) then epilogue(i-1) (warps 2..5, software-pipelined) ============
    const int q = warp & 3;               // TMEM lane quarter
    const int row = q * 32 + lane;        // tile row = TMEM lane
    const int ul = row >> 6;              // unit within the tile
    const uint32_t t_lane = (uint32_t)(q * 32) << 16;
    uint8_t* orow = sO + row * C::kRowBytes;
    const uint32_t oswz = (uint32_t)((row * C::kRowBytes) >> 7) & (C::kChunks - 1);
    const bool leader = (threadIdx.x == 64);
    if constexpr (ADD) {
      // Load the CTA's two (bias + mask) * log2e tiles into TMEM once: every tile of this
      // CTA has the same (w, h) pair per slot (period-aligned grid). Each unit's table is
      // read coalesced into the (not yet used) staging tile as f16, then each thread
      // moves its own row to its TMEM lane as fp32.
      const int ct = threadIdx.x - 64;             // 0..127 within the softmax warps
      const uint32_t rswz = (uint32_t)(row & 7);
#pragma unroll 1
      for (int u = 0; u < 2; ++u) {
        const int uu = 2 * (int)blockIdx.x + u;
        const int hd = uu % add.heads;
        const int w = (uu / add.heads) % add.mask_windows;
        const float* __restrict__ bt = add.bias ? add.bias + (size_t)hd * L * L : nullptr;
        const float* __restrict__ mt = add.mask ? add.mask + (size_t)w * L * L : nullptr;
        for (int e = ct; e < L * L; e += 128) {
          const float av = ((bt ? __ldg(bt + e) : 0.f) + (mt ? __ldg(mt + e) : 0.f)) * 1.4426950408889634f;
          const int r = e / L, j = e % L;
          *reinterpret_cast<__half*>(sO + r * 128 + ((((j >> 3) ^ (r & 7))) << 4) + (j & 7) * 2) =
              __float2half_rn(av);
        }
        named_sync(3, 128);
        if (ul == u) {
          const int r = row & 63;
          uint32_t fv[64];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 hv = *reinterpret_cast<const uint4*>(sO + r * 128 + ((c ^ rswz) << 4));
            const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int j = 8 * c + 2 * t;
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&hw[t]));
              fv[j] = __float_as_uint((r < L && j < L) ? f.x : 0.f);
              fv[j + 1] = __float_as_uint((r < L && j + 1 < L) ? f.y : 0.f);
            }
          }
#pragma unroll
          for (int g = 0; g < 4; ++g) tmem_st16(tmem + t_lane + C::kTmemAdd + g * 16, &fv[g * 16]);
          tmem_wait_st();
        }
        named_sync(3, 128);
      }
    }
    float inv_prev = 0.f;
    for (int i = 0; i <= n_local; ++i) {
      float inv_cur = 0.f;
      if (i < n_local) {
        mbar_wait(&bars->s_full, i & 1);
        tc_fence_after();
        uint32_t s[64];
        uint32_t ad[ADD ? 64 : 1];
#pragma unroll
        for (int g = 0; g < 4; ++g)
          if (LK == 0 || g * 16 < LK) {
            tmem_ld16(tmem + t_lane + g * 16, *reinterpret_cast<uint32_t(*)[16]>(&s[g * 16]));
            if constexpr (ADD)
              tmem_ld16(tmem + t_lane + C::kTmemAdd + g * 16,
                        *reinterpret_cast<uint32_t(*)[16]>(&ad[g * 16]));
          }
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bars->s_empty);
        float mx = -INFINITY;
        if constexpr (ADD) {
          // t = scale*log2e*S + (bias+mask)*log2e, kept in s[] (packed f32x2 FMA)
          const float2 sc2 = make_float2(scale_log2, scale_log2);
#pragma unroll
          for (int j = 0; j < 64; j += 2) {
            const float2 t2 = __ffma2_rn(make_float2(__uint_as_float(s[j]), __uint_as_float(s[j + 1])), sc2,
                                         make_float2(__uint_as_float(ad[j]), __uint_as_float(ad[j + 1])));
            s[j] = __float_as_uint(t2.x);
            s[j + 1] = __float_as_uint(t2.y);
            if (j + 1 < L) mx = fmaxf(mx, fmaxf(t2.x, t2.y));
            else if (j < L) mx = fmaxf(mx, t2.x);
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
        const float2 sl22 = make_float2(sl2, sl2), nm2 = make_float2(-mxs, -mxs);
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
          // packed f32x2 math; a quarter of the exponentials on the FMA pipe (poly)
          const float2 a = __ffma2_rn(make_float2(__uint_as_float(s[j]), __uint_as_float(s[j + 1])), sl22, nm2);
          float2 pp = (j & 7) == 6 ? ex2_poly2(a) : make_float2(ex2(a.x), ex2(a.y));
          const float p0 = j < L ? pp.x : 0.f;
          const float p1 = j + 1 < L ? pp.y : 0.f;
          sum2 = __fadd2_rn(sum2, make_float2(p0, p1));
          if constexpr (kBF16) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
            pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h2);
          } else {
            __half2 h2 = __floats2half2_rn(p0, p1);
            pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h2);
          }
        }
        inv_cur = __frcp_rn(sum2.x + sum2.y);
        // P(i) -> TMEM (own unit's 32 columns) once PV(i-1) has consumed P(i-1)
        if (i > 0) {
          mbar_wait(&bars->pv_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
          tc_fence_after();
        }
        tmem_st32(tmem + t_lane + C::kTmemP, pk);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->p_full);
      }
      if (i > 0) {
        // ---- epilogue of tile i-1 (its PV ran while we did softmax(i)) ----
        const int e = i - 1;
        const int tile = blockIdx.x + e * gridDim.x;
        mbar_wait(&bars->pv_done[e & 1], (e >> 1) & 1);
        tc_fence_after();
        uint32_t o[D];
#pragma unroll
        for (int g = 0; g < D / 16; ++g)
          tmem_ld16(tmem + t_lane + ((e & 1) ? C::kTmemO1 : C::kTmemO0) + g * 16,
                    *reinterpret_cast<uint32_t(*)[16]>(&o[g * 16]));
        tmem_wait_ld();
        tc_fence_before();
        uint32_t ob[D / 2];
#pragma unroll
        for (int j = 0; j < D; j += 2) {
          const float a = __uint_as_float(o[j]) * inv_prev;
          const float b = __uint_as_float(o[j + 1]) * inv_prev;
          if constexpr (kBF16) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
            ob[j >> 1] = *reinterpret_cast<uint32_t*>(&h2);
          } else {
            __half2 h2 = __floats2half2_rn(a, b);
            ob[j >> 1] = *reinterpret_cast<uint32_t*>(&h2);
          }
        }
        if (leader) bulk_wait_read<0>();   // previous store finished reading the staging tile
        named_sync(1, 128);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c) {
          uint4 v = make_uint4(ob[4 * c], ob[4 * c + 1], ob[4 * c + 2], ob[4 * c + 3]);
          *reinterpret_cast<uint4*>(orow + ((c ^ oswz) << 4)) = v;
        }
        fence_proxy_async_smem();
        named_sync(2, 128);
        if (leader) {
          store_tile<kUnitRows * C::kRowBytes>(&tm_o, sO, tile, lay.mode, lay.heads);
          bulk_commit();
        }
      }
      inv_prev = inv_cur;
    }
    if (leader) bulk_wait_read<0>();  // smem reads done; the grid's completion flushes the writes
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

// ---- host side ---------------------------------------------------------------
// Period (in tiles) after which the (window mod nW, head) pair of a tile slot repeats.
int add_period_tiles(const Geom& g, bool has_bias, bool has_mask) {
  if (!has_bias && !has_mask) return 1;
  const int64_t pu = (int64_t)g.heads * (has_mask ? g.mask_windows : 1);
  const int64_t pt = (pu % 2 == 0) ? pu / 2 : pu;
  return pt > (1 << 30) ? (1 << 30) : (int)pt;
}

template <typename T, int D, int LK, bool ADD>
int launch_t(const Geom& g, int dtype, const void* q, const void* k, const void* v, void* o,
             const float* bias, const float* mask, int layout, cudaStream_t s) {
  CUtensorMap mq, mk, mv, mo;
  int rc;
  if (layout == kUnits) {
    if ((rc = get_units_map(&mq, q, dtype, g.units, g.L, g.d, kUnitRows, 2))) return rc;
    if ((rc = get_units_map(&mk, k, dtype, g.units, g.L, g.d, kUnitRows, 2))) return rc;
    if ((rc = get_units_map(&mv, v, dtype, g.units, g.L, g.d, kUnitRows, 2))) return rc;
    if ((rc = get_units_map(&mo, o, dtype, g.units, g.L, g.d, kUnitRows, 2))) return rc;
  } else {  // q = packed qkv [N][L][3][h][d]; o = [N][L][h][d]
    const int64_t N = g.units / g.heads;
    const size_t hd = (size_t)g.heads * g.d;
    const uint8_t* qkv = static_cast<const uint8_t*>(q);
    if ((rc = get_tokens_map(&mq, qkv, dtype, N, g.L, 3, g.heads, g.d, kUnitRows))) return rc;
    if ((rc = get_tokens_map(&mk, qkv + hd * 2, dtype, N, g.L, 3, g.heads, g.d, kUnitRows))) return rc;
    if ((rc = get_tokens_map(&mv, qkv + hd * 4, dtype, N, g.L, 3, g.heads, g.d, kUnitRows))) return rc;
    if ((rc = get_tokens_map(&mo, o, dtype, N, g.L, 1, g.heads, g.d, kUnitRows))) return rc;
  }
  auto kern = fwd_tc_kernel<T, D, LK, ADD>;
  constexpr int smem = Cfg<D, ADD>::kSmem;
  if ((rc = ensure_smem_attr((const void*)kern, (int)(smem), "cudaFuncSetAttribute(fwd_tc)"))) return rc;
  const int n_tiles = (int)((g.units + 1) / 2);
  const int per_sm = Cfg<D, ADD>::kCtasPerSm;
  int grid = std::max(1, std::min(n_tiles, device_sm_count() * per_sm));
  if (ADD && n_tiles > grid) {
    const int pt = add_period_tiles(g, bias != nullptr, mask != nullptr);
    grid = (grid / pt) * pt;  // tc_fwd_supported guarantees pt <= grid
  }
  const float scale_log2 = g.scale * 1.4426950408889634f;
  AddArgs add{bias, mask, g.heads, mask ? g.mask_windows : 1};
  LayoutArgs lay{layout, g.heads};
  rc = check_cuda(launch_pdl(kern, dim3(grid), dim3(kThreads), smem, s, mq, mk, mv, mo, n_tiles,
                             (int)g.L, scale_log2, add, lay),
                  "fwd_tc_kernel launch");
  if (rc) return rc;
  count_launch();
  return check_cuda(cudaGetLastError(), "fwd_tc_kernel launch");
}

template <typename T, int D, bool ADD>
int dispatch_l(const Geom& g, int dtype, const void* q, const void* k, const void* v, void* o,
               const float* b, const float* m, int lay, cudaStream_t s) {
  if (g.L == 49) return launch_t<T, D, 49, ADD>(g, dtype, q, k, v, o, b, m, lay, s);
  if (g.L == 64) return launch_t<T, D, 64, ADD>(g, dtype, q, k, v, o, b, m, lay, s);
  return launch_t<T, D, 0, ADD>(g, dtype, q, k, v, o, b, m, lay, s);
}

template <typename T>
int dispatch_d(const Geom& g, int dtype, const void* q, const void* k, const void* v, void* o,
               const float* b, const float* m, int lay, cudaStream_t s) {
  const bool add = b || m;
  switch (g.d) {
    case 16: return add ? dispatch_l<T, 16, true>(g, dtype, q, k, v, o, b, m, lay, s)
                        : dispatch_l<T, 16, false>(g, dtype, q, k, v, o, b, m, lay, s);
    case 32: return add ? dispatch_l<T, 32, true>(g, dtype, q, k, v, o, b, m, lay, s)
                        : dispatch_l<T, 32, false>(g, dtype, q, k, v, o, b, m, lay, s);
    case 64: return add ? dispatch_l<T, 64, true>(g, dtype, q, k, v, o, b, m, lay, s)
                        : dispatch_l<T, 64, false>(g, dtype, q, k, v, o, b, m, lay, s);
  }
  return fail(FWA_ERR_CAPACITY, "tcgen05 forward: unsupported head_dim");
}

}  // namespace

bool tc_fwd_supported(const Geom& g, int dtype, bool has_bias, bool has_mask) {
  if (dtype != FWA_F16 && dtype != FWA_BF16) return false;
  if (has_bias || has_mask) {
    const int64_t n_tiles = (g.units + 1) / 2;
    const int cap = device_sm_count() * (g.d <= 32 ? 2 : 1);
    if (n_tiles > cap && add_period_tiles(g, has_bias, has_mask) > cap) return false;
  }
  if (g.L < 1 || g.L > kUnitRows) return false;
  if (g.d != 16 && g.d != 32 && g.d != 64) return false;
  if (g.units > (int64_t)1 << 31) return false;
  return true;
}

size_t tc_fwd_smem(const Geom& g, int) {
  return g.d == 16 ? Cfg<16>::kSmem : g.d == 32 ? Cfg<32>::kSmem : Cfg<64>::kSmem;
}

int tc_fwd_tmem_cols(const Geom& g) {
  return g.d == 16 ? Cfg<16>::kTmemCols : g.d == 32 ? Cfg<32>::kTmemCols : Cfg<64>::kTmemCols;
}

int launch_fwd_tc(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                  const float* bias, const float* mask, void* o, cudaStream_t s, int layout) {
  const bool bf = dtype == FWA_BF16;
  return bf ? dispatch_d<__nv_bfloat16>(g, dtype, q, k, v, o, bias, mask, layout, s)
            : dispatch_d<__half>(g, dtype, q, k, v, o, bias, mask, layout, s);
  return fail(FWA_ERR_CAPACITY, "tcgen05 forward: unsupported head_dim");
}

}  // namespace fwa
