// fwa_tc_flat.cu — "flat-row" forward for large windows (64 < L <= 256, L % 16 == 0; e.g.
// Swin-B 12x12 = 144, 16x16 = 256) on tcgen05 + TMA (sm_100a), f16/bf16, optional Swin
// bias / shifted-window mask.
//
// For the [units][L][d] layout the units are contiguous, so Q/K/V/O are one flat
// [units*L][d] row matrix. Each CTA owns a contiguous unit range [ua, ub) and walks
// its rows in 128-row blocks that ignore unit boundaries: a block holds the tail of one
// unit and the head of the next (<= 3 units for L < 128). Every TMEM lane therefore
// carries a real query row — the per-unit tiling of fwa_tc_fwd_large.cu runs L=144 as a
// 128-row tile plus a 16-row tile whose softmax leaves 3 of 4 warps idle.
//
//   S = Q_blk K_u^T   one lane-masked SS MMA chain per unit segment (lanes of the
//                     segment written; tcgen05 disable-output-lane mask), N = L
//   softmax           thread = row = TMEM lane; pass 1 row max (with bias/mask: x = S*c +
//                     add, add read once from an f16 table and written back over S),
//                     pass 2 exp2 + row sum (packed f32x2; 3/8 of the exponentials as a
//                     polynomial on the FMA pipe for d <= 32), P as 16-bit pairs in TMEM
//   O = P V_u         lane-masked TS MMA chain per segment (A = P in TMEM), N = d
//   epilogue          1/rowsum, convert, swizzled staging, TMA store (a CTA's last
//                     block stores 16-row pieces so it never touches the next range)
//
// S and PV are issued from separate warps (S(b) as soon as its TMEM slot is free, PV(b) as
// soon as the softmax publishes P) and two softmax warpgroups alternate blocks. For L up to
// ~150 the TMEM is split into two S slots and two P/O slots: the S slot frees as soon as
// the softmax has read it and a separate epilogue warpgroup drains O; larger L use two or
// three 256-column buffers with P and O inside the consumed S columns. K/V of a unit are
// loaded once into a ring and released after the PV of the last block that touches the
// unit. HBM: Q, K, V read once, O written once.
#include <cuda.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <type_traits>

#include "fwa_common.cuh"
#include "fwa_flat.cuh"
#include "fwa_sm100.cuh"

#ifdef FWA_TRACE
__device__ long long g_flat_trace[8][64];
extern "C" int fwa_flat_trace_copy(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_flat_trace, sizeof(g_flat_trace));
}
#define FTRACE(ev, b)                                                      \
  do {                                                                     \
    if (blockIdx.x == 0 && (b) < 64) g_flat_trace[ev][b] = clock64();     \
  } while (0)
#else
#define FTRACE(ev, b) \
  do {                \
  } while (0)
#endif

namespace fwa {
namespace {

using namespace sm100;

// warps: 0 producer, 1 S issuer, 2..9 softmax (+ epilogue unless split), 10 PV issuer,
// 11..14 epilogue (split mode)
constexpr int kRows = 128;

template <int D, int L>
struct FCfg {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kQBytes = kRows * kRowBytes;
  static constexpr int kKVBytes = L * kRowBytes;
  static constexpr int kKVSlot = (kKVBytes + 1023) / 1024 * 1024;
  static constexpr int kQStages = D >= 64 ? 2 : 4;
  static constexpr int kFixed = 1024 + kQStages * kQBytes + 2 * kQBytes + 1536;   // + barriers, sInv
  static constexpr int kKVAvail = (227 * 1024 - kFixed) / (2 * kKVSlot);
  static constexpr int kKVStages = kKVAvail < 8 ? kKVAvail : 8;
  static constexpr int kSmem = kFixed + kKVStages * 2 * kKVSlot;
  static constexpr uint32_t kSwz = D == 16 ? 6u : (D == 32 ? 4u : 2u);
  static constexpr int kChunks = kRowBytes / 16;
  static constexpr uint32_t kOCol = ((L / 2 + 15) / 16) * 16;
  // TMEM buffer = S [0, L), then P over [0, L/2) and O at [kOCol, kOCol + D); three buffers
  // when they fit in 512 columns (S of block b+2 is issued while b+1 and b are in flight)
  static constexpr int kBW = ((L > (int)kOCol + D ? L : (int)kOCol + D) + 15) / 16 * 16;
  // split mode (L up to ~150): two S slots [0, 2L) plus two P/O slots (P then O) of kPW
  // columns. The S slot frees as soon as the softmax has read S, so S(b+2) runs while P(b)
  // still waits for PV, and a separate epilogue warpgroup drains O.
  static constexpr int kPW = (int)kOCol + D;
  static constexpr bool kSplit = 2 * L + 2 * kPW <= 512;
  static constexpr int kNB = kSplit ? 2 : (3 * kBW <= 512 ? 3 : 2);
  static constexpr int kThreads = kSplit ? 480 : 352;
  // columns [kPolyFrom, 32) of each 32-column piece exponentiate on the FMA pipe (ex2_poly2):
  // measured best 37.5 % for d <= 32, 25 % for d = 64 (whose PV leaves less FMA slack)
  static constexpr int kPolyFrom = D >= 64 ? 24 : 20;
  // units resident between the oldest block awaiting PV and the newest S
  static constexpr int kNeedKV = (L - std::gcd(128, L) + (kNB + 1) * kRows + L - 1) / L;
  static constexpr bool kFits = kKVStages >= kNeedKV && kBW <= 256 && kSmem <= 227 * 1024;
};

struct FBarriers {
  uint64_t q_full[4], q_empty[4], kv_full[8], kv_empty[8];
  uint64_t s_full[3], p_ready[3], o_full[3], buf_free[3];
  uint32_t tmem_base;
};

template <typename T>
__device__ __forceinline__ uint32_t fpack2(float a, float b) {
  if constexpr (DT<T>::id == FWA_BF16) {
    __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  } else {
    __half2 h2 = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  }
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// tcgen05 disable-output-lane word w (lanes 32w..32w+31): bit set = lane outside [lo, hi)
__device__ __forceinline__ uint32_t lane_off(int w, int lo, int hi) {
  const int a = max(lo - 32 * w, 0), b = min(hi - 32 * w, 32);
  if (b <= a) return 0xffffffffu;
  const uint32_t in = (b - a == 32) ? 0xffffffffu : (((1u << (b - a)) - 1u) << a);
  return ~in;
}

// 32 lanes x 32-bit, 32 consecutive columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// Streams one TMEM row segment [0, N) in 32-column pieces (the last may be 16 wide): the
// next piece's tcgen05.ld is in flight while f(first column, values) runs on this one.
template <int N, typename F>
__device__ __forceinline__ void srow_stream(uint32_t taddr, F&& f) {
  uint32_t buf[2][32];
  constexpr int kPieces = (N + 31) / 32;
  auto load = [&](int c, uint32_t (&r)[32]) {
    if (c * 32 + 32 <= N) tmem_ld32(taddr + c * 32, r);
    else tmem_ld16(taddr + c * 32, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
  };
  load(0, buf[0]);
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < kPieces; ++c) {
    if (c + 1 < kPieces) load(c + 1, buf[(c + 1) & 1]);
    f(c * 32, buf[c & 1]);
    tmem_wait_ld();
  }
}

// Swin bias / shifted-window mask (ADD): `add` = (bias[h] + mask[w]) * log2e as f16, laid
// out [w][h][L][L] (w = window index mod the mask period, h = head; unit u = (n, h) with
// n = u / heads, w = n % n_w). Each softmax thread reads its row's L values from L2.
struct FlatAdd {
  const __half* table;
  int heads;
  int n_w;
};

// volatile loads: kept in program order (plain __ldg gets hoisted for the whole row,
// which spills at L >= 128)
__device__ __forceinline__ uint4 ldv4_nc(const __half* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// srow_stream plus the matching 16 f16 of this row's add table per 16-column piece (two
// 8-column chunks of the chunk-major table, coalesced across the warp). The first two pieces'
// loads are issued by the caller before it waits for S (`pre`) and three pieces stay in
// flight, so the L2 latency overlaps the barrier wait and the math of earlier pieces.
template <int N, typename F>
__device__ __forceinline__ void srow_stream_add(uint32_t taddr, const __half* arow,
                                                const uint4 (&pre)[2][2], F&& f) {
  uint32_t buf[2][16];
  uint4 ab[3][2];
  constexpr int kPieces = N / 16;
  ab[0][0] = pre[0][0];
  ab[0][1] = pre[0][1];
  ab[1][0] = pre[1][0];
  ab[1][1] = pre[1][1];
  tmem_ld16(taddr, buf[0]);
  if (kPieces > 2) {
    ab[2][0] = ldv4_nc(arow + 4 * (N * 8));
    ab[2][1] = ldv4_nc(arow + 5 * (N * 8));
  }
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < kPieces; ++c) {
    if (c + 1 < kPieces) tmem_ld16(taddr + (c + 1) * 16, buf[(c + 1) & 1]);
    f(c * 16, buf[c & 1], ab[c % 3]);
    if (c + 3 < kPieces) {
      ab[c % 3][0] = ldv4_nc(arow + (2 * (c + 3)) * (N * 8));
      ab[c % 3][1] = ldv4_nc(arow + (2 * (c + 3) + 1) * (N * 8));
    }
    tmem_wait_ld();
  }
}

// pieces mode: Q and O through per-segment boxes (fwa_flat.cuh)
struct FwdPieceMaps {
  RowMaps q, o;
};
template <bool PC>
using FwdPM = std::conditional_t<PC, FwdPieceMaps, NoRowMaps>;

template <typename T, int D, int L, bool ADD, bool PC>
__global__ void __launch_bounds__(FCfg<D, L>::kThreads, 1)
fwd_flat_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                const __grid_constant__ CUtensorMap tm_o16, int64_t n_units, float scale_log2,
                FlatAdd add, FlatMap fm, const __grid_constant__ FwdPM<PC> pm) {
  using C = FCfg<D, L>;
  constexpr bool kBF16 = DT<T>::id == FWA_BF16;
  constexpr int QS = C::kQStages, KS = C::kKVStages, NB = C::kNB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;                              // [KS] K slots
  uint8_t* sV = sK + KS * C::kKVSlot;              // [KS] V slots
  uint8_t* sQ = sV + KS * C::kKVSlot;              // [QS] Q blocks
  uint8_t* sO = sQ + QS * C::kQBytes;              // [2] output staging (one per group)
  FBarriers* bars = reinterpret_cast<FBarriers*>(sO + 2 * C::kQBytes);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // this CTA's unit range and its 128-row blocks
  const int64_t ua = (int64_t)blockIdx.x * n_units / gridDim.x;
  const int64_t ub = (int64_t)(blockIdx.x + 1) * n_units / gridDim.x;
  const int r0 = (int)(ua * L), r1 = (int)(ub * L);
  const int nblk = (r1 - r0 + kRows - 1) / kRows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < QS; ++s) {
      mbar_init(&bars->q_full[s], 1);
      mbar_init(&bars->q_empty[s], 1);
    }
    for (int s = 0; s < KS; ++s) {
      mbar_init(&bars->kv_full[s], 1);
      mbar_init(&bars->kv_empty[s], 1);
    }
    for (int s = 0; s < 3; ++s) {
      mbar_init(&bars->s_full[s], 1);
      mbar_init(&bars->p_ready[s], 128);
      mbar_init(&bars->o_full[s], 1);
      mbar_init(&bars->buf_free[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_o);
    tma_prefetch_desc(&tm_o16);
  }
  if (warp == 1) tmem_alloc(&bars->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  float* sInv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);   // [2][128]
  // TMEM columns of block b: S, P (16-bit pairs), O
  auto s_col = [&](int b) -> uint32_t { return C::kSplit ? (b & 1) * L : (b % NB) * C::kBW; };
  auto p_col = [&](int b) -> uint32_t { return C::kSplit ? 2 * L + (b & 1) * C::kPW : (b % NB) * C::kBW; };
  auto o_col = [&](int b) -> uint32_t { return p_col(b) + C::kOCol; };
  griddep_launch_dependents();

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0 && nblk > 0) {
      griddep_wait();
      // streamed once: evict_first -- except token-major rows (one head's 64 B of a 768 B
      // token row), whose neighbours are the next units' rows: kept at normal priority
      const uint64_t pol = (PC && fm.tok) ? policy_evict_normal() : policy_evict_first();
      int next = 0;  // next local unit to load
      const int n_loc = (int)(ub - ua);
      for (int b = 0; b < nblk; ++b) {
        const int rs = r0 + b * kRows;
        const int last = (min(rs + kRows, r1) - 1) / L - (int)ua;
        for (; next <= last && next < n_loc; ++next) {
          const int s = next % KS;
          mbar_wait(&bars->kv_empty[s], ((next / KS) & 1) ^ 1);
          mbar_arrive_expect_tx(&bars->kv_full[s], 2 * C::kKVBytes);
          if constexpr (PC) {
            int un, uh;
            vunit_nh(fm, (int)(ua + next), un, uh);
            ld_unit_rows<L>(sK + s * C::kKVSlot, &tm_k, &bars->kv_full[s], fm, un, uh, 0, pol);
            ld_unit_rows<L>(sV + s * C::kKVSlot, &tm_v, &bars->kv_full[s], fm, un, uh, 0, pol);
          } else {
            const int row = (int)((ua + next) * L);
            tma_load_3d(sK + s * C::kKVSlot, &tm_k, &bars->kv_full[s], 0, row, 0, pol);
            tma_load_3d(sV + s * C::kKVSlot, &tm_v, &bars->kv_full[s], 0, row, 0, pol);
          }
        }
        const int qs = b % QS;
        mbar_wait(&bars->q_empty[qs], ((b / QS) & 1) ^ 1);
        if constexpr (PC) {   // rows not contiguous in memory: one box per unit segment
          const int nrows = min(rs + kRows, r1) - rs;
          mbar_arrive_expect_tx(&bars->q_full[qs], nrows * C::kRowBytes);
          ld_segments<L, C::kRowBytes>(sQ + qs * C::kQBytes, pm.q, &bars->q_full[qs], fm, rs, nrows, pol);
        } else {
          mbar_arrive_expect_tx(&bars->q_full[qs], C::kQBytes);
          tma_load_3d(sQ + qs * C::kQBytes, &tm_q, &bars->q_full[qs], 0, rs, 0, pol);
        }
      }
    }
  } else if (warp == 1) {
    // ===== S issuer: S(b) into TMEM buffer b % NB as soon as its inputs and buffer are ready =====
    if (nblk > 0) {
      constexpr uint32_t idS = make_idesc_f16(kBF16, 128, L, false, false);
      constexpr uint32_t sbo = 8 * C::kRowBytes;
      for (int b = 0; b < nblk; ++b) {
        const int j = b % NB, qs = b % QS;
        const int rs = r0 + b * kRows, re = min(rs + kRows, r1);
        const int u0 = rs / L, u1 = (re - 1) / L;
        mbar_wait(&bars->q_full[qs], (b / QS) & 1);
        for (int u = u0; u <= u1; ++u) {
          const int lu = u - (int)ua;
          mbar_wait(&bars->kv_full[lu % KS], (lu / KS) & 1);
        }
        FTRACE(0, b);
        if (C::kSplit) {
          if (b >= 2) mbar_wait(&bars->p_ready[b & 1], ((b >> 1) - 1) & 1);   // S slot read
        } else if (b >= NB) {
          mbar_wait(&bars->buf_free[j], ((b / NB) - 1) & 1);
        }
        tc_fence_after();
        FTRACE(1, b);
        const uint64_t a_q = make_sdesc(smem_u32(sQ + qs * C::kQBytes), 16, sbo, C::kSwz);
        for (int u = u0; u <= u1; ++u) {
          const int lo = max(u * L, rs) - rs, hi = min((u + 1) * L, re) - rs;
          const uint32_t m0 = lane_off(0, lo, hi), m1 = lane_off(1, lo, hi);
          const uint32_t m2 = lane_off(2, lo, hi), m3 = lane_off(3, lo, hi);
          const uint64_t b_k = make_sdesc(smem_u32(sK + ((u - (int)ua) % KS) * C::kKVSlot), 16, sbo, C::kSwz);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              mma_f16_ss_m(tmem + s_col(b), desc_add(a_q, kk * 2), desc_add(b_k, kk * 2), idS, kk > 0,
                           m0, m1, m2, m3);
          }
          __syncwarp();
        }
        if (elect_one()) {
          mma_commit(&bars->s_full[j]);
          mma_commit(&bars->q_empty[qs]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 10) {
    // ===== PV issuer: O(b) = P(b) V as soon as the softmax of b has published P =====
    if (nblk > 0) {
      constexpr uint32_t idO = make_idesc_f16(kBF16, 128, D, false, true);
      constexpr uint32_t sbo = 8 * C::kRowBytes;
      for (int b = 0; b < nblk; ++b) {
        const int j = b % NB;
        const int rs = r0 + b * kRows, re = min(rs + kRows, r1);
        const int u0 = rs / L, u1 = (re - 1) / L;
        mbar_wait(&bars->p_ready[j], (b / NB) & 1);
        tc_fence_after();
        FTRACE(2, b);
        const uint32_t tp = tmem + p_col(b), to = tmem + o_col(b);
        for (int u = u0; u <= u1; ++u) {
          const int lo = max(u * L, rs) - rs, hi = min((u + 1) * L, re) - rs;
          const uint32_t m0 = lane_off(0, lo, hi), m1 = lane_off(1, lo, hi);
          const uint32_t m2 = lane_off(2, lo, hi), m3 = lane_off(3, lo, hi);
          const uint64_t b_v = make_sdesc(smem_u32(sV + ((u - (int)ua) % KS) * C::kKVSlot), C::kKVSlot, sbo, C::kSwz);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < L / 16; ++kk)
              mma_f16_ts_m(to, tp + kk * 8, desc_add(b_v, (kk * 16 * C::kRowBytes) >> 4), idO,
                           kk > 0, m0, m1, m2, m3);
          }
          __syncwarp();
        }
        // units whose last block is b: their K/V slots may be refilled (S(b+1) does not use them)
        const int nxt_u0 = (b + 1 < nblk) ? (rs + kRows) / L : u1 + 1;
        if (elect_one()) {
          mma_commit(&bars->o_full[j]);
          for (int u = u0; u <= u1 && u < nxt_u0; ++u)
            mma_commit(&bars->kv_empty[(u - (int)ua) % KS]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 10) {
    // ===== softmax + epilogue: group g takes blocks b = g, g+2, ... =====
    const int g = (warp - 2) >> 2;
    const int qd = warp & 3;
    const int r_in = qd * 32 + lane;
    const uint32_t t_lane = (uint32_t)(qd * 32) << 16;
    const uint32_t oswz = (uint32_t)((r_in * C::kRowBytes) >> 7) & (C::kChunks - 1);
    uint8_t* stage = sO + g * C::kQBytes;
    const bool leader = (warp & 3) == 0 && lane == 0;   // one thread per group
    for (int b = g; b < nblk; b += 2) {
      const int j = b % NB;
      const uint32_t tb = tmem + t_lane + s_col(b);
      const uint32_t tpw = tmem + t_lane + p_col(b);
      float mx = -INFINITY;
      // this row's (bias + mask) * log2e (f16, L2-resident table); rows past the range clamp;
      // its first pieces are requested before waiting for S
      const __half* arow = nullptr;
      uint4 apre[2][2];
      if constexpr (ADD) {
        // 32-bit index math (rows < 2^31 is a precondition of the flat kernels)
        const int grow = min(r0 + b * kRows + r_in, r1 - 1);
        const int u = grow / L, i = grow - (grow / L) * L;
        int n, hd;
        if constexpr (PC) {
          vunit_nh(fm, u, n, hd);
        } else {
          hd = u % add.heads;
          n = u / add.heads;
        }
        const int nw = n % add.n_w;
        arow = add.table + (int64_t)(nw * add.heads + hd) * L * L + i * 8;
        apre[0][0] = ldv4_nc(arow);
        apre[0][1] = ldv4_nc(arow + 1 * (L * 8));
        apre[1][0] = ldv4_nc(arow + 2 * (L * 8));
        apre[1][1] = ldv4_nc(arow + 3 * (L * 8));
      }
      mbar_wait(&bars->s_full[j], (b / NB) & 1);
      tc_fence_after();
      if (leader) FTRACE(3, b);
      // scores in the exp2 domain: s * scale * log2e (+ add)
      const float2 sc2 = make_float2(scale_log2, scale_log2);
      if constexpr (ADD) {
        // pass 1 with the add row: x = s*scale*log2e + add is written back over S (TMEM) so
        // pass 2 reads it without touching the table again
        srow_stream_add<L>(tb, arow, apre, [&](int c0, const uint32_t* r, const uint4* a4) {
          uint32_t xs[16];
#pragma unroll
          for (int t = 0; t < 16; t += 2) {
            const uint32_t* aw = reinterpret_cast<const uint32_t*>(&a4[t / 8]);
            const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&aw[(t % 8) / 2]));
            const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[t]), __uint_as_float(r[t + 1])), sc2, a);
            mx = fmax3(mx, x.x, x.y);
            xs[t] = __float_as_uint(x.x);
            xs[t + 1] = __float_as_uint(x.y);
          }
          tmem_st16(tb + c0, xs);
        });
        tmem_wait_st();
      } else {
        srow_stream<L>(tb, [&](int c0, const uint32_t* r) {   // pass 1: row max
#pragma unroll
          for (int t = 0; t < 32; t += 2)
            if (c0 + t < L) mx = fmax3(mx, __uint_as_float(r[t]), __uint_as_float(r[t + 1]));
        });
      }
      const float mxs = ADD ? mx : mx * scale_log2;
      float2 sum2 = make_float2(0.f, 0.f);
      const float2 nm2 = make_float2(-mxs, -mxs);
      if (C::kSplit && b >= 2) mbar_wait(&bars->buf_free[b & 1], ((b >> 1) - 1) & 1);   // P/O slot
      // pass 2: p = 2^(x - m) -> P (x = s*scale*log2e, or the biased x already in TMEM)
      const float2 sx2 = ADD ? make_float2(1.f, 1.f) : sc2;
      srow_stream<L>(tb, [&](int c0, const uint32_t* r) {
        uint32_t pk[16];
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          if (c0 + t < L) {
            // pairs on packed f32x2 FMA; a quarter of the exponentials (columns 24..31 of
            // each piece) on the FMA pipe instead of the MUFU
            const float2 a = __ffma2_rn(make_float2(__uint_as_float(r[t]), __uint_as_float(r[t + 1])), sx2, nm2);
            const float2 p = t >= C::kPolyFrom ? ex2_poly2(a) : make_float2(ex2(a.x), ex2(a.y));
            sum2 = __fadd2_rn(sum2, p);
            pk[t >> 1] = fpack2<T>(p.x, p.y);
          }
        }
        if (c0 + 32 <= L) {
          tmem_st16(tpw + c0 / 2, pk);
        } else {
          tmem_st8(tpw + c0 / 2, pk);
        }
      });
      tmem_wait_st();
      if (leader) FTRACE(4, b);
      const float inv = __frcp_rn(sum2.x + sum2.y);
      if (C::kSplit) sInv[(b & 1) * 128 + r_in] = inv;
      tc_fence_before();
      mbar_arrive(&bars->p_ready[j]);
      if (C::kSplit) continue;   // the epilogue warpgroup drains O

      // ---- epilogue of block b ----
      const int rs = r0 + b * kRows, nrows = min(kRows, r1 - rs);
      mbar_wait(&bars->o_full[j], (b / NB) & 1);
      tc_fence_after();
      if (leader) FTRACE(5, b);
      uint32_t o[D];
#pragma unroll
      for (int q = 0; q < D / 16; ++q)
        tmem_ld16(tmem + t_lane + o_col(b) + q * 16, *reinterpret_cast<uint32_t(*)[16]>(&o[q * 16]));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars->buf_free[j]);
      if (leader) bulk_wait_read<0>();           // previous store out of this staging buffer
      named_sync(1 + g, 128);
      uint8_t* orow = stage + r_in * C::kRowBytes;
#pragma unroll
      for (int c = 0; c < C::kChunks; ++c)
        *reinterpret_cast<uint4*>(orow + ((c ^ oswz) << 4)) = make_uint4(
            fpack2<T>(__uint_as_float(o[8 * c]) * inv, __uint_as_float(o[8 * c + 1]) * inv),
            fpack2<T>(__uint_as_float(o[8 * c + 2]) * inv, __uint_as_float(o[8 * c + 3]) * inv),
            fpack2<T>(__uint_as_float(o[8 * c + 4]) * inv, __uint_as_float(o[8 * c + 5]) * inv),
            fpack2<T>(__uint_as_float(o[8 * c + 6]) * inv, __uint_as_float(o[8 * c + 7]) * inv));
      fence_proxy_async_smem();
      named_sync(3 + g, 128);
      if (leader) {
        if constexpr (PC) {
          st_segments<L, C::kRowBytes, false>(pm.o, stage, fm, rs, nrows, 0);
        } else if (nrows == kRows) {
          tma_store_3d(&tm_o, stage, 0, rs, 0);
        } else {
          for (int t = 0; t < nrows; t += 16)
            tma_store_3d(&tm_o16, stage + t * C::kRowBytes, 0, rs + t, 0);
        }
        bulk_commit();
      }
      if (leader) FTRACE(6, b);
    }
    if (leader) bulk_wait_read<0>();
  } else if (C::kSplit && warp >= 11) {
    // ===== split mode: epilogue warpgroup (warps 11..14 = lane quarters 3, 0, 1, 2) =====
    const int qd = warp & 3;
    const int r_in = qd * 32 + lane;
    const uint32_t t_lane = (uint32_t)(qd * 32) << 16;
    const uint32_t oswz = (uint32_t)((r_in * C::kRowBytes) >> 7) & (C::kChunks - 1);
    const bool leader = warp == 12 && lane == 0;
    for (int b = 0; b < nblk; ++b) {
      const int rs = r0 + b * kRows, nrows = min(kRows, r1 - rs);
      mbar_wait(&bars->o_full[b & 1], (b >> 1) & 1);
      mbar_wait(&bars->p_ready[b & 1], (b >> 1) & 1);   // orders the softmax's sInv store
      tc_fence_after();
      if (leader) FTRACE(5, b);
      uint32_t o[D];
#pragma unroll
      for (int q = 0; q < D / 16; ++q)
        tmem_ld16(tmem + t_lane + o_col(b) + q * 16, *reinterpret_cast<uint32_t(*)[16]>(&o[q * 16]));
      tmem_wait_ld();
      const float inv = sInv[(b & 1) * 128 + r_in];
      tc_fence_before();
      mbar_arrive(&bars->buf_free[b & 1]);   // P/O slot reusable
      uint8_t* stage = sO + (b & 1) * C::kQBytes;
      if (leader) bulk_wait_read<1>();       // the store that last used this staging buffer
      named_sync(1, 128);
      uint8_t* orow = stage + r_in * C::kRowBytes;
#pragma unroll
      for (int c = 0; c < C::kChunks; ++c)
        *reinterpret_cast<uint4*>(orow + ((c ^ oswz) << 4)) = make_uint4(
            fpack2<T>(__uint_as_float(o[8 * c]) * inv, __uint_as_float(o[8 * c + 1]) * inv),
            fpack2<T>(__uint_as_float(o[8 * c + 2]) * inv, __uint_as_float(o[8 * c + 3]) * inv),
            fpack2<T>(__uint_as_float(o[8 * c + 4]) * inv, __uint_as_float(o[8 * c + 5]) * inv),
            fpack2<T>(__uint_as_float(o[8 * c + 6]) * inv, __uint_as_float(o[8 * c + 7]) * inv));
      fence_proxy_async_smem();
      named_sync(2, 128);
      if (leader) {
        if constexpr (PC) {
          st_segments<L, C::kRowBytes, false>(pm.o, stage, fm, rs, nrows, 0);
        } else if (nrows == kRows) {
          tma_store_3d(&tm_o, stage, 0, rs, 0);
        } else {
          for (int t = 0; t < nrows; t += 16)
            tma_store_3d(&tm_o16, stage + t * C::kRowBytes, 0, rs + t, 0);
        }
        bulk_commit();
      }
      if (leader) FTRACE(6, b);
    }
    if (leader) bulk_wait_read<0>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// (bias[h] + mask[w]) * log2e -> f16 table [n_w][h][L][L] (either input may be null)
// One (window, head) plane per blockIdx.y; thread v = (8-column chunk k, row i), i fastest:
// the table is stored chunk-major, plane[k][i][8], so the softmax threads of a warp (32
// consecutive rows) read one 512-byte run per 16-byte load instead of 32 rows 2L bytes apart
// (that uncoalesced load was most of the bias cost of the forward: 230 vs 154 us).
__global__ void flat_add_table_kernel(const float* __restrict__ bias, const float* __restrict__ mask,
                                      int heads, int n_w, int L, __half* __restrict__ out) {
  const int LL = L * L, plane = blockIdx.y;   // plane = w * heads + h
  const int h = plane % heads, w = plane / heads;
  const float* bp = bias ? bias + (size_t)h * LL : nullptr;
  const float* mp = mask ? mask + (size_t)w * LL : nullptr;
  uint4* o = reinterpret_cast<uint4*>(out + (size_t)plane * LL);
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < LL / 8; v += gridDim.x * blockDim.x) {
    const int k = v / L, i = v - k * L;         // output (chunk k, row i)
    const int src = i * L + k * 8;              // row-major (i, 8k .. 8k+7)
    float a[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) a[t] = 0.f;
    if (bp) {
      const float4 x = *reinterpret_cast<const float4*>(bp + src), y = *reinterpret_cast<const float4*>(bp + src + 4);
      a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w; a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
    }
    if (mp) {
      const float4 x = *reinterpret_cast<const float4*>(mp + src), y = *reinterpret_cast<const float4*>(mp + src + 4);
      a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w; a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
    }
    const float kl = 1.4426950408889634f;
    __half2 r[4] = {__floats2half2_rn(a[0] * kl, a[1] * kl), __floats2half2_rn(a[2] * kl, a[3] * kl),
                    __floats2half2_rn(a[4] * kl, a[5] * kl), __floats2half2_rn(a[6] * kl, a[7] * kl)};
    o[v] = *reinterpret_cast<uint4*>(r);
  }
}

__host__ __device__ constexpr bool flat_pc_built_rt(int D, int L) {
  return D == 32 && (L == 128 || L == 144 || L == 192 || L == 256);
}

template <typename T, int D, int L, bool PC>
int launch_flat_kern(const Geom& g, const CUtensorMap* m, const FlatAdd& fa, const FlatMap& fm,
                     const FwdPM<PC>& pm, bool add, cudaStream_t s) {
  using C = FCfg<D, L>;
  auto kern = add ? fwd_flat_kernel<T, D, L, true, PC> : fwd_flat_kernel<T, D, L, false, PC>;
  int rc;
  if ((rc = ensure_smem_attr((const void*)kern, (int)(C::kSmem), "cudaFuncSetAttribute(fwd_flat)"))) return rc;
  // every CTA gets >= 1 unit (ranges are balanced to within one unit)
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(g.units, device_sm_count()));
  rc = check_cuda(launch_pdl(kern, dim3(grid), dim3(C::kThreads), (size_t)C::kSmem, s, m[0], m[1],
                             m[2], m[3], m[4], (int64_t)g.units, g.scale * 1.4426950408889634f, fa, fm,
                             pm),
                  "fwd_flat_kernel launch");
  if (rc) return rc;
  count_launch();
  return FWA_OK;
}

template <typename T, int D, int L>
int launch_flat_t(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                  const float* bias, const float* mask, void* o, cudaStream_t s, int layout) {
  using C = FCfg<D, L>;
  if constexpr (!C::kFits) {
    return fail(FWA_ERR_CAPACITY, "flat forward: shape does not fit");
  } else {
    const FlatMap fm{layout == kTokens ? 1 : 0, 0, g.heads, (int)(g.units / g.heads)};
    const bool pc = fm.tok || (flat_force_pieces() && flat_pc_built_rt(D, L));
    if (pc && !flat_pc_built_rt(D, L))
      return fail(FWA_ERR_CAPACITY, "flat forward: no token-major build for this shape");
    const bool add = bias || mask;
    FlatAdd fa{g.add_table, g.heads, g.add_nw};
    if (add && !fa.table) return fail(FWA_ERR_SHAPE, "flat forward: bias/mask given without the add table");
    CUtensorMap m[5];
    int rc;
    const int64_t N = fm.n_win;
    const size_t hdb = (size_t)g.heads * D * 2;
    const uint8_t* qkv = static_cast<const uint8_t*>(q);
    if (!fm.tok) {
      const int rows = (int)(g.units * L);
      if ((rc = get_units_map(&m[0], q, dtype, 1, rows, D, kRows, 1))) return rc;
      if ((rc = get_units_map(&m[1], k, dtype, 1, rows, D, L, 1))) return rc;
      if ((rc = get_units_map(&m[2], v, dtype, 1, rows, D, L, 1))) return rc;
      if ((rc = get_units_map(&m[3], o, dtype, 1, rows, D, kRows, 1))) return rc;
      if ((rc = get_units_map(&m[4], o, dtype, 1, rows, D, 16, 1))) return rc;
    } else {   // q = packed qkv [N][L][3][h][d]; o = [N][L][h][d]
      if ((rc = get_tokens_map(&m[1], qkv + hdb, dtype, N, L, 3, g.heads, D, L))) return rc;
      if ((rc = get_tokens_map(&m[2], qkv + 2 * hdb, dtype, N, L, 3, g.heads, D, L))) return rc;
      m[0] = m[3] = m[4] = m[1];   // unused: Q / O go through the per-segment maps
    }
    if (!pc) return launch_flat_kern<T, D, L, false>(g, m, fa, fm, NoRowMaps{}, add, s);
    if constexpr (flat_pc_built_rt(D, L)) {
      static_assert(sizeof(FwdPieceMaps) <= 4096, "kernel parameter budget");
      FwdPieceMaps pm;
      if (fm.tok) {
        if ((rc = get_row_maps(&pm.q, qkv, dtype, true, N, L, 3, g.heads, D))) return rc;
        if ((rc = get_row_maps(&pm.o, o, dtype, true, N, L, 1, g.heads, D))) return rc;
      } else {
        if ((rc = get_row_maps(&pm.q, q, dtype, false, g.units, L, 1, 1, D))) return rc;
        if ((rc = get_row_maps(&pm.o, o, dtype, false, g.units, L, 1, 1, D))) return rc;
      }
      return launch_flat_kern<T, D, L, true>(g, m, fa, fm, pm, add, s);
    }
    return fail(FWA_ERR_CAPACITY, "flat forward: no pieces build for this shape");
  }
}

template <typename T, int D>
int flat_l(const Geom& g, int dtype, const void* q, const void* k, const void* v, const float* bias,
           const float* mask, void* o, cudaStream_t s, int layout) {
  switch (g.L) {
    case 80: return launch_flat_t<T, D, 80>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 96: return launch_flat_t<T, D, 96>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 112: return launch_flat_t<T, D, 112>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 128: return launch_flat_t<T, D, 128>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 144: return launch_flat_t<T, D, 144>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 160: return launch_flat_t<T, D, 160>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 176: return launch_flat_t<T, D, 176>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 192: return launch_flat_t<T, D, 192>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 208: return launch_flat_t<T, D, 208>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 224: return launch_flat_t<T, D, 224>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 240: return launch_flat_t<T, D, 240>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 256: return launch_flat_t<T, D, 256>(g, dtype, q, k, v, bias, mask, o, s, layout);
  }
  return fail(FWA_ERR_CAPACITY, "flat forward: unsupported L");
}

template <int D>
constexpr bool fits_d(int L) {
  switch (L) {
    case 80: return FCfg<D, 80>::kFits;
    case 96: return FCfg<D, 96>::kFits;
    case 112: return FCfg<D, 112>::kFits;
    case 128: return FCfg<D, 128>::kFits;
    case 144: return FCfg<D, 144>::kFits;
    case 160: return FCfg<D, 160>::kFits;
    case 176: return FCfg<D, 176>::kFits;
    case 192: return FCfg<D, 192>::kFits;
    case 208: return FCfg<D, 208>::kFits;
    case 224: return FCfg<D, 224>::kFits;
    case 240: return FCfg<D, 240>::kFits;
    case 256: return FCfg<D, 256>::kFits;
  }
  return false;
}

template <int D>
constexpr int smem_d(int L) {
  switch (L) {
    case 80: return FCfg<D, 80>::kSmem;
    case 96: return FCfg<D, 96>::kSmem;
    case 112: return FCfg<D, 112>::kSmem;
    case 128: return FCfg<D, 128>::kSmem;
    case 144: return FCfg<D, 144>::kSmem;
    case 160: return FCfg<D, 160>::kSmem;
    case 176: return FCfg<D, 176>::kSmem;
    case 192: return FCfg<D, 192>::kSmem;
    case 208: return FCfg<D, 208>::kSmem;
    case 224: return FCfg<D, 224>::kSmem;
    case 240: return FCfg<D, 240>::kSmem;
    case 256: return FCfg<D, 256>::kSmem;
  }
  return 0;
}

}  // namespace

bool flat_force_pieces() {
  static const bool on = [] {
    const char* e = getenv("FWA_FLAT_PIECES");
    return e && e[0] == '1';
  }();
  return on;
}

namespace {

bool flat_disabled() {
  static const bool off = [] {
    const char* e = getenv("FWA_NO_FLAT");
    return e && e[0] == '1';
  }();
  return off;
}

}  // namespace

size_t flat_add_table_bytes(const Geom& g, bool has_mask) {
  const int64_t n_w = has_mask ? std::max(1, g.mask_windows) : 1;
  return ((size_t)n_w * g.heads * g.L * g.L * sizeof(__half) + 255) / 256 * 256;
}

int flat_build_add_table(const Geom& g, const float* bias, const float* mask, __half* out,
                         cudaStream_t s) {
  const int n_w = mask ? std::max(1, g.mask_windows) : 1;
  const int64_t n = (int64_t)n_w * g.heads * g.L * g.L;
  (void)n;
  const int per_plane = (g.L * g.L / 8 + 255) / 256;
  flat_add_table_kernel<<<dim3(per_plane, n_w * g.heads), 256, 0, s>>>(bias, mask, g.heads, n_w, g.L, out);
  int rc = check_cuda(cudaGetLastError(), "flat_add_table_kernel launch");
  if (rc) return rc;
  count_launch();
  return FWA_OK;
}

bool tc_fwd_flat_supported(const Geom& g, int dtype, bool has_bias, bool has_mask) {
  (void)has_bias;
  (void)has_mask;   // Swin bias / shifted-window mask: the ADD variant
  if (flat_disabled()) return false;
  if (dtype != FWA_F16 && dtype != FWA_BF16) return false;
  if (g.L <= 64 || g.L > 256 || g.L % 16 != 0) return false;
  if (g.units * (int64_t)g.L >= ((int64_t)1 << 31)) return false;
  switch (g.d) {
    case 16: return fits_d<16>(g.L);
    case 32: return fits_d<32>(g.L);
    case 64: return fits_d<64>(g.L);
  }
  return false;
}

size_t tc_fwd_flat_smem(const Geom& g) {
  switch (g.d) {
    case 16: return smem_d<16>(g.L);
    case 32: return smem_d<32>(g.L);
    case 64: return smem_d<64>(g.L);
  }
  return 0;
}

bool tc_fwd_flat_tokens_supported(const Geom& g, int dtype, bool has_bias, bool has_mask) {
  return tc_fwd_flat_supported(g, dtype, has_bias, has_mask) && flat_pc_built_rt(g.d, g.L);
}

int launch_fwd_tc_flat(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                       const float* bias, const float* mask, void* o, cudaStream_t s, int layout) {
  const bool bf = dtype == FWA_BF16;
  switch (g.d) {
    case 16: return bf ? flat_l<__nv_bfloat16, 16>(g, dtype, q, k, v, bias, mask, o, s, layout)
                       : flat_l<__half, 16>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 32: return bf ? flat_l<__nv_bfloat16, 32>(g, dtype, q, k, v, bias, mask, o, s, layout)
                       : flat_l<__half, 32>(g, dtype, q, k, v, bias, mask, o, s, layout);
    case 64: return bf ? flat_l<__nv_bfloat16, 64>(g, dtype, q, k, v, bias, mask, o, s, layout)
                       : flat_l<__half, 64>(g, dtype, q, k, v, bias, mask, o, s, layout);
  }
  return fail(FWA_ERR_CAPACITY, "flat forward: unsupported head_dim");
}

}  // namespace fwa
