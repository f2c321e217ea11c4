// fwa_tc_flat_bwd.cu — "flat-row" backward for large windows (64 < L <= 256, L % 16 == 0,
// TMEM 2L + (1 + 3*ceil(L/128))*d <= 512 columns with two dV sets, else one; e.g. Swin-B
// 12x12: L = 144, d = 32) on tcgen05 + TMA (sm_100a), f16/bf16, optional Swin bias /
// shifted-window mask / deterministic dBias (d = 32).
//
// As in fwa_tc_flat.cu the CTA owns a contiguous unit range and walks its flat
// [units*L][d] rows in 128-row query blocks that straddle unit boundaries, so every
// TMEM lane / softmax thread carries a real query row. Per block b (segments = the
// units it intersects, lane-masked MMAs per segment; masks from a smem lookup table):
//
//   S  = Q_b K_u^T, dP = dO_b V_u^T          TMEM [0, L), [L, 2L)      (SS, N = L)
//   softmax warps (8: two per lane quarter, each owns half of the row's keys; row
//   max / sum / rho combined through smem; packed f32x2 math, 1/4 of the exponentials
//   as a polynomial on the FMA pipe):
//     [bias/mask: x = S*c + (bias + mask)*log2e from an f16 table, written back over S]
//     p = 2^(x - m) (unnormalized)            -> smem sP (16-key 32-byte-swizzle atoms)
//     dO_b rows scaled by 1/l in place        (so dV += p^T (dO/l) = P^T dO)
//     rho = sum_j p dP / l, dS = (scale/l) p (dP - rho) -> smem sDS
//     [dBias: this CTA's [heads][L][L] fp32 slice += dS/scale (vector L2 reductions)]
//   dV_u += p^T dO'_b, dK_u += dS^T Q_b        M = keys (A read MN-major from sP/sDS),
//                                              K = the segment's query rows, TMEM accumulators
//   dQ_b  = dS K_u                             (SS, masked per segment) -> TMEM
//   4 drain warps: dQ_b per block; dK_u / dV_u when unit u's last rows are done.
//
// Two warps issue the MMAs: one S(b), dP(b) as soon as block b-1's softmax has released the
// S/dP columns, the other the gradient MMAs of each block as soon as its P and dS are in
// smem (one issue stream was the measured bottleneck), so the softmax of b+1 overlaps the
// gradients of b. dV has two accumulator sets (unit parity) when TMEM allows, so all
// dV MMAs of a block go first and release sP early; dK has one set: a block that finishes
// unit u and starts u+1 issues u's dK, commits it for draining, issues dQ_b (covering the
// drain) and only then starts u+1. HBM: Q, K, V, dO read once; dQ, dK, dV written once
// (7 L d per unit). K and V share one ring of unit slots; where that ring cannot hold the
// units in flight (L = 208/256 at d = 32, L = 96/112 at d = 64) V gets its own, shallower
// ring, released by dP instead of by the gradients. Timing-experiment builds: -DFWA_TRACE (phase stamps of CTA 0),
// -DFWA_TC_ONLY (softmax math skipped), -DFWA_NO_DRAIN, -DFWA_PROBE, -DFWA_NO_MMA_FENCE.
#include <cuda.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <numeric>

#include "fwa_common.cuh"
#include "fwa_flat.cuh"
#include "fwa_sm100.cuh"

#ifdef FWA_TRACE
__device__ long long g_bflat_trace[16][64];
extern "C" int fwa_bflat_trace_copy(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_bflat_trace, sizeof(g_bflat_trace));
}
#define BTRACE(ev, b)                                                   \
  do {                                                                  \
    if (blockIdx.x == 0 && (b) < 64) g_bflat_trace[ev][b] = clock64();  \
  } while (0)
#ifdef FWA_PROBE
// serialize: wait until every MMA issued so far has executed, then stamp event ev
#define BPROBE(ev, b)                                   \
  do {                                                  \
    if (elect_one()) mma_commit(&bars->probe);          \
    __syncwarp();                                       \
    mbar_wait(&bars->probe, probe_ph);                  \
    probe_ph ^= 1;                                      \
    if (lane == 0) BTRACE(ev, b);                       \
  } while (0)
#endif
#else
#define BTRACE(ev, b) \
  do {                \
  } while (0)
#endif
#ifndef BPROBE
#define BPROBE(ev, b) \
  do {                \
  } while (0)
#endif

#ifdef FWA_NO_MMA_FENCE
#define MMA_FENCE_AFTER() \
  do {                    \
  } while (0)
#else
#define MMA_FENCE_AFTER() tc_fence_after()
#endif

namespace fwa {
namespace {

using namespace sm100;

// warps: 0 producer, 1 S/dP issuer, 2..9 softmax, 10..13 drain, 14 gradient-MMA issuer
constexpr int kBThreads = 480;
constexpr int kRows = 128;

__host__ __device__ constexpr int span_units(int L, int rows) {
  return (L - std::gcd(128, L) + rows + L - 1) / L;
}

template <int D, int L>
struct BFCfg {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTile = kRows * kRowBytes;        // one 128-row Q or dO block
  static constexpr int kNKT = (L + 127) / 128;           // 128-key tiles (M of dK/dV)
  // P / dS tiles: [128 rows][L keys] in 32-byte-swizzle atoms of 16 keys x 8 rows, atom
  // columns of 16 keys 4 KB apart (K-major for dQ, MN-major for dV/dK). 16-key atoms keep
  // L = 144 at 36 KB per tile (64-key atoms: 48 KB), which makes room for two dS buffers.
  static constexpr int kAtoms = (L + 15) / 16;
  static constexpr int kPBytes = kAtoms * 4096;
  // the MN-major dK/dV reads of key tile kt span atoms [8kt, 8kt+8): up to kOver bytes past
  // the last tile (garbage keys feed only lanes >= L, never stored) -- must stay in smem
  static constexpr int kOver = (kNKT * 8 - kAtoms) * 4096;
  static constexpr int kKVBytes = L * kRowBytes;
  static constexpr int kKVSlot = (kKVBytes + 1023) / 1024 * 1024;
  // dS buffers: 1 (K/V and Q/dO prefetch depth measured to matter more) or 2
  static constexpr int kDSB = 1;
  // sP, sDS[kDSB], staging, + 5 KB: row partials, barriers, lane-mask table
  static constexpr int kBase = 1024 + (1 + kDSB) * kPBytes + kTile + 5120;
  // units touched between the oldest block with pending gradients and the newest S
  static constexpr int kNeedKV = span_units(L, 2 * kRows);
  // Q/dO stages: 3 when the K/V ring still holds kNeedKV units (the Q/dO slot of block b+2
  // frees only when the gradients of block b-1 have executed), else 2
  static constexpr int kQS = (kBase + 3 * 2 * kTile + kNeedKV * 2 * kKVSlot <= 227 * 1024) ? 3 : 2;
  static constexpr int kFixed = kBase + kQS * 2 * kTile;
  static constexpr int kKVAvail = (227 * 1024 - kFixed) / (2 * kKVSlot);
  // K and V rings: V(u) is read only by dP (freed when the dP of u's last block executed), K(u)
  // also by dQ of the gradients one block later. Same depth when kNeedKV K/V pairs fit; else
  // (L = 208/256 at d = 32, L = 96/112 at d = 64) kNeedKV K slots and one block's worth of V
  static constexpr int kVNeed = span_units(L, kRows);
  static constexpr bool kSplitKV = kKVAvail < kNeedKV;
  static constexpr int kKS = kSplitKV ? kNeedKV : (kKVAvail < 6 ? kKVAvail : 6);
  static constexpr int kVS = kSplitKV ? kVNeed : kKS;
  static_assert(kDSB == 1, "two dS buffers need the ds_ready aliasing guard (single issuing warp)");
  static constexpr int kSmem = kFixed + (kKS + kVS) * kKVSlot;
  static constexpr uint32_t kSwz = D == 16 ? 6u : (D == 32 ? 4u : 2u);
  static constexpr int kChunks = kRowBytes / 16;
  // TMEM columns: S, dP, dQ, dV (two sets, by unit parity, when they fit), dK
  // S and dP in their own columns when they fit; else (L = 192..256) dP reuses the S columns
  // once the softmax has read S (one extra MMA latency per block)
  static constexpr bool kSharedSdP = 2 * L + D + 2 * kNKT * D > 512;
  static constexpr int kSdP = kSharedSdP ? L : 2 * L;
  static constexpr bool kDV2 = kSdP + D + 3 * kNKT * D <= 512;
  static constexpr int kVSets = kDV2 ? 2 : 1;
  static constexpr uint32_t kTS = 0, kTDP = kSharedSdP ? 0 : L, kTDQ = kSdP;
  static constexpr uint32_t kTDV = kSdP + D, kTDK = kSdP + D + kVSets * kNKT * D;
  static constexpr int kCols = kSdP + D + (kVSets + 1) * kNKT * D;
  static constexpr bool kFits = (L % 16 == 0) && kCols <= 512 && kKS >= kNeedKV && kKS <= 6 &&
                                kVS <= 6 && kSmem <= 227 * 1024 && kOver <= kQS * 2 * kTile;
};

struct BFBarriers {
  uint64_t qd_full[3], qd_empty[3], k_full[6], k_empty[6], v_full[6], v_empty[6];
  uint64_t s_full, dp_full, p_ready, ds_ready, p_free, ds_free[2], s_read;
  uint64_t acc_full, acc_free, dq_full, dq_free, dsr_free;
  uint64_t probe;
  uint32_t tmem_base;
};
// the 5 KB reserve of kBase: row partials [3][2][128] f32, barriers, 81-entry lane-mask table
static_assert(3 * 2 * 128 * 4 + sizeof(BFBarriers) + 16 + 81 * 16 <= 5120, "flat bwd smem reserve");

template <typename T>
__device__ __forceinline__ uint32_t bpack2(float a, float b) {
  if constexpr (DT<T>::id == FWA_BF16) {
    __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  } else {
    __half2 h2 = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h2);
  }
}
template <typename T>
__device__ __forceinline__ float2 bunpack2(uint32_t w) {
  if constexpr (DT<T>::id == FWA_BF16) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
  } else {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
}

__device__ __forceinline__ float bfmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// disable-output-lane word w: bit set = lane outside [lo, hi)
__device__ __forceinline__ uint32_t blane_off(int w, int lo, int hi) {
  const int a = max(lo - 32 * w, 0), b = min(hi - 32 * w, 32);
  if (b <= a) return 0xffffffffu;
  const uint32_t in = (b - a == 32) ? 0xffffffffu : (((1u << (b - a)) - 1u) << a);
  return ~in;
}

// byte offset of (row r, 8-key chunk at key `key`) in a [128 rows][keys] tile of 32-byte
// swizzle atoms (16 keys x 8 rows, 256 B; 16-byte half index XOR address bit 7)
__device__ __forceinline__ int patom_off(int r, int key) {
  return (key >> 4) * 4096 + (r >> 3) * 256 + (r & 7) * 32 + ((((key >> 3) & 1) ^ ((r >> 2) & 1)) << 4);
}

// TMEM load of N (multiple of 8) consecutive columns into v[0..N); the start column is
// OFF (0 or 8) mod 16, so .x16 loads stay 16-column aligned
template <int N, int OFF>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t* v) {
  static_assert(N % 8 == 0 && (OFF == 0 || OFF == 8), "8-column granularity");
  constexpr int c0 = OFF == 8 ? 8 : 0;
  if constexpr (OFF == 8) tmem_ld8(taddr, v);
#pragma unroll
  for (int c = c0; c + 16 <= N; c += 16) tmem_ld16(taddr + c, *reinterpret_cast<uint32_t(*)[16]>(v + c));
  if constexpr ((N - c0) % 16 == 8) tmem_ld8(taddr + (N - 8), v + (N - 8));
}

// NKT key tiles x N query steps of M=128, K=16 SS MMAs (A MN-major from a P/dS tile:
// key tile kt 8 atoms = 32 KB apart, step 512 B; B = 16 query rows of dO'/Q); the first
// MMA of each key tile accumulates iff acc_first.
template <int NKT, int D, int RB, int N>
__device__ __forceinline__ void mma_steps_n(uint32_t dcol, uint64_t a0, uint64_t b0, uint32_t id,
                                            uint32_t acc_first) {
#pragma unroll
  for (int kt = 0; kt < NKT; ++kt)
#pragma unroll
    for (int st = 0; st < N; ++st)
      mma_f16_ss(dcol + kt * D, desc_add(a0, (kt * 8 * 4096 + st * 512) >> 4),
                 desc_add(b0, (st * 16 * RB) >> 4), id, st > 0 ? 1u : acc_first);
}
template <int NKT, int D, int RB>
__device__ __forceinline__ void mma_steps(int n, uint32_t dcol, uint64_t a0, uint64_t b0, uint32_t id,
                                          uint32_t acc_first) {
  switch (n) {
    case 1: mma_steps_n<NKT, D, RB, 1>(dcol, a0, b0, id, acc_first); break;
    case 2: mma_steps_n<NKT, D, RB, 2>(dcol, a0, b0, id, acc_first); break;
    case 3: mma_steps_n<NKT, D, RB, 3>(dcol, a0, b0, id, acc_first); break;
    case 4: mma_steps_n<NKT, D, RB, 4>(dcol, a0, b0, id, acc_first); break;
    case 5: mma_steps_n<NKT, D, RB, 5>(dcol, a0, b0, id, acc_first); break;
    case 6: mma_steps_n<NKT, D, RB, 6>(dcol, a0, b0, id, acc_first); break;
    case 7: mma_steps_n<NKT, D, RB, 7>(dcol, a0, b0, id, acc_first); break;
    case 8: mma_steps_n<NKT, D, RB, 8>(dcol, a0, b0, id, acc_first); break;
    default: break;
  }
}

// Streams N (multiple of 8) columns in 8-column pieces, the next piece's tcgen05.ld in
// flight while f(piece index, values) runs on the current one.
template <int N, typename F>
__device__ __forceinline__ void tmem_stream(uint32_t taddr, F&& f) {
  uint32_t buf[2][8];
  tmem_ld8(taddr, buf[0]);
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < N / 8; ++c) {
    if (c + 1 < N / 8) tmem_ld8(taddr + (c + 1) * 8, buf[(c + 1) & 1]);
    f(c, buf[c & 1]);
    tmem_wait_ld();
  }
}

// Swin bias / shifted-window mask for the backward: the same f16 (bias + mask) * log2e
// table as the forward; with dBias each CTA accumulates P (dP - rho) of its rows into its
// own [heads][L][L] fp32 slice of `ws` (reduced over CTAs in a fixed order afterwards).
struct FlatBAdd {
  const __half* table;
  int heads;
  int n_w;
  float* ws;
  int slice_heads;   // heads per CTA partial: [slice_heads][L][L] (see range_heads)
  int half_parts;    // partials in f16 (when fp32 slices of all CTAs would not fit in L2)
  int lazy_init;     // unit-major walk with >= heads units per CTA: the first unit of each head
                     // stores its rows (initialising the slice), later units reduce into them
};

// Gradient outputs for the drain's direct stores: base pointers (token-major: dq = dqkv and
// dk / dv offset by h*d / 2*h*d elements) and the row pitch in slots (3 for dqkv, else 1)
struct GradOut {
  uint8_t* dq;
  uint8_t* dk;
  uint8_t* dv;
  int S;
};

// pieces mode: Q, dO, dQ through per-segment boxes (fwa_flat.cuh)
struct BwdPieceMaps {
  RowMaps q, dout, dq;
};
template <bool PC>
using BwdPM = std::conditional_t<PC, BwdPieceMaps, NoRowMaps>;

template <typename T, int D, int L, bool ADD, bool DBIAS, bool PC>
__global__ void __launch_bounds__(kBThreads, 1)
bwd_flat_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dq16,
                const __grid_constant__ CUtensorMap tm_dk, const __grid_constant__ CUtensorMap tm_dk16,
                const __grid_constant__ CUtensorMap tm_dv, const __grid_constant__ CUtensorMap tm_dv16,
                int64_t n_units, float scale, FlatBAdd add, FlatMap fm,
                const __grid_constant__ BwdPM<PC> pm, GradOut go) {
  using C = BFCfg<D, L>;
  constexpr bool kBF16 = DT<T>::id == FWA_BF16;
  constexpr int QS = C::kQS, KS = C::kKS, VS = C::kVS, NKT = C::kNKT;
  constexpr int H = L / 2;  // keys per softmax thread (one half of the row)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sP = smem;
  uint8_t* sDS = sP + C::kPBytes;                    // [kDSB] dS tiles
  uint8_t* sQD = sDS + C::kDSB * C::kPBytes;         // [QS][Q | dO] blocks
  uint8_t* sK = sQD + QS * 2 * C::kTile;             // [KS] K slots
  uint8_t* sV = sK + KS * C::kKVSlot;                // [VS] V slots
  uint8_t* sSt = sV + VS * C::kKVSlot;               // dQ / dK / dV store staging
  float* red = reinterpret_cast<float*>(sSt + C::kTile);    // [3][2][128] row partials
  BFBarriers* bars = reinterpret_cast<BFBarriers*>(red + 3 * 2 * 128);
  // disable-output-lane masks for lane ranges [16a, 16b): segment bounds are multiples of 16
  // (L % 16 == 0), so the MMA warp looks them up instead of recomputing them per MMA chain
  uint4* lmtab = reinterpret_cast<uint4*>((reinterpret_cast<uintptr_t>(bars + 1) + 15) & ~uintptr_t(15));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  const int64_t ua = (int64_t)blockIdx.x * n_units / gridDim.x;
  const int64_t ub = (int64_t)(blockIdx.x + 1) * n_units / gridDim.x;
  const int r0 = (int)(ua * L), r1 = (int)(ub * L);
  const int nblk = (r1 - r0 + kRows - 1) / kRows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < QS; ++s) {
      mbar_init(&bars->qd_full[s], 1);
      mbar_init(&bars->qd_empty[s], 1);
    }
    for (int s = 0; s < KS; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->p_ready, 256);
    mbar_init(&bars->s_read, 256);
    mbar_init(&bars->ds_ready, 256);
    mbar_init(&bars->p_free, 1);
    mbar_init(&bars->ds_free[0], 1);
    mbar_init(&bars->ds_free[1], 1);
    mbar_init(&bars->acc_full, 1);
    mbar_init(&bars->acc_free, 128);
    mbar_init(&bars->dq_full, 1);
    mbar_init(&bars->dq_free, 128);
    mbar_init(&bars->dsr_free, 128);
    mbar_init(&bars->probe, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 1) tmem_alloc(&bars->tmem_base, 512);
  for (int t = threadIdx.x; t < 81; t += kBThreads) {
    const int lo = (t / 9) * 16, hi = (t % 9) * 16;
    lmtab[t] = make_uint4(blane_off(0, lo, hi), blane_off(1, lo, hi), blane_off(2, lo, hi), blane_off(3, lo, hi));
  }
  if (DBIAS && !add.lazy_init) {
    griddep_wait();   // the slice may still be read by the previous call's reduction
    const int eb = add.half_parts ? 2 : 4;
    float4* z = reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(add.ws) +
                                          (size_t)blockIdx.x * add.slice_heads * L * L * eb);
    for (int i = threadIdx.x; i < add.slice_heads * L * L * eb / 16; i += kBThreads)
      z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  griddep_launch_dependents();

  if (warp == 0) {
   if constexpr (PC) {
    // ===================== TMA producer (pieces mode) =====================
    // the whole warp runs the loop: lane 0 keeps the K/V ring and the barrier bookkeeping,
    // lanes 0-3 issue the <= 4 per-segment Q / dO boxes of a block concurrently (one thread
    // issuing them serially was measured as most of the pieces mode's overhead)
    if (nblk > 0) {
      griddep_wait();
      const uint64_t pol = fm.tok ? policy_evict_normal() : policy_evict_first();
      const int n_loc = (int)(ub - ua);
      int next = 0;
      for (int b = 0; b < nblk; ++b) {
        const int rs = r0 + b * kRows;
        const int last = (min(rs + kRows, r1) - 1) / L - (int)ua;
        const int first = next;
        for (; next <= last && next < n_loc; ++next) {   // K first: S(b) needs Q and K only
          const int s = next % KS;
          mbar_wait(&bars->k_empty[s], ((next / KS) & 1) ^ 1);
          if (lane == 0) mbar_arrive_expect_tx(&bars->k_full[s], (C::kSplitKV ? 1 : 2) * C::kKVBytes);
          __syncwarp();
          if (lane < (C::kSplitKV ? 1 : 2)) {   // lane 0: K, lane 1: V (one ring)
            int un, uh;
            vunit_nh(fm, (int)(ua + next), un, uh);
            ld_unit_rows<L>((lane ? sV : sK) + s * C::kKVSlot, lane ? &tm_v : &tm_k, &bars->k_full[s],
                            fm, un, uh, 0, pol);
          }
          __syncwarp();
        }
        const int qs = b % QS;
        const int nrows = min(rs + kRows, r1) - rs;
        mbar_wait(&bars->qd_empty[qs], ((b / QS) & 1) ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&bars->qd_full[qs], 2 * nrows * C::kRowBytes);
        __syncwarp();
        if (lane < 4) {   // lane = 2 * segment + tensor (0: Q, 1: dO)
          const RowMaps& rm = (lane & 1) ? pm.dout : pm.q;
          uint8_t* dst = sQD + qs * 2 * C::kTile + (lane & 1) * C::kTile;
          int seg = 0;
          for_segments<L>(fm, rs, nrows, [&](int n, int hd, int i, int off, int len) {
            if (seg++ == (lane >> 1))
              ld_unit_rows<L>(dst + off * C::kRowBytes, &rm.m[len / 16 - 1], &bars->qd_full[qs], fm, n, hd, i, pol);
          });
        }
        __syncwarp();
        if (lane == 0) {
          for (int u = first; C::kSplitKV && u < next; ++u) {   // V free once dP of u's last block ran
            const int s = u % VS;
            int un, uh;
            vunit_nh(fm, (int)(ua + u), un, uh);
            mbar_wait(&bars->v_empty[s], ((u / VS) & 1) ^ 1);
            mbar_arrive_expect_tx(&bars->v_full[s], C::kKVBytes);
            ld_unit_rows<L>(sV + s * C::kKVSlot, &tm_v, &bars->v_full[s], fm, un, uh, 0, pol);
          }
        }
        __syncwarp();
      }
    }
   } else {
    // ===================== TMA producer =====================
    // warp-wide loop: lane 0 keeps the barrier bookkeeping; lanes 0 / 1 issue the K / V and
    // Q / dO loads of a step concurrently
    if (nblk > 0) {
      griddep_wait();
      const uint64_t pol = policy_evict_first();   // streamed once
      const int n_loc = (int)(ub - ua);
      int next = 0;
      for (int b = 0; b < nblk; ++b) {
        const int rs = r0 + b * kRows;
        const int last = (min(rs + kRows, r1) - 1) / L - (int)ua;
        const int first = next;
        for (; next <= last && next < n_loc; ++next) {   // K first: S(b) needs Q and K only
          const int s = next % KS;
          mbar_wait(&bars->k_empty[s], ((next / KS) & 1) ^ 1);
          if (lane == 0) mbar_arrive_expect_tx(&bars->k_full[s], (C::kSplitKV ? 1 : 2) * C::kKVBytes);
          __syncwarp();
          if (lane == 0)
            tma_load_3d(sK + s * C::kKVSlot, &tm_k, &bars->k_full[s], 0, (int)((ua + next) * L), 0, pol);
          if (!C::kSplitKV && lane == 1)   // one ring: V rides on K's barriers (measured faster)
            tma_load_3d(sV + s * C::kKVSlot, &tm_v, &bars->k_full[s], 0, (int)((ua + next) * L), 0, pol);
          __syncwarp();
        }
        const int qs = b % QS;
        mbar_wait(&bars->qd_empty[qs], ((b / QS) & 1) ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&bars->qd_full[qs], 2 * C::kTile);
        __syncwarp();
        if (lane == 0) tma_load_3d(sQD + qs * 2 * C::kTile, &tm_q, &bars->qd_full[qs], 0, rs, 0, pol);
        if (lane == 1)
          tma_load_3d(sQD + qs * 2 * C::kTile + C::kTile, &tm_do, &bars->qd_full[qs], 0, rs, 0, pol);
        __syncwarp();
        if (lane == 0) {
          for (int u = first; C::kSplitKV && u < next; ++u) {   // V free once dP of u's last block ran
            const int s = u % VS;
            mbar_wait(&bars->v_empty[s], ((u / VS) & 1) ^ 1);
            mbar_arrive_expect_tx(&bars->v_full[s], C::kKVBytes);
            tma_load_3d(sV + s * C::kKVSlot, &tm_v, &bars->v_full[s], 0, (int)((ua + u) * L), 0, pol);
          }
        }
        __syncwarp();
      }
    }
   }
  } else if (warp == 1 || warp == 14) {
    // ===== MMA issuer: S(b), dP(b), then the gradients of block b-1 =====
    if (nblk > 0) {
      constexpr uint32_t idS = make_idesc_f16(kBF16, 128, L, false, false);
      constexpr uint32_t idMN = make_idesc_f16(kBF16, 128, D, true, true);   // dV, dK
      constexpr uint32_t idQ = make_idesc_f16(kBF16, 128, D, false, true);   // dQ
      constexpr uint32_t sbo = 8 * C::kRowBytes;
      const uint32_t p0 = smem_u32(sP), ds0 = smem_u32(sDS);
      int n_done = 0;  // units whose dK/dV were committed for draining
      uint32_t probe_ph = 0;
      (void)probe_ph;
      auto kslot = [&](int u) { return (u - (int)ua) % KS; };
      auto vslot = [&](int u) { return (u - (int)ua) % VS; };
      auto issue_SdP = [&](int b) {
        const int qs = b % QS;
        const int rs = r0 + b * kRows, re = min(rs + kRows, r1);
        const int u0 = rs / L, u1 = (re - 1) / L;
        mbar_wait(&bars->qd_full[qs], (b / QS) & 1);
        for (int u = u0; u <= u1; ++u) {
          const int lu = u - (int)ua;
          mbar_wait(&bars->k_full[lu % KS], (lu / KS) & 1);
        }
        if (b > 0) mbar_wait(&bars->ds_ready, (b - 1) & 1);   // S / dP of b-1 consumed
        MMA_FENCE_AFTER();
        if (lane == 0) BTRACE(0, b);
        const uint32_t q0 = smem_u32(sQD + qs * 2 * C::kTile), do0 = q0 + C::kTile;
        for (int u = u0; u <= u1; ++u) {
          const int lo = max(u * L, rs) - rs, hi = min((u + 1) * L, re) - rs;
          const uint4 mm = lmtab[(lo >> 4) * 9 + (hi >> 4)];
          const uint32_t m0 = mm.x, m1 = mm.y, m2 = mm.z, m3 = mm.w;
          const uint64_t a_q = make_sdesc(q0, 16, sbo, C::kSwz);
          const uint64_t b_k = make_sdesc(smem_u32(sK + kslot(u) * C::kKVSlot), 16, sbo, C::kSwz);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              mma_f16_ss_m(tmem + C::kTS, a_q + ((kk * 32) >> 4), b_k + ((kk * 32) >> 4), idS, kk > 0,
                           m0, m1, m2, m3);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(&bars->s_full);
        __syncwarp();
#ifdef FWA_TC_ONLY
        if (lane == 0) BTRACE(4, b);
#endif
        if constexpr (C::kSplitKV) {
          for (int u = u0; u <= u1; ++u) {
            const int lu = u - (int)ua;
            mbar_wait(&bars->v_full[lu % VS], (lu / VS) & 1);
          }
        }
        if constexpr (C::kSharedSdP) {   // dP goes into the S columns: the softmax must have read S
          mbar_wait(&bars->s_read, b & 1);
        }
        if constexpr (C::kSplitKV || C::kSharedSdP) MMA_FENCE_AFTER();
        for (int u = u0; u <= u1; ++u) {
          const int lo = max(u * L, rs) - rs, hi = min((u + 1) * L, re) - rs;
          const uint4 mm = lmtab[(lo >> 4) * 9 + (hi >> 4)];
          const uint32_t m0 = mm.x, m1 = mm.y, m2 = mm.z, m3 = mm.w;
          const uint64_t a_do = make_sdesc(do0, 16, sbo, C::kSwz);
          const uint64_t b_v = make_sdesc(smem_u32(sV + vslot(u) * C::kKVSlot), 16, sbo, C::kSwz);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              mma_f16_ss_m(tmem + C::kTDP, a_do + ((kk * 32) >> 4), b_v + ((kk * 32) >> 4), idS, kk > 0,
                           m0, m1, m2, m3);
          }
          __syncwarp();
        }
        if (elect_one()) {
          mma_commit(&bars->dp_full);
          // V of the units whose last rows were in this block: read by nothing after this dP
          if constexpr (C::kSplitKV) {
            const int nxt_u0 = (b + 1 < nblk) ? (rs + kRows) / L : u1 + 1;
            for (int u = u0; u <= u1 && u < nxt_u0; ++u) mma_commit(&bars->v_empty[vslot(u)]);
          }
        }
        __syncwarp();
#ifdef FWA_TC_ONLY
        if (lane == 0) BTRACE(5, b);
#endif
        BPROBE(15, b);
      };
      auto issue_dQ = [&](int c) {
        const int rs = r0 + c * kRows, re = min(rs + kRows, r1);
        const int u0 = rs / L, u1 = (re - 1) / L;
        if (c > 0) mbar_wait(&bars->dq_free, (c - 1) & 1);   // dQ(c-1) pulled out of TMEM
        MMA_FENCE_AFTER();
        for (int u = u0; u <= u1; ++u) {
          const int lo = max(u * L, rs) - rs, hi = min((u + 1) * L, re) - rs;
          const uint4 mm = lmtab[(lo >> 4) * 9 + (hi >> 4)];
          const uint32_t m0 = mm.x, m1 = mm.y, m2 = mm.z, m3 = mm.w;
          const uint64_t a_ds = make_sdesc(ds0 + (c % C::kDSB) * C::kPBytes, 16, 256, 6);
          const uint64_t b_k = make_sdesc(smem_u32(sK + kslot(u) * C::kKVSlot), C::kKVSlot, sbo, C::kSwz);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < L / 16; ++kk)
              mma_f16_ss_m(tmem + C::kTDQ, desc_add(a_ds, (kk * 4096) >> 4),
                           desc_add(b_k, (kk * 16 * C::kRowBytes) >> 4), idQ, kk > 0, m0, m1, m2, m3);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(&bars->dq_full);
        __syncwarp();
      };
      auto issue_grads = [&](int c) {
        const int qs = c % QS;
        const int rs = r0 + c * kRows, re = min(rs + kRows, r1);
        const int u0 = rs / L, u1 = (re - 1) / L;
        mbar_wait(&bars->p_ready, c & 1);
        if constexpr (!C::kDV2) {
          // (with kDSB = 1, ds_ready(c+1) needs ds_free(c), committed below: no phase aliasing)
          mbar_wait(&bars->ds_ready, c & 1);
        }
        MMA_FENCE_AFTER();
        if (lane == 0) BTRACE(1, c);
        const uint32_t q0 = smem_u32(sQD + qs * 2 * C::kTile), do0 = q0 + C::kTile;
        const uint64_t a_p = make_sdesc(p0, 4096, 256, 6);
        const uint64_t a_ds = make_sdesc(ds0 + (c % C::kDSB) * C::kPBytes, 4096, 256, 6);
        const uint64_t b_do = make_sdesc(do0, C::kTile, sbo, C::kSwz);
        const uint64_t b_q = make_sdesc(q0, C::kTile, sbo, C::kSwz);
        // dV_kt(+)= p^T dO' / dK_kt(+)= dS^T Q over the segment's 16-row query steps
        // dV_kt(+)= p^T dO' / dK_kt(+)= dS^T Q over the segment's 16-row query steps
        // [k_lo, k_hi): straight-line MMAs per step count (no per-MMA predicate or branch)
        auto mma_dv = [&](uint32_t col, int k_lo, int k_hi, int first) {
          const uint64_t a0 = desc_add(a_p, (k_lo * 512) >> 4);
          const uint64_t b0 = desc_add(b_do, (k_lo * 16 * C::kRowBytes) >> 4);
          if (elect_one())
            mma_steps<NKT, D, C::kRowBytes>(k_hi - k_lo, tmem + col, a0, b0, idMN, first == k_lo ? 0u : 1u);
          __syncwarp();
        };
        auto mma_dk = [&](int k_lo, int k_hi, int first) {
          const uint64_t a0 = desc_add(a_ds, (k_lo * 512) >> 4);
          const uint64_t b0 = desc_add(b_q, (k_lo * 16 * C::kRowBytes) >> 4);
          if (elect_one())
            mma_steps<NKT, D, C::kRowBytes>(k_hi - k_lo, tmem + C::kTDK, a0, b0, idMN, first == k_lo ? 0u : 1u);
          __syncwarp();
        };
        if constexpr (C::kDV2) {
          // all dV first, as soon as p and the 1/l-scaled dO are in smem (p_ready; dS is not
          // needed), so sP is released for the softmax of c+1 while that of c still computes
          // dS. A unit starting here reuses the dV set of the unit two before it: wait until
          // the drain has read the last finished unit (drains run in unit order).
          bool any_start = false;
          for (int u = u0; u <= u1; ++u) any_start |= max(u * L, rs) == u * L;
          if (any_start && n_done > 0) {
            mbar_wait(&bars->acc_free, (n_done - 1) & 1);
            MMA_FENCE_AFTER();
          }
          for (int u = u0; u <= u1; ++u) {
            const int g_lo = max(u * L, rs), g_hi = min((u + 1) * L, re);
            const int k_lo = (g_lo - rs) / 16, k_hi = (g_hi - rs) / 16;
            mma_dv(C::kTDV + ((u - (int)ua) & 1) * NKT * D, k_lo, k_hi, g_lo == u * L ? k_lo : -1);
          }
          if (elect_one()) mma_commit(&bars->p_free);
          __syncwarp();
          if (lane == 0) BTRACE(8, c);
          BPROBE(4, c);
          // (with kDSB = 1, ds_ready(c+1) needs ds_free(c), committed below: no phase aliasing)
          mbar_wait(&bars->ds_ready, c & 1);
          MMA_FENCE_AFTER();
        }
        bool dq_issued = false;
        for (int u = u0; u <= u1; ++u) {
          const int g_lo = max(u * L, rs), g_hi = min((u + 1) * L, re);   // global rows
          const bool starts = g_lo == u * L, ends = g_hi == (u + 1) * L;
          if (starts && n_done > 0) {   // dK (and single-set dV) of the previous unit drained?
            if (lane == 0 && u > u0) BTRACE(11, c);
            mbar_wait(&bars->acc_free, (n_done - 1) & 1);
            MMA_FENCE_AFTER();
            if (lane == 0 && u > u0) BTRACE(12, c);
          }
          const int k_lo = (g_lo - rs) / 16, k_hi = (g_hi - rs) / 16;   // 16-row query steps
          const int first = starts ? k_lo : -1;
          if constexpr (!C::kDV2) mma_dv(C::kTDV, k_lo, k_hi, first);
          mma_dk(k_lo, k_hi, first);
          if (lane == 0) BTRACE(u == u0 ? 9 : 13, c);
          BPROBE(u == u0 ? 5 : 7, c);
          if (ends) {
            if (elect_one()) mma_commit(&bars->acc_full);
            __syncwarp();
            ++n_done;
          }
          if (!dq_issued) {   // dQ right after the first segment: covers the drain of its unit
            issue_dQ(c);
            dq_issued = true;
            if (lane == 0) BTRACE(10, c);
            BPROBE(6, c);
          }
        }
        // block c's P / dS / Q / dO fully read; release its units whose last rows were here
        const int nxt_u0 = (c + 1 < nblk) ? (rs + kRows) / L : u1 + 1;
        if (elect_one()) {
          if constexpr (!C::kDV2) mma_commit(&bars->p_free);
          mma_commit(&bars->ds_free[c % C::kDSB]);
          mma_commit(&bars->qd_empty[qs]);
          for (int u = u0; u <= u1 && u < nxt_u0; ++u) mma_commit(&bars->k_empty[kslot(u)]);
        }
        __syncwarp();
        if (lane == 0) BTRACE(2, c);
#ifdef FWA_TC_ONLY
        mbar_wait(&bars->ds_free[c % C::kDSB], (c / C::kDSB) & 1);   // timing experiment: when did the TC finish grads(c)?
        if (lane == 0) BTRACE(14, c);
#endif
      };
      // two issuing warps: S/dP of the next block never queues behind the gradient MMAs
      // of the previous one in a single instruction stream (ordering between the two is
      // carried by the barriers: S(b+1) after ds_ready(b), gradients(c) after p/ds_ready(c))
      if (warp == 1) {
        for (int b = 0; b < nblk; ++b) issue_SdP(b);
      } else {
        for (int c = 0; c < nblk; ++c) issue_grads(c);
      }
    }
  } else if (warp < 10) {
    // ===== softmax / dS: warp pair (w, w+4) share a lane quarter, each owns half the keys =====
    const int hf = (warp - 2) >> 2;
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t t_lane = (uint32_t)(qd * 32) << 16;
    const float sl2 = scale * 1.4426950408889634f;
    float* rmax = red;
    float* rsum = red + 256;
    float* rrho = red + 512;
    const uint32_t ts = tmem + t_lane + C::kTS + hf * H;
    const uint32_t tdp = tmem + t_lane + C::kTDP + hf * H;
    uint32_t pk[H / 2];   // this half row of p (then dS) as 16-bit pairs
    for (int b = 0; b < nblk; ++b) {
      const int qs = b % QS;
      // this row's (unit, query) -> (head, window); rows past the range clamp to the last one
      const int grow = min(r0 + b * kRows + r, r1 - 1);
      const int urow = grow / L, irow = grow - (grow / L) * L;
      int nrow = 0, hrow = 0;
      if constexpr (ADD && PC) {
        vunit_nh(fm, urow, nrow, hrow);
      } else if constexpr (ADD) {
        hrow = urow % add.heads;
        nrow = urow / add.heads;
      }
      uint4 arow_half[ADD ? H / 8 : 1];
      if constexpr (ADD) {
        const int wrow = nrow % add.n_w;
        // chunk-major table (fwa_tc_flat.cu): 8-column chunk k of row i at plane + (k*L + i)*8
        const uint4* ap = reinterpret_cast<const uint4*>(
            add.table + (int64_t)(wrow * add.heads + hrow) * L * L + irow * 8) + hf * (H / 8) * L;
#pragma unroll
        for (int c = 0; c < H / 8; ++c) arow_half[c] = __ldg(ap + c * L);
      }
      mbar_wait(&bars->s_full, b & 1);
      tc_fence_after();
      const bool trc = warp == 4 && lane == 0;
      if (trc) BTRACE(3, b);
#ifdef FWA_TC_ONLY
      // timing experiment: keep the barrier protocol, skip the math
      if constexpr (C::kSharedSdP) mbar_arrive(&bars->s_read);
      if (b > 0) mbar_wait(&bars->p_free, (b - 1) & 1);
      mbar_wait(&bars->dp_full, b & 1);
      tc_fence_after();
      mbar_arrive(&bars->p_ready);
      tc_fence_before();
      if (b >= C::kDSB) mbar_wait(&bars->ds_free[b % C::kDSB], ((b / C::kDSB) - 1) & 1);
      mbar_arrive(&bars->ds_ready);
      continue;
#endif
      float mx = -INFINITY;
      if constexpr (ADD) {
        // S read 1 with this half row of (bias + mask) * log2e: x = s*scale*log2e + add is
        // written back over S so read 2 does not touch the table again
        const float2 sc2a = make_float2(sl2, sl2);
        tmem_stream<H>(ts, [&](int c, const uint32_t* x) {
          const uint4 aw = arow_half[c];
          const uint32_t a4[4] = {aw.x, aw.y, aw.z, aw.w};
          uint32_t xs[8];
#pragma unroll
          for (int t = 0; t < 8; t += 2) {
            const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&a4[t / 2]));
            const float2 v = __ffma2_rn(make_float2(__uint_as_float(x[t]), __uint_as_float(x[t + 1])), sc2a, a);
            mx = bfmax3(mx, v.x, v.y);
            xs[t] = __float_as_uint(v.x);
            xs[t + 1] = __float_as_uint(v.y);
          }
          tmem_st8(ts + c * 8, xs);
        });
        tmem_wait_st();
      } else {
        tmem_stream<H>(ts, [&](int c, const uint32_t* x) {   // S read 1: row max
#pragma unroll
          for (int t = 0; t < 8; t += 2) mx = bfmax3(mx, __uint_as_float(x[t]), __uint_as_float(x[t + 1]));
        });
      }
      rmax[hf * 128 + r] = mx;
      named_sync(1, 256);
      mx = fmaxf(rmax[r], rmax[128 + r]);
      const float mxs = ADD ? mx : mx * sl2;
      float2 s2 = make_float2(0.f, 0.f);
      const float2 sc2 = ADD ? make_float2(1.f, 1.f) : make_float2(sl2, sl2), nm2 = make_float2(-mxs, -mxs);
      tmem_stream<H>(ts, [&](int c, const uint32_t* x) {   // S read 2: p = 2^(s c - m c)
#pragma unroll
        for (int t = 0; t < 8; t += 2) {
          const float2 a = __ffma2_rn(make_float2(__uint_as_float(x[t]), __uint_as_float(x[t + 1])), sc2, nm2);
          // a quarter of the exponentials on the FMA pipe
          const float2 p = t == 6 ? ex2_poly2(a) : make_float2(ex2(a.x), ex2(a.y));
          s2 = __fadd2_rn(s2, p);
          pk[c * 4 + (t >> 1)] = bpack2<T>(p.x, p.y);
        }
      });
      if constexpr (C::kSharedSdP) {   // S fully read: its columns may take dP
        tc_fence_before();
        mbar_arrive(&bars->s_read);
      }
      rsum[hf * 128 + r] = s2.x + s2.y;
      // p -> sP once the gradient MMAs of b-1 stopped reading it
      if (b > 0) mbar_wait(&bars->p_free, (b - 1) & 1);
#pragma unroll
      for (int c8 = 0; c8 < H / 8; ++c8) {
        const int key = hf * H + c8 * 8;
        *reinterpret_cast<uint4*>(sP + patom_off(r, key)) =
            make_uint4(pk[4 * c8], pk[4 * c8 + 1], pk[4 * c8 + 2], pk[4 * c8 + 3]);
      }
      if (trc) BTRACE(4, b);
      named_sync(1, 256);
      const float inv_l = __frcp_rn(rsum[r] + rsum[128 + r]);
      // dO rows *= 1/l (after dP consumed dO): this half of the row's 16-byte chunks
      mbar_wait(&bars->dp_full, b & 1);
      tc_fence_after();
      {
        uint8_t* row = sQD + qs * 2 * C::kTile + C::kTile + r * C::kRowBytes;
#pragma unroll
        for (int c = hf * (C::kChunks / 2); c < (hf + 1) * (C::kChunks / 2); ++c) {
          uint4 w = *reinterpret_cast<uint4*>(row + c * 16);
          uint32_t* e = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 f = bunpack2<T>(e[t]);
            e[t] = bpack2<T>(f.x * inv_l, f.y * inv_l);
          }
          *reinterpret_cast<uint4*>(row + c * 16) = w;
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&bars->p_ready);
      if (trc) BTRACE(5, b);
      float2 rho2 = make_float2(0.f, 0.f);
      tmem_stream<H>(tdp, [&](int c, const uint32_t* x) {   // dP read 1: sum_j p dP
#pragma unroll
        for (int t = 0; t < 8; t += 2)
          rho2 = __ffma2_rn(bunpack2<T>(pk[c * 4 + (t >> 1)]),
                            make_float2(__uint_as_float(x[t]), __uint_as_float(x[t + 1])), rho2);
      });
      rrho[hf * 128 + r] = rho2.x + rho2.y;
      named_sync(1, 256);
      const float g = scale * inv_l;
      const float rg = (rrho[r] + rrho[128 + r]) * inv_l * g;   // rho * scale / l
      const float2 g2 = make_float2(g, g), nrg2 = make_float2(-rg, -rg);
      tmem_stream<H>(tdp, [&](int c, const uint32_t* x) {   // dP read 2: dS
#pragma unroll
        for (int t = 0; t < 8; t += 2) {
          const float2 d = __ffma2_rn(make_float2(__uint_as_float(x[t]), __uint_as_float(x[t + 1])), g2, nrg2);
          const float2 v = __fmul2_rn(bunpack2<T>(pk[c * 4 + (t >> 1)]), d);
          pk[c * 4 + (t >> 1)] = bpack2<T>(v.x, v.y);
        }
      });
      tc_fence_before();   // S / dP reads done before ds_ready lets S(b+1) overwrite them
      if (b >= C::kDSB) mbar_wait(&bars->ds_free[b % C::kDSB], ((b / C::kDSB) - 1) & 1);   // buffer read
      if constexpr (DBIAS) {   // ... and by the drain warps' dBias reductions
        if (b > 0) mbar_wait(&bars->dsr_free, (b - 1) & 1);
      }
      uint8_t* sDSb = sDS + (b % C::kDSB) * C::kPBytes;
#pragma unroll
      for (int c8 = 0; c8 < H / 8; ++c8) {
        const int key = hf * H + c8 * 8;
        *reinterpret_cast<uint4*>(sDSb + patom_off(r, key)) =
            make_uint4(pk[4 * c8], pk[4 * c8 + 1], pk[4 * c8 + 2], pk[4 * c8 + 3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&bars->ds_ready);
      if (trc) BTRACE(6, b);
    }
  } else {
    // ===== drain warps: dK/dV of finished units, dQ of every block =====
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t t_lane = (uint32_t)(qd * 32) << 16;
    const bool leader = warp == 12 && lane == 0;
    (void)leader;
    // Direct stores: each drain thread writes its own row straight from registers (rows are
    // 32-128 contiguous bytes; a warp's 32 rows are contiguous in the flat layout), so emits
    // need no staging buffer, no bulk-store wait and no drain-group barrier (measured against
    // smem staging + TMA stores: equal on the plain backward, 3-8 % faster with dBias and in
    // the token-major layout).
    auto pack_row = [&](const uint32_t* x, int c) {
      return make_uint4(bpack2<T>(__uint_as_float(x[8 * c]), __uint_as_float(x[8 * c + 1])),
                        bpack2<T>(__uint_as_float(x[8 * c + 2]), __uint_as_float(x[8 * c + 3])),
                        bpack2<T>(__uint_as_float(x[8 * c + 4]), __uint_as_float(x[8 * c + 5])),
                        bpack2<T>(__uint_as_float(x[8 * c + 6]), __uint_as_float(x[8 * c + 7])));
    };
    auto put_row = [&](uint8_t* dst, const uint32_t* x) {
      const uint64_t spol = DBIAS ? policy_evict_first() : 0;
#pragma unroll
      for (int c = 0; c < C::kChunks; ++c) st_global_v4<DBIAS>(dst + c * 16, pack_row(x, c), spol);
    };
    // row kt*128 + r of unit u (dK / dV)
    auto put_unit_row = [&](uint8_t* base, const uint32_t* x, int u, int i) {
      if constexpr (PC) {
        int un, uh;
        vunit_nh(fm, u, un, uh);
        put_row(base + unit_row_offset<L>(fm, un, uh, i, go.S, C::kRowBytes), x);
      } else {
        put_row(base + ((int64_t)u * L + i) * C::kRowBytes, x);
      }
    };
    int n_unit = 0;
    for (int b = 0; b < nblk; ++b) {
      const int rs = r0 + b * kRows, re = min(rs + kRows, r1);
      const int u0 = rs / L, u1 = (re - 1) / L;
      for (int u = u0; u <= u1; ++u) {
        if ((u + 1) * L > re) continue;   // unit continues into the next block
        mbar_wait(&bars->acc_full, n_unit & 1);
        tc_fence_after();
#ifdef FWA_NO_DRAIN
        mbar_arrive(&bars->acc_free);
        ++n_unit;
        continue;
#endif
#pragma unroll
        for (int kt = 0; kt < NKT; ++kt) {
          uint32_t gv[D], gk[D];
#pragma unroll
          for (int q = 0; q < D / 16; ++q) {
            tmem_ld16(tmem + t_lane + C::kTDV + (C::kDV2 ? ((u - (int)ua) & 1) * NKT * D : 0) + kt * D + q * 16,
                      *reinterpret_cast<uint32_t(*)[16]>(&gv[q * 16]));
            tmem_ld16(tmem + t_lane + C::kTDK + kt * D + q * 16, *reinterpret_cast<uint32_t(*)[16]>(&gk[q * 16]));
          }
          tmem_wait_ld();
          if (kt == NKT - 1) {
            tc_fence_before();
            mbar_arrive(&bars->acc_free);
          }
          const int nr = min(kRows, L - kt * kRows);
          if (r < nr) {
            put_unit_row(go.dv, gv, u, kt * kRows + r);
            put_unit_row(go.dk, gk, u, kt * kRows + r);
          }
        }
        ++n_unit;
      }
      mbar_wait(&bars->dq_full, b & 1);
      tc_fence_after();
#ifdef FWA_NO_DRAIN
      mbar_arrive(&bars->dq_free);
#else
      uint32_t gq[D];
#pragma unroll
      for (int q = 0; q < D / 16; ++q)
        tmem_ld16(tmem + t_lane + C::kTDQ + q * 16, *reinterpret_cast<uint32_t(*)[16]>(&gq[q * 16]));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars->dq_free);
      if (r < re - rs) {
        const int vr = rs + r, v = vr / L;
        put_unit_row(go.dq, gq, v, vr - v * L);
      }
#endif
      if (leader) BTRACE(7, b);
      if constexpr (DBIAS) {
        // dBias partial of block b: += dS / scale = P (dP - rho) for this CTA's rows, read back
        // from sDS here, off the softmax's path (it waits dsr_free only before overwriting
        // sDS with block b+1). A warp's vector reductions cover 8 rows x 64 contiguous bytes:
        // 16 full 32-byte sectors per instruction (one row per lane, each lane on its own half
        // sector, measured 1.9x slower in L2: tools/micro/red_rate.cu). Per address one
        // thread per block, blocks ordered through ds_ready / dsr_free: deterministic.
        mbar_wait(&bars->ds_ready, b & 1);   // sDS(b) visible (cannot have advanced: dsr_free)
        const int wq = warp - 10, rr = lane & 7;
        const float is = 1.f / scale;
        const float2 is2 = make_float2(is, is);
        const uint64_t rpol = policy_evict_last();   // 4.3 KB/row slices stay resident in L2
        float4* slice = reinterpret_cast<float4*>(add.ws + (size_t)blockIdx.x * add.slice_heads * L * L);
        uint4* sliceh = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(add.ws) +
                                                 (size_t)blockIdx.x * add.slice_heads * L * L);
        int h0, h1;
        range_heads(fm, ua, ub, h0, h1);
        (void)h1;
#pragma unroll 1
        for (int grp = 0; grp < 4; ++grp) {
          const int lr = wq * 32 + grp * 8 + rr;   // block row
          const int g = rs + lr;
          if (g < r1) {
            const int u = g / L, i = g - (g / L) * L;
            int uh;
            if constexpr (PC) {
              int un;
              vunit_nh(fm, u, un, uh);
            } else {
              uh = u % add.heads;
            }
            // first unit of its head in this CTA: plain stores initialise the slice row (its
            // rows precede every reduction into them in the walk; the producer's griddep_wait
            // precedes all of this, so the previous call's reduce has finished reading)
            const bool first = add.lazy_init && (u - (int)ua) < add.heads;
            if (add.half_parts) {
              // f16 partials (8 keys per vector reduction): the slices of stages with many
              // heads stay in L2; a partial sums <= units-per-CTA / heads terms
              uint4* wp = sliceh + ((uh - h0) * L + i) * (L / 8);
#pragma unroll 2
              for (int it = 0; it < (L / 8 + 3) / 4; ++it) {
                const int c8 = it * 4 + (lane >> 3);   // 8-key column
                if (c8 < L / 8) {
                  const uint4 w = *reinterpret_cast<const uint4*>(sDS + patom_off(lr, c8 * 8));
                  const uint32_t wi[4] = {w.x, w.y, w.z, w.w};
                  uint32_t ho[4];
#pragma unroll
                  for (int t = 0; t < 4; ++t) {
                    const float2 f = __fmul2_rn(bunpack2<T>(wi[t]), is2);
                    __half2 h2 = __floats2half2_rn(f.x, f.y);
                    ho[t] = *reinterpret_cast<uint32_t*>(&h2);
                  }
                  if (first) st_global_v4<true>(wp + c8, make_uint4(ho[0], ho[1], ho[2], ho[3]), rpol);
                  else red_add_v4_f16x2_hint(wp + c8, make_uint4(ho[0], ho[1], ho[2], ho[3]), rpol);
                }
              }
            } else {
              float4* wp = slice + ((uh - h0) * L + i) * (L / 4);
#pragma unroll 3
              for (int it = 0; it < L / 16; ++it) {
                const int c = it * 4 + (lane >> 3);   // 4-key column (float4 of the slice row)
                const uint2 w = *reinterpret_cast<const uint2*>(sDS + patom_off(lr, c * 4) + (c & 1) * 8);
                const float2 a = __fmul2_rn(bunpack2<T>(w.x), is2), e = __fmul2_rn(bunpack2<T>(w.y), is2);
                if (first)
                  st_global_v4<true>(wp + c, make_uint4(__float_as_uint(a.x), __float_as_uint(a.y),
                                                        __float_as_uint(e.x), __float_as_uint(e.y)), rpol);
                else
                  red_add_v4_hint(wp + c, make_float4(a.x, a.y, e.x, e.y), rpol);
              }
            }
          }
        }
        mbar_arrive(&bars->dsr_free);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// dbias[h][i][j] = sum over the CTAs c whose unit range covers head h of their partial
// ws[c][h - h0(c)][i][j], deterministic. A block covers 32 consecutive 16-byte vectors of the
// output (threadIdx.x: 8 f16 or 4 fp32 partial values per load, contiguous across the warp) x
// 8 CTA groups (threadIdx.y: group g sums CTAs g, g+8, ... in ascending order); the group
// sums are added in g order -- a fixed association. (One thread per element issued 2-4 byte
// loads and 148 dependent steps: 48 us for the 98 MB of f16 partials at Swin-B stage 3.)
template <typename P>
__global__ void __launch_bounds__(256) bflat_dbias_reduce_kernel(const P* __restrict__ ws, int grid,
                                                                 int64_t n_units, FlatMap fm,
                                                                 int slice_heads, int LL,
                                                                 float* __restrict__ dbias) {
  constexpr int V = 16 / sizeof(P);
  __shared__ float part[8][32 * V + 1];
  const int LLv = LL / V;
  const int64_t nv = (int64_t)fm.heads * LLv;
  const int64_t e = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int g = threadIdx.y;
  float acc[V];
#pragma unroll
  for (int t = 0; t < V; ++t) acc[t] = 0.f;
  const int hd = e < nv ? (int)(e / LLv) : 0;
  const int ij = e < nv ? (int)(e - (int64_t)hd * LLv) * V : 0;
  auto add = [&](int c, int h0) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(ws + ((size_t)c * slice_heads + (hd - h0)) * LL + ij));
    if constexpr (sizeof(P) == 4) {
      acc[0] += __uint_as_float(w.x);
      acc[1] += __uint_as_float(w.y);
      acc[2] += __uint_as_float(w.z);
      acc[3] += __uint_as_float(w.w);
    } else {
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&ww[t]));
        acc[2 * t] += f.x;
        acc[2 * t + 1] += f.y;
      }
    }
  };
  if (e < nv) {
    if (!fm.head_major) {   // every CTA covers every head: no range test in the loop
#pragma unroll 4
      for (int c = g; c < grid; c += 8) add(c, 0);
    } else {
      // head-major: the CTAs covering head hd are the contiguous range [c_lo, c_hi]
      // (ua(c) = floor(c U / G) < (hd + 1) N and ub(c) = floor((c + 1) U / G) > hd N)
      const int64_t U = n_units, N = fm.n_win;
      const int c_lo = (int)(((hd * N + 1) * grid + U - 1) / U) - 1;
      const int c_hi = (int)((((int64_t)hd + 1) * N * grid + U - 1) / U) - 1;
      for (int c = max(c_lo, 0) + g; c <= min(c_hi, grid - 1); c += 8)
        add(c, (int)((int64_t)c * U / grid / N));
    }
  }
#pragma unroll
  for (int t = 0; t < V; ++t) part[g][threadIdx.x * V + t] = acc[t];
  __syncthreads();
  if (g == 0 && e < nv) {
    float out[V];
#pragma unroll
    for (int t = 0; t < V; ++t) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += part[k][threadIdx.x * V + t];
      out[t] = s;
    }
    float4* o = reinterpret_cast<float4*>(dbias + (size_t)hd * LL + ij);
#pragma unroll
    for (int t = 0; t < V / 4; ++t) o[t] = make_float4(out[4 * t], out[4 * t + 1], out[4 * t + 2], out[4 * t + 3]);
  }
}

// pieces-mode (head-major dBias walk, token-major layout) instances: Swin's d = 32 windows
__host__ __device__ constexpr bool bflat_pc_built_rt(int D, int L) {
  return D == 32 && (L == 128 || L == 144 || L == 192 || L == 256);
}
template <int D, int L>
constexpr bool bflat_pc_built() {
  return bflat_pc_built_rt(D, L);
}

// Walk order of a dBias call. Unit-major (the physical order, flat addressing) unless a CTA's
// unit range is shorter than the head count: then every CTA would keep (and zero) a partial
// for every head although it touches only a few, and the head-major walk (each CTA covers 1-2
// heads: pieces addressing) wins. Measured on B200 (tools/time_layers.py, bf16, bias + dBias):
// Swin-B stage 4 (64, 32, 144, 32) 180 -> 145 us head-major; stage 3 (256, 16, 144, 32) 224 us
// unit-major vs 250 us head-major, stage 1 815 vs 870 us (the pieces addressing costs more
// than the partial traffic it saves once a CTA spans all heads). Head-major needs a 128-row
// block to hold at most one row per (head, query) slot (L >= 128). FWA_FLAT_WALK=head / unit
// forces either.
int bflat_walk_override() {
  static const int v = [] {
    const char* e = getenv("FWA_FLAT_WALK");
    if (!e) return 0;
    return e[0] == 'h' ? 1 : (e[0] == 'u' ? -1 : 0);
  }();
  return v;
}

int bflat_grid(const Geom& g);

FlatMap bflat_map(const Geom& g, bool want_db, bool tok) {
  FlatMap fm;
  fm.tok = tok ? 1 : 0;
  const bool can = want_db && g.L >= 128 && g.heads > 1 && bflat_pc_built_rt(g.d, g.L);
  const int ov = bflat_walk_override();
  fm.head_major = (can && (ov > 0 || (ov == 0 && g.units / bflat_grid(g) < g.heads))) ? 1 : 0;
  fm.heads = g.heads;
  fm.n_win = (int)(g.units / g.heads);
  return fm;
}

int bflat_grid(const Geom& g) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(g.units, device_sm_count()));
}

// f16 dBias partials (a) when the fp32 ones of all CTAs would exceed half of L2 (Swin-B
// stages 2-4: 98 / 196 / 392 MB fp32), so the slices stay resident while Q/K/V/dO stream
// through, and (b) always for bf16 inputs: half the vector reductions (stage 1: 811 -> 746 us)
// at no cost in accuracy -- dS is formed from bf16 operands, whose 8-bit mantissa dominates
// the error (tools/dbias_precision.py: relative RMS error vs fp32 torch 2.31e-3 with fp32
// partials, 2.46e-3 with f16; fp16 inputs keep fp32 partials where they fit: 6.0e-4 vs 1.0e-3).
// The workspace query (no dtype) sizes by rule (a) alone, an upper bound for both.
// FWA_DBIAS_PARTS=f32 / f16 forces either.
bool bflat_half_parts(const Geom& g, int grid, int slice_heads, bool bf16) {
  static const int force = [] {
    const char* e = getenv("FWA_DBIAS_PARTS");
    if (!e) return 0;
    return e[1] == '1' ? 1 : (e[1] == '3' ? -1 : 0);   // "f16" -> 1, "f32" -> -1
  }();
  if (force) return force > 0;
  if (bf16) return true;
  const int64_t l2 = device_l2_bytes() > 0 ? device_l2_bytes() : (int64_t)126 << 20;
  return (int64_t)grid * slice_heads * g.L * g.L * 4 > l2 / 2;
}

// FWA_DBIAS_ZERO=1: zero the partial slices up front instead of first-touch stores (A/B)
bool bflat_eager_zero() {
  static const bool on = [] {
    const char* e = getenv("FWA_DBIAS_ZERO");
    return e && e[0] == '1';
  }();
  return on;
}

int bflat_slice_heads(const FlatMap& fm, int64_t units, int grid) {
  int sh = 1;
  for (int c = 0; c < grid; ++c) {
    int h0, h1;
    range_heads(fm, (int64_t)c * units / grid, (int64_t)(c + 1) * units / grid, h0, h1);
    sh = std::max(sh, h1 - h0 + 1);
  }
  return sh;
}

template <bool PC>
using BFlatKern = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap,
                           CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, int64_t, float, FlatBAdd,
                           FlatMap, BwdPM<PC>, GradOut);

template <typename T, int D, int L, bool PC>
int launch_bflat_kern(const Geom& g, const CUtensorMap* m, const FlatBAdd& fa, const FlatMap& fm,
                      const BwdPM<PC>& pm, const GradOut& go, bool add, bool want_db, int grid,
                      cudaStream_t s) {
  using C = BFCfg<D, L>;
  // kernel variants: plain, + bias/mask, + bias/mask + dBias (bias/mask only for d = 32)
  BFlatKern<PC> kern = bwd_flat_kernel<T, D, L, false, false, PC>;
  if constexpr (D == 32) {
    if (add) kern = want_db ? bwd_flat_kernel<T, D, L, true, true, PC> : bwd_flat_kernel<T, D, L, true, false, PC>;
  }
  int rc;
  if ((rc = ensure_smem_attr((const void*)kern, (int)(C::kSmem), "cudaFuncSetAttribute(bwd_flat)"))) return rc;
  rc = check_cuda(launch_pdl(kern, dim3(grid), dim3(kBThreads), (size_t)C::kSmem, s, m[0], m[1], m[2],
                             m[3], m[4], m[5], m[6], m[7], m[8], m[9], (int64_t)g.units, g.scale, fa, fm,
                             pm, go),
                  "bwd_flat_kernel launch");
  if (rc) return rc;
  count_launch();
  return FWA_OK;
}

template <typename T, int D, int L>
int launch_bflat_t(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                   const void* dout, const float* bias, const float* mask, void* dq, void* dk,
                   void* dv, float* dbias, float* ws, cudaStream_t s, int layout) {
  using C = BFCfg<D, L>;
  if constexpr (!C::kFits) {
    return fail(FWA_ERR_CAPACITY, "flat backward: shape does not fit");
  } else {
    const bool add = bias || mask;
    const bool want_db = dbias != nullptr;
    const FlatMap fm = bflat_map(g, want_db, layout == kTokens);
    const bool pc = fm.tok || fm.head_major || (flat_force_pieces() && bflat_pc_built<D, L>());
    if (pc && !bflat_pc_built<D, L>())
      return fail(FWA_ERR_CAPACITY, "flat backward: no token-major / head-major build for this shape");
    CUtensorMap m[10];
    int rc;
    const int64_t N = fm.n_win;
    const size_t hdb = (size_t)g.heads * D * 2;
    const uint8_t* qkv = static_cast<const uint8_t*>(q);
    uint8_t* dqkv = static_cast<uint8_t*>(dq);
    if (!fm.tok) {
      const int rows = (int)(g.units * L);
      if ((rc = get_units_map(&m[0], q, dtype, 1, rows, D, kRows, 1))) return rc;
      if ((rc = get_units_map(&m[1], k, dtype, 1, rows, D, L, 1))) return rc;
      if ((rc = get_units_map(&m[2], v, dtype, 1, rows, D, L, 1))) return rc;
      if ((rc = get_units_map(&m[3], dout, dtype, 1, rows, D, kRows, 1))) return rc;
      void* outs[3] = {dq, dk, dv};
      for (int i = 0; i < 3; ++i) {
        if ((rc = get_units_map(&m[4 + 2 * i], outs[i], dtype, 1, rows, D, kRows, 1))) return rc;
        if ((rc = get_units_map(&m[5 + 2 * i], outs[i], dtype, 1, rows, D, 16, 1))) return rc;
      }
    } else {   // q = packed qkv [N][L][3][h][d], dout [N][L][h][d], dq = packed dqkv
      if ((rc = get_tokens_map(&m[1], qkv + hdb, dtype, N, L, 3, g.heads, D, L))) return rc;
      if ((rc = get_tokens_map(&m[2], qkv + 2 * hdb, dtype, N, L, 3, g.heads, D, L))) return rc;
      const int big = std::min(kRows, L);
      if ((rc = get_tokens_map(&m[6], dqkv + hdb, dtype, N, L, 3, g.heads, D, big))) return rc;
      if ((rc = get_tokens_map(&m[7], dqkv + hdb, dtype, N, L, 3, g.heads, D, 16))) return rc;
      if ((rc = get_tokens_map(&m[8], dqkv + 2 * hdb, dtype, N, L, 3, g.heads, D, big))) return rc;
      if ((rc = get_tokens_map(&m[9], dqkv + 2 * hdb, dtype, N, L, 3, g.heads, D, 16))) return rc;
      m[0] = m[3] = m[4] = m[5] = m[1];   // unused: Q / dO / dQ go through per-segment maps
    }
    FlatBAdd fa{g.add_table, g.heads, g.add_nw, ws, 1, 0, 0};
    if (add) {
      if constexpr (D != 32) return fail(FWA_ERR_CAPACITY, "flat backward: bias/mask need d = 32");
      if (!fa.table) return fail(FWA_ERR_SHAPE, "flat backward: bias/mask given without the add table");
    }
    GradOut go;
    if (fm.tok) {
      uint8_t* base = static_cast<uint8_t*>(dq);
      go = GradOut{base, base + hdb, base + 2 * hdb, 3};
    } else {
      go = GradOut{static_cast<uint8_t*>(dq), static_cast<uint8_t*>(dk), static_cast<uint8_t*>(dv), 1};
    }
    const int grid = bflat_grid(g);
    if (want_db) {
      fa.slice_heads = bflat_slice_heads(fm, g.units, grid);
      fa.half_parts = bflat_half_parts(g, grid, fa.slice_heads, DT<T>::id == FWA_BF16) ? 1 : 0;
      // every CTA's first `heads` units cover every (head, row) of its slice exactly once
      fa.lazy_init = (!fm.head_major && g.units / grid >= g.heads && !bflat_eager_zero()) ? 1 : 0;
    }
    if (!pc) {
      if ((rc = launch_bflat_kern<T, D, L, false>(g, m, fa, fm, NoRowMaps{}, go, add, want_db, grid, s))) return rc;
    } else {
      if constexpr (bflat_pc_built<D, L>()) {
        BwdPieceMaps pm;
        if (fm.tok) {
          if ((rc = get_row_maps(&pm.q, qkv, dtype, true, N, L, 3, g.heads, D))) return rc;
          if ((rc = get_row_maps(&pm.dout, dout, dtype, true, N, L, 1, g.heads, D))) return rc;
          if ((rc = get_row_maps(&pm.dq, dqkv, dtype, true, N, L, 3, g.heads, D))) return rc;
        } else {
          if ((rc = get_row_maps(&pm.q, q, dtype, false, g.units, L, 1, 1, D))) return rc;
          if ((rc = get_row_maps(&pm.dout, dout, dtype, false, g.units, L, 1, 1, D))) return rc;
          if ((rc = get_row_maps(&pm.dq, dq, dtype, false, g.units, L, 1, 1, D))) return rc;
        }
        if ((rc = launch_bflat_kern<T, D, L, true>(g, m, fa, fm, pm, go, add, want_db, grid, s))) return rc;
      } else {
        return fail(FWA_ERR_CAPACITY, "flat backward: no pieces build for this shape");
      }
    }
    if (want_db) {
      const int LL = L * L;
      const int64_t n = (int64_t)g.heads * LL;
      if (grid > 1024) return fail(FWA_ERR_CAPACITY, "flat backward: dBias reduce supports <= 1024 CTAs");
      const unsigned rgrid = (unsigned)((n / (fa.half_parts ? 8 : 4) + 31) / 32);
      if (fa.half_parts)
        bflat_dbias_reduce_kernel<__half><<<rgrid, dim3(32, 8), 0, s>>>(reinterpret_cast<const __half*>(ws), grid,
                                                                 g.units, fm, fa.slice_heads, LL, dbias);
      else
        bflat_dbias_reduce_kernel<float><<<rgrid, dim3(32, 8), 0, s>>>(ws, grid, g.units, fm, fa.slice_heads, LL,
                                                                dbias);
      if ((rc = check_cuda(cudaGetLastError(), "bflat_dbias_reduce_kernel launch"))) return rc;
      count_launch();
    }
    return FWA_OK;
  }
}

#define FWA_FLAT_LS(X) X(80) X(96) X(112) X(128) X(144) X(160) X(176) X(192) X(208) X(224) X(240) X(256)

template <typename T, int D>
int bflat_l(const Geom& g, int dtype, const void* q, const void* k, const void* v, const void* dout,
            const float* bias, const float* mask, void* dq, void* dk, void* dv, float* dbias,
            float* ws, cudaStream_t s, int layout) {
  switch (g.L) {
#define FWA_CASE(LL) \
  case LL: return launch_bflat_t<T, D, LL>(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s, layout);
    FWA_FLAT_LS(FWA_CASE)
#undef FWA_CASE
  }
  return fail(FWA_ERR_CAPACITY, "flat backward: unsupported L");
}

template <int D>
constexpr bool bfits_d(int L) {
  switch (L) {
#define FWA_CASE(LL) \
  case LL: return BFCfg<D, LL>::kFits;
    FWA_FLAT_LS(FWA_CASE)
#undef FWA_CASE
  }
  return false;
}

template <int D>
constexpr int bsmem_d(int L) {
  switch (L) {
#define FWA_CASE(LL) \
  case LL: return BFCfg<D, LL>::kSmem;
    FWA_FLAT_LS(FWA_CASE)
#undef FWA_CASE
  }
  return 0;
}

template <int D>
constexpr bool bpc_d(int L) {
  switch (L) {
#define FWA_CASE(LL) \
  case LL: return bflat_pc_built<D, LL>();
    FWA_FLAT_LS(FWA_CASE)
#undef FWA_CASE
  }
  return false;
}

bool bflat_disabled() {
  static const bool off = [] {
    const char* e = getenv("FWA_NO_FLAT");
    return e && e[0] == '1';
  }();
  return off;
}

}  // namespace

bool tc_bwd_flat_supported(const Geom& g, int dtype, bool has_bias, bool has_mask, bool want_dbias) {
  if (bflat_disabled()) return false;
  if (want_dbias && !has_bias) return false;
  // bias/mask variants are built for d = 32 (Swin); with dBias, the rows of one 128-row block
  // must hit distinct [head][query] slices of the per-CTA partials (no two threads on one row)
  if ((has_bias || has_mask) && g.d != 32) return false;
  if (want_dbias && g.heads < 2 && g.L < 128) return false;
  if (dtype != FWA_F16 && dtype != FWA_BF16) return false;
  if (g.L <= 64 || g.L > 256 || g.L % 16 != 0) return false;
  if (g.units * (int64_t)g.L >= ((int64_t)1 << 31)) return false;
  switch (g.d) {
    case 16: return bfits_d<16>(g.L);
    case 32: return bfits_d<32>(g.L);
    case 64: return bfits_d<64>(g.L);
  }
  return false;
}

size_t tc_bwd_flat_smem(const Geom& g) {
  switch (g.d) {
    case 16: return bsmem_d<16>(g.L);
    case 32: return bsmem_d<32>(g.L);
    case 64: return bsmem_d<64>(g.L);
  }
  return 0;
}

size_t tc_bwd_flat_workspace_bytes(const Geom& g) {
  // dBias partials: [grid][slice_heads][L][L] fp32 (head-major walk: 1-2 heads per CTA)
  const int grid = bflat_grid(g);
  const FlatMap fm = bflat_map(g, true, false);
  const int sh = bflat_slice_heads(fm, g.units, grid);
  return (size_t)grid * sh * g.L * g.L * (bflat_half_parts(g, grid, sh, false) ? 2 : 4);
}

bool tc_bwd_flat_tokens_supported(const Geom& g, int dtype, bool has_bias, bool has_mask,
                                  bool want_dbias) {
  if (!tc_bwd_flat_supported(g, dtype, has_bias, has_mask, want_dbias)) return false;
  return g.d == 32 && bpc_d<32>(g.L);
}

int launch_bwd_tc_flat(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                       const void* dout, const float* bias, const float* mask, void* dq, void* dk,
                       void* dv, float* dbias, float* ws, cudaStream_t s, int layout) {
  const bool bf = dtype == FWA_BF16;
  switch (g.d) {
    case 16: return bf ? bflat_l<__nv_bfloat16, 16>(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s, layout)
                       : bflat_l<__half, 16>(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s, layout);
    case 32: return bf ? bflat_l<__nv_bfloat16, 32>(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s, layout)
                       : bflat_l<__half, 32>(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s, layout);
    case 64: return bf ? bflat_l<__nv_bfloat16, 64>(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s, layout)
                       : bflat_l<__half, 64>(g, dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, ws, s, layout);
  }
  return fail(FWA_ERR_CAPACITY, "flat backward: unsupported head_dim");
}

}  // namespace fwa
