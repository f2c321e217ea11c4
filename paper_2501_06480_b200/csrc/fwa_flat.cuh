// fwa_flat.cuh — unit walk order and row addressing shared by the flat-row large-window
// kernels (fwa_tc_flat.cu, fwa_tc_flat_bwd.cu).
//
// A CTA walks a contiguous range of *virtual* units in 128-row blocks that straddle unit
// boundaries. A virtual unit v names one (window n, head hd) unit:
//   unit-major (default)  v = n * heads + hd   (= the physical unit of [N][h][L][d])
//   head-major            v = hd * N + n       (a CTA's range covers 1-2 heads: the dBias
//                                               backward keeps a [2][L][L] partial per CTA
//                                               instead of [heads][L][L])
// and rows are addressed either in the flat [units * L][d] row matrix of [N][h][L][d]
// (3-D tensor maps (d, rows, 1)) or in a token-major tensor [N][L][S][h][d] (the packed
// qkv-Linear output, S = 3, or the proj-Linear input, S = 1; 4-D maps (d, h, L, N)).
// When virtual rows are not contiguous in memory (head-major or token-major: "pieces"),
// a 128-row block moves as one TMA box per unit segment it holds (<= 2 for L >= 128), the
// box height picked from a set of maps with 16, 32, ..., 128-row boxes (L % 16 == 0 keeps
// every segment a multiple of 16 rows). Measured: per-16-row boxes made the L = 144
// forward 1.8x slower than one 128-row box (TMA op cost, not bytes).
#pragma once

#include <type_traits>

#include "fwa_sm100.cuh"

namespace fwa {

struct FlatMap {
  int tok;         // 1: token-major 4-D maps; 0: flat [units * L][d] 3-D maps
  int head_major;  // virtual unit order (see above)
  int heads;       // h
  int n_win;       // N (windows)
};

// FWA_FLAT_PIECES=1: force the pieces addressing on the plain layout (A/B timing)
bool flat_force_pieces();

__device__ __forceinline__ void vunit_nh(const FlatMap& m, int v, int& n, int& hd) {
  if (m.head_major) {
    hd = v / m.n_win;
    n = v - hd * m.n_win;
  } else {
    n = v / m.heads;
    hd = v - n * m.heads;
  }
}

// TMA load / store of the box at rows [i, i + box) of unit (n, hd)
template <int L>
__device__ __forceinline__ void ld_unit_rows(void* dst, const CUtensorMap* m, uint64_t* bar,
                                             const FlatMap& fm, int n, int hd, int i,
                                             uint64_t pol) {
  if (fm.tok)
    sm100::tma_load_4d(dst, m, bar, 0, hd, i, n, pol);
  else
    sm100::tma_load_3d(dst, m, bar, 0, (n * fm.heads + hd) * L + i, 0, pol);
}

__device__ __forceinline__ void tma_store_4d_hint(const CUtensorMap* m, const void* src, int c0,
                                                  int c1, int c2, int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint"
      " [%0, {%2, %3, %4, %5}], [%1], %6;" ::"l"(reinterpret_cast<uint64_t>(m)),
      "r"(sm100::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
      : "memory");
}

template <int L, bool HINT>
__device__ __forceinline__ void st_unit_rows(const CUtensorMap* m, const void* src,
                                             const FlatMap& fm, int n, int hd, int i,
                                             uint64_t pol) {
  if (fm.tok) {
    if constexpr (HINT) tma_store_4d_hint(m, src, 0, hd, i, n, pol);
    else sm100::tma_store_4d(m, src, 0, hd, i, n);
  } else {
    const int row = (n * fm.heads + hd) * L + i;
    if constexpr (HINT) sm100::tma_store_3d_hint(m, src, 0, row, 0, pol);
    else sm100::tma_store_3d(m, src, 0, row, 0);
  }
}

// Tensor maps of one operand with 16, 32, ..., 128-row boxes (pieces mode)
struct RowMaps {
  CUtensorMap m[8];
};
struct NoRowMaps {};

// Walks the unit segments of virtual rows [rs, rs + nrows) (nrows % 16 == 0):
// op(n, hd, i, off, len) for rows [i, i + len) of unit (n, hd) at block row off.
// One division per call; the loop only increments.
template <int L, typename Op>
__device__ __forceinline__ void for_segments(const FlatMap& fm, int rs, int nrows, Op&& op) {
  const int v = rs / L;
  int i = rs - v * L, n, hd;
  vunit_nh(fm, v, n, hd);
  for (int off = 0; off < nrows;) {
    const int len = min(L - i, nrows - off);
    op(n, hd, i, off, len);
    off += len;
    i = 0;   // next virtual unit
    if (fm.head_major) {
      if (++n == fm.n_win) { n = 0; ++hd; }
    } else {
      if (++hd == fm.heads) { hd = 0; ++n; }
    }
  }
}

// Virtual rows [rs, rs + nrows) (nrows <= 128): load into dst (rows consecutive) ...
template <int L, int RB>
__device__ __forceinline__ void ld_segments(uint8_t* dst, const RowMaps& rm, uint64_t* bar,
                                            const FlatMap& fm, int rs, int nrows, uint64_t pol) {
  for_segments<L>(fm, rs, nrows, [&](int n, int hd, int i, int off, int len) {
    ld_unit_rows<L>(dst + off * RB, &rm.m[len / 16 - 1], bar, fm, n, hd, i, pol);
  });
}
// prefetch the descriptors those segment boxes will use (hides a descriptor-cache miss
// behind the barrier wait that precedes the copy)
template <int L>
__device__ __forceinline__ void prefetch_segments(const RowMaps& rm, const FlatMap& fm, int rs,
                                                  int nrows) {
  for_segments<L>(fm, rs, nrows, [&](int, int, int, int, int len) {
    sm100::tma_prefetch_desc(&rm.m[len / 16 - 1]);
  });
}
// ... or store them from src
template <int L, int RB, bool HINT>
__device__ __forceinline__ void st_segments(const RowMaps& rm, const uint8_t* src,
                                            const FlatMap& fm, int rs, int nrows, uint64_t pol) {
  for_segments<L>(fm, rs, nrows, [&](int n, int hd, int i, int off, int len) {
    st_unit_rows<L, HINT>(&rm.m[len / 16 - 1], src + off * RB, fm, n, hd, i, pol);
  });
}

// Byte offset of row i of unit (n, hd): flat [units][L] rows or token-major rows of S x h
// slots (the drain's direct global stores)
template <int L>
__device__ __forceinline__ int64_t unit_row_offset(const FlatMap& fm, int n, int hd, int i, int S,
                                                   int row_bytes) {
  if (fm.tok) return ((int64_t)(n * L + i) * S * fm.heads + hd) * row_bytes;
  return ((int64_t)(n * fm.heads + hd) * L + i) * row_bytes;
}

// 16-byte global store, optionally with an L2 eviction-priority hint
template <bool HINT>
__device__ __forceinline__ void st_global_v4(void* p, uint4 v, uint64_t pol) {
  if constexpr (HINT)
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
  else
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// Heads spanned by the virtual units [ua, ub) (their dBias partial slices)
__host__ __device__ inline void range_heads(const FlatMap& fm, int64_t ua, int64_t ub, int& h0,
                                            int& h1) {
  if (fm.head_major) {
    h0 = (int)(ua / fm.n_win);
    h1 = (int)((ub - 1) / fm.n_win);
  } else {
    h0 = 0;
    h1 = fm.heads - 1;
  }
}

}  // namespace fwa
