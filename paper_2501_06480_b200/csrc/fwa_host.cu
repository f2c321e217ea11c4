// fwa_host.cu — host helpers shared by the TMA kernels: tensor-map encode + cache, PDL launch.
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "fwa_common.cuh"
#include "fwa_flat.cuh"

namespace fwa {
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

struct MapKey {
  uintptr_t ptr;
  int64_t units;
  int32_t dtype, L, d, box_rows, box_units;
  int32_t kind, S, h;   // kind 0: [units][L][d] 3-D map; 1: token-major 4-D map (S, h)
  bool operator==(const MapKey& o) const { return std::memcmp(this, &o, sizeof(MapKey)) == 0; }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<uintptr_t>()(k.ptr);
    h ^= std::hash<int64_t>()(k.units) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h ^= (size_t)k.L * 1315423911u ^ (size_t)k.d * 2654435761u ^ (size_t)k.dtype ^
         ((size_t)k.box_rows << 20) ^ ((size_t)k.box_units << 28) ^ ((size_t)k.kind << 40) ^
         ((size_t)k.S << 44) ^ ((size_t)k.h << 48);
    return h;
  }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash>& map_cache() {
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> m;
  return m;
}

}  // namespace

// 3-D map over [units][L][d] (16-bit elements) with box (d, box_rows, box_units);
// swizzle = the row width (32/64/128 B) so the smem image is the UMMA canonical layout.
int get_units_map(CUtensorMap* out, const void* ptr, int dtype, int64_t units, int L, int d,
                  int box_rows, int box_units) {
  MapKey key;
  std::memset(&key, 0, sizeof(key));
  key.ptr = (uintptr_t)ptr;
  key.units = units;
  key.dtype = dtype;
  key.L = L;
  key.d = d;
  key.box_rows = box_rows;
  key.box_units = box_units;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = map_cache().find(key);
    if (it != map_cache().end()) {
      *out = it->second;
      return FWA_OK;
    }
  }
  EncodeFn enc = get_encode();
  if (!enc) return fail(FWA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t gdim[3] = {(cuuint64_t)d, (cuuint64_t)L, (cuuint64_t)units};
  const cuuint64_t gstride[2] = {(cuuint64_t)d * 2, (cuuint64_t)L * d * 2};
  const cuuint32_t box[3] = {(cuuint32_t)d, (cuuint32_t)box_rows, (cuuint32_t)box_units};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapSwizzle swz = d == 16   ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : d == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                           : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(out, dtype == FWA_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                          : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   3, const_cast<void*>(ptr), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(FWA_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> lk(g_map_mu);
  if (map_cache().size() > 1024) map_cache().clear();
  map_cache().emplace(key, *out);
  return FWA_OK;
}

// 4-D map over a token-major tensor [N][L][S][h][d] (S = 3 for packed qkv, 1 for O/dO)
// starting at `base` (already offset to the q/k/v slice): dims (d, h, L, N), box (d, 1, rows, 1).
int get_tokens_map(CUtensorMap* out, const void* base, int dtype, int64_t N, int L, int S, int h,
                   int d, int box_rows) {
  MapKey key;
  std::memset(&key, 0, sizeof(key));
  key.ptr = (uintptr_t)base;
  key.units = N;
  key.dtype = dtype;
  key.L = L;
  key.d = d;
  key.box_rows = box_rows;
  key.kind = 1;
  key.S = S;
  key.h = h;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = map_cache().find(key);
    if (it != map_cache().end()) {
      *out = it->second;
      return FWA_OK;
    }
  }
  EncodeFn enc = get_encode();
  if (!enc) return fail(FWA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t gdim[4] = {(cuuint64_t)d, (cuuint64_t)h, (cuuint64_t)L, (cuuint64_t)N};
  const cuuint64_t gstride[3] = {(cuuint64_t)d * 2, (cuuint64_t)S * h * d * 2,
                                 (cuuint64_t)L * S * h * d * 2};
  const cuuint32_t box[4] = {(cuuint32_t)d, 1, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUtensorMapSwizzle swz = d == 16   ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : d == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                           : CU_TENSOR_MAP_SWIZZLE_128B;
  // a token row holds one head's d features (32-128 B) between other heads / q, k, v:
  // promoting each row request to a 256 B L2 fetch pulls neighbours that are evicted again
  // before their own unit runs (measured: 2x the DRAM reads in the L = 144 backward)
  static const CUtensorMapL2promotion promo = [] {
    const char* e = getenv("FWA_TOK_PROMO");
    if (!e) return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    return e[0] == '2' ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
           : e[0] == '1' ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
           : e[0] == '6' ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  }();
  CUresult r = enc(out, dtype == FWA_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                          : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   4, const_cast<void*>(base), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(FWA_ERR_CUDA, "cuTensorMapEncodeTiled (token layout) failed (" +
                                  std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> lk(g_map_mu);
  if (map_cache().size() > 1024) map_cache().clear();
  map_cache().emplace(key, *out);
  return FWA_OK;
}

// Maps with 16, 32, ..., 128-row boxes of one operand (pieces mode of the flat kernels):
// flat rows of [units][L][d] (tok = false; N = units) or token-major [N][L][S][h][d].
int get_row_maps(RowMaps* out, const void* base, int dtype, bool tok, int64_t N, int L, int S,
                 int h, int d) {
  for (int k = 0; k < 8; ++k) {
    const int rows = 16 * (k + 1);
    int rc;
    if (rows > L) {
      out->m[k] = out->m[k > 0 ? k - 1 : 0];   // never used: segments are <= L rows
      continue;
    }
    if (tok)
      rc = get_tokens_map(&out->m[k], base, dtype, N, L, S, h, d, rows);
    else
      rc = get_units_map(&out->m[k], base, dtype, 1, (int)(N * L), d, rows, 1);
    if (rc) return rc;
  }
  return FWA_OK;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("FWA_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

}  // namespace fwa
