// fwa_common.cuh — shared device/host helpers for libfwa (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../../include/fwa.h"

namespace fwa {

// Device-side error flags (bit 0: a TMA kernel found its dynamic smem misaligned).
// Kernels get the address as an argument; read through fwa_device_flags().
unsigned int* device_flags_ptr();

// ---- dtype traits ---------------------------------------------------------
template <typename T> struct DT;
template <> struct DT<float> {
  static constexpr int id = FWA_F32;
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <> struct DT<__half> {
  static constexpr int id = FWA_F16;
  __device__ __forceinline__ static float to_f(__half x) { return __half2float(x); }
  __device__ __forceinline__ static __half from_f(float x) { return __float2half_rn(x); }
};
template <> struct DT<__nv_bfloat16> {
  static constexpr int id = FWA_BF16;
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

inline int elem_bytes(int dtype) { return dtype == FWA_F32 ? 4 : 2; }

// ---- host-side error plumbing ---------------------------------------------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);
void count_launch(int64_t n = 1);
// Raise a kernel's dynamic-smem limit once per (device, kernel); thread-safe.
int ensure_smem_attr(const void* func, int bytes, const char* what);

// Problem geometry shared by the kernels.
struct Geom {
  int64_t units;   // N * h
  int32_t heads;
  int32_t L;
  int32_t d;
  float scale;
  int32_t mask_windows;
  // large-window (flat) kernels with bias/mask: the (bias[h] + mask[w]) * log2e f16 table
  // [add_nw][heads][L][L] built by flat_build_add_table (caller-owned memory), else null
  const __half* add_table = nullptr;
  int32_t add_nw = 1;
};

// ---- kernel launchers (defined in the .cu files) --------------------------
int launch_fwd_generic(const Geom& g, int dtype, const void* q, const void* k,
                       const void* v, const float* bias, const float* mask,
                       void* o, cudaStream_t s);
size_t fwd_generic_smem(const Geom& g);

int launch_bwd_generic(const Geom& g, int dtype, const void* q, const void* k,
                       const void* v, const void* dout, const float* bias,
                       const float* mask, void* dq, void* dk, void* dv,
                       float* dbias, float* ws, cudaStream_t s);
size_t bwd_generic_smem(const Geom& g);
bool bwd_generic_fits(const Geom& g);
int bwd_generic_grid(const Geom& g);

// tcgen05 / TMA forward (fwa_tc_fwd.cu)
bool tc_fwd_supported(const Geom& g, int dtype, bool has_bias, bool has_mask);
size_t tc_fwd_smem(const Geom& g, int dtype);
int tc_fwd_tmem_cols(const Geom& g);
int launch_fwd_tc(const Geom& g, int dtype, const void* q, const void* k,
                  const void* v, const float* bias, const float* mask, void* o,
                  cudaStream_t s, int layout = 0);

// fwa_host.cu: cached 3-D tensor map over [units][L][d] 16-bit data
int get_units_map(CUtensorMap* out, const void* ptr, int dtype, int64_t units, int L, int d,
                  int box_rows, int box_units);

// 4-D map over a token-major [N][L][S][h][d] tensor (fused qkv / proj layouts).
int get_tokens_map(CUtensorMap* out, const void* base, int dtype, int64_t N, int L, int S, int h,
                   int d, int box_rows);

// 8 maps with 16..128-row boxes of one operand (fwa_flat.cuh RowMaps; pieces mode)
struct RowMaps;
int get_row_maps(RowMaps* out, const void* base, int dtype, bool tok, int64_t N, int L, int S,
                 int h, int d);

// Operand layout of the TMA kernels: kUnits = [N][h][L][d] (the reference's batched
// layout); kTokens = token-major, read from the packed qkv-Linear output [N][L][3][h][d]
// and written as [N][L][h][d] (= the proj-Linear input): no permute copies.
enum Layout { kUnits = 0, kTokens = 1 };
struct LayoutArgs {
  int mode;   // Layout
  int heads;  // h (kTokens: unit u = (u / h, u % h))
};

// FWA_NO_PDL=1 in the environment disables PDL (diagnostics).
bool pdl_enabled();

// Launch with programmatic dependent launch (PDL) enabled: the kernel must execute
// griddepcontrol.wait before touching global memory.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// tcgen05 / TMA forward for 64 < L <= 256 (fwa_tc_fwd_large.cu)
bool tc_fwd_large_supported(const Geom& g, int dtype, bool has_bias, bool has_mask);
size_t tc_fwd_large_smem(const Geom& g);
int launch_fwd_tc_large(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                        const float* bias, const float* mask, void* o, cudaStream_t s);

// flat-row forward for 64 < L <= 256, L % 16 == 0 (fwa_tc_flat.cu); taken by
// launch_fwd_tc_large when supported (FWA_NO_FLAT=1 disables it)
bool tc_fwd_flat_supported(const Geom& g, int dtype, bool has_bias, bool has_mask);
size_t tc_fwd_flat_smem(const Geom& g);
int launch_fwd_tc_flat(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                       const float* bias, const float* mask, void* o, cudaStream_t s, int layout = 0);
// token-major layout (fwa_fwd_qkv) on the flat forward: d = 32, L in {128, 144, 192, 256}
bool tc_fwd_flat_tokens_supported(const Geom& g, int dtype, bool has_bias, bool has_mask);

// (bias[h] + mask[w]) * log2e as f16 [n_w][h][L][L] (n_w = mask windows, or 1 without a
// mask) into caller-owned memory of flat_add_table_bytes(g, has_mask) bytes
size_t flat_add_table_bytes(const Geom& g, bool has_mask);
int flat_build_add_table(const Geom& g, const float* bias, const float* mask, __half* out,
                         cudaStream_t s);

// tcgen05 / TMA backward (fwa_tc_bwd.cu)
bool tc_bwd_supported(const Geom& g, int dtype, bool has_bias, bool has_mask, bool want_dbias);
size_t tc_bwd_smem(const Geom& g);
int tc_bwd_tmem_cols(const Geom& g);
size_t tc_bwd_workspace_bytes(const Geom& g, bool has_mask, bool want_dbias);
int launch_bwd_tc(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                  const void* dout, const float* bias, const float* mask, void* dq, void* dk,
                  void* dv, float* dbias, float* ws, cudaStream_t s, int layout = 0);

// tcgen05 / TMA backward for 64 < L <= 256 (fwa_tc_bwd_large.cu)
bool tc_bwd_large_supported(const Geom& g, int dtype, bool has_bias, bool has_mask, bool want_dbias);
size_t tc_bwd_large_smem(const Geom& g);
int launch_bwd_tc_large(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                        const void* dout, const float* bias, const float* mask, void* dq, void* dk,
                        void* dv, float* dbias, float* ws, cudaStream_t s);

// flat-row backward (fwa_tc_flat_bwd.cu); taken by launch_bwd_tc_large when supported
bool tc_bwd_flat_supported(const Geom& g, int dtype, bool has_bias, bool has_mask, bool want_dbias);
size_t tc_bwd_flat_smem(const Geom& g);
size_t tc_bwd_flat_workspace_bytes(const Geom& g);
int launch_bwd_tc_flat(const Geom& g, int dtype, const void* q, const void* k, const void* v,
                       const void* dout, const float* bias, const float* mask, void* dq, void* dk,
                       void* dv, float* dbias, float* ws, cudaStream_t s, int layout = 0);
// token-major layout (fwa_bwd_qkv) on the flat backward: d = 32, L in {128, 144, 192, 256}
bool tc_bwd_flat_tokens_supported(const Geom& g, int dtype, bool has_bias, bool has_mask,
                                  bool want_dbias);

int device_sm_count();
int64_t device_l2_bytes();
size_t device_max_smem_optin();

}  // namespace fwa
