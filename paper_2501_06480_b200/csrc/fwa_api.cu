// fwa_api.cu — the C-ABI (include/fwa.h): validation, kernel selection, errors.
//
// Validation mirrors the reference's checks and their order so the Python
// layer can raise the same exception classes:
//   TileConfig.__post_init__      flash.py:49-55   -> FWA_ERR_INVALID_RANGE
//   TileConfig.chunk_width        flash.py:57-66   -> FWA_ERR_SHAPE
//   _check_qkv_2d / dO shape      flash.py:322-327, :202-203 -> FWA_ERR_SHAPE
//   _check_budget (before work)   flash.py:98-103  -> FWA_ERR_CAPACITY
#include <math.h>
#include <stdio.h>

#include <atomic>
#include <mutex>
#include <string>

#include <algorithm>
#include <map>
#include <utility>

#include "fwa_common.cuh"

namespace fwa {

__device__ unsigned int g_fwa_device_flags = 0;
static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}
int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FWA_OK;
  return fail(FWA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
struct DevInfo {
  int sm = 0;
  int64_t l2 = 0;
  size_t smem_optin = 0;
};
DevInfo query_dev(int dev) {
  DevInfo d;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) d.sm = v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) == cudaSuccess) d.l2 = v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess)
    d.smem_optin = (size_t)v;
  return d;
}
// Per-device caches (a process may drive several GPUs, or call from several threads):
// device attributes, the function attributes already raised on each device, and the
// address of the device-side error word. All behind one mutex; a lookup costs a lock.
constexpr int kMaxDevices = 64;
std::mutex g_dev_mu;
DevInfo g_dev_info[kMaxDevices];
bool g_dev_known[kMaxDevices] = {};
unsigned int* g_flags_ptr[kMaxDevices] = {};
std::map<std::pair<int, const void*>, int>& smem_attrs() {
  static std::map<std::pair<int, const void*>, int> m;
  return m;
}
int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}
DevInfo dev_info() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_dev_known[dev]) {
    g_dev_info[dev] = query_dev(dev);
    g_dev_known[dev] = true;
  }
  return g_dev_info[dev];
}
}  // namespace

int ensure_smem_attr(const void* func, int bytes, const char* what) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  int& have = smem_attrs()[{dev, func}];
  if (have >= bytes) return FWA_OK;
  const int rc = check_cuda(
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), what);
  if (rc == FWA_OK) have = bytes;
  return rc;
}

int device_sm_count() { return dev_info().sm > 0 ? dev_info().sm : 148; }
int64_t device_l2_bytes() { return dev_info().l2; }
size_t device_max_smem_optin() {
  return dev_info().smem_optin ? dev_info().smem_optin : (size_t)227 * 1024;
}

namespace {

int64_t paper_peak(int L, int C, int cw, int eb, bool bwd) {
  return ((bwd ? 2 : 1) * (int64_t)L * L + 2 * (int64_t)L * cw) * eb;
}

// Reference-ordered validation; fills g and picks kernels. No device work.
int validate(const fwa_desc* d, Geom* g, bool need_mask_windows_if_mask, const float* mask) {
  if (!d) return fail(FWA_ERR_SHAPE, "null descriptor");
  if (d->dtype != FWA_F32 && d->dtype != FWA_F16 && d->dtype != FWA_BF16)
    return fail(FWA_ERR_INVALID_RANGE, "dtype must be FWA_F32, FWA_F16 or FWA_BF16");
  if (d->chunks < 1)
    return fail(FWA_ERR_INVALID_RANGE, "chunk count must be >= 1, got " + std::to_string(d->chunks));
  if (!isfinite(d->scale) || d->scale <= 0.f)
    return fail(FWA_ERR_INVALID_RANGE, "scale must be finite and > 0");
  if (d->num_windows < 1 || d->heads < 1 || d->seq_len < 1 || d->head_dim < 1)
    return fail(FWA_ERR_SHAPE, "N, heads, L and d must all be >= 1 (got N=" +
                                   std::to_string(d->num_windows) + ", h=" +
                                   std::to_string(d->heads) + ", L=" + std::to_string(d->seq_len) +
                                   ", d=" + std::to_string(d->head_dim) + ")");
  const int C = d->head_dim, r = d->chunks;
  if (r > C)
    return fail(FWA_ERR_SHAPE, "chunk count " + std::to_string(r) + " exceeds feature count " +
                                   std::to_string(C));
  const int cw = (C + r - 1) / r;
  if ((int64_t)cw * (r - 1) >= C)
    return fail(FWA_ERR_SHAPE, "chunk count " + std::to_string(r) +
                                   " leaves an empty chunk for " + std::to_string(C) + " features");
  if (need_mask_windows_if_mask && mask && d->mask_windows < 1)
    return fail(FWA_ERR_SHAPE, "mask given but mask_windows < 1");
  if (d->kernel < FWA_KERNEL_AUTO || d->kernel > FWA_KERNEL_TC)
    return fail(FWA_ERR_INVALID_RANGE, "unknown kernel selector");
  g->units = d->num_windows * d->heads;
  g->heads = d->heads;
  g->L = d->seq_len;
  g->d = d->head_dim;
  g->scale = d->scale;
  g->mask_windows = mask ? d->mask_windows : 1;
  return FWA_OK;
}

int pick_fwd(const fwa_desc* d, const Geom& g, bool has_bias, bool has_mask, int* kernel,
             size_t* smem, int* tmem) {
  const bool tc_small = tc_fwd_supported(g, d->dtype, has_bias, has_mask);
  const bool tc_large = !tc_small && tc_fwd_large_supported(g, d->dtype, has_bias, has_mask);
  const bool tc_ok = tc_small || tc_large;
  if (d->kernel == FWA_KERNEL_TC && !tc_ok)
    return fail(FWA_ERR_CAPACITY, "tcgen05 forward does not support this shape/dtype (L=" +
                                      std::to_string(g.L) + ", d=" + std::to_string(g.d) + ")");
  if (tc_ok && d->kernel != FWA_KERNEL_GENERIC) {
    *kernel = FWA_KERNEL_TC;
    *smem = tc_small ? tc_fwd_smem(g, d->dtype) : tc_fwd_large_smem(g);
    *tmem = tc_small ? tc_fwd_tmem_cols(g)
                     : (tc_fwd_flat_supported(g, d->dtype, has_bias, has_mask) ? 512 : 256);
    return FWA_OK;
  }
  *kernel = FWA_KERNEL_GENERIC;
  *smem = fwd_generic_smem(g);
  *tmem = 0;
  if (*smem > device_max_smem_optin())
    return fail(FWA_ERR_CAPACITY, "forward pass needs " + std::to_string(*smem) +
                                      " bytes of shared memory, device provides " +
                                      std::to_string(device_max_smem_optin()));
  return FWA_OK;
}

int pick_bwd(const fwa_desc* d, const Geom& g, bool has_bias, bool has_mask, bool want_dbias,
             int* kernel, size_t* smem, int* tmem) {
  const bool tc_small = tc_bwd_supported(g, d->dtype, has_bias, has_mask, want_dbias);
  const bool tc_large =
      !tc_small && tc_bwd_large_supported(g, d->dtype, has_bias, has_mask, want_dbias);
  const bool tc_ok = tc_small || tc_large;
  if (d->kernel == FWA_KERNEL_TC && !tc_ok)
    return fail(FWA_ERR_CAPACITY, "tcgen05 backward does not support this shape/dtype (L=" +
                                      std::to_string(g.L) + ", d=" + std::to_string(g.d) + ")");
  if (tc_ok && d->kernel != FWA_KERNEL_GENERIC) {
    *kernel = FWA_KERNEL_TC;
    *smem = tc_small ? tc_bwd_smem(g) : tc_bwd_large_smem(g);
    *tmem = tc_small ? tc_bwd_tmem_cols(g) : 512;
    return FWA_OK;
  }
  *kernel = FWA_KERNEL_GENERIC;
  *smem = bwd_generic_smem(g);
  *tmem = 0;
  if (*smem > device_max_smem_optin())
    return fail(FWA_ERR_CAPACITY, "backward pass needs " + std::to_string(*smem) +
                                      " bytes of shared memory, device provides " +
                                      std::to_string(device_max_smem_optin()));
  return FWA_OK;
}

// The large-window (flat) kernels read bias/mask through one f16 (bias + mask) * log2e
// table [n_w][h][L][L]; the L <= 64 and SIMT kernels read the fp32 bias/mask directly.
bool fwd_uses_table(const fwa_desc* d, const Geom& g, bool has_bias, bool has_mask) {
  if (!(has_bias || has_mask) || d->kernel == FWA_KERNEL_GENERIC) return false;
  if (tc_fwd_supported(g, d->dtype, has_bias, has_mask)) return false;
  return tc_fwd_flat_supported(g, d->dtype, has_bias, has_mask);
}
bool bwd_uses_table(const fwa_desc* d, const Geom& g, bool has_bias, bool has_mask, bool want_dbias) {
  if (!(has_bias || has_mask) || d->kernel == FWA_KERNEL_GENERIC) return false;
  if (tc_bwd_supported(g, d->dtype, has_bias, has_mask, want_dbias)) return false;
  return tc_bwd_flat_supported(g, d->dtype, has_bias, has_mask, want_dbias);
}
// dBias partials of the kernel pick_bwd chooses (0 without dBias)
size_t dbias_partial_bytes(const fwa_desc* d, const Geom& g, bool has_bias, bool has_mask,
                           bool want_dbias) {
  if (!want_dbias) return 0;
  int kern = 0, tmem = 0;
  size_t smem = 0;
  if (pick_bwd(d, g, has_bias, has_mask, true, &kern, &smem, &tmem) != FWA_OK) return 0;
  if (kern == FWA_KERNEL_GENERIC)
    return (size_t)bwd_generic_grid(g) * g.heads * g.L * g.L * sizeof(float);
  if (tc_bwd_supported(g, d->dtype, has_bias, has_mask, true))
    return tc_bwd_workspace_bytes(g, has_mask, true);
  return tc_bwd_flat_workspace_bytes(g);
}
size_t round256(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace
}  // namespace fwa

using namespace fwa;

extern "C" const char* fwa_last_error(void) { return g_last_error.c_str(); }
extern "C" int fwa_abi_version(void) { return FWA_ABI_VERSION; }
extern "C" int64_t fwa_launch_count(void) { return g_launches.load(); }

namespace fwa {
unsigned int* device_flags_ptr() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_flags_ptr[dev]) {
    void* a = nullptr;
    if (cudaGetSymbolAddress(&a, g_fwa_device_flags) == cudaSuccess)
      g_flags_ptr[dev] = (unsigned int*)a;
  }
  return g_flags_ptr[dev];
}
}  // namespace fwa

extern "C" int fwa_device_flags(uint32_t* flags) {
  unsigned int v = 0;
  int rc = check_cuda(cudaMemcpyFromSymbol(&v, g_fwa_device_flags, sizeof(v)), "fwa_device_flags");
  if (flags) *flags = v;
  return rc;
}

extern "C" int fwa_device_info(int32_t* sm_count, int64_t* l2_bytes) {
  if (sm_count) *sm_count = device_sm_count();
  if (l2_bytes) *l2_bytes = device_l2_bytes();
  return FWA_OK;
}

extern "C" int fwa_footprint(const fwa_desc* desc, fwa_footprint_t* out) {
  Geom g;
  int rc = validate(desc, &g, false, nullptr);
  if (rc) return rc;
  if (!out) return fail(FWA_ERR_SHAPE, "null footprint output");
  const int eb = elem_bytes(desc->dtype);
  const int cw = (g.d + desc->chunks - 1) / desc->chunks;
  out->paper_peak_fwd = paper_peak(g.L, g.d, cw, eb, false);
  out->paper_peak_bwd = paper_peak(g.L, g.d, cw, eb, true);
  const int64_t lcd = g.units * g.L * (int64_t)g.d * eb;
  out->hbm_bytes_fwd = 4 * lcd;
  out->hbm_bytes_bwd = 7 * lcd;
  size_t smem = 0;
  int kern = 0, tmem = 0;
  rc = pick_fwd(desc, g, false, false, &kern, &smem, &tmem);
  if (rc) return rc;
  out->kernel_fwd = kern;
  out->smem_bytes_fwd = (int64_t)smem;
  out->tmem_cols_fwd = tmem;
  rc = pick_bwd(desc, g, false, false, false, &kern, &smem, &tmem);
  if (rc) return rc;
  out->kernel_bwd = kern;
  out->smem_bytes_bwd = (int64_t)smem;
  out->tmem_cols_bwd = tmem;
  return FWA_OK;
}

// Resolve the add table of a flat-kernel call: the caller's prebuilt desc->add_table, else
// built into the head of `workspace`. Returns the workspace bytes it used.
static int resolve_table(const fwa_desc* desc, Geom* g, const float* bias, const float* mask,
                         void* workspace, size_t workspace_bytes, size_t* used, cudaStream_t s) {
  *used = 0;
  g->add_nw = mask ? std::max(1, desc->mask_windows) : 1;
  if (desc->add_table) {
    g->add_table = static_cast<const __half*>(desc->add_table);
    return FWA_OK;
  }
  const size_t need = round256(flat_add_table_bytes(*g, mask != nullptr));
  if (!workspace || workspace_bytes < need)
    return fail(FWA_ERR_CAPACITY, "bias/mask on the large-window kernels need " +
                                      std::to_string(need) + " workspace bytes (add table), got " +
                                      std::to_string(workspace ? workspace_bytes : 0));
  int rc = flat_build_add_table(*g, bias, mask, static_cast<__half*>(workspace), s);
  if (rc) return rc;
  g->add_table = static_cast<const __half*>(workspace);
  *used = need;
  return FWA_OK;
}

extern "C" int fwa_fwd(const fwa_desc* desc, const void* q, const void* k, const void* v,
                       const float* bias, const float* mask, void* o, void* workspace,
                       size_t workspace_bytes, void* stream) {
  Geom g;
  int rc = validate(desc, &g, true, mask);
  if (rc) return rc;
  if (!q || !k || !v || !o) return fail(FWA_ERR_SHAPE, "null q/k/v/o pointer");
  int kern = 0, tmem = 0;
  size_t smem = 0;
  rc = pick_fwd(desc, g, bias != nullptr, mask != nullptr, &kern, &smem, &tmem);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (fwd_uses_table(desc, g, bias != nullptr, mask != nullptr)) {
    size_t used = 0;
    if ((rc = resolve_table(desc, &g, bias, mask, workspace, workspace_bytes, &used, s))) return rc;
  }
  if (kern == FWA_KERNEL_TC) {
    if (tc_fwd_supported(g, desc->dtype, bias != nullptr, mask != nullptr))
      return launch_fwd_tc(g, desc->dtype, q, k, v, bias, mask, o, s);
    return launch_fwd_tc_large(g, desc->dtype, q, k, v, bias, mask, o, s);
  }
  return launch_fwd_generic(g, desc->dtype, q, k, v, bias, mask, o, s);
}

extern "C" size_t fwa_add_table_bytes(const fwa_desc* desc, int has_bias, int has_mask) {
  Geom g;
  if (validate(desc, &g, false, nullptr)) return 0;
  g.mask_windows = has_mask ? std::max(1, desc->mask_windows) : 1;
  if (!fwd_uses_table(desc, g, has_bias, has_mask) &&
      !bwd_uses_table(desc, g, has_bias, has_mask, false) &&
      !bwd_uses_table(desc, g, has_bias, has_mask, has_bias))
    return 0;
  return round256(flat_add_table_bytes(g, has_mask));
}

extern "C" int fwa_build_add_table(const fwa_desc* desc, const float* bias, const float* mask,
                                   void* table, size_t table_bytes, void* stream) {
  Geom g;
  int rc = validate(desc, &g, true, mask);
  if (rc) return rc;
  if (!bias && !mask) return fail(FWA_ERR_SHAPE, "add table needs a bias or a mask");
  const size_t need = round256(flat_add_table_bytes(g, mask != nullptr));
  if (!table || table_bytes < need)
    return fail(FWA_ERR_CAPACITY, "add table needs " + std::to_string(need) + " bytes, got " +
                                      std::to_string(table ? table_bytes : 0));
  return flat_build_add_table(g, bias, mask, static_cast<__half*>(table), (cudaStream_t)stream);
}

extern "C" size_t fwa_fwd_workspace_bytes(const fwa_desc* desc, int has_bias, int has_mask) {
  Geom g;
  if (validate(desc, &g, false, nullptr)) return 0;
  g.mask_windows = has_mask ? std::max(1, desc->mask_windows) : 1;
  if (desc->add_table || !fwd_uses_table(desc, g, has_bias, has_mask)) return 0;
  return round256(flat_add_table_bytes(g, has_mask));
}

extern "C" size_t fwa_bwd_workspace_bytes(const fwa_desc* desc, int has_bias, int has_mask,
                                          int want_dbias) {
  Geom g;
  if (validate(desc, &g, false, nullptr)) return 0;
  g.mask_windows = has_mask ? std::max(1, desc->mask_windows) : 1;
  size_t b = 0;
  if (!desc->add_table && bwd_uses_table(desc, g, has_bias, has_mask, want_dbias))
    b = round256(flat_add_table_bytes(g, has_mask));
  return b + dbias_partial_bytes(desc, g, has_bias, has_mask, want_dbias);
}

extern "C" int fwa_bwd(const fwa_desc* desc, const void* q, const void* k, const void* v,
                       const void* dout, const float* bias, const float* mask, void* dq, void* dk,
                       void* dv, float* dbias, void* workspace, size_t workspace_bytes,
                       void* stream) {
  Geom g;
  int rc = validate(desc, &g, true, mask);
  if (rc) return rc;
  if (!q || !k || !v || !dout || !dq || !dk || !dv)
    return fail(FWA_ERR_SHAPE, "null q/k/v/dO/dq/dk/dv pointer");
  int kern = 0, tmem = 0;
  size_t smem = 0;
  rc = pick_bwd(desc, g, bias != nullptr, mask != nullptr, dbias != nullptr, &kern, &smem, &tmem);
  if (rc) return rc;
  const size_t need =
      fwa_bwd_workspace_bytes(desc, bias != nullptr, mask != nullptr, dbias != nullptr);
  if (need && (!workspace || workspace_bytes < need))
    return fail(FWA_ERR_CAPACITY, "backward workspace needs " + std::to_string(need) +
                                      " bytes, got " + std::to_string(workspace_bytes));
  cudaStream_t s = (cudaStream_t)stream;
  size_t used = 0;
  if (bwd_uses_table(desc, g, bias != nullptr, mask != nullptr, dbias != nullptr) &&
      (rc = resolve_table(desc, &g, bias, mask, workspace, workspace_bytes, &used, s)))
    return rc;
  float* parts = workspace ? reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + used)
                           : nullptr;
  if (kern == FWA_KERNEL_TC) {
    if (tc_bwd_supported(g, desc->dtype, bias != nullptr, mask != nullptr, dbias != nullptr))
      return launch_bwd_tc(g, desc->dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, parts, s);
    return launch_bwd_tc_large(g, desc->dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, parts, s);
  }
  return launch_bwd_generic(g, desc->dtype, q, k, v, dout, bias, mask, dq, dk, dv, dbias, parts, s);
}

// ---- token-major ("qkv") layout: fused with the Swin qkv / proj Linears ----------
// qkv: [N][L][3][h][d] (qkv-Linear output), o / dout: [N][L][h][d] (proj-Linear input),
// dqkv: [N][L][3][h][d]. tcgen05 kernels only: the tile kernels (L <= 64, d in {16,32,64})
// and the flat-row kernels in pieces mode (d = 32, L in {128, 144, 192, 256}), f16/bf16;
// other shapes return FWA_ERR_CAPACITY so the caller can fall back to fwa_fwd/fwa_bwd.
extern "C" int fwa_fwd_qkv(const fwa_desc* desc, const void* qkv, const float* bias,
                           const float* mask, void* o, void* workspace, size_t workspace_bytes,
                           void* stream) {
  Geom g;
  int rc = validate(desc, &g, true, mask);
  if (rc) return rc;
  if (!qkv || !o) return fail(FWA_ERR_SHAPE, "null qkv/o pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const bool hb = bias != nullptr, hm = mask != nullptr;
  if (desc->kernel != FWA_KERNEL_GENERIC && tc_fwd_supported(g, desc->dtype, hb, hm))
    return launch_fwd_tc(g, desc->dtype, qkv, nullptr, nullptr, bias, mask, o, s, kTokens);
  if (desc->kernel != FWA_KERNEL_GENERIC && tc_fwd_flat_tokens_supported(g, desc->dtype, hb, hm)) {
    size_t used = 0;
    if ((hb || hm) && (rc = resolve_table(desc, &g, bias, mask, workspace, workspace_bytes, &used, s)))
      return rc;
    return launch_fwd_tc_flat(g, desc->dtype, qkv, nullptr, nullptr, bias, mask, o, s, kTokens);
  }
  return fail(FWA_ERR_CAPACITY, "fused qkv layout needs a tcgen05 forward (L <= 64 with d in "
                                "{16,32,64}, or d = 32 with L in {128,144,192,256}; f16/bf16)");
}

extern "C" int fwa_bwd_qkv(const fwa_desc* desc, const void* qkv, const void* dout,
                           const float* bias, const float* mask, void* dqkv, float* dbias,
                           void* workspace, size_t workspace_bytes, void* stream) {
  Geom g;
  int rc = validate(desc, &g, true, mask);
  if (rc) return rc;
  if (!qkv || !dout || !dqkv) return fail(FWA_ERR_SHAPE, "null qkv/dO/dqkv pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const bool hb = bias != nullptr, hm = mask != nullptr, db = dbias != nullptr;
  const bool small = desc->kernel != FWA_KERNEL_GENERIC && tc_bwd_supported(g, desc->dtype, hb, hm, db);
  const bool flat = !small && desc->kernel != FWA_KERNEL_GENERIC &&
                    tc_bwd_flat_tokens_supported(g, desc->dtype, hb, hm, db);
  if (!small && !flat)
    return fail(FWA_ERR_CAPACITY, "fused qkv layout needs a tcgen05 backward (L <= 64 with d in "
                                  "{16,32,64}, or d = 32 with L in {128,144,192,256}; f16/bf16)");
  const size_t need = fwa_bwd_workspace_bytes(desc, hb, hm, db);
  if (need && (!workspace || workspace_bytes < need))
    return fail(FWA_ERR_CAPACITY, "backward workspace needs " + std::to_string(need) + " bytes");
  if (small)
    return launch_bwd_tc(g, desc->dtype, qkv, nullptr, nullptr, dout, bias, mask, dqkv, nullptr,
                         nullptr, dbias, (float*)workspace, s, kTokens);
  size_t used = 0;
  if ((hb || hm) && (rc = resolve_table(desc, &g, bias, mask, workspace, workspace_bytes, &used, s)))
    return rc;
  float* parts = workspace ? reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + used)
                           : nullptr;
  return launch_bwd_tc_flat(g, desc->dtype, qkv, nullptr, nullptr, dout, bias, mask, dqkv, nullptr,
                            nullptr, dbias, parts, s, kTokens);
}
