/*
 * fwa.h — C-ABI of the B200-native Flash Window Attention library (libfwa.so).
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary.
 * Every device pointer is caller-owned: the library never allocates device
 * memory (scratch comes from the caller's `workspace`, sized by the
 * fwa_*_workspace_bytes queries) and never changes process-wide CUDA state
 * (memory pools, limits). Every call is stream-ordered on the `stream`
 * argument (a cudaStream_t passed as void*), re-entrant and thread-safe
 * (per-device caches behind a mutex), and returns an fwa_status.
 * On a non-zero status, fwa_last_error() returns a thread-local message.
 *
 * The reference (`flashwin`, pure Python) has no FFI; its "operator API" is
 * the Python signatures re-exported at pkg/src/flashwin/__init__.py:19-45.
 * Each entry point below names the reference interface it replaces. The
 * Python host layer (paper_2501_06480_b200/) binds these with ctypes and
 * mirrors the reference signatures on top.
 *
 * Layouts (row-major, contiguous):
 *   q, k, v, o, dO, dq, dk, dv : [num_windows][heads][seq_len][head_dim]
 *                                 (the reference's batched (B,h,L,C), flash.py:269-275)
 *   bias  (optional)           : float32 [heads][seq_len][seq_len]
 *   mask  (optional)           : float32 [mask_windows][seq_len][seq_len];
 *                                 window n uses mask[n % mask_windows]
 */
#ifndef FWA_H_
#define FWA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FWA_ABI_VERSION 2

/* Status codes. The Python layer maps them back onto the reference's
 * exception classes (pkg/src/flashwin/errors.py:4-33). */
typedef enum {
  FWA_OK = 0,
  FWA_ERR_SHAPE = 1,         /* ShapeError       (flash.py:322-327, :59-65, :202-203) */
  FWA_ERR_CAPACITY = 2,      /* CapacityError    (flash.py:98-103), raised before any work */
  FWA_ERR_INVALID_RANGE = 3, /* InvalidRangeError(flash.py:49-55, :287-288) */
  FWA_ERR_CONTEXT = 4,       /* ContextError     (flash.py:197-200) */
  FWA_ERR_CUDA = 5,          /* CUDA runtime / launch failure */
  FWA_ERR_PARTITION = 6      /* PartitionError   (windowing.py:35-39) */
} fwa_status;

typedef enum { FWA_F32 = 0, FWA_F16 = 1, FWA_BF16 = 2 } fwa_dtype;

/* Kernel selection. AUTO picks the tcgen05/TMA kernel when the shape and
 * dtype allow it, else the generic SIMT kernel (a GPU path, not a CPU one). */
typedef enum {
  FWA_KERNEL_AUTO = 0,
  FWA_KERNEL_GENERIC = 1,
  FWA_KERNEL_TC = 2
} fwa_kernel;

/* Problem descriptor: the reference's (B,h,L,C) + TileConfig (flash.py:41-55). */
typedef struct {
  int64_t num_windows;  /* N (B in the reference's batched API) */
  int32_t heads;        /* h */
  int32_t seq_len;      /* L = k*k */
  int32_t head_dim;     /* d (C per head in the reference) */
  int32_t dtype;        /* fwa_dtype of q/k/v/o/dO/dq/dk/dv */
  float scale;          /* TileConfig.scale: finite, > 0 */
  int32_t chunks;       /* TileConfig.r: feature chunks, validated like flash.py:57-66 */
  int32_t mask_windows; /* nW of the mask tensor; 0 when mask == NULL */
  int32_t kernel;       /* fwa_kernel */
  int32_t reserved;     /* 0 */
  /* Optional prebuilt score addend for the large-window kernels: the output of
   * fwa_build_add_table for this call's bias/mask (e.g. built once per layer and
   * shared by its forward and backward). NULL = built per call in `workspace`. */
  const void* add_table;
} fwa_desc;

/* Per-launch facts (analogue of peak_sram_forward/backward, flash.py:84-95,
 * reported for the kernel that would actually run). */
typedef struct {
  int32_t kernel_fwd;         /* fwa_kernel chosen for the forward */
  int32_t kernel_bwd;         /* fwa_kernel chosen for the backward */
  int64_t smem_bytes_fwd;     /* dynamic shared memory per CTA */
  int64_t smem_bytes_bwd;
  int32_t tmem_cols_fwd;      /* TMEM columns per CTA (0 for the SIMT kernel) */
  int32_t tmem_cols_bwd;
  int64_t paper_peak_fwd;     /* (L^2 + 2 L cw) * elem_bytes, flash.py:84-88 */
  int64_t paper_peak_bwd;     /* (2 L^2 + 2 L cw) * elem_bytes, flash.py:91-95 */
  int64_t hbm_bytes_fwd;      /* algorithmic: 4 * N*h*L*d * elem_bytes */
  int64_t hbm_bytes_bwd;      /* algorithmic: 7 * N*h*L*d * elem_bytes */
} fwa_footprint_t;

/* Window geometry: the reference's WindowConfig(H,W,C,k) (windowing.py:17-41)
 * plus a batch axis and Swin's cyclic shift (extension). */
typedef struct {
  int64_t batch;     /* B images */
  int32_t height;    /* H */
  int32_t width;     /* W */
  int32_t channels;  /* C */
  int32_t window;    /* k; must divide H and W, else FWA_ERR_PARTITION */
  int32_t shift;     /* cyclic shift s (0 = none); 0 <= s < k */
  int32_t elem_bytes;/* 1, 2, 4 or 8: the copy is bitwise */
} fwa_win_desc;

/* ---- hot path --------------------------------------------------------- */

/* Forward over all (window, head) units.
 * Replaces flash_forward (flash.py:141-184) and batched_flash_forward
 * (flash.py:269-319): O = softmax(scale*Q K^T [+ bias[h]] [+ mask[n % nW]]) V.
 * Validation (shape/range/capacity) completes before any work is enqueued.
 * `workspace` must hold fwa_fwd_workspace_bytes(desc, bias != NULL, mask != NULL)
 * bytes (NULL when that is 0: always for L <= 64 or without bias/mask). */
int fwa_fwd(const fwa_desc* desc, const void* q, const void* k, const void* v,
            const float* bias, const float* mask, void* o, void* workspace,
            size_t workspace_bytes, void* stream);

size_t fwa_fwd_workspace_bytes(const fwa_desc* desc, int has_bias, int has_mask);

/* Backward: recomputes P on chip (no O / LSE read), returns dQ, dK, dV and,
 * when dbias != NULL, dBias[h][L][L] = sum_n dS[n,h]. Replaces flash_backward
 * (flash.py:187-266). dBias is deterministic (bitwise repeatable): per-CTA
 * fp32 partials in `workspace`, each address accumulated in a fixed order
 * (the large-window kernel's vector L2 reductions are issued by one thread
 * per (block, row) and ordered block after block by the kernel's mbarriers),
 * then summed over CTAs in ascending order. `workspace` must hold
 * fwa_bwd_workspace_bytes(desc, bias != NULL, mask != NULL, dbias != NULL)
 * bytes (may be NULL when that is 0). */
int fwa_bwd(const fwa_desc* desc, const void* q, const void* k, const void* v,
            const void* dout, const float* bias, const float* mask, void* dq,
            void* dk, void* dv, float* dbias, void* workspace,
            size_t workspace_bytes, void* stream);

size_t fwa_bwd_workspace_bytes(const fwa_desc* desc, int has_bias, int has_mask,
                               int want_dbias);

/* The large-window kernels' score addend (bias[h] + mask[n % nW]) * log2e as f16
 * [nW][h][L][L]. fwa_add_table_bytes is 0 when no kernel of this shape reads it;
 * a table built once can be passed to the forward and backward of the same layer
 * through desc->add_table (saves one build per call). */
size_t fwa_add_table_bytes(const fwa_desc* desc, int has_bias, int has_mask);
int fwa_build_add_table(const fwa_desc* desc, const float* bias, const float* mask,
                        void* table, size_t table_bytes, void* stream);

/* Shape/budget query, no device work (peak_sram_forward/backward + _check_budget,
 * flash.py:84-103). Returns FWA_ERR_CAPACITY when no kernel can run the shape. */
int fwa_footprint(const fwa_desc* desc, fwa_footprint_t* out);

/* ---- fused layouts (no reference counterpart) ------- */

/* Same math as fwa_fwd, reading Q/K/V straight from the Swin qkv-Linear output
 * qkv [num_windows][seq_len][3][heads][head_dim] and writing O as
 * [num_windows][seq_len][heads][head_dim] (the proj-Linear input): the two
 * permute copies around window attention disappear. tcgen05 path only
 * (seq_len <= 64, head_dim in {16,32,64}, f16/bf16); FWA_ERR_CAPACITY otherwise. */
int fwa_fwd_qkv(const fwa_desc* desc, const void* qkv, const float* bias,
                const float* mask, void* o, void* workspace, size_t workspace_bytes,
                void* stream);

/* Backward in the same layouts: dout [N][L][h][d] -> dqkv [N][L][3][h][d]. */
int fwa_bwd_qkv(const fwa_desc* desc, const void* qkv, const void* dout,
                const float* bias, const float* mask, void* dqkv, float* dbias,
                void* workspace, size_t workspace_bytes, void* stream);

/* ---- window partition / reverse (windowing.py:44-70) ------------------ */

/* in [B][H][W][C] -> out [B*nW][k*k][C]; with shift s the image is first
 * rolled by (-s,-s) (Swin's cyclic shift). Bitwise copy. */
int fwa_window_partition(const fwa_win_desc* desc, const void* in, void* out,
                         void* stream);

/* Inverse: in [B*nW][k*k][C] -> out [B][H][W][C], then roll by (+s,+s). */
int fwa_window_reverse(const fwa_win_desc* desc, const void* in, void* out,
                       void* stream);

/* ---- Swin bias / mask helpers (extension, SPEC.md:14 excludes them upstream) */

/* table [(2k-1)^2][heads] float32 -> bias [heads][k*k][k*k] float32. */
int fwa_bias_gather(const float* table, int32_t window, int32_t heads,
                    float* bias, void* stream);

/* dbias [heads][L][L] -> dtable [(2k-1)^2][heads] (overwritten), summed in a
 * fixed order (deterministic). */
int fwa_bias_scatter(const float* dbias, int32_t window, int32_t heads,
                     float* dtable, void* stream);

/* Swin shifted-window mask [nW][L][L]: 0 within a region, `neg` across. */
int fwa_shift_mask(int32_t height, int32_t width, int32_t window, int32_t shift,
                   float neg, float* mask, void* stream);

/* ---- deterministic inputs (tensor.py:118-138) ------------------------- */

/* SplitMix64 fill: element i = lo + (hi-lo) * (mix(state + (i+1)*G) >> 11) * 2^-53,
 * computed in float64, then rounded f64 -> f32 -> dtype (round-to-nearest-even
 * at each step). Bit-identical to the CPU generator for the same state. */
int fwa_fill_uniform(uint64_t state, int64_t count, double lo, double hi,
                     int32_t dtype, void* out, void* stream);

/* ---- misc ------------------------------------------------------------- */
const char* fwa_last_error(void);
int fwa_abi_version(void);
/* Number of hot-path kernel launches this process has enqueued (bench's gpu_launches). */
int64_t fwa_launch_count(void);
/* Device-side error flags (synchronising read; 0 = healthy). */
int fwa_device_flags(uint32_t* flags);
/* Multiprocessor count and L2 bytes of the current device (for grid sizing / flushes). */
int fwa_device_info(int32_t* sm_count, int64_t* l2_bytes);

#ifdef __cplusplus
}
#endif

#endif /* FWA_H_ */
