// fwa_tc_fwd.cu — tcgen05/TMA forward (placeholder until the kernel lands).
#include "fwa_common.cuh"

namespace fwa {
bool tc_fwd_supported(const Geom&, int) { return false; }
size_t tc_fwd_smem(const Geom&, int) { return 0; }
int tc_fwd_tmem_cols(const Geom&) { return 0; }
int launch_fwd_tc(const Geom&, int, const void*, const void*, const void*, const float*,
                  const float*, void*, cudaStream_t) {
  return fail(FWA_ERR_CAPACITY, "tcgen05 forward not built");
}
}  // namespace fwa
