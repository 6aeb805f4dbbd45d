// placeholder: tcgen05 path (filled in next)
#include "ss_common.cuh"
#include "ss_internal.h"
namespace ss {
bool topk_tc_supported(const TopkArgs&) { return false; }
int topk_tc_slices(const TopkArgs&, int) { return 1; }
int launch_topk_tc(const TopkArgs&, uint64_t*, int, cudaStream_t) {
  return set_error(SS_ERR_UNSUPPORTED, "tcgen05 path not built");
}
}  // namespace ss
