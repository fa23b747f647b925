#include "kernels.cuh"
namespace nsg {
int launch_rss_rows(const nsg_spec&, const void*, void*, const void*, void*, int64_t, int64_t, cudaStream_t) {
  return fail(NSG_ERR_SPEC, "RSS not built yet");
}
int launch_rss_items(const nsg_spec&, void*, int64_t, int64_t, cudaStream_t) {
  return fail(NSG_ERR_SPEC, "RSS not built yet");
}
}  // namespace nsg
