#include "kernels.cuh"
namespace nsg {
size_t segments_ws_bytes(int64_t, int64_t) { return 0; }
int launch_segments(const nsg_spec&, const uint32_t*, int64_t, const void*, void*, const void*, void*, void*, size_t,
                    cudaStream_t) {
  return fail(NSG_ERR_SPEC, "segmented sort not built yet");
}
}  // namespace nsg
