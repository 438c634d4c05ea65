// k_large.cu -- placeholder until the tcgen05 kernel lands.
#include <cuda_runtime.h>

#include <string>

#include "mlpv_internal.cuh"

namespace mlpv {
cudaError_t prepare_large(const DevNet& net, const void* const* W_host, void** Wt_dev, std::string* why) {
  (void)net; (void)W_host; (void)Wt_dev;
  *why = "tcgen05 kernel not built yet";
  return cudaSuccess;
}
cudaError_t launch_large(const DevNet&, const void* const*, const void*, int, const DevPert&, const DevProp&,
                         const DevCov&, const DevResult&, BaseWS, const uint64_t*, int64_t, int, void*, int,
                         cudaStream_t, bool* supported, std::string* why) {
  *supported = false;
  *why = "tcgen05 kernel not built yet";
  return cudaSuccess;
}
}  // namespace mlpv
