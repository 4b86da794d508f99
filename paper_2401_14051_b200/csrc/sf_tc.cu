// sf_tc.cu — tensor-core backbone (placeholder until the tcgen05 kernel lands).
#include "sf_internal.h"

namespace sfb {
bool tc_supported(const sf_backbone_config&) { return false; }
void tc_prepare(sf_backbone&, cudaStream_t) {}
void tc_release(sf_backbone&) {}
void launch_backbone_tc(const sf_backbone&, int64_t, const float*, const double*, float*, double*,
                        cudaStream_t) {
    fail(SF_ERR_INVALID_ARGUMENT, "bf16 tensor-core backbone not built");
}
}  // namespace sfb
