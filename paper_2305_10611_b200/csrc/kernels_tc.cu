// kernels_tc.cu — tcgen05 tensor-core kernels for recognised plan shapes (in progress; plans
// without a tensor-core kernel run on the FP32 plan VM).
#include "tc.h"

namespace mbx {
void tc_prepare(mbx_ctx*, PlanEntry& pe) { pe.tc_kind = -1; }
cudaError_t tc_launch(mbx_ctx*, const PlanEntry&, const BatchLaunch&) { return cudaErrorNotSupported; }
void tc_release(PlanEntry&) {}
}  // namespace mbx
