// tc.h — tensor-core (tcgen05) kernels for recognised plan shapes (kernels_tc.cu).
#pragma once
#include "ctx.h"

namespace mbx {
// Inspects a freshly compiled plan; if a tensor-core kernel implements it, packs what it needs
// (e.g. split-bf16 weights are packed at first launch) and sets pe.tc_kind.
void tc_prepare(mbx_ctx* c, PlanEntry& pe);
// Launches the plan's tensor-core kernel for one batch.
cudaError_t tc_launch(mbx_ctx* c, const PlanEntry& pe, const BatchLaunch& L);
void tc_release(PlanEntry& pe);
}  // namespace mbx
