// devplan.h — device-side form of a backend::ExecutablePlan, shared by the host compiler
// (backend.cpp) and the kernels (kernels.cu).  Plain-old-data, copied to HBM once per plan.
//
// A plan is the reference's interpretable kernel plan (proj/include/mbatch/backend.hpp:101-132):
// steps of kOp / kFusedDense / kChain over refs to shared inputs (S), batched inputs (B) and
// per-instance temporaries (T).  The plan compiler (backend.cpp: compile_plan) adds:
//   * temp_off: each step's slot in the per-instance temp block (on-chip, in shared memory),
//   * split:    whether a step is column-local w.r.t. the plan's output "unit" columns, so a
//               launch can spread one batch over (node tiles) x (column tiles) CTAs,
//   * shapes of every ref, so the kernel never consults the host plan.
#pragma once
#include <stdint.h>

namespace mbx {

constexpr int kMaxIn = 8;
constexpr int kMaxChain = 8;
constexpr int kMaxSteps = 40;
constexpr int kMaxOut = 4;
constexpr int kMaxShared = 16;
constexpr int kMaxBatched = 8;
constexpr int kMaxTM = 8;  // node tile of the plan VM

enum RefKind : int32_t { kRefShared = 0, kRefBatched = 1, kRefTemp = 2 };
enum StepKind : int32_t { kStepOp = 0, kStepFused = 1, kStepChain = 2 };
enum Op : int32_t { kDense = 0, kAdd, kMul, kSigmoid, kTanh, kRelu, kConcat, kArgmax, kFill };

struct DRef {
  int32_t kind, index, col_off, cols;  // cols < 0: whole tensor
  int32_t rows_r, cols_r;              // resolved shape of the (sliced) operand
};

struct DLink {
  int32_t op, has_rhs;
  DRef rhs;
};

struct DStep {
  int32_t kind, op, rows, cols, nin, nchain;
  int32_t temp_off;  // float offset inside the per-instance temp block
  int32_t split;     // computed per column tile (1) or in full by every CTA (0)
  DRef ins[kMaxIn];
  DLink chain[kMaxChain];
};

struct DPlan {
  int32_t nsteps, nout, nshared, nbatched;
  int32_t temp_floats;   // per-instance temp block size
  int32_t unit;          // width of the column-split space (0: no split)
  int32_t ghost;
  int32_t pad_;
  DStep steps[kMaxSteps];
  DRef outputs[kMaxOut];
  int32_t out_split[kMaxOut];
};

}  // namespace mbx
