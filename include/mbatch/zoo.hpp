// mbatch/zoo.hpp — the evaluation models (reference: proj/include/mbatch/zoo.hpp,
// proj/src/zoo.cpp) as compiled models for the B200 runtime.
//
// The reference parses each model's text IR and compiles it (duplication, coarsening, hoisting,
// ghosts, phases, kernel generation).  Here each model is delivered in compiled form: its kernel
// library (signature names, shared/batched split, lowered ExecutablePlans), static blocks with
// bindings and hoist depths, stage phases, and an AOT-lowered C++ body that emits the same DFG
// the reference executor would (ACRoBat's own AOT approach).  Parity with the
// reference compiler's artefacts is checked in tests/ against golden dumps of the reference.
#pragma once

#include <string>
#include <vector>

#include "mbatch/runtime.hpp"

namespace mbatch {
namespace zoo {

using runtime::CompiledModel;
using runtime::ExecOptions;
using runtime::HostValue;
using runtime::InstanceInput;
using runtime::ParamEnv;

// name in {rnn, birnn, treelstm, mvrnn, nestedrnn, drnn, stackrnn, fig5}; any hidden size
// (the reference's "small" / "large" are 32 / 64).  Classes C = 8.
CompiledModel get_model(const std::string& name, int hidden, const ExecOptions& opts = {});
std::vector<std::string> model_names();  // the seven evaluation models

// Parameters drawn uniformly from [-0.5, 0.5) from mt19937(seed*7919+17) in module order
// (zoo.cpp:332-341).
ParamEnv make_params(const CompiledModel& model, unsigned seed);
// Per-instance inputs from mt19937(seed*104729+31*i+7): lists of length U[4,12], full binary
// trees with U[4,16] leaves, fuel U[3,4], sel = i%2 (zoo.cpp:343-401).
std::vector<InstanceInput> make_inputs(const CompiledModel& model, unsigned seed, int batch);

}  // namespace zoo
}  // namespace mbatch
