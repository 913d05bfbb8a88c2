// mbatch/runtime.hpp — lazy batching runtime (fibers, inline-depth DFG construction, depth /
// agenda scheduling, device flushes), API-compatible with the reference's
// proj/include/mbatch/runtime.hpp and proj/include/mbatch/kernelgen.hpp (type and function names,
// trace and node-table semantics).  What differs is where the work happens: every flush runs its
// batches as sm_100a kernels over an HBM arena, and models are AOT-lowered C++ programs
// (zoo.hpp) instead of an interpreted IR — the compiled artefacts the executor consumes
// (kernel signatures, lowered plans, block bindings, hoist depths, phases) are the reference's.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "mbatch/backend.hpp"

namespace mbatch {

namespace kernelgen {

using backend::ExecutablePlan;
using backend::PlanRef;
using backend::Shape;

// proj/include/mbatch/kernelgen.hpp:18-44
struct KernelSignature {
  int id = -1;
  std::string name;
  std::vector<std::pair<std::string, Shape>> shared_params;
  std::vector<std::pair<std::string, Shape>> batched_params;
  std::vector<Shape> outputs;
  bool ghost = false;
};

struct BlockBinding {
  int sig_id = -1;
  std::vector<int> shared_input_pos, batched_input_pos;
};

struct KernelLibrary {
  std::vector<KernelSignature> signatures;
  std::map<int, BlockBinding> binding_of_block;
  std::vector<ExecutablePlan> plans;  // indexed by sig id
  int ghost_sig = -1;
  const ExecutablePlan& plan(int sig) const { return plans.at(sig); }
};

}  // namespace kernelgen

namespace runtime {

using backend::GatherMode;
using backend::Shape;
using backend::TensorHandle;

struct HostValue {
  enum class Kind { kTensor, kInt, kFloat, kList, kTuple, kAdt };
  Kind kind = Kind::kTensor;
  Shape shape;
  std::vector<float> data;
  // Tensor data borrowed from the caller instead of `data` (the C ABI's instance inputs: valid
  // for the duration of the evaluate call, so the floats are copied once, into the pinned
  // staging buffer, not first into a vector).
  const float* ext = nullptr;
  long ival = 0;
  double fval = 0.0;
  std::vector<HostValue> items;
  std::string ctor;

  static HostValue tensor(Shape s, std::vector<float> d);
  static HostValue scalar(long v);
  static HostValue list(std::vector<HostValue> items);
  static HostValue tuple(std::vector<HostValue> items);
  static HostValue adt(std::string ctor, std::vector<HostValue> fields);
};

bool bitwise_equal(const HostValue& a, const HostValue& b);

struct ExecOptions {
  enum class Scheduler { kDepth, kAgenda };
  Scheduler scheduler = Scheduler::kDepth;
  GatherMode gather = GatherMode::kFused;
  bool coarsen = true;          // compile-time (fixed: blocks are the coarsened ones)
  bool ghost = true;            // compile-time (ghost units are part of the lowered program)
  bool phases = true;
  bool hoist = true;
  bool horizontal_fuse = true;  // compile-time (plans carry the fused denses)
  unsigned seed = 0;
  // B200 additions
  bool record_nodes = true;     // keep EvalResult::nodes
  bool time_kernels = false;    // CUDA-event span of the device work
  bool time_batches = false;    // CUDA events around every batch launch
  bool inputs_resident = false; // inputs already materialised by an identical previous call
  bool outputs_on_device = false; // outputs stay in the arena: no read-back, EvalResult::outputs empty
  // Return once the device work and the output read-back are enqueued (no final sync, outputs not
  // decoded): the caller synchronises the context's stream before reusing the context.  Used by
  // the throughput pool to keep two mini-batches in flight per worker.
  bool defer_sync = false;
};

// Static block of the compiled model (the reference's analysis::StaticBlock + hoist depth).
struct StaticBlockInfo {
  int id = -1;
  std::string func;
  int sig = -1;
  int hoist = -1;  // static depth, -1 = dynamic
  std::vector<std::string> inputs;
  int num_outputs = 0;
};

struct ParamDecl {
  std::string name;
  Shape shape;                     // tensors
  bool is_instance_input = false;
};

class Program;  // AOT-lowered model body (zoo.cpp)

struct CompiledModel {
  std::string name;
  int hidden = 0;
  std::vector<ParamDecl> params;   // module order (params and instance inputs)
  kernelgen::KernelLibrary kernels;
  std::vector<StaticBlockInfo> blocks;
  std::vector<int> stage_phase;    // main stage -> phase
  std::shared_ptr<const Program> program;
  ExecOptions opts;
  // analysis::static_nesting_estimate of the model's functions (analysis.cpp:1293-1324): the
  // entry 0, a callee in another call-graph SCC its caller's level (+1 when it recurses); the
  // zoo programs carry their modules' values.
  std::map<std::string, int> nesting;
};

struct TensorRef {
  int node = -1;
  int out = 0;
  TensorHandle handle;
};

struct DFGNode {
  int id = -1;
  int sig_id = -1;
  int block_id = -1;
  int instance = -1;
  int phase = 0;
  int depth = 0;
  bool ghost = false;
  bool executed = false;
  std::vector<TensorRef> shared_ins, batched_ins;
  std::vector<int> producers;
  std::vector<TensorHandle> outputs;
};

struct BatchRecord {
  int phase = 0;
  int depth = 0;
  int sig = -1;
  int size = 0;
  bool ghost = false;
  std::vector<int> node_ids;
};

struct ScheduleTrace {
  std::vector<BatchRecord> batches;
  long kernel_launches = 0;
  long total_nodes = 0;
  long scheduler_ops = 0;
  long sync_points = 0;
  long gather_bytes = 0;
  long dfg_edges = 0;
  std::vector<int> flush_boundaries;
};

struct Timing {
  double host_total_us = 0;     // evaluate_batch wall time
  double host_dfg_us = 0;       // fibers + DFG + scheduling + launch (host)
  double device_span_us = 0;    // sum over flushes of first-to-last batch (CUDA events)
  long h2d_bytes = 0, d2h_bytes = 0;
  long device_launches = 0;     // CUDA kernels issued
  // host_dfg_us split: fiber execution + DFG build, scheduling, offset tables, kernel issue
  double host_fibers_us = 0, host_sched_us = 0, host_prepare_us = 0, host_issue_us = 0;
  std::vector<double> batch_us; // per non-ghost batch (time_batches)
};

struct EvalResult {
  std::vector<HostValue> outputs;
  ScheduleTrace trace;
  std::vector<DFGNode> nodes;
  Timing timing;
};

std::vector<BatchRecord> schedule_depth(const std::vector<const DFGNode*>& nodes, long& scheduler_ops);
std::vector<BatchRecord> schedule_agenda(const std::vector<const DFGNode*>& nodes, long& scheduler_ops);

using ParamEnv = std::map<std::string, HostValue>;
using InstanceInput = std::map<std::string, HostValue>;

// Instance inputs / outputs in the C ABI's flat hostval encoding (include/mbx.h: int32 tokens +
// float data, depth-first; per instance its @main instance inputs in module order).  Evaluating
// from the encoding skips building HostValue trees on the way in and out (mbx_evaluate_batch).
struct EncodedValues {
  int count = 0;  // instances (inputs) / values (outputs)
  const int32_t* toks = nullptr;
  int64_t ntok = 0;
  const float* data = nullptr;  // borrowed for the call
  int64_t ndata = 0;
};
struct EncodedOutputs {
  std::vector<int32_t> toks;
  std::vector<float> data;
};

// A device session: context + the model's parameters resident in the arena (module order,
// offsets identical to the reference's Executor, proj/src/executor.cpp:153-158) + the model's
// registered plans.  device < 0 runs the host logic only (no kernels; tensor values are zero),
// which reproduces traces of models without tensor-dependent control flow on a CPU.
class Session {
 public:
  Session(const CompiledModel& model, int device = 0, int precision = MBX_PREC_FP32);
  // Uses an existing context (not owned); parameters are allocated at its current arena end.
  Session(const CompiledModel& model, mbx_ctx* ctx);
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;
  void set_params(const ParamEnv& params);
  EvalResult evaluate(const std::vector<InstanceInput>& inputs, const ExecOptions& opts);
  // The same from / to the flat encoding (EvalResult::outputs stays empty; *out gets them).
  EvalResult evaluate_encoded(const EncodedValues& inputs, const ExecOptions& opts, EncodedOutputs* out);
  const CompiledModel& model() const { return model_; }
  mbx_ctx* ctx() const { return ctx_; }
  int64_t params_end() const { return params_end_; }
  const std::map<std::string, TensorHandle>& param_handles() const { return param_handles_; }
  const std::vector<int>& plan_ids() const { return plan_ids_; }
  // DFG node objects of earlier evaluations, kept with their vectors' capacity so the next
  // evaluation's node construction allocates nothing (implementation detail of the executor).
  std::vector<DFGNode>& node_pool() { return node_pool_; }
  int64_t node_hint() const { return node_hint_; }
  int64_t fiber_hint() const { return fiber_hint_; }
  void set_hints(int64_t nodes, int64_t fibers) {
    node_hint_ = nodes;
    fiber_hint_ = fibers;
  }

 private:
  std::vector<DFGNode> node_pool_;
  int64_t node_hint_ = 0, fiber_hint_ = 0;
  const CompiledModel& model_;
  mbx_ctx* ctx_ = nullptr;
  bool owned_ = true;
  void init();
  std::map<std::string, TensorHandle> param_handles_;
  int64_t params_end_ = 0;
  std::vector<int> plan_ids_;  // sig id -> registered plan id
};

// Reference-compatible entry points: a fresh session per call (params re-uploaded, like the
// reference materialising them per Executor).
EvalResult evaluate_batch(const CompiledModel& model, const ParamEnv& params,
                          const std::vector<InstanceInput>& inputs);

// Unbatched evaluation (the reference's sequential oracle entry point, runtime.hpp:141-144):
// every instance evaluated on its own, one instance per mini-batch, on the device; outputs equal
// evaluate_batch's bit for bit in FP32 (the reference's batched == unbatched property).
std::vector<HostValue> reference_evaluate(const CompiledModel& model, const ParamEnv& params,
                                          const std::vector<InstanceInput>& inputs);

// Exact invocation counts per kernel signature over a sample run, plus the static nesting-depth
// estimate for comparison; ranked by count (pipeline.cpp:99-123).
struct ProfileReport {
  std::map<int, long> counts;          // sig id -> invocations (non-ghost DFG nodes)
  std::map<int, int> static_estimate;  // sig id -> nesting level of its blocks' functions (max)
  std::vector<int> ranking;            // sig ids, most-invoked first (ties: lower id)
};
ProfileReport profile_invocations(const CompiledModel& model, const ParamEnv& params,
                                  const std::vector<InstanceInput>& inputs);
// The same over the DFG node table of a finished evaluation (record_nodes).
ProfileReport profile_from_nodes(const CompiledModel& model, const std::vector<DFGNode>& nodes);

}  // namespace runtime
}  // namespace mbatch
