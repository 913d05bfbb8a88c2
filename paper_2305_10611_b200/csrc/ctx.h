// ctx.h — internal state of an mbx_ctx: device, stream, HBM arena, index staging, plan registry.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

#include "devplan.h"
#include "kernels.h"
#include "mbatch/backend.hpp"

namespace mbx {

// A registered plan: the host plan, its compiled device form and its launch configuration.
struct PlanEntry {
  mbatch::backend::ExecutablePlan plan;       // as registered (reference semantics, arena parity)
  mbatch::backend::ExecutablePlan exec_plan;  // what the kernels run (shared prefix hoisted out)
  // Shared-prefix hoisting: steps whose operands are all shared compute the same value for every
  // instance (e.g. the TreeLSTM leaf cell's [hz|hz].W); they run once per launch as `prefix_plan`
  // (b = 1) into `prefix_scratch`, and exec_plan reads them as extra shared inputs.
  int prefix_plan = -1;
  std::vector<int64_t> prefix_sizes;  // floats per hoisted boundary tensor
  float* prefix_scratch = nullptr;
  // Shared offsets + upload epoch the scratch currently holds the prefix for (see persist_end).
  mutable std::vector<int64_t> prefix_key;
  DPlan hplan{};
  DPlan* dplan = nullptr;            // device copy
  int64_t temp_floats_per_inst = 0;  // sum of step output sizes (reference arena parity)
  std::vector<mbatch::backend::Shape> out_shapes;
  int tm = 1, threads = 256, smem = 0, unit_chunk = 0, max_split = 1;
  // Column-split head / reduction tail (see split_at_reduction in backend.cpp): a plan whose
  // trailing steps need whole rows (a small dense over a gate result, argmax) runs as two plans,
  // the head split over columns across CTAs, the tail per node.  Head outputs the tail reads
  // live in the plan's (reference-reserved) temporary region, or are original outputs.
  int head_plan = -1, tail_plan = -1;
  int head_nout_orig = 0;                    // head outputs [0, n) are original outputs
  std::vector<int> head_orig_out;            // original output index of head output k < n
  std::vector<int64_t> bnd_size;             // head outputs [n, ...): boundary sizes (floats)
  std::vector<int> tail_in_src;              // tail extra batched input j: >= 0 original output, < 0 -1-boundary
  std::vector<int> tail_orig_out;            // original output index of tail output k
  bool force_vm = false;                     // exact FP32 plan VM only (decision-feeding heads)
  // dense (1 x K . K x N, N <= 32) + argmax plans (NestedRNN's decision tail): a dedicated exact
  // kernel (launch_dense_argmax) instead of the general plan VM.  da_out[k]: 0 row, 1 decision.
  bool da = false;
  int da_k = 0, da_n = 0, da_a_batched = 0, da_a_idx = 0, da_w_idx = 0, da_out[2] = {0, 0};
  // MV-RNN combine cell [x0.M0, x1.M1 per instance, concat, . W, chain] (kernels_mv.cu), and the
  // per-instance matrix add [B0 + B1] it can absorb when the flush issues the two back to back.
  bool mv = false, mv_add = false;
  int mv_x[2] = {0, 0}, mv_m[2] = {0, 0}, mv_first = 0, mv_w = 0, mv_k = 0, mv_n = 0, mv_u = 0;
  int mv_nlinks = 0, mv_link_op[4] = {0, 0, 0, 0}, mv_link_rhs[4] = {-1, -1, -1, -1};
  float* mv_wt = nullptr;                   // W^T (launch_mv_transpose)
  mutable std::vector<int64_t> mv_wt_key;   // {W offset, upload epoch} it holds (session parameters)
  // [concat of whole rows] plans (BiRNN's output concat): concat_rows_kernel.
  bool cat = false;
  int cat_n = 0, cat_kind[8] = {}, cat_idx[8] = {}, cat_cols[8] = {};
  int tc_kind = -1;                  // tensor-core kernel for this plan (kernels_tc.cu), -1 none
  bool tc_small = false;             // gate plan served by the bit-exact kernel in every precision
  bool tc_exact = false;             // the bit-exact CUDA-core gate kernel exists (FP32 contexts use it)
  void* tc_state = nullptr;          // packed weights etc., owned by kernels_tc
};

// Pinned host staging + device mirror for per-launch index arrays (offset tables).
struct MetaRing {
  char* host = nullptr;
  char* dev = nullptr;
  size_t cap = 0, cursor = 0, committed = 0;
};

// One batched launch of a registered plan whose offsets are already staged.
struct BatchLaunch {
  int plan_id = -1;
  int b = 0;
  size_t shared_meta = 0, batched_meta = 0, out_meta = 0;
  size_t prefix_out_meta = 0;  // hoisted shared prefix: its output offsets (scratch)
  // EXPLICIT gathers to run first: (slot size, src offsets meta, dst offset)
  struct Gather { int size; size_t src_meta; int64_t dst; };
  std::vector<Gather> gathers;
  std::vector<BatchLaunch> sub;  // head / tail launches of a split plan
  unsigned shadow_out = 0;       // pointwise launches: bit k = also write output slot k's shadow
  int img_slot = -1;             // pointwise launches: output slot scattered into operand images
  size_t img_dst_meta = 0;       // ... and its per-row destinations (int4, staged)
  // Merged launch (merge_launches: several independent batches of one plan as one launch): node
  // i's output k is at out_node_meta[i * nout + k] instead of out_meta[k] + i * size_k.
  bool out_node = false;
  size_t out_node_meta = 0;
};

// One persistent multi-level launch covering launches [start, start + n) of a flush.
struct LevelsRun {
  int start = 0, n = 0, groups = 1, cfg = 0;
  size_t table = 0;
};

}  // namespace mbx

struct mbx_ctx {
  int device = 0;
  bool dry = false;  // device < 0: host bookkeeping only (offsets, traces), no CUDA calls
  int precision = MBX_PREC_FP32;
  cudaStream_t stream = nullptr;
  bool owns_stream = true;       // false: a pool's shared stream (mbx_pool_create)
  cudaEvent_t ev_sync = nullptr;  // waits for this context's own work only (shared streams)
  // Mini-batch inputs go H2D on a copy stream while the host builds the DFG; the kernel stream
  // waits for that copy (event) only right before the first kernel that needs it, so a shared
  // stream is not held up by one worker's copy.
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy = nullptr;
  bool copy_pending = false;
  // Inputs already in pinned host memory (the caller's): one H2D of the whole data stream into
  // in_dev, then a scatter kernel to the arena offsets (both on copy_stream) — no host memcpy.
  float* in_dev = nullptr;
  size_t in_dev_cap = 0;  // floats
  int64_t* scat_host = nullptr;  // pinned (src, size, dst) triples
  int64_t* scat_dev = nullptr;
  size_t scat_cap = 0;  // triples
  // Contexts on one device that run concurrently (a pool's workers, each on its own stream):
  // launches that need all their CTAs resident at once (mbx_tc_levels: grid barrier, cross-CTA
  // counters) are chained through a per-device lane — each waits for the previous one to
  // complete — so two of them are never partially resident together; everything else overlaps.
  bool serialize_persistent = true;  // every context: any two may run concurrently on a device
  // SMs one persistent launch may occupy: 148, or 74 for pool contexts (mbx_pool_create), whose
  // persistent launches then run two at a time on the device's two lanes (persistent_lane_begin).
  int sm_budget = 148;
  // Second kernel stream: a flush issues independent chains of launches (BiRNN's two directions)
  // on stream and stream2 (runtime.cpp assign_streams); issue_slot selects the per-slot scratch
  // (readiness counters, exchange buffers) of the persistent launches issued on each.
  cudaStream_t stream2 = nullptr;
  int issue_slot = 0;
  bool prefer_pair = false;  // this flush has two independent runs: plan them to fit together
  std::vector<cudaEvent_t> ev_pool;  // cross-stream dependency events, reused flush to flush
  cudaEvent_t ev_persist = nullptr;
  // HBM arena: one virtual-address reservation, physical chunks mapped on demand, so offsets
  // (the reference's TensorHandle::offset) are stable while the arena grows.
  CUdeviceptr base = 0;
  size_t reserve_bytes = 0, mapped_bytes = 0, chunk_bytes = 0;
  std::vector<CUmemGenericAllocationHandle> chunks;
  int64_t used = 0;  // floats
  mbx::MetaRing meta;
  // D2H staging for packed outputs / decisions.
  float* d2h_host = nullptr;
  float* d2h_dev = nullptr;
  size_t d2h_cap = 0;  // floats
  // Pinned staging for a mini-batch's instance inputs (one H2D copy per evaluation).
  float* in_host = nullptr;
  size_t in_cap = 0;  // floats
  std::vector<mbx::PlanEntry> plans;
  std::map<std::vector<int32_t>, int> plan_by_enc;
  std::string err;
  int64_t launches = 0;
  // `launches` right after the last kernel that wrote arbitrary arena tensors (primop / fill): a
  // kernel issued next must not read shared inputs early under PDL.
  int64_t write_launch = -1;
  // Bumped by every host write into existing tensors (uploads, primops); tensor-core weight
  // packs made under an older epoch are re-packed.
  uint64_t upload_epoch = 0;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  // Arena floats [0, persist_end) hold session parameters that only change through host writes
  // (which bump upload_epoch); set by runtime::Session.  Lets a hoisted all-shared prefix whose
  // inputs all lie below it be computed once per upload epoch.
  int64_t persist_end = 0;
  // Split-K partial accumulators of the tensor-core kernels (L2-resident scratch).
  float* tc_part = nullptr;
  size_t tc_part_bytes = 0;
  // Split-bf16 shadow of the arena (tensor-core precisions): a second reservation of the same
  // size mapped in lockstep, 4 bytes per arena float — for each 8-float group at float offset g,
  // bytes [4g, 4g + 16) hold the 8 bf16 "hi" parts and [4g + 16, 4g + 32) the "lo" parts.
  // Producers write it for rows a later tensor-core level gathers (plan_shadows), which then
  // arrive MMA-ready.
  CUdeviceptr shadow_base = 0;
  std::vector<CUmemGenericAllocationHandle> shadow_chunks;
  // Operand images of the tensor-core levels whose gathered rows all have one producer each
  // (plan_shadows): per flush, [level][tile][K rank][chunk][hi | lo] split-bf16 B operands in
  // the canonical UMMA layout, filled by the producers, loaded by the consumer with bulk copies.
  unsigned char* img_buf = nullptr;
  size_t img_cap = 0;
  // mbx_flush_begin .. mbx_flush_end: exec_batched calls are prepared (offsets, handles) and
  // queued, then planned and issued together like a runtime flush (persistent multi-level
  // launches, operand images).
  bool flush_active = false;
  std::vector<mbx::BatchLaunch> pending;
};

namespace mbx {

// Throws mbatch::Error on CUDA failure.
void cuda_check(cudaError_t e, const char* what);
// The per-device persistent-launch lane (see mbx_ctx::serialize_persistent): returns the stream
// to launch on (the lane's, ordered after c->stream's work so far); persistent_lane_end orders
// c->stream's later work after the launch.
cudaStream_t persistent_lane_begin(mbx_ctx* c, bool half);
void persistent_lane_end(mbx_ctx* c);
void persistent_lane_forget(mbx_ctx* c);  // before destroying c (its event may be the lane's last)
// Waits for everything this context enqueued so far (an event: on a pool's shared stream it does
// not wait for work other workers enqueue later).
void stream_wait_own(mbx_ctx* c, const char* what);
void cu_check(CUresult r, const char* what);

float* arena_ptr(mbx_ctx* c);
// Bump allocation in floats (maps more physical memory when needed).
int64_t arena_alloc(mbx_ctx* c, int64_t floats);
void arena_check(const mbx_ctx* c, int64_t off, int64_t n);

// Index staging: reserve bytes (8-aligned) in the pinned ring; returns the byte offset.
size_t meta_stage(mbx_ctx* c, const void* src, size_t bytes);
// Guarantees `bytes` of contiguous free space (may synchronize and recycle the ring).
void meta_reserve(mbx_ctx* c, size_t bytes);
// Issues one H2D copy for everything staged since the last commit.
void meta_commit(mbx_ctx* c);
template <class T>
const T* meta_dev(mbx_ctx* c, size_t off) { return reinterpret_cast<const T*>(c->meta.dev + off); }

void ensure_d2h(mbx_ctx* c, size_t floats);
void ensure_input_stage(mbx_ctx* c, size_t floats);

// Plan registry (backend.cpp).
int register_plan(mbx_ctx* c, const mbatch::backend::ExecutablePlan& plan);



// Host half of exec_batched: validation, gather accounting, reference-order allocation of
// scratch / output regions / temporaries, staging of offset tables.  Fills `out_off`
// (b * nout) and returns the launch record (not yet issued).
BatchLaunch prepare_batch(mbx_ctx* c, int plan_id, int b, const int64_t* shared_off,
                          const int64_t* batched_off, int gather_mode, int64_t* out_off,
                          int64_t* gather_bytes);
// Device half: enqueues the gather copies and the plan kernel (meta must be committed).
void issue_batch(mbx_ctx* c, const BatchLaunch& L);
// Issues Ls[i] — together with Ls[i + 1] in one launch when the two fuse (an MV-RNN combine
// cell and the matrix add of the same nodes) — and returns how many launches it consumed.
int issue_batches(mbx_ctx* c, const std::vector<BatchLaunch>& Ls, size_t i);
// Whether launch L can be merged with other independent launches of its plan (merge_launches):
// the exact small gate kernel, the dense + argmax kernel, and split plans made of them.
bool mergeable(const mbx_ctx* c, const BatchLaunch& L);
// Whether two launches of one plan read the same shared operands.
bool same_shared(const mbx_ctx* c, const BatchLaunch& a, const BatchLaunch& b);
// One launch over the nodes of g (mergeable launches of one plan, same shared operands, no node
// reading another's output): node tables concatenated, per-node output offsets.
BatchLaunch merge_launches(mbx_ctx* c, const std::vector<const BatchLaunch*>& g);
// The exact small gate kernel serves this plan's batches in every precision (tc_launch).
bool tc_small_kernel(const PlanEntry& pe);
void issue_prefix(mbx_ctx* c, const BatchLaunch& L);

// Persistent multi-level launches (kernels_tc.cu): if launches [i, i+n) (n >= 1) are consecutive
// batches of one tensor-core gate plan over the same weights that one mbx_tc_levels launch can
// run, stages its level table (before meta_commit) into *table, sets its node-tile groups
// (grid x) and returns n; else 0.
int plan_levels(mbx_ctx* c, const std::vector<BatchLaunch>& Ls, size_t i, size_t* table, int* groups, int* cfg);
// After every run of the flush is planned (before meta_commit): marks the levels whose gathered
// rows all have split-bf16 shadows written earlier in the flush (they skip the conversion), and
// makes those rows' producers (pointwise launches, levels of a run) write the shadows.
void plan_shadows(mbx_ctx* c, std::vector<BatchLaunch>& Ls, const std::vector<LevelsRun>& runs);
// Plans and issues the launches queued by mbx_flush_begin .. (exec_batched in flush mode):
// persistent multi-level runs, operand images / shadows, one offset-table H2D, then the kernels.
void issue_pending(mbx_ctx* c);
// Issues queued launches (if any) before an operation that reads or writes the arena.
inline void settle(mbx_ctx* c) {
  if (!c->pending.empty()) issue_pending(c);
}
// Enqueues that launch (meta committed).
void issue_levels(mbx_ctx* c, const std::vector<BatchLaunch>& Ls, size_t i, int n, size_t table, int groups,
                  int cfg);

}  // namespace mbx
