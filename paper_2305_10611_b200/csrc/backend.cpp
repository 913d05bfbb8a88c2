// backend.cpp — device arena, plan compiler/registry and the host half of exec_batched.
//
// Reference interfaces replaced (proj/include/mbatch/backend.hpp):
//   Arena (:63-88)            -> HBM arena in one CUDA VMM reservation (stable offsets)
//   exec_primop (:92-93)      -> one-step plan on the FP32 plan VM (kernels_vm.cu)
//   exec_batched (:149-150)   -> prepare_batch (validation, gather accounting, allocation in the
//                                reference's order) + issue_batch (device launch)
// Error texts are the reference's, so callers matching on them keep working.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>

#include "ctx.h"
#include "tc.h"

namespace mbx {

std::atomic<int64_t> g_launches{0};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw mbatch::Error(std::string("cuda error in ") + what + ": " + cudaGetErrorString(e));
}
void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw mbatch::Error(std::string("cuda driver error ") + std::to_string(int(r)) + " in " + what);
}

namespace {
// One per device: a stream of its own that every co-residency-requiring launch of every context
// on the device goes through (in host submission order), so two such kernels never run
// concurrently, back-to-back kernels in it start with little gap, and the contexts' own streams
// stay free for everything else.
// Two lanes: launches of at most half the SMs alternate between them (two run at once, and
// together they always fit: no grid can wait for SMs the other holds); a larger launch takes
// lane 0 after lane 1's work and lane 1 follows it (it runs alone).
struct PersistentLane {
  std::mutex mu;  // held from begin to end: the dependency edges enclose one launch
  cudaStream_t stream[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  int next = 0;
  int cur = 0;          // lane of the launch between begin and end
  bool whole = false;   // ... and whether it is a whole-device launch
};
PersistentLane& lane_of(int device) {
  static std::mutex m;
  static std::map<int, std::unique_ptr<PersistentLane>> lanes;
  std::lock_guard<std::mutex> lock(m);
  auto& p = lanes[device];
  if (!p) p = std::make_unique<PersistentLane>();
  return *p;
}
}  // namespace

cudaStream_t persistent_lane_begin(mbx_ctx* c, bool half) {
  if (!c->serialize_persistent || c->dry) return c->stream;
  PersistentLane& L = lane_of(c->device);
  std::unique_lock<std::mutex> lock(L.mu);  // released on every error path below
  if (!L.stream[0]) {
    // Highest priority: when SMs free up, the block scheduler places the lane kernel's CTAs first
    // (its resident CTAs wait at the grid barrier for the rest).
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    for (int k = 0; k < 2; ++k) {
      cuda_check(cudaStreamCreateWithPriority(&L.stream[k], cudaStreamNonBlocking, hi), "persistent lane stream");
      cuda_check(cudaEventCreateWithFlags(&L.done[k], cudaEventDisableTiming), "persistent lane event");
    }
  }
  if (!c->ev_persist) cuda_check(cudaEventCreateWithFlags(&c->ev_persist, cudaEventDisableTiming), "event");
  // Half-lane launches: two such grids always fit together (the caller checked SMs and clusters,
  // or the context planned for half the device); anything else runs alone.
  L.whole = !half;
  if (L.whole) {
    L.cur = 0;
    cuda_check(cudaStreamWaitEvent(L.stream[0], L.done[1], 0), "persistent lane wait");  // runs alone
  } else {
    L.cur = L.next;
    L.next ^= 1;
  }
  // The launch follows this context's work so far ...
  cuda_check(cudaEventRecord(c->ev_persist, c->stream), "persistent lane record");
  cuda_check(cudaStreamWaitEvent(L.stream[L.cur], c->ev_persist, 0), "persistent lane wait");
  lock.release();  // held until persistent_lane_end
  return L.stream[L.cur];
}

void persistent_lane_end(mbx_ctx* c) {
  if (!c->serialize_persistent || c->dry) return;
  PersistentLane& L = lane_of(c->device);
  std::unique_lock<std::mutex> lock(L.mu, std::adopt_lock);  // taken by persistent_lane_begin
  // ... and this context's later work follows the launch.  (The lock is released even if these
  // throw after a sticky device error, so the other workers fail instead of blocking.)
  cuda_check(cudaEventRecord(L.done[L.cur], L.stream[L.cur]), "persistent lane record");
  if (L.whole) cuda_check(cudaStreamWaitEvent(L.stream[1], L.done[0], 0), "persistent lane wait");
  cuda_check(cudaStreamWaitEvent(c->stream, L.done[L.cur], 0), "persistent lane wait");
}

void persistent_lane_forget(mbx_ctx* c) { (void)c; }

void stream_wait_own(mbx_ctx* c, const char* what) {
  if (c->dry) return;
  if (!c->ev_sync) {
    cuda_check(cudaStreamSynchronize(c->stream), what);
    return;
  }
  cuda_check(cudaEventRecord(c->ev_sync, c->stream), what);
  cuda_check(cudaEventSynchronize(c->ev_sync), what);
}

float* arena_ptr(mbx_ctx* c) { return reinterpret_cast<float*>(c->base); }

// Driver VMM entry points, resolved through the runtime (cudaGetDriverEntryPoint) so the library
// has no link-time dependency on libcuda and loads on GPU-less hosts.
struct VmmApi {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
};

static const VmmApi& vmm() {
  static VmmApi api = [] {
    VmmApi a;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      cuda_check(cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q), name);
      if (q != cudaDriverEntryPointSuccess || !*fn) throw mbatch::Error(std::string("driver entry point missing: ") + name);
    };
    get("cuMemCreate", reinterpret_cast<void**>(&a.create));
    get("cuMemMap", reinterpret_cast<void**>(&a.map));
    get("cuMemSetAccess", reinterpret_cast<void**>(&a.set_access));
    get("cuMemAddressReserve", reinterpret_cast<void**>(&a.reserve));
    get("cuMemAddressFree", reinterpret_cast<void**>(&a.addr_free));
    get("cuMemUnmap", reinterpret_cast<void**>(&a.unmap));
    get("cuMemRelease", reinterpret_cast<void**>(&a.release));
    get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&a.granularity));
    return a;
  }();
  return api;
}

void arena_init(mbx_ctx* c) {
  if (c->dry) return;
  const VmmApi& api = vmm();
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = c->device;
  size_t gran = 0;
  cu_check(api.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
  c->chunk_bytes = ((size_t(256) << 20) + gran - 1) / gran * gran;
  c->reserve_bytes = size_t(128) << 30;  // 128 GiB of address space; physical memory on demand
  cu_check(api.reserve(&c->base, c->reserve_bytes, 0, 0, 0), "cuMemAddressReserve");
  // The split-bf16 shadow (same byte size, same offsets; mapped in lockstep with the arena).
  cu_check(api.reserve(&c->shadow_base, c->reserve_bytes, 0, 0, 0), "cuMemAddressReserve (shadow)");
}

void arena_release(mbx_ctx* c) {
  if (c->dry || !c->base) return;
  const VmmApi& api = vmm();
  for (size_t k = 0; k < c->chunks.size(); ++k) {
    api.unmap(c->base + k * c->chunk_bytes, c->chunk_bytes);
    api.release(c->chunks[k]);
  }
  c->chunks.clear();
  for (size_t k = 0; k < c->shadow_chunks.size(); ++k) {
    api.unmap(c->shadow_base + k * c->chunk_bytes, c->chunk_bytes);
    api.release(c->shadow_chunks[k]);
  }
  c->shadow_chunks.clear();
  api.addr_free(c->base, c->reserve_bytes);
  if (c->shadow_base) api.addr_free(c->shadow_base, c->reserve_bytes);
  c->base = 0;
  c->shadow_base = 0;
}

static void arena_map_to(mbx_ctx* c, size_t bytes) {
  if (c->dry) return;
  const VmmApi& api = vmm();
  while (c->mapped_bytes < bytes) {
    if (c->mapped_bytes + c->chunk_bytes > c->reserve_bytes) throw mbatch::Error("arena reservation exhausted");
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = c->device;
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (int shadow = 0; shadow < 2; ++shadow) {
      const CUdeviceptr at = (shadow ? c->shadow_base : c->base) + c->mapped_bytes;
      CUmemGenericAllocationHandle h;
      cu_check(api.create(&h, c->chunk_bytes, &prop, 0), "cuMemCreate");
      cu_check(api.map(at, c->chunk_bytes, 0, h, 0), "cuMemMap");
      cu_check(api.set_access(at, c->chunk_bytes, &acc, 1), "cuMemSetAccess");
      (shadow ? c->shadow_chunks : c->chunks).push_back(h);
    }
    c->mapped_bytes += c->chunk_bytes;
  }
}

int64_t arena_alloc(mbx_ctx* c, int64_t floats) {
  MBATCH_CHECK(floats >= 0, "negative allocation");
  int64_t off = c->used;
  size_t need = size_t(off + floats) * sizeof(float);
  if (need > c->mapped_bytes) arena_map_to(c, need);
  c->used += floats;
  return off;
}

void arena_check(const mbx_ctx* c, int64_t off, int64_t n) {
  MBATCH_CHECK(off >= 0 && off + n <= c->used, "tensor handle out of arena bounds");
}

void meta_reserve(mbx_ctx* c, size_t bytes) {
  bytes = (bytes + 7) & ~size_t(7);
  if (c->meta.cursor + bytes <= c->meta.cap) return;
  meta_commit(c);
  if (!c->dry) cuda_check(cudaStreamSynchronize(c->stream), "meta recycle");
  c->meta.cursor = c->meta.committed = 0;
  if (bytes > c->meta.cap) {
    size_t cap = std::max(bytes, c->meta.cap * 2);
    if (c->dry) {
      std::free(c->meta.host);
      c->meta.host = static_cast<char*>(std::malloc(cap));
    } else {
      if (c->meta.host) cudaFreeHost(c->meta.host);
      if (c->meta.dev) cudaFree(c->meta.dev);
      cuda_check(cudaMallocHost(&c->meta.host, cap), "meta host");
      cuda_check(cudaMalloc(&c->meta.dev, cap), "meta dev");
    }
    c->meta.cap = cap;
  }
}

size_t meta_stage(mbx_ctx* c, const void* src, size_t bytes) {
  size_t b8 = (bytes + 7) & ~size_t(7);
  if (c->meta.cursor + b8 > c->meta.cap) meta_reserve(c, b8);
  size_t off = c->meta.cursor;
  if (bytes) std::memcpy(c->meta.host + off, src, bytes);
  c->meta.cursor += b8;
  return off;
}

void meta_commit(mbx_ctx* c) {
  if (c->dry) {
    c->meta.committed = c->meta.cursor;
    return;
  }
  if (c->copy_pending) {  // the mini-batch's inputs (copy stream) before any kernel reads them
    cuda_check(cudaStreamWaitEvent(c->stream, c->ev_copy, 0), "input copy wait");
    c->copy_pending = false;
  }
  if (c->meta.cursor > c->meta.committed) {
    cuda_check(cudaMemcpyAsync(c->meta.dev + c->meta.committed, c->meta.host + c->meta.committed,
                               c->meta.cursor - c->meta.committed, cudaMemcpyHostToDevice, c->stream),
               "meta H2D");
    c->meta.committed = c->meta.cursor;
  }
}

void ensure_input_stage(mbx_ctx* c, size_t floats) {
  if (floats <= c->in_cap) return;
  size_t cap = std::max(floats, c->in_cap * 2);
  if (c->dry) {
    std::free(c->in_host);
    c->in_host = static_cast<float*>(std::malloc(cap * sizeof(float)));
  } else {
    cuda_check(cudaStreamSynchronize(c->stream), "input stage grow");
    if (c->in_host) cudaFreeHost(c->in_host);
    cuda_check(cudaMallocHost(&c->in_host, cap * sizeof(float)), "input stage");
  }
  c->in_cap = cap;
}

void ensure_d2h(mbx_ctx* c, size_t floats) {
  if (c->dry || floats <= c->d2h_cap) return;
  cuda_check(cudaStreamSynchronize(c->stream), "d2h grow");
  size_t cap = std::max(floats, c->d2h_cap * 2);
  if (c->d2h_host) cudaFreeHost(c->d2h_host);
  if (c->d2h_dev) cudaFree(c->d2h_dev);
  cuda_check(cudaMallocHost(&c->d2h_host, cap * sizeof(float)), "d2h host");
  cuda_check(cudaMalloc(&c->d2h_dev, cap * sizeof(float)), "d2h dev");
  c->d2h_cap = cap;
}

// ---------------------------------------------------------------------------------------------
// Plan compiler: ExecutablePlan -> DPlan (shapes, temp layout, column-split analysis)

namespace {

using mbatch::backend::ExecutablePlan;
using mbatch::backend::OpCode;
using mbatch::backend::PlanRef;
using mbatch::backend::PlanStep;
using mbatch::backend::Shape;

Shape ref_shape(const ExecutablePlan& p, const PlanRef& r, size_t cur_step) {
  Shape s;
  switch (r.kind) {
    case PlanRef::Kind::kShared:
      MBATCH_CHECK(r.index >= 0 && size_t(r.index) < p.shared_shapes.size(), "plan: shared ref out of range");
      s = p.shared_shapes[r.index];
      break;
    case PlanRef::Kind::kBatched:
      MBATCH_CHECK(r.index >= 0 && size_t(r.index) < p.batched_shapes.size(), "plan: batched ref out of range");
      s = p.batched_shapes[r.index];
      break;
    case PlanRef::Kind::kTemp:
      MBATCH_CHECK(r.index >= 0 && size_t(r.index) < cur_step, "plan: temp ref to a later step");
      s = p.steps[r.index].out_shape;
      break;
  }
  if (r.cols >= 0) {
    MBATCH_CHECK(s.rows == 1, "column slices require row vectors");
    MBATCH_CHECK(r.col_off >= 0 && r.col_off + r.cols <= s.cols, "plan: column slice out of range");
    s = Shape{1, r.cols};
  }
  return s;
}

DRef to_dref(const ExecutablePlan& p, const PlanRef& r, size_t cur) {
  Shape s = ref_shape(p, r, cur);
  DRef d{};
  d.kind = r.kind == PlanRef::Kind::kShared ? kRefShared : r.kind == PlanRef::Kind::kBatched ? kRefBatched : kRefTemp;
  d.index = r.index;
  d.col_off = r.col_off;
  d.cols = r.cols;
  d.rows_r = s.rows;
  d.cols_r = s.cols;
  return d;
}

void split_analysis(const ExecutablePlan& p, DPlan& d) {
  const size_t n = p.steps.size();
  d.unit = 0;
  if (p.outputs.empty()) return;
  Shape o0 = ref_shape(p, p.outputs[0], n);
  if (o0.rows != 1) return;
  const int U = o0.cols;
  std::vector<bool> capable(n, false), full(n, false);
  for (size_t s = 0; s < n; ++s) {
    const PlanStep& st = p.steps[s];
    if (st.out_shape.rows != 1) continue;
    if (st.kind == PlanStep::Kind::kFusedDense) {
      bool ok = true;
      for (size_t w = 1; w < st.ins.size(); ++w) ok = ok && ref_shape(p, st.ins[w], s).cols == U;
      capable[s] = ok;
    } else if (st.kind == PlanStep::Kind::kChain) {
      capable[s] = st.out_shape.cols == U;
    } else if (st.op == OpCode::kDense) {
      capable[s] = st.out_shape.cols == U;
    } else if (mbatch::backend::is_elementwise(st.op)) {
      capable[s] = st.out_shape.cols == U;
    }
  }
  auto temp_ins = [&](size_t s) {
    std::vector<std::pair<PlanRef, bool>> v;  // (ref, is_dense_A)
    const PlanStep& st = p.steps[s];
    for (size_t i = 0; i < st.ins.size(); ++i) {
      bool dense_a = (st.kind == PlanStep::Kind::kFusedDense || (st.kind == PlanStep::Kind::kOp && st.op == OpCode::kDense)) && i == 0;
      if (st.ins[i].kind == PlanRef::Kind::kTemp) v.push_back({st.ins[i], dense_a});
    }
    for (auto& l : st.chain)
      if (l.rhs && l.rhs->kind == PlanRef::Kind::kTemp) v.push_back({*l.rhs, false});
    return v;
  };
  // A split consumer may read a producer's columns only if the column maps line up.
  auto aligned = [&](const PlanRef& r) {
    const PlanStep& prod = p.steps[r.index];
    if (r.cols < 0) return prod.out_shape.cols == U;
    if (r.cols != U || r.col_off % U != 0) return false;
    if (prod.kind == PlanStep::Kind::kFusedDense) {
      int col = 0;
      for (size_t w = 1; w < prod.ins.size(); ++w) {
        if (col == r.col_off) return true;
        col += ref_shape(p, prod.ins[w], r.index).cols;
      }
      return false;
    }
    return prod.out_shape.cols == U && r.col_off == 0;
  };
  bool changed = true;
  while (changed) {
    changed = false;
    for (size_t s = 0; s < n; ++s) {
      bool split = capable[s] && !full[s];
      for (auto& [r, dense_a] : temp_ins(s)) {
        bool need = dense_a || !split || !aligned(r);
        if (need && !full[r.index]) { full[r.index] = true; changed = true; }
      }
    }
    for (size_t k = 0; k < p.outputs.size(); ++k) {
      const PlanRef& r = p.outputs[k];
      if (r.kind != PlanRef::Kind::kTemp) continue;
      if (!aligned(r) && !full[r.index]) { full[r.index] = true; changed = true; }
    }
  }
  bool any_dense_split = false;
  for (size_t s = 0; s < n; ++s) {
    d.steps[s].split = capable[s] && !full[s];
    const PlanStep& st = p.steps[s];
    if (d.steps[s].split && (st.kind == PlanStep::Kind::kFusedDense || (st.kind == PlanStep::Kind::kOp && st.op == OpCode::kDense)))
      any_dense_split = true;
  }
  for (size_t k = 0; k < p.outputs.size(); ++k) {
    const PlanRef& r = p.outputs[k];
    d.out_split[k] = r.kind == PlanRef::Kind::kTemp && d.steps[r.index].split && aligned(r);
  }
  // Column tiling pays when a contraction is split (its weight slice is read once per tile) or
  // when the plan is purely column-local (no redundant full steps); otherwise run unsplit.
  bool all_split = true;
  for (size_t s = 0; s < n; ++s) all_split = all_split && d.steps[s].split;
  if (any_dense_split || all_split) d.unit = U;
  else
    for (size_t s = 0; s < n; ++s) d.steps[s].split = 0;
}

// Splits `p` into a prefix of steps whose operands are all shared (computed once per launch) and
// the rest, which reads the prefix's boundary tensors as extra shared inputs.  Returns false when
// nothing worth hoisting (no contraction in the shared part) exists.
bool hoist_shared_prefix(const ExecutablePlan& p, ExecutablePlan& prefix, ExecutablePlan& rest,
                         std::vector<int64_t>& boundary_sizes) {
  const size_t n = p.steps.size();
  std::vector<bool> so(n, false);
  bool has_dense = false;
  auto refs_of = [&](const PlanStep& st) {
    std::vector<PlanRef> r = st.ins;
    for (auto& l : st.chain)
      if (l.rhs) r.push_back(*l.rhs);
    return r;
  };
  for (size_t s = 0; s < n; ++s) {
    bool all = true;
    for (auto& r : refs_of(p.steps[s]))
      all = all && (r.kind == PlanRef::Kind::kShared || (r.kind == PlanRef::Kind::kTemp && so[r.index]));
    so[s] = all;
    const PlanStep& st = p.steps[s];
    if (all && (st.kind == PlanStep::Kind::kFusedDense || (st.kind == PlanStep::Kind::kOp && st.op == OpCode::kDense)))
      has_dense = true;
  }
  if (!has_dense) return false;
  for (auto& o : p.outputs)
    if (o.kind == PlanRef::Kind::kTemp && so[o.index]) return false;
  bool any_rest = false;
  for (size_t s = 0; s < n; ++s) any_rest = any_rest || !so[s];
  if (!any_rest) return false;
  // Boundary: shared-only steps read by the rest.
  std::vector<int> bidx(n, -1), pidx(n, -1), ridx(n, -1);
  prefix = ExecutablePlan{};
  prefix.shared_shapes = p.shared_shapes;
  rest = ExecutablePlan{};
  rest.shared_shapes = p.shared_shapes;
  rest.batched_shapes = p.batched_shapes;
  boundary_sizes.clear();
  for (size_t s = 0; s < n; ++s) {
    if (!so[s]) continue;
    pidx[s] = int(prefix.steps.size());
    PlanStep st = p.steps[s];
    for (auto& r : st.ins)
      if (r.kind == PlanRef::Kind::kTemp) r.index = pidx[r.index];
    for (auto& l : st.chain)
      if (l.rhs && l.rhs->kind == PlanRef::Kind::kTemp) l.rhs->index = pidx[l.rhs->index];
    prefix.steps.push_back(st);
  }
  // One boundary tensor per distinct (step, column slice) the rest reads, so a hoisted fused
  // dense exposes one (1, N_g) output per gate and the prefix launch can split its columns.
  std::map<std::tuple<int, int, int>, int> boundary;  // (step, col_off, cols) -> shared index
  (void)bidx;
  for (size_t s = 0; s < n; ++s) {
    if (so[s]) continue;
    for (auto& r : refs_of(p.steps[s]))
      if (r.kind == PlanRef::Kind::kTemp && so[r.index]) {
        auto key = std::make_tuple(r.index, r.cols >= 0 ? r.col_off : 0, r.cols);
        if (boundary.count(key)) continue;
        boundary[key] = int(rest.shared_shapes.size());
        Shape sh = p.steps[r.index].out_shape;
        if (r.cols >= 0) sh = Shape{1, r.cols};
        rest.shared_shapes.push_back(sh);
        prefix.outputs.push_back(PlanRef{PlanRef::Kind::kTemp, pidx[r.index], r.col_off, r.cols});
        boundary_sizes.push_back(sh.size());
      }
  }
  auto remap = [&](PlanRef r) {
    if (r.kind != PlanRef::Kind::kTemp) return r;
    if (so[r.index]) {
      const int idx = boundary.at(std::make_tuple(r.index, r.cols >= 0 ? r.col_off : 0, r.cols));
      r = PlanRef{PlanRef::Kind::kShared, idx, 0, -1};
    } else {
      r.index = ridx[r.index];
    }
    return r;
  };
  for (size_t s = 0; s < n; ++s) {
    if (so[s]) continue;
    ridx[s] = int(rest.steps.size());
    PlanStep st = p.steps[s];
    for (auto& r : st.ins) r = remap(r);
    for (auto& l : st.chain)
      if (l.rhs) l.rhs = remap(*l.rhs);
    rest.steps.push_back(st);
  }
  for (auto& o : p.outputs) rest.outputs.push_back(remap(o));
  return true;
}


// Splits `p` at the first step that needs a whole row of an earlier step (the dense over the
// mixed hidden state and the argmax of NestedRNN's decision cell, zoo.cpp:145-174): every step
// before it is column-local, so the head can spread over CTAs by columns, which the plan as a
// whole cannot.  Head outputs: the original outputs it computes, then the boundary temporaries
// the tail reads (each once); tail inputs: the original batched inputs, then those temporaries.
// Returns false when no split point leaves a head with a contraction.
bool split_at_reduction(const ExecutablePlan& p, ExecutablePlan& head, ExecutablePlan& tail, std::vector<int>& head_orig_out,
                        std::vector<int>& head_bnd_step, std::vector<int>& tail_in_src, std::vector<int>& tail_orig_out) {
  const size_t n = p.steps.size();
  if (p.ghost || n < 3) return false;
  auto refs_of = [&](const PlanStep& st) {
    std::vector<PlanRef> r = st.ins;
    for (auto& l : st.chain)
      if (l.rhs) r.push_back(*l.rhs);
    return r;
  };
  auto is_dense = [](const PlanStep& st) {
    return st.kind == PlanStep::Kind::kFusedDense || (st.kind == PlanStep::Kind::kOp && st.op == OpCode::kDense);
  };
  // Split point: the first dense whose row operand is a temporary and whose width differs from the
  // plan's unit (the head's first dense's width), i.e. a reduction over a whole computed row.
  int first_dense = -1;
  for (size_t s = 0; s < n; ++s)
    if (is_dense(p.steps[s])) { first_dense = int(s); break; }
  if (first_dense < 0) return false;
  int cut = -1;
  for (size_t s = size_t(first_dense) + 1; s < n; ++s) {
    const PlanStep& st = p.steps[s];
    if (is_dense(st) && st.ins[0].kind == PlanRef::Kind::kTemp) { cut = int(s); break; }
    if (st.kind == PlanStep::Kind::kOp && st.op == OpCode::kArgmax) { cut = int(s); break; }
  }
  if (cut <= first_dense) return false;
  head = ExecutablePlan{};
  head.shared_shapes = p.shared_shapes;
  head.batched_shapes = p.batched_shapes;
  for (int s = 0; s < cut; ++s) head.steps.push_back(p.steps[size_t(s)]);
  head_orig_out.clear();
  head_bnd_step.clear();
  tail_in_src.clear();
  tail_orig_out.clear();
  for (size_t k = 0; k < p.outputs.size(); ++k) {
    const PlanRef& o = p.outputs[k];
    if (o.kind == PlanRef::Kind::kTemp && o.index < cut) {
      head.outputs.push_back(o);
      head_orig_out.push_back(int(k));
    }
  }
  // Temporaries of the head the tail reads: one tail batched input per step (slices kept).
  std::map<int, int> tin;  // head step -> tail batched index
  tail = ExecutablePlan{};
  tail.shared_shapes = p.shared_shapes;
  tail.batched_shapes = p.batched_shapes;
  for (size_t s = size_t(cut); s < n; ++s)
    for (auto& r : refs_of(p.steps[s]))
      if (r.kind == PlanRef::Kind::kTemp && r.index < cut && !tin.count(r.index)) {
        tin[r.index] = int(tail.batched_shapes.size());
        tail.batched_shapes.push_back(p.steps[size_t(r.index)].out_shape);
        int src = -1;
        for (size_t k = 0; k < p.outputs.size(); ++k) {
          const PlanRef& o = p.outputs[k];
          if (o.kind == PlanRef::Kind::kTemp && o.index == r.index && o.cols < 0) src = int(k);
        }
        if (src < 0) {  // not an original output: a boundary output of the head
          src = -1 - int(head_bnd_step.size());
          head_bnd_step.push_back(r.index);
          head.outputs.push_back(PlanRef{PlanRef::Kind::kTemp, r.index, 0, -1});
        }
        tail_in_src.push_back(src);
      }
  if (tin.empty()) return false;
  auto remap = [&](PlanRef r) {
    if (r.kind != PlanRef::Kind::kTemp) return r;
    if (r.index < cut) return PlanRef{PlanRef::Kind::kBatched, tin.at(r.index), r.col_off, r.cols};
    r.index -= cut;
    return r;
  };
  for (size_t s = size_t(cut); s < n; ++s) {
    PlanStep st = p.steps[s];
    for (auto& r : st.ins) r = remap(r);
    for (auto& l : st.chain)
      if (l.rhs) l.rhs = remap(*l.rhs);
    tail.steps.push_back(st);
  }
  for (size_t k = 0; k < p.outputs.size(); ++k) {
    const PlanRef& o = p.outputs[k];
    if (o.kind == PlanRef::Kind::kTemp && o.index < cut) continue;
    tail.outputs.push_back(remap(o));
    tail_orig_out.push_back(int(k));
  }
  return !head.outputs.empty() && !tail.outputs.empty();
}
}  // namespace

DPlan compile_plan(const ExecutablePlan& p, int64_t& temp_per_inst, std::vector<Shape>& out_shapes) {
  DPlan d{};
  MBATCH_CHECK(p.steps.size() <= size_t(kMaxSteps), "plan: too many steps for the device plan VM");
  MBATCH_CHECK(p.outputs.size() <= size_t(kMaxOut), "plan: too many outputs");
  MBATCH_CHECK(p.shared_shapes.size() <= size_t(kMaxShared), "plan: too many shared inputs");
  MBATCH_CHECK(p.batched_shapes.size() <= size_t(kMaxBatched), "plan: too many batched inputs");
  d.ghost = p.ghost;
  d.nsteps = int(p.steps.size());
  d.nout = int(p.outputs.size());
  d.nshared = int(p.shared_shapes.size());
  d.nbatched = int(p.batched_shapes.size());
  int64_t off = 0;
  temp_per_inst = 0;
  for (size_t s = 0; s < p.steps.size(); ++s) {
    const PlanStep& st = p.steps[s];
    DStep& ds = d.steps[s];
    ds.kind = st.kind == PlanStep::Kind::kOp ? kStepOp : st.kind == PlanStep::Kind::kFusedDense ? kStepFused : kStepChain;
    ds.op = int(st.op);
    ds.rows = st.out_shape.rows;
    ds.cols = st.out_shape.cols;
    MBATCH_CHECK(st.ins.size() <= size_t(kMaxIn) && st.chain.size() <= size_t(kMaxChain), "plan: step too wide");
    ds.nin = int(st.ins.size());
    ds.nchain = int(st.chain.size());
    std::vector<Shape> in_shapes;
    for (size_t i = 0; i < st.ins.size(); ++i) {
      ds.ins[i] = to_dref(p, st.ins[i], s);
      in_shapes.push_back(Shape{ds.ins[i].rows_r, ds.ins[i].cols_r});
    }
    switch (st.kind) {
      case PlanStep::Kind::kOp: {
        MBATCH_CHECK(st.op != OpCode::kFill, "plan: fill is not a batched step");
        Shape expect = mbatch::backend::infer_shape(st.op, in_shapes);
        MBATCH_CHECK(expect == st.out_shape, std::string(mbatch::backend::op_name(st.op)) + ": output shape mismatch");
        break;
      }
      case PlanStep::Kind::kFusedDense: {
        MBATCH_CHECK(st.ins.size() >= 2 && in_shapes[0].rows == 1, "plan: fused dense needs (1,k) x weights");
        int total = 0;
        for (size_t w = 1; w < in_shapes.size(); ++w) {
          MBATCH_CHECK(in_shapes[w].rows == in_shapes[0].cols, "dense: shape mismatch, expected (m,k)x(k,n), got " +
                                                                    in_shapes[0].str() + " x " + in_shapes[w].str());
          total += in_shapes[w].cols;
        }
        MBATCH_CHECK(st.out_shape == (Shape{1, total}), "dense: output shape mismatch");
        break;
      }
      case PlanStep::Kind::kChain: {
        MBATCH_CHECK(st.ins.size() == 1 && in_shapes[0] == st.out_shape, "plan: chain base shape mismatch");
        for (size_t l = 0; l < st.chain.size(); ++l) {
          MBATCH_CHECK(mbatch::backend::is_elementwise(st.chain[l].op), "op not fusable in an elementwise chain");
          ds.chain[l].op = int(st.chain[l].op);
          ds.chain[l].has_rhs = st.chain[l].rhs.has_value();
          if (st.chain[l].rhs) {
            ds.chain[l].rhs = to_dref(p, *st.chain[l].rhs, s);
            MBATCH_CHECK(ds.chain[l].rhs.rows_r * ds.chain[l].rhs.cols_r == st.out_shape.size(),
                         std::string(mbatch::backend::op_name(st.chain[l].op)) + ": shape mismatch in chain");
          }
        }
        break;
      }
    }
    ds.temp_off = int32_t(off);
    off += st.out_shape.size();
  }
  d.temp_floats = int32_t(off);
  temp_per_inst = off;
  out_shapes.clear();
  for (size_t k = 0; k < p.outputs.size(); ++k) {
    MBATCH_CHECK(p.outputs[k].kind == PlanRef::Kind::kTemp, "plan outputs must be step results");
    d.outputs[k] = to_dref(p, p.outputs[k], p.steps.size());
    out_shapes.push_back(Shape{d.outputs[k].rows_r, d.outputs[k].cols_r});
  }
  split_analysis(p, d);
  return d;
}

// Set while the head / tail of a split plan are registered (they stay on the exact FP32 VM).
static thread_local bool force_vm_next = false;

// [dense(row . shared W), argmax(that row)] with the row 1 x K and W K x N (N <= 32): NestedRNN's
// decision tail after the head / tail split.  Whole operands only (no column slices).
static void detect_dense_argmax(PlanEntry& pe) {
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  static const bool off = std::getenv("MBX_NO_DENSE_ARGMAX") != nullptr;  // experiment knob
  const ExecutablePlan& p = pe.exec_plan;
  if (off || pe.tc_kind != -1 || pe.prefix_plan >= 0 || p.ghost || p.steps.size() != 2 || p.outputs.empty() || p.outputs.size() > 2) return;
  const PlanStep& d = p.steps[0];
  const PlanStep& m = p.steps[1];
  if (d.kind != PlanStep::Kind::kOp || d.op != OpCode::kDense || d.ins.size() != 2) return;
  if (m.kind != PlanStep::Kind::kOp || m.op != OpCode::kArgmax || m.ins.size() != 1) return;
  const PlanRef &a = d.ins[0], &w = d.ins[1], &r = m.ins[0];
  if (r.kind != PlanRef::Kind::kTemp || r.index != 0 || r.cols >= 0) return;
  if (w.kind != PlanRef::Kind::kShared || w.cols >= 0 || a.cols >= 0 || a.kind == PlanRef::Kind::kTemp) return;
  const auto& as = a.kind == PlanRef::Kind::kBatched ? p.batched_shapes[size_t(a.index)] : p.shared_shapes[size_t(a.index)];
  const auto& ws = p.shared_shapes[size_t(w.index)];
  if (as.rows != 1 || as.cols != ws.rows || ws.cols < 1 || ws.cols > 32) return;
  // The kernel stages W, the row and the transposed products in shared memory; larger plans keep
  // the plan VM (any K).
  if (dense_argmax_smem(ws.rows, ws.cols) > 227 * 1024) return;
  int outs[2] = {0, 0};
  for (size_t k = 0; k < p.outputs.size(); ++k) {
    const PlanRef& o = p.outputs[k];
    if (o.kind != PlanRef::Kind::kTemp || o.cols >= 0 || o.index < 0 || o.index > 1) return;
    outs[k] = o.index;
  }
  pe.da = true;
  pe.da_k = ws.rows;
  pe.da_n = ws.cols;
  pe.da_a_batched = a.kind == PlanRef::Kind::kBatched ? 1 : 0;
  pe.da_a_idx = a.index;
  pe.da_w_idx = w.index;
  pe.da_out[0] = outs[0];
  pe.da_out[1] = outs[1];
}

// MV-RNN's combine cell (proj/src/zoo.cpp:124-136): [dense(B x0, B M0), dense(B x1, B M1),
// concat of the two, dense(that, S W), optional chain of shared-row add/mul and unaries], whole
// operands only.  Runs on mv_cell_kernel (exact FP32, every precision).
static bool detect_mv_cell(PlanEntry& pe, const ExecutablePlan& p) {
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  using RK = PlanRef::Kind;
  if (p.ghost || p.outputs.size() != 1 || p.steps.size() < 4 || p.steps.size() > 5) return false;
  auto whole = [](const PlanRef& r) { return r.cols < 0; };
  auto op_step = [](const PlanStep& s, OpCode op, size_t nin) { return s.kind == PlanStep::Kind::kOp && s.op == op && s.ins.size() == nin; };
  int K = -1, N = -1;
  for (int g = 0; g < 2; ++g) {
    const PlanStep& s = p.steps[size_t(g)];
    if (!op_step(s, OpCode::kDense, 2)) return false;
    const PlanRef &x = s.ins[0], &m = s.ins[1];
    if (x.kind != RK::kBatched || m.kind != RK::kBatched || !whole(x) || !whole(m)) return false;
    const auto &xs = p.batched_shapes[size_t(x.index)], &ms = p.batched_shapes[size_t(m.index)];
    if (xs.rows != 1 || xs.cols != ms.rows) return false;
    if (g == 0) {
      K = ms.rows;
      N = ms.cols;
    } else if (ms.rows != K || ms.cols != N) {
      return false;
    }
    pe.mv_x[g] = x.index;
    pe.mv_m[g] = m.index;
  }
  const PlanStep& cat = p.steps[2];
  if (!op_step(cat, OpCode::kConcat, 2)) return false;
  const PlanRef &c0 = cat.ins[0], &c1 = cat.ins[1];
  if (c0.kind != RK::kTemp || c1.kind != RK::kTemp || !whole(c0) || !whole(c1) || c0.index + c1.index != 1) return false;
  pe.mv_first = c0.index == 0 ? 0 : 1;
  const PlanStep& d = p.steps[3];
  if (!op_step(d, OpCode::kDense, 2)) return false;
  const PlanRef &a = d.ins[0], &w = d.ins[1];
  if (a.kind != RK::kTemp || a.index != 2 || !whole(a) || w.kind != RK::kShared || !whole(w)) return false;
  const auto& ws = p.shared_shapes[size_t(w.index)];
  if (ws.rows != 2 * N) return false;
  const int U = ws.cols;
  pe.mv_w = w.index;
  pe.mv_nlinks = 0;
  int last = 3;
  if (p.steps.size() == 5) {
    const PlanStep& ch = p.steps[4];
    if (ch.kind != PlanStep::Kind::kChain || ch.ins.size() != 1 || ch.ins[0].kind != RK::kTemp || ch.ins[0].index != 3 ||
        !whole(ch.ins[0]) || ch.chain.size() > 4)
      return false;
    for (const auto& l : ch.chain) {
      int rhs = -1;
      if (l.rhs) {
        const PlanRef& r = *l.rhs;
        if (r.kind != RK::kShared || !whole(r) || p.shared_shapes[size_t(r.index)].size() != U) return false;
        if (l.op != OpCode::kAdd && l.op != OpCode::kMul) return false;
        rhs = r.index;
      } else if (l.op != OpCode::kSigmoid && l.op != OpCode::kTanh && l.op != OpCode::kRelu) {
        return false;
      }
      pe.mv_link_op[pe.mv_nlinks] = int(l.op);
      pe.mv_link_rhs[pe.mv_nlinks] = rhs;
      ++pe.mv_nlinks;
    }
    last = 4;
  }
  const PlanRef& o = p.outputs[0];
  if (o.kind != RK::kTemp || o.index != last || !whole(o)) return false;
  if (!mv_cell_supported(K, N, U)) return false;
  pe.mv_k = K;
  pe.mv_n = N;
  pe.mv_u = U;
  return true;
}

// [add(B0, B1)] over two batched matrices: the MV-RNN matrix add (zoo.cpp:135) that
// issue_pending folds into the preceding combine-cell launch of the same nodes.
static bool detect_mv_add(const ExecutablePlan& p) {
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  if (p.ghost || p.steps.size() != 1 || p.outputs.size() != 1 || p.batched_shapes.size() != 2 || !p.shared_shapes.empty()) return false;
  const PlanStep& s = p.steps[0];
  if (s.kind != PlanStep::Kind::kOp || s.op != OpCode::kAdd || s.ins.size() != 2) return false;
  for (const auto& r : s.ins)
    if (r.kind != PlanRef::Kind::kBatched || r.cols >= 0) return false;
  if (s.ins[0].index + s.ins[1].index != 1 || !(p.batched_shapes[0] == p.batched_shapes[1])) return false;
  const PlanRef& o = p.outputs[0];
  return o.kind == PlanRef::Kind::kTemp && o.index == 0 && o.cols < 0;
}

// [concat(whole 1 x c rows, shared or batched)] -> output: concat_rows_kernel.
static bool detect_concat(PlanEntry& pe, const ExecutablePlan& p) {
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  if (p.ghost || p.steps.size() != 1 || p.outputs.size() != 1) return false;
  const PlanStep& st = p.steps[0];
  if (st.kind != PlanStep::Kind::kOp || st.op != OpCode::kConcat || st.ins.size() > 8 || st.out_shape.rows != 1) return false;
  const PlanRef& o = p.outputs[0];
  if (o.kind != PlanRef::Kind::kTemp || o.index != 0 || o.cols >= 0) return false;
  pe.cat_n = 0;
  for (const auto& r : st.ins) {
    if (r.cols >= 0 || r.kind == PlanRef::Kind::kTemp) return false;
    const auto& sh = r.kind == PlanRef::Kind::kBatched ? p.batched_shapes[size_t(r.index)] : p.shared_shapes[size_t(r.index)];
    if (sh.rows != 1) return false;
    pe.cat_kind[pe.cat_n] = r.kind == PlanRef::Kind::kBatched ? 1 : 0;
    pe.cat_idx[pe.cat_n] = r.index;
    pe.cat_cols[pe.cat_n] = sh.cols;
    ++pe.cat_n;
  }
  return true;
}

int register_plan(mbx_ctx* c, const ExecutablePlan& plan) {
  std::vector<int32_t> enc = mbatch::backend::encode_plan(plan);
  auto it = c->plan_by_enc.find(enc);
  if (it != c->plan_by_enc.end()) return it->second;
  PlanEntry pe;
  pe.plan = plan;
  pe.hplan = compile_plan(plan, pe.temp_floats_per_inst, pe.out_shapes);
  pe.exec_plan = plan;
  ExecutablePlan prefix, rest;
  std::vector<int64_t> bsizes;
  if (!plan.ghost && hoist_shared_prefix(plan, prefix, rest, bsizes)) {
    pe.prefix_plan = register_plan(c, prefix);
    pe.exec_plan = rest;
    pe.prefix_sizes = bsizes;
    int64_t tmp = 0;
    std::vector<Shape> tmp_shapes;
    pe.hplan = compile_plan(rest, tmp, tmp_shapes);
    int64_t total = 0;
    for (int64_t s : bsizes) total += s;
    if (!c->dry) cuda_check(cudaMalloc(&pe.prefix_scratch, size_t(total) * sizeof(float)), "prefix scratch");
  }
  pe.mv = !force_vm_next && pe.prefix_plan < 0 && detect_mv_cell(pe, plan);
  pe.mv_add = detect_mv_add(plan);
  pe.cat = pe.prefix_plan < 0 && detect_concat(pe, plan);
  if (!plan.ghost && !pe.mv && pe.prefix_plan < 0 && pe.hplan.unit <= 0 && !force_vm_next) {
    ExecutablePlan head, tail;
    std::vector<int> hoo, hbs, tis, too;
    if (split_at_reduction(plan, head, tail, hoo, hbs, tis, too)) {
      force_vm_next = true;  // decision-feeding: exact FP32 plan VM for both halves
      const int hid = register_plan(c, head);
      const int tid = register_plan(c, tail);
      force_vm_next = false;
      const PlanEntry& hpe = c->plans[size_t(hid)];
      const PlanEntry& tpe = c->plans[size_t(tid)];
      if (hpe.hplan.unit > 0 && hpe.prefix_plan < 0 && tpe.prefix_plan < 0) {  // the head splits over columns
        pe.head_plan = hid;
        pe.tail_plan = tid;
        pe.head_nout_orig = int(hoo.size());
        pe.head_orig_out = hoo;
        pe.bnd_size.clear();
        for (int st : hbs) pe.bnd_size.push_back(plan.steps[size_t(st)].out_shape.size());
        pe.tail_in_src = tis;
        pe.tail_orig_out = too;
      }
    }
  }
  pe.force_vm = force_vm_next;
  if (!plan.ghost) {
    if (!c->dry) {
      cuda_check(cudaMalloc(&pe.dplan, sizeof(DPlan)), "plan alloc");
      cuda_check(cudaMemcpy(pe.dplan, &pe.hplan, sizeof(DPlan), cudaMemcpyHostToDevice), "plan upload");
    }
    const int64_t tf = std::max<int64_t>(1, pe.hplan.temp_floats);
    const int64_t budget = 192 * 1024 / 4;
    MBATCH_CHECK(tf <= budget, "plan: per-instance temporaries exceed shared memory");
    pe.tm = int(std::min<int64_t>(kMaxTM, std::max<int64_t>(1, budget / tf)));
    pe.smem = int(pe.tm * tf * 4);
    pe.threads = 256;
    if (pe.hplan.unit > 0) {
      pe.unit_chunk = pe.hplan.unit >= 64 ? 32 : pe.hplan.unit;
      pe.max_split = (pe.hplan.unit + pe.unit_chunk - 1) / pe.unit_chunk;
    } else {
      pe.unit_chunk = 0;
      pe.max_split = 1;
    }
    tc_prepare(c, pe);  // force_vm plans get only the bit-exact gate kernel, if any
    detect_dense_argmax(pe);
  }
  int id = int(c->plans.size());
  c->plans.push_back(std::move(pe));
  c->plan_by_enc[enc] = id;
  return id;
}

BatchLaunch prepare_batch(mbx_ctx* c, int plan_id, int b, const int64_t* shared_off,
                          const int64_t* batched_off, int gather_mode, int64_t* out_off,
                          int64_t* gather_bytes) {
  MBATCH_CHECK(b > 0, "exec_batched: empty batch");
  MBATCH_CHECK(plan_id >= 0 && size_t(plan_id) < c->plans.size(), "exec_batched: unknown plan");
  const PlanEntry& pe = c->plans[plan_id];
  const ExecutablePlan& p = pe.plan;
  BatchLaunch L;
  L.plan_id = plan_id;
  L.b = b;
  if (gather_bytes) *gather_bytes = 0;
  if (p.ghost) return L;
  const int ns = int(p.shared_shapes.size()), nb = int(p.batched_shapes.size()), no = int(p.outputs.size());
  for (int s = 0; s < ns; ++s) arena_check(c, shared_off[s], p.shared_shapes[s].size());
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < nb; ++j) arena_check(c, batched_off[int64_t(i) * nb + j], p.batched_shapes[j].size());

  // Effective node rows: the caller's, or (EXPLICIT gathers) the packed copies.
  thread_local std::vector<int64_t> eff;
  eff.assign(batched_off, batched_off + int64_t(b) * nb);
  if (gather_mode == MBX_GATHER_EXPLICIT) {
    for (int j = 0; j < nb; ++j) {
      const int64_t size = p.batched_shapes[j].size();
      bool contiguous = true;
      for (int i = 0; i + 1 < b; ++i)
        contiguous = contiguous && batched_off[int64_t(i + 1) * nb + j] == batched_off[int64_t(i) * nb + j] + size;
      if (contiguous) continue;
      const int64_t region = arena_alloc(c, int64_t(b) * size);
      std::vector<int64_t> src(b);
      for (int i = 0; i < b; ++i) {
        src[i] = batched_off[int64_t(i) * nb + j];
        eff[int64_t(i) * nb + j] = region + int64_t(i) * size;
      }
      L.gathers.push_back({int(size), meta_stage(c, src.data(), src.size() * 8), region});
      if (gather_bytes) *gather_bytes += int64_t(b) * size * int64_t(sizeof(float));
    }
  }
  thread_local std::vector<int64_t> bases;
  bases.resize(size_t(no));
  for (int k = 0; k < no; ++k) {
    const int64_t size = pe.out_shapes[k].size();
    bases[k] = arena_alloc(c, int64_t(b) * size);
    for (int i = 0; i < b; ++i) out_off[int64_t(i) * no + k] = bases[k] + int64_t(i) * size;
  }
  // Per-instance step temporaries: the reference allocates them in the arena (exec_batched.cpp:
  // 106); here they live on chip, but the offsets are reserved so every later handle offset
  // equals the reference's.
  const int64_t temps = arena_alloc(c, int64_t(b) * pe.temp_floats_per_inst);
  if (pe.head_plan >= 0) {
    // Split plan: head (columns across CTAs) then tail (per node).  The boundary tensors the tail
    // reads go into the reserved temporary region (batch-contiguous per boundary), so no
    // allocation the reference does not make.
    const PlanEntry& hp = c->plans[size_t(pe.head_plan)];
    const PlanEntry& tp = c->plans[size_t(pe.tail_plan)];
    std::vector<int64_t> bnd_base;
    int64_t cur = temps;
    for (int64_t sz : pe.bnd_size) {
      bnd_base.push_back(cur);
      cur += int64_t(b) * sz;
    }
    MBATCH_CHECK(cur <= temps + int64_t(b) * pe.temp_floats_per_inst, "split plan: boundary exceeds temporaries");
    BatchLaunch LH, LT;
    LH.plan_id = pe.head_plan;
    LH.b = b;
    LT.plan_id = pe.tail_plan;
    LT.b = b;
    LH.shared_meta = meta_stage(c, shared_off, size_t(ns) * 8);
    LH.batched_meta = meta_stage(c, eff.data(), eff.size() * 8);
    std::vector<int64_t> hout;
    for (int k : pe.head_orig_out) hout.push_back(bases[size_t(k)]);
    for (int64_t bb : bnd_base) hout.push_back(bb);
    LH.out_meta = meta_stage(c, hout.data(), hout.size() * 8);
    const int ntb = int(tp.plan.batched_shapes.size());
    std::vector<int64_t> tb(size_t(b) * ntb);
    for (int i = 0; i < b; ++i) {
      for (int j = 0; j < nb; ++j) tb[size_t(i) * ntb + j] = eff[size_t(i) * nb + j];
      for (size_t j = 0; j < pe.tail_in_src.size(); ++j) {
        const int src = pe.tail_in_src[j];
        const int64_t size = tp.plan.batched_shapes[size_t(nb) + j].size();
        const int64_t base = src >= 0 ? bases[size_t(src)] : bnd_base[size_t(-1 - src)];
        tb[size_t(i) * ntb + nb + j] = base + int64_t(i) * size;
      }
    }
    LT.shared_meta = meta_stage(c, shared_off, size_t(ns) * 8);
    LT.batched_meta = meta_stage(c, tb.data(), tb.size() * 8);
    std::vector<int64_t> tout;
    for (int k : pe.tail_orig_out) tout.push_back(bases[size_t(k)]);
    LT.out_meta = meta_stage(c, tout.data(), tout.size() * 8);
    (void)hp;
    L.sub.push_back(LH);
    L.sub.push_back(LT);
    return L;
  }
  if (pe.prefix_plan >= 0) {
    // The hoisted prefix writes its boundary tensors into the plan's scratch; the main kernel
    // reads them as extra shared inputs (offsets relative to the arena base).
    std::vector<int64_t> sh(shared_off, shared_off + ns), pouts;
    int64_t off = c->dry ? 0 : (reinterpret_cast<float*>(pe.prefix_scratch) - arena_ptr(c));
    for (int64_t s : pe.prefix_sizes) {
      sh.push_back(off);
      pouts.push_back(off);
      off += s;
    }
    L.shared_meta = meta_stage(c, sh.data(), sh.size() * 8);
    L.prefix_out_meta = meta_stage(c, pouts.data(), pouts.size() * 8);
  } else {
    L.shared_meta = meta_stage(c, shared_off, size_t(ns) * 8);
  }
  L.batched_meta = meta_stage(c, eff.data(), eff.size() * 8);
  L.out_meta = meta_stage(c, bases.data(), bases.size() * 8);
  return L;
}

// Shared-memory floats the plan VM may use to stage shared weights (after its temps): up to
// 128 KiB, within the 227 KiB per-CTA limit.
static int vm_weight_stage_floats(int temp_floats) {
  const int budget = (227 * 1024) / 4 - 256 - ((temp_floats + 3) & ~3);
  return std::max(0, std::min(budget, 32 * 1024));
}

// The hoisted all-shared prefix of a plan (e.g. the TreeLSTM leaf cell's [hz|hz] . W), computed
// once per parameter upload; issued before the batch (or the fused launch) that reads it.
void issue_prefix(mbx_ctx* c, const BatchLaunch& L) {
  PlanEntry& pe = c->plans[L.plan_id];
  float* arena = arena_ptr(c);
  bool prefix_cached = false;
  if (pe.prefix_plan >= 0) {
    // The prefix reads shared inputs only; if they are all session parameters its result is a
    // function of the parameters alone and the scratch still holds it.
    const PlanEntry& pp = c->plans[pe.prefix_plan];
    const int64_t* sh = reinterpret_cast<const int64_t*>(c->meta.host + L.shared_meta);
    std::vector<int64_t> key;
    bool persistent = true;
    for (size_t k = 0; k < pp.plan.shared_shapes.size(); ++k) {
      key.push_back(sh[k]);
      persistent = persistent && sh[k] + pp.plan.shared_shapes[k].size() <= c->persist_end;
    }
    key.push_back(int64_t(c->upload_epoch));
    prefix_cached = persistent && key == pe.prefix_key;
    pe.prefix_key = persistent ? key : std::vector<int64_t>{};
  }
  if (pe.prefix_plan >= 0 && !prefix_cached) {
    const PlanEntry& pp = c->plans[pe.prefix_plan];
    VmLaunch v{};
    v.plan = pp.dplan;
    v.arena = arena;
    v.b = 1;
    v.tm = 1;
    v.nsplit = pp.max_split;
    v.unit_chunk = pp.max_split > 1 ? pp.unit_chunk : pp.hplan.unit;
    if (pp.max_split > 1) {  // spread the one-row contraction over ~148 CTAs
      const int unit = pp.hplan.unit;
      v.unit_chunk = std::max(8, ((unit + 147) / 148 + 7) / 8 * 8);
      v.nsplit = (unit + v.unit_chunk - 1) / v.unit_chunk;
    }
    v.threads = pp.threads;
    v.temp_floats_total = int(std::max<int64_t>(1, pp.hplan.temp_floats));
    v.wst_floats = vm_weight_stage_floats(v.temp_floats_total);
    v.smem_bytes = (((v.temp_floats_total + 3) & ~3) + v.wst_floats) * 4;
    v.shared_off = meta_dev<int64_t>(c, L.shared_meta);
    v.batched_off = nullptr;
    v.out_base = meta_dev<int64_t>(c, L.prefix_out_meta);
    cuda_check(launch_plan_vm(v, c->stream), "shared prefix");
    ++c->launches;
    ++g_launches;
  }
}

// The MV-RNN combine cell, and with `add` the next batch's matrix add over the same nodes.
static void issue_mv(mbx_ctx* c, const BatchLaunch& L, const BatchLaunch* add) {
  PlanEntry& pe = c->plans[L.plan_id];
  MvCellLaunch m{};
  m.arena = arena_ptr(c);
  m.shared_off = meta_dev<int64_t>(c, L.shared_meta);
  m.batched_off = meta_dev<int64_t>(c, L.batched_meta);
  m.b = L.b;
  m.nb = int(pe.exec_plan.batched_shapes.size());
  for (int g = 0; g < 2; ++g) {
    m.x[g] = pe.mv_x[g];
    m.m[g] = pe.mv_m[g];
  }
  m.first = pe.mv_first;
  m.w = pe.mv_w;
  m.K = pe.mv_k;
  m.N = pe.mv_n;
  m.U = pe.mv_u;
  m.nlinks = pe.mv_nlinks;
  for (int l = 0; l < 4; ++l) {
    m.link_op[l] = pe.mv_link_op[l];
    m.link_rhs[l] = pe.mv_link_rhs[l];
  }
  m.cell_out = meta_dev<int64_t>(c, L.out_meta);
  m.add_out = add ? meta_dev<int64_t>(c, add->out_meta) : nullptr;
  // W^T: transposed once per parameter upload when W is a session parameter, else per launch.
  const int64_t w_off = reinterpret_cast<const int64_t*>(c->meta.host + L.shared_meta)[pe.mv_w];
  const bool persistent = w_off + int64_t(2) * pe.mv_n * pe.mv_u <= c->persist_end;
  if (!pe.mv_wt) cuda_check(cudaMalloc(&pe.mv_wt, mv_wt_floats(pe.mv_n, pe.mv_u) * sizeof(float)), "mv W^T");
  const std::vector<int64_t> key{w_off, int64_t(c->upload_epoch)};
  const bool fresh = !persistent || pe.mv_wt_key != key;
  if (fresh) {
    cuda_check(launch_mv_transpose(arena_ptr(c) + w_off, pe.mv_wt, pe.mv_n, pe.mv_u, c->stream), "mv W^T");
    ++c->launches;
    ++g_launches;
  }
  pe.mv_wt_key = persistent ? key : std::vector<int64_t>{};
  m.wt = pe.mv_wt;
  // PDL (the W^T slice streams in while the previous kernel finishes) unless that kernel wrote
  // W^T or arbitrary arena tensors.
  m.pdl = pdl_enabled() && !fresh && c->write_launch != c->launches;
  cuda_check(launch_mv_cell(m, c->stream), "mv cell");
  ++c->launches;
  ++g_launches;
}

// Whether batch `a` (an [add(B0, B1)] plan) adds exactly the two matrices combine-cell batch `L`
// reads, node for node (the MV-RNN add one depth after the cell, zoo.cpp:134-135).
static bool mv_pair(const mbx_ctx* c, const BatchLaunch& L, const BatchLaunch& a) {
  const PlanEntry& pe = c->plans[L.plan_id];
  const PlanEntry& pa = c->plans[a.plan_id];
  if (!pe.mv || !pa.mv_add || a.b != L.b || !L.gathers.empty() || !a.gathers.empty()) return false;
  if (a.shadow_out != 0 || a.img_slot >= 0) return false;  // a later tensor-core level gathers its rows
  if (!(pa.plan.batched_shapes[0] == mbatch::backend::Shape{pe.mv_k, pe.mv_n})) return false;
  const int nb = int(pe.exec_plan.batched_shapes.size());
  const int64_t* cb = reinterpret_cast<const int64_t*>(c->meta.host + L.batched_meta);
  const int64_t* ab = reinterpret_cast<const int64_t*>(c->meta.host + a.batched_meta);
  for (int i = 0; i < L.b; ++i) {
    const int64_t m0 = cb[int64_t(i) * nb + pe.mv_m[0]], m1 = cb[int64_t(i) * nb + pe.mv_m[1]];
    const int64_t a0 = ab[2 * int64_t(i)], a1 = ab[2 * int64_t(i) + 1];
    if (!((a0 == m0 && a1 == m1) || (a0 == m1 && a1 == m0))) return false;  // fp32 + is commutative
  }
  return true;
}

int issue_batches(mbx_ctx* c, const std::vector<BatchLaunch>& Ls, size_t i) {
  if (!c->dry && i + 1 < Ls.size() && mv_pair(c, Ls[i], Ls[i + 1])) {
    issue_mv(c, Ls[i], &Ls[i + 1]);
    return 2;
  }
  issue_batch(c, Ls[i]);
  return 1;
}

static bool leaf_mergeable(const mbx_ctx* c, const BatchLaunch& L) {
  const PlanEntry& pe = c->plans[size_t(L.plan_id)];
  if (pe.plan.ghost || !L.gathers.empty() || !L.sub.empty() || pe.prefix_plan >= 0 || L.shadow_out != 0 ||
      L.img_slot >= 0 || L.out_node)
    return false;
  if (pe.da) return pe.tc_kind < 0 && !pe.tc_small && !pe.tc_exact;  // issue_batch's dense + argmax branch
  return tc_small_kernel(pe);
}

bool mergeable(const mbx_ctx* c, const BatchLaunch& L) {
  if (!L.sub.empty()) {
    if (!L.gathers.empty()) return false;
    for (const auto& S : L.sub)
      if (!leaf_mergeable(c, S)) return false;
    return true;
  }
  return leaf_mergeable(c, L);
}

bool same_shared(const mbx_ctx* c, const BatchLaunch& a, const BatchLaunch& b) {
  if (a.plan_id != b.plan_id || a.sub.size() != b.sub.size()) return false;
  if (!a.sub.empty()) {
    for (size_t s = 0; s < a.sub.size(); ++s)
      if (!same_shared(c, a.sub[s], b.sub[s])) return false;
    return true;
  }
  const size_t ns = c->plans[size_t(a.plan_id)].exec_plan.shared_shapes.size();
  return std::memcmp(c->meta.host + a.shared_meta, c->meta.host + b.shared_meta, ns * 8) == 0;
}

BatchLaunch merge_launches(mbx_ctx* c, const std::vector<const BatchLaunch*>& g) {
  MBATCH_CHECK(!g.empty(), "merge_launches: empty group");
  const BatchLaunch& f = *g[0];
  BatchLaunch M;
  M.plan_id = f.plan_id;
  for (const BatchLaunch* L : g) M.b += L->b;
  if (!f.sub.empty()) {  // split plan: merge the heads and the tails
    for (size_t s = 0; s < f.sub.size(); ++s) {
      std::vector<const BatchLaunch*> part;
      for (const BatchLaunch* L : g) part.push_back(&L->sub[s]);
      M.sub.push_back(merge_launches(c, part));
    }
    return M;
  }
  const PlanEntry& pe = c->plans[size_t(f.plan_id)];
  const size_t nb = pe.exec_plan.batched_shapes.size(), no = pe.out_shapes.size();
  std::vector<int64_t> rows, outs;
  rows.reserve(size_t(M.b) * nb);
  outs.reserve(size_t(M.b) * no);
  for (const BatchLaunch* L : g) {
    const int64_t* b = reinterpret_cast<const int64_t*>(c->meta.host + L->batched_meta);
    rows.insert(rows.end(), b, b + size_t(L->b) * nb);
    const int64_t* o = reinterpret_cast<const int64_t*>(c->meta.host + L->out_meta);
    for (int i = 0; i < L->b; ++i)
      for (size_t k = 0; k < no; ++k) outs.push_back(o[k] + int64_t(i) * pe.out_shapes[k].size());
  }
  M.shared_meta = f.shared_meta;
  M.out_meta = f.out_meta;
  M.batched_meta = meta_stage(c, rows.data(), rows.size() * 8);
  M.out_node_meta = meta_stage(c, outs.data(), outs.size() * 8);
  M.out_node = true;
  return M;
}

void issue_pending(mbx_ctx* c) {
  std::vector<BatchLaunch> Ls;
  Ls.swap(c->pending);
  if (Ls.empty()) return;
  std::vector<LevelsRun> runs;
  std::vector<int> run_at(Ls.size(), -1);
  for (size_t i = 0; i < Ls.size();) {
    LevelsRun r;
    r.start = int(i);
    r.n = plan_levels(c, Ls, i, &r.table, &r.groups, &r.cfg);
    if (r.n >= 1) {
      run_at[i] = int(runs.size());
      runs.push_back(r);
      i += size_t(r.n);
    } else {
      ++i;
    }
  }
  plan_shadows(c, Ls, runs);
  meta_commit(c);
  for (size_t i = 0; i < Ls.size();) {
    if (run_at[i] >= 0) {
      const LevelsRun& r = runs[size_t(run_at[i])];
      issue_levels(c, Ls, i, r.n, r.table, r.groups, r.cfg);
      i += size_t(r.n);
    } else {
      i += size_t(issue_batches(c, Ls, i));
    }
  }
}

void issue_batch(mbx_ctx* c, const BatchLaunch& L) {
  const PlanEntry& pe = c->plans[L.plan_id];
  if (pe.plan.ghost || c->dry) return;
  float* arena = arena_ptr(c);
  for (const auto& g : L.gathers) {
    cuda_check(launch_gather_rows(arena, meta_dev<int64_t>(c, g.src_meta), g.dst, L.b, g.size, c->stream), "gather");
    ++c->launches;
    ++g_launches;
  }
  if (!L.sub.empty()) {  // split plan: head, then tail
    for (const auto& S : L.sub) issue_batch(c, S);
    return;
  }
  issue_prefix(c, L);
  if (pe.mv) {
    issue_mv(c, L, nullptr);
    return;
  }
  if (pe.cat) {
    ConcatLaunch cl{};
    cl.shared_off = meta_dev<int64_t>(c, L.shared_meta);
    cl.batched_off = meta_dev<int64_t>(c, L.batched_meta);
    cl.out_base = meta_dev<int64_t>(c, L.out_meta);
    cl.b = L.b;
    cl.nb = int(pe.exec_plan.batched_shapes.size());
    cl.nin = pe.cat_n;
    cl.width = int(pe.out_shapes[0].cols);
    for (int k = 0; k < pe.cat_n; ++k) {
      cl.kind[k] = pe.cat_kind[k];
      cl.idx[k] = pe.cat_idx[k];
      cl.cols[k] = pe.cat_cols[k];
    }
    cuda_check(launch_concat_rows(arena, cl, c->stream), "concat");
    ++c->launches;
    ++g_launches;
    return;
  }
  // tc_kind 2 (pointwise) is exact and runs in every precision; tc_kind 1 (tensor cores) only
  // when the context allows split-bf16 / bf16 contractions.
  // The bit-exact gate kernel runs for small / decision plans in every precision and for every
  // gate plan in FP32 contexts; pointwise plans always; tensor cores in the other precisions.
  // BF16X6 runs the tensor cores only in persistent levels runs (3-part operands); its single
  // batches take the exact kernels like FP32.
  const bool exact_batches = c->precision == MBX_PREC_FP32 || c->precision == MBX_PREC_BF16X6;
  if (pe.tc_kind == 2 || pe.tc_small || (pe.tc_exact && exact_batches) || (!exact_batches && pe.tc_kind == 1)) {
    cuda_check(tc_launch(c, pe, L), "tensor-core plan kernel");
    ++c->launches;
    ++g_launches;
    return;
  }
  if (pe.da) {
    // PDL (W streams in while the previous kernel finishes) when W is a session parameter and the
    // previous kernel did not write arena tensors.
    const int64_t w_off = reinterpret_cast<const int64_t*>(c->meta.host + L.shared_meta)[pe.da_w_idx];
    const int da_pdl = pdl_enabled() && w_off + int64_t(pe.da_k) * pe.da_n <= c->persist_end && c->write_launch != c->launches;
    cuda_check(launch_dense_argmax(arena, meta_dev<int64_t>(c, L.shared_meta), meta_dev<int64_t>(c, L.batched_meta),
                                   L.b, int(pe.exec_plan.batched_shapes.size()), pe.da_a_batched, pe.da_a_idx,
                                   pe.da_w_idx, pe.da_k, pe.da_n, meta_dev<int64_t>(c, L.out_meta),
                                   L.out_node ? meta_dev<int64_t>(c, L.out_node_meta) : nullptr,
                                   int(pe.exec_plan.outputs.size()), pe.da_out[0], pe.da_out[1], da_pdl, c->stream),
               "dense + argmax");
    ++c->launches;
    ++g_launches;
    return;
  }
  VmLaunch v{};
  v.plan = pe.dplan;
  v.arena = arena;
  v.b = L.b;
  // Node tile: as many nodes per CTA as fill ~one wave (weight-tile reuse), no more; a plan that
  // splits over columns keeps every split and grows the node tile instead (each CTA streams its
  // weight slice once per tile, so one node per CTA would re-read the weights per node).
  v.tm = pe.max_split > 1 ? std::clamp((L.b * pe.max_split + 295) / 296, 1, pe.tm) : std::clamp((L.b + 147) / 148, 1, pe.tm);
  const int ntiles = (L.b + v.tm - 1) / v.tm;
  // Column tiles: enough CTAs for ~2 waves over 148 SMs, and together they must cover the unit.
  v.nsplit = pe.max_split > 1 ? std::clamp((296 + ntiles - 1) / ntiles, 1, pe.max_split) : 1;
  if (v.nsplit > 1) {
    const int unit = pe.hplan.unit;
    v.unit_chunk = ((unit + v.nsplit - 1) / v.nsplit + 7) / 8 * 8;
    v.nsplit = (unit + v.unit_chunk - 1) / v.unit_chunk;
  } else {
    v.unit_chunk = pe.hplan.unit;
  }
  v.threads = pe.threads;
  // Temporaries of the tile this launch actually uses (pe.smem is sized for the largest tile):
  // the rest of shared memory stages weights.
  v.temp_floats_total = int(std::max<int64_t>(1, pe.hplan.temp_floats)) * v.tm;
  v.wst_floats = vm_weight_stage_floats(v.temp_floats_total);
  v.smem_bytes = (((v.temp_floats_total + 3) & ~3) + v.wst_floats) * 4;
  v.shared_off = meta_dev<int64_t>(c, L.shared_meta);
  v.batched_off = meta_dev<int64_t>(c, L.batched_meta);
  v.out_base = meta_dev<int64_t>(c, L.out_meta);
  cuda_check(launch_plan_vm(v, c->stream), "plan VM");
  ++c->launches;
  ++g_launches;
}

}  // namespace mbx

// =============================================================================================
// mbatch::backend C++ surface

namespace mbatch {
namespace backend {

const char* op_name(OpCode op) {
  switch (op) {
    case OpCode::kDense: return "dense";
    case OpCode::kAdd: return "add";
    case OpCode::kMul: return "mul";
    case OpCode::kSigmoid: return "sigmoid";
    case OpCode::kTanh: return "tanh";
    case OpCode::kRelu: return "relu";
    case OpCode::kConcat: return "concat";
    case OpCode::kArgmax: return "argmax";
    case OpCode::kFill: return "fill";
  }
  return "?";
}

bool is_elementwise(OpCode op) {
  switch (op) {
    case OpCode::kAdd: case OpCode::kMul: case OpCode::kSigmoid: case OpCode::kTanh: case OpCode::kRelu:
      return true;
    default:
      return false;
  }
}

int op_arity(OpCode op) {
  switch (op) {
    case OpCode::kDense: case OpCode::kAdd: case OpCode::kMul: case OpCode::kConcat: return 2;
    case OpCode::kSigmoid: case OpCode::kTanh: case OpCode::kRelu: case OpCode::kArgmax: return 1;
    case OpCode::kFill: return 0;
  }
  return -1;
}

std::string Shape::str() const {
  std::ostringstream os;
  os << "(" << rows << ", " << cols << ")";
  return os.str();
}

Shape infer_shape(OpCode op, const std::vector<Shape>& in) {
  MBATCH_CHECK(static_cast<int>(in.size()) == op_arity(op), std::string(op_name(op)) + ": bad arity");
  switch (op) {
    case OpCode::kDense:
      MBATCH_CHECK(in[0].cols == in[1].rows, std::string("dense: shape mismatch, expected (m,k)x(k,n), got ") +
                                                  in[0].str() + " x " + in[1].str());
      return Shape{in[0].rows, in[1].cols};
    case OpCode::kAdd:
    case OpCode::kMul:
      MBATCH_CHECK(in[0] == in[1], std::string(op_name(op)) + ": shape mismatch, expected " + in[0].str() +
                                       ", actual " + in[1].str());
      return in[0];
    case OpCode::kSigmoid: case OpCode::kTanh: case OpCode::kRelu:
      return in[0];
    case OpCode::kConcat:
      MBATCH_CHECK(in[0].rows == in[1].rows, std::string("concat: row mismatch, ") + in[0].str() + " vs " + in[1].str());
      return Shape{in[0].rows, in[0].cols + in[1].cols};
    case OpCode::kArgmax:
      MBATCH_CHECK(in[0].rows == 1, "argmax: expected a (1,n) tensor, got " + in[0].str());
      return Shape{1, 1};
    case OpCode::kFill:
      return Shape{};
  }
  throw Error("unknown op");
}

static void put_ref(std::vector<int32_t>& e, const PlanRef& r) {
  e.push_back(r.kind == PlanRef::Kind::kShared ? 0 : r.kind == PlanRef::Kind::kBatched ? 1 : 2);
  e.push_back(r.index);
  e.push_back(r.col_off);
  e.push_back(r.cols);
}

std::vector<int32_t> encode_plan(const ExecutablePlan& p) {
  std::vector<int32_t> e;
  e.push_back(p.ghost ? 1 : 0);
  e.push_back(int32_t(p.shared_shapes.size()));
  for (auto& s : p.shared_shapes) { e.push_back(s.rows); e.push_back(s.cols); }
  e.push_back(int32_t(p.batched_shapes.size()));
  for (auto& s : p.batched_shapes) { e.push_back(s.rows); e.push_back(s.cols); }
  e.push_back(int32_t(p.steps.size()));
  for (auto& st : p.steps) {
    e.push_back(st.kind == PlanStep::Kind::kOp ? 0 : st.kind == PlanStep::Kind::kFusedDense ? 1 : 2);
    e.push_back(int32_t(st.op));
    e.push_back(st.out_shape.rows);
    e.push_back(st.out_shape.cols);
    e.push_back(int32_t(st.ins.size()));
    for (auto& r : st.ins) put_ref(e, r);
    e.push_back(int32_t(st.chain.size()));
    for (auto& l : st.chain) {
      e.push_back(int32_t(l.op));
      e.push_back(l.rhs ? 1 : 0);
      put_ref(e, l.rhs ? *l.rhs : PlanRef{});
    }
  }
  e.push_back(int32_t(p.outputs.size()));
  for (auto& r : p.outputs) put_ref(e, r);
  return e;
}

ExecutablePlan decode_plan(const int32_t* e, int64_t n) {
  int64_t i = 0;
  auto get = [&]() -> int32_t {
    MBATCH_CHECK(i < n, "plan encoding truncated");
    return e[i++];
  };
  auto ref = [&]() {
    PlanRef r;
    int k = get();
    MBATCH_CHECK(k >= 0 && k <= 2, "plan encoding: bad ref kind");
    r.kind = k == 0 ? PlanRef::Kind::kShared : k == 1 ? PlanRef::Kind::kBatched : PlanRef::Kind::kTemp;
    r.index = get();
    r.col_off = get();
    r.cols = get();
    return r;
  };
  auto op = [&]() {
    int o = get();
    MBATCH_CHECK(o >= 0 && o <= 8, "plan encoding: bad op");
    return OpCode(o);
  };
  ExecutablePlan p;
  p.ghost = get() != 0;
  int ns = get();
  for (int k = 0; k < ns; ++k) { int r = get(); int c = get(); p.shared_shapes.push_back({r, c}); }
  int nb = get();
  for (int k = 0; k < nb; ++k) { int r = get(); int c = get(); p.batched_shapes.push_back({r, c}); }
  int nst = get();
  for (int s = 0; s < nst; ++s) {
    PlanStep st;
    int k = get();
    MBATCH_CHECK(k >= 0 && k <= 2, "plan encoding: bad step kind");
    st.kind = k == 0 ? PlanStep::Kind::kOp : k == 1 ? PlanStep::Kind::kFusedDense : PlanStep::Kind::kChain;
    st.op = op();
    st.out_shape.rows = get();
    st.out_shape.cols = get();
    int nin = get();
    for (int q = 0; q < nin; ++q) st.ins.push_back(ref());
    int nc = get();
    for (int q = 0; q < nc; ++q) {
      ChainLink l;
      l.op = op();
      int has = get();
      PlanRef r = ref();
      if (has) l.rhs = r;
      st.chain.push_back(l);
    }
    p.steps.push_back(std::move(st));
  }
  int no = get();
  for (int k = 0; k < no; ++k) p.outputs.push_back(ref());
  MBATCH_CHECK(i == n, "plan encoding has trailing data");
  return p;
}

// ---- Arena ------------------------------------------------------------------------------------

static void throw_if(int rc, mbx_ctx* c) {
  if (rc != 0) throw Error(mbx_last_error(c));
}

static int env_precision() {
  const char* e = std::getenv("MBX_PRECISION");
  if (!e || std::strcmp(e, "fp32") == 0) return MBX_PREC_FP32;
  if (std::strcmp(e, "bf16x3") == 0) return MBX_PREC_BF16X3;
  if (std::strcmp(e, "bf16") == 0) return MBX_PREC_BF16;
  if (std::strcmp(e, "bf16x6") == 0) return MBX_PREC_BF16X6;
  throw Error(std::string("MBX_PRECISION: unknown precision ") + e);
}
Arena::Arena(int64_t initial_capacity) : owned_(true) {
  (void)initial_capacity;  // HBM is mapped on demand; offsets never move
  const char* dev = std::getenv("MBX_DEVICE");
  mbx_ctx* c = nullptr;
  if (mbx_ctx_create(dev ? std::atoi(dev) : 0, env_precision(), &c) != 0) throw Error(mbx_last_error(nullptr));
  ctx_ = c;
}
Arena::Arena(Device d) : owned_(true) {
  mbx_ctx* c = nullptr;
  if (mbx_ctx_create(d.id, d.precision, &c) != 0) throw Error(mbx_last_error(nullptr));
  ctx_ = c;
}
Float* Arena::ptr(const TensorHandle& h) {
  check(h);
  float* p = nullptr;
  throw_if(mbx_arena_device_ptr(ctx_, h.offset, h.size(), &p), ctx_);
  return p;
}
const Float* Arena::ptr(const TensorHandle& h) const { return const_cast<Arena*>(this)->ptr(h); }
std::vector<long> Arena::read_ints(const std::vector<TensorHandle>& hs) const {
  std::vector<int64_t> offs, vals(hs.size());
  for (const auto& h : hs) {
    check(h);
    offs.push_back(h.offset);
  }
  throw_if(mbx_read_ints(ctx_, offs.data(), int(offs.size()), vals.data()), ctx_);
  return std::vector<long>(vals.begin(), vals.end());
}
FlushScope::FlushScope(Arena& a) : a_(a) { throw_if(mbx_flush_begin(a.ctx()), a.ctx()); }
FlushScope::~FlushScope() noexcept(false) {
  const int rc = mbx_flush_end(a_.ctx());
  if (rc != 0 && !std::uncaught_exceptions()) throw Error(mbx_last_error(a_.ctx()));
}
Arena::~Arena() {
  if (owned_) mbx_ctx_destroy(ctx_);
}
TensorHandle Arena::alloc(Shape shape) {
  int64_t off = 0;
  throw_if(mbx_arena_alloc(ctx_, shape.rows, shape.cols, &off), ctx_);
  return TensorHandle{off, shape};
}
int64_t Arena::used() const { return mbx_arena_used(ctx_); }
void Arena::check(const TensorHandle& h) const {
  MBATCH_CHECK(h.valid() && h.offset + h.size() <= used(), "tensor handle out of arena bounds");
}
void Arena::upload(const TensorHandle& h, const Float* src) {
  check(h);
  throw_if(mbx_arena_upload(ctx_, h.offset, src, h.size()), ctx_);
}
void Arena::download(const TensorHandle& h, Float* dst) const {
  check(h);
  throw_if(mbx_arena_download(ctx_, h.offset, dst, h.size()), ctx_);
}
std::vector<Float> Arena::read(const TensorHandle& h) const {
  std::vector<Float> v(h.size());
  download(h, v.data());
  return v;
}
void Arena::sync() const { throw_if(mbx_sync(ctx_), ctx_); }

void exec_primop(Arena& arena, OpCode op, const std::vector<TensorHandle>& inputs, const TensorHandle& out,
                 Float fill_value) {
  std::vector<int64_t> offs;
  std::vector<int> rows, cols;
  for (auto& h : inputs) {
    offs.push_back(h.offset);
    rows.push_back(h.shape.rows);
    cols.push_back(h.shape.cols);
  }
  throw_if(mbx_exec_primop(arena.ctx(), int(op), int(inputs.size()), offs.data(), rows.data(), cols.data(),
                           out.offset, out.shape.rows, out.shape.cols, fill_value),
           arena.ctx());
}

BatchedResult exec_batched(Arena& arena, const ExecutablePlan& plan, const std::vector<BatchedCall>& instances,
                           GatherMode mode) {
  MBATCH_CHECK(!instances.empty(), "exec_batched: empty batch");
  BatchedResult res;
  if (plan.ghost) {
    res.outputs.resize(instances.size());
    return res;
  }
  const size_t b = instances.size();
  const BatchedCall& first = instances[0];
  MBATCH_CHECK(first.shared.size() == plan.shared_shapes.size() && first.batched.size() == plan.batched_shapes.size(),
               "exec_batched: arity mismatch");
  for (size_t i = 1; i < b; ++i)
    for (size_t s = 0; s < first.shared.size(); ++s)
      MBATCH_CHECK(instances[i].shared[s] == first.shared[s],
                   "shared-param handle mismatch across instances (analysis bug)");
  for (size_t s = 0; s < first.shared.size(); ++s)
    MBATCH_CHECK(first.shared[s].shape == plan.shared_shapes[s], "exec_batched: shared input shape mismatch, expected " +
                                                                     plan.shared_shapes[s].str() + ", actual " +
                                                                     first.shared[s].shape.str());
  std::vector<int64_t> shared, batched;
  for (auto& call : instances)
    for (auto& h : call.shared) shared.push_back(h.offset);
  for (auto& call : instances) {
    MBATCH_CHECK(call.batched.size() == plan.batched_shapes.size(), "exec_batched: arity mismatch");
    for (size_t j = 0; j < call.batched.size(); ++j) {
      MBATCH_CHECK(call.batched[j].shape == plan.batched_shapes[j], "exec_batched: batched input shape mismatch, expected " +
                                                                        plan.batched_shapes[j].str() + ", actual " +
                                                                        call.batched[j].shape.str());
      batched.push_back(call.batched[j].offset);
    }
  }
  mbx_ctx* c = arena.ctx();
  std::vector<int32_t> enc = encode_plan(plan);
  int pid = -1;
  throw_if(mbx_plan_register(c, enc.data(), int64_t(enc.size()), &pid), c);
  std::vector<int64_t> outs(b * plan.outputs.size());
  int64_t gb = 0;
  throw_if(mbx_exec_batched(c, pid, int(b), shared.data(), batched.data(),
                            mode == GatherMode::kFused ? MBX_GATHER_FUSED : MBX_GATHER_EXPLICIT, outs.data(), &gb),
           c);
  res.gather_bytes = gb;
  const auto& shapes = c->plans[pid].out_shapes;
  res.outputs.resize(b);
  for (size_t i = 0; i < b; ++i)
    for (size_t k = 0; k < plan.outputs.size(); ++k)
      res.outputs[i].push_back(TensorHandle{outs[i * plan.outputs.size() + k], shapes[k]});
  return res;
}

}  // namespace backend
}  // namespace mbatch
