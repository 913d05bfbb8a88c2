// runtime.cpp — the lazy batching executor on the device: fibers build per-instance DFGs with
// inline depths; when every fiber is blocked the pending window is scheduled by depth and each
// batch becomes one device launch over the HBM arena.
//
// Reference behaviour reproduced (proj/src/executor.cpp, proj/src/schedule.cpp):
//   run loop / sync points / deadlock checks ..... executor.cpp:161-220
//   inline depth + memoised all-shared blocks ..... executor.cpp:368-427
//   flush window, batch formation, launches ....... executor.cpp:711-758
//   schedule_depth / schedule_agenda .............. schedule.cpp:13-138
// Device-side differences: inputs are staged once per mini-batch into pinned memory and copied
// with one H2D transfer; every flush stages all of its offset tables, commits them with one H2D
// copy and then issues its batches back to back; scalar decisions and final outputs are packed
// on the device and read back with one D2H copy each.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cstring>
#include <unordered_map>

#include "ctx.h"
#include "exec.h"

namespace mbatch {
namespace runtime {

// ---- coroutine frame pool (exec.h) ---------------------------------------------------------
namespace {
struct FramePool {
  static constexpr size_t kClass = 64, kClasses = 64;  // 64-byte classes up to 4 KiB
  std::vector<void*> free_[kClasses];
  ~FramePool() {
    for (auto& v : free_)
      for (void* p : v) ::operator delete(p);
  }
};
thread_local FramePool g_frames;
}  // namespace

void* frame_alloc(size_t bytes) {
  const size_t c = (bytes + FramePool::kClass - 1) / FramePool::kClass;
  if (c < FramePool::kClasses) {
    auto& v = g_frames.free_[c];
    if (!v.empty()) {
      void* p = v.back();
      v.pop_back();
      return p;
    }
    return ::operator new(c * FramePool::kClass);
  }
  return ::operator new(bytes);
}

void frame_free(void* p, size_t bytes) noexcept {
  const size_t c = (bytes + FramePool::kClass - 1) / FramePool::kClass;
  if (c < FramePool::kClasses) {
    try {
      g_frames.free_[c].push_back(p);
      return;
    } catch (...) {
    }
  }
  ::operator delete(p);
}


// ---------------------------------------------------------------------------------------------
// Host values (proj/src/pipeline.cpp:9-63)

HostValue HostValue::tensor(Shape s, std::vector<float> d) {
  HostValue v;
  v.kind = Kind::kTensor;
  v.shape = s;
  v.data = std::move(d);
  MBATCH_CHECK(static_cast<int>(v.data.size()) == s.size(), "host tensor size mismatch");
  return v;
}
HostValue HostValue::scalar(long x) { HostValue v; v.kind = Kind::kInt; v.ival = x; return v; }
HostValue HostValue::list(std::vector<HostValue> items) { HostValue v; v.kind = Kind::kList; v.items = std::move(items); return v; }
HostValue HostValue::tuple(std::vector<HostValue> items) { HostValue v; v.kind = Kind::kTuple; v.items = std::move(items); return v; }
HostValue HostValue::adt(std::string ctor, std::vector<HostValue> fields) {
  HostValue v;
  v.kind = Kind::kAdt;
  v.ctor = std::move(ctor);
  v.items = std::move(fields);
  return v;
}

bool bitwise_equal(const HostValue& a, const HostValue& b) {
  if (a.kind != b.kind) return false;
  switch (a.kind) {
    case HostValue::Kind::kTensor:
      return a.shape == b.shape && a.data.size() == b.data.size() &&
             std::memcmp(a.data.data(), b.data.data(), a.data.size() * sizeof(float)) == 0;
    case HostValue::Kind::kInt: return a.ival == b.ival;
    case HostValue::Kind::kFloat: return std::memcmp(&a.fval, &b.fval, sizeof(double)) == 0;
    default:
      if (a.ctor != b.ctor || a.items.size() != b.items.size()) return false;
      for (size_t i = 0; i < a.items.size(); ++i)
        if (!bitwise_equal(a.items[i], b.items[i])) return false;
      return true;
  }
}

// ---------------------------------------------------------------------------------------------
// Schedulers

namespace {

// Shared-argument identity (schedule.cpp:13-25): FNV-1a over (node+1, out, offset+1) per ref.
uint64_t shared_key(const DFGNode& n) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    h ^= v;
    h *= 1099511628211ull;
  };
  for (const auto& r : n.shared_ins) {
    mix(static_cast<uint64_t>(r.node + 1));
    mix(static_cast<uint64_t>(r.out));
    mix(static_cast<uint64_t>(r.handle.offset + 1));
  }
  return h;
}

struct DepthKey {
  int phase, depth, sig;
  uint64_t shared;
  bool operator<(const DepthKey& o) const {
    if (phase != o.phase) return phase < o.phase;
    if (depth != o.depth) return depth < o.depth;
    if (sig != o.sig) return sig < o.sig;
    return shared < o.shared;
  }
};

}  // namespace

// Buckets by (phase, depth) index first (both small non-negative integers), then (signature,
// shared key) within — the same buckets in the same (key-ascending) order as the tree below, with
// no tree of buckets per node.  Falls back to the tree for negative or sparse depth ranges.
static bool schedule_depth_dense(const std::vector<const DFGNode*>& nodes, long& scheduler_ops,
                                 std::vector<BatchRecord>& out) {
  int maxp = 0, maxd = 0;
  for (const DFGNode* n : nodes) {
    if (n->phase < 0 || n->depth < 0) return false;
    maxp = std::max(maxp, n->phase);
    maxd = std::max(maxd, n->depth);
  }
  const size_t npd = size_t(maxp + 1) * size_t(maxd + 1);
  if (npd > 4 * nodes.size() + 64) return false;
  struct Sub {
    int sig;
    uint64_t shared;
    bool ghost;
    std::vector<int> ids;
  };
  std::vector<std::vector<Sub>> pd(npd);
  for (const DFGNode* n : nodes) {
    auto& v = pd[size_t(n->phase) * size_t(maxd + 1) + size_t(n->depth)];
    const uint64_t sk = shared_key(*n);
    Sub* b = nullptr;
    for (auto& x : v)
      if (x.sig == n->sig_id && x.shared == sk) {
        b = &x;
        break;
      }
    if (!b) b = &v.emplace_back(Sub{n->sig_id, sk, n->ghost, {}});
    b->ids.push_back(n->id);  // the window is in id order: ids stay ascending
    ++scheduler_ops;
  }
  for (size_t k = 0; k < npd; ++k) {
    auto& v = pd[k];
    if (v.empty()) continue;
    std::sort(v.begin(), v.end(), [](const Sub& a, const Sub& b) {
      return a.sig != b.sig ? a.sig < b.sig : a.shared < b.shared;
    });
    for (auto& x : v) {
      BatchRecord b;
      b.phase = int(k / size_t(maxd + 1));
      b.depth = int(k % size_t(maxd + 1));
      b.sig = x.sig;
      b.ghost = x.ghost;
      b.size = static_cast<int>(x.ids.size());
      b.node_ids = std::move(x.ids);
      scheduler_ops += b.size;
      out.push_back(std::move(b));
    }
  }
  return true;
}

std::vector<BatchRecord> schedule_depth(const std::vector<const DFGNode*>& nodes, long& scheduler_ops) {
  {
    std::vector<BatchRecord> out;
    long ops = scheduler_ops;
    if (schedule_depth_dense(nodes, ops, out)) {
      scheduler_ops = ops;
      return out;
    }
  }
  std::map<DepthKey, std::pair<bool, std::vector<int>>> buckets;
  for (const DFGNode* n : nodes) {
    auto& b = buckets[DepthKey{n->phase, n->depth, n->sig_id, shared_key(*n)}];
    if (b.second.empty()) b.first = n->ghost;
    b.second.push_back(n->id);
    ++scheduler_ops;
  }
  std::vector<BatchRecord> out;
  out.reserve(buckets.size());
  for (auto& [key, val] : buckets) {
    std::sort(val.second.begin(), val.second.end());
    BatchRecord b;
    b.phase = key.phase;
    b.depth = key.depth;
    b.sig = key.sig;
    b.ghost = val.first;
    b.size = static_cast<int>(val.second.size());
    b.node_ids = std::move(val.second);
    scheduler_ops += b.size;
    out.push_back(std::move(b));
  }
  return out;
}

std::vector<BatchRecord> schedule_agenda(const std::vector<const DFGNode*>& nodes, long& scheduler_ops) {
  std::unordered_map<int, const DFGNode*> in_window;
  for (const DFGNode* n : nodes) in_window[n->id] = n;
  std::unordered_map<int, int> missing;
  std::unordered_map<int, std::vector<int>> consumers;
  for (const DFGNode* n : nodes) {
    ++scheduler_ops;
    int cnt = 0;
    for (int p : n->producers) {
      auto it = in_window.find(p);
      if (it == in_window.end() || it->second->executed) continue;
      ++cnt;
      consumers[p].push_back(n->id);
      ++scheduler_ops;
    }
    missing[n->id] = cnt;
  }
  std::map<int, std::map<uint64_t, std::vector<int>>> ready;
  int ready_count = 0;
  auto push_ready = [&](const DFGNode* n) {
    ready[n->sig_id][shared_key(*n)].push_back(n->id);
    ++ready_count;
    ++scheduler_ops;
  };
  for (const DFGNode* n : nodes)
    if (missing[n->id] == 0) push_ready(n);
  std::vector<BatchRecord> out;
  std::unordered_map<int, bool> done;
  while (ready_count > 0) {
    int best_sig = -1;
    size_t best = 0;
    for (const auto& [sig, groups] : ready) {
      size_t total = 0;
      for (const auto& [k, ids] : groups) total += ids.size();
      if (total > best) {
        best = total;
        best_sig = sig;
      }
    }
    MBATCH_CHECK(best_sig >= 0, "agenda scheduler: ready set corrupt");
    auto groups = std::move(ready[best_sig]);
    ready.erase(best_sig);
    for (auto& [k, ids] : groups) {
      std::sort(ids.begin(), ids.end());
      ready_count -= static_cast<int>(ids.size());
      BatchRecord b;
      const DFGNode* first = in_window.at(ids[0]);
      b.phase = first->phase;
      b.depth = first->depth;
      b.sig = best_sig;
      b.ghost = first->ghost;
      b.size = static_cast<int>(ids.size());
      b.node_ids = ids;
      out.push_back(std::move(b));
      for (int id : ids) {
        done[id] = true;
        ++scheduler_ops;
        for (int cons : consumers[id])
          if (--missing[cons] == 0) push_ready(in_window.at(cons));
      }
    }
  }
  for (const DFGNode* n : nodes) MBATCH_CHECK(done.count(n->id), "agenda scheduler: cycle detected in DFG");
  return out;
}

// ---------------------------------------------------------------------------------------------
// Session

Session::Session(const CompiledModel& model, int device, int precision) : model_(model) {
  if (mbx_ctx_create(device, precision, &ctx_) != 0) throw Error(std::string("mbx_ctx_create failed: ") + mbx_last_error(nullptr));
  try {
    init();
  } catch (...) {
    mbx_ctx_destroy(ctx_);
    throw;
  }
}

Session::Session(const CompiledModel& model, mbx_ctx* ctx) : model_(model), ctx_(ctx), owned_(false) { init(); }

void Session::init() {
  for (const auto& plan : model_.kernels.plans) plan_ids_.push_back(mbx::register_plan(ctx_, plan));
  for (const auto& d : model_.params) {
    if (d.is_instance_input) continue;
    int64_t off = mbx::arena_alloc(ctx_, d.shape.size());
    param_handles_[d.name] = TensorHandle{off, d.shape};
  }
  params_end_ = ctx_->used;
}

Session::~Session() {
  if (owned_) mbx_ctx_destroy(ctx_);
}

void Session::set_params(const ParamEnv& params) {
  for (const auto& d : model_.params) {
    if (d.is_instance_input) continue;
    auto it = params.find(d.name);
    MBATCH_CHECK(it != params.end(), "missing model parameter " + d.name);
    MBATCH_CHECK(it->second.kind == HostValue::Kind::kTensor && it->second.shape == d.shape,
                 "parameter " + d.name + " has the wrong shape");
    const TensorHandle& h = param_handles_.at(d.name);
    if (mbx_arena_upload(ctx_, h.offset, it->second.data.data(), h.size()) != 0) throw Error(mbx_last_error(ctx_));
  }
  if (mbx_sync(ctx_) != 0) throw Error(mbx_last_error(ctx_));
}

EvalResult Session::evaluate(const std::vector<InstanceInput>& inputs, const ExecOptions& opts) {
  MBATCH_CHECK(!inputs.empty(), "evaluate_batch: need at least one instance");
  if (mbx_arena_rewind(ctx_, params_end_) != 0) throw Error(mbx_last_error(ctx_));
  ctx_->persist_end = params_end_;  // nothing below the rewind point is written by this evaluation
  Executor ex(*this, inputs, opts);
  return ex.run();
}

EvalResult Session::evaluate_encoded(const EncodedValues& inputs, const ExecOptions& opts, EncodedOutputs* out) {
  MBATCH_CHECK(inputs.count >= 1, "evaluate_batch: need at least one instance");
  if (mbx_arena_rewind(ctx_, params_end_) != 0) throw Error(mbx_last_error(ctx_));
  ctx_->persist_end = params_end_;
  Executor ex(*this, inputs, opts, out);
  return ex.run();
}

EvalResult evaluate_batch(const CompiledModel& model, const ParamEnv& params, const std::vector<InstanceInput>& inputs) {
  Session s(model, 0, MBX_PREC_FP32);
  s.set_params(params);
  return s.evaluate(inputs, model.opts);
}

std::vector<HostValue> reference_evaluate(const CompiledModel& model, const ParamEnv& params,
                                          const std::vector<InstanceInput>& inputs) {
  Session s(model, 0, MBX_PREC_FP32);
  s.set_params(params);
  std::vector<HostValue> out;
  out.reserve(inputs.size());
  for (const auto& in : inputs) {
    EvalResult r = s.evaluate({in}, model.opts);
    out.push_back(std::move(r.outputs.at(0)));
  }
  return out;
}

ProfileReport profile_from_nodes(const CompiledModel& model, const std::vector<DFGNode>& nodes) {
  ProfileReport rep;
  for (const auto& n : nodes)
    if (!n.ghost) ++rep.counts[n.sig_id];
  for (const auto& blk : model.blocks) {
    auto b = model.kernels.binding_of_block.find(blk.id);
    if (b == model.kernels.binding_of_block.end()) continue;
    const int sig = b->second.sig_id;
    auto it = model.nesting.find(blk.func);
    const int level = it == model.nesting.end() ? 0 : it->second;
    auto cur = rep.static_estimate.find(sig);
    if (cur == rep.static_estimate.end() || level > cur->second) rep.static_estimate[sig] = level;
  }
  for (const auto& [sig, count] : rep.counts) rep.ranking.push_back(sig);
  std::sort(rep.ranking.begin(), rep.ranking.end(), [&](int a, int b) {
    if (rep.counts.at(a) != rep.counts.at(b)) return rep.counts.at(a) > rep.counts.at(b);
    return a < b;
  });
  return rep;
}

ProfileReport profile_invocations(const CompiledModel& model, const ParamEnv& params,
                                  const std::vector<InstanceInput>& inputs) {
  Session s(model, 0, MBX_PREC_FP32);
  s.set_params(params);
  ExecOptions o = model.opts;
  o.record_nodes = true;
  EvalResult res = s.evaluate(inputs, o);
  return profile_from_nodes(model, res.nodes);
}

// ---------------------------------------------------------------------------------------------
// Executor

using clk = std::chrono::steady_clock;

struct Executor::Impl {
  Executor& ex;
  Session& s;
  const CompiledModel& m;
  ExecOptions opts;
  mbx_ctx* c;
  const std::vector<InstanceInput>& inputs;
  const EncodedValues* enc = nullptr;  // encoded inputs (inputs is empty then)
  EncodedOutputs* enc_out = nullptr;
  int batch = 0;                       // instances
  std::vector<std::pair<int64_t, std::pair<const float*, int64_t>>> enc_tensors;  // (offset, (src, n))
  ScheduleTrace trace;
  std::unordered_map<std::string, int> memo;
  std::vector<const StaticBlockInfo*> block_by_id;
  std::vector<const kernelgen::BlockBinding*> binding_by_id;
  // input staging (pinned)
  int64_t input_base = 0;
  std::vector<std::pair<int64_t, const HostValue*>> input_tensors;
  Timing timing;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> flush_events;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> batch_events;
  std::vector<int> batch_share;  // batches one timed launch covers (multi-level launches > 1)

  Impl(Executor& e, Session& sess, const std::vector<InstanceInput>& in, const ExecOptions& o)
      : ex(e), s(sess), m(sess.model()), opts(o), c(sess.ctx()), inputs(in), batch(int(in.size())) {
    int maxid = -1;
    for (const auto& b : m.blocks) maxid = std::max(maxid, b.id);
    block_by_id.assign(maxid + 1, nullptr);
    binding_by_id.assign(maxid + 1, nullptr);
    for (const auto& b : m.blocks) {
      block_by_id[b.id] = &b;
      auto it = m.kernels.binding_of_block.find(b.id);
      if (it != m.kernels.binding_of_block.end()) binding_by_id[b.id] = &it->second;
    }
  }

  ~Impl() {
    for (auto* v : {&flush_events, &batch_events})
      for (auto& [a, b] : *v) {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
  }

  Val materialize(const HostValue& hv) {
    switch (hv.kind) {
      case HostValue::Kind::kTensor: {
        int64_t off = mbx::arena_alloc(c, hv.shape.size());
        input_tensors.push_back({off, &hv});
        return Val::tensor(TensorRef{-1, 0, TensorHandle{off, hv.shape}});
      }
      case HostValue::Kind::kInt: return Val::integer(hv.ival);
      case HostValue::Kind::kFloat: return Val::real(hv.fval);
      case HostValue::Kind::kList: {
        // The reference builds cons cells back to front, so later elements get lower offsets.
        std::vector<Val> items(hv.items.size());
        for (size_t k = hv.items.size(); k-- > 0;) items[k] = materialize(hv.items[k]);
        return Val::list(std::move(items));
      }
      case HostValue::Kind::kTuple:
      case HostValue::Kind::kAdt: {
        std::vector<Val> items;
        for (const auto& f : hv.items) items.push_back(materialize(f));
        if (hv.kind == HostValue::Kind::kTuple) return Val::tuple(std::move(items));
        return Val::seq(Val::kAdt, std::move(items), ctor_id(hv.ctor));
      }
    }
    throw Error("unreachable");
  }

  // The zoo programs' ADTs are binary trees (zoo.cpp): constructors Leaf and Node.
  static int ctor_id(const std::string& name) {
    MBATCH_CHECK(name == "Leaf" || name == "Node", "unknown ADT constructor " + name);
    return name == "Node" ? 1 : 0;
  }
  // ADT constructor of the flat encoding (0 Leaf, 1 Node, -1 named: length + bytes).
  int read_ctor(int64_t& ti) {
    const int32_t* t = enc->toks;
    MBATCH_CHECK(ti < enc->ntok, "hostval encoding truncated");
    const int id = t[ti++];
    if (id >= 0) return id ? 1 : 0;
    MBATCH_CHECK(ti < enc->ntok, "hostval encoding truncated");
    const int len = t[ti++];
    MBATCH_CHECK(len >= 0 && ti + len <= enc->ntok, "hostval encoding truncated");
    std::string name;
    for (int k = 0; k < len; ++k) name.push_back(char(t[ti++]));
    return ctor_id(name);
  }

  // The flat-encoding counterpart of materialize(decode(...)): same arena order (list elements
  // back to front, like the reference's cons cells), same errors as the C ABI's decoder.
  void skip_enc(int64_t& ti, int64_t& di) {
    const int32_t* t = enc->toks;
    MBATCH_CHECK(ti < enc->ntok, "hostval encoding truncated");
    const int kind = t[ti++];
    if (kind == 0) {
      MBATCH_CHECK(ti + 2 <= enc->ntok, "hostval encoding truncated");
      di += int64_t(t[ti]) * t[ti + 1];
      ti += 2;
    } else if (kind == 1) {
      ++ti;
    } else if (kind == 5 || kind == 6) {
      MBATCH_CHECK(ti + 2 <= enc->ntok, "hostval encoding truncated");
      ti += 2;
    } else if (kind >= 2 && kind <= 4) {
      if (kind == 4) read_ctor(ti);
      MBATCH_CHECK(ti < enc->ntok, "hostval encoding truncated");
      const int n = t[ti++];
      for (int k = 0; k < n; ++k) skip_enc(ti, di);
    } else {
      throw Error("hostval encoding: bad kind " + std::to_string(kind));
    }
  }
  Val materialize_enc(int64_t& ti, int64_t& di) {
    const int32_t* t = enc->toks;
    MBATCH_CHECK(ti < enc->ntok, "hostval encoding truncated");
    const int kind = t[ti++];
    switch (kind) {
      case 0: {
        MBATCH_CHECK(ti + 2 <= enc->ntok, "hostval encoding truncated");
        const int r = t[ti++], cc = t[ti++];
        const int64_t n = int64_t(r) * cc;
        MBATCH_CHECK(r >= 0 && cc >= 0 && di + n <= enc->ndata, "hostval data truncated");
        const int64_t off = mbx::arena_alloc(c, n);
        enc_tensors.push_back({off, {enc->data + di, n}});
        di += n;
        return Val::tensor(TensorRef{-1, 0, TensorHandle{off, Shape{r, cc}}});
      }
      case 1: MBATCH_CHECK(ti < enc->ntok, "hostval encoding truncated"); return Val::integer(t[ti++]);
      case 5:
      case 6: {
        MBATCH_CHECK(ti + 2 <= enc->ntok, "hostval encoding truncated");
        const uint64_t bits = uint64_t(uint32_t(t[ti])) | (uint64_t(uint32_t(t[ti + 1])) << 32);
        ti += 2;
        if (kind == 6) return Val::integer(long(int64_t(bits)));
        double x;
        std::memcpy(&x, &bits, sizeof x);
        return Val::real(x);
      }
      case 2: {
        MBATCH_CHECK(ti < enc->ntok, "hostval encoding truncated");
        const int n = t[ti++];
        std::vector<std::pair<int64_t, int64_t>> at(static_cast<size_t>(n));
        for (int k = 0; k < n; ++k) {
          at[size_t(k)] = {ti, di};
          skip_enc(ti, di);
        }
        const int64_t tend = ti, dend = di;
        std::vector<Val> items(static_cast<size_t>(n));
        for (int k = n; k-- > 0;) {
          int64_t a = at[size_t(k)].first, b = at[size_t(k)].second;
          items[size_t(k)] = materialize_enc(a, b);
        }
        ti = tend;
        di = dend;
        return Val::list(std::move(items));
      }
      case 3:
      case 4: {
        int ctor = 0;
        if (kind == 4) ctor = read_ctor(ti);
        MBATCH_CHECK(ti < enc->ntok, "hostval encoding truncated");
        const int n = t[ti++];
        std::vector<Val> items;
        items.reserve(size_t(n));
        for (int k = 0; k < n; ++k) items.push_back(materialize_enc(ti, di));
        if (kind == 3) return Val::tuple(std::move(items));
        return Val::seq(Val::kAdt, std::move(items), ctor ? 1 : 0);
      }
    }
    throw Error("hostval encoding: bad kind " + std::to_string(kind));
  }

  // to_host + the C ABI's encode in one pass.
  void to_tokens(const Val& v, const std::vector<float>& buf, size_t& cursor, size_t& ti,
                 const std::vector<TensorHandle>& hs, EncodedOutputs& out) {
    switch (v.kind) {
      case Val::kTensor: {
        const TensorHandle& h = hs[ti++];
        out.toks.push_back(0);
        out.toks.push_back(h.shape.rows);
        out.toks.push_back(h.shape.cols);
        out.data.insert(out.data.end(), buf.begin() + cursor, buf.begin() + cursor + h.size());
        cursor += h.size();
        return;
      }
      case Val::kInt:
        if (v.i >= INT32_MIN && v.i <= INT32_MAX) {
          out.toks.push_back(1);
          out.toks.push_back(int32_t(v.i));
        } else {
          out.toks.push_back(6);
          out.toks.push_back(int32_t(uint32_t(uint64_t(v.i) & 0xffffffffu)));
          out.toks.push_back(int32_t(uint32_t(uint64_t(v.i) >> 32)));
        }
        return;
      case Val::kFloat:
        out.toks.push_back(5);
        out.toks.push_back(int32_t(uint32_t(uint64_t(v.i) & 0xffffffffu)));
        out.toks.push_back(int32_t(uint32_t(uint64_t(v.i) >> 32)));
        return;
      default:
        if (v.kind == Val::kList) out.toks.push_back(2);
        else if (v.kind == Val::kTuple) out.toks.push_back(3);
        else {
          out.toks.push_back(4);
          out.toks.push_back(v.ctor == 1 ? 1 : 0);
        }
        out.toks.push_back(int32_t(v.size()));
        for (size_t k = 0; k < v.size(); ++k) to_tokens(v.at(k), buf, cursor, ti, hs, out);
    }
  }

  // Encoded inputs whose data stream lies in pinned host memory: one H2D of the stream plus a
  // device scatter, both on the copy stream.  Returns false when the data is pageable.
  bool upload_pinned() {
    if (!enc || c->dry || !c->copy_stream || enc_tensors.empty() || !input_tensors.empty()) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, enc->data) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.type != cudaMemoryTypeHost) return false;
    const size_t nd = size_t(enc->ndata), nt = enc_tensors.size();
    cudaStream_t cs = c->copy_stream;
    {
      // When the tensors sit in the arena in stream order (runs that continue each other in both),
      // a few direct H2D copies replace the staging copy + scatter kernel.
      struct Run { int64_t src, size, dst; };
      std::vector<Run> runs;
      for (size_t k = 0; k < nt && runs.size() <= 8; ++k) {
        const int64_t src = int64_t(enc_tensors[k].second.first - enc->data), size = enc_tensors[k].second.second,
                      dst = enc_tensors[k].first;
        if (!runs.empty() && runs.back().src + runs.back().size == src && runs.back().dst + runs.back().size == dst)
          runs.back().size += size;
        else
          runs.push_back({src, size, dst});
      }
      if (runs.size() <= 8 && !std::getenv("MBX_INPUT_SCATTER")) {  // (env: force the scatter path)
        float* arena = mbx::arena_ptr(c);
        int64_t bytes = 0;
        for (const Run& r : runs) {
          mbx::cuda_check(cudaMemcpyAsync(arena + r.dst, enc->data + r.src, size_t(r.size) * sizeof(float),
                                          cudaMemcpyHostToDevice, cs),
                          "input H2D");
          bytes += r.size * int64_t(sizeof(float));
        }
        mbx::cuda_check(cudaEventRecord(c->ev_copy, cs), "input copy event");
        c->copy_pending = true;
        timing.h2d_bytes += long(bytes);
        return true;
      }
    }
    if (nd > c->in_dev_cap) {
      if (c->in_dev) cudaFree(c->in_dev);
      c->in_dev_cap = std::max(nd, c->in_dev_cap * 2);
      mbx::cuda_check(cudaMalloc(&c->in_dev, c->in_dev_cap * sizeof(float)), "pinned input staging");
    }
    if (nt > c->scat_cap) {
      if (c->scat_host) cudaFreeHost(c->scat_host);
      if (c->scat_dev) cudaFree(c->scat_dev);
      c->scat_cap = std::max(nt, c->scat_cap * 2);
      mbx::cuda_check(cudaMallocHost(&c->scat_host, c->scat_cap * 3 * sizeof(int64_t)), "scatter table");
      mbx::cuda_check(cudaMalloc(&c->scat_dev, c->scat_cap * 3 * sizeof(int64_t)), "scatter table");
    }
    for (size_t k = 0; k < nt; ++k) {
      c->scat_host[3 * k] = int64_t(enc_tensors[k].second.first - enc->data);
      c->scat_host[3 * k + 1] = enc_tensors[k].second.second;
      c->scat_host[3 * k + 2] = enc_tensors[k].first;
    }
    mbx::cuda_check(cudaMemcpyAsync(c->in_dev, enc->data, nd * sizeof(float), cudaMemcpyHostToDevice, cs), "input H2D");
    mbx::cuda_check(cudaMemcpyAsync(c->scat_dev, c->scat_host, nt * 3 * sizeof(int64_t), cudaMemcpyHostToDevice, cs),
                    "scatter table H2D");
    mbx::cuda_check(mbx::launch_scatter_ranges(c->in_dev, c->scat_dev, int(nt), mbx::arena_ptr(c), cs), "input scatter");
    ++c->launches;
    ++timing.device_launches;
    mbx::cuda_check(cudaEventRecord(c->ev_copy, cs), "input copy event");
    c->copy_pending = true;
    timing.h2d_bytes += long(nd * sizeof(float) + nt * 3 * sizeof(int64_t));
    return true;
  }

  void upload_inputs() {
    int64_t n = c->used - input_base;
    if (n <= 0 || opts.inputs_resident) return;
    if (upload_pinned()) return;
    mbx::ensure_input_stage(c, size_t(n));
    for (auto& [off, hv] : input_tensors)
      std::memcpy(c->in_host + (off - input_base), hv->ext ? hv->ext : hv->data.data(),
                  size_t(hv->shape.size()) * sizeof(float));
    for (auto& [off, src] : enc_tensors)
      std::memcpy(c->in_host + (off - input_base), src.first, size_t(src.second) * sizeof(float));
    if (opts.inputs_resident) return;
    if (!c->dry) {
      cudaStream_t cs = c->copy_stream ? c->copy_stream : c->stream;
      mbx::cuda_check(cudaMemcpyAsync(mbx::arena_ptr(c) + input_base, c->in_host, size_t(n) * sizeof(float),
                                      cudaMemcpyHostToDevice, cs),
                      "input H2D");
      if (c->copy_stream) {
        mbx::cuda_check(cudaEventRecord(c->ev_copy, cs), "input copy event");
        c->copy_pending = true;  // the kernel stream waits at the first meta_commit
      }
    }
    timing.h2d_bytes += n * long(sizeof(float));
  }

  TensorHandle resolve(const TensorRef& r) const {
    if (r.node < 0) return r.handle;
    const DFGNode& n = ex.nodes_[r.node];
    MBATCH_CHECK(n.executed, "use of unmaterialized tensor (scheduling bug)");
    return n.outputs.at(r.out);
  }

  // A DFG node from the session's pool (vectors cleared, capacity kept) or a fresh one.
  DFGNode recycled_node() {
    auto& pool = s.node_pool();
    if (pool.empty()) return DFGNode{};
    DFGNode n = std::move(pool.back());
    pool.pop_back();
    n.id = n.sig_id = n.block_id = n.instance = -1;
    n.phase = n.depth = 0;
    n.ghost = n.executed = false;
    n.shared_ins.clear();
    n.batched_ins.clear();
    n.producers.clear();
    n.outputs.clear();
    return n;
  }

  // -- DFG construction (executor.cpp:368-443) --------------------------------------------
  int emit(Fiber& fb, int blk_id, std::initializer_list<const Val*> ins) {
    const StaticBlockInfo& blk = *block_by_id.at(blk_id);
    const kernelgen::BlockBinding& bind = *binding_by_id[blk_id];
    const Val* const* in = ins.begin();
    if (ins.size() != blk.inputs.size()) throw Error("block " + std::to_string(blk_id) + ": input arity");
    auto& nodes = ex.nodes_;
    const bool all_shared = bind.batched_input_pos.empty();
    std::string memo_key;
    if (all_shared) {
      memo_key = std::to_string(blk.id) + "|";
      for (int pos : bind.shared_input_pos) {
        const TensorRef& r = in[pos]->t;
        memo_key += std::to_string(r.node) + ":" + std::to_string(r.out) + ":" + std::to_string(r.handle.offset) + ";";
      }
      auto it = memo.find(memo_key);
      if (it != memo.end()) return it->second;
    }
    // Built in place at the end of the node table (storage recycled from the session's pool).
    DFGNode& node = nodes.emplace_back(recycled_node());
    node.shared_ins.reserve(bind.shared_input_pos.size());
    node.batched_ins.reserve(bind.batched_input_pos.size());
    node.producers.reserve(bind.shared_input_pos.size() + bind.batched_input_pos.size() + 1);
    for (int pos : bind.shared_input_pos) node.shared_ins.push_back(in[pos]->t);
    for (int pos : bind.batched_input_pos) node.batched_ins.push_back(in[pos]->t);
    node.id = static_cast<int>(nodes.size()) - 1;
    node.sig_id = bind.sig_id;
    node.block_id = blk.id;
    node.instance = fb.instance;
    node.phase = fb.phase;
    for (const auto& r : node.shared_ins)
      if (r.node >= 0) node.producers.push_back(r.node);
    for (const auto& r : node.batched_ins)
      if (r.node >= 0) node.producers.push_back(r.node);
    if (fb.pending_ghost >= 0) {
      node.producers.push_back(fb.pending_ghost);
      fb.pending_ghost = -1;
    }
    auto floor = [&](int base) {
      int d = base;
      for (int p : node.producers) {
        const DFGNode& prod = nodes[p];
        if (!prod.executed && prod.phase == node.phase) d = std::max(d, prod.depth + 1);
      }
      return d;
    };
    if (opts.hoist && blk.hoist >= 0) {
      node.depth = floor(blk.hoist);
    } else {
      node.depth = floor(fb.depth_counter + 1);
      fb.depth_counter = node.depth;
    }
    fb.last_node = node.id;
    if (all_shared) memo[memo_key] = node.id;
    return node.id;
  }

  void ghosts(Fiber& fb, int count) {
    auto& nodes = ex.nodes_;
    for (int k = 0; k < count; ++k) {
      DFGNode node = recycled_node();
      node.id = static_cast<int>(nodes.size());
      node.sig_id = m.kernels.ghost_sig;
      node.instance = fb.instance;
      node.phase = fb.phase;
      node.ghost = true;
      node.depth = ++fb.depth_counter;
      int prev = fb.pending_ghost >= 0 ? fb.pending_ghost : fb.last_node;
      if (prev >= 0 && !nodes[prev].executed) node.producers.push_back(prev);
      fb.pending_ghost = node.id;
      nodes.push_back(std::move(node));
    }
  }

  void stage(Fiber& fb, int st) {
    int phase = opts.phases ? m.stage_phase.at(st) : 0;
    if (phase != fb.phase) {
      MBATCH_CHECK(phase > fb.phase, "phases must be non-decreasing");
      fb.phase = phase;
      fb.depth_counter = 0;
      fb.last_node = -1;
      fb.pending_ghost = -1;
    }
  }

  // -- fibers ----------------------------------------------------------------------------
  void resume_fiber(Fiber& fb) {
    std::coroutine_handle<> h = fb.resume_point ? fb.resume_point : std::coroutine_handle<>(fb.root.h);
    fb.resume_point = nullptr;
    h.resume();
    if (fb.root.h.done()) {
      if (fb.root.h.promise().exc) std::rethrow_exception(fb.root.h.promise().exc);
      fb.result = std::move(fb.root.h.promise().value);
      fb.has_result = true;
      fb.status = FiberStatus::kDone;
      if (fb.parent >= 0) {
        Fiber& parent = *ex.fibers_[fb.parent];
        if (--parent.pending_children == 0 && parent.status == FiberStatus::kBlockedJoin)
          parent.status = FiberStatus::kRunnable;
      }
    }
  }

  void run_runnable() {
    bool progressed = true;
    while (progressed) {
      progressed = false;
      for (size_t i = 0; i < ex.fibers_.size(); ++i) {
        Fiber& fb = *ex.fibers_[i];
        if (fb.status != FiberStatus::kRunnable) continue;
        progressed = true;
        resume_fiber(fb);
      }
    }
  }

  // -- two-stream issue ---------------------------------------------------------------------
  // Two or more runs of consecutive tensor-core batches (length >= 2) over different weights:
  // the flush may run them at once (assign_streams), so they are planned to fit together.
  bool pair_candidates(const std::vector<mbx::BatchLaunch>& L) const {
    std::vector<std::pair<int, size_t>> seen;  // (plan, shared_meta of the run's first batch)
    for (size_t i = 0; i < L.size();) {
      const mbx::PlanEntry& pe = c->plans[size_t(L[i].plan_id)];
      size_t j = i + 1;
      if (pe.tc_kind == 1 && !pe.tc_small) {
        const size_t ns = pe.exec_plan.shared_shapes.size();
        while (j < L.size() && L[j].plan_id == L[i].plan_id &&
               std::memcmp(c->meta.host + L[j].shared_meta, c->meta.host + L[i].shared_meta, ns * 8) == 0)
          ++j;
        if (j - i >= 2) {
          bool fresh = true;
          for (const auto& [p, off] : seen)
            if (p == L[i].plan_id && std::memcmp(c->meta.host + off, c->meta.host + L[i].shared_meta, ns * 8) == 0)
              fresh = false;
          if (fresh) seen.push_back({L[i].plan_id, L[i].shared_meta});
        }
      }
      i = j;
    }
    return seen.size() >= 2;
  }

  size_t ev_next_ = 0;
  cudaEvent_t take_event() {
    if (ev_next_ == c->ev_pool.size()) {
      cudaEvent_t e;
      mbx::cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      c->ev_pool.push_back(e);
    }
    return c->ev_pool[ev_next_++];
  }

  // Independent chains of a flush on two streams: an issue unit (a persistent run, or one
  // launch) depends on an earlier unit when one of its input rows lies in that unit's output
  // regions.  A unit with no dependency goes to the stream the previous unit did not use; one
  // whose dependencies all sit on one stream follows them; otherwise the primary stream, waiting
  // for the other's units it reads.  Only when the flush has two persistent runs (BiRNN's two
  // directions: each run and its input transform on its own stream) and no MV-RNN fusion pairs.
  bool assign_streams(const std::vector<mbx::BatchLaunch>& L, const std::vector<mbx::LevelsRun>& runs,
                      const std::vector<int>& run_at, std::vector<int>& ustream, std::vector<std::vector<int>>& uwait,
                      std::vector<char>& usignal) {
    int persistent = 0;
    for (const auto& r : runs) persistent += r.n > 1;
    if (persistent < 2) return false;
    // Kept on one stream: MV-RNN cell + add pairs (fused at issue), merged sinks, hoisted
    // prefixes (their cached scratch), and single tensor-core batches outside persistent runs
    // (the context's split-K scratch).
    for (size_t i = 0; i < L.size(); ++i) {
      const mbx::PlanEntry& pe = c->plans[size_t(L[i].plan_id)];
      if (pe.mv || pe.mv_add || L[i].out_node || pe.prefix_plan >= 0) return false;
      if (run_at[i] < 0 && pe.tc_kind == 1 && !pe.tc_small) {
        bool in_run = false;
        for (const auto& r : runs) in_run = in_run || (int(i) >= r.start && int(i) < r.start + r.n);
        if (!in_run) return false;
      }
    }
    struct Region {
      int64_t lo, hi;
      int unit;
    };
    std::vector<Region> regions;
    std::vector<std::pair<size_t, size_t>> units;  // [begin, end) launches
    for (size_t i = 0; i < L.size();) {
      const size_t n = run_at[i] >= 0 ? size_t(runs[size_t(run_at[i])].n) : 1;
      units.push_back({i, i + n});
      i += n;
    }
    auto for_leaves = [&](const mbx::BatchLaunch& l, auto&& f) {
      if (l.sub.empty()) f(l);
      else
        for (const auto& sl : l.sub) f(sl);
    };
    for (size_t u = 0; u < units.size(); ++u)
      for (size_t j = units[u].first; j < units[u].second; ++j)
        for_leaves(L[j], [&](const mbx::BatchLaunch& l) {
          const mbx::PlanEntry& pe = c->plans[size_t(l.plan_id)];
          if (pe.plan.ghost) return;
          const int64_t* ob = reinterpret_cast<const int64_t*>(c->meta.host + l.out_meta);
          for (size_t k = 0; k < pe.out_shapes.size(); ++k)
            regions.push_back({ob[k], ob[k] + int64_t(l.b) * pe.out_shapes[k].size(), int(u)});
          for (const auto& g : l.gathers) regions.push_back({g.dst, g.dst + int64_t(l.b) * g.size, int(u)});
        });
    std::sort(regions.begin(), regions.end(), [](const Region& a, const Region& b) { return a.lo < b.lo; });
    auto owner = [&](int64_t off) -> int {
      auto it = std::upper_bound(regions.begin(), regions.end(), off, [](int64_t v, const Region& r) { return v < r.lo; });
      if (it == regions.begin()) return -1;
      --it;
      return off < it->hi ? it->unit : -1;
    };
    ustream.assign(units.size(), 0);
    uwait.assign(units.size(), {});
    usignal.assign(units.size(), 0);
    bool any2 = false;
    for (size_t u = 0; u < units.size(); ++u) {
      std::vector<int> deps;
      auto add = [&](int64_t off) {
        const int v = owner(off);
        if (v >= 0 && v != int(u) && std::find(deps.begin(), deps.end(), v) == deps.end()) deps.push_back(v);
      };
      for (size_t j = units[u].first; j < units[u].second; ++j)
        for_leaves(L[j], [&](const mbx::BatchLaunch& l) {
          const mbx::PlanEntry& pe = c->plans[size_t(l.plan_id)];
          if (pe.plan.ghost) return;
          const size_t ns = pe.exec_plan.shared_shapes.size(), nb = pe.exec_plan.batched_shapes.size();
          const int64_t* sh = reinterpret_cast<const int64_t*>(c->meta.host + l.shared_meta);
          const int64_t* bt = reinterpret_cast<const int64_t*>(c->meta.host + l.batched_meta);
          for (size_t k = 0; k < ns; ++k) add(sh[k]);
          for (size_t k = 0; k < size_t(l.b) * nb; ++k) add(bt[k]);
        });
      // Runs over the same weights follow each other (one weight pack, made by the first).
      const int r0 = run_at[units[u].first];
      if (r0 >= 0)
        for (size_t v = 0; v < u; ++v) {
          const int rv = run_at[units[v].first];
          if (rv < 0 || L[units[v].first].plan_id != L[units[u].first].plan_id) continue;
          const size_t ns = c->plans[size_t(L[units[u].first].plan_id)].exec_plan.shared_shapes.size();
          if (std::memcmp(c->meta.host + L[units[v].first].shared_meta, c->meta.host + L[units[u].first].shared_meta,
                          ns * 8) == 0 &&
              std::find(deps.begin(), deps.end(), int(v)) == deps.end())
            deps.push_back(int(v));
        }
      int s = 0;
      bool on0 = false, on1 = false;
      for (int v : deps) (ustream[size_t(v)] ? on1 : on0) = true;
      if (deps.empty()) s = u == 0 ? 0 : 1 - ustream[u - 1];
      else if (on1 && !on0) s = 1;
      ustream[u] = s;
      for (int v : deps)
        if (ustream[size_t(v)] != s) {
          uwait[u].push_back(v);
          usignal[size_t(v)] = 1;
        }
      any2 = any2 || s == 1;
    }
    return any2;
  }

  // -- flush (executor.cpp:711-758) -------------------------------------------------------
  size_t exec_lo_ = 0;  // every node below this index is executed
  bool flush(int phase_limit) {
    auto& nodes = ex.nodes_;
    std::vector<const DFGNode*> window;
    while (exec_lo_ < nodes.size() && nodes[exec_lo_].executed) ++exec_lo_;  // (nodes before: all executed)
    for (size_t k = exec_lo_; k < nodes.size(); ++k)
      if (!nodes[k].executed && nodes[k].phase <= phase_limit) window.push_back(&nodes[k]);
    if (window.empty()) return false;
    trace.flush_boundaries.push_back(static_cast<int>(trace.batches.size()));
    auto ts0 = clk::now();
    std::vector<BatchRecord> batches;
    if (opts.scheduler == ExecOptions::Scheduler::kDepth) {
      batches = schedule_depth(window, trace.scheduler_ops);
    } else {
      std::map<int, std::vector<const DFGNode*>> by_phase;
      for (const DFGNode* n : window) by_phase[n->phase].push_back(n);
      for (auto& [p, group] : by_phase)
        for (auto& b : schedule_agenda(group, trace.scheduler_ops)) batches.push_back(std::move(b));
    }
    auto ts1 = clk::now();
    timing.host_sched_us += std::chrono::duration<double, std::micro>(ts1 - ts0).count();
    // Reserve index staging for the whole window so nothing recycles mid-flush.
    size_t meta_bytes = 0;
    for (const auto& b : batches) {
      if (b.ghost) continue;
      const auto& plan = m.kernels.plan(b.sig);
      const size_t nb = plan.batched_shapes.size();
      meta_bytes += 8 * (plan.shared_shapes.size() + size_t(b.size) * nb * 2 + plan.outputs.size()) + 512 + 64 +
                    16 * size_t(b.size) + 16;  // operand-image destinations (plan_shadows)
      // merge_launches: concatenated node tables + per-node output offsets (split plans: both halves)
      const mbx::PlanEntry& pe = c->plans[size_t(s.plan_ids()[b.sig])];
      for (int q : {pe.head_plan, pe.tail_plan, pe.head_plan < 0 ? int(s.plan_ids()[b.sig]) : -1})
        if (q >= 0)
          meta_bytes += 8 * size_t(b.size) * (c->plans[size_t(q)].exec_plan.batched_shapes.size() +
                                               c->plans[size_t(q)].out_shapes.size()) + 16;
    }
    mbx::meta_reserve(c, meta_bytes);

    std::vector<mbx::BatchLaunch> launches;
    launches.reserve(batches.size());
    std::vector<size_t> lbatch;  // launch -> its batch in trace.batches
    lbatch.reserve(batches.size());
    std::vector<TensorHandle> first_shared;
    std::vector<int64_t> shared, batched, outs;
    for (auto& batch : batches) {
      if (batch.ghost) {
        for (int id : batch.node_ids) nodes[id].executed = true;
        trace.batches.push_back(std::move(batch));
        continue;
      }
      const auto& plan = m.kernels.plan(batch.sig);
      const size_t ns = plan.shared_shapes.size(), nb = plan.batched_shapes.size(), no = plan.outputs.size();
      const int b = batch.size;
      shared.assign(ns, 0);
      batched.assign(size_t(b) * nb, 0);
      outs.assign(size_t(b) * no, 0);
      const DFGNode& first = nodes[batch.node_ids[0]];
      MBATCH_CHECK(first.shared_ins.size() == ns && first.batched_ins.size() == nb, "exec_batched: arity mismatch");
      first_shared.resize(ns);
      for (size_t k = 0; k < ns; ++k) {
        first_shared[k] = resolve(first.shared_ins[k]);
        shared[k] = first_shared[k].offset;
      }
      for (int i = 0; i < b; ++i) {
        const DFGNode& n = nodes[batch.node_ids[i]];
        if (i > 0)
          for (size_t k = 0; k < ns; ++k)
            MBATCH_CHECK(resolve(n.shared_ins[k]) == first_shared[k],
                         "shared-param handle mismatch across instances (analysis bug)");
        for (size_t j = 0; j < nb; ++j) batched[size_t(i) * nb + j] = resolve(n.batched_ins[j]).offset;
      }
      int64_t gb = 0;
      launches.push_back(mbx::prepare_batch(c, s.plan_ids()[batch.sig], b, shared.data(), batched.data(),
                                            opts.gather == GatherMode::kFused ? MBX_GATHER_FUSED : MBX_GATHER_EXPLICIT,
                                            outs.data(), &gb));
      const auto& shapes = c->plans[s.plan_ids()[batch.sig]].out_shapes;
      for (int i = 0; i < b; ++i) {
        DFGNode& n = nodes[batch.node_ids[i]];
        n.outputs.resize(no);
        for (size_t k = 0; k < no; ++k) n.outputs[k] = TensorHandle{outs[size_t(i) * no + k], shapes[k]};
        n.executed = true;
      }
      trace.gather_bytes += gb;
      ++trace.kernel_launches;
      lbatch.push_back(trace.batches.size());
      trace.batches.push_back(std::move(batch));
    }
    if (!c->dry && !opts.time_batches) hoist_sinks(launches, lbatch);
    // Runs of consecutive batches of one tensor-core gate plan (e.g. every TreeLSTM internal
    // depth) become one persistent multi-level launch; their level tables are staged here, then
    // the split-bf16 shadows of the rows they gather are planned.
    std::vector<mbx::LevelsRun> runs;
    std::vector<int> run_at(launches.size(), -1);
    c->prefer_pair = !opts.time_batches && pair_candidates(launches);
    for (size_t i = 0; i < launches.size();) {
      mbx::LevelsRun r;
      r.start = int(i);
      r.n = mbx::plan_levels(c, launches, i, &r.table, &r.groups, &r.cfg);
      if (r.n >= 1) {
        run_at[i] = int(runs.size());
        runs.push_back(r);
        i += size_t(r.n);
      } else {
        ++i;
      }
    }
    c->prefer_pair = false;  // (planning only; the C-ABI flush scope plans single-stream)
    mbx::plan_shadows(c, launches, runs);
    timing.h2d_bytes += long(c->meta.cursor - c->meta.committed);
    mbx::meta_commit(c);
    auto ts2 = clk::now();
    timing.host_prepare_us += std::chrono::duration<double, std::micro>(ts2 - ts1).count();
    struct IssueClock {
      Timing& t;
      clk::time_point a = clk::now();
      ~IssueClock() { t.host_issue_us += std::chrono::duration<double, std::micro>(clk::now() - a).count(); }
    } issue_clock{timing};
    if (!c->dry && !launches.empty()) {
      cudaEvent_t a = nullptr, e = nullptr;
      if (opts.time_kernels) {
        cudaEventCreate(&a);
        cudaEventCreate(&e);
        cudaEventRecord(a, c->stream);
      }
      int64_t before = c->launches;
      std::vector<int> unit_stream;  // per issue unit (a run or a launch): 0 / 1
      std::vector<std::vector<int>> unit_waits;  // units on the other stream it waits for
      std::vector<char> unit_signal;             // a unit on the other stream waits for it
      const bool dual = !opts.time_batches && assign_streams(launches, runs, run_at, unit_stream, unit_waits, unit_signal);
      std::vector<cudaEvent_t> unit_ev(dual ? unit_stream.size() : 0, nullptr);
      if (dual) {
        if (!c->stream2) mbx::cuda_check(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking), "second stream");
        cudaEvent_t ev_start = take_event();
        mbx::cuda_check(cudaEventRecord(ev_start, c->stream), "flush start");  // offsets + inputs committed
        mbx::cuda_check(cudaStreamWaitEvent(c->stream2, ev_start, 0), "flush start");
      }
      bool used2 = false;
      size_t unit = 0;
      for (size_t i = 0; i < launches.size(); ++unit) {
        const mbx::LevelsRun* run = run_at[i] >= 0 ? &runs[size_t(run_at[i])] : nullptr;
        int n = run ? run->n : 1;
        const bool on2 = dual && unit_stream[unit] == 1;
        if (dual) {
          cudaStream_t own = on2 ? c->stream2 : c->stream;
          for (int w : unit_waits[unit]) mbx::cuda_check(cudaStreamWaitEvent(own, unit_ev[size_t(w)], 0), "cross-stream wait");
        }
        if (on2) {
          std::swap(c->stream, c->stream2);
          c->issue_slot = 1;
          used2 = true;
        }
        struct Restore {  // back to the primary stream even if the issue throws
          mbx_ctx* c;
          bool on;
          ~Restore() {
            if (on) {
              std::swap(c->stream, c->stream2);
              c->issue_slot = 0;
            }
          }
        } restore{c, on2};
        cudaEvent_t x = nullptr, y = nullptr;
        if (opts.time_batches) {
          cudaEventCreate(&x);
          cudaEventCreate(&y);
          cudaEventRecord(x, c->stream);
        }
        if (run) mbx::issue_levels(c, launches, i, n, run->table, run->groups, run->cfg);
        else n = mbx::issue_batches(c, launches, i);
        if (dual && unit_signal[unit]) {
          unit_ev[unit] = take_event();
          mbx::cuda_check(cudaEventRecord(unit_ev[unit], c->stream), "unit done");
        }
        if (opts.time_batches) {
          cudaEventRecord(y, c->stream);
          batch_events.push_back({x, y});
          batch_share.push_back(n);
        }
        i += size_t(n);
      }
      if (used2) {  // the rest of this context's work (read-backs, the next flush) follows both
        cudaEvent_t e = take_event();
        mbx::cuda_check(cudaEventRecord(e, c->stream2), "second stream done");
        mbx::cuda_check(cudaStreamWaitEvent(c->stream, e, 0), "second stream done");
      }
      ev_next_ = 0;  // reusable: every recorded event is ordered before later work of this context
      timing.device_launches += long(c->launches - before);
      if (opts.time_kernels) {
        cudaEventRecord(e, c->stream);
        flush_events.push_back({a, e});
      }
    }
    return true;
  }

  // Issue order of a flush (the trace keeps the reference's order).  A batch no later batch of
  // the flush reads (a sink: NestedRNN's decision cells, whose results only the host and the
  // next flush consume) need not run at its depth; mergeable sinks (the exact decision kernels)
  // move behind the other batches and the sinks of one plan run as ONE launch.  NestedRNN: the
  // inner steps between decision cells become one persistent levels run and a flush's ~10
  // decision batches one head + one tail launch (instead of ~10 of each interleaved with
  // single-level runs).  Results are unchanged: every node reads the same inputs.
  std::vector<int> node_launch_;
  void hoist_sinks(std::vector<mbx::BatchLaunch>& launches, const std::vector<size_t>& lbatch) {
    const size_t n = launches.size();
    if (n < 2) return;
    auto& nodes = ex.nodes_;
    if (node_launch_.size() < nodes.size()) node_launch_.resize(nodes.size(), -1);
    for (size_t li = 0; li < n; ++li)
      for (int id : trace.batches[lbatch[li]].node_ids) node_launch_[size_t(id)] = int(li);
    std::vector<char> consumed(n, 0);
    for (size_t li = 0; li < n; ++li)
      for (int id : trace.batches[lbatch[li]].node_ids)
        for (int p : nodes[size_t(id)].producers) {
          const int q = node_launch_[size_t(p)];
          if (q >= 0 && q != int(li)) consumed[size_t(q)] = 1;
        }
    for (size_t li = 0; li < n; ++li)
      for (int id : trace.batches[lbatch[li]].node_ids) node_launch_[size_t(id)] = -1;
    std::vector<size_t> keep, moved;
    for (size_t li = 0; li < n; ++li) (!consumed[li] && mbx::mergeable(c, launches[li]) ? moved : keep).push_back(li);
    if (moved.empty() || (moved.size() == 1 && (keep.empty() || moved[0] > keep.back()))) return;
    // Sinks grouped by plan and shared operands (first-appearance order), each group one launch.
    std::vector<std::vector<size_t>> groups;
    for (size_t li : moved) {
      bool placed = false;
      for (auto& gr : groups)
        if (mbx::same_shared(c, launches[gr[0]], launches[li])) {
          gr.push_back(li);
          placed = true;
          break;
        }
      if (!placed) groups.push_back({li});
    }
    std::vector<mbx::BatchLaunch> out;
    out.reserve(keep.size() + groups.size());
    for (size_t li : keep) out.push_back(std::move(launches[li]));
    for (const auto& gr : groups) {
      if (gr.size() == 1) {
        out.push_back(std::move(launches[gr[0]]));
        continue;
      }
      std::vector<const mbx::BatchLaunch*> g;
      for (size_t li : gr) g.push_back(&launches[li]);
      out.push_back(mbx::merge_launches(c, g));
    }
    launches.swap(out);
  }

  // Reads the scalar decision of every blocked fiber whose value is now materialised with one
  // pack kernel + one D2H copy (instead of one synchronising read per fiber).
  bool wake_blocked() {
    std::vector<Fiber*> ready;
    for (auto& fb : ex.fibers_)
      if (fb->status == FiberStatus::kBlockedValue && is_materialized(fb->wait_ref)) ready.push_back(fb.get());
    if (ready.empty()) return false;
    std::vector<int64_t> offs;
    for (Fiber* fb : ready) offs.push_back(resolve(fb->wait_ref).offset);
    std::vector<float> vals = read_floats(offs);
    for (size_t k = 0; k < ready.size(); ++k) {
      ready[k]->wait_value = static_cast<long>(vals[k]);
      ready[k]->wait_value_ready = true;
      ready[k]->status = FiberStatus::kRunnable;
    }
    return true;
  }

  bool is_materialized(const TensorRef& r) const { return r.node < 0 || ex.nodes_[r.node].executed; }

  // Gathers single floats at arena offsets to the host (one kernel, one copy, one sync).
  std::vector<float> read_floats(const std::vector<int64_t>& offs) {
    std::vector<float> out(offs.size(), 0.0f);
    if (offs.empty() || c->dry) return out;
    std::vector<int64_t> ranges;
    for (size_t k = 0; k < offs.size(); ++k) {
      ranges.push_back(offs[k]);
      ranges.push_back(1);
      ranges.push_back(int64_t(k));
    }
    pack_to_host(ranges, out.data(), out.size());
    return out;
  }

  // sync = false (defer_sync): the read-back is enqueued, the copy out of the pinned buffer is
  // the caller's business after it synchronises.
  void pack_to_host(const std::vector<int64_t>& ranges, float* dst, size_t total, bool sync = true) {
    // Ranges that continue each other in the arena and in the output (batch-contiguous output
    // regions: TreeLSTM's logits are one run) go out as a few direct D2H copies: no pack kernel.
    std::vector<int64_t> runs;
    for (size_t k = 0; k + 2 < ranges.size() && runs.size() <= 24; k += 3) {
      const size_t r = runs.size();
      if (r && runs[r - 3] + runs[r - 2] == ranges[k] && runs[r - 1] + runs[r - 2] == ranges[k + 2])
        runs[r - 2] += ranges[k + 1];
      else
        runs.insert(runs.end(), {ranges[k], ranges[k + 1], ranges[k + 2]});
    }
    if (runs.size() <= 24) {
      mbx::ensure_d2h(c, total);
      if (c->copy_pending) {  // (meta_commit's job on the other path: inputs before any read)
        mbx::cuda_check(cudaStreamWaitEvent(c->stream, c->ev_copy, 0), "input copy wait");
        c->copy_pending = false;
      }
      for (size_t k = 0; k < runs.size(); k += 3)
        mbx::cuda_check(cudaMemcpyAsync(c->d2h_host + runs[k + 2], mbx::arena_ptr(c) + runs[k],
                                        size_t(runs[k + 1]) * sizeof(float), cudaMemcpyDeviceToHost, c->stream),
                        "D2H");
      if (sync) {
        mbx::stream_wait_own(c, "D2H sync");
        std::memcpy(dst, c->d2h_host, total * sizeof(float));
      }
      timing.d2h_bytes += long(total * sizeof(float));
      return;
    }
    {
      // Permuted but compact (one batch's output region read in instance order): one D2H of the
      // covering span, the permutation done on the host.
      int64_t lo = INT64_MAX, hi = 0;
      for (size_t k = 0; k + 2 < ranges.size(); k += 3) {
        lo = std::min(lo, ranges[k]);
        hi = std::max(hi, ranges[k] + ranges[k + 1]);
      }
      const int64_t span = hi - lo;
      if (span > 0 && size_t(span) <= 4 * total + 1024) {
        mbx::ensure_d2h(c, std::max(total, size_t(span)));
        if (c->copy_pending) {
          mbx::cuda_check(cudaStreamWaitEvent(c->stream, c->ev_copy, 0), "input copy wait");
          c->copy_pending = false;
        }
        mbx::cuda_check(cudaMemcpyAsync(c->d2h_host, mbx::arena_ptr(c) + lo, size_t(span) * sizeof(float),
                                        cudaMemcpyDeviceToHost, c->stream),
                        "D2H");
        if (sync) {
          mbx::stream_wait_own(c, "D2H sync");
          for (size_t k = 0; k + 2 < ranges.size(); k += 3)
            std::memcpy(dst + ranges[k + 2], c->d2h_host + (ranges[k] - lo), size_t(ranges[k + 1]) * sizeof(float));
        }
        timing.d2h_bytes += long(span * int64_t(sizeof(float)));
        return;
      }
    }
    mbx::meta_reserve(c, ranges.size() * 8 + 64);
    size_t moff = mbx::meta_stage(c, ranges.data(), ranges.size() * 8);
    mbx::meta_commit(c);
    mbx::ensure_d2h(c, total);
    mbx::cuda_check(mbx::launch_pack_ranges(mbx::arena_ptr(c), mbx::meta_dev<int64_t>(c, moff),
                                            int(ranges.size() / 3), c->d2h_dev, c->stream),
                    "pack ranges");
    ++c->launches;
    ++timing.device_launches;
    mbx::cuda_check(cudaMemcpyAsync(c->d2h_host, c->d2h_dev, total * sizeof(float), cudaMemcpyDeviceToHost, c->stream),
                    "D2H");
    if (sync) {
      mbx::stream_wait_own(c, "D2H sync");
      std::memcpy(dst, c->d2h_host, total * sizeof(float));
    }
    timing.d2h_bytes += long(total * sizeof(float));
    timing.h2d_bytes += long(ranges.size() * 8);
  }

  void collect_tensors(const Val& v, std::vector<TensorHandle>& out) {
    if (v.kind == Val::kTensor) out.push_back(resolve(v.t));
    for (size_t k = 0; k < v.size(); ++k) collect_tensors(v.at(k), out);
  }

  HostValue to_host(const Val& v, const std::vector<float>& buf, size_t& cursor, size_t& ti,
                    const std::vector<TensorHandle>& hs) {
    switch (v.kind) {
      case Val::kTensor: {
        const TensorHandle& h = hs[ti++];
        std::vector<float> d(buf.begin() + cursor, buf.begin() + cursor + h.size());
        cursor += h.size();
        return HostValue::tensor(h.shape, std::move(d));
      }
      case Val::kInt: return HostValue::scalar(v.i);
      case Val::kFloat: {
        HostValue h;
        h.kind = HostValue::Kind::kFloat;
        h.fval = v.real_value();
        return h;
      }
      default: {
        std::vector<HostValue> items;
        for (size_t k = 0; k < v.size(); ++k) items.push_back(to_host(v.at(k), buf, cursor, ti, hs));
        if (v.kind == Val::kList) return HostValue::list(std::move(items));
        if (v.kind == Val::kTuple) return HostValue::tuple(std::move(items));
        return HostValue::adt(v.ctor == 1 ? "Node" : "Leaf", std::move(items));
      }
    }
  }
};

Executor::Executor(Session& s, const std::vector<InstanceInput>& inputs, const ExecOptions& opts)
    : impl_(std::make_unique<Impl>(*this, s, inputs, opts)) {}

namespace {
const std::vector<InstanceInput> kNoInputs;
}

Executor::Executor(Session& s, const EncodedValues& inputs, const ExecOptions& opts, EncodedOutputs* out)
    : impl_(std::make_unique<Impl>(*this, s, kNoInputs, opts)) {
  impl_->enc = &inputs;
  impl_->enc_out = out;
  impl_->batch = inputs.count;
}
Executor::~Executor() = default;

int Executor::emit(Fiber& fb, int blk, std::initializer_list<const Val*> inputs) { return impl_->emit(fb, blk, inputs); }
void Executor::stage(Fiber& fb, int st) { impl_->stage(fb, st); }
void Executor::ghosts(Fiber& fb, int count) { impl_->ghosts(fb, count); }
bool Executor::ghost_enabled() const { return impl_->opts.ghost; }
bool Executor::hoist_enabled() const { return impl_->opts.hoist; }

long Executor::read_scalar_now(const TensorRef& r) {
  std::vector<float> v = impl_->read_floats({impl_->resolve(r).offset});
  return static_cast<long>(v[0]);
}

JoinAwait Executor::concurrent(Fiber& fb, std::vector<Call> calls) {
  // A single call is not a fork (executor.cpp:524-528): run it as a one-child group anyway is
  // not equivalent, so callers only use this for groups of >= 2 calls.
  fb.children.clear();
  for (auto& call : calls) {
    auto child = std::make_unique<Fiber>();
    child->id = static_cast<int>(fibers_.size());
    child->instance = fb.instance;
    child->parent = fb.id;
    child->phase = fb.phase;
    child->depth_counter = fb.depth_counter;
    Fiber* raw = child.get();
    child->root = call(*raw);
    fb.children.push_back(child->id);
    fibers_.push_back(std::move(child));
  }
  return JoinAwait{this, &fb};
}

void JoinAwait::await_suspend(std::coroutine_handle<> h) {
  fb->status = FiberStatus::kBlockedJoin;
  fb->pending_children = static_cast<int>(fb->children.size());
  fb->resume_point = h;
}

std::vector<Val> JoinAwait::await_resume() {
  std::vector<Val> out;
  out.reserve(fb->children.size());
  auto& fibers = ex->fibers();
  for (int id : fb->children) {
    Fiber& child = *fibers[id];
    MBATCH_CHECK(child.has_result, "joined child fiber without a result");
    out.push_back(child.result);
    fb->depth_counter = std::max(fb->depth_counter, child.depth_counter);
  }
  fb->children.clear();
  return out;
}

bool ScalarAwait::await_ready() { return ex->is_materialized(ref); }
void ScalarAwait::await_suspend(std::coroutine_handle<> h) {
  fb->status = FiberStatus::kBlockedValue;
  fb->wait_ref = ref;
  fb->wait_value_ready = false;
  fb->resume_point = h;
}
long ScalarAwait::await_resume() {
  if (fb->wait_value_ready) {
    fb->wait_value_ready = false;
    return fb->wait_value;
  }
  return ex->read_scalar_now(ref);
}

EvalResult Executor::run() {
  Impl& I = *impl_;
  auto t0 = clk::now();
  const CompiledModel& m = I.m;
  I.input_base = I.c->used;
  std::vector<Val> param_vals;
  nodes_.reserve(I.s.node_hint());    // the previous evaluation's node count: no regrowth
  fibers_.reserve(I.s.fiber_hint());
  int64_t eti = 0, edi = 0;  // encoded inputs: cursor into the token / data streams
  const char* flat_env = std::getenv("MBX_FLAT_DFG");  // 0: the coroutine path (tests compare both)
  const bool flat_ok = !flat_env || std::atoi(flat_env) != 0;
  const bool flat = flat_ok && m.program->has_flat();
  std::vector<std::vector<Val>> flat_args;
  std::vector<Fiber*> flat_roots;
  for (size_t i = 0; i < size_t(I.batch); ++i) {
    auto fb = std::make_unique<Fiber>();
    fb->id = static_cast<int>(fibers_.size());
    fb->instance = static_cast<int>(i);
    std::vector<Val> args;
    for (const auto& d : m.params) {
      if (d.is_instance_input) {
        if (I.enc) {
          args.push_back(I.materialize_enc(eti, edi));
          continue;
        }
        auto it = I.inputs[i].find(d.name);
        MBATCH_CHECK(it != I.inputs[i].end(), "missing instance input " + d.name);
        args.push_back(I.materialize(it->second));
      } else {
        args.push_back(Val::tensor(TensorRef{-1, 0, I.s.param_handles().at(d.name)}));
      }
    }
    Fiber* raw = fb.get();
    if (flat) {
      flat_roots.push_back(raw);
      flat_args.push_back(std::move(args));
    } else {
      fb->root = m.program->run(*this, *raw, std::move(args));
    }
    fibers_.push_back(std::move(fb));
  }
  if (I.enc) MBATCH_CHECK(eti == I.enc->ntok && edi == I.enc->ndata, "hostval encoding: trailing data");
  I.upload_inputs();
  if (flat) {
    auto tf = clk::now();
    m.program->run_flat(*this, flat_roots, flat_args);
    for (Fiber* fb : flat_roots) MBATCH_CHECK(fb->status == FiberStatus::kDone, "flat DFG builder left a fiber running");
    I.timing.host_fibers_us += std::chrono::duration<double, std::micro>(clk::now() - tf).count();
  }

  while (true) {
    auto tf = clk::now();
    I.run_runnable();
    I.timing.host_fibers_us += std::chrono::duration<double, std::micro>(clk::now() - tf).count();
    bool all_done = true;
    for (const auto& fb : fibers_) all_done = all_done && fb->status == FiberStatus::kDone;
    if (all_done) break;
    int phase_limit = INT_MAX;
    for (const auto& fb : fibers_)
      if (fb->status != FiberStatus::kDone) phase_limit = std::min(phase_limit, fb->phase);
    bool executed = I.flush(phase_limit);
    ++I.trace.sync_points;
    bool woke = I.wake_blocked();
    if (!woke) {
      MBATCH_CHECK(executed, "fiber deadlock: all fibers blocked with an empty pending DFG");
      MBATCH_CHECK(false, "fiber deadlock: flush made no fiber runnable");
    }
  }
  I.flush(INT_MAX);

  // Outputs: one pack + one D2H for every tensor of every instance result.
  std::vector<TensorHandle> hs;
  for (size_t i = 0; i < size_t(I.batch); ++i) I.collect_tensors(fibers_[i]->result, hs);
  std::vector<int64_t> ranges;
  size_t total = 0;
  for (const auto& h : hs) {
    ranges.push_back(h.offset);
    ranges.push_back(h.size());
    ranges.push_back(int64_t(total));
    total += size_t(h.size());
  }
  auto t_host = clk::now();
  // Outputs left on the device: no read-back and no host values (the result carries none).
  const bool keep = I.opts.outputs_on_device && !I.c->dry;
  std::vector<float> buf(keep ? 0 : total, 0.0f);
  const bool defer = I.opts.defer_sync && !I.c->dry;
  if (!I.c->dry && total > 0 && !I.opts.outputs_on_device) I.pack_to_host(ranges, buf.data(), total, !defer);
  else if (!I.c->dry && !defer) mbx::stream_wait_own(I.c, "final sync");
  if (I.c->copy_pending) {  // inputs no kernel read: the pinned staging is reused next call
    mbx::cuda_check(cudaEventSynchronize(I.c->ev_copy), "input copy");
    I.c->copy_pending = false;
  }

  EvalResult res;
  size_t cursor = 0, ti = 0;
  if (!defer && !keep) {  // deferred: the outputs are read back but not decoded
    if (I.enc_out) {
      for (size_t i = 0; i < size_t(I.batch); ++i) I.to_tokens(fibers_[i]->result, buf, cursor, ti, hs, *I.enc_out);
      I.enc_out->toks.shrink_to_fit();
    } else {
      for (size_t i = 0; i < size_t(I.batch); ++i) res.outputs.push_back(I.to_host(fibers_[i]->result, buf, cursor, ti, hs));
    }
  }
  I.trace.total_nodes = static_cast<long>(nodes_.size());
  for (const auto& n : nodes_) I.trace.dfg_edges += static_cast<long>(n.producers.size());
  res.trace = std::move(I.trace);
  I.s.set_hints(int64_t(nodes_.size()), int64_t(fibers_.size()));
  if (I.opts.record_nodes) {
    res.nodes = std::move(nodes_);
  } else {  // back to the session's pool for the next evaluation
    auto& pool = I.s.node_pool();
    pool.reserve(pool.size() + nodes_.size());
    for (auto& n : nodes_) pool.push_back(std::move(n));
    nodes_.clear();
  }
  for (auto& [a, b] : I.flush_events) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    I.timing.device_span_us += ms * 1000.0;
  }
  for (size_t k = 0; k < I.batch_events.size(); ++k) {
    float ms = 0;
    cudaEventElapsedTime(&ms, I.batch_events[k].first, I.batch_events[k].second);
    const int n = I.batch_share[k];
    for (int j = 0; j < n; ++j) I.timing.batch_us.push_back(ms * 1000.0 / n);
  }
  I.timing.host_dfg_us = std::chrono::duration<double, std::micro>(t_host - t0).count();
  I.timing.host_total_us = std::chrono::duration<double, std::micro>(clk::now() - t0).count();
  res.timing = I.timing;
  return res;
}

}  // namespace runtime
}  // namespace mbatch
