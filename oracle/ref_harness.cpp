// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// Driver around the UNMODIFIED reference library (compiled from /root/reference/proj/src by
// oracle/Makefile).  It never changes reference behaviour; it only
//   * builds a zoo model at an arbitrary hidden size H (token substitution on the reference's own
//     zoo text at H=32, see `model_source`),
//   * runs runtime::compile / evaluate_batch / reference_evaluate exactly as metrics::run_once
//     does (proj/src/metrics.cpp:71-102), and
//   * dumps the compiled kernel library, the schedule trace, the DFG node table and the outputs
//     as JSON (`dump`), or times the batched and unbatched CPU paths (`time`).
// The dumps are the golden fixtures under tests/golden/ and the parity target of the B200 path.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <regex>

#include <json.hpp>

#include "mbatch/runtime.hpp"
#include "mbatch/zoo.hpp"

using namespace mbatch;
using json = nlohmann::ordered_json;

namespace {

// The reference zoo only emits H in {32, 64} (proj/src/zoo.cpp:306-307).  Its templates substitute
// {2H}, {H}, {C}=8; at "small" that is 64, 32, 8.  Re-substituting the numeric tokens 64 -> 2H and
// 32 -> H yields the template at any H (checked: H=64 reproduces get_model(name, "large")).
std::string model_source(const std::string& name, int hidden) {
  std::string src = zoo::get_model(name, "small").source;
  std::regex tok("\\b(64|32)\\b");
  std::string out;
  auto begin = std::sregex_iterator(src.begin(), src.end(), tok);
  size_t last = 0;
  for (auto it = begin; it != std::sregex_iterator(); ++it) {
    out += src.substr(last, it->position() - last);
    out += it->str() == "64" ? std::to_string(2 * hidden) : std::to_string(hidden);
    last = it->position() + it->length();
  }
  out += src.substr(last);
  return out;
}

struct Args {
  std::string cmd = "dump", model = "treelstm", out;
  int hidden = 32, batch = 8, reps = 3, warmup = 1;
  unsigned seed = 1;
  bool nodes = true, outputs = true, verify = true;
  runtime::ExecOptions opts;
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc > 1) a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::runtime_error("missing value for " + k);
      return argv[++i];
    };
    if (k == "--model") a.model = next();
    else if (k == "--hidden") a.hidden = std::stoi(next());
    else if (k == "--batch") a.batch = std::stoi(next());
    else if (k == "--seed") a.seed = static_cast<unsigned>(std::stoul(next()));
    else if (k == "--reps") a.reps = std::stoi(next());
    else if (k == "--warmup") a.warmup = std::max(1, std::stoi(next()));
    else if (k == "--out") a.out = next();
    else if (k == "--scheduler") a.opts.scheduler = next() == "agenda" ? runtime::ExecOptions::Scheduler::kAgenda
                                                                        : runtime::ExecOptions::Scheduler::kDepth;
    else if (k == "--gather") a.opts.gather = next() == "explicit" ? backend::GatherMode::kExplicit
                                                                    : backend::GatherMode::kFused;
    else if (k == "--no-coarsen") a.opts.coarsen = false;
    else if (k == "--no-ghost") a.opts.ghost = false;
    else if (k == "--no-phases") a.opts.phases = false;
    else if (k == "--no-hoist") a.opts.hoist = false;
    else if (k == "--no-hfuse") a.opts.horizontal_fuse = false;
    else if (k == "--no-nodes") a.nodes = false;
    else if (k == "--no-outputs") a.outputs = false;
    else if (k == "--no-verify") a.verify = false;
    else throw std::runtime_error("unknown flag " + k);
  }
  return a;
}

const char* kind_name(backend::PlanRef::Kind k) {
  switch (k) {
    case backend::PlanRef::Kind::kShared: return "S";
    case backend::PlanRef::Kind::kBatched: return "B";
    case backend::PlanRef::Kind::kTemp: return "T";
  }
  return "?";
}

json ref_json(const backend::PlanRef& r) { return json::array({kind_name(r.kind), r.index, r.col_off, r.cols}); }
json shape_json(const backend::Shape& s) { return json::array({s.rows, s.cols}); }

json plan_json(const backend::ExecutablePlan& p) {
  json j;
  j["ghost"] = p.ghost;
  j["shared_shapes"] = json::array();
  for (auto& s : p.shared_shapes) j["shared_shapes"].push_back(shape_json(s));
  j["batched_shapes"] = json::array();
  for (auto& s : p.batched_shapes) j["batched_shapes"].push_back(shape_json(s));
  j["steps"] = json::array();
  for (auto& st : p.steps) {
    json s;
    s["kind"] = st.kind == backend::PlanStep::Kind::kOp ? "op"
                : st.kind == backend::PlanStep::Kind::kFusedDense ? "fused_dense" : "chain";
    s["op"] = backend::op_name(st.op);
    s["ins"] = json::array();
    for (auto& r : st.ins) s["ins"].push_back(ref_json(r));
    s["chain"] = json::array();
    for (auto& l : st.chain) {
      json c;
      c["op"] = backend::op_name(l.op);
      c["rhs"] = l.rhs ? ref_json(*l.rhs) : json(nullptr);
      s["chain"].push_back(c);
    }
    s["out"] = shape_json(st.out_shape);
    j["steps"].push_back(s);
  }
  j["outputs"] = json::array();
  for (auto& r : p.outputs) j["outputs"].push_back(ref_json(r));
  return j;
}

json host_json(const runtime::HostValue& v) {
  using K = runtime::HostValue::Kind;
  json j;
  switch (v.kind) {
    case K::kTensor: {
      j["k"] = "t";
      j["s"] = shape_json(v.shape);
      json d = json::array();
      for (float f : v.data) d.push_back(f);
      j["d"] = d;
      break;
    }
    case K::kInt: j["k"] = "i"; j["v"] = v.ival; break;
    case K::kFloat: j["k"] = "f"; j["v"] = v.fval; break;
    case K::kList: case K::kTuple: case K::kAdt: {
      j["k"] = v.kind == K::kList ? "l" : v.kind == K::kTuple ? "u" : "a";
      if (v.kind == K::kAdt) j["c"] = v.ctor;
      j["items"] = json::array();
      for (auto& it : v.items) j["items"].push_back(host_json(it));
      break;
    }
  }
  return j;
}

// FNV-1a over the float bit patterns of every tensor, depth-first in value order.
void digest(const runtime::HostValue& v, uint64_t& h) {
  auto mix = [&](uint64_t x) { h ^= x; h *= 1099511628211ull; };
  if (v.kind == runtime::HostValue::Kind::kTensor) {
    for (float f : v.data) { uint32_t b; std::memcpy(&b, &f, 4); mix(b); }
  } else if (v.kind == runtime::HostValue::Kind::kInt) {
    mix(static_cast<uint64_t>(v.ival));
  }
  for (auto& it : v.items) digest(it, h);
}

std::string hex64(uint64_t h) { char buf[32]; std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)h); return buf; }

int run(const Args& a) {
  std::string src = model_source(a.model, a.hidden);
  ir::Program prog = ir::parse_program(src);
  runtime::CompiledModel m = runtime::compile(prog, a.opts);
  zoo::ModelSpec spec = zoo::get_model(a.model, "small");
  auto params = zoo::make_params(spec, m.typed.program, a.seed);
  auto inputs = zoo::make_inputs(spec, m.typed.program, a.seed, a.batch);

  if (a.cmd == "source") { std::cout << src; return 0; }

  if (a.cmd == "time") {
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point t0) { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); };
    runtime::EvalResult res = runtime::evaluate_batch(m, params, inputs);  // warm-up
    for (int w = 1; w < a.warmup; ++w) res = runtime::evaluate_batch(m, params, inputs);
    double best_b = 1e300, sum_b = 0, best_u = 1e300, sum_u = 0;
    for (int r = 0; r < a.reps; ++r) {
      auto t0 = clk::now();
      res = runtime::evaluate_batch(m, params, inputs);
      double t = ms(t0); best_b = std::min(best_b, t); sum_b += t;
    }
    int ureps = a.verify ? a.reps : 0;
    for (int r = 0; r < ureps; ++r) {
      auto t0 = clk::now();
      auto ref = runtime::reference_evaluate(m, params, inputs);
      double t = ms(t0); best_u = std::min(best_u, t); sum_u += t;
    }
    json j;
    j["model"] = a.model; j["hidden"] = a.hidden; j["batch"] = a.batch; j["seed"] = a.seed;
    j["reps"] = a.reps;
    j["warmup"] = a.warmup;
    j["nodes"] = res.trace.total_nodes;
    j["launches"] = res.trace.kernel_launches;
    j["sync_points"] = res.trace.sync_points;
    j["batched_ms_best"] = best_b; j["batched_ms_mean"] = sum_b / a.reps;
    if (ureps) { j["unbatched_ms_best"] = best_u; j["unbatched_ms_mean"] = sum_u / ureps; }
    std::cout << j.dump() << std::endl;
    return 0;
  }

  runtime::EvalResult res = runtime::evaluate_batch(m, params, inputs);
  json j;
  j["model"] = a.model; j["hidden"] = a.hidden; j["batch"] = a.batch; j["seed"] = a.seed;
  j["opts"] = {{"scheduler", a.opts.scheduler == runtime::ExecOptions::Scheduler::kDepth ? "depth" : "agenda"},
               {"gather", a.opts.gather == backend::GatherMode::kFused ? "fused" : "explicit"},
               {"coarsen", a.opts.coarsen}, {"ghost", a.opts.ghost}, {"phases", a.opts.phases},
               {"hoist", a.opts.hoist}, {"horizontal_fuse", a.opts.horizontal_fuse}};
  j["params"] = json::array();
  j["instance_inputs"] = json::array();
  for (auto& d : m.module.params) {
    if (d.is_instance_input) j["instance_inputs"].push_back(d.name);
    else j["params"].push_back({{"name", d.name}, {"shape", shape_json(d.type->shape)}});
  }
  // Digests of the seeded synthetic inputs, so a re-implementation of the zoo generators can be
  // checked without shipping the tensors.
  uint64_t hp = 1469598103934665603ull, hi = 1469598103934665603ull;
  for (auto& d : m.module.params)
    if (!d.is_instance_input) digest(params.at(d.name), hp);
  for (auto& inst : inputs)
    for (auto& d : m.module.params)
      if (d.is_instance_input) digest(inst.at(d.name), hi);
  j["digests"] = {{"params", hex64(hp)}, {"inputs", hex64(hi)}};

  j["signatures"] = json::array();
  for (auto& s : m.kernels.signatures) {
    json sj;
    sj["id"] = s.id; sj["name"] = s.name; sj["ghost"] = s.ghost;
    sj["shared"] = json::array();
    for (auto& [n, sh] : s.shared_params) sj["shared"].push_back({n, sh.rows, sh.cols});
    sj["batched"] = json::array();
    for (auto& [n, sh] : s.batched_params) sj["batched"].push_back({n, sh.rows, sh.cols});
    sj["outputs"] = json::array();
    for (auto& sh : s.outputs) sj["outputs"].push_back(shape_json(sh));
    sj["structural_key"] = s.structural_key;
    j["signatures"].push_back(sj);
  }
  j["ghost_sig"] = m.kernels.ghost_sig;
  j["plans"] = json::array();
  for (auto& p : m.kernels.plans) j["plans"].push_back(plan_json(p));
  j["blocks"] = json::array();
  for (auto& b : m.blocks.blocks) {
    json bj;
    auto& bind = m.kernels.binding_of_block.at(b.id);
    bj["id"] = b.id; bj["func"] = b.func; bj["sig"] = bind.sig_id;
    bj["inputs"] = b.inputs; bj["outputs"] = b.outputs;
    bj["shared_pos"] = bind.shared_input_pos; bj["batched_pos"] = bind.batched_input_pos;
    auto h = m.hoist.static_depth.find(b.id);
    bj["hoist"] = (a.opts.hoist && h != m.hoist.static_depth.end()) ? json(h->second) : json(nullptr);
    bj["prim_sites"] = b.prim_sites; bj["trigger_site"] = b.trigger_site;
    j["blocks"].push_back(bj);
  }
  j["stage_phase"] = m.phases.stage_phase;

  const auto& t = res.trace;
  json tj;
  tj["batches"] = json::array();
  for (auto& b : t.batches)
    tj["batches"].push_back({{"phase", b.phase}, {"depth", b.depth}, {"sig", b.sig}, {"size", b.size},
                             {"ghost", b.ghost}, {"nodes", b.node_ids}});
  tj["kernel_launches"] = t.kernel_launches; tj["total_nodes"] = t.total_nodes;
  tj["scheduler_ops"] = t.scheduler_ops; tj["sync_points"] = t.sync_points;
  tj["gather_bytes"] = t.gather_bytes; tj["dfg_edges"] = t.dfg_edges;
  tj["flush_boundaries"] = t.flush_boundaries;
  j["trace"] = tj;

  if (a.nodes) {
    j["nodes"] = json::array();
    for (auto& n : res.nodes) {
      json nj;
      nj["id"] = n.id; nj["sig"] = n.sig_id; nj["block"] = n.block_id; nj["inst"] = n.instance;
      nj["phase"] = n.phase; nj["depth"] = n.depth; nj["ghost"] = n.ghost;
      nj["shared"] = json::array();
      for (auto& r : n.shared_ins) nj["shared"].push_back({r.node, r.out, r.handle.offset});
      nj["batched"] = json::array();
      for (auto& r : n.batched_ins) nj["batched"].push_back({r.node, r.out, r.handle.offset});
      nj["producers"] = n.producers;
      nj["outputs"] = json::array();
      for (auto& h : n.outputs) nj["outputs"].push_back({h.offset, h.shape.rows, h.shape.cols});
      j["nodes"].push_back(nj);
    }
  }
  if (a.outputs) {
    j["outputs"] = json::array();
    for (auto& o : res.outputs) j["outputs"].push_back(host_json(o));
  }
  uint64_t ho = 1469598103934665603ull;
  for (auto& o : res.outputs) digest(o, ho);
  j["digests"]["outputs"] = hex64(ho);
  if (a.verify) {
    auto ref = runtime::reference_evaluate(m, params, inputs);
    bool ok = ref.size() == res.outputs.size();
    for (size_t i = 0; ok && i < ref.size(); ++i) ok = runtime::bitwise_equal(ref[i], res.outputs[i]);
    j["batched_equals_unbatched"] = ok;
  }
  if (a.out.empty()) {
    std::cout << j.dump() << std::endl;
  } else {
    std::ofstream f(a.out);
    f << j.dump() << std::endl;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(parse(argc, argv));
  } catch (const std::exception& e) {
    std::cerr << "mbatch_ref: " << e.what() << std::endl;
    return 2;
  }
}
