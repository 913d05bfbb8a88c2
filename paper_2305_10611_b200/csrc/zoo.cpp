// zoo.cpp — the evaluation models compiled for the B200 runtime.
//
// For each model of the reference zoo (proj/src/zoo.cpp:26-279) this file provides what the
// reference's compile pipeline (proj/src/pipeline.cpp:65-97) would hand the executor:
//   * the kernel library: signature names, shared/batched parameter split, lowered plans
//     (proj/src/kernelgen.cpp: build_dag + lower_block_to_kernel),
//   * the static blocks with their bindings and hoist depths (proj/src/analysis.cpp),
//   * the phase of each top-level stage of @main,
//   * an AOT-lowered body: C++ coroutines that walk the instance input and emit one DFG node per
//     static-block invocation in the order the reference interpreter reaches the block's trigger
//     site, suspending on scalar() and forking concurrent calls onto child fibers.
// tests/test_zoo_parity.py checks every artefact against the reference compiler's own dump
// (tests/golden/*.json) and every trace against the reference executor's.
#include "mbatch/zoo.hpp"

#include <deque>
#include <random>

#include "exec.h"

namespace mbatch {
namespace zoo {

using backend::ChainLink;
using backend::ExecutablePlan;
using backend::OpCode;
using backend::PlanRef;
using backend::PlanStep;
using backend::Shape;
using runtime::Call;
using runtime::Executor;
using runtime::Fiber;
using runtime::Task;
using runtime::Val;

namespace {

// ---- plan construction helpers ------------------------------------------------------------

PlanRef S(int i) { return PlanRef{PlanRef::Kind::kShared, i, 0, -1}; }
PlanRef B(int i) { return PlanRef{PlanRef::Kind::kBatched, i, 0, -1}; }
PlanRef T(int i) { return PlanRef{PlanRef::Kind::kTemp, i, 0, -1}; }
PlanRef Tc(int i, int off, int cols) { return PlanRef{PlanRef::Kind::kTemp, i, off, cols}; }
ChainLink L(OpCode op) { return ChainLink{op, std::nullopt}; }
ChainLink L(OpCode op, PlanRef rhs) { return ChainLink{op, rhs}; }

struct PlanBuilder {
  ExecutablePlan p;
  PlanBuilder(std::vector<Shape> shared, std::vector<Shape> batched) {
    p.shared_shapes = std::move(shared);
    p.batched_shapes = std::move(batched);
  }
  PlanBuilder& op(OpCode o, std::vector<PlanRef> ins, Shape out) {
    PlanStep s;
    s.kind = PlanStep::Kind::kOp;
    s.op = o;
    s.ins = std::move(ins);
    s.out_shape = out;
    p.steps.push_back(std::move(s));
    return *this;
  }
  PlanBuilder& fused(std::vector<PlanRef> ins, Shape out) {
    PlanStep s;
    s.kind = PlanStep::Kind::kFusedDense;
    s.op = OpCode::kDense;
    s.ins = std::move(ins);
    s.out_shape = out;
    p.steps.push_back(std::move(s));
    return *this;
  }
  PlanBuilder& chain(PlanRef base, std::vector<ChainLink> links, Shape out) {
    PlanStep s;
    s.kind = PlanStep::Kind::kChain;
    s.op = OpCode::kAdd;
    s.ins = {base};
    s.chain = std::move(links);
    s.out_shape = out;
    p.steps.push_back(std::move(s));
    return *this;
  }
  ExecutablePlan outputs(std::vector<PlanRef> outs) {
    p.outputs = std::move(outs);
    return p;
  }
};

// dense(B0, S0) followed by an elementwise tail: bias_dense / *_bias_dense signatures.
ExecutablePlan dense_tail(Shape w, Shape bias, Shape x, std::vector<ChainLink> tail, std::vector<Shape> extra_batched = {}) {
  std::vector<Shape> batched{x};
  for (auto& s : extra_batched) batched.push_back(s);
  std::vector<Shape> shared{w};
  if (bias.size() > 0) shared.push_back(bias);
  Shape out{1, w.cols};
  return PlanBuilder(shared, batched).op(OpCode::kDense, {B(0), S(0)}, out).chain(T(0), std::move(tail), out).outputs({T(1)});
}

// ---- compiled-model assembly ----------------------------------------------------------------

struct ModelBuilder {
  runtime::CompiledModel m;
  ModelBuilder(const std::string& name, int H) {
    m.name = name;
    m.hidden = H;
  }
  void param(const std::string& n, int r, int c) { m.params.push_back({n, Shape{r, c}, false}); }
  void input(const std::string& n) { m.params.push_back({n, Shape{}, true}); }
  int sig(const std::string& name, std::vector<std::pair<std::string, Shape>> shared,
          std::vector<std::pair<std::string, Shape>> batched, std::vector<Shape> outs, ExecutablePlan plan) {
    kernelgen::KernelSignature s;
    s.id = static_cast<int>(m.kernels.signatures.size());
    s.name = name;
    s.shared_params = std::move(shared);
    s.batched_params = std::move(batched);
    s.outputs = std::move(outs);
    m.kernels.signatures.push_back(s);
    m.kernels.plans.push_back(std::move(plan));
    return s.id;
  }
  void ghost() {
    kernelgen::KernelSignature g;
    g.id = static_cast<int>(m.kernels.signatures.size());
    g.name = "ghost";
    g.ghost = true;
    m.kernels.ghost_sig = g.id;
    m.kernels.signatures.push_back(g);
    ExecutablePlan p;
    p.ghost = true;
    m.kernels.plans.push_back(p);
  }
  void block(int id, const std::string& func, int sig, std::vector<std::string> inputs, std::vector<int> shared_pos,
             std::vector<int> batched_pos, int hoist, int nout) {
    runtime::StaticBlockInfo b;
    b.id = id;
    b.func = func;
    b.sig = sig;
    b.hoist = hoist;
    b.inputs = std::move(inputs);
    b.num_outputs = nout;
    m.blocks.push_back(b);
    kernelgen::BlockBinding bind;
    bind.sig_id = sig;
    bind.shared_input_pos = std::move(shared_pos);
    bind.batched_input_pos = std::move(batched_pos);
    m.kernels.binding_of_block[id] = bind;
  }
};

std::pair<std::string, Shape> P(const std::string& n, int r, int c) { return {n, Shape{r, c}}; }

// =============================================================================================
// Model bodies.  Each Program receives @main's parameters in module order.

// Programs without awaits (rnn, birnn, fig5): each root fiber runs start to finish when the first
// scheduler pass resumes it, in instance order — run_flat calls the same body in that order.
class StraightProgram : public runtime::Program {
 public:
  virtual Val body(Executor& ex, Fiber& fb, std::vector<Val>& a) const = 0;
  Task run(Executor& ex, Fiber& fb, std::vector<Val> a) const override { co_return body(ex, fb, a); }
  bool has_flat() const override { return true; }
  void run_flat(Executor& ex, std::vector<Fiber*>& roots, std::vector<std::vector<Val>>& args) const override {
    for (size_t i = 0; i < roots.size(); ++i) {
      Fiber& fb = *roots[i];
      fb.result = body(ex, fb, args[i]);
      fb.has_result = true;
      fb.status = runtime::FiberStatus::kDone;
    }
  }
};

// ---- rnn (zoo.cpp:26-45) / birnn (zoo.cpp:47-76) ----------------------------------------------
// @rnn: per element, inp_linear = bias + dense(inp, i_wt) [hoisted block], then
// new_state = sigmoid(inp_linear + dense(state, h_wt)) [recurrent block].
std::vector<Val> rnn_chain(Executor& ex, Fiber& fb, const Val& inps, Val state, const Val& bias, const Val& i_wt,
                           const Val& h_wt, int blk_in, int blk_rec) {
  std::vector<Val> out;
  for (size_t k = 0; k < inps.size(); ++k) {
    const Val& inp = inps.at(k);
    Val inp_linear = Executor::out(ex.emit(fb, blk_in, {&inp, &i_wt, &bias}), 0);
    Val ns = Executor::out(ex.emit(fb, blk_rec, {&state, &h_wt, &inp_linear}), 0);
    out.push_back(ns);
    state = ns;
  }
  return out;
}

class RnnProgram : public StraightProgram {
 public:
  Val body(Executor& ex, Fiber& fb, std::vector<Val>& a) const override {
    // a: rnn_bias, rnn_i_wt, rnn_h_wt, rnn_init, c_wt, cbias, inps
    ex.stage(fb, 0);
    std::vector<Val> res = rnn_chain(ex, fb, a[6], a[3], a[0], a[1], a[2], 1, 2);
    ex.stage(fb, 1);
    int start = fb.depth_counter, deepest = start;  // @map: shared start depth
    std::vector<Val> out;
    for (auto& p : res) {
      fb.depth_counter = start;
      out.push_back(Executor::out(ex.emit(fb, 0, {&p, &a[4], &a[5]}), 0));
      deepest = std::max(deepest, fb.depth_counter);
    }
    fb.depth_counter = deepest;
    return Val::list(std::move(out));
  }
};

class BirnnProgram : public StraightProgram {
 public:
  Val body(Executor& ex, Fiber& fb, std::vector<Val>& a) const override {
    // a: f_bias, f_i_wt, f_h_wt, f_init, b_bias, b_i_wt, b_h_wt, b_init, inps_list
    ex.stage(fb, 0);
    std::vector<Val> rev(a[8].items->rbegin(), a[8].items->rend());
    Val rinps = Val::list(rev);
    ex.stage(fb, 1);
    std::vector<Val> fwd = rnn_chain(ex, fb, a[8], a[3], a[0], a[1], a[2], 1, 2);
    ex.stage(fb, 2);
    std::vector<Val> bwd = rnn_chain(ex, fb, rinps, a[7], a[4], a[5], a[6], 3, 4);
    ex.stage(fb, 3);
    std::reverse(bwd.begin(), bwd.end());
    int start = fb.depth_counter, deepest = start;  // @map2
    std::vector<Val> out;
    for (size_t k = 0; k < fwd.size(); ++k) {
      fb.depth_counter = start;
      out.push_back(Executor::out(ex.emit(fb, 0, {&fwd[k], &bwd[k]}), 0));
      deepest = std::max(deepest, fb.depth_counter);
    }
    fb.depth_counter = deepest;
    return Val::list(std::move(out));
  }
};

// ---- treelstm (zoo.cpp:78-117) ------------------------------------------------------------
struct TreeLstmParams {
  Val x_wt, x_bias, xn, i_wt, fl_wt, fr_wt, u_wt, hz, cz, c_wt, cbias;
};

Task tlstm(Executor& ex, Fiber& fb, const TreeLstmParams& P, Val t) {
  if (t.ctor == 0) {  // Leaf(x): xt = x_bias + dense(x, x_wt) [hoisted 0]; tcell__c0 [hoisted 1]
    Val xt = Executor::out(ex.emit(fb, 3, {&t.at(0), &P.x_wt, &P.x_bias}), 0);
    int n = ex.emit(fb, 1, {&P.hz, &P.hz, &P.i_wt, &xt, &P.fl_wt, &P.fr_wt, &P.u_wt, &P.cz, &P.cz});
    co_return Val::tuple({Executor::out(n, 1), Executor::out(n, 0)});  // (tanh(c), c)
  }
  // The children's calls capture one pointer each (fits std::function's inline storage): the
  // subtrees live in this frame until the join, and tlstm copies its argument at the call.
  struct Sub { Executor* ex; const TreeLstmParams* P; const Val* t; };
  const Sub sl{&ex, &P, &t.at(0)}, sr{&ex, &P, &t.at(1)};
  std::vector<Call> calls;
  calls.reserve(2);
  calls.push_back([a = &sl](Fiber& f) { return tlstm(*a->ex, f, *a->P, *a->t); });
  calls.push_back([a = &sr](Fiber& f) { return tlstm(*a->ex, f, *a->P, *a->t); });
  runtime::JoinAwait join = ex.concurrent(fb, std::move(calls));
  std::vector<Val> res = co_await join;
  const Val &lh = res[0].at(0), &lc = res[0].at(1), &rh = res[1].at(0), &rc = res[1].at(1);
  int n = ex.emit(fb, 2, {&lh, &rh, &P.i_wt, &P.xn, &P.fl_wt, &P.fr_wt, &P.u_wt, &lc, &rc});
  co_return Val::tuple({Executor::out(n, 1), Executor::out(n, 0)});
}

// The fiber scheduler's order for tlstm without coroutines (Program::run_flat): light fibers in
// creation order, resumed in passes over the growing list exactly as run_runnable does — a tree
// node's fiber spawns its two children (appended) and blocks; leaves emit and finish in the same
// pass; a parent resumes in the pass after its last child finished (its depth counter the max of
// its children's), emits its cell, and finishes; a root then takes stage 1 and the classifier.
struct FlatTree {
  Fiber* fb;
  const Val* t;
  int parent;
  int state;  // 0: not started, 1: resumed after its join
  int kids[2];
  int inst;   // instance (its params)
  Val res[2]; // the finished subtree's pair (e.g. (h, c)): no tuple allocated per tree node
};

// Tree nodes below the roots (one child fiber each).
inline size_t count_subtrees(const Val& t) {
  if (t.ctor == 0) return 0;
  return 2 + count_subtrees(t.at(0)) + count_subtrees(t.at(1));
}

template <class Leaf, class Node, class Root>
void run_tree_flat(Executor& ex, std::vector<Fiber*>& roots, const std::vector<const Val*>& trees, Leaf leaf, Node node,
                   Root root_done) {
  // The child fibers: one block per call, reused across calls on this thread (sized up front so
  // the pointers into it stay valid; fibers are plain records here, no coroutine frames).
  size_t nsub = 0;
  for (const Val* t : trees) nsub += count_subtrees(*t);
  thread_local std::vector<Fiber> extra;
  extra.clear();
  extra.resize(nsub);
  size_t next_extra = 0;
  thread_local std::vector<FlatTree> F;
  F.clear();
  F.reserve(roots.size() + nsub);
  for (size_t i = 0; i < roots.size(); ++i) F.push_back(FlatTree{roots[i], trees[i], -1, 0, {-1, -1}, int(i), {}});
  // A pass of run_runnable visits, in index order, the fibers made runnable in the previous pass
  // (parents whose last child finished: lower indices than anything created since), then every
  // fiber created during this pass (appended, runnable).  No rescans of blocked fibers.
  std::vector<int> cur(roots.size()), next;
  for (size_t i = 0; i < roots.size(); ++i) cur[i] = int(i);
  auto resume = [&](size_t i) {
    Fiber& fb = *F[i].fb;
    const bool is_root = F[i].parent < 0;
    if (F[i].state == 0) {
      if (is_root) ex.stage(fb, 0);
      const Val& t = *F[i].t;
      if (t.ctor != 0) {  // Node(l, r): concurrent children, then join
        for (int k = 0; k < 2; ++k) {
          Fiber& cf = extra[next_extra++];
          cf.instance = fb.instance;
          cf.phase = fb.phase;
          cf.depth_counter = fb.depth_counter;
          F[i].kids[k] = int(F.size());
          F.push_back(FlatTree{&cf, &t.at(size_t(k)), int(i), 0, {-1, -1}, F[i].inst, {}});
        }
        fb.status = runtime::FiberStatus::kBlockedJoin;
        fb.pending_children = 2;
        F[i].state = 1;
        return;
      }
      leaf(fb, F[i].inst, t, F[i].res);
    } else {
      const FlatTree &a = F[size_t(F[i].kids[0])], &b = F[size_t(F[i].kids[1])];
      fb.depth_counter = std::max(fb.depth_counter, a.fb->depth_counter);
      fb.depth_counter = std::max(fb.depth_counter, b.fb->depth_counter);
      node(fb, F[i].inst, a.res, b.res, F[i].res);
    }
    if (is_root) root_done(fb, F[i].inst, F[i].res);
    fb.status = runtime::FiberStatus::kDone;
    fb.has_result = true;
    const int p = F[i].parent;
    if (p >= 0) {
      Fiber& pf = *F[size_t(p)].fb;
      if (--pf.pending_children == 0 && pf.status == runtime::FiberStatus::kBlockedJoin) {
        pf.status = runtime::FiberStatus::kRunnable;
        next.push_back(p);
      }
    }
  };
  while (!cur.empty()) {
    const size_t created = F.size();
    next.clear();
    for (int i : cur) resume(size_t(i));
    for (size_t i = created; i < F.size(); ++i) resume(i);
    std::sort(next.begin(), next.end());
    cur.swap(next);
  }
}

class TreeLstmProgram : public runtime::Program {
 public:
  bool has_flat() const override { return true; }
  void run_flat(Executor& ex, std::vector<Fiber*>& roots, std::vector<std::vector<Val>>& args) const override {
    std::vector<TreeLstmParams> P;
    std::vector<const Val*> trees;
    P.reserve(args.size());
    for (auto& a : args) {
      P.push_back(TreeLstmParams{a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9], a[10]});
      trees.push_back(&a[11]);
    }
    run_tree_flat(
        ex, roots, trees,
        [&](Fiber& fb, int i, const Val& t, Val* res) {  // tlstm's Leaf branch: res = (tanh(c), c)
          const TreeLstmParams& p = P[size_t(i)];
          Val xt = Executor::out(ex.emit(fb, 3, {&t.at(0), &p.x_wt, &p.x_bias}), 0);
          int n = ex.emit(fb, 1, {&p.hz, &p.hz, &p.i_wt, &xt, &p.fl_wt, &p.fr_wt, &p.u_wt, &p.cz, &p.cz});
          res[0] = Executor::out(n, 1);
          res[1] = Executor::out(n, 0);
        },
        [&](Fiber& fb, int i, const Val* l, const Val* r, Val* res) {  // tlstm's Node branch after the join
          const TreeLstmParams& p = P[size_t(i)];
          int n = ex.emit(fb, 2, {&l[0], &r[0], &p.i_wt, &p.xn, &p.fl_wt, &p.fr_wt, &p.u_wt, &l[1], &r[1]});
          res[0] = Executor::out(n, 1);
          res[1] = Executor::out(n, 0);
        },
        [&](Fiber& fb, int i, const Val* res) {  // TreeLstmProgram::run after co_await tlstm
          const TreeLstmParams& p = P[size_t(i)];
          ex.stage(fb, 1);
          fb.result = Executor::out(ex.emit(fb, 0, {&res[0], &p.c_wt, &p.cbias}), 0);
        });
  }
  Task run(Executor& ex, Fiber& fb, std::vector<Val> a) const override {
    TreeLstmParams P{a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9], a[10]};
    ex.stage(fb, 0);
    Val res = co_await tlstm(ex, fb, P, a[11]);
    ex.stage(fb, 1);
    co_return Executor::out(ex.emit(fb, 0, {&res.at(0), &P.c_wt, &P.cbias}), 0);
  }
};

// ---- mvrnn (zoo.cpp:119-143) --------------------------------------------------------------
struct MvParams {
  Val v_wt, vbias, c_wt, cbias;
};

Task mv(Executor& ex, Fiber& fb, const MvParams& P, Val t) {
  if (t.ctor == 0) co_return Val::tuple({t.at(0), t.at(1)});
  struct Sub { Executor* ex; const MvParams* P; const Val* t; };
  const Sub sl{&ex, &P, &t.at(0)}, sr{&ex, &P, &t.at(1)};
  std::vector<Call> calls;
  calls.reserve(2);
  calls.push_back([a = &sl](Fiber& f) { return mv(*a->ex, f, *a->P, *a->t); });
  calls.push_back([a = &sr](Fiber& f) { return mv(*a->ex, f, *a->P, *a->t); });
  runtime::JoinAwait join = ex.concurrent(fb, std::move(calls));
  std::vector<Val> res = co_await join;
  const Val &lv = res[0].at(0), &lm = res[0].at(1), &rv = res[1].at(0), &rm = res[1].at(1);
  // block inputs: lres.0, rres.1, rres.0, lres.1, v_wt, vbias
  int n1 = ex.emit(fb, 1, {&lv, &rm, &rv, &lm, &P.v_wt, &P.vbias});
  int n2 = ex.emit(fb, 2, {&lm, &rm});
  co_return Val::tuple({Executor::out(n1, 0), Executor::out(n2, 0)});
}

class MvRnnProgram : public runtime::Program {
 public:
  bool has_flat() const override { return true; }
  void run_flat(Executor& ex, std::vector<Fiber*>& roots, std::vector<std::vector<Val>>& args) const override {
    std::vector<MvParams> P;
    std::vector<const Val*> trees;
    P.reserve(args.size());
    for (auto& a : args) {
      P.push_back(MvParams{a[0], a[1], a[2], a[3]});
      trees.push_back(&a[4]);
    }
    run_tree_flat(
        ex, roots, trees,
        [&](Fiber&, int, const Val& t, Val* res) {  // mv's Leaf branch: (vector, matrix)
          res[0] = t.at(0);
          res[1] = t.at(1);
        },
        [&](Fiber& fb, int i, const Val* l, const Val* r, Val* res) {  // mv's Node branch
          const MvParams& p = P[size_t(i)];
          int n1 = ex.emit(fb, 1, {&l[0], &r[1], &r[0], &l[1], &p.v_wt, &p.vbias});
          int n2 = ex.emit(fb, 2, {&l[1], &r[1]});
          res[0] = Executor::out(n1, 0);
          res[1] = Executor::out(n2, 0);
        },
        [&](Fiber& fb, int i, const Val* res) {  // MvRnnProgram::run after co_await mv
          const MvParams& p = P[size_t(i)];
          ex.stage(fb, 1);
          fb.result = Executor::out(ex.emit(fb, 0, {&res[0], &p.c_wt, &p.cbias}), 0);
        });
  }
  Task run(Executor& ex, Fiber& fb, std::vector<Val> a) const override {
    MvParams P{a[0], a[1], a[2], a[3]};
    ex.stage(fb, 0);
    Val res = co_await mv(ex, fb, P, a[4]);
    ex.stage(fb, 1);
    co_return Executor::out(ex.emit(fb, 0, {&res.at(0), &P.c_wt, &P.cbias}), 0);
  }
};

// ---- nestedrnn (zoo.cpp:145-174) ----------------------------------------------------------
class NestedRnnProgram : public runtime::Program {
 public:
  Task run(Executor& ex, Fiber& fb, std::vector<Val> a) const override {
    // a: zb, z_wt, hb, h_wt, rb, r_wt, n_wt, ibias, i_wt, outer_init, xs
    ex.stage(fb, 0);
    Val h = a[9];
    const Val& xs = a[10];
    for (size_t k = 0; k < xs.size(); ++k) {
      const Val& x = xs.at(k);
      int n1 = ex.emit(fb, 1, {&x, &h, &a[1], &a[0], &a[3], &a[2], &a[5], &a[4], &a[6]});
      Val hmix = Executor::out(n1, 0);
      long n = co_await ex.scalar(fb, Executor::out(n1, 1));
      Val s = hmix;
      for (long it = n + 25; it > 0; --it) s = Executor::out(ex.emit(fb, 0, {&s, &a[8], &a[7]}), 0);  // @inner
      h = s;
    }
    co_return h;
  }
};

// ---- drnn (zoo.cpp:176-209) ---------------------------------------------------------------
struct DrnnParams {
  Val obias, o_wt, d_wt, lbias, l_wt, rbias, r_wt;
};

Task drnn_gen(Executor& ex, Fiber& fb, const DrnnParams& P, Val h, long fuel) {
  Val o = Executor::out(ex.emit(fb, 0, {&h, &P.o_wt, &P.obias}), 0);
  if (fuel <= 0) co_return Val::list({o});
  long d = co_await ex.scalar(fb, Executor::out(ex.emit(fb, 1, {&o, &P.d_wt}), 0));
  if (d == 0) co_return Val::list({o});
  Val lh = Executor::out(ex.emit(fb, 2, {&o, &P.l_wt, &P.lbias}), 0);
  Val rh = Executor::out(ex.emit(fb, 3, {&o, &P.r_wt, &P.rbias}), 0);
  // The two recursive calls are annotated concurrent(0), but in ANF each is preceded by its own
  // `fuel - 1`, so they are not a run of adjacent calls and the reference executor runs them
  // inline, one after the other (executor.cpp:522-531).
  Val lt = co_await drnn_gen(ex, fb, P, lh, fuel - 1);
  Val rt = co_await drnn_gen(ex, fb, P, rh, fuel - 1);
  std::vector<Val> out{o};
  for (auto& v : *lt.items) out.push_back(v);
  for (auto& v : *rt.items) out.push_back(v);
  co_return Val::list(std::move(out));
}

class DrnnProgram : public runtime::Program {
 public:
  Task run(Executor& ex, Fiber& fb, std::vector<Val> a) const override {
    // a: obias, o_wt, d_wt, lbias, l_wt, rbias, r_wt, root_bias, root_wt, x, fuel
    DrnnParams P{a[0], a[1], a[2], a[3], a[4], a[5], a[6]};
    ex.stage(fb, 0);
    Val h0 = Executor::out(ex.emit(fb, 4, {&a[9], &a[8], &a[7]}), 0);
    co_return co_await drnn_gen(ex, fb, P, h0, a[10].i);
  }
};

// ---- stackrnn (zoo.cpp:211-240) -----------------------------------------------------------
class StackRnnProgram : public runtime::Program {
 public:
  Task run(Executor& ex, Fiber& fb, std::vector<Val> a) const override {
    // a: hbias, s_wt, a_wt, ebias, e_wt, pbias, p_wt, rbias, r_wt, obias, o_wt, init, c_wt, cbias, toks
    ex.stage(fb, 0);
    Val h = a[11];
    const Val& toks = a[14];
    for (size_t k = 0; k < toks.size(); ++k) {
      const Val& x = toks.at(k);
      int n1 = ex.emit(fb, 1, {&x, &h, &a[1], &a[0], &a[2]});
      Val h2 = Executor::out(n1, 0);
      long act = co_await ex.scalar(fb, Executor::out(n1, 1));
      Val h0, h1;
      if (act == 0) {
        h0 = Executor::out(ex.emit(fb, 2, {&h2, &a[4], &a[3]}), 0);
        h1 = Executor::out(ex.emit(fb, 3, {&h2, &a[6], &a[5]}), 0);
      } else {
        // Ghost unit balancing the one-unit branch against the two-unit one (Fig. 5,
        // analysis.cpp:1083-1212); a scheduling-only node.
        if (ex.ghost_enabled()) ex.ghosts(fb, 1);
        h0 = Executor::out(ex.emit(fb, 4, {&h2, &a[8], &a[7]}), 0);
        h1 = h0;
      }
      h = Executor::out(ex.emit(fb, 5, {&h0, &h1, &a[10], &a[9]}), 0);
    }
    ex.stage(fb, 1);
    co_return Executor::out(ex.emit(fb, 0, {&h, &a[12], &a[13]}), 0);
  }
};

// ---- fig5 (zoo.cpp:243-259) ---------------------------------------------------------------
class Fig5Program : public StraightProgram {
 public:
  Val body(Executor& ex, Fiber& fb, std::vector<Val>& a) const override {
    // a: a_wt, abias, b_wt, bbias, x, sel
    ex.stage(fb, 0);
    Val r;
    if (a[5].i == 0) {
      // Without hoisting the branches hold 1 and 2 units: pad the short one (Fig. 5).  With
      // hoisting the common block sits at static depth 2 in both branches and no ghost is needed.
      if (ex.ghost_enabled() && !ex.hoist_enabled()) ex.ghosts(fb, 1);
      r = Executor::out(ex.emit(fb, 0, {&a[4], &a[2], &a[3]}), 0);
    } else {
      Val e = Executor::out(ex.emit(fb, 1, {&a[4], &a[0], &a[1]}), 0);
      r = Executor::out(ex.emit(fb, 0, {&e, &a[2], &a[3]}), 0);
    }
    ex.stage(fb, 1);
    return Executor::out(ex.emit(fb, 0, {&r, &a[2], &a[3]}), 0);
  }
};

}  // namespace

// =============================================================================================

std::vector<std::string> model_names() { return {"rnn", "birnn", "treelstm", "mvrnn", "nestedrnn", "drnn", "stackrnn"}; }

CompiledModel get_model(const std::string& name, int H, const ExecOptions& opts) {
  MBATCH_CHECK(H >= 1, "hidden size must be positive");
  const int C = 8, H2 = 2 * H;
  const Shape h1{1, H}, hh{H, H}, h2h{H2, H}, hc{H, C}, c1{1, C};
  ModelBuilder mb(name, H);
  auto& m = mb.m;
  m.opts = opts;
  using O = OpCode;
  if (name == "rnn") {
    mb.param("rnn_bias", 1, H); mb.param("rnn_i_wt", H, H); mb.param("rnn_h_wt", H, H); mb.param("rnn_init", 1, H);
    mb.param("c_wt", H, C); mb.param("cbias", 1, C); mb.input("inps");
    mb.sig("relu_bias_dense", {P("c_wt", H, C), P("cbias", 1, C)}, {P("p", 1, H)}, {c1}, dense_tail(hc, c1, h1, {L(O::kAdd, S(1)), L(O::kRelu)}));
    mb.sig("bias_dense", {P("i_wt", H, H), P("bias", 1, H)}, {P("inp", 1, H)}, {h1}, dense_tail(hh, h1, h1, {L(O::kAdd, S(1))}));
    mb.sig("sigmoid_add_dense", {P("h_wt", H, H)}, {P("state", 1, H), P("inp_linear", 1, H)}, {h1},
           dense_tail(hh, Shape{}, h1, {L(O::kAdd, B(1)), L(O::kSigmoid)}, {h1}));
    mb.ghost();
    mb.block(0, "main", 0, {"p", "c_wt", "cbias"}, {1, 2}, {0}, -1, 1);
    mb.block(1, "rnn", 1, {"inp", "i_wt", "bias"}, {1, 2}, {0}, 0, 1);
    mb.block(2, "rnn", 2, {"state", "h_wt", "inp_linear"}, {1}, {0, 2}, -1, 1);
    m.stage_phase = {0, 1};
    m.program = std::make_shared<RnnProgram>();
    m.nesting = {{"main", 0}, {"rnn", 1}};
  } else if (name == "birnn") {
    for (const char* d : {"f", "b"}) {
      std::string p = std::string(d) + "_rnn_";
      mb.param(p + "bias", 1, H); mb.param(p + "i_wt", H, H); mb.param(p + "h_wt", H, H); mb.param(p + "init", 1, H);
    }
    mb.input("inps_list");
    mb.sig("concat", {}, {P("ft", 1, H), P("bt", 1, H)}, {Shape{1, H2}},
           PlanBuilder({}, {h1, h1}).op(O::kConcat, {B(0), B(1)}, Shape{1, H2}).outputs({T(0)}));
    mb.sig("bias_dense", {P("i_wt", H, H), P("bias", 1, H)}, {P("inp", 1, H)}, {h1}, dense_tail(hh, h1, h1, {L(O::kAdd, S(1))}));
    mb.sig("sigmoid_add_dense", {P("h_wt", H, H)}, {P("state", 1, H), P("inp_linear", 1, H)}, {h1},
           dense_tail(hh, Shape{}, h1, {L(O::kAdd, B(1)), L(O::kSigmoid)}, {h1}));
    mb.ghost();
    mb.block(0, "main", 0, {"ft", "bt"}, {}, {0, 1}, -1, 1);
    mb.block(1, "rnn__c0", 1, {"inp", "i_wt", "bias"}, {1, 2}, {0}, 0, 1);
    mb.block(2, "rnn__c0", 2, {"state", "h_wt", "inp_linear"}, {1}, {0, 2}, -1, 1);
    mb.block(3, "rnn__c1", 1, {"inp", "i_wt", "bias"}, {1, 2}, {0}, 0, 1);
    mb.block(4, "rnn__c1", 2, {"state", "h_wt", "inp_linear"}, {1}, {0, 2}, -1, 1);
    m.stage_phase = {0, 0, 1, 2};
    m.program = std::make_shared<BirnnProgram>();
    m.nesting = {{"main", 0}, {"rnn__c0", 1}, {"rnn__c1", 1}};
  } else if (name == "treelstm") {
    mb.param("x_wt", H, H); mb.param("x_bias", 1, H); mb.param("xn", 1, H);
    mb.param("i_wt", H2, H); mb.param("fl_wt", H2, H); mb.param("fr_wt", H2, H); mb.param("u_wt", H2, H);
    mb.param("hz", 1, H); mb.param("cz", 1, H); mb.param("c_wt", H, C); mb.param("cbias", 1, C); mb.input("t");
    mb.sig("relu_bias_dense", {P("c_wt", H, C), P("cbias", 1, C)}, {P("%t0", 1, H)}, {c1}, dense_tail(hc, c1, h1, {L(O::kAdd, S(1)), L(O::kRelu)}));
    // The tcell block (zoo.cpp:84-92): concat, 4-gate fused dense, gates, c, tanh(c).
    // `x` is the ref carrying xt; `lc`/`rc` the cell-state refs; g the fused dense input refs.
    auto tcell_plan = [&](std::vector<Shape> shared, std::vector<Shape> batched, PlanRef lh, PlanRef rh,
                          std::vector<PlanRef> w, PlanRef x, PlanRef lc, PlanRef rc) {
      PlanBuilder b(std::move(shared), std::move(batched));
      b.op(O::kConcat, {lh, rh}, Shape{1, H2});
      b.fused({T(0), w[0], w[1], w[2], w[3]}, Shape{1, 4 * H});
      b.op(O::kAdd, {Tc(1, 0, H), x}, h1).chain(T(2), {L(O::kSigmoid)}, h1);          // i
      b.op(O::kAdd, {Tc(1, H, H), x}, h1).chain(T(4), {L(O::kSigmoid)}, h1);          // fl
      b.op(O::kAdd, {Tc(1, 2 * H, H), x}, h1).chain(T(6), {L(O::kSigmoid)}, h1);      // fr
      b.op(O::kAdd, {Tc(1, 3 * H, H), x}, h1).chain(T(8), {L(O::kTanh), L(O::kMul, T(3))}, h1);  // u*i
      b.op(O::kMul, {T(5), lc}, h1).op(O::kMul, {T(7), rc}, h1);
      b.chain(T(11), {L(O::kAdd, T(10)), L(O::kAdd, T(9))}, h1);  // c
      b.op(O::kTanh, {T(12)}, h1);
      return b.outputs({T(12), T(13)});
    };
    mb.sig("add_mul_sigmoid_add",
           {P("lh", 1, H), P("rh", 1, H), P("i_wt", H2, H), P("fl_wt", H2, H), P("fr_wt", H2, H), P("u_wt", H2, H), P("lc", 1, H), P("rc", 1, H)},
           {P("xt", 1, H)}, {h1, h1},
           tcell_plan({h1, h1, h2h, h2h, h2h, h2h, h1, h1}, {h1}, S(0), S(1), {S(2), S(3), S(4), S(5)}, B(0), S(6), S(7)));
    mb.sig("add_mul_sigmoid_bias",
           {P("i_wt", H2, H), P("xt", 1, H), P("fl_wt", H2, H), P("fr_wt", H2, H), P("u_wt", H2, H)},
           {P("lh", 1, H), P("rh", 1, H), P("lc", 1, H), P("rc", 1, H)}, {h1, h1},
           tcell_plan({h2h, h1, h2h, h2h, h2h}, {h1, h1, h1, h1}, B(0), B(1), {S(0), S(2), S(3), S(4)}, S(1), B(2), B(3)));
    mb.sig("bias_dense", {P("x_wt", H, H), P("x_bias", 1, H)}, {P("x", 1, H)}, {h1}, dense_tail(hh, h1, h1, {L(O::kAdd, S(1))}));
    mb.ghost();
    const std::vector<std::string> cell_in{"lh", "rh", "i_wt", "xt", "fl_wt", "fr_wt", "u_wt", "lc", "rc"};
    mb.block(0, "main", 0, {"%t0", "c_wt", "cbias"}, {1, 2}, {0}, -1, 1);
    mb.block(1, "tcell__c0", 1, cell_in, {0, 1, 2, 4, 5, 6, 7, 8}, {3}, 1, 2);
    mb.block(2, "tcell__c1", 2, cell_in, {2, 3, 4, 5, 6}, {0, 1, 7, 8}, -1, 2);
    mb.block(3, "tlstm", 3, {"x", "x_wt", "x_bias"}, {1, 2}, {0}, 0, 1);
    m.stage_phase = {0, 1};
    m.program = std::make_shared<TreeLstmProgram>();
    m.nesting = {{"main", 0}, {"tlstm", 1}, {"tcell__c0", 1}, {"tcell__c1", 1}};
  } else if (name == "mvrnn") {
    mb.param("v_wt", H2, H); mb.param("vbias", 1, H); mb.param("c_wt", H, C); mb.param("cbias", 1, C); mb.input("t");
    mb.sig("relu_bias_dense", {P("c_wt", H, C), P("cbias", 1, C)}, {P("%t0", 1, H)}, {c1}, dense_tail(hc, c1, h1, {L(O::kAdd, S(1)), L(O::kRelu)}));
    mb.sig("tanh_bias_dense_concat", {P("v_wt", H2, H), P("vbias", 1, H)},
           {P("%t6", 1, H), P("%t7", H, H), P("%t8", 1, H), P("%t9", H, H)}, {h1},
           PlanBuilder({h2h, h1}, {h1, hh, h1, hh})
               .op(O::kDense, {B(0), B(1)}, h1)
               .op(O::kDense, {B(2), B(3)}, h1)
               .op(O::kConcat, {T(0), T(1)}, Shape{1, H2})
               .op(O::kDense, {T(2), S(0)}, h1)
               .chain(T(3), {L(O::kAdd, S(1)), L(O::kTanh)}, h1)
               .outputs({T(4)}));
    mb.sig("add", {}, {P("%t13", H, H), P("%t14", H, H)}, {hh}, PlanBuilder({}, {hh, hh}).op(O::kAdd, {B(0), B(1)}, hh).outputs({T(0)}));
    mb.ghost();
    mb.block(0, "main", 0, {"%t0", "c_wt", "cbias"}, {1, 2}, {0}, -1, 1);
    mb.block(1, "mv", 1, {"%t6", "%t7", "%t8", "%t9", "v_wt", "vbias"}, {4, 5}, {0, 1, 2, 3}, -1, 1);
    mb.block(2, "mv", 2, {"%t13", "%t14"}, {}, {0, 1}, -1, 1);
    m.stage_phase = {0, 1};
    m.program = std::make_shared<MvRnnProgram>();
    m.nesting = {{"main", 0}, {"mv", 1}};
  } else if (name == "nestedrnn") {
    mb.param("zb", 1, H); mb.param("z_wt", H2, H); mb.param("hb", 1, H); mb.param("h_wt", H2, H);
    mb.param("rb", 1, H); mb.param("r_wt", H2, H); mb.param("n_wt", H, 11); mb.param("ibias", 1, H);
    mb.param("i_wt", H, H); mb.param("outer_init", 1, H); mb.input("xs");
    mb.sig("sigmoid_bias_dense", {P("i_wt", H, H), P("ibias", 1, H)}, {P("s", 1, H)}, {h1},
           dense_tail(hh, h1, h1, {L(O::kAdd, S(1)), L(O::kSigmoid)}));
    mb.sig("add_mul_sigmoid_bias",
           {P("z_wt", H2, H), P("zb", 1, H), P("h_wt", H2, H), P("hb", 1, H), P("r_wt", H2, H), P("rb", 1, H), P("n_wt", H, 11)},
           {P("x", 1, H), P("h", 1, H)}, {h1, Shape{1, 1}},
           PlanBuilder({h2h, h1, h2h, h1, h2h, h1, Shape{H, 11}}, {h1, h1})
               .op(O::kConcat, {B(0), B(1)}, Shape{1, H2})
               .fused({T(0), S(0), S(2), S(4)}, Shape{1, 3 * H})
               .op(O::kAdd, {S(1), Tc(1, 0, H)}, h1).chain(T(2), {L(O::kSigmoid)}, h1)       // z
               .op(O::kAdd, {S(3), Tc(1, H, H)}, h1).chain(T(4), {L(O::kTanh)}, h1)          // hc
               .op(O::kAdd, {S(5), Tc(1, 2 * H, H)}, h1).chain(T(6), {L(O::kSigmoid)}, h1)   // zr
               .op(O::kMul, {T(3), T(5)}, h1)
               .op(O::kMul, {T(7), B(1)}, h1)
               .chain(T(9), {L(O::kAdd, T(8))}, h1)                                          // hmix
               .op(O::kDense, {T(10), S(6)}, Shape{1, 11})
               .op(O::kArgmax, {T(11)}, Shape{1, 1})
               .outputs({T(10), T(12)}));
    mb.ghost();
    mb.block(0, "inner", 0, {"s", "i_wt", "ibias"}, {1, 2}, {0}, -1, 1);
    mb.block(1, "outer", 1, {"x", "h", "z_wt", "zb", "h_wt", "hb", "r_wt", "rb", "n_wt"}, {2, 3, 4, 5, 6, 7, 8}, {0, 1}, -1, 2);
    m.stage_phase = {0};
    m.program = std::make_shared<NestedRnnProgram>();
    m.nesting = {{"main", 0}, {"outer", 1}, {"inner", 2}};
  } else if (name == "drnn") {
    mb.param("obias", 1, H); mb.param("o_wt", H, H); mb.param("d_wt", H, 2); mb.param("lbias", 1, H);
    mb.param("l_wt", H, H); mb.param("rbias", 1, H); mb.param("r_wt", H, H); mb.param("root_bias", 1, H);
    mb.param("root_wt", H, H); mb.input("x"); mb.input("fuel");
    mb.sig("tanh_bias_dense", {P("o_wt", H, H), P("obias", 1, H)}, {P("h", 1, H)}, {h1}, dense_tail(hh, h1, h1, {L(O::kAdd, S(1)), L(O::kTanh)}));
    mb.sig("argmax_dense", {P("d_wt", H, 2)}, {P("o", 1, H)}, {Shape{1, 1}},
           PlanBuilder({Shape{H, 2}}, {h1}).op(O::kDense, {B(0), S(0)}, Shape{1, 2}).op(O::kArgmax, {T(0)}, Shape{1, 1}).outputs({T(1)}));
    mb.ghost();
    mb.block(0, "gen", 0, {"h", "o_wt", "obias"}, {1, 2}, {0}, -1, 1);
    mb.block(1, "gen", 1, {"o", "d_wt"}, {1}, {0}, -1, 1);
    mb.block(2, "gen", 0, {"o", "l_wt", "lbias"}, {1, 2}, {0}, -1, 1);
    mb.block(3, "gen", 0, {"o", "r_wt", "rbias"}, {1, 2}, {0}, -1, 1);
    mb.block(4, "main", 0, {"x", "root_wt", "root_bias"}, {1, 2}, {0}, 0, 1);
    m.stage_phase = {0};
    m.program = std::make_shared<DrnnProgram>();
    m.nesting = {{"main", 0}, {"gen", 1}};
  } else if (name == "stackrnn") {
    mb.param("hbias", 1, H); mb.param("s_wt", H2, H); mb.param("a_wt", H, 2); mb.param("ebias", 1, H);
    mb.param("e_wt", H, H); mb.param("pbias", 1, H); mb.param("p_wt", H, H); mb.param("rbias", 1, H);
    mb.param("r_wt", H, H); mb.param("obias", 1, H); mb.param("o_wt", H2, H); mb.param("init", 1, H);
    mb.param("c_wt", H, C); mb.param("cbias", 1, C); mb.input("toks");
    mb.sig("relu_bias_dense", {P("c_wt", H, C), P("cbias", 1, C)}, {P("res", 1, H)}, {c1}, dense_tail(hc, c1, h1, {L(O::kAdd, S(1)), L(O::kRelu)}));
    mb.sig("sigmoid_bias_dense_concat", {P("s_wt", H2, H), P("hbias", 1, H), P("a_wt", H, 2)}, {P("x", 1, H), P("h", 1, H)},
           {h1, Shape{1, 1}},
           PlanBuilder({h2h, h1, Shape{H, 2}}, {h1, h1})
               .op(O::kConcat, {B(0), B(1)}, Shape{1, H2})
               .op(O::kDense, {T(0), S(0)}, h1)
               .chain(T(1), {L(O::kAdd, S(1)), L(O::kSigmoid)}, h1)
               .op(O::kDense, {T(2), S(2)}, Shape{1, 2})
               .op(O::kArgmax, {T(3)}, Shape{1, 1})
               .outputs({T(2), T(4)}));
    mb.sig("tanh_bias_dense", {P("e_wt", H, H), P("ebias", 1, H)}, {P("h2", 1, H)}, {h1}, dense_tail(hh, h1, h1, {L(O::kAdd, S(1)), L(O::kTanh)}));
    mb.sig("relu_bias_dense_2", {P("p_wt", H, H), P("pbias", 1, H)}, {P("h2", 1, H)}, {h1}, dense_tail(hh, h1, h1, {L(O::kAdd, S(1)), L(O::kRelu)}));
    mb.sig("sigmoid_bias_dense_concat_2", {P("o_wt", H2, H), P("obias", 1, H)}, {P("%t20", 1, H), P("%t21", 1, H)}, {h1},
           PlanBuilder({h2h, h1}, {h1, h1})
               .op(O::kConcat, {B(0), B(1)}, Shape{1, H2})
               .op(O::kDense, {T(0), S(0)}, h1)
               .chain(T(1), {L(O::kAdd, S(1)), L(O::kSigmoid)}, h1)
               .outputs({T(2)}));
    mb.ghost();
    mb.block(0, "main", 0, {"res", "c_wt", "cbias"}, {1, 2}, {0}, -1, 1);
    mb.block(1, "srnn", 1, {"x", "h", "s_wt", "hbias", "a_wt"}, {2, 3, 4}, {0, 1}, -1, 2);
    mb.block(2, "srnn", 2, {"h2", "e_wt", "ebias"}, {1, 2}, {0}, -1, 1);
    mb.block(3, "srnn", 3, {"h2", "p_wt", "pbias"}, {1, 2}, {0}, -1, 1);
    mb.block(4, "srnn", 2, {"h2", "r_wt", "rbias"}, {1, 2}, {0}, -1, 1);
    mb.block(5, "srnn", 4, {"%t20", "%t21", "o_wt", "obias"}, {2, 3}, {0, 1}, -1, 1);
    m.stage_phase = {0, 1};
    m.program = std::make_shared<StackRnnProgram>();
    m.nesting = {{"main", 0}, {"srnn", 1}};
  } else if (name == "fig5") {
    mb.param("a_wt", H, H); mb.param("abias", 1, H); mb.param("b_wt", H, H); mb.param("bbias", 1, H);
    mb.input("x"); mb.input("sel");
    mb.sig("sigmoid_bias_dense", {P("b_wt", H, H), P("bbias", 1, H)}, {P("v", 1, H)}, {h1}, dense_tail(hh, h1, h1, {L(O::kAdd, S(1)), L(O::kSigmoid)}));
    mb.sig("relu_bias_dense", {P("a_wt", H, H), P("abias", 1, H)}, {P("v", 1, H)}, {h1}, dense_tail(hh, h1, h1, {L(O::kAdd, S(1)), L(O::kRelu)}));
    mb.ghost();
    mb.block(0, "common", 0, {"v", "b_wt", "bbias"}, {1, 2}, {0}, 2, 1);
    mb.block(1, "extra", 1, {"v", "a_wt", "abias"}, {1, 2}, {0}, 0, 1);
    m.stage_phase = {0, 1};
    m.program = std::make_shared<Fig5Program>();
    m.nesting = {{"main", 0}, {"common", 0}, {"extra", 0}};
  } else {
    throw Error("unknown model '" + name + "'");
  }
  (void)h2h;
  return m;
}

// ---- seeded synthetic inputs (zoo.cpp:281-401) --------------------------------------------

namespace {

HostValue random_tensor(std::mt19937& rng, Shape s) {
  std::uniform_real_distribution<float> dist(-0.5f, 0.5f);
  std::vector<float> v(s.size());
  for (auto& x : v) x = dist(rng);
  return HostValue::tensor(s, std::move(v));
}

HostValue random_tree(std::mt19937& rng, int leaves, const std::function<HostValue(std::mt19937&)>& leaf_fn) {
  if (leaves == 1) return leaf_fn(rng);
  std::uniform_int_distribution<int> split(1, leaves - 1);
  int left = split(rng);
  HostValue l = random_tree(rng, left, leaf_fn);
  HostValue r = random_tree(rng, leaves - left, leaf_fn);
  return HostValue::adt("Node", {std::move(l), std::move(r)});
}

}  // namespace

ParamEnv make_params(const CompiledModel& model, unsigned seed) {
  std::mt19937 rng(seed * 7919u + 17u);
  ParamEnv env;
  for (const auto& d : model.params)
    if (!d.is_instance_input) env[d.name] = random_tensor(rng, d.shape);
  return env;
}

std::vector<InstanceInput> make_inputs(const CompiledModel& model, unsigned seed, int batch) {
  const int H = model.hidden;
  std::vector<InstanceInput> out;
  for (int i = 0; i < batch; ++i) {
    std::mt19937 rng(seed * 104729u + 31u * i + 7u);
    InstanceInput inst;
    for (const auto& d : model.params) {
      if (!d.is_instance_input) continue;
      if (d.name == "inps" || d.name == "inps_list" || d.name == "xs" || d.name == "toks") {
        std::uniform_int_distribution<int> len_dist(4, 12);
        int len = len_dist(rng);
        std::vector<HostValue> items;
        for (int k = 0; k < len; ++k) items.push_back(random_tensor(rng, Shape{1, H}));
        inst[d.name] = HostValue::list(std::move(items));
      } else if (d.name == "t") {
        std::uniform_int_distribution<int> leaves_dist(4, 16);
        int leaves = leaves_dist(rng);
        const bool mv = model.name == "mvrnn";
        auto leaf_fn = [H, mv](std::mt19937& r) {
          std::vector<HostValue> f;
          f.push_back(random_tensor(r, Shape{1, H}));
          if (mv) f.push_back(random_tensor(r, Shape{H, H}));
          return HostValue::adt("Leaf", std::move(f));
        };
        inst[d.name] = random_tree(rng, leaves, leaf_fn);
      } else if (d.name == "x") {
        inst[d.name] = random_tensor(rng, Shape{1, H});
      } else if (d.name == "fuel") {
        std::uniform_int_distribution<int> fd(3, 4);
        inst[d.name] = HostValue::scalar(fd(rng));
      } else if (d.name == "sel") {
        inst[d.name] = HostValue::scalar(i % 2);
      } else {
        std::uniform_int_distribution<int> dd(0, 7);
        inst[d.name] = HostValue::scalar(dd(rng));
      }
    }
    out.push_back(std::move(inst));
  }
  return out;
}

}  // namespace zoo

namespace runtime {
std::shared_ptr<const Program> make_program(const std::string& name, int hidden) {
  return zoo::get_model(name, hidden).program;
}
}  // namespace runtime
}  // namespace mbatch
