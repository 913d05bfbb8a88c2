// exec.h — internals of the lazy batching executor shared by runtime.cpp (the executor) and
// zoo.cpp (the AOT-lowered model programs that run on its fibers).
//
// Semantics follow the reference executor (proj/src/executor.cpp):
//   * one fiber per instance, round-robin resumption in fiber-index order (:334-345),
//   * a static block emits one DFG node; inline depth = static hoist depth, or
//     ++depth_counter, floored by pending same-phase producers (:368-427),
//   * concurrent calls fork child fibers that copy the counter and join at the max (:522-556),
//   * @map elements share the start depth (:636-668), ghosts (:429-443), phases (:464-474),
//   * scalar() suspends the fiber until a flush materialises the value (:124-131, :772-778),
//   * when every live fiber is blocked the pending DFG is flushed (:183-208).
#pragma once

#include <coroutine>
#include <exception>
#include <functional>
#include <cstring>
#include <memory>
#include <vector>

#include "mbatch/runtime.hpp"

namespace mbatch {
namespace runtime {

// Per-thread size-class free lists (runtime.cpp) for the small objects the fibers churn through:
// coroutine frames, fibers, the shared item lists of tuple / list values.
void* frame_alloc(size_t bytes);
void frame_free(void* p, size_t bytes) noexcept;

template <class T>
struct PoolAlloc {
  using value_type = T;
  PoolAlloc() = default;
  template <class U>
  PoolAlloc(const PoolAlloc<U>&) {}
  T* allocate(size_t n) { return static_cast<T*>(frame_alloc(n * sizeof(T))); }
  void deallocate(T* p, size_t n) noexcept { frame_free(p, n * sizeof(T)); }
  template <class U>
  bool operator==(const PoolAlloc<U>&) const { return true; }
  template <class U>
  bool operator!=(const PoolAlloc<U>&) const { return false; }
};

struct Val {
  enum Kind : uint8_t { kTensor, kInt, kList, kTuple, kAdt, kFloat };  // kFloat: double bits in i
  Kind kind = kInt;
  int ctor = 0;  // kAdt: 0 Leaf, 1 Node
  long i = 0;
  TensorRef t;
  std::shared_ptr<const std::vector<Val>> items;

  static Val tensor(TensorRef r) { Val v; v.kind = kTensor; v.t = r; return v; }
  static Val integer(long x) { Val v; v.kind = kInt; v.i = x; return v; }
  static Val real(double x) { Val v; v.kind = kFloat; std::memcpy(&v.i, &x, sizeof x); return v; }
  double real_value() const { double x; std::memcpy(&x, &i, sizeof x); return x; }
  static Val seq(Kind k, std::vector<Val> it, int ctor = 0) {
    Val v;
    v.kind = k;
    v.ctor = ctor;
    v.items = std::allocate_shared<const std::vector<Val>>(PoolAlloc<std::vector<Val>>(), std::move(it));
    return v;
  }
  static Val list(std::vector<Val> it) { return seq(kList, std::move(it)); }
  static Val tuple(std::vector<Val> it) { return seq(kTuple, std::move(it)); }
  const Val& at(size_t k) const { return (*items)[k]; }
  size_t size() const { return items ? items->size() : 0; }
};

// Coroutine frames of the zoo programs are allocated per call (one per block-calling function,
// one per forked child fiber): the per-thread free lists make them ~free.
struct Task {
  struct promise_type {
    static void* operator new(size_t n) { return frame_alloc(n); }
    static void operator delete(void* p, size_t n) noexcept { frame_free(p, n); }
    Val value;
    std::exception_ptr exc;
    std::coroutine_handle<> continuation;
    Task get_return_object() { return Task{std::coroutine_handle<promise_type>::from_promise(*this)}; }
    std::suspend_always initial_suspend() noexcept { return {}; }
    struct FinalAwaiter {
      bool await_ready() noexcept { return false; }
      std::coroutine_handle<> await_suspend(std::coroutine_handle<promise_type> h) noexcept {
        auto c = h.promise().continuation;
        return c ? c : std::noop_coroutine();
      }
      void await_resume() noexcept {}
    };
    FinalAwaiter final_suspend() noexcept { return {}; }
    void return_value(Val v) { value = std::move(v); }
    void unhandled_exception() { exc = std::current_exception(); }
  };
  std::coroutine_handle<promise_type> h;
  Task() = default;
  explicit Task(std::coroutine_handle<promise_type> handle) : h(handle) {}
  Task(Task&& o) noexcept : h(o.h) { o.h = nullptr; }
  Task& operator=(Task&& o) noexcept {
    if (h) h.destroy();
    h = o.h;
    o.h = nullptr;
    return *this;
  }
  Task(const Task&) = delete;
  ~Task() {
    if (h) h.destroy();
  }
  bool await_ready() { return false; }
  std::coroutine_handle<> await_suspend(std::coroutine_handle<> parent) {
    h.promise().continuation = parent;
    return h;
  }
  Val await_resume() {
    if (h.promise().exc) std::rethrow_exception(h.promise().exc);
    return std::move(h.promise().value);
  }
};

enum class FiberStatus { kRunnable, kBlockedValue, kBlockedJoin, kDone };

struct Fiber {
  static void* operator new(size_t n) { return frame_alloc(n); }
  static void operator delete(void* p, size_t n) noexcept { frame_free(p, n); }
  int id = -1;
  int instance = -1;
  int parent = -1;
  FiberStatus status = FiberStatus::kRunnable;
  Task root;
  std::coroutine_handle<> resume_point;
  TensorRef wait_ref;
  long wait_value = 0;
  bool wait_value_ready = false;
  int pending_children = 0;
  std::vector<int> children;
  Val result;
  bool has_result = false;
  int phase = 0;
  int depth_counter = 0;
  int last_node = -1;
  int pending_ghost = -1;
};

class Executor;

struct ScalarAwait {
  Executor* ex;
  Fiber* fb;
  TensorRef ref;
  bool await_ready();
  void await_suspend(std::coroutine_handle<> h);
  long await_resume();
};

struct JoinAwait {
  Executor* ex;
  Fiber* fb;
  bool await_ready() { return fb->children.empty(); }
  void await_suspend(std::coroutine_handle<> h);
  std::vector<Val> await_resume();
};

using Call = std::function<Task(Fiber&)>;

class Program {
 public:
  virtual ~Program() = default;
  // Body of @main for one instance; `args` are main's parameters in module order.
  virtual Task run(Executor& ex, Fiber& fb, std::vector<Val> args) const = 0;
  // Programs without tensor-dependent control flow (no scalar awaits) can build the whole DFG
  // without coroutines: run_flat makes the same emits, in the same order, from the same fiber
  // states (phase, depth counter, join maxima) the fiber scheduler (run_runnable) would produce,
  // and leaves each root fiber done with its result.  tests/test_flat_builder.py checks node
  // tables and traces against the coroutine path.
  virtual bool has_flat() const { return false; }
  virtual void run_flat(Executor& ex, std::vector<Fiber*>& roots, std::vector<std::vector<Val>>& args) const {
    (void)ex, (void)roots, (void)args;
  }
};

class Executor {
 public:
  // -- program-facing API ------------------------------------------------------------------
  // Emits the DFG node of static block `blk` (inputs in the block's input order) and returns
  // its node id (executor.cpp:368-427).
  int emit(Fiber& fb, int blk, std::initializer_list<const Val*> inputs);
  static Val out(int node, int k) { return Val::tensor(TensorRef{node, k, {}}); }
  // Top-level stage boundary of @main (executor.cpp:464-474).
  void stage(Fiber& fb, int stage);
  void ghosts(Fiber& fb, int count);  // executor.cpp:429-443
  ScalarAwait scalar(Fiber& fb, const Val& t) { return ScalarAwait{this, &fb, t.t}; }
  // Compile-time options the lowered program depends on (ghost insertion, hoisting).
  bool ghost_enabled() const;
  bool hoist_enabled() const;
  // A concurrent group of calls (executor.cpp:522-556).
  JoinAwait concurrent(Fiber& fb, std::vector<Call> calls);

  // -- runtime side -----------------------------------------------------------------------
  Executor(Session& s, const std::vector<InstanceInput>& inputs, const ExecOptions& opts);
  // Inputs (and outputs, into *out) in the flat hostval encoding.
  Executor(Session& s, const EncodedValues& inputs, const ExecOptions& opts, EncodedOutputs* out);
  ~Executor();
  EvalResult run();

  bool is_materialized(const TensorRef& r) const { return r.node < 0 || nodes_[r.node].executed; }
  long read_scalar_now(const TensorRef& r);
  std::vector<std::unique_ptr<Fiber>>& fibers() { return fibers_; }

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
  std::vector<DFGNode> nodes_;
  std::vector<std::unique_ptr<Fiber>> fibers_;
  friend struct Impl;
};

// Model programs (zoo.cpp).
std::shared_ptr<const Program> make_program(const std::string& name, int hidden);

}  // namespace runtime
}  // namespace mbatch
