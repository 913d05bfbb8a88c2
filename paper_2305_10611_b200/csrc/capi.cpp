#include <climits>
// capi.cpp — the C ABI (include/mbx.h).  Every entry point catches mbatch::Error (and any other
// exception) and turns it into a nonzero status plus mbx_last_error(ctx), so the boundary never
// throws; the C++ surface (include/mbatch/*.hpp) rethrows the same text.
#include <atomic>
#include <cstdlib>
#include <array>
#include <cstring>
#include <malloc.h>
#include <memory>

#include "ctx.h"
#include "exec.h"
#include "mbatch/zoo.hpp"
#include "tc.h"

namespace mbx {
extern std::atomic<int64_t> g_launches;
void arena_init(mbx_ctx* c);
void arena_release(mbx_ctx* c);
}  // namespace mbx

using mbatch::Error;
using mbatch::runtime::HostValue;

namespace {

thread_local std::string g_err;  // errors before a context exists

template <class F>
int guarded(mbx_ctx* c, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    else g_err = e.what();
    return 1;
  } catch (...) {
    if (c) c->err = "unknown error";
    else g_err = "unknown error";
    return 1;
  }
}

// Scalars: kind 1 = int32, kind 6 = int64 (lo, hi), kind 5 = float64 (lo, hi bits).  ADT
// constructors: 0 Leaf, 1 Node, -1 = named (length, one token per byte).
void push64(std::vector<int32_t>& t, uint64_t bits) {
  t.push_back(int32_t(uint32_t(bits & 0xffffffffu)));
  t.push_back(int32_t(uint32_t(bits >> 32)));
}
uint64_t read64(const int32_t* t, int64_t nt, int64_t& ti) {
  MBATCH_CHECK(ti + 2 <= nt, "hostval encoding truncated");
  const uint64_t v = uint64_t(uint32_t(t[ti])) | (uint64_t(uint32_t(t[ti + 1])) << 32);
  ti += 2;
  return v;
}

void encode(const HostValue& v, std::vector<int32_t>& t, std::vector<float>& d) {
  switch (v.kind) {
    case HostValue::Kind::kTensor:
      t.push_back(0); t.push_back(v.shape.rows); t.push_back(v.shape.cols);
      d.insert(d.end(), v.data.begin(), v.data.end());
      return;
    case HostValue::Kind::kInt:
      if (v.ival >= INT32_MIN && v.ival <= INT32_MAX) {
        t.push_back(1);
        t.push_back(int32_t(v.ival));
      } else {
        t.push_back(6);
        push64(t, uint64_t(int64_t(v.ival)));
      }
      return;
    case HostValue::Kind::kFloat: {
      uint64_t bits;
      std::memcpy(&bits, &v.fval, sizeof bits);
      t.push_back(5);
      push64(t, bits);
      return;
    }
    case HostValue::Kind::kList: t.push_back(2); break;
    case HostValue::Kind::kTuple: t.push_back(3); break;
    case HostValue::Kind::kAdt:
      t.push_back(4);
      if (v.ctor == "Leaf" || v.ctor == "Node") {
        t.push_back(v.ctor == "Node" ? 1 : 0);
      } else {
        t.push_back(-1);
        t.push_back(int32_t(v.ctor.size()));
        for (unsigned char ch : v.ctor) t.push_back(int32_t(ch));
      }
      break;
  }
  t.push_back(int32_t(v.items.size()));
  for (auto& it : v.items) encode(it, t, d);
}

HostValue decode(const int32_t* t, int64_t nt, int64_t& ti, const float* d, int64_t nd, int64_t& di) {
  MBATCH_CHECK(ti < nt, "hostval encoding truncated");
  int kind = t[ti++];
  switch (kind) {
    case 0: {
      MBATCH_CHECK(ti + 2 <= nt, "hostval encoding truncated");
      int r = t[ti++], c = t[ti++];
      int64_t n = int64_t(r) * c;
      MBATCH_CHECK(r >= 0 && c >= 0 && di + n <= nd, "hostval data truncated");
      HostValue v;
      v.kind = HostValue::Kind::kTensor;
      v.shape = {r, c};
      v.ext = d + di;  // borrowed for the call
      di += n;
      return v;
    }
    case 1: MBATCH_CHECK(ti < nt, "hostval encoding truncated"); return HostValue::scalar(t[ti++]);
    case 6: return HostValue::scalar(long(int64_t(read64(t, nt, ti))));
    case 5: {
      const uint64_t bits = read64(t, nt, ti);
      HostValue v;
      v.kind = HostValue::Kind::kFloat;
      std::memcpy(&v.fval, &bits, sizeof bits);
      return v;
    }
    case 2: case 3: case 4: {
      std::string ctor = "Leaf";
      if (kind == 4) {
        MBATCH_CHECK(ti < nt, "hostval encoding truncated");
        const int id = t[ti++];
        if (id >= 0) {
          ctor = id ? "Node" : "Leaf";
        } else {
          MBATCH_CHECK(ti < nt, "hostval encoding truncated");
          const int len = t[ti++];
          MBATCH_CHECK(len >= 0 && ti + len <= nt, "hostval encoding truncated");
          ctor.clear();
          for (int k = 0; k < len; ++k) ctor.push_back(char(t[ti++]));
        }
      }
      MBATCH_CHECK(ti < nt, "hostval encoding truncated");
      int n = t[ti++];
      std::vector<HostValue> items;
      for (int k = 0; k < n; ++k) items.push_back(decode(t, nt, ti, d, nd, di));
      if (kind == 2) return HostValue::list(std::move(items));
      if (kind == 3) return HostValue::tuple(std::move(items));
      return HostValue::adt(ctor, std::move(items));
    }
  }
  throw Error("hostval encoding: bad kind " + std::to_string(kind));
}

}  // namespace

struct mbx_model {
  mbx_ctx* ctx = nullptr;
  mbatch::runtime::CompiledModel cm;
  std::unique_ptr<mbatch::runtime::Session> session;
  std::vector<std::string> param_names;
};

struct mbx_result {
  mbatch::runtime::EvalResult r;
  std::vector<int32_t> out_tok;
  std::vector<float> out_data;
};

extern "C" {

const char* mbx_version(void) { return "mbx 0.1 (sm_100a)"; }
int64_t mbx_kernel_launch_count(void) { return mbx::g_launches.load(); }

int mbx_ctx_create(int device, int precision, mbx_ctx** out) {
  *out = nullptr;
  // The runtime builds and frees a few hundred KB of DFG state per mini-batch on every worker
  // thread: keep those blocks in the malloc arenas (no mmap/munmap or trim syscalls, which
  // serialise in the kernel across threads).  Process-wide, set once.
  static const bool tuned = [] {
    if (std::getenv("MBX_NO_MALLOPT")) return false;
    mallopt(M_MMAP_THRESHOLD, 64 << 20);
    mallopt(M_TRIM_THRESHOLD, 512 << 20);
    return true;
  }();
  (void)tuned;
  auto c = std::make_unique<mbx_ctx>();
  c->device = device;
  c->dry = device < 0;
  c->precision = precision;
  // MBX_SM_BUDGET=74: plan persistent launches for half the device, as pool contexts do
  // (measurements of the pool's configurations on one context).
  if (const char* e = std::getenv("MBX_SM_BUDGET")) c->sm_budget = std::max(16, std::min(148, std::atoi(e)));
  int rc = guarded(nullptr, [&] {
    MBATCH_CHECK(precision >= MBX_PREC_FP32 && precision <= MBX_PREC_BF16X6, "unknown precision");
    if (!c->dry) {
      mbx::cuda_check(cudaSetDevice(device), "cudaSetDevice");
      mbx::cuda_check(cudaFree(nullptr), "context init");
      mbx::cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
      mbx::cuda_check(cudaEventCreateWithFlags(&c->ev_sync, cudaEventDisableTiming), "event");
      mbx::cuda_check(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "copy stream");
      mbx::cuda_check(cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming), "event");
      mbx::arena_init(c.get());
    }
    mbx::meta_reserve(c.get(), size_t(8) << 20);
  });
  if (rc) return rc;
  *out = c.release();
  return 0;
}

void mbx_ctx_destroy(mbx_ctx* c) {
  if (!c) return;
  if (!c->dry) {
    cudaStreamSynchronize(c->stream);
    if (c->stream2) cudaStreamSynchronize(c->stream2);
    mbx::persistent_lane_forget(c);
    if (c->ev_persist) cudaEventDestroy(c->ev_persist);
    for (auto& pe : c->plans) {
      if (pe.dplan) cudaFree(pe.dplan);
      if (pe.prefix_scratch) cudaFree(pe.prefix_scratch);
      if (pe.mv_wt) cudaFree(pe.mv_wt);
      mbx::tc_release(pe);
    }
    if (c->meta.host) cudaFreeHost(c->meta.host);
    if (c->meta.dev) cudaFree(c->meta.dev);
    if (c->d2h_host) cudaFreeHost(c->d2h_host);
    if (c->d2h_dev) cudaFree(c->d2h_dev);
    if (c->in_host) cudaFreeHost(c->in_host);
    if (c->tc_part) cudaFree(c->tc_part);
    if (c->img_buf) cudaFree(c->img_buf);
    try { mbx::arena_release(c); } catch (...) {}
    if (c->ev_sync) cudaEventDestroy(c->ev_sync);
    if (c->copy_stream) {
      cudaStreamSynchronize(c->copy_stream);
      cudaStreamDestroy(c->copy_stream);
    }
    if (c->ev_copy) cudaEventDestroy(c->ev_copy);
    if (c->in_dev) cudaFree(c->in_dev);
    if (c->scat_host) cudaFreeHost(c->scat_host);
    if (c->scat_dev) cudaFree(c->scat_dev);
    if (c->stream2) {
      cudaStreamSynchronize(c->stream2);
      cudaStreamDestroy(c->stream2);
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    if (c->owns_stream) cudaStreamDestroy(c->stream);
  } else {
    std::free(c->meta.host);
    std::free(c->in_host);
  }
  delete c;
}

const char* mbx_last_error(const mbx_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }
void mbx_pool_set_error(const char* msg) { g_err = msg ? msg : ""; }

int mbx_ctx_set_precision(mbx_ctx* c, int precision) {
  return guarded(c, [&] {
    mbx::settle(c);
    MBATCH_CHECK(precision >= MBX_PREC_FP32 && precision <= MBX_PREC_BF16X6, "unknown precision");
    c->precision = precision;
  });
}

int mbx_sync(mbx_ctx* c) {
  return guarded(c, [&] {
    mbx::settle(c);
    if (!c->dry) mbx::cuda_check(cudaStreamSynchronize(c->stream), "sync");
  });
}

void* mbx_ctx_stream(mbx_ctx* c) { return c ? reinterpret_cast<void*>(c->stream) : nullptr; }

int mbx_arena_alloc(mbx_ctx* c, int rows, int cols, int64_t* offset) {
  return guarded(c, [&] {
    MBATCH_CHECK(rows >= 0 && cols >= 0, "negative shape");
    *offset = mbx::arena_alloc(c, int64_t(rows) * cols);
  });
}

int64_t mbx_arena_used(const mbx_ctx* c) { return c->used; }

int mbx_arena_upload(mbx_ctx* c, int64_t off, const float* src, int64_t n) {
  return guarded(c, [&] {
    mbx::settle(c);
    mbx::arena_check(c, off, n);
    ++c->upload_epoch;
    if (c->dry || n == 0) return;
    mbx::cuda_check(cudaMemcpyAsync(mbx::arena_ptr(c) + off, src, size_t(n) * 4, cudaMemcpyHostToDevice, c->stream), "upload");
    mbx::cuda_check(cudaStreamSynchronize(c->stream), "upload sync");
  });
}

int mbx_arena_download(mbx_ctx* c, int64_t off, float* dst, int64_t n) {
  return guarded(c, [&] {
    mbx::settle(c);
    mbx::arena_check(c, off, n);
    if (c->dry) {
      std::memset(dst, 0, size_t(n) * 4);
      return;
    }
    mbx::meta_commit(c);
    mbx::cuda_check(cudaMemcpyAsync(dst, mbx::arena_ptr(c) + off, size_t(n) * 4, cudaMemcpyDeviceToHost, c->stream), "download");
    mbx::cuda_check(cudaStreamSynchronize(c->stream), "download sync");
  });
}

int mbx_arena_device_ptr(mbx_ctx* c, int64_t off, int64_t n, float** out) {
  return guarded(c, [&] {
    mbx::arena_check(c, off, n);
    *out = c->dry ? nullptr : mbx::arena_ptr(c) + off;
  });
}

int mbx_arena_rewind(mbx_ctx* c, int64_t used) {
  return guarded(c, [&] {
    mbx::settle(c);
    MBATCH_CHECK(used >= 0 && used <= c->used, "rewind past the arena end");
    c->used = used;
    c->persist_end = std::min(c->persist_end, used);  // memory above may be reused now
  });
}

int mbx_plan_register(mbx_ctx* c, const int32_t* enc, int64_t n, int* plan_id) {
  return guarded(c, [&] { *plan_id = mbx::register_plan(c, mbatch::backend::decode_plan(enc, n)); });
}

int mbx_exec_batched(mbx_ctx* c, int plan_id, int b, const int64_t* shared_off, const int64_t* batched_off,
                     int gather_mode, int64_t* out_off, int64_t* gather_bytes) {
  return guarded(c, [&] {
    MBATCH_CHECK(b > 0, "exec_batched: empty batch");
    MBATCH_CHECK(plan_id >= 0 && size_t(plan_id) < c->plans.size(), "exec_batched: unknown plan");
    const auto& pe = c->plans.at(plan_id);
    const size_t ns = pe.plan.shared_shapes.size();
    for (int i = 1; i < b; ++i)
      for (size_t s = 0; s < ns; ++s)
        MBATCH_CHECK(shared_off[size_t(i) * ns + s] == shared_off[s],
                     "shared-param handle mismatch across instances (analysis bug)");
    size_t bytes = 8 * (pe.plan.shared_shapes.size() + size_t(b) * pe.plan.batched_shapes.size() * 2 + pe.plan.outputs.size()) + 512;
    if (c->flush_active) {
      // Queued: its offset tables stay staged until mbx_flush_end plans the whole sequence (level
      // tables and operand-image destinations are staged then, so keep room for them too).
      bytes += 64 /* one level-table entry */ + 16 * size_t(b) + 64;
      if (c->meta.cursor + bytes > c->meta.cap) mbx::issue_pending(c);  // the ring may recycle now
      mbx::meta_reserve(c, bytes);
      c->pending.push_back(
          mbx::prepare_batch(c, plan_id, b, shared_off, batched_off, gather_mode, out_off, gather_bytes));
      return;
    }
    mbx::meta_reserve(c, bytes);
    mbx::BatchLaunch L = mbx::prepare_batch(c, plan_id, b, shared_off, batched_off, gather_mode, out_off, gather_bytes);
    mbx::meta_commit(c);
    mbx::issue_batch(c, L);
  });
}

int mbx_flush_begin(mbx_ctx* c) {
  return guarded(c, [&] {
    mbx::settle(c);
    c->flush_active = true;
  });
}

int mbx_flush_end(mbx_ctx* c) {
  return guarded(c, [&] {
    c->flush_active = false;
    mbx::settle(c);
  });
}

int mbx_read_ints(mbx_ctx* c, const int64_t* offs, int n, int64_t* out) {
  return guarded(c, [&] {
    MBATCH_CHECK(n >= 0, "read_ints: negative count");
    for (int k = 0; k < n; ++k) mbx::arena_check(c, offs[k], 1);
    mbx::settle(c);
    if (n == 0) return;
    if (c->dry) {
      for (int k = 0; k < n; ++k) out[k] = 0;
      return;
    }
    // One pack kernel + one D2H for every value (executor.cpp:235-238 reads them one by one).
    std::vector<int64_t> ranges;
    ranges.reserve(size_t(n) * 3);
    for (int k = 0; k < n; ++k) {
      ranges.push_back(offs[k]);
      ranges.push_back(1);
      ranges.push_back(k);
    }
    mbx::meta_reserve(c, ranges.size() * 8);
    const size_t meta = mbx::meta_stage(c, ranges.data(), ranges.size() * 8);
    mbx::meta_commit(c);
    mbx::ensure_d2h(c, size_t(n));
    mbx::cuda_check(mbx::launch_pack_ranges(mbx::arena_ptr(c), mbx::meta_dev<int64_t>(c, meta), n, c->d2h_dev, c->stream),
                    "read_ints pack");
    ++c->launches;
    ++mbx::g_launches;
    mbx::cuda_check(cudaMemcpyAsync(c->d2h_host, c->d2h_dev, size_t(n) * 4, cudaMemcpyDeviceToHost, c->stream),
                    "read_ints D2H");
    mbx::cuda_check(cudaStreamSynchronize(c->stream), "read_ints sync");
    for (int k = 0; k < n; ++k) out[k] = static_cast<long>(c->d2h_host[k]);  // read_scalar_int
  });
}

int mbx_exec_primop(mbx_ctx* c, int op, int nin, const int64_t* in_off, const int* in_rows, const int* in_cols,
                    int64_t out_off, int out_rows, int out_cols, float fill) {
  using namespace mbatch::backend;
  return guarded(c, [&] {
    mbx::settle(c);
    MBATCH_CHECK(op >= 0 && op <= 8, "unknown op");
    OpCode o = OpCode(op);
    std::vector<Shape> shapes;
    for (int i = 0; i < nin; ++i) shapes.push_back(Shape{in_rows[i], in_cols[i]});
    const Shape out{out_rows, out_cols};
    if (o != OpCode::kFill) {
      Shape expect = infer_shape(o, shapes);
      MBATCH_CHECK(expect == out, std::string(op_name(o)) + ": output shape mismatch");
    }
    for (int i = 0; i < nin; ++i) mbx::arena_check(c, in_off[i], shapes[i].size());
    mbx::arena_check(c, out_off, out.size());
    ++c->upload_epoch;
    if (c->dry) return;
    if (o == OpCode::kFill) {
      mbx::cuda_check(mbx::launch_fill(mbx::arena_ptr(c), out_off, out.size(), fill, c->stream), "fill");
      c->write_launch = ++c->launches;
      ++mbx::g_launches;
      return;
    }
    const int64_t b_off = nin > 1 ? in_off[1] : in_off[0];
    const int br = nin > 1 ? in_rows[1] : 0, bc = nin > 1 ? in_cols[1] : 0;
    mbx::meta_commit(c);
    mbx::cuda_check(mbx::launch_primop(mbx::arena_ptr(c), op, in_off[0], in_rows[0], in_cols[0], b_off, br, bc, out_off,
                                       out_rows, out_cols, c->stream),
                    "primop");
    c->write_launch = ++c->launches;
    ++mbx::g_launches;
  });
}

// ---- models ------------------------------------------------------------------------------

int mbx_model_create(mbx_ctx* c, const char* name, int hidden, mbx_model** out) {
  *out = nullptr;
  auto m = std::make_unique<mbx_model>();
  int rc = guarded(c, [&] {
    m->ctx = c;
    m->cm = mbatch::zoo::get_model(name, hidden);
    m->session = std::make_unique<mbatch::runtime::Session>(m->cm, c);
    for (auto& d : m->cm.params)
      if (!d.is_instance_input) m->param_names.push_back(d.name);
  });
  if (rc) return rc;
  *out = m.release();
  return 0;
}

void mbx_model_destroy(mbx_model* m) { delete m; }

int mbx_model_make_params(mbx_model* m, unsigned seed) {
  return guarded(m->ctx, [&] { m->session->set_params(mbatch::zoo::make_params(m->cm, seed)); });
}

int mbx_model_set_param(mbx_model* m, const char* name, const float* data, int64_t n) {
  return guarded(m->ctx, [&] {
    auto it = m->session->param_handles().find(name);
    MBATCH_CHECK(it != m->session->param_handles().end(), std::string("unknown model parameter ") + name);
    MBATCH_CHECK(n == it->second.size(), std::string("parameter ") + name + " has the wrong size");
    if (mbx_arena_upload(m->ctx, it->second.offset, data, n) != 0) throw Error(m->ctx->err);
  });
}

int mbx_model_num_params(const mbx_model* m) { return int(m->param_names.size()); }
const char* mbx_model_param_name(const mbx_model* m, int i) { return m->param_names.at(size_t(i)).c_str(); }

int mbx_model_make_inputs(mbx_model* m, unsigned seed, int batch, int32_t* toks, int64_t* ntok, float* data, int64_t* ndata) {
  return guarded(m->ctx, [&] {
    auto inputs = mbatch::zoo::make_inputs(m->cm, seed, batch);
    std::vector<int32_t> t;
    std::vector<float> d;
    for (auto& inst : inputs)
      for (auto& decl : m->cm.params)
        if (decl.is_instance_input) encode(inst.at(decl.name), t, d);
    if (toks) {
      MBATCH_CHECK(*ntok >= int64_t(t.size()) && *ndata >= int64_t(d.size()), "buffers too small");
      std::memcpy(toks, t.data(), t.size() * 4);
      std::memcpy(data, d.data(), d.size() * 4);
    }
    *ntok = int64_t(t.size());
    *ndata = int64_t(d.size());
  });
}

int mbx_model_num_sigs(const mbx_model* m) { return int(m->cm.kernels.signatures.size()); }
const char* mbx_model_sig_name(const mbx_model* m, int sig) { return m->cm.kernels.signatures.at(size_t(sig)).name.c_str(); }

int mbx_model_plan_encoding(const mbx_model* m, int sig, int32_t* enc, int64_t* n) {
  return guarded(m->ctx, [&] {
    auto e = mbatch::backend::encode_plan(m->cm.kernels.plans.at(size_t(sig)));
    if (enc) {
      MBATCH_CHECK(*n >= int64_t(e.size()), "buffer too small");
      std::memcpy(enc, e.data(), e.size() * 4);
    }
    *n = int64_t(e.size());
  });
}

void mbx_options_default(mbx_options* o) {
  o->scheduler = MBX_SCHED_DEPTH;
  o->gather = MBX_GATHER_FUSED;
  o->hoist = 1;
  o->phases = 1;
  o->record_nodes = 1;
  o->time_kernels = 0;
  o->time_batches = 0;
  o->inputs_resident = 0;
  o->outputs_on_device = 0;
  o->defer_sync = 0;
  o->ghost = 1;
}

int mbx_evaluate_batch(mbx_model* m, int batch, const int32_t* toks, int64_t ntok, const float* data, int64_t ndata,
                       const mbx_options* opts, mbx_result** out) {
  *out = nullptr;
  auto res = std::make_unique<mbx_result>();
  int rc = guarded(m->ctx, [&] {
    mbx::settle(m->ctx);
    MBATCH_CHECK(batch >= 1, "evaluate_batch: need at least one instance");
    // The inputs are materialised straight from the encoding (no HostValue trees; the tensor
    // data is copied once, into pinned staging) and the outputs encoded straight from the run.
    mbatch::runtime::EncodedValues enc;
    enc.count = batch;
    enc.toks = toks;
    enc.ntok = ntok;
    enc.data = data;
    enc.ndata = ndata;
    mbatch::runtime::ExecOptions o;
    mbx_options d;
    mbx_options_default(&d);
    const mbx_options& oo = opts ? *opts : d;
    o.scheduler = oo.scheduler == MBX_SCHED_AGENDA ? mbatch::runtime::ExecOptions::Scheduler::kAgenda
                                                   : mbatch::runtime::ExecOptions::Scheduler::kDepth;
    o.gather = oo.gather == MBX_GATHER_EXPLICIT ? mbatch::backend::GatherMode::kExplicit : mbatch::backend::GatherMode::kFused;
    o.hoist = oo.hoist != 0;
    o.phases = oo.phases != 0;
    o.record_nodes = oo.record_nodes != 0;
    o.time_kernels = oo.time_kernels != 0;
    o.time_batches = oo.time_batches != 0;
    o.inputs_resident = oo.inputs_resident != 0;
    o.outputs_on_device = oo.outputs_on_device != 0;
    o.defer_sync = oo.defer_sync != 0;
    o.ghost = oo.ghost != 0;
    mbatch::runtime::EncodedOutputs out;
    res->r = m->session->evaluate_encoded(enc, o, &out);
    res->out_tok = std::move(out.toks);
    res->out_data = std::move(out.data);
  });
  if (rc) return rc;
  *out = res.release();
  return 0;
}

// Splits hostval-encoded inputs into per-instance (token, data) spans: each instance is its
// model's instance inputs in module order.
static std::vector<std::array<int64_t, 4>> instance_spans(const mbx_model* m, int batch, const int32_t* toks,
                                                           int64_t ntok, const float* data, int64_t ndata) {
  int ninputs = 0;
  for (const auto& d : m->cm.params) ninputs += d.is_instance_input ? 1 : 0;
  std::vector<std::array<int64_t, 4>> spans;
  int64_t ti = 0, di = 0;
  for (int i = 0; i < batch; ++i) {
    const int64_t t0 = ti, d0 = di;
    for (int k = 0; k < ninputs; ++k) (void)decode(toks, ntok, ti, data, ndata, di);
    spans.push_back({t0, ti - t0, d0, di - d0});
  }
  MBATCH_CHECK(ti == ntok && di == ndata, "hostval encoding: trailing values after the last instance");
  return spans;
}

int mbx_reference_evaluate(mbx_model* m, int batch, const int32_t* toks, int64_t ntok, const float* data,
                           int64_t ndata, mbx_result** out) {
  *out = nullptr;
  auto res = std::make_unique<mbx_result>();
  int rc = guarded(m->ctx, [&] {
    mbx::settle(m->ctx);
    MBATCH_CHECK(batch >= 1, "evaluate_batch: need at least one instance");
    mbatch::runtime::ExecOptions o;
    o.ghost = true;
    for (const auto& sp : instance_spans(m, batch, toks, ntok, data, ndata)) {
      mbatch::runtime::EncodedValues enc;
      enc.count = 1;
      enc.toks = toks + sp[0];
      enc.ntok = sp[1];
      enc.data = data + sp[2];
      enc.ndata = sp[3];
      mbatch::runtime::EncodedOutputs eo;
      mbatch::runtime::EvalResult r = m->session->evaluate_encoded(enc, o, &eo);
      res->out_tok.insert(res->out_tok.end(), eo.toks.begin(), eo.toks.end());
      res->out_data.insert(res->out_data.end(), eo.data.begin(), eo.data.end());
      res->r.timing.device_launches += r.timing.device_launches;
    }
  });
  if (rc) return rc;
  *out = res.release();
  return 0;
}

int mbx_profile_invocations(mbx_model* m, int batch, const int32_t* toks, int64_t ntok, const float* data,
                            int64_t ndata, int64_t* counts, int32_t* levels, int32_t* ranking, int* nranked) {
  return guarded(m->ctx, [&] {
    mbx::settle(m->ctx);
    MBATCH_CHECK(batch >= 1, "evaluate_batch: need at least one instance");
    mbatch::runtime::EncodedValues enc;
    enc.count = batch;
    enc.toks = toks;
    enc.ntok = ntok;
    enc.data = data;
    enc.ndata = ndata;
    mbatch::runtime::ExecOptions o;
    o.ghost = true;
    o.record_nodes = true;
    mbatch::runtime::EncodedOutputs eo;
    mbatch::runtime::EvalResult r = m->session->evaluate_encoded(enc, o, &eo);
    const auto rep = mbatch::runtime::profile_from_nodes(m->cm, r.nodes);
    const int nsig = int(m->cm.kernels.signatures.size());
    for (int k = 0; k < nsig; ++k) {
      auto c = rep.counts.find(k);
      auto l = rep.static_estimate.find(k);
      counts[k] = c == rep.counts.end() ? 0 : c->second;
      levels[k] = l == rep.static_estimate.end() ? -1 : l->second;
    }
    *nranked = int(rep.ranking.size());
    for (size_t k = 0; k < rep.ranking.size(); ++k) ranking[k] = rep.ranking[k];
  });
}

void mbx_result_destroy(mbx_result* r) { delete r; }

int mbx_result_outputs(const mbx_result* r, int32_t* toks, int64_t* ntok, float* data, int64_t* ndata) {
  if (toks) {
    if (*ntok < int64_t(r->out_tok.size()) || *ndata < int64_t(r->out_data.size())) return 1;
    std::memcpy(toks, r->out_tok.data(), r->out_tok.size() * 4);
    std::memcpy(data, r->out_data.data(), r->out_data.size() * 4);
  }
  *ntok = int64_t(r->out_tok.size());
  *ndata = int64_t(r->out_data.size());
  return 0;
}

int mbx_result_counters(const mbx_result* r, int64_t* o) {
  const auto& t = r->r.trace;
  o[0] = t.kernel_launches;
  o[1] = t.total_nodes;
  o[2] = t.scheduler_ops;
  o[3] = t.sync_points;
  o[4] = t.gather_bytes;
  o[5] = t.dfg_edges;
  o[6] = int64_t(t.batches.size());
  o[7] = int64_t(t.flush_boundaries.size());
  o[8] = r->r.timing.device_launches;
  return 0;
}

int mbx_result_batches(const mbx_result* r, int32_t* rows5, int32_t* ids) {
  size_t k = 0;
  for (size_t b = 0; b < r->r.trace.batches.size(); ++b) {
    const auto& br = r->r.trace.batches[b];
    rows5[5 * b] = br.phase;
    rows5[5 * b + 1] = br.depth;
    rows5[5 * b + 2] = br.sig;
    rows5[5 * b + 3] = br.size;
    rows5[5 * b + 4] = br.ghost ? 1 : 0;
    for (int id : br.node_ids) ids[k++] = id;
  }
  return 0;
}

int mbx_result_flush_boundaries(const mbx_result* r, int32_t* out) {
  for (size_t k = 0; k < r->r.trace.flush_boundaries.size(); ++k) out[k] = r->r.trace.flush_boundaries[k];
  return 0;
}

int mbx_result_nodes(const mbx_result* r, int32_t* hdr, int64_t* refs, int64_t* nrefs) {
  int64_t need = 0;
  for (const auto& n : r->r.nodes)
    need += 3 * int64_t(n.shared_ins.size() + n.batched_ins.size() + n.outputs.size()) + int64_t(n.producers.size());
  if (!hdr) {
    *nrefs = need;
    return 0;
  }
  if (*nrefs < need) return 1;
  int64_t k = 0;
  for (size_t i = 0; i < r->r.nodes.size(); ++i) {
    const auto& n = r->r.nodes[i];
    int32_t* h = hdr + 11 * i;
    h[0] = n.id; h[1] = n.sig_id; h[2] = n.block_id; h[3] = n.instance; h[4] = n.phase; h[5] = n.depth;
    h[6] = n.ghost; h[7] = int32_t(n.shared_ins.size()); h[8] = int32_t(n.batched_ins.size());
    h[9] = int32_t(n.producers.size()); h[10] = int32_t(n.outputs.size());
    for (auto& t : n.shared_ins) { refs[k++] = t.node; refs[k++] = t.out; refs[k++] = t.handle.offset; }
    for (auto& t : n.batched_ins) { refs[k++] = t.node; refs[k++] = t.out; refs[k++] = t.handle.offset; }
    for (int p : n.producers) refs[k++] = p;
    for (auto& o : n.outputs) { refs[k++] = o.offset; refs[k++] = o.shape.rows; refs[k++] = o.shape.cols; }
  }
  *nrefs = need;
  return 0;
}

int mbx_result_batch_times(const mbx_result* r, double* us) {
  for (size_t k = 0; k < r->r.timing.batch_us.size(); ++k) us[k] = r->r.timing.batch_us[k];
  return int(r->r.timing.batch_us.size());
}

int mbx_result_timing(const mbx_result* r, double* o) {
  o[0] = r->r.timing.host_total_us;
  o[1] = r->r.timing.host_dfg_us;
  o[2] = r->r.timing.device_span_us;
  o[3] = double(r->r.timing.h2d_bytes);
  o[4] = double(r->r.timing.d2h_bytes);
  return 0;
}

int mbx_result_host_breakdown(const mbx_result* r, double* o) {
  o[0] = r->r.timing.host_fibers_us;
  o[1] = r->r.timing.host_sched_us;
  o[2] = r->r.timing.host_prepare_us;
  o[3] = r->r.timing.host_issue_us;
  return 0;
}

}  // extern "C"
