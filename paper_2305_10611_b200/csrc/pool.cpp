// pool.cpp — throughput mode: many independent mini-batches on one GPU, host work in parallel.
//
// The reference evaluates one mini-batch per call on one host thread (runtime::evaluate_batch,
// proj/src/executor.cpp:782-787); its host side (fibers, inline-depth DFG, scheduling) is the
// part that does not shrink with a faster device.  A pool runs T worker threads, each with its
// own context (arena, offset-table ring, plan registry, model + parameters) and the same model,
// all issuing into ONE device stream: the device work of different mini-batches is serialised in
// submission order (so the persistent multi-level kernels, which need every CTA resident, never
// overlap), while their host work (input decode, fibers, scheduling, offset tables) overlaps.
// Mini-batch i runs on worker i % T, so a worker's inputs can stay resident across calls
// (inputs_resident).  Each worker waits only for its own work (event sync, not stream sync).
#include <atomic>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ctx.h"
#include "mbx.h"

struct mbx_pool {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::vector<mbx_ctx*> ctxs;
  std::vector<mbx_model*> models;
  std::string err;
};

extern "C" {

int mbx_pool_create(int device, int precision, const char* model, int hidden, unsigned param_seed, int threads,
                    mbx_pool** out) {
  *out = nullptr;
  auto p = std::make_unique<mbx_pool>();
  p->device = device;
  if (threads < 1) threads = 1;
  auto fail = [&](const char* what) {
    for (auto* m : p->models) mbx_model_destroy(m);
    for (auto* c : p->ctxs) mbx_ctx_destroy(c);
    if (p->stream) cudaStreamDestroy(p->stream);
    mbx_pool_set_error(what);
    return 1;
  };
  if (device >= 0) {
    if (cudaSetDevice(device) != cudaSuccess) return fail("cudaSetDevice");
    if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess) return fail("stream");
  }
  for (int t = 0; t < threads; ++t) {
    mbx_ctx* c = nullptr;
    if (mbx_ctx_create(device, precision, &c)) return fail(mbx_last_error(nullptr));
    if (device >= 0) {
      cudaStreamSynchronize(c->stream);
      cudaStreamDestroy(c->stream);
      c->stream = p->stream;
      c->owns_stream = false;
    }
    p->ctxs.push_back(c);
    mbx_model* m = nullptr;
    if (mbx_model_create(c, model, hidden, &m)) return fail(mbx_last_error(c));
    p->models.push_back(m);
    if (mbx_model_make_params(m, param_seed)) return fail(mbx_last_error(c));
  }
  *out = p.release();
  return 0;
}

void mbx_pool_destroy(mbx_pool* p) {
  if (!p) return;
  if (p->stream) cudaStreamSynchronize(p->stream);
  for (auto* m : p->models) mbx_model_destroy(m);
  for (auto* c : p->ctxs) mbx_ctx_destroy(c);
  if (p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

const char* mbx_pool_last_error(const mbx_pool* p) { return p ? p->err.c_str() : ""; }
int mbx_pool_threads(const mbx_pool* p) { return p ? int(p->ctxs.size()) : 0; }
void* mbx_pool_stream(mbx_pool* p) { return p ? reinterpret_cast<void*>(p->stream) : nullptr; }
mbx_model* mbx_pool_model(mbx_pool* p, int worker) {
  return p && worker >= 0 && worker < int(p->models.size()) ? p->models[size_t(worker)] : nullptr;
}

int mbx_pool_run(mbx_pool* p, int n, int batch, const int32_t* const* toks, const int64_t* ntok,
                 const float* const* data, const int64_t* ndata, const mbx_options* opts, int64_t* total_nodes) {
  const int T = int(p->ctxs.size());
  std::atomic<int64_t> nodes{0};
  std::vector<std::string> errs(static_cast<size_t>(T));
  auto work = [&](int w) {
    for (int i = w; i < n; i += T) {
      mbx_result* r = nullptr;
      if (mbx_evaluate_batch(p->models[size_t(w)], batch, toks[i], ntok[i], data[i], ndata[i], opts, &r)) {
        errs[size_t(w)] = mbx_last_error(p->ctxs[size_t(w)]);
        return;
      }
      int64_t cnt[9];
      mbx_result_counters(r, cnt);
      nodes += cnt[1];
      mbx_result_destroy(r);
    }
  };
  std::vector<std::thread> th;
  for (int w = 1; w < T && w < n; ++w) th.emplace_back(work, w);
  work(0);
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (!e.empty()) {
      p->err = e;
      return 1;
    }
  if (total_nodes) *total_nodes = nodes.load();
  return 0;
}

}  // extern "C"
