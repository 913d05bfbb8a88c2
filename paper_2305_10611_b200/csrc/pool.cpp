// pool.cpp — throughput mode: many independent mini-batches on one GPU, host work in parallel.
//
// The reference evaluates one mini-batch per call on one host thread (runtime::evaluate_batch,
// proj/src/executor.cpp:782-787); its host side (fibers, inline-depth DFG, scheduling) is the
// part that does not shrink with a faster device.  A pool runs T worker threads, each with its
// own context (stream, arena, offset-table ring, plan registry, model + parameters): host work
// overlaps, and so does device work of different mini-batches — except the launches that need
// all their CTAs resident at once (the persistent mbx_tc_levels kernels), which are chained
// through the per-device persistent lane (mbx_ctx::serialize_persistent) so two of them are
// never partially resident together.  Mini-batch i runs on worker i % T, so a worker's inputs
// can stay resident across calls (inputs_resident).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ctx.h"
#include "mbx.h"

constexpr int kInFlight = 2;  // contexts (mini-batches in flight) per worker

struct mbx_pool {
  int device = 0;
  int threads = 1;
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
  // Two contexts per worker: a worker builds its next mini-batch's DFG on one while the device
  // still runs the previous one on the other (deferred sync), so each keeps two in flight.
  for (int t = 0; t < threads * kInFlight; ++t) {
    mbx_ctx* c = nullptr;
    if (mbx_ctx_create(device, precision, &c)) return fail(mbx_last_error(nullptr));
    p->ctxs.push_back(c);
    // Persistent launches on half the SMs, two at a time (several workers keep both lanes busy).
    static const bool half = [] {
      const char* e = std::getenv("MBX_POOL_HALF");
      return !e || std::atoi(e) != 0;
    }();
    if (half && threads > 1) c->sm_budget = 74;
    mbx_model* m = nullptr;
    if (mbx_model_create(c, model, hidden, &m)) return fail(mbx_last_error(c));
    p->models.push_back(m);
    if (mbx_model_make_params(m, param_seed)) return fail(mbx_last_error(c));
  }
  p->threads = threads;
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
int mbx_pool_threads(const mbx_pool* p) { return p ? p->threads : 0; }
void* mbx_pool_stream(mbx_pool* p) { return p ? reinterpret_cast<void*>(p->stream) : nullptr; }
mbx_model* mbx_pool_model(mbx_pool* p, int worker) {
  return p && worker >= 0 && worker < p->threads ? p->models[size_t(worker) * kInFlight] : nullptr;
}

int mbx_pool_run(mbx_pool* p, int n, int batch, const int32_t* const* toks, const int64_t* ntok,
                 const float* const* data, const int64_t* ndata, const mbx_options* opts, int64_t* total_nodes) {
  return mbx_pool_run_timed(p, n, batch, toks, ntok, data, ndata, opts, total_nodes, nullptr);
}

int mbx_pool_run_timed(mbx_pool* p, int n, int batch, const int32_t* const* toks, const int64_t* ntok,
                       const float* const* data, const int64_t* ndata, const mbx_options* opts,
                       int64_t* total_nodes, double* device_ms) {
  const int T = p->threads;
  const int C = int(p->ctxs.size());
  // Device time of the whole run: an event in every context stream before any work (the streams
  // are idle, so they fire at once) and after all of it; the span is first start -> last end.
  std::vector<cudaEvent_t> ev0(size_t(C), nullptr), ev1(size_t(C), nullptr);
  const bool timed = device_ms && p->device >= 0;
  if (timed)
    for (int w = 0; w < C; ++w) {
      cudaEventCreate(&ev0[size_t(w)]);
      cudaEventCreate(&ev1[size_t(w)]);
      cudaEventRecord(ev0[size_t(w)], p->ctxs[size_t(w)]->stream);
    }
  mbx_options o;
  mbx_options_default(&o);
  if (opts) o = *opts;
  o.defer_sync = 1;
  std::atomic<int64_t> nodes{0};
  std::vector<std::string> errs(static_cast<size_t>(T));
  auto work = [&](int w) {
    int k = 0;
    for (int i = w; i < n; i += T, ++k) {
      const int ci = w * kInFlight + (k % kInFlight);
      mbx_ctx* c = p->ctxs[size_t(ci)];
      // The context's previous mini-batch must be done before its arena and staging are reused.
      if (k >= kInFlight && mbx_sync(c)) {
        errs[size_t(w)] = mbx_last_error(c);
        return;
      }
      mbx_result* r = nullptr;
      if (mbx_evaluate_batch(p->models[size_t(ci)], batch, toks[i], ntok[i], data[i], ndata[i], &o, &r)) {
        errs[size_t(w)] = mbx_last_error(c);
        return;
      }
      int64_t cnt[9];
      mbx_result_counters(r, cnt);
      nodes += cnt[1];
      mbx_result_destroy(r);
    }
    for (int q = 0; q < kInFlight; ++q) mbx_sync(p->ctxs[size_t(w * kInFlight + q)]);
  };
  std::vector<std::thread> th;
  for (int w = 1; w < T && w < n; ++w) th.emplace_back(work, w);
  work(0);
  for (auto& t : th) t.join();
  if (timed) {
    double span = 0.0;
    for (int w = 0; w < C; ++w) {
      cudaEventRecord(ev1[size_t(w)], p->ctxs[size_t(w)]->stream);
      cudaEventSynchronize(ev1[size_t(w)]);
    }
    for (int a = 0; a < C; ++a)
      for (int b = 0; b < C; ++b) {
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, ev0[size_t(a)], ev1[size_t(b)]) == cudaSuccess) span = std::max(span, double(ms));
      }
    *device_ms = span;
    for (int w = 0; w < C; ++w) {
      cudaEventDestroy(ev0[size_t(w)]);
      cudaEventDestroy(ev1[size_t(w)]);
    }
  }
  for (auto& e : errs)
    if (!e.empty()) {
      p->err = e;
      return 1;
    }
  if (total_nodes) *total_nodes = nodes.load();
  return 0;
}

}  // extern "C"
