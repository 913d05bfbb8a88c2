/* mbx.h — C ABI of the B200 batched-execution library (libmbx.so).
 *
 * This is the drop-in boundary for the reference's batched-execution hot path.  The reference
 * (`mbatch`, /root/reference/proj) is C++ calling C++; every entry point below replaces one
 * reference interface, cited per function.  The C++ surface with the reference's own names and
 * types (include/mbatch/{backend,runtime,zoo}.hpp) is a thin layer over these functions.
 *
 * Conventions
 *   - Every function returns an int status: 0 = OK, nonzero = error.  The C ABI never throws;
 *     the message (same text as the reference's mbatch::Error, e.g. "shared-param handle
 *     mismatch across instances (analysis bug)") is returned by mbx_last_error(ctx).
 *   - Tensors live in a per-context device arena addressed by float offsets, exactly as the
 *     reference's TensorHandle{offset, shape} (proj/include/mbatch/backend.hpp:53-59).
 *   - Host values (model inputs / outputs) cross the ABI in the "hostval" encoding: an int32
 *     token stream plus a float32 data stream, depth-first:
 *        tensor: 0, rows, cols (rows*cols floats from the data stream) | int: 1, value
 *        | int64: 6, lo, hi | float64: 5, lo, hi (bits of the double)
 *        list: 2, n, items... | tuple: 3, n, items...
 *        | adt: 4, ctor (0 Leaf, 1 Node, -1 named: length, one token per byte), n, fields...
 *   - One context = one device + one CUDA stream + one arena; a context is used by one host
 *     thread at a time (the reference executor is single-threaded).
 */
#ifndef MBX_H
#define MBX_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mbx_ctx mbx_ctx;
typedef struct mbx_model mbx_model;
typedef struct mbx_result mbx_result;

/* Op codes = backend::OpCode (proj/include/mbatch/backend.hpp:27-37). */
enum { MBX_DENSE = 0, MBX_ADD, MBX_MUL, MBX_SIGMOID, MBX_TANH, MBX_RELU, MBX_CONCAT, MBX_ARGMAX, MBX_FILL };
/* GatherMode (backend.hpp:100). */
enum { MBX_GATHER_FUSED = 0, MBX_GATHER_EXPLICIT = 1 };
/* Arithmetic of the dense contractions.
 *   FP32: CUDA-core, reference accumulation order, glibc-exact activations -> bitwise equal to
 *         the reference.
 *   BF16X3: tcgen05 tensor cores on split bf16 operands (hi*hi + hi*lo + lo*hi, fp32 TMEM
 *         accumulation) where a tensor-core kernel exists for the plan, FP32 elsewhere.
 *   BF16: tcgen05 single bf16 pass (fastest, widest tolerance). */
enum { MBX_PREC_FP32 = 0, MBX_PREC_BF16X3 = 1, MBX_PREC_BF16 = 2, MBX_PREC_BF16X6 = 3 };
/* ExecOptions::Scheduler (proj/include/mbatch/runtime.hpp:45-55). */
enum { MBX_SCHED_DEPTH = 0, MBX_SCHED_AGENDA = 1 };

const char* mbx_version(void);
/* Number of kernel launches this process has issued through libmbx (all contexts). */
int64_t mbx_kernel_launch_count(void);

/* ---- context -------------------------------------------------------------------------- */
int mbx_ctx_create(int device, int precision, mbx_ctx** out);
void mbx_ctx_destroy(mbx_ctx* ctx);
const char* mbx_last_error(const mbx_ctx* ctx);
int mbx_ctx_set_precision(mbx_ctx* ctx, int precision);
int mbx_sync(mbx_ctx* ctx);
/* The context's CUDA stream (cudaStream_t), for callers that time or order work around it. */
void* mbx_ctx_stream(mbx_ctx* ctx);

/* ---- arena: backend::Arena (backend.hpp:63-88) ----------------------------------------- */
/* Bump-allocates rows*cols floats; *offset gets the element offset (Arena::alloc). */
int mbx_arena_alloc(mbx_ctx* ctx, int rows, int cols, int64_t* offset);
int64_t mbx_arena_used(const mbx_ctx* ctx);                                  /* Arena::used */
/* Host <-> device copies of arena ranges; bounds-checked like Arena::ptr
 * ("tensor handle out of arena bounds").  download synchronizes the stream. */
int mbx_arena_upload(mbx_ctx* ctx, int64_t offset, const float* src, int64_t n);
int mbx_arena_download(mbx_ctx* ctx, int64_t offset, float* dst, int64_t n);
/* Arena::ptr: the device address of arena[off, off + n) (bounds-checked; NULL in dry contexts). */
int mbx_arena_device_ptr(mbx_ctx* ctx, int64_t offset, int64_t n, float** out);
/* Drops every allocation at or above `used` (session reuse; params below stay resident). */
int mbx_arena_rewind(mbx_ctx* ctx, int64_t used);

/* ---- plans: backend::ExecutablePlan (backend.hpp:101-132) ------------------------------
 * Flat int32 encoding:
 *   ghost, nshared, (rows, cols)*nshared, nbatched, (rows, cols)*nbatched, nsteps,
 *   per step: kind(0 op,1 fused_dense,2 chain), op, out_rows, out_cols, nin, ref*nin,
 *             nchain, (op, has_rhs, ref)*nchain,
 *   nout, ref*nout
 * with ref = kind(0 shared,1 batched,2 temp), index, col_off, cols(-1 = whole tensor). */
int mbx_plan_register(mbx_ctx* ctx, const int32_t* enc, int64_t n, int* plan_id);

/* backend::exec_batched (proj/src/exec_batched.cpp:23-157) over b instances.
 *   shared_off[b * nshared]    each instance's shared-input offsets (row-major); they must be
 *                              identical across instances, else the call fails with
 *                              "shared-param handle mismatch across instances (analysis bug)"
 *   batched_off[b * nbatched]  arena offsets of each instance's batched inputs (row-major)
 *   out_off[b * nout]          receives each instance's output handle offsets (batch-contiguous
 *                              per output slot, as the reference lays them out)
 *   *gather_bytes              0 in FUSED mode; EXPLICIT-mode copy bytes otherwise.
 * Allocates scratch/outputs/temporaries in the arena in the reference's order, so handle
 * offsets equal the reference's.  Asynchronous: enqueues device work on the context stream. */
int mbx_exec_batched(mbx_ctx* ctx, int plan_id, int b, const int64_t* shared_off,
                     const int64_t* batched_off, int gather_mode, int64_t* out_off,
                     int64_t* gather_bytes);

/* Flush scope (runtime::Executor::flush, proj/src/executor.cpp:711-758): between
 * mbx_flush_begin and mbx_flush_end, mbx_exec_batched validates, allocates and returns each
 * batch's output handles at once (same offsets as outside a flush) but queues the device work;
 * mbx_flush_end plans the queued batches together — consecutive batches of one tensor-core gate
 * plan become one persistent multi-level launch (e.g. every TreeLSTM depth), gathered operands
 * are written MMA-ready by their producers — and issues them with one offset-table H2D.  Every
 * other call on the context (downloads, uploads, primops, mbx_read_ints, mbx_sync, evaluation)
 * issues the queued work first, so the results are the same as without the scope. */
int mbx_flush_begin(mbx_ctx* ctx);
int mbx_flush_end(mbx_ctx* ctx);

/* Decision read-back (Executor::read_scalar_int, proj/src/executor.cpp:235-238): out[k] =
 * (long)arena[offs[k]] for every k, with one pack kernel and one D2H for all n values
 * (synchronises). */
int mbx_read_ints(mbx_ctx* ctx, const int64_t* offs, int n, int64_t* out);

/* backend::exec_primop (proj/src/backend.cpp:105-181) on arena tensors. */
int mbx_exec_primop(mbx_ctx* ctx, int op, int nin, const int64_t* in_off, const int* in_rows,
                    const int* in_cols, int64_t out_off, int out_rows, int out_cols, float fill);

/* ---- whole-model runtime: runtime::evaluate_batch (proj/src/executor.cpp:782-787) --------- */
/* Zoo model `name` (rnn, birnn, treelstm, mvrnn, nestedrnn, drnn, stackrnn, fig5) at hidden
 * size `hidden` (zoo::get_model, proj/src/zoo.cpp:305-322, any H).  Registers the model's
 * kernel library (signatures + lowered plans) with the context. */
int mbx_model_create(mbx_ctx* ctx, const char* name, int hidden, mbx_model** out);
void mbx_model_destroy(mbx_model* m);
/* zoo::make_params(seed) (zoo.cpp:332-341), uploaded to the device arena (params resident). */
int mbx_model_make_params(mbx_model* m, unsigned seed);
/* Sets one parameter from host memory (n = rows*cols floats). */
int mbx_model_set_param(mbx_model* m, const char* name, const float* data, int64_t n);
int mbx_model_num_params(const mbx_model* m);
const char* mbx_model_param_name(const mbx_model* m, int i);
/* zoo::make_inputs(seed, batch) (zoo.cpp:343-401) in hostval encoding; two-call protocol:
 * call with NULL buffers to get sizes, then with buffers of those sizes. */
int mbx_model_make_inputs(mbx_model* m, unsigned seed, int batch, int32_t* toks, int64_t* ntok,
                          float* data, int64_t* ndata);
/* Kernel library introspection: number of signatures, name of signature i, and its lowered
 * plan in the mbx_plan_register encoding (two-call size protocol). */
int mbx_model_num_sigs(const mbx_model* m);
const char* mbx_model_sig_name(const mbx_model* m, int sig);
int mbx_model_plan_encoding(const mbx_model* m, int sig, int32_t* enc, int64_t* n);

typedef struct {
  int32_t scheduler;    /* MBX_SCHED_* */
  int32_t gather;       /* MBX_GATHER_* */
  int32_t hoist;        /* honour static hoist depths (ExecOptions::hoist) */
  int32_t phases;       /* program phases (ExecOptions::phases) */
  int32_t record_nodes; /* keep the DFG node table in the result (oracle checks) */
  int32_t time_kernels; /* CUDA-event timing of the device work (per flush) */
  int32_t time_batches; /* CUDA-event timing of every batch launch (mbx_result_batch_times) */
  int32_t inputs_resident;   /* inputs already in the arena from an identical previous call:
                                skip their H2D copy (device-resident benchmarking) */
  int32_t outputs_on_device; /* leave outputs in the arena (no D2H; the result carries no output values) */
  int32_t ghost;        /* ghost units of the lowered program (ExecOptions::ghost) */
  int32_t defer_sync;   /* return with the work and the output read-back enqueued; outputs not
                           decoded; synchronise (mbx_sync) before reusing the context */
} mbx_options;
void mbx_options_default(mbx_options* o);

/* Runs one mini-batch end to end: host inputs -> device (pinned staging, one copy), fibers +
 * inline-depth DFG construction, depth scheduling, batched kernels, outputs -> host. */
int mbx_evaluate_batch(mbx_model* m, int batch, const int32_t* toks, int64_t ntok,
                       const float* data, int64_t ndata, const mbx_options* opts,
                       mbx_result** out);
/* runtime::reference_evaluate (runtime.hpp:141-144): every instance evaluated on its own (one
 * instance per mini-batch, no cross-instance batching).  The result carries outputs only (read
 * with mbx_result_outputs; its trace is empty); in FP32 they equal mbx_evaluate_batch's bitwise. */
int mbx_reference_evaluate(mbx_model* m, int batch, const int32_t* toks, int64_t ntok,
                           const float* data, int64_t ndata, mbx_result** out);
/* runtime::profile_invocations (runtime.hpp:146-154): over one evaluation of the inputs, per
 * signature k < mbx_model_num_sigs: counts[k] = non-ghost DFG nodes, levels[k] = static nesting
 * estimate of its blocks' functions (-1: no block); ranking[0 .. *nranked) = invoked signatures,
 * most-invoked first (ties: lower id). */
int mbx_profile_invocations(mbx_model* m, int batch, const int32_t* toks, int64_t ntok,
                            const float* data, int64_t ndata, int64_t* counts, int32_t* levels,
                            int32_t* ranking, int* nranked);
void mbx_result_destroy(mbx_result* r);
/* Outputs, hostval-encoded (two-call size protocol). */
int mbx_result_outputs(const mbx_result* r, int32_t* toks, int64_t* ntok, float* data,
                       int64_t* ndata);
/* runtime::ScheduleTrace counters (runtime.hpp:94-112), in this order:
 * kernel_launches, total_nodes, scheduler_ops, sync_points, gather_bytes, dfg_edges,
 * num_batches, num_flushes, device_launches (CUDA kernels actually issued). */
int mbx_result_counters(const mbx_result* r, int64_t* out9);
/* Batch rows (phase, depth, sig, size, ghost) * num_batches and node ids in batch order. */
int mbx_result_batches(const mbx_result* r, int32_t* rows5, int32_t* node_ids);
int mbx_result_flush_boundaries(const mbx_result* r, int32_t* out);
/* DFG node table (record_nodes): per node
 *   id, sig, block, instance, phase, depth, ghost, nshared, nbatched, nprod, nout
 * (11 int32) into `hdr`, and the variable parts concatenated into `refs` (int64):
 *   shared (node, out, offset) * nshared, batched (node, out, offset) * nbatched,
 *   producers * nprod, outputs (offset, rows, cols) * nout.  Two-call size protocol on refs. */
int mbx_result_nodes(const mbx_result* r, int32_t* hdr, int64_t* refs, int64_t* nrefs);
/* Timing of this evaluation in microseconds: host total, host DFG+schedule, device kernel span
 * (first to last batch, CUDA events), H2D bytes, D2H bytes. */
int mbx_result_timing(const mbx_result* r, double* out5);
/* Split of the host DFG time in microseconds: fiber execution + DFG construction, depth
 * scheduling, offset-table preparation, kernel issue. */
int mbx_result_host_breakdown(const mbx_result* r, double* out4);
/* Per non-ghost batch, in trace order: device duration in microseconds (time_batches). */
int mbx_result_batch_times(const mbx_result* r, double* us);

/* ---- throughput mode: many mini-batches on one GPU, host work on T threads ----------------
 * T worker contexts (each: stream, arena, plan registry, model `model` at `hidden` with
 * parameters from zoo::make_params(param_seed)); launches needing co-resident CTAs are chained
 * through a per-device lane, everything else overlaps across workers.  mbx_pool_run evaluates
 * mini-batch i (hostval-encoded toks[i] / data[i]) on worker i % T with `opts`; returns the
 * total DFG node count.  Same semantics per mini-batch as mbx_evaluate_batch. */
typedef struct mbx_pool mbx_pool;
int mbx_pool_create(int device, int precision, const char* model, int hidden, unsigned param_seed,
                    int threads, mbx_pool** out);
void mbx_pool_destroy(mbx_pool* p);
const char* mbx_pool_last_error(const mbx_pool* p);
void mbx_pool_set_error(const char* msg); /* error text of a failed mbx_pool_create: mbx_last_error(NULL) */
int mbx_pool_threads(const mbx_pool* p);
void* mbx_pool_stream(mbx_pool* p);
mbx_model* mbx_pool_model(mbx_pool* p, int worker);
int mbx_pool_run(mbx_pool* p, int n, int batch, const int32_t* const* toks, const int64_t* ntok,
                 const float* const* data, const int64_t* ndata, const mbx_options* opts,
                 int64_t* total_nodes);
/* Same, and the device time of the run (first worker-stream start to last worker-stream end,
 * CUDA events) in *device_ms. */
int mbx_pool_run_timed(mbx_pool* p, int n, int batch, const int32_t* const* toks, const int64_t* ntok,
                       const float* const* data, const int64_t* ndata, const mbx_options* opts,
                       int64_t* total_nodes, double* device_ms);

#ifdef __cplusplus
}
#endif
#endif
